// Host-side scheduling layer of the B200 verification-step engine.
//
// Mirrors the reference operator API (namespace moesim in
// /root/reference/proj/core/include/moesim/*.hpp) — same type and function
// names, argument meaning and exception types — so the reference's own tests
// read the same against it. Internals are B200-first: per-layer dense tables
// (N <= 1024 experts) instead of node-based std::map/std::set/std::deque,
// residency as a bitmap that is uploaded to the GPU once per step, and an
// HBM slot allocator behind every admit/evict so that each load the
// Asynchronous Execution Engine decides is a real cudaMemcpyAsync into a
// concrete device slot.
//
// Reference counterparts:
//   HardwareProfile/RatioEstimates/BalancerInput/...  workload_balancer.hpp:15-93
//   predicted_times / count_prefetch / solve_threshold /
//   update_ratio_estimates                            workload_balancer.cpp:39-199
//   PolicyKind/PolicySpec/choose_threshold/
//   estimator_config_for/is_utility_family            policies.hpp:18-59, policies.cpp:41-84
//   EstimatorConfig/ExpertUtilityState                utility_estimator.hpp:14-30
//   ExpertKey/IoEvent/PrefetchQueues/ResidencyPool/
//   drain_prefetch/apply_eviction                     execution_engine.hpp:19-159
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <unordered_map>
#include <stdexcept>
#include <unordered_set>
#include <utility>
#include <vector>

namespace moespac {

// ---------------------------------------------------------------- balancer
struct HardwareProfile {
  std::int64_t t_cpu_unit_ns = 0;
  std::int64_t t_gpu_unit_ns = 0;
  std::int64_t t_io_unit_ns = 0;
  std::int64_t t_draft_unit_ns = 0;
  std::int64_t expert_bytes = 0;
  int n_layers = 1;
  std::int64_t vram_capacity_bytes = 0;
  void validate() const;
};

struct RatioEstimates {
  std::vector<double> cpu_ratio;  // non-decreasing in tau (index tau-1)
  std::vector<double> gpu_ratio;  // non-increasing in tau
  int cap() const { return static_cast<int>(cpu_ratio.size()); }
  void validate() const;
  static RatioEstimates uniform(int cap, double rc = 0.5, double rg = 0.5);
};

// Residency view handed to the balancer. The reference passes an
// unordered_set<int>; the engine passes its bitmap directly.
class ResidentView {
 public:
  ResidentView() = default;
  explicit ResidentView(const std::unordered_set<int>* set) : set_(set) {}
  ResidentView(const std::uint32_t* bits, int n) : bits_(bits), n_(n) {}
  bool contains(int e) const {
    if (bits_) return e >= 0 && e < n_ && ((bits_[e >> 5] >> (e & 31)) & 1u);
    return set_ && set_->count(e) != 0;
  }

 private:
  const std::unordered_set<int>* set_ = nullptr;
  const std::uint32_t* bits_ = nullptr;
  int n_ = 0;
};

struct BalancerInput {
  std::span<const int> scores;
  const std::unordered_set<int>* resident = nullptr;  // reference-style view
  ResidentView resident_view;                         // engine-style view
  int gamma = 1;
  int top_k = 1;
  int b_est = 1;
  const RatioEstimates* ratios = nullptr;
  const HardwareProfile* profile = nullptr;
  std::int64_t vram_left_bytes = 0;
  int utility_cap = 1;
  std::int64_t draft_credit_ns = 0;

  ResidentView residents() const {
    return resident ? ResidentView(resident) : resident_view;
  }
  static std::int64_t default_draft_credit(int gamma, const HardwareProfile& p) {
    return gamma * p.t_draft_unit_ns / p.n_layers;
  }
};

struct ThresholdDecision {
  int tau = 1;
  bool fallback = false;
  std::int64_t predicted_t_cpu_ns = 0;
  std::int64_t predicted_t_gpu_ns = 0;
  int n_prefetch = 0;
};

struct PredictedTimes {
  std::int64_t cpu_ns = 0;
  std::int64_t gpu_ns = 0;
};

PredictedTimes predicted_times(int tau, const BalancerInput& input);
int count_prefetch(int tau, std::span<const int> scores, const std::unordered_set<int>& resident);
int count_prefetch(int tau, std::span<const int> scores, const ResidentView& resident);
ThresholdDecision solve_threshold(const BalancerInput& input, int* eval_count = nullptr);
void update_ratio_estimates(RatioEstimates& ratios, int tau_used, double observed_rc,
                            double observed_rg, double smoothing);

// ---------------------------------------------------------------- policies
enum class PolicyKind {
  moe_spac,
  on_demand_gpu,
  lru_cache,
  static_split,
  ar_mode,
  fixed_tau,
  fixed_boundaries,
  binary_utility,
};

struct EstimatorConfig {
  int utility_cap = 4;
  double forgetting = 0.1;
  int gamma = 8;
  bool adaptive_boundaries = true;
  int init_up = -1;
  int init_down = -1;
  void validate() const;
};

struct ExpertUtilityState {
  int score = 0;
  int up_boundary = 0;
  int down_boundary = 0;
  int last_freq = 0;
};

struct PolicySpec {
  PolicyKind kind = PolicyKind::moe_spac;
  int fixed_tau = 2;
  int fixed_up = 3;
  int fixed_down = 1;
  void validate(int utility_cap) const;
};

bool is_utility_family(PolicyKind kind);
EstimatorConfig estimator_config_for(const PolicySpec& spec, EstimatorConfig base);
ThresholdDecision choose_threshold(const PolicySpec& spec, const BalancerInput& input);

// ---------------------------------------------------------------- engine
struct ExpertKey {
  int layer = 0;
  int expert = 0;
  auto operator<=>(const ExpertKey&) const = default;
};

struct IoEvent {
  enum class Kind { load, evict };
  Kind kind = Kind::load;
  ExpertKey key;
  std::int64_t start_ns = 0;
  std::int64_t duration_ns = 0;
};

// K-level FIFO of pending prefetch requests (execution_engine.hpp:33-61).
// Storage: one contiguous vector per level plus a key->level table; N is
// small (<= 1024 per layer) so erase-by-scan beats node containers.
class PrefetchQueues {
 public:
  explicit PrefetchQueues(int utility_cap);
  void enqueue(ExpertKey key, int score);
  bool contains(ExpertKey key) const { return level_of_.count(pack(key)) != 0; }
  int level_of(ExpertKey key) const;
  std::size_t pending() const { return level_of_.size(); }
  int cap() const { return static_cast<int>(levels_.size()); }

  template <typename Visitor>
  void drain(int tau, Visitor&& visit);
  template <typename Pred>
  void scrub(Pred&& keep);

 private:
  static std::uint64_t pack(ExpertKey k) {
    return (static_cast<std::uint64_t>(static_cast<std::uint32_t>(k.layer)) << 32) |
           static_cast<std::uint32_t>(k.expert);
  }
  std::vector<std::vector<ExpertKey>> levels_;  // FIFO order, index = level-1
  std::vector<std::size_t> head_;                // consumed prefix per level
  std::unordered_map<std::uint64_t, int> level_of_;
};

// Score-tagged resident set with frozen protection (execution_engine.hpp:63-116).
// Entries live in a flat vector kept sorted by key; eviction order is
// (score asc, key asc), exactly the order the reference's
// map<int, set<ExpertKey>> walk produces.
class ResidencyPool {
 public:
  ResidencyPool(int utility_cap, std::int64_t expert_bytes, std::int64_t capacity_bytes);

  int frozen_score() const { return cap_ + 1; }
  std::int64_t total_bytes() const { return total_bytes_; }
  std::int64_t capacity_bytes() const { return capacity_bytes_; }
  std::int64_t free_bytes() const { return capacity_bytes_ - total_bytes_; }
  std::int64_t expert_bytes() const { return expert_bytes_; }
  std::size_t size() const { return entries_.size(); }

  bool resident(ExpertKey key) const { return index(key) >= 0; }
  int score_of(ExpertKey key) const;
  bool admit(ExpertKey key, int score);
  std::vector<ExpertKey> evict_below(int tau);
  std::vector<ExpertKey> evict_for_room(std::int64_t needed_bytes, int tau);
  void freeze(ExpertKey key);
  void thaw_and_recycle(ExpertKey key);
  bool retag(ExpertKey key, int new_score);
  std::unordered_set<int> layer_residents(int layer) const;
  std::vector<std::pair<ExpertKey, int>> entries() const { return entries_; }

  // Engine extensions: residency bitmap of one layer, and the admit/evict
  // observer the device slot allocator hangs off.
  void layer_bitmap(int layer, std::uint32_t* bits, int n_experts) const;
  using Observer = std::function<void(ExpertKey, bool admitted)>;
  void set_observer(Observer obs) { observer_ = std::move(obs); }

 private:
  int index(ExpertKey key) const;
  ExpertKey pop_lowest(int tau);  // lowest (score, key) below tau, non-frozen
  int cap_;
  std::int64_t expert_bytes_;
  std::int64_t capacity_bytes_;
  std::int64_t total_bytes_ = 0;
  std::vector<std::pair<ExpertKey, int>> entries_;  // sorted by key
  Observer observer_;
};

std::vector<IoEvent> drain_prefetch(PrefetchQueues& queues, int tau, std::int64_t io_budget_ns,
                                    const HardwareProfile& profile, ResidencyPool& pool,
                                    std::int64_t start_ns = 0);
std::vector<IoEvent> apply_eviction(ResidencyPool& pool, int tau, std::int64_t start_ns = 0);

template <typename Visitor>
void PrefetchQueues::drain(int tau, Visitor&& visit) {
  for (int level = cap(); level >= std::max(tau, 1); --level) {
    auto& q = levels_[level - 1];
    std::size_t& h = head_[level - 1];
    while (h < q.size()) {
      const ExpertKey key = q[h];
      if (!visit(key, level)) return;
      ++h;
      level_of_.erase(pack(key));
    }
    q.clear();
    h = 0;
  }
}

template <typename Pred>
void PrefetchQueues::scrub(Pred&& keep) {
  for (int level = 1; level <= cap(); ++level) {
    auto& q = levels_[level - 1];
    std::size_t& h = head_[level - 1];
    std::size_t w = 0;
    for (std::size_t r = h; r < q.size(); ++r) {
      if (keep(q[r], level)) q[w++] = q[r];
      else level_of_.erase(pack(q[r]));
    }
    q.resize(w);
    h = 0;
  }
}

}  // namespace moespac
