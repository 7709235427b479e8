// Host scheduling layer — see scheduler.hpp. Every function names the
// reference routine whose semantics it reproduces. Built with
// -ffp-contract=off: predicted_times' llround and the ratio EMA must round
// exactly like the reference's separate IEEE operations.
#include "scheduler.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <optional>

namespace moespac {

// ------------------------------------------------------------ balancer

// workload_balancer.cpp:12-18
void HardwareProfile::validate() const {
  const bool pos = t_cpu_unit_ns > 0 && t_gpu_unit_ns > 0 && t_io_unit_ns > 0 &&
                   t_draft_unit_ns > 0 && expert_bytes > 0 && vram_capacity_bytes > 0;
  if (!pos) throw std::invalid_argument("HardwareProfile: all units must be positive");
  if (n_layers < 1) throw std::invalid_argument("HardwareProfile: n_layers must be >= 1");
}

// workload_balancer.cpp:20-30
void RatioEstimates::validate() const {
  const std::size_t n = cpu_ratio.size();
  if (n == 0 || n != gpu_ratio.size())
    throw std::invalid_argument("RatioEstimates: shape mismatch");
  for (std::size_t i = 0; i < n; ++i) {
    const double c = cpu_ratio[i], g = gpu_ratio[i];
    if (!(c >= 0.0 && c <= 1.0 && g >= 0.0 && g <= 1.0))
      throw std::invalid_argument("RatioEstimates: ratios must be in [0,1]");
    if (i && (c < cpu_ratio[i - 1] || g > gpu_ratio[i - 1]))
      throw std::invalid_argument("RatioEstimates: non-monotone estimate");
  }
}

RatioEstimates RatioEstimates::uniform(int cap, double rc, double rg) {
  RatioEstimates r;
  r.cpu_ratio = std::vector<double>(static_cast<std::size_t>(cap), rc);
  r.gpu_ratio = std::vector<double>(static_cast<std::size_t>(cap), rg);
  return r;
}

// Eq. 7-8, workload_balancer.cpp:39-52. The products are
// evaluated left to right in double, then rounded half away from zero.
PredictedTimes predicted_times(int tau, const BalancerInput& in) {
  if (tau < 1 || tau > in.utility_cap)
    throw std::out_of_range("predicted_times: tau out of [1,K]");
  const double rc = in.ratios->cpu_ratio.at(static_cast<std::size_t>(tau - 1));
  const double rg = in.ratios->gpu_ratio.at(static_cast<std::size_t>(tau - 1));
  double cpu = rc * in.gamma;
  cpu = cpu * in.top_k;
  cpu = cpu * static_cast<double>(in.profile->t_cpu_unit_ns);
  double gpu = rg * in.b_est;
  gpu = gpu * static_cast<double>(in.profile->t_gpu_unit_ns);
  return {std::llround(cpu), std::llround(gpu)};
}

int count_prefetch(int tau, std::span<const int> scores, const ResidentView& resident) {
  int n = 0;
  const int N = static_cast<int>(scores.size());
  for (int e = 0; e < N; ++e) n += (scores[e] >= tau && !resident.contains(e)) ? 1 : 0;
  return n;
}

// workload_balancer.cpp:54-60
int count_prefetch(int tau, std::span<const int> scores, const std::unordered_set<int>& resident) {
  return count_prefetch(tau, scores, ResidentView(&resident));
}

namespace {

// Lazily tabulated T_cpu/T_gpu and feasibility over tau in [1, K]
// (memoised like the reference Evaluator, workload_balancer.cpp:66-102, so
// eval counts are comparable).
class Tabulated {
 public:
  explicit Tabulated(const BalancerInput& in)
      : in_(in), res_(in.residents()), t_(static_cast<std::size_t>(in.utility_cap)),
        have_(static_cast<std::size_t>(in.utility_cap), 0) {}

  const PredictedTimes& at(int tau) {
    const std::size_t i = static_cast<std::size_t>(tau - 1);
    if (!have_.at(i)) {
      t_[i] = predicted_times(tau, in_);
      have_[i] = 1;
      ++evals_;
    }
    return t_[i];
  }
  std::int64_t gap(int tau) {
    const PredictedTimes& p = at(tau);
    return p.cpu_ns - p.gpu_ns;
  }
  // Eq. 10 (I/O window incl. draft credit) and Eq. 11 (VRAM).
  bool ok(int tau) {
    const PredictedTimes& p = at(tau);
    const std::int64_t n = count_prefetch(tau, in_.scores, res_);
    const std::int64_t window = std::max(p.cpu_ns, p.gpu_ns) + in_.draft_credit_ns;
    return in_.profile->t_io_unit_ns * n <= window && in_.profile->expert_bytes * n <= in_.vram_left_bytes;
  }
  int evals() const { return evals_; }

 private:
  const BalancerInput& in_;
  ResidentView res_;
  std::vector<PredictedTimes> t_;
  std::vector<char> have_;
  int evals_ = 0;
};

ThresholdDecision finish(Tabulated& tab, const BalancerInput& in, int tau, bool fallback) {
  ThresholdDecision d;
  d.tau = tau;
  d.fallback = fallback;
  const PredictedTimes& p = tab.at(tau);
  d.predicted_t_cpu_ns = p.cpu_ns;
  d.predicted_t_gpu_ns = p.gpu_ns;
  d.n_prefetch = count_prefetch(tau, in.scores, in.residents());
  return d;
}

}  // namespace

// Appendix C solve (workload_balancer.cpp:106-167): the gap T_cpu - T_gpu is
// monotone in tau, so locate its sign change by bisection, then take the
// closest feasible tau on each side of it and keep the one with the smaller
// |gap| (the lower tau on a tie). Nothing feasible -> tau = K, fallback.
ThresholdDecision solve_threshold(const BalancerInput& in, int* eval_count) {
  in.ratios->validate();
  in.profile->validate();
  const int K = in.utility_cap;
  Tabulated tab(in);

  int lo = 1, hi = K + 1;  // invariant: gap(<lo) < 0, gap(>=hi) >= 0
  while (hi > lo) {
    const int mid = lo + (hi - lo) / 2;
    if (tab.gap(mid) < 0) lo = mid + 1;
    else hi = mid;
  }
  const int cross = lo;

  int left = 0, right = 0;  // 0 = none
  for (int t = std::min(cross - 1, K); t > 0 && !left; --t)
    if (tab.ok(t)) left = t;
  for (int t = cross; t <= K && !right; ++t)
    if (tab.ok(t)) right = t;

  ThresholdDecision d;
  if (!left && !right) {
    d = finish(tab, in, K, true);
  } else if (left && right) {
    const std::int64_t gl = std::llabs(tab.gap(left)), gr = std::llabs(tab.gap(right));
    d = finish(tab, in, gr < gl ? right : left, false);
  } else {
    d = finish(tab, in, left ? left : right, false);
  }
  if (eval_count) *eval_count = tab.evals();
  return d;
}

// workload_balancer.cpp:169-199 — EMA at the used tau, then re-impose
// monotonicity around the one entry that moved.
void update_ratio_estimates(RatioEstimates& r, int tau_used, double obs_rc, double obs_rg,
                            double smoothing) {
  r.validate();
  if (tau_used < 1 || tau_used > r.cap())
    throw std::out_of_range("update_ratio_estimates: tau out of range");
  if (obs_rc < 0.0 || obs_rc > 1.0 || obs_rg < 0.0 || obs_rg > 1.0)
    throw std::invalid_argument("update_ratio_estimates: observations in [0,1]");
  if (smoothing < 0.0 || smoothing > 1.0)
    throw std::invalid_argument("update_ratio_estimates: smoothing in [0,1]");
  const std::size_t a = static_cast<std::size_t>(tau_used - 1);
  const double keep = 1.0 - smoothing;
  const double c0 = keep * r.cpu_ratio[a], c1 = smoothing * obs_rc;
  const double g0 = keep * r.gpu_ratio[a], g1 = smoothing * obs_rg;
  const double c = c0 + c1, g = g0 + g1;
  r.cpu_ratio[a] = c;
  r.gpu_ratio[a] = g;
  for (std::size_t i = 0; i < r.cpu_ratio.size(); ++i) {
    if (i < a) {
      r.cpu_ratio[i] = std::min(r.cpu_ratio[i], c);
      r.gpu_ratio[i] = std::max(r.gpu_ratio[i], g);
    } else if (i > a) {
      r.cpu_ratio[i] = std::max(r.cpu_ratio[i], c);
      r.gpu_ratio[i] = std::min(r.gpu_ratio[i], g);
    }
  }
}

// ------------------------------------------------------------ policies

// utility_estimator.cpp:12-21
void EstimatorConfig::validate() const {
  if (utility_cap < 1) throw std::invalid_argument("EstimatorConfig: utility cap K must be >= 1");
  if (!(forgetting >= 0.0 && forgetting <= 1.0))
    throw std::invalid_argument("EstimatorConfig: forgetting factor must be in [0,1]");
  if (gamma < 1) throw std::invalid_argument("EstimatorConfig: gamma must be >= 1");
  if (utility_cap > gamma) throw std::invalid_argument("EstimatorConfig: requires K <= gamma");
}

// policies.cpp:7-13
void PolicySpec::validate(int utility_cap) const {
  if (kind == PolicyKind::fixed_tau && (fixed_tau < 1 || fixed_tau > utility_cap))
    throw std::invalid_argument("PolicySpec: fixed_tau must be in [1,K]");
  if (kind == PolicyKind::fixed_boundaries && (fixed_up < 1 || fixed_down < 1))
    throw std::invalid_argument("PolicySpec: fixed boundaries must be >= 1");
}

// policies.cpp:41-52
bool is_utility_family(PolicyKind k) {
  return k == PolicyKind::moe_spac || k == PolicyKind::ar_mode || k == PolicyKind::fixed_tau ||
         k == PolicyKind::fixed_boundaries || k == PolicyKind::binary_utility;
}

// policies.cpp:54-69
EstimatorConfig estimator_config_for(const PolicySpec& spec, EstimatorConfig base) {
  if (spec.kind == PolicyKind::binary_utility) {
    base.utility_cap = 1;
  } else if (spec.kind == PolicyKind::fixed_boundaries) {
    base.adaptive_boundaries = false;
    base.init_up = spec.fixed_up;
    base.init_down = spec.fixed_down;
  }
  return base;
}

// policies.cpp:71-84
ThresholdDecision choose_threshold(const PolicySpec& spec, const BalancerInput& in) {
  if (spec.kind != PolicyKind::fixed_tau) return solve_threshold(in);
  ThresholdDecision d;
  d.tau = spec.fixed_tau;
  const PredictedTimes p = predicted_times(d.tau, in);
  d.predicted_t_cpu_ns = p.cpu_ns;
  d.predicted_t_gpu_ns = p.gpu_ns;
  d.n_prefetch = count_prefetch(d.tau, in.scores, in.residents());
  return d;
}

// ------------------------------------------------------------ engine

// execution_engine.cpp:7-11
PrefetchQueues::PrefetchQueues(int utility_cap) {
  if (utility_cap < 1) throw std::invalid_argument("PrefetchQueues: utility cap must be >= 1");
  levels_.resize(static_cast<std::size_t>(utility_cap));
  head_.assign(static_cast<std::size_t>(utility_cap), 0);
}

// execution_engine.cpp:13-25 — a request lives at one level; re-enqueueing
// at a higher level moves it to the back of that level's FIFO.
void PrefetchQueues::enqueue(ExpertKey key, int score) {
  if (score < 1 || score > cap()) throw std::out_of_range("PrefetchQueues: score must be in [1,K]");
  const std::uint64_t id = pack(key);
  auto it = level_of_.find(id);
  if (it != level_of_.end()) {
    if (it->second >= score) return;
    auto& q = levels_[static_cast<std::size_t>(it->second - 1)];
    std::size_t& h = head_[static_cast<std::size_t>(it->second - 1)];
    for (std::size_t i = h; i < q.size(); ++i)
      if (q[i] == key) {
        q.erase(q.begin() + static_cast<std::ptrdiff_t>(i));
        break;
      }
    it->second = score;
  } else {
    level_of_.emplace(id, score);
  }
  levels_[static_cast<std::size_t>(score - 1)].push_back(key);
}

int PrefetchQueues::level_of(ExpertKey key) const {
  auto it = level_of_.find(pack(key));
  if (it == level_of_.end()) throw std::out_of_range("PrefetchQueues: request not pending");
  return it->second;
}

// execution_engine.cpp:34-42
ResidencyPool::ResidencyPool(int utility_cap, std::int64_t expert_bytes, std::int64_t capacity_bytes)
    : cap_(utility_cap), expert_bytes_(expert_bytes), capacity_bytes_(capacity_bytes) {
  if (utility_cap < 1) throw std::invalid_argument("ResidencyPool: utility cap must be >= 1");
  if (expert_bytes <= 0 || capacity_bytes < 0)
    throw std::invalid_argument("ResidencyPool: invalid byte sizes");
}

int ResidencyPool::index(ExpertKey key) const {
  auto it = std::lower_bound(entries_.begin(), entries_.end(), key,
                             [](const std::pair<ExpertKey, int>& a, const ExpertKey& k) { return a.first < k; });
  if (it == entries_.end() || it->first != key) return -1;
  return static_cast<int>(it - entries_.begin());
}

int ResidencyPool::score_of(ExpertKey key) const {
  const int i = index(key);
  if (i < 0) throw std::out_of_range("ResidencyPool: expert not resident");
  return entries_[static_cast<std::size_t>(i)].second;
}

// execution_engine.cpp:63-75
bool ResidencyPool::admit(ExpertKey key, int score) {
  if (score < 0 || score > cap_) throw std::out_of_range("ResidencyPool: admit score must be in [0,K]");
  if (index(key) >= 0) {
    retag(key, score);
    return true;
  }
  if (total_bytes_ + expert_bytes_ > capacity_bytes_) return false;
  auto it = std::lower_bound(entries_.begin(), entries_.end(), key,
                             [](const std::pair<ExpertKey, int>& a, const ExpertKey& k) { return a.first < k; });
  entries_.insert(it, {key, score});
  total_bytes_ += expert_bytes_;
  if (observer_) observer_(key, true);
  return true;
}

ExpertKey ResidencyPool::pop_lowest(int tau) {
  int best = -1;
  for (std::size_t i = 0; i < entries_.size(); ++i) {
    const int s = entries_[i].second;
    if (s >= tau || s == frozen_score()) continue;
    // entries_ is key-sorted, so the first minimum seen has the lowest key.
    if (best < 0 || s < entries_[static_cast<std::size_t>(best)].second) best = static_cast<int>(i);
  }
  if (best < 0) return {-1, -1};
  const ExpertKey key = entries_[static_cast<std::size_t>(best)].first;
  entries_.erase(entries_.begin() + best);
  total_bytes_ -= expert_bytes_;
  if (observer_) observer_(key, false);
  return key;
}

// execution_engine.cpp:77-90 — every non-frozen resident below tau, in
// (score, key) order.
std::vector<ExpertKey> ResidencyPool::evict_below(int tau) {
  std::vector<ExpertKey> out;
  for (ExpertKey k = pop_lowest(tau); k.layer >= 0; k = pop_lowest(tau)) out.push_back(k);
  return out;
}

// execution_engine.cpp:92-109 — lazy reclamation, lowest (score, key) first,
// stops as soon as needed_bytes fit.
std::vector<ExpertKey> ResidencyPool::evict_for_room(std::int64_t needed_bytes, int tau) {
  std::vector<ExpertKey> out;
  while (free_bytes() < needed_bytes) {
    const ExpertKey k = pop_lowest(tau);
    if (k.layer < 0) break;
    out.push_back(k);
  }
  return out;
}

// execution_engine.cpp:111-118
void ResidencyPool::freeze(ExpertKey key) {
  const int i = index(key);
  if (i < 0) throw std::logic_error("ResidencyPool: freezing a non-resident expert");
  entries_[static_cast<std::size_t>(i)].second = frozen_score();
}

// execution_engine.cpp:120-126
void ResidencyPool::thaw_and_recycle(ExpertKey key) {
  const int i = index(key);
  if (i < 0) throw std::logic_error("ResidencyPool: recycling a non-resident expert");
  entries_[static_cast<std::size_t>(i)].second = 0;
}

// execution_engine.cpp:128-139
bool ResidencyPool::retag(ExpertKey key, int new_score) {
  if (new_score < 0 || new_score > cap_) throw std::out_of_range("ResidencyPool: retag score must be in [0,K]");
  const int i = index(key);
  if (i < 0) return false;
  int& s = entries_[static_cast<std::size_t>(i)].second;
  if (s != frozen_score()) s = new_score;
  return true;
}

// execution_engine.cpp:141-146
std::unordered_set<int> ResidencyPool::layer_residents(int layer) const {
  std::unordered_set<int> ids;
  for (const auto& [k, s] : entries_)
    if (k.layer == layer) ids.insert(k.expert);
  return ids;
}

void ResidencyPool::layer_bitmap(int layer, std::uint32_t* bits, int n_experts) const {
  std::fill(bits, bits + (n_experts + 31) / 32, 0u);
  for (const auto& [k, s] : entries_)
    if (k.layer == layer && k.expert >= 0 && k.expert < n_experts)
      bits[k.expert >> 5] |= 1u << (k.expert & 31);
}

// execution_engine.cpp:152-171
std::vector<IoEvent> drain_prefetch(PrefetchQueues& queues, int tau, std::int64_t io_budget_ns,
                                    const HardwareProfile& profile, ResidencyPool& pool,
                                    std::int64_t start_ns) {
  if (io_budget_ns < 0) throw std::invalid_argument("drain_prefetch: negative io budget");
  std::vector<IoEvent> loads;
  std::int64_t clock = 0;
  queues.drain(tau, [&](ExpertKey key, int level) {
    if (pool.resident(key)) return true;  // stale: consumed silently
    if (clock + profile.t_io_unit_ns > io_budget_ns) return false;
    if (!pool.admit(key, level)) return false;  // VRAM full: keep the request
    loads.push_back({IoEvent::Kind::load, key, start_ns + clock, profile.t_io_unit_ns});
    clock += profile.t_io_unit_ns;
    return true;
  });
  return loads;
}

// execution_engine.cpp:173-181
std::vector<IoEvent> apply_eviction(ResidencyPool& pool, int tau, std::int64_t start_ns) {
  if (tau < 1 || tau > pool.frozen_score() - 1) throw std::out_of_range("apply_eviction: tau must be in [1,K]");
  std::vector<IoEvent> ev;
  for (ExpertKey k : pool.evict_below(tau)) ev.push_back({IoEvent::Kind::evict, k, start_ns, 0});
  return ev;
}

}  // namespace moespac
