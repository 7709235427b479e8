// Verification-step scheduler: the host half of Simulation::run_utility_step
// (/root/reference/proj/core/src/sim_core.cpp:157-316), split into the two
// phases SURVEY.md §0 item 8 validated as decision-exact:
//
//   decide()  — for every layer, before any of this step's routing is known:
//               snapshot scores -> choose_threshold -> retag -> evict_for_room
//               -> scrub/enqueue -> drain_prefetch. Produces the residency
//               bitmaps, per-layer tau, and the ordered load/evict lists that
//               the device engine turns into cudaMemcpyAsync on copy streams
//               (runs while the draft model would be drafting).
//   observe() — after the GPU ran K1/K2/K3 for the step: consumes the K2
//               counters (or host freqs in host-only mode), applies
//               freeze/thaw, the ratio EMA and b_est, and emits the same
//               LayerTiming/StepReport/SimEvent records the reference does,
//               so decision parity is checked record-for-record.
//
// Expert-parallel mode (shard_world G > 1): expert e lives on
// shard e % G. Every rank runs the bookkeeping for all G shards (cheap,
// deterministic) so every rank derives identical tau/residency with zero
// communication; each shard owns a ResidencyPool/PrefetchQueues pair with
// per-GPU capacity min(|shard|, C1) slots, tau is solved on the global score
// vector. G == 1 reproduces the reference exactly.
#pragma once

#include <cstdint>
#include <vector>

#include "scheduler.hpp"

namespace moespac {

struct SchedConfig {
  int n_layers = 1;
  int n_experts = 8;
  int top_k = 2;
  int gamma = 8;
  HardwareProfile profile;  // n_layers / vram_capacity derived
  EstimatorConfig estimator;
  PolicySpec policy;
  double cache_ratio = 0.17;
  double ratio_smoothing = 0.3;
  int shard_world = 1;
  void validate() const;
};

// sim_core.hpp:38-61 (same fields)
struct LayerTiming {
  std::int64_t t_cpu_ns = 0, t_gpu_ns = 0, t_io_used_ns = 0, stall_ns = 0, bubble_ns = 0, wall_ns = 0;
  int tau = 0;
  bool fallback = false;
  int n_prefetch = 0;
};

struct StepReport {
  std::vector<LayerTiming> layers;
  std::int64_t draft_ns = 0;
  int accepted_tokens = 0;
  std::int64_t cache_hits = 0, cache_misses = 0;
  double accuracy = 0.0;
  std::int64_t faults_fn = 0, faults_fp = 0;
  int n_experts = 0;
  std::int64_t step_wall_ns = 0;
};

// sim_core.hpp:65-73
struct SimEvent {
  enum class Kind { draft, cpu, gpu, stall, load, evict };
  Kind kind;
  int step, layer, expert;
  std::int64_t start_ns, duration_ns;
};
std::int64_t recompute_total_time(const std::vector<SimEvent>& log);

// Realized split of one layer (sim_core.cpp:233-283); produced by K2 on the
// device or by split_on_host() in host-only mode.
struct LayerOutcome {
  std::int32_t distinct = 0, distinct_hits = 0, hit_tokens = 0, miss_tokens = 0;
  std::int32_t agree = 0, faults_fn = 0, faults_fp = 0, n_local_hits = 0;
};

struct SlotLoad {
  int layer, expert, shard, slot;
};

int layer_capacity_experts(double cache_ratio, int n_experts);  // sim_core.cpp:31-34

class StepScheduler {
 public:
  explicit StepScheduler(const SchedConfig& cfg);

  // Phase 1. scores: [L][N] snapshot (the estimator state after the previous
  // step; all zero before the first step).
  void decide(const std::int32_t* scores);
  // Phase 2 with device counters [L] (K2 output) — or host freqs [L][N].
  StepReport observe(const LayerOutcome* outcomes, int accepted_count);
  StepReport observe_freqs(const std::int32_t* freqs, int accepted_count);
  LayerOutcome split_on_host(int layer, const std::int32_t* freqs) const;

  // Decision outputs of the last decide().
  const std::vector<std::uint32_t>& resident_bits() const { return resident_bits_; }  // [L][W]
  const std::vector<std::uint32_t>& loaded_bits() const { return loaded_bits_; }      // [L][W]
  const std::vector<std::int32_t>& taus() const { return taus_; }                     // [L]
  const std::vector<SlotLoad>& loads() const { return loads_; }  // ordered as drained
  const std::vector<ThresholdDecision>& decisions() const { return decisions_; }
  // experts evicted from layer l's pools by the last decide(), in order
  const std::vector<int>& evicted(int layer) const { return layers_[static_cast<std::size_t>(layer)].evicted; }
  // slot of expert e of layer l within its shard pool, -1 if not resident.
  const std::vector<std::int32_t>& slot_table() const { return slot_of_; }  // [L][N]
  int slots_per_layer(int shard) const { return shard_slots_[static_cast<std::size_t>(shard)]; }
  int words() const { return words_; }

  const std::vector<SimEvent>& event_log() const { return events_; }
  std::int64_t total_time_ns() const { return clock_ns_; }
  std::int64_t total_tokens() const { return tokens_; }
  const SchedConfig& config() const { return cfg_; }
  const RatioEstimates& ratios(int layer) const { return layers_[static_cast<std::size_t>(layer)].ratios; }
  int b_est(int layer) const { return layers_[static_cast<std::size_t>(layer)].b_est; }
  const ResidencyPool& pool(int layer, int shard = 0) const {
    return layers_[static_cast<std::size_t>(layer)].pools[static_cast<std::size_t>(shard)];
  }
  int steps() const { return step_; }

 private:
  struct Layer {
    RatioEstimates ratios;
    std::vector<PrefetchQueues> queues;  // per shard
    std::vector<ResidencyPool> pools;    // per shard
    std::vector<std::vector<int>> free_slots;  // per shard, LIFO
    int b_est = 1;
    // last decide() bookkeeping for observe()
    std::vector<int> evicted, loaded;  // expert ids in decision order
    std::int64_t draft_credit = 0;
    std::vector<int> snapshot;  // scores used for the decision
  };
  void admit_slot(int layer, ExpertKey key, bool admitted);

  SchedConfig cfg_;
  int cap_ = 1;        // utility cap K after policy
  int c1_ = 0;         // layer_capacity_experts at G=1
  int words_ = 1;
  bool ar_ = false;
  std::vector<int> shard_slots_;
  std::vector<Layer> layers_;
  std::vector<std::uint32_t> resident_bits_, loaded_bits_;
  std::vector<std::int32_t> taus_, slot_of_;
  std::vector<SlotLoad> loads_;
  std::vector<ThresholdDecision> decisions_;
  std::vector<SimEvent> events_;
  std::int64_t clock_ns_ = 0, tokens_ = 0;
  int step_ = 0;
  bool decided_ = false;
};

}  // namespace moespac
