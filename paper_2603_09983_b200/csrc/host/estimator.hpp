// Speculative Utility Estimator, host operator API — the reference's
// LayerEstimator (/root/reference/proj/core/include/moesim/
// utility_estimator.hpp:33-58, core/src/utility_estimator.cpp:23-107) with
// the same names, semantics and exception classes.
//
// On the B200 path the estimator state of every layer lives in HBM and K2
// updates it in place each step (router_hist.cu, bit-exact with this class);
// this class is the host-side face of that state: the operator for callers
// that drive the estimator directly (the reference's own test scenarios, the
// oracle checks) and the checkpoint codec of the engine
// (moespac_ctx_estimator_dump / _load: one `dump` per layer, the reference's
// text format "<layer> <expert> <score> <up> <down> <last_freq>").
#pragma once

#include <cstdint>
#include <iosfwd>
#include <span>
#include <vector>

#include "scheduler.hpp"  // EstimatorConfig, ExpertUtilityState

namespace moespac {

class LayerEstimator {
 public:
  LayerEstimator(int n_experts, EstimatorConfig config);  // utility_estimator.cpp:23-33

  // utility_estimator.cpp:47-72: inertial transition (score +-1 within [0, K]
  // when the fluctuation reaches a boundary), then the boundary on the side
  // of the fluctuation is recalibrated max(1, floor((1-l)*theta + l*|delta|))
  // in fp64 without contraction.
  void observe_step(std::span<const int> freqs);
  std::vector<int> snapshot_scores() const;  // :74-79

  int n_experts() const { return static_cast<int>(states_.size()); }
  const EstimatorConfig& config() const { return config_; }
  const ExpertUtilityState& state(int expert) const { return states_.at(static_cast<std::size_t>(expert)); }

  // Checkpoint (:81-107): one line per expert; load reads n_experts records
  // (any order) and throws std::runtime_error on a truncated or malformed
  // checkpoint or an out-of-range expert id.
  void dump(std::ostream& out, int layer) const;
  static LayerEstimator load(std::istream& in, int n_experts, const EstimatorConfig& config);

  // Device layout of the engine's estimator state: int32 [N][4] =
  // score, up, down, last_freq (router_hist.cu K2).
  void to_device_layout(std::int32_t* out) const;
  void from_device_layout(const std::int32_t* in);

 private:
  EstimatorConfig config_;
  std::vector<ExpertUtilityState> states_;
};

}  // namespace moespac
