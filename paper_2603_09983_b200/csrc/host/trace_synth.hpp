// Synthetic routing workload: the reference's TraceGenerator
// (/root/reference/proj/core/src/trace_model.cpp:59-109) split at the point
// where the B200 path takes over. The host keeps the strictly sequential
// mt19937_64 stream and the glibc log/cos noise (not bit-reproducible on the
// GPU, SURVEY.md §7 hard part (ii)) and emits the noisy fp64 logits
// logits[l][t][e] = latent[l][e] + route_noise * gumbel; the top-k selection
// that the reference does next (:87-104) is K1's job on the device.
#pragma once

#include <cstdint>
#include <random>
#include <vector>

namespace moespac {

struct TraceSynthConfig {
  int n_layers = 1, n_experts = 8, top_k = 2, gamma = 8;
  double alpha = 0.8, drift_scale = 0.02, route_noise = 0.2;
  int shift_period = 0;
  std::uint64_t seed = 1;
  void validate() const;  // TraceConfig::validate, trace_model.cpp:12-24
};

class TraceSynth {
 public:
  explicit TraceSynth(const TraceSynthConfig& cfg);
  // logits: [L][gamma+1][N]; returns the accepted count in [1, gamma+1].
  int next(double* logits);
  const TraceSynthConfig& config() const { return cfg_; }

 private:
  double u01();
  double normal();
  double gumbel();
  void redraw();
  TraceSynthConfig cfg_;
  std::mt19937_64 rng_;
  std::vector<double> latent_;  // [L][N]
  int step_ = 0;
};

}  // namespace moespac
