#include "trace_synth.hpp"

#include <cmath>
#include <stdexcept>

namespace moespac {

void TraceSynthConfig::validate() const {
  if (n_layers < 1) throw std::invalid_argument("TraceConfig: n_layers >= 1");
  if (n_experts < 1) throw std::invalid_argument("TraceConfig: n_experts >= 1");
  if (top_k < 1 || top_k > n_experts) throw std::invalid_argument("TraceConfig: requires 1 <= k <= N");
  if (gamma < 1) throw std::invalid_argument("TraceConfig: gamma >= 1");
  if (!(alpha >= 0.0 && alpha <= 1.0)) throw std::invalid_argument("TraceConfig: alpha in [0,1]");
  if (drift_scale < 0.0 || route_noise < 0.0) throw std::invalid_argument("TraceConfig: noise scales must be >= 0");
  if (shift_period < 0) throw std::invalid_argument("TraceConfig: shift_period >= 0");
}

TraceSynth::TraceSynth(const TraceSynthConfig& cfg) : cfg_(cfg), rng_(cfg.seed) {
  cfg_.validate();
  latent_.resize(static_cast<size_t>(cfg_.n_layers) * cfg_.n_experts);
  redraw();
}

// 53-bit mantissa draw (trace_model.cpp:30-32)
double TraceSynth::u01() { return static_cast<double>(rng_() >> 11) * 0x1.0p-53; }

// Box-Muller, one variate per call, u1 redrawn while zero (:34-41)
double TraceSynth::normal() {
  double a = u01();
  const double b = u01();
  while (a == 0.0) a = u01();
  return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * 3.141592653589793 * b);
}

// standard Gumbel via double log (:43-47)
double TraceSynth::gumbel() {
  double u = u01();
  while (u == 0.0) u = u01();
  return -std::log(-std::log(u));
}

void TraceSynth::redraw() {
  for (double& v : latent_) v = normal();
}

int TraceSynth::next(double* logits) {
  ++step_;
  if (cfg_.shift_period > 0 && step_ > 1 && (step_ - 1) % cfg_.shift_period == 0) redraw();
  if (cfg_.drift_scale > 0.0)
    for (double& v : latent_) v += cfg_.drift_scale * normal();
  const int T = cfg_.gamma + 1, N = cfg_.n_experts;
  double* out = logits;
  for (int l = 0; l < cfg_.n_layers; ++l) {
    const double* lat = latent_.data() + static_cast<size_t>(l) * N;
    for (int t = 0; t < T; ++t)
      for (int e = 0; e < N; ++e) *out++ = lat[e] + (cfg_.route_noise > 0.0 ? cfg_.route_noise * gumbel() : 0.0);
  }
  // accepted drafts + bonus token (sample_accept_length, :51-57)
  int acc = 0;
  while (acc < cfg_.gamma && u01() < cfg_.alpha) ++acc;
  return acc + 1;
}

}  // namespace moespac
