// Routing workload, host operator API — the reference's trace_model
// (/root/reference/proj/core/include/moesim/trace_model.hpp:15-83):
// StepActivations / Trace, sample_accept_length, TraceGenerator::next_step,
// activation_frequencies, read_trace / write_trace, same names and
// semantics.
//
// On the B200 path the generator's host half (latent walk + Gumbel noise,
// TraceSynth) feeds noisy fp64 logits to K1, which does the top-k on the
// device, and K2 builds the frequency map there. These host versions are the
// operator API for callers that want activations rather than logits — the
// reference's test scenarios, trace export (#moetrace v1) — and equal the
// device results bit for bit (tests/test_cpp_api.py, tests/test_gpu_kernels.py).
#pragma once

#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "trace_io.hpp"
#include "trace_synth.hpp"

namespace moespac {

using TraceConfig = TraceSynthConfig;

// experts[layer][token] = top_k distinct ids, ascending; accepted in [1, gamma+1]
struct StepActivations {
  std::vector<std::vector<std::vector<int>>> experts;
  int accepted_count = 1;
  bool operator==(const StepActivations&) const = default;
};

struct Trace {
  int n_layers = 0, n_experts = 0, top_k = 0, gamma = 0;
  std::vector<StepActivations> steps;
  bool operator==(const Trace&) const = default;
};

// trace_model.cpp:51-57: leading accepted drafts (each with probability
// alpha, stopping at the first rejection) + 1.
int sample_accept_length(double alpha, int gamma, std::mt19937_64& rng);

// trace_model.cpp:59-109 (+ generate, :111-120).
class TraceGenerator {
 public:
  explicit TraceGenerator(TraceConfig config);
  StepActivations next_step();
  Trace generate(int n_steps);
  const TraceConfig& config() const { return synth_.config(); }

 private:
  TraceSynth synth_;              // latent walk + noise: the same rng stream
  std::vector<double> logits_;    // [L][gamma+1][N] of the current step
};

// trace_model.cpp:122-130 (std::out_of_range for a bad layer).
std::vector<int> activation_frequencies(const StepActivations& acts, int layer, int n_experts);

// trace_model.cpp:132-254, through the flat codec of trace_io.hpp.
Trace read_trace_steps(const std::string& path);
void write_trace_steps(const Trace& trace, const std::string& path);

}  // namespace moespac
