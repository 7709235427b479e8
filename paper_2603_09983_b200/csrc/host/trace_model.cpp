#include "trace_model.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace moespac {

int sample_accept_length(double alpha, int gamma, std::mt19937_64& rng) {
  if (!(alpha >= 0.0 && alpha <= 1.0) || gamma < 0)
    throw std::invalid_argument("sample_accept_length: invalid parameters");
  int accepted = 0;
  while (accepted < gamma && static_cast<double>(rng() >> 11) * 0x1.0p-53 < alpha) ++accepted;
  return accepted + 1;
}

TraceGenerator::TraceGenerator(TraceConfig config) : synth_(config) {
  logits_.resize(static_cast<std::size_t>(config.n_layers) * (config.gamma + 1) * config.n_experts);
}

StepActivations TraceGenerator::next_step() {
  const TraceConfig& c = synth_.config();
  const int T = c.gamma + 1, N = c.n_experts, k = c.top_k;
  StepActivations acts;
  acts.accepted_count = synth_.next(logits_.data());
  acts.experts.assign(static_cast<std::size_t>(c.n_layers), std::vector<std::vector<int>>(static_cast<std::size_t>(T)));
  std::vector<int> order(static_cast<std::size_t>(N));
  for (int l = 0; l < c.n_layers; ++l)
    for (int t = 0; t < T; ++t) {
      const double* row = logits_.data() + (static_cast<std::size_t>(l) * T + t) * N;
      std::iota(order.begin(), order.end(), 0);
      // k largest by (value desc, id asc) — IEEE comparisons, so -0 == +0 ties
      std::partial_sort(order.begin(), order.begin() + k, order.end(), [&](int a, int b) {
        if (row[a] != row[b]) return row[a] > row[b];
        return a < b;
      });
      std::vector<int>& tok = acts.experts[static_cast<std::size_t>(l)][static_cast<std::size_t>(t)];
      tok.assign(order.begin(), order.begin() + k);
      std::sort(tok.begin(), tok.end());
    }
  return acts;
}

Trace TraceGenerator::generate(int n_steps) {
  const TraceConfig& c = synth_.config();
  Trace tr;
  tr.n_layers = c.n_layers;
  tr.n_experts = c.n_experts;
  tr.top_k = c.top_k;
  tr.gamma = c.gamma;
  tr.steps.reserve(static_cast<std::size_t>(std::max(0, n_steps)));
  for (int i = 0; i < n_steps; ++i) tr.steps.push_back(next_step());
  return tr;
}

std::vector<int> activation_frequencies(const StepActivations& acts, int layer, int n_experts) {
  if (layer < 0 || layer >= static_cast<int>(acts.experts.size()))
    throw std::out_of_range("activation_frequencies: layer out of range");
  std::vector<int> f(static_cast<std::size_t>(n_experts), 0);
  for (const std::vector<int>& tok : acts.experts[static_cast<std::size_t>(layer)])
    for (int e : tok) ++f.at(static_cast<std::size_t>(e));
  return f;
}

Trace read_trace_steps(const std::string& path) {
  const TraceData d = read_trace(path);
  Trace tr;
  tr.n_layers = d.n_layers;
  tr.n_experts = d.n_experts;
  tr.top_k = d.top_k;
  tr.gamma = d.gamma;
  const int T = d.gamma + 1;
  std::size_t i = 0;
  for (std::int64_t s = 0; s < d.steps(); ++s) {
    StepActivations a;
    a.accepted_count = d.accepted[static_cast<std::size_t>(s)];
    a.experts.assign(static_cast<std::size_t>(d.n_layers), std::vector<std::vector<int>>(static_cast<std::size_t>(T)));
    for (auto& layer : a.experts)
      for (auto& tok : layer) {
        tok.assign(d.ids.begin() + static_cast<std::ptrdiff_t>(i), d.ids.begin() + static_cast<std::ptrdiff_t>(i + d.top_k));
        i += static_cast<std::size_t>(d.top_k);
      }
    tr.steps.push_back(std::move(a));
  }
  return tr;
}

void write_trace_steps(const Trace& trace, const std::string& path) {
  TraceData d;
  d.n_layers = trace.n_layers;
  d.n_experts = trace.n_experts;
  d.top_k = trace.top_k;
  d.gamma = trace.gamma;
  for (const StepActivations& a : trace.steps) {
    d.accepted.push_back(a.accepted_count);
    for (const auto& layer : a.experts)
      for (const auto& tok : layer) d.ids.insert(d.ids.end(), tok.begin(), tok.end());
  }
  write_trace(d, path);
}

}  // namespace moespac
