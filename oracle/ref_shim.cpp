// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim around the *unmodified* reference library `moesim_core`,
// compiled from /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libmoesim_ref.so. It lets pytest (ctypes) and bench.py's
// reference arm drive the reference's own code on identical inputs:
//   - TraceGenerator::next_step            proj/core/src/trace_model.cpp:73-109
//   - LayerEstimator::observe_step         proj/core/src/utility_estimator.cpp:47-72
//   - solve_threshold / choose_threshold   proj/core/src/workload_balancer.cpp:106-167,
//                                          proj/core/src/policies.cpp:71-84
//   - update_ratio_estimates               proj/core/src/workload_balancer.cpp:169-199
//   - Simulation::run_utility_step         proj/core/src/sim_core.cpp:157-316
//   - write_trace / read_trace              proj/core/src/trace_model.cpp:132-254
//   - summarize / emit / parse_metrics     proj/core/src/metrics_report.cpp:12-183
// Only the shim is ours; every algorithm runs inside the reference objects.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>

#include "moesim/config.hpp"
#include "moesim/execution_engine.hpp"
#include "moesim/metrics_report.hpp"
#include "moesim/policies.hpp"
#include "moesim/sim_core.hpp"
#include "moesim/trace_model.hpp"
#include "moesim/utility_estimator.hpp"
#include "moesim/workload_balancer.hpp"

using namespace moesim;

extern "C" {

// Mirrors SimConfig (proj/core/include/moesim/sim_core.hpp:23-36) flattened to
// C. Same layout as moespac_sched_config in include/moespac/moespac.h.
struct ref_sim_config {
  int32_t n_layers, n_experts, top_k, gamma;
  double alpha, drift_scale, route_noise;
  int32_t shift_period, _pad0;
  uint64_t seed;
  int64_t t_cpu_unit_ns, t_gpu_unit_ns, t_io_unit_ns, t_draft_unit_ns, expert_bytes;
  int32_t utility_cap, adaptive_boundaries;
  double forgetting;
  int32_t init_up, init_down;
  int32_t policy, fixed_tau, fixed_up, fixed_down;
  double cache_ratio;
  int64_t token_budget;
  int32_t max_steps, warmup_steps;
  double ratio_smoothing;
};

static thread_local std::string g_err;
const char* ref_last_error() { return g_err.c_str(); }

}  // extern "C"

namespace {

SimConfig to_sim(const ref_sim_config& c) {
  SimConfig s = default_sim_config();
  s.trace.n_layers = c.n_layers;
  s.trace.n_experts = c.n_experts;
  s.trace.top_k = c.top_k;
  s.trace.gamma = c.gamma;
  s.trace.alpha = c.alpha;
  s.trace.drift_scale = c.drift_scale;
  s.trace.route_noise = c.route_noise;
  s.trace.shift_period = c.shift_period;
  s.trace.seed = c.seed;
  s.profile.t_cpu_unit_ns = c.t_cpu_unit_ns;
  s.profile.t_gpu_unit_ns = c.t_gpu_unit_ns;
  s.profile.t_io_unit_ns = c.t_io_unit_ns;
  s.profile.t_draft_unit_ns = c.t_draft_unit_ns;
  s.profile.expert_bytes = c.expert_bytes;
  s.estimator.utility_cap = c.utility_cap;
  s.estimator.forgetting = c.forgetting;
  s.estimator.gamma = c.gamma;
  s.estimator.adaptive_boundaries = c.adaptive_boundaries != 0;
  s.estimator.init_up = c.init_up;
  s.estimator.init_down = c.init_down;
  s.policy.kind = static_cast<PolicyKind>(c.policy);
  s.policy.fixed_tau = c.fixed_tau;
  s.policy.fixed_up = c.fixed_up;
  s.policy.fixed_down = c.fixed_down;
  s.cache_ratio = c.cache_ratio;
  s.token_budget = c.token_budget;
  s.max_steps = c.max_steps;
  s.warmup_steps = c.warmup_steps;
  s.ratio_smoothing = c.ratio_smoothing;
  return s;
}

Trace trace_from_arrays(const ref_sim_config& c, const int32_t* ids,
                        const int32_t* accepted, int n_steps) {
  Trace t;
  t.n_layers = c.n_layers;
  t.n_experts = c.n_experts;
  t.top_k = c.top_k;
  t.gamma = c.gamma;
  const int T = c.gamma + 1;
  size_t pos = 0;
  for (int s = 0; s < n_steps; ++s) {
    StepActivations a;
    a.accepted_count = accepted[s];
    a.experts.resize(c.n_layers);
    for (int l = 0; l < c.n_layers; ++l) {
      a.experts[l].resize(T);
      for (int tok = 0; tok < T; ++tok) {
        a.experts[l][tok].assign(ids + pos, ids + pos + c.top_k);
        pos += c.top_k;
      }
    }
    t.steps.push_back(std::move(a));
  }
  return t;
}

}  // namespace

extern "C" {

// ids: [n_steps][L][T][k] int32 (ascending per token), accepted: [n_steps].
int ref_trace_generate(const ref_sim_config* c, int n_steps, int32_t* ids,
                       int32_t* accepted) {
  try {
    SimConfig s = to_sim(*c);
    TraceGenerator gen(s.trace);
    size_t pos = 0;
    for (int i = 0; i < n_steps; ++i) {
      StepActivations a = gen.next_step();
      accepted[i] = a.accepted_count;
      for (const auto& layer : a.experts)
        for (const auto& tok : layer)
          for (int e : tok) ids[pos++] = e;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Wall-clock cost of TraceGenerator::next_step (ns per step, 1 thread).
double ref_trace_time_ns(const ref_sim_config* c, int n_steps) {
  SimConfig s = to_sim(*c);
  TraceGenerator gen(s.trace);
  auto t0 = std::chrono::steady_clock::now();
  int sink = 0;
  for (int i = 0; i < n_steps; ++i) sink += gen.next_step().accepted_count;
  auto t1 = std::chrono::steady_clock::now();
  if (sink < 0) return -1;
  return std::chrono::duration<double, std::nano>(t1 - t0).count() / n_steps;
}

// Runs the reference Simulation over a given trace.
// layer_rec: [S][L][10] = tau, fallback, n_prefetch, t_cpu, t_gpu, t_io_used,
//            stall, wall, bubble, (unused 0)
// step_rec:  [S][8] = accepted, hits, misses, faults_fn, faults_fp,
//            step_wall, draft_ns, n_layers
// step_acc:  [S] accuracy
// events:    [ev_cap][6] = kind, step, layer, expert, start_ns, duration_ns
// Returns the number of steps run (<0 on error).
int ref_sim_run(const ref_sim_config* c, const int32_t* ids,
                const int32_t* accepted, int n_steps, int64_t* layer_rec,
                int64_t* step_rec, double* step_acc, int64_t* events,
                int64_t ev_cap, int64_t* n_events, int64_t* total_time_ns) {
  try {
    SimConfig s = to_sim(*c);
    Simulation sim(s, trace_from_arrays(*c, ids, accepted, n_steps));
    int steps = 0;
    while (auto rep = sim.run_step()) {
      int64_t* sr = step_rec + 8 * steps;
      sr[0] = rep->accepted_tokens;
      sr[1] = rep->cache_hits;
      sr[2] = rep->cache_misses;
      sr[3] = rep->faults_fn;
      sr[4] = rep->faults_fp;
      sr[5] = rep->step_wall_ns;
      sr[6] = rep->draft_ns;
      sr[7] = static_cast<int64_t>(rep->layers.size());
      step_acc[steps] = rep->accuracy;
      for (size_t l = 0; l < rep->layers.size(); ++l) {
        const LayerTiming& lt = rep->layers[l];
        int64_t* r = layer_rec + (static_cast<size_t>(steps) * c->n_layers + l) * 10;
        r[0] = lt.tau;
        r[1] = lt.fallback;
        r[2] = lt.n_prefetch;
        r[3] = lt.t_cpu_ns;
        r[4] = lt.t_gpu_ns;
        r[5] = lt.t_io_used_ns;
        r[6] = lt.stall_ns;
        r[7] = lt.wall_ns;
        r[8] = lt.bubble_ns;
        r[9] = 0;
      }
      ++steps;
    }
    const auto& log = sim.event_log();
    int64_t n = 0;
    for (const SimEvent& e : log) {
      if (n < ev_cap) {
        int64_t* r = events + 6 * n;
        r[0] = static_cast<int64_t>(e.kind);
        r[1] = e.step;
        r[2] = e.layer;
        r[3] = e.expert;
        r[4] = e.start_ns;
        r[5] = e.duration_ns;
      }
      ++n;
    }
    *n_events = n;
    *total_time_ns = sim.total_time_ns();
    return steps;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Host cost of the reference verification-step scheduler
// (Simulation::run_step -> run_utility_step), ns per step, 1 thread.
double ref_sim_time_ns(const ref_sim_config* c, const int32_t* ids,
                       const int32_t* accepted, int n_steps) {
  try {
    SimConfig s = to_sim(*c);
    Simulation sim(s, trace_from_arrays(*c, ids, accepted, n_steps));
    auto t0 = std::chrono::steady_clock::now();
    int steps = 0;
    while (sim.run_step()) ++steps;
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::nano>(t1 - t0).count() /
           (steps > 0 ? steps : 1);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// LayerEstimator over a sequence of frequency vectors.
// state: [n][4] (score, up, down, last_freq) in/out; freqs: [n_steps][n].
int ref_estimator_run(int n, int cap, double lambda, int gamma, int adaptive,
                      int init_up, int init_down, int32_t* state,
                      const int32_t* freqs, int n_steps) {
  try {
    EstimatorConfig cfg;
    cfg.utility_cap = cap;
    cfg.forgetting = lambda;
    cfg.gamma = gamma;
    cfg.adaptive_boundaries = adaptive != 0;
    cfg.init_up = init_up;
    cfg.init_down = init_down;
    std::ostringstream ck;
    for (int i = 0; i < n; ++i)
      ck << 0 << ' ' << i << ' ' << state[4 * i] << ' ' << state[4 * i + 1]
         << ' ' << state[4 * i + 2] << ' ' << state[4 * i + 3] << '\n';
    std::istringstream in(ck.str());
    LayerEstimator est = LayerEstimator::load(in, n, cfg);
    for (int s = 0; s < n_steps; ++s)
      est.observe_step(std::span<const int>(freqs + static_cast<size_t>(s) * n, n));
    for (int i = 0; i < n; ++i) {
      const ExpertUtilityState& st = est.state(i);
      state[4 * i] = st.score;
      state[4 * i + 1] = st.up_boundary;
      state[4 * i + 2] = st.down_boundary;
      state[4 * i + 3] = st.last_freq;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Fresh-estimator initial state (constructor semantics).
int ref_estimator_init(int n, int cap, double lambda, int gamma, int adaptive,
                       int init_up, int init_down, int32_t* state) {
  try {
    EstimatorConfig cfg;
    cfg.utility_cap = cap;
    cfg.forgetting = lambda;
    cfg.gamma = gamma;
    cfg.adaptive_boundaries = adaptive != 0;
    cfg.init_up = init_up;
    cfg.init_down = init_down;
    LayerEstimator est(n, cfg);
    for (int i = 0; i < n; ++i) {
      const ExpertUtilityState& st = est.state(i);
      state[4 * i] = st.score;
      state[4 * i + 1] = st.up_boundary;
      state[4 * i + 2] = st.down_boundary;
      state[4 * i + 3] = st.last_freq;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// solve_threshold on one instance. out: tau, fallback, pred_cpu, pred_gpu,
// n_prefetch, evals.
int ref_solve_threshold(const int32_t* scores, int n, const uint8_t* resident,
                        int gamma, int top_k, int b_est, const double* rc,
                        const double* rg, int cap, int64_t t_cpu, int64_t t_gpu,
                        int64_t t_io, int64_t expert_bytes, int64_t vram_left,
                        int64_t draft_credit, int64_t* out) {
  try {
    std::vector<int> sc(scores, scores + n);
    std::unordered_set<int> res;
    for (int i = 0; i < n; ++i)
      if (resident[i]) res.insert(i);
    RatioEstimates r;
    r.cpu_ratio.assign(rc, rc + cap);
    r.gpu_ratio.assign(rg, rg + cap);
    HardwareProfile p;
    p.t_cpu_unit_ns = t_cpu;
    p.t_gpu_unit_ns = t_gpu;
    p.t_io_unit_ns = t_io;
    p.t_draft_unit_ns = 1;
    p.expert_bytes = expert_bytes;
    p.n_layers = 1;
    p.vram_capacity_bytes = 1;
    BalancerInput in;
    in.scores = sc;
    in.resident = &res;
    in.gamma = gamma;
    in.top_k = top_k;
    in.b_est = b_est;
    in.ratios = &r;
    in.profile = &p;
    in.vram_left_bytes = vram_left;
    in.utility_cap = cap;
    in.draft_credit_ns = draft_credit;
    int evals = 0;
    ThresholdDecision d = solve_threshold(in, &evals);
    out[0] = d.tau;
    out[1] = d.fallback;
    out[2] = d.predicted_t_cpu_ns;
    out[3] = d.predicted_t_gpu_ns;
    out[4] = d.n_prefetch;
    out[5] = evals;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_update_ratio_estimates(double* rc, double* rg, int cap, int tau,
                               double obs_rc, double obs_rg, double smoothing) {
  try {
    RatioEstimates r;
    r.cpu_ratio.assign(rc, rc + cap);
    r.gpu_ratio.assign(rg, rg + cap);
    update_ratio_estimates(r, tau, obs_rc, obs_rg, smoothing);
    std::memcpy(rc, r.cpu_ratio.data(), sizeof(double) * cap);
    std::memcpy(rg, r.gpu_ratio.data(), sizeof(double) * cap);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_layer_capacity_experts(double cache_ratio, int n_experts) {
  SimConfig s = default_sim_config();
  s.cache_ratio = cache_ratio;
  s.trace.n_experts = n_experts;
  return layer_capacity_experts(s);
}


// ---- trace wire format and run metrics (status: 0 ok, -1 runtime_error,
// -2 invalid_argument, -3 out_of_range, -4 other; message in ref_last_error)
static int classify(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return -2;
  if (dynamic_cast<const std::out_of_range*>(&e)) return -3;
  if (dynamic_cast<const std::runtime_error*>(&e)) return -1;
  return -4;
}

int ref_write_trace(const char* path, int L, int N, int k, int gamma, int n_steps, const int32_t* ids,
                    const int32_t* accepted) {
  try {
    Trace t;
    t.n_layers = L;
    t.n_experts = N;
    t.top_k = k;
    t.gamma = gamma;
    size_t pos = 0;
    for (int s = 0; s < n_steps; ++s) {
      StepActivations a;
      a.accepted_count = accepted[s];
      a.experts.resize(static_cast<size_t>(L));
      for (int l = 0; l < L; ++l) {
        a.experts[static_cast<size_t>(l)].resize(static_cast<size_t>(gamma + 1));
        for (auto& tok : a.experts[static_cast<size_t>(l)]) {
          tok.resize(static_cast<size_t>(k));
          for (int& e : tok) e = ids[pos++];
        }
      }
      t.steps.push_back(std::move(a));
    }
    write_trace(t, path);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_read_trace(const char* path, int32_t* shape4, int64_t* n_steps, int32_t* ids, int32_t* accepted,
                   int64_t cap_steps) {
  try {
    const Trace t = read_trace(path);
    shape4[0] = t.n_layers;
    shape4[1] = t.n_experts;
    shape4[2] = t.top_k;
    shape4[3] = t.gamma;
    *n_steps = static_cast<int64_t>(t.steps.size());
    if (ids && static_cast<int64_t>(t.steps.size()) <= cap_steps) {
      size_t pos = 0;
      for (size_t s = 0; s < t.steps.size(); ++s) {
        accepted[s] = t.steps[s].accepted_count;
        for (const auto& layer : t.steps[s].experts)
          for (const auto& tok : layer)
            for (int e : tok) ids[pos++] = e;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// StepReport / LayerTiming flattened (sim_core.hpp:38-61)
struct ref_step_report {
  int64_t draft_ns, cache_hits, cache_misses, faults_fn, faults_fp, step_wall_ns;
  double accuracy;
  int32_t accepted_tokens, n_experts, n_layers, _pad;
};
struct ref_layer_timing {
  int64_t t_cpu_ns, t_gpu_ns, t_io_used_ns, stall_ns, bubble_ns, wall_ns;
  int32_t tau, fallback, n_prefetch, _pad;
};
// RunSummary numbers: vals[10] = axis_value, tps, latency_s, hit_rate,
// bubble_ratio, fault_rate, fn_rate, fp_rate, mean_accuracy, (unused);
// ints[2] = total_tokens, total_time_ns
static void put_summary(const RunSummary& r, double* v, int64_t* i) {
  const double x[10] = {r.axis_value, r.tps, r.latency_s, r.hit_rate, r.bubble_ratio,
                        r.fault_rate, r.fn_rate, r.fp_rate, r.mean_accuracy, 0.0};
  std::memcpy(v, x, sizeof(x));
  i[0] = r.total_tokens;
  i[1] = r.total_time_ns;
}

int ref_summarize(const ref_step_report* reps, const ref_layer_timing* layers, int n, double* vals, int64_t* ints,
                  double* series) {
  try {
    std::vector<StepReport> v(static_cast<size_t>(n));
    const ref_layer_timing* lt = layers;
    for (int i = 0; i < n; ++i) {
      StepReport& s = v[static_cast<size_t>(i)];
      s.draft_ns = reps[i].draft_ns;
      s.accepted_tokens = reps[i].accepted_tokens;
      s.cache_hits = reps[i].cache_hits;
      s.cache_misses = reps[i].cache_misses;
      s.accuracy = reps[i].accuracy;
      s.faults_fn = reps[i].faults_fn;
      s.faults_fp = reps[i].faults_fp;
      s.n_experts = reps[i].n_experts;
      s.step_wall_ns = reps[i].step_wall_ns;
      s.layers.resize(static_cast<size_t>(reps[i].n_layers));
      for (auto& x : s.layers) {
        x.t_cpu_ns = lt->t_cpu_ns;
        x.t_gpu_ns = lt->t_gpu_ns;
        x.t_io_used_ns = lt->t_io_used_ns;
        x.stall_ns = lt->stall_ns;
        x.bubble_ns = lt->bubble_ns;
        x.wall_ns = lt->wall_ns;
        x.tau = lt->tau;
        x.fallback = lt->fallback != 0;
        x.n_prefetch = lt->n_prefetch;
        ++lt;
      }
    }
    const RunSummary r = summarize(v);
    put_summary(r, vals, ints);
    if (series) std::memcpy(series, r.accuracy_series.data(), sizeof(double) * r.accuracy_series.size());
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

// axis: n NUL-terminated names at a 64-byte stride; series concatenated.
int ref_emit(const double* vals, const int64_t* ints, const char* axis, const double* series, const int64_t* n_series,
             int n, int format, const char* path) {
  try {
    std::vector<RunSummary> v(static_cast<size_t>(n));
    const double* sp = series;
    for (int i = 0; i < n; ++i) {
      RunSummary& r = v[static_cast<size_t>(i)];
      r.axis_name = std::string(axis + 64 * i);
      const double* x = vals + 10 * i;
      r.axis_value = x[0];
      r.tps = x[1];
      r.latency_s = x[2];
      r.hit_rate = x[3];
      r.bubble_ratio = x[4];
      r.fault_rate = x[5];
      r.fn_rate = x[6];
      r.fp_rate = x[7];
      r.mean_accuracy = x[8];
      r.total_tokens = ints[2 * i];
      r.total_time_ns = ints[2 * i + 1];
      r.accuracy_series.assign(sp, sp + n_series[i]);
      sp += n_series[i];
    }
    emit(v, format == 0 ? MetricsFormat::csv : MetricsFormat::jsonl, path);
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

int ref_parse(const char* path, double* vals, int64_t* ints, char* axis, double* series, int64_t* n_series, int cap,
              int64_t series_cap, int* n_out) {
  try {
    const std::vector<RunSummary> v = parse_metrics(path);
    *n_out = static_cast<int>(v.size());
    if (static_cast<int>(v.size()) > cap) return 0;
    int64_t used = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      put_summary(v[i], vals + 10 * i, ints + 2 * i);
      std::memset(axis + 64 * i, 0, 64);
      std::strncpy(axis + 64 * i, v[i].axis_name.c_str(), 63);
      n_series[i] = static_cast<int64_t>(v[i].accuracy_series.size());
      if (used + n_series[i] <= series_cap)
        std::memcpy(series + used, v[i].accuracy_series.data(), sizeof(double) * v[i].accuracy_series.size());
      used += n_series[i];
    }
    return 0;
  } catch (const std::exception& e) {
    return classify(e);
  }
}

}  // extern "C"
