// extern "C" boundary (include/moespac/moespac.h). Every entry point
// converts C++ exceptions into moespac_status, following the reference's
// exception classes.
#include <cstdlib>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/moespac/moespac.h"
#include <cmath>

#include "host/engine.hpp"
#include "host/metrics.hpp"
#include "host/trace_io.hpp"
#include "host/step_scheduler.hpp"
#include "host/trace_model.hpp"
#include "host/trace_synth.hpp"
#include "kernels/launch.hpp"

using namespace moespac;

struct moespac_sched {
  StepScheduler s;
  explicit moespac_sched(const SchedConfig& c) : s(c) {}
};
struct moespac_trace_synth {
  TraceSynth t;
  explicit moespac_trace_synth(const TraceSynthConfig& c) : t(c) {}
};
struct moespac_loopback {
  LoopbackGroup g;
  moespac_loopback(int dev, int world, size_t n) : g(dev, world, n) {}
};
struct moespac_ctx {
  Engine e;
  moespac_ctx(int dev, const moespac_model_desc& m, const moespac_sched_config& c, int r, int w) : e(dev, m, c, r, w) {}
};

namespace {

thread_local std::string g_last_error;

template <typename F>
moespac_status guard(F&& f) {
  try {
    f();
    g_last_error.clear();
    return MOESPAC_OK;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return MOESPAC_E_RANGE;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return MOESPAC_E_INVALID;
  } catch (const std::logic_error& e) {
    g_last_error = e.what();
    return MOESPAC_E_LOGIC;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return MOESPAC_E_CUDA;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    return MOESPAC_E_NCCL;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of memory";
    return MOESPAC_E_NOMEM;
  } catch (const std::runtime_error& e) {
    g_last_error = e.what();
    return MOESPAC_E_IO;
  } catch (...) {
    g_last_error = "unknown error";
    return MOESPAC_E_LOGIC;
  }
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device entry points fail loudly without an sm_100 device (no CPU fallback).
void require_device() {
  int dev = 0, n = 0;
  cuda_ok(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
  if (n < 1) throw CudaError("no CUDA device");
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  int major = 0;
  cuda_ok(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev), "attr");
  if (major != 10) throw CudaError("moespac kernels are built for sm_100a only");
}

SchedConfig to_sched(const moespac_sched_config& c, int world) {
  SchedConfig s;
  s.n_layers = c.n_layers;
  s.n_experts = c.n_experts;
  s.top_k = c.top_k;
  s.gamma = c.gamma;
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
  s.ratio_smoothing = c.ratio_smoothing;
  s.shard_world = world;
  return s;
}

void fill_report(const StepReport& sr, moespac_step_report* rep, moespac_layer_timing* layers,
                 const StepScheduler& s) {
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->draft_ns = sr.draft_ns;
    rep->cache_hits = sr.cache_hits;
    rep->cache_misses = sr.cache_misses;
    rep->faults_fn = sr.faults_fn;
    rep->faults_fp = sr.faults_fp;
    rep->step_wall_ns = sr.step_wall_ns;
    rep->accuracy = sr.accuracy;
    rep->accepted_tokens = sr.accepted_tokens;
    rep->n_experts = sr.n_experts;
    rep->n_layers = static_cast<int32_t>(sr.layers.size());
    rep->n_loads = static_cast<int32_t>(s.loads().size());
  }
  if (layers)
    for (size_t l = 0; l < sr.layers.size(); ++l) {
      const LayerTiming& lt = sr.layers[l];
      moespac_layer_timing& o = layers[l];
      o.t_cpu_ns = lt.t_cpu_ns;
      o.t_gpu_ns = lt.t_gpu_ns;
      o.t_io_used_ns = lt.t_io_used_ns;
      o.stall_ns = lt.stall_ns;
      o.bubble_ns = lt.bubble_ns;
      o.wall_ns = lt.wall_ns;
      o.tau = lt.tau;
      o.fallback = lt.fallback;
      o.n_prefetch = lt.n_prefetch;
      o.n_loads = 0;
      for (const SlotLoad& ld : s.loads())
        if (ld.layer == static_cast<int>(l)) ++o.n_loads;
    }
}

}  // namespace

extern "C" {

const char* moespac_last_error(void) { return g_last_error.c_str(); }
int moespac_abi_version(void) { return MOESPAC_ABI_VERSION; }

void moespac_default_sched_config(moespac_sched_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->n_layers = 48;
  c->n_experts = 128;
  c->top_k = 8;
  c->gamma = 8;
  c->alpha = 0.8;
  c->drift_scale = 0.02;
  c->route_noise = 0.2;
  c->seed = 1;
  c->t_cpu_unit_ns = 100000;
  c->t_gpu_unit_ns = 40000;
  c->t_io_unit_ns = 400000;
  c->t_draft_unit_ns = 300000;
  c->expert_bytes = 25000000;
  c->utility_cap = 4;
  c->adaptive_boundaries = 1;
  c->forgetting = 0.1;
  c->init_up = -1;
  c->init_down = -1;
  c->policy = 0;
  c->fixed_tau = 2;
  c->fixed_up = 3;
  c->fixed_down = 1;
  c->cache_ratio = 0.17;
  c->token_budget = 512;
  c->max_steps = 0;
  c->warmup_steps = 32;
  c->ratio_smoothing = 0.3;
}

// ------------------------------------------------------------ scheduler
moespac_status moespac_sched_create(const moespac_sched_config* cfg, int shard_world, moespac_sched** out) {
  return guard([&] {
    if (!cfg || !out) throw std::invalid_argument("moespac_sched_create: null argument");
    *out = new moespac_sched(to_sched(*cfg, shard_world));
  });
}

void moespac_sched_destroy(moespac_sched* s) { delete s; }

moespac_status moespac_sched_decide(moespac_sched* s, const int32_t* scores) {
  return guard([&] { s->s.decide(scores); });
}

moespac_status moespac_sched_tables(const moespac_sched* s, int32_t* taus, uint32_t* rb, uint32_t* lb,
                                    int32_t* slots) {
  return guard([&] {
    const StepScheduler& x = s->s;
    if (taus) std::memcpy(taus, x.taus().data(), sizeof(int32_t) * x.taus().size());
    if (rb) std::memcpy(rb, x.resident_bits().data(), sizeof(uint32_t) * x.resident_bits().size());
    if (lb) std::memcpy(lb, x.loaded_bits().data(), sizeof(uint32_t) * x.loaded_bits().size());
    if (slots) std::memcpy(slots, x.slot_table().data(), sizeof(int32_t) * x.slot_table().size());
  });
}

moespac_status moespac_sched_decisions(const moespac_sched* s, int64_t* out) {
  return guard([&] {
    size_t i = 0;
    for (const ThresholdDecision& d : s->s.decisions()) {
      out[i++] = d.tau;
      out[i++] = d.fallback;
      out[i++] = d.predicted_t_cpu_ns;
      out[i++] = d.predicted_t_gpu_ns;
      out[i++] = d.n_prefetch;
    }
  });
}

int64_t moespac_sched_loads(const moespac_sched* s, int32_t* out, int64_t cap) {
  const auto& loads = s->s.loads();
  const int64_t n = static_cast<int64_t>(loads.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    out[4 * i] = loads[static_cast<size_t>(i)].layer;
    out[4 * i + 1] = loads[static_cast<size_t>(i)].expert;
    out[4 * i + 2] = loads[static_cast<size_t>(i)].shard;
    out[4 * i + 3] = loads[static_cast<size_t>(i)].slot;
  }
  return n;
}

moespac_status moespac_sched_observe(moespac_sched* s, const moespac_layer_outcome* o, int accepted,
                                     moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] {
    static_assert(sizeof(moespac_layer_outcome) == sizeof(LayerOutcome), "outcome layout");
    const StepReport sr = s->s.observe(reinterpret_cast<const LayerOutcome*>(o), accepted);
    fill_report(sr, rep, layers, s->s);
  });
}

moespac_status moespac_sched_observe_freqs(moespac_sched* s, const int32_t* freqs, int accepted,
                                           moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] {
    const StepReport sr = s->s.observe_freqs(freqs, accepted);
    fill_report(sr, rep, layers, s->s);
  });
}

int64_t moespac_sched_events(const moespac_sched* s, int64_t* out, int64_t cap) {
  const auto& ev = s->s.event_log();
  const int64_t n = static_cast<int64_t>(ev.size());
  for (int64_t i = 0; i < n && i < cap; ++i) {
    const SimEvent& e = ev[static_cast<size_t>(i)];
    int64_t* r = out + 6 * i;
    r[0] = static_cast<int64_t>(e.kind);
    r[1] = e.step;
    r[2] = e.layer;
    r[3] = e.expert;
    r[4] = e.start_ns;
    r[5] = e.duration_ns;
  }
  return n;
}

int64_t moespac_sched_total_time_ns(const moespac_sched* s) { return s->s.total_time_ns(); }

moespac_status moespac_sched_ratios(const moespac_sched* s, int layer, double* rc, double* rg, int32_t* b_est) {
  return guard([&] {
    if (layer < 0 || layer >= s->s.config().n_layers) throw std::out_of_range("moespac_sched_ratios: layer");
    const RatioEstimates& r = s->s.ratios(layer);
    if (rc) std::memcpy(rc, r.cpu_ratio.data(), sizeof(double) * r.cpu_ratio.size());
    if (rg) std::memcpy(rg, r.gpu_ratio.data(), sizeof(double) * r.gpu_ratio.size());
    if (b_est) *b_est = s->s.b_est(layer);
  });
}

moespac_status moespac_solve_threshold(const int32_t* scores, int n, const uint8_t* resident, int gamma, int top_k,
                                       int b_est, const double* rc, const double* rg, int cap, int64_t t_cpu,
                                       int64_t t_gpu, int64_t t_io, int64_t expert_bytes, int64_t vram_left,
                                       int64_t draft_credit, int64_t* out) {
  return guard([&] {
    std::vector<uint32_t> bits(static_cast<size_t>((n + 31) / 32), 0u);
    for (int i = 0; i < n; ++i)
      if (resident[i]) bits[static_cast<size_t>(i >> 5)] |= 1u << (i & 31);
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
    in.scores = std::span<const int>(scores, static_cast<size_t>(n));
    in.resident_view = ResidentView(bits.data(), n);
    in.gamma = gamma;
    in.top_k = top_k;
    in.b_est = b_est;
    in.ratios = &r;
    in.profile = &p;
    in.vram_left_bytes = vram_left;
    in.utility_cap = cap;
    in.draft_credit_ns = draft_credit;
    int evals = 0;
    const ThresholdDecision d = solve_threshold(in, &evals);
    out[0] = d.tau;
    out[1] = d.fallback;
    out[2] = d.predicted_t_cpu_ns;
    out[3] = d.predicted_t_gpu_ns;
    out[4] = d.n_prefetch;
    out[5] = evals;
  });
}

moespac_status moespac_update_ratio_estimates(double* rc, double* rg, int cap, int tau, double orc, double org,
                                              double smoothing) {
  return guard([&] {
    RatioEstimates r;
    r.cpu_ratio.assign(rc, rc + cap);
    r.gpu_ratio.assign(rg, rg + cap);
    update_ratio_estimates(r, tau, orc, org, smoothing);
    std::memcpy(rc, r.cpu_ratio.data(), sizeof(double) * static_cast<size_t>(cap));
    std::memcpy(rg, r.gpu_ratio.data(), sizeof(double) * static_cast<size_t>(cap));
  });
}

int moespac_layer_capacity_experts(double cache_ratio, int n_experts) {
  return layer_capacity_experts(cache_ratio, n_experts);
}

// ------------------------------------------------------------ workload
static TraceSynthConfig synth_config(const moespac_sched_config* cfg) {
  TraceSynthConfig c;
  c.n_layers = cfg->n_layers;
  c.n_experts = cfg->n_experts;
  c.top_k = cfg->top_k;
  c.gamma = cfg->gamma;
  c.alpha = cfg->alpha;
  c.drift_scale = cfg->drift_scale;
  c.route_noise = cfg->route_noise;
  c.shift_period = cfg->shift_period;
  c.seed = cfg->seed;
  return c;
}

moespac_status moespac_trace_generate(const moespac_sched_config* cfg, int64_t n_steps, int32_t* ids,
                                      int32_t* accepted) {
  return guard([&] {
    if (!cfg || n_steps < 0) throw std::invalid_argument("moespac_trace_generate: arguments");
    TraceGenerator gen(synth_config(cfg));
    const int L = cfg->n_layers, T = cfg->gamma + 1, k = cfg->top_k;
    for (int64_t s = 0; s < n_steps; ++s) {
      const StepActivations a = gen.next_step();
      if (accepted) accepted[s] = a.accepted_count;
      if (ids)
        for (int l = 0; l < L; ++l)
          for (int t = 0; t < T; ++t)
            std::copy(a.experts[static_cast<size_t>(l)][static_cast<size_t>(t)].begin(),
                      a.experts[static_cast<size_t>(l)][static_cast<size_t>(t)].end(),
                      ids + ((s * L + l) * T + t) * k);
    }
  });
}

moespac_status moespac_trace_synth_create(const moespac_sched_config* cfg, moespac_trace_synth** out) {
  return guard([&] {
    if (!cfg || !out) throw std::invalid_argument("moespac_trace_synth_create: null argument");
    TraceSynthConfig c;
    c.n_layers = cfg->n_layers;
    c.n_experts = cfg->n_experts;
    c.top_k = cfg->top_k;
    c.gamma = cfg->gamma;
    c.alpha = cfg->alpha;
    c.drift_scale = cfg->drift_scale;
    c.route_noise = cfg->route_noise;
    c.shift_period = cfg->shift_period;
    c.seed = cfg->seed;
    *out = new moespac_trace_synth(c);
  });
}

moespac_status moespac_trace_synth_next(moespac_trace_synth* s, double* logits, int32_t* accepted) {
  return guard([&] { *accepted = s->t.next(logits); });
}

void moespac_trace_synth_destroy(moespac_trace_synth* s) { delete s; }

// ------------------------------------------------------------ kernels
moespac_status moespac_router_topk(const double* logits, int rows, int n, int k, int gate_mode, int32_t* ids,
                                   float* gates, void* stream) {
  return guard([&] {
    if (rows < 0 || n < 1 || n > 1024 || k < 1 || k > n) throw std::invalid_argument("moespac_router_topk: shape");
    if (gate_mode != 0 && gate_mode != 1) throw std::invalid_argument("moespac_router_topk: gate_mode");
    require_device();
    cuda_ok(launch_router_topk(logits, rows, n, k, gate_mode, ids, gates, static_cast<cudaStream_t>(stream)),
            "router_topk");
  });
}

moespac_status moespac_hist_scan_observe(const moespac_k2_args* a, void* stream) {
  return guard([&] {
    if (a->n_layers < 1 || a->tokens < 1 || a->top_k < 1 || a->n_experts < 1 || a->n_experts > 4096 ||
        a->tokens * a->top_k > 2048)
      throw std::invalid_argument("moespac_hist_scan_observe: shape");
    if (a->shard_world < 1 || a->shard_rank < 0 || a->shard_rank >= a->shard_world)
      throw std::invalid_argument("moespac_hist_scan_observe: shard");
    require_device();
    dev::K2Args k{};
    k.ids = a->ids_dev;
    k.L = a->n_layers;
    k.T = a->tokens;
    k.k = a->top_k;
    k.N = a->n_experts;
    k.resident_bits = a->resident_bits_dev;
    k.loaded_bits = a->loaded_bits_dev;
    k.taus = a->taus_dev;
    k.est_state = a->est_state_dev;
    k.utility_cap = a->utility_cap;
    k.adaptive = a->adaptive_boundaries;
    k.forgetting = a->forgetting;
    k.shard_rank = a->shard_rank;
    k.shard_world = a->shard_world;
    k.freqs = a->freqs_dev;
    k.offsets = a->offsets_dev;
    k.perm = a->perm_dev;
    k.hit_list = a->hit_list_dev;
    k.hit_ord = a->hit_ord_dev;
    k.counters = a->counters_dev;
    k.scores_out = a->scores_out_dev;
    cuda_ok(launch_hist_scan_observe(k, static_cast<cudaStream_t>(stream)), "hist_scan_observe");
  });
}

moespac_status moespac_estimator_init(int32_t* st, int n, int gamma, int init_up, int init_down, void* stream) {
  return guard([&] {
    if (n < 1 || gamma < 1) throw std::invalid_argument("moespac_estimator_init: shape");
    require_device();
    cuda_ok(launch_estimator_init(st, n, init_up >= 0 ? init_up : gamma / 2, init_down >= 0 ? init_down : gamma / 2,
                                  static_cast<cudaStream_t>(stream)),
            "estimator_init");
  });
}

size_t moespac_ffn_workspace_bytes(int tokens, int d, int n_experts, int n_shared, int grid) {
  return static_cast<size_t>(grid + n_experts + n_shared) * tokens * d * 4;
}

int64_t moespac_expert_image_elems(int d, int ffn) { return 3LL * d * ffn; }

static int device_sms() {
  int dev = 0, sms = 0;
  cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
  cuda_ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
  return sms;
}

int moespac_ffn_resolve(int kernel, int d, int ffn) { return ffn_resolve(kernel, d, ffn); }

moespac_status moespac_build_hT(const uint16_t* h, int tokens, int d, uint16_t* hT, void* stream) {
  return guard([&] {
    if (tokens < 1 || tokens > kFfnMaxTokens || d % 64) throw std::invalid_argument("moespac_build_hT: shape");
    require_device();
    cuda_ok(launch_build_hT(h, tokens, d, hT, static_cast<cudaStream_t>(stream)), "build_hT");
  });
}

moespac_status moespac_expert_ffn(const moespac_ffn_args* a, void* stream) {
  return guard([&] {
    const int kern = ffn_resolve(a->kernel, a->d_model, a->d_ffn);
    if (!ffn_shape_ok(kern, a->d_model, a->d_ffn) || a->tokens < 1 || a->tokens > kFfnMaxTokens)
      throw std::invalid_argument("moespac_expert_ffn: unsupported shape for this kernel (1 <= tokens <= 16)");
    if (kern == kFfnTensorCore && !a->hT_dev) throw std::invalid_argument("moespac_expert_ffn: hT_dev required");
    require_device();
    int dev = 0, optin = 0;
    cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_ok(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
    const FfnPlan plan = kern == kFfnTensorCore ? ffn_tc_plan(a->tokens, a->d_model, static_cast<size_t>(optin), a->accum)
                                                : ffn_plan(a->tokens, a->d_model, static_cast<size_t>(optin));
    if (!plan.n_stages) throw std::invalid_argument("moespac_expert_ffn: tokens x d_model too large for shared memory");
    const int grid = a->grid > 0 ? a->grid : device_sms();
    if (plan.acc_mode == 3 && !ffn_tg_grid_ok(a->n_experts + a->n_shared_units, a->d_ffn, grid))
      throw std::invalid_argument("moespac_expert_ffn: grid too small for the grouped accumulator (use accum 3)");
    dev::FfnArgs f{};
    f.h = a->h_dev;
    f.T = a->tokens;
    f.d = a->d_model;
    f.ffn = a->d_ffn;
    f.k = a->top_k;
    f.N = a->n_experts;
    f.perm = a->perm_dev;
    f.offsets = a->offsets_dev;
    f.gates = a->gates_dev;
    f.hit_list = a->hit_list_dev;
    f.counters = a->counters_dev;
    f.slot_of = a->slot_of_dev;
    f.pool = a->pool_dev;
    f.shared_w = a->shared_dev;
    f.n_shared = a->n_shared_units;
    f.expert_elems = 3LL * a->d_model * a->d_ffn;
    f.partial = a->workspace_dev;
    f.n_stages = plan.n_stages;
    f.ring_bytes = plan.n_stages * 1024;
    f.global_acc = plan.global_acc ? 1 : 0;
    f.acc_mode = plan.acc_mode;
    f.hT = a->hT_dev;
    f.dbg = reinterpret_cast<unsigned long long*>(a->debug_ts_dev);
    f.l2_policy = a->l2_policy;
    // grouped-K3 profiling knobs, as the engine reads them (engine.cpp)
    if (const char* e = std::getenv("MOESPAC_TAIL_ABSORB")) f.tail_absorb = std::atoi(e);
    if (const char* e = std::getenv("MOESPAC_DRAIN_LATE")) f.drain_late = std::atoi(e);
    if (const char* e = std::getenv("MOESPAC_DRAIN_SC")) f.drain_sc = std::atoi(e);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_ok(kern == kFfnTensorCore ? launch_expert_ffn_tc(f, grid, plan.smem, st) : launch_expert_ffn(f, grid, plan.smem, st),
            "expert_ffn");
  });
}

moespac_status moespac_ffn_combine(const moespac_combine_args* a, void* stream) {
  return guard([&] {
    if (a->d_model % 4 || a->tokens < 1) throw std::invalid_argument("moespac_ffn_combine: shape");
    require_device();
    dev::CombineArgs c{};
    c.h_in = a->h_in_dev;
    c.y_extra = a->y_extra_dev;
    c.T = a->tokens;
    c.d = a->d_model;
    c.ffn = a->d_ffn;
    c.k = a->top_k;
    c.ids = a->ids_dev;
    c.hit_ord = a->hit_ord_dev;
    c.counters = a->counters_dev;
    c.n_shared = a->n_shared_units;
    c.grid = a->grid > 0 ? a->grid : device_sms();
    if (ffn_resolve(a->kernel, a->d_model, a->d_ffn) == kFfnTensorCore) {
      int dev = 0, optin = 0;
      cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
      cuda_ok(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev), "attr");
      c.per_cta = ffn_tc_plan(a->tokens, a->d_model, static_cast<size_t>(optin), a->accum).acc_mode == 3 ? 1 : 0;
      c.unit_rows = 8;
    } else {
      c.unit_rows = 16;
    }
    c.partial = a->workspace_dev;
    c.y_out = a->y_dev;
    c.h_out = a->h_out_dev;
    cuda_ok(launch_combine(c, static_cast<cudaStream_t>(stream)), "combine");
  });
}

moespac_status moespac_pack_expert(const uint16_t* wg, const uint16_t* wu, const uint16_t* wd, int d, int ffn,
                                   int kernel, uint16_t* out, void* stream) {
  return guard([&] {
    const int kern = ffn_resolve(kernel, d, ffn);
    if (!ffn_shape_ok(kern, d, ffn)) throw std::invalid_argument("moespac_pack_expert: shape");
    require_device();
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_ok(kern == kFfnTensorCore ? launch_pack_expert_tc(wg, wu, wd, d, ffn, out, st)
                                   : launch_pack_expert(wg, wu, wd, d, ffn, out, st),
            "pack_expert");
  });
}

moespac_status moespac_unpack_expert(const uint16_t* image, int d, int ffn, int kernel, uint16_t* wg, uint16_t* wu,
                                     uint16_t* wd, void* stream) {
  return guard([&] {
    const int kern = ffn_resolve(kernel, d, ffn);
    if (!ffn_shape_ok(kern, d, ffn)) throw std::invalid_argument("moespac_unpack_expert: shape");
    require_device();
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    cuda_ok(kern == kFfnTensorCore ? launch_unpack_expert_tc(image, d, ffn, wg, wu, wd, st)
                                   : launch_unpack_expert(image, d, ffn, wg, wu, wd, st),
            "unpack_expert");
  });
}

moespac_status moespac_fill_synthetic(uint16_t* dst, int64_t n, uint64_t seed, float stdv, void* stream) {
  return guard([&] {
    if (n < 0) throw std::invalid_argument("moespac_fill_synthetic: n");
    require_device();
    cuda_ok(launch_fill_synthetic(dst, n, seed, stdv, static_cast<cudaStream_t>(stream)), "fill_synthetic");
  });
}

// ------------------------------------------------------------ context
moespac_status moespac_ctx_create(int device, const moespac_model_desc* m, const moespac_sched_config* cfg,
                                  int rank, int world, moespac_ctx** out) {
  return guard([&] {
    if (!m || !cfg || !out) throw std::invalid_argument("moespac_ctx_create: null argument");
    *out = new moespac_ctx(device, *m, *cfg, rank, world);
  });
}

void moespac_ctx_destroy(moespac_ctx* c) { delete c; }

moespac_status moespac_ctx_host_arena(moespac_ctx* c, int64_t n_images, uint16_t** arena) {
  return guard([&] { *arena = c->e.host_arena(n_images); });
}

moespac_status moespac_ctx_fill_synthetic(moespac_ctx* c, uint64_t seed, float stdv) {
  return guard([&] { c->e.fill_synthetic(seed, stdv); });
}

moespac_status moespac_ctx_estimator_dump(moespac_ctx* c, const char* path) {
  return guard([&] {
    if (!path) throw std::invalid_argument("moespac_ctx_estimator_dump: path");
    c->e.estimator_dump(path);
  });
}

moespac_status moespac_ctx_estimator_load(moespac_ctx* c, const char* path) {
  return guard([&] {
    if (!path) throw std::invalid_argument("moespac_ctx_estimator_load: path");
    c->e.estimator_load(path);
  });
}

moespac_status moespac_ctx_set_shared_gate(moespac_ctx* c, int layer, const uint16_t* w_sg) {
  return guard([&] { c->e.set_shared_gate(layer, w_sg); });
}

moespac_status moespac_ctx_set_shared(moespac_ctx* c, int layer, const uint16_t* units) {
  return guard([&] { c->e.set_shared(layer, units); });
}

moespac_status moespac_ctx_finalize(moespac_ctx* c) {
  return guard([&] { c->e.finalize(); });
}

moespac_status moespac_nccl_unique_id(void* out) {
  moespac_status st = MOESPAC_OK;
  moespac_status g = guard([&] { st = nccl_unique_id(out); });
  return g != MOESPAC_OK ? g : st;
}

moespac_status moespac_ctx_set_nccl(moespac_ctx* c, const void* uid, int nranks, int rank) {
  return guard([&] { c->e.set_nccl(uid, nranks, rank); });
}

moespac_status moespac_ctx_set_timing(moespac_ctx* c, int enabled) {
  return guard([&] { c->e.set_timing(enabled != 0); });
}

moespac_status moespac_ctx_set_cold_threads(moespac_ctx* c, int threads) {
  return guard([&] { c->e.set_cold_threads(threads); });
}

moespac_status moespac_ctx_set_cold_staging(moespac_ctx* c, int slots, double fraction) {
  return guard([&] { c->e.set_cold_staging(slots, fraction); });
}

moespac_status moespac_ctx_set_k3_trace(moespac_ctx* c, void* dev_buf) {
  return guard([&] { c->e.set_k3_trace(static_cast<unsigned long long*>(dev_buf)); });
}

moespac_status moespac_ctx_set_l2_prefetch(moespac_ctx* c, int bytes) {
  return guard([&] {
    if (bytes < 0) throw std::invalid_argument("moespac_ctx_set_l2_prefetch: bytes must be >= 0");
    c->e.set_l2_prefetch(bytes);
  });
}

moespac_status moespac_ctx_set_draft_window(moespac_ctx* c, int enabled) {
  return guard([&] { c->e.set_draft_window(enabled != 0); });
}

moespac_status moespac_ctx_set_draft_model(moespac_ctx* c, int64_t n_params, int d_draft) {
  return guard([&] {
    if (n_params < 0) throw std::invalid_argument("moespac_ctx_set_draft_model: n_params must be >= 0");
    c->e.set_draft_model(n_params, d_draft);
  });
}

moespac_status moespac_draft_gemv(const uint16_t* w, int64_t rows, int d, const float* y_prev, const uint16_t* x0,
                                  float scale, float* y, void* stream) {
  return guard([&] {
    if (!draft_d_ok(d) || rows < 1) throw std::invalid_argument("moespac_draft_gemv: shape");
    if (!y_prev && !x0) throw std::invalid_argument("moespac_draft_gemv: y_prev or x0 required");
    require_device();
    int dev = 0, sms = 148;
    cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    cuda_ok(launch_draft_gemv(w, rows, d, y_prev, x0, scale, y, sms, static_cast<cudaStream_t>(stream)),
            "draft_gemv");
  });
}

moespac_status moespac_ctx_set_timeline(moespac_ctx* c, int enabled) {
  return guard([&] {
    c->e.timeline_clear();
    c->e.set_timeline(enabled != 0);
  });
}

int64_t moespac_ctx_timeline_events(const moespac_ctx* c, int64_t* out, int64_t cap) {
  return c->e.timeline_events(out, cap);
}

int64_t moespac_ctx_timeline_layers(const moespac_ctx* c, moespac_layer_timing* out, int64_t cap) {
  return c->e.timeline_layers(out, cap);
}

int64_t moespac_ctx_timeline_steps(const moespac_ctx* c, int64_t* out, int64_t cap) {
  return c->e.timeline_steps(out, cap);
}

moespac_status moespac_ctx_set_graph(moespac_ctx* c, int enabled) {
  return guard([&] { c->e.set_graph(enabled != 0); });
}

moespac_status moespac_ctx_set_pdl(moespac_ctx* c, int enabled) {
  return guard([&] { c->e.set_pdl(enabled != 0); });
}

void* moespac_ctx_stream(const moespac_ctx* c) { return c->e.stream(); }

int moespac_ctx_parallel_mode(const moespac_ctx* c) {
  return c->e.unit_split() ? MOESPAC_PAR_UNITS : MOESPAC_PAR_EXPERT;
}

int moespac_ctx_k3_variant(const moespac_ctx* c) {
  if (c->e.ffn_kernel() != kFfnTensorCore) return MOESPAC_K3_CUDACORE;
  switch (c->e.ffn_acc_mode()) {
    case 0: return MOESPAC_K3_TC_SMEM;
    case 1: return MOESPAC_K3_TC_L2;
    case 2: return MOESPAC_K3_TC_TMEM;
    default: return MOESPAC_K3_GROUPED;
  }
}

moespac_status moespac_step(moespac_ctx* c, const double* logits, const uint16_t* h_in, int accepted, uint16_t* h_out,
                            moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] { c->e.step(logits, true, h_in, true, accepted, h_out, true, rep, layers); });
}

moespac_status moespac_ctx_set_router(moespac_ctx* c, int layer, const uint16_t* w) {
  return guard([&] {
    if (!w) throw std::invalid_argument("moespac_ctx_set_router: weights");
    c->e.set_router(layer, w);
  });
}

moespac_status moespac_step_model(moespac_ctx* c, const uint16_t* h_in, int accepted, uint16_t* h_out,
                                  moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] { c->e.step_model(h_in, true, accepted, h_out, true, rep, layers); });
}

moespac_status moespac_loopback_create(int device, int world, int64_t max_elems, moespac_loopback** out) {
  return guard([&] {
    if (!out || max_elems < 1) throw std::invalid_argument("moespac_loopback_create: arguments");
    require_device();
    *out = new moespac_loopback(device, world, static_cast<size_t>(max_elems));
  });
}

void moespac_loopback_destroy(moespac_loopback* g) { delete g; }

moespac_status moespac_ctx_set_loopback(moespac_ctx* c, moespac_loopback* g) {
  return guard([&] {
    if (!g) throw std::invalid_argument("moespac_ctx_set_loopback: group");
    c->e.set_loopback(&g->g);
  });
}

moespac_status moespac_step_model_device(moespac_ctx* c, const uint16_t* h_in, int accepted, uint16_t* h_out,
                                         moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] { c->e.step_model(h_in, false, accepted, h_out, false, rep, layers); });
}

moespac_status moespac_step_ids(moespac_ctx* c, const int32_t* ids, const float* gates, const uint16_t* h_in,
                                int accepted, uint16_t* h_out, moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] { c->e.step_ids(ids, gates, h_in, true, accepted, h_out, true, rep, layers); });
}

moespac_status moespac_step_device(moespac_ctx* c, const double* logits, const uint16_t* h_in, int accepted,
                                   uint16_t* h_out, moespac_step_report* rep, moespac_layer_timing* layers) {
  return guard([&] { c->e.step(logits, false, h_in, false, accepted, h_out, false, rep, layers); });
}

moespac_status moespac_ctx_step_tables(const moespac_ctx* c, int32_t* taus, uint32_t* rb, uint32_t* lb,
                                      int32_t* slots) {
  return guard([&] { c->e.step_tables(taus, rb, lb, slots); });
}

moespac_status moespac_ctx_get_views(const moespac_ctx* c, moespac_ctx_views* out) {
  return guard([&] { c->e.views(out); });
}

const moespac_sched* moespac_ctx_sched(const moespac_ctx* c) {
  // moespac_sched is layout-compatible with a StepScheduler (single member).
  return reinterpret_cast<const moespac_sched*>(&c->e.sched());
}

}  // extern "C"

// ------------------------------------------------------------------ routing traces
moespac_status moespac_trace_write(const char* path, int L, int N, int k, int gamma, int64_t n_steps,
                                   const int32_t* ids, const int32_t* accepted) {
  return guard([&] {
    if (!path || n_steps < 0 || (n_steps > 0 && (!ids || !accepted)))
      throw std::invalid_argument("moespac_trace_write: arguments");
    TraceData tr;
    tr.n_layers = L;
    tr.n_experts = N;
    tr.top_k = k;
    tr.gamma = gamma;
    tr.accepted.assign(accepted, accepted + n_steps);
    tr.ids.assign(ids, ids + n_steps * L * (gamma + 1) * k);
    write_trace(tr, path);
  });
}

moespac_status moespac_trace_read(const char* path, int32_t* shape4, int64_t* n_steps, int32_t* ids,
                                  int32_t* accepted, int64_t cap_steps) {
  return guard([&] {
    if (!path) throw std::invalid_argument("moespac_trace_read: path");
    const TraceData tr = read_trace(path);
    if (shape4) {
      shape4[0] = tr.n_layers;
      shape4[1] = tr.n_experts;
      shape4[2] = tr.top_k;
      shape4[3] = tr.gamma;
    }
    if (n_steps) *n_steps = tr.steps();
    if (ids || accepted) {
      if (cap_steps < tr.steps()) throw std::out_of_range("moespac_trace_read: buffer too small");
      if (ids) std::memcpy(ids, tr.ids.data(), sizeof(int32_t) * tr.ids.size());
      if (accepted) std::memcpy(accepted, tr.accepted.data(), sizeof(int32_t) * tr.accepted.size());
    }
  });
}

// ------------------------------------------------------------------ run metrics
namespace {

void to_c(const RunSummary& s, moespac_run_summary* o) {
  std::memset(o, 0, sizeof(*o));
  std::strncpy(o->axis_name, s.axis_name.c_str(), sizeof(o->axis_name) - 1);
  o->axis_value = s.axis_value;
  o->tps = s.tps;
  o->latency_s = s.latency_s;
  o->hit_rate = s.hit_rate;
  o->bubble_ratio = s.bubble_ratio;
  o->fault_rate = s.fault_rate;
  o->fn_rate = s.fn_rate;
  o->fp_rate = s.fp_rate;
  o->mean_accuracy = s.mean_accuracy;
  o->total_tokens = s.total_tokens;
  o->total_time_ns = s.total_time_ns;
  o->n_series = static_cast<int64_t>(s.accuracy_series.size());
}

}  // namespace

moespac_status moespac_summarize(const moespac_step_report* reps, const moespac_layer_timing* layers, int64_t n,
                                 int measured, moespac_run_summary* out, double* series) {
  return guard([&] {
    if (n < 0 || (n > 0 && !reps) || !out) throw std::invalid_argument("moespac_summarize: arguments");
    std::vector<StepReport> v(static_cast<size_t>(n));
    const moespac_layer_timing* lt = layers;
    for (int64_t i = 0; i < n; ++i) {
      const moespac_step_report& r = reps[i];
      StepReport& s = v[static_cast<size_t>(i)];
      s.draft_ns = r.draft_ns;
      s.accepted_tokens = r.accepted_tokens;
      s.cache_hits = r.cache_hits;
      s.cache_misses = r.cache_misses;
      s.accuracy = r.accuracy;
      s.faults_fn = r.faults_fn;
      s.faults_fp = r.faults_fp;
      s.n_experts = r.n_experts;
      s.step_wall_ns = measured && r.gpu_ms_total > 0.f ? std::llround(static_cast<double>(r.gpu_ms_total) * 1e6)
                                                        : r.step_wall_ns;
      if (lt) {
        s.layers.resize(static_cast<size_t>(r.n_layers));
        for (int l = 0; l < r.n_layers; ++l, ++lt) {
          LayerTiming& x = s.layers[static_cast<size_t>(l)];
          x.t_cpu_ns = lt->t_cpu_ns;
          x.t_gpu_ns = lt->t_gpu_ns;
          x.t_io_used_ns = lt->t_io_used_ns;
          x.stall_ns = lt->stall_ns;
          x.bubble_ns = lt->bubble_ns;
          x.wall_ns = lt->wall_ns;
          x.tau = lt->tau;
          x.fallback = lt->fallback != 0;
          x.n_prefetch = lt->n_prefetch;
        }
      } else {
        s.layers.resize(static_cast<size_t>(r.n_layers));
      }
    }
    const RunSummary rs = summarize(v);
    to_c(rs, out);
    if (series) std::memcpy(series, rs.accuracy_series.data(), sizeof(double) * rs.accuracy_series.size());
  });
}

moespac_status moespac_metrics_emit(const moespac_run_summary* summaries, const double* series, int64_t n, int format,
                                    const char* path) {
  return guard([&] {
    if (!path || n < 0 || (n > 0 && !summaries) || (format != 0 && format != 1))
      throw std::invalid_argument("moespac_metrics_emit: arguments");
    std::vector<RunSummary> v(static_cast<size_t>(n));
    const double* sp = series;
    for (int64_t i = 0; i < n; ++i) {
      const moespac_run_summary& c = summaries[i];
      RunSummary& s = v[static_cast<size_t>(i)];
      s.axis_name.assign(c.axis_name, strnlen(c.axis_name, sizeof(c.axis_name)));
      s.axis_value = c.axis_value;
      s.tps = c.tps;
      s.latency_s = c.latency_s;
      s.hit_rate = c.hit_rate;
      s.bubble_ratio = c.bubble_ratio;
      s.fault_rate = c.fault_rate;
      s.fn_rate = c.fn_rate;
      s.fp_rate = c.fp_rate;
      s.mean_accuracy = c.mean_accuracy;
      s.total_tokens = c.total_tokens;
      s.total_time_ns = c.total_time_ns;
      if (c.n_series > 0) {
        if (!sp) throw std::invalid_argument("moespac_metrics_emit: series required");
        s.accuracy_series.assign(sp, sp + c.n_series);
        sp += c.n_series;
      }
    }
    emit(v, format == 0 ? MetricsFormat::csv : MetricsFormat::jsonl, path);
  });
}

moespac_status moespac_metrics_parse(const char* path, moespac_run_summary* out, int64_t cap, double* series,
                                     int64_t series_cap, int64_t* n_out) {
  return guard([&] {
    if (!path) throw std::invalid_argument("moespac_metrics_parse: path");
    const std::vector<RunSummary> v = parse_metrics(path);
    if (n_out) *n_out = static_cast<int64_t>(v.size());
    if (!out) return;
    if (cap < static_cast<int64_t>(v.size())) throw std::out_of_range("moespac_metrics_parse: buffer too small");
    int64_t used = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      to_c(v[i], &out[i]);
      const int64_t ns = static_cast<int64_t>(v[i].accuracy_series.size());
      if (series) {
        if (used + ns > series_cap) throw std::out_of_range("moespac_metrics_parse: series buffer too small");
        std::memcpy(series + used, v[i].accuracy_series.data(), sizeof(double) * static_cast<size_t>(ns));
      }
      used += ns;
    }
  });
}
