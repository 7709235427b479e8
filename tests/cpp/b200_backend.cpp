// The reference-side binding of INTEGRATION.md, as a translation unit that
// compiles against the reference's own headers
// (/root/reference/proj/core/include/moesim) and this repository's C ABI
// (include/moespac/moespac.h). tests/test_cpp_api.py compiles it (syntax +
// types; it links nothing) whenever /root/reference is mounted.
//
// B200Backend replaces Simulation::run_utility_step
// (core/src/sim_core.cpp:157-316) for the utility-family policies: one
// context per GPU, one moespac_step per verification step, the reports
// copied back into the reference's StepReport / LayerTiming.
#include <cstdint>
#include <stdexcept>
#include <vector>

#include "moesim/sim_core.hpp"
#include "moespac/moespac.h"

namespace moesim {

class B200Backend {
 public:
  // d_model / d_ffn / gate_mode describe the real expert FFN the reference
  // models as a constant (sim_core.cpp:253-254).
  B200Backend(const SimConfig& c, int d_model, int d_ffn, int gate_mode, int device = 0) : n_layers_(c.trace.n_layers) {
    moespac_sched_config cfg;
    moespac_default_sched_config(&cfg);  // == default_sim_config() (config.cpp:11-39)
    cfg.n_layers = c.trace.n_layers;
    cfg.n_experts = c.trace.n_experts;
    cfg.top_k = c.trace.top_k;
    cfg.gamma = c.trace.gamma;
    cfg.alpha = c.trace.alpha;
    cfg.drift_scale = c.trace.drift_scale;
    cfg.route_noise = c.trace.route_noise;
    cfg.shift_period = c.trace.shift_period;
    cfg.seed = c.trace.seed;
    cfg.t_cpu_unit_ns = c.profile.t_cpu_unit_ns;
    cfg.t_gpu_unit_ns = c.profile.t_gpu_unit_ns;
    cfg.t_io_unit_ns = c.profile.t_io_unit_ns;
    cfg.t_draft_unit_ns = c.profile.t_draft_unit_ns;
    cfg.expert_bytes = c.profile.expert_bytes;
    cfg.utility_cap = c.estimator.utility_cap;
    cfg.adaptive_boundaries = c.estimator.adaptive_boundaries ? 1 : 0;
    cfg.forgetting = c.estimator.forgetting;
    cfg.init_up = c.estimator.init_up;
    cfg.init_down = c.estimator.init_down;
    cfg.policy = static_cast<int32_t>(c.policy.kind);
    cfg.fixed_tau = c.policy.fixed_tau;
    cfg.fixed_up = c.policy.fixed_up;
    cfg.fixed_down = c.policy.fixed_down;
    cfg.cache_ratio = c.cache_ratio;
    cfg.ratio_smoothing = c.ratio_smoothing;
    moespac_model_desc m{};
    m.n_layers = cfg.n_layers;
    m.n_experts = cfg.n_experts;
    m.top_k = cfg.top_k;
    m.gamma = cfg.gamma;
    m.d_model = d_model;
    m.d_ffn = d_ffn;
    m.gate_mode = gate_mode;
    m.ffn_kernel = MOESPAC_FFN_AUTO;
    check(moespac_ctx_create(device, &m, &cfg, /*shard_rank=*/0, /*shard_world=*/1, &ctx_));
    uint16_t* arena = nullptr;  // pinned master copy of every expert
    check(moespac_ctx_host_arena(ctx_, int64_t(cfg.n_layers) * cfg.n_experts, &arena));
    arena_ = arena;
    image_elems_ = moespac_expert_image_elems(d_model, d_ffn);
  }
  ~B200Backend() { moespac_ctx_destroy(ctx_); }
  B200Backend(const B200Backend&) = delete;
  B200Backend& operator=(const B200Backend&) = delete;

  // expert (l, e)'s image, in moespac_pack_expert's layout, goes here before finalize()
  uint16_t* expert_image(int layer, int expert, int n_experts) {
    return arena_ + (int64_t(layer) * n_experts + expert) * image_elems_;
  }
  void finalize() { check(moespac_ctx_finalize(ctx_)); }

  // replaces run_utility_step: logits = router scores of the gamma+1
  // verified tokens [L][gamma+1][N], hidden states in / out [gamma+1][d]
  StepReport step(const double* logits, const uint16_t* h_in, int accepted, uint16_t* h_out) {
    moespac_step_report r;
    std::vector<moespac_layer_timing> lt(static_cast<size_t>(n_layers_));
    check(moespac_step(ctx_, logits, h_in, accepted, h_out, &r, lt.data()));
    StepReport rep;
    rep.draft_ns = r.draft_ns;
    rep.accepted_tokens = r.accepted_tokens;
    rep.cache_hits = r.cache_hits;
    rep.cache_misses = r.cache_misses;
    rep.accuracy = r.accuracy;
    rep.faults_fn = r.faults_fn;
    rep.faults_fp = r.faults_fp;
    rep.n_experts = r.n_experts;
    rep.step_wall_ns = r.step_wall_ns;
    for (const moespac_layer_timing& x : lt) {
      LayerTiming y;
      y.t_cpu_ns = x.t_cpu_ns;
      y.t_gpu_ns = x.t_gpu_ns;
      y.t_io_used_ns = x.t_io_used_ns;
      y.stall_ns = x.stall_ns;
      y.bubble_ns = x.bubble_ns;
      y.wall_ns = x.wall_ns;
      y.tau = x.tau;
      y.fallback = x.fallback != 0;
      y.n_prefetch = x.n_prefetch;
      rep.layers.push_back(y);
    }
    return rep;
  }

  // LayerEstimator::dump / load for the whole model (utility_estimator.cpp:81-107)
  void checkpoint(const char* path) { check(moespac_ctx_estimator_dump(ctx_, path)); }
  void restore(const char* path) { check(moespac_ctx_estimator_load(ctx_, path)); }

 private:
  static void check(moespac_status s) {
    switch (s) {  // the reference's exception classes
      case MOESPAC_OK:
        return;
      case MOESPAC_E_INVALID:
        throw std::invalid_argument(moespac_last_error());
      case MOESPAC_E_RANGE:
        throw std::out_of_range(moespac_last_error());
      case MOESPAC_E_LOGIC:
        throw std::logic_error(moespac_last_error());
      default:
        throw std::runtime_error(moespac_last_error());
    }
  }
  moespac_ctx* ctx_ = nullptr;
  uint16_t* arena_ = nullptr;
  int64_t image_elems_ = 0;
  int n_layers_ = 0;
};

// Simulation::run_step (sim_core.cpp:137-144) would dispatch the utility
// family here; the reactive baselines stay on the reference path.
StepReport run_step_on_b200(B200Backend& backend, const double* logits, const uint16_t* h_in, int accepted,
                            uint16_t* h_out) {
  return backend.step(logits, h_in, accepted, h_out);
}

}  // namespace moesim
