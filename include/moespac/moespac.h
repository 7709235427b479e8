/*
 * moespac.h — C ABI of the B200-native MoE-SpAc verification-step hot path.
 *
 * This is the drop-in boundary for the reference's verification-step path
 * (/root/reference/proj/core — C++ namespace `moesim`). The reference exposes
 * only a C++ API; every entry point below names the reference routine it
 * replaces (file:line relative to /root/reference/proj). INTEGRATION.md shows
 * the binding a maintainer adds on the reference side.
 *
 * Conventions:
 *  - Every function returns moespac_status and never throws. Error classes map
 *    1:1 onto the reference's exceptions: MOESPAC_E_INVALID <-
 *    std::invalid_argument, MOESPAC_E_RANGE <- std::out_of_range,
 *    MOESPAC_E_LOGIC <- std::logic_error, MOESPAC_E_IO <- std::runtime_error;
 *    plus MOESPAC_E_CUDA / MOESPAC_E_NCCL / MOESPAC_E_NOMEM. The message of the
 *    last failure on the calling thread is moespac_last_error().
 *  - Plain pointers and sizes only. "_dev" pointers are device (HBM) memory,
 *    "_host" pointers host memory. `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).
 *  - The caller owns I/O buffers; a context owns expert slot pools, copy
 *    streams, estimator state and scheduler state. One context per device,
 *    driven by one host thread (not reentrant), mirroring the reference's
 *    single-mutator rule.
 *  - There is no CPU fallback: device entry points fail with
 *    MOESPAC_E_CUDA when no usable sm_100 device is present.
 */
#ifndef MOESPAC_MOESPAC_H
#define MOESPAC_MOESPAC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOESPAC_ABI_VERSION 2

typedef enum moespac_status {
  MOESPAC_OK = 0,
  MOESPAC_E_INVALID = 1,
  MOESPAC_E_RANGE = 2,
  MOESPAC_E_LOGIC = 3,
  MOESPAC_E_IO = 4,
  MOESPAC_E_CUDA = 5,
  MOESPAC_E_NCCL = 6,
  MOESPAC_E_NOMEM = 7
} moespac_status;

const char* moespac_last_error(void);
int moespac_abi_version(void);

/* ------------------------------------------------------------------ config
 * moespac_sched_config mirrors moesim::SimConfig (core/include/moesim/
 * sim_core.hpp:23-36) with TraceConfig, HardwareProfile, EstimatorConfig and
 * PolicySpec flattened; moespac_default_sched_config() == default_sim_config()
 * (core/src/config.cpp:11-39). `policy` uses moesim::PolicyKind numbering
 * (core/include/moesim/policies.hpp:18-27). */
typedef struct moespac_sched_config {
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
} moespac_sched_config;

void moespac_default_sched_config(moespac_sched_config* out);

/* LayerTiming / StepReport (core/include/moesim/sim_core.hpp:38-61). */
typedef struct moespac_layer_timing {
  int64_t t_cpu_ns, t_gpu_ns, t_io_used_ns, stall_ns, bubble_ns, wall_ns;
  int32_t tau, fallback, n_prefetch, n_loads;
} moespac_layer_timing;

typedef struct moespac_step_report {
  int64_t draft_ns, cache_hits, cache_misses, faults_fn, faults_fp, step_wall_ns;
  double accuracy;
  int32_t accepted_tokens, n_experts, n_layers, n_loads;
  /* measured on the device for this step (0 when timing is off) */
  float gpu_ms_total, gpu_ms_router, gpu_ms_hist, gpu_ms_ffn, gpu_ms_combine, gpu_ms_h2d_loads;
  /* algorithmic K3 bytes this step on this rank: (local hit experts + shared
   * units) x image bytes, summed over layers; and the kernel launches issued */
  int64_t ffn_bytes, h2d_bytes, d2h_bytes;
  int32_t kernel_launches;
  /* cold path: (layer, expert) misses computed on the host cores this step
   * and the host time spent on them */
  int32_t cold_experts;
  float cpu_ms_cold;
  /* K3 launches this step (one per layer) */
  int32_t ffn_launches;
  /* draft phase this step: device time (timing on) and draft-model weight
   * bytes streamed (moespac_ctx_set_draft_model; 0 for the emulated window) */
  float gpu_ms_draft;
  int64_t draft_bytes;
  /* cold experts of this step run on the device from the staging ring
   * (moespac_ctx_set_cold_staging); cold_experts counts the host-run ones */
  int32_t staged_experts;
} moespac_step_report;

/* Realized split of one layer (core/src/sim_core.cpp:233-283), as K2 emits it. */
typedef struct moespac_layer_outcome {
  int32_t distinct, distinct_hits, hit_tokens, miss_tokens, agree, faults_fn, faults_fp, n_local_hits;
} moespac_layer_outcome;

/* ------------------------------------------------------------------ host scheduler
 * Heterogeneous Workload Balancer + Asynchronous Execution Engine bookkeeping,
 * host only (no device needed). Replaces the per-layer decision half of
 * Simulation::run_utility_step (core/src/sim_core.cpp:177-228) and its
 * accounting half (:229-297). shard_world > 1 runs expert-partitioned
 * bookkeeping (expert e on shard e % shard_world). */
typedef struct moespac_sched moespac_sched;

moespac_status moespac_sched_create(const moespac_sched_config* cfg, int shard_world, moespac_sched** out);
void moespac_sched_destroy(moespac_sched* s);
/* Phase 1: scores_host [L][N] = estimator snapshot after the previous step. */
moespac_status moespac_sched_decide(moespac_sched* s, const int32_t* scores_host);
/* Decision tables of the last decide(): taus [L], resident/loaded bitmaps
 * [L][ceil(N/32)], slot table [L][N] (slot within the owning shard, -1 if not
 * resident). Any pointer may be NULL. */
moespac_status moespac_sched_tables(const moespac_sched* s, int32_t* taus, uint32_t* resident_bits,
                                    uint32_t* loaded_bits, int32_t* slot_table);
/* Per-layer ThresholdDecision: [L][5] = tau, fallback, pred_cpu_ns, pred_gpu_ns, n_prefetch. */
moespac_status moespac_sched_decisions(const moespac_sched* s, int64_t* out);
/* Ordered loads of the last decide(): [n][4] = layer, expert, shard, slot. Returns n (or -1). */
int64_t moespac_sched_loads(const moespac_sched* s, int32_t* out, int64_t cap);
/* Phase 2 with K2 counters [L], or with host frequencies [L][N]. */
moespac_status moespac_sched_observe(moespac_sched* s, const moespac_layer_outcome* outcomes, int accepted,
                                     moespac_step_report* rep, moespac_layer_timing* layers);
moespac_status moespac_sched_observe_freqs(moespac_sched* s, const int32_t* freqs_host, int accepted,
                                           moespac_step_report* rep, moespac_layer_timing* layers);
/* SimEvent log (sim_core.hpp:65-73): [n][6] = kind, step, layer, expert, start_ns, duration_ns. */
int64_t moespac_sched_events(const moespac_sched* s, int64_t* out, int64_t cap);
int64_t moespac_sched_total_time_ns(const moespac_sched* s);
moespac_status moespac_sched_ratios(const moespac_sched* s, int layer, double* cpu_ratio, double* gpu_ratio,
                                    int32_t* b_est);

/* solve_threshold (core/src/workload_balancer.cpp:106-167). resident: [n] bytes.
 * out[6] = tau, fallback, pred_cpu_ns, pred_gpu_ns, n_prefetch, evals. */
moespac_status moespac_solve_threshold(const int32_t* scores, int n, const uint8_t* resident, int gamma,
                                       int top_k, int b_est, const double* cpu_ratio, const double* gpu_ratio,
                                       int cap, int64_t t_cpu_unit_ns, int64_t t_gpu_unit_ns,
                                       int64_t t_io_unit_ns, int64_t expert_bytes, int64_t vram_left_bytes,
                                       int64_t draft_credit_ns, int64_t* out);
/* update_ratio_estimates (core/src/workload_balancer.cpp:169-199), in place. */
moespac_status moespac_update_ratio_estimates(double* cpu_ratio, double* gpu_ratio, int cap, int tau_used,
                                              double observed_rc, double observed_rg, double smoothing);
/* layer_capacity_experts (core/src/sim_core.cpp:31-34). */
int moespac_layer_capacity_experts(double cache_ratio, int n_experts);

/* ------------------------------------------------------------------ synthetic workload
 * The host half of TraceGenerator::next_step (core/src/trace_model.cpp:73-109):
 * the latent random walk and per-token Gumbel noise from the same
 * mt19937_64 stream, emitted as noisy fp64 logits [L][gamma+1][N] for K1 (the
 * top-k selection itself runs on the device). Uses the trace fields of cfg. */
/* The whole generator on the host (TraceGenerator::next_step, trace_model.cpp:
 * 73-109, incl. its top-k): ids [n_steps][L][gamma+1][k] ascending per
 * token, accepted [n_steps] (either may be NULL). The operator for trace
 * export; the device path takes logits (below) and selects with K1. */
moespac_status moespac_trace_generate(const moespac_sched_config* cfg, int64_t n_steps, int32_t* ids,
                                      int32_t* accepted);
typedef struct moespac_trace_synth moespac_trace_synth;
moespac_status moespac_trace_synth_create(const moespac_sched_config* cfg, moespac_trace_synth** out);
moespac_status moespac_trace_synth_next(moespac_trace_synth* s, double* logits_host, int32_t* accepted);
void moespac_trace_synth_destroy(moespac_trace_synth* s);

/* ------------------------------------------------------------------ routing traces
 * The reference's line format `#moetrace v1` (core/src/trace_model.cpp:132-254):
 * ids [n_steps][n_layers][gamma+1][top_k] in file order, accepted [n_steps].
 * read: call once with ids == NULL to get shape[4] = layers, experts, k,
 * gamma and *n_steps, then with buffers of cap_steps steps. Parse errors are
 * MOESPAC_E_IO with the reference's message ("read_trace: <path>:<line>: ..."). */
moespac_status moespac_trace_write(const char* path, int n_layers, int n_experts, int top_k, int gamma,
                                   int64_t n_steps, const int32_t* ids, const int32_t* accepted);
moespac_status moespac_trace_read(const char* path, int32_t* shape4, int64_t* n_steps, int32_t* ids,
                                  int32_t* accepted, int64_t cap_steps);

/* ------------------------------------------------------------------ run metrics
 * RunSummary / summarize / emit / parse_metrics in the reference's
 * `#moesim-metrics v1` schema (core/src/metrics_report.cpp:12-183).
 * summarize: n step reports with their layer timings [n][n_layers];
 * measured != 0 replaces each step's modeled wall time by its device time
 * (gpu_ms_total, needs moespac_ctx_set_timing) for tps / latency. series
 * [n] receives the per-step accuracy series (may be NULL).
 * emit: format 0 = CSV, 1 = JSONL; series = the n summaries' accuracy
 * series concatenated (lengths in n_series). parse: up to cap summaries,
 * their series concatenated into series (series_cap values); *n_out = count. */
typedef struct moespac_run_summary {
  char axis_name[64];
  double axis_value, tps, latency_s, hit_rate, bubble_ratio, fault_rate, fn_rate, fp_rate, mean_accuracy;
  int64_t total_tokens, total_time_ns;
  int64_t n_series;
} moespac_run_summary;
moespac_status moespac_summarize(const moespac_step_report* reps, const moespac_layer_timing* layers, int64_t n,
                                 int measured, moespac_run_summary* out, double* series);
moespac_status moespac_metrics_emit(const moespac_run_summary* summaries, const double* series, int64_t n, int format,
                                    const char* path);
moespac_status moespac_metrics_parse(const char* path, moespac_run_summary* out, int64_t cap, double* series,
                                     int64_t series_cap, int64_t* n_out);

/* ------------------------------------------------------------------ device kernels (stateless)
 * K1 — router top-k + gates. Replaces the selection block of
 * TraceGenerator::next_step (core/src/trace_model.cpp:87-104).
 * logits_dev [rows][n_experts] fp64 -> ids_dev [rows][top_k] ascending,
 * gates_dev [rows][top_k] fp32 (may be NULL). gate_mode 0: softmax over the
 * selected k (Eq. 3); 1: softmax over all N, not renormalised. n_experts <= 1024. */
moespac_status moespac_router_topk(const double* logits_dev, int rows, int n_experts, int top_k, int gate_mode,
                                   int32_t* ids_dev, float* gates_dev, void* stream);

/* K2 — per layer: activation histogram (trace_model.cpp:122-130), exclusive
 * scan, (expert, token, slot)-sorted permutation, LayerEstimator::observe_step
 * (utility_estimator.cpp:47-72) in place on est_state_dev, and the realized
 * split / accuracy / fault counters (sim_core.cpp:233-283). One launch for all
 * layers. */
typedef struct moespac_k2_args {
  const int32_t* ids_dev;          /* [L][T][k] */
  int32_t n_layers, tokens, top_k, n_experts;
  const uint32_t* resident_bits_dev; /* [L][W] after this step's loads */
  const uint32_t* loaded_bits_dev;   /* [L][W] loaded this step, or NULL */
  const int32_t* taus_dev;           /* [L] */
  int32_t* est_state_dev;            /* [L][N][4] score, up, down, last_freq */
  int32_t utility_cap, adaptive_boundaries;
  double forgetting;
  int32_t shard_rank, shard_world;
  int32_t* freqs_dev;      /* [L][N] */
  int32_t* offsets_dev;    /* [L][N+1] */
  int32_t* perm_dev;       /* [L][T*k] */
  int32_t* hit_list_dev;   /* [L][N] */
  int32_t* hit_ord_dev;    /* [L][N] */
  int32_t* counters_dev;   /* [L][8] = moespac_layer_outcome */
  int32_t* scores_out_dev; /* [L][N] */
} moespac_k2_args;
moespac_status moespac_hist_scan_observe(const moespac_k2_args* a, void* stream);

/* LayerEstimator constructor state (utility_estimator.cpp:23-33) for n experts. */
moespac_status moespac_estimator_init(int32_t* est_state_dev, int n, int gamma, int init_up, int init_down,
                                      void* stream);

/* K3 — grouped SwiGLU expert FFN over the resident activated experts of one
 * layer (replaces the modeled charge at core/src/sim_core.cpp:253-254).
 * Two kernels, one contract: MOESPAC_FFN_TENSOR (tcgen05.mma, TMEM
 * accumulators; needs d % 128 == 0, ffn % 64 == 0) and MOESPAC_FFN_CUDACORE
 * (weight-streaming GEMV on the CUDA cores; d % 512 == 0, ffn % 16 == 0).
 * Expert images must be packed for the kernel that reads them. */
#define MOESPAC_FFN_AUTO 0
#define MOESPAC_FFN_CUDACORE 1
#define MOESPAC_FFN_TENSOR 2
int moespac_ffn_resolve(int kernel, int d_model, int d_ffn);
/* h [T][d] bf16 -> h^T UMMA operand image (16 * d bf16) for the tensor kernel. */
moespac_status moespac_build_hT(const uint16_t* h_dev, int tokens, int d_model, uint16_t* hT_dev, void* stream);
typedef struct moespac_ffn_args {
  const uint16_t* h_dev;       /* [T][d] bf16 */
  int32_t tokens, d_model, d_ffn, top_k, n_experts;
  const int32_t* perm_dev, *offsets_dev;
  const float* gates_dev;      /* [T][k] */
  const int32_t* hit_list_dev, *counters_dev; /* one layer's K2 outputs */
  const int32_t* slot_of_dev;  /* [N] */
  const uint16_t* pool_dev;    /* tiled expert images, one per slot */
  const uint16_t* shared_dev;  /* tiled shared-expert units */
  int32_t n_shared_units;
  float* workspace_dev;        /* moespac_ffn_workspace_bytes() */
  int32_t grid;                /* 0 = one CTA per SM */
  int32_t kernel;              /* MOESPAC_FFN_* (image layout must match) */
  const uint16_t* hT_dev;      /* tensor-core kernel: moespac_build_hT(h) image */
  uint64_t* debug_ts_dev;      /* optional [grid][32] per-CTA profiling record (%globaltimer stamps, wait counters), or NULL */
  int32_t accum;               /* tensor-core kernel: 0 auto, 1 shared-memory, 2 L2 (partial-block), 3 TMEM accumulator
                                  per expert (d <= 2048), 4 grouped: whole-CTA TMEM accumulator (d <= 2048; auto's choice) */
  int32_t l2_policy;           /* weight stream L2 policy: 0 evict_first (default), 1 evict_normal */
} moespac_ffn_args;
size_t moespac_ffn_workspace_bytes(int tokens, int d_model, int n_experts, int n_shared_units, int grid);
int64_t moespac_expert_image_elems(int d_model, int d_ffn);
moespac_status moespac_expert_ffn(const moespac_ffn_args* a, void* stream);

/* Combine: y = sum of the K3 partials in fixed order; writes y_dev [T][d] fp32
 * and/or h_out_dev = bf16(h_in + y + y_extra). ids/hit_ord from K1/K2. */
typedef struct moespac_combine_args {
  const uint16_t* h_in_dev;
  const float* y_extra_dev;
  int32_t tokens, d_model, d_ffn, top_k;
  const int32_t* ids_dev, *hit_ord_dev, *counters_dev;
  int32_t n_shared_units, grid;
  const float* workspace_dev;
  float* y_dev;
  uint16_t* h_out_dev;
  int32_t accum;               /* the accum selector the K3 launch used (decides the partial-block layout) */
  int32_t kernel;              /* the MOESPAC_FFN_* kernel the K3 launch used */
} moespac_combine_args;
moespac_status moespac_ffn_combine(const moespac_combine_args* a, void* stream);

/* Standard layouts (w_gate, w_up: [ffn][d]; w_down: [d][ffn]) -> tiled image. */
moespac_status moespac_pack_expert(const uint16_t* w_gate_dev, const uint16_t* w_up_dev,
                                   const uint16_t* w_down_dev, int d_model, int d_ffn, int kernel,
                                   uint16_t* image_dev, void* stream);
/* Inverse of moespac_pack_expert: tiled image -> standard layouts (export /
 * checkpointing of the resident pool; parity checks on synthetic images). */
moespac_status moespac_unpack_expert(const uint16_t* image_dev, int d_model, int d_ffn, int kernel,
                                     uint16_t* w_gate_dev, uint16_t* w_up_dev, uint16_t* w_down_dev, void* stream);
moespac_status moespac_fill_synthetic(uint16_t* dev, int64_t n_elems, uint64_t seed, float stdv, void* stream);

/* ------------------------------------------------------------------ engine context
 * The full verification step on one device: K1 -> K2 -> per layer
 * [wait own loads] K3 -> combine (-> NCCL all-gather + ordered sum in the multi-GPU modes),
 * with the host scheduler deciding every layer's tau and loads during the
 * draft window and the Asynchronous Execution Engine issuing each load as a
 * pinned-host -> HBM cudaMemcpyAsync on a copy stream. Replaces
 * Simulation::run_utility_step (core/src/sim_core.cpp:157-316). */
typedef struct moespac_model_desc {
  int32_t n_layers, n_experts, top_k, gamma;
  int32_t d_model, d_ffn;
  int32_t n_shared_units; /* shared experts expressed in units of d_ffn rows */
  int32_t gate_mode;      /* see moespac_router_topk */
  int32_t ffn_kernel;     /* MOESPAC_FFN_*; expert images use its layout */
  int32_t parallel_mode;  /* world > 1 only — MOESPAC_PAR_*; see below */
  int32_t shared_gate;    /* MOESPAC_SHARED_GATE_*: how shared units enter the layer output */
} moespac_model_desc;

/* Shared-expert gate (SURVEY.md §8 gate flags): NONE adds the shared units
 * with weight 1 (DeepSeek-V2-Lite); SIGMOID scales them per token by
 * sigmoid(w_sg . h_t) with a per-layer gate vector w_sg [d_model]
 * (Qwen1.5-MoE's shared_expert_gate; set with moespac_ctx_set_shared_gate;
 * grouped tensor-core K3 only: d_model <= 2048). */
#define MOESPAC_SHARED_GATE_NONE 0
#define MOESPAC_SHARED_GATE_SIGMOID 1

/* Multi-GPU modes (shard_world > 1 in moespac_ctx_create):
 * EXPERT: expert e lives on rank e % world (its own slot pool, the
 *   balancer solves tau on the global scores).
 * UNITS: every rank holds every expert (the budget must cover all of them:
 *   cache_ratio 1.0) and each layer's (expert, 8-row unit) work list is cut
 *   across the ranks' K3 CTAs as one virtual grid, so the per-GPU work is
 *   balanced whatever the routing; tensor-core K3 only.
 * AUTO: UNITS when it applies, else EXPERT. Both combine with one
 *   all-gather (NCCL) of the per-rank fp32 partial outputs per layer, then
 *   every rank sums them in rank order (deterministic; the loopback group
 *   runs the same ordered-sum kernel, so it pins the NCCL path's bits). */
#define MOESPAC_PAR_AUTO 0
#define MOESPAC_PAR_EXPERT 1
#define MOESPAC_PAR_UNITS 2

typedef struct moespac_ctx moespac_ctx;

/* expert_bytes in cfg is overridden by the real image size. */
moespac_status moespac_ctx_create(int device, const moespac_model_desc* model, const moespac_sched_config* cfg,
                                  int shard_rank, int shard_world, moespac_ctx** out);
void moespac_ctx_destroy(moespac_ctx* c);
/* Pinned host master copy: n_images tiled expert images; expert (l, e) is
 * image (l*N + e) % n_images. Returns the host pointer for the caller to fill. */
moespac_status moespac_ctx_host_arena(moespac_ctx* c, int64_t n_images, uint16_t** arena_host);
/* Fill arena images + shared units with synthetic weights (seeded per image). */
moespac_status moespac_ctx_fill_synthetic(moespac_ctx* c, uint64_t seed, float stdv);
/* Shared units of layer l from a device buffer [n_shared_units][image]. */
moespac_status moespac_ctx_set_shared(moespac_ctx* c, int layer, const uint16_t* units_dev);
/* Shared-expert gate vector of layer l, [d_model] bf16 (host or device
 * pointer), for MOESPAC_SHARED_GATE_SIGMOID (filled synthetically by
 * moespac_ctx_fill_synthetic otherwise). */
moespac_status moespac_ctx_set_shared_gate(moespac_ctx* c, int layer, const uint16_t* w_sg);
/* Estimator checkpoint (LayerEstimator::dump / load, utility_estimator.cpp:
 * 81-107): the device estimator state of every layer in the reference's text
 * format, layer after layer, one line "<layer> <expert> <score> <up> <down>
 * <last_freq>" per expert. load parses every layer before changing anything
 * (MOESPAC_E_IO with the reference's message on a truncated / malformed
 * checkpoint), uploads it, and the next step decides from its scores. The
 * residency pools, queues and ratio estimates are not part of it (the
 * reference does not serialise them either). */
moespac_status moespac_ctx_estimator_dump(moespac_ctx* c, const char* path);
moespac_status moespac_ctx_estimator_load(moespac_ctx* c, const char* path);
/* Upload the warm-fill residents (sim_core.cpp:108-111) from the arena. */
moespac_status moespac_ctx_finalize(moespac_ctx* c);
/* Expert-parallel combine over NCCL: 128-byte ncclUniqueId from rank 0. */
moespac_status moespac_nccl_unique_id(void* out128);
moespac_status moespac_ctx_set_nccl(moespac_ctx* c, const void* unique_id128, int nranks, int rank);
/* In-process stand-in for the expert-parallel all-gather: `world` contexts on
 * ONE device (one host thread each) exchange their per-layer partial outputs
 * through device slots instead of NCCL (which refuses two ranks on one GPU).
 * Test harness for the expert-parallel device path on a single GPU;
 * max_elems >= tokens * d_model. Use instead of moespac_ctx_set_nccl. */
typedef struct moespac_loopback moespac_loopback;
moespac_status moespac_loopback_create(int device, int world, int64_t max_elems, moespac_loopback** out);
void moespac_loopback_destroy(moespac_loopback* g);
moespac_status moespac_ctx_set_loopback(moespac_ctx* c, moespac_loopback* g);
/* Per-kernel CUDA-event timing in moespac_step_report (off by default). While
 * timing is on, layer kernels are launched without programmatic dependent
 * launch so each K3 event pair brackets exactly that kernel. */
moespac_status moespac_ctx_set_timing(moespac_ctx* c, int enabled);
/* Host threads for the cold-expert path (activations whose expert is not
 * resident are computed on the CPU from the pinned arena, in parallel with
 * the device, and added by the combine): -1 = all cores (default), 0 = off
 * (misses are counted but not computed). Takes effect at moespac_ctx_finalize. */
moespac_status moespac_ctx_set_cold_threads(moespac_ctx* c, int threads);
/* Cold experts staged through HBM: of each layer's misses, a fixed fraction
 * (spread evenly over the misses in expert order, at most slots/2 per layer)
 * is copied pinned host -> a staging ring of `slots` expert images (two
 * layers in flight, outside the cache budget's slots) on a side stream and
 * run by that layer's K3 with the resident experts; the rest stay on the
 * host cores. The misses' decisions and accounting are unchanged (the
 * reference's HWB decides residency; this only chooses where a miss is
 * computed: host DRAM -> cores, or host DRAM -> PCIe -> tensor cores).
 * slots even, >= 0 (0 = off, the default); fraction in [0, 1]. Takes effect
 * at moespac_ctx_finalize. Replaces nothing in the reference (its misses are
 * modeled as CPU time, core/src/sim_core.cpp:253-254). */
moespac_status moespac_ctx_set_cold_staging(moespac_ctx* c, int slots, double fraction);
/* Emulated draft window (off by default): each step first holds the compute
 * stream for gamma * t_draft_unit_ns (the reference's modeled draft phase,
 * sim_core.cpp:167-172) while the copy engine works through the step's
 * expert loads — the overlap the balancer's draft credit assumes. Steps then
 * measure draft + verification, the reference's TPS definition. */
moespac_status moespac_ctx_set_draft_window(moespac_ctx* c, int enabled);
/* Real draft phase (replaces the modeled window of
 * sim_core.cpp:167-172): a dense draft model of n_params bf16 weights (rows
 * of d_draft) on the same GPU; each step first runs gamma autoregressive
 * draft passes — one weight-streaming GEMV over all n_params per draft token,
 * each fed by the previous pass's output — on the compute stream, while the
 * copy engine works through the step's expert loads. Steps then measure
 * draft + verification. n_params = 0 turns it off. (Qwen3-4B-FP8, the
 * paper's draft, streams ~4 GB per token: n_params 2e9 bf16, d_draft 2560.) */
moespac_status moespac_ctx_set_draft_model(moespac_ctx* c, int64_t n_params, int d_draft);
/* One draft pass as a stateless kernel (the draft model's building block):
 * y [R] fp32 = W [R][D] bf16 . x, x = bf16(scale * y_prev[0:D]) or x0 [D]
 * bf16 when y_prev is NULL. D as moespac_ctx_set_draft_model's d_draft. */
moespac_status moespac_draft_gemv(const uint16_t* w_dev, int64_t rows, int d, const float* y_prev_dev,
                                  const uint16_t* x0_dev, float scale, float* y_dev, void* stream);
/* Measured timeline: while on, every step appends
 * device-measured records in the reference's SimEvent schema
 * (sim_core.hpp:65-73): [n][6] = kind (0 draft, 1 cpu, 2 gpu, 3 stall,
 * 4 load, 5 evict), step, layer, expert, start_ns, duration_ns — gpu = K3 +
 * combine of the layer on the compute stream, stall = the compute stream's
 * wait for the layer's loads, load = one H2D copy on the copy stream, cpu =
 * the host cold path of the layer (host clock; start = the layer's K3
 * start), draft = the draft phase. Starts are on the context's measured
 * clock (sum of earlier steps' totals). Implies per-kernel events (PDL off).
 * timeline_layers: measured moespac_layer_timing per (step, layer) (ns;
 * wall = previous layer's end -> this layer's end). timeline_steps:
 * [n][6] = total, draft, prologue (H2D + K1 + K2), sum of layer walls,
 * epilogue (D2H), step index — total == draft + prologue + walls + epilogue.
 * Each getter returns the record count (out may be NULL). */
moespac_status moespac_ctx_set_timeline(moespac_ctx* c, int enabled);
int64_t moespac_ctx_timeline_events(const moespac_ctx* c, int64_t* out, int64_t cap);
int64_t moespac_ctx_timeline_layers(const moespac_ctx* c, moespac_layer_timing* out, int64_t cap);
int64_t moespac_ctx_timeline_steps(const moespac_ctx* c, int64_t* out, int64_t cap);
/* Launch-latency path (on by default): a step with no expert loads, no host
 * cold path, no draft phase and no per-kernel timing enqueues the same device
 * work every time, so the context captures it once into a CUDA graph
 * (programmatic dependencies included) and replays it with one launch. */
moespac_status moespac_ctx_set_graph(moespac_ctx* c, int enabled);
/* Programmatic dependent launch between layer kernels (on by default). */
moespac_status moespac_ctx_set_pdl(moespac_ctx* c, int enabled);
/* Profiling hook: device buffer of [n_layers][grid][32] uint64 that every
 * following step's tensor-core K3 launches fill with per-CTA %globaltimer
 * stamps and wait counters (layer l at offset l*grid*32), or NULL to stop. */
moespac_status moespac_ctx_set_k3_trace(moespac_ctx* c, void* dev_buf);
/* Cross-layer L2 prefetch budget per K3 CTA in bytes (tensor-core K3; 0 =
 * off): after its last weight copy, each CTA prefetches into L2 the part of
 * its next-layer work that follows the next CTA's own ring fill, so HBM
 * keeps working through the launch tail and the layer handoff. Default: 128
 * KiB for the grouped K3 (-2.5 to -3% step time measured at d = 2048; within
 * noise on the Mixtral shape, 5.13 vs 5.12 ms), 0 for the per-segment K3 (no
 * gain there). */
moespac_status moespac_ctx_set_l2_prefetch(moespac_ctx* c, int bytes);
/* The context's compute stream (cudaStream_t as void*) — every kernel of a
 * step runs on it, so events recorded there bracket whole steps. */
void* moespac_ctx_stream(const moespac_ctx* c);
/* Which K3 the context's plan picked (for reports and profiles):
 * CUDA-core GEMV, tcgen05 kernel with its per-segment accumulator (shared
 * memory / L2 partial block / TMEM), or the grouped tcgen05 kernel. */
#define MOESPAC_K3_CUDACORE 0
#define MOESPAC_K3_TC_SMEM 1
#define MOESPAC_K3_TC_L2 2
#define MOESPAC_K3_TC_TMEM 3
#define MOESPAC_K3_GROUPED 4
int moespac_ctx_k3_variant(const moespac_ctx* c);
/* The multi-GPU mode the context resolved to (MOESPAC_PAR_EXPERT or
 * MOESPAC_PAR_UNITS; MOESPAC_PAR_EXPERT for a single device). */
int moespac_ctx_parallel_mode(const moespac_ctx* c);

/* One verification step end to end with HOST buffers: H2D logits [L][T][N]
 * fp64 and h_in [T][d] bf16, run, D2H h_out [T][d] bf16 + the step's
 * scores/counters. `accepted` = tokens accepted this step (trace record). */
moespac_status moespac_step(moespac_ctx* c, const double* logits_host, const uint16_t* h_in_host, int accepted,
                            uint16_t* h_out_host, moespac_step_report* rep, moespac_layer_timing* layers);
/* Same with device-resident inputs/outputs. */
moespac_status moespac_step_device(moespac_ctx* c, const double* logits_dev, const uint16_t* h_in_dev,
                                   int accepted, uint16_t* h_out_dev, moespac_step_report* rep,
                                   moespac_layer_timing* layers);

/* Trace replay: one verification step with recorded routing instead of K1
 * over logits — ids [L][T][k] (any order within a token; sorted here),
 * gates [L][T][k] or NULL for uniform 1/k — host buffers as moespac_step. */
moespac_status moespac_step_ids(moespac_ctx* c, const int32_t* ids_host, const float* gates_host,
                                const uint16_t* h_in_host, int accepted, uint16_t* h_out_host,
                                moespac_step_report* rep, moespac_layer_timing* layers);

/* Model mode (the router GEMV s = W_g h of Eq. 3, feeding K1):
 * router weights of layer l, [n_experts][d_model] bf16 (host or device
 * pointer; d_model % 256 == 0), then steps whose routing is computed on the
 * device from each layer's input h_l — K0 GEMV (fp32, fixed summation order)
 * -> K1 -> K2 for that layer -> K3 — instead of from trace logits. Needs the
 * cold-expert host path off (moespac_ctx_set_cold_threads(ctx, 0)). */
moespac_status moespac_ctx_set_router(moespac_ctx* c, int layer, const uint16_t* w_router);
moespac_status moespac_step_model(moespac_ctx* c, const uint16_t* h_in_host, int accepted, uint16_t* h_out_host,
                                  moespac_step_report* rep, moespac_layer_timing* layers);
moespac_status moespac_step_model_device(moespac_ctx* c, const uint16_t* h_in_dev, int accepted, uint16_t* h_out_dev,
                                         moespac_step_report* rep, moespac_layer_timing* layers);

/* Device views of the last step (for parity checks; pointers owned by ctx). */
typedef struct moespac_ctx_views {
  const int32_t* ids_dev;       /* [L][T][k] */
  const float* gates_dev;       /* [L][T][k] */
  const int32_t* freqs_dev;     /* [L][N] */
  const int32_t* offsets_dev;   /* [L][N+1] */
  const int32_t* perm_dev;      /* [L][T*k] */
  const int32_t* counters_dev;  /* [L][8] */
  const int32_t* est_state_dev; /* [L][N][4] */
  const uint16_t* h_dev;        /* [L+1][T][d] bf16 layer inputs / final output */
  const float* y_dev;           /* [L][T][d] fp32 MoE outputs (multi-GPU: the ordered sum over ranks) */
  const uint16_t* pool_dev;     /* [L][slots][image] */
  const double* logits_dev;     /* [L][T][N] router logits (trace input, or K0's output in model mode) */
  int64_t slots_per_layer, image_elems;
  const uint16_t* shared_dev;   /* [L][n_shared_units][image] shared-expert units */
  const uint16_t* shared_gate_dev; /* [L][d] bf16 shared-expert gate vectors (SIGMOID), else NULL */
} moespac_ctx_views;
moespac_status moespac_ctx_get_views(const moespac_ctx* c, moespac_ctx_views* out);
/* Decision tables the last executed step ran with (the context's scheduler
 * already holds the next step's decisions, made while that step's layers
 * ran). Same layouts as moespac_sched_tables. */
moespac_status moespac_ctx_step_tables(const moespac_ctx* c, int32_t* taus, uint32_t* resident_bits,
                                       uint32_t* loaded_bits, int32_t* slot_table);
/* Host scheduler of the context (read-only use of the moespac_sched_* getters). */
const moespac_sched* moespac_ctx_sched(const moespac_ctx* c);

#ifdef __cplusplus
}
#endif

#endif /* MOESPAC_MOESPAC_H */
