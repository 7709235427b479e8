// Device engine: one verification step of the MoE-SpAc hot path on one B200.
// See include/moespac/moespac.h (moespac_ctx_*) for the contract and
// DESIGN.md for the HBM layout.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <array>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "../../../include/moespac/moespac.h"
#include "step_scheduler.hpp"

namespace moespac {

struct NcclApi;  // dlopen'ed libnccl (no link-time dependency)

// In-process stand-in for the per-layer NCCL all-gather: `world` contexts on
// one device, each driven by its own host thread, exchange their partial
// outputs through device slots and CUDA events; every rank then sums the
// slots in rank order with the same kernel the NCCL path uses. Test harness for the expert-parallel device path where only
// one GPU is available (NCCL refuses two ranks on one device).
class LoopbackGroup {
 public:
  LoopbackGroup(int device, int world, size_t max_elems);
  ~LoopbackGroup();
  // buf [n] -> slots [world][stride()] (rank order); release() after reading them
  const float* all_gather(int rank, const float* buf, size_t n, cudaStream_t stream);
  void release(int rank, cudaStream_t stream);
  size_t stride() const { return max_; }
  int world() const { return world_; }

 private:
  void barrier();
  int device_, world_;
  size_t max_;
  float* slots_ = nullptr;  // [world][max]
  std::vector<cudaEvent_t> put_, done_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  unsigned long long gen_ = 0;
};
class ColdExecutor;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

moespac_status nccl_unique_id(void* out128);

class Engine {
 public:
  Engine(int device, const moespac_model_desc& m, const moespac_sched_config& cfg, int rank, int world);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  uint16_t* host_arena(int64_t n_images);
  void fill_synthetic(uint64_t seed, float stdv);
  void set_shared(int layer, const uint16_t* units_dev);
  void set_shared_gate(int layer, const uint16_t* w_sg);
  // estimator checkpoint in the reference's text format (one
  // LayerEstimator::dump per layer, utility_estimator.cpp:81-107)
  void estimator_dump(const char* path);
  void estimator_load(const char* path);
  void finalize();
  void set_nccl(const void* uid, int nranks, int rank);
  void set_timing(bool on) { timing_ = on; }
  void set_pdl(bool on) {
    pdl_ = on;
    drop_graph();
  }
  void set_k3_trace(unsigned long long* buf) {
    k3_trace_ = buf;
    drop_graph();
  }
  void set_draft_window(bool on) { draft_window_ = on; }
  // real draft phase: gamma weight-streaming GEMV passes over n_params bf16
  // draft weights (rows of d_draft) before each verification step
  void set_draft_model(int64_t n_params, int d_draft);
  // measured SimEvent-shaped timeline (implies per-kernel events, PDL off)
  void set_timeline(bool on) { timeline_ = on; }
  int64_t timeline_events(int64_t* out, int64_t cap) const;
  int64_t timeline_layers(moespac_layer_timing* out, int64_t cap) const;
  int64_t timeline_steps(int64_t* out, int64_t cap) const;
  void timeline_clear() {
    tl_events_.clear();
    tl_layers_.clear();
    tl_steps_.clear();
    tl_clock_ns_ = 0;
  }
  void set_loopback(LoopbackGroup* g) {
    if (!g || g->world() != world_) throw std::invalid_argument("moespac_ctx_set_loopback: group size != shard world");
    loop_ = g;
  }
  void set_l2_prefetch(int bytes) {
    l2_prefetch_ = bytes;
    drop_graph();
  }
  // launch-latency path: replay a captured CUDA graph of steps without loads
  // or host work (on by default; MOESPAC_GRAPH=0)
  void set_graph(bool on) {
    use_graph_ = on;
    drop_graph();
  }
  // host threads for cold (non-resident) experts: -1 auto, 0 = off (misses
  // are then counted but not computed); takes effect at finalize()
  void set_cold_threads(int n) { cold_threads_ = n; }
  // cold experts staged through HBM (moespac_ctx_set_cold_staging); before finalize()
  void set_cold_staging(int slots, double fraction) {
    if (finalized_) throw std::logic_error("moespac_ctx_set_cold_staging: context already finalized");
    if (slots < 0 || slots % 2 || !(fraction >= 0.0 && fraction <= 1.0))
      throw std::invalid_argument("moespac_ctx_set_cold_staging: slots must be even and >= 0, fraction in [0, 1]");
    stage_slots_ = slots;
    stage_frac_ = fraction;
  }
  void step(const double* logits, bool logits_host, const uint16_t* h_in, bool h_in_host, int accepted,
            uint16_t* h_out, bool h_out_host, moespac_step_report* rep, moespac_layer_timing* layers);
  // Trace replay (#moetrace v1, trace_io.hpp): routing ids [L][T][k] (and
  // gates, or uniform 1/k when null) from the host instead of K1 over logits.
  void step_ids(const int32_t* ids, const float* gates, const uint16_t* h_in, bool h_in_host, int accepted,
                uint16_t* h_out, bool h_out_host, moespac_step_report* rep, moespac_layer_timing* layers);
  // Model mode (router GEMV): routing from W_g h_l on
  // the device, layer by layer, instead of trace logits.
  void set_router(int layer, const uint16_t* w_dev);
  void step_model(const uint16_t* h_in, bool h_in_host, int accepted, uint16_t* h_out, bool h_out_host,
                  moespac_step_report* rep, moespac_layer_timing* layers);
  void views(moespac_ctx_views* v) const;
  // decision tables the last executed step ran with
  void step_tables(int32_t* taus, uint32_t* rb, uint32_t* lb, int32_t* slots) const;
  int ffn_kernel() const { return kernel_; }
  int ffn_acc_mode() const { return acc_mode_; }
  bool unit_split() const { return split_; }
  const StepScheduler& sched() const { return *sched_; }
  void* stream() const { return compute_; }

 private:
  void check(cudaError_t e, const char* what) const;
  int64_t image_of(int layer, int expert) const {
    return (static_cast<int64_t>(layer) * m_.n_experts + expert) % n_images_;
  }
  uint16_t* slot_ptr(int layer, int slot) const {
    return pool_ + (static_cast<int64_t>(layer) * slots_ + slot) * image_elems_;
  }

  int kernel_ = 0;
  int device_ = 0, rank_ = 0, world_ = 1, sms_ = 148, T_ = 0, W_ = 1, stages_ = 6;
  // expert shard of this rank: (rank, world) in the expert-partitioned mode,
  // (0, 1) in the unit-split mode (every expert on every rank)
  int shard_rank_ = 0, shard_world_ = 1;
  bool split_ = false;
  bool ar_ = false;  // AR policy: T = 1 token per step
  size_t ffn_smem_ = 0;
  moespac_model_desc m_{};
  std::unique_ptr<StepScheduler> sched_;
  int64_t image_elems_ = 0, slots_ = 0, n_images_ = 0;
  bool synthetic_ = false, finalized_ = false, timing_ = false, global_acc_ = false;
  uint64_t synth_seed_ = 0;
  float synth_std_ = 0.02f;

  // HBM
  uint16_t* pool_ = nullptr;    // [L][slots][image]
  uint16_t* shared_ = nullptr;  // [L][n_shared][image]
  uint16_t* sg_w_ = nullptr;    // [L][d] bf16 shared-expert gate vectors (MOESPAC_SHARED_GATE_SIGMOID)
  double* logits_d_ = nullptr;
  int32_t *ids_d_ = nullptr, *freqs_d_ = nullptr, *offsets_d_ = nullptr, *perm_d_ = nullptr;
  int32_t *hit_list_d_ = nullptr, *hit_ord_d_ = nullptr, *est_d_ = nullptr;
  float *gates_d_ = nullptr, *y_d_ = nullptr, *work_d_ = nullptr;
  float* gather_d_ = nullptr;   // [world][T][d] all-gathered rank partials (NCCL)
  uint16_t* h_d_ = nullptr;     // [L+1][T][d]
  uint16_t* hT_d_ = nullptr;    // h^T UMMA image of the current layer input (tensor-core K3)
  uint8_t* tables_d_ = nullptr; // resident bits | loaded bits | taus | slot table
  int32_t* out_d_ = nullptr;    // scores_out [L][N] | counters [L][8]
  size_t tables_bytes_ = 0, out_bytes_ = 0, work_bytes_ = 0;
  // host
  uint16_t* arena_h_ = nullptr;
  uint8_t* tables_h_ = nullptr;
  int32_t* out_h_ = nullptr;
  std::vector<int32_t> scores_;  // [L][N] snapshot for the next decide()

  cudaStream_t compute_ = nullptr, copy_ = nullptr;
  std::vector<cudaEvent_t> load_done_, ffn_beg_, ffn_end_;
  cudaEvent_t ev_[7] = {};  // step begin, draft end, K1 end, K2 end, layers end, step end, draft begin
  cudaEvent_t copy_ev_[2] = {};  // timing: first / last expert load on the copy stream
  cudaEvent_t k2_done_ = nullptr;
  bool decided_ = false;  // next step's decisions already made
  bool pdl_ = true;                         // programmatic dependent launch between layer kernels
  unsigned long long* k3_trace_ = nullptr;  // profiling: [L][grid][32]
  int l2_prefetch_ = -1;  // per-CTA next-layer L2 prefetch (bytes); -1: per-kernel default
  int cold_threads_ = -1;
  bool cold_trace_ = false;  // MOESPAC_COLD_TRACE: per-step host timing of the cold path on stderr
  bool step_trace_ = false;  // MOESPAC_STEP_TRACE: per-step host timing of the device-only path on stderr
  int ffn_accum_ = 0;
  int group_units_ = 0;  // grouped K3 units per group (MOESPAC_GROUP_UNITS profiling knob; 0 = 8)
  int tail_absorb_ = -1;  // grouped K3: remainder units joining the last group (MOESPAC_TAIL_ABSORB; -1 = per shape)
  int drain_late_ = 0;    // grouped K3: D2 drained after the whole last DN pass (MOESPAC_DRAIN_LATE, profiling)
  int drain_sc_ = 0;      // grouped K3: M-tiles per drain chunk (MOESPAC_DRAIN_SC, profiling; 0 = kernel default)
  const int32_t* replay_ids_ = nullptr;  // set for the duration of step_ids()
  const float* replay_gates_ = nullptr;
  uint16_t* wg_d_ = nullptr;      // [L][N][d] bf16 router weights (model mode)
  std::vector<bool> router_set_;
  bool model_mode_ = false;       // set for the duration of step_model()
  bool draft_window_ = false;  // emulated γ·t_draft spin on the compute stream before K1
  // draft model (draft.cu): weights [R][D] bf16, y ping-pong [2][R] fp32, x0 [D]
  uint16_t* draft_w_ = nullptr;
  float* draft_y_ = nullptr;
  uint16_t* draft_x0_ = nullptr;
  int64_t draft_R_ = 0;
  int draft_D_ = 0;
  float draft_scale_ = 1.f;
  // measured timeline
  bool timeline_ = false;
  std::vector<cudaEvent_t> wait_beg_, layer_end_, ld_beg_, ld_end_;
  // cross-step loads: next step's loads of layer l issued during this step
  // after its last reader of the layer's slots (xload_ev_[l])
  std::vector<cudaEvent_t> xload_ev_;
  std::vector<uint8_t> preloaded_;  // [L] loads of the coming step already on the copy stream
  bool cross_step_ = true;          // MOESPAC_CROSS_STEP=0 disables
  // captured step graph (launch-latency path)
  void drop_graph();
  bool drafted_any() const { return T_ > 1 && (draft_R_ > 0 || draft_window_); }
  bool use_graph_ = true;
  cudaGraphExec_t graph_exec_ = nullptr;
  int graph_warm_ = 0;
  std::vector<std::array<int64_t, 6>> tl_events_;
  std::vector<ThresholdDecision> sched_decisions_;  // decisions of the step being executed
  std::vector<moespac_layer_timing> tl_layers_;
  std::vector<std::array<int64_t, 6>> tl_steps_;  // total, draft, prologue, sum of layer walls, epilogue, step
  int64_t tl_clock_ns_ = 0;
  int acc_mode_ = 0;

  std::unique_ptr<ColdExecutor> cold_;
  // cold-expert staging ring: stage_slots_ images after the pool's L x slots_
  // (two halves, layers alternating), filled on stage_ behind the event of
  // the combine two layers back (its last reader)
  int stage_slots_ = 0;
  double stage_frac_ = 0.0;
  int64_t pool_images_ = 0;       // images allocated in pool_ (L x slots_ + staging)
  cudaStream_t stage_ = nullptr;
  std::vector<cudaEvent_t> stage_ev_, stage_done_;  // [L] combine(l) done / layer l's staged copies landed
  int32_t* xt_d_ = nullptr;       // [L][3N + 8] routing tables incl. staged experts: hit_list | hit_ord | slot_of | counters
  int32_t* xt_h_ = nullptr;       // pinned host copy
  float* ycold_h_ = nullptr;   // pinned, mapped [L][T][d] host-computed cold-expert outputs
  float* ycold_d_ = nullptr;   // device alias of ycold_h_ (read by the combine)
  uint16_t* hcold_h_ = nullptr;  // pinned, mapped [L+1][T][d] layer inputs for the cold path
  uint16_t* hcold_d_ = nullptr;  // device alias of hcold_h_ (written by the combine)
  uint8_t* route_h_ = nullptr;   // pinned ids [L][T][k] | gates [L][T][k]
  std::vector<cudaEvent_t> h_ready_;
  std::unique_ptr<NcclApi> nccl_;
  LoopbackGroup* loop_ = nullptr;  // test harness instead of NCCL (not owned)
  void* comm_ = nullptr;
};

}  // namespace moespac
