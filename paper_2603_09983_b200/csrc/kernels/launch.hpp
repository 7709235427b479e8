// Kernel argument blocks and host-side launcher declarations.
#pragma once
#include <cstddef>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

namespace moespac {
namespace dev {

struct K2Args {
  const int32_t* ids;            // [L][T][k]
  int L, T, k, N;
  const uint32_t* resident_bits;  // [L][W] after this step's loads
  const uint32_t* loaded_bits;    // [L][W] loaded this step (may be null)
  const int32_t* taus;            // [L]
  int32_t* est_state;             // [L][N][4] score, up, down, last_freq (in/out)
  int utility_cap, adaptive;
  double forgetting;
  int shard_rank, shard_world;
  int32_t* freqs;      // [L][N]
  int32_t* offsets;    // [L][N+1]
  int32_t* perm;       // [L][T*k]
  int32_t* hit_list;   // [L][N] local-shard resident activated experts, ascending
  int32_t* hit_ord;    // [L][N] ordinal in hit_list or -1
  int32_t* counters;   // [L][8] distinct, hits, hit_tok, miss_tok, agree, fn, fp, n_local_hits
  int32_t* scores_out; // [L][N] post-update scores (next step's snapshot)
  float* gates;        // [L][T][k] (route_layer_kernel only: K1 gates of the layer)
};

struct FfnArgs {
  const uint16_t* h;        // [T][d] bf16 layer input
  int T, d, ffn, k, N;
  const int32_t* perm;      // [T*k]
  const int32_t* offsets;   // [N+1]
  const float* gates;       // [T][k]
  const int32_t* hit_list;  // [N]
  const int32_t* counters;  // [8], counters[7] = number of local hits
  const int32_t* slot_of;   // [N] slot of each expert in `pool` (-1 if absent)
  const uint16_t* pool;     // tiled expert images, stride expert_elems
  const uint16_t* shared_w; // tiled shared-expert units, stride expert_elems
  int n_shared;
  const uint16_t* shared_gate_w;  // [d] bf16: shared units weighted by sigmoid(w . h_t) (null: weight 1)
  long long expert_elems;   // 3*ffn*d
  float* partial;           // [(grid + N + n_shared)][T][d]
  int n_stages;             // CUDA-core kernel: ring stages
  int ring_bytes;           // tensor-core kernel: byte-ring size
  int global_acc;           // 1: accumulate down-proj partials in `partial` (large T*d)
  int acc_mode;             // tensor-core kernel: 0 shared-memory, 1 global (L2), 2 TMEM accumulator,
                            // 3 grouped (whole-CTA TMEM accumulator, expert_ffn_grouped.cu)
  const uint16_t* hT;       // tcgen05 variant: h^T UMMA image [d/64][16 tok][64] (build_hT)
  unsigned long long* dbg;  // optional per-CTA profiling record [grid][32]
  int l2_policy;            // weight stream L2 policy: 0 evict_first, 1 evict_normal
  // Next layer (tensor-core kernel): once a CTA has issued its last weight
  // copy it prefetches into L2 pf_bytes of what the same CTA index will
  // stream in the next layer — skipping the first ring_bytes, which that CTA
  // loads into its ring itself on entry — so HBM keeps working through this
  // launch's tail and the layer-to-layer handoff. nx_counters == null: off.
  const int32_t* nx_counters;
  const int32_t* nx_hit_list;
  const int32_t* nx_slot_of;
  const uint16_t* nx_pool;
  const uint16_t* nx_shared_w;
  int pf_bytes;
  // unit-split multi-GPU mode: this launch's CTAs are [cta_base, cta_base +
  // grid) of a virtual grid of cta_total CTAs over the layer's work units
  // (cta_total 0: the launch grid itself)
  int cta_base, cta_total;
  // grouped K3: units per group (8: one M = 128 gate|up tile per group
  // round; 0 / 16: up to two tiles, one round for CTAs with <= 16 units)
  int group_units;
  // grouped K3: a last remainder of <= tail_absorb units joins the group
  // before it as a second M-tile instead of running a round of its own
  int tail_absorb;
  int tg_n8;  // grouped K3 N = 8 mode (ffn_tg_n8(d, T), set by the launcher)
  // grouped K3: drain D2 only after the whole last DN pass (profiling A/B;
  // 0 = drain each M-tile chunk as soon as its entry completes)
  int drain_late;
  int drain_sc;  // grouped K3: M-tiles per drain chunk (0 = 4; halved until two fit the h^T slices)
};

struct CombineArgs {
  const uint16_t* h_in;     // [T][d] bf16 (residual; may be null)
  const float* y_extra;     // [T][d] fp32 added before rounding (cold path / remote); may be null
  int T, d, ffn, k;
  const int32_t* ids;       // [T][k]
  const int32_t* hit_ord;   // [N]
  const int32_t* counters;  // counters[7] = local hits
  int n_shared;
  int grid;                 // K3 grid size
  int per_cta;              // 1: one partial block per K3 CTA (grouped K3), else per (CTA, entry) pair
  int unit_rows;            // ffn rows per K3 work unit: 8 (tensor-core K3s) or 16 (CUDA-core K3)
  int cta_base, grid_local; // unit-split mode: the K3 launch was CTAs [cta_base, cta_base + grid_local) of `grid`
  const float* partial;
  float* y_out;             // [T][d] fp32 (may be null)
  uint16_t* h_out;          // [T][d] bf16 (may be null)
  uint16_t* hT_out;         // optional h^T UMMA image of h_out (next layer's tensor-core K3 operand)
  uint16_t* h_host;         // optional second copy of h_out in mapped host memory (cold path input)
  unsigned long long* dbg;  // optional per-CTA profiling record (K3 trace rows, slots 26-29), or null
};

}  // namespace dev

cudaError_t launch_router_topk(const double* logits, int rows, int N, int k, int gate_mode, int32_t* ids,
                               float* gates, cudaStream_t stream);
cudaError_t launch_hist_scan_observe(const dev::K2Args& a, cudaStream_t stream);
cudaError_t launch_estimator_init(int32_t* st, int n, int up, int down, cudaStream_t stream);
// model mode: K0 router GEMV (d % 256 == 0, T <= 16) and one layer's K1 + K2
cudaError_t launch_router_gemv(const uint16_t* wg, const uint16_t* h, int T, int N, int d, double* logits,
                               cudaStream_t stream, bool pdl = false);
cudaError_t launch_route_layer(const double* logits_l, int k, int gate_mode, const dev::K2Args& a, int l,
                               cudaStream_t stream, bool pdl = false);
struct FfnPlan {
  int n_stages;     // CUDA-core: ring stages; tensor-core: ring KiB
  bool global_acc;
  size_t smem;
  int acc_mode = 0; // tensor-core: 0 shared-memory, 1 global (L2), 2 TMEM accumulator, 3 grouped
};
size_t ffn_smem_bytes(int T, int d, int n_stages, bool global_acc);
FfnPlan ffn_plan(int T, int d, size_t smem_limit);
cudaError_t launch_expert_ffn(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl = false);
size_t ffn_tc_smem_bytes(int T, int d, int ring_bytes, int acc_mode);
FfnPlan ffn_tc_plan(int T, int d, size_t smem_limit, int accum = 0);
cudaError_t launch_expert_ffn_tc(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl = false);
// grouped K3 N = 8 mode: needed for d > 2048 (D2 in TMEM); at d <= 2048
// only with MOESPAC_TG_N8=1 (measured neutral there: Qwen1.5 1.036 vs 1.039
// ms per step, tiny within noise — the freed 32 KiB of h^T do not pay)
inline bool ffn_tg_n8_small() {
  static const bool on = [] {
    const char* e = std::getenv("MOESPAC_TG_N8");
    return e && e[0] == '1';
  }();
  return on;
}
inline bool ffn_tg_n8(int d, int T) { return d > 2048 || (T <= 8 && ffn_tg_n8_small()); }
size_t ffn_tg_smem_bytes(int T, int d, int ring_bytes);
int ffn_tg_ring_bytes(int T, int d, size_t smem_limit);
bool ffn_tg_grid_ok(int n_entries, int d_ffn, int grid);
cudaError_t launch_expert_ffn_tg(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl = false);
cudaError_t launch_build_hT(const uint16_t* h, int T, int d, uint16_t* out, cudaStream_t stream, bool pdl = false);
cudaError_t launch_pack_expert_tc(const uint16_t* wg, const uint16_t* wu, const uint16_t* wd, int d, int ffn,
                                  uint16_t* out, cudaStream_t stream);
cudaError_t launch_combine(const dev::CombineArgs& a, cudaStream_t stream, bool pdl = false);
cudaError_t launch_residual(const uint16_t* h_in, const float* y, uint16_t* h_out, uint16_t* hT_out, int d, int n,
                            cudaStream_t stream, bool pdl = false);
cudaError_t launch_sum_slots(const float* slots, int world, size_t stride, float* out, size_t n, cudaStream_t stream);
// expert-parallel combine: ordered sum of the all-gathered rank partials + residual + h^T (n = T*d, even)
cudaError_t launch_gather_sum_residual(const float* parts, int world, size_t stride, const uint16_t* h_in, float* y_out,
                                       uint16_t* h_out, uint16_t* hT_out, int d, int n, cudaStream_t stream);
cudaError_t launch_pack_expert(const uint16_t* wg, const uint16_t* wu, const uint16_t* wd, int d, int ffn,
                               uint16_t* out, cudaStream_t stream);
cudaError_t launch_unpack_expert(const uint16_t* image, int d, int ffn, uint16_t* wg, uint16_t* wu, uint16_t* wd,
                                 cudaStream_t stream);
cudaError_t launch_unpack_expert_tc(const uint16_t* image, int d, int ffn, uint16_t* wg, uint16_t* wu, uint16_t* wd,
                                    cudaStream_t stream);
cudaError_t launch_fill_synthetic(uint16_t* out, long long n, uint64_t seed, float stdv, cudaStream_t stream);
cudaError_t launch_draft_window(long long ns, cudaStream_t stream);
// draft model (draft.cu): one weight-streaming GEMV pass per draft token
bool draft_d_ok(int D);  // D % 256 == 0, D / 256 in {1, 2, 4, 6, 8, 10, 12, 16}
cudaError_t launch_draft_gemv(const uint16_t* W, long long R, int D, const float* y_prev, const uint16_t* x0,
                              float scale, float* y, int grid, cudaStream_t stream, bool pdl = false);

constexpr int kFfnMaxTokens = 16;
constexpr int kFfnChunkRows = 16;

// K3 variants: the tensor-core kernel (tcgen05/TMEM, image layout v2:
// d % 128 == 0, ffn % 64 == 0) and the CUDA-core GEMV (layout v1:
// d % 512 == 0, ffn % 16 == 0). 0 picks tcgen05 when the shape allows.
enum FfnKernel { kFfnAuto = 0, kFfnCudaCore = 1, kFfnTensorCore = 2 };
inline int ffn_resolve(int kernel, int d, int ffn) {
  if (kernel == kFfnAuto) return (d % 128 == 0 && ffn % 64 == 0) ? kFfnTensorCore : kFfnCudaCore;
  return kernel;
}
inline bool ffn_shape_ok(int kernel, int d, int ffn) {
  return kernel == kFfnTensorCore ? (d % 128 == 0 && ffn % 64 == 0 && d >= 128)
                                  : (d % 512 == 0 && ffn % 16 == 0 && ffn > 0);
}

}  // namespace moespac
