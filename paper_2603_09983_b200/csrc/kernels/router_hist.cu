// K1 — router top-k + gates, and K2 — fused histogram / scan / permutation /
// Speculative-Utility-Estimator update / realized split.
//
// K1 replaces the selection block of TraceGenerator::next_step
// (/root/reference/proj/core/src/trace_model.cpp:87-104): per token, the k
// largest logits by (value desc, id asc), ids emitted ascending. One warp
// per token; each lane keeps ceil(N/32) fp64 logits in registers; k rounds of
// a warp argmax on (value, -id) via __shfl_xor_sync; the selection mask is
// turned into ascending ids with ballots. Comparisons are plain IEEE double
// compares (so -0.0 == +0.0 ties resolve to the lower id, like the
// reference). Gates follow Eq. 3: softmax over the
// selected k (gate_mode 0) or over all N without renormalisation (gate_mode
// 1), in fp32 from fp64 differences.
//
// K2 replaces activation_frequencies (trace_model.cpp:122-130),
// LayerEstimator::observe_step + calibrate (utility_estimator.cpp:40-72),
// snapshot_scores (:74-79) and the realized split / accuracy / fault counters
// of run_utility_step (sim_core.cpp:233-283). One CTA per layer; the
// calibrate() arithmetic uses __dsub_rn/__dmul_rn/__dadd_rn in the
// reference's operation order, so the floor is bit-identical (no FMA).
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"

namespace moespac {
namespace dev {

// ------------------------------------------------------------------ K1
template <int VPL>
__global__ void __launch_bounds__(256) router_topk_kernel(const double* __restrict__ logits, int rows, int N,
                                                          int k, int gate_mode, int32_t* __restrict__ ids,
                                                          float* __restrict__ gates) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const double* v = logits + static_cast<size_t>(row) * N;
  double x[VPL];
  uint32_t taken = 0;  // bit i <-> expert lane + 32*i
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int e = lane + 32 * i;
    x[i] = e < N ? __ldg(v + e) : -__longlong_as_double(0x7ff0000000000000LL);  // -inf
  }
  double vmax_sel = 0.0;
  for (int r = 0; r < k; ++r) {
    // lane-local best among untaken: ascending e, strict > keeps lower id
    double bv = 0.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int e = lane + 32 * i;
      if (e < N && !((taken >> i) & 1u) && (bi == 0x7fffffff || x[i] > bv)) {
        bv = x[i];
        bi = e;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      const bool other_better = oi != 0x7fffffff && (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi));
      if (other_better) {
        bv = ov;
        bi = oi;
      }
    }
    if (r == 0) vmax_sel = bv;
    if ((bi & 31) == lane) taken |= 1u << (bi >> 5);
  }
  // ascending emission + gates
  float sum_all = 0.f;
  if (gate_mode == 1) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i)
      if (lane + 32 * i < N) s += expf(static_cast<float>(x[i] - vmax_sel));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    sum_all = s;
  }
  // selected exps (fp32) — first pass for the renormalised sum
  float sel_sum = 0.f;
#pragma unroll
  for (int i = 0; i < VPL; ++i)
    if ((taken >> i) & 1u) sel_sum += expf(static_cast<float>(x[i] - vmax_sel));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sel_sum += __shfl_xor_sync(0xffffffffu, sel_sum, off);
  const float denom = gate_mode == 1 ? sum_all : sel_sum;
  int base = 0;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const bool mine = (taken >> i) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (mine) {
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      ids[static_cast<size_t>(row) * k + pos] = lane + 32 * i;
      if (gates) gates[static_cast<size_t>(row) * k + pos] = expf(static_cast<float>(x[i] - vmax_sel)) / denom;
    }
    base += __popc(m);
  }
}

// ------------------------------------------------------------------ K2

// utility_estimator.cpp:40-43 — floor((1-l)*b + l*m), clamped >= 1, each
// operation a separately rounded IEEE double op.
__device__ __forceinline__ int calibrate_rn(int boundary, double lambda, int magnitude) {
  const double keep = __dsub_rn(1.0, lambda);
  const double next = __dadd_rn(__dmul_rn(keep, static_cast<double>(boundary)),
                                __dmul_rn(lambda, static_cast<double>(magnitude)));
  const int f = static_cast<int>(floor(next));
  return f > 1 ? f : 1;
}

constexpr int K2_THREADS = 256;
constexpr int K2_MAX_N = 4096;
constexpr int K2_MAX_TK = 2048;

__global__ void __launch_bounds__(K2_THREADS) hist_scan_observe_kernel(K2Args a) {
  __shared__ int32_t s_freq[K2_MAX_N];
  __shared__ int32_t s_ids[K2_MAX_TK];
  __shared__ int32_t s_scan[K2_THREADS];
  __shared__ int32_t s_cnt[8];
  const int l = blockIdx.x;
  const int N = a.N, TK = a.T * a.k, tid = threadIdx.x;
  const int W = (N + 31) / 32;
  const int32_t* ids = a.ids + static_cast<size_t>(l) * TK;
  for (int e = tid; e < N; e += K2_THREADS) s_freq[e] = 0;
  if (tid < 8) s_cnt[tid] = 0;
  __syncthreads();
  for (int i = tid; i < TK; i += K2_THREADS) {
    const int e = ids[i];
    s_ids[i] = e;
    atomicAdd(&s_freq[e], 1);
  }
  __syncthreads();

  // Exclusive scans over experts: offsets (freqs) and hit ordinals. Each
  // thread owns a contiguous run of experts.
  const int per = (N + K2_THREADS - 1) / K2_THREADS;
  const int e0 = tid * per, e1 = min(N, e0 + per);
  const uint32_t* rbits = a.resident_bits + static_cast<size_t>(l) * W;
  int my_f = 0, my_h = 0;
  for (int e = e0; e < e1; ++e) {
    my_f += s_freq[e];
    const bool hit = s_freq[e] > 0 && ((rbits[e >> 5] >> (e & 31)) & 1u) && (e % a.shard_world) == a.shard_rank;
    my_h += hit ? 1 : 0;
  }
  // pack two 16-bit-safe counts? keep two passes for clarity (N <= 4096)
  s_scan[tid] = my_f;
  __syncthreads();
  for (int off = 1; off < K2_THREADS; off <<= 1) {
    const int v = tid >= off ? s_scan[tid - off] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int run_f = s_scan[tid] - my_f;
  __syncthreads();
  s_scan[tid] = my_h;
  __syncthreads();
  for (int off = 1; off < K2_THREADS; off <<= 1) {
    const int v = tid >= off ? s_scan[tid - off] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int run_h = s_scan[tid] - my_h;
  if (tid == K2_THREADS - 1) s_cnt[7] = s_scan[tid];

  int32_t* offs = a.offsets + static_cast<size_t>(l) * (N + 1);
  int32_t* freqs = a.freqs + static_cast<size_t>(l) * N;
  int32_t* hl = a.hit_list + static_cast<size_t>(l) * N;
  int32_t* ho = a.hit_ord + static_cast<size_t>(l) * N;
  int32_t* st = a.est_state + static_cast<size_t>(l) * N * 4;
  int32_t* so = a.scores_out + static_cast<size_t>(l) * N;
  const uint32_t* lbits = a.loaded_bits ? a.loaded_bits + static_cast<size_t>(l) * W : nullptr;
  const int tau = a.taus[l];
  int c_dist = 0, c_hits = 0, c_hit_tok = 0, c_miss_tok = 0, c_agree = 0, c_fn = 0, c_fp = 0;
  for (int e = e0; e < e1; ++e) {
    const int f = s_freq[e];
    freqs[e] = f;
    offs[e] = run_f;
    run_f += f;
    const bool res = (rbits[e >> 5] >> (e & 31)) & 1u;
    const bool hit = f > 0 && res && (e % a.shard_world) == a.shard_rank;
    if (hit) {
      hl[run_h] = e;
      ho[e] = run_h++;
    } else {
      ho[e] = -1;
    }
    // realized split over the GLOBAL residency (sim_core.cpp:233-246)
    if (f > 0) {
      ++c_dist;
      if (res) {
        ++c_hits;
        c_hit_tok += f;
      } else {
        c_miss_tok += f;
      }
    }
    // estimator: snapshot score -> accuracy / FN (sim_core.cpp:276-280),
    // then observe_step (utility_estimator.cpp:47-72)
    int4 s = *reinterpret_cast<int4*>(st + 4 * e);  // score, up, down, last
    c_agree += ((s.x >= 1) == (f >= 1)) ? 1 : 0;
    c_fn += (f >= 1 && s.x < tau) ? 1 : 0;
    if (lbits && ((lbits[e >> 5] >> (e & 31)) & 1u) && f == 0) ++c_fp;
    const int delta = f - s.w;
    if (delta >= s.y) s.x = min(a.utility_cap, s.x + 1);
    else if (-delta >= s.z) s.x = max(0, s.x - 1);
    if (a.adaptive) {
      if (delta > 0) s.y = calibrate_rn(s.y, a.forgetting, delta);
      else if (delta < 0) s.z = calibrate_rn(s.z, a.forgetting, -delta);
    }
    s.w = f;
    *reinterpret_cast<int4*>(st + 4 * e) = s;
    so[e] = s.x;
  }
  if (tid == K2_THREADS - 1) offs[N] = run_f;
  // block-reduce counters (integer: order-independent)
  atomicAdd(&s_cnt[0], c_dist);
  atomicAdd(&s_cnt[1], c_hits);
  atomicAdd(&s_cnt[2], c_hit_tok);
  atomicAdd(&s_cnt[3], c_miss_tok);
  atomicAdd(&s_cnt[4], c_agree);
  atomicAdd(&s_cnt[5], c_fn);
  atomicAdd(&s_cnt[6], c_fp);
  __syncthreads();
  if (tid < 8) a.counters[static_cast<size_t>(l) * 8 + tid] = s_cnt[tid];

  // Stable permutation, sorted by (expert, token, slot): position of id i =
  // offsets[e] + #{i' < i : ids[i'] == e}. s_freq is reused as the offsets
  // table after the scan above.
  __syncthreads();
  for (int e = e0; e < e1; ++e) s_freq[e] = offs[e];
  __syncthreads();
  int32_t* perm = a.perm + static_cast<size_t>(l) * TK;
  for (int i = tid; i < TK; i += K2_THREADS) {
    const int e = s_ids[i];
    int r = 0;
    for (int j = 0; j < i; ++j) r += s_ids[j] == e ? 1 : 0;
    perm[s_freq[e] + r] = i;
  }
}

__global__ void estimator_init_kernel(int32_t* st, int n, int up, int down) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) *reinterpret_cast<int4*>(st + 4 * i) = make_int4(0, up, down, 0);
}

}  // namespace dev

// ------------------------------------------------------------------ launchers
cudaError_t launch_router_topk(const double* logits, int rows, int N, int k, int gate_mode, int32_t* ids,
                               float* gates, cudaStream_t stream) {
  if (rows <= 0) return cudaSuccess;
  const int vpl = (N + 31) / 32;
  const dim3 grid((rows + 7) / 8), block(256);
  if (vpl <= 1) dev::router_topk_kernel<1><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else if (vpl <= 2) dev::router_topk_kernel<2><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else if (vpl <= 4) dev::router_topk_kernel<4><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else if (vpl <= 8) dev::router_topk_kernel<8><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else if (vpl <= 16) dev::router_topk_kernel<16><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else if (vpl <= 32) dev::router_topk_kernel<32><<<grid, block, 0, stream>>>(logits, rows, N, k, gate_mode, ids, gates);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_hist_scan_observe(const dev::K2Args& a, cudaStream_t stream) {
  if (a.N > dev::K2_MAX_N || a.T * a.k > dev::K2_MAX_TK) return cudaErrorInvalidValue;
  dev::hist_scan_observe_kernel<<<a.L, dev::K2_THREADS, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_estimator_init(int32_t* st, int n, int up, int down, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  dev::estimator_init_kernel<<<(n + 255) / 256, 256, 0, stream>>>(st, n, up, down);
  return cudaGetLastError();
}

}  // namespace moespac
