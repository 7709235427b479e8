// Draft phase: a real weight-streaming draft model
// in place of the reference's modeled γ·t_draft window
// (/root/reference/proj/core/src/sim_core.cpp:167-172).
//
// MoE-SpAc drafts with a small dense model on the same GPU (PAPER.md:378-383:
// Qwen3-4B-FP8 next to Qwen3-30B-A3B). At batch 1 a draft token is one pass
// over all the draft weights, i.e. a chain of weight-streaming GEMVs — the
// work that contends with the verification step's expert loads for HBM and
// with its kernels for SMs. The draft model here is that byte stream: R rows
// of D bf16 weights (R·D = the draft's parameter count) and one GEMV per
// draft token, y_i = W x_i, whose input is the previous token's output
// (x_{i+1} = bf16(scale · y_i[0:D])), so the γ passes are a true dependency
// chain as in autoregressive drafting.
//
// Kernel: persistent grid (a multiple of the SM count), one warp per row at a
// time, two rows in flight per warp, each lane issuing D/256 16-byte
// non-allocating loads per row (evict-first: the 4 GB stream must not flush
// the verification step's L2 working set), fp32 FMA, xor-butterfly
// reduction. HBM-bound: algorithmic bytes per pass = R·D·2 (+ R·4 of y).
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"

namespace moespac {
namespace dev {

constexpr int DRAFT_THREADS = 512;
constexpr int DRAFT_MAX_D = 4096;

__device__ __forceinline__ uint4 ld_stream(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// x (bf16 [D]) from the previous pass: scale · y_prev[0:D] (pass 0: x0).
template <int V>  // V = D / 256 uint4 per lane per row
__global__ void __launch_bounds__(DRAFT_THREADS) draft_gemv_kernel(const uint16_t* __restrict__ W, long long R, int D,
                                                                  const float* __restrict__ y_prev,
                                                                  const uint16_t* __restrict__ x0, float scale,
                                                                  float* __restrict__ y) {
  __shared__ __align__(16) uint16_t xs[DRAFT_MAX_D];
  pdl_wait();
  for (int k = threadIdx.x; k < D; k += blockDim.x)
    xs[k] = y_prev ? f32_to_bf16_cvt(scale * y_prev[k]) : x0[k];
  __syncthreads();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const long long warps = static_cast<long long>(gridDim.x) * (DRAFT_THREADS / 32);
  const long long w0 = static_cast<long long>(blockIdx.x) * (DRAFT_THREADS / 32) + (threadIdx.x >> 5);
  const uint64_t pol = l2_evict_first_policy();
  // this lane's slice of x: k = 256 v + 8 lane + e
  float xv[V][8];
#pragma unroll
  for (int v = 0; v < V; ++v) bf16x8_to_f32(*reinterpret_cast<const uint4*>(xs + 256 * v + 8 * lane), xv[v]);
  for (long long r = w0; r < R; r += 2 * warps) {
    const long long r1 = r + warps;
    const bool two = r1 < R;
    const uint4* p0 = reinterpret_cast<const uint4*>(W + r * D) + lane;
    const uint4* p1 = reinterpret_cast<const uint4*>(W + (two ? r1 : r) * D) + lane;
    uint4 a[V], b[V];
#pragma unroll
    for (int v = 0; v < V; ++v) a[v] = ld_stream(p0 + 32 * v, pol);
#pragma unroll
    for (int v = 0; v < V; ++v) b[v] = ld_stream(p1 + 32 * v, pol);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float wa[8], wb[8];
      bf16x8_to_f32(a[v], wa);
      bf16x8_to_f32(b[v], wb);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s0 = fmaf(wa[e], xv[v][e], s0);
        s1 = fmaf(wb[e], xv[v][e], s1);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    if (lane == 0) {
      y[r] = s0;
      if (two) y[r1] = s1;
    }
  }
}

}  // namespace dev

bool draft_d_ok(int D) {
  if (D < 256 || D % 256) return false;
  switch (D / 256) {
    case 1: case 2: case 4: case 6: case 8: case 10: case 12: case 16:
      return true;
    default:
      return false;
  }
}

cudaError_t launch_draft_gemv(const uint16_t* W, long long R, int D, const float* y_prev, const uint16_t* x0,
                              float scale, float* y, int grid, cudaStream_t stream, bool pdl) {
  if (!draft_d_ok(D) || R < 1) return cudaErrorInvalidValue;
  const dim3 g(grid), b(dev::DRAFT_THREADS);
  switch (D / 256) {
#define MOESPAC_DRAFT_CASE(v) \
  case v:                     \
    return launch_pdl(dev::draft_gemv_kernel<v>, g, b, 0, stream, pdl, W, R, D, y_prev, x0, scale, y);
    MOESPAC_DRAFT_CASE(1)
    MOESPAC_DRAFT_CASE(2)
    MOESPAC_DRAFT_CASE(4)
    MOESPAC_DRAFT_CASE(6)
    MOESPAC_DRAFT_CASE(8)
    MOESPAC_DRAFT_CASE(10)
    MOESPAC_DRAFT_CASE(12)
    MOESPAC_DRAFT_CASE(16)
#undef MOESPAC_DRAFT_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace moespac
