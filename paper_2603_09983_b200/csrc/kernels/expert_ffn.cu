// K3 — grouped SwiGLU expert FFN over the HBM-resident (hit) experts of one
// layer, plus the deterministic combine.
//
// Replaces the modeled FFN charge of run_utility_step
// (/root/reference/proj/core/src/sim_core.cpp:253-254) with the real
// computation of Eq. 3 and App. D:
//     y_t = sum_{i in TopK(t)} g_{t,i} * W_down^i (silu(W_gate^i h_t) * (W_up^i h_t)).
//
// Shape of the work: at verification batches (T <= 16 tokens, T_e <= T tokens
// per expert) every expert is a weight-streaming GEMV — arithmetic intensity
// ~T_e FLOP/B against a ridge of ~250 — so the kernel is built to stream each
// resident expert's 3*d*ffn bf16 weights from HBM exactly once:
//
//  * Tiled expert image. Each expert is stored in HBM as ffn/16 "chunks" of
//    3*16*d contiguous bf16: d/256 gate|up tiles ([32 rows][256 cols]: rows
//    0-15 gate, 16-31 up) then d/512 down tiles ([8][1024] or [16][512] of
//    W_down^T). Every tile is 16 KiB, so one TMA bulk copy per tile.
//  * Persistent CTAs, one per SM. The layer's chunk list (hit experts in
//    ascending id, then shared-expert units) is split into equal contiguous
//    ranges — byte-balanced because every chunk has the same size.
//  * Warp-specialised: warp 8 is the TMA producer (cp.async.bulk into a
//    6-deep 16 KiB ring, mbarrier complete_tx, L2 evict_first), warps 0-7
//    consume. Tokens' hidden states sit in shared memory for the whole launch.
//  * Gate/up: warp w owns ffn rows {w, w+8} of the chunk (gate and up), lane
//    owns 8 columns per tile, fp32 accumulation; butterfly reduction, then
//    a = silu(g)*u*gate_t into shared memory.
//  * Down: each thread owns 4 output columns of a tile and accumulates the
//    chunk's 16 ffn rows into a per-expert fp32 accumulator in shared
//    memory; when the CTA leaves an expert it writes one partial block
//    P[cta + expert_ordinal][t][d] (index unique along the staircase).
//  * Combine: y_t = sum over the token's experts (ascending id) and over the
//    CTAs that covered them (ascending), fixed order => deterministic; fused
//    with the residual add + bf16 round, or fp32 partial out for the
//    multi-GPU all-gather + ordered sum.
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"

namespace moespac {
namespace dev {

constexpr int FFN_CONSUMER_WARPS = 8;
constexpr int FFN_CONSUMERS = FFN_CONSUMER_WARPS * 32;
constexpr int FFN_THREADS = FFN_CONSUMERS + 32;
constexpr int TILE_BYTES = 16384;
constexpr int TILE_ELEMS = TILE_BYTES / 2;
constexpr int FC = 16;    // ffn rows per chunk
constexpr int MAX_T = 16;


// NT bucket used by dispatch_chunk (padding rows need ysum storage).
__host__ __device__ __forceinline__ int token_bucket(int t) { return t <= 9 ? t : (t <= 12 ? 12 : 16); }

struct Geo {
  int d, cpe, gu_tiles, dn_tiles, DW, DR, nsub, rows_per_tile_group, tp;
  long long chunk_elems;
};

__device__ __forceinline__ Geo make_geo(int d, int ffn, int T) {
  Geo g;
  g.tp = token_bucket(T);
  g.d = d;
  g.cpe = ffn / FC;
  g.gu_tiles = d / 256;
  g.dn_tiles = d / 512;
  g.DW = d < 1024 ? d : 1024;
  g.DR = TILE_ELEMS / g.DW;          // 8 or 16
  g.nsub = FFN_CONSUMERS / (g.DW / 4);  // 1 or 2
  g.rows_per_tile_group = FC / g.DR;    // down tiles per column tile: 2 or 1
  g.chunk_elems = 3LL * FC * d;
  return g;
}

__device__ __forceinline__ long long owner_of(long long q, long long n, int G) {
  return ((q + 1) * G - 1) / n;
}

__device__ __forceinline__ float silu(float x) { return x / (1.f + __expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

__device__ __forceinline__ float dot8(const uint4& w, const float (&x)[8]) {
  float s = bf_lo(w.x) * x[0];
  s = fmaf(bf_hi(w.x), x[1], s);
  s = fmaf(bf_lo(w.y), x[2], s);
  s = fmaf(bf_hi(w.y), x[3], s);
  s = fmaf(bf_lo(w.z), x[4], s);
  s = fmaf(bf_hi(w.z), x[5], s);
  s = fmaf(bf_lo(w.w), x[6], s);
  s = fmaf(bf_hi(w.w), x[7], s);
  return s;
}

struct Smem {
  uint8_t* ring;
  uint64_t* full;
  uint64_t* empty;
  uint16_t* h;     // [T][d]
  float* ysum;     // [nsub][TP][d], TP = token_bucket(T); unused in global mode
  float* yglob;    // global-accumulation mode: this CTA's partial block for the current entry
  float* a;        // [MAX_T][FC]
  int* tok;        // [MAX_T]
  float* gate;     // [MAX_T]
  int* ntok;       // [1]
};

struct Pipe {
  int stage;
  uint32_t ph;
  __device__ __forceinline__ void advance(int n) {
    if (++stage == n) {
      stage = 0;
      ph ^= 1u;
    }
  }
};

// One chunk (16 ffn rows of one expert) for NT tokens.
template <int NT>
__device__ __forceinline__ void chunk_compute(const Geo& g, const Smem& s, Pipe& p, int n_stages, int warp, int lane,
                                              int tid) {
  // ---------------- gate / up ----------------
  float acc[4][NT];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[i][t] = 0.f;
  const uint4* h4 = reinterpret_cast<const uint4*>(s.h);
  const int hrow4 = g.d / 8;
  int tokoff[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) tokoff[t] = s.tok[t] * hrow4;
  for (int ct = 0; ct < g.gu_tiles; ++ct) {
    mbar_wait(&s.full[p.stage], p.ph);
    const uint4* tile = reinterpret_cast<const uint4*>(s.ring + static_cast<size_t>(p.stage) * TILE_BYTES);
    const uint4 wg0 = tile[warp * 32 + lane];
    const uint4 wg1 = tile[(warp + 8) * 32 + lane];
    const uint4 wu0 = tile[(warp + 16) * 32 + lane];
    const uint4 wu1 = tile[(warp + 24) * 32 + lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.empty[p.stage]);
    p.advance(n_stages);
    const int col4 = ct * 32 + lane;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const uint4 hv = h4[tokoff[t] + col4];
      float x[8] = {bf_lo(hv.x), bf_hi(hv.x), bf_lo(hv.y), bf_hi(hv.y),
                    bf_lo(hv.z), bf_hi(hv.z), bf_lo(hv.w), bf_hi(hv.w)};
      acc[0][t] += dot8(wg0, x);
      acc[1][t] += dot8(wg1, x);
      acc[2][t] += dot8(wu0, x);
      acc[3][t] += dot8(wu1, x);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[i][t] = warp_sum(acc[i][t]);
  // all consumers finished reading s.a from the previous chunk's down phase
  named_bar_sync(1, FFN_CONSUMERS);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    if (lane == t) {
      const float gt = s.gate[t];
      s.a[t * FC + warp] = silu(acc[0][t]) * acc[2][t] * gt;
      s.a[t * FC + warp + 8] = silu(acc[1][t]) * acc[3][t] * gt;
    }
  }
  named_bar_sync(1, FFN_CONSUMERS);

  // ---------------- down ----------------
  const int cg = tid % (g.DW / 4);
  const int rsub = tid / (g.DW / 4);
  float* yrow[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t)
    yrow[t] = s.yglob ? s.yglob + static_cast<size_t>(s.tok[t]) * g.d
                      : s.ysum + (static_cast<size_t>(rsub) * g.tp + t) * g.d;
  for (int ct2 = 0; ct2 < g.d / g.DW; ++ct2) {
    float acc2[NT][4];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[t][j] = 0.f;
    for (int fg = 0; fg < g.rows_per_tile_group; ++fg) {
      mbar_wait(&s.full[p.stage], p.ph);
      const uint2* tile = reinterpret_cast<const uint2*>(s.ring + static_cast<size_t>(p.stage) * TILE_BYTES);
      uint2 w[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) w[r] = tile[(rsub + r * g.nsub) * (g.DW / 4) + cg];
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.empty[p.stage]);
      p.advance(n_stages);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int f = fg * g.DR + rsub + r * g.nsub;
        const float w0 = bf_lo(w[r].x), w1 = bf_hi(w[r].x), w2 = bf_lo(w[r].y), w3 = bf_hi(w[r].y);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float av = s.a[t * FC + f];
          acc2[t][0] = fmaf(w0, av, acc2[t][0]);
          acc2[t][1] = fmaf(w1, av, acc2[t][1]);
          acc2[t][2] = fmaf(w2, av, acc2[t][2]);
          acc2[t][3] = fmaf(w3, av, acc2[t][3]);
        }
      }
    }
    const int col = ct2 * g.DW + cg * 4;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      float4* dst = reinterpret_cast<float4*>(yrow[t] + col);
      float4 v = *dst;
      v.x += acc2[t][0];
      v.y += acc2[t][1];
      v.z += acc2[t][2];
      v.w += acc2[t][3];
      *dst = v;
    }
  }
}

__device__ __forceinline__ void dispatch_chunk(int nt, const Geo& g, const Smem& s, Pipe& p, int ns, int warp,
                                               int lane, int tid) {
  switch (nt) {
    case 1: chunk_compute<1>(g, s, p, ns, warp, lane, tid); break;
    case 2: chunk_compute<2>(g, s, p, ns, warp, lane, tid); break;
    case 3: chunk_compute<3>(g, s, p, ns, warp, lane, tid); break;
    case 4: chunk_compute<4>(g, s, p, ns, warp, lane, tid); break;
    case 5: chunk_compute<5>(g, s, p, ns, warp, lane, tid); break;
    case 6: chunk_compute<6>(g, s, p, ns, warp, lane, tid); break;
    case 7: chunk_compute<7>(g, s, p, ns, warp, lane, tid); break;
    case 8: chunk_compute<8>(g, s, p, ns, warp, lane, tid); break;
    case 9: chunk_compute<9>(g, s, p, ns, warp, lane, tid); break;
    case 10: case 11: case 12: chunk_compute<12>(g, s, p, ns, warp, lane, tid); break;
    default: chunk_compute<16>(g, s, p, ns, warp, lane, tid); break;
  }
}

__device__ __forceinline__ const uint16_t* entry_weights(const FfnArgs& a, int o, int n_hits) {
  if (o < n_hits) {
    const int e = a.hit_list[o];
    return a.pool + static_cast<long long>(a.slot_of[e]) * a.expert_elems;
  }
  return a.shared_w + static_cast<long long>(o - n_hits) * a.expert_elems;
}

__global__ void __launch_bounds__(FFN_THREADS, 1) expert_ffn_kernel(FfnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const Geo g = make_geo(a.d, a.ffn, a.T);
  const int ns = a.n_stages;
  const bool global_acc = a.global_acc != 0;
  Smem s;
  s.yglob = nullptr;
  uint8_t* ptr = smem_raw;
  s.ring = ptr;
  ptr += static_cast<size_t>(ns) * TILE_BYTES;
  s.full = reinterpret_cast<uint64_t*>(ptr);
  ptr += 8 * ns;
  s.empty = reinterpret_cast<uint64_t*>(ptr);
  ptr += 8 * ns;
  s.ysum = reinterpret_cast<float*>(ptr);
  if (!global_acc) ptr += static_cast<size_t>(g.nsub) * g.tp * a.d * 4;
  s.a = reinterpret_cast<float*>(ptr);
  ptr += MAX_T * FC * 4;
  s.gate = reinterpret_cast<float*>(ptr);
  ptr += MAX_T * 4;
  s.tok = reinterpret_cast<int*>(ptr);
  ptr += MAX_T * 4;
  s.ntok = reinterpret_cast<int*>(ptr);
  ptr += 16;
  s.h = reinterpret_cast<uint16_t*>(ptr);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_hits = a.counters[7];
  const long long n_entries = n_hits + a.n_shared;
  const long long n = n_entries * g.cpe;
  const int G = gridDim.x, b = blockIdx.x;
  const long long q0 = n > 0 ? (b * n) / G : 0;
  const long long q1 = n > 0 ? ((b + 1) * n) / G : 0;
  if (q0 >= q1) return;

  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], FFN_CONSUMER_WARPS);
    }
    fence_mbar_init();
    pdl_trigger();
  }
  pdl_wait();  // h and the partial workspace come from the previous kernel
  // hidden states of all T tokens -> smem (bf16), ysum <- 0
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.h);
    uint4* dst = reinterpret_cast<uint4*>(s.h);
    const int n4 = a.T * a.d / 8;
    for (int i = tid; i < n4; i += FFN_THREADS) dst[i] = src[i];
    float4* ys = reinterpret_cast<float4*>(s.ysum);
    const int ny = global_acc ? 0 : g.nsub * g.tp * a.d / 4;
    for (int i = tid; i < ny; i += FFN_THREADS) ys[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();

  if (warp == FFN_CONSUMER_WARPS) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      Pipe p{0, 0u};
      const int tiles = g.gu_tiles + g.dn_tiles;
      for (long long q = q0; q < q1; ++q) {
        const int o = static_cast<int>(q / g.cpe), c = static_cast<int>(q % g.cpe);
        const uint16_t* base = entry_weights(a, o, n_hits) + c * g.chunk_elems;
        for (int t = 0; t < tiles; ++t) {
          mbar_wait(&s.empty[p.stage], p.ph ^ 1u);
          mbar_arrive_expect_tx(&s.full[p.stage], TILE_BYTES);
          bulk_g2s(s.ring + static_cast<size_t>(p.stage) * TILE_BYTES, base + static_cast<long long>(t) * TILE_ELEMS,
                   TILE_BYTES, &s.full[p.stage], pol);
          p.advance(ns);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  Pipe p{0, 0u};
  int cur = -1;
  auto flush = [&](int o) {
    named_bar_sync(1, FFN_CONSUMERS);
    if (global_acc) return;  // already accumulated in place
    const int nt = *s.ntok;
    float* P = a.partial + static_cast<long long>(b + o) * a.T * a.d;
    for (int t = 0; t < nt; ++t) {
      const int tg = s.tok[t];
      for (int c = tid * 4; c < a.d; c += FFN_CONSUMERS * 4) {
        float4 v = *reinterpret_cast<float4*>(s.ysum + static_cast<size_t>(t) * a.d + c);
        *reinterpret_cast<float4*>(s.ysum + static_cast<size_t>(t) * a.d + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 1; r < g.nsub; ++r) {
          float* y2 = s.ysum + (static_cast<size_t>(r) * g.tp + t) * a.d + c;
          const float4 u = *reinterpret_cast<float4*>(y2);
          *reinterpret_cast<float4*>(y2) = make_float4(0.f, 0.f, 0.f, 0.f);
          v.x += u.x;
          v.y += u.y;
          v.z += u.z;
          v.w += u.w;
        }
        *reinterpret_cast<float4*>(P + static_cast<long long>(tg) * a.d + c) = v;
      }
    }
  };
  for (long long q = q0; q < q1; ++q) {
    const int o = static_cast<int>(q / g.cpe);
    if (o != cur) {
      if (cur >= 0) flush(cur);
      named_bar_sync(1, FFN_CONSUMERS);
      if (tid < MAX_T) {
        int nt, tok = 0;
        float gt = 0.f;
        if (o < n_hits) {
          const int e = a.hit_list[o];
          const int p0 = a.offsets[e];
          nt = a.offsets[e + 1] - p0;
          if (tid < nt) {
            const int idx = a.perm[p0 + tid];
            tok = idx / a.k;
            gt = a.gates[idx];
          }
        } else {
          nt = a.T;
          if (tid < nt) {
            tok = tid;
            gt = 1.f;
          }
        }
        if (tid >= nt) {  // padding lanes of a bucketed NT: valid row, zero gate
          tok = 0;
          gt = 0.f;
        }
        s.tok[tid] = tok;
        s.gate[tid] = gt;
        if (tid == 0) *s.ntok = nt;
      }
      named_bar_sync(1, FFN_CONSUMERS);
      if (global_acc) {
        // zero this entry's rows of the CTA-exclusive partial block
        s.yglob = a.partial + static_cast<long long>(b + o) * a.T * a.d;
        const int nt = *s.ntok;
        for (int t = 0; t < nt; ++t)
          for (int c = tid * 4; c < a.d; c += FFN_CONSUMERS * 4)
            *reinterpret_cast<float4*>(s.yglob + static_cast<size_t>(s.tok[t]) * a.d + c) =
                make_float4(0.f, 0.f, 0.f, 0.f);
        named_bar_sync(1, FFN_CONSUMERS);
      }
      cur = o;
    }
    dispatch_chunk(*s.ntok, g, s, p, ns, warp, lane, tid);
  }
  flush(cur);
}

// ---------------------------------------------------------------- combine

// One CTA per (token, 128-column slice); the partial rows of the token (its
// experts in ascending id, each over the CTAs that covered it in ascending
// order) are dealt round-robin to the warps, then the warp sums are added in
// warp order — a fixed summation tree, so the result is deterministic.
// 4 warps next to the per-segment K3 (its 200-register CTA leaves room for
// no more), 8 next to the grouped K3 (82 registers): twice the partial rows
// in flight per output column. The row lists and the cross-warp sums share
// one shared-memory block (lists are dead once the loads are issued).
constexpr int COMBINE_BATCH = 16;  // partial rows in flight per warp
constexpr int COMBINE_ROWS = 192;  // row list capacity over all warps (else streamed)

template <int WARPS>
struct CombineSmem {
  union {
    float4 red[WARPS][32];
    int rows[WARPS][COMBINE_ROWS / WARPS];
  };
};

template <int WARPS>
__device__ __forceinline__ void combine_store(const CombineArgs& a, float4 acc, const float4 (*red)[32], int t,
                                              int c, uint2 hv, float4 ex);

// (<= 112 registers: see expert_ffn_tc_kernel)
template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32) combine_kernel(CombineArgs a) {
  constexpr int COMBINE_WARPS = WARPS, COMBINE_LIST = COMBINE_ROWS / WARPS;
  __shared__ CombineSmem<WARPS> sm;
  auto& rows = sm.rows;
  if (threadIdx.x == 0) pdl_trigger();
  unsigned long long* dbg = a.dbg ? a.dbg + (blockIdx.y * gridDim.x + blockIdx.x) * 32 : nullptr;
  auto stamp = [&](int slot) {
    if (dbg && threadIdx.x == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt)::"memory");
      dbg[slot] = tt;
    }
  };
  stamp(26);
  if (dbg && threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    dbg[29] = smid;
  }
  const int t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.y * 128 + lane * 4;
  const int qpe = a.ffn / (a.per_cta || a.unit_rows == 8 ? 8 : FC);  // work units per entry (tensor-core K3s: 8 rows)
  // The routing (K2 outputs: counters, ids, hit order) was final several
  // kernels ago, so the row list is built before waiting for the K3 launch
  // whose partials it sums: only the partial loads sit on the critical path.
  const int n_hits = a.counters[7];
  const int n = (n_hits + a.n_shared) * qpe;
  const int G = a.grid;
  // unit-split mode: only this GPU's K3 CTAs [cb0, cb1) of the virtual grid
  const int cb0 = a.cta_base, cb1 = a.grid_local > 0 ? a.cta_base + a.grid_local : G;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  // warp 0's residual and host-cold inputs, loaded right after the wait
  // (alongside the partial rows, not after the sums)
  uint2 hv = make_uint2(0u, 0u);
  float4 ex = make_float4(0.f, 0.f, 0.f, 0.f);
  auto preload = [&]() {
    if (warp != 0 || c >= a.d) return;
    const size_t off = static_cast<size_t>(t) * a.d + c;
    if (a.h_out && a.h_in) hv = __ldcg(reinterpret_cast<const uint2*>(a.h_in + off));
    if (a.y_extra) ex = __ldcg(reinterpret_cast<const float4*>(a.y_extra + off));
  };
  if (n > 0 && c < a.d) {
    // 1) this warp's partial rows, in the fixed order (experts ascending,
    //    covering CTAs ascending, dealt round-robin to the warps)
    //    Grouped K3 (per_cta): one block per CTA holding the CTA's sum over
    //    all its experts; a CTA covering two of the token's experts is listed
    //    once (entries ascend, so their CTA ranges do too).
    int idx = 0, my_n = 0, last_b = -1;
    auto list_entry = [&](int o) {
      const int lo = ((o * qpe + 1) * G - 1) / n;
      const int hi = (((o + 1) * qpe) * G - 1) / n;
      for (int b = lo; b <= hi; ++b) {
        // with fewer work units than CTAs some CTAs own nothing
        if ((b * n) / G == ((b + 1) * n) / G || b < cb0 || b >= cb1) continue;
        if (a.per_cta) {
          if (b <= last_b) continue;
          last_b = b;
        }
        if ((idx++ % COMBINE_WARPS) != warp) continue;
        if (lane == 0 && my_n < COMBINE_LIST) rows[warp][my_n] = a.per_cta ? b - cb0 : b - cb0 + o;
        ++my_n;
      }
    };
    for (int j = 0; j < a.k; ++j) {
      const int o = a.hit_ord[a.ids[t * a.k + j]];
      if (o >= 0) list_entry(o);
    }
    for (int sidx = 0; sidx < a.n_shared; ++sidx) list_entry(n_hits + sidx);
    __syncwarp();
    pdl_wait();  // partials of the K3 launch just before
    preload();
    stamp(27);
    auto row_ptr = [&](int r) {
      return reinterpret_cast<const float4*>(a.partial + (static_cast<long long>(r) * a.T + t) * a.d + c);
    };
    if (my_n <= COMBINE_LIST) {
      // 2) COMBINE_BATCH independent loads in flight, summed in list order
      for (int base = 0; base < my_n; base += COMBINE_BATCH) {
        float4 v[COMBINE_BATCH];
#pragma unroll
        for (int u = 0; u < COMBINE_BATCH; ++u)
          if (base + u < my_n) v[u] = __ldcg(row_ptr(rows[warp][base + u]));
#pragma unroll
        for (int u = 0; u < COMBINE_BATCH; ++u)
          if (base + u < my_n) {
            acc.x += v[u].x;
            acc.y += v[u].y;
            acc.z += v[u].z;
            acc.w += v[u].w;
          }
      }
    } else {  // long lists: same order, one row at a time
      idx = 0;
      last_b = -1;
      auto add_entry = [&](int o) {
        const int lo = ((o * qpe + 1) * G - 1) / n;
        const int hi = (((o + 1) * qpe) * G - 1) / n;
        for (int b = lo; b <= hi; ++b) {
          if ((b * n) / G == ((b + 1) * n) / G || b < cb0 || b >= cb1) continue;
          if (a.per_cta) {
            if (b <= last_b) continue;
            last_b = b;
          }
          if ((idx++ % COMBINE_WARPS) != warp) continue;
          const float4 v = __ldcg(row_ptr(a.per_cta ? b - cb0 : b - cb0 + o));
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
      };
      for (int j = 0; j < a.k; ++j) {
        const int o = a.hit_ord[a.ids[t * a.k + j]];
        if (o >= 0) add_entry(o);
      }
      for (int sidx = 0; sidx < a.n_shared; ++sidx) add_entry(n_hits + sidx);
    }
  }
  if (!(n > 0 && c < a.d)) {  // (no partials to read; still order after K3)
    pdl_wait();
    preload();
  }
  __syncthreads();  // every warp is past its row list (the sums reuse that memory)
  sm.red[warp][lane] = acc;
  __syncthreads();
  stamp(28);
  if (warp != 0 || c >= a.d) return;
  combine_store<WARPS>(a, acc, sm.red, t, c, hv, ex);
  if (lane == 0) stamp(30);
}

// warp 0 of a combine CTA: cross-warp sum, y / residual / bf16 / h^T stores
template <int WARPS>
__device__ __forceinline__ void combine_store(const CombineArgs& a, float4 acc, const float4 (*red)[32], int t,
                                              int c, uint2 hv, float4 ex) {
  const int lane = threadIdx.x & 31;
  for (int w = 1; w < WARPS; ++w) {
    const float4 v = red[w][lane];
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  const size_t off = static_cast<size_t>(t) * a.d + c;
  if (a.y_extra) {  // cold experts computed on the host (added after the fixed-order device sum)
    acc.x += ex.x;
    acc.y += ex.y;
    acc.z += ex.z;
    acc.w += ex.w;
  }
  if (a.y_out) *reinterpret_cast<float4*>(a.y_out + off) = acc;
  if (a.h_out) {
    float4 r = acc;
    if (a.h_in) {
      r.x += bf_lo(hv.x);
      r.y += bf_hi(hv.x);
      r.z += bf_lo(hv.y);
      r.w += bf_hi(hv.y);
    }
    uint2 o;
    o.x = static_cast<uint32_t>(f32_to_bf16_rn(r.x)) | (static_cast<uint32_t>(f32_to_bf16_rn(r.y)) << 16);
    o.y = static_cast<uint32_t>(f32_to_bf16_rn(r.z)) | (static_cast<uint32_t>(f32_to_bf16_rn(r.w)) << 16);
    *reinterpret_cast<uint2*>(a.h_out + off) = o;
    if (a.h_host) *reinterpret_cast<uint2*>(a.h_host + off) = o;
    if (a.hT_out) {
      // the next layer's h^T UMMA image (tensor-core K3): 4 consecutive k of
      // token t share one 8-byte run (k % 8 in {0..3} or {4..7})
      const int kt = c >> 6, j = (c >> 3) & 7, e = c & 7;
      const int w = kt * 1024 + (t >> 3) * 512 + j * 64 + (t & 7) * 8 + e;
      *reinterpret_cast<uint2*>(a.hT_out + w) = o;
    }
  }
}

// h_out = bf16(h_in + y) — residual after an expert-parallel all-reduce.
__global__ void residual_kernel(const uint16_t* h_in, const float* y, uint16_t* h_out, uint16_t* hT_out, int d,
                                int n) {
  pdl_wait();
  pdl_trigger();
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i >= n) return;
  const uint32_t hv = *reinterpret_cast<const uint32_t*>(h_in + i);
  const float a = bf_lo(hv) + y[i], b = bf_hi(hv) + y[i + 1];
  const uint32_t o = static_cast<uint32_t>(f32_to_bf16_rn(a)) | (static_cast<uint32_t>(f32_to_bf16_rn(b)) << 16);
  *reinterpret_cast<uint32_t*>(h_out + i) = o;
  if (hT_out) {
    const int t = i / d, c = i % d;
    const int kt = c >> 6, j = (c >> 3) & 7, e = c & 7;
    *reinterpret_cast<uint32_t*>(hT_out + kt * 1024 + (t >> 3) * 512 + j * 64 + (t & 7) * 8 + e) = o;
  }
}

// ---------------------------------------------------------------- packing
// Standard layouts (wg, wu: [ffn][d], wd: [d][ffn]) <-> tiled expert image:
// kUnpack = false packs (image element idx gathers its source element), true
// unpacks (the same index map, scattered back).
template <bool kUnpack>
__global__ void pack_expert_kernel(uint16_t* __restrict__ wg, uint16_t* __restrict__ wu, uint16_t* __restrict__ wd,
                                   int d, int ffn, uint16_t* __restrict__ out) {
  const long long total = 3LL * ffn * d;
  const long long chunk = 3LL * FC * d;
  const long long gu = 2LL * FC * d;
  const int DW = d < 1024 ? d : 1024;
  const int DR = TILE_ELEMS / DW;
  const int nrg = FC / DR;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = idx / chunk;
    const long long r = idx % chunk;
    uint16_t* src;
    if (r < gu) {
      const long long tile = r / TILE_ELEMS, within = r % TILE_ELEMS;
      const int row = static_cast<int>(within / 256), col = static_cast<int>(within % 256);
      const long long src_col = tile * 256 + col;
      src = row < FC ? &wg[(c * FC + row) * d + src_col] : &wu[(c * FC + row - FC) * d + src_col];
    } else {
      const long long r2 = r - gu;
      const long long tile = r2 / TILE_ELEMS, within = r2 % TILE_ELEMS;
      const int row = static_cast<int>(within / DW), col = static_cast<int>(within % DW);
      const long long ct2 = tile / nrg, fg = tile % nrg;
      const long long f = c * FC + fg * DR + row;
      src = &wd[(ct2 * DW + col) * ffn + f];
    }
    if (kUnpack)
      *src = out[idx];
    else
      out[idx] = *src;
  }
}

// Deterministic synthetic bf16 weights ~ N(0, std^2) (Irwin-Hall of 4
// hashed uniforms), written straight into tiled images.
__device__ __forceinline__ uint32_t mix32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return static_cast<uint32_t>(x);
}

__global__ void fill_synthetic_kernel(uint16_t* out, long long n, uint64_t seed, float stdv) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint64_t base = seed * 0x9E3779B97F4A7C15ULL + static_cast<uint64_t>(i) * 4;
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += static_cast<float>(mix32(base + j)) * 2.3283064365386963e-10f;
    out[i] = f32_to_bf16_rn((s - 2.f) * 1.7320508f * stdv);
  }
}

}  // namespace dev

// ---------------------------------------------------------------- launchers
size_t ffn_smem_bytes(int T, int d, int n_stages, bool global_acc) {
  const int DW = d < 1024 ? d : 1024;
  const int nsub = dev::FFN_CONSUMERS / (DW / 4);
  return static_cast<size_t>(n_stages) * dev::TILE_BYTES + 16ull * n_stages +
         (global_acc ? 0 : static_cast<size_t>(nsub) * dev::token_bucket(T) * d * 4) + dev::MAX_T * dev::FC * 4 + dev::MAX_T * 8 + 16 +
         static_cast<size_t>(T) * d * 2;
}

FfnPlan ffn_plan(int T, int d, size_t smem_limit) {
  // Prefer the shared-memory accumulator with a >= 4-deep ring; otherwise
  // accumulate in the CTA's exclusive partial block (L2-resident) and keep
  // the deep ring. Global mode needs one accumulator copy (d >= 1024).
  for (int ns = 6; ns >= 4; --ns)
    if (ffn_smem_bytes(T, d, ns, false) <= smem_limit) return {ns, false, ffn_smem_bytes(T, d, ns, false)};
  if (d >= 1024)
    for (int ns = 6; ns >= 2; --ns)
      if (ffn_smem_bytes(T, d, ns, true) <= smem_limit) return {ns, true, ffn_smem_bytes(T, d, ns, true)};
  for (int ns = 3; ns >= 2; --ns)
    if (ffn_smem_bytes(T, d, ns, false) <= smem_limit) return {ns, false, ffn_smem_bytes(T, d, ns, false)};
  return {0, false, 0};
}

cudaError_t launch_expert_ffn(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl) {
  if (const cudaError_t e = smem_optin_once<dev::expert_ffn_kernel>(232448); e != cudaSuccess) return e;
  return launch_pdl(dev::expert_ffn_kernel, dim3(grid), dim3(dev::FFN_THREADS), smem, stream, pdl, a);
}

cudaError_t launch_combine(const dev::CombineArgs& a, cudaStream_t stream, bool pdl) {
  if (a.per_cta)
    return launch_pdl(dev::combine_kernel<8>, dim3(a.T, (a.d + 127) / 128), dim3(8 * 32), 0, stream, pdl, a);
  return launch_pdl(dev::combine_kernel<4>, dim3(a.T, (a.d + 127) / 128), dim3(4 * 32), 0, stream, pdl,
                    a);
}

cudaError_t launch_residual(const uint16_t* h_in, const float* y, uint16_t* h_out, uint16_t* hT_out, int d, int n,
                            cudaStream_t stream, bool pdl) {
  return launch_pdl(dev::residual_kernel, dim3((n / 2 + 255) / 256), dim3(256), 0, stream, pdl, h_in, y, h_out,
                    hT_out, d, n);
}

namespace dev {
// out[i] = sum over q = 0..world-1 (in that order) of slots[q * stride + i]
__global__ void sum_slots_kernel(const float* __restrict__ slots, int world, size_t stride, float* __restrict__ out,
                                 size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = slots[i];
  for (int q = 1; q < world; ++q) s += slots[q * stride + i];
  out[i] = s;
}
}  // namespace dev

cudaError_t launch_sum_slots(const float* slots, int world, size_t stride, float* out, size_t n, cudaStream_t stream) {
  dev::sum_slots_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(slots, world, stride, out, n);
  return cudaGetLastError();
}

namespace dev {
// Expert-parallel combine after the all-gather of the ranks' fp32 partial
// outputs ([world][stride], rank order): y = sum over ranks 0..world-1 in
// that order (the same bits on every rank, for NCCL and the in-process
// loopback alike), h_out = bf16(h_in + y), and the next layer's h^T image.
__global__ void gather_sum_residual_kernel(const float* __restrict__ parts, int world, size_t stride,
                                           const uint16_t* __restrict__ h_in, float* __restrict__ y_out,
                                           uint16_t* __restrict__ h_out, uint16_t* __restrict__ hT_out, int d, int n) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i >= n) return;
  float2 y = *reinterpret_cast<const float2*>(parts + i);
  for (int q = 1; q < world; ++q) {
    const float2 p = *reinterpret_cast<const float2*>(parts + q * stride + i);
    y.x += p.x;
    y.y += p.y;
  }
  *reinterpret_cast<float2*>(y_out + i) = y;
  const uint32_t hv = *reinterpret_cast<const uint32_t*>(h_in + i);
  const uint32_t o = static_cast<uint32_t>(f32_to_bf16_rn(bf_lo(hv) + y.x)) |
                     (static_cast<uint32_t>(f32_to_bf16_rn(bf_hi(hv) + y.y)) << 16);
  *reinterpret_cast<uint32_t*>(h_out + i) = o;
  if (hT_out) {
    const int t = i / d, c = i % d;
    const int kt = c >> 6, j = (c >> 3) & 7, e = c & 7;
    *reinterpret_cast<uint32_t*>(hT_out + kt * 1024 + (t >> 3) * 512 + j * 64 + (t & 7) * 8 + e) = o;
  }
}
}  // namespace dev

cudaError_t launch_gather_sum_residual(const float* parts, int world, size_t stride, const uint16_t* h_in, float* y_out,
                                       uint16_t* h_out, uint16_t* hT_out, int d, int n, cudaStream_t stream) {
  dev::gather_sum_residual_kernel<<<static_cast<unsigned>((n / 2 + 255) / 256), 256, 0, stream>>>(
      parts, world, stride, h_in, y_out, h_out, hT_out, d, n);
  return cudaGetLastError();
}

namespace dev {
// Emulated draft window (the reference's modeled γ·t_draft, sim_core.cpp:
// 167-172): one warp holds the compute stream for `ns` nanoseconds of
// %globaltimer while the copy engine works through the step's expert loads.
__global__ void draft_window_kernel(long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0)::"memory");
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  } while (static_cast<long long>(t - t0) < ns);
}
}  // namespace dev

cudaError_t launch_draft_window(long long ns, cudaStream_t stream) {
  if (ns <= 0) return cudaSuccess;
  dev::draft_window_kernel<<<1, 32, 0, stream>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_pack_expert(const uint16_t* wg, const uint16_t* wu, const uint16_t* wd, int d, int ffn,
                               uint16_t* out, cudaStream_t stream) {
  dev::pack_expert_kernel<false><<<1184, 256, 0, stream>>>(const_cast<uint16_t*>(wg), const_cast<uint16_t*>(wu),
                                                           const_cast<uint16_t*>(wd), d, ffn, out);
  return cudaGetLastError();
}

cudaError_t launch_unpack_expert(const uint16_t* image, int d, int ffn, uint16_t* wg, uint16_t* wu, uint16_t* wd,
                                 cudaStream_t stream) {
  dev::pack_expert_kernel<true><<<1184, 256, 0, stream>>>(wg, wu, wd, d, ffn, const_cast<uint16_t*>(image));
  return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(uint16_t* out, long long n, uint64_t seed, float stdv, cudaStream_t stream) {
  dev::fill_synthetic_kernel<<<1184, 256, 0, stream>>>(out, n, seed, stdv);
  return cudaGetLastError();
}

}  // namespace moespac
