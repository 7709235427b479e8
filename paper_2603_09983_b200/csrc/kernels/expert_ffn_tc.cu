// K3 (tensor-core variant) — grouped SwiGLU expert FFN on the 5th-gen tensor
// cores: TMA bulk copies -> shared-memory UMMA operands -> tcgen05.mma ->
// TMEM accumulators -> tcgen05.ld epilogue.
//
// Same contract and partial-block protocol as the CUDA-core kernel in
// expert_ffn.cu (the combine kernel is shared); what changes is where the
// multiply-adds run. At verification batches (T <= 16) the contraction is a
// GEMV, so the tensor cores are idle most of the time either way — the point
// of this variant is that the SMs no longer unpack bf16 and issue FFMA for
// every weight element, which is what bounded the CUDA-core kernel (ncu:
// issue-bound at ~58% of HBM). Here an SM issues ~10 instructions per 16 KiB
// of weights and the kernel is bounded by the TMA weight stream.
//
// Tiled expert image (v2), per chunk of 64 ffn rows (ffn % 64 == 0):
//   d/64 gate|up K-tiles, each [128 rows][64 k] bf16 in UMMA K-major
//     core-matrix order (8 rows x 16 B core matrices; row-group outer:
//     byte = g*1024 + j*128 + r*16 + e*2); rows are quarter-major and
//     octet-interleaved: rows 32q..32q+31 = gate f 16q+0..7, up f 16q+0..7,
//     gate f 16q+8..15, up f 16q+8..15, so a quarter is one 4 KiB run and an
//     8-row half of it (gate + up octet) one 2 KiB run;
//   d/128 down M-tiles, each [128 out rows][64 f] of W_down, core matrices
//     k-chunk outer (byte = j*2048 + g*128 + r*16 + e*2) so that a 16-row
//     quarter of the chunk (k-chunks 2q, 2q+1) is one contiguous 4 KiB run.
// Work unit = 16 ffn rows (a "quarter"), as in the CUDA-core kernel; a CTA
// covering part of a chunk loads only its quarters' rows (2 gate/up copies +
// 1 down copy per tile) and skips the down k-steps it does not own.
//
// Operands per MMA (cta_group::1, kind::f16, M=128, N=16, K=16):
//   gate/up: A = weight tile (smem), B = h^T for all T tokens (zero-padded
//            to 16; a 2 KiB slice per K-tile, streamed with the weights from
//            an L2-resident image built per layer), D1 = TMEM [128][16].
//   down:    A = W_down tile (smem), B = a^T split into bf16 hi + lo parts
//            (a = silu(g) * u * gate_t; two MMAs keep ~16 mantissa bits),
//            D2 = TMEM [128][16] per M-tile, 8 M-tiles per pass, 2 passes
//            in flight.
// Warp roles: 0 = TMA producer, 1 = MMA issuer (+ TMEM owner), 2-5 = epilogue
// (TMEM lane quarters 2,3,0,1).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"
#include "tcgen05.cuh"

namespace moespac {
namespace dev {
namespace tc {

constexpr int THREADS = 192;
constexpr int EPI_THREADS = 128;
constexpr int A_BYTES = 16384;
constexpr int B_BYTES = 2048;
constexpr int UBYTES = 2048;     // one 8-row unit (gate + up octet) of a 128-row gate|up tile, or 8 k of a down tile
constexpr int NSLOT = 32;        // ring entries in flight (mbarrier pairs)
constexpr int FCH = 64;  // ffn rows per chunk
constexpr int UROWS = 8;          // ffn rows per work unit
constexpr int TMEM_COLS = 512;
constexpr int D2_COL0 = 256;
constexpr int ACC_SMEM = 0, ACC_GLOBAL = 1, ACC_TMEM = 2, ACC_GROUP = 3;  // FfnArgs::acc_mode
constexpr int TMEM_ACC_MAX_D = (512 - D2_COL0) / 16 * 128;  // TMEM mode: D2 for all M-tiles fits
constexpr int PASS_TILES = 8;
constexpr int ENT_PRE = 8;  // entries whose routing is staged in the prologue
struct Ring {
  int stage = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void advance(int ns) {
    if (++stage == ns) {
      stage = 0;
      ph ^= 1u;
    }
  }
};

// Iterates the CTA's work as segments (entry, chunk, unit range); a unit
// is 8 ffn rows (image layout v3: one 2 KiB run per tile), 8 per chunk.
struct Seg {
  int o, c, qa, qb;  // units [qa, qb) of chunk c of entry o
};

struct SegIter {
  long long q, q1;
  int qpe;  // units per entry = ffn / 8
  __device__ __forceinline__ bool next(Seg& s) {
    if (q >= q1) return false;
    const int o = static_cast<int>(q / qpe);
    const int qi = static_cast<int>(q % qpe);
    const int c = qi / 8;
    const int qa = qi % 8;
    const long long chunk_end = static_cast<long long>(o) * qpe + (c + 1) * 8;
    const long long end = chunk_end < q1 ? chunk_end : q1;
    s = {o, c, qa, qa + static_cast<int>(end - q)};
    q = end;
    return true;
  }
};

// Ring entries. One entry carries m consecutive K-tiles (gate/up: A parts
// of the segment's quarters + the matching h^T slices) or m consecutive
// M-tiles (down) of one segment, so the per-entry bookkeeping of the
// producer and MMA warps (~500 cycles of dependent single-warp work) is
// amortised over >= 24 KiB whatever the segment's width: m grows as the
// segment narrows.
__device__ __forceinline__ int pow2_divisor(int x, int cap) {
  int m = 1;
  while (m < cap && x % (2 * m) == 0) m *= 2;
  return m;
}
__device__ __forceinline__ int tiles_per_entry(int nu, int cap) {
  const int t = nu >= 6 ? 2 : (nu >= 3 ? 4 : 8);
  return t < cap ? t : cap;
}
struct Geom {  // one entry: bytes, tiles, read window (bytes from the entry start)
  uint32_t size, win;
  int m;
};
// hb: h^T bytes per K-tile carried in the entry — 2 KiB (16 token rows), or
// 1 KiB when T <= 8: only the first 8-row token group is copied and the
// descriptor's second group (SBO = 1 KiB) reads whatever follows, which only
// feeds D1 columns of tokens >= T (the epilogue selects 0 for those).
__device__ __forceinline__ Geom gu_geom(int nu, int cap, uint32_t hb) {
  const int m = tiles_per_entry(nu, cap);
  const uint32_t a = static_cast<uint32_t>(nu) * 2048u;
  const uint32_t size = static_cast<uint32_t>(m) * (a + hb);
  // tile j's A descriptor reads the 16 KiB window at j*a - qa*2048; the last
  // h^T slice's second token group reads 1 KiB past the entry when hb = 1 KiB
  const uint32_t w = static_cast<uint32_t>(m - 1) * a + 16384u;
  const uint32_t ws = size + (hb < 2048u ? 1024u : 0u);
  return {size, ws > w ? ws : w, m};
}
__device__ __forceinline__ Geom dn_geom(int nu, int cap) {
  const int m = tiles_per_entry(nu, cap);
  // a down K-step reads two units: one unit past the segment at either end
  // (its a^T rows are 0)
  const uint32_t size = static_cast<uint32_t>(m) * static_cast<uint32_t>(nu) * 2048u;
  return {size, size + 2048u, m};
}
__device__ __forceinline__ uint32_t ring_place(uint32_t& head, const Geom& g, uint32_t rb) {
  uint32_t e = head;
  if (e + g.win > rb) e = 0;
  head = e + ((g.size + 1023u) & ~1023u);
  return e;
}

constexpr int DBG = 32;  // debug slots per CTA

__device__ __forceinline__ void stamp(const FfnArgs& a, int slot) {
  if (a.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    a.dbg[blockIdx.x * DBG + slot] = t;
  }
}

// mbarrier wait that, in profiling mode, accumulates the cycles spent
// blocked into debug slot `slot` (slots 8..15: per-role wait counters)
__device__ __forceinline__ void wait_acc(const FfnArgs& a, uint64_t* bar, uint32_t parity, long long& acc) {
  if (a.dbg) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}

__device__ __forceinline__ const uint16_t* entry_weights(const FfnArgs& a, int o, int n_hits) {
  if (o < n_hits) return a.pool + static_cast<long long>(a.slot_of[a.hit_list[o]]) * a.expert_elems;
  return a.shared_w + static_cast<long long>(o - n_hits) * a.expert_elems;
}

// <= 200 registers: with 2 of its warps on one SM sub-partition (16K registers)
// a 4-warp combine CTA (<= 112 regs) must still fit next to it, or PDL cannot
// overlap the combine with this kernel's tail (measured: +3 us per layer).
__global__ void __maxnreg__(200) expert_ffn_tc_kernel(FfnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int d = a.d, T = a.T;
  const int ktiles = d / 64, mtiles = d / 128;
  const int passes = (mtiles + PASS_TILES - 1) / PASS_TILES;
  const long long chunk_elems = 3LL * FCH * d;
  const int qpe = a.ffn / UROWS;

  // [a^T 16 KiB][ring][ysum][small]: the a^T buffers sit right before the
  // ring so that a shifted A descriptor of a partial entry (up to 12 KiB
  // before the entry) still addresses this CTA's shared memory.
  const uint32_t RB = static_cast<uint32_t>(a.ring_bytes);
  const uint32_t hb = a.T <= 8 ? 1024u : static_cast<uint32_t>(B_BYTES);  // h^T bytes per K-tile in an entry
  uint8_t* p = smem_raw;
  uint8_t* aT = p;  // [2 buf][2 part][4096]
  p += 2 * 2 * 4096;
  uint8_t* ring = p;
  p += RB;
  // down-projection accumulator across the segments of an entry:
  // shared memory (ysum), the partial block in global memory, or TMEM
  const int mode = a.acc_mode;
  float* ysum = reinterpret_cast<float*>(p);  // [T][d] (shared-memory mode)
  if (mode == ACC_SMEM) p += static_cast<size_t>(T) * d * 4;
  float* gate_s = reinterpret_cast<float*>(p);  // [2 slots][16] per-token gate of the entry
  p += 2 * 16 * 4;
  int* tok_s = reinterpret_cast<int*>(p);  // [2 slots][16] token list of the entry (for flush)
  p += 2 * 16 * 4;
  int* misc = reinterpret_cast<int*>(p);  // [1] tmem base, [2..3] ntok per slot
  p += 16;
  // routing of this CTA's first ENT_PRE entries, read once in the prologue
  float* ent_gate = reinterpret_cast<float*>(p);  // [ENT_PRE][16]
  p += ENT_PRE * 16 * 4;
  int* ent_tok = reinterpret_cast<int*>(p);  // [ENT_PRE][16]
  p += ENT_PRE * 16 * 4;
  int* ent_n = reinterpret_cast<int*>(p);  // [ENT_PRE]
  p += ENT_PRE * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;
  uint64_t* empty = full + NSLOT;
  uint64_t* d1_full = empty + NSLOT; // [2]
  uint64_t* d1_empty = d1_full + 2; // [2]
  uint64_t* at_full = d1_empty + 2; // [2]
  uint64_t* at_empty = at_full + 2; // [2]
  uint64_t* d2_full = at_empty + 2; // [2]
  uint64_t* d2_empty = d2_full + 2; // [2]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    stamp(a, 0);
    if (a.dbg) a.dbg[blockIdx.x * DBG + 7] = static_cast<unsigned long long>(clock64());
  }
  const int n_hits = a.counters[7];
  const long long n = static_cast<long long>(n_hits + a.n_shared) * qpe;
  // b: this CTA's partial blocks (local); bg / G: its share of the layer's
  // units (a virtual grid across GPUs in the unit-split mode)
  const int b = blockIdx.x;
  const int G = a.cta_total > 0 ? a.cta_total : static_cast<int>(gridDim.x);
  const long long bg = a.cta_base + b;
  const long long q0 = n > 0 ? (bg * n) / G : 0;
  const long long q1 = n > 0 ? ((bg + 1) * n) / G : 0;
  if (q0 >= q1) return;

  if (tid == 0) {
    for (int i = 0; i < NSLOT; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&d1_full[i], 1);
      mbar_init(&d1_empty[i], 4);
      mbar_init(&at_full[i], 1);
      mbar_init(&at_empty[i], 1);
      mbar_init(&d2_full[i], 1);
      mbar_init(&d2_empty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&misc[1])),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (mode == ACC_SMEM) {
    float4* ys = reinterpret_cast<float4*>(ysum);
    for (int i = tid; i < T * d / 4; i += THREADS) ys[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  {  // a^T columns of tokens >= T stay zero for the whole launch; the ring
     // starts zeroed so that the unit a partial down K-step reads past the
     // segment (a^T = 0 there) is finite even before the ring has wrapped
    uint4* z = reinterpret_cast<uint4*>(aT);
    for (int i = tid; i < 2 * 2 * 4096 / 16; i += THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
    uint4* zr = reinterpret_cast<uint4*>(ring);
    for (uint32_t i = tid; i < RB / 16; i += THREADS) zr[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async();
  }
  {
    // Stage the routing (token list, per-token gate) of the first ENT_PRE
    // entries of this CTA's range, one thread per entry, so that expert
    // switches in the epilogue are shared-memory lookups. K2 wrote these
    // several kernels ago, so no programmatic-dependency wait is needed.
    const int o0 = static_cast<int>(q0 / qpe);
    const int e = tid - 64;
    const int o = o0 + e;
    if (e >= 0 && e < ENT_PRE && static_cast<long long>(o) * qpe < q1) {
      for (int t = 0; t < 16; ++t) {
        ent_gate[e * 16 + t] = 0.f;
        ent_tok[e * 16 + t] = 0;
      }
      int nt;
      if (o < n_hits) {
        const int ex = a.hit_list[o];
        const int p0 = a.offsets[ex];
        nt = a.offsets[ex + 1] - p0;
        for (int j = 0; j < nt; ++j) {
          const int idx = a.perm[p0 + j];
          ent_tok[e * 16 + j] = idx / a.k;
          ent_gate[e * 16 + idx / a.k] = a.gates[idx];
        }
      } else {
        nt = T;
        for (int j = 0; j < T; ++j) {
          ent_tok[e * 16 + j] = j;
          ent_gate[e * 16 + j] = 1.f;
        }
      }
      ent_n[e] = nt;
    }
  }
  __syncwarp();  // bar.sync is warp-aligned: a warp arriving in pieces is counted once per piece
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = static_cast<uint32_t>(misc[1]);
  if (tid == 0) {
    pdl_trigger();  // the combine may launch and park on its own wait
    stamp(a, 1);
  }
  // Everything below except the producer's first weight copies depends on
  // the previous kernel (h^T image, partial workspace): wait for it.
  if (warp != 0) pdl_wait();
  if (tid == 32) {
    stamp(a, 22);  // predecessor complete (PDL) as seen by this CTA
    if (a.dbg) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.dbg[blockIdx.x * DBG + 24] = smid;
    }
  }

  // All three roles walk the same software-pipelined sequence of segments:
  //   GU(0), GU(1), DN(0), GU(2), DN(1), ..., DN(last)
  // so the tensor core streams chunk i+1's gate/up tiles while the epilogue
  // turns chunk i's D1 into a^T; DN(i) then finds a^T(i) ready.
  // tiles per ring entry are powers of two dividing the tile counts (and
  // the D2 pass, so a down entry never straddles two passes)
  const int kcap = pow2_divisor(ktiles, 8), mcap = pow2_divisor(mtiles, PASS_TILES);
  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    // The whole warp walks the loop in convergent flow (addresses stay in
    // uniform registers); one elected lane issues each copy. Entries are
    // allocated back to back in a byte ring (a partial segment's tiles cost
    // only its quarters' bytes) and released in order by the MMA commits.
    {
      const bool leader = elect_one();
      long long w_empty = 0;
      const uint64_t pol = a.l2_policy == 1 ? l2_evict_normal_policy() : l2_evict_first_policy();
      const uint8_t* hTb = reinterpret_cast<const uint8_t*>(a.hT);
      uint32_t head = 0, idx = 0, tail = 0;
      // In-flight entry table, one ring slot per lane (NSLOT == 32): lane s
      // holds the offset / size / sequence number of the entry in slot s,
      // so "does the new entry overlap any in-flight one" is one warp vote
      // (no shared-memory FIFO: the producer's shared-memory loads would
      // queue behind the epilogue's shared-memory traffic).
      uint32_t my_off = 0, my_size = 0, my_idx = 0xFFFFFFFFu;
      // place an entry; waits (oldest first) for the MMA to release what it
      // would overwrite. Returns false (nothing placed) if it would wait and
      // !may_wait.
      auto reserve = [&](const Geom& g, bool may_wait, uint32_t& e) -> bool {
        e = head;
        if (e + g.win > RB) e = 0;
        for (;;) {
          const bool mine = my_idx != 0xFFFFFFFFu && my_idx >= tail && my_off < e + g.size && e < my_off + my_size;
          const bool over = idx - tail >= static_cast<uint32_t>(NSLOT) || __any_sync(0xffffffffu, mine);
          if (!over) break;
          if (!may_wait) return false;
          wait_acc(a, &empty[tail % NSLOT], (tail / NSLOT) & 1u, w_empty);
          ++tail;
        }
        if (lane == static_cast<int>(idx % NSLOT)) {
          my_off = e;
          my_size = g.size;
          my_idx = idx;
        }
        head = e + ((g.size + 1023u) & ~1023u);
        return true;
      };
      // A parts of tiles [t0, t0 + m) of a segment, one tile per lane: a
      // thread's bulk copies issue one after another, copies from different
      // lanes overlap (tools/tma_probe.cu: 2 x 16 KiB from two lanes stream
      // ~8% faster per SM than one 32 KiB copy, and far faster than
      // sub-16 KiB runs from one lane)
      auto copy_tiles = [&](const uint8_t* base, int t0, int m, int qa, int nq, uint32_t e, uint64_t* bar) {
        __syncwarp();  // after the leader's expect_tx
        const uint32_t ab = static_cast<uint32_t>(nq) * UBYTES;
        for (int j = lane; j < m; j += 32)
          bulk_g2s(ring + e + j * ab, base + static_cast<size_t>(t0 + j) * A_BYTES + qa * UBYTES, ab, bar, pol);
      };
      // entry image bases, one lane per entry of the CTA's range, looked up
      // once: a segment change then costs a shuffle instead of two dependent
      // global loads (hit list -> slot) on the producer's critical path
      const int o_first = q1 > q0 ? static_cast<int>(q0 / qpe) : 0;
      const int n_ent = q1 > q0 ? static_cast<int>((q1 - 1) / qpe) - o_first + 1 : 0;
      unsigned long long my_ent = 0;
      if (lane < n_ent) my_ent = reinterpret_cast<unsigned long long>(entry_weights(a, o_first + lane, n_hits));
      auto seg_base = [&](const Seg& s) {  // (warp-uniform)
        const uint16_t* w =
            n_ent <= 32 ? reinterpret_cast<const uint16_t*>(__shfl_sync(0xffffffffu, my_ent, (s.o - o_first) & 31))
                        : entry_weights(a, s.o, n_hits);
        return reinterpret_cast<const uint8_t*>(w + s.c * chunk_elems);
      };
      SegIter it{q0, q1, qpe};
      Seg cur, prev;
      bool more = it.next(cur), has_prev = false;
      const uint8_t* cur_base = seg_base(cur);
      const uint8_t* prev_base = cur_base;
      // Weights do not depend on the previous kernel: put as many of the
      // first segment's gate/up weight copies in flight as fit without
      // waiting, then wait for the predecessor, then add their h^T slices.
      int kt0 = 0;
      {
        const int nq = cur.qb - cur.qa;
        const Geom g = gu_geom(nq, kcap, hb);
        int np = 0;
        uint32_t e;
        while (kt0 < ktiles && reserve(g, false, e)) {
          if (leader) mbar_arrive_expect_tx(&full[idx % NSLOT], g.size);
          copy_tiles(cur_base, kt0, g.m, cur.qa, nq, e, &full[idx % NSLOT]);
          ++idx;
          ++np;
          kt0 += g.m;
        }
        pdl_wait();
        // the prefetched entries lie back to back from offset 0 (no wrap)
        const uint32_t span = (g.size + 1023u) & ~1023u, ab = static_cast<uint32_t>(g.m * nq) * UBYTES;
        if (hb == B_BYTES) {
          for (int j = lane; j < np; j += 32)
            bulk_g2s(ring + j * span + ab, hTb + static_cast<size_t>(j * g.m) * B_BYTES,
                     static_cast<uint32_t>(g.m) * B_BYTES, &full[j], pol);
        } else {
          for (int c = lane; c < np * g.m; c += 32) {
            const int j = c / g.m, jj = c - j * g.m;
            bulk_g2s(ring + j * span + ab + jj * hb, hTb + static_cast<size_t>(j * g.m + jj) * B_BYTES, hb, &full[j],
                     pol);
          }
        }
      }
      while (more || has_prev) {
        if (more) {
          const int nq = cur.qb - cur.qa;
          const Geom g = gu_geom(nq, kcap, hb);
          const uint32_t ab = static_cast<uint32_t>(g.m * nq) * UBYTES;
          for (int kt = kt0; kt < ktiles; kt += g.m) {
            uint32_t e;
            reserve(g, true, e);
            uint64_t* bar = &full[idx % NSLOT];
            if (leader) mbar_arrive_expect_tx(bar, g.size);
            copy_tiles(cur_base, kt, g.m, cur.qa, nq, e, bar);
            if (hb == B_BYTES) {
              if (lane == 31)  // (m <= 8 < 31: a lane with no tile copy)
                bulk_g2s(ring + e + ab, hTb + static_cast<size_t>(kt) * B_BYTES,
                         static_cast<uint32_t>(g.m) * B_BYTES, bar, pol);
            } else if (lane >= 16 && lane < 16 + g.m) {  // one 1 KiB slice per lane
              const int jj = lane - 16;
              bulk_g2s(ring + e + ab + jj * hb, hTb + static_cast<size_t>(kt + jj) * B_BYTES, hb, bar, pol);
            }
            ++idx;
          }
          kt0 = 0;
        }
        if (has_prev) {
          const int nq = prev.qb - prev.qa;
          const Geom g = dn_geom(nq, mcap);
          const uint8_t* dbase = prev_base + static_cast<size_t>(ktiles) * A_BYTES;
          for (int mt = 0; mt < mtiles; mt += g.m) {
            uint32_t e;
            reserve(g, true, e);
            uint64_t* bar = &full[idx % NSLOT];
            if (leader) mbar_arrive_expect_tx(bar, g.size);
            copy_tiles(dbase, mt, g.m, prev.qa, nq, e, bar);
            ++idx;
          }
        }
        has_prev = more;
        prev = cur;
        prev_base = cur_base;
        if (more) {
          more = it.next(cur);
          if (more) cur_base = seg_base(cur);
        }
      }
      if (a.nx_counters && a.pf_bytes > 0) {
        // ---- cross-layer L2 prefetch (see FfnArgs::pf_bytes): the next
        // layer's routing is final (K2 ran for all layers), so walk this CTA
        // index's next-layer segments in stream order and prefetch their
        // gate/up runs, then their down runs, up to the byte budget.
        const int nh = a.nx_counters[7];
        const long long nn = static_cast<long long>(nh + a.n_shared) * qpe;
        const long long p0 = nn > 0 ? (bg * nn) / G : 0;
        const long long p1 = nn > 0 ? ((bg + 1) * nn) / G : 0;
        SegIter pit{p0, p1, qpe};
        Seg s;
        // (the next CTA fills its ring with the first ring_bytes itself)
        long long budget = a.pf_bytes, skip = RB;
        while (budget > 0 && pit.next(s)) {
          const uint16_t* w = s.o < nh ? a.nx_pool + static_cast<long long>(a.nx_slot_of[a.nx_hit_list[s.o]]) *
                                                          a.expert_elems
                                       : a.nx_shared_w + static_cast<long long>(s.o - nh) * a.expert_elems;
          const uint8_t* base = reinterpret_cast<const uint8_t*>(w + s.c * chunk_elems);
          const int nq = s.qb - s.qa;
          const uint32_t run = static_cast<uint32_t>(nq) * UBYTES;
          for (int t = 0; t < ktiles + mtiles && budget > 0; ++t) {
            if (skip > 0) {
              skip -= run;
              continue;
            }
            if (leader)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + static_cast<size_t>(t) * A_BYTES +
                                                                              s.qa * UBYTES),
                           "r"(run)
                           : "memory");
            budget -= run;
          }
        }
      }
      if (a.dbg && leader) a.dbg[blockIdx.x * DBG + 8] = static_cast<unsigned long long>(w_empty);
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // Whole warp in convergent flow so descriptors are warp-uniform (no
    // per-MMA R2UR waterfall); one elected lane issues MMAs and commits.
    // Entry offsets follow the producer's allocation rule.
    {
      const bool leader = elect_one();
      long long w_full = 0, w_at = 0, w_d2e = 0, w_d1e = 0;
      Phase d1e[2], ate[2], d2e[2];
      int c3 = 0;  // D2 pass buffer counter
      int ent_done = 0, last_dn_o = -1;  // TMEM mode: entries committed, entry of the last DN
      uint32_t head = 0, idx = 0;
      SegIter it{q0, q1, qpe};
      Seg cur, prev;
      bool more = it.next(cur), has_prev = false;
      int i = 0;
      const uint32_t ring_addr = smem_u32(ring);
      const uint32_t at_addr = smem_u32(aT);
      while (more || has_prev) {
        if (more) {  // GU(i): D1[i & 1] = W_gu x h^T
          const int b1 = i & 1;
          wait_acc(a, &d1_empty[b1], d1e[b1].bit ^ 1u, w_d1e);
          d1e[b1].flip();
          fence_after();
          const uint32_t d1 = tmem + static_cast<uint32_t>(b1 * 16);
          const int nq = cur.qb - cur.qa;
          const Geom g = gu_geom(nq, kcap, hb);
          const uint32_t ab = static_cast<uint32_t>(nq) * UBYTES;
          for (int kt = 0; kt < ktiles; kt += g.m) {
            const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
            wait_acc(a, &full[slot], (idx / NSLOT) & 1u, w_full);
            ++idx;
            if (i == 0 && kt == 0 && leader) stamp(a, 2);
            fence_after();
            // shifted base: rows of unit qa of tile j land at off + j*ab
            const uint32_t va = ring_addr + off - static_cast<uint32_t>(cur.qa) * UBYTES;
            const uint32_t vb = ring_addr + off + static_cast<uint32_t>(g.m) * ab;
            if (leader) {
              for (int j = 0; j < g.m; ++j) {
                const uint64_t adesc = smem_desc(va + j * ab, 128, 1024), bdesc = smem_desc(vb + j * hb, 128, 1024);
#pragma unroll
                for (int k = 0; k < 4; ++k)  // +256 B per K=16 step = +16 in the start-address field
                  mma_bf16(d1, adesc + 16 * k, bdesc + 16 * k, (kt | j | k) != 0);
              }
              mma_commit(&empty[slot]);
            }
            __syncwarp();
          }
          if (leader) mma_commit(&d1_full[b1]);
          __syncwarp();
          if (i == 0 && leader) stamp(a, 3);
          if (i < 5 && leader) {  // per-segment trace: GU(i) issued
            const int gs[5] = {15, 19, 23, 25, 31};
            stamp(a, gs[i]);
          }
        }
        if (has_prev) {  // DN(i-1): D2 = W_down x a^T(i-1), hi + lo
          const int ab_ = (i - 1) & 1;
          wait_acc(a, &at_full[ab_], ate[ab_].bit, w_at);
          ate[ab_].flip();
          fence_after();
          const uint32_t ahi = at_addr + static_cast<uint32_t>(ab_) * 8192u;
          const uint64_t bhi = smem_desc(ahi, 256, 128), blo = smem_desc(ahi + 4096u, 256, 128);
          const int nq = prev.qb - prev.qa;
          const Geom g = dn_geom(nq, mcap);
          const uint32_t tb = static_cast<uint32_t>(nq) * UBYTES;
          // K-steps (16 f = 2 units) overlapping the segment's units
          const int k0 = prev.qa >> 1, k1 = (prev.qb + 1) >> 1;
          if (mode == ACC_TMEM) {
            // D2[mt] accumulates the whole entry's down projection in TMEM
            // (all M-tiles resident); drained once, at the entry's last
            // segment in this CTA
            const bool first = prev.o != last_dn_o, last = !more || cur.o != prev.o;
            if (first && ent_done > 0) {
              wait_acc(a, &d2_empty[0], static_cast<uint32_t>(ent_done - 1) & 1u, w_d2e);
              fence_after();
            }
            for (int mt = 0; mt < mtiles; mt += g.m) {
              const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
              wait_acc(a, &full[slot], (idx / NSLOT) & 1u, w_full);
              ++idx;
              if (i == 1 && mt == 0 && leader) stamp(a, 16);
              fence_after();
              const uint32_t va = ring_addr + off - static_cast<uint32_t>(prev.qa) * UBYTES;
              if (leader) {
                for (int j = 0; j < g.m; ++j) {
                  const uint32_t d2 = tmem + D2_COL0 + static_cast<uint32_t>((mt + j) * 16);
                  const uint64_t adn = smem_desc(va + j * tb, 2048, 128);
                  for (int k = k0; k < k1; ++k) {
                    mma_bf16(d2, adn + 256 * k, bhi + 32 * k, (first && k == k0) ? 0u : 1u);
                    mma_bf16(d2, adn + 256 * k, blo + 32 * k, 1u);
                  }
                }
                mma_commit(&empty[slot]);
              }
              __syncwarp();
            }
            if (last) {
              if (leader) mma_commit(&d2_full[0]);
              __syncwarp();
              ++ent_done;
            }
            last_dn_o = prev.o;
          }
          for (int ps = 0; ps < (mode == ACC_TMEM ? 0 : passes); ++ps) {
            const int pb = c3 & 1;
            wait_acc(a, &d2_empty[pb], d2e[pb].bit ^ 1u, w_d2e);
            d2e[pb].flip();
            fence_after();
            const int mt_end = min(mtiles, (ps + 1) * PASS_TILES);
            for (int mt = ps * PASS_TILES; mt < mt_end; mt += g.m) {
              const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
              wait_acc(a, &full[slot], (idx / NSLOT) & 1u, w_full);
              ++idx;
              if (i == 1 && mt == 0 && leader) stamp(a, 16);
              fence_after();
              const uint32_t va = ring_addr + off - static_cast<uint32_t>(prev.qa) * UBYTES;
              if (leader) {
                for (int j = 0; j < g.m; ++j) {
                  const uint32_t d2 =
                      tmem + D2_COL0 + static_cast<uint32_t>(pb * 128 + (mt + j - ps * PASS_TILES) * 16);
                  const uint64_t adn = smem_desc(va + j * tb, 2048, 128);
                  for (int k = k0; k < k1; ++k) {  // +4096 B (A) / +512 B (a^T) per K=16 step
                    mma_bf16(d2, adn + 256 * k, bhi + 32 * k, k == k0 ? 0u : 1u);
                    mma_bf16(d2, adn + 256 * k, blo + 32 * k, 1u);
                  }
                }
                mma_commit(&empty[slot]);
              }
              __syncwarp();
            }
            if (leader) mma_commit(&d2_full[pb]);
            __syncwarp();
            ++c3;
          }
          if (leader) mma_commit(&at_empty[ab_]);
          __syncwarp();
          if (i == 1 && leader) stamp(a, 17);
        }
        has_prev = more;
        prev = cur;
        if (more) more = it.next(cur);
        ++i;
      }
      if (a.dbg && leader) {
        a.dbg[blockIdx.x * DBG + 9] = static_cast<unsigned long long>(w_full);
        a.dbg[blockIdx.x * DBG + 10] = static_cast<unsigned long long>(w_at);
        a.dbg[blockIdx.x * DBG + 11] = static_cast<unsigned long long>(w_d2e);
        a.dbg[blockIdx.x * DBG + 12] = static_cast<unsigned long long>(w_d1e);
      }
    }
  } else {
    // ------------------------------------------------ epilogue (4 warps)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int et = tid - 64; // 0..127
    Phase d1f[2], atf[2], d2f[2];
    long long w_d1f = 0, w_d2f = 0;
    int c3 = 0, ent_e = 0;  // ent_e: TMEM mode, entries drained
    int cur_entry = -1, eslot = 1;
    int seg_slot[2] = {0, 0};
    // per-entry token data, two slots (entry being drained / entry being fed)
    const int o_first = static_cast<int>(q0 / qpe);
    auto load_entry = [&](int o, int slot) {
      named_bar_sync(2, EPI_THREADS);
      const int pre = o - o_first;
      if (pre < ENT_PRE) {
        if (et < 16) {
          gate_s[slot * 16 + et] = ent_gate[pre * 16 + et];
          tok_s[slot * 16 + et] = ent_tok[pre * 16 + et];
        }
        if (et == 0) misc[2 + slot] = ent_n[pre];
        named_bar_sync(2, EPI_THREADS);
        if (mode == ACC_GLOBAL) {
          float* P = a.partial + static_cast<long long>(b + o) * T * d;
          const int nt = misc[2 + slot];
          for (int t = 0; t < nt; ++t)
            for (int c = et * 4; c < d; c += EPI_THREADS * 4)
              *reinterpret_cast<float4*>(P + static_cast<long long>(tok_s[slot * 16 + t]) * d + c) =
                  make_float4(0.f, 0.f, 0.f, 0.f);
          named_bar_sync(2, EPI_THREADS);
        }
        return;
      }
      if (et < 16) {
        gate_s[slot * 16 + et] = 0.f;
        tok_s[slot * 16 + et] = 0;
      }
      named_bar_sync(2, EPI_THREADS);
      if (et == 0) {
        int nt = 0;
        if (o < n_hits) {
          const int e = a.hit_list[o];
          const int p0 = a.offsets[e];
          nt = a.offsets[e + 1] - p0;
          for (int i = 0; i < nt; ++i) {
            const int idx = a.perm[p0 + i];
            tok_s[slot * 16 + i] = idx / a.k;
            gate_s[slot * 16 + idx / a.k] = a.gates[idx];
          }
        } else {
          nt = T;
          for (int i = 0; i < T; ++i) {
            tok_s[slot * 16 + i] = i;
            gate_s[slot * 16 + i] = 1.f;
          }
        }
        misc[2 + slot] = nt;
      }
      named_bar_sync(2, EPI_THREADS);
      if (mode == ACC_GLOBAL) {  // zero this entry's rows of the CTA-exclusive partial block
        float* P = a.partial + static_cast<long long>(b + o) * T * d;
        const int nt = misc[2 + slot];
        for (int t = 0; t < nt; ++t)
          for (int c = et * 4; c < d; c += EPI_THREADS * 4)
            *reinterpret_cast<float4*>(P + static_cast<long long>(tok_s[slot * 16 + t]) * d + c) =
                make_float4(0.f, 0.f, 0.f, 0.f);
        named_bar_sync(2, EPI_THREADS);
      }
    };
    auto flush = [&](int o, int slot) {
      named_bar_sync(2, EPI_THREADS);
      if (mode == ACC_SMEM) {
        const int nt = misc[2 + slot];
        float* P = a.partial + static_cast<long long>(b + o) * T * d;
        for (int t = 0; t < nt; ++t) {
          const int tg = tok_s[slot * 16 + t];
          for (int c = et * 4; c < d; c += EPI_THREADS * 4) {
            float4* src = reinterpret_cast<float4*>(ysum + static_cast<size_t>(tg) * d + c);
            *reinterpret_cast<float4*>(P + static_cast<long long>(tg) * d + c) = *src;
            *src = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      named_bar_sync(2, EPI_THREADS);
    };
    SegIter it{q0, q1, qpe};
    Seg cur, prev;
    bool more = it.next(cur), has_prev = false;
    int i = 0;
    while (more || has_prev) {
      if (more) {
        // ---- A(i): D1 -> a^T (bf16 hi/lo) for DN(i)
        if (cur.o != cur_entry) {
          eslot ^= 1;
          load_entry(cur.o, eslot);
          cur_entry = cur.o;
        }
        seg_slot[i & 1] = eslot;
        const float* gs = gate_s + eslot * 16;
        const int b1 = i & 1;
        wait_acc(a, &d1_full[b1], d1f[b1].bit, w_d1f);
        d1f[b1].flip();
        fence_after();
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(b1 * 16), v);
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d1_empty[b1]);
        const int ab = i & 1;
        // a^T buffer ab is free once DN(i-2) completed
        mbar_wait(&at_empty[ab], atf[ab].bit ^ 1u);
        atf[ab].flip();
        // This warp's TMEM lanes are chunk quarter q, octet-interleaved:
        // lanes 8h..8h+7 hold the gate rows f = 16q + 8h + (lane & 7), lanes
        // 8h+8..8h+15 the up rows of the same f (h = lane >> 4).
        if (2 * q + 1 >= cur.qa && 2 * q < cur.qb) {
          // the quarter overlaps the segment; a unit of it outside the
          // segment gets a = 0 (a down K-step covers both of its units)
          const int unit = 2 * q + (lane >> 4);
          const bool inside = unit >= cur.qa && unit < cur.qb;
          const int f = 16 * q + ((lane >> 4) << 3) + (lane & 7);
          const int up = (lane >> 3) & 1;
          uint16_t* hi = reinterpret_cast<uint16_t*>(aT + static_cast<size_t>(ab) * 8192);
          uint16_t* lo = hi + 2048;
          float gts[16];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 x = reinterpret_cast<const float4*>(gs)[j];
            gts[4 * j] = x.x;
            gts[4 * j + 1] = x.y;
            gts[4 * j + 2] = x.z;
            gts[4 * j + 3] = x.w;
          }
          // gate lanes take the even tokens, up lanes the odd ones (t = 2j +
          // up), one xor-8 shuffle each; branch-free so the eight chains
          // interleave (a serial branchy token loop took ~2 us per segment)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int t = 2 * j + up;
            const float pv = __shfl_xor_sync(0xffffffffu, up ? v[2 * j] : v[2 * j + 1], 8);
            const float g = up ? pv : v[2 * j];
            const float u = up ? v[2 * j + 1] : pv;
            const float gt = up ? gts[2 * j + 1] : gts[2 * j];
            const float sv = __fdividef(g, 1.f + __expf(-g)) * u * gt;
            const float av = (inside && t < T && gt != 0.f) ? sv : 0.f;
            const uint16_t h16 = f32_to_bf16_cvt(av);
            const float rem = av - __uint_as_float(static_cast<uint32_t>(h16) << 16);
            // byte = j*256 + tg*128 + r*16 + e*2 (token = 8 tg + r, f = 8 j + e)
            const int off = (f >> 3) * 128 + (t >> 3) * 64 + (t & 7) * 8 + (f & 7);
            hi[off] = h16;
            lo[off] = f32_to_bf16_cvt(rem);
          }
        }
        fence_proxy_async();
        named_bar_sync(2, EPI_THREADS);
        if (et == 0) {
          mbar_arrive(&at_full[ab]);
          if (i == 0) stamp(a, 4);
        }
      }
      if (has_prev && mode == ACC_TMEM) {
        // ---- D(i-1), TMEM mode: at the entry's last segment here, drain
        // D2 (all M-tiles) straight into this CTA's partial block
        if (!more || cur.o != prev.o) {
          wait_acc(a, &d2_full[0], static_cast<uint32_t>(ent_e) & 1u, w_d2f);
          if (i == 1 && et == 0) stamp(a, 18);
          fence_after();
          const int slot = seg_slot[(i - 1) & 1];
          uint32_t tmask = 0;  // tokens of this entry
          for (int tt = 0; tt < misc[2 + slot]; ++tt) tmask |= 1u << tok_s[slot * 16 + tt];
          float* P = a.partial + static_cast<long long>(b + prev.o) * T * d + 32 * q + lane;
          const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(D2_COL0);
          for (int mt = 0; mt < mtiles; mt += 2) {  // two M-tiles per TMEM wait
            uint32_t y0[16], y1[16];
            const bool two = mt + 1 < mtiles;
            if (T <= 8) {
              tmem_ld8_nw(tbase + static_cast<uint32_t>(mt * 16), y0);
              if (two) tmem_ld8_nw(tbase + static_cast<uint32_t>((mt + 1) * 16), y1);
            } else {
              tmem_ld16_nw(tbase + static_cast<uint32_t>(mt * 16), y0);
              if (two) tmem_ld16_nw(tbase + static_cast<uint32_t>((mt + 1) * 16), y1);
            }
            tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (t < T && ((tmask >> t) & 1u)) {
                __stcg(P + static_cast<long long>(t) * d + mt * 128, __uint_as_float(y0[t]));
                if (two) __stcg(P + static_cast<long long>(t) * d + mt * 128 + 128, __uint_as_float(y1[t]));
              }
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d2_empty[0]);
          ++ent_e;
          if (i == 1 && et == 0) stamp(a, 20);
        }
      }
      if (has_prev && mode != ACC_TMEM) {
        // ---- D(i-1): D2 passes -> per-expert fp32 accumulator
        for (int ps = 0; ps < passes; ++ps) {
          const int pb = c3 & 1;
          wait_acc(a, &d2_full[pb], d2f[pb].bit, w_d2f);
          d2f[pb].flip();
          if (i == 1 && et == 0) stamp(a, 18 + (ps == 0 ? 0 : 1));
          fence_after();
          const int mt0 = ps * PASS_TILES, mt_end = min(mtiles, mt0 + PASS_TILES);
          const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(D2_COL0 + pb * 128);
          float* P = a.partial + static_cast<long long>(b + prev.o) * T * d;
          const float* gsl = gate_s + seg_slot[(i - 1) & 1] * 16;
          // four M-tiles per tcgen05.wait::ld (the drain is load-latency
          // bound: one TMEM round trip per wait, ~4x fewer than per tile)
          for (int mb = mt0; mb < mt_end; mb += 4) {
            uint32_t y[4][16];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (mb + j < mt_end) {  // only the first T token columns matter
                if (T <= 8)
                  tmem_ld8_nw(tbase + static_cast<uint32_t>((mb + j - mt0) * 16), y[j]);
                else
                  tmem_ld16_nw(tbase + static_cast<uint32_t>((mb + j - mt0) * 16), y[j]);
              }
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (mb + j >= mt_end) break;
              const int orow = (mb + j) * 128 + 32 * q + lane;
              if (mode == ACC_GLOBAL) {
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  if (t < T && gsl[t] != 0.f) P[static_cast<long long>(t) * d + orow] += __uint_as_float(y[j][t]);
              } else {
                // all loads, then all stores: the T read-modify-writes of a
                // row are independent (a += chain would serialise on each LDS)
                float* r0 = ysum + orow;
                float o0[16];
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  if (t < T) o0[t] = r0[static_cast<size_t>(t) * d];
#pragma unroll
                for (int t = 0; t < 16; ++t)
                  if (t < T) r0[static_cast<size_t>(t) * d] = o0[t] + __uint_as_float(y[j][t]);
              }
            }
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d2_empty[pb]);
          ++c3;
        }
        if (i == 1 && et == 0) stamp(a, 20);
        if (!more || cur.o != prev.o) flush(prev.o, seg_slot[(i - 1) & 1]);
        if (i == 1 && et == 0) stamp(a, 21);
      }
      has_prev = more;
      prev = cur;
      if (more) more = it.next(cur);
      ++i;
    }
    if (a.dbg && tid == 64) {
      a.dbg[blockIdx.x * DBG + 13] = static_cast<unsigned long long>(w_d1f);
      a.dbg[blockIdx.x * DBG + 14] = static_cast<unsigned long long>(w_d2f);
    }
  }
  if (tid == 64) {
    stamp(a, 5);  // epilogue finished (all flushes written)
  }
  __syncwarp();  // bar.sync is warp-aligned: a warp arriving in pieces is counted once per piece
  fence_before();
  __syncthreads();
  if (tid == 0) {
    stamp(a, 6);
    if (a.dbg) a.dbg[blockIdx.x * DBG + 7] = static_cast<unsigned long long>(clock64()) - a.dbg[blockIdx.x * DBG + 7];
  }
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// h [T][d] bf16 -> h^T image: per K-tile of 64, [tg 2][j 8][r 8][e 8] bf16
// (token = 8 tg + r, k = 64 kt + 8 j + e), tokens >= T zero.
__global__ void build_hT_kernel(const uint16_t* __restrict__ h, int T, int d, uint16_t* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int total = (d / 64) * 1024;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int kt = i >> 10, w = i & 1023;
    const int tg = w >> 9, j = (w >> 6) & 7, r = (w >> 3) & 7, e = w & 7;
    const int t = tg * 8 + r, k = kt * 64 + j * 8 + e;
    out[i] = t < T ? h[static_cast<size_t>(t) * d + k] : static_cast<uint16_t>(0);
  }
}

// Standard layouts <-> v2 tiled image (see file header); kUnpack scatters
// the image back through the same index map.
template <bool kUnpack>
__global__ void pack_expert_tc_kernel(uint16_t* __restrict__ wg, uint16_t* __restrict__ wu, uint16_t* __restrict__ wd,
                                      int d, int ffn, uint16_t* __restrict__ out) {
  const long long total = 3LL * ffn * d;
  const long long chunk = 3LL * FCH * d;
  const long long gu = 2LL * FCH * d;
  for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = idx / chunk, r0 = idx % chunk;
    uint16_t* src;
    if (r0 < gu) {
      const long long kt = r0 / 8192;
      const int w = static_cast<int>(r0 % 8192);
      const int g = w >> 9, j = (w >> 6) & 7, r = (w >> 3) & 7, e = w & 7;
      // quarter q = row / 32, octet-interleaved: gate f 0-7, up f 0-7, gate f 8-15, up f 8-15
      const int row = g * 8 + r;
      const int qq = row >> 5, s = row & 31;
      const long long f = c * FCH + qq * 16 + ((s >> 4) << 3) + (s & 7);
      const long long k = kt * 64 + j * 8 + e;
      src = ((s >> 3) & 1) ? &wu[f * d + k] : &wg[f * d + k];
    } else {
      const long long r2 = r0 - gu;
      const long long mt = r2 / 8192;
      const int w = static_cast<int>(r2 % 8192);
      const int j = w >> 10, g = (w >> 6) & 15, r = (w >> 3) & 7, e = w & 7;
      const long long orow = mt * 128 + g * 8 + r;
      const long long f = c * FCH + j * 8 + e;
      src = &wd[orow * ffn + f];
    }
    if (kUnpack)
      *src = out[idx];
    else
      out[idx] = *src;
  }
}

}  // namespace tc
}  // namespace dev

size_t ffn_tc_smem_bytes(int T, int d, int ring_bytes, int acc_mode) {
  return 2 * 2 * 4096 + static_cast<size_t>(ring_bytes) +
         (acc_mode == dev::tc::ACC_SMEM ? static_cast<size_t>(T) * d * 4 : 0) + 2 * 16 * 4 * 2 + 16 +
         dev::tc::ENT_PRE * (16 * 8 + 4) + 8 + 8 * (2 * dev::tc::NSLOT + 12);
}

// accum: 0 auto, 1 shared-memory accumulator, 2 global (L2) accumulator,
// 3 TMEM accumulator, 4 grouped (whole-CTA TMEM accumulator, separate
// kernel). Auto: grouped when d <= 2048, else TMEM when D2 for every M-tile fits next to the
// D1 buffers (d <= 2048) — no per-segment accumulate pass at all and the
// whole remaining shared memory for the ring; else shared memory when it
// leaves a >= 64 KiB ring; else global. Measured: the L2 accumulator puts
// dependent global read-modify-writes on the drain's critical path and loses
// ~30% even with a deeper ring, so it is only the fallback for large T x d.
FfnPlan ffn_tc_plan(int T, int d, size_t smem_limit, int accum) {
  // Leave room on the SM for one combine CTA (3 KiB static + 1 KiB reserve)
  // next to the K3 CTA (+1 KiB reserve) of 228 KiB: programmatic dependent
  // launch only overlaps the two kernels when they can co-reside.
  // (the grouped K3 sits next to the 8-warp combine: 4 KiB static + 1 KiB)
  constexpr size_t kSmPerSm = 233472, kReserve = 1024, kCombine = 3072 + 1024, kCombine8 = 4096 + 1024 + 256;
  const size_t limit_grouped = std::min(smem_limit, kSmPerSm - kReserve - kCombine8);
  if (smem_limit > kSmPerSm - kReserve - kCombine) smem_limit = kSmPerSm - kReserve - kCombine;
  auto ring_for = [&](int mode) -> int {
    const size_t fixed = ffn_tc_smem_bytes(T, d, 0, mode);
    if (fixed + 32768 > smem_limit) return 0;
    return static_cast<int>(((smem_limit - fixed) / 1024) * 1024);
  };
  auto plan = [&](int mode, int rb) {
    FfnPlan p{rb / 1024, mode == dev::tc::ACC_GLOBAL, ffn_tc_smem_bytes(T, d, rb, mode)};
    p.acc_mode = mode;
    return p;
  };
  const bool tmem_ok = d <= dev::tc::TMEM_ACC_MAX_D;
  // the grouped kernel holds D2 for every M-tile in TMEM: d <= 2048 at
  // N = 16, or d <= 4096 with T <= 8 tokens at N = 8 (the Mixtral shape:
  // measured 5.44 -> 5.22 ms per step against the per-segment kernel)
  const bool grouped_ok = tmem_ok || (d <= 4096 && T <= 8);
  if (accum == 4 || (accum == 0 && grouped_ok)) {
    // grouped kernel (expert_ffn_grouped.cu): whole-CTA TMEM accumulator
    const int rb = ffn_tg_ring_bytes(T, d, limit_grouped);
    if (rb > 0) {
      FfnPlan p{rb / 1024, false, ffn_tg_smem_bytes(T, d, rb)};
      p.acc_mode = dev::tc::ACC_GROUP;
      return p;
    }
    if (accum == 4) return {0, false, 0};
  }
  if (accum == 3 || (accum == 0 && tmem_ok)) {
    if (!tmem_ok) return {0, false, 0};
    const int rb = ring_for(dev::tc::ACC_TMEM);
    if (rb >= 32768) return plan(dev::tc::ACC_TMEM, rb);
    return {0, false, 0};
  }
  if (accum != 2) {
    const int rb = ring_for(dev::tc::ACC_SMEM);
    if (rb >= (accum == 1 ? 32768 : 65536)) return plan(dev::tc::ACC_SMEM, rb);
  }
  const int rb = ring_for(dev::tc::ACC_GLOBAL);
  if (rb >= 32768) return plan(dev::tc::ACC_GLOBAL, rb);
  return {0, false, 0};
}

cudaError_t launch_expert_ffn_tc(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl) {
  if (a.acc_mode == dev::tc::ACC_GROUP) return launch_expert_ffn_tg(a, grid, smem, stream, pdl);
  if (const cudaError_t e = smem_optin_once<dev::tc::expert_ffn_tc_kernel>(232448); e != cudaSuccess) return e;
  return launch_pdl(dev::tc::expert_ffn_tc_kernel, dim3(grid), dim3(dev::tc::THREADS), smem, stream, pdl, a);
}

cudaError_t launch_build_hT(const uint16_t* h, int T, int d, uint16_t* out, cudaStream_t stream, bool pdl) {
  return launch_pdl(dev::tc::build_hT_kernel, dim3((d / 64 * 1024 + 255) / 256), dim3(256), 0, stream, pdl, h, T, d,
                    out);
}

cudaError_t launch_pack_expert_tc(const uint16_t* wg, const uint16_t* wu, const uint16_t* wd, int d, int ffn,
                                  uint16_t* out, cudaStream_t stream) {
  dev::tc::pack_expert_tc_kernel<false><<<1184, 256, 0, stream>>>(
      const_cast<uint16_t*>(wg), const_cast<uint16_t*>(wu), const_cast<uint16_t*>(wd), d, ffn, out);
  return cudaGetLastError();
}

cudaError_t launch_unpack_expert_tc(const uint16_t* image, int d, int ffn, uint16_t* wg, uint16_t* wu, uint16_t* wd,
                                    cudaStream_t stream) {
  dev::tc::pack_expert_tc_kernel<true><<<1184, 256, 0, stream>>>(wg, wu, wd, d, ffn, const_cast<uint16_t*>(image));
  return cudaGetLastError();
}

}  // namespace moespac
