// K3 (grouped tensor-core variant, d <= 2048) — grouped SwiGLU expert FFN
// whose down-projection accumulator is the whole CTA's work, held in TMEM.
//
// Same image layout (v2, see expert_ffn_tc.cu) and the same byte-balanced
// split of the layer's (expert, 16-row ffn quarter) units over a persistent
// grid as the per-segment kernel; what changes is how a CTA walks its range:
//
//  * Groups, not chunk segments. The CTA's quarters are taken four at a time
//    in global order, whatever chunk or expert they belong to, and packed into
//    the four 32-row slots of one M = 128 gate|up tile (slot s = rows
//    32s..32s+31: gate and up rows of the same 16 ffn rows, octet-interleaved). A
//    CTA with 5-6 quarters runs two full-width GU passes instead of 2-3
//    partial chunk segments.
//  * One accumulator. The gate of token t for expert e is applied in the
//    SwiGLU epilogue (a = silu(g)·u·g_{t,e}, 0 for tokens not routed to e),
//    so the down projections of different experts can share one D2
//    accumulator: D2[d][16 tokens] in TMEM columns 256-511 sums every group
//    of the CTA and is drained once, at the end, through shared memory with
//    bulk stores — one partial block per CTA instead of one per
//    (CTA, expert) pair.
//  * h^T resident. The layer's h^T image (d/64 slices of 2 KiB) is loaded
//    into shared memory once, one mbarrier per slice, instead of riding along
//    with every GU entry (that re-streamed 64 KiB from L2 per segment: up to a
//    third of a narrow segment's bytes).
//
// The combine reads, for token t, the partial blocks of the CTAs whose
// range covers a quarter of one of t's experts, in ascending CTA order.
//
// Warp roles (192 threads): 0 TMA producer, 1 MMA issuer (TMEM owner),
// 2-5 epilogue (TMEM lane quarters 2, 3, 0, 1 = group slots).
#include <cstdint>

#include "common.cuh"
#include "k3_stream.cuh"
#include "launch.hpp"
#include "tcgen05.cuh"

namespace moespac {
namespace dev {
namespace tg {

using tc::elect_one;
using tc::fence_after;
using tc::fence_before;
using tc::fence_proxy_async;
using tc::mma_bf16;
using tc::mma_commit;
using tc::Phase;
using tc::smem_desc;

constexpr int THREADS = 192;
constexpr int EPI_THREADS = 128;
constexpr int NSLOT = 32;      // ring entries in flight (mbarrier pairs)
constexpr int TILE = k3s::TILE;  // one gate|up K-tile or down M-tile of a 64-row chunk
constexpr int UB = k3s::UB;      // one 8-row unit (gate + up octet) of a gate|up tile, or 8 k of a down tile
constexpr int GMAX = 16;       // units per group: up to two M = 128 gate|up tiles (8 units each)
constexpr int HTS = 2048;      // h^T slice of one K-tile (16 tokens x 64 k); 1 KiB (8 tokens) in N = 8 mode
constexpr int ENT_MAX = 32;    // entries one CTA may touch (one producer lane each)
constexpr int MAX_KT = 64;     // d <= 2048 (d <= 4096 in N = 8 mode, T <= 8)
constexpr int D2_COL0 = 256;
constexpr int TMEM_COLS = 512;
constexpr int DBG = 32;
constexpr int D2E = 32;        // entries of a CTA's last DN pass (<= d/128 M-tiles)

// ---------------------------------------------------------------- groups
// Work unit = 8 ffn rows of one expert; groups of <= gmax (8 or 16) units,
// at most two chunk pieces each (k3_stream.cuh). (A CTA's 9 units always fit
// one 16-unit group; measured, a third piece per group made the producer's
// per-copy bookkeeping ~4% slower on the Qwen3 shape.)
using k3s::Grp;
using k3s::GroupIt;

__device__ __forceinline__ int pow2_divisor(int x, int cap) {
  int m = 1;
  while (m < cap && x % (2 * m) == 0) m *= 2;
  return m;
}
// tiles per ring entry: >= 24-32 KiB of weights per entry whatever the width
// (capped by the power-of-two divisor of the tile count), so the
// single-warp producer/MMA bookkeeping per entry is amortised
__device__ __forceinline__ int tiles_per_entry(int nu, int cap) {
  const int t = nu >= 12 ? 1 : (nu >= 8 ? 2 : (nu >= 4 ? 4 : (nu >= 2 ? 8 : 16)));
  return t < cap ? t : cap;
}
struct Geom {
  uint32_t size, win;  // bytes; read window from the entry start
  int m;
};
__device__ __forceinline__ Geom gu_geom(int nu, int cap) {
  const int m = tiles_per_entry(nu, cap);
  const uint32_t a = static_cast<uint32_t>(nu) * UB;
  const uint32_t size = static_cast<uint32_t>(m) * a;
  // the last tile's M = 128 A operands read 16 KiB each (one or two of them)
  const uint32_t w = static_cast<uint32_t>(m - 1) * a + static_cast<uint32_t>((nu + 7) / 8) * TILE;
  return {size, size > w ? size : w, m};
}
__device__ __forceinline__ Geom dn_geom(int nu, int cap) {
  const int m = tiles_per_entry(nu, cap);
  const uint32_t size = static_cast<uint32_t>(m) * static_cast<uint32_t>(nu) * UB;
  return {size, size, m};
}
__device__ __forceinline__ uint32_t ring_place(uint32_t& head, const Geom& g, uint32_t rb) {
  uint32_t e = head;
  if (e + g.win > rb) e = 0;
  head = e + ((g.size + 1023u) & ~1023u);
  return e;
}

__device__ __forceinline__ void stamp(const FfnArgs& a, int slot) {
  if (a.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    a.dbg[blockIdx.x * DBG + slot] = t;
  }
}
__device__ __forceinline__ void wait_acc(const FfnArgs& a, uint64_t* bar, uint32_t parity, long long& acc) {
  if (a.dbg) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}

__device__ __forceinline__ void bulk_s2g(void* gmem_dst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
}
// (the source reads only: kernel completion makes the writes visible to the
// dependent combine)
__device__ __forceinline__ void bulk_commit_wait_all() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// <= 200 registers so a 4-warp combine CTA still fits next to this CTA
// (programmatic dependent launch overlaps the two only when they co-reside).
__global__ void __maxnreg__(200) expert_ffn_tg_kernel(FfnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int d = a.d, T = a.T;
  // N = 8 mode (d > 2048, T <= 8): MMAs over 8 token columns, so D2 takes 8
  // TMEM columns per M-tile and fits 32 M-tiles (d = 4096) in columns
  // 256-511; the resident h^T keeps only the first 8 token rows (1 KiB per
  // K-tile)
  const bool n8 = a.tg_n8 != 0;
  const uint32_t hsz = n8 ? 1024u : static_cast<uint32_t>(HTS);
  const uint32_t idesc = n8 ? tc::IDESC_N8 : tc::IDESC;
  const int d2w = n8 ? 8 : 16;
  const int ktiles = d / 64, mtiles = d / 128;
  const long long chunk_bytes = 3LL * 64 * d * 2;
  const int upe = a.ffn / 8;
  const int gmax = a.group_units == 16 ? 16 : 8;  // measured: 8 (one tile per group round) is faster
  const uint32_t RB = static_cast<uint32_t>(a.ring_bytes);

  // [a^T 2 x (hi, lo) x 4 KiB][h^T ktiles x 2 KiB][ring][2 KiB zeros][entry gates][entry masks][misc][mbarriers]
  uint8_t* p = smem_raw;
  uint8_t* aT = p;
  p += 2 * 2 * 4096;
  uint8_t* hts = p;
  p += static_cast<size_t>(ktiles) * hsz;
  uint8_t* ring = p;
  p += RB;
  uint8_t* zeros = p;  // the missing half of an odd group's last down K-step (finite, times a^T = 0)
  p += UB;
  float* ent_gate = reinterpret_cast<float*>(p);  // [ENT_MAX][16]
  p += ENT_MAX * 16 * 4;
  uint32_t* ent_mask = reinterpret_cast<uint32_t*>(p);  // [ENT_MAX] tokens routed to the entry
  p += ENT_MAX * 4;
  int* misc = reinterpret_cast<int*>(p);  // [1] TMEM base
  p += 16;
  float* sg_part = reinterpret_cast<float*>(p);  // [4 warps][16 tokens] shared-gate partial dots
  p += 4 * 16 * 4;
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;
  uint64_t* empty = full + NSLOT;
  uint64_t* d1_full = empty + NSLOT;  // [2]
  uint64_t* d1_empty = d1_full + 2;   // [2]
  uint64_t* at_full = d1_empty + 2;   // [2]
  uint64_t* at_empty = at_full + 2;   // [2]
  uint64_t* d2e = at_empty + 2;       // [D2E]: the last DN pass's entries, one each
  uint64_t* ht_full = d2e + D2E;      // [ktiles]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    stamp(a, 0);
    if (a.dbg) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.dbg[blockIdx.x * DBG + 24] = smid;
    }
  }
  const int n_hits = a.counters[7];
  const long long n = static_cast<long long>(n_hits + a.n_shared) * upe;
  // b: this CTA's partial block (local); bg / G: its share of the layer's
  // units (a virtual grid across GPUs in the unit-split mode)
  const int b = blockIdx.x;
  const int G = a.cta_total > 0 ? a.cta_total : static_cast<int>(gridDim.x);
  const long long bg = a.cta_base + b;
  const long long u0 = n > 0 ? (bg * n) / G : 0;
  const long long u1 = n > 0 ? ((bg + 1) * n) / G : 0;
  if (u0 >= u1) return;
  const int o_first = static_cast<int>(u0 / upe);
  const int n_ent = static_cast<int>((u1 - 1) / upe) - o_first + 1;
  if (n_ent > ENT_MAX) __trap();  // the host plan rules this out (ffn_tg_grid_ok)

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
    }
    for (int i = 0; i < D2E; ++i) mbar_init(&d2e[i], 1);
    for (int i = 0; i < ktiles; ++i) mbar_init(&ht_full[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  __syncthreads();
  if (tid == 0) pdl_trigger();  // the combine may launch and park on its own wait

  const int kcap = pow2_divisor(ktiles, 16), mcap = pow2_divisor(mtiles, 16);
  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    // Starts streaming weights right away (they do not depend on the
    // previous kernel); the h^T slices follow the programmatic-dependency
    // wait, which it takes the first time the ring is full (or at the end).
    const bool leader = elect_one();
    long long w_empty = 0;
    const uint64_t pol = a.l2_policy == 1 ? l2_evict_normal_policy() : l2_evict_first_policy();
    const uint64_t pol_h = l2_evict_normal_policy();
    // entry image bases, one lane per entry of this CTA's range
    unsigned long long my_base = 0;
    if (lane < n_ent) {
      const int o = o_first + lane;
      const uint16_t* w = o < n_hits ? a.pool + static_cast<long long>(a.slot_of[a.hit_list[o]]) * a.expert_elems
                                     : a.shared_w + static_cast<long long>(o - n_hits) * a.expert_elems;
      my_base = reinterpret_cast<unsigned long long>(w);
    }
    bool waited = false;
    // (Measured: an own-stream L2 prefetch issued here, at the first full
    // ring before the input wait, made the layer 7-15% slower for 128-384
    // KiB per CTA on the Qwen3 / DeepSeek-V2-Lite shapes; not used.)
    auto wait_pred = [&]() {
      pdl_wait();
      {  // one slice per lane: bulk copies issued by one thread serialise
        const uint8_t* hTb = reinterpret_cast<const uint8_t*>(a.hT);
        for (int kt = lane; kt < ktiles; kt += 32) {
          mbar_arrive_expect_tx(&ht_full[kt], hsz);
          bulk_g2s(hts + kt * hsz, hTb + static_cast<size_t>(kt) * HTS, hsz, &ht_full[kt], pol_h);
        }
      }
      waited = true;
      stamp(a, 22);
    };
    uint32_t head = 0, idx = 0, tail = 0;
    // in-flight entry table, one ring slot per lane (NSLOT == 32): the
    // "does the new entry overlap an unreleased one" test is one warp vote
    uint32_t my_off = 0, my_size = 0, my_idx = 0xFFFFFFFFu;
    auto reserve = [&](const Geom& g) -> uint32_t {
      uint32_t e = head;
      if (e + g.win > RB) e = 0;
      for (;;) {
        const bool mine = my_idx != 0xFFFFFFFFu && my_idx >= tail && my_off < e + g.size && e < my_off + my_size;
        const bool over = idx - tail >= static_cast<uint32_t>(NSLOT) || __any_sync(0xffffffffu, mine);
        if (!over) break;
        if (!waited) wait_pred();
        wait_acc(a, &empty[tail % NSLOT], (tail / NSLOT) & 1u, w_empty);
        ++tail;
      }
      if (lane == static_cast<int>(idx % NSLOT)) {
        my_off = e;
        my_size = g.size;
        my_idx = idx;
      }
      head = e + ((g.size + 1023u) & ~1023u);
      return e;
    };
    // chunk bases of a group's pieces (warp-uniform: every lane shuffles)
    auto piece_bases = [&](const Grp& g, const uint8_t* (&pb)[2]) {
      const unsigned long long b0 = __shfl_sync(0xffffffffu, my_base, g.o[0] - o_first);
      const unsigned long long b1 = __shfl_sync(0xffffffffu, my_base, g.np > 1 ? g.o[1] - o_first : 0);
      pb[0] = reinterpret_cast<const uint8_t*>(b0) + static_cast<long long>(g.c[0]) * chunk_bytes;
      pb[1] = reinterpret_cast<const uint8_t*>(b1) + static_cast<long long>(g.np > 1 ? g.c[1] : 0) * chunk_bytes;
    };
    // tiles [t0, t0 + m) (tile index within the chunk: K-tiles then M-tiles)
    // of every piece, slot-packed: tile j of the entry at j * nu * 2 KiB.
    // One bulk copy per (tile, piece), one copy per lane: a thread's bulk
    // copies issue one after another (~0.1-0.3 us each, tools/tma_probe.cu),
    // copies from different lanes overlap — with one issuing lane, split runs
    // capped the stream at 8-40 GB/s per SM. (Measured: issuing a one-piece
    // group's entry as ONE 5-D TMA tensor copy instead — n runs x m tiles —
    // changed nothing on Qwen3 / DeepSeek-V2-Lite step time; removed.)
    auto copy_entry = [&](const Grp& g, const uint8_t* const (&pb)[2], int t0, int m, uint32_t e, uint64_t* bar) {
      const uint32_t ab = static_cast<uint32_t>(g.nu) * UB;
      const uint32_t n0 = static_cast<uint32_t>(g.n[0]) * UB;
      __syncwarp();  // after the leader's expect_tx
      for (int c = lane; c < m * g.np; c += 32) {
        const int j = g.np > 1 ? c >> 1 : c;
        if (g.np == 1 || (c & 1) == 0)
          bulk_g2s(ring + e + j * ab, pb[0] + static_cast<size_t>(t0 + j) * TILE + g.pa[0] * UB, n0, bar, pol);
        else
          bulk_g2s(ring + e + j * ab + n0, pb[1] + static_cast<size_t>(t0 + j) * TILE,
                   static_cast<uint32_t>(g.n[1]) * UB, bar, pol);
      }
    };
    GroupIt it{u0, u1, upe, gmax, a.tail_absorb};
    Grp cur, prev;
    bool more = it.next(cur), has_prev = false;
    const uint8_t* cb[2];
    const uint8_t* pbs[2];
    piece_bases(cur, cb);
    while (more || has_prev) {
      if (more) {  // GU(i)
        const Geom g = gu_geom(cur.nu, kcap);
        for (int kt = 0; kt < ktiles; kt += g.m) {
          const uint32_t e = reserve(g);
          uint64_t* bar = &full[idx % NSLOT];
          if (leader) mbar_arrive_expect_tx(bar, g.size);
          copy_entry(cur, cb, kt, g.m, e, bar);
          ++idx;
        }
      }
      if (has_prev) {  // DN(i-1)
        const Geom g = dn_geom(prev.nu, mcap);
        for (int mt = 0; mt < mtiles; mt += g.m) {
          const uint32_t e = reserve(g);
          uint64_t* bar = &full[idx % NSLOT];
          if (leader) mbar_arrive_expect_tx(bar, g.size);
          copy_entry(prev, pbs, ktiles + mt, g.m, e, bar);
          ++idx;
          if (mt == 0 && !more && leader) stamp(a, 11);  // last round's DN: first entry issued
        }
      }
      has_prev = more;
      if (more) {
        prev = cur;
        pbs[0] = cb[0];
        pbs[1] = cb[1];
        more = it.next(cur);
        if (more) piece_bases(cur, cb);
      }
    }
    if (leader) stamp(a, 15);  // last weight copy issued
    if (a.nx_counters && a.pf_bytes > 0) {
      // ---- cross-layer L2 prefetch: the next layer's routing is final (K2
      // ran for all layers), so walk what this CTA index streams next layer
      // and prefetch its runs into L2 (HBM otherwise idles through this
      // launch's tail and the layer handoff); the next CTA fills its ring
      // with the first ring_bytes itself right after entry
      const k3s::StreamSrc nx{a.nx_counters, a.nx_hit_list, a.nx_slot_of, a.nx_pool, a.nx_shared_w,
                              a.n_shared,    a.expert_elems, d,            a.ffn};
      k3s::prefetch_stream_l2(nx, bg, G, gmax, RB, a.pf_bytes, lane);
    }
    if (!waited) wait_pred();
    if (a.dbg && leader) a.dbg[blockIdx.x * DBG + 8] = static_cast<unsigned long long>(w_empty);
  } else {
    // TMEM allocation (MMA warp) and routing staging (epilogue warps) run
    // while the producer's first copies are in flight.
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&misc[1])),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      // entry r (= o_first + r): per-token gate (0 for tokens not routed to
      // it) and the token mask; one warp per entry, one lane per routed slot
      const int ew = warp - 2;
      {  // a^T columns of tokens >= T stay zero for the whole launch; so does the zero buffer
        uint4* z = reinterpret_cast<uint4*>(aT);
        for (int i = tid - 64; i < 2 * 2 * 4096 / 16; i += EPI_THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
        uint4* zz = reinterpret_cast<uint4*>(zeros);
        for (int i = tid - 64; i < UB / 16; i += EPI_THREADS) zz[i] = make_uint4(0u, 0u, 0u, 0u);
      }
      for (int r = ew; r < n_ent; r += 4) {
        const int o = o_first + r;
        if (lane < 16) ent_gate[r * 16 + lane] = 0.f;
        __syncwarp();
        uint32_t bit = 0;
        if (o < n_hits) {
          const int e = a.hit_list[o];
          const int p0 = a.offsets[e];
          const int nt = a.offsets[e + 1] - p0;
          if (lane < nt) {
            const int ix = a.perm[p0 + lane];
            const int t = ix / a.k;
            ent_gate[r * 16 + t] = a.gates[ix];
            bit = 1u << t;
          }
        } else if (lane < T) {
          ent_gate[r * 16 + lane] = 1.f;
          bit = 1u << lane;
        }
        bit = __reduce_or_sync(0xffffffffu, bit);
        if (lane == 0) ent_mask[r] = bit;
        __syncwarp();
      }
    }
    fence_before();
    named_bar_sync(1, 32 + EPI_THREADS);
    fence_after();
    const uint32_t tmem = static_cast<uint32_t>(misc[1]);

    if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      // whole warp in convergent flow (warp-uniform descriptors); one elected
      // lane issues the MMAs and commits
      const bool leader = elect_one();
      long long w_full = 0, w_at = 0, w_d1e = 0;
      Phase d1e[2], ate[2];
      uint32_t head = 0, idx = 0;
      int ht_ok = 0;  // h^T slices [0, ht_ok) known to have landed
      const uint32_t ring_addr = smem_u32(ring), at_addr = smem_u32(aT), ht_addr = smem_u32(hts);
      const uint32_t zero_addr = smem_u32(zeros);
      GroupIt it{u0, u1, upe, gmax, a.tail_absorb};
      Grp cur, prev;
      bool more = it.next(cur), has_prev = false;
      int i = 0;
      while (more || has_prev) {
        if (more) {  // GU(i): D1[i & 1] = W_gu(group) x h^T, one or two M = 128 tiles
          const int b1 = i & 1;
          wait_acc(a, &d1_empty[b1], d1e[b1].bit ^ 1u, w_d1e);
          d1e[b1].flip();
          fence_after();
          const uint32_t d1 = tmem + static_cast<uint32_t>(b1 * 32);
          const int nt = (cur.nu + 7) / 8;
          const Geom g = gu_geom(cur.nu, kcap);
          const uint32_t ab = static_cast<uint32_t>(cur.nu) * UB;
          for (int kt = 0; kt < ktiles; kt += g.m) {
            const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
            wait_acc(a, &full[slot], (idx / NSLOT) & 1u, w_full);
            ++idx;
            for (; ht_ok < kt + g.m; ++ht_ok) mbar_wait(&ht_full[ht_ok], 0);
            if (i == 0 && kt == 0 && leader) stamp(a, 2);
            fence_after();
            if (leader) {
              for (int j = 0; j < g.m; ++j) {
                const uint64_t bdesc = smem_desc(ht_addr + (kt + j) * hsz, 128, 1024);
                for (int t = 0; t < nt; ++t) {
                  const uint64_t adesc = smem_desc(ring_addr + off + j * ab + t * TILE, 128, 1024);
#pragma unroll
                  for (int k = 0; k < 4; ++k)  // +256 B per K=16 step = +16 in the start-address field
                    tc::mma_bf16_id(d1 + 16 * t, adesc + 16 * k, bdesc + 16 * k, (kt | j | k) != 0, idesc);
                }
              }
              mma_commit(&empty[slot]);
            }
            __syncwarp();
          }
          if (leader) mma_commit(&d1_full[b1]);
          __syncwarp();
          if (i == 0 && leader) stamp(a, 3);
          if (i == 1 && leader) stamp(a, 5);  // GU(1) issued
        }
        if (has_prev) {  // DN(i-1): D2 += W_down(group) x a^T(i-1), hi + lo
          const int ab_ = (i - 1) & 1;
          wait_acc(a, &at_full[ab_], ate[ab_].bit, w_at);
          ate[ab_].flip();
          fence_after();
          const uint32_t ahi = at_addr + static_cast<uint32_t>(ab_) * 8192u;
          const uint64_t bhi = smem_desc(ahi, 256, 128), blo = smem_desc(ahi + 4096u, 256, 128);
          const Geom g = dn_geom(prev.nu, mcap);
          const uint32_t ab = static_cast<uint32_t>(prev.nu) * UB;
          const bool last = !more;  // D2 M-tiles are final as this pass's entries complete
          for (int mt = 0; mt < mtiles; mt += g.m) {
            const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
            wait_acc(a, &full[slot], (idx / NSLOT) & 1u, w_full);
            ++idx;
            fence_after();
            if (leader) {
              for (int j = 0; j < g.m; ++j) {
                const uint32_t d2 = tmem + D2_COL0 + static_cast<uint32_t>((mt + j) * d2w);
                // K-step s2 = units 2 s2, 2 s2 + 1 (two 8-k core-matrix columns,
                // LBO apart); an odd group's last step takes its second
                // column from the zero buffer (a^T rows there are 0 too)
                for (int s2 = 0; 2 * s2 < prev.nu; ++s2) {
                  const uint32_t run = ring_addr + off + j * ab + 2 * s2 * UB;
                  const uint32_t lbo = 2 * s2 + 1 < prev.nu ? UB : zero_addr - run;
                  const uint64_t adn = smem_desc(run, lbo, 128);
                  tc::mma_bf16_id(d2, adn, bhi + 32 * s2, (i == 1 && s2 == 0) ? 0u : 1u, idesc);  // +512 B of a^T per step
                  tc::mma_bf16_id(d2, adn, blo + 32 * s2, 1u, idesc);
                }
              }
              mma_commit(&empty[slot]);
              if (last) mma_commit(&d2e[mt / g.m]);
            }
            __syncwarp();
          }
          if (leader) mma_commit(&at_empty[ab_]);
          __syncwarp();
        }
        has_prev = more;
        if (more) {
          prev = cur;
          more = it.next(cur);
        }
        ++i;
      }
      if (a.dbg && leader) {
        a.dbg[blockIdx.x * DBG + 9] = static_cast<unsigned long long>(w_full);
        a.dbg[blockIdx.x * DBG + 10] = static_cast<unsigned long long>(w_at);
        a.dbg[blockIdx.x * DBG + 12] = static_cast<unsigned long long>(w_d1e);
      }
      named_bar_sync(3, EPI_THREADS + 32);  // the epilogue has drained D2
      fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
      if (lane == 0) stamp(a, 23);
    } else {
      // ------------------------------------------------ epilogue (4 warps)
      pdl_wait();  // partial blocks are still being read by the previous combine
      const int q = warp & 3;   // TMEM lane quarter = group slot
      const int et = tid - 64;  // 0..127
      if (a.shared_gate_w && o_first + n_ent - 1 >= n_hits) {
        // ---- sigmoid shared-expert gate (Qwen1.5-MoE): g_t = sigmoid(w_sg . h_t)
        // from the resident h^T slices, one fixed order for every CTA (thread
        // et: 8-k chunks et, et + 128, ...; xor butterfly; warps in order);
        // it replaces the weight-1 gates the staging gave the shared entries
        for (int kt = 0; kt < ktiles; ++kt) mbar_wait(&ht_full[kt], 0);
        float acc[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) acc[t] = 0.f;
        const uint16_t* ht16 = reinterpret_cast<const uint16_t*>(hts);
        for (int c8 = et; c8 < d / 8; c8 += EPI_THREADS) {
          const int kt = c8 >> 3, j = c8 & 7;
          const uint4 wv = *reinterpret_cast<const uint4*>(a.shared_gate_w + static_cast<size_t>(c8) * 8);
          float w8[8];
          bf16x8_to_f32(wv, w8);
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            if (t < T) {
              const uint4 hv = *reinterpret_cast<const uint4*>(ht16 + kt * (hsz / 2) + (t >> 3) * 512 + j * 64 + (t & 7) * 8);
              float h8[8];
              bf16x8_to_f32(hv, h8);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[t] = fmaf(w8[e], h8[e], acc[t]);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
        }
        if (lane == 0) {
#pragma unroll
          for (int t = 0; t < 16; ++t) sg_part[q * 16 + t] = acc[t];
        }
        named_bar_sync(2, EPI_THREADS);
        const float z = lane < T ? ((sg_part[lane] + sg_part[16 + lane]) + sg_part[32 + lane]) + sg_part[48 + lane] : 0.f;
        const float sg = lane < T ? 1.f / (1.f + expf(-z)) : 0.f;
        for (int r = warp - 2; r < n_ent; r += 4)
          if (o_first + r >= n_hits && lane < 16) ent_gate[r * 16 + lane] = sg;
        named_bar_sync(2, EPI_THREADS);
      }
      Phase d1f[2], atf[2];
      long long w_d1f = 0, w_d2f = 0;
      GroupIt it{u0, u1, upe, gmax, a.tail_absorb};
      Grp g;
      int i = 0;
      while (it.next(g)) {
        // ---- A(i): D1 -> a^T (bf16 hi/lo) for DN(i)
        const int b1 = i & 1;
        wait_acc(a, &d1_full[b1], d1f[b1].bit, w_d1f);
        d1f[b1].flip();
        if (i == 0 && et == 0) stamp(a, 17);
        fence_after();
        const int nt = (g.nu + 7) / 8;
        float v[2][16];
        tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(b1 * 32), v[0]);
        if (nt > 1) tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(b1 * 32 + 16), v[1]);
        if (i == 0 && et == 0 && a.dbg) {  // after the TMEM data is in registers
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt) : "f"(v[0][0]), "f"(v[0][15]) : "memory");
          a.dbg[blockIdx.x * DBG + 25] = tt;
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d1_empty[b1]);
        const int ab = i & 1;
        mbar_wait(&at_empty[ab], atf[ab].bit ^ 1u);  // DN(i-2) done with this buffer
        atf[ab].flip();
        if (i == 0 && et == 0) stamp(a, 16);
        uint16_t* hi = reinterpret_cast<uint16_t*>(aT + static_cast<size_t>(ab) * 8192);
        uint16_t* lo = hi + 2048;
        const int up = (lane >> 3) & 1;
#pragma unroll
        for (int t16 = 0; t16 < 2; ++t16) {
          if (t16 >= nt) break;
          // this warp's TMEM lanes of tile t16 are group slots 8 t16 + 2q
          // (lanes 0-15) and 8 t16 + 2q + 1 (lanes 16-31); in a slot, lanes
          // 0-7 hold the gate rows of f = 8 slot + (lane & 7), lanes 8-15
          // the up rows of the same f. Slots past the group's last unit get
          // a = 0 (an odd group's last down K-step reads them).
          const int slot = 8 * t16 + 2 * q + (lane >> 4);
          const bool valid = slot < g.nu;
          const float* gs = ent_gate + (valid ? static_cast<int>((g.us + slot) / upe) - o_first : 0) * 16;
          const int f = 8 * slot + (lane & 7);
          float gts[16];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 x = reinterpret_cast<const float4*>(gs)[j];
            gts[4 * j] = x.x;
            gts[4 * j + 1] = x.y;
            gts[4 * j + 2] = x.z;
            gts[4 * j + 3] = x.w;
          }
          // gate lanes take the even tokens, up lanes the odd ones: token
          // t = 2j + up, its partner value crosses with one xor-8 shuffle.
          // Branch-free (tokens >= T and unrouted entries select 0) so the
          // eight independent chains interleave.
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int t = 2 * j + up;
            const float pv = __shfl_xor_sync(0xffffffffu, up ? v[t16][2 * j] : v[t16][2 * j + 1], 8);
            const float gv = up ? pv : v[t16][2 * j];
            const float uv = up ? v[t16][2 * j + 1] : pv;
            const float gt = up ? gts[2 * j + 1] : gts[2 * j];
            const float sv = __fdividef(gv, 1.f + __expf(-gv)) * uv * gt;
            const float av = (valid && t < T && gt != 0.f) ? sv : 0.f;
            const uint16_t h16 = f32_to_bf16_cvt(av);
            const float rem = av - __uint_as_float(static_cast<uint32_t>(h16) << 16);
            // byte = j*256 + tg*128 + r*16 + e*2 (token = 8 tg + r, f = 8 j + e)
            const int off = (f >> 3) * 128 + (t >> 3) * 64 + (t & 7) * 8 + (f & 7);
            hi[off] = h16;
            lo[off] = f32_to_bf16_cvt(rem);
          }
        }
        if (i == 0 && et == 0) stamp(a, 21);
        fence_proxy_async();
        named_bar_sync(2, EPI_THREADS);
        if (et == 0) {
          mbar_arrive(&at_full[ab]);
          if (i == 0) stamp(a, 4);
        }
        ++i;
      }
      // ---- drain, overlapped with the last DN pass: D2 M-tiles [mt, mt + nm)
      // are final once the pass's entry holding M-tile mt + nm - 1 has
      // completed (the MMA warp commits each of that pass's entries to its own
      // mbarrier), so while the pass's later entries still stream, chunks of
      // sc M-tiles are read from TMEM, staged [T][nm * 128] fp32 in the h^T
      // slices (dead once the last gate|up MMAs are done: every DN MMA is
      // issued after them, two buffers) and stored, one bulk copy per touched
      // token row. A pass of one entry (a short last group) — or two buffers
      // not fitting in the h^T slices — drains after the whole pass instead:
      // all M-tiles staged in the idle ring, one d * 4-byte copy per row.
      uint32_t tmask = 0;  // tokens this CTA touched
      for (int r = 0; r < n_ent; ++r) tmask |= ent_mask[r];
      const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(D2_COL0);
      const Geom gl = dn_geom(g.nu, mcap);  // g: the last group (GroupIt leaves it)
      const int n_last = (mtiles + gl.m - 1) / gl.m;
      const uint32_t hts_bytes = static_cast<uint32_t>(ktiles) * hsz;
      int sc = a.drain_sc > 0 ? a.drain_sc : 4;
      while (sc > 1 && 2u * sc * 512u * static_cast<uint32_t>(T) > hts_bytes) sc >>= 1;
      const bool early = !a.drain_late && n_last > 1 && 2u * sc * 512u * static_cast<uint32_t>(T) <= hts_bytes;
      if (!early) sc = mtiles;
      float* stg0 = reinterpret_cast<float*>(early ? hts : ring);
      const bool issuer = q == 0 && lane < T;  // one lane per token row
      int c = 0;
      for (int mt = 0; mt < mtiles; mt += sc, ++c) {
        const int nm = mtiles - mt < sc ? mtiles - mt : sc;
        wait_acc(a, &d2e[early ? (mt + nm - 1) / gl.m : n_last - 1], 0, w_d2f);
        if (mt == 0 && et == 0) stamp(a, 18);
        fence_after();
        // buffer c & 1 was last read by chunk c - 2's stores
        if (c >= 2 && issuer) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (c >= 2) named_bar_sync(2, EPI_THREADS);
        float* s = stg0 + static_cast<size_t>(c & 1) * sc * 128 * T;
        // four M-tiles per tcgen05.wait::ld (the loads are latency bound)
        for (int m4 = 0; m4 < nm; m4 += 4) {
          const int n4 = nm - m4 < 4 ? nm - m4 : 4;
          uint32_t y[4][16];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < n4) {
              if (T <= 8)
                tc::tmem_ld8_nw(tbase + static_cast<uint32_t>((mt + m4 + j) * d2w), y[j]);
              else
                tc::tmem_ld16_nw(tbase + static_cast<uint32_t>((mt + m4 + j) * d2w), y[j]);
            }
          tc::tmem_wait_ld();
          float* r0 = s + 128 * m4 + 32 * q + lane;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (j < n4) {
#pragma unroll
              for (int t = 0; t < 16; ++t)
                if (t < T) r0[static_cast<size_t>(t) * nm * 128 + 128 * j] = __uint_as_float(y[j][t]);
            }
        }
        fence_proxy_async();
        if (mt + nm >= mtiles) {
          if (et == 0) stamp(a, 1);
          // TMEM is dead past this barrier: warp 1 (also arriving) deallocates
          // it while the last rows are stored
          fence_before();
          named_bar_sync(3, EPI_THREADS + 32);
        }
        named_bar_sync(2, EPI_THREADS);
        if (issuer) {
          if ((tmask >> lane) & 1u)
            bulk_s2g(a.partial + (static_cast<long long>(b) * T + lane) * d + mt * 128,
                     s + static_cast<size_t>(lane) * nm * 128, static_cast<uint32_t>(nm) * 512u);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      if (et == 0) stamp(a, 19);
      // (the source reads only: kernel completion makes the writes visible to
      // the dependent combine)
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (et == 0) stamp(a, 20);
      if (a.dbg && tid == 64) {
        a.dbg[blockIdx.x * DBG + 13] = static_cast<unsigned long long>(w_d1f);
        a.dbg[blockIdx.x * DBG + 14] = static_cast<unsigned long long>(w_d2f);
      }
    }
  }
  __syncwarp();  // bar.sync is warp-aligned: a warp arriving in pieces is counted once per piece
  __syncthreads();
  if (tid == 0) stamp(a, 6);
}

}  // namespace tg
}  // namespace dev

size_t ffn_tg_smem_bytes(int T, int d, int ring_bytes) {
  const size_t hsz = ffn_tg_n8(d, T) ? 1024 : dev::tg::HTS;  // (N = 8 mode keeps 8 token rows of h^T)
  return 2 * 2 * 4096 + static_cast<size_t>(d / 64) * hsz + static_cast<size_t>(ring_bytes) + dev::tg::UB +
         dev::tg::ENT_MAX * (16 * 4 + 4) + 16 + 4 * 16 * 4 + 8 +
         8 * (2 * dev::tg::NSLOT + 8 + dev::tg::D2E + dev::tg::MAX_KT);
}

// Every CTA's range must touch <= ENT_MAX entries (one producer lane each).
bool ffn_tg_grid_ok(int n_entries, int d_ffn, int grid) {
  const long long upe = d_ffn / 8, n = static_cast<long long>(n_entries) * upe;
  const long long maxu = (n + grid - 1) / grid;
  return grid > 0 && (maxu > 0 ? (maxu - 1) / upe + 2 : 1) <= dev::tg::ENT_MAX;
}

// Grouped mode: d <= 2048 (D2 for all d/128 M-tiles fits in TMEM columns
// 256-511), the drain's [T][d] fp32 staging fits in the ring, and the ring
// holds the widest entry window (58 KiB: 3 or 7 units x 8 or 4 tiles, the
// last tile read as a full 16 KiB A operand).
int ffn_tg_ring_bytes(int T, int d, size_t smem_limit) {
  // D2 (all d/128 M-tiles) in TMEM columns 256-511: 16 columns per M-tile
  // (d <= 2048), or 8 in N = 8 mode (d <= 4096, T <= 8)
  if (d % 128 || T > 16 || d > 4096 || (d > 2048 && T > 8)) return 0;
  const size_t fixed = ffn_tg_smem_bytes(T, d, 0);
  if (fixed >= smem_limit) return 0;
  const int rb = static_cast<int>(((smem_limit - fixed) / 1024) * 1024);
  const int need = static_cast<int>(T) * d * 4 > 59392 ? T * d * 4 : 59392;
  return rb >= need ? rb : 0;
}

cudaError_t launch_expert_ffn_tg(const dev::FfnArgs& a, int grid, size_t smem, cudaStream_t stream, bool pdl) {
  if (const cudaError_t e = smem_optin_once<dev::tg::expert_ffn_tg_kernel>(232448); e != cudaSuccess) return e;
  dev::FfnArgs b = a;
  b.tg_n8 = ffn_tg_n8(a.d, a.T) ? 1 : 0;  // (the same rule sized its shared memory)
  return launch_pdl(dev::tg::expert_ffn_tg_kernel, dim3(grid), dim3(dev::tg::THREADS), smem, stream, pdl, b);
}

}  // namespace moespac
