// K3 persistent (grouped tensor-core variant, d <= 2048, all layers in one
// launch): the grouped K3 of expert_ffn_grouped.cu with the layer loop and
// the combine moved inside the kernel.
//
// Per layer the separate kernels cost a K3 grid completion, a combine
// kernel, a second grid completion and the next K3's prologue (~6 us of a
// ~34 us Qwen3 layer) during which HBM mostly idles. Here the
// 148 CTAs (one per SM, all co-resident) stay up for the whole step:
//
//   * the producer streams its work of layer l+1 into the byte ring as soon
//     as it has issued layer l's — only the h^T slices of layer l+1 wait for
//     the layer handoff;
//   * the epilogue drains the CTA's D2 accumulator to its partial block,
//     arrives on grid barrier 1, sums its slice of the layer output over the
//     partial blocks (fixed order: the token's covering CTAs ascending,
//     dealt to 4 threads per output, reduced 0..3), writes h_{l+1}, the
//     h^T image of layer l+1 and y_l, and arrives on grid barrier 2; the
//     producer polls barrier 2 between ring waits and then loads h^T.
//
// Grid barriers are monotonic counters in global memory (release/acquire,
// zeroed by the host before the launch); every CTA arrives once per layer
// whether or not it has work in that layer. A spin that does not complete
// within ~4 s traps instead of hanging the device.
//
// Same image layout (v3), work units, groups, byte ring, SwiGLU epilogue and
// D2 accumulator as the grouped kernel; see that file's header.
#include <cstdint>

#include "common.cuh"
#include "launch.hpp"
#include "tcgen05.cuh"

namespace moespac {
namespace dev {
namespace tp {

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
constexpr int NSLOT = 32;
constexpr int TILE = 16384;
constexpr int UB = 2048;
constexpr int UPC = 8;
constexpr int GMAX = 8;
constexpr int HTS = 2048;
constexpr int ENT_MAX = 32;
constexpr int MAX_KT = 32;
constexpr int D2_COL0 = 256;
constexpr int TMEM_COLS = 512;
constexpr int ROWMAX = 256;  // partial rows of one token (<= grid)
constexpr int DBG = 32;

struct Grp {
  long long us;
  int nu, np;
  int o[2], c[2], pa[2], n[2];
};

struct GroupIt {
  long long u, u1;
  int upe;
  __device__ __forceinline__ bool next(Grp& g) {
    if (u >= u1) return false;
    const long long ue = u + GMAX < u1 ? u + GMAX : u1;
    g.us = u;
    g.nu = static_cast<int>(ue - u);
    const int o = static_cast<int>(u / upe), ui = static_cast<int>(u % upe);
    const long long cend = static_cast<long long>(o) * upe + (ui / UPC + 1) * UPC;
    const long long e = cend < ue ? cend : ue;
    g.o[0] = o;
    g.c[0] = ui / UPC;
    g.pa[0] = ui % UPC;
    g.n[0] = static_cast<int>(e - u);
    g.np = e < ue ? 2 : 1;
    g.o[1] = static_cast<int>(e / upe);
    g.c[1] = static_cast<int>(e % upe) / UPC;
    g.pa[1] = 0;
    g.n[1] = static_cast<int>(ue - e);
    u = ue;
    return true;
  }
};

__device__ __forceinline__ int pow2_divisor(int x, int cap) {
  int m = 1;
  while (m < cap && x % (2 * m) == 0) m *= 2;
  return m;
}
__device__ __forceinline__ int tiles_per_entry(int nu, int cap) {
  const int t = nu >= 8 ? 2 : (nu >= 4 ? 4 : 8);
  return t < cap ? t : cap;
}
struct Geom {
  uint32_t size, win;
  int m;
};
__device__ __forceinline__ Geom gu_geom(int nu, int cap) {
  const int m = tiles_per_entry(nu, cap);
  const uint32_t a = static_cast<uint32_t>(nu) * UB;
  const uint32_t size = static_cast<uint32_t>(m) * a;
  const uint32_t w = static_cast<uint32_t>(m - 1) * a + TILE;
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

__device__ __forceinline__ void stamp(const PersistArgs& a, int layer, int slot) {
  if (a.dbg) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    a.dbg[(static_cast<size_t>(layer) * gridDim.x + blockIdx.x) * DBG + slot] = t;
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void spin_until(const unsigned* p, unsigned target) {
  const long long t0 = clock64();
  while (static_cast<int>(ld_acquire(p) - target) < 0) {
    __nanosleep(20);
    if (clock64() - t0 > (1ll << 33)) __trap();  // ~4 s: fail loudly instead of hanging
  }
}

// per-layer view of the step's routing tables
struct LayerView {
  int n_hits;
  long long n;  // work units
  long long u0, u1;
  int o_first, n_ent;
};
__device__ __forceinline__ LayerView layer_view(const PersistArgs& a, int l, int upe) {
  LayerView v;
  v.n_hits = a.counters[l * 8 + 7];
  v.n = static_cast<long long>(v.n_hits + a.n_shared) * upe;
  const int G = gridDim.x, b = blockIdx.x;
  v.u0 = v.n > 0 ? (b * v.n) / G : 0;
  v.u1 = v.n > 0 ? ((b + 1) * v.n) / G : 0;
  v.o_first = v.u0 < v.u1 ? static_cast<int>(v.u0 / upe) : 0;
  v.n_ent = v.u0 < v.u1 ? static_cast<int>((v.u1 - 1) / upe) - v.o_first + 1 : 0;
  return v;
}

// routing of layer l into staging slot l & 1: per entry of the CTA's range
// the per-token gate (0 if not routed) and token mask; entries r0, r0 + step, ...
__device__ __forceinline__ void stage_layer(const PersistArgs& a, int l, int upe, float* ent_gate, uint32_t* ent_mask,
                                            int r0, int step, int lane) {
  const LayerView v = layer_view(a, l, upe);
  const int N = a.N, T = a.T, k = a.k;
  float* eg = ent_gate + (l & 1) * ENT_MAX * 16;
  uint32_t* em = ent_mask + (l & 1) * ENT_MAX;
  const int32_t* hit_l = a.hit_list + static_cast<size_t>(l) * N;
  const int32_t* off_l = a.offsets + static_cast<size_t>(l) * (N + 1);
  const int32_t* perm_l = a.perm + static_cast<size_t>(l) * T * k;
  const float* gates_l = a.gates + static_cast<size_t>(l) * T * k;
  for (int r = r0; r < v.n_ent; r += step) {
    const int o = v.o_first + r;
    if (lane < 16) eg[r * 16 + lane] = 0.f;
    __syncwarp();
    uint32_t bit = 0;
    if (o < v.n_hits) {
      const int e = hit_l[o];
      const int p0 = off_l[e];
      const int nt = off_l[e + 1] - p0;
      if (lane < nt) {
        const int ix = perm_l[p0 + lane];
        const int t = ix / k;
        eg[r * 16 + t] = gates_l[ix];
        bit = 1u << t;
      }
    } else if (lane < T) {
      eg[r * 16 + lane] = 1.f;
      bit = 1u << lane;
    }
    bit = __reduce_or_sync(0xffffffffu, bit);
    if (lane == 0) em[r] = bit;
    __syncwarp();
  }
}

// partial rows of token t in layer l: the CTAs covering any of its entries,
// ascending (entries ascend, so their CTA ranges do too)
__device__ __forceinline__ int row_list(const PersistArgs& a, int l, int t, int upe, int* out) {
  const LayerView v = layer_view(a, l, upe);
  const int G = gridDim.x, k = a.k;
  const int32_t* ids_l = a.ids + (static_cast<size_t>(l) * a.T + t) * k;
  const int32_t* ord_l = a.hit_ord + static_cast<size_t>(l) * a.N;
  const int n = static_cast<int>(v.n);  // n * (grid + 1) < 2^31 (host plan)
  const bool all_busy = n >= G;         // no CTA with an empty range
  int nr = 0, last = -1;
  auto add = [&](int o) {
    const int lo = ((o * upe + 1) * G - 1) / n;
    const int hi = (((o + 1) * upe) * G - 1) / n;
    for (int c = lo > last + 1 ? lo : last + 1; c <= hi; ++c) {
      if (!all_busy && (c * n) / G == ((c + 1) * n) / G) continue;
      last = c;
      if (nr < ROWMAX) out[nr] = c;
      ++nr;
    }
  };
  if (v.n > 0) {
    for (int j = 0; j < k; ++j) {
      const int o = ord_l[ids_l[j]];
      if (o >= 0) add(o);
    }
    for (int s = 0; s < a.n_shared; ++s) add(v.n_hits + s);
  }
  return nr;
}

__device__ __forceinline__ void named_bar_arrive(int id, int threads) {
  __syncwarp();
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__global__ void __maxnreg__(200) expert_ffn_persistent_kernel(PersistArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const int d = a.d, T = a.T, L = a.L, N = a.N, k = a.k;
  const int ktiles = d / 64, mtiles = d / 128;
  const long long chunk_bytes = 3LL * 64 * d * 2;
  const int upe = a.ffn / 8;
  const uint32_t RB = static_cast<uint32_t>(a.ring_bytes);
  const int G = gridDim.x, b = blockIdx.x;

  // [a^T 16 KiB][h^T][ring][zeros][entry gates x2][entry masks x2][rows 2 x ROWMAX][misc][mbarriers]
  uint8_t* p = smem_raw;
  uint8_t* aT = p;
  p += 2 * 2 * 4096;
  uint8_t* hts = p;
  p += static_cast<size_t>(ktiles) * HTS;
  uint8_t* ring = p;
  p += RB;
  uint8_t* zeros = p;
  p += UB;
  float* ent_gate = reinterpret_cast<float*>(p);  // [2][ENT_MAX][16] (layer parity)
  p += 2 * ENT_MAX * 16 * 4;
  uint32_t* ent_mask = reinterpret_cast<uint32_t*>(p);  // [2][ENT_MAX]
  p += 2 * ENT_MAX * 4;
  int* rows = reinterpret_cast<int*>(p);  // [2][ROWMAX] partial rows of the slice's tokens
  p += 2 * ROWMAX * 4;
  int* misc = reinterpret_cast<int*>(p);  // [1] TMEM base, [2..3] row counts, [4..5] slice tokens
  p += 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(p) + 7) & ~uintptr_t(7));
  uint64_t* full = bars;
  uint64_t* empty = full + NSLOT;
  uint64_t* d1_full = empty + NSLOT;  // [2]
  uint64_t* d1_empty = d1_full + 2;   // [2]
  uint64_t* at_full = d1_empty + 2;   // [2]
  uint64_t* at_empty = at_full + 2;   // [2]
  uint64_t* d2_full = at_empty + 2;   // [1]
  uint64_t* d2_empty = d2_full + 1;   // [1] (4 epilogue warps)
  uint64_t* ht_free = d2_empty + 1;   // [1] last gate|up MMA of a layer done
  uint64_t* ht_full = ht_free + 1;    // [ktiles]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
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
    mbar_init(d2_full, 1);
    mbar_init(d2_empty, 4);
    mbar_init(ht_free, 1);
    for (int i = 0; i < ktiles; ++i) mbar_init(&ht_full[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  __syncthreads();

  const int kcap = pow2_divisor(ktiles, 8), mcap = pow2_divisor(mtiles, 8);
  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    const bool leader = elect_one();
    const uint64_t pol = l2_evict_first_policy();
    const uint64_t pol_h = l2_evict_normal_policy();
    uint32_t head = 0, idx = 0, tail = 0;
    uint32_t my_off = 0, my_size = 0, my_idx = 0xFFFFFFFFu;
    int processed = 0;          // layers with work in this CTA whose h^T was loaded
    int ht_layer = -1;          // layer whose h^T load is pending (-1: none)
    auto try_ht = [&](bool block) {
      // h^T of layer ht_layer: needs barrier 2 of the previous layer (all
      // CTAs wrote their slice of it) and the CTA's previous h^T consumer done
      if (ht_layer < 0) return;
      const int l = ht_layer;
      for (;;) {
        int ok = 1;
        if (lane == 0) {
          if (l > 0 && static_cast<int>(ld_acquire(a.sync + 1) - static_cast<unsigned>(l * G)) < 0) ok = 0;
          if (ok && processed > 0 && !mbar_try_wait(ht_free, static_cast<uint32_t>(processed - 1) & 1u)) ok = 0;
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (ok) break;
        if (!block) return;
        __nanosleep(20);
      }
      asm volatile("fence.proxy.async;" ::: "memory");  // generic writes (other CTAs' combine) -> TMA reads
      if (leader) {
        const uint8_t* hTb = reinterpret_cast<const uint8_t*>(a.hT + static_cast<size_t>(l & 1) * 16 * d);
        for (int kt = 0; kt < ktiles; ++kt) {
          mbar_arrive_expect_tx(&ht_full[kt], HTS);
          bulk_g2s(hts + kt * HTS, hTb + static_cast<size_t>(kt) * HTS, HTS, &ht_full[kt], pol_h);
        }
      }
      __syncwarp();
      if (lane == 0) stamp(a, l, 5);
      ++processed;
      ht_layer = -1;
    };
    auto reserve = [&](const Geom& g) -> uint32_t {
      uint32_t e = head;
      if (e + g.win > RB) e = 0;
      for (;;) {
        const bool mine = my_idx != 0xFFFFFFFFu && my_idx >= tail && my_off < e + g.size && e < my_off + my_size;
        const bool over = idx - tail >= static_cast<uint32_t>(NSLOT) || __any_sync(0xffffffffu, mine);
        if (!over) break;
        // wait for the oldest entry, polling the pending h^T load meanwhile
        const uint32_t par = (tail / NSLOT) & 1u;
        for (;;) {
          int done = lane == 0 ? static_cast<int>(mbar_try_wait(&empty[tail % NSLOT], par)) : 0;
          done = __shfl_sync(0xffffffffu, done, 0);
          if (done) break;
          try_ht(false);
        }
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
    for (int l = 0; l < L; ++l) {
      const LayerView v = layer_view(a, l, upe);
      if (v.u0 >= v.u1) continue;
      try_ht(true);  // a previous layer's h^T still pending: its MMAs come first in the stream
      ht_layer = l;
      if (v.n_ent > ENT_MAX) __trap();
      const uint16_t* pool_l = a.pool + static_cast<long long>(l) * a.pool_layer_elems;
      const uint16_t* shared_l = a.shared_w + static_cast<long long>(l) * a.n_shared * a.expert_elems;
      const int32_t* slot_l = a.slot_of + static_cast<size_t>(l) * N;
      const int32_t* hit_l = a.hit_list + static_cast<size_t>(l) * N;
      unsigned long long my_base = 0;
      if (lane < v.n_ent) {
        const int o = v.o_first + lane;
        const uint16_t* w = o < v.n_hits ? pool_l + static_cast<long long>(slot_l[hit_l[o]]) * a.expert_elems
                                         : shared_l + static_cast<long long>(o - v.n_hits) * a.expert_elems;
        my_base = reinterpret_cast<unsigned long long>(w);
      }
      auto piece_bases = [&](const Grp& g, const uint8_t* (&pb)[2]) {
        const unsigned long long b0 = __shfl_sync(0xffffffffu, my_base, g.o[0] - v.o_first);
        const unsigned long long b1 = __shfl_sync(0xffffffffu, my_base, g.np > 1 ? g.o[1] - v.o_first : 0);
        pb[0] = reinterpret_cast<const uint8_t*>(b0) + static_cast<long long>(g.c[0]) * chunk_bytes;
        pb[1] = reinterpret_cast<const uint8_t*>(b1) + static_cast<long long>(g.np > 1 ? g.c[1] : 0) * chunk_bytes;
      };
      auto copy_entry = [&](const Grp& g, const uint8_t* const (&pb)[2], int t0, int m, uint32_t e, uint64_t* bar) {
        if (!leader) return;
        const uint32_t ab = static_cast<uint32_t>(g.nu) * UB;
        const uint32_t n0 = static_cast<uint32_t>(g.n[0]) * UB;
        for (int j = 0; j < m; ++j) {
          bulk_g2s(ring + e + j * ab, pb[0] + static_cast<size_t>(t0 + j) * TILE + g.pa[0] * UB, n0, bar, pol);
          if (g.np > 1)
            bulk_g2s(ring + e + j * ab + n0, pb[1] + static_cast<size_t>(t0 + j) * TILE,
                     static_cast<uint32_t>(g.n[1]) * UB, bar, pol);
        }
      };
      if (l == 0) try_ht(true);  // layer 0's h^T was written before this launch
      GroupIt it{v.u0, v.u1, upe};
      Grp cur, prev;
      bool more = it.next(cur), has_prev = false;
      const uint8_t* cb[2];
      const uint8_t* pbs[2];
      piece_bases(cur, cb);
      while (more || has_prev) {
        if (more) {
          const Geom g = gu_geom(cur.nu, kcap);
          for (int kt = 0; kt < ktiles; kt += g.m) {
            const uint32_t e = reserve(g);
            uint64_t* bar = &full[idx % NSLOT];
            if (leader) mbar_arrive_expect_tx(bar, g.size);
            copy_entry(cur, cb, kt, g.m, e, bar);
            __syncwarp();
            ++idx;
          }
        }
        if (has_prev) {
          const Geom g = dn_geom(prev.nu, mcap);
          for (int mt = 0; mt < mtiles; mt += g.m) {
            const uint32_t e = reserve(g);
            uint64_t* bar = &full[idx % NSLOT];
            if (leader) mbar_arrive_expect_tx(bar, g.size);
            copy_entry(prev, pbs, ktiles + mt, g.m, e, bar);
            __syncwarp();
            ++idx;
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
      if (lane == 0) stamp(a, l, 6);
    }
    try_ht(true);
  } else {
    if (warp == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&misc[1])),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      uint4* z = reinterpret_cast<uint4*>(aT);
      for (int i = tid - 64; i < 2 * 2 * 4096 / 16; i += EPI_THREADS) z[i] = make_uint4(0u, 0u, 0u, 0u);
      uint4* zz = reinterpret_cast<uint4*>(zeros);
      for (int i = tid - 64; i < UB / 16; i += EPI_THREADS) zz[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_before();
    named_bar_sync(1, 32 + EPI_THREADS);
    fence_after();
    const uint32_t tmem = static_cast<uint32_t>(misc[1]);

    if (warp == 1) {
      // ------------------------------------------------ MMA issuer
      const bool leader = elect_one();
      Phase d1e[2], ate[2];
      uint32_t head = 0, idx = 0;
      int gb = 0, processed = 0;  // groups of earlier layers (D1 / a^T buffer parity), layers done
      const uint32_t ring_addr = smem_u32(ring), at_addr = smem_u32(aT), ht_addr = smem_u32(hts);
      const uint32_t zero_addr = smem_u32(zeros);
      const int Q = T * d / 4, dq = d / 4;
      const int s0 = static_cast<int>((static_cast<long long>(b) * Q) / G);
      const int s1 = static_cast<int>((static_cast<long long>(b + 1) * Q) / G);
      // between its last down projection of layer l and the h^T of layer
      // l+1 this warp is idle: it stages layer l+1's routing and the row
      // lists of layer l's combine for the epilogue
      auto side_work = [&](int l) {
        if (l > 0) named_bar_sync(4, 32 + EPI_THREADS);  // combine of layer l-1 done with rows / misc
        if (l + 1 < L) stage_layer(a, l + 1, upe, ent_gate, ent_mask, 0, 1, lane);
        if (lane < 2) {
          const int t = (lane == 0 ? s0 : s1 - 1) / dq;
          misc[4 + lane] = t;
          misc[2 + lane] = s0 < s1 ? row_list(a, l, t, upe, rows + lane * ROWMAX) : 0;
        }
        named_bar_arrive(3, 32 + EPI_THREADS);
      };
      for (int l = 0; l < L; ++l) {
        const LayerView v = layer_view(a, l, upe);
        if (v.u0 >= v.u1) {
          side_work(l);
          continue;
        }
        const uint32_t hpar = static_cast<uint32_t>(processed) & 1u;
        int ht_ok = 0, i = 0;  // i: this layer's loop step (GU(i), DN(i-1))
        bool first_dn = true;
        GroupIt it{v.u0, v.u1, upe};
        Grp cur, prev;
        bool more = it.next(cur), has_prev = false;
        while (more || has_prev) {
          if (more) {
            const int b1 = (gb + i) & 1;
            mbar_wait(&d1_empty[b1], d1e[b1].bit ^ 1u);
            d1e[b1].flip();
            fence_after();
            const uint32_t d1 = tmem + static_cast<uint32_t>(b1 * 16);
            const Geom g = gu_geom(cur.nu, kcap);
            const uint32_t ab = static_cast<uint32_t>(cur.nu) * UB;
            for (int kt = 0; kt < ktiles; kt += g.m) {
              const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
              mbar_wait(&full[slot], (idx / NSLOT) & 1u);
              ++idx;
              for (; ht_ok < kt + g.m; ++ht_ok) mbar_wait(&ht_full[ht_ok], hpar);
              fence_after();
              if (leader) {
                for (int j = 0; j < g.m; ++j) {
                  const uint64_t adesc = smem_desc(ring_addr + off + j * ab, 128, 1024);
                  const uint64_t bdesc = smem_desc(ht_addr + (kt + j) * HTS, 128, 1024);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk) mma_bf16(d1, adesc + 16 * kk, bdesc + 16 * kk, (kt | j | kk) != 0);
                }
                mma_commit(&empty[slot]);
              }
              __syncwarp();
            }
            if (leader) {
              mma_commit(&d1_full[b1]);
              if (it.u >= it.u1) mma_commit(ht_free);  // the layer's last gate|up pass
            }
            __syncwarp();
          }
          if (has_prev) {
            const int ab_ = (gb + i - 1) & 1;
            mbar_wait(&at_full[ab_], ate[ab_].bit);
            ate[ab_].flip();
            fence_after();
            if (first_dn) {
              // D2 of the previous layer drained by the epilogue
              if (processed > 0) mbar_wait(d2_empty, static_cast<uint32_t>(processed - 1) & 1u);
              fence_after();
            }
            const uint32_t ahi = at_addr + static_cast<uint32_t>(ab_) * 8192u;
            const uint64_t bhi = smem_desc(ahi, 256, 128), blo = smem_desc(ahi + 4096u, 256, 128);
            const Geom g = dn_geom(prev.nu, mcap);
            const uint32_t ab = static_cast<uint32_t>(prev.nu) * UB;
            for (int mt = 0; mt < mtiles; mt += g.m) {
              const uint32_t off = ring_place(head, g, RB), slot = idx % NSLOT;
              mbar_wait(&full[slot], (idx / NSLOT) & 1u);
              ++idx;
              fence_after();
              if (leader) {
                for (int j = 0; j < g.m; ++j) {
                  const uint32_t d2 = tmem + D2_COL0 + static_cast<uint32_t>((mt + j) * 16);
                  for (int s2 = 0; 2 * s2 < prev.nu; ++s2) {
                    const uint32_t run = ring_addr + off + j * ab + 2 * s2 * UB;
                    const uint32_t lbo = 2 * s2 + 1 < prev.nu ? UB : zero_addr - run;
                    const uint64_t adn = smem_desc(run, lbo, 128);
                    mma_bf16(d2, adn, bhi + 32 * s2, (first_dn && s2 == 0) ? 0u : 1u);
                    mma_bf16(d2, adn, blo + 32 * s2, 1u);
                  }
                }
                mma_commit(&empty[slot]);
              }
              __syncwarp();
            }
            first_dn = false;
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
        if (leader) mma_commit(d2_full);
        __syncwarp();
        if (lane == 0) stamp(a, l, 3);
        gb += i - 1;  // the loop ran one step per group plus the final DN
        ++processed;
        side_work(l);
      }
    } else {
      // ------------------------------------------------ epilogue (4 warps) + in-kernel combine
      const int q = warp & 3;
      const int et = tid - 64;
      Phase d1f[2], atf[2];
      int i = 0, processed = 0;
      const int Q = T * d / 4;  // float4 outputs per layer
      const int s0 = static_cast<int>((static_cast<long long>(b) * Q) / G);
      const int s1 = static_cast<int>((static_cast<long long>(b + 1) * Q) / G);
      const int dq = d / 4;
      stage_layer(a, 0, upe, ent_gate, ent_mask, warp - 2, 4, lane);
      named_bar_sync(2, EPI_THREADS);
      for (int l = 0; l < L; ++l) {
        const LayerView v = layer_view(a, l, upe);
        const float* eg = ent_gate + (l & 1) * ENT_MAX * 16;
        const uint32_t* em = ent_mask + (l & 1) * ENT_MAX;
        if (v.u0 < v.u1) {
          GroupIt it{v.u0, v.u1, upe};
          Grp g;
          while (it.next(g)) {
            const int b1 = i & 1;
            mbar_wait(&d1_full[b1], d1f[b1].bit);
            d1f[b1].flip();
            fence_after();
            float vv[16];
            tc::tmem_ld16(tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(b1 * 16), vv);
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&d1_empty[b1]);
            const int ab = i & 1;
            mbar_wait(&at_empty[ab], atf[ab].bit ^ 1u);
            atf[ab].flip();
            {
              const int slot = 2 * q + (lane >> 4);
              const bool valid = slot < g.nu;
              const float* gs = eg + (valid ? static_cast<int>((g.us + slot) / upe) - v.o_first : 0) * 16;
              const int f = 8 * slot + (lane & 7);
              const int up = (lane >> 3) & 1;
              uint16_t* hi = reinterpret_cast<uint16_t*>(aT + static_cast<size_t>(ab) * 8192);
              uint16_t* lo = hi + 2048;
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                if (t < T) {
                  const float pv = __shfl_xor_sync(0xffffffffu, vv[t], 8);
                  if ((t & 1) == up) {
                    const float gv = up ? pv : vv[t];
                    const float uv = up ? vv[t] : pv;
                    const float gt = valid ? gs[t] : 0.f;
                    const float av = gt != 0.f ? __fdividef(gv, 1.f + __expf(-gv)) * uv * gt : 0.f;
                    const uint16_t h16 = f32_to_bf16_rn(av);
                    const float rem = av - __uint_as_float(static_cast<uint32_t>(h16) << 16);
                    const int off = (f >> 3) * 128 + (t >> 3) * 64 + (t & 7) * 8 + (f & 7);
                    hi[off] = h16;
                    lo[off] = f32_to_bf16_rn(rem);
                  }
                }
              }
            }
            fence_proxy_async();
            named_bar_sync(2, EPI_THREADS);
            if (et == 0) mbar_arrive(&at_full[ab]);
            ++i;
          }
          // ---- drain D2 (this CTA's sum over its experts) -> partial block
          mbar_wait(d2_full, static_cast<uint32_t>(processed) & 1u);
          fence_after();
          uint32_t tmask = 0;
          for (int r = 0; r < v.n_ent; ++r) tmask |= em[r];
          const uint32_t tbase = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(D2_COL0);
          float* P = a.partial + static_cast<long long>(b) * T * d + 32 * q + lane;
          for (int mt = 0; mt < mtiles; mt += 2) {
            uint32_t y0[16], y1[16];
            const bool two = mt + 1 < mtiles;
            if (T <= 8) {
              tc::tmem_ld8_nw(tbase + static_cast<uint32_t>(mt * 16), y0);
              if (two) tc::tmem_ld8_nw(tbase + static_cast<uint32_t>((mt + 1) * 16), y1);
            } else {
              tc::tmem_ld16_nw(tbase + static_cast<uint32_t>(mt * 16), y0);
              if (two) tc::tmem_ld16_nw(tbase + static_cast<uint32_t>((mt + 1) * 16), y1);
            }
            tc::tmem_wait_ld();
#pragma unroll
            for (int t = 0; t < 16; ++t)
              if (t < T && ((tmask >> t) & 1u)) {
                __stcg(P + static_cast<long long>(t) * d + mt * 128, __uint_as_float(y0[t]));
                if (two) __stcg(P + static_cast<long long>(t) * d + mt * 128 + 128, __uint_as_float(y1[t]));
              }
          }
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(d2_empty);
          if (et == 0) stamp(a, l, 4);
          ++processed;
        }
        if (et == 0) stamp(a, l, 0);
        // ---- grid barrier 1: every CTA's partial block of layer l written
        named_bar_sync(2, EPI_THREADS);
        if (et == 0) {
          __threadfence();
          red_release_add(a.sync, 1u);
        }
        if (et == 0) spin_until(a.sync, static_cast<unsigned>((l + 1) * G));
        named_bar_sync(2, EPI_THREADS);
        named_bar_sync(3, 32 + EPI_THREADS);  // the MMA warp staged layer l+1 and this layer's row lists
        if (et == 0) stamp(a, l, 1);
        // ---- combine of this CTA's output slice [s0, s1): 4 threads per
        // float4, rows dealt round-robin, partial sums added 0..3
        const int t_first = misc[4];
        for (int base = s0; base < s1; base += EPI_THREADS / 4) {
          const int oi = base + (et >> 2);
          const int r4 = et & 3;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          const bool live = oi < s1;
          const int t = live ? oi / dq : t_first;
          const int c = (live ? oi % dq : 0) * 4;
          const int li = t == t_first ? 0 : 1;
          const int nr = misc[2 + li] < ROWMAX ? misc[2 + li] : ROWMAX;
          const int* rl = rows + li * ROWMAX;
          if (live) {
            for (int j0 = r4; j0 < nr; j0 += 4 * 16) {
              float4 vb[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) {
                const int j = j0 + 4 * u;
                if (j < nr)
                  vb[u] = __ldcg(reinterpret_cast<const float4*>(a.partial + (static_cast<long long>(rl[j]) * T + t) * d + c));
              }
#pragma unroll
              for (int u = 0; u < 16; ++u)
                if (j0 + 4 * u < nr) {
                  acc.x += vb[u].x;
                  acc.y += vb[u].y;
                  acc.z += vb[u].z;
                  acc.w += vb[u].w;
                }
            }
          }
          // fixed-order reduction of the 4 quarter sums (lanes 4m..4m+3)
          float4 s = acc;
#pragma unroll
          for (int r = 1; r < 4; ++r) {
            const int src = (lane & ~3) + r;
            const float x = __shfl_sync(0xffffffffu, acc.x, src), yv = __shfl_sync(0xffffffffu, acc.y, src);
            const float z = __shfl_sync(0xffffffffu, acc.z, src), w = __shfl_sync(0xffffffffu, acc.w, src);
            s.x += x;
            s.y += yv;
            s.z += z;
            s.w += w;
          }
          if (live && r4 == 0) {
            const size_t off = static_cast<size_t>(t) * d + c;
            *reinterpret_cast<float4*>(a.y + static_cast<size_t>(l) * T * d + off) = s;
            const uint2 hv = __ldcg(reinterpret_cast<const uint2*>(a.h + static_cast<size_t>(l) * T * d + off));
            float4 r = s;
            r.x += bf_lo(hv.x);
            r.y += bf_hi(hv.x);
            r.z += bf_lo(hv.y);
            r.w += bf_hi(hv.y);
            uint2 o;
            o.x = static_cast<uint32_t>(f32_to_bf16_rn(r.x)) | (static_cast<uint32_t>(f32_to_bf16_rn(r.y)) << 16);
            o.y = static_cast<uint32_t>(f32_to_bf16_rn(r.z)) | (static_cast<uint32_t>(f32_to_bf16_rn(r.w)) << 16);
            *reinterpret_cast<uint2*>(a.h + static_cast<size_t>(l + 1) * T * d + off) = o;
            if (l + 1 < L) {
              uint16_t* hT_n = a.hT + static_cast<size_t>((l + 1) & 1) * 16 * d;
              const int kt = c >> 6, jj = (c >> 3) & 7, e = c & 7;
              *reinterpret_cast<uint2*>(hT_n + kt * 1024 + (t >> 3) * 512 + jj * 64 + (t & 7) * 8 + e) = o;
            }
          }
        }
        // ---- grid barrier 2 (arrive): h_{l+1} / h^T of layer l+1 written
        if (l + 1 < L) named_bar_arrive(4, 32 + EPI_THREADS);  // row lists / misc free again
        named_bar_sync(2, EPI_THREADS);
        if (et == 0) {
          __threadfence();
          red_release_add(a.sync + 1, 1u);
        }
        if (et == 0) stamp(a, l, 2);
      }
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(static_cast<uint32_t>(misc[1])),
                 "r"(TMEM_COLS));
  }
}

}  // namespace tp
}  // namespace dev

size_t ffn_tp_smem_bytes(int d, int ring_bytes) {
  return 2 * 2 * 4096 + static_cast<size_t>(d / 64) * dev::tp::HTS + static_cast<size_t>(ring_bytes) + dev::tp::UB +
         2 * dev::tp::ENT_MAX * (16 * 4 + 4) + 2 * dev::tp::ROWMAX * 4 + 32 + 8 +
         8 * (2 * dev::tp::NSLOT + 11 + dev::tp::MAX_KT);
}

// The persistent kernel needs no co-resident combine CTA: the whole SM's
// shared memory minus the per-CTA reserve.
int ffn_tp_ring_bytes(int T, int d, size_t smem_limit) {
  if (d > dev::tp::MAX_KT * 64 || d % 128 || T > 16) return 0;
  const size_t fixed = ffn_tp_smem_bytes(d, 0);
  if (fixed >= smem_limit) return 0;
  const int rb = static_cast<int>(((smem_limit - fixed) / 1024) * 1024);
  return rb >= 45056 ? rb : 0;
}

bool ffn_tp_ok(int n_entries, int d_ffn, int grid, int sms) {
  // co-residency of the whole grid (spin barriers) and the per-CTA entry limit
  const long long upe = d_ffn / 8, n = static_cast<long long>(n_entries) * upe;
  const long long maxu = (n + grid - 1) / grid;
  return grid > 0 && grid <= sms && grid <= dev::tp::ROWMAX && n * (grid + 1) < (1ll << 31) &&
         (maxu > 0 ? (maxu - 1) / upe + 2 : 1) <= dev::tp::ENT_MAX;
}

cudaError_t launch_expert_ffn_persistent(const dev::PersistArgs& a, int grid, size_t smem, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(dev::tp::expert_ffn_persistent_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  // the spin barriers need every CTA resident: no programmatic overlap with
  // the predecessor (its CTAs could hold SMs), grid <= SM count
  return launch_pdl(dev::tp::expert_ffn_persistent_kernel, dim3(grid), dim3(dev::tp::THREADS), smem, stream, false, a);
}

}  // namespace moespac
