// The grouped K3's weight stream (expert_ffn_grouped.cu), shared with the
// kernels that prefetch it into L2 ahead of the launch that streams it.
//
// A layer's work is the list of 8-row units (8 gate + 8 up rows and the
// matching 8 down columns of one expert: 2 KiB per 16 KiB tile of the image)
// over (hit experts ascending, then shared units); CTA b of a G-CTA (virtual)
// grid streams units [b*n/G, (b+1)*n/G) in groups of <= gmax units, each group
// cut so that it spans at most two 64-row chunk pieces.
#pragma once
#include <cstdint>

namespace moespac {
namespace dev {
namespace k3s {

constexpr int TILE = 16384;  // one gate|up K-tile or down M-tile of a 64-row chunk
constexpr int UB = 2048;     // one 8-row unit of a tile
constexpr int UPC = 8;       // units per 64-row chunk

struct Grp {
  long long us;                 // first unit (global order)
  int nu, np;
  int o[2], c[2], pa[2], n[2];  // piece p: units [pa, pa + n) of chunk c of entry o
};

struct GroupIt {
  long long u, u1;
  int upe;    // units per entry = ffn / 8
  int gmax;   // units per group (8 or 16)
  int absorb = 0;  // a remainder of <= absorb units joins the group before it (a second M-tile)
  __device__ __forceinline__ bool next(Grp& g) {
    if (u >= u1) return false;
    const int o = static_cast<int>(u / upe), ui = static_cast<int>(u % upe);
    // end of u's chunk, and of the chunk after it (a group has <= 2 pieces)
    const long long cend = static_cast<long long>(o) * upe + (ui / UPC + 1) * UPC;
    long long ue = u + gmax < u1 ? u + gmax : u1;
    if (u1 - ue <= absorb) ue = u1;
    if (ue > cend + UPC) ue = cend + UPC;
    g.us = u;
    g.nu = static_cast<int>(ue - u);
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

// Where a layer's weight stream lives (a launch's routing tables and buffers).
struct StreamSrc {
  const int32_t* counters;  // counters[7] = hit experts
  const int32_t* hit_list;
  const int32_t* slot_of;
  const uint16_t* pool;
  const uint16_t* shared_w;
  int n_shared;
  long long expert_elems;
  int d, ffn;
};

// L2 prefetch of CTA bg's stream (of a G-CTA grid) in approximately stream
// order (group by group, each piece's tiles in order), skipping the first
// `skip` bytes and stopping after `budget` bytes. Run r is issued by lane
// r % 32 of the calling warp (all 32 lanes call).
__device__ __forceinline__ void prefetch_stream_l2(const StreamSrc& s, long long bg, int G, int gmax, long long skip,
                                                   long long budget, int lane) {
  const int upe = s.ffn / 8, ntile = s.d / 64 + s.d / 128;
  const long long chunk_bytes = 3LL * 64 * s.d * 2;
  const int nh = s.counters[7];
  const long long nn = static_cast<long long>(nh + s.n_shared) * upe;
  const long long p0 = nn > 0 ? (bg * nn) / G : 0, p1 = nn > 0 ? ((bg + 1) * nn) / G : 0;
  GroupIt it{p0, p1, upe, gmax};
  Grp g;
  int rc = 0;
  while (budget > 0 && it.next(g)) {
    for (int i = 0; i < g.np && budget > 0; ++i) {
      const int o = g.o[i];
      const uint16_t* w = o < nh ? s.pool + static_cast<long long>(s.slot_of[s.hit_list[o]]) * s.expert_elems
                                 : s.shared_w + static_cast<long long>(o - nh) * s.expert_elems;
      const uint8_t* base = reinterpret_cast<const uint8_t*>(w) + g.c[i] * chunk_bytes + g.pa[i] * UB;
      const uint32_t run = static_cast<uint32_t>(g.n[i]) * UB;
      for (int t = 0; t < ntile && budget > 0; ++t) {
        if (skip > 0) {
          skip -= run;
          continue;
        }
        if ((rc++ & 31) == lane)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + static_cast<size_t>(t) * TILE), "r"(run)
                       : "memory");
        budget -= run;
      }
    }
  }
}

}  // namespace k3s
}  // namespace dev
}  // namespace moespac
