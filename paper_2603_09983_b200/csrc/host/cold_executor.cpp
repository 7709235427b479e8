// Cold-expert executor — see cold_executor.hpp. Compiled with
// -O3 -mavx2 -mfma (build.py) so the fp32 dot/axpy loops vectorise; reads
// the expert images in their device tile order (no host-side relayout), so
// a miss costs exactly one pass over the expert's bytes in host DRAM.
#include "cold_executor.hpp"

#include <immintrin.h>
#include <pthread.h>
#include <sched.h>

#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace moespac {

namespace {

inline float bf(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

inline float silu(float x) { return x / (1.f + std::exp(-x)); }

// Spin on pred with _mm_pause for at most kSpinNs; true if pred came true.
template <typename Pred>
bool spin_until(Pred pred) {
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned i = 0;; ++i) {
    if (pred()) return true;
    _mm_pause();
    if ((i & 63u) == 63u &&
        std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count() >
            ColdExecutor::kSpinNs)
      return pred();
  }
}

}  // namespace

ColdExecutor::ColdExecutor(int threads, int layout, int d, int ffn, int T)
    : layout_(layout), d_(d), ffn_(ffn), T_(T), rows_(layout == 2 ? 64 : 16) {
  __builtin_cpu_init();
  bf16_dot_ = __builtin_cpu_supports("avx512bf16") && !std::getenv("MOESPAC_COLD_SCALAR");
  if (threads < 1) threads = 1;
  // Worker w >= 1 is pinned to its own CPU of the process's allowed set,
  // skipping the first one, which is left to the driver thread (worker 0,
  // which also issues the layer's CUDA work): a static chunk partition waits
  // for its slowest worker, so a worker preempted or migrated mid-layer
  // stalls the layer (measured: 17-65% window-to-window spread unpinned).
  // MOESPAC_COLD_PIN=0 disables it.
  cpu_set_t allowed;
  CPU_ZERO(&allowed);
  std::vector<int> cpus;
  if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0)
    for (int c = 0; c < CPU_SETSIZE; ++c)
      if (CPU_ISSET(c, &allowed)) cpus.push_back(c);
  const char* pin_env = std::getenv("MOESPAC_COLD_PIN");
  pin_ = !(pin_env && pin_env[0] == '0') && static_cast<int>(cpus.size()) >= threads;
  part_.assign(static_cast<size_t>(threads), std::vector<float>(static_cast<size_t>(T) * d));
  scratch_.assign(static_cast<size_t>(threads), std::vector<float>());
  hf_.assign(static_cast<size_t>(T) * d, 0.f);
  // Workers spin briefly on the job generation before sleeping: a layer's
  // cold work arrives every few hundred microseconds, and a condition-
  // variable wake-up per layer and worker cost tens of microseconds each.
  for (int w = 1; w < threads; ++w) workers_.emplace_back([this, w, cpu = pin_ ? cpus[static_cast<size_t>(w)] : -1] {
      if (cpu >= 0) {
        cpu_set_t one;
        CPU_ZERO(&one);
        CPU_SET(cpu, &one);
        pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
      }
      int seen = 0;
      for (;;) {
        const bool got = spin_until(
            [&] { return gen_a_.load(std::memory_order_acquire) != seen || stop_a_.load(std::memory_order_acquire); });
        if (!got) {
          std::unique_lock<std::mutex> lk(mu_);
          cv_.wait(lk, [&] { return stop_a_.load() || gen_a_.load() != seen; });
        }
        if (stop_a_.load(std::memory_order_acquire)) return;
        seen = gen_a_.load(std::memory_order_acquire);
        work(w);
        if (pending_a_.fetch_sub(1, std::memory_order_acq_rel) == 1) {
          std::lock_guard<std::mutex> lk(mu_);
          done_cv_.notify_all();
        }
      }
    });
}

ColdExecutor::~ColdExecutor() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_a_.store(true, std::memory_order_release);
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

// AVX-512 BF16 path for the tensor-core image (layout 2), chosen at run time
// when the host has VDPBF16PS: the image's core matrices are 8 rows x 8
// bf16 = 128 contiguous bytes, i.e. two 512-bit registers of 4 rows x 8 k;
// one dot-product instruction against a token's 8 h values (16 bytes,
// broadcast to the four 128-bit lanes) accumulates 32 products. The down
// projection takes a = silu(g)·u·gate as bf16 hi + lo (two passes), as K3
// does on the device, so both sides round a the same way.
__attribute__((target("avx512f,avx512bw,avx512vl,avx512bf16"))) static void chunk_tc_bf16(
    const ColdItem& it, int c, int d, const uint16_t* hb, float* y, float* acc, uint16_t* abf) {
  const int R = 64, n = it.n_tok;
  const uint16_t* base = it.image + static_cast<size_t>(c) * 3 * R * d;
  const int ktiles = d / 64;
  // ---- gate|up: acc[row-slot f][i] per token, gate rows then up rows
  for (int g = 0; g < 16; ++g) {
    __m512 s0[16], s1[16];
    for (int i = 0; i < n; ++i) {
      s0[i] = _mm512_setzero_ps();
      s1[i] = _mm512_setzero_ps();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
      const uint16_t* gp = base + static_cast<size_t>(kt) * 8192 + g * 512;
      for (int j = 0; j < 8; ++j) {
        const __m512bh w0 = reinterpret_cast<__m512bh>(_mm512_loadu_si512(gp + j * 64));
        const __m512bh w1 = reinterpret_cast<__m512bh>(_mm512_loadu_si512(gp + j * 64 + 32));
        for (int i = 0; i < n; ++i) {
          const __m512bh hv = reinterpret_cast<__m512bh>(_mm512_broadcast_i32x4(
              _mm_loadu_si128(reinterpret_cast<const __m128i*>(hb + static_cast<size_t>(it.tok[i]) * d + kt * 64 + j * 8))));
          s0[i] = _mm512_dpbf16_ps(s0[i], w0, hv);
          s1[i] = _mm512_dpbf16_ps(s1[i], w1, hv);
        }
      }
    }
    for (int i = 0; i < n; ++i) {
      alignas(64) float v[32];
      _mm512_store_ps(v, s0[i]);
      _mm512_store_ps(v + 16, s1[i]);
      for (int r = 0; r < 8; ++r) {
        const float tot = (v[4 * r] + v[4 * r + 1]) + (v[4 * r + 2] + v[4 * r + 3]);
        const int row = g * 8 + r;  // quarter-major, octet-interleaved (see the scalar path)
        const int qq = row >> 5, sr = row & 31;
        const int fl = qq * 16 + ((sr >> 4) << 3) + (sr & 7);
        acc[((((sr >> 3) & 1) ? R + fl : fl)) * 16 + i] = tot;
      }
    }
  }
  // ---- a = silu(g) u gate as bf16 hi + lo, [i][f]
  for (int i = 0; i < n; ++i)
    for (int f = 0; f < R; ++f) {
      const float gv = acc[f * 16 + i], uv = acc[(R + f) * 16 + i];
      const float av = gv / (1.f + std::exp(-gv)) * uv * it.gate[i];
      uint32_t u;
      std::memcpy(&u, &av, 4);
      const uint32_t hiu = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;  // round to nearest even
      float hi;
      std::memcpy(&hi, &hiu, 4);
      const float rem = av - hi;
      uint32_t ru;
      std::memcpy(&ru, &rem, 4);
      abf[(i * 2 + 0) * R + f] = static_cast<uint16_t>(hiu >> 16);
      abf[(i * 2 + 1) * R + f] = static_cast<uint16_t>((ru + 0x7fffu + ((ru >> 16) & 1u)) >> 16);
    }
  // ---- down: y[tok][o] += sum_f W[o][f] a[f]
  const uint16_t* dbase = base + static_cast<size_t>(ktiles) * 8192;
  for (int mt = 0; mt < d / 128; ++mt) {
    const uint16_t* tile = dbase + static_cast<size_t>(mt) * 8192;
    for (int go = 0; go < 16; ++go) {
      __m512 s0[16], s1[16];
      for (int i = 0; i < n; ++i) {
        s0[i] = _mm512_setzero_ps();
        s1[i] = _mm512_setzero_ps();
      }
      for (int j = 0; j < 8; ++j) {
        const uint16_t* gp = tile + j * 1024 + go * 64;
        const __m512bh w0 = reinterpret_cast<__m512bh>(_mm512_loadu_si512(gp));
        const __m512bh w1 = reinterpret_cast<__m512bh>(_mm512_loadu_si512(gp + 32));
        for (int i = 0; i < n; ++i)
          for (int part = 0; part < 2; ++part) {
            const __m512bh av = reinterpret_cast<__m512bh>(_mm512_broadcast_i32x4(
                _mm_loadu_si128(reinterpret_cast<const __m128i*>(abf + (i * 2 + part) * R + j * 8))));
            s0[i] = _mm512_dpbf16_ps(s0[i], w0, av);
            s1[i] = _mm512_dpbf16_ps(s1[i], w1, av);
          }
      }
      for (int i = 0; i < n; ++i) {
        alignas(64) float v[32];
        _mm512_store_ps(v, s0[i]);
        _mm512_store_ps(v + 16, s1[i]);
        float* yr = y + static_cast<size_t>(it.tok[i]) * d + mt * 128 + go * 8;
        for (int r = 0; r < 8; ++r) yr[r] += (v[4 * r] + v[4 * r + 1]) + (v[4 * r + 2] + v[4 * r + 3]);
      }
    }
  }
}

// One chunk of one expert: gate/up rows -> a = silu(g) * u * gate -> down.
void ColdExecutor::chunk(const ColdItem& it, int c, const float* hf, float* y, std::vector<float>& scr) const {
  const int d = d_, R = rows_, n = it.n_tok;
  scr.resize(static_cast<size_t>(2 * R) * 16 + static_cast<size_t>(d) + static_cast<size_t>(2 * 16 * R));
  float* acc = scr.data();        // [2R][16] gate rows then up rows, per token
  float* wrow = acc + 2 * R * 16;  // one unpacked row [d] (or [64] for layout 2 runs)
  std::memset(acc, 0, sizeof(float) * 2 * R * 16);
  if (layout_ == 2 && bf16_dot_) {
    chunk_tc_bf16(it, c, d, hb_, y, acc, reinterpret_cast<uint16_t*>(wrow + d));
    return;
  }
  const uint16_t* base = it.image + static_cast<size_t>(c) * 3 * R * d;
  if (layout_ == 2) {
    // gate|up K-tiles [128 rows][64 k]: element (row, kk) at
    // (row>>3)*512 + (kk>>3)*64 + (row&7)*8 + (kk&7); rows ordered by quarter
    for (int kt = 0; kt < d / 64; ++kt) {
      const uint16_t* tile = base + static_cast<size_t>(kt) * 8192;
      for (int row = 0; row < 128; ++row) {
        float w[64];
        const uint16_t* rp = tile + (row >> 3) * 512 + (row & 7) * 8;
        for (int j = 0; j < 8; ++j)
          for (int e = 0; e < 8; ++e) w[j * 8 + e] = bf(rp[j * 64 + e]);
        // 16-row quarter q = row / 32, octet-interleaved: gate rows f 0-7,
        // up rows f 0-7, gate rows f 8-15, up rows f 8-15 (f within the quarter)
        const int qq = row >> 5, s = row & 31;
        const int fl = qq * 16 + ((s >> 4) << 3) + (s & 7);
        float* ar = acc + (((s >> 3) & 1) ? R + fl : fl) * 16;
        for (int i = 0; i < n; ++i) {
          const float* hv = hf + static_cast<size_t>(it.tok[i]) * d + kt * 64;
          float s = 0.f;
          for (int k = 0; k < 64; ++k) s += w[k] * hv[k];
          ar[i] += s;
        }
      }
    }
  } else {
    // gate|up tiles [32 rows][256 cols] row-major: rows 0-15 gate, 16-31 up
    for (int ct = 0; ct < d / 256; ++ct) {
      const uint16_t* tile = base + static_cast<size_t>(ct) * 8192;
      for (int row = 0; row < 32; ++row) {
        float w[256];
        for (int k = 0; k < 256; ++k) w[k] = bf(tile[row * 256 + k]);
        float* ar = acc + row * 16;
        for (int i = 0; i < n; ++i) {
          const float* hv = hf + static_cast<size_t>(it.tok[i]) * d + ct * 256;
          float s = 0.f;
          for (int k = 0; k < 256; ++k) s += w[k] * hv[k];
          ar[i] += s;
        }
      }
    }
  }
  // a[f][i] (stored over the gate accumulators)
  for (int f = 0; f < R; ++f)
    for (int i = 0; i < n; ++i) acc[f * 16 + i] = silu(acc[f * 16 + i]) * acc[(R + f) * 16 + i] * it.gate[i];
  if (layout_ == 2) {
    // down M-tiles [128 out][64 f]: element (o, f) at (f>>3)*1024 + (o>>3)*64 + (o&7)*8 + (f&7)
    const uint16_t* dbase = base + static_cast<size_t>(d / 64) * 8192;
    for (int mt = 0; mt < d / 128; ++mt) {
      const uint16_t* tile = dbase + static_cast<size_t>(mt) * 8192;
      for (int o = 0; o < 128; ++o) {
        float w[64];
        const uint16_t* rp = tile + (o >> 3) * 64 + (o & 7) * 8;
        for (int j = 0; j < 8; ++j)
          for (int e = 0; e < 8; ++e) w[j * 8 + e] = bf(rp[j * 1024 + e]);
        const int orow = mt * 128 + o;
        for (int i = 0; i < n; ++i) {
          float s = 0.f;
          for (int f = 0; f < 64; ++f) s += w[f] * acc[f * 16 + i];
          y[static_cast<size_t>(it.tok[i]) * d + orow] += s;
        }
      }
    }
  } else {
    // down tiles of W_down^T: [DR f-rows][DW out cols]
    const int DW = d < 1024 ? d : 1024, DR = 8192 / DW, nrg = 16 / DR;
    const uint16_t* dbase = base + static_cast<size_t>(d / 256) * 8192;
    for (int t2 = 0; t2 < d / 512; ++t2) {
      const uint16_t* tile = dbase + static_cast<size_t>(t2) * 8192;
      const int ct2 = t2 / nrg, fg = t2 % nrg;
      for (int row = 0; row < DR; ++row) {
        const int f = fg * DR + row;
        for (int col = 0; col < DW; ++col) wrow[col] = bf(tile[row * DW + col]);
        for (int i = 0; i < n; ++i) {
          const float av = acc[f * 16 + i];
          float* yr = y + static_cast<size_t>(it.tok[i]) * d + ct2 * DW;
          for (int col = 0; col < DW; ++col) yr[col] += wrow[col] * av;
        }
      }
    }
  }
}

void ColdExecutor::work(int w) {
  std::vector<float>& part = part_[static_cast<size_t>(w)];
  std::fill(part.begin(), part.end(), 0.f);
  const int W = threads();
  for (size_t u = static_cast<size_t>(w); u < units_.size(); u += static_cast<size_t>(W))
    chunk((*items_)[static_cast<size_t>(units_[u].first)], units_[u].second, hf_.data(), part.data(),
          scratch_[static_cast<size_t>(w)]);
}

void ColdExecutor::run(const std::vector<ColdItem>& items, const uint16_t* h, float* y) {
  const size_t TD = static_cast<size_t>(T_) * d_;
  for (size_t i = 0; i < TD; ++i) hf_[i] = bf(h[i]);
  hb_ = h;
  units_.clear();
  const int cpe = ffn_ / rows_;
  for (size_t i = 0; i < items.size(); ++i)
    for (int c = 0; c < cpe; ++c) units_.emplace_back(static_cast<int>(i), c);
  items_ = &items;
  pending_a_.store(static_cast<int>(workers_.size()), std::memory_order_relaxed);
  {
    std::lock_guard<std::mutex> lk(mu_);
    gen_a_.fetch_add(1, std::memory_order_acq_rel);
  }
  cv_.notify_all();
  work(0);
  if (!spin_until([&] { return pending_a_.load(std::memory_order_acquire) == 0; })) {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_a_.load() == 0; });
  }
  // fixed-order reduction over workers
  std::memcpy(y, part_[0].data(), sizeof(float) * TD);
  for (size_t w = 1; w < part_.size(); ++w) {
    const float* p = part_[w].data();
    for (size_t i = 0; i < TD; ++i) y[i] += p[i];
  }
}

}  // namespace moespac
