/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the verification-step MoE
 * hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * (paper_2603_09983_b200/) never links or calls it.
 *
 * Plain-C restatement of the reference algorithm, each function citing the
 * reference file:line it follows (paths relative to /root/reference):
 *
 *   orc_mt64_*            std::mt19937_64 (C++ [rand.eng.mers], as used by
 *                         proj/core/include/moesim/trace_model.hpp:74)
 *   orc_gen_*             TraceGenerator + uniform01/gaussian/gumbel,
 *                         proj/core/src/trace_model.cpp:30-109, additionally
 *                         emitting the noisy fp64 logits that K1 consumes
 *   orc_router_topk       top-k block, trace_model.cpp:87-104
 *                         (value desc, id asc; ids sorted ascending) plus
 *                         Eq. 3 gates — gates UNPINNED by
 *                         the reference (no gating code exists there)
 *   orc_hist_scan         activation_frequencies, trace_model.cpp:122-130,
 *                         plus the (expert, token, slot)-sorted permutation
 *                         (permutation order UNPINNED: new in this design)
 *   orc_estimator_*       LayerEstimator ctor/calibrate/observe_step,
 *                         proj/core/src/utility_estimator.cpp:23-72
 *   orc_realized_split    realized split + accuracy/fault counters,
 *                         proj/core/src/sim_core.cpp:233-283
 *   orc_expert_apply      SwiGLU expert, PAPER.md:971 (W_up·x, W_gate·x,
 *                         W_down·x) — numerics UNPINNED by the reference
 *                         (its FFN is the modeled constant sim_core.cpp:253)
 *
 * Parity pinning: tests/test_oracle.py checks this file against the compiled
 * reference (oracle/_ref/libmoesim_ref.so, built from the reference sources by
 * oracle/Makefile) and against the committed fixtures in tests/golden/.
 * Build with -ffp-contract=off: calibrate()'s floor is FMA-sensitive
 * (SURVEY.md §0 item 6).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- std::mt19937_64 ---------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* trace_model.cpp:30-32 */
static double uniform01(orc_mt64* g) { return (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53; }

/* trace_model.cpp:34-41 */
static double gaussian(orc_mt64* g) {
  double u1 = uniform01(g);
  double u2 = uniform01(g);
  while (u1 == 0.0) u1 = uniform01(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* trace_model.cpp:43-47 */
static double gumbel(orc_mt64* g) {
  double u = uniform01(g);
  while (u == 0.0) u = uniform01(g);
  return -log(-log(u));
}

/* ---------------- trace generator (trace_model.cpp:59-109) ---------------- */
typedef struct {
  int L, N, k, gamma, shift_period, step;
  double alpha, drift, noise;
  orc_mt64 rng;
  double* logits; /* [L][N] latent */
} orc_gen;

static void redraw(orc_gen* g) {
  for (int i = 0; i < g->L * g->N; ++i) g->logits[i] = gaussian(&g->rng);
}

orc_gen* orc_gen_create(int L, int N, int k, int gamma, double alpha, double drift,
                        double noise, int shift_period, uint64_t seed) {
  if (L < 1 || N < 1 || k < 1 || k > N || gamma < 1 || alpha < 0 || alpha > 1 || drift < 0 ||
      noise < 0 || shift_period < 0)
    return NULL;
  orc_gen* g = (orc_gen*)calloc(1, sizeof(orc_gen));
  g->L = L; g->N = N; g->k = k; g->gamma = gamma; g->alpha = alpha;
  g->drift = drift; g->noise = noise; g->shift_period = shift_period;
  orc_mt64_seed(&g->rng, seed);
  g->logits = (double*)malloc(sizeof(double) * (size_t)L * N);
  redraw(g);
  return g;
}

void orc_gen_destroy(orc_gen* g) {
  if (!g) return;
  free(g->logits);
  free(g);
}

/* Selection by (value desc, id asc) == the partial_sort comparator at
 * trace_model.cpp:96-100; the k chosen ids are then sorted ascending (:104). */
static void topk_row(const double* v, int N, int k, int32_t* ids, uint8_t* taken) {
  memset(taken, 0, (size_t)N);
  for (int r = 0; r < k; ++r) {
    int best = -1;
    for (int e = 0; e < N; ++e) {
      if (taken[e]) continue;
      if (best < 0 || v[e] > v[best]) best = e; /* strict >: ties keep lower id */
    }
    taken[best] = 1;
  }
  int j = 0;
  for (int e = 0; e < N; ++e)
    if (taken[e]) ids[j++] = e;
}

/* One step. noisy: [L][T][N] (may be NULL), ids: [L][T][k]. Returns accepted. */
int orc_gen_next(orc_gen* g, double* noisy, int32_t* ids) {
  const int T = g->gamma + 1, N = g->N, k = g->k;
  ++g->step;
  if (g->shift_period > 0 && g->step > 1 && (g->step - 1) % g->shift_period == 0) redraw(g);
  if (g->drift > 0.0)
    for (int i = 0; i < g->L * N; ++i) g->logits[i] += g->drift * gaussian(&g->rng);
  double* row = (double*)malloc(sizeof(double) * N);
  uint8_t* taken = (uint8_t*)malloc((size_t)N);
  for (int l = 0; l < g->L; ++l)
    for (int t = 0; t < T; ++t) {
      for (int e = 0; e < N; ++e) {
        double nz = g->noise > 0.0 ? g->noise * gumbel(&g->rng) : 0.0;
        row[e] = g->logits[(size_t)l * N + e] + nz; /* trace_model.cpp:94 */
      }
      if (noisy) memcpy(noisy + ((size_t)l * T + t) * N, row, sizeof(double) * N);
      topk_row(row, N, k, ids + ((size_t)l * T + t) * k, taken);
    }
  free(row);
  free(taken);
  /* sample_accept_length, trace_model.cpp:51-57 */
  int acc = 0;
  while (acc < g->gamma && uniform01(&g->rng) < g->alpha) ++acc;
  return acc + 1;
}

/* ---------------- K1 oracle: router top-k + gates ----------------
 * gate_mode 0: softmax over the selected k (Eq. 3, renormalized top-k)
 * gate_mode 1: softmax over all N, selected entries not renormalized
 *              (Qwen1.5-MoE / DeepSeek-V2-Lite convention). */
void orc_router_topk(const double* logits, int rows, int N, int k, int gate_mode, int32_t* ids,
                     double* gates) {
  uint8_t* taken = (uint8_t*)malloc((size_t)N);
  for (int r = 0; r < rows; ++r) {
    const double* v = logits + (size_t)r * N;
    int32_t* id = ids + (size_t)r * k;
    topk_row(v, N, k, id, taken);
    if (!gates) continue;
    double m = v[id[0]];
    for (int j = 1; j < k; ++j) m = v[id[j]] > m ? v[id[j]] : m;
    double s = 0.0;
    if (gate_mode == 1) {
      for (int e = 0; e < N; ++e) m = v[e] > m ? v[e] : m;
      for (int e = 0; e < N; ++e) s += exp(v[e] - m);
    } else {
      for (int j = 0; j < k; ++j) s += exp(v[id[j]] - m);
    }
    for (int j = 0; j < k; ++j) gates[(size_t)r * k + j] = exp(v[id[j]] - m) / s;
  }
  free(taken);
}

/* ---------------- K2 oracle: histogram, scan, permutation ----------------
 * freqs: activation_frequencies (trace_model.cpp:122-130) over all T tokens.
 * offsets: exclusive scan, [N+1]. perm[p] = t*k + j sorted by (expert, t, j). */
void orc_hist_scan(const int32_t* ids, int T, int k, int N, int32_t* freqs, int32_t* offsets,
                   int32_t* perm) {
  memset(freqs, 0, sizeof(int32_t) * N);
  for (int i = 0; i < T * k; ++i) freqs[ids[i]]++;
  offsets[0] = 0;
  for (int e = 0; e < N; ++e) offsets[e + 1] = offsets[e] + freqs[e];
  int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * N);
  memcpy(cur, offsets, sizeof(int32_t) * N);
  for (int i = 0; i < T * k; ++i) perm[cur[ids[i]]++] = i; /* i = t*k + j, ascending */
  free(cur);
}

/* ---------------- estimator (utility_estimator.cpp:23-72) ---------------- */
void orc_estimator_init(int32_t* st, int N, int gamma, int init_up, int init_down) {
  for (int i = 0; i < N; ++i) {
    st[4 * i + 0] = 0;
    st[4 * i + 1] = init_up >= 0 ? init_up : gamma / 2;
    st[4 * i + 2] = init_down >= 0 ? init_down : gamma / 2;
    st[4 * i + 3] = 0;
  }
}

/* utility_estimator.cpp:40-43; the two products and the sum are separate
 * IEEE double operations (no contraction). */
static int calibrate(int boundary, double lambda, int magnitude) {
  volatile double a = (1.0 - lambda) * (double)boundary;
  volatile double b = lambda * (double)magnitude;
  double next = a + b;
  int f = (int)floor(next);
  return f > 1 ? f : 1;
}

void orc_estimator_observe(int32_t* st, const int32_t* freqs, int N, int cap, double lambda,
                           int adaptive) {
  for (int i = 0; i < N; ++i) {
    int32_t* s = st + 4 * i;
    const int delta = freqs[i] - s[3];
    if (delta >= s[1]) s[0] = s[0] + 1 < cap ? s[0] + 1 : cap;
    else if (-delta >= s[2]) s[0] = s[0] - 1 > 0 ? s[0] - 1 : 0;
    if (adaptive) {
      if (delta > 0) s[1] = calibrate(s[1], lambda, delta);
      else if (delta < 0) s[2] = calibrate(s[2], lambda, -delta);
    }
    s[3] = freqs[i];
  }
}

/* ---------------- realized split (sim_core.cpp:233-283) ----------------
 * out: distinct, distinct_hits, hit_tokens, miss_tokens, agree, faults_fn,
 *      faults_fp (loaded this step and unactivated), 0 */
void orc_realized_split(const int32_t* freqs, const int32_t* scores, const uint8_t* resident,
                        const uint8_t* loaded, int N, int tau, int64_t* out) {
  memset(out, 0, sizeof(int64_t) * 8);
  for (int e = 0; e < N; ++e) {
    if (freqs[e] > 0) {
      out[0]++;
      if (resident[e]) { out[1]++; out[2] += freqs[e]; }
      else out[3] += freqs[e];
    }
    if ((scores[e] >= 1) == (freqs[e] >= 1)) out[4]++;
    if (freqs[e] >= 1 && scores[e] < tau) out[5]++;
    if (loaded && loaded[e] && freqs[e] == 0) out[6]++;
  }
}

/* ---------------- expert FFN oracle ---------------- */
static inline float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40); /* NaN */
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

/* y[tok[i]] += gate[i] * W_down · (silu(W_gate · h) ⊙ (W_up · h)) for the n
 * tokens of one expert, in fp64. Standard (untiled) layouts:
 * wg, wu: [ffn][d]; wd: [d][ffn]; h: [T][d] bf16; y: [T][d] fp64. */
void orc_expert_apply(const uint16_t* h, int d, int ffn, const int32_t* tok, const double* gate,
                      int n, const uint16_t* wg, const uint16_t* wu, const uint16_t* wd,
                      double* y, int n_threads) {
  double* a = (double*)malloc(sizeof(double) * (size_t)n * ffn);
#ifdef _OPENMP
  if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for num_threads(n_threads) schedule(static)
#endif
  for (int f = 0; f < ffn; ++f) {
    for (int i = 0; i < n; ++i) {
      const uint16_t* x = h + (size_t)tok[i] * d;
      double g = 0.0, u = 0.0;
      for (int c = 0; c < d; ++c) {
        double xv = bf16_to_f32(x[c]);
        g += (double)bf16_to_f32(wg[(size_t)f * d + c]) * xv;
        u += (double)bf16_to_f32(wu[(size_t)f * d + c]) * xv;
      }
      a[(size_t)i * ffn + f] = g / (1.0 + exp(-g)) * u;
    }
  }
#ifdef _OPENMP
#pragma omp parallel for num_threads(n_threads) schedule(static)
#endif
  for (int r = 0; r < d; ++r) {
    for (int i = 0; i < n; ++i) {
      double acc = 0.0;
      for (int f = 0; f < ffn; ++f)
        acc += (double)bf16_to_f32(wd[(size_t)r * ffn + f]) * a[(size_t)i * ffn + f];
      y[(size_t)tok[i] * d + r] += gate[i] * acc;
    }
  }
  free(a);
}

/* Router GEMV s = W_g h (Eq. 3). The
 * reference has no router weights (its logits are a synthetic random walk),
 * so this is parity-unpinned against the reference and pinned instead to the
 * device K0's summation order (router_hist.cu, router_gemv_kernel): for each
 * (t, e), lane j in 0..31 accumulates k = 256 i + 8 j + q (i ascending,
 * q = 0..7) with fmaf in fp32, then a xor butterfly over m = 16, 8, 4, 2, 1
 * adds lane L ^ m into lane L. W [N][d], h [T][d] bf16; d % 256 == 0. */
void orc_router_gemv(const uint16_t* W, const uint16_t* h, int T, int N, int d, double* logits) {
  for (int t = 0; t < T; ++t)
    for (int e = 0; e < N; ++e) {
      float v[32], nv[32];
      for (int j = 0; j < 32; ++j) {
        float acc = 0.f;
        for (int i = 0; i < d / 256; ++i)
          for (int q = 0; q < 8; ++q) {
            const int k = 256 * i + 8 * j + q;
            acc = fmaf(bf16_to_f32(W[(size_t)e * d + k]), bf16_to_f32(h[(size_t)t * d + k]), acc);
          }
        v[j] = acc;
      }
      for (int m = 16; m > 0; m >>= 1) {
        for (int L = 0; L < 32; ++L) nv[L] = v[L] + v[L ^ m];
        memcpy(v, nv, sizeof(v));
      }
      logits[(size_t)t * N + e] = (double)v[0];
    }
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
