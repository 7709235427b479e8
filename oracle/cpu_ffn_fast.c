/*
 * TEST INFRASTRUCTURE ONLY — timed CPU baseline for bench.py (cpu_baseline and
 * --impl reference legs). Same SwiGLU math as orc_expert_apply in
 * moespac_oracle.c, fp32 accumulation, compiled with
 * -O3 -ffast-math -mavx2 -mfma so the host cores get a fair, vectorised
 * kernel. Never linked into the product.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline float bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

/* Same math in fp32 with vectorisable loops: the timed CPU baseline
 * (bench.py cpu_baseline / --impl reference), all host threads. */
void orc_expert_apply_f32(const uint16_t* h, int d, int ffn, const int32_t* tok,
                          const float* gate, int n, const uint16_t* wg, const uint16_t* wu,
                          const uint16_t* wd, float* y, int n_threads) {
  float* a = (float*)malloc(sizeof(float) * (size_t)n * ffn);
  float* hx = (float*)malloc(sizeof(float) * (size_t)n * d);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < d; ++c) hx[(size_t)i * d + c] = bf16_to_f32(h[(size_t)tok[i] * d + c]);
#ifdef _OPENMP
  if (n_threads <= 0) n_threads = omp_get_max_threads();
#pragma omp parallel for num_threads(n_threads) schedule(static)
#endif
  for (int f = 0; f < ffn; ++f) {
    const uint16_t* rg = wg + (size_t)f * d;
    const uint16_t* ru = wu + (size_t)f * d;
    for (int i = 0; i < n; ++i) {
      const float* x = hx + (size_t)i * d;
      float g = 0.f, u = 0.f;
      for (int c = 0; c < d; ++c) {
        g += bf16_to_f32(rg[c]) * x[c];
        u += bf16_to_f32(ru[c]) * x[c];
      }
      a[(size_t)i * ffn + f] = g / (1.f + expf(-g)) * u;
    }
  }
#ifdef _OPENMP
#pragma omp parallel for num_threads(n_threads) schedule(static)
#endif
  for (int r = 0; r < d; ++r) {
    const uint16_t* rw = wd + (size_t)r * ffn;
    for (int i = 0; i < n; ++i) {
      const float* av = a + (size_t)i * ffn;
      float acc = 0.f;
      for (int f = 0; f < ffn; ++f) acc += bf16_to_f32(rw[f]) * av[f];
      y[(size_t)tok[i] * d + r] += gate[i] * acc;
    }
  }
  free(a);
  free(hx);
}

