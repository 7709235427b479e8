// TMA bulk-copy streaming probe (profiling, not part of the library).
//
// One CTA per SM streams its own contiguous slice of a large HBM buffer into
// a shared-memory ring with cp.async.bulk (global -> shared, mbarrier
// complete_tx), consuming nothing: the question is how many bytes per SM a
// bulk-copy ring of a given size and copy granularity keeps in flight, i.e.
// the streaming ceiling of a K3-style producer. Optionally each ring slot is
// filled by `pieces` copies of size/pieces bytes strided `stride` apart (the
// grouped K3's per-tile unit runs).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
//   ./tma_probe            (prints one JSON line per configuration)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_nohint(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void stream_kernel(const uint8_t* __restrict__ buf, long long per_cta, int slot_bytes, int nslot,
                              int pieces, long long stride, int issuers, int hint, unsigned long long* out_ns) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(slot_bytes) * nslot);
  if (threadIdx.x == 0) {
    for (int i = 0; i < nslot; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0)::"memory");
  const uint8_t* base = buf + blockIdx.x * per_cta;
  const long long n = per_cta / slot_bytes;
  const uint32_t pb = static_cast<uint32_t>(slot_bytes / pieces);
  // slot s of round r covers bytes [(r*nslot + s) * slot_bytes, +slot_bytes)
  // of the CTA's slice; with pieces > 1 they are gathered from pieces runs of
  // pb bytes `stride` apart (wrapping inside the slice)
  for (long long i = 0; i < n; ++i) {
    const int s = static_cast<int>(i % nslot);
    if (i >= nslot) mbar_wait(&bars[s], static_cast<uint32_t>(((i / nslot) - 1) & 1));
    if (lane == 0) mbar_expect(&bars[s], static_cast<uint32_t>(slot_bytes));
    __syncwarp();
    for (int p = lane; p < pieces && lane < issuers; p += issuers) {
      long long off = i * slot_bytes;
      if (pieces > 1) off = ((i * pieces + p) * stride) % per_cta;
      const uint8_t* src = base + (pieces > 1 ? off : off + p * pb);
      if (hint)
        bulk_g2s(sm + static_cast<size_t>(s) * slot_bytes + p * pb, src, pb, &bars[s], pol);
      else
        bulk_g2s_nohint(sm + static_cast<size_t>(s) * slot_bytes + p * pb, src, pb, &bars[s]);
    }
    __syncwarp();
  }
  for (long long i = n > nslot ? n - nslot : 0; i < n; ++i) {
    const int s = static_cast<int>(i % nslot);
    mbar_wait(&bars[s], static_cast<uint32_t>((i / nslot) & 1));
  }
  if (lane != 0) return;
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1)::"memory");
  out_ns[blockIdx.x * 2] = t0;
  out_ns[blockIdx.x * 2 + 1] = t1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long per_cta = 8LL << 20;  // 8 MiB per SM -> ~1.2 GB total, >> L2
  uint8_t* buf = nullptr;
  cudaMalloc(&buf, per_cta * sms);
  cudaMemset(buf, 1, per_cta * sms);
  unsigned long long* ns = nullptr;
  cudaMalloc(&ns, sms * 2 * sizeof(unsigned long long));
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int slot, nslot, pieces; long long stride; int issuers, hint; };
  const Cfg cfgs[] = {
      {2048, 64, 1, 0, 1, 1},   {4096, 32, 1, 0, 1, 1},   {8192, 16, 1, 0, 1, 1},   {16384, 8, 1, 0, 1, 1},
      {32768, 4, 1, 0, 1, 1},   {65536, 3, 1, 0, 1, 1},   {2048, 64, 1, 0, 1, 0},   {16384, 8, 1, 0, 1, 0},
      // slots filled by strided runs (the K3 unit-run shapes), 1 / 4 / 8 / 16 issuing lanes
      {32768, 4, 2, 16384, 1, 1}, {32768, 4, 2, 16384, 2, 1},
      {16384, 8, 8, 16384, 1, 1}, {16384, 8, 8, 16384, 4, 1}, {16384, 8, 8, 16384, 8, 1},
      {32768, 4, 16, 16384, 1, 1}, {32768, 4, 16, 16384, 16, 1}, {16384, 8, 8, 16384, 8, 0},
      {32768, 4, 4, 16384, 1, 1}, {32768, 4, 4, 16384, 4, 1},
  };
  for (const Cfg& c : cfgs) {
    const size_t smem = static_cast<size_t>(c.slot) * c.nslot + 8 * c.nslot;
    if (smem > 232448) continue;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      stream_kernel<<<sms, 32, smem>>>(buf, per_cta, c.slot, c.nslot, c.pieces, c.stride, c.issuers, c.hint, ns);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("{\"slot\": %d, \"nslot\": %d, \"ring_KiB\": %zu, \"pieces\": %d, \"issuers\": %d, \"hint\": %d, \"GBps\": %.1f, \"per_sm_GBps\": %.1f, \"err\": \"%s\"}\n",
           c.slot, c.nslot, static_cast<size_t>(c.slot) * c.nslot / 1024, c.pieces, c.issuers, c.hint,
           per_cta * sms / (best * 1e-3) / 1e9, per_cta / (best * 1e-3) / 1e9, cudaGetErrorString(err));
    fflush(stdout);
  }
  return 0;
}
