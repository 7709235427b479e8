// tcgen05.mma throughput probe (profiling, not part of the library).
//
// One CTA per SM, one elected thread issuing a chain of kind::f16
// tcgen05.mma (A and B from shared memory, fp32 accumulator in TMEM) back to
// back, then one commit and its wait: cycles per MMA as a function of M, N
// and whether consecutive MMAs read the same or different A tiles. The K3
// kernels issue M = 128, N = 16 (tokens), K = 16 MMAs; the question is what
// one of them costs the tensor pipe when it is not waiting for data.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../csrc/kernels -o mma_probe mma_probe.cu
//   ./mma_probe            (prints one JSON line per configuration)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "tcgen05.cuh"

using namespace moespac::dev;

// kind::f16 MMA with a run-time instruction descriptor (M, N vary here)
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void mma_kernel(int n_mma, int m, int n, int distinct_a, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  // [A: 32 tiles x 4 KiB (M = 128 x K = 16 bf16 each)][B: 64 KiB]
  uint8_t* a_base = sm;
  uint8_t* b_base = sm + 32 * 4096;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (32 * 4096 + 65536) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) {
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(n) >> 3) << 17) |
                           ((static_cast<uint32_t>(m) >> 4) << 24);
    const uint32_t a_addr = smem_u32(a_base), b_addr = smem_u32(b_base);
    const uint64_t bdesc = tc::smem_desc(b_addr, 128, 1024);
    const bool leader = tc::elect_one();
    long long t0 = 0, t1 = 0;
    if (leader) {
      t0 = clock64();
      for (int i = 0; i < n_mma; ++i) {
        const uint64_t adesc = tc::smem_desc(a_addr + (distinct_a ? (i & 31) * 4096u : 0u), 128, 1024);
        mma_f16(tmem, adesc, bdesc, i > 0 ? 1u : 0u, idesc);
      }
      tc::mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (leader) {
      t1 = clock64();
      out[blockIdx.x] = t1 - t0;
    }
    __syncwarp();
    tc::fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d_out = nullptr;
  cudaMalloc(&d_out, sizeof(long long) * sms);
  long long* h_out = new long long[sms];
  const size_t smem = 32 * 4096 + 65536;
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  struct Cfg { int m, n, distinct, grid; };
  const Cfg cfgs[] = {
      {128, 16, 1, 1}, {128, 16, 0, 1}, {64, 16, 1, 1}, {128, 32, 1, 1}, {128, 64, 1, 1},
      {128, 128, 1, 1}, {128, 256, 1, 1}, {128, 16, 1, 0}, {64, 16, 1, 0}, {128, 256, 1, 0},
  };
  const int n_mma = 4096;
  for (const Cfg& c : cfgs) {
    const int grid = c.grid ? c.grid : sms;
    long long best = -1;
    for (int rep = 0; rep < 3; ++rep) {
      mma_kernel<<<grid, 128, smem>>>(n_mma, c.m, c.n, c.distinct, d_out);
      cudaDeviceSynchronize();
      cudaMemcpy(h_out, d_out, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h_out[i] > mx ? h_out[i] : mx;
      if (best < 0 || mx < best) best = mx;
    }
    const cudaError_t err = cudaGetLastError();
    printf("{\"M\": %d, \"N\": %d, \"K\": 16, \"distinct_A\": %d, \"ctas\": %d, \"mma\": %d, \"cycles_per_mma\": %.2f, "
           "\"dense_flop_per_cycle_per_sm\": %.1f, \"err\": \"%s\"}\n",
           c.m, c.n, c.distinct, grid, n_mma, static_cast<double>(best) / n_mma,
           2.0 * c.m * c.n * 16 / (static_cast<double>(best) / n_mma), cudaGetErrorString(err));
    fflush(stdout);
  }
  delete[] h_out;
  return 0;
}
