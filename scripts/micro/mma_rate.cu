// Microbenchmark (diagnostics): issue-to-completion time of a chain of
// tcgen05.mma.cta_group::1.kind::f16 (M = 128, K = 16) for N = 32..256,
// A from shared memory or from tensor memory, one CTA per SM on 128 SMs:
// the recurrence's per-step MMA chain is 32 x (128 x 64 x 16).
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((16 >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) k(int N, int nmma, int amode, int reps, unsigned long long* out, int nacc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0x3c003c00u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  unsigned long long tot = 0;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
    for (int r = 0; r < reps; ++r) {
      const unsigned long long t0 = gt();
      for (int i = 0; i < nmma; ++i) {
        const uint32_t a_s = su(s) + (i % 4) * 32 + (i / 4 % 2) * 16384;
        const uint64_t bd = desc(su(s) + 32768 + (i % 4) * 32);
        if (amode == 0) {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + 256 + (i % nacc) * (256 / nacc)),
                       "l"(desc(a_s)), "l"(bd), "r"(idesc), "r"(i >= nacc ? 1 : 0));
        } else {
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem + 256 + (i % nacc) * (256 / nacc)),
                       "r"(tmem + (i % 32) * 8), "l"(bd), "r"(idesc), "r"(i >= nacc ? 1 : 0));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     "selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(su(&bar)), "r"(r & 1) : "memory");
      tot += gt() - t0;
    }
    out[blockIdx.x] = tot / reps;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  for (int amode = 0; amode < 1; ++amode)
    for (int N : {64, 256})
    for (int nmma : {1, 2, 8, 32, 128, 512}) {
      const int nacc = 1;
      k<<<128, 128, 66 * 1024>>>(N, nmma, amode, 50, out, nacc);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h(128);
      cudaMemcpy(h.data(), out, 128 * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (auto v : h) m += (double)v;
      m /= 128;
      const double fl = 2.0 * 128 * N * 16 * nmma;
      printf("A %s N %3d x %2d MMAs, %d accumulators: %6.0f ns  (%.0f ns/MMA, %.1f TFLOP/s per SM) %s\n",
             amode ? "tmem" : "smem", N, nmma, nacc, m, m / nmma, fl / m / 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
