// Microbenchmark (diagnostics): per-CTA ingest of 128 KB (8 k-blocks of a
// 128-row x 64-column bf16 tile, the recurrence's per-step A) into shared
// memory, 128 CTAs at once, by
//   mode 0: 2-D TMA boxes {64 cols, 128 rows}, SWIZZLE_128B (as rec_tc.cu)
//   mode 1: 1-D bulk copies of 16 KB contiguous chunks (a pre-blocked tape)
//   mode 2: 2-D TMA boxes {64 cols, 32 rows} (4 per k-block)
//   mode 3: as 0, but each repetition first rewrites the source (every CTA
//           its 32-row x 64-column slice, as the recurrence's producers),
//           publishes it (release counter) and waits for all 128 writers
//           (acquire) -- the timer starts after that wait
//   mode 4: as 3 with the writes to a fresh slot of a 16-step tape
// from a 512 KB source (all CTAs read the same h_t, K-slice = CTA % 4).
// Prints the mean time from the first issue to the last byte landed.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap m128,
                                            const __grid_constant__ CUtensorMap m32,
                                            const __nv_bfloat16* blocked, int mode, int reps,
                                            unsigned long long* out, __nv_bfloat16* src,
                                            unsigned* cnt, const __grid_constant__ CUtensorMap mtape) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  const int ks = blockIdx.x % 4;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    if (mode >= 3) {
      // my slice: rows 32 (b % 4).., columns 64 (b / 4)..  (b < 128)
      const int b = blockIdx.x, row0 = 32 * (b % 4), col0 = 64 * (b / 4);
      const int slot = mode == 4 ? (r % 16) : 0;
      for (int e = threadIdx.x; e < 32 * 16; e += blockDim.x) {  // 16 x 4-element groups per row
        const int rr = row0 + e / 16, cc = col0 + 4 * (e % 16);
        __nv_bfloat162* d = (__nv_bfloat162*)(src + ((size_t)slot * 128 + rr) * 2048 + cc);
        d[0] = __floats2bfloat162_rn((float)r, 1.f);
        d[1] = __floats2bfloat162_rn(2.f, 3.f);
      }
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned v = 0;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
        } while (v < (unsigned)(gridDim.x * (r + 1)));
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      const unsigned long long t0 = gt();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)),
                   "r"(131072) : "memory");
      for (int i = 0; i < 8; ++i) {
        const int col = (ks * 8 + i) * 64;
        if (mode == 0 || mode >= 3) {
          const int row = mode == 4 ? (r % 16) * 128 : 0;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(su(s + i * 16384)),
              "l"((uint64_t)(mode == 4 ? &mtape : &m128)), "r"(su(&bar)), "r"(col), "r"(row) : "memory");
        } else if (mode == 1) {
          const __nv_bfloat16* src = blocked + (size_t)(ks * 8 + i) * 8192;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
              ::"r"(su(s + i * 16384)), "l"(src), "r"(16384), "r"(su(&bar)) : "memory");
        } else {
          for (int q = 0; q < 4; ++q)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4}], [%2];" ::"r"(su(s + i * 16384 + q * 4096)),
                "l"((uint64_t)&m32), "r"(su(&bar)), "r"(col), "r"(32 * q) : "memory");
        }
      }
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     "selp.u32 %0, 1, 0, p;\n}" : "=r"(done) : "r"(su(&bar)), "r"(r & 1) : "memory");
      tot += gt() - t0;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / reps;
}

int main() {
  const int rows = 128, cols = 2048;
  __nv_bfloat16 *a, *blk;
  cudaMalloc(&a, rows * cols * 2);
  cudaMalloc(&blk, rows * cols * 2);
  cudaMemset(a, 0, rows * cols * 2);
  cudaMemset(blk, 0, rows * cols * 2);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m128, m32;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box128[2] = {64, 128}, box32[2] = {64, 32}, es[2] = {1, 1};
  enc(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, strides, box128, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, a, dims, strides, box32, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 8);
  __nv_bfloat16* tape;
  cudaMalloc(&tape, 16 * 128 * 2048 * 2);
  CUtensorMap mt;
  cuuint64_t dims_t[2] = {(cuuint64_t)cols, (cuuint64_t)16 * 128};
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, tape, dims_t, strides, box128, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned* cnt;
  cudaMalloc(&cnt, 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072 + 1024);
  for (int grid : {1, 32, 128, 148})
    for (int mode = 0; mode < 5; ++mode) {
      if (mode >= 3 && grid != 128) continue;
      cudaMemset(cnt, 0, 4);
      // (mode 3 writes the 2-D source the 128-row map reads: a)
      k<<<grid, 128, 131072 + 1024>>>(m128, m32, blk, mode, 20, out, mode == 3 ? a : tape, cnt, mt);
      cudaDeviceSynchronize();
      std::vector<unsigned long long> h(grid);
      cudaMemcpy(h.data(), out, grid * 8, cudaMemcpyDeviceToHost);
      double m = 0;
      for (auto v : h) m += (double)v;
      m /= grid;
      printf("grid %3d mode %d (%s): %.0f ns per 128 KB = %.1f GB/s per SM (err %s)\n", grid, mode,
             mode == 0 ? "2-D TMA 128-row boxes" : mode == 1 ? "1-D bulk 16 KB" : mode == 2 ? "2-D TMA 32-row boxes" : mode == 3 ? "fresh (same slot)" : "fresh (tape slot)",
             m, 131072.0 / m, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
