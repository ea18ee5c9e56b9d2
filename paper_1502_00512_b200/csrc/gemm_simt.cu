// fp32 SIMT GEMM for the parity precision mode (DL_FP32).
//
// Replaces mat.hpp:116-184 (matmul_nt / matmul_nn / matmul_tn_add) when the
// caller needs reference-grade fp32 numbers: every product is accumulated
// in fp32 FMA over a fixed k order (reference: double accumulation, rounded
// once), which stays within the 1e-4 relative tolerance of the north star.
// The throughput path is the tcgen05 kernel in gemm_tc.cu.
#include "common.cuh"

namespace dl {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, TPB = 256;

__global__ void __launch_bounds__(TPB)
gemm_f32_kernel(GemmDesc g, int kchunk) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const float* A = static_cast<const float*>(g.A);
  const float* B = static_cast<const float*>(g.B);
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int kb = blockIdx.z * kchunk;
  const int ke = min(g.K, kb + kchunk);

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  for (int k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int i = 0; i < (BM * BK) / TPB; ++i) {
      const int e = tid + i * TPB;
      int m, k;
      if (g.a_major == K_MAJOR) { m = e / BK; k = e % BK; }
      else { k = e / BM; m = e % BM; }
      const int gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gm < g.M && gk < ke)
        v = g.a_major == K_MAJOR ? A[(int64_t)gm * g.lda + gk]
                                 : A[(int64_t)gk * g.lda + gm];
      As[k][m] = v;
    }
#pragma unroll
    for (int i = 0; i < (BN * BK) / TPB; ++i) {
      const int e = tid + i * TPB;
      int n, k;
      if (g.b_major == K_MAJOR) { n = e / BK; k = e % BK; }
      else { k = e / BN; n = e % BN; }
      const int gn = n0 + n, gk = k0 + k;
      float v = 0.f;
      if (gn < g.N && gk < ke)
        v = g.b_major == K_MAJOR ? B[(int64_t)gn * g.ldb + gk]
                                 : B[(int64_t)gk * g.ldb + gn];
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  float* C = g.C + (int64_t)blockIdx.z * g.split_stride;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= g.N) continue;
      float v = acc[i][j];
      if (g.do_clip) {
        v = clip1(v, g.clip);
        bad |= !isfinite(v);
      }
      C[(int64_t)m * g.ldc + n] = v;
    }
  }
  if (g.do_clip && g.nonfinite && __syncthreads_or(bad) && tid == 0)
    atomicExch(g.nonfinite, 1);
}

}  // namespace

void gemm_f32(const GemmDesc& g, cudaStream_t st) {
  const int splits = g.k_splits < 1 ? 1 : g.k_splits;
  int kchunk = (g.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM, splits);
  gemm_f32_kernel<<<grid, TPB, 0, st>>>(g, kchunk);
  DL_CUDA(cudaGetLastError());
}

}  // namespace dl
