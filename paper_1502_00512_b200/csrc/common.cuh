// Shared internals of libdesklm_cuda.so (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace dl {

using bf16 = __nv_bfloat16;

// Status-carrying exception used inside the runtime; mapped to DL_E* codes
// at the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define DL_CUDA(x)                                                        \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess)                                                \
      throw ::dl::Error(3, std::string("CUDA: ") + cudaGetErrorString(e_) + \
                               " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

#define DL_REQUIRE(cond, code, msg) \
  do {                              \
    if (!(cond)) throw ::dl::Error((code), (msg)); \
  } while (0)

constexpr int kNumSMs = 148;

// Operand storage order for the generic GEMMs.  A is M x K, B is N x K
// logically; K_MAJOR means K is the contiguous index (row-major [M][K]),
// MN_MAJOR means M (or N) is contiguous (row-major [K][M]).
enum Major : int { K_MAJOR = 0, MN_MAJOR = 1 };

__device__ __forceinline__ float act_f(int act, float x) {
  // rnn.hpp:37-42 (float): 1/(1+exp(-x)) or tanh
  return act == 0 ? 1.0f / (1.0f + expf(-x)) : tanhf(x);
}
__device__ __forceinline__ float act_deriv_f(int act, float y) {
  // rnn.hpp:45-49, expressed through the output y
  return act == 0 ? y * (1.0f - y) : 1.0f - y * y;
}
// std::min(c, std::max(-c, x)): NaN maps to -c exactly like the reference
// (rnn.hpp:131-134 with std::max/min's comparison order).
__device__ __forceinline__ float clip1(float x, float c) {
  const float t = (-c < x) ? x : -c;
  return (t < c) ? t : c;
}

// float(eta * g / denom) exactly as the reference computes it (double
// multiply, IEEE double divide, round to float), with one reciprocal per row
// instead of a divide per element: q*inv is within 1.5 double ulps of the
// correctly rounded quotient, so rounding it to float gives the same float
// unless the quotient lies within a few double ulps of a float rounding
// midpoint -- only then is the exact division performed.
__device__ __forceinline__ float rms_step(double eta, float g, double denom, double inv) {
  const double q = eta * (double)g;
  const double r = q * inv;
  const float f = (float)r;
  const float af = fabsf(f);
  if (!(af < 3.0e38f) || af < 1.0e-30f) return (float)(q / denom);  // inf/NaN/tiny: exact
  const double up = (double)__int_as_float(__float_as_int(af) + 1) - (double)af;
  const double dn = (double)af - (double)__int_as_float(__float_as_int(af) - 1);
  const double ar = fabs(r), fd = (double)af;
  const double tol = ar * 0x1p-49;
  if (fabs(ar - (fd + 0.5 * up)) <= tol || fabs(ar - (fd - 0.5 * dn)) <= tol)
    return (float)(q / denom);
  return f;
}

// ---------------------------------------------------------------- launches
// GEMM problem description shared by the SIMT (fp32) and tcgen05 (bf16)
// kernels.  C (+ split * split_stride) receives fp32 results; for k_splits>1
// the caller reduces the slices.
// dS of one logit (backprop.hpp:179-186) from the row's lse (fp32) and
// scale: scale * 2^((s - lse) log2 e); the target column subtracts the scale
// afterwards.  Shared by the in-place softmax rows kernel and the dh GEMM's
// operand transform so both produce the same bits.
constexpr float kDsLog2e = 1.4426950408889634f;
__device__ __forceinline__ float ds_of_logit(float s, float lse, float sc) {
  return sc * exp2f((s - lse) * kDsLog2e);
}

struct GemmDesc {
  int M, N, K;
  int a_major, b_major;
  const void* A;  // float* (fp32 path) or bf16* (tc path)
  const void* B;
  int64_t lda, ldb;  // elements between consecutive rows of the stored matrix
  float* C;
  int64_t ldc;
  int64_t split_stride;
  int k_splits;
  // optional fused clip (only valid with k_splits == 1)
  float clip;
  int do_clip;
  int* nonfinite;  // set to 1 if any clipped value is non-finite
  // logits epilogue (tc path): per-row online (max, sum-exp) partials per
  // N tile, the target logit and an optional bf16 copy of the logits.
  int logits;
  bf16* S;
  int64_t lds;
  float2* part;          // [n_tiles][M]
  const uint32_t* tgt;   // [M] target column per row
  float* tgt_logit;      // [M]
  // shifted-exponential logits (bf16 trainer path, "pfac"): with shift set
  // the epilogue stores E = 2^(min((s - shift[r]) log2 e, 120)) in bf16
  // instead of s, and the partials become (tile max of s, sum of E)
  const float* shift;
  int part_n;            // (shift) partials per row: part is [M][part_n]
  // fp32 epilogue: row r of the product is multiplied by row_scale[r]
  // (the dh GEMM over E: dS = diag(row_scale) E)
  const float* row_scale;
  // + row_resid[r] * resid_w[resid_idx[r]][n] (bf16 rows, ld = N): the part
  // of the target column's dS that E' rounded away (k_pfac_rows), so dh's
  // dominant term is formed in fp32
  const float* row_resid;
  const uint32_t* resid_idx;
  const bf16* resid_w;
  int raster;            // 0: M-tiles fastest, 1: N-tiles fastest
  int no_pair;           // 1: keep the single-CTA kernel (no cta_group::2 tiles)
  // bf16 gradient epilogue (dW_out in throughput mode): clipped values to Cb
  // (ld = ldc) and per-(half N tile, row) sums of squares to rowsq
  // [2*n_tiles][M] (double), for the dense rmsprop's mean_sq
  bf16* Cb;
  double* rowsq;
  // fused dense rmsprop (dW_out, bf16 trainer path; rmsprop.hpp:94-107):
  // the epilogue clips, publishes per-(half N tile, row) sums of squares to
  // rowsq, waits on rms_cnt[M block] until every N tile of its rows has
  // published, then updates the fp32 master rms_w, the bf16 shadow rms_wb
  // and m_out rms_m in place.  The gradient is never stored.
  int rms;
  float* rms_w;
  bf16* rms_wb;
  float* rms_m;
  unsigned* rms_cnt;  // [ceil(M / 256)], zero at launch
  double rho, eps, eta;
  // dS on the fly (the dh GEMM over bf16 logits, A K-major; pair tiles):
  // each A tile is rewritten in shared memory before the MMAs as
  //   bf16(xf_sc[r] * exp2((s - xf_lse[r]) * log2 e) - (k == xf_tgt[r] ? xf_sc[r] : 0))
  // (backprop.hpp:179-186) and the CTAs of N tile 0 store it to xf_out
  // (ld = lda) for the dW_out GEMM.
  int xf;
  const float* xf_lse;
  const float* xf_sc;
  const uint32_t* xf_tgt;
  bf16* xf_out;
  unsigned long long* trace;  // DL_GEMM_TRACE diagnostics (fused kernel), or null
  int trace_warps;            // DL_GEMM_TRACE_WARPS: trace three warps of one CTA
};

// whether gemm_tc runs an M x N GEMM on CTA-pair tiles (the xf transform
// and the fused rmsprop epilogue exist only there)
bool tc_pair_tiles(int M, int N);

// 3xTF32 tensor-core GEMM for the fp32 parity mode (gemm_tc.cu): same
// GemmDesc contract as gemm_f32 (fp32 operands and output, clip / split-K)
bool tf32x3_ok(const GemmDesc& g);
int tf32_splits(int K, int desired);
int gemm_tf32x3(const GemmDesc& g, cudaStream_t st);

// gemm_simt.cu
void gemm_f32(const GemmDesc& g, cudaStream_t st);
// gemm_tc.cu  (returns the number of N-tiles used for logits partials)
int gemm_tc(const GemmDesc& g, cudaStream_t st);
int tc_n_tiles(int N);
int tc_splits(int K, int desired);
bool tc_rms_fusable(int M, int N);

}  // namespace dl
