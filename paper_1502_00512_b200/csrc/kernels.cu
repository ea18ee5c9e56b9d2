// Bandwidth-bound kernels of the RNNLM window: recurrence epilogues (split-K
// reduction + embedding gather + activation), softmax/LSE rows, the sparse
// embedding gradient, clip/finite, rmsprop and the device-side offset-stream
// schedule.  Each kernel cites the reference code it replaces (paths
// relative to /root/reference/proj/include/desklm).
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include <cstdlib>

#include "kernels.cuh"

namespace dl {
namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide deterministic reductions (fixed tree for a fixed block size).
template <int NT>
__device__ double block_sum_d(double v, double* red) {
  v = warp_sum_d(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < NT / 32 ? red[l] : 0.0;
    v = warp_sum_d(v);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}
template <int NT>
__device__ double block_max_d(double v, double* red) {
  v = warp_max_d(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < NT / 32 ? red[l] : -INFINITY;
    v = warp_max_d(v);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// max of a and sum of b over the block in one pass (fixed tree)
template <int NT>
__device__ void block_max_sum_d(double& a, double& b, double* red) {
  a = warp_max_d(a);
  b = warp_sum_d(b);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) { red[w] = a; red[16 + w] = b; }
  __syncthreads();
  if (w == 0) {
    double x = l < NT / 32 ? red[l] : -INFINITY;
    double y = l < NT / 32 ? red[16 + l] : 0.0;
    x = warp_max_d(x);
    y = warp_sum_d(y);
    if (l == 0) { red[0] = x; red[16] = y; }
  }
  __syncthreads();
  a = red[0];
  b = red[16];
}

// ---------------------------------------------------------------- casts
__global__ void k_f32_to_bf16(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

__global__ void k_fill_f32(float* __restrict__ x, float v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// ------------------------------------------------------- recurrence steps
// Forward step epilogue (backprop.hpp:102-112, rnn.hpp:209-216):
//   pre = sum_s partial[s] (fixed order), rounded to float;
//   pre += W_in[x_b] (float);  h = act(pre)
__global__ void k_rec_fwd(const float* __restrict__ part, int splits, int64_t split_stride,
                          int64_t Bn, int64_t H, const float* __restrict__ w_in,
                          const uint32_t* __restrict__ x, int act, float* __restrict__ h,
                          bf16* __restrict__ hb) {
  const int64_t n = Bn * H;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / H, j = i % H;
    float pre = part[i];
    for (int s = 1; s < splits; ++s) pre += part[s * split_stride + i];
    pre += w_in[(int64_t)x[b] * H + j];
    const float y = act_f(act, pre);
    h[i] = y;
    if (hb) hb[i] = __float2bfloat16_rn(y);
  }
}

// Backward step epilogue (backprop.hpp:207-218):
//   dh = dh_out_t (+ sum_s partial[s] = dpre_{t+1} . W_rec when chained)
//   dpre = dh * act'(h_{t+1})
__global__ void k_rec_bwd(const float* __restrict__ part, int splits, int64_t split_stride,
                          int64_t n, const float* __restrict__ dh_out,
                          const float* __restrict__ hnext, int act, float* __restrict__ dpre,
                          bf16* __restrict__ dpreb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float dh = 0.f;
    if (splits > 0) {
      dh = part[i];
      for (int s = 1; s < splits; ++s) dh += part[s * split_stride + i];
    }
    dh += dh_out[i];
    const float d = dh * act_deriv_f(act, hnext[i]);
    dpre[i] = d;
    if (dpreb) dpreb[i] = __float2bfloat16_rn(d);
  }
}

// Split-K reduction with optional clip and finite flag (dW_rec, dh_out).
__global__ void k_reduce(const float* __restrict__ part, int splits, int64_t split_stride,
                         int64_t n, float* __restrict__ out, float clip, int do_clip,
                         int* nonfinite) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float v = part[i];
    for (int s = 1; s < splits; ++s) v += part[s * split_stride + i];
    if (do_clip) {
      v = clip1(v, clip);
      bad |= !isfinite(v);
    }
    out[i] = v;
  }
  if (do_clip && nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
}

// The dW_rec split-K reduction + clip (rnn.hpp:158-159) with the W_rec
// rmsprop step (rmsprop.hpp:113-133, k_rms_rec's arithmetic) in the same
// pass, for the trainer path with a finite clip (every clipped component
// finite: the all-finite check cannot fail); g_rec is still written.
__global__ void k_reduce_rms_rec(const float* __restrict__ part, int splits, int64_t split_stride,
                                 int64_t n, float* __restrict__ g_out, float clip,
                                 float* __restrict__ w, bf16* __restrict__ wb,
                                 float* __restrict__ m, double rho, double eps, double eta) {
  auto one = [&](float& wi, float& mi, float gf) {
    const double gi = (double)gf;
    mi = (float)(rho * (double)mi + (1.0 - rho) * gi * gi);
    wi = wi - (float)(eta * gi / sqrt((double)mi + eps));
  };
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4* p4 = reinterpret_cast<const float4*>(part);
    float4 v = p4[i];
#pragma unroll 4
    for (int sp = 1; sp < splits; ++sp) {
      const float4 q = p4[sp * (split_stride / 4) + i];
      v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
    }
    v = make_float4(clip1(v.x, clip), clip1(v.y, clip), clip1(v.z, clip), clip1(v.w, clip));
    reinterpret_cast<float4*>(g_out)[i] = v;
    float4 mq = reinterpret_cast<float4*>(m)[i];
    float4 wq = reinterpret_cast<float4*>(w)[i];
    one(wq.x, mq.x, v.x);
    one(wq.y, mq.y, v.y);
    one(wq.z, mq.z, v.z);
    one(wq.w, mq.w, v.w);
    reinterpret_cast<float4*>(m)[i] = mq;
    reinterpret_cast<float4*>(w)[i] = wq;
    if (wb) {
      __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(wb + 4 * i);
      b2[0] = __floats2bfloat162_rn(wq.x, wq.y);
      b2[1] = __floats2bfloat162_rn(wq.z, wq.w);
    }
  }
}

// ---------------------------------------------------------- softmax rows
// fp32 path: S holds fp32 logits [M x V].  Per row (backprop.hpp:162-186):
//   mx = max_w s (double), z = sum exp(s - mx) (double), lse = mx + log z
//   loss_row = w ? scale*(lse - s_y) : 0 ;  logp_row = s_y - lse
//   grads: dS = w ? float(scale*exp(s - lse)) - [w==y] float(scale) : 0
constexpr int kRowThreads = 512;
#ifndef DL_SOFTMAX_UNROLL
#define DL_SOFTMAX_UNROLL 4  // 16-byte loads in flight per thread in the dS pass
#endif

// Vocabulary-sharded rows: every rank holds a V/G column
// block of the logits.  lse over the full vocabulary is the log-sum-exp of
// the G block lse values (gathered, rank order); the target logit was summed
// over ranks (only its owner contributes).
__device__ __forceinline__ double lse_of_blocks(const double* __restrict__ lse_all, int G,
                                                int64_t M, int64_t r) {
  double mx = -INFINITY;
  for (int g = 0; g < G; ++g) mx = fmax(mx, lse_all[g * M + r]);
  double z = 0.0;
  for (int g = 0; g < G; ++g) z += exp(lse_all[g * M + r] - mx);
  return mx + log(z);
}

__global__ void __launch_bounds__(kRowThreads)
k_softmax_rows_f32(float* __restrict__ S, int64_t V, int64_t M, const uint32_t* __restrict__ tgt,
                   const uint8_t* __restrict__ wts, double scale, int grads,
                   double* __restrict__ loss_row, double* __restrict__ logp_row,
                   const double* __restrict__ lse_all, int G, const float* __restrict__ tgt_logit) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  float* s = S + r * V;
  const bool active = wts == nullptr || wts[r] != 0;
  if (!active) {
    if (loss_row) loss_row[r] = 0.0;
    if (logp_row) logp_row[r] = NAN;
    if (grads)
      for (int64_t w = threadIdx.x; w < V; w += blockDim.x) s[w] = 0.f;
    return;
  }
  double lse;
  if (lse_all) {
    lse = lse_of_blocks(lse_all, G, M, r);
  } else {
    double mx = -INFINITY;
    for (int64_t w = threadIdx.x; w < V; w += blockDim.x) mx = fmax(mx, (double)s[w]);
    mx = block_max_d<kRowThreads>(mx, red);
    double z = 0.0;
    for (int64_t w = threadIdx.x; w < V; w += blockDim.x) z += exp((double)s[w] - mx);
    z = block_sum_d<kRowThreads>(z, red);
    lse = mx + log(z);
  }
  const uint32_t y = tgt[r];  // sharded: column inside this block, or ~0u
  const double sy = lse_all ? (double)tgt_logit[r] : (double)s[y];
  if (threadIdx.x == 0) {
    if (loss_row) loss_row[r] = scale * (lse - sy);
    if (logp_row) logp_row[r] = sy - lse;
  }
  if (grads) {
    __syncthreads();  // everyone has read s[y]
    for (int64_t w = threadIdx.x; w < V; w += blockDim.x) {
      float d = (float)(scale * exp((double)s[w] - lse));
      if (w == y) d -= (float)scale;
      s[w] = d;
    }
  }
}

// bf16 path: the tcgen05 logits epilogue left per-(N tile, row) partials
// (max, sum-exp) and the fp32 target logit; combine them into lse, then
// overwrite the bf16 logits with bf16 dS in place.
__global__ void __launch_bounds__(kRowThreads)
k_softmax_rows_bf16(bf16* __restrict__ S, int64_t V, int64_t M, const float2* __restrict__ part,
                    int n_tiles, const float* __restrict__ tgt_logit,
                    const uint32_t* __restrict__ tgt, const uint8_t* __restrict__ wts,
                    double scale, int grads, double* __restrict__ loss_row,
                    double* __restrict__ logp_row, const double* __restrict__ lse_all, int G) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  bf16* s = S ? S + r * V : nullptr;
  const bool active = wts == nullptr || wts[r] != 0;
  if (!active) {
    if (threadIdx.x == 0) {
      if (loss_row) loss_row[r] = 0.0;
      if (logp_row) logp_row[r] = NAN;
    }
    if (grads) {
      const bf16 z = __float2bfloat16_rn(0.f);
      for (int64_t w = threadIdx.x; w < V; w += blockDim.x) s[w] = z;
    }
    return;
  }
  double lse;
  if (lse_all) {
    lse = lse_of_blocks(lse_all, G, M, r);
  } else {
    double mx = -INFINITY;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
      mx = fmax(mx, (double)part[r * n_tiles + t].x);
    mx = block_max_d<kRowThreads>(mx, red);
    double z = 0.0;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
      const float2 p = part[r * n_tiles + t];
      if (p.y > 0.f) z += (double)p.y * exp((double)p.x - mx);
    }
    z = block_sum_d<kRowThreads>(z, red);
    lse = mx + log(z);
  }
  const double sy = (double)tgt_logit[r];
  if (threadIdx.x == 0) {
    if (loss_row) loss_row[r] = scale * (lse - sy);
    if (logp_row) logp_row[r] = sy - lse;
  }
  if (grads) {
    const uint32_t y = tgt[r];
    const float lsef = (float)lse, scf = (float)scale;

    if ((V % 8) == 0) {
      // four 16-byte loads in flight per thread before any store (the row
      // streams at HBM speed only with enough bytes outstanding)
      uint4* s8 = reinterpret_cast<uint4*>(s);
      const int64_t n8 = V / 8;
      constexpr int U = DL_SOFTMAX_UNROLL;
      for (int64_t q0 = threadIdx.x; q0 < n8; q0 += (int64_t)U * blockDim.x) {
        uint4 u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int64_t q = q0 + (int64_t)j * blockDim.x;
          if (q < n8) u[j] = __ldcs(s8 + q);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int64_t q = q0 + (int64_t)j * blockDim.x;
          if (q >= n8) continue;
          __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u[j]);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            float2 f = __bfloat1622float2(h2[k]);
            const int64_t w0 = q * 8 + 2 * k;
            f.x = ds_of_logit(f.x, lsef, scf) - (w0 == y ? scf : 0.f);
            f.y = ds_of_logit(f.y, lsef, scf) - (w0 + 1 == y ? scf : 0.f);
            h2[k] = __float22bfloat162_rn(f);
          }
          s8[q] = u[j];
        }
      }
    } else {
      for (int64_t w = threadIdx.x; w < V; w += blockDim.x) {
        const float f = __bfloat162float(s[w]);
        s[w] = __float2bfloat16_rn(ds_of_logit(f, lsef, scf) - (w == y ? scf : 0.f));
      }
    }
  }
}

// The row half of k_softmax_rows_bf16 when dS is formed on the fly in the
// dh GEMM's operand path (gemm_tc.cu, GemmDesc::xf): per row the
// log-sum-exp from the logits epilogue's partials (backprop.hpp:168-178),
// loss / log-prob, and the transform's constants lse (fp32, as the in-place
// kernel uses it) and the row scale (0 for masked rows).
__global__ void __launch_bounds__(kRowThreads)
k_lse_rows_bf16(int64_t M, const float2* __restrict__ part, int n_tiles,
                const float* __restrict__ tgt_logit, const uint8_t* __restrict__ wts,
                double scale, double* __restrict__ loss_row, double* __restrict__ logp_row,
                float* __restrict__ lse_f, float* __restrict__ sc_f,
                const double* __restrict__ lse_all, int G) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const bool active = wts == nullptr || wts[r] != 0;
  if (!active) {
    if (threadIdx.x == 0) {
      if (loss_row) loss_row[r] = 0.0;
      if (logp_row) logp_row[r] = NAN;
      lse_f[r] = 0.f;
      sc_f[r] = 0.f;
    }
    return;
  }
  double lse;
  if (lse_all) {
    lse = lse_of_blocks(lse_all, G, M, r);
  } else {
    double mx = -INFINITY;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
      mx = fmax(mx, (double)part[r * n_tiles + t].x);
    mx = block_max_d<kRowThreads>(mx, red);
    double z = 0.0;
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
      const float2 p = part[r * n_tiles + t];
      if (p.y > 0.f) z += (double)p.y * exp((double)p.x - mx);
    }
    z = block_sum_d<kRowThreads>(z, red);
    lse = mx + log(z);
  }
  if (threadIdx.x == 0) {
    const double sy = (double)tgt_logit[r];
    if (loss_row) loss_row[r] = scale * (lse - sy);
    if (logp_row) logp_row[r] = sy - lse;
    lse_f[r] = (float)lse;
    sc_f[r] = (float)scale;
  }
}

// ------------------------------------------- shifted-exponential softmax
// The bf16 trainer's output layer without a pass over the logits
// (backprop.hpp:157-189 restated): the logits GEMM epilogue stores
// E = e^(s - c_r) in bf16 for a per-row shift c_r fixed before the GEMM, so
//   p = e^(s - lse) = E * e^(c_r - lse)   and   dS = scale (p - 1[y])
//                                              = diag(sigma) E'
// with sigma_r = scale e^(c_r - lse_r) and E' = E except at the target
// column, which k_pfac_rows overwrites with (p_y - 1) / e^(c_r - lse_r)
// (computed from the fp32 target logit, not from the rounded E).  The row
// factor then moves out of both gradient GEMMs: dh = diag(sigma) (E' W_out)
// (the dh epilogue's row_scale) and dW_out = E'^T (diag(sigma) Hs) (its B
// operand scaled once: TB x H values instead of TB x V).
//
// c_r = the row's target logit (dot of the bf16 operands the GEMM uses):
// E stays within range for every logit less than 83 nats above the
// target's (the epilogue caps the exponent at 2^120 and redoes a half tile
// past the cap against its own maximum); a row with such a tile or whose
// sum of E exceeds e^40 (sigma = scale e^(c - lse) would underflow) is
// rescaled to one new shift (pfac_row_lse).
__global__ void __launch_bounds__(256)
k_target_shift(const bf16* __restrict__ hs, const bf16* __restrict__ w, int64_t H, int64_t M,
               const uint32_t* __restrict__ tgt, int64_t V, float* __restrict__ shift) {
  const int64_t r = blockIdx.x * 8 + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (r >= M) return;
  const uint32_t y = tgt[r];
  float acc = 0.f;
  if (y < V) {
    const bf16* a = hs + r * H;
    const bf16* b = w + (int64_t)y * H;
    if ((H % 8) == 0) {
      for (int64_t k = 8 * lane; k < H; k += 256) {
        const uint4 qa = *reinterpret_cast<const uint4*>(a + k);
        const uint4 qb = *reinterpret_cast<const uint4*>(b + k);
        const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&qa);
        const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&qb);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 fa = __bfloat1622float2(pa[j]), fb = __bfloat1622float2(pb[j]);
          acc = fmaf(fa.x, fb.x, acc);
          acc = fmaf(fa.y, fb.y, acc);
        }
      }
    } else {
      for (int64_t k = lane; k < H; k += 32)
        acc = fmaf(__bfloat162float(a[k]), __bfloat162float(b[k]), acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) shift[r] = acc;
}

constexpr int kPfacThreads = 256;

// The row's log-sum-exp relative to its shift from the logits epilogue's
// partials (row-major [M][n_tiles]: .x the half tile's shift offset in
// nats -- 0 unless one of its logits was more than 83 nats above the shift
// and the epilogue redid it against its own maximum -- .y its sum of E).
// A row with an offset tile, or whose sum exceeds e^repair_nats (a target
// far less likely than the rest of the row: sigma = scale e^(c - lse) would
// leave fp32's range), is rescaled in place to E / z = p with one factor
// per half tile, the shift becoming the lse itself -- one streaming pass
// over the row, nothing recomputed.  repaired[0] counts those rows,
// repaired[1] the ones with offset tiles.  pw: columns per partial.
// Block-uniform.
__device__ void pfac_row_lse(bf16* erow, int64_t V, int64_t r, const float2* __restrict__ part,
                             int n_tiles, int pw, double& c, double& z, float repair_nats,
                             int* repaired, double* red, float* fac) {
  const float2* pr = part + r * n_tiles;
  // the offsets' maximum and the plain sum in one reduction (offsets are 0
  // but in the rare redone tiles)
  double om = 0.0;
  z = 0.0;
  for (int t = threadIdx.x; t < n_tiles; t += kPfacThreads) {
    const float2 q = pr[t];
    om = fmax(om, (double)q.x);
    z += (double)q.y;
  }
  block_max_sum_d<kPfacThreads>(om, z, red);
  if (om > 0.0) {
    z = 0.0;
    for (int t = threadIdx.x; t < n_tiles; t += kPfacThreads)
      z += (double)pr[t].y * exp((double)pr[t].x - om);
    z = block_sum_d<kPfacThreads>(z, red);
  }
  if (om == 0.0 && log(z) <= (double)repair_nats) return;
  // tile t's elements are e^(s - c - x_t): times e^(x_t - om - ln z) they
  // become e^(s - lse)
  const double lz = log(z);
  for (int t = threadIdx.x; t < n_tiles; t += kPfacThreads)
    fac[t] = (float)exp((double)pr[t].x - om - lz);
  __syncthreads();
  for (int64_t v = threadIdx.x; v < V; v += kPfacThreads)
    erow[v] = __float2bfloat16_rn(__bfloat162float(erow[v]) * fac[v / pw]);
  c += om + lz;
  z = 1.0;
  if (threadIdx.x == 0 && repaired) atomicAdd(repaired + (om > 0.0 ? 1 : 0), 1);
  __syncthreads();  // (fac is reused by the caller's next row)
}

// Vocabulary-sharded output layer: this rank's block log-sum-exp (after the
// repair), exchanged before k_pfac_rows; shift[r] updated when repaired.
__global__ void __launch_bounds__(kPfacThreads)
k_pfac_lse(bf16* __restrict__ E, int64_t V, int64_t M, const float2* __restrict__ part,
           int n_tiles, int pw, const uint8_t* __restrict__ wts, float* __restrict__ shift,
           double* __restrict__ lse_loc, float repair_nats, int* __restrict__ repaired) {
  extern __shared__ float fac[];
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const bool active = wts == nullptr || wts[r] != 0;
  double c = (double)shift[r], z;
  pfac_row_lse(E + r * V, V, r, part, n_tiles, pw, c, z, active ? repair_nats : INFINITY,
               repaired, red, fac);
  if (threadIdx.x == 0) {
    lse_loc[r] = c + log(z);
    shift[r] = (float)c;
  }
}

__global__ void __launch_bounds__(kPfacThreads)
k_pfac_rows(bf16* __restrict__ E, int64_t V, int64_t M, int64_t H, const float2* __restrict__ part,
            int n_tiles, int pw, const float* __restrict__ tgt_logit, const uint32_t* __restrict__ tgt,
            const uint8_t* __restrict__ wts, double scale, double* __restrict__ loss_row,
            double* __restrict__ logp_row, const float* __restrict__ shift,
            float* __restrict__ sigma, float* __restrict__ resid, const float* __restrict__ hs,
            bf16* __restrict__ hs_sc, const bf16* __restrict__ hs_bf, float repair_nats,
            int* __restrict__ repaired, const double* __restrict__ lse_all, int G) {
  extern __shared__ float fac[];
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const bool active = wts == nullptr || wts[r] != 0;
  bf16* hrow = hs_sc + r * H;
  if (!active) {
    // dS row = 0: sigma = 0 and a zero row of the scaled B operand (E stays
    // finite: its exponent is capped in the epilogue)
    if (threadIdx.x == 0) {
      if (loss_row) loss_row[r] = 0.0;
      if (logp_row) logp_row[r] = NAN;
      sigma[r] = 0.f;
      resid[r] = 0.f;
    }
    const bf16 z = __float2bfloat16_rn(0.f);
    for (int64_t k = threadIdx.x; k < H; k += kPfacThreads) hrow[k] = z;
    return;
  }
  double c = (double)shift[r], lse;
  bf16* erow = E + r * V;
  if (lse_all) {
    lse = lse_of_blocks(lse_all, G, M, r);  // (shift repaired by k_pfac_lse)
  } else {
    double z;
    pfac_row_lse(erow, V, r, part, n_tiles, pw, c, z, repair_nats, repaired, red, fac);
    lse = c + log(z);
  }
  const double sy = (double)tgt_logit[r];
  const float sg = (float)(scale * exp(c - lse));
  if (threadIdx.x == 0) {
    if (loss_row) loss_row[r] = scale * (lse - sy);
    if (logp_row) logp_row[r] = sy - lse;
    sigma[r] = sg;
    // the target column (its owner's block): sigma * E'[y] = scale (p_y - 1);
    // what the bf16 rounding of E'[y] loses goes to the dh epilogue as resid
    // (dW_out keeps the rounded value: an error of the order of its bf16 Hs)
    const uint32_t y = tgt[r];
    float rsd = 0.f;
    if (y < V) {
      const double ds = scale * expm1(sy - lse);
      const bf16 e = __float2bfloat16_rn(sg > 0.f ? (float)(ds / (double)sg) : 0.f);
      erow[y] = e;
      rsd = (float)(ds - (double)sg * (double)__bfloat162float(e));
    }
    resid[r] = rsd;
  }
  // the dW_out GEMM's B operand: diag(sigma) Hs, rounded once to bf16 (from
  // the bf16 copy when the fp32 rows are not at hand: gathered windows)
  for (int64_t k = threadIdx.x; k < H; k += kPfacThreads)
    hrow[k] = __float2bfloat16_rn(sg * (hs ? hs[r * H + k] : __bfloat162float(hs_bf[r * H + k])));
}

// Sharded output layer helpers.  Targets inside [v0, v0 + Vo) become local
// columns, all others ~0u (matches no column).
__global__ void k_shard_targets(const uint32_t* __restrict__ y, int64_t M, int64_t v0, int64_t Vo,
                                uint32_t* __restrict__ loc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = (int64_t)y[i] - v0;
    loc[i] = (l >= 0 && l < Vo) ? (uint32_t)l : ~0u;
  }
}

// Block log-sum-exp of one row from the tcgen05 epilogue's partials.
__global__ void __launch_bounds__(256)
k_block_lse_bf16(const float2* __restrict__ part, int n_tiles, int64_t M,
                 double* __restrict__ lse) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  double mx = -INFINITY;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x)
    mx = fmax(mx, (double)part[r * n_tiles + t].x);
  mx = block_max_d<256>(mx, red);
  double z = 0.0;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const float2 p = part[r * n_tiles + t];
    if (p.y > 0.f) z += (double)p.y * exp((double)p.x - mx);
  }
  z = block_sum_d<256>(z, red);
  if (threadIdx.x == 0) lse[r] = mx + log(z);
}

// fp32: block log-sum-exp in double over the row's Vo logits, plus the
// target logit (0 when the target is not in this block).
__global__ void __launch_bounds__(kRowThreads)
k_block_lse_f32(const float* __restrict__ S, int64_t V, const uint32_t* __restrict__ loc,
                double* __restrict__ lse, float* __restrict__ tgt_logit) {
  __shared__ double red[32];
  const int64_t r = blockIdx.x;
  const float* s = S + r * V;
  double mx = -INFINITY;
  for (int64_t w = threadIdx.x; w < V; w += blockDim.x) mx = fmax(mx, (double)s[w]);
  mx = block_max_d<kRowThreads>(mx, red);
  double z = 0.0;
  for (int64_t w = threadIdx.x; w < V; w += blockDim.x) z += exp((double)s[w] - mx);
  z = block_sum_d<kRowThreads>(z, red);
  if (threadIdx.x == 0) {
    lse[r] = mx + log(z);
    const uint32_t y = loc[r];
    tgt_logit[r] = y < V ? s[y] : 0.f;
  }
}

// Deterministic sum of per-row losses (fixed order / fixed tree) and count
// of scored rows; accumulates into acc[0] (loss) and cnt[0].
__global__ void k_sum_rows(const double* __restrict__ v, const uint8_t* __restrict__ wts,
                           int64_t n, double* acc, unsigned long long* cnt) {
  __shared__ double red[32];
  double s = 0.0, c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    s += v[i];
    c += (wts == nullptr || wts[i]) ? 1.0 : 0.0;
  }
  s = block_sum_d<1024>(s, red);
  c = block_sum_d<1024>(c, red);
  if (threadIdx.x == 0) {
    acc[0] += s;
    if (cnt) cnt[0] += (unsigned long long)c;
  }
}

// ------------------------------------------------------- embedding grads
// SparseRowGrads for W_in (rnn.hpp:89-127, input_backward rnn.hpp:218-222):
// positions are sorted by (word, processing order) where the processing
// order of position (t, b) is (T-1-t)*B + b (the backward loop runs t
// descending, b ascending), so every word's row is summed in exactly the
// reference's float order.
// With G data-parallel ranks the gathered window is rank-blocked ([G][T][B])
// and the global stream index is r*B + b, so processing order i maps to
// t = T-1 - i/(G*B), r = (i % (G*B)) / B, b = i % B.
constexpr int kSortThreads = 1024;
constexpr int kEmbedShort = 64;  // segments up to this many rows: k_embed_short

__device__ __forceinline__ int64_t gathered_pos(int64_t i, int64_t T, int64_t B, int64_t G) {
  const int64_t GB = G * B;
  const int64_t t = T - 1 - i / GB, bg = i % GB;
  return (bg / B) * T * B + t * B + (bg % B);
}

// Sort by a stable block radix sort on the word id (values = processing
// index, so equal words keep processing order), for n <= 1024 * IPT
// positions; emits segment heads, words and the position order.
template <int IPT>
struct EmbedRadix {
  using Sort = cub::BlockRadixSort<uint32_t, kSortThreads, IPT, int>;
  using Scan = cub::BlockScan<int, kSortThreads>;
  struct Smem {
    union {
      typename Sort::TempStorage sort;
      typename Scan::TempStorage scan;
    } u;
    uint32_t last[kSortThreads];
  };
};

template <int IPT>
__global__ void __launch_bounds__(kSortThreads)
k_embed_radix(const uint32_t* __restrict__ x, int64_t T, int64_t B, int64_t G, int end_bit,
              int* __restrict__ seg_start, int* __restrict__ n_seg, int* __restrict__ order_pos,
              uint32_t* __restrict__ seg_word, int* __restrict__ long_list,
              int* __restrict__ n_long) {
  using R = EmbedRadix<IPT>;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  typename R::Smem& sm = *reinterpret_cast<typename R::Smem*>(sm_raw);
  const int n = (int)(G * T * B);
  const uint32_t pad = (1u << end_bit) - 1u;  // > every word id
  uint32_t key[IPT];
  int val[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = threadIdx.x * IPT + k;
    key[k] = i < n ? x[gathered_pos(i, T, B, G)] : pad;
    val[k] = i;
  }
  typename R::Sort(sm.u.sort).Sort(key, val, 0, end_bit);
  sm.last[threadIdx.x] = key[IPT - 1];
  __syncthreads();
  int head[IPT], cnt = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = threadIdx.x * IPT + k;
    const uint32_t prev = k > 0 ? key[k - 1] : (threadIdx.x > 0 ? sm.last[threadIdx.x - 1] : ~0u);
    head[k] = (i < n) && key[k] != prev;
    cnt += head[k];
  }
  int off, total;
  typename R::Scan(sm.u.scan).ExclusiveSum(cnt, off, total);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = threadIdx.x * IPT + k;
    if (i < n) {
      order_pos[i] = (int)gathered_pos(val[k], T, B, G);
      if (head[k]) {
        seg_start[off] = i;
        seg_word[off] = key[k];
        ++off;
      }
    }
  }
  if (threadIdx.x == 0) {
    *n_seg = total;
    seg_start[total] = n;
  }
  // the segments longer than kEmbedShort rows, for k_embed_long (any order)
  __shared__ int n_long_sm;
  if (threadIdx.x == 0) n_long_sm = 0;
  __syncthreads();
  for (int sl = threadIdx.x; sl < total; sl += kSortThreads)
    if (seg_start[sl + 1] - seg_start[sl] > kEmbedShort) long_list[atomicAdd(&n_long_sm, 1)] = sl;
  __syncthreads();
  if (threadIdx.x == 0) *n_long = n_long_sm;
}

// Row sums per segment in processing order, then clip (rnn.hpp:155-162),
// in two kernels by segment length:
//   k_embed_short: a warp per (segment of <= kEmbedShort rows, 1024-column
//     chunk), grid-stride; each row's columns are 8 float4 loads per lane,
//     all in flight, rows added in order;
//   k_embed_long: a block per (long segment, 32-column chunk); seven warps
//     stage the next pass of rows x 32 columns in shared memory with every
//     load in flight (lane = column) while warp 0 adds the current pass in
//     order (double-buffered).
// Both sum every word's rows in exactly the reference's float order.
constexpr int kShortWarps = 8;     // warps per k_embed_short block
constexpr int kLongPass = 7 * 24;  // rows staged per pass in k_embed_long (7 warps x 24)

__global__ void __launch_bounds__(32 * kShortWarps)
k_embed_short(const float* __restrict__ dpre, int64_t H, const int* __restrict__ seg_start,
              const int* __restrict__ n_seg, const int* __restrict__ order_pos,
              const float* __restrict__ order_scale, float* __restrict__ rows, float clip,
              int* nonfinite) {
  const int ns = __ldg(n_seg);
  const int lane = threadIdx.x % 32;
  const int64_t nchunk = (H + 1023) / 1024;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nw = (int64_t)gridDim.x * blockDim.x / 32;
  bool bad = false;
  for (int64_t w = gw; w < ns * nchunk; w += nw) {
    const int slot = (int)(w / nchunk);
    const int64_t c0 = (w % nchunk) * 1024;
    const int a = __ldg(seg_start + slot), e = __ldg(seg_start + slot + 1);
    if (e - a > kEmbedShort) continue;  // k_embed_long
    if ((H % 4) != 0) {
      // unaligned rows: one column per lane
      for (int64_t j = c0 + lane; j < min(H, c0 + 1024); j += 32) {
        float acc = 0.f;
        for (int i = a; i < e; ++i) {
          const float v = dpre[(int64_t)order_pos[i] * H + j];
          acc = __fadd_rn(acc, order_scale ? __fmul_rn(order_scale[i], v) : v);
        }
        acc = clip1(acc, clip);
        bad |= !isfinite(acc);
        rows[(int64_t)slot * H + j] = acc;
      }
      continue;
    }
    float4 acc[8], v[8], nv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto load_row = [&](int i, float4 (&dst)[8]) {
      const float* src = dpre + (int64_t)__ldg(order_pos + i) * H;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t j = c0 + 4 * (lane + 32 * q);
        if (j < H) dst[q] = __ldg(reinterpret_cast<const float4*>(src + j));
      }
    };
    load_row(a, v);
    float sc = order_scale ? __ldg(order_scale + a) : 1.0f;
    for (int i = a; i < e; ++i) {
      // the next row's loads go out before this row's adds
      float nsc = 1.0f;
      if (i + 1 < e) {
        load_row(i + 1, nv);
        nsc = order_scale ? __ldg(order_scale + i + 1) : 1.0f;
      }
      // (a scaled row is the reference's axpy_row: acc += s * x, two roundings)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        acc[q].x = __fadd_rn(acc[q].x, __fmul_rn(sc, v[q].x));
        acc[q].y = __fadd_rn(acc[q].y, __fmul_rn(sc, v[q].y));
        acc[q].z = __fadd_rn(acc[q].z, __fmul_rn(sc, v[q].z));
        acc[q].w = __fadd_rn(acc[q].w, __fmul_rn(sc, v[q].w));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = nv[q];
      sc = nsc;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = c0 + 4 * (lane + 32 * q);
      if (j >= H) continue;
      const float4 o = make_float4(clip1(acc[q].x, clip), clip1(acc[q].y, clip),
                                   clip1(acc[q].z, clip), clip1(acc[q].w, clip));
      bad |= !isfinite(o.x) || !isfinite(o.y) || !isfinite(o.z) || !isfinite(o.w);
      *reinterpret_cast<float4*>(rows + (int64_t)slot * H + j) = o;
    }
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
}

__global__ void __launch_bounds__(256)
k_embed_long(const float* __restrict__ dpre, int64_t H, const int* __restrict__ seg_start,
             const int* __restrict__ long_list, const int* __restrict__ n_long,
             const int* __restrict__ order_pos, const float* __restrict__ order_scale,
             float* __restrict__ rows, float clip, int* nonfinite) {
  // warps 1..7 stage pass p+1 (kLongPass rows x 32 columns, every load in
  // flight, the row positions of pass p+2 already in registers) while warp 0
  // adds pass p in order from the other buffer: a word with ~18,000 records
  // (NCE's eos noise) is bound by its add chain, not by one L2 round trip
  // per pass
  constexpr int kPer = kLongPass / 7;  // rows per staging warp per pass
  __shared__ float tile[2][kLongPass][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t nchunk = (H + 31) / 32;
  const int64_t items = (int64_t)__ldg(n_long) * nchunk;
  bool bad = false;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int slot = __ldg(long_list + it / nchunk);
    const int64_t j = (it % nchunk) * 32 + lane;
    const int a = __ldg(seg_start + slot), e = __ldg(seg_start + slot + 1);
    const int npass = (e - a + kLongPass - 1) / kLongPass;
    int pos[kPer];
    float sc[kPer];
    auto fetch = [&](int p) {  // row positions / scales of pass p (staging warps)
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = a + p * kLongPass + (warp - 1) + 7 * u;
        pos[u] = (p < npass && i < e) ? __ldg(order_pos + i) : -1;
        sc[u] = (p < npass && i < e && order_scale) ? __ldg(order_scale + i) : 1.0f;
      }
    };
    float v[kPer], vs[kPer];
    auto load = [&] {  // pass rows (positions in pos) -> v, loads left in flight
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        v[u] = (pos[u] >= 0 && j < H) ? __ldg(dpre + (int64_t)pos[u] * H + j) : 0.f;
        vs[u] = sc[u];
      }
    };
    auto store = [&](int b) {  // (the first use of the loaded values)
#pragma unroll
      for (int u = 0; u < kPer; ++u) tile[b][(warp - 1) + 7 * u][lane] = __fmul_rn(vs[u], v[u]);
    };
    if (warp > 0) {
      fetch(0);
      load();
      store(0);
      fetch(1);
      load();  // pass 1, stored during pass 0's adds
      fetch(2);
    }
    __syncthreads();
    float acc = 0.f;
    for (int p = 0; p < npass; ++p) {
      if (warp > 0) {
        // pass p+1's values were loaded an iteration ago; pass p+2's loads
        // go out now and land while the next passes are added
        if (p + 1 < npass) store((p + 1) & 1);
        if (p + 2 < npass) {
          load();
          fetch(p + 3);
        }
      } else {
        const int cnt = min(kLongPass, e - a - p * kLongPass);
        const float(*t)[32] = tile[p & 1];
        int r = 0;
        for (; r + 16 <= cnt; r += 16) {
          float x[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) x[u] = t[r + u][lane];
#pragma unroll
          for (int u = 0; u < 16; ++u) acc = __fadd_rn(acc, x[u]);
        }
        for (; r < cnt; ++r) acc = __fadd_rn(acc, t[r][lane]);
      }
      __syncthreads();
    }
    if (warp == 0 && j < H) {
      acc = clip1(acc, clip);
      bad |= !isfinite(acc);
      rows[(int64_t)slot * H + j] = acc;
    }
  }
  if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicExch(nonfinite, 1);
}

// Dense scatter of the compact rows (tests / dl_get_grads).
__global__ void k_embed_dense(const float* __restrict__ rows, const uint32_t* __restrict__ words,
                              const int* __restrict__ n_seg, int64_t H, float* __restrict__ dense) {
  const int slot = blockIdx.x;
  if (slot >= *n_seg) return;
  for (int64_t j = threadIdx.x; j < H; j += blockDim.x)
    dense[(int64_t)words[slot] * H + j] = rows[(int64_t)slot * H + j];
}

// --------------------------------------------------------------- rmsprop
// rmsprop.hpp:118-124: per-element W_rec update in double, stored float.
__global__ void k_rms_rec(float* __restrict__ w, bf16* __restrict__ wb, float* __restrict__ m,
                          const float* __restrict__ g, int64_t n, double rho, double eps,
                          double eta, const int* __restrict__ nonfinite) {
  if (nonfinite && *nonfinite) return;
  auto one = [&](float& wi, float& mi, float gf) {
    const double gi = (double)gf;
    mi = (float)(rho * (double)mi + (1.0 - rho) * gi * gi);
    wi = wi - (float)(eta * gi / sqrt((double)mi + eps));
  };
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = (n % 4) == 0 ? n / 4 : 0;
  // four independent elements per thread (float4), all loads issued first
  for (int64_t i = tid; i < n4; i += nth) {
    const float4 gq = reinterpret_cast<const float4*>(g)[i];
    float4 mq = reinterpret_cast<float4*>(m)[i];
    float4 wq = reinterpret_cast<float4*>(w)[i];
    one(wq.x, mq.x, gq.x);
    one(wq.y, mq.y, gq.y);
    one(wq.z, mq.z, gq.z);
    one(wq.w, mq.w, gq.w);
    reinterpret_cast<float4*>(m)[i] = mq;
    reinterpret_cast<float4*>(w)[i] = wq;
    if (wb) {
      __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(wb + 4 * i);
      b2[0] = __floats2bfloat162_rn(wq.x, wq.y);
      b2[1] = __floats2bfloat162_rn(wq.z, wq.w);
    }
  }
  for (int64_t i = 4 * n4 + tid; i < n; i += nth) {
    float wi = w[i], mi = m[i];
    one(wi, mi, g[i]);
    m[i] = mi;
    w[i] = wi;
    if (wb) wb[i] = __float2bfloat16_rn(wi);
  }
}

// rmsprop.hpp:84 first loop: every W_in accumulator decays.
__global__ void k_rms_decay(float* __restrict__ m, int64_t n, double rho,
                            const int* __restrict__ nonfinite) {
  if (nonfinite && *nonfinite) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m[i] = (float)(rho * (double)m[i]);
}

// The same update with a block per row (H / 8 threads, two float4 per
// thread): the row's gradient and master are loaded once, together, before
// the block's sum of squares -- the one-warp-per-row kernel below keeps only
// a warp's loads in flight per row and re-reads g for the update.
template <int VPT>
__global__ void k_rms_rows_blk(float* __restrict__ w, bf16* __restrict__ wb,
                               float* __restrict__ m, const float* __restrict__ g,
                               const uint32_t* __restrict__ words,
                               const int* __restrict__ n_rows_dev, int64_t n_rows, int64_t H,
                               double rho, double eps, double eta, int dense,
                               const int* __restrict__ nonfinite) {
  if (nonfinite && *nonfinite) return;
  __shared__ double red[32];
  const int64_t rows = n_rows_dev ? (int64_t)*n_rows_dev : n_rows;
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32, nw = blockDim.x / 32;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t word = words ? (int64_t)words[r] : r;
    const float4* g4 = reinterpret_cast<const float4*>(g + r * H);
    float4* w4 = reinterpret_cast<float4*>(w + word * H);
    float4 q[VPT], o[VPT];
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      q[v] = g4[threadIdx.x + v * blockDim.x];
      o[v] = w4[threadIdx.x + v * blockDim.x];
    }
    double s = 0.0;
#pragma unroll
    for (int v = 0; v < VPT; ++v)
      s += (double)q[v].x * (double)q[v].x + (double)q[v].y * (double)q[v].y +
           (double)q[v].z * (double)q[v].z + (double)q[v].w * (double)q[v].w;
    s = warp_sum_d(s);
    if (lane == 0) red[wid] = s;
    __syncthreads();
    double tot = 0.0;
    for (int i = 0; i < nw; ++i) tot += red[i];  // fixed order, every thread
    const double ms = tot / (double)H;
    float mw;
    if (dense) mw = (float)(rho * (double)m[word] + (1.0 - rho) * ms);
    else mw = m[word] + (float)((1.0 - rho) * ms);
    const double denom = sqrt((double)mw + eps);
    const double inv = 1.0 / denom;
#pragma unroll
    for (int v = 0; v < VPT; ++v) {
      o[v].x -= rms_step(eta, q[v].x, denom, inv);
      o[v].y -= rms_step(eta, q[v].y, denom, inv);
      o[v].z -= rms_step(eta, q[v].z, denom, inv);
      o[v].w -= rms_step(eta, q[v].w, denom, inv);
      const int64_t j = threadIdx.x + v * blockDim.x;
      w4[j] = o[v];
      if (wb) {
        __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(wb + word * H + 4 * j);
        b2[0] = __floats2bfloat162_rn(o[v].x, o[v].y);
        b2[1] = __floats2bfloat162_rn(o[v].z, o[v].w);
      }
    }
    __syncthreads();  // every thread has read m[word] and red[]
    if (threadIdx.x == 0) m[word] = mw;
  }
}

// rmsprop.hpp:85-91: touched rows add (1-rho)*mean(g^2) to the decayed
// scalar, then divide the whole row's step by sqrt(m + eps).
// rmsprop.hpp:94-107 (dense=1): m = float(rho*m + (1-rho)*mean(g^2)).
// One warp per row.
__global__ void k_rms_rows(float* __restrict__ w, bf16* __restrict__ wb, float* __restrict__ m,
                           const float* __restrict__ g, const uint32_t* __restrict__ words,
                           const int* __restrict__ n_rows_dev, int64_t n_rows, int64_t H,
                           double rho, double eps, double eta, int dense,
                           const int* __restrict__ nonfinite) {
  if (nonfinite && *nonfinite) return;
  const int64_t rows = n_rows_dev ? (int64_t)*n_rows_dev : n_rows;
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = warp0; r < rows; r += nwarps) {
    const float* gr = g + r * H;
    const int64_t word = words ? (int64_t)words[r] : r;
    double s = 0.0;
    if ((H % 4) == 0) {
      const float4* g4 = reinterpret_cast<const float4*>(gr);
      for (int64_t j = lane; j < H / 4; j += 32) {
        const float4 q = g4[j];
        s += (double)q.x * (double)q.x + (double)q.y * (double)q.y +
             (double)q.z * (double)q.z + (double)q.w * (double)q.w;
      }
    } else {
      for (int64_t j = lane; j < H; j += 32) s += (double)gr[j] * (double)gr[j];
    }
    s = warp_sum_d(s);
    const double ms = s / (double)H;
    float mw;
    if (dense) mw = (float)(rho * (double)m[word] + (1.0 - rho) * ms);
    else mw = m[word] + (float)((1.0 - rho) * ms);
    const double denom = sqrt((double)mw + eps);
    const double inv = 1.0 / denom;
    float* wr = w + word * H;
    bf16* wbr = wb ? wb + word * H : nullptr;
    if ((H % 4) == 0) {
      const float4* g4 = reinterpret_cast<const float4*>(gr);
      float4* w4 = reinterpret_cast<float4*>(wr);
      for (int64_t j = lane; j < H / 4; j += 32) {
        const float4 q = g4[j];
        float4 o = w4[j];
        o.x -= rms_step(eta, q.x, denom, inv);
        o.y -= rms_step(eta, q.y, denom, inv);
        o.z -= rms_step(eta, q.z, denom, inv);
        o.w -= rms_step(eta, q.w, denom, inv);
        w4[j] = o;
        if (wbr) {
          __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(wbr + 4 * j);
          b2[0] = __floats2bfloat162_rn(o.x, o.y);
          b2[1] = __floats2bfloat162_rn(o.z, o.w);
        }
      }
    } else {
      for (int64_t j = lane; j < H; j += 32) {
        const float o = wr[j] - rms_step(eta, gr[j], denom, inv);
        wr[j] = o;
        if (wbr) wbr[j] = __float2bfloat16_rn(o);
      }
    }
    if (lane == 0) m[word] = mw;
  }
}

// Dense W_out rows (rmsprop.hpp:94-107) for H = 128*NV4: one warp per row,
// the gradient row held in registers (each lane: NV4 float4), so every load
// of a row is issued before the first use -- enough bytes in flight to run
// at HBM speed from only one 256-thread block per SM, which co-resides with
// the tensor-core GEMM it overlaps.
template <int NV4>
__global__ void __launch_bounds__(128, NV4 > 8 ? 3 : 4)
k_rms_dense_rows(float* __restrict__ w, bf16* __restrict__ wb, float* __restrict__ m,
                 const float* __restrict__ g, int64_t V, double rho, double eps, double eta,
                 const int* __restrict__ nonfinite) {
  if (nonfinite && *nonfinite) return;
  constexpr int64_t H = 128 * NV4;
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = warp0; r < V; r += nwarps) {
    const float4* g4 = reinterpret_cast<const float4*>(g + r * H);
    float4* w4 = reinterpret_cast<float4*>(w + r * H);
    float4 q[NV4];
#pragma unroll
    for (int k = 0; k < NV4; ++k) q[k] = __ldcs(g4 + lane + 32 * k);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < NV4; ++k)
      s += (double)q[k].x * (double)q[k].x + (double)q[k].y * (double)q[k].y +
           (double)q[k].z * (double)q[k].z + (double)q[k].w * (double)q[k].w;
    s = warp_sum_d(s);
    const float mw = (float)(rho * (double)m[r] + (1.0 - rho) * (s / (double)H));
    const double denom = sqrt((double)mw + eps);
    const double inv = 1.0 / denom;
#pragma unroll
    for (int k = 0; k < NV4; ++k) {
      float4 o = w4[lane + 32 * k];
      o.x -= rms_step(eta, q[k].x, denom, inv);
      o.y -= rms_step(eta, q[k].y, denom, inv);
      o.z -= rms_step(eta, q[k].z, denom, inv);
      o.w -= rms_step(eta, q[k].w, denom, inv);
      w4[lane + 32 * k] = o;
      if (wb) {
        __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(wb + r * H + 4 * (lane + 32 * k));
        b2[0] = __floats2bfloat162_rn(o.x, o.y);
        b2[1] = __floats2bfloat162_rn(o.z, o.w);
      }
    }
    if (lane == 0) m[r] = mw;
  }
}

// Dense W_out rmsprop (rmsprop.hpp:94-107) from the bf16 gradient the dW_out
// GEMM epilogue wrote, with mean_sq assembled from its per-(half tile, row)
// partial sums of squares (fixed order): one pass over the row, 12 B/elem
// (g 2, w 4+4, shadow 2).  One warp per row.
__global__ void __launch_bounds__(256)
k_rms_dense_g16(float* __restrict__ w, bf16* __restrict__ wb, float* __restrict__ m,
                const bf16* __restrict__ g, const double* __restrict__ rowsq, int nsub,
                int64_t V, int64_t H, double rho, double eps, double eta) {
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = warp0; r < V; r += nwarps) {
    double s = 0.0;
    for (int k = 0; k < nsub; ++k) s += rowsq[(int64_t)k * V + r];
    const float mw = (float)(rho * (double)m[r] + (1.0 - rho) * (s / (double)H));
    const double denom = sqrt((double)mw + eps);
    const double inv = 1.0 / denom;
    const uint4* g8 = reinterpret_cast<const uint4*>(g + r * H);
    float4* w4 = reinterpret_cast<float4*>(w + r * H);
    uint4* b8 = reinterpret_cast<uint4*>(wb + r * H);
#pragma unroll 2
    for (int64_t j = lane; j < H / 8; j += 32) {
      const uint4 q = __ldcs(g8 + j);
      float4 o0 = w4[2 * j], o1 = w4[2 * j + 1];
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&q);
      const float2 a = __bfloat1622float2(q2[0]), b = __bfloat1622float2(q2[1]);
      const float2 c = __bfloat1622float2(q2[2]), d = __bfloat1622float2(q2[3]);
      o0.x -= rms_step(eta, a.x, denom, inv);
      o0.y -= rms_step(eta, a.y, denom, inv);
      o0.z -= rms_step(eta, b.x, denom, inv);
      o0.w -= rms_step(eta, b.y, denom, inv);
      o1.x -= rms_step(eta, c.x, denom, inv);
      o1.y -= rms_step(eta, c.y, denom, inv);
      o1.z -= rms_step(eta, d.x, denom, inv);
      o1.w -= rms_step(eta, d.y, denom, inv);
      w4[2 * j] = o0;
      w4[2 * j + 1] = o1;
      uint4 ob;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(o0.x, o0.y), p1 = __floats2bfloat162_rn(o0.z, o0.w);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(o1.x, o1.y), p3 = __floats2bfloat162_rn(o1.z, o1.w);
      ob.x = *reinterpret_cast<uint32_t*>(&p0);
      ob.y = *reinterpret_cast<uint32_t*>(&p1);
      ob.z = *reinterpret_cast<uint32_t*>(&p2);
      ob.w = *reinterpret_cast<uint32_t*>(&p3);
      b8[j] = ob;
    }
    if (lane == 0) m[r] = mw;
  }
}

// Dense W_out rmsprop (rmsprop.hpp:94-107) from an unclipped bf16 gradient
// (the data-parallel path: dW_out summed over ranks in bf16): clip
// (rnn.hpp:158-159), mean_sq in fp64, then the row's update -- two passes
// over the row's gradient (the second from L1/L2).  One warp per row.
__global__ void __launch_bounds__(256)
k_rms_dense_g16c(float* __restrict__ w, bf16* __restrict__ wb, float* __restrict__ m,
                 const bf16* __restrict__ g, int64_t V, int64_t H, float clip, double rho,
                 double eps, double eta) {
  const int lane = threadIdx.x % 32;
  const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t nwarps = (int64_t)gridDim.x * blockDim.x / 32;
  for (int64_t r = warp0; r < V; r += nwarps) {
    const uint4* g8 = reinterpret_cast<const uint4*>(g + r * H);
    double s = 0.0;
    for (int64_t j = lane; j < H / 8; j += 32) {
      const uint4 q = __ldg(g8 + j);
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(q2[k]);
        const float a = clip1(f.x, clip), b = clip1(f.y, clip);
        s += (double)a * (double)a + (double)b * (double)b;
      }
    }
    s = warp_sum_d(s);
    const float mw = (float)(rho * (double)m[r] + (1.0 - rho) * (s / (double)H));
    const double denom = sqrt((double)mw + eps);
    const double inv = 1.0 / denom;
    float4* w4 = reinterpret_cast<float4*>(w + r * H);
    uint4* b8 = reinterpret_cast<uint4*>(wb + r * H);
    for (int64_t j = lane; j < H / 8; j += 32) {
      const uint4 q = __ldg(g8 + j);
      const __nv_bfloat162* q2 = reinterpret_cast<const __nv_bfloat162*>(&q);
      float gg[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(q2[k]);
        gg[2 * k] = clip1(f.x, clip);
        gg[2 * k + 1] = clip1(f.y, clip);
      }
      float4 o0 = w4[2 * j], o1 = w4[2 * j + 1];
      o0.x -= rms_step(eta, gg[0], denom, inv);
      o0.y -= rms_step(eta, gg[1], denom, inv);
      o0.z -= rms_step(eta, gg[2], denom, inv);
      o0.w -= rms_step(eta, gg[3], denom, inv);
      o1.x -= rms_step(eta, gg[4], denom, inv);
      o1.y -= rms_step(eta, gg[5], denom, inv);
      o1.z -= rms_step(eta, gg[6], denom, inv);
      o1.w -= rms_step(eta, gg[7], denom, inv);
      w4[2 * j] = o0;
      w4[2 * j + 1] = o1;
      uint4 ob;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(o0.x, o0.y), p1 = __floats2bfloat162_rn(o0.z, o0.w);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(o1.x, o1.y), p3 = __floats2bfloat162_rn(o1.z, o1.w);
      ob.x = *reinterpret_cast<uint32_t*>(&p0);
      ob.y = *reinterpret_cast<uint32_t*>(&p1);
      ob.z = *reinterpret_cast<uint32_t*>(&p2);
      ob.w = *reinterpret_cast<uint32_t*>(&p3);
      b8[j] = ob;
    }
    if (lane == 0) m[r] = mw;
  }
}

__global__ void k_count_skip(const int* __restrict__ nonfinite, unsigned long long* skipped) {
  if (*nonfinite) skipped[0] += 1ull;
}

__global__ void k_accum_loss(double* acc, const double* v, unsigned long long* cnt,
                             const unsigned long long* vc) {
  acc[0] += v[0];
  cnt[0] += vc[0];
}

// dst = src ? *src : value  (device-side flags inside graphs)
__global__ void k_set_flag(int* dst, const int* src, int value) {
  dst[0] = src ? src[0] : value;
}

// ----------------------------------------------------- offset streams
// Window build for group g = window % noffset (trainer.hpp:376-389): the
// rank's streams are s = g*Bg + rank*B + b; pos = cursor[s] + t; x =
// ids[pos % L], y = ids[(pos+1) % L], w = (y != bos).  Also gathers h0.
__global__ void k_window_build(const uint32_t* __restrict__ ids, int64_t L,
                               const int64_t* __restrict__ cursors, const float* __restrict__ hidden,
                               const int64_t* __restrict__ win_counter, int noffset, int64_t B,
                               int64_t T, int64_t H, uint32_t bos, uint32_t* __restrict__ x,
                               uint32_t* __restrict__ y, uint8_t* __restrict__ w,
                               float* __restrict__ h0, bf16* __restrict__ h0b) {
  const int64_t g = *win_counter % noffset;
  const int64_t s0 = g * B;  // cursors / hidden hold this rank's streams only
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < T * B; i += nthreads) {
    const int64_t t = i / B, b = i % B;
    const int64_t pos = cursors[s0 + b] + t;
    const uint32_t xi = ids[pos % L];
    const uint32_t yi = ids[(pos + 1) % L];
    x[i] = xi;
    y[i] = yi;
    w[i] = yi == bos ? 0 : 1;
  }
  for (int64_t i = tid; i < B * H; i += nthreads) {
    const float v = hidden[s0 * H + i];
    h0[i] = v;
    if (h0b) h0b[i] = __float2bfloat16_rn(v);  // the recurrence's first A operand
  }
}

// After the window (trainer.hpp:396-405), one block per stream: hidden <-
// h_final (or act(0) on a wrap), then the stream's cursor += T (-= L on a
// wrap).  The window counter advances in k_window_tail.
__global__ void k_window_finish(int64_t* __restrict__ cursors, float* __restrict__ hidden,
                                const float* __restrict__ h_final,
                                const int64_t* __restrict__ win_counter, int noffset, int64_t B,
                                int64_t T, int64_t H, int64_t L, float a0) {
  const int64_t s0 = (*win_counter % noffset) * B;
  for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
    const int64_t cur = cursors[s0 + b];
    const bool wrap = cur + T >= L;
    float* dst = hidden + (s0 + b) * H;
    const float* src = h_final + b * H;
    if ((H % 4) == 0) {
      for (int64_t i = threadIdx.x; i < H / 4; i += blockDim.x)
        reinterpret_cast<float4*>(dst)[i] =
            wrap ? make_float4(a0, a0, a0, a0) : reinterpret_cast<const float4*>(src)[i];
    } else {
      for (int64_t i = threadIdx.x; i < H; i += blockDim.x) dst[i] = wrap ? a0 : src[i];
    }
    __syncthreads();  // every thread has read the old cursor
    if (threadIdx.x == 0) cursors[s0 + b] = wrap ? cur + T - L : cur + T;
    __syncthreads();
  }
}

// window counter += 1; skipped += the update's non-finite verdict
__global__ void k_window_tail(int64_t* win_counter, const int* __restrict__ nonfinite,
                              unsigned long long* skipped) {
  if (nonfinite && skipped && *nonfinite) skipped[0] += 1ull;
  win_counter[0] += 1;
}

}  // namespace

// ------------------------------------------------------------ launchers
static inline int grid_for(int64_t n, int tpb = 256, int cap = 148 * 16) {
  int64_t g = (n + tpb - 1) / tpb;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// out[c][r] = in[r][c] for an fp32 rows x cols matrix (32 x 32 tiles through
// shared memory): the 3xTF32 GEMM's MN-major operands made K-major
// (kind::tf32 reads K-major tiles only).
__global__ void k_transpose_f32(const float* __restrict__ in, int64_t rows, int64_t cols,
                                int64_t ld_in, float* __restrict__ out, int64_t ld_out) {
  __shared__ float t[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < rows && c < cols) ? in[r * ld_in + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[c * ld_out + r] = t[threadIdx.x][i];
  }
}

void transpose_f32(const float* in, int64_t rows, int64_t cols, int64_t ld_in, float* out,
                   int64_t ld_out, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  k_transpose_f32<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ld_in, out, ld_out);
}

void f32_to_bf16(const float* x, bf16* y, int64_t n, cudaStream_t st) {
  k_f32_to_bf16<<<grid_for(n), 256, 0, st>>>(x, y, n);
}
void fill_f32(float* x, float v, int64_t n, cudaStream_t st) {
  k_fill_f32<<<grid_for(n), 256, 0, st>>>(x, v, n);
}
void rec_fwd(const float* part, int splits, int64_t ss, int64_t Bn, int64_t H, const float* w_in,
             const uint32_t* x, int act, float* h, bf16* hb, cudaStream_t st) {
  k_rec_fwd<<<grid_for(Bn * H), 256, 0, st>>>(part, splits, ss, Bn, H, w_in, x, act, h, hb);
}
void rec_bwd(const float* part, int splits, int64_t ss, int64_t n, const float* dh_out,
             const float* hnext, int act, float* dpre, bf16* dpreb, cudaStream_t st) {
  k_rec_bwd<<<grid_for(n), 256, 0, st>>>(part, splits, ss, n, dh_out, hnext, act, dpre, dpreb);
}
void reduce_rms_rec(const float* part, int splits, int64_t ss, int64_t n, float* g_out, float clip,
                    float* w, bf16* wb, float* m, double rho, double eps, double eta,
                    cudaStream_t st) {
  k_reduce_rms_rec<<<grid_for(n / 4), 256, 0, st>>>(part, splits, ss, n, g_out, clip, w, wb, m,
                                                    rho, eps, eta);
}
void reduce_splits(const float* part, int splits, int64_t ss, int64_t n, float* out, float clip,
                   int do_clip, int* nonfinite, cudaStream_t st) {
  k_reduce<<<grid_for(n), 256, 0, st>>>(part, splits, ss, n, out, clip, do_clip, nonfinite);
}
void softmax_rows_f32(float* S, int64_t M, int64_t V, const uint32_t* tgt, const uint8_t* wts,
                      double scale, int grads, double* loss_row, double* logp_row,
                      cudaStream_t st, const double* lse_all, int G, const float* tgt_logit) {
  if (M <= 0) return;
  k_softmax_rows_f32<<<(unsigned)M, kRowThreads, 0, st>>>(S, V, M, tgt, wts, scale, grads,
                                                          loss_row, logp_row, lse_all, G,
                                                          tgt_logit);
}
void softmax_rows_bf16(bf16* S, int64_t M, int64_t V, const float2* part, int n_tiles,
                       const float* tgt_logit, const uint32_t* tgt, const uint8_t* wts,
                       double scale, int grads, double* loss_row, double* logp_row,
                       cudaStream_t st, const double* lse_all, int G) {
  if (M <= 0) return;
  k_softmax_rows_bf16<<<(unsigned)M, kRowThreads, 0, st>>>(S, V, M, part, n_tiles, tgt_logit, tgt,
                                                           wts, scale, grads, loss_row, logp_row,
                                                           lse_all, G);
}
void lse_rows_bf16(int64_t M, const float2* part, int n_tiles, const float* tgt_logit,
                   const uint8_t* wts, double scale, double* loss_row, double* logp_row,
                   float* lse_f, float* sc_f, cudaStream_t st, const double* lse_all, int G) {
  if (M <= 0) return;
  k_lse_rows_bf16<<<(unsigned)M, kRowThreads, 0, st>>>(M, part, n_tiles, tgt_logit, wts, scale,
                                                       loss_row, logp_row, lse_f, sc_f, lse_all,
                                                       G);
}
void target_shift(const bf16* hs, const bf16* w, int64_t H, int64_t M, const uint32_t* tgt,
                  int64_t V, float* shift, cudaStream_t st) {
  if (M <= 0) return;
  k_target_shift<<<(unsigned)((M + 7) / 8), 256, 0, st>>>(hs, w, H, M, tgt, V, shift);
}
void pfac_rows(bf16* E, int64_t M, int64_t V, int64_t H, const float2* part, int n_tiles,
               const float* tgt_logit, const uint32_t* tgt, const uint8_t* wts, double scale,
               double* loss_row, double* logp_row, const float* shift, float* sigma,
               float* resid, const float* hs, bf16* hs_sc, const bf16* hs_bf, float repair_nats,
               int* repaired, cudaStream_t st, const double* lse_all, int G) {
  if (M <= 0) return;
  const int pw = (V >= 256 ? 256 : V >= 128 ? 128 : 64) / 2;  // (tc_n_tiles' half tiles)
  k_pfac_rows<<<(unsigned)M, kPfacThreads, n_tiles * sizeof(float), st>>>(
      E, V, M, H, part, n_tiles, pw, tgt_logit, tgt, wts, scale, loss_row, logp_row, shift, sigma,
      resid, hs, hs_sc, hs_bf, repair_nats, repaired, lse_all, G);
}
void pfac_lse(bf16* E, int64_t M, int64_t V, const float2* part, int n_tiles, const uint8_t* wts,
              float* shift, double* lse_loc, float repair_nats, int* repaired, cudaStream_t st) {
  if (M <= 0) return;
  const int pw = (V >= 256 ? 256 : V >= 128 ? 128 : 64) / 2;  // (tc_n_tiles' half tiles)
  k_pfac_lse<<<(unsigned)M, kPfacThreads, n_tiles * sizeof(float), st>>>(
      E, V, M, part, n_tiles, pw, wts, shift, lse_loc, repair_nats, repaired);
}
void shard_targets(const uint32_t* y, int64_t M, int64_t v0, int64_t Vo, uint32_t* loc,
                   cudaStream_t st) {
  if (M <= 0) return;
  k_shard_targets<<<grid_for(M), 256, 0, st>>>(y, M, v0, Vo, loc);
}
void block_lse_bf16(const float2* part, int n_tiles, int64_t M, double* lse, cudaStream_t st) {
  if (M <= 0) return;
  k_block_lse_bf16<<<(unsigned)M, 256, 0, st>>>(part, n_tiles, M, lse);
}
void block_lse_f32(const float* S, int64_t M, int64_t V, const uint32_t* loc, double* lse,
                   float* tgt_logit, cudaStream_t st) {
  if (M <= 0) return;
  k_block_lse_f32<<<(unsigned)M, kRowThreads, 0, st>>>(S, V, loc, lse, tgt_logit);
}
void sum_rows(const double* v, const uint8_t* wts, int64_t n, double* acc,
              unsigned long long* cnt, cudaStream_t st) {
  k_sum_rows<<<1, 1024, 0, st>>>(v, wts, n, acc, cnt);
}
void embed_sort(const uint32_t* x, int64_t T, int64_t B, int64_t G, int64_t V, EmbedWs& ws,
                uint32_t* words, int* n_rows, cudaStream_t st) {
  const int64_t n = G * T * B;
  DL_REQUIRE(n <= 16 * kSortThreads, 1, "window too large for the embedding sort (G*T*B <= 16384)");
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= V) ++end_bit;  // 2^end_bit - 1 >= V pads past every id
#define DL_RADIX(IPT)                                                                          \
  if (n <= (IPT) * kSortThreads) {                                                             \
    static bool attr = false;                                                                  \
    const size_t smem = sizeof(typename EmbedRadix<IPT>::Smem);                                \
    if (!attr) {                                                                               \
      DL_CUDA(cudaFuncSetAttribute(k_embed_radix<IPT>,                                         \
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));   \
      attr = true;                                                                             \
    }                                                                                          \
    k_embed_radix<IPT><<<1, kSortThreads, smem, st>>>(x, T, B, G, end_bit, ws.seg_start,       \
                                                      n_rows, ws.order_pos, words,             \
                                                      ws.long_list(), ws.n_long());            \
  } else
  DL_RADIX(2) DL_RADIX(4) DL_RADIX(8) DL_RADIX(16) {}
#undef DL_RADIX
}
int embed_short_max() { return kEmbedShort; }

void embed_rows(int64_t n, const float* dpre, int64_t H, float clip, EmbedWs& ws, float* rows,
                int* n_rows, int* nonfinite, cudaStream_t st, const float* order_scale) {
  if (n <= 0) return;
  const int64_t nchunk = (H + 1023) / 1024;
  const int64_t warps = std::min<int64_t>(n * nchunk, 148 * 64);
  k_embed_short<<<(unsigned)((warps + kShortWarps - 1) / kShortWarps), 32 * kShortWarps, 0, st>>>(
      dpre, H, ws.seg_start, n_rows, ws.order_pos, order_scale, rows, clip, nonfinite);
  k_embed_long<<<148 * 2, 256, 0, st>>>(
      dpre, H, ws.seg_start, ws.long_list(), ws.n_long(), ws.order_pos, order_scale, rows, clip,
      nonfinite);
}
void embed_grads(const uint32_t* x, int64_t T, int64_t B, int64_t G, int64_t V, const float* dpre,
                 int64_t H, float clip, EmbedWs& ws, float* rows, uint32_t* words, int* n_rows,
                 int* nonfinite, cudaStream_t st) {
  embed_sort(x, T, B, G, V, ws, words, n_rows, st);
  embed_rows(G * T * B, dpre, H, clip, ws, rows, n_rows, nonfinite, st);
}
void embed_dense(const float* rows, const uint32_t* words, const int* n_rows, int64_t max_rows,
                 int64_t H, float* dense, cudaStream_t st) {
  if (max_rows <= 0) return;
  k_embed_dense<<<(unsigned)max_rows, 256, 0, st>>>(rows, words, n_rows, H, dense);
}
void rms_rec(float* w, bf16* wb, float* m, const float* g, int64_t n, double rho, double eps,
             double eta, const int* nonfinite, cudaStream_t st) {
  k_rms_rec<<<grid_for(n), 256, 0, st>>>(w, wb, m, g, n, rho, eps, eta, nonfinite);
}
void rms_decay(float* m, int64_t n, double rho, const int* nonfinite, cudaStream_t st) {
  k_rms_decay<<<grid_for(n), 256, 0, st>>>(m, n, rho, nonfinite);
}
// DL_DENSE_ROWS=1 selects the register-resident one-warp-per-row W_out
// kernel (fewer warps; measured slower than k_rms_rows on B200).
static const bool use_dense_rows_kernel = [] {
  const char* e = std::getenv("DL_DENSE_ROWS");
  return e && std::atoi(e) != 0;
}();

// DL_WARP_ROWS=1: the one-warp-per-row kernel for every H
static const bool use_warp_rows_kernel = [] {
  const char* e = std::getenv("DL_WARP_ROWS");
  return e && std::atoi(e) != 0;
}();

void rms_rows(float* w, bf16* wb, float* m, const float* g, const uint32_t* words,
              const int* n_rows_dev, int64_t n_rows, int64_t H, double rho, double eps, double eta,
              int dense, const int* nonfinite, cudaStream_t st) {
  if (use_dense_rows_kernel && dense && !words && !n_rows_dev && (H == 1024 || H == 2048)) {
    const int blocks = 148 * (H == 1024 ? 4 : 3);
    if (H == 1024)
      k_rms_dense_rows<8><<<blocks, 128, 0, st>>>(w, wb, m, g, n_rows, rho, eps, eta, nonfinite);
    else
      k_rms_dense_rows<16><<<blocks, 128, 0, st>>>(w, wb, m, g, n_rows, rho, eps, eta, nonfinite);
    return;
  }
  // (a few thousand rows at most -- the W_in rows of a window: a block per
  // row; tens of thousands -- NCE's W_out rows: the warp kernel measured
  // 0.321 vs 0.330 ms at C3)
  if (H % 256 == 0 && H / 8 >= 64 && H / 8 <= 1024 && n_rows <= 4096 && !use_warp_rows_kernel) {
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(n_rows, 148 * 16));
    k_rms_rows_blk<2><<<blocks, (unsigned)(H / 8), 0, st>>>(w, wb, m, g, words, n_rows_dev,
                                                            n_rows, H, rho, eps, eta, dense,
                                                            nonfinite);
    return;
  }
  const int64_t warps = n_rows;
  int blocks = (int)std::min<int64_t>((warps * 32 + 255) / 256, 148 * 8);
  if (blocks < 1) blocks = 1;
  k_rms_rows<<<blocks, 256, 0, st>>>(w, wb, m, g, words, n_rows_dev, n_rows, H, rho, eps, eta,
                                     dense, nonfinite);
}
void count_skip(const int* nonfinite, unsigned long long* skipped, cudaStream_t st) {
  k_count_skip<<<1, 1, 0, st>>>(nonfinite, skipped);
}
void rms_dense_g16c(float* w, bf16* wb, float* m, const bf16* g, int64_t V, int64_t H,
                    float clip, double rho, double eps, double eta, cudaStream_t st) {
  if (V <= 0) return;
  const int blocks = (int)std::min<int64_t>((V + 7) / 8, 148 * 8);
  k_rms_dense_g16c<<<blocks, 256, 0, st>>>(w, wb, m, g, V, H, clip, rho, eps, eta);
}
void rms_dense_g16(float* w, bf16* wb, float* m, const bf16* g, const double* rowsq, int nsub,
                   int64_t V, int64_t H, double rho, double eps, double eta, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((V * 32 + 255) / 256, 148 * 8);
  k_rms_dense_g16<<<blocks, 256, 0, st>>>(w, wb, m, g, rowsq, nsub, V, H, rho, eps, eta);
}
void accum_loss(double* acc, const double* v, unsigned long long* cnt,
                const unsigned long long* vc, cudaStream_t st) {
  k_accum_loss<<<1, 1, 0, st>>>(acc, v, cnt, vc);
}
void set_flag(int* dst, const int* src, int value, cudaStream_t st) {
  k_set_flag<<<1, 1, 0, st>>>(dst, src, value);
}
void window_build(const uint32_t* ids, int64_t L, const int64_t* cursors, const float* hidden,
                  const int64_t* win_counter, int noffset, int64_t B, int64_t T, int64_t H,
                  uint32_t bos, uint32_t* x, uint32_t* y, uint8_t* w, float* h0, cudaStream_t st,
                  bf16* h0b) {
  k_window_build<<<grid_for(std::max(T * B, B * H)), 256, 0, st>>>(
      ids, L, cursors, hidden, win_counter, noffset, B, T, H, bos, x, y, w, h0, h0b);
}
void window_finish(int64_t* cursors, float* hidden, const float* h_final, int64_t* win_counter,
                   int noffset, int64_t B, int64_t T, int64_t H, int64_t L, float a0,
                   cudaStream_t st, const int* nonfinite, unsigned long long* skipped) {
  k_window_finish<<<(unsigned)std::min<int64_t>(B, 148 * 4), 256, 0, st>>>(
      cursors, hidden, h_final, win_counter, noffset, B, T, H, L, a0);
  k_window_tail<<<1, 1, 0, st>>>(win_counter, nonfinite, skipped);
}

}  // namespace dl
