// NCE output layer of the RNNLM window (LossMode::kNce, the reference's
// default training mode): backprop.hpp:126-156 (loss), :193-203 (backward);
// StandardAdapter::score / score_backward rnn.hpp:246-255; nce.hpp:31-36,
// 103-129 (softplus / sigmoid / the loss); SparseRowGrads rnn.hpp:89-127.
//
// The noise ids are drawn on the host with the reference's mt19937_64 +
// AliasSampler (runtime.cu), in the reference's order (t, then b, then the
// sample; masked positions draw nothing), and arrive as records:
//   forward order   r = p * (k+1) + j   (p = the p-th unmasked position in
//                   t-major order, j = 0 the target, 1..k the noise words)
//   processing order q (t descending, b ascending, j ascending) -- the order
//                   score_backward visits them, hence the float summation
//                   order of every sparse W_out row.
// Kernels:
//   k_nce_scores  score[r] = float(dot_acc<double>(h_row, W_out[w]))  -- the
//                 reference's 8 fixed double lanes (mat.hpp:59-78), no FMA
//   k_nce_loss    per position: a = s - ln(k q(w)); loss terms softplus;
//                 ds = float(-scale*sigmoid(-a_t)) / float(scale*sigmoid(a))
//   k_nce_dh      dh[row] = sum over the position's records of ds * W_out[w]
//                 (float axpy order, mat.hpp:80-84)
//   W_out rows    records stably radix-sorted by word (cub), segment heads,
//                 then the segmented ds * h sums of kernels.cu (embed_rows).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace dl {
namespace {

__device__ __forceinline__ float ld_f(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ld_f(const bf16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float4 ld_f4(const float* row, int64_t i4) {
  return __ldg(reinterpret_cast<const float4*>(row) + i4);
}
__device__ __forceinline__ float4 ld_f4(const bf16* row, int64_t i4) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(row) + i4);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

// one record per 8 threads: thread q owns the reference's lane q.  W (the
// output rows) is the fp32 master, or (bf16 mode) its bf16 shadow: half the
// bytes of the row gathers that bound this kernel and k_nce_dh
template <typename X, typename W>
__global__ void k_nce_scores(const X* __restrict__ h, const W* __restrict__ w_out,
                             int64_t H, const uint32_t* __restrict__ rec_word,
                             const uint32_t* __restrict__ rec_row, int64_t N,
                             float* __restrict__ score) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = gt / 8;
  const int q = (int)(gt % 8);
  const bool valid = r < N;
  double s = 0.0;
  const X* x = nullptr;
  const W* y = nullptr;
  const int64_t H8 = (H / 8) * 8;
  if (valid) {
    x = h + (int64_t)rec_row[r] * H;
    y = w_out + (int64_t)rec_word[r] * H;
    for (int64_t i = 0; i < H8; i += 8)
      s = __dadd_rn(s, __dmul_rn((double)x[i + q], (double)ld_f(y + i + q)));
  }
  // ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)) + tail
  const int base = (threadIdx.x % 32) & ~7;
  double l[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) l[k] = __shfl_sync(0xffffffffu, s, base + k);
  if (valid && q == 0) {
    double tail = 0.0;
    for (int64_t i = H8; i < H; ++i)
      tail = __dadd_rn(tail, __dmul_rn((double)x[i], (double)ld_f(y + i)));
    const double tot = __dadd_rn(__dadd_rn(__dadd_rn(l[0], l[1]), __dadd_rn(l[2], l[3])),
                                 __dadd_rn(__dadd_rn(l[4], l[5]), __dadd_rn(l[6], l[7])));
    score[r] = (float)__dadd_rn(tot, tail);
  }
}

__device__ __forceinline__ double softplus_d(double x) {
  return x > 0 ? x + log1p(exp(-x)) : log1p(exp(x));
}
__device__ __forceinline__ double sigmoid_d(double x) { return 1.0 / (1.0 + exp(-x)); }

// a warp per position: the records' terms in parallel (lane = record within
// a 32-record chunk), their sum in the reference's record order by lane 0
// (backprop.hpp:136-150: L += scale softplus(..) in j order)
__global__ void k_nce_loss(const float* __restrict__ score, const uint32_t* __restrict__ rec_word,
                           const double* __restrict__ ln_kq, int64_t P, int K1, double scale,
                           double* __restrict__ loss_pos, float* __restrict__ ds) {
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (p >= P) return;  // (whole warps)
  const int64_t r0 = p * K1;
  double L = 0.0;
  for (int j0 = 0; j0 < K1; j0 += 32) {
    const int j = j0 + lane;
    double t = 0.0;
    if (j < K1) {
      const double a = (double)score[r0 + j] - ln_kq[rec_word[r0 + j]];
      if (j == 0) {  // the target record
        t = scale * softplus_d(-a);
        ds[r0] = (float)(-scale * sigmoid_d(-a));
      } else {
        t = scale * softplus_d(a);
        ds[r0 + j] = (float)(scale * sigmoid_d(a));
      }
    }
    const int n = min(32, K1 - j0);
    for (int i = 0; i < n; ++i) {
      const double ti = __shfl_sync(0xffffffffu, t, i);
      L = (j0 == 0 && i == 0) ? ti : L + ti;
    }
  }
  if (lane == 0) loss_pos[p] = L;
}

// dh[row] = sum_j ds_j * W_out[w_j] in record order (float, two roundings)
template <typename W>
__global__ void k_nce_dh(const W* __restrict__ w_out, int64_t H,
                         const uint32_t* __restrict__ rec_word, const uint32_t* __restrict__ rec_row,
                         const float* __restrict__ ds, int K1, float* __restrict__ dh) {
  const int64_t p = blockIdx.x;
  const int64_t r0 = p * K1;
  float* out = dh + (int64_t)rec_row[r0] * H;
  if ((H % 4) == 0) {
    // float4 columns; eight records' rows in flight before their adds
    const int64_t H4 = H / 4;
    for (int64_t i4 = threadIdx.x; i4 < H4; i4 += blockDim.x) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      auto add = [&](float d, float4 w) {
        acc.x = __fadd_rn(acc.x, __fmul_rn(d, w.x));
        acc.y = __fadd_rn(acc.y, __fmul_rn(d, w.y));
        acc.z = __fadd_rn(acc.z, __fmul_rn(d, w.z));
        acc.w = __fadd_rn(acc.w, __fmul_rn(d, w.w));
      };
      int j = 0;
      for (; j + 8 <= K1; j += 8) {
        float4 w[8];
        float d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          d[u] = __ldg(ds + r0 + j + u);
          w[u] = ld_f4(w_out + (int64_t)__ldg(rec_word + r0 + j + u) * H, i4);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) add(d[u], w[u]);
      }
      for (; j < K1; ++j)
        add(__ldg(ds + r0 + j), ld_f4(w_out + (int64_t)__ldg(rec_word + r0 + j) * H, i4));
      reinterpret_cast<float4*>(out)[i4] = acc;
    }
    return;
  }
  for (int64_t i = threadIdx.x; i < H; i += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < K1; ++j)
      acc = __fadd_rn(acc, __fmul_rn(ds[r0 + j], ld_f(w_out + (int64_t)rec_word[r0 + j] * H + i)));
    out[i] = acc;
  }
}

// sort input in processing order: key = word, value = q
__global__ void k_nce_sort_in(const uint32_t* __restrict__ proc_r,
                              const uint32_t* __restrict__ rec_word, int64_t N,
                              uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= N) return;
  keys[q] = rec_word[proc_r[q]];
  vals[q] = (uint32_t)q;
}

// after the stable sort: segment-head flags, and the rows / factors of the
// segmented sums in sorted order
__global__ void k_nce_sorted(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                             const uint32_t* __restrict__ proc_r,
                             const uint32_t* __restrict__ rec_row, const float* __restrict__ ds,
                             int64_t N, int* __restrict__ head, int* __restrict__ order_pos,
                             float* __restrict__ order_scale) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
  const uint32_t r = proc_r[vals[i]];
  order_pos[i] = (int)rec_row[r];
  order_scale[i] = ds[r];
}

__global__ void k_nce_heads(const uint32_t* __restrict__ keys, const int* __restrict__ head,
                            const int* __restrict__ slot, int64_t N, int* __restrict__ seg_start,
                            uint32_t* __restrict__ words, int* __restrict__ n_seg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (head[i]) {
    seg_start[slot[i]] = (int)i;
    words[slot[i]] = keys[i];
  }
  if (i == N - 1) {
    const int total = slot[i] + head[i];
    *n_seg = total;
    seg_start[total] = (int)N;
  }
}

__global__ void k_nce_long(const int* __restrict__ seg_start, const int* __restrict__ n_seg,
                           int short_max, int* __restrict__ long_list, int* __restrict__ n_long) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= *n_seg) return;
  if (seg_start[s + 1] - seg_start[s] > short_max) long_list[atomicAdd(n_long, 1)] = s;
}

// Unmasked positions of the window in t-major order (one block): pos_of[p] =
// t*B + b of the p-th, first[t] = index of row t's first one (first[T] = P).
__global__ void k_nce_positions(const uint8_t* __restrict__ w, int64_t T, int64_t B,
                                uint32_t* __restrict__ pos_of, int* __restrict__ first) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x % 32, wid = threadIdx.x / 32, nw = blockDim.x / 32;
  const int64_t n = T * B;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t i = base + threadIdx.x;
    const int f = (i < n && w[i]) ? 1 : 0;
    // block-wide exclusive scan of f
    int x = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < nw) warp_tot[lane] = v;  // inclusive warp prefix
    }
    __syncthreads();
    const int excl = carry + (wid > 0 ? warp_tot[wid - 1] : 0) + x - f;
    if (i < n) {
      if (i % B == 0) first[i / B] = excl;  // row t starts here
      if (f) pos_of[excl] = (uint32_t)i;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_tot[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) first[T] = carry;
}

// Records of the window from the raw mt19937_64 outputs (2 per draw, in
// the reference's draw order): AliasSampler::sample (rng.hpp:91-94) with
// uniform_index / uniform01 (rng.hpp:37-50) -- the same IEEE double
// operations as the host, so the words are identical.
__global__ void k_nce_records(const uint32_t* __restrict__ y, const uint32_t* __restrict__ pos_of,
                              const int* __restrict__ first, int64_t B, int64_t P, int K1,
                              const unsigned long long* __restrict__ raw,
                              const double* __restrict__ prob, const uint32_t* __restrict__ alias,
                              int64_t V, uint32_t* __restrict__ rec_word,
                              uint32_t* __restrict__ rec_row, uint32_t* __restrict__ proc_r,
                              int64_t T) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= P * K1) return;
  const int64_t p = r / K1;
  const int j = (int)(r % K1);
  const uint32_t idx = pos_of[p];
  uint32_t word;
  if (j == 0) {
    word = y[idx];
  } else {
    const int64_t d = p * (K1 - 1) + (j - 1);
    const double u1 = (double)(raw[2 * d] >> 11) * 0x1.0p-53;
    const uint64_t i = (uint64_t)(u1 * (double)V);
    const double u2 = (double)(raw[2 * d + 1] >> 11) * 0x1.0p-53;
    word = u2 < prob[i] ? (uint32_t)i : alias[i];
  }
  rec_word[r] = word;
  rec_row[r] = idx;
  // processing order: rows t descending, positions ascending, records ascending
  const int64_t t = idx / B;
  const int64_t q_pos = (P - first[t + 1]) + (p - first[t]);
  proc_r[q_pos * K1 + j] = (uint32_t)r;
  (void)T;
}

}  // namespace

void nce_records(const uint8_t* w, const uint32_t* y, int64_t T, int64_t B, int64_t P, int K1,
                 const unsigned long long* raw, const double* prob, const uint32_t* alias,
                 int64_t V, uint32_t* pos_of, int* first, uint32_t* rec_word, uint32_t* rec_row,
                 uint32_t* proc_r, cudaStream_t st) {
  k_nce_positions<<<1, 1024, 0, st>>>(w, T, B, pos_of, first);
  const int64_t N = P * K1;
  if (N > 0)
    k_nce_records<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
        y, pos_of, first, B, P, K1, raw, prob, alias, V, rec_word, rec_row, proc_r, T);
}

void nce_scores(const float* h, const float* w_out, int64_t H, const uint32_t* rec_word,
                const uint32_t* rec_row, int64_t N, float* score, cudaStream_t st,
                const bf16* w_bf) {
  if (N <= 0) return;
  const int64_t threads = N * 8;
  const unsigned g = (unsigned)((threads + 255) / 256);
  if (w_bf)
    k_nce_scores<<<g, 256, 0, st>>>(h, w_bf, H, rec_word, rec_row, N, score);
  else
    k_nce_scores<<<g, 256, 0, st>>>(h, w_out, H, rec_word, rec_row, N, score);
}

void nce_loss(const float* score, const uint32_t* rec_word, const double* ln_kq, int64_t P,
              int K1, double scale, double* loss_pos, float* ds, cudaStream_t st) {
  if (P <= 0) return;
  k_nce_loss<<<(unsigned)((P * 32 + 127) / 128), 128, 0, st>>>(score, rec_word, ln_kq, P, K1,
                                                               scale, loss_pos, ds);
}

void nce_dh(const float* w_out, int64_t H, const uint32_t* rec_word, const uint32_t* rec_row,
            const float* ds, int64_t P, int K1, float* dh, cudaStream_t st, const bf16* w_bf) {
  if (P <= 0) return;
  if (w_bf)
    k_nce_dh<<<(unsigned)P, 256, 0, st>>>(w_bf, H, rec_word, rec_row, ds, K1, dh);
  else
    k_nce_dh<<<(unsigned)P, 256, 0, st>>>(w_out, H, rec_word, rec_row, ds, K1, dh);
}

size_t nce_sort_temp_bytes(int64_t N) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)N);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const int*)nullptr, (int*)nullptr, (int)N);
  return std::max(a, b);
}

void nce_out_rows(const NceRecs& R, int64_t N, int64_t V, const float* h, int64_t H, float clip,
                  EmbedWs& ws, float* order_scale, float* rows, uint32_t* words, int* n_rows,
                  int* nonfinite, cudaStream_t st) {
  if (N <= 0) {
    DL_CUDA(cudaMemsetAsync(n_rows, 0, sizeof(int), st));
    return;
  }
  const unsigned g = (unsigned)((N + 255) / 256);
  k_nce_sort_in<<<g, 256, 0, st>>>(R.proc_r, R.rec_word, N, R.keys_in, R.vals_in);
  int end_bit = 1;
  while ((int64_t(1) << end_bit) <= V) ++end_bit;
  size_t tb = R.temp_bytes;
  DL_CUDA(cub::DeviceRadixSort::SortPairs(R.temp, tb, R.keys_in, R.keys_out, R.vals_in,
                                          R.vals_out, (int)N, 0, end_bit, st));
  k_nce_sorted<<<g, 256, 0, st>>>(R.keys_out, R.vals_out, R.proc_r, R.rec_row, R.ds, N, R.head,
                                  ws.order_pos, order_scale);
  tb = R.temp_bytes;
  DL_CUDA(cub::DeviceScan::ExclusiveSum(R.temp, tb, R.head, R.slot, (int)N, st));
  k_nce_heads<<<g, 256, 0, st>>>(R.keys_out, R.head, R.slot, N, ws.seg_start, words, n_rows);
  DL_CUDA(cudaMemsetAsync(ws.n_long(), 0, sizeof(int), st));
  k_nce_long<<<g, 256, 0, st>>>(ws.seg_start, n_rows, embed_short_max(), ws.long_list(),
                                ws.n_long());
  embed_rows(N, h, H, clip, ws, rows, n_rows, nonfinite, st, order_scale);
}

// NoiseModel (nce.hpp:41-66) + AliasSampler (rng.hpp:54-89) tables, host side:
// q = max(count/total, floor) renormalised, ln(k q), and the alias tables
// built with the reference's small/large stack discipline (bit-identical
// sampling).
void noise_tables(const double* counts, int64_t V, int k, double floor, std::vector<double>& lnkq,
                  std::vector<double>& prob, std::vector<uint32_t>& alias) {
  double total = 0.0;
  for (int64_t w = 0; w < V; ++w) {
    DL_REQUIRE(counts[w] >= 0.0, 1, "NoiseModel: negative count");
    total += counts[w];
  }
  DL_REQUIRE(total > 0.0, 1, "NoiseModel: zero total");
  std::vector<double> q(V);
  double qsum = 0.0;
  for (int64_t w = 0; w < V; ++w) {
    q[w] = std::max(counts[w] / total, floor);
    qsum += q[w];
  }
  for (int64_t w = 0; w < V; ++w) q[w] /= qsum;
  noise_tables_q(q.data(), V, k, lnkq, prob, alias);
}

// ln(k q) and AliasSampler(q) from NoiseModel's normalised distribution
// (nce.hpp:60-64; rng.hpp:54-89): the caller already built q.
void noise_tables_q(const double* q, int64_t V, int k, std::vector<double>& lnkq,
                    std::vector<double>& prob, std::vector<uint32_t>& alias) {
  lnkq.assign(V, 0.0);
  for (int64_t w = 0; w < V; ++w) {
    DL_REQUIRE(q[w] > 0.0, 1, "NoiseModel: distribution must be positive");
    lnkq[w] = std::log(static_cast<double>(k) * q[w]);
  }
  double tw = 0.0;
  for (int64_t i = 0; i < V; ++i) tw += q[i];
  std::vector<double> scaled(V);
  prob.assign(V, 0.0);
  alias.assign(V, 0);
  std::vector<uint32_t> small, large;
  small.reserve(V);
  large.reserve(V);
  for (int64_t i = 0; i < V; ++i) {
    scaled[i] = q[i] * static_cast<double>(V) / tw;
    (scaled[i] < 1.0 ? small : large).push_back(static_cast<uint32_t>(i));
  }
  while (!small.empty() && !large.empty()) {
    const uint32_t sm = small.back();
    small.pop_back();
    const uint32_t lg = large.back();
    large.pop_back();
    prob[sm] = scaled[sm];
    alias[sm] = lg;
    scaled[lg] = (scaled[lg] + scaled[sm]) - 1.0;
    (scaled[lg] < 1.0 ? small : large).push_back(lg);
  }
  for (uint32_t i : large) prob[i] = 1.0;
  for (uint32_t i : small) prob[i] = 1.0;
}

}  // namespace dl
