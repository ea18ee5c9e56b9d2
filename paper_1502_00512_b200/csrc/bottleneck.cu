// Bottleneck / tied-embedding model on the device (compress.hpp:38-415).
//
//   h_{t+1} = act(E[x_t] . U + W_rec . h_t),  z = h . D,  s_w = E[w] . z
//
// E [V x P] is both the input embedding and the output layer, U [P x H],
// W_rec [H x H], D [H x P].  One window (bptt_run over BottleneckAdapter,
// backprop.hpp:76-222 + compress.hpp:121-244, softmax mode) is laid out as
// whole-window GEMMs around the shared recurrence kernels:
//
//   forward   Eg = E[x] (gather, T*B x P); XU = Eg . U (all steps at once);
//             h_{t+1} = act(h_t . W_rec^T + XU_t)   (rec kernels: XU is the
//             "W_in" table indexed by position, x = 0..T*B-1)
//             Z = Hs . D;  logits = Z . E^T -> softmax rows (dS in place)
//   backward  dZ = dS . E;  gE = dS^T . Z;  dh_out = dZ . D^T;  gD = Hs^T . dZ
//             dpre_t = (dh_out_t + dpre_{t+1} . W_rec) * act'(h_{t+1})
//             gRec = sum_t dpre_t^T . h_t;  gU = Eg^T . dpre;  din = dpre . U^T
//             gE[x] += din (deterministic segmented sums by word, the
//             reference's first-touch order), then every gradient is clipped
//             and checked for non-finite values (compress.hpp:96-114)
//   update    bottleneck_update (compress.hpp:296-309): E dense rows (one
//             accumulator per word), U / W_rec / D per element
//
// NCE mode (LossMode::kNce, the reference Trainer's default): the same
// window with the output side replaced by the engine's NCE kernels (nce.cu)
// over z and E: host-drawn reference noise (mt19937_64 + AliasSampler),
// 8-lane double scores float(z_b . E[w]), dz from the records, and a sparse
// embedding gradient -- the output records' rows plus the input rows, each
// summed per word in the reference's processing order -- applied with the
// sparse row update (rmsprop.hpp:77-92: every accumulator decays, touched
// rows step).
//
// The GEMMs are the engine's: tcgen05 (bf16 operands, fp32 accumulate) in
// the BF16 mode, the fp32 SIMT kernel in the parity mode.  All buffers are
// device resident; host arrays are only read/written by the C ABI calls.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <tuple>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/desklm_cuda.h"
#include "kernels.cuh"

using namespace dl;

struct dl_bn {
  int device = 0;
  int64_t V = 0, H = 0, P = 0;
  int act = 0;
  int precision = DL_FP32;
  cudaStream_t st = nullptr;
  std::string err;
  double rho = 0.9995, eps = 1e-6;
  uint64_t launches = 0;
  // parameters (fp32 masters) and their bf16 operand copies
  float *e = nullptr, *u = nullptr, *w_rec = nullptr, *d = nullptr;
  bf16 *e_bf = nullptr, *u_bf = nullptr, *w_rec_bf = nullptr, *d_bf = nullptr;
  // rmsprop accumulators (compress.hpp:252-278)
  float *m_e = nullptr, *m_u = nullptr, *m_rec = nullptr, *m_d = nullptr;
  // gradients
  float *g_e = nullptr, *g_u = nullptr, *g_rec = nullptr, *g_d = nullptr;
  int* nonfinite = nullptr;
  bool have_grads = false;
  // window buffers, sized for capN = T*B rows (and capT steps)
  int64_t capN = 0, capT = 0;
  uint32_t *x = nullptr, *y = nullptr, *iota = nullptr;
  uint8_t* w = nullptr;
  float* htape = nullptr;  // [(T+1) x B x H]
  bf16* htape_bf = nullptr;
  float* eg = nullptr;  // [N x P]
  bf16* eg_bf = nullptr;
  float* xu = nullptr;  // [N x H]
  float* z = nullptr;   // [N x P]
  bf16* z_bf = nullptr;
  void* S = nullptr;  // logits / dS [N x V] (fp32, or bf16 in the BF16 mode)
  float2* part = nullptr;
  int part_tiles = 0;
  float* tgt_logit = nullptr;
  float* dz = nullptr;
  bf16* dz_bf = nullptr;
  float* dh = nullptr;
  float* dpre = nullptr;
  bf16* dpre_bf = nullptr;
  float* din = nullptr;
  double* loss_row = nullptr;
  double* logp_row = nullptr;
  double* d_loss = nullptr;
  unsigned long long* d_pos = nullptr;
  EmbedWs ews{};
  float* in_rows = nullptr;
  uint32_t* in_words = nullptr;
  int* in_n = nullptr;
  float* splitws = nullptr;
  size_t split_cap = 0;
  unsigned* bar_counter = nullptr;
  // NCE mode
  int loss_mode = 1;  // 1 softmax, 0 NCE
  int nce_k = 0;
  std::vector<double> nz_prob;
  double *ln_kq_d = nullptr, *nz_prob_d = nullptr;
  uint32_t* nz_alias_d = nullptr;
  std::mt19937_64 rng{1};
  int64_t nce_cap = 0, nce_P = 0, nce_N = 0;
  unsigned long long* raw_d = nullptr;
  std::vector<unsigned long long> raw_h;
  uint32_t *pos_of_d = nullptr, *rec_word = nullptr, *rec_row = nullptr, *proc_r = nullptr;
  int* first_d = nullptr;
  float *score = nullptr, *ds = nullptr, *nce_scale = nullptr, *out_rows = nullptr;
  double* loss_pos = nullptr;
  uint32_t *keys_in = nullptr, *vals_in = nullptr, *keys_out = nullptr, *vals_out = nullptr;
  uint32_t* out_words = nullptr;
  int *head = nullptr, *slot = nullptr, *out_n = nullptr;
  void* sort_temp = nullptr;
  size_t sort_temp_bytes = 0;
  EmbedWs nce_ws{};
  uint8_t* touched = nullptr;  // [V] rows of the sparse embedding gradient
  bool e_sparse = false;       // the last window's embedding gradient is sparse
  // softmax-mode training windows replay one CUDA graph per (T, B, scale,
  // clip, eta); buffers are sized by an eager run first
  std::map<std::tuple<int64_t, int64_t, double, float, double>, cudaGraphExec_t> graphs;
  std::map<std::tuple<int64_t, int64_t, double, float, double>, uint64_t> graph_launches;
  bool use_graphs = true;
  // device-resident epoch schedule (dl_bn_trainer_*): the stream, the
  // offset-stream cursors and hidden carry, the window counter and the run's
  // loss / position / skipped-update sums; softmax windows replay one graph
  int64_t L = 0;
  int noffset = 0, minibatch = 0, unroll = 0;
  double clip = 1.0;
  uint32_t bos = 1;
  uint32_t* ids = nullptr;
  std::vector<uint32_t> h_ids;  // (NCE: the host mirrors the schedule to draw)
  int64_t* cursors = nullptr;
  float* hidden = nullptr;
  int64_t* win_counter = nullptr;
  double* t_loss = nullptr;
  unsigned long long *t_pos = nullptr, *t_skipped = nullptr;
  cudaGraphExec_t tgraph = nullptr;
  double tgraph_eta = 0.0;
  uint64_t tgraph_launches = 0;
  bool tgraph_sized = false;
};

namespace {

thread_local std::string g_bn_err;

int bn_fail(dl_bn* c, int code, const std::string& m) {
  g_bn_err = m;
  if (c) c->err = m;
  return code;
}

template <class F>
int bn_guarded(dl_bn* c, F&& f) {
  try {
    if (c) DL_CUDA(cudaSetDevice(c->device));
    f();
    return DL_OK;
  } catch (const Error& e) {
    return bn_fail(c, e.code, e.what());
  } catch (const std::exception& e) {
    return bn_fail(c, DL_EDEVICE, e.what());
  }
}

template <class T>
T* bn_alloc(size_t n) {
  void* p = nullptr;
  DL_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return static_cast<T*>(p);
}

template <class T>
void bn_free(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

bool tcm(const dl_bn* c) { return c->precision == DL_BF16; }

// ------------------------------------------------------------- kernels
// gathered embedding rows Eg[n] = E[x[n]] (BottleneckAdapter::gather,
// compress.hpp:159-168), fp32 and (optionally) the bf16 operand copy
__global__ void k_gather_rows(const float* __restrict__ e, const uint32_t* __restrict__ x,
                              int64_t n, int64_t P, float* __restrict__ out,
                              bf16* __restrict__ outb) {
  const int64_t total = n * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / P, k = i - r * P;
    const float v = e[(int64_t)x[r] * P + k];
    out[i] = v;
    if (outb) outb[i] = __float2bfloat16_rn(v);
  }
}

__global__ void k_iota(uint32_t* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (uint32_t)i;
}

// gE[words[s]] += rows[s] for the window's distinct input words (each word
// once, so no two slots touch the same row)
__global__ void k_add_rows(const float* __restrict__ rows, const uint32_t* __restrict__ words,
                           const int* __restrict__ n_seg, int64_t P, float* __restrict__ dense,
                           uint8_t* __restrict__ touched) {
  const int slot = blockIdx.x;
  if (slot >= *n_seg) return;
  if (touched && threadIdx.x == 0) touched[words[slot]] = 1;
  float* dst = dense + (int64_t)words[slot] * P;
  const float* src = rows + (int64_t)slot * P;
  for (int64_t j = threadIdx.x; j < P; j += blockDim.x) dst[j] += src[j];
}

// update_rows_sparse (rmsprop.hpp:77-92) over a dense gradient with a
// touched-row mask: every accumulator decays, m = float(rho m); a touched
// row then takes m += float((1-rho) mean_sq) and w -= float(eta g / sqrt(m +
// eps)).  One warp per row; skipped entirely on a non-finite gradient.
__global__ void k_rms_rows_masked(float* __restrict__ w, bf16* __restrict__ wb,
                                  float* __restrict__ m, const float* __restrict__ g,
                                  const uint8_t* __restrict__ touched, int64_t V, int64_t P,
                                  double rho, double eps, double eta,
                                  const int* __restrict__ nonfinite) {
  if (*nonfinite) return;
  const int lane = threadIdx.x % 32;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < V; r += nw) {
    float mr = (float)(rho * (double)m[r]);
    if (touched[r]) {
      const float* gr = g + r * P;
      double sq = 0.0;
      for (int64_t i = lane; i < P; i += 32) sq += (double)gr[i] * (double)gr[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
      mr = mr + (float)((1.0 - rho) * (sq / (double)P));
      const double denom = sqrt((double)mr + eps), inv = 1.0 / denom;
      float* wr = w + r * P;
      for (int64_t i = lane; i < P; i += 32) {
        const float v = wr[i] - rms_step(eta, gr[i], denom, inv);
        wr[i] = v;
        if (wb) wb[r * P + i] = __float2bfloat16_rn(v);
      }
    }
    if (lane == 0) m[r] = mr;
  }
}

// dequantize_matrix (compress.hpp:481-488) on the device: code i is bits
// [i*bits, (i+1)*bits) of the packed payload, least-significant bit first;
// value = float(double(min) + step * code).
__global__ void k_dequant(const uint8_t* __restrict__ codes, int64_t nbytes, int64_t n, int bits,
                          float mn, double step, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bit = i * bits;
    const int64_t b0 = bit >> 3;
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (b0 + j < nbytes) word |= (uint32_t)codes[b0 + j] << (8 * j);
    const uint32_t code = (word >> (bit & 7)) & ((1u << bits) - 1u);
    out[i] = (float)((double)mn + step * (double)code);
  }
}

unsigned grid_n(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// ------------------------------------------------------------- GEMMs
GemmDesc mk(int M, int N, int K, int am, const void* A, int64_t lda, int bm, const void* B,
            int64_t ldb, float* C, int64_t ldc) {
  GemmDesc g{};
  g.M = M; g.N = N; g.K = K;
  g.a_major = am; g.b_major = bm;
  g.A = A; g.B = B; g.lda = lda; g.ldb = ldb;
  g.C = C; g.ldc = ldc;
  g.k_splits = 1;
  return g;
}

int splits_for(const dl_bn* c, int M, int N, int K, int max_splits) {
  const int bn = tcm(c) ? (N >= 256 ? 256 : (N >= 128 ? 128 : 64)) : 128;
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  int s = std::max(1, std::min(max_splits, kNumSMs / std::max(1, tiles)));
  if (tcm(c)) s = tc_splits(K, s);
  else s = std::max(1, std::min(s, (K + 63) / 64));
  return s;
}

void drop_graphs(dl_bn* c);

// Grow the split-K workspace: recorded graphs hold the old pointer, so they
// are dropped (growth happens in eager windows only -- every graphed shape
// has run eagerly first)
void grow_splitws(dl_bn* c, size_t need) {
  if (need <= c->split_cap) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  DL_CUDA(cudaStreamIsCapturing(c->st, &cs));
  DL_REQUIRE(cs == cudaStreamCaptureStatusNone, DL_EDEVICE, "split workspace grown inside a capture");
  DL_CUDA(cudaStreamSynchronize(c->st));
  drop_graphs(c);
  bn_free(c->splitws);
  c->splitws = bn_alloc<float>(need);
  c->split_cap = need;
}

void run_gemm(dl_bn* c, const GemmDesc& g) {
  c->launches++;
  if (tcm(c)) gemm_tc(g, c->st);
  else gemm_f32(g, c->st);
}

// C [M x N] (ldc = N) = op(A) . op(B), split over K when the tile grid is
// small; the split partials are summed in fixed order.
void mm(dl_bn* c, int M, int N, int K, int am, const void* A, int64_t lda, int bm, const void* B,
        int64_t ldb, float* C, int max_splits = 16) {
  GemmDesc g = mk(M, N, K, am, A, lda, bm, B, ldb, C, N);
  const int s = splits_for(c, M, N, K, max_splits);
  if (s > 1) {
    const size_t need = (size_t)s * M * N;
    grow_splitws(c, need);
    g.C = c->splitws;
    g.k_splits = s;
    g.split_stride = (int64_t)M * N;
    run_gemm(c, g);
    reduce_splits(c->splitws, s, (int64_t)M * N, (int64_t)M * N, C, 0.f, 0, nullptr, c->st);
    c->launches++;
  } else {
    run_gemm(c, g);
  }
}

// ------------------------------------------------------------- buffers
void drop_graphs(dl_bn* c) {
  for (auto& kv : c->graphs)
    if (kv.second) cudaGraphExecDestroy(kv.second);
  c->graphs.clear();
  if (c->tgraph) cudaGraphExecDestroy(c->tgraph);
  c->tgraph = nullptr;
  c->tgraph_sized = false;
}

void ensure_window(dl_bn* c, int64_t T, int64_t N) {
  if (N <= c->capN && T <= c->capT) return;
  DL_CUDA(cudaStreamSynchronize(c->st));
  drop_graphs(c);
  const int64_t n = std::max(N, c->capN), t = std::max(T, c->capT);
  const int64_t H = c->H, P = c->P, V = c->V;
  for (void** p : {(void**)&c->x, (void**)&c->y, (void**)&c->iota, (void**)&c->w,
                   (void**)&c->htape, (void**)&c->htape_bf, (void**)&c->eg, (void**)&c->eg_bf,
                   (void**)&c->xu, (void**)&c->z, (void**)&c->z_bf, (void**)&c->S,
                   (void**)&c->part, (void**)&c->tgt_logit, (void**)&c->dz, (void**)&c->dz_bf,
                   (void**)&c->dh, (void**)&c->dpre, (void**)&c->dpre_bf, (void**)&c->din,
                   (void**)&c->loss_row, (void**)&c->logp_row, (void**)&c->ews.seg_start,
                   (void**)&c->ews.order_pos, (void**)&c->in_rows, (void**)&c->in_words,
                   (void**)&c->in_n})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  c->x = bn_alloc<uint32_t>(n);
  c->y = bn_alloc<uint32_t>(n);
  c->iota = bn_alloc<uint32_t>(n);
  c->w = bn_alloc<uint8_t>(n);
  // the tape holds T+1 states of n / T rows; sized for the largest row count
  // any call uses (n rows per state covers every T >= 1)
  c->htape = bn_alloc<float>((n + n) * H);
  c->eg = bn_alloc<float>(n * P);
  c->xu = bn_alloc<float>(n * H);
  c->z = bn_alloc<float>(n * P);
  c->dz = bn_alloc<float>(n * P);
  c->dh = bn_alloc<float>(n * H);
  c->dpre = bn_alloc<float>(n * H);
  c->din = bn_alloc<float>(n * P);
  c->loss_row = bn_alloc<double>(n);
  c->logp_row = bn_alloc<double>(n);
  c->tgt_logit = bn_alloc<float>(n);
  c->ews.seg_start = bn_alloc<int>(2 * n + 2);
  c->ews.order_pos = bn_alloc<int>(n);
  c->ews.cap = n;
  c->in_rows = bn_alloc<float>(n * P);
  c->in_words = bn_alloc<uint32_t>(n);
  c->in_n = bn_alloc<int>(1);
  bn_free(c->pos_of_d);
  bn_free(c->first_d);
  c->pos_of_d = bn_alloc<uint32_t>(n);
  c->first_d = bn_alloc<int>(t + 1);
  if (tcm(c)) {
    c->htape_bf = bn_alloc<bf16>((n + n) * H);
    c->eg_bf = bn_alloc<bf16>(n * P);
    c->z_bf = bn_alloc<bf16>(n * P);
    c->dz_bf = bn_alloc<bf16>(n * P);
    c->dpre_bf = bn_alloc<bf16>(n * H);
    c->S = bn_alloc<bf16>(n * V);
    c->part_tiles = tc_n_tiles((int)V);
    c->part = bn_alloc<float2>((size_t)c->part_tiles * n);
  } else {
    c->S = bn_alloc<float>(n * V);
  }
  k_iota<<<grid_n(n), 256, 0, c->st>>>(c->iota, n);
  c->capN = n;
  c->capT = t;
}

// NCE record buffers for up to N = T*B*(k+1) records
void nce_reserve(dl_bn* c, int64_t N) {
  if (N <= c->nce_cap) return;
  DL_CUDA(cudaStreamSynchronize(c->st));
  for (void** p : {(void**)&c->rec_word, (void**)&c->rec_row, (void**)&c->proc_r,
                   (void**)&c->score, (void**)&c->ds, (void**)&c->nce_scale, (void**)&c->loss_pos,
                   (void**)&c->keys_in, (void**)&c->vals_in, (void**)&c->keys_out,
                   (void**)&c->vals_out, (void**)&c->head, (void**)&c->slot, &c->sort_temp,
                   (void**)&c->nce_ws.seg_start, (void**)&c->nce_ws.order_pos,
                   (void**)&c->out_rows, (void**)&c->out_words, (void**)&c->out_n,
                   (void**)&c->raw_d})
    if (*p) {
      cudaFree(*p);
      *p = nullptr;
    }
  c->rec_word = bn_alloc<uint32_t>(N);
  c->rec_row = bn_alloc<uint32_t>(N);
  c->proc_r = bn_alloc<uint32_t>(N);
  c->score = bn_alloc<float>(N);
  c->ds = bn_alloc<float>(N);
  c->nce_scale = bn_alloc<float>(N);
  c->loss_pos = bn_alloc<double>(N);
  c->keys_in = bn_alloc<uint32_t>(N);
  c->vals_in = bn_alloc<uint32_t>(N);
  c->keys_out = bn_alloc<uint32_t>(N);
  c->vals_out = bn_alloc<uint32_t>(N);
  c->head = bn_alloc<int>(N);
  c->slot = bn_alloc<int>(N);
  c->sort_temp_bytes = nce_sort_temp_bytes(N);
  c->sort_temp = bn_alloc<uint8_t>(c->sort_temp_bytes);
  c->nce_ws.seg_start = bn_alloc<int>(2 * N + 2);
  c->nce_ws.order_pos = bn_alloc<int>(N);
  c->nce_ws.cap = N;
  c->out_rows = bn_alloc<float>(N * c->P);
  c->out_words = bn_alloc<uint32_t>(N);
  c->out_n = bn_alloc<int>(1);
  c->raw_d = bn_alloc<unsigned long long>(2 * N);
  c->nce_cap = N;
}

void refresh_shadows(dl_bn* c) {
  if (!tcm(c)) return;
  f32_to_bf16(c->e, c->e_bf, c->V * c->P, c->st);
  f32_to_bf16(c->u, c->u_bf, c->P * c->H, c->st);
  f32_to_bf16(c->w_rec, c->w_rec_bf, c->H * c->H, c->st);
  f32_to_bf16(c->d, c->d_bf, c->H * c->P, c->st);
  c->launches += 4;
}

float act0(int act) { return act == 0 ? 0.5f : 0.0f; }

// ------------------------------------------------------------- forward
// Recurrence over T steps of Bn rows from htape[0]: the input term of row
// (t, b) is XU[t*Bn + b] (compress.hpp:170-174 hoisted out of the loop).
void recurrence_fwd(dl_bn* c, int64_t T, int64_t Bn) {
  const int64_t H = c->H, BH = Bn * H;
  if (tcm(c)) {
    f32_to_bf16(c->htape, c->htape_bf, BH, c->st);
    c->launches++;
    if (rec_window_tc(0, (int)T, (int)Bn, (int)H, c->act, c->htape_bf, (T + 1) * Bn, c->w_rec_bf,
                      c->xu, c->iota, nullptr, nullptr, c->htape, c->htape_bf, c->bar_counter,
                      c->st)) {
      c->launches++;
      return;
    }
  }
  for (int64_t t = 0; t < T; ++t) {
    const int s = splits_for(c, (int)Bn, (int)H, (int)H, 32);
    const size_t need = (size_t)s * BH;
    grow_splitws(c, need);
    GemmDesc g = tcm(c) ? mk((int)Bn, (int)H, (int)H, K_MAJOR, c->htape_bf + t * BH, H, K_MAJOR,
                             c->w_rec_bf, H, c->splitws, H)
                        : mk((int)Bn, (int)H, (int)H, K_MAJOR, c->htape + t * BH, H, K_MAJOR,
                             c->w_rec, H, c->splitws, H);
    g.k_splits = s;
    g.split_stride = BH;
    run_gemm(c, g);
    rec_fwd(c->splitws, s, BH, Bn, H, c->xu + t * BH, c->iota, c->act, c->htape + (t + 1) * BH,
            tcm(c) ? c->htape_bf + (t + 1) * BH : nullptr, c->st);
    c->launches++;
  }
}

// Eg, XU for N positions of ids x (device)
void input_side(dl_bn* c, int64_t N) {
  k_gather_rows<<<grid_n(N * c->P), 256, 0, c->st>>>(c->e, c->x, N, c->P, c->eg,
                                                      tcm(c) ? c->eg_bf : nullptr);
  c->launches++;
  // XU = Eg . U  [N x H]  (matmul_nn, compress.hpp:173)
  if (tcm(c))
    mm(c, (int)N, (int)c->H, (int)c->P, K_MAJOR, c->eg_bf, c->P, MN_MAJOR, c->u_bf, c->H, c->xu);
  else
    mm(c, (int)N, (int)c->H, (int)c->P, K_MAJOR, c->eg, c->P, MN_MAJOR, c->u, c->H, c->xu);
}

// Z = Hs . D and the softmax rows over E (compress.hpp:195-202, 227-230);
// writes loss_row / logp_row, leaves dS in S when grads
void output_side(dl_bn* c, int64_t N, const float* hs, const bf16* hs_bf, double scale,
                 bool grads) {
  const int64_t H = c->H, P = c->P, V = c->V;
  if (tcm(c)) {
    mm(c, (int)N, (int)P, (int)H, K_MAJOR, hs_bf, H, MN_MAJOR, c->d_bf, P, c->z);
    f32_to_bf16(c->z, c->z_bf, N * P, c->st);
    c->launches++;
    GemmDesc g = mk((int)N, (int)V, (int)P, K_MAJOR, c->z_bf, P, K_MAJOR, c->e_bf, P, nullptr, 0);
    g.logits = 1;
    g.S = grads ? static_cast<bf16*>(c->S) : nullptr;
    g.lds = V;
    g.part = c->part;
    g.part_n = c->part_tiles;
    g.tgt = c->y;
    g.tgt_logit = c->tgt_logit;
    run_gemm(c, g);
    softmax_rows_bf16(grads ? static_cast<bf16*>(c->S) : nullptr, N, V, c->part, c->part_tiles,
                      c->tgt_logit, c->y, c->w, scale, grads ? 1 : 0, c->loss_row, c->logp_row,
                      c->st);
  } else {
    mm(c, (int)N, (int)P, (int)H, K_MAJOR, hs, H, MN_MAJOR, c->d, P, c->z);
    GemmDesc g = mk((int)N, (int)V, (int)P, K_MAJOR, c->z, P, K_MAJOR, c->e, P,
                    static_cast<float*>(c->S), V);
    run_gemm(c, g);
    softmax_rows_f32(static_cast<float*>(c->S), N, V, c->y, c->w, scale, grads ? 1 : 0,
                     c->loss_row, c->logp_row, c->st);
  }
  c->launches++;
}

void check_ids(const dl_bn* c, const uint32_t* ids, int64_t n, const char* what) {
  for (int64_t i = 0; i < n; ++i)
    DL_REQUIRE(ids[i] < (uint64_t)c->V, DL_EDATA, std::string(what) + ": id out of vocabulary range");
}

// ------------------------------------------------------------- window
void run_window(dl_bn* c, int64_t T, int64_t B, double scale, float clip, bool grads) {
  const int64_t H = c->H, P = c->P, V = c->V, N = T * B, BH = B * H;
  cudaStream_t st = c->st;
  const bool nce = c->loss_mode == 0;
  const bool t16 = tcm(c);
  input_side(c, N);
  recurrence_fwd(c, T, B);
  const float* Hs = c->htape + BH;
  const bf16* Hs_bf = t16 ? c->htape_bf + BH : nullptr;
  DL_CUDA(cudaMemsetAsync(c->d_loss, 0, sizeof(double), st));
  DL_CUDA(cudaMemsetAsync(c->d_pos, 0, sizeof(unsigned long long), st));
  const int K1 = c->nce_k + 1;
  if (nce) {
    // Z = Hs . D, then the NCE records over z and E (backprop.hpp:126-156;
    // compress.hpp:204-207)
    if (t16)
      mm(c, (int)N, (int)P, (int)H, K_MAJOR, Hs_bf, H, MN_MAJOR, c->d_bf, P, c->z);
    else
      mm(c, (int)N, (int)P, (int)H, K_MAJOR, Hs, H, MN_MAJOR, c->d, P, c->z);
    nce_records(c->w, c->y, T, B, c->nce_P, K1, c->raw_d, c->nz_prob_d, c->nz_alias_d, V,
                c->pos_of_d, c->first_d, c->rec_word, c->rec_row, c->proc_r, st);
    nce_scores(c->z, c->e, P, c->rec_word, c->rec_row, c->nce_N, c->score, st);
    nce_loss(c->score, c->rec_word, c->ln_kq_d, c->nce_P, K1, scale, c->loss_pos, c->ds, st);
    sum_rows(c->loss_pos, nullptr, c->nce_P, c->d_loss, c->d_pos, st);
    c->launches += 5;
  } else {
    output_side(c, N, Hs, Hs_bf, scale, grads);
    sum_rows(c->loss_row, c->w, N, c->d_loss, c->d_pos, st);
    c->launches++;
  }
  if (!grads) return;
  DL_CUDA(cudaMemsetAsync(c->nonfinite, 0, sizeof(int), st));
  c->e_sparse = nce;
  if (nce) {
    // score_backward of every record (compress.hpp:209-219): dz[b] += ds E[w];
    // the embedding rows sum ds * z[b] per word in processing order
    DL_CUDA(cudaMemsetAsync(c->dz, 0, N * P * sizeof(float), st));
    nce_dh(c->e, P, c->rec_word, c->rec_row, c->ds, c->nce_P, K1, c->dz, st);
    DL_CUDA(cudaMemsetAsync(c->g_e, 0, V * P * sizeof(float), st));
    DL_CUDA(cudaMemsetAsync(c->touched, 0, V, st));
    NceRecs R{c->rec_word, c->rec_row, c->proc_r, c->ds, c->keys_in, c->vals_in, c->keys_out,
              c->vals_out, c->head, c->slot, c->sort_temp, c->sort_temp_bytes};
    nce_out_rows(R, c->nce_N, V, c->z, P, FLT_MAX, c->nce_ws, c->nce_scale, c->out_rows,
                 c->out_words, c->out_n, nullptr, st);
    k_add_rows<<<(unsigned)std::max<int64_t>(c->nce_N, 1), 128, 0, st>>>(
        c->out_rows, c->out_words, c->out_n, P, c->g_e, c->touched);
    c->launches += 10;
    if (t16) {
      f32_to_bf16(c->dz, c->dz_bf, N * P, st);
      c->launches++;
    }
  } else if (t16) {
    // softmax_backward (compress.hpp:237-243):
    //   dZ = dS . E  [N x P];  gE = dS^T . Z  [V x P]
    mm(c, (int)N, (int)P, (int)V, K_MAJOR, c->S, V, MN_MAJOR, c->e_bf, P, c->dz);
    mm(c, (int)V, (int)P, (int)N, MN_MAJOR, c->S, V, MN_MAJOR, c->z_bf, P, c->g_e);
    f32_to_bf16(c->dz, c->dz_bf, N * P, st);
    c->launches++;
  } else {
    // softmax_backward, fp32
    mm(c, (int)N, (int)P, (int)V, K_MAJOR, c->S, V, MN_MAJOR, c->e, P, c->dz);
    mm(c, (int)V, (int)P, (int)N, MN_MAJOR, c->S, V, MN_MAJOR, c->z, P, c->g_e);
  }
  // out_end (compress.hpp:221-225): dh_out = dZ . D^T [N x H]; gD = Hs^T . dZ
  if (t16) {
    mm(c, (int)N, (int)H, (int)P, K_MAJOR, c->dz_bf, P, K_MAJOR, c->d_bf, P, c->dh);
    mm(c, (int)H, (int)P, (int)N, MN_MAJOR, Hs_bf, H, MN_MAJOR, c->dz_bf, P, c->g_d);
  } else {
    mm(c, (int)N, (int)H, (int)P, K_MAJOR, c->dz, P, K_MAJOR, c->d, P, c->dh);
    mm(c, (int)H, (int)P, (int)N, MN_MAJOR, Hs, H, MN_MAJOR, c->dz, P, c->g_d);
  }
  // backward recurrence (backprop.hpp:197-219)
  const bool persist = t16 && rec_window_tc(1, (int)T, (int)B, (int)H, c->act, c->dpre_bf, N,
                                            c->w_rec_bf, nullptr, nullptr, c->dh, c->htape,
                                            c->dpre, c->dpre_bf, c->bar_counter, st);
  if (persist) c->launches++;
  for (int64_t t = persist ? -1 : T - 1; t >= 0; --t) {
    int s = 0;
    if (t < T - 1) {
      s = splits_for(c, (int)B, (int)H, (int)H, 32);
      const size_t need = (size_t)s * BH;
      grow_splitws(c, need);
      GemmDesc g = t16 ? mk((int)B, (int)H, (int)H, K_MAJOR, c->dpre_bf + (t + 1) * BH, H, MN_MAJOR,
                            c->w_rec_bf, H, c->splitws, H)
                       : mk((int)B, (int)H, (int)H, K_MAJOR, c->dpre + (t + 1) * BH, H, MN_MAJOR,
                            c->w_rec, H, c->splitws, H);
      g.k_splits = s;
      g.split_stride = BH;
      run_gemm(c, g);
    }
    rec_bwd(c->splitws, s, BH, BH, c->dh + t * BH, c->htape + (t + 1) * BH, c->act,
            c->dpre + t * BH, t16 ? c->dpre_bf + t * BH : nullptr, st);
    c->launches++;
  }
  // gRec = sum_t dpre_t^T . h_t; gU = Eg^T . dpre (compress.hpp:179);
  // din = dpre . U^T (compress.hpp:182)
  if (t16) {
    mm(c, (int)H, (int)H, (int)N, MN_MAJOR, c->dpre_bf, H, MN_MAJOR, c->htape_bf, H, c->g_rec);
    mm(c, (int)P, (int)H, (int)N, MN_MAJOR, c->eg_bf, P, MN_MAJOR, c->dpre_bf, H, c->g_u);
    mm(c, (int)N, (int)P, (int)H, K_MAJOR, c->dpre_bf, H, K_MAJOR, c->u_bf, H, c->din);
  } else {
    mm(c, (int)H, (int)H, (int)N, MN_MAJOR, c->dpre, H, MN_MAJOR, c->htape, H, c->g_rec);
    mm(c, (int)P, (int)H, (int)N, MN_MAJOR, c->eg, P, MN_MAJOR, c->dpre, H, c->g_u);
    mm(c, (int)N, (int)P, (int)H, K_MAJOR, c->dpre, H, K_MAJOR, c->u, H, c->din);
  }
  // embedding rows of the input side: per-word sums of din in the
  // reference's processing order, added to the dense gradient
  embed_grads(c->x, T, B, 1, V, c->din, P, FLT_MAX, c->ews, c->in_rows, c->in_words, c->in_n,
              nullptr, st);
  k_add_rows<<<(unsigned)N, 128, 0, st>>>(c->in_rows, c->in_words, c->in_n, P, c->g_e,
                                          nce ? c->touched : nullptr);
  c->launches += 4;
  // BottleneckGrads::clip + finite (compress.hpp:96-114)
  reduce_splits(c->g_e, 1, 0, V * P, c->g_e, clip, 1, c->nonfinite, st);
  reduce_splits(c->g_u, 1, 0, P * H, c->g_u, clip, 1, c->nonfinite, st);
  reduce_splits(c->g_rec, 1, 0, H * H, c->g_rec, clip, 1, c->nonfinite, st);
  reduce_splits(c->g_d, 1, 0, H * P, c->g_d, clip, 1, c->nonfinite, st);
  c->launches += 4;
  c->have_grads = true;
}

// bottleneck_update (compress.hpp:296-309); skipped on the device when any
// gradient is non-finite
void run_update(dl_bn* c, double eta) {
  cudaStream_t st = c->st;
  const bool t16 = tcm(c);
  if (c->e_sparse)
    k_rms_rows_masked<<<148 * 8, 256, 0, st>>>(c->e, t16 ? c->e_bf : nullptr, c->m_e, c->g_e,
                                               c->touched, c->V, c->P, c->rho, c->eps, eta,
                                               c->nonfinite);
  else
    rms_rows(c->e, t16 ? c->e_bf : nullptr, c->m_e, c->g_e, nullptr, nullptr, c->V, c->P, c->rho,
             c->eps, eta, 1, c->nonfinite, st);
  rms_rec(c->u, t16 ? c->u_bf : nullptr, c->m_u, c->g_u, c->P * c->H, c->rho, c->eps, eta,
          c->nonfinite, st);
  rms_rec(c->w_rec, t16 ? c->w_rec_bf : nullptr, c->m_rec, c->g_rec, c->H * c->H, c->rho, c->eps,
          eta, c->nonfinite, st);
  rms_rec(c->d, t16 ? c->d_bf : nullptr, c->m_d, c->g_d, c->H * c->P, c->rho, c->eps, eta,
          c->nonfinite, st);
  c->launches += 4;
}

// The window's noise draws (t, b, then sample; masked positions draw
// nothing): 2 raw mt19937_64 outputs per draw, turned into words on the
// device with the alias tables (nce.cu k_nce_records).  (Pageable source:
// the copy has consumed raw_h when cudaMemcpyAsync returns.)
void nce_draws(dl_bn* c, const uint8_t* weights, int64_t N) {
  DL_REQUIRE(c->nce_k > 0 && !c->nz_prob.empty(), 1,
             "bptt: NCE mode needs noise model and rng (dl_bn_set_noise)");
  int64_t Pn = 0;
  for (int64_t i = 0; i < N; ++i) Pn += weights[i] ? 1 : 0;
  nce_reserve(c, std::max<int64_t>(N * (c->nce_k + 1), 1));
  const int64_t ND = 2 * Pn * c->nce_k;
  c->raw_h.resize(std::max<int64_t>(ND, 1));
  for (int64_t i = 0; i < ND; ++i) c->raw_h[i] = c->rng();
  if (ND > 0)
    DL_CUDA(cudaMemcpyAsync(c->raw_d, c->raw_h.data(), ND * 8, cudaMemcpyHostToDevice, c->st));
  c->nce_P = Pn;
  c->nce_N = Pn * (c->nce_k + 1);
}

void upload(dl_bn* c, float* dst, const float* src, int64_t n) {
  DL_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyHostToDevice, c->st));
}
void download(dl_bn* c, float* dst, const float* src, int64_t n) {
  if (dst) DL_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToHost, c->st));
}

}  // namespace

extern "C" {

const char* dl_bn_last_error(const dl_bn* c) { return c ? c->err.c_str() : g_bn_err.c_str(); }

int dl_bn_create(dl_bn** out, int device, int64_t V, int64_t H, int64_t P, int act,
                 int precision) {
  if (!out) return bn_fail(nullptr, DL_EINVAL, "dl_bn_create: null out");
  *out = nullptr;
  if (V < 1 || H < 1 || P < 1) return bn_fail(nullptr, DL_EINVAL, "BottleneckParams: V,H,P >= 1");
  if (P > H) return bn_fail(nullptr, DL_EINVAL, "BottleneckParams: P must not exceed H");
  if (act != 0 && act != 1) return bn_fail(nullptr, DL_EINVAL, "dl_bn_create: act must be 0 or 1");
  if (precision != DL_FP32 && precision != DL_BF16)
    return bn_fail(nullptr, DL_EINVAL, "dl_bn_create: precision must be DL_FP32 or DL_BF16");
  if (precision == DL_BF16 && (H % 8 || P % 8 || V % 8))
    return bn_fail(nullptr, DL_EINVAL, "dl_bn_create: BF16 mode needs V, H, P multiples of 8");
  dl_bn* c = new dl_bn();
  c->device = device;
  c->V = V; c->H = H; c->P = P;
  c->act = act;
  c->precision = precision;
  const int rc = bn_guarded(c, [&] {
    DL_CUDA(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    c->e = bn_alloc<float>(V * P);
    c->u = bn_alloc<float>(P * H);
    c->w_rec = bn_alloc<float>(H * H);
    c->d = bn_alloc<float>(H * P);
    c->m_e = bn_alloc<float>(V);
    c->m_u = bn_alloc<float>(P * H);
    c->m_rec = bn_alloc<float>(H * H);
    c->m_d = bn_alloc<float>(H * P);
    c->g_e = bn_alloc<float>(V * P);
    c->g_u = bn_alloc<float>(P * H);
    c->g_rec = bn_alloc<float>(H * H);
    c->g_d = bn_alloc<float>(H * P);
    c->nonfinite = bn_alloc<int>(1);
    c->d_loss = bn_alloc<double>(1);
    c->d_pos = bn_alloc<unsigned long long>(1);
    c->bar_counter = bn_alloc<unsigned>(256);
    DL_CUDA(cudaMemsetAsync(c->bar_counter, 0, 256 * sizeof(unsigned), c->st));
    if (precision == DL_BF16) {
      c->e_bf = bn_alloc<bf16>(V * P);
      c->u_bf = bn_alloc<bf16>(P * H);
      c->w_rec_bf = bn_alloc<bf16>(H * H);
      c->d_bf = bn_alloc<bf16>(H * P);
    }
    DL_CUDA(cudaMemsetAsync(c->e, 0, V * P * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->u, 0, P * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->w_rec, 0, H * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->d, 0, H * P * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_e, 0, V * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_u, 0, P * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_rec, 0, H * H * 4, c->st));
    DL_CUDA(cudaMemsetAsync(c->m_d, 0, H * P * 4, c->st));
    refresh_shadows(c);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
  if (rc != DL_OK) {
    g_bn_err = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return DL_OK;
}

int dl_bn_destroy(dl_bn* c) {
  if (!c) return DL_OK;
  cudaSetDevice(c->device);
  if (c->st) cudaStreamSynchronize(c->st);
  drop_graphs(c);
  for (void* p : {(void*)c->e, (void*)c->u, (void*)c->w_rec, (void*)c->d, (void*)c->e_bf,
                  (void*)c->u_bf, (void*)c->w_rec_bf, (void*)c->d_bf, (void*)c->m_e,
                  (void*)c->m_u, (void*)c->m_rec, (void*)c->m_d, (void*)c->g_e, (void*)c->g_u,
                  (void*)c->g_rec, (void*)c->g_d, (void*)c->nonfinite, (void*)c->x, (void*)c->y,
                  (void*)c->iota, (void*)c->w, (void*)c->htape, (void*)c->htape_bf, (void*)c->eg,
                  (void*)c->eg_bf, (void*)c->xu, (void*)c->z, (void*)c->z_bf, c->S,
                  (void*)c->part, (void*)c->tgt_logit, (void*)c->dz, (void*)c->dz_bf,
                  (void*)c->dh, (void*)c->dpre, (void*)c->dpre_bf, (void*)c->din,
                  (void*)c->loss_row, (void*)c->logp_row, (void*)c->d_loss, (void*)c->d_pos,
                  (void*)c->ews.seg_start, (void*)c->ews.order_pos, (void*)c->in_rows,
                  (void*)c->in_words, (void*)c->in_n, (void*)c->splitws, (void*)c->bar_counter,
                  (void*)c->ln_kq_d, (void*)c->nz_prob_d, (void*)c->nz_alias_d, (void*)c->raw_d,
                  (void*)c->pos_of_d, (void*)c->first_d, (void*)c->rec_word, (void*)c->rec_row,
                  (void*)c->proc_r, (void*)c->score, (void*)c->ds, (void*)c->nce_scale,
                  (void*)c->loss_pos, (void*)c->keys_in, (void*)c->vals_in, (void*)c->keys_out,
                  (void*)c->vals_out, (void*)c->head, (void*)c->slot, c->sort_temp,
                  (void*)c->nce_ws.seg_start, (void*)c->nce_ws.order_pos, (void*)c->out_rows,
                  (void*)c->out_words, (void*)c->out_n, (void*)c->touched, (void*)c->ids,
                  (void*)c->cursors, (void*)c->hidden, (void*)c->win_counter, (void*)c->t_loss,
                  (void*)c->t_pos, (void*)c->t_skipped})
    if (p) cudaFree(p);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
  return DL_OK;
}

int dl_bn_set_params(dl_bn* c, const float* e, const float* u, const float* w_rec,
                     const float* d) {
  if (!c || !e || !u || !w_rec || !d) return bn_fail(c, DL_EINVAL, "dl_bn_set_params: null argument");
  return bn_guarded(c, [&] {
    upload(c, c->e, e, c->V * c->P);
    upload(c, c->u, u, c->P * c->H);
    upload(c, c->w_rec, w_rec, c->H * c->H);
    upload(c, c->d, d, c->H * c->P);
    refresh_shadows(c);
    c->have_grads = false;
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_set_params_quantized(dl_bn* c, const dl_qmatrix m[4]) {
  if (!c || !m) return bn_fail(c, DL_EINVAL, "dl_bn_set_params_quantized: null argument");
  const int64_t rows[4] = {c->V, c->P, c->H, c->H}, cols[4] = {c->P, c->H, c->H, c->P};
  for (int k = 0; k < 4; ++k) {
    if (m[k].bits < 1 || m[k].bits > 16) return bn_fail(c, DL_EDATA, "quantized model: bits out of range");
    if (!m[k].codes) return bn_fail(c, DL_EINVAL, "dl_bn_set_params_quantized: null codes");
  }
  return bn_guarded(c, [&] {
    float* dst[4] = {c->e, c->u, c->w_rec, c->d};
    for (int k = 0; k < 4; ++k) {
      const int64_t n = rows[k] * cols[k];
      const int64_t nbytes = (n * m[k].bits + 7) / 8;
      uint8_t* dcodes = bn_alloc<uint8_t>(nbytes);
      DL_CUDA(cudaMemcpyAsync(dcodes, m[k].codes, nbytes, cudaMemcpyHostToDevice, c->st));
      // QuantizedMatrix::step (compress.hpp:431-436)
      const double range = (double)m[k].max - (double)m[k].min;
      const double step = range > 0.0 ? range / (double)((1u << m[k].bits) - 1u) : 0.0;
      k_dequant<<<grid_n(n), 256, 0, c->st>>>(dcodes, nbytes, n, m[k].bits, m[k].min, step, dst[k]);
      c->launches++;
      DL_CUDA(cudaStreamSynchronize(c->st));
      cudaFree(dcodes);
    }
    refresh_shadows(c);
    c->have_grads = false;
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_get_params(dl_bn* c, float* e, float* u, float* w_rec, float* d) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_get_params: null ctx");
  return bn_guarded(c, [&] {
    download(c, e, c->e, c->V * c->P);
    download(c, u, c->u, c->P * c->H);
    download(c, w_rec, c->w_rec, c->H * c->H);
    download(c, d, c->d, c->H * c->P);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_set_opt(dl_bn* c, const float* m_e, const float* m_u, const float* m_rec,
                  const float* m_d, double rho, double eps) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_set_opt: null ctx");
  if (!(rho > 0.0 && rho < 1.0)) return bn_fail(c, DL_EINVAL, "opt state: rho must be in (0, 1)");
  if (!(eps > 0.0)) return bn_fail(c, DL_EINVAL, "opt state: eps must be > 0");
  return bn_guarded(c, [&] {
    c->rho = rho;
    c->eps = eps;
    if (m_e) upload(c, c->m_e, m_e, c->V);
    else DL_CUDA(cudaMemsetAsync(c->m_e, 0, c->V * 4, c->st));
    if (m_u) upload(c, c->m_u, m_u, c->P * c->H);
    else DL_CUDA(cudaMemsetAsync(c->m_u, 0, c->P * c->H * 4, c->st));
    if (m_rec) upload(c, c->m_rec, m_rec, c->H * c->H);
    else DL_CUDA(cudaMemsetAsync(c->m_rec, 0, c->H * c->H * 4, c->st));
    if (m_d) upload(c, c->m_d, m_d, c->H * c->P);
    else DL_CUDA(cudaMemsetAsync(c->m_d, 0, c->H * c->P * 4, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_get_opt(dl_bn* c, float* m_e, float* m_u, float* m_rec, float* m_d) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_get_opt: null ctx");
  return bn_guarded(c, [&] {
    download(c, m_e, c->m_e, c->V);
    download(c, m_u, c->m_u, c->P * c->H);
    download(c, m_rec, c->m_rec, c->H * c->H);
    download(c, m_d, c->m_d, c->H * c->P);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

}  // extern "C"

namespace {
// dl_bn_window / dl_bn_train_window: validate, copy the window in, run it
// (+ bottleneck_update when eta > 0) and read loss, positions, the update's
// verdict and h_final back with one synchronisation.
int bn_window_call(dl_bn* c, int64_t T, int64_t B, const uint32_t* inputs,
                   const uint32_t* targets, const uint8_t* weights, const float* h0,
                   float* h_final, double loss_scale, float clip, bool grads, double eta,
                   double* loss, uint64_t* positions, int* applied) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_window: null ctx");
  if (T < 1 || B < 1) return bn_fail(c, DL_EINVAL, "bptt: empty window");
  if (!inputs || !targets || !weights || !h0)
    return bn_fail(c, DL_EINVAL, "bptt: window size mismatch");
  return bn_guarded(c, [&] {
    const int64_t N = T * B;
    check_ids(c, inputs, N, "bptt");
    for (int64_t i = 0; i < N; ++i)
      if (weights[i]) DL_REQUIRE(targets[i] < (uint64_t)c->V, DL_EDATA, "bptt: id out of vocabulary range");
    ensure_window(c, T, N);
    cudaStream_t st = c->st;
    if (c->loss_mode == 0) nce_draws(c, weights, N);
    DL_CUDA(cudaMemcpyAsync(c->x, inputs, N * 4, cudaMemcpyHostToDevice, st));
    DL_CUDA(cudaMemcpyAsync(c->y, targets, N * 4, cudaMemcpyHostToDevice, st));
    DL_CUDA(cudaMemcpyAsync(c->w, weights, N, cudaMemcpyHostToDevice, st));
    DL_CUDA(cudaMemcpyAsync(c->htape, h0, B * c->H * 4, cudaMemcpyHostToDevice, st));
    auto body = [&] {
      run_window(c, T, B, loss_scale, clip, grads);
      if (grads && eta > 0.0) run_update(c, eta);
    };
    // softmax training windows: one graph per shape/hyper-parameters, after
    // an eager run has sized every buffer
    const auto key = std::make_tuple(T, B, loss_scale, clip, eta);
    const bool graphable = c->use_graphs && c->loss_mode == 1 && grads && eta > 0.0;
    auto it = graphable ? c->graphs.find(key) : c->graphs.end();
    if (it != c->graphs.end()) {
      DL_CUDA(cudaGraphLaunch(it->second, st));
      c->launches += c->graph_launches[key];
      c->e_sparse = false;
      c->have_grads = true;
    } else if (graphable && c->graphs.count(std::make_tuple(T, B, -1.0, 0.f, 0.0))) {
      cudaGraph_t gr = nullptr;
      const uint64_t l0 = c->launches;
      DL_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      body();
      DL_CUDA(cudaStreamEndCapture(st, &gr));
      c->graph_launches[key] = c->launches - l0;
      cudaGraphExec_t ex = nullptr;
      DL_CUDA(cudaGraphInstantiate(&ex, gr, 0));
      cudaGraphDestroy(gr);
      c->graphs[key] = ex;
      DL_CUDA(cudaGraphLaunch(ex, st));
    } else {
      body();
      // (a marker: this shape has run eagerly, so its buffers are sized)
      if (graphable) c->graphs[std::make_tuple(T, B, -1.0, 0.f, 0.0)] = nullptr;
    }
    struct { double l; unsigned long long p; int bad; } res{};
    DL_CUDA(cudaMemcpyAsync(&res.l, c->d_loss, sizeof res.l, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaMemcpyAsync(&res.p, c->d_pos, sizeof res.p, cudaMemcpyDeviceToHost, st));
    if (grads && eta > 0.0)
      DL_CUDA(cudaMemcpyAsync(&res.bad, c->nonfinite, sizeof res.bad, cudaMemcpyDeviceToHost, st));
    if (h_final)
      DL_CUDA(cudaMemcpyAsync(h_final, c->htape + T * B * c->H, B * c->H * 4,
                              cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    if (eta > 0.0) c->have_grads = false;
    if (loss) *loss = res.l;
    if (positions) *positions = res.p;
    if (applied) *applied = res.bad ? 0 : 1;
  });
}
}  // namespace

extern "C" {

int dl_bn_window(dl_bn* c, int64_t T, int64_t B, const uint32_t* inputs,
                 const uint32_t* targets, const uint8_t* weights, const float* h0,
                 float* h_final, double loss_scale, float clip, int compute_grads, double* loss,
                 uint64_t* positions) {
  return bn_window_call(c, T, B, inputs, targets, weights, h0, h_final, loss_scale, clip,
                        compute_grads != 0, 0.0, loss, positions, nullptr);
}

int dl_bn_get_grads(dl_bn* c, float* g_e, float* g_u, float* g_rec, float* g_d) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_get_grads: null ctx");
  if (!c->have_grads) return bn_fail(c, DL_EINVAL, "dl_bn_get_grads: no gradients (run a window)");
  return bn_guarded(c, [&] {
    download(c, g_e, c->g_e, c->V * c->P);
    download(c, g_u, c->g_u, c->P * c->H);
    download(c, g_rec, c->g_rec, c->H * c->H);
    download(c, g_d, c->g_d, c->H * c->P);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_rmsprop(dl_bn* c, double eta, int* applied) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_rmsprop: null ctx");
  if (!c->have_grads) return bn_fail(c, DL_EINVAL, "dl_bn_rmsprop: no gradients (run a window)");
  return bn_guarded(c, [&] {
    run_update(c, eta);
    int nf = 0;
    DL_CUDA(cudaMemcpyAsync(&nf, c->nonfinite, sizeof nf, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
    c->have_grads = false;
    if (applied) *applied = nf ? 0 : 1;
  });
}

int dl_bn_train_window(dl_bn* c, int64_t T, int64_t B, const uint32_t* inputs,
                       const uint32_t* targets, const uint8_t* weights, const float* h0,
                       float* h_final, double loss_scale, float clip, double eta, double* loss,
                       uint64_t* positions, int* applied) {
  if (!(eta > 0.0)) return bn_fail(c, DL_EINVAL, "config: eta must be > 0");
  return bn_window_call(c, T, B, inputs, targets, weights, h0, h_final, loss_scale, clip, true,
                        eta, loss, positions, applied);
}

// ------------------------------------------------------------- trainer
// Trainer<BottleneckTraits>::run_epoch on the device (trainer.hpp:350-410
// over compress.hpp:389-415): the stream, the offset-stream cursors
// floor(i*L/N), the hidden carry and the window counter live in HBM; each
// window is window_build -> bptt_run -> bottleneck_update -> window_finish,
// with the loss / skipped-update sums kept on the device.  Softmax windows
// replay one CUDA graph; NCE windows draw their noise on the host (the
// reference's generator order), which mirrors the schedule for the targets.
int dl_bn_trainer_init(dl_bn* c, const uint32_t* ids, int64_t L, int noffset, int minibatch,
                       int unroll, double clip, uint32_t bos) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_trainer_init: null ctx");
  if (noffset < 1 || minibatch < 1 || unroll < 1)
    return bn_fail(c, DL_EINVAL, "config: noffset, minibatch, unroll must be >= 1");
  if (!(clip > 0.0)) return bn_fail(c, DL_EINVAL, "config: clip must be > 0");
  const int64_t N = (int64_t)noffset * minibatch;
  if (!ids || L < N)
    return bn_fail(c, DL_EINVAL, "trainer: training stream shorter than the stream count");
  for (int64_t i = 0; i < L; ++i)
    if (ids[i] >= (uint64_t)c->V) return bn_fail(c, DL_EDATA, "trainer: id out of vocabulary range");
  return bn_guarded(c, [&] {
    DL_CUDA(cudaStreamSynchronize(c->st));
    drop_graphs(c);
    for (void** p : {(void**)&c->ids, (void**)&c->cursors, (void**)&c->hidden})
      if (*p) {
        cudaFree(*p);
        *p = nullptr;
      }
    c->L = L;
    c->noffset = noffset;
    c->minibatch = minibatch;
    c->unroll = unroll;
    c->clip = clip;
    c->bos = bos;
    c->ids = bn_alloc<uint32_t>(L);
    c->h_ids.assign(ids, ids + L);
    DL_CUDA(cudaMemcpyAsync(c->ids, c->h_ids.data(), L * 4, cudaMemcpyHostToDevice, c->st));
    c->cursors = bn_alloc<int64_t>(N);
    c->hidden = bn_alloc<float>(N * c->H);
    if (!c->win_counter) c->win_counter = bn_alloc<int64_t>(1);
    if (!c->t_loss) c->t_loss = bn_alloc<double>(1);
    if (!c->t_pos) c->t_pos = bn_alloc<unsigned long long>(1);
    if (!c->t_skipped) c->t_skipped = bn_alloc<unsigned long long>(1);
    std::vector<int64_t> cur(N);
    for (int64_t i = 0; i < N; ++i) cur[i] = i * L / N;  // trainer.hpp:194-195
    DL_CUDA(cudaMemcpyAsync(c->cursors, cur.data(), N * 8, cudaMemcpyHostToDevice, c->st));
    fill_f32(c->hidden, act0(c->act), N * c->H, c->st);
    c->launches++;
    ensure_window(c, unroll, (int64_t)unroll * minibatch);
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_trainer_get_state(dl_bn* c, int64_t* cursors, float* hidden) {
  if (!c || !c->cursors) return bn_fail(c, DL_EINVAL, "trainer not initialised");
  return bn_guarded(c, [&] {
    const int64_t N = (int64_t)c->noffset * c->minibatch;
    if (cursors) DL_CUDA(cudaMemcpyAsync(cursors, c->cursors, N * 8, cudaMemcpyDeviceToHost, c->st));
    if (hidden) DL_CUDA(cudaMemcpyAsync(hidden, c->hidden, N * c->H * 4, cudaMemcpyDeviceToHost, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

int dl_bn_trainer_set_state(dl_bn* c, const int64_t* cursors, const float* hidden) {
  if (!c || !c->cursors) return bn_fail(c, DL_EINVAL, "trainer not initialised");
  const int64_t N = (int64_t)c->noffset * c->minibatch;
  if (cursors)
    for (int64_t i = 0; i < N; ++i)
      if (cursors[i] < 0 || cursors[i] >= c->L)
        return bn_fail(c, DL_EDATA, "trainer checkpoint: cursor out of range");
  return bn_guarded(c, [&] {
    if (cursors) DL_CUDA(cudaMemcpyAsync(c->cursors, cursors, N * 8, cudaMemcpyHostToDevice, c->st));
    if (hidden) DL_CUDA(cudaMemcpyAsync(c->hidden, hidden, N * c->H * 4, cudaMemcpyHostToDevice, c->st));
    DL_CUDA(cudaStreamSynchronize(c->st));
  });
}

namespace {
void bn_trainer_window(dl_bn* c, double eta) {
  const int64_t B = c->minibatch, T = c->unroll, H = c->H;
  cudaStream_t st = c->st;
  window_build(c->ids, c->L, c->cursors, c->hidden, c->win_counter, c->noffset, B, T, H, c->bos,
               c->x, c->y, c->w, c->htape, st);
  c->launches++;
  run_window(c, T, B, 1.0 / (double)(B * T), (float)c->clip, true);
  run_update(c, eta);
  accum_loss(c->t_loss, c->d_loss, c->t_pos, c->d_pos, st);
  window_finish(c->cursors, c->hidden, c->htape + T * B * H, c->win_counter, c->noffset, B, T, H,
                c->L, act0(c->act), st, c->nonfinite, c->t_skipped);
  c->launches += 3;
}
}  // namespace

int dl_bn_trainer_run(dl_bn* c, int64_t first, int64_t count, double eta, double* loss_sum,
                      uint64_t* positions, uint64_t* skipped) {
  if (!c || !c->ids) return bn_fail(c, DL_EINVAL, "trainer not initialised");
  if (!(eta > 0.0)) return bn_fail(c, DL_EINVAL, "config: eta must be > 0");
  if (first < 0 || count < 0) return bn_fail(c, DL_EINVAL, "dl_bn_trainer_run: negative window");
  return bn_guarded(c, [&] {
    cudaStream_t st = c->st;
    const int64_t B = c->minibatch, T = c->unroll, N = (int64_t)c->noffset * B;
    DL_CUDA(cudaMemcpyAsync(c->win_counter, &first, 8, cudaMemcpyHostToDevice, st));
    DL_CUDA(cudaMemsetAsync(c->t_loss, 0, 8, st));
    DL_CUDA(cudaMemsetAsync(c->t_pos, 0, 8, st));
    DL_CUDA(cudaMemsetAsync(c->t_skipped, 0, 8, st));
    ensure_window(c, T, T * B);
    if (c->loss_mode == 0) {
      // the host mirrors the schedule (cursors; trainer.hpp:374-406) for the
      // window's targets / mask, then draws in the reference's order
      std::vector<int64_t> cur(N);
      DL_CUDA(cudaMemcpyAsync(cur.data(), c->cursors, N * 8, cudaMemcpyDeviceToHost, st));
      DL_CUDA(cudaStreamSynchronize(st));
      std::vector<uint8_t> w(T * B);
      const int64_t L = c->L;
      for (int64_t i = 0; i < count; ++i) {
        const int64_t s0 = ((first + i) % c->noffset) * B;
        for (int64_t t = 0; t < T; ++t)
          for (int64_t b = 0; b < B; ++b)
            w[t * B + b] = c->h_ids[(cur[s0 + b] + t + 1) % L] == c->bos ? 0 : 1;
        nce_draws(c, w.data(), T * B);
        bn_trainer_window(c, eta);
        for (int64_t b = 0; b < B; ++b) {
          int64_t v = cur[s0 + b] + T;
          cur[s0 + b] = v >= L ? v - L : v;
        }
      }
    } else if (c->use_graphs && count > 0) {
      // one eager window sizes every lazily grown buffer, then one graph
      // (build -> window -> update -> sums -> finish) replays the rest
      int64_t i = 0;
      if (!c->tgraph_sized) {
        bn_trainer_window(c, eta);
        c->tgraph_sized = true;
        ++i;
      }
      if (i < count && (!c->tgraph || c->tgraph_eta != eta)) {
        if (c->tgraph) cudaGraphExecDestroy(c->tgraph);
        c->tgraph = nullptr;
        cudaGraph_t gr = nullptr;
        const uint64_t l0 = c->launches;
        DL_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
          bn_trainer_window(c, eta);
        } catch (...) {
          cudaStreamEndCapture(st, &gr);
          if (gr) cudaGraphDestroy(gr);
          throw;
        }
        DL_CUDA(cudaStreamEndCapture(st, &gr));
        c->tgraph_launches = c->launches - l0;
        c->launches = l0;  // counted when replayed
        DL_CUDA(cudaGraphInstantiate(&c->tgraph, gr, 0));
        cudaGraphDestroy(gr);
        c->tgraph_eta = eta;
      }
      for (; i < count; ++i) {
        DL_CUDA(cudaGraphLaunch(c->tgraph, st));
        c->launches += c->tgraph_launches;
      }
    } else {
      for (int64_t i = 0; i < count; ++i) bn_trainer_window(c, eta);
    }
    c->have_grads = false;
    struct { double l; unsigned long long p, s; } res{};
    DL_CUDA(cudaMemcpyAsync(&res.l, c->t_loss, 8, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaMemcpyAsync(&res.p, c->t_pos, 8, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaMemcpyAsync(&res.s, c->t_skipped, 8, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    if (loss_sum) *loss_sum += res.l;
    if (positions) *positions += res.p;
    if (skipped) *skipped += res.s;
  });
}

// sharded_perplexity over the bottleneck adapter (eval.hpp:151-222): S
// slices walked cold in lockstep, banked so that each output GEMM scores
// several steps at once
// Lock-step forward scorer over S streams (the bottleneck adapter's
// softmax_scores_t + lse_column, eval.hpp:176-220 / :725-751): in[j*S+s]
// input ids, tgt[j*S+s] target or -1; h0 (S x H) may be NULL for act(0).
int dl_bn_score(dl_bn* c, int64_t S, int64_t steps, const uint32_t* in, const int64_t* tgt,
                const float* h0, float* h_final, double* logp, double* total_logprob,
                uint64_t* predicted) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_score: null ctx");
  if (S < 1 || steps < 0 || (steps > 0 && (!in || !tgt)))
    return bn_fail(c, DL_EINVAL, "dl_bn_score: bad shape");
  std::vector<uint32_t> yv(S * steps);
  std::vector<uint8_t> wv(S * steps);
  for (int64_t i = 0; i < S * steps; ++i) {
    if (in[i] >= (uint64_t)c->V || tgt[i] >= c->V)
      return bn_fail(c, DL_EDATA, "score: id out of vocabulary range");
    yv[i] = tgt[i] >= 0 ? (uint32_t)tgt[i] : 0u;
    wv[i] = tgt[i] >= 0 ? 1 : 0;
  }
  double tot = 0.0;
  uint64_t pred = 0;
  return bn_guarded(c, [&] {
    const int64_t H = c->H, SH = S * H;
    const int64_t bank = std::max<int64_t>(1, std::min<int64_t>(steps, 4096 / S));
    ensure_window(c, bank, bank * S);
    cudaStream_t st = c->st;
    if (h0) DL_CUDA(cudaMemcpyAsync(c->htape, h0, SH * 4, cudaMemcpyHostToDevice, st));
    else fill_f32(c->htape, act0(c->act), SH, st);
    std::vector<double> lp(bank * S);
    for (int64_t j0 = 0; j0 < steps; j0 += bank) {
      const int64_t nb = std::min(bank, steps - j0), N = nb * S;
      DL_CUDA(cudaMemcpyAsync(c->x, in + j0 * S, N * 4, cudaMemcpyHostToDevice, st));
      DL_CUDA(cudaMemcpyAsync(c->y, yv.data() + j0 * S, N * 4, cudaMemcpyHostToDevice, st));
      DL_CUDA(cudaMemcpyAsync(c->w, wv.data() + j0 * S, N, cudaMemcpyHostToDevice, st));
      input_side(c, N);
      recurrence_fwd(c, nb, S);
      output_side(c, N, c->htape + SH, tcm(c) ? c->htape_bf + SH : nullptr, 1.0, false);
      DL_CUDA(cudaMemcpyAsync(c->htape, c->htape + nb * SH, SH * 4, cudaMemcpyDeviceToDevice, st));
      DL_CUDA(cudaMemcpyAsync(lp.data(), c->logp_row, N * 8, cudaMemcpyDeviceToHost, st));
      DL_CUDA(cudaStreamSynchronize(st));
      for (int64_t i = 0; i < N; ++i) {
        const bool scored = wv[j0 * S + i] != 0;
        if (logp) logp[j0 * S + i] = scored ? lp[i] : NAN;
        if (scored) {
          tot += lp[i];
          ++pred;
        }
      }
    }
    if (h_final) DL_CUDA(cudaMemcpyAsync(h_final, c->htape, SH * 4, cudaMemcpyDeviceToHost, st));
    DL_CUDA(cudaStreamSynchronize(st));
    if (total_logprob) *total_logprob = tot;
    if (predicted) *predicted = pred;
  });
}

int dl_bn_sharded_perplexity(dl_bn* c, const uint32_t* ids, int64_t n, int shards, uint32_t bos,
                             double* total_logprob, uint64_t* predicted, double* perplexity) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_sharded_perplexity: null ctx");
  if (!ids || n < 2) return bn_fail(c, DL_EINVAL, "sharded perplexity: stream too short");
  if (shards < 1) return bn_fail(c, DL_EINVAL, "sharded perplexity: shards must be >= 1");
  const int64_t S = std::min<int64_t>(shards, n / 2);
  std::vector<int64_t> begin(S + 1);
  for (int64_t s = 0; s <= S; ++s) begin[s] = s * n / S;
  int64_t max_len = 0;
  for (int64_t s = 0; s < S; ++s) max_len = std::max(max_len, begin[s + 1] - begin[s]);
  const int64_t steps = std::max<int64_t>(0, max_len - 1);
  std::vector<uint32_t> in(S * steps);
  std::vector<int64_t> tg(S * steps);
  for (int64_t j = 0; j < steps; ++j)
    for (int64_t s = 0; s < S; ++s) {
      const int64_t len = begin[s + 1] - begin[s], i = j * S + s;
      in[i] = 0;
      tg[i] = -1;
      if (j + 1 < len) {
        const uint32_t x = ids[begin[s] + j], y = ids[begin[s] + j + 1];
        if (x >= (uint64_t)c->V || y >= (uint64_t)c->V)
          return bn_fail(c, DL_EDATA, "sharded perplexity: id out of vocabulary range");
        in[i] = x;
        if (y != bos) tg[i] = y;
      }
    }
  double tot = 0.0;
  uint64_t pred = 0;
  const int rc = dl_bn_score(c, S, steps, in.data(), tg.data(), nullptr, nullptr, nullptr, &tot,
                             &pred);
  if (rc != DL_OK) return rc;
  if (pred == 0) return bn_fail(c, DL_EINVAL, "sharded perplexity: no predicted tokens");
  if (total_logprob) *total_logprob = tot;
  if (predicted) *predicted = pred;
  if (perplexity) *perplexity = std::exp(-tot / (double)pred);
  return DL_OK;
}

int dl_bn_set_loss_mode(dl_bn* c, int mode) {
  if (!c) return bn_fail(c, DL_EINVAL, "dl_bn_set_loss_mode: null ctx");
  if (mode != 0 && mode != 1) return bn_fail(c, DL_EINVAL, "loss mode must be 0 (NCE) or 1 (softmax)");
  c->loss_mode = mode;
  return DL_OK;
}

namespace {
int bn_noise(dl_bn* c, const double* counts, int64_t V, int k, double floor, bool dist) {
  if (!c || !counts) return bn_fail(c, DL_EINVAL, "dl_bn_set_noise: null argument");
  if (V != c->V) return bn_fail(c, DL_EINVAL, "NoiseModel: vocabulary size mismatch");
  if (k < 1) return bn_fail(c, DL_EINVAL, "NoiseModel: k >= 1");
  if (!dist && !(floor > 0.0)) return bn_fail(c, DL_EINVAL, "NoiseModel: floor must be > 0");
  return bn_guarded(c, [&] {
    std::vector<double> lnkq, prob;
    std::vector<uint32_t> alias;
    if (dist) noise_tables_q(counts, V, k, lnkq, prob, alias);
    else noise_tables(counts, V, k, floor, lnkq, prob, alias);
    if (!c->ln_kq_d) c->ln_kq_d = bn_alloc<double>(V);
    if (!c->nz_prob_d) c->nz_prob_d = bn_alloc<double>(V);
    if (!c->nz_alias_d) c->nz_alias_d = bn_alloc<uint32_t>(V);
    if (!c->touched) c->touched = bn_alloc<uint8_t>(V);
    DL_CUDA(cudaMemcpy(c->ln_kq_d, lnkq.data(), V * 8, cudaMemcpyHostToDevice));
    DL_CUDA(cudaMemcpy(c->nz_prob_d, prob.data(), V * 8, cudaMemcpyHostToDevice));
    DL_CUDA(cudaMemcpy(c->nz_alias_d, alias.data(), V * 4, cudaMemcpyHostToDevice));
    c->nz_prob = std::move(prob);
    c->nce_k = k;
  });
}
}  // namespace

int dl_bn_set_noise(dl_bn* c, const double* counts, int64_t V, int k, double floor) {
  return bn_noise(c, counts, V, k, floor, false);
}

int dl_bn_set_noise_dist(dl_bn* c, const double* q, int64_t V, int k) {
  return bn_noise(c, q, V, k, 0.0, true);
}

int dl_bn_set_rng_state(dl_bn* c, const uint64_t state[313]) {
  if (!c || !state) return bn_fail(c, DL_EINVAL, "dl_bn_set_rng_state: null argument");
  std::stringstream ss;
  for (int i = 0; i < 313; ++i) ss << state[i] << ' ';
  ss >> c->rng;
  if (!ss) return bn_fail(c, DL_EINVAL, "dl_bn_set_rng_state: bad state");
  return DL_OK;
}

int dl_bn_get_rng_state(const dl_bn* c, uint64_t state[313]) {
  if (!c || !state) return bn_fail(nullptr, DL_EINVAL, "dl_bn_get_rng_state: null argument");
  std::stringstream ss;
  ss << c->rng;
  for (int i = 0; i < 313; ++i) ss >> state[i];
  return DL_OK;
}

uint64_t dl_bn_launch_count(const dl_bn* c) { return c ? c->launches : 0; }

void* dl_bn_cuda_stream(const dl_bn* c) { return c ? (void*)c->st : nullptr; }

}  // extern "C"
