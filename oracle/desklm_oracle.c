/*
 * oracle/desklm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference desklm algorithm for the RNNLM
 * training/scoring hot path.  It is the *checker* the parity tests compare
 * the CUDA path against (and the "port" CPU baseline); it is never linked
 * into, called by, or used as a fallback for the product library
 * (paper_1502_00512_b200/libdesklm_cuda.so).
 *
 * Pinning: every function here is checked bit-for-bit against the reference
 * itself, compiled from /root/reference/proj/include into oracle/_ref
 * (oracle/ref_shim.cpp) with the same flags (-O3 -ffp-contract=off), and
 * against the committed golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Reference anchors (all paths relative to /root/reference/proj/include/desklm):
 *   mt19937_64 / uniform01 / uniform / uniform_index   rng.hpp:37-50
 *   random_stream (test fixture)                       ../../tests/oracles/helpers.hpp:36-52
 *   RnnParams::init_uniform                            rnn.hpp:79-83
 *   activate / activate_deriv                          rnn.hpp:37-49
 *   dot_acc (8 fixed double lanes + tail)              mat.hpp:59-78
 *   matmul_nt / matmul_nn / matmul_tn_add              mat.hpp:116-184
 *   bptt_run, softmax branch                           backprop.hpp:76-222
 *   bptt_run, NCE branch; NoiseModel; AliasSampler    backprop.hpp:126-156, 193-203;
 *                                                      nce.hpp:31-93; rng.hpp:54-101
 *   StandardGrads::clip / SparseRowGrads               rnn.hpp:89-162
 *   rmsprop_update (+ sparse / dense row updates)      rmsprop.hpp:77-133
 *   sharded_perplexity / lse_column                    eval.hpp:48-57, 151-222
 *   rnn_perplexity                                     eval.hpp:84-145
 *   Trainer ctor / train / run_epoch / validate        trainer.hpp:178-270, 350-410
 *
 * Status codes: 0 ok, 1 invalid argument, 2 data error.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 (fully specified by the C++ standard). */
typedef struct {
  uint64_t x[312];
  int p;
} orc_mt64;

void orc_mt_seed(orc_mt64* m, uint64_t seed) {
  m->x[0] = seed;
  for (int i = 1; i < 312; ++i)
    m->x[i] = 6364136223846793005ULL * (m->x[i - 1] ^ (m->x[i - 1] >> 62)) +
              (uint64_t)i;
  m->p = 312;
}

static void mt_twist(orc_mt64* m) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  const uint64_t MAT = 0xB5026F5AA96619E9ULL;
  for (int i = 0; i < 312; ++i) {
    const uint64_t y = (m->x[i] & UM) | (m->x[(i + 1) % 312] & LM);
    m->x[i] = m->x[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? MAT : 0ULL);
  }
  m->p = 0;
}

uint64_t orc_mt_next(orc_mt64* m) {
  if (m->p >= 312) mt_twist(m);
  uint64_t z = m->x[m->p++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

/* rng.hpp:37-50 */
static double uniform01(orc_mt64* m) {
  return (double)(orc_mt_next(m) >> 11) * 0x1.0p-53;
}
static double uniform(orc_mt64* m, double lo, double hi) {
  return lo + (hi - lo) * uniform01(m);
}
static uint64_t uniform_index(orc_mt64* m, uint64_t n) {
  return (uint64_t)(uniform01(m) * (double)n);
}

/* rnn.hpp:79-83: one generator, w_in then w_rec then w_out, row-major. */
int orc_init_uniform(int64_t V, int64_t H, uint64_t seed, double range,
                     float* w_in, float* w_rec, float* w_out) {
  if (V < 1 || H < 1) return 1;
  orc_mt64 m;
  orc_mt_seed(&m, seed);
  for (int64_t i = 0; i < V * H; ++i) w_in[i] = (float)uniform(&m, -range, range);
  for (int64_t i = 0; i < H * H; ++i) w_rec[i] = (float)uniform(&m, -range, range);
  for (int64_t i = 0; i < V * H; ++i) w_out[i] = (float)uniform(&m, -range, range);
  return 0;
}

/* helpers.hpp:36-52 on an existing generator.  Returns the length; writes at
 * most cap ids. */
static int64_t random_stream_rng(orc_mt64* m, uint64_t v, uint64_t min_tokens,
                                 uint64_t max_len, uint32_t* out, uint64_t cap) {
  const uint64_t body = v - 3;
  uint64_t n = 0;
#define PUSH(val)                     \
  do {                                \
    if (n < cap) out[n] = (val);      \
    ++n;                              \
  } while (0)
  while (n < min_tokens) {
    PUSH(1u);
    const uint64_t len = 1 + uniform_index(m, max_len);
    for (uint64_t i = 0; i < len; ++i) {
      const uint32_t r1 = (uint32_t)uniform_index(m, body);
      const uint32_t r2 = (uint32_t)uniform_index(m, body);
      PUSH(3u + (r1 < r2 ? r1 : r2));
    }
    PUSH(2u);
  }
#undef PUSH
  return (int64_t)n;
}

int64_t orc_random_stream(uint64_t seed, uint64_t v, uint64_t min_tokens,
                          uint64_t max_len, uint32_t* out, uint64_t cap) {
  orc_mt64 m;
  orc_mt_seed(&m, seed);
  return random_stream_rng(&m, v, min_tokens, max_len, out, cap);
}

int orc_random_stream_pair(uint64_t seed, uint64_t v, uint64_t min_a,
                           uint64_t min_b, uint32_t* out_a, uint64_t cap_a,
                           int64_t* len_a, uint32_t* out_b, uint64_t cap_b,
                           int64_t* len_b) {
  orc_mt64 m;
  orc_mt_seed(&m, seed);
  *len_a = random_stream_rng(&m, v, min_a, 12, out_a, cap_a);
  *len_b = random_stream_rng(&m, v, min_b, 12, out_b, cap_b);
  return 0;
}

/* ----------------------------------------------------------- dense math */
/* mat.hpp:59-78 */
static double dot_acc(const float* x, const float* y, int64_t n) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    s0 += (double)x[i + 0] * (double)y[i + 0];
    s1 += (double)x[i + 1] * (double)y[i + 1];
    s2 += (double)x[i + 2] * (double)y[i + 2];
    s3 += (double)x[i + 3] * (double)y[i + 3];
    s4 += (double)x[i + 4] * (double)y[i + 4];
    s5 += (double)x[i + 5] * (double)y[i + 5];
    s6 += (double)x[i + 6] * (double)y[i + 6];
    s7 += (double)x[i + 7] * (double)y[i + 7];
  }
  double tail = 0;
  for (; i < n; ++i) tail += (double)x[i] * (double)y[i];
  return ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)) + tail;
}

/* The three GEMMs split their work over OpenMP threads by output element
 * (matmul_nt), output column block (matmul_nn) or output row
 * (matmul_tn_add): every output element still sees exactly the reference's
 * sequence of operations, so the results do not depend on the thread count
 * (as parallel_rows, mat.hpp:95-114).  Small products stay serial. */
#define ORC_PAR_MIN 262144

/* C[MxN] = A[MxK] . B[NxK]^T, rounded to float (mat.hpp:116-134). */
static void matmul_nt(const float* A, const float* B, float* C, int64_t M,
                      int64_t N, int64_t K) {
#pragma omp parallel for collapse(2) schedule(static) if (M * N * K >= ORC_PAR_MIN)
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) C[i * N + j] = (float)dot_acc(A + i * K, B + j * K, K);
}

/* C[MxN] (=|+=) A[MxK] . B[KxN] with a double row accumulator; zero A
 * entries are skipped (mat.hpp:136-166). */
static void matmul_nn(const float* A, const float* B, float* C, int64_t M,
                      int64_t N, int64_t K, int accumulate, double* acc) {
  const int64_t JB = 256;
  for (int64_t i = 0; i < M; ++i) {
#pragma omp parallel for schedule(static) if (N * K >= ORC_PAR_MIN)
    for (int64_t j0 = 0; j0 < N; j0 += JB) {
      const int64_t j1 = j0 + JB < N ? j0 + JB : N;
      for (int64_t j = j0; j < j1; ++j) acc[j] = accumulate ? (double)C[i * N + j] : 0.0;
      for (int64_t k = 0; k < K; ++k) {
        const double a = (double)A[i * K + k];
        if (a == 0.0) continue;
        const float* bk = B + k * N;
        for (int64_t j = j0; j < j1; ++j) acc[j] += a * (double)bk[j];
      }
      for (int64_t j = j0; j < j1; ++j) C[i * N + j] = (float)acc[j];
    }
  }
}

/* C[MxN] += A[KxM]^T . B[KxN], float accumulate, k outer (mat.hpp:168-184);
 * each row of C accumulates its k terms in the same ascending order. */
static void matmul_tn_add(const float* A, const float* B, float* C, int64_t K,
                          int64_t M, int64_t N) {
#pragma omp parallel for schedule(static) if (M * N * K >= ORC_PAR_MIN)
  for (int64_t i = 0; i < M; ++i) {
    float* ci = C + i * N;
    for (int64_t k = 0; k < K; ++k) {
      const float a = A[k * M + i];
      if (a == 0.0f) continue;
      const float* bk = B + k * N;
      for (int64_t j = 0; j < N; ++j) ci[j] += a * bk[j];
    }
  }
}

/* rnn.hpp:37-49 (float instantiation) */
static float act_f(int act, float x) {
  if (act == 0) return 1.0f / (1.0f + expf(-x));
  return tanhf(x);
}
static float act_deriv_f(int act, float y) {
  if (act == 0) return y * (1.0f - y);
  return 1.0f - y * y;
}

/* std::min(c, std::max(-c, x)) -- note a NaN becomes -c (rnn.hpp:131-134). */
static float clip1(float x, float c) {
  const float t = (-c < x) ? x : -c;
  return (t < c) ? t : c;
}

/* ------------------------------------------------------------- bptt_run */
/* Softmax-mode window (backprop.hpp:76-222).  Sparse W_in gradient is
 * reported in slot (first-touch) order like SparseRowGrads; g_in_words and
 * g_in_data must hold T*B rows. */
int orc_bptt(int64_t V, int64_t H, int act, const float* w_in,
             const float* w_rec, const float* w_out, int64_t T, int64_t B,
             const uint32_t* inputs, const uint32_t* targets,
             const uint8_t* weights, const float* h0, double loss_scale,
             float clip, int compute_grads, int threads, float* h_final,
             int64_t* g_in_rows, uint32_t* g_in_words, float* g_in_data,
             float* g_rec, float* g_out, double* loss, uint64_t* positions) {
  (void)threads;
  if (T < 1 || B < 1) return 1;
  const int64_t BH = B * H;
  float* h = (float*)malloc(sizeof(float) * (T + 1) * BH);
  float* pre = (float*)malloc(sizeof(float) * BH);
  float* scores = (float*)malloc(sizeof(float) * B * V);
  float* dsc = compute_grads ? (float*)calloc((size_t)(T * B * V), sizeof(float)) : NULL;
  memcpy(h, h0, sizeof(float) * BH);
  /* forward (backprop.hpp:97-115) */
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(h + t * BH, w_rec, pre, B, H, H);
    for (int64_t b = 0; b < B; ++b) {
      const float* e = w_in + (int64_t)inputs[t * B + b] * H;
      for (int64_t i = 0; i < H; ++i) pre[b * H + i] += e[i];
    }
    for (int64_t i = 0; i < BH; ++i) h[(t + 1) * BH + i] = act_f(act, pre[i]);
  }
  if (h_final) memcpy(h_final, h + T * BH, sizeof(float) * BH);
  /* softmax loss (backprop.hpp:157-189) */
  double L = 0.0;
  uint64_t pos = 0;
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(h + (t + 1) * BH, w_out, scores, B, V, H);
    for (int64_t b = 0; b < B; ++b) {
      const int64_t idx = t * B + b;
      if (!weights[idx]) continue;
      ++pos;
      const float* s = scores + b * V;
      double mx = (double)s[0];
      for (int64_t w = 1; w < V; ++w) mx = (mx < (double)s[w]) ? (double)s[w] : mx;
      double z = 0.0;
      for (int64_t w = 0; w < V; ++w) z += exp((double)s[w] - mx);
      const double lse = mx + log(z);
      const uint32_t y = targets[idx];
      L += loss_scale * (lse - (double)s[y]);
      if (compute_grads) {
        float* d = dsc + idx * V;
        for (int64_t w = 0; w < V; ++w)
          d[w] = (float)(loss_scale * exp((double)s[w] - lse));
        d[y] -= (float)loss_scale;
      }
    }
  }
  *loss = L;
  *positions = pos;
  if (compute_grads) {
    /* backward (backprop.hpp:193-220) */
    float* dh = (float*)calloc((size_t)BH, sizeof(float));
    float* dpre = (float*)malloc(sizeof(float) * BH);
    double* acc = (double*)malloc(sizeof(double) * (V > H ? V : H));
    int32_t* slot_of = (int32_t*)malloc(sizeof(int32_t) * V);
    for (int64_t w = 0; w < V; ++w) slot_of[w] = -1;
    int64_t nrows = 0;
    memset(g_rec, 0, sizeof(float) * H * H);
    memset(g_out, 0, sizeof(float) * V * H);
    for (int64_t t = T - 1; t >= 0; --t) {
      const float* dst = dsc + t * B * V;
      const float* ht1 = h + (t + 1) * BH;
      /* softmax_backward (rnn.hpp:253-258) */
      matmul_tn_add(dst, ht1, g_out, B, V, H);
      matmul_nn(dst, w_out, dh, B, H, V, 1, acc);
      for (int64_t i = 0; i < BH; ++i) dpre[i] = dh[i] * act_deriv_f(act, ht1[i]);
      matmul_tn_add(dpre, h + t * BH, g_rec, B, H, H);
      /* input_backward -> SparseRowGrads::axpy_row (rnn.hpp:106-110, 218-222) */
      for (int64_t b = 0; b < B; ++b) {
        const uint32_t w = inputs[t * B + b];
        if (slot_of[w] < 0) {
          slot_of[w] = (int32_t)nrows;
          g_in_words[nrows] = w;
          memset(g_in_data + nrows * H, 0, sizeof(float) * H);
          ++nrows;
        }
        float* r = g_in_data + (int64_t)slot_of[w] * H;
        for (int64_t i = 0; i < H; ++i) r[i] += 1.0f * dpre[b * H + i];
      }
      if (t > 0) matmul_nn(dpre, w_rec, dh, B, H, H, 0, acc);
    }
    *g_in_rows = nrows;
    /* StandardGrads::clip (rnn.hpp:155-162) */
    for (int64_t i = 0; i < nrows * H; ++i) g_in_data[i] = clip1(g_in_data[i], clip);
    for (int64_t i = 0; i < H * H; ++i) g_rec[i] = clip1(g_rec[i], clip);
    for (int64_t i = 0; i < V * H; ++i) g_out[i] = clip1(g_out[i], clip);
    free(dh);
    free(dpre);
    free(acc);
    free(slot_of);
  }
  free(h);
  free(pre);
  free(scores);
  free(dsc);
  return 0;
}

/* ------------------------------------------------------------------ NCE */
/* NoiseModel (nce.hpp:41-66): q = max(count/total, floor) renormalised,
 * ln_kq = log(k q); AliasSampler (rng.hpp:54-89) built from q with the same
 * small/large stack discipline, so sampling is bit-identical. */
int orc_noise_build(int64_t V, const double* counts, int k, double floor, double* q,
                    double* ln_kq, double* prob, uint32_t* alias) {
  if (k < 1 || V < 1) return 1;
  double total = 0.0;
  for (int64_t w = 0; w < V; ++w) {
    if (counts[w] < 0.0) return 1;
    total += counts[w];
  }
  if (total <= 0.0) return 1;
  double qsum = 0.0;
  for (int64_t w = 0; w < V; ++w) {
    const double v = counts[w] / total;
    q[w] = v > floor ? v : floor;  /* std::max(count/total, floor) */
    qsum += q[w];
  }
  for (int64_t w = 0; w < V; ++w) {
    q[w] /= qsum;
    ln_kq[w] = log((double)k * q[w]);
  }
  /* AliasSampler(q) */
  double tw = 0.0;
  for (int64_t w = 0; w < V; ++w) tw += q[w];
  double* scaled = (double*)malloc(sizeof(double) * V);
  uint32_t* small = (uint32_t*)malloc(sizeof(uint32_t) * V);
  uint32_t* large = (uint32_t*)malloc(sizeof(uint32_t) * V);
  int64_t ns = 0, nl = 0;
  for (int64_t i = 0; i < V; ++i) {
    prob[i] = 0.0;
    alias[i] = 0;
    scaled[i] = q[i] * (double)V / tw;
    if (scaled[i] < 1.0) small[ns++] = (uint32_t)i;
    else large[nl++] = (uint32_t)i;
  }
  while (ns > 0 && nl > 0) {
    const uint32_t sm = small[--ns];
    const uint32_t lg = large[--nl];
    prob[sm] = scaled[sm];
    alias[sm] = lg;
    scaled[lg] = (scaled[lg] + scaled[sm]) - 1.0;
    if (scaled[lg] < 1.0) small[ns++] = lg;
    else large[nl++] = lg;
  }
  for (int64_t i = 0; i < nl; ++i) prob[large[i]] = 1.0;
  for (int64_t i = 0; i < ns; ++i) prob[small[i]] = 1.0;
  free(scaled);
  free(small);
  free(large);
  return 0;
}

/* AliasSampler::sample (rng.hpp:91-94) */
static uint32_t alias_sample(orc_mt64* m, int64_t V, const double* prob, const uint32_t* alias) {
  const uint64_t i = uniform_index(m, (uint64_t)V);
  return uniform01(m) < prob[i] ? (uint32_t)i : alias[i];
}

/* the mt19937_64 state crosses the C boundary as 312 words + position */
static void mt_load(orc_mt64* m, const uint64_t* st) {
  memcpy(m->x, st, sizeof(uint64_t) * 312);
  m->p = (int)st[312];
}
static void mt_store(const orc_mt64* m, uint64_t* st) {
  memcpy(st, m->x, sizeof(uint64_t) * 312);
  st[312] = (uint64_t)m->p;
}
void orc_mt_state(uint64_t seed, uint64_t* st) {
  orc_mt64 m;
  orc_mt_seed(&m, seed);
  mt_store(&m, st);
}
int orc_noise_sample(int64_t V, const double* prob, const uint32_t* alias, uint64_t* rng,
                     int64_t n, uint32_t* out) {
  orc_mt64 m;
  mt_load(&m, rng);
  for (int64_t i = 0; i < n; ++i) out[i] = alias_sample(&m, V, prob, alias);
  mt_store(&m, rng);
  return 0;
}

/* nce.hpp:31-36 */
static double softplus(double x) {
  if (x > 0) return x + log1p(exp(-x));
  return log1p(exp(x));
}
static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* NCE-mode window (backprop.hpp:76-156, 193-222).  rng: 313-word state, in
 * and out (draws: t, then b, then sample; masked positions draw nothing).
 * The sparse W_out gradient comes back in slot (first-touch) order like the
 * W_in rows: g_out_words / g_out_data must hold T*B*(k+1) rows; noise_out
 * (optional) receives the k draws of every unmasked position in order. */
int orc_bptt_nce(int64_t V, int64_t H, int act, const float* w_in, const float* w_rec,
                 const float* w_out, int64_t T, int64_t B, const uint32_t* inputs,
                 const uint32_t* targets, const uint8_t* weights, const float* h0,
                 double loss_scale, float clip, int compute_grads, int k, const double* ln_kq,
                 const double* prob, const uint32_t* alias, uint64_t* rng, float* h_final,
                 int64_t* g_in_rows, uint32_t* g_in_words, float* g_in_data, float* g_rec,
                 int64_t* g_out_rows, uint32_t* g_out_words, float* g_out_data,
                 uint32_t* noise_out, double* loss, uint64_t* positions) {
  if (T < 1 || B < 1 || k < 1) return 1;
  const int64_t BH = B * H, K1 = k + 1;
  orc_mt64 m;
  mt_load(&m, rng);
  float* h = (float*)malloc(sizeof(float) * (T + 1) * BH);
  float* pre = (float*)malloc(sizeof(float) * BH);
  /* per (t, b): k+1 records (word, ds); n_rec[t*B+b] = 0 when masked */
  uint32_t* rw = (uint32_t*)malloc(sizeof(uint32_t) * T * B * K1);
  float* rds = (float*)malloc(sizeof(float) * T * B * K1);
  int* has = (int*)calloc((size_t)(T * B), sizeof(int));
  memcpy(h, h0, sizeof(float) * BH);
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(h + t * BH, w_rec, pre, B, H, H);
    for (int64_t b = 0; b < B; ++b) {
      const float* e = w_in + (int64_t)inputs[t * B + b] * H;
      for (int64_t i = 0; i < H; ++i) pre[b * H + i] += e[i];
    }
    for (int64_t i = 0; i < BH; ++i) h[(t + 1) * BH + i] = act_f(act, pre[i]);
  }
  if (h_final) memcpy(h_final, h + T * BH, sizeof(float) * BH);
  double L = 0.0;
  uint64_t pos = 0, nd = 0;
  for (int64_t t = 0; t < T; ++t) {
    const float* ht = h + (t + 1) * BH;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t idx = t * B + b;
      if (!weights[idx]) continue;
      ++pos;
      has[idx] = 1;
      const uint32_t y = targets[idx];
      /* StandardAdapter::score: float(dot_acc<double>) (rnn.hpp:246-249) */
      const double st = (double)(float)dot_acc(ht + b * H, w_out + (int64_t)y * H, H);
      const double at = st - ln_kq[y];
      L += loss_scale * softplus(-at);
      rw[idx * K1] = y;
      rds[idx * K1] = (float)(-loss_scale * sigmoid(-at));
      for (int j = 0; j < k; ++j) {
        const uint32_t w = alias_sample(&m, V, prob, alias);
        if (noise_out) noise_out[nd++] = w;
        const double s = (double)(float)dot_acc(ht + b * H, w_out + (int64_t)w * H, H);
        const double a = s - ln_kq[w];
        L += loss_scale * softplus(a);
        rw[idx * K1 + 1 + j] = w;
        rds[idx * K1 + 1 + j] = (float)(loss_scale * sigmoid(a));
      }
    }
  }
  mt_store(&m, rng);
  *loss = L;
  *positions = pos;
  if (compute_grads) {
    float* dh = (float*)calloc((size_t)BH, sizeof(float));
    float* dpre = (float*)malloc(sizeof(float) * BH);
    double* acc = (double*)malloc(sizeof(double) * H);
    int32_t* slot_in = (int32_t*)malloc(sizeof(int32_t) * V);
    int32_t* slot_out = (int32_t*)malloc(sizeof(int32_t) * V);
    for (int64_t w = 0; w < V; ++w) slot_in[w] = slot_out[w] = -1;
    int64_t nin = 0, nout = 0;
    memset(g_rec, 0, sizeof(float) * H * H);
    for (int64_t t = T - 1; t >= 0; --t) {
      const float* ht1 = h + (t + 1) * BH;
      /* score_backward per record (rnn.hpp:251-255): sparse row axpy, then
       * dh[b] += ds * W_out[w] (float axpy) */
      for (int64_t b = 0; b < B; ++b) {
        const int64_t idx = t * B + b;
        if (!has[idx]) continue;
        for (int64_t r = 0; r < K1; ++r) {
          const uint32_t w = rw[idx * K1 + r];
          const float ds = rds[idx * K1 + r];
          if (slot_out[w] < 0) {
            slot_out[w] = (int32_t)nout;
            g_out_words[nout] = w;
            memset(g_out_data + nout * H, 0, sizeof(float) * H);
            ++nout;
          }
          float* gr = g_out_data + (int64_t)slot_out[w] * H;
          const float* hb = ht1 + b * H;
          const float* wr = w_out + (int64_t)w * H;
          float* db = dh + b * H;
          for (int64_t i = 0; i < H; ++i) gr[i] += ds * hb[i];
          for (int64_t i = 0; i < H; ++i) db[i] += ds * wr[i];
        }
      }
      for (int64_t i = 0; i < BH; ++i) dpre[i] = dh[i] * act_deriv_f(act, ht1[i]);
      matmul_tn_add(dpre, h + t * BH, g_rec, B, H, H);
      for (int64_t b = 0; b < B; ++b) {
        const uint32_t w = inputs[t * B + b];
        if (slot_in[w] < 0) {
          slot_in[w] = (int32_t)nin;
          g_in_words[nin] = w;
          memset(g_in_data + nin * H, 0, sizeof(float) * H);
          ++nin;
        }
        float* r = g_in_data + (int64_t)slot_in[w] * H;
        for (int64_t i = 0; i < H; ++i) r[i] += 1.0f * dpre[b * H + i];
      }
      if (t > 0) matmul_nn(dpre, w_rec, dh, B, H, H, 0, acc);
    }
    *g_in_rows = nin;
    *g_out_rows = nout;
    for (int64_t i = 0; i < nin * H; ++i) g_in_data[i] = clip1(g_in_data[i], clip);
    for (int64_t i = 0; i < H * H; ++i) g_rec[i] = clip1(g_rec[i], clip);
    for (int64_t i = 0; i < nout * H; ++i) g_out_data[i] = clip1(g_out_data[i], clip);
    free(dh);
    free(dpre);
    free(acc);
    free(slot_in);
    free(slot_out);
  }
  free(h);
  free(pre);
  free(rw);
  free(rds);
  free(has);
  return 0;
}

/* -------------------------------------------------------------- rmsprop */
static double mean_sq(const float* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += (double)x[i] * (double)x[i];
  return s / (double)n;
}

static int all_finite(const float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite((double)x[i])) return 0;
  return 1;
}

/* rmsprop.hpp:77-92 */
static void update_rows_sparse(float* w, int64_t H, int64_t nrows,
                               const uint32_t* words, const float* data,
                               float* m, int64_t V, double rho, double eps,
                               double eta) {
  for (int64_t i = 0; i < V; ++i) m[i] = (float)(rho * m[i]);
  for (int64_t s = 0; s < nrows; ++s) {
    const uint32_t word = words[s];
    const float* row = data + s * H;
    m[word] += (float)((1.0 - rho) * mean_sq(row, H));
    const double denom = sqrt((double)m[word] + eps);
    float* wr = w + (int64_t)word * H;
    for (int64_t i = 0; i < H; ++i) wr[i] -= (float)(eta * (double)row[i] / denom);
  }
}

/* rmsprop.hpp:94-107 */
static void update_rows_dense(float* w, int64_t V, int64_t H, const float* g,
                              float* m, double rho, double eps, double eta) {
  for (int64_t word = 0; word < V; ++word) {
    const float* row = g + word * H;
    m[word] = (float)(rho * (double)m[word] + (1.0 - rho) * mean_sq(row, H));
    const double denom = sqrt((double)m[word] + eps);
    float* wr = w + word * H;
    for (int64_t i = 0; i < H; ++i) wr[i] -= (float)(eta * (double)row[i] / denom);
  }
}

/* rmsprop.hpp:113-133.  out_dense selects the dense W_out gradient (softmax
 * mode) or sparse rows (NCE mode). */
int orc_rmsprop(int64_t V, int64_t H, float* w_in, float* w_rec, float* w_out,
                float* m_rec, float* m_in, float* m_out, double rho, double eps,
                double eta, int64_t n_in_rows, const uint32_t* in_words,
                const float* in_data, const float* g_rec, int out_dense,
                int64_t n_out_rows, const uint32_t* out_words,
                const float* out_data, int* applied) {
  const int fin = all_finite(in_data, n_in_rows * H) && all_finite(g_rec, H * H) &&
                  (out_dense ? all_finite(out_data, V * H)
                             : all_finite(out_data, n_out_rows * H));
  if (!fin) {
    *applied = 0;
    return 0;
  }
  for (int64_t i = 0; i < H * H; ++i) {
    const double gi = (double)g_rec[i];
    m_rec[i] = (float)(rho * (double)m_rec[i] + (1.0 - rho) * gi * gi);
    w_rec[i] -= (float)(eta * gi / sqrt((double)m_rec[i] + eps));
  }
  update_rows_sparse(w_in, H, n_in_rows, in_words, in_data, m_in, V, rho, eps, eta);
  if (out_dense)
    update_rows_dense(w_out, V, H, out_data, m_out, rho, eps, eta);
  else
    update_rows_sparse(w_out, H, n_out_rows, out_words, out_data, m_out, V, rho,
                       eps, eta);
  *applied = 1;
  return 0;
}

/* --------------------------------------------------------------- scoring */
/* eval.hpp:48-57 over a contiguous score vector. */
static double lse_vec(const float* s, int64_t n) {
  double mx = -INFINITY;
  for (int64_t w = 0; w < n; ++w) mx = (mx < (double)s[w]) ? (double)s[w] : mx;
  double z = 0.0;
  for (int64_t w = 0; w < n; ++w) z += exp((double)s[w] - mx);
  return mx + log(z);
}

/* Per-token log-probs of the sharded walk (eval.hpp:151-222).  out[j*S+s]
 * is ln p or NaN for skipped targets; totals mirror PerplexityResult. */
int orc_sharded_logprobs(int64_t V, int64_t H, int act, const float* w_in,
                         const float* w_rec, const float* w_out,
                         const uint32_t* ids, int64_t n, int shards,
                         uint32_t bos, double* out, int64_t cap, int64_t* S_out,
                         int64_t* steps_out, double* total_logprob,
                         uint64_t* predicted) {
  if (n < 2 || shards < 1) return 1;
  const int64_t S = shards < n / 2 ? shards : n / 2;
  int64_t* begin = (int64_t*)malloc(sizeof(int64_t) * (S + 1));
  for (int64_t s = 0; s <= S; ++s) begin[s] = s * n / S;
  int64_t max_len = 0;
  for (int64_t s = 0; s < S; ++s)
    if (begin[s + 1] - begin[s] > max_len) max_len = begin[s + 1] - begin[s];
  *S_out = S;
  *steps_out = max_len - 1;
  if (out && (max_len - 1) * S > cap) {
    free(begin);
    return 1;
  }
  const float a0 = act_f(act, 0.0f);
  float* h = (float*)malloc(sizeof(float) * S * H);
  float* pre = (float*)malloc(sizeof(float) * S * H);
  float* sc = (float*)malloc(sizeof(float) * V);
  uint32_t* in = (uint32_t*)malloc(sizeof(uint32_t) * S);
  int64_t* tgt = (int64_t*)malloc(sizeof(int64_t) * S);
  for (int64_t i = 0; i < S * H; ++i) h[i] = a0;
  double total = 0.0;
  uint64_t pred = 0;
  int rc = 0;
  for (int64_t j = 0; j + 1 < max_len; ++j) {
    int any = 0;
    for (int64_t s = 0; s < S; ++s) {
      const int64_t len = begin[s + 1] - begin[s];
      if (j + 1 < len) {
        const uint32_t x = ids[begin[s] + j], y = ids[begin[s] + j + 1];
        if (x >= (uint64_t)V || y >= (uint64_t)V) {
          rc = 2;
          goto done;
        }
        in[s] = x;
        tgt[s] = (y == bos) ? -1 : (int64_t)y;
      } else {
        in[s] = 0;
        tgt[s] = -1;
      }
      any = any || tgt[s] >= 0;
    }
    matmul_nt(h, w_rec, pre, S, H, H);
    for (int64_t s = 0; s < S; ++s)
      for (int64_t i = 0; i < H; ++i) {
        const float p = pre[s * H + i] + w_in[(int64_t)in[s] * H + i];
        h[s * H + i] = act_f(act, p);
      }
    for (int64_t s = 0; s < S; ++s) {
      double v = NAN;
      if (any && tgt[s] >= 0) {
        /* scores_t column s: W_out . h_s (eval.hpp:207, rnn.hpp:248-251) */
#pragma omp parallel for schedule(static) if (V * H >= ORC_PAR_MIN)
        for (int64_t w = 0; w < V; ++w) sc[w] = (float)dot_acc(w_out + w * H, h + s * H, H);
        v = (double)sc[tgt[s]] - lse_vec(sc, V);
        total += v;
        ++pred;
      }
      if (out) out[j * S + s] = v;
    }
  }
  *total_logprob = total;
  *predicted = pred;
  if (pred == 0) rc = 1;
done:
  free(begin);
  free(h);
  free(pre);
  free(sc);
  free(in);
  free(tgt);
  return rc;
}

int orc_sharded_ppl(int64_t V, int64_t H, int act, const float* w_in,
                    const float* w_rec, const float* w_out, const uint32_t* ids,
                    int64_t n, int shards, uint32_t bos, int threads,
                    double* total_logprob, uint64_t* predicted, double* ppl) {
  (void)threads;
  int64_t S, steps;
  const int rc = orc_sharded_logprobs(V, H, act, w_in, w_rec, w_out, ids, n,
                                      shards, bos, NULL, 0, &S, &steps,
                                      total_logprob, predicted);
  if (rc) return rc;
  *ppl = exp(-*total_logprob / (double)*predicted);
  return 0;
}

/* eval.hpp:84-145: single stream, state never reset after the start; every
 * non-bos target scored (banking does not change the numbers). */
int orc_rnn_ppl(int64_t V, int64_t H, int act, const float* w_in,
                const float* w_rec, const float* w_out, const uint32_t* ids,
                int64_t n, uint32_t bos, int threads, double* total_logprob,
                uint64_t* predicted, double* ppl) {
  (void)threads;
  if (n < 2) return 1;
  float* h = (float*)malloc(sizeof(float) * H);
  float* pre = (float*)malloc(sizeof(float) * H);
  float* sc = (float*)malloc(sizeof(float) * V);
  const float a0 = act_f(act, 0.0f);
  for (int64_t i = 0; i < H; ++i) h[i] = a0;
  double total = 0.0;
  uint64_t pred = 0;
  int rc = 0;
  for (int64_t i = 0; i + 1 < n; ++i) {
    if (ids[i] >= (uint64_t)V || ids[i + 1] >= (uint64_t)V) {
      rc = 2;
      break;
    }
    matmul_nt(h, w_rec, pre, 1, H, H);
    for (int64_t j = 0; j < H; ++j) h[j] = act_f(act, pre[j] + w_in[(int64_t)ids[i] * H + j]);
    const uint32_t y = ids[i + 1];
    if (y == bos) continue;
    for (int64_t w = 0; w < V; ++w) sc[w] = (float)dot_acc(w_out + w * H, h, H);
    total += (double)sc[y] - lse_vec(sc, V);
    ++pred;
  }
  free(h);
  free(pre);
  free(sc);
  if (rc) return rc;
  if (pred == 0) return 1;
  *total_logprob = total;
  *predicted = pred;
  *ppl = exp(-total / (double)pred);
  return 0;
}

/* -------------------------------------------------------------- trainer */
/* Window construction for streams s0..s0+B-1 (trainer.hpp:376-387). */
void orc_window_build(const uint32_t* ids, int64_t L, const int64_t* cursors,
                      int64_t s0, int64_t B, int64_t T, uint32_t bos,
                      uint32_t* inputs, uint32_t* targets, uint8_t* weights) {
  for (int64_t t = 0; t < T; ++t)
    for (int64_t b = 0; b < B; ++b) {
      const int64_t pos = cursors[s0 + b] + t;
      const uint32_t x = ids[pos % L];
      const uint32_t y = ids[(pos + 1) % L];
      inputs[t * B + b] = x;
      targets[t * B + b] = y;
      weights[t * B + b] = (y == bos) ? 0 : 1;
    }
}

/* Mirrors the ref_train_config layout in oracle/ref_shim.cpp. */
typedef struct {
  int64_t nstate, nproj;
  int32_t noffset, minibatch, unroll, mode;
  double eta, rho, eps, clip;
  int32_t nce_k, max_epochs;
  double noise_floor;
  uint64_t seed;
  int32_t act, valid_shards;
  double divergence_factor;
  int64_t valid_limit;
  double init_range;
  int32_t threads, pad_;
} orc_train_config;

/* State of Trainer::rng_ after the last orc_train (313 words: the 312 state
 * words and the position, as `os << rng_` writes them, trainer.hpp:283-285):
 * it only advances in NCE mode (2 outputs per noise draw). */
static uint64_t g_train_rng[313];
void orc_last_train_rng(uint64_t* out) { memcpy(out, g_train_rng, sizeof g_train_rng); }

/* Trainer<StandardTraits> in softmax mode: constructor (trainer.hpp:178-212),
 * train() (:233-270), run_epoch() (:350-410), validate() (:223-228).
 * Params (inout), opt state (out), cursors (out, N), hidden (out, N*H),
 * logs (7 doubles/epoch).  Returns 2 on divergence (DataError). */
int orc_train(const orc_train_config* c, int64_t V, float* w_in, float* w_rec,
              float* w_out, const uint32_t* ids, int64_t L,
              const uint32_t* valid, int64_t n_valid, int run_epochs,
              float* m_rec, float* m_in, float* m_out, int64_t* cursors,
              float* hidden, double* logs, int* n_logs, double* initial_ppl,
              double* eta_out, double* best_out, int* bad_out, int* epoch_out) {
  const int64_t H = c->nstate, B = c->minibatch, T = c->unroll;
  const int64_t N = (int64_t)c->noffset * B;
  if (c->mode != 0 && c->mode != 1) return 1;
  if (L < N) return 1;
  const int nce = c->mode == 0;
  for (int64_t i = 0; i < N; ++i) cursors[i] = i * L / N;
  const float a0 = act_f(c->act, 0.0f);
  for (int64_t i = 0; i < N * H; ++i) hidden[i] = a0;
  const int64_t nv = (c->valid_limit > 0 && n_valid > c->valid_limit) ? c->valid_limit : n_valid;
  if (nv < 2) return 1;
  memset(m_rec, 0, sizeof(float) * H * H);
  memset(m_in, 0, sizeof(float) * V);
  memset(m_out, 0, sizeof(float) * V);
  double eta = c->eta, best = 0.0, initial = 0.0;
  int bad = 0, epoch = 0;
  *n_logs = 0;
  int rc = 0;
  uint32_t* xin = (uint32_t*)malloc(sizeof(uint32_t) * T * B);
  uint32_t* yt = (uint32_t*)malloc(sizeof(uint32_t) * T * B);
  uint8_t* wt = (uint8_t*)malloc(T * B);
  float* h0 = (float*)malloc(sizeof(float) * B * H);
  float* hf = (float*)malloc(sizeof(float) * B * H);
  uint32_t* gw = (uint32_t*)malloc(sizeof(uint32_t) * T * B);
  float* gd = (float*)malloc(sizeof(float) * T * B * H);
  float* grec = (float*)malloc(sizeof(float) * H * H);
  float* gout = (float*)malloc(sizeof(float) * V * H);
  /* NCE: NoiseModel::from_stream (nce.hpp:69-76, trainer.hpp:207-209) and
   * Trainer::rng_(seed) (trainer.hpp:184) */
  const int K1 = nce ? c->nce_k + 1 : 1;
  double *nq = NULL, *nlnkq = NULL, *nprob = NULL;
  uint32_t *nalias = NULL, *gow = NULL;
  float* god = NULL;
  uint64_t rng[313];
  if (nce) {
    double* counts = (double*)calloc((size_t)V, sizeof(double));
    for (int64_t i = 0; i < L; ++i)
      if (ids[i] != 1u) counts[ids[i]] += 1.0;
    nq = (double*)malloc(sizeof(double) * V);
    nlnkq = (double*)malloc(sizeof(double) * V);
    nprob = (double*)malloc(sizeof(double) * V);
    nalias = (uint32_t*)malloc(sizeof(uint32_t) * V);
    rc = orc_noise_build(V, counts, c->nce_k, c->noise_floor, nq, nlnkq, nprob, nalias);
    free(counts);
    orc_mt_state(c->seed, rng);
    gow = (uint32_t*)malloc(sizeof(uint32_t) * T * B * K1);
    god = (float*)malloc(sizeof(float) * T * B * K1 * H);
    if (rc) goto done;
  }
  if (run_epochs) {
    double tl;
    uint64_t pr;
    double ppl;
    if (orc_sharded_ppl(V, H, c->act, w_in, w_rec, w_out, valid, nv, c->valid_shards, 1, 1, &tl, &pr, &ppl)) {
      rc = 1;
      goto done;
    }
    initial = best = ppl;
    while (epoch < c->max_epochs && bad < 2) {
      const int64_t rounds = (L + N * T - 1) / (N * T);
      double loss_sum = 0.0;
      int64_t windows = 0, skipped = 0;
      for (int64_t r = 0; r < rounds; ++r)
        for (int64_t g = 0; g < c->noffset; ++g) {
          const int64_t s0 = g * B;
          orc_window_build(ids, L, cursors, s0, B, T, 1, xin, yt, wt);
          memcpy(h0, hidden + s0 * H, sizeof(float) * B * H);
          double loss;
          uint64_t pos;
          int64_t nrows;
          int applied;
          if (nce) {
            int64_t nout;
            orc_bptt_nce(V, H, c->act, w_in, w_rec, w_out, T, B, xin, yt, wt, h0,
                         1.0 / (double)(B * T), (float)c->clip, 1, c->nce_k, nlnkq, nprob,
                         nalias, rng, hf, &nrows, gw, gd, grec, &nout, gow, god, NULL, &loss,
                         &pos);
            orc_rmsprop(V, H, w_in, w_rec, w_out, m_rec, m_in, m_out, c->rho, c->eps, eta,
                        nrows, gw, gd, grec, 0, nout, gow, god, &applied);
          } else {
            orc_bptt(V, H, c->act, w_in, w_rec, w_out, T, B, xin, yt, wt, h0,
                     1.0 / (double)(B * T), (float)c->clip, 1, 1, hf, &nrows, gw,
                     gd, grec, gout, &loss, &pos);
            orc_rmsprop(V, H, w_in, w_rec, w_out, m_rec, m_in, m_out, c->rho,
                        c->eps, eta, nrows, gw, gd, grec, 1, 0, NULL, gout, &applied);
          }
          loss_sum += loss;
          ++windows;
          if (!applied) ++skipped;
          for (int64_t b = 0; b < B; ++b) {
            memcpy(hidden + (s0 + b) * H, hf + b * H, sizeof(float) * H);
            cursors[s0 + b] += T;
            if (cursors[s0 + b] >= L) {
              cursors[s0 + b] -= L;
              for (int64_t i = 0; i < H; ++i) hidden[(s0 + b) * H + i] = a0;
            }
          }
        }
      if (orc_sharded_ppl(V, H, c->act, w_in, w_rec, w_out, valid, nv, c->valid_shards, 1, 1, &tl, &pr, &ppl)) {
        rc = 1;
        goto done;
      }
      double* lg = logs + 7 * (*n_logs);
      lg[0] = ++epoch;
      lg[1] = windows > 0 ? loss_sum / (double)windows : 0.0;
      lg[2] = ppl;
      lg[3] = eta;
      lg[4] = 0.0;
      lg[5] = 0.0;
      lg[6] = (double)skipped;
      ++*n_logs;
      if (ppl > c->divergence_factor * initial) {
        rc = 2;
        goto done;
      }
      if (ppl < best) {
        best = ppl;
        bad = 0;
      } else {
        ++bad;
        eta *= 0.5;
      }
    }
  }
done:
  if (nce) memcpy(g_train_rng, rng, sizeof g_train_rng);
  else orc_mt_state(c->seed, g_train_rng);
  *initial_ppl = initial;
  *eta_out = eta;
  *best_out = best;
  *bad_out = bad;
  *epoch_out = epoch;
  free(xin);
  free(yt);
  free(wt);
  free(h0);
  free(hf);
  free(gw);
  free(gd);
  free(grec);
  free(gout);
  free(nq);
  free(nlnkq);
  free(nprob);
  free(nalias);
  free(gow);
  free(god);
  return rc;
}

/* ------------------------------------------------------- bottleneck model */
/* Tied-embedding bottleneck model (compress.hpp:38-415):
 *   pre = float(h . W_rec^T); pre = float(double(pre) + E[x] . U);
 *   h' = act(pre); z = float(h' . D); s_w = float(E[w] . z).
 * E is V x P, U is P x H, W_rec is H x H, D is H x P (row-major). */

/* BottleneckParams::init_uniform (compress.hpp:78-82): e, u, w_rec, d. */
int orc_bn_init_uniform(int64_t V, int64_t H, int64_t P, uint64_t seed, double range,
                        float* e, float* u, float* w_rec, float* d) {
  if (V < 1 || H < 1 || P < 1 || P > H) return 1;
  orc_mt64 m;
  orc_mt_seed(&m, seed);
  for (int64_t i = 0; i < V * P; ++i) e[i] = (float)uniform(&m, -range, range);
  for (int64_t i = 0; i < P * H; ++i) u[i] = (float)uniform(&m, -range, range);
  for (int64_t i = 0; i < H * H; ++i) w_rec[i] = (float)uniform(&m, -range, range);
  for (int64_t i = 0; i < H * P; ++i) d[i] = (float)uniform(&m, -range, range);
  return 0;
}

/* BottleneckAdapter::input_forward (compress.hpp:170-174): gathered rows
 * then matmul_nn accumulate into pre. */
static void bn_input_forward(const float* e, const float* u, int64_t H, int64_t P,
                             const uint32_t* words, int64_t B, float* eb, float* pre,
                             double* acc) {
  for (int64_t b = 0; b < B; ++b) memcpy(eb + b * P, e + (int64_t)words[b] * P, sizeof(float) * P);
  matmul_nn(eb, u, pre, B, H, P, 1, acc);
}

/* Softmax-mode window, bptt_run (backprop.hpp:76-222) over the bottleneck
 * adapter (compress.hpp:121-244): dense embedding gradient g_e [V x P]
 * (output side matmul_tn_add, input side row adds), g_u [P x H],
 * g_rec [H x H], g_d [H x P]; clipped at the end (compress.hpp:96-104). */
int orc_bn_bptt(int64_t V, int64_t H, int64_t P, int act, const float* e, const float* u,
                const float* w_rec, const float* d, int64_t T, int64_t B,
                const uint32_t* inputs, const uint32_t* targets, const uint8_t* weights,
                const float* h0, double loss_scale, float clip, int compute_grads,
                float* h_final, float* g_e, float* g_u, float* g_rec, float* g_d,
                double* loss, uint64_t* positions) {
  if (T < 1 || B < 1 || P < 1 || P > H) return 1;
  const int64_t BH = B * H, BP = B * P;
  const int64_t W = V > H ? V : H;
  float* h = (float*)malloc(sizeof(float) * (T + 1) * BH);
  float* z = (float*)malloc(sizeof(float) * T * BP);
  float* pre = (float*)malloc(sizeof(float) * BH);
  float* eb = (float*)malloc(sizeof(float) * BP);
  float* scores = (float*)malloc(sizeof(float) * B * V);
  double* acc = (double*)malloc(sizeof(double) * W);
  float* dsc = compute_grads ? (float*)calloc((size_t)(T * B * V), sizeof(float)) : NULL;
  memcpy(h, h0, sizeof(float) * BH);
  /* forward: bptt_run loop + out_begin (compress.hpp:195-202) */
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(h + t * BH, w_rec, pre, B, H, H);
    bn_input_forward(e, u, H, P, inputs + t * B, B, eb, pre, acc);
    for (int64_t i = 0; i < BH; ++i) h[(t + 1) * BH + i] = act_f(act, pre[i]);
    matmul_nn(h + (t + 1) * BH, d, z + t * BP, B, P, H, 0, acc);
  }
  if (h_final) memcpy(h_final, h + T * BH, sizeof(float) * BH);
  /* softmax loss: softmax_scores = z . E^T (compress.hpp:227-230) */
  double L = 0.0;
  uint64_t pos = 0;
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(z + t * BP, e, scores, B, V, P);
    for (int64_t b = 0; b < B; ++b) {
      const int64_t idx = t * B + b;
      if (!weights[idx]) continue;
      ++pos;
      const float* s = scores + b * V;
      double mx = (double)s[0];
      for (int64_t w = 1; w < V; ++w) mx = (mx < (double)s[w]) ? (double)s[w] : mx;
      double zz = 0.0;
      for (int64_t w = 0; w < V; ++w) zz += exp((double)s[w] - mx);
      const double lse = mx + log(zz);
      const uint32_t y = targets[idx];
      L += loss_scale * (lse - (double)s[y]);
      if (compute_grads) {
        float* dd = dsc + idx * V;
        for (int64_t w = 0; w < V; ++w) dd[w] = (float)(loss_scale * exp((double)s[w] - lse));
        dd[y] -= (float)loss_scale;
      }
    }
  }
  *loss = L;
  *positions = pos;
  if (compute_grads) {
    float* dh = (float*)calloc((size_t)BH, sizeof(float));
    float* dpre = (float*)malloc(sizeof(float) * BH);
    float* dz = (float*)malloc(sizeof(float) * BP);
    float* din = (float*)malloc(sizeof(float) * BP);
    memset(g_e, 0, sizeof(float) * V * P);
    memset(g_u, 0, sizeof(float) * P * H);
    memset(g_rec, 0, sizeof(float) * H * H);
    memset(g_d, 0, sizeof(float) * H * P);
    for (int64_t t = T - 1; t >= 0; --t) {
      const float* dst = dsc + t * B * V;
      const float* ht1 = h + (t + 1) * BH;
      const float* zt = z + t * BP;
      /* softmax_backward (compress.hpp:237-243) */
      matmul_nn(dst, e, dz, B, P, V, 0, acc);
      matmul_tn_add(dst, zt, g_e, B, V, P);
      /* out_end (compress.hpp:221-225): dh += dz . D^T (double, one rounding) */
      for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < H; ++i)
          dh[b * H + i] = (float)((double)dh[b * H + i] + dot_acc(dz + b * P, d + i * P, P));
      matmul_tn_add(ht1, dz, g_d, B, H, P);
      for (int64_t i = 0; i < BH; ++i) dpre[i] = dh[i] * act_deriv_f(act, ht1[i]);
      matmul_tn_add(dpre, h + t * BH, g_rec, B, H, H);
      /* input_backward (compress.hpp:176-193) */
      const uint32_t* words = inputs + t * B;
      for (int64_t b = 0; b < B; ++b)
        memcpy(eb + b * P, e + (int64_t)words[b] * P, sizeof(float) * P);
      matmul_tn_add(eb, dpre, g_u, B, P, H);
      matmul_nt(dpre, u, din, B, P, H);
      for (int64_t b = 0; b < B; ++b) {
        float* dstrow = g_e + (int64_t)words[b] * P;
        for (int64_t k = 0; k < P; ++k) dstrow[k] += din[b * P + k];
      }
      if (t > 0) matmul_nn(dpre, w_rec, dh, B, H, H, 0, acc);
    }
    for (int64_t i = 0; i < V * P; ++i) g_e[i] = clip1(g_e[i], clip);
    for (int64_t i = 0; i < P * H; ++i) g_u[i] = clip1(g_u[i], clip);
    for (int64_t i = 0; i < H * H; ++i) g_rec[i] = clip1(g_rec[i], clip);
    for (int64_t i = 0; i < H * P; ++i) g_d[i] = clip1(g_d[i], clip);
    free(dh);
    free(dpre);
    free(dz);
    free(din);
  }
  free(h);
  free(z);
  free(pre);
  free(eb);
  free(scores);
  free(acc);
  free(dsc);
  return 0;
}

/* rms_dense_elem (compress.hpp:282-292) */
static void rms_elem(float* w, const float* g, float* m, int64_t n, double rho, double eps,
                     double eta) {
  for (int64_t i = 0; i < n; ++i) {
    const double gi = (double)g[i];
    m[i] = (float)(rho * (double)m[i] + (1.0 - rho) * gi * gi);
    w[i] -= (float)(eta * gi / sqrt((double)m[i] + eps));
  }
}

/* bottleneck_update, dense embedding gradient (compress.hpp:296-309). */
int orc_bn_update(int64_t V, int64_t H, int64_t P, float* e, float* u, float* w_rec, float* d,
                  float* m_e, float* m_u, float* m_rec, float* m_d, double rho, double eps,
                  double eta, const float* g_e, const float* g_u, const float* g_rec,
                  const float* g_d, int* applied) {
  if (!(all_finite(g_e, V * P) && all_finite(g_u, P * H) && all_finite(g_rec, H * H) &&
        all_finite(g_d, H * P))) {
    *applied = 0;
    return 0;
  }
  update_rows_dense(e, V, P, g_e, m_e, rho, eps, eta);
  rms_elem(u, g_u, m_u, P * H, rho, eps, eta);
  rms_elem(w_rec, g_rec, m_rec, H * H, rho, eps, eta);
  rms_elem(d, g_d, m_d, H * P, rho, eps, eta);
  *applied = 1;
  return 0;
}

/* sharded_perplexity (eval.hpp:151-222) over the bottleneck adapter:
 * scores_t = E . z (compress.hpp:232-235). */
int orc_bn_sharded_ppl(int64_t V, int64_t H, int64_t P, int act, const float* e,
                       const float* u, const float* w_rec, const float* d,
                       const uint32_t* ids, int64_t n, int shards, uint32_t bos,
                       double* total_logprob, uint64_t* predicted, double* ppl) {
  if (n < 2 || shards < 1) return 1;
  const int64_t S = shards < n / 2 ? shards : n / 2;
  int64_t max_len = 0;
  for (int64_t s = 0; s < S; ++s) {
    const int64_t len = (s + 1) * n / S - s * n / S;
    if (len > max_len) max_len = len;
  }
  const float a0 = act_f(act, 0.0f);
  const int64_t W = V > H ? V : H;
  float* h = (float*)malloc(sizeof(float) * S * H);
  float* pre = (float*)malloc(sizeof(float) * S * H);
  float* eb = (float*)malloc(sizeof(float) * S * P);
  float* z = (float*)malloc(sizeof(float) * S * P);
  float* sc = (float*)malloc(sizeof(float) * V);
  double* acc = (double*)malloc(sizeof(double) * W);
  uint32_t* in = (uint32_t*)malloc(sizeof(uint32_t) * S);
  int64_t* tgt = (int64_t*)malloc(sizeof(int64_t) * S);
  for (int64_t i = 0; i < S * H; ++i) h[i] = a0;
  double total = 0.0;
  uint64_t pred = 0;
  int rc = 0;
  for (int64_t j = 0; j + 1 < max_len; ++j) {
    int any = 0;
    for (int64_t s = 0; s < S; ++s) {
      const int64_t b0 = s * n / S, len = (s + 1) * n / S - b0;
      if (j + 1 < len) {
        const uint32_t x = ids[b0 + j], y = ids[b0 + j + 1];
        if (x >= (uint64_t)V || y >= (uint64_t)V) {
          rc = 2;
          goto done;
        }
        in[s] = x;
        tgt[s] = (y == bos) ? -1 : (int64_t)y;
      } else {
        in[s] = 0;
        tgt[s] = -1;
      }
      any = any || tgt[s] >= 0;
    }
    matmul_nt(h, w_rec, pre, S, H, H);
    bn_input_forward(e, u, H, P, in, S, eb, pre, acc);
    for (int64_t i = 0; i < S * H; ++i) h[i] = act_f(act, pre[i]);
    if (!any) continue;
    matmul_nn(h, d, z, S, P, H, 0, acc);
    for (int64_t s = 0; s < S; ++s) {
      if (tgt[s] < 0) continue;
      for (int64_t w = 0; w < V; ++w) sc[w] = (float)dot_acc(e + w * P, z + s * P, P);
      total += (double)sc[tgt[s]] - lse_vec(sc, V);
      ++pred;
    }
  }
  *total_logprob = total;
  *predicted = pred;
  if (pred == 0) rc = 1;
  else *ppl = exp(-total / (double)pred);
done:
  free(h);
  free(pre);
  free(eb);
  free(z);
  free(sc);
  free(acc);
  free(in);
  free(tgt);
  return rc;
}

/* NCE-mode window over the bottleneck adapter (backprop.hpp:126-156,
 * 193-222; compress.hpp:204-225): scores float(dot_acc(z_b, E[w])), the
 * embedding gradient as one SparseRowGrads in first-touch slot order over
 * both sides (per step t: the output records, then the input rows) --
 * g_e_words / g_e_data must hold T*B*(k+2) rows. */
int orc_bn_bptt_nce(int64_t V, int64_t H, int64_t P, int act, const float* e, const float* u,
                    const float* w_rec, const float* d, int64_t T, int64_t B,
                    const uint32_t* inputs, const uint32_t* targets, const uint8_t* weights,
                    const float* h0, double loss_scale, float clip, int compute_grads, int k,
                    const double* ln_kq, const double* prob, const uint32_t* alias,
                    uint64_t* rng, float* h_final, int64_t* g_e_rows, uint32_t* g_e_words,
                    float* g_e_data, float* g_u, float* g_rec, float* g_d, double* loss,
                    uint64_t* positions) {
  if (T < 1 || B < 1 || k < 1 || P < 1 || P > H) return 1;
  const int64_t BH = B * H, BP = B * P, K1 = k + 1;
  orc_mt64 m;
  mt_load(&m, rng);
  float* h = (float*)malloc(sizeof(float) * (T + 1) * BH);
  float* z = (float*)malloc(sizeof(float) * T * BP);
  float* pre = (float*)malloc(sizeof(float) * BH);
  float* eb = (float*)malloc(sizeof(float) * BP);
  double* acc = (double*)malloc(sizeof(double) * (V > H ? V : H));
  uint32_t* rw = (uint32_t*)malloc(sizeof(uint32_t) * T * B * K1);
  float* rds = (float*)malloc(sizeof(float) * T * B * K1);
  int* has = (int*)calloc((size_t)(T * B), sizeof(int));
  memcpy(h, h0, sizeof(float) * BH);
  for (int64_t t = 0; t < T; ++t) {
    matmul_nt(h + t * BH, w_rec, pre, B, H, H);
    bn_input_forward(e, u, H, P, inputs + t * B, B, eb, pre, acc);
    for (int64_t i = 0; i < BH; ++i) h[(t + 1) * BH + i] = act_f(act, pre[i]);
    matmul_nn(h + (t + 1) * BH, d, z + t * BP, B, P, H, 0, acc);
  }
  if (h_final) memcpy(h_final, h + T * BH, sizeof(float) * BH);
  double L = 0.0;
  uint64_t pos = 0;
  for (int64_t t = 0; t < T; ++t) {
    const float* zt = z + t * BP;
    for (int64_t b = 0; b < B; ++b) {
      const int64_t idx = t * B + b;
      if (!weights[idx]) continue;
      ++pos;
      has[idx] = 1;
      const uint32_t y = targets[idx];
      const double st = (double)(float)dot_acc(zt + b * P, e + (int64_t)y * P, P);
      const double at = st - ln_kq[y];
      L += loss_scale * softplus(-at);
      rw[idx * K1] = y;
      rds[idx * K1] = (float)(-loss_scale * sigmoid(-at));
      for (int j = 0; j < k; ++j) {
        const uint32_t w = alias_sample(&m, V, prob, alias);
        const double s = (double)(float)dot_acc(zt + b * P, e + (int64_t)w * P, P);
        const double a = s - ln_kq[w];
        L += loss_scale * softplus(a);
        rw[idx * K1 + 1 + j] = w;
        rds[idx * K1 + 1 + j] = (float)(loss_scale * sigmoid(a));
      }
    }
  }
  mt_store(&m, rng);
  *loss = L;
  *positions = pos;
  if (compute_grads) {
    float* dh = (float*)calloc((size_t)BH, sizeof(float));
    float* dpre = (float*)malloc(sizeof(float) * BH);
    float* dz = (float*)malloc(sizeof(float) * BP);
    float* din = (float*)malloc(sizeof(float) * BP);
    int32_t* slot = (int32_t*)malloc(sizeof(int32_t) * V);
    for (int64_t w = 0; w < V; ++w) slot[w] = -1;
    int64_t ne = 0;
#define BN_ROW(w_)                                                     \
  do {                                                                 \
    if (slot[(w_)] < 0) {                                              \
      slot[(w_)] = (int32_t)ne;                                        \
      g_e_words[ne] = (w_);                                            \
      memset(g_e_data + ne * P, 0, sizeof(float) * P);                 \
      ++ne;                                                            \
    }                                                                  \
  } while (0)
    memset(g_u, 0, sizeof(float) * P * H);
    memset(g_rec, 0, sizeof(float) * H * H);
    memset(g_d, 0, sizeof(float) * H * P);
    for (int64_t t = T - 1; t >= 0; --t) {
      const float* ht1 = h + (t + 1) * BH;
      const float* zt = z + t * BP;
      memset(dz, 0, sizeof(float) * BP);
      /* score_backward per record (compress.hpp:209-219) */
      for (int64_t b = 0; b < B; ++b) {
        const int64_t idx = t * B + b;
        if (!has[idx]) continue;
        for (int64_t r = 0; r < K1; ++r) {
          const uint32_t w = rw[idx * K1 + r];
          const float ds = rds[idx * K1 + r];
          const float* er = e + (int64_t)w * P;
          float* db = dz + b * P;
          for (int64_t i = 0; i < P; ++i) db[i] += ds * er[i];
          BN_ROW(w);
          float* gr = g_e_data + (int64_t)slot[w] * P;
          const float* zb = zt + b * P;
          for (int64_t i = 0; i < P; ++i) gr[i] += ds * zb[i];
        }
      }
      /* out_end (compress.hpp:221-225) */
      for (int64_t b = 0; b < B; ++b)
        for (int64_t i = 0; i < H; ++i)
          dh[b * H + i] = (float)((double)dh[b * H + i] + dot_acc(dz + b * P, d + i * P, P));
      matmul_tn_add(ht1, dz, g_d, B, H, P);
      for (int64_t i = 0; i < BH; ++i) dpre[i] = dh[i] * act_deriv_f(act, ht1[i]);
      matmul_tn_add(dpre, h + t * BH, g_rec, B, H, H);
      const uint32_t* words = inputs + t * B;
      for (int64_t b = 0; b < B; ++b)
        memcpy(eb + b * P, e + (int64_t)words[b] * P, sizeof(float) * P);
      matmul_tn_add(eb, dpre, g_u, B, P, H);
      matmul_nt(dpre, u, din, B, P, H);
      for (int64_t b = 0; b < B; ++b) {
        BN_ROW(words[b]);
        float* gr = g_e_data + (int64_t)slot[words[b]] * P;
        for (int64_t i = 0; i < P; ++i) gr[i] += 1.0f * din[b * P + i];
      }
      if (t > 0) matmul_nn(dpre, w_rec, dh, B, H, H, 0, acc);
    }
#undef BN_ROW
    *g_e_rows = ne;
    for (int64_t i = 0; i < ne * P; ++i) g_e_data[i] = clip1(g_e_data[i], clip);
    for (int64_t i = 0; i < P * H; ++i) g_u[i] = clip1(g_u[i], clip);
    for (int64_t i = 0; i < H * H; ++i) g_rec[i] = clip1(g_rec[i], clip);
    for (int64_t i = 0; i < H * P; ++i) g_d[i] = clip1(g_d[i], clip);
    free(dh);
    free(dpre);
    free(dz);
    free(din);
    free(slot);
  }
  free(h);
  free(z);
  free(pre);
  free(eb);
  free(acc);
  free(rw);
  free(rds);
  free(has);
  return 0;
}

/* bottleneck_update with a sparse embedding gradient (compress.hpp:303-304). */
int orc_bn_update_sparse(int64_t V, int64_t H, int64_t P, float* e, float* u, float* w_rec,
                         float* d, float* m_e, float* m_u, float* m_rec, float* m_d, double rho,
                         double eps, double eta, int64_t n_rows, const uint32_t* words,
                         const float* rows, const float* g_u, const float* g_rec,
                         const float* g_d, int* applied) {
  if (!(all_finite(rows, n_rows * P) && all_finite(g_u, P * H) && all_finite(g_rec, H * H) &&
        all_finite(g_d, H * P))) {
    *applied = 0;
    return 0;
  }
  update_rows_sparse(e, P, n_rows, words, rows, m_e, V, rho, eps, eta);
  rms_elem(u, g_u, m_u, P * H, rho, eps, eta);
  rms_elem(w_rec, g_rec, m_rec, H * H, rho, eps, eta);
  rms_elem(d, g_d, m_d, H * P, rho, eps, eta);
  *applied = 1;
  return 0;
}

/* ln_z_samples (eval.hpp:805-857) for the standard model: one pass, state
 * carried across sentences, ln Z = lse over W_out . h (float scores, double
 * lse) of the states after ids[i], i % stride == 0, stride = max(1, n/count). */
int orc_ln_z_samples(int64_t V, int64_t H, int act, const float* w_in, const float* w_rec,
                     const float* w_out, const uint32_t* ids, int64_t n, int64_t count,
                     double* out, int64_t* n_out) {
  if (n < 1 || count < 1) return 1;
  const int64_t stride = (n / count) > 1 ? n / count : 1;
  float* h = (float*)malloc(sizeof(float) * H);
  float* pre = (float*)malloc(sizeof(float) * H);
  float* sc = (float*)malloc(sizeof(float) * V);
  const float a0 = act_f(act, 0.0f);
  for (int64_t j = 0; j < H; ++j) h[j] = a0;
  int64_t ns = 0;
  int rc = 0;
  for (int64_t i = 0; i < n && ns < count; ++i) {
    if (ids[i] >= (uint64_t)V) {
      rc = 2;
      break;
    }
    matmul_nt(h, w_rec, pre, 1, H, H);
    for (int64_t j = 0; j < H; ++j) h[j] = act_f(act, pre[j] + w_in[(int64_t)ids[i] * H + j]);
    if (i % stride != 0) continue;
    for (int64_t w = 0; w < V; ++w) sc[w] = (float)dot_acc(w_out + w * H, h, H);
    out[ns++] = lse_vec(sc, V);
  }
  *n_out = ns;
  free(h);
  free(pre);
  free(sc);
  return rc;
}
