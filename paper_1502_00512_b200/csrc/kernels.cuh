// Launchers for the bandwidth-bound kernels (kernels.cu).
#pragma once

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace dl {

struct EmbedWs {
  int* seg_start;  // [T*B + 1] segment heads, then [T*B] long-segment slots, then their count
  int* order_pos;  // [T*B]
  int* long_list() const { return seg_start + cap + 1; }
  int* n_long() const { return seg_start + 2 * cap + 1; }
  int64_t cap;     // T*B (positions the buffers hold)
};

// NCE records of one window (nce.cu): forward-order words / h rows / ds,
// the processing-order -> forward map, and sort scratch
struct NceRecs {
  const uint32_t* rec_word;  // [N] forward order r = p*(k+1) + j
  const uint32_t* rec_row;   // [N] t*B + b of the record's position
  const uint32_t* proc_r;    // [N] processing order q -> r
  const float* ds;           // [N] dloss/dscore, forward order
  uint32_t *keys_in, *vals_in, *keys_out, *vals_out;
  int *head, *slot;
  void* temp;
  size_t temp_bytes;
};

void nce_records(const uint8_t* w, const uint32_t* y, int64_t T, int64_t B, int64_t P, int K1,
                 const unsigned long long* raw, const double* prob, const uint32_t* alias,
                 int64_t V, uint32_t* pos_of, int* first, uint32_t* rec_word, uint32_t* rec_row,
                 uint32_t* proc_r, cudaStream_t st);
// w_bf: score / backpropagate against the bf16 shadow of W_out (bf16 mode)
void nce_scores(const float* h, const float* w_out, int64_t H, const uint32_t* rec_word,
                const uint32_t* rec_row, int64_t N, float* score, cudaStream_t st,
                const bf16* w_bf = nullptr);
void nce_loss(const float* score, const uint32_t* rec_word, const double* ln_kq, int64_t P,
              int K1, double scale, double* loss_pos, float* ds, cudaStream_t st);
void nce_dh(const float* w_out, int64_t H, const uint32_t* rec_word, const uint32_t* rec_row,
            const float* ds, int64_t P, int K1, float* dh, cudaStream_t st,
            const bf16* w_bf = nullptr);
size_t nce_sort_temp_bytes(int64_t N);
// sparse W_out gradient rows (slot order = by word), clipped: rows / words /
// *n_rows on the device
void nce_out_rows(const NceRecs& R, int64_t N, int64_t V, const float* h, int64_t H, float clip,
                  struct EmbedWs& ws, float* order_scale, float* rows, uint32_t* words,
                  int* n_rows, int* nonfinite, cudaStream_t st);
int embed_short_max();
// NoiseModel + AliasSampler tables (host; nce.cu)
void noise_tables(const double* counts, int64_t V, int k, double floor, std::vector<double>& lnkq,
                  std::vector<double>& prob, std::vector<uint32_t>& alias);
void noise_tables_q(const double* q, int64_t V, int k, std::vector<double>& lnkq,
                    std::vector<double>& prob, std::vector<uint32_t>& alias);

void f32_to_bf16(const float* x, bf16* y, int64_t n, cudaStream_t st);
// out [cols x rows] (ld_out) = transpose of in [rows x cols] (ld_in), fp32
void transpose_f32(const float* in, int64_t rows, int64_t cols, int64_t ld_in, float* out,
                   int64_t ld_out, cudaStream_t st);
void fill_f32(float* x, float v, int64_t n, cudaStream_t st);
void rec_fwd(const float* part, int splits, int64_t split_stride, int64_t Bn, int64_t H,
             const float* w_in, const uint32_t* x, int act, float* h, bf16* hb, cudaStream_t st);
void rec_bwd(const float* part, int splits, int64_t split_stride, int64_t n, const float* dh_out,
             const float* hnext, int act, float* dpre, bf16* dpreb, cudaStream_t st);
void reduce_splits(const float* part, int splits, int64_t split_stride, int64_t n, float* out,
                   float clip, int do_clip, int* nonfinite, cudaStream_t st);
// the dW_rec reduction + clip and the W_rec rmsprop step in one pass (finite
// clip, n and split_stride multiples of 4)
void reduce_rms_rec(const float* part, int splits, int64_t split_stride, int64_t n, float* g_out,
                    float clip, float* w, bf16* wb, float* m, double rho, double eps, double eta,
                    cudaStream_t st);
// lse_all != nullptr: vocabulary-sharded rows -- lse from the G gathered
// block values [G][M], target logit from tgt_logit, tgt = local columns.
void softmax_rows_f32(float* S, int64_t M, int64_t V, const uint32_t* tgt, const uint8_t* wts,
                      double scale, int grads, double* loss_row, double* logp_row,
                      cudaStream_t st, const double* lse_all = nullptr, int G = 0,
                      const float* tgt_logit = nullptr);
// per-row lse / loss / log-prob and the dS transform's (lse, scale) for the
// dh GEMM's on-the-fly softmax (GemmDesc::xf)
void lse_rows_bf16(int64_t M, const float2* part, int n_tiles, const float* tgt_logit,
                   const uint8_t* wts, double scale, double* loss_row, double* logp_row,
                   float* lse_f, float* sc_f, cudaStream_t st, const double* lse_all = nullptr,
                   int G = 1);
void softmax_rows_bf16(bf16* S, int64_t M, int64_t V, const float2* part, int n_tiles,
                       const float* tgt_logit, const uint32_t* tgt, const uint8_t* wts,
                       double scale, int grads, double* loss_row, double* logp_row,
                       cudaStream_t st, const double* lse_all = nullptr, int G = 0);
// shifted-exponential softmax of the bf16 trainer (kernels.cu k_pfac_rows):
// shift[r] = the row's target logit (bf16 operands, fp32 dot) before the
// logits GEMM; after it, per row: lse, loss / log-prob, sigma[r] =
// scale e^(shift - lse) (0 masked), E's target column patched so that
// sigma E' = dS (resid[r]: the patch's bf16 rounding error), and hs_sc =
// bf16(sigma h) (dW_out's B operand).  Rows whose sum of E exceeds
// e^repair_nats, or with a half tile the epilogue redid against its own
// maximum, are rescaled in place to one shift (counted in repaired[0] /
// repaired[1]).
void target_shift(const bf16* hs, const bf16* w, int64_t H, int64_t M, const uint32_t* tgt,
                  int64_t V, float* shift, cudaStream_t st);
void pfac_rows(bf16* E, int64_t M, int64_t V, int64_t H, const float2* part, int n_tiles,
               const float* tgt_logit, const uint32_t* tgt, const uint8_t* wts, double scale,
               double* loss_row, double* logp_row, const float* shift, float* sigma,
               float* resid, const float* hs, bf16* hs_sc, const bf16* hs_bf, float repair_nats,
               int* repaired, cudaStream_t st, const double* lse_all = nullptr, int G = 1);
// vocabulary-sharded: this rank's block lse (lse_loc) after the rescales, for
// the exchange before pfac_rows(..., lse_all, G)
void pfac_lse(bf16* E, int64_t M, int64_t V, const float2* part, int n_tiles, const uint8_t* wts,
              float* shift, double* lse_loc, float repair_nats, int* repaired, cudaStream_t st);
void shard_targets(const uint32_t* y, int64_t M, int64_t v0, int64_t Vo, uint32_t* loc,
                   cudaStream_t st);
void block_lse_bf16(const float2* part, int n_tiles, int64_t M, double* lse, cudaStream_t st);
void block_lse_f32(const float* S, int64_t M, int64_t V, const uint32_t* loc, double* lse,
                   float* tgt_logit, cudaStream_t st);
void sum_rows(const double* v, const uint8_t* wts, int64_t n, double* acc,
              unsigned long long* cnt, cudaStream_t st);
// x / dpre: G rank-blocked windows [G][T][B] (G = 1 on one GPU)
// W_in gradient rows: embed_sort (stable radix sort of the window's ids,
// depends on x only) then embed_rows (segmented sums of dpre + clip);
// embed_grads = both
void embed_sort(const uint32_t* x, int64_t T, int64_t B, int64_t G, int64_t V, EmbedWs& ws,
                uint32_t* words, int* n_rows, cudaStream_t st);
// (order_scale: optional per-sorted-record factor -- the NCE W_out rows sum
// ds * h, SparseRowGrads::axpy_row rnn.hpp:113-116)
void embed_rows(int64_t n, const float* dpre, int64_t H, float clip, EmbedWs& ws, float* rows,
                int* n_rows, int* nonfinite, cudaStream_t st, const float* order_scale = nullptr);
void embed_grads(const uint32_t* x, int64_t T, int64_t B, int64_t G, int64_t V, const float* dpre, int64_t H,
                 float clip, EmbedWs& ws, float* rows, uint32_t* words, int* n_rows,
                 int* nonfinite, cudaStream_t st);
void embed_dense(const float* rows, const uint32_t* words, const int* n_rows, int64_t max_rows,
                 int64_t H, float* dense, cudaStream_t st);
void rms_rec(float* w, bf16* wb, float* m, const float* g, int64_t n, double rho, double eps,
             double eta, const int* nonfinite, cudaStream_t st);
void rms_decay(float* m, int64_t n, double rho, const int* nonfinite, cudaStream_t st);
void rms_rows(float* w, bf16* wb, float* m, const float* g, const uint32_t* words,
              const int* n_rows_dev, int64_t n_rows, int64_t H, double rho, double eps, double eta,
              int dense, const int* nonfinite, cudaStream_t st);
void count_skip(const int* nonfinite, unsigned long long* skipped, cudaStream_t st);
// dense W_out rmsprop from bf16 gradients + per-(half tile, row) sums of
// squares [nsub][V] (H % 8 == 0)
// data-parallel bf16 path: unclipped summed bf16 gradient, clip + update (H % 8 == 0)
void rms_dense_g16c(float* w, bf16* wb, float* m, const bf16* g, int64_t V, int64_t H,
                    float clip, double rho, double eps, double eta, cudaStream_t st);
void rms_dense_g16(float* w, bf16* wb, float* m, const bf16* g, const double* rowsq, int nsub,
                   int64_t V, int64_t H, double rho, double eps, double eta, cudaStream_t st);

// rec_tc.cu: one recurrence step, tcgen05 + split-K cluster/DSMEM reduction.
// mode 0: out = act(A . W_rec^T + W_in[x]); mode 1: out = (A . W_rec +
// dh_out) * act'(hnext).  A is [M x H] bf16, K-major.
void rec_plan(int M, int H, int& bn, int& S);
// All T steps in one persistent cluster launch (W_rec slice resident in
// shared memory, grid barrier per step).  mode 0: A tape = h (bf16) rows
// [(T+1) x M]; writes htape[s+1].  mode 1: A tape = dpre (bf16) [T x M];
// writes dpre[s] for s = T-1..0.  Returns false if it cannot run (caller
// falls back to rec_step_tc per step).
bool rec_window_tc(int mode, int T, int M, int H, int act, const bf16* a_tape, int64_t a_rows,
                   const bf16* w_rec_bf, const float* w_in, const uint32_t* x,
                   const float* dh_out, const float* htape, float* out, bf16* outb,
                   unsigned* counter, cudaStream_t st);
void rec_step_tc(int mode, int M, int H, int act, const bf16* A, const bf16* w_rec_bf,
                 const float* w_in, const uint32_t* x, const float* dh_out, const float* hnext,
                 float* out, bf16* outb, cudaStream_t st);
void set_flag(int* dst, const int* src, int value, cudaStream_t st);
void accum_loss(double* acc, const double* v, unsigned long long* cnt,
                const unsigned long long* vc, cudaStream_t st);
void window_build(const uint32_t* ids, int64_t L, const int64_t* cursors, const float* hidden,
                  const int64_t* win_counter, int noffset, int64_t B, int64_t T, int64_t H,
                  uint32_t bos, uint32_t* x, uint32_t* y, uint8_t* w, float* h0, cudaStream_t st,
                  bf16* h0b = nullptr);
// hidden carry + cursor advance; then the window counter (and, with
// nonfinite / skipped, the skipped-update count) in one tail kernel
void window_finish(int64_t* cursors, float* hidden, const float* h_final, int64_t* win_counter,
                   int noffset, int64_t B, int64_t T, int64_t H, int64_t L, float a0,
                   cudaStream_t st, const int* nonfinite = nullptr,
                   unsigned long long* skipped = nullptr);

}  // namespace dl
