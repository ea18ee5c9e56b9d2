/*
 * desklm_cuda.h -- C ABI of the B200-native RNNLM training / scoring path.
 *
 * This is the drop-in boundary between the desklm host API (C++ Trainer /
 * Traits / Adapter, /root/reference/proj/include/desklm) and the sm_100a
 * kernels in libdesklm_cuda.so.  Plain pointers and sizes only; every host
 * array is borrowed for the duration of the call; all device memory is owned
 * by the opaque context.  Each entry point names the reference interface it
 * replaces (paths relative to /root/reference/proj/include/desklm).
 *
 * Status codes mirror the reference's error classes (util.hpp:32-48,
 * tools/desklm.cpp:1382-1390):
 *   DL_OK 0, DL_EINVAL 1 (std::invalid_argument, CLI exit 1),
 *   DL_EDATA 2 (DataError, CLI exit 2), DL_EDEVICE 3 (CUDA/NCCL failure).
 * dl_last_error() returns the message of the last failure on that context
 * (or the last global failure when ctx is NULL).
 *
 * Threading: one context per (host thread, GPU); calls on a context are
 * serialised on its CUDA stream; value-returning calls synchronise.
 */
#ifndef DESKLM_CUDA_H
#define DESKLM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dl_ctx dl_ctx;

enum { DL_OK = 0, DL_EINVAL = 1, DL_EDATA = 2, DL_EDEVICE = 3 };

/* Arithmetic of the GEMMs.  DL_FP32: fp32 SIMT kernels (parity mode,
 * reference tolerance 1e-4).  DL_BF16: tcgen05/TMEM tensor-core kernels with
 * bf16 operands, fp32 accumulation, fp32 master weights (throughput mode).
 * DL_TF32X3: the fp32 mode with its GEMMs on the tensor cores as 3xTF32
 * (tcgen05 kind::tf32: hi.hi + hi.lo + lo.hi of the split fp32 operands,
 * fp32 accumulation in K chunks summed round-to-nearest) -- fp32-class
 * numbers at 5-10x the SIMT speed; everything else as DL_FP32. */
enum { DL_FP32 = 0, DL_BF16 = 1, DL_TF32X3 = 2 };

/* Activation (rnn.hpp:35: enum class Activation { kSigmoid, kTanh }). */
enum { DL_SIGMOID = 0, DL_TANH = 1 };

const char* dl_last_error(const dl_ctx* ctx);
const char* dl_version(void);

/* ---- model / optimiser state ------------------------------------------ */

/* Replaces the StandardAdapter view construction (rnn.hpp:187-189) and
 * RnnParams<float> storage (rnn.hpp:61-84): V x H W_in, H x H W_rec,
 * V x H word-major W_out live in HBM for the context's lifetime. */
int dl_create(dl_ctx** out, int device, int64_t V, int64_t H, int act,
              int precision);
int dl_destroy(dl_ctx* ctx);

/* Upload / download RnnParams<float> (row-major, W_out word-major V x H as
 * in memory, rnn.hpp:61-77).  Download is what write_params (rnn.hpp:263)
 * serialises. */
int dl_set_params(dl_ctx* ctx, const float* w_in, const float* w_rec,
                  const float* w_out);
int dl_get_params(dl_ctx* ctx, float* w_in, float* w_rec, float* w_out);

/* Host-only: RnnParams<float>::init_uniform (rnn.hpp:79-83) -- one
 * std::mt19937_64(seed) drawn over w_in, w_rec, w_out in order, uniform in
 * [-range, range) exactly as rng.hpp:37-44; bit-identical to the reference. */
int dl_init_uniform(int64_t V, int64_t H, uint64_t seed, double range,
                    float* w_in, float* w_rec, float* w_out);

/* RmspropState (rmsprop.hpp:37-59): m_rec H x H, m_in V, m_out V. */
int dl_set_opt(dl_ctx* ctx, const float* m_rec, const float* m_in,
               const float* m_out, double rho, double eps);
int dl_get_opt(dl_ctx* ctx, float* m_rec, float* m_in, float* m_out);

/* ---- one truncated-BPTT window ----------------------------------------- */

/* bptt_run<StandardAdapter<float>> in softmax mode (backprop.hpp:76-222,
 * BpttOptions backprop.hpp:52-61, WindowBatch backprop.hpp:36-50):
 * t-major (index t*B+b) inputs/targets/weights, h0 B x H, optional h_final.
 * With compute_grads the clipped gradients stay on the device for
 * dl_rmsprop / dl_get_grads.  *loss = scaled summed loss, *positions =
 * unmasked count (BpttResult, backprop.hpp:63-66). */
int dl_window(dl_ctx* ctx, int64_t T, int64_t B, const uint32_t* inputs,
              const uint32_t* targets, const uint8_t* weights,
              const float* h0, float* h_final, double loss_scale, float clip,
              int compute_grads, double* loss, uint64_t* positions);

/* Dense copies of the last window's clipped gradients (tests; the
 * reference's StandardGrads, rnn.hpp:147-172, with SparseRowGrads::to_dense
 * for W_in).  Any pointer may be NULL. */
int dl_get_grads(dl_ctx* ctx, float* g_in_dense, float* g_rec, float* g_out);

/* Test hook: load externally computed (already clipped) gradients in the
 * reference's StandardGrads form -- sparse W_in rows (n_in_rows rows of H,
 * words in_words), dense W_rec, dense W_out -- so rmsprop parity can be
 * checked on identical inputs. */
int dl_set_grads(dl_ctx* ctx, int64_t n_in_rows, const uint32_t* in_words,
                 const float* in_rows, const float* g_rec, const float* g_out);

/* rmsprop_update (rmsprop.hpp:113-133) with the device-resident gradients
 * of the last dl_window.  *applied = 0 mirrors the reference's `false`
 * (non-finite gradient: parameters and accumulators untouched). */
int dl_rmsprop(dl_ctx* ctx, double eta, int* applied);

/* One training step of Trainer::run_epoch (trainer.hpp:391-397): bptt_run on
 * the window (as dl_window with compute_grads = 1) followed by
 * Traits::update = rmsprop_update (rmsprop.hpp:113-133) with eta.  Same
 * results as dl_window + dl_rmsprop; in DL_BF16 mode with a finite clip the
 * dense W_out update runs inside the dW_out GEMM's epilogue (the gradient is
 * never stored).  *applied as for dl_rmsprop. */
int dl_train_window(dl_ctx* ctx, int64_t T, int64_t B, const uint32_t* inputs,
                    const uint32_t* targets, const uint8_t* weights,
                    const float* h0, float* h_final, double loss_scale, float clip,
                    double eta, double* loss, uint64_t* positions, int* applied);

/* ---- scoring ------------------------------------------------------------ */

/* Lock-step forward scorer over S streams for `steps` steps (the inner loop
 * of sharded_perplexity, eval.hpp:176-220; rnn_perplexity eval.hpp:84-145;
 * the RNN half of rescore_nbest eval.hpp:725-751).  in[j*S+s] is the input
 * id, tgt[j*S+s] the target id or -1 (not scored).  h0 (S x H) may be NULL
 * for act(0).  logp (steps x S, NaN where skipped) and h_final may be NULL.
 * Sums are over scored positions in (j, s) order. */
int dl_score(dl_ctx* ctx, int64_t S, int64_t steps, const uint32_t* in,
             const int64_t* tgt, const float* h0, float* h_final, double* logp,
             double* total_logprob, uint64_t* predicted);

/* sharded_perplexity (eval.hpp:151-222) and rnn_perplexity
 * (eval.hpp:84-145) with the reference's argument meaning and errors. */
int dl_sharded_perplexity(dl_ctx* ctx, const uint32_t* ids, int64_t n,
                          int shards, uint32_t bos_id, double* total_logprob,
                          uint64_t* predicted, double* perplexity);
int dl_rnn_perplexity(dl_ctx* ctx, const uint32_t* ids, int64_t n,
                      uint32_t bos_id, double* total_logprob,
                      uint64_t* predicted, double* perplexity);

/* ln_z_samples (eval.hpp:805-857): ln Z at up to `count` hidden states taken
 * at stride max(1, n / count) from one pass over the stream (state carried
 * across sentences).  out: count doubles; *n_out: states taken.  The host
 * drift_stats (eval.hpp:859-880) runs on these. */
int dl_ln_z_samples(dl_ctx* ctx, const uint32_t* ids, int64_t n, int64_t count, double* out,
                    int64_t* n_out);

/* RnnHitScorer (eval.hpp:476-510) over one stream: after each input id
 * in[j], the raw scores float(h . W_out[w]) (8-lane double dot, as
 * Adapter::score) of the candidates cand[j*K .. j*K+K) (-1 = none) into
 * out[j*K + k]; the host ranks them (hit_rate, eval.hpp:544-592). */
int dl_score_candidates(dl_ctx* ctx, const uint32_t* in, int64_t steps, int64_t K,
                        const int64_t* cand, float* out);

/* ---- device-resident trainer (Trainer<Traits>::run_epoch) -------------- */

/* Uploads the training IdStream once and sets up the offset-stream schedule
 * of trainer.hpp:188-198 / :350-410: N = noffset*minibatch streams with
 * cursors floor(i*L/N), hidden = act(0).  With a communicator of G ranks
 * (dl_comm_init) the global minibatch is G*minibatch and this rank owns
 * streams [rank*minibatch, (rank+1)*minibatch) of every group. */
int dl_trainer_init(dl_ctx* ctx, const uint32_t* ids, int64_t L, int noffset,
                    int minibatch, int unroll, double clip, uint32_t bos_id);

/* Runs windows [first, first+count) of the epoch schedule (window w is
 * group w % noffset), each = window build + bptt_run + rmsprop_update +
 * hidden carry + cursor advance with wrap reset, entirely on the device
 * (captured in a CUDA graph).  Adds the windows' losses (sum over windows)
 * and skipped updates to the outputs. */
int dl_trainer_run(dl_ctx* ctx, int64_t first, int64_t count, double eta,
                   double* loss_sum, uint64_t* skipped);

/* Host-only: this rank's initial cursors (noffset*minibatch of them,
 * group-major) -- floor(i*L/N) of trainer.hpp:194-195 over the global
 * stream index i = g*G*minibatch + rank*minibatch + b. */
int dl_rank_cursors(int64_t L, int noffset, int minibatch, int nranks, int rank,
                    int64_t* out);

/* Schedule state for checkpoints (RTRN cursors + hidden, trainer.hpp:286-288).
 * Arrays cover this rank's streams (N/G of them, group-major). */
int dl_trainer_get_state(dl_ctx* ctx, int64_t* cursors, float* hidden);
int dl_trainer_set_state(dl_ctx* ctx, const int64_t* cursors,
                         const float* hidden);

/* ---- multi-GPU ----------------------------------------------------------- */

/* NCCL communicator for data-parallel streams (gradient allreduce before
 * clip).  Rank 0 calls dl_comm_unique_id and broadcasts the 128 bytes.  A
 * one-rank communicator is a real NCCL communicator: the multi-rank code
 * paths (collectives, gathered windows, the sharded output layer) run on a
 * single GPU with identity exchanges. */
int dl_comm_unique_id(uint8_t id[128]);
int dl_comm_init(dl_ctx* ctx, const uint8_t id[128], int nranks, int rank);

/* In-process rank groups: G contexts on ONE device act as G ranks (one host
 * thread per context, collectives through device memory with a host
 * barrier) so the multi-rank paths can be exercised on a single GPU.  Same
 * semantics as dl_comm_init otherwise. */
int dl_local_group_create(int G, void** group);
int dl_local_group_destroy(void* group);
int dl_comm_init_local(dl_ctx* ctx, void* group, int rank);

/* ---- NCE (LossMode::kNce, the reference's default training mode) ------- */

/* Loss mode of the following windows: 0 = NCE (backprop.hpp:126-156), 1 =
 * exact softmax (the default of a fresh context).  TrainConfig::mode,
 * trainer.hpp:53. */
int dl_set_loss_mode(dl_ctx* ctx, int mode);

/* NoiseModel(counts, k, floor) (nce.hpp:41-66): unigram counts of the
 * training stream (NoiseModel::from_stream counts every non-bos token),
 * k noise samples per position.  Sampling uses the AliasSampler of
 * rng.hpp:54-94 on the host, the ln(k q) table lives on the device. */
int dl_set_noise(dl_ctx* ctx, const double* counts, int64_t V, int k, double floor);

/* The same noise model from its normalised distribution q (NoiseModel::q,
 * nce.hpp:54-64, already floored and renormalised by the caller, e.g. a
 * reference NoiseModel): ln(k q) and the AliasSampler(q) tables are built
 * from q exactly as the reference builds them. */
int dl_set_noise_dist(dl_ctx* ctx, const double* q, int64_t V, int k);

/* The std::mt19937_64 the noise draws come from (BpttOptions::rng,
 * backprop.hpp:52-61; Trainer::rng_, trainer.hpp:184, :284, :314): 312 state
 * words then the position, as the libstdc++ stream operators write them.
 * Every NCE window advances it by 2 draws per noise sample. */
int dl_set_rng_state(dl_ctx* ctx, const uint64_t state[313]);
int dl_get_rng_state(const dl_ctx* ctx, uint64_t state[313]);
/* state of std::mt19937_64(seed) (host helper) */
int dl_rng_seed_state(uint64_t seed, uint64_t state[313]);

/* Vocabulary-sharded softmax (no reference counterpart: the reference's
 * output layer, rnn.hpp:245-258 / backprop.hpp:162-186, is one V x H
 * matrix).  With on != 0, after dl_comm_init(_local) with G ranks, rank r
 * holds only W_out / m_out rows [r*V/G, (r+1)*V/G); every rank runs the same
 * windows (identical inputs, no minibatch split).  Per window the ranks
 * exchange G x TB block log-sum-exps and the target logits (forward) and sum
 * dh = dS . W_out (backward); W_in / W_rec stay replicated and bit-identical.
 * dl_set_params / dl_set_opt read, and dl_get_params / dl_get_opt /
 * dl_get_grads write, only this rank's W_out / m_out rows of the full V-row
 * host arrays.  Resets W_out and m_out to zero: call before dl_set_params.
 * dl_comm_init(_local) turns sharding off again.
 * on == 2: data-parallel streams with a vocabulary-parallel output layer --
 * every rank trains its own B streams (global minibatch G*B, as without
 * sharding) and keeps W_out rows [r*V/G, (r+1)*V/G).  Per window the hidden
 * states, targets and weights of all ranks are all-gathered, each rank
 * scores the whole global window against its block (the same G x rows
 * log-sum-exp exchange), the partial dh is reduce-scattered back to the
 * rank owning the rows, and W_rec / W_in are summed as in plain data
 * parallel: no V x H gradient crosses the links and the dense W_out update
 * is split G ways.  Scoring calls keep the on == 1 semantics (identical
 * inputs on every rank). */
int dl_set_vocab_shard(dl_ctx* ctx, int on);

/* ---- instrumentation ----------------------------------------------------- */

/* Test hook for the GEMM engine behind every matmul_* of mat.hpp:116-184:
 * C[M x N] = A . B^T with A K-major [M x K] (a_major 0) or MN-major [K x M]
 * (1), likewise B ([N x K] / [K x N]); fp32 host data (rounded to bf16 in
 * DL_BF16 mode).  splits > 1 exercises split-K.  With tgt != NULL (DL_BF16)
 * the online-LSE logits epilogue runs and Cout receives M*N bf16 logits
 * (widened), then M log-probs of tgt, then M target logits. */
int dl_test_gemm(dl_ctx* ctx, int M, int N, int K, int a_major, int b_major,
                 const float* A, const float* B, float* Cout, int splits,
                 const uint32_t* tgt);

/* Test hook for the data-parallel W_in gradient (SparseRowGrads over the
 * gathered window, rnn.hpp:89-127): G rank-blocked windows x_all [G][T][B]
 * and dpre_all [G][T][B][H] -> clipped dense g_in [V x H], each word's row
 * summed in the reference's order (t descending, global stream ascending). */
int dl_test_embed(dl_ctx* ctx, int G, int64_t T, int64_t B,
                  const uint32_t* x_all, const float* dpre_all, float clip,
                  float* g_in_dense);

/* Kernel launches issued on the context's streams since creation (graph
 * replays count every kernel node). */
uint64_t dl_launch_count(const dl_ctx* ctx);
/* The context's cudaStream_t (as void*), for CUDA-event timing by callers. */
void* dl_cuda_stream(const dl_ctx* ctx);
/* Average device time (ms) of the named kernel class over the last
 * dl_trainer_run / dl_window when profiling is on ("logits", "dh", "dw_out",
 * "recurrence", "rmsprop", ...); returns -1 if unknown. */
int dl_set_profiling(dl_ctx* ctx, int on);
double dl_kernel_ms(const dl_ctx* ctx, const char* name);

/* ------------------------------------------------------------------
 * Bottleneck / tied-embedding model (compress.hpp:38-415), a second model
 * family on the same engine: BottleneckParams {E [V x P], U [P x H],
 * W_rec [H x H], D [H x P]} with h' = act(E[x] . U + W_rec . h),
 * z = h' . D, s_w = E[w] . z.  One context per (host thread, GPU); the
 * device boundary is again per window and per scoring call.  Replaces the
 * reference's BottleneckAdapter / BottleneckTraits seams:
 *   dl_bn_create / dl_bn_set_params   BottleneckParams (compress.hpp:54-83)
 *   dl_bn_set_opt / dl_bn_get_opt     BottleneckOptState (compress.hpp:252-278)
 *   dl_bn_window                      bptt_run(BottleneckAdapter), softmax mode
 *                                     (backprop.hpp:76-222, compress.hpp:121-244)
 *   dl_bn_get_grads                   BottleneckGrads, dense E (compress.hpp:87-115)
 *   dl_bn_rmsprop                     bottleneck_update (compress.hpp:296-309)
 *   dl_bn_sharded_perplexity          sharded_perplexity(BottleneckAdapter)
 *                                     (eval.hpp:151-222)
 * Same status codes and error behaviour as the standard model's calls;
 * P > H is rejected like the reference constructor (compress.hpp:72-73).
 * ------------------------------------------------------------------ */
typedef struct dl_bn dl_bn;

int dl_bn_create(dl_bn** out, int device, int64_t V, int64_t H, int64_t P, int act,
                 int precision);
int dl_bn_destroy(dl_bn* ctx);
const char* dl_bn_last_error(const dl_bn* ctx);
/* e [V x P], u [P x H], w_rec [H x H], d [H x P], row-major fp32 */
int dl_bn_set_params(dl_bn* ctx, const float* e, const float* u, const float* w_rec,
                     const float* d);
int dl_bn_get_params(dl_bn* ctx, float* e, float* u, float* w_rec, float* d);
/* RNQZ load path (read_quantized + dequantize_model, compress.hpp:481-523):
 * the four linearly quantised matrices e, u, w_rec, d (packed codes,
 * least-significant bit first, as in the file) are dequantised on the
 * device into the fp32 parameters. */
typedef struct dl_qmatrix {
  int bits;              /* 1..16 */
  float min, max;        /* QuantizedMatrix::min / max */
  const uint8_t* codes;  /* ceil(rows * cols * bits / 8) bytes */
} dl_qmatrix;
int dl_bn_set_params_quantized(dl_bn* ctx, const dl_qmatrix m[4]);
/* m_e [V], m_u [P x H], m_rec [H x H], m_d [H x P]; NULL = zeros */
int dl_bn_set_opt(dl_bn* ctx, const float* m_e, const float* m_u, const float* m_rec,
                  const float* m_d, double rho, double eps);
int dl_bn_get_opt(dl_bn* ctx, float* m_e, float* m_u, float* m_rec, float* m_d);
/* One softmax-mode window; arrays as dl_window. */
int dl_bn_window(dl_bn* ctx, int64_t T, int64_t B, const uint32_t* inputs,
                 const uint32_t* targets, const uint8_t* weights, const float* h0,
                 float* h_final, double loss_scale, float clip, int compute_grads,
                 double* loss, uint64_t* positions);
/* Clipped gradients of the last window: dense g_e [V x P], g_u, g_rec, g_d. */
int dl_bn_get_grads(dl_bn* ctx, float* g_e, float* g_u, float* g_rec, float* g_d);
/* *applied = 0 mirrors bottleneck_update returning false (non-finite). */
int dl_bn_rmsprop(dl_bn* ctx, double eta, int* applied);
/* dl_bn_window + dl_bn_rmsprop in one call. */
int dl_bn_train_window(dl_bn* ctx, int64_t T, int64_t B, const uint32_t* inputs,
                       const uint32_t* targets, const uint8_t* weights, const float* h0,
                       float* h_final, double loss_scale, float clip, double eta,
                       double* loss, uint64_t* positions, int* applied);
/* Trainer<BottleneckTraits>::run_epoch on the device (trainer.hpp:350-410
 * over compress.hpp:389-415), as dl_trainer_init / _run / _get_state /
 * _set_state: the stream and the offset-stream schedule (cursors
 * floor(i*L/N), hidden act(0)) live on the device; window w of a run is
 * group w % noffset, built, trained (loss_scale 1/(minibatch*unroll), clip)
 * and carried on the device (softmax windows replay one CUDA graph; NCE
 * windows draw their noise on the host in the reference's order).
 * dl_bn_trainer_run adds the windows' loss sum, target positions and
 * skipped (non-finite) updates to the outputs (any may be NULL). */
int dl_bn_trainer_init(dl_bn* ctx, const uint32_t* ids, int64_t L, int noffset, int minibatch,
                       int unroll, double clip, uint32_t bos);
int dl_bn_trainer_run(dl_bn* ctx, int64_t first, int64_t count, double eta, double* loss_sum,
                      uint64_t* positions, uint64_t* skipped);
/* cursors [noffset*minibatch], hidden [noffset*minibatch x H]; NULL skips */
int dl_bn_trainer_get_state(dl_bn* ctx, int64_t* cursors, float* hidden);
int dl_bn_trainer_set_state(dl_bn* ctx, const int64_t* cursors, const float* hidden);
int dl_bn_sharded_perplexity(dl_bn* ctx, const uint32_t* ids, int64_t n, int shards,
                             uint32_t bos, double* total_logprob, uint64_t* predicted,
                             double* perplexity);
/* Lock-step scorer over S streams, as dl_score (sharded_perplexity /
 * rnn_perplexity / rescore_nbest over the BottleneckAdapter, eval.hpp:84-222,
 * :693-790): per-token log-probs (NaN where tgt = -1), sums in (j, s) order. */
int dl_bn_score(dl_bn* ctx, int64_t S, int64_t steps, const uint32_t* in, const int64_t* tgt,
                const float* h0, float* h_final, double* logp, double* total_logprob,
                uint64_t* predicted);
/* NCE mode (LossMode::kNce) for the bottleneck model: as dl_set_loss_mode /
 * dl_set_noise / dl_{set,get}_rng_state of the standard model (the noise
 * model over E, sparse embedding gradient; backprop.hpp:126-156,
 * compress.hpp:204-225). */
int dl_bn_set_loss_mode(dl_bn* ctx, int mode);
int dl_bn_set_noise(dl_bn* ctx, const double* counts, int64_t V, int k, double floor);
int dl_bn_set_noise_dist(dl_bn* ctx, const double* q, int64_t V, int k);
int dl_bn_set_rng_state(dl_bn* ctx, const uint64_t state[313]);
int dl_bn_get_rng_state(const dl_bn* ctx, uint64_t state[313]);
uint64_t dl_bn_launch_count(const dl_bn* ctx);
void* dl_bn_cuda_stream(const dl_bn* ctx);

#ifdef __cplusplus
}
#endif

#endif /* DESKLM_CUDA_H */
