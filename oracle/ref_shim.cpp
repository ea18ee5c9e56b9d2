// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (never shipped, never timed
// as the product).
//
// A C-ABI shim that compiles the *unmodified* reference library
// (/root/reference/proj/include/desklm, header-only C++20) into
// oracle/_ref/libdesklm_ref.so so that Python tests can run the reference's
// own code on the same inputs the CUDA path sees.  No reference source is
// copied into this repository: the headers are pulled in with -I at build
// time by oracle/Makefile.  Every entry point below calls straight into the
// reference's public API:
//
//   ref_init_uniform      -> RnnParams<float>::init_uniform      rnn.hpp:79-83
//   ref_random_stream     -> testutil::random_stream             tests/oracles/helpers.hpp:36-52
//   ref_bptt              -> bptt_run(StandardAdapter<float>)    backprop.hpp:76-222
//   ref_rmsprop           -> rmsprop_update                      rmsprop.hpp:113-133
//   ref_sharded_ppl       -> sharded_perplexity                  eval.hpp:151-222
//   ref_rnn_ppl           -> rnn_perplexity                      eval.hpp:84-145
//   ref_sharded_logprobs  -> the sharded_perplexity loop, per token, built from
//                            the same primitives (matmul_nt, input_forward,
//                            activate, softmax_scores_t, lse_column)
//   ref_train             -> Trainer<StandardTraits>::train + save_checkpoint
//                                                                trainer.hpp:178-341
//   ref_write_params      -> write_params (RNLM)                 rnn.hpp:263-285
//   ref_write_rmsprop     -> write_rmsprop (ROPT)                rmsprop.hpp:139-149
//   ref_rescore           -> read_nbest + rescore_nbest + write_nbest
//                                                                eval.hpp:612-790
//
// Errors: C++ exceptions are caught and mapped to the same status codes the
// CUDA C-ABI uses (1 = std::invalid_argument, 2 = DataError, 3 = other).

#include <cstdint>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "desklm/desklm.hpp"
#include "oracles/helpers.hpp"

using namespace desklm;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

RnnParams<float> make_params(std::int64_t V, std::int64_t H, int act,
                             const float* w_in, const float* w_rec,
                             const float* w_out) {
  RnnParams<float> p(V, H, static_cast<Activation>(act));
  std::memcpy(p.w_in.a.data(), w_in, sizeof(float) * V * H);
  std::memcpy(p.w_rec.a.data(), w_rec, sizeof(float) * H * H);
  std::memcpy(p.w_out.a.data(), w_out, sizeof(float) * V * H);
  return p;
}

}  // namespace

extern "C" {

// Field order is the RTRN config echo order (trainer.hpp:412-432).
struct ref_train_config {
  std::int64_t nstate;
  std::int64_t nproj;
  std::int32_t noffset;
  std::int32_t minibatch;
  std::int32_t unroll;
  std::int32_t mode;  // 0 nce, 1 softmax
  double eta;
  double rho;
  double eps;
  double clip;
  std::int32_t nce_k;
  std::int32_t max_epochs;
  double noise_floor;
  std::uint64_t seed;
  std::int32_t act;
  std::int32_t valid_shards;
  double divergence_factor;
  std::int64_t valid_limit;
  double init_range;
  std::int32_t threads;
  std::int32_t pad_;
};

const char* ref_last_error() { return g_err.c_str(); }

int ref_init_uniform(std::int64_t V, std::int64_t H, std::uint64_t seed,
                     double range, float* w_in, float* w_rec, float* w_out) {
  return guarded([&] {
    RnnParams<float> p(V, H);
    p.init_uniform(seed, range);
    std::memcpy(w_in, p.w_in.a.data(), sizeof(float) * V * H);
    std::memcpy(w_rec, p.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(w_out, p.w_out.a.data(), sizeof(float) * V * H);
  });
}

// Writes up to `cap` ids; returns the full stream length (or -1 on error).
std::int64_t ref_random_stream(std::uint64_t seed, std::uint64_t v,
                               std::uint64_t min_tokens,
                               std::uint64_t max_sentence_len,
                               std::uint32_t* out, std::uint64_t cap) {
  std::int64_t n = -1;
  guarded([&] {
    std::mt19937_64 rng(seed);
    IdStream s = testutil::random_stream(rng, v, min_tokens, max_sentence_len);
    n = static_cast<std::int64_t>(s.ids.size());
    std::memcpy(out, s.ids.data(),
                sizeof(std::uint32_t) * std::min<std::uint64_t>(cap, s.ids.size()));
  });
  return n;
}

// Two consecutive random_stream draws from one generator, as the trainer
// tests do (train stream then valid stream, test_trainer.cpp:167-169).
int ref_random_stream_pair(std::uint64_t seed, std::uint64_t v,
                           std::uint64_t min_a, std::uint64_t min_b,
                           std::uint32_t* out_a, std::uint64_t cap_a,
                           std::int64_t* len_a, std::uint32_t* out_b,
                           std::uint64_t cap_b, std::int64_t* len_b) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    IdStream a = testutil::random_stream(rng, v, min_a);
    IdStream b = testutil::random_stream(rng, v, min_b);
    *len_a = static_cast<std::int64_t>(a.ids.size());
    *len_b = static_cast<std::int64_t>(b.ids.size());
    std::memcpy(out_a, a.ids.data(),
                sizeof(std::uint32_t) * std::min<std::uint64_t>(cap_a, a.ids.size()));
    std::memcpy(out_b, b.ids.data(),
                sizeof(std::uint32_t) * std::min<std::uint64_t>(cap_b, b.ids.size()));
  });
}

// mt19937_64 state as 312 words + position (the libstdc++ stream order).
static std::mt19937_64 rng_from(const std::uint64_t* st) {
  std::stringstream ss;
  for (int i = 0; i < 313; ++i) ss << st[i] << ' ';
  std::mt19937_64 r;
  ss >> r;
  return r;
}
static void rng_to(const std::mt19937_64& r, std::uint64_t* st) {
  std::stringstream ss;
  ss << r;
  for (int i = 0; i < 313; ++i) ss >> st[i];
}

void ref_mt_state(std::uint64_t seed, std::uint64_t* st) { rng_to(std::mt19937_64(seed), st); }

// NoiseModel(counts, k, floor) (nce.hpp:41-66): ln(k q) per word and n draws
// of its alias sampler from the given rng state (state updated in place).
int ref_noise_sample(std::int64_t V, const double* counts, int k, double floor,
                     std::uint64_t* rng, std::int64_t n, std::uint32_t* out,
                     double* ln_kq) {
  return guarded([&] {
    NoiseModel nm(std::vector<double>(counts, counts + V), k, floor);
    std::mt19937_64 r = rng_from(rng);
    for (std::int64_t i = 0; i < n; ++i) out[i] = nm.sample(r);
    for (std::int64_t w = 0; w < V; ++w) ln_kq[w] = nm.ln_kq(static_cast<WordId>(w));
    rng_to(r, rng);
  });
}

// One NCE-mode window (backprop.hpp:126-156).  The sparse W_out gradient
// rows come back in slot order like W_in's (g_out_words/g_out_data hold
// T*B*(k+1) rows).
int ref_bptt_nce(std::int64_t V, std::int64_t H, int act, const float* w_in,
                 const float* w_rec, const float* w_out, std::int64_t T, std::int64_t B,
                 const std::uint32_t* inputs, const std::uint32_t* targets,
                 const std::uint8_t* weights, const float* h0, double loss_scale, float clip,
                 int compute_grads, const double* counts, int k, double floor,
                 std::uint64_t* rng, float* h_final, std::int64_t* g_in_rows,
                 std::uint32_t* g_in_words, float* g_in_data, float* g_rec,
                 std::int64_t* g_out_rows, std::uint32_t* g_out_words, float* g_out_data,
                 double* loss, std::uint64_t* positions) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    WindowBatch wb;
    wb.resize(T, B);
    std::memcpy(wb.inputs.data(), inputs, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.targets.data(), targets, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.weights.data(), weights, T * B);
    Mat<float> h0m(B, H);
    std::memcpy(h0m.a.data(), h0, sizeof(float) * B * H);
    StandardAdapter<float> a(p);
    NoiseModel nm(std::vector<double>(counts, counts + V), k, floor);
    std::mt19937_64 r = rng_from(rng);
    BpttOptions<float> opt;
    opt.mode = LossMode::kNce;
    opt.noise = &nm;
    opt.rng = &r;
    opt.loss_scale = loss_scale;
    opt.clip = clip;
    opt.compute_grads = compute_grads != 0;
    StandardGrads<float> g;
    Mat<float> hf;
    const BpttResult res = bptt_run(a, wb, h0m, compute_grads ? &g : nullptr,
                                    h_final ? &hf : nullptr, opt);
    rng_to(r, rng);
    *loss = res.loss;
    *positions = res.positions;
    if (h_final) std::memcpy(h_final, hf.a.data(), sizeof(float) * B * H);
    if (compute_grads) {
      *g_in_rows = static_cast<std::int64_t>(g.w_in.rows());
      for (std::size_t s2 = 0; s2 < g.w_in.rows(); ++s2) g_in_words[s2] = g.w_in.words[s2];
      std::memcpy(g_in_data, g.w_in.data.data(), sizeof(float) * g.w_in.data.size());
      std::memcpy(g_rec, g.w_rec.a.data(), sizeof(float) * H * H);
      *g_out_rows = static_cast<std::int64_t>(g.w_out_sp.rows());
      for (std::size_t s2 = 0; s2 < g.w_out_sp.rows(); ++s2) g_out_words[s2] = g.w_out_sp.words[s2];
      std::memcpy(g_out_data, g.w_out_sp.data.data(), sizeof(float) * g.w_out_sp.data.size());
    }
  });
}

// One softmax-mode window.  Sparse W_in gradient is exported in the
// reference's slot order (first touch, t descending then b ascending).
// g_in_words/g_in_data must hold T*B rows; *g_in_rows receives the count.
int ref_bptt(std::int64_t V, std::int64_t H, int act, const float* w_in,
             const float* w_rec, const float* w_out, std::int64_t T,
             std::int64_t B, const std::uint32_t* inputs,
             const std::uint32_t* targets, const std::uint8_t* weights,
             const float* h0, double loss_scale, float clip,
             int compute_grads, int threads, float* h_final,
             std::int64_t* g_in_rows, std::uint32_t* g_in_words,
             float* g_in_data, float* g_rec, float* g_out, double* loss,
             std::uint64_t* positions) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    WindowBatch wb;
    wb.resize(T, B);
    std::memcpy(wb.inputs.data(), inputs, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.targets.data(), targets, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.weights.data(), weights, T * B);
    Mat<float> h0m(B, H);
    std::memcpy(h0m.a.data(), h0, sizeof(float) * B * H);
    StandardAdapter<float> a(p);
    BpttOptions<float> opt;
    opt.mode = LossMode::kSoftmax;
    opt.loss_scale = loss_scale;
    opt.clip = clip;
    opt.threads = threads;
    opt.compute_grads = compute_grads != 0;
    StandardGrads<float> g;
    Mat<float> hf;
    const BpttResult r = bptt_run(a, wb, h0m, compute_grads ? &g : nullptr,
                                  h_final ? &hf : nullptr, opt);
    *loss = r.loss;
    *positions = r.positions;
    if (h_final) std::memcpy(h_final, hf.a.data(), sizeof(float) * B * H);
    if (compute_grads) {
      *g_in_rows = static_cast<std::int64_t>(g.w_in.rows());
      for (std::size_t s = 0; s < g.w_in.rows(); ++s) g_in_words[s] = g.w_in.words[s];
      std::memcpy(g_in_data, g.w_in.data.data(), sizeof(float) * g.w_in.data.size());
      std::memcpy(g_rec, g.w_rec.a.data(), sizeof(float) * H * H);
      std::memcpy(g_out, g.w_out_dense.a.data(), sizeof(float) * V * H);
    }
  });
}

// rmsprop_update with a sparse W_in gradient (slot order as given) and a
// dense (out_dense=1) or sparse W_out gradient.  Returns the status code;
// *applied mirrors the reference's bool result.
int ref_rmsprop(std::int64_t V, std::int64_t H, float* w_in, float* w_rec,
                float* w_out, float* m_rec, float* m_in, float* m_out,
                double rho, double eps, double eta, std::int64_t n_in_rows,
                const std::uint32_t* in_words, const float* in_data,
                const float* g_rec, int out_dense, std::int64_t n_out_rows,
                const std::uint32_t* out_words, const float* out_data,
                int* applied) {
  return guarded([&] {
    RnnParams<float> p = make_params(V, H, 0, w_in, w_rec, w_out);
    RmspropState s(V, H, rho, eps);
    std::memcpy(s.m_rec.a.data(), m_rec, sizeof(float) * H * H);
    std::memcpy(s.m_in.data(), m_in, sizeof(float) * V);
    std::memcpy(s.m_out.data(), m_out, sizeof(float) * V);
    StandardGrads<float> g;
    StandardAdapter<float> a(p);
    a.grads_reset(g, out_dense != 0);
    for (std::int64_t r = 0; r < n_in_rows; ++r)
      g.w_in.axpy_row(in_words[r], 1.0f, in_data + r * H);
    std::memcpy(g.w_rec.a.data(), g_rec, sizeof(float) * H * H);
    if (out_dense) {
      std::memcpy(g.w_out_dense.a.data(), out_data, sizeof(float) * V * H);
    } else {
      for (std::int64_t r = 0; r < n_out_rows; ++r)
        g.w_out_sp.axpy_row(out_words[r], 1.0f, out_data + r * H);
    }
    *applied = rmsprop_update(p, g, s, eta) ? 1 : 0;
    std::memcpy(w_in, p.w_in.a.data(), sizeof(float) * V * H);
    std::memcpy(w_rec, p.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(w_out, p.w_out.a.data(), sizeof(float) * V * H);
    std::memcpy(m_rec, s.m_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(m_in, s.m_in.data(), sizeof(float) * V);
    std::memcpy(m_out, s.m_out.data(), sizeof(float) * V);
  });
}

int ref_sharded_ppl(std::int64_t V, std::int64_t H, int act, const float* w_in,
                    const float* w_rec, const float* w_out,
                    const std::uint32_t* ids, std::int64_t n, int shards,
                    std::uint32_t bos, int threads, double* total_logprob,
                    std::uint64_t* predicted, double* ppl) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    IdStream s;
    s.ids.assign(ids, ids + n);
    StandardAdapter<float> a(p);
    const PerplexityResult r = sharded_perplexity(a, s, shards, bos, threads);
    *total_logprob = r.total_logprob;
    *predicted = r.predicted;
    *ppl = r.perplexity;
  });
}

int ref_rnn_ppl(std::int64_t V, std::int64_t H, int act, const float* w_in,
                const float* w_rec, const float* w_out, const std::uint32_t* ids,
                std::int64_t n, std::uint32_t bos, int threads,
                double* total_logprob, std::uint64_t* predicted, double* ppl) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    IdStream s;
    s.ids.assign(ids, ids + n);
    StandardAdapter<float> a(p);
    const PerplexityResult r = rnn_perplexity(a, s, bos, threads);
    *total_logprob = r.total_logprob;
    *predicted = r.predicted;
    *ppl = r.perplexity;
  });
}

// Per-token log-probabilities of the sharded walk (eval.hpp:151-222):
// out[j*S + s] = ln p(tgt | history) or NaN where the target is skipped.
// out must hold (max_len-1)*S doubles; *S_out / *steps_out report the shape.
int ref_sharded_logprobs(std::int64_t V, std::int64_t H, int act,
                         const float* w_in, const float* w_rec,
                         const float* w_out, const std::uint32_t* ids,
                         std::int64_t n, int shards, std::uint32_t bos,
                         double* out, std::int64_t cap, std::int64_t* S_out,
                         std::int64_t* steps_out) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    StandardAdapter<float> model(p);
    const std::int64_t S = std::min<std::int64_t>(shards, n / 2);
    if (S < 1) throw std::invalid_argument("sharded logprobs: stream too short");
    std::vector<std::int64_t> begin(S + 1);
    for (std::int64_t s = 0; s <= S; ++s) begin[s] = s * n / S;
    std::int64_t max_len = 0;
    for (std::int64_t s = 0; s < S; ++s)
      max_len = std::max(max_len, begin[s + 1] - begin[s]);
    *S_out = S;
    *steps_out = max_len - 1;
    if ((max_len - 1) * S > cap) throw std::invalid_argument("sharded logprobs: cap");
    const float a0 = activate(p.act, 0.0f);
    Mat<float> h(S, H), pre(S, H), scores_t(V, S);
    h.fill(a0);
    std::vector<WordId> in(S, 0);
    std::vector<std::int64_t> tgt(S, -1);
    for (std::int64_t j = 0; j + 1 < max_len; ++j) {
      for (std::int64_t s = 0; s < S; ++s) {
        const std::int64_t len = begin[s + 1] - begin[s];
        if (j + 1 < len) {
          const WordId x = ids[begin[s] + j];
          const WordId y = ids[begin[s] + j + 1];
          in[s] = x;
          tgt[s] = y == bos ? -1 : static_cast<std::int64_t>(y);
        } else {
          in[s] = 0;
          tgt[s] = -1;
        }
      }
      matmul_nt<double>(h, p.w_rec, pre, false, 1);
      model.input_forward(in, pre, 1);
      for (std::int64_t s = 0; s < S; ++s)
        for (std::int64_t i = 0; i < H; ++i)
          h.at(s, i) = activate(p.act, pre.at(s, i));
      StandardAdapter<float>::OutCtx octx{};
      model.softmax_scores_t(octx, h, scores_t, 1);
      for (std::int64_t s = 0; s < S; ++s) {
        double v = std::numeric_limits<double>::quiet_NaN();
        if (tgt[s] >= 0)
          v = static_cast<double>(scores_t.at(tgt[s], s)) -
              detail::lse_column(scores_t, s);
        out[j * S + s] = v;
      }
    }
  });
}

// Runs Trainer<StandardTraits> for cfg->max_epochs (with early stopping as
// the reference does) on a make_vocab(V) vocabulary; returns the RTRN
// checkpoint bytes and the epoch logs (7 doubles per epoch: epoch,
// train_loss, valid_ppl, eta, seconds, tokens_per_sec, skipped).
}  // extern "C"

namespace {

TrainConfig to_cfg(const ref_train_config* c) {
  TrainConfig cfg;
  cfg.nstate = c->nstate;
  cfg.nproj = c->nproj;
  cfg.noffset = c->noffset;
  cfg.minibatch = c->minibatch;
  cfg.unroll = c->unroll;
  cfg.mode = static_cast<LossMode>(c->mode);
  cfg.eta = c->eta;
  cfg.rho = c->rho;
  cfg.eps = c->eps;
  cfg.clip = c->clip;
  cfg.nce_k = c->nce_k;
  cfg.max_epochs = c->max_epochs;
  cfg.noise_floor = c->noise_floor;
  cfg.seed = c->seed;
  cfg.act = static_cast<Activation>(c->act);
  cfg.valid_shards = c->valid_shards;
  cfg.divergence_factor = c->divergence_factor;
  cfg.valid_limit = c->valid_limit;
  cfg.init_range = c->init_range;
  cfg.threads = c->threads;
  return cfg;
}

// Trainer<Traits>::train + save_checkpoint; logs as 7 doubles per epoch.
template <class Traits>
void run_trainer(const TrainConfig& cfg, const typename Traits::Params& p, std::int64_t V,
                 const std::uint32_t* train_ids, std::int64_t n_train,
                 const std::uint32_t* valid_ids, std::int64_t n_valid, int run_epochs,
                 std::uint8_t* ckpt, std::uint64_t cap, std::uint64_t* ckpt_len, double* logs,
                 int* n_logs, double* initial_ppl) {
  IdStream tr, va;
  tr.ids.assign(train_ids, train_ids + n_train);
  va.ids.assign(valid_ids, valid_ids + n_valid);
  Trainer<Traits> t(cfg, p, testutil::make_vocab(V), tr, va);
  if (run_epochs) t.train(nullptr);
  std::ostringstream os(std::ios::binary);
  t.save_checkpoint(os);
  const std::string b = os.str();
  *ckpt_len = b.size();
  if (b.size() <= cap) std::memcpy(ckpt, b.data(), b.size());
  *n_logs = static_cast<int>(t.logs().size());
  for (std::size_t i = 0; i < t.logs().size(); ++i) {
    const EpochLog& l = t.logs()[i];
    double* o = logs + 7 * i;
    o[0] = l.epoch;
    o[1] = l.train_loss;
    o[2] = l.valid_ppl;
    o[3] = l.eta;
    o[4] = l.seconds;
    o[5] = l.tokens_per_sec;
    o[6] = static_cast<double>(l.skipped_updates);
  }
  *initial_ppl = t.initial_ppl();
}

}  // namespace

extern "C" {

int ref_train(const ref_train_config* c, std::int64_t V, const float* w_in,
              const float* w_rec, const float* w_out,
              const std::uint32_t* train_ids, std::int64_t n_train,
              const std::uint32_t* valid_ids, std::int64_t n_valid,
              int run_epochs, std::uint8_t* ckpt, std::uint64_t cap,
              std::uint64_t* ckpt_len, double* logs, int* n_logs,
              double* initial_ppl) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, c->nstate, c->act, w_in, w_rec, w_out);
    run_trainer<StandardTraits>(to_cfg(c), p, V, train_ids, n_train, valid_ids, n_valid,
                                run_epochs, ckpt, cap, ckpt_len, logs, n_logs, initial_ppl);
  });
}

// Trainer<BottleneckTraits> (compress.hpp:389-415; test_compress.cpp:427-460).
int ref_bn_train(const ref_train_config* c, std::int64_t V, std::int64_t P, const float* e,
                 const float* u, const float* w_rec, const float* d,
                 const std::uint32_t* train_ids, std::int64_t n_train,
                 const std::uint32_t* valid_ids, std::int64_t n_valid, int run_epochs,
                 std::uint8_t* ckpt, std::uint64_t cap, std::uint64_t* ckpt_len, double* logs,
                 int* n_logs, double* initial_ppl) {
  return guarded([&] {
    BottleneckParams<float> p(V, c->nstate, P, static_cast<Activation>(c->act));
    std::memcpy(p.e.a.data(), e, sizeof(float) * V * P);
    std::memcpy(p.u.a.data(), u, sizeof(float) * P * c->nstate);
    std::memcpy(p.w_rec.a.data(), w_rec, sizeof(float) * c->nstate * c->nstate);
    std::memcpy(p.d.a.data(), d, sizeof(float) * c->nstate * P);
    run_trainer<BottleneckTraits>(to_cfg(c), p, V, train_ids, n_train, valid_ids, n_valid,
                                  run_epochs, ckpt, cap, ckpt_len, logs, n_logs, initial_ppl);
  });
}

// RNLM bytes for params over make_vocab(V).
int ref_write_params(std::int64_t V, std::int64_t H, int act, const float* w_in,
                     const float* w_rec, const float* w_out, std::uint8_t* buf,
                     std::uint64_t cap, std::uint64_t* len) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    std::ostringstream os(std::ios::binary);
    write_params(os, p, testutil::make_vocab(V));
    const std::string b = os.str();
    *len = b.size();
    if (b.size() <= cap) std::memcpy(buf, b.data(), b.size());
  });
}

int ref_write_rmsprop(std::int64_t V, std::int64_t H, double rho, double eps,
                      const float* m_rec, const float* m_in, const float* m_out,
                      std::uint8_t* buf, std::uint64_t cap, std::uint64_t* len) {
  return guarded([&] {
    RmspropState s(V, H, rho, eps);
    std::memcpy(s.m_rec.a.data(), m_rec, sizeof(float) * H * H);
    std::memcpy(s.m_in.data(), m_in, sizeof(float) * V);
    std::memcpy(s.m_out.data(), m_out, sizeof(float) * V);
    std::ostringstream os(std::ios::binary);
    write_rmsprop(os, s);
    const std::string b = os.str();
    *len = b.size();
    if (b.size() <= cap) std::memcpy(buf, b.data(), b.size());
  });
}

// n-best rescoring (RNN only, exact or fast) over make_vocab(V) words.
// Input/output are the reference's tab-separated text formats.
int ref_rescore(std::int64_t V, std::int64_t H, int act, const float* w_in,
                const float* w_rec, const float* w_out, const char* nbest_text,
                double lm_scale, double wip, int fast, char* out,
                std::uint64_t cap, std::uint64_t* len) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    std::istringstream is(nbest_text);
    auto utts = read_nbest(is);
    RescoreConfig rc;
    rc.lambda = 1.0;
    rc.lm_scale = lm_scale;
    rc.wip = wip;
    rc.fast = fast != 0;
    StandardAdapter<float> a(p);
    rescore_nbest(utts, a, testutil::make_vocab(V), nullptr, rc);
    std::ostringstream os;
    write_nbest(os, utts);
    const std::string b = os.str();
    *len = b.size();
    if (b.size() + 1 <= cap) std::memcpy(out, b.c_str(), b.size() + 1);
  });
}

// ----- bottleneck model (compress.hpp) -----
//   ref_bn_init_uniform   -> BottleneckParams<float>::init_uniform  compress.hpp:78-82
//   ref_bn_bptt           -> bptt_run(BottleneckAdapter<float>)     backprop.hpp:76-222
//   ref_bn_update         -> bottleneck_update                      compress.hpp:296-309
//   ref_bn_sharded_ppl    -> sharded_perplexity(BottleneckAdapter)  eval.hpp:151-222
//   ref_bn_write          -> write_bottleneck + write_bottleneck_opt compress.hpp:315-368

static BottleneckParams<float> make_bn(std::int64_t V, std::int64_t H, std::int64_t P, int act,
                                       const float* e, const float* u, const float* w_rec,
                                       const float* d) {
  BottleneckParams<float> p(V, H, P, static_cast<Activation>(act));
  std::memcpy(p.e.a.data(), e, sizeof(float) * V * P);
  std::memcpy(p.u.a.data(), u, sizeof(float) * P * H);
  std::memcpy(p.w_rec.a.data(), w_rec, sizeof(float) * H * H);
  std::memcpy(p.d.a.data(), d, sizeof(float) * H * P);
  return p;
}

int ref_bn_init_uniform(std::int64_t V, std::int64_t H, std::int64_t P, std::uint64_t seed,
                        double range, float* e, float* u, float* w_rec, float* d) {
  return guarded([&] {
    BottleneckParams<float> p(V, H, P);
    p.init_uniform(seed, range);
    std::memcpy(e, p.e.a.data(), sizeof(float) * V * P);
    std::memcpy(u, p.u.a.data(), sizeof(float) * P * H);
    std::memcpy(w_rec, p.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(d, p.d.a.data(), sizeof(float) * H * P);
  });
}

int ref_bn_bptt(std::int64_t V, std::int64_t H, std::int64_t P, int act, const float* e,
                const float* u, const float* w_rec, const float* d, std::int64_t T,
                std::int64_t B, const std::uint32_t* inputs, const std::uint32_t* targets,
                const std::uint8_t* weights, const float* h0, double loss_scale, float clip,
                int compute_grads, float* h_final, float* g_e, float* g_u, float* g_rec,
                float* g_d, double* loss, std::uint64_t* positions) {
  return guarded([&] {
    const BottleneckParams<float> p = make_bn(V, H, P, act, e, u, w_rec, d);
    WindowBatch wb;
    wb.resize(T, B);
    std::memcpy(wb.inputs.data(), inputs, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.targets.data(), targets, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.weights.data(), weights, T * B);
    Mat<float> h0m(B, H);
    std::memcpy(h0m.a.data(), h0, sizeof(float) * B * H);
    BottleneckAdapter<float> a(p);
    BpttOptions<float> opt;
    opt.mode = LossMode::kSoftmax;
    opt.loss_scale = loss_scale;
    opt.clip = clip;
    opt.compute_grads = compute_grads != 0;
    BottleneckGrads<float> g;
    Mat<float> hf;
    const BpttResult res = bptt_run(a, wb, h0m, compute_grads ? &g : nullptr,
                                    h_final ? &hf : nullptr, opt);
    *loss = res.loss;
    *positions = res.positions;
    if (h_final) std::memcpy(h_final, hf.a.data(), sizeof(float) * B * H);
    if (compute_grads) {
      std::memcpy(g_e, g.e_dense.a.data(), sizeof(float) * V * P);
      std::memcpy(g_u, g.u.a.data(), sizeof(float) * P * H);
      std::memcpy(g_rec, g.w_rec.a.data(), sizeof(float) * H * H);
      std::memcpy(g_d, g.d.a.data(), sizeof(float) * H * P);
    }
  });
}

int ref_bn_update(std::int64_t V, std::int64_t H, std::int64_t P, float* e, float* u,
                  float* w_rec, float* d, float* m_e, float* m_u, float* m_rec, float* m_d,
                  double rho, double eps, double eta, const float* g_e, const float* g_u,
                  const float* g_rec, const float* g_d, int* applied) {
  return guarded([&] {
    BottleneckParams<float> p = make_bn(V, H, P, 0, e, u, w_rec, d);
    BottleneckOptState s(V, H, P, rho, eps);
    std::memcpy(s.m_e.data(), m_e, sizeof(float) * V);
    std::memcpy(s.m_u.a.data(), m_u, sizeof(float) * P * H);
    std::memcpy(s.m_rec.a.data(), m_rec, sizeof(float) * H * H);
    std::memcpy(s.m_d.a.data(), m_d, sizeof(float) * H * P);
    BottleneckGrads<float> g;
    g.e_is_dense = true;
    g.e_dense = Mat<float>(V, P);
    g.u = Mat<float>(P, H);
    g.w_rec = Mat<float>(H, H);
    g.d = Mat<float>(H, P);
    std::memcpy(g.e_dense.a.data(), g_e, sizeof(float) * V * P);
    std::memcpy(g.u.a.data(), g_u, sizeof(float) * P * H);
    std::memcpy(g.w_rec.a.data(), g_rec, sizeof(float) * H * H);
    std::memcpy(g.d.a.data(), g_d, sizeof(float) * H * P);
    *applied = bottleneck_update(p, g, s, eta) ? 1 : 0;
    std::memcpy(e, p.e.a.data(), sizeof(float) * V * P);
    std::memcpy(u, p.u.a.data(), sizeof(float) * P * H);
    std::memcpy(w_rec, p.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(d, p.d.a.data(), sizeof(float) * H * P);
    std::memcpy(m_e, s.m_e.data(), sizeof(float) * V);
    std::memcpy(m_u, s.m_u.a.data(), sizeof(float) * P * H);
    std::memcpy(m_rec, s.m_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(m_d, s.m_d.a.data(), sizeof(float) * H * P);
  });
}

int ref_bn_sharded_ppl(std::int64_t V, std::int64_t H, std::int64_t P, int act, const float* e,
                       const float* u, const float* w_rec, const float* d,
                       const std::uint32_t* ids, std::int64_t n, int shards, std::uint32_t bos,
                       double* total_logprob, std::uint64_t* predicted, double* ppl) {
  return guarded([&] {
    const BottleneckParams<float> p = make_bn(V, H, P, act, e, u, w_rec, d);
    IdStream st;
    st.ids.assign(ids, ids + n);
    BottleneckAdapter<float> a(p);
    const PerplexityResult r = sharded_perplexity(a, st, shards, bos);
    *total_logprob = r.total_logprob;
    *predicted = r.predicted;
    *ppl = r.perplexity;
  });
}

// RNBL (params + vocabulary "w<i>") followed by RBOP, as two byte strings
// concatenated: *len_params gives the split.
int ref_bn_write(std::int64_t V, std::int64_t H, std::int64_t P, int act, const float* e,
                 const float* u, const float* w_rec, const float* d, double rho, double eps,
                 const float* m_e, const float* m_u, const float* m_rec, const float* m_d,
                 std::uint8_t* buf, std::uint64_t cap, std::uint64_t* len_params,
                 std::uint64_t* len) {
  return guarded([&] {
    const BottleneckParams<float> p = make_bn(V, H, P, act, e, u, w_rec, d);
    std::ostringstream os(std::ios::binary);
    write_bottleneck(os, p, testutil::make_vocab(V));
    *len_params = os.str().size();
    BottleneckOptState s(V, H, P, rho, eps);
    std::memcpy(s.m_e.data(), m_e, sizeof(float) * V);
    std::memcpy(s.m_u.a.data(), m_u, sizeof(float) * P * H);
    std::memcpy(s.m_rec.a.data(), m_rec, sizeof(float) * H * H);
    std::memcpy(s.m_d.a.data(), m_d, sizeof(float) * H * P);
    write_bottleneck_opt(os, s);
    const std::string b = os.str();
    *len = b.size();
    if (b.size() <= cap) std::memcpy(buf, b.data(), b.size());
  });
}

// bptt_run(BottleneckAdapter) in NCE mode; the sparse embedding gradient in
// SparseRowGrads slot order (g_e_words / g_e_data hold T*B*(k+2) rows).
int ref_bn_bptt_nce(std::int64_t V, std::int64_t H, std::int64_t P, int act, const float* e,
                    const float* u, const float* w_rec, const float* d, std::int64_t T,
                    std::int64_t B, const std::uint32_t* inputs, const std::uint32_t* targets,
                    const std::uint8_t* weights, const float* h0, double loss_scale, float clip,
                    int compute_grads, const double* counts, int k, double floor,
                    std::uint64_t* rng, float* h_final, std::int64_t* g_e_rows,
                    std::uint32_t* g_e_words, float* g_e_data, float* g_u, float* g_rec,
                    float* g_d, double* loss, std::uint64_t* positions) {
  return guarded([&] {
    const BottleneckParams<float> p = make_bn(V, H, P, act, e, u, w_rec, d);
    WindowBatch wb;
    wb.resize(T, B);
    std::memcpy(wb.inputs.data(), inputs, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.targets.data(), targets, sizeof(std::uint32_t) * T * B);
    std::memcpy(wb.weights.data(), weights, T * B);
    Mat<float> h0m(B, H);
    std::memcpy(h0m.a.data(), h0, sizeof(float) * B * H);
    BottleneckAdapter<float> a(p);
    NoiseModel nm(std::vector<double>(counts, counts + V), k, floor);
    std::mt19937_64 r = rng_from(rng);
    BpttOptions<float> opt;
    opt.mode = LossMode::kNce;
    opt.noise = &nm;
    opt.rng = &r;
    opt.loss_scale = loss_scale;
    opt.clip = clip;
    opt.compute_grads = compute_grads != 0;
    BottleneckGrads<float> g;
    Mat<float> hf;
    const BpttResult res = bptt_run(a, wb, h0m, compute_grads ? &g : nullptr,
                                    h_final ? &hf : nullptr, opt);
    rng_to(r, rng);
    *loss = res.loss;
    *positions = res.positions;
    if (h_final) std::memcpy(h_final, hf.a.data(), sizeof(float) * B * H);
    if (compute_grads) {
      *g_e_rows = static_cast<std::int64_t>(g.e_sp.rows());
      for (std::size_t s2 = 0; s2 < g.e_sp.rows(); ++s2) g_e_words[s2] = g.e_sp.words[s2];
      std::memcpy(g_e_data, g.e_sp.data.data(), sizeof(float) * g.e_sp.data.size());
      std::memcpy(g_u, g.u.a.data(), sizeof(float) * P * H);
      std::memcpy(g_rec, g.w_rec.a.data(), sizeof(float) * H * H);
      std::memcpy(g_d, g.d.a.data(), sizeof(float) * H * P);
    }
  });
}

// bottleneck_update with a sparse embedding gradient.
int ref_bn_update_sparse(std::int64_t V, std::int64_t H, std::int64_t P, float* e, float* u,
                         float* w_rec, float* d, float* m_e, float* m_u, float* m_rec,
                         float* m_d, double rho, double eps, double eta, std::int64_t n_rows,
                         const std::uint32_t* words, const float* rows, const float* g_u,
                         const float* g_rec, const float* g_d, int* applied) {
  return guarded([&] {
    BottleneckParams<float> p = make_bn(V, H, P, 0, e, u, w_rec, d);
    BottleneckOptState s(V, H, P, rho, eps);
    std::memcpy(s.m_e.data(), m_e, sizeof(float) * V);
    std::memcpy(s.m_u.a.data(), m_u, sizeof(float) * P * H);
    std::memcpy(s.m_rec.a.data(), m_rec, sizeof(float) * H * H);
    std::memcpy(s.m_d.a.data(), m_d, sizeof(float) * H * P);
    BottleneckGrads<float> g;
    g.e_is_dense = false;
    g.e_sp.reset(P);
    for (std::int64_t i = 0; i < n_rows; ++i) g.e_sp.axpy_row(words[i], 1.0f, rows + i * P);
    g.u = Mat<float>(P, H);
    g.w_rec = Mat<float>(H, H);
    g.d = Mat<float>(H, P);
    std::memcpy(g.u.a.data(), g_u, sizeof(float) * P * H);
    std::memcpy(g.w_rec.a.data(), g_rec, sizeof(float) * H * H);
    std::memcpy(g.d.a.data(), g_d, sizeof(float) * H * P);
    *applied = bottleneck_update(p, g, s, eta) ? 1 : 0;
    std::memcpy(e, p.e.a.data(), sizeof(float) * V * P);
    std::memcpy(u, p.u.a.data(), sizeof(float) * P * H);
    std::memcpy(w_rec, p.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(d, p.d.a.data(), sizeof(float) * H * P);
    std::memcpy(m_e, s.m_e.data(), sizeof(float) * V);
    std::memcpy(m_u, s.m_u.a.data(), sizeof(float) * P * H);
    std::memcpy(m_rec, s.m_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(m_d, s.m_d.a.data(), sizeof(float) * H * P);
  });
}

// ln_z_samples(StandardAdapter) + drift_stats (eval.hpp:805-880); stats =
// {mean, median, q25, q75, iqr, contexts} (only when >= 100 samples).
int ref_ln_z_samples(std::int64_t V, std::int64_t H, int act, const float* w_in,
                     const float* w_rec, const float* w_out, const std::uint32_t* ids,
                     std::int64_t n, std::int64_t count, double* out, std::int64_t* n_out,
                     double* stats) {
  return guarded([&] {
    const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
    IdStream st;
    st.ids.assign(ids, ids + n);
    StandardAdapter<float> a(p);
    const std::vector<double> z = ln_z_samples(a, st, static_cast<std::size_t>(count));
    *n_out = static_cast<std::int64_t>(z.size());
    std::memcpy(out, z.data(), sizeof(double) * z.size());
    if (z.size() >= 100) {
      const DriftStats d = drift_stats(z);
      stats[0] = d.mean;
      stats[1] = d.median;
      stats[2] = d.q25;
      stats[3] = d.q75;
      stats[4] = d.iqr;
      stats[5] = static_cast<double>(d.contexts);
    }
  });
}

// quantize_model + write_quantized (RNQZ) of a bottleneck model, and the
// dequantize_model round trip (compress.hpp:417-621).
int ref_bn_quantize(std::int64_t V, std::int64_t H, std::int64_t P, int act, const float* e,
                    const float* u, const float* w_rec, const float* d, int bits,
                    std::uint8_t* buf, std::uint64_t cap, std::uint64_t* len, float* de,
                    float* du, float* dw_rec, float* dd) {
  return guarded([&] {
    const BottleneckParams<float> p = make_bn(V, H, P, act, e, u, w_rec, d);
    const QuantizedModel q = quantize_model(p, testutil::make_vocab(V), bits);
    std::ostringstream os(std::ios::binary);
    write_quantized(os, q);
    const std::string b = os.str();
    *len = b.size();
    if (b.size() != quantized_size_bytes(q)) throw std::runtime_error("size mismatch");
    if (b.size() <= cap) std::memcpy(buf, b.data(), b.size());
    std::istringstream is(b);
    auto [p2, v2] = dequantize_model(read_quantized(is));
    std::memcpy(de, p2.e.a.data(), sizeof(float) * V * P);
    std::memcpy(du, p2.u.a.data(), sizeof(float) * P * H);
    std::memcpy(dw_rec, p2.w_rec.a.data(), sizeof(float) * H * H);
    std::memcpy(dd, p2.d.a.data(), sizeof(float) * H * P);
  });
}

// ----- n-gram side of the interpolation / hit-rate scorers (ngram.hpp,
// eval.hpp:231-592) -----
//   ref_ngram_query   count_ngrams + estimate_kn over a training stream
//                     (make_vocab(V)), then logprob(ctx, w) for each query
//                     (contexts: ctx_len ids each, -1 padded on the left) and
//                     shortlist(ctx, k) per context
//   ref_interp_terms  interpolation_terms + tune_lambda (RNN vocabulary
//                     make_vocab(Vr), n-gram vocabulary make_vocab(Vf))
//   ref_hit_rate      hit_rate with RnnHitScorer (kind 0) or NgramHitScorer (1)

static NGramModel build_ngram(const std::uint32_t* train, std::int64_t n_train, std::int64_t V,
                              int order) {
  IdStream tr;
  tr.ids.assign(train, train + n_train);
  return estimate_kn(count_ngrams(tr, order), testutil::make_vocab(V));
}

int ref_ngram_query(const std::uint32_t* train, std::int64_t n_train, std::int64_t V, int order,
                    std::int64_t nq, int ctx_len, const std::int64_t* ctx,
                    const std::uint32_t* words, double* logp, int k, std::uint32_t* shortlists,
                    const std::uint32_t* eval, std::int64_t n_eval, double* ppl) {
  return guarded([&] {
    const NGramModel m = build_ngram(train, n_train, V, order);
    for (std::int64_t q = 0; q < nq; ++q) {
      std::vector<WordId> c;
      for (int i = 0; i < ctx_len; ++i)
        if (ctx[q * ctx_len + i] >= 0) c.push_back(static_cast<WordId>(ctx[q * ctx_len + i]));
      logp[q] = m.logprob(c, words[q]);
      const std::vector<WordId> sl = m.shortlist(c, static_cast<std::size_t>(k));
      for (int i = 0; i < k; ++i)
        shortlists[q * k + i] = i < (int)sl.size() ? sl[i] : 0xffffffffu;
    }
    IdStream ev;
    ev.ids.assign(eval, eval + n_eval);
    const PerplexityResult r = ngram_perplexity_full(m, ev);
    ppl[0] = r.total_logprob;
    ppl[1] = static_cast<double>(r.predicted);
    ppl[2] = r.perplexity;
  });
}

int ref_interp_terms(std::int64_t Vr, std::int64_t H, int act, const float* w_in,
                     const float* w_rec, const float* w_out, std::int64_t Vf,
                     const std::uint32_t* train, std::int64_t n_train, int order,
                     const std::uint32_t* eval, std::int64_t n_eval, double* a, double* b,
                     std::int64_t* n_terms, double* lambda_ppl) {
  return guarded([&] {
    const RnnParams<float> p = make_params(Vr, H, act, w_in, w_rec, w_out);
    StandardAdapter<float> ad(p);
    const NGramModel m = build_ngram(train, n_train, Vf, order);
    const VocabMap map = make_vocab_map(testutil::make_vocab(Vr), testutil::make_vocab(Vf));
    IdStream ev;
    ev.ids.assign(eval, eval + n_eval);
    const std::vector<InterpTerm> t = interpolation_terms(ad, map, m, ev);
    *n_terms = static_cast<std::int64_t>(t.size());
    for (std::size_t i = 0; i < t.size(); ++i) {
      a[i] = t[i].a;
      b[i] = t[i].b;
    }
    double best = 0.0;
    lambda_ppl[0] = tune_lambda(t, &best);
    lambda_ppl[1] = best;
  });
}

int ref_hit_rate(std::int64_t V, std::int64_t H, int act, const float* w_in, const float* w_rec,
                 const float* w_out, const std::uint32_t* train, std::int64_t n_train, int order,
                 const std::uint32_t* eval, std::int64_t n_eval, int shortlist_k, int top_k,
                 int kind, std::uint64_t* positions, std::uint64_t* hits) {
  return guarded([&] {
    const NGramModel m = build_ngram(train, n_train, V, order);
    IdStream ev;
    ev.ids.assign(eval, eval + n_eval);
    HitRateResult r;
    if (kind == 0) {
      const RnnParams<float> p = make_params(V, H, act, w_in, w_rec, w_out);
      StandardAdapter<float> ad(p);
      RnnHitScorer<StandardAdapter<float>> sc(ad);
      r = hit_rate(ev, m, static_cast<std::size_t>(shortlist_k),
                   static_cast<std::size_t>(top_k), sc);
    } else {
      NgramHitScorer sc(m);
      r = hit_rate(ev, m, static_cast<std::size_t>(shortlist_k),
                   static_cast<std::size_t>(top_k), sc);
    }
    *positions = r.positions;
    *hits = r.hits;
  });
}

// The SURVEY §8d C1 PPL-match corpus: TextGenerator(GenConfig{}, gen_seed)
// text -> normalize_text -> build_vocab(train, V) -> encode (train and
// valid under the train vocabulary).
int ref_gen_corpus(std::uint64_t gen_seed, std::int64_t train_tokens, std::uint64_t train_seed,
                   std::int64_t valid_tokens, std::uint64_t valid_seed, std::int64_t V,
                   std::uint32_t* out_train, std::int64_t cap_train, std::int64_t* n_train,
                   std::uint32_t* out_valid, std::int64_t cap_valid, std::int64_t* n_valid) {
  return guarded([&] {
    TextGenerator gen(GenConfig{}, gen_seed);
    const SentenceCorpus tr = normalize_text(gen.generate(train_tokens, train_seed));
    const SentenceCorpus va = normalize_text(gen.generate(valid_tokens, valid_seed));
    const Vocabulary vocab = build_vocab(tr, static_cast<std::size_t>(V));
    const IdStream a = encode(tr, vocab), b = encode(va, vocab);
    *n_train = static_cast<std::int64_t>(a.ids.size());
    *n_valid = static_cast<std::int64_t>(b.ids.size());
    std::memcpy(out_train, a.ids.data(), sizeof(std::uint32_t) * std::min<std::int64_t>(*n_train, cap_train));
    std::memcpy(out_valid, b.ids.data(), sizeof(std::uint32_t) * std::min<std::int64_t>(*n_valid, cap_valid));
  });
}

}  // extern "C"
