// desklm_b200/traits.hpp -- the B200 model family for the reference's own
// desklm::Trainer<Traits>, scorers and CLI dispatch.
//
// Include after the reference headers are on the include path
// (-I /root/reference/proj/include): this header plugs the device path into
// the reference's plug-in seams instead of mirroring them:
//
//   Traits concept  trainer.hpp:117-156   -> GpuStandardTraits / GpuBottleneckTraits
//   Adapter seam    rnn.hpp:174-259       -> GpuAdapter / GpuBottleneckAdapter
//   bptt_run        backprop.hpp:76-222   -> bptt_run(const GpuAdapter&, ...) overloads
//   sharded_perplexity / rnn_perplexity    eval.hpp:84-222  -> overloads
//   rescore_nbest   eval.hpp:693-790      -> overloads (all hypotheses as lock-step streams)
//   with_model      tools/desklm.cpp:142-163 -> with_gpu_model (RNLM / RNBL / RNQZ)
//
// so that, unchanged,
//
//   desklm::Trainer<desklm::b200::GpuStandardTraits> tr(
//       cfg, desklm::b200::GpuParams(p0, desklm::b200::Precision::kBf16), vocab, train, valid);
//   tr.train(&std::cerr);  tr.save_checkpoint(path);  tr.load_checkpoint(path);
//
// runs the reference's epoch loop (run_epoch, validation, learning-rate
// schedule, RTRN checkpoints byte-compatible with StandardTraits') with every
// window on the GPU.  The overloads are found by argument-dependent lookup
// from inside the reference's templates and win over its generic templates
// as non-template functions with identical argument types.
//
// Parameters, gradients and optimiser state stay on the device: GpuParams /
// GpuOpt hold the context; the host copies exist only while a checkpoint is
// written or read (read_params / read_opt return host values that are
// uploaded into the trainer's context when the trainer assigns them).
// The Trainer keeps its schedule and hidden state on the host and calls the
// device once per window (dl_window + dl_rmsprop); desklm::b200::Trainer
// (gpu.hpp) is the device-resident epoch loop for throughput.
#ifndef DESKLM_B200_TRAITS_HPP
#define DESKLM_B200_TRAITS_HPP

#include <algorithm>
#include <cmath>
#include <cstring>
#include <istream>
#include <memory>
#include <optional>
#include <ostream>
#include <sstream>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "desklm/compress.hpp"
#include "desklm/eval.hpp"
#include "desklm/trainer.hpp"
#include "desklm_b200/gpu.hpp"

namespace desklm {
namespace b200 {

namespace detail {
// mt19937_64 <-> the library's 313-word state (the stream operators' text)
inline void rng_to_words(const std::mt19937_64& r, std::uint64_t st[313]) {
  std::stringstream ss;
  ss << r;
  for (int i = 0; i < 313; ++i) ss >> st[i];
}
inline void words_to_rng(const std::uint64_t st[313], std::mt19937_64& r) {
  std::stringstream ss;
  for (int i = 0; i < 313; ++i) ss << st[i] << ' ';
  ss >> r;
}
// Library errors -> the reference's exception classes (util.hpp:32-48):
// usage errors std::invalid_argument, data errors desklm::DataError.
inline void chk(int rc, const dl_ctx* ctx) {
  if (rc == DL_OK) return;
  const std::string m = dl_last_error(ctx) ? dl_last_error(ctx) : "";
  if (rc == DL_EINVAL) throw std::invalid_argument(m);
  if (rc == DL_EDATA) throw ::desklm::DataError(m);
  throw std::runtime_error("desklm_cuda: " + m);
}
inline void chk_bn(int rc, const dl_bn* ctx) {
  if (rc == DL_OK) return;
  const std::string m = dl_bn_last_error(ctx) ? dl_bn_last_error(ctx) : "";
  if (rc == DL_EINVAL) throw std::invalid_argument(m);
  if (rc == DL_EDATA) throw ::desklm::DataError(m);
  throw std::runtime_error("desklm_cuda: " + m);
}
}  // namespace detail

// ======================================================= standard model
// Per-context state the device path keeps beside the weights: which loss
// mode / noise model was last configured (NoiseModel identity).
struct GpuContext {
  Model model;
  int loss_mode = -1;
  const NoiseModel* noise = nullptr;
  GpuContext(std::int64_t V, std::int64_t H, int act, Precision p, int device)
      : model(V, H, act, p, device) {}
};

// RnnParams<float> on the device (rnn.hpp:61-84).  v, h and act are the
// reference fields; the weights live in the context.  A value read from a
// checkpoint (read_params) holds host weights until it is assigned into a
// GpuParams that owns a context, which then receives them.
struct GpuParams {
  std::int64_t v = 0, h = 0;
  Activation act = Activation::kSigmoid;
  Precision precision = Precision::kBf16;
  int device = 0;
  std::shared_ptr<GpuContext> ctx;
  std::shared_ptr<RnnParams<float>> pending;

  GpuParams() = default;
  explicit GpuParams(const RnnParams<float>& p, Precision prec = Precision::kBf16,
                     int dev = 0)
      : v(p.v), h(p.h), act(p.act), precision(prec), device(dev) {
    ctx = std::make_shared<GpuContext>(p.v, p.h, static_cast<int>(p.act), prec, dev);
    ctx->model.upload(p);
  }
  static GpuParams from_host(RnnParams<float> p) {
    GpuParams g;
    g.v = p.v;
    g.h = p.h;
    g.act = p.act;
    g.pending = std::make_shared<RnnParams<float>>(std::move(p));
    return g;
  }
  GpuParams(GpuParams&&) = default;
  GpuParams(const GpuParams&) = default;
  GpuParams& operator=(const GpuParams&) = default;
  // Trainer::load_checkpoint assigns read_params' value: keep this context
  // (precision, device) and upload the checkpoint's weights into it
  GpuParams& operator=(GpuParams&& o) {
    if (ctx && !o.ctx && o.pending && o.v == v && o.h == h) {
      act = o.pending->act;
      ctx->model.upload(*o.pending);
      return *this;
    }
    v = o.v;
    h = o.h;
    act = o.act;
    precision = o.precision;
    device = o.device;
    ctx = std::move(o.ctx);
    pending = std::move(o.pending);
    return *this;
  }
  GpuContext& context() const {
    auto& self = const_cast<GpuParams&>(*this);
    if (!self.ctx) {
      if (!self.pending) throw std::invalid_argument("GpuParams: empty parameters");
      self.ctx = std::make_shared<GpuContext>(v, h, static_cast<int>(act), precision, device);
      self.ctx->model.upload(*self.pending);
    }
    self.pending.reset();
    return *self.ctx;
  }
  dl_ctx* handle() const { return context().model.get(); }
  RnnParams<float> download() const {
    RnnParams<float> p(v, h, act);
    if (pending && !ctx) return *pending;
    context().model.download(p);
    return p;
  }
};

// Gradients of the last window stay on the device (StandardGrads,
// rnn.hpp:147-172); this records which context holds them.
struct GpuGrads {
  std::shared_ptr<GpuContext> ctx;
  bool valid = false;
};

// RmspropState (rmsprop.hpp:37-59) on the device, bound to the parameters'
// context by make_opt; read_opt's value holds host accumulators until it is
// assigned into a bound GpuOpt.
struct GpuOpt {
  std::int64_t v = 0, h = 0;
  double rho = 0.9995, eps = 1e-6;
  std::shared_ptr<GpuContext> ctx;
  std::shared_ptr<RmspropState> pending;

  GpuOpt() = default;
  GpuOpt(const GpuOpt&) = default;
  GpuOpt& operator=(const GpuOpt&) = default;
  GpuOpt(GpuOpt&&) = default;
  GpuOpt& operator=(GpuOpt&& o) {
    if (ctx && !o.ctx && o.pending) {
      if (o.pending->v != v || o.pending->h != h)
        throw ::desklm::DataError("rmsprop state: shape mismatch");
      rho = o.pending->rho;
      eps = o.pending->eps;
      upload(*o.pending);
      return *this;
    }
    v = o.v;
    h = o.h;
    rho = o.rho;
    eps = o.eps;
    ctx = std::move(o.ctx);
    pending = std::move(o.pending);
    return *this;
  }
  void upload(const RmspropState& s) const {
    detail::chk(dl_set_opt(ctx->model.get(), s.m_rec.a.data(), s.m_in.data(), s.m_out.data(),
                           s.rho, s.eps),
                ctx->model.get());
  }
  RmspropState download() const {
    if (!ctx) {
      if (pending) return *pending;
      throw std::invalid_argument("GpuOpt: unbound optimiser state");
    }
    RmspropState s(v, h, rho, eps);
    detail::chk(dl_get_opt(ctx->model.get(), s.m_rec.a.data(), s.m_in.data(), s.m_out.data()),
                ctx->model.get());
    return s;
  }
};

// The engine plug-in (StandardAdapter's role, rnn.hpp:179-259) for the
// device model.  The device boundary is per window / per scoring batch, so
// only the shape accessors of the adapter contract are exposed.
class GpuAdapter {
 public:
  using RealT = float;
  using AccT = double;
  using Grads = GpuGrads;
  explicit GpuAdapter(const GpuParams& p) : p_(&p) {}
  std::int64_t hidden() const { return p_->h; }
  std::int64_t vocab() const { return p_->v; }
  Activation activation() const { return p_->act; }
  GpuContext& context() const { return p_->context(); }
  dl_ctx* handle() const { return p_->handle(); }
  const GpuParams& params() const { return *p_; }

 private:
  const GpuParams* p_;
};

// bptt_run (backprop.hpp:76-222) for the device model: one dl_window call.
// NCE mode: the noise model is the caller's NoiseModel (its normalised q,
// dl_set_noise_dist) and the draws come from *opt.rng, which advances by
// exactly the reference's 2 outputs per noise sample.
inline ::desklm::BpttResult bptt_run(const GpuAdapter& model, const WindowBatch& wb,
                                     const Mat<float>& h0, GpuGrads* grads,
                                     Mat<float>* h_final, const BpttOptions<float>& opt) {
  if (wb.T < 1 || wb.B < 1) throw std::invalid_argument("bptt: empty window");
  const std::int64_t H = model.hidden();
  if (h0.rows != wb.B || h0.cols != H)
    throw std::invalid_argument("bptt: initial state shape mismatch");
  GpuContext& c = model.context();
  dl_ctx* ctx = c.model.get();
  const int mode = opt.mode == LossMode::kNce ? 0 : 1;
  if (c.loss_mode != mode) {
    detail::chk(dl_set_loss_mode(ctx, mode), ctx);
    c.loss_mode = mode;
  }
  if (mode == 0) {
    if (opt.noise == nullptr || opt.rng == nullptr)
      throw std::invalid_argument("bptt: NCE mode needs noise model and rng");
    if (c.noise != opt.noise) {
      std::vector<double> q(static_cast<std::size_t>(model.vocab()));
      for (std::size_t w = 0; w < q.size(); ++w) q[w] = opt.noise->q(static_cast<WordId>(w));
      detail::chk(dl_set_noise_dist(ctx, q.data(), model.vocab(), opt.noise->k()), ctx);
      c.noise = opt.noise;
    }
    std::uint64_t st[313];
    detail::rng_to_words(*opt.rng, st);
    detail::chk(dl_set_rng_state(ctx, st), ctx);
  }
  if (h_final && (h_final->rows != wb.B || h_final->cols != H)) *h_final = Mat<float>(wb.B, H);
  ::desklm::BpttResult r;
  std::uint64_t pos = 0;
  const bool g = grads != nullptr && opt.compute_grads;
  detail::chk(dl_window(ctx, wb.T, wb.B, wb.inputs.data(), wb.targets.data(), wb.weights.data(),
                        h0.a.data(), h_final ? h_final->a.data() : nullptr, opt.loss_scale,
                        static_cast<float>(opt.clip), g ? 1 : 0, &r.loss, &pos),
              ctx);
  r.positions = static_cast<std::size_t>(pos);
  if (mode == 0) {
    std::uint64_t st[313];
    detail::chk(dl_get_rng_state(ctx, st), ctx);
    detail::words_to_rng(st, *opt.rng);
  }
  if (grads) {
    grads->ctx = model.params().ctx;
    grads->valid = g;
  }
  return r;
}

// rmsprop_update (rmsprop.hpp:113-133) on the device: false = rejected
// non-finite gradient, parameters and accumulators untouched.
inline bool rmsprop_update(GpuParams& p, const GpuGrads& g, GpuOpt& o, double eta) {
  if (!g.valid || g.ctx.get() != &p.context())
    throw std::invalid_argument("rmsprop: no device gradients for these parameters");
  if (o.pending) {
    o.ctx = p.ctx;
    const RmspropState s = *o.pending;
    o.pending.reset();
    o.upload(s);
  }
  int applied = 0;
  detail::chk(dl_rmsprop(p.handle(), eta, &applied), p.handle());
  return applied != 0;
}

// sharded_perplexity (eval.hpp:151-222) / rnn_perplexity (eval.hpp:84-145).
inline ::desklm::PerplexityResult sharded_perplexity(const GpuAdapter& model,
                                                     const IdStream& stream, int shards,
                                                     WordId bos_id = Vocabulary::kBosId,
                                                     int threads = 1) {
  (void)threads;
  ::desklm::PerplexityResult r;
  std::uint64_t pred = 0;
  dl_ctx* ctx = model.handle();
  detail::chk(dl_sharded_perplexity(ctx, stream.ids.data(),
                                    static_cast<std::int64_t>(stream.ids.size()), shards, bos_id,
                                    &r.total_logprob, &pred, &r.perplexity),
              ctx);
  r.predicted = static_cast<std::size_t>(pred);
  return r;
}

inline ::desklm::PerplexityResult rnn_perplexity(const GpuAdapter& model, const IdStream& stream,
                                                 WordId bos_id = Vocabulary::kBosId,
                                                 int threads = 1) {
  (void)threads;
  ::desklm::PerplexityResult r;
  std::uint64_t pred = 0;
  dl_ctx* ctx = model.handle();
  detail::chk(dl_rnn_perplexity(ctx, stream.ids.data(),
                                static_cast<std::int64_t>(stream.ids.size()), bos_id,
                                &r.total_logprob, &pred, &r.perplexity),
              ctx);
  r.predicted = static_cast<std::size_t>(pred);
  return r;
}

// Model family for desklm::Trainer (trainer.hpp:117-156).
struct GpuStandardTraits {
  using Params = GpuParams;
  using Grads = GpuGrads;
  using Adapter = GpuAdapter;
  using Opt = GpuOpt;

  static std::int64_t hidden(const Params& p) { return p.h; }
  static std::int64_t vocab(const Params& p) { return p.v; }
  static Activation activation(const Params& p) { return p.act; }
  static Opt make_opt(const Params& p, double rho, double eps) {
    Opt o;
    o.v = p.v;
    o.h = p.h;
    o.rho = rho;
    o.eps = eps;
    p.context();
    o.ctx = p.ctx;
    o.upload(RmspropState(p.v, p.h, rho, eps));  // zero accumulators
    return o;
  }
  static bool update(Params& p, const Grads& g, Opt& o, double eta) {
    return rmsprop_update(p, g, o, eta);
  }
  static void write_params(std::ostream& os, const Params& p, const Vocabulary& v) {
    ::desklm::write_params(os, p.download(), v);
  }
  static std::pair<Params, Vocabulary> read_params(std::istream& is) {
    auto [p, v] = ::desklm::read_params(is);
    return {GpuParams::from_host(std::move(p)), std::move(v)};
  }
  static void write_opt(std::ostream& os, const Opt& o) {
    ::desklm::write_rmsprop(os, o.download());
  }
  static Opt read_opt(std::istream& is) {
    RmspropState s = ::desklm::read_rmsprop(is);
    Opt o;
    o.v = s.v;
    o.h = s.h;
    o.rho = s.rho;
    o.eps = s.eps;
    o.pending = std::make_shared<RmspropState>(std::move(s));
    return o;
  }
};

// rescore_nbest (eval.hpp:693-790) for the device models: every hypothesis
// is one stream (bos + words + eos, hidden state act(0)); all of them are
// scored by one lock-step device call.  Exact mode needs, per position,
// ln p(y) of the mapped target (or of the RNN's <unk> when the n-gram maps
// the target outside the RNN vocabulary), which the scorer returns; the
// n-gram interpolation and the stable sort are the reference's host logic.
// Fast mode (raw scores as if normalised) scores one candidate per position
// with the 8-lane double dot product (dl_score_candidates).
namespace detail {
template <class ScoreFn, class CandFn>
void rescore_device(std::vector<NBestUtt>& utts, std::int64_t V, const Vocabulary& rnn_vocab,
                    const NGramModel* ngram, const RescoreConfig& cfg, ScoreFn&& score_exact,
                    CandFn&& score_fast) {
  if (static_cast<std::int64_t>(rnn_vocab.size()) != V)
    throw std::invalid_argument("rescore: vocabulary/model size mismatch");
  if (cfg.lambda < 0.0 || cfg.lambda > 1.0)
    throw std::invalid_argument("rescore: lambda must be in [0, 1]");
  const Vocabulary& enc_vocab = ngram != nullptr ? ngram->vocab() : rnn_vocab;
  VocabMap map;
  if (ngram != nullptr) map = make_vocab_map(rnn_vocab, ngram->vocab());
  // encode every hypothesis; RNN inputs / targets per position
  std::vector<std::vector<WordId>> seqs;
  for (const NBestUtt& u : utts)
    for (const NBestHyp& hyp : u.hyps) {
      std::vector<WordId> ids;
      ids.reserve(hyp.words.size() + 2);
      ids.push_back(enc_vocab.bos_id());
      for (const std::string& w : hyp.words) ids.push_back(enc_vocab.id_or_unk(w));
      ids.push_back(enc_vocab.eos_id());
      seqs.push_back(std::move(ids));
    }
  if (seqs.empty()) return;
  auto to_rnn = [&](WordId x) -> WordId {
    if (ngram == nullptr) return x;
    const std::int64_t xr = map.full_to_rnn[x];
    return xr >= 0 ? static_cast<WordId>(xr) : map.rnn_unk;
  };
  auto rnn_target = [&](WordId y) -> WordId {
    if (ngram == nullptr) return y;
    const std::int64_t yr = map.full_to_rnn[y];
    return (yr >= 0 && static_cast<WordId>(yr) != map.rnn_unk) ? static_cast<WordId>(yr)
                                                                 : map.rnn_unk;
  };
  const std::int64_t S = static_cast<std::int64_t>(seqs.size());
  std::int64_t steps = 0;
  for (const auto& s : seqs) steps = std::max<std::int64_t>(steps, s.size() - 1);
  std::vector<std::uint32_t> in(static_cast<std::size_t>(S * steps), 0);
  std::vector<std::int64_t> tg(static_cast<std::size_t>(S * steps), -1);
  for (std::int64_t s = 0; s < S; ++s)
    for (std::size_t i = 0; i + 1 < seqs[s].size(); ++i) {
      in[i * S + s] = to_rnn(seqs[s][i]);
      tg[i * S + s] = rnn_target(seqs[s][i + 1]);
    }
  // ln p_rnn (exact) or the raw score (fast) of the chosen target
  std::vector<double> lp(static_cast<std::size_t>(S * steps), 0.0);
  if (!cfg.fast) score_exact(S, steps, in, tg, lp);
  else score_fast(S, steps, seqs, in, tg, lp);
  std::int64_t s = 0;
  for (NBestUtt& u : utts) {
    for (NBestHyp& hyp : u.hyps) {
      const auto& ids = seqs[s];
      std::vector<WordId> ctx;
      double total = 0.0;
      for (std::size_t i = 0; i + 1 < ids.size(); ++i) {
        const WordId x = ids[i], y = ids[i + 1];
        const double p_rnn = std::exp(lp[i * S + s]);  // exp(s - lse) or exp(raw)
        if (ngram == nullptr) {
          total += std::log(p_rnn);
          continue;
        }
        if (x == enc_vocab.bos_id())
          ctx.assign(1, x);
        else {
          ctx.push_back(x);
          const auto cap = static_cast<std::size_t>(ngram->order() - 1);
          if (cap > 0 && ctx.size() > cap)
            ctx.erase(ctx.begin(), ctx.end() - static_cast<std::ptrdiff_t>(cap));
        }
        const double pn = std::exp(ngram->logprob(ctx, y));
        const std::int64_t yr = map.full_to_rnn[y];
        double a;
        if (yr >= 0 && static_cast<WordId>(yr) != map.rnn_unk) {
          a = p_rnn;
        } else {
          double z_out = 0.0;
          for (WordId f : map.oor_ids) z_out += std::exp(ngram->logprob(ctx, f));
          a = z_out > 0.0 ? p_rnn * pn / z_out : 0.0;
        }
        const double p = cfg.lambda * a + (1.0 - cfg.lambda) * pn;
        if (!(p > 0.0)) throw ::desklm::DataError("rescore: non-positive probability");
        total += std::log(p);
      }
      hyp.new_lm = total;
      hyp.new_total = hyp.acoustic + cfg.lm_scale * total +
                      cfg.wip * static_cast<double>(hyp.words.size());
      ++s;
    }
    std::stable_sort(u.hyps.begin(), u.hyps.end(), [](const NBestHyp& a, const NBestHyp& b) {
      return a.new_total > b.new_total;
    });
    for (std::size_t i = 0; i < u.hyps.size(); ++i) u.hyps[i].rank = i + 1;
  }
}
}  // namespace detail

inline void rescore_nbest(std::vector<NBestUtt>& utts, const GpuAdapter& rnn,
                          const Vocabulary& rnn_vocab, const NGramModel* ngram,
                          const RescoreConfig& cfg) {
  dl_ctx* ctx = rnn.handle();
  detail::rescore_device(
      utts, rnn.vocab(), rnn_vocab, ngram, cfg,
      [&](std::int64_t S, std::int64_t steps, const std::vector<std::uint32_t>& in,
          const std::vector<std::int64_t>& tg, std::vector<double>& lp) {
        double tot = 0.0;
        std::uint64_t pred = 0;
        detail::chk(dl_score(ctx, S, steps, in.data(), tg.data(), nullptr, nullptr, lp.data(),
                             &tot, &pred),
                    ctx);
      },
      [&](std::int64_t S, std::int64_t steps, const std::vector<std::vector<WordId>>& seqs,
          const std::vector<std::uint32_t>& in, const std::vector<std::int64_t>& tg,
          std::vector<double>& lp) {
        (void)steps;
        // one stream per hypothesis: raw score float(h . W_out[target])
        for (std::int64_t s = 0; s < S; ++s) {
          const std::int64_t n = static_cast<std::int64_t>(seqs[s].size()) - 1;
          std::vector<std::uint32_t> x(n);
          std::vector<std::int64_t> cand(n);
          for (std::int64_t i = 0; i < n; ++i) {
            x[i] = in[i * S + s];
            cand[i] = tg[i * S + s];
          }
          std::vector<float> out(n);
          detail::chk(dl_score_candidates(ctx, x.data(), n, 1, cand.data(), out.data()), ctx);
          for (std::int64_t i = 0; i < n; ++i) lp[i * S + s] = static_cast<double>(out[i]);
        }
      });
}

// ===================================================== bottleneck model
// BottleneckParams<float> on the device (compress.hpp:38-83): E [V x P],
// U [P x H], W_rec [H x H], D [H x P].  Scoring (RNBL / RNQZ models through
// with_gpu_model) and the training seam of Trainer<GpuBottleneckTraits>.
struct GpuBnContext {
  BottleneckModel model;
  int loss_mode = -1;
  const NoiseModel* noise = nullptr;
  GpuBnContext(std::int64_t V, std::int64_t H, std::int64_t P, int act, Precision prec, int dev)
      : model(V, H, P, act, prec, dev) {}
};

struct GpuBnParams {
  std::int64_t v = 0, h = 0, p = 0;
  Activation act = Activation::kSigmoid;
  Precision precision = Precision::kBf16;
  int device = 0;
  std::shared_ptr<GpuBnContext> ctx;
  std::shared_ptr<BottleneckParams<float>> pending;

  GpuBnParams() = default;
  explicit GpuBnParams(const BottleneckParams<float>& bp, Precision prec = Precision::kBf16,
                       int dev = 0)
      : v(bp.v), h(bp.h), p(bp.p), act(bp.act), precision(prec), device(dev) {
    ctx = std::make_shared<GpuBnContext>(bp.v, bp.h, bp.p, static_cast<int>(bp.act), prec, dev);
    ctx->model.upload(bp);
  }
  // RNQZ: the packed codes are dequantised on the device (dl_bn_set_params_quantized)
  explicit GpuBnParams(const QuantizedModel& q, Precision prec = Precision::kBf16, int dev = 0)
      : v(q.v), h(q.h), p(q.p), act(q.act), precision(prec), device(dev) {
    ctx = std::make_shared<GpuBnContext>(q.v, q.h, q.p, static_cast<int>(q.act), prec, dev);
    const QuantizedMatrix* mats[4] = {&q.e, &q.u, &q.w_rec, &q.d};
    dl_qmatrix m[4];
    for (int i = 0; i < 4; ++i) {
      m[i].bits = mats[i]->bits;
      m[i].min = mats[i]->min;
      m[i].max = mats[i]->max;
      m[i].codes = mats[i]->codes.data();  // packed LSB first, as in the file
    }
    detail::chk_bn(dl_bn_set_params_quantized(ctx->model.get(), m), ctx->model.get());
  }
  static GpuBnParams from_host(BottleneckParams<float> bp) {
    GpuBnParams g;
    g.v = bp.v;
    g.h = bp.h;
    g.p = bp.p;
    g.act = bp.act;
    g.pending = std::make_shared<BottleneckParams<float>>(std::move(bp));
    return g;
  }
  GpuBnParams(GpuBnParams&&) = default;
  GpuBnParams(const GpuBnParams&) = default;
  GpuBnParams& operator=(const GpuBnParams&) = default;
  GpuBnParams& operator=(GpuBnParams&& o) {
    if (ctx && !o.ctx && o.pending && o.v == v && o.h == h && o.p == p) {
      act = o.pending->act;
      ctx->model.upload(*o.pending);
      return *this;
    }
    v = o.v;
    h = o.h;
    p = o.p;
    act = o.act;
    precision = o.precision;
    device = o.device;
    ctx = std::move(o.ctx);
    pending = std::move(o.pending);
    return *this;
  }
  GpuBnContext& context() const {
    auto& self = const_cast<GpuBnParams&>(*this);
    if (!self.ctx) {
      if (!self.pending) throw std::invalid_argument("GpuBnParams: empty parameters");
      self.ctx =
          std::make_shared<GpuBnContext>(v, h, p, static_cast<int>(act), precision, device);
      self.ctx->model.upload(*self.pending);
    }
    self.pending.reset();
    return *self.ctx;
  }
  dl_bn* handle() const { return context().model.get(); }
  BottleneckParams<float> download() const {
    if (pending && !ctx) return *pending;
    BottleneckParams<float> bp(v, h, p, act);
    context().model.download(bp);
    return bp;
  }
};

struct GpuBnGrads {
  std::shared_ptr<GpuBnContext> ctx;
  bool valid = false;
};

struct GpuBnOpt {
  std::int64_t v = 0, h = 0, p = 0;
  double rho = 0.9995, eps = 1e-6;
  std::shared_ptr<GpuBnContext> ctx;
  std::shared_ptr<BottleneckOptState> pending;

  GpuBnOpt() = default;
  GpuBnOpt(const GpuBnOpt&) = default;
  GpuBnOpt& operator=(const GpuBnOpt&) = default;
  GpuBnOpt(GpuBnOpt&&) = default;
  GpuBnOpt& operator=(GpuBnOpt&& o) {
    if (ctx && !o.ctx && o.pending) {
      rho = o.pending->rho;
      eps = o.pending->eps;
      upload(*o.pending);
      return *this;
    }
    v = o.v;
    h = o.h;
    p = o.p;
    rho = o.rho;
    eps = o.eps;
    ctx = std::move(o.ctx);
    pending = std::move(o.pending);
    return *this;
  }
  void upload(const BottleneckOptState& s) const {
    detail::chk_bn(dl_bn_set_opt(ctx->model.get(), s.m_e.data(), s.m_u.a.data(),
                                 s.m_rec.a.data(), s.m_d.a.data(), s.rho, s.eps),
                   ctx->model.get());
  }
  BottleneckOptState download() const {
    if (!ctx) {
      if (pending) return *pending;
      throw std::invalid_argument("GpuBnOpt: unbound optimiser state");
    }
    BottleneckOptState s(v, h, p, rho, eps);
    detail::chk_bn(dl_bn_get_opt(ctx->model.get(), s.m_e.data(), s.m_u.a.data(),
                                 s.m_rec.a.data(), s.m_d.a.data()),
                   ctx->model.get());
    return s;
  }
};

class GpuBottleneckAdapter {
 public:
  using RealT = float;
  using AccT = double;
  using Grads = GpuBnGrads;
  explicit GpuBottleneckAdapter(const GpuBnParams& p) : p_(&p) {}
  std::int64_t hidden() const { return p_->h; }
  std::int64_t vocab() const { return p_->v; }
  std::int64_t proj() const { return p_->p; }
  Activation activation() const { return p_->act; }
  GpuBnContext& context() const { return p_->context(); }
  dl_bn* handle() const { return p_->handle(); }
  const GpuBnParams& params() const { return *p_; }

 private:
  const GpuBnParams* p_;
};

inline ::desklm::BpttResult bptt_run(const GpuBottleneckAdapter& model, const WindowBatch& wb,
                                     const Mat<float>& h0, GpuBnGrads* grads,
                                     Mat<float>* h_final, const BpttOptions<float>& opt) {
  if (wb.T < 1 || wb.B < 1) throw std::invalid_argument("bptt: empty window");
  const std::int64_t H = model.hidden();
  if (h0.rows != wb.B || h0.cols != H)
    throw std::invalid_argument("bptt: initial state shape mismatch");
  GpuBnContext& c = model.context();
  dl_bn* ctx = c.model.get();
  const int mode = opt.mode == LossMode::kNce ? 0 : 1;
  if (c.loss_mode != mode) {
    detail::chk_bn(dl_bn_set_loss_mode(ctx, mode), ctx);
    c.loss_mode = mode;
  }
  if (mode == 0) {
    if (opt.noise == nullptr || opt.rng == nullptr)
      throw std::invalid_argument("bptt: NCE mode needs noise model and rng");
    if (c.noise != opt.noise) {
      std::vector<double> q(static_cast<std::size_t>(model.vocab()));
      for (std::size_t w = 0; w < q.size(); ++w) q[w] = opt.noise->q(static_cast<WordId>(w));
      detail::chk_bn(dl_bn_set_noise_dist(ctx, q.data(), model.vocab(), opt.noise->k()), ctx);
      c.noise = opt.noise;
    }
    std::uint64_t st[313];
    detail::rng_to_words(*opt.rng, st);
    detail::chk_bn(dl_bn_set_rng_state(ctx, st), ctx);
  }
  if (h_final && (h_final->rows != wb.B || h_final->cols != H)) *h_final = Mat<float>(wb.B, H);
  ::desklm::BpttResult r;
  std::uint64_t pos = 0;
  const bool g = grads != nullptr && opt.compute_grads;
  detail::chk_bn(dl_bn_window(ctx, wb.T, wb.B, wb.inputs.data(), wb.targets.data(),
                              wb.weights.data(), h0.a.data(),
                              h_final ? h_final->a.data() : nullptr, opt.loss_scale,
                              static_cast<float>(opt.clip), g ? 1 : 0, &r.loss, &pos),
                 ctx);
  r.positions = static_cast<std::size_t>(pos);
  if (mode == 0) {
    std::uint64_t st[313];
    detail::chk_bn(dl_bn_get_rng_state(ctx, st), ctx);
    detail::words_to_rng(st, *opt.rng);
  }
  if (grads) {
    grads->ctx = model.params().ctx;
    grads->valid = g;
  }
  return r;
}

// bottleneck_update (compress.hpp:296-309) on the device.
inline bool bottleneck_update(GpuBnParams& p, const GpuBnGrads& g, GpuBnOpt& o, double eta) {
  if (!g.valid || g.ctx.get() != &p.context())
    throw std::invalid_argument("bottleneck update: no device gradients for these parameters");
  if (o.pending) {
    o.ctx = p.ctx;
    const BottleneckOptState s = *o.pending;
    o.pending.reset();
    o.upload(s);
  }
  int applied = 0;
  detail::chk_bn(dl_bn_rmsprop(p.handle(), eta, &applied), p.handle());
  return applied != 0;
}

inline ::desklm::PerplexityResult sharded_perplexity(const GpuBottleneckAdapter& model,
                                                     const IdStream& stream, int shards,
                                                     WordId bos_id = Vocabulary::kBosId,
                                                     int threads = 1) {
  (void)threads;
  ::desklm::PerplexityResult r;
  std::uint64_t pred = 0;
  dl_bn* ctx = model.handle();
  detail::chk_bn(dl_bn_sharded_perplexity(ctx, stream.ids.data(),
                                          static_cast<std::int64_t>(stream.ids.size()), shards,
                                          bos_id, &r.total_logprob, &pred, &r.perplexity),
                 ctx);
  r.predicted = static_cast<std::size_t>(pred);
  return r;
}

// rnn_perplexity (eval.hpp:84-145): one stream walked cold from its start,
// every token an input, non-bos targets scored.
inline ::desklm::PerplexityResult rnn_perplexity(const GpuBottleneckAdapter& model,
                                                 const IdStream& stream,
                                                 WordId bos_id = Vocabulary::kBosId,
                                                 int threads = 1) {
  (void)threads;
  const auto& ids = stream.ids;
  if (ids.size() < 2) throw std::invalid_argument("rnn perplexity: stream too short");
  const std::int64_t n = static_cast<std::int64_t>(ids.size()) - 1;
  std::vector<std::int64_t> tg(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < n; ++i)
    tg[i] = ids[i + 1] == bos_id ? std::int64_t{-1} : static_cast<std::int64_t>(ids[i + 1]);
  ::desklm::PerplexityResult r;
  std::uint64_t pred = 0;
  dl_bn* ctx = model.handle();
  detail::chk_bn(dl_bn_score(ctx, 1, n, ids.data(), tg.data(), nullptr, nullptr, nullptr,
                             &r.total_logprob, &pred),
                 ctx);
  if (pred == 0) throw std::invalid_argument("rnn perplexity: no predicted tokens");
  r.predicted = static_cast<std::size_t>(pred);
  r.perplexity = std::exp(-r.total_logprob / static_cast<double>(r.predicted));
  return r;
}

inline void rescore_nbest(std::vector<NBestUtt>& utts, const GpuBottleneckAdapter& rnn,
                          const Vocabulary& rnn_vocab, const NGramModel* ngram,
                          const RescoreConfig& cfg) {
  if (cfg.fast)
    throw std::invalid_argument("rescore: fast mode is not available for the bottleneck model");
  dl_bn* ctx = rnn.handle();
  detail::rescore_device(
      utts, rnn.vocab(), rnn_vocab, ngram, cfg,
      [&](std::int64_t S, std::int64_t steps, const std::vector<std::uint32_t>& in,
          const std::vector<std::int64_t>& tg, std::vector<double>& lp) {
        double tot = 0.0;
        std::uint64_t pred = 0;
        detail::chk_bn(dl_bn_score(ctx, S, steps, in.data(), tg.data(), nullptr, nullptr,
                                   lp.data(), &tot, &pred),
                       ctx);
      },
      [](std::int64_t, std::int64_t, const std::vector<std::vector<WordId>>&,
         const std::vector<std::uint32_t>&, const std::vector<std::int64_t>&,
         std::vector<double>&) {});
}

struct GpuBottleneckTraits {
  using Params = GpuBnParams;
  using Grads = GpuBnGrads;
  using Adapter = GpuBottleneckAdapter;
  using Opt = GpuBnOpt;

  static std::int64_t hidden(const Params& p) { return p.h; }
  static std::int64_t vocab(const Params& p) { return p.v; }
  static Activation activation(const Params& p) { return p.act; }
  static Opt make_opt(const Params& p, double rho, double eps) {
    Opt o;
    o.v = p.v;
    o.h = p.h;
    o.p = p.p;
    o.rho = rho;
    o.eps = eps;
    p.context();
    o.ctx = p.ctx;
    o.upload(BottleneckOptState(p.v, p.h, p.p, rho, eps));
    return o;
  }
  static bool update(Params& p, const Grads& g, Opt& o, double eta) {
    return bottleneck_update(p, g, o, eta);
  }
  static void write_params(std::ostream& os, const Params& p, const Vocabulary& v) {
    write_bottleneck(os, p.download(), v);
  }
  static std::pair<Params, Vocabulary> read_params(std::istream& is) {
    auto [p, v] = read_bottleneck(is);
    return {GpuBnParams::from_host(std::move(p)), std::move(v)};
  }
  static void write_opt(std::ostream& os, const Opt& o) { write_bottleneck_opt(os, o.download()); }
  static Opt read_opt(std::istream& is) {
    BottleneckOptState s = read_bottleneck_opt(is);
    Opt o;
    o.v = s.v;
    o.h = s.h;
    o.p = s.p;
    o.rho = s.rho;
    o.eps = s.eps;
    o.pending = std::make_shared<BottleneckOptState>(std::move(s));
    return o;
  }
};

// tools/desklm.cpp:142-163 with_model for the device: reads a recurrent model
// of any on-disk flavour -- standard "RNLM", bottleneck "RNBL", or quantised
// "RNQZ" (dequantised on the device) -- and invokes fn(adapter, vocabulary).
template <class Fn>
void with_gpu_model(const std::string& bytes, Precision prec, Fn&& fn, int device = 0) {
  if (bytes.size() < 4) throw ::desklm::DataError("model file too short to identify");
  const std::string_view magic(bytes.data(), 4);
  std::istringstream is(bytes);
  if (magic == "RNLM") {
    auto [p, v] = ::desklm::read_params(is);
    const GpuParams gp(p, prec, device);
    const GpuAdapter a(gp);
    fn(a, v);
  } else if (magic == "RNBL") {
    auto [p, v] = read_bottleneck(is);
    const GpuBnParams gp(p, prec, device);
    const GpuBottleneckAdapter a(gp);
    fn(a, v);
  } else if (magic == "RNQZ") {
    const QuantizedModel q = read_quantized(is);
    const GpuBnParams gp(q, prec, device);
    const GpuBottleneckAdapter a(gp);
    const Vocabulary v(q.words);
    fn(a, v);
  } else {
    throw ::desklm::DataError("unrecognized model header (want RNLM, RNBL, or RNQZ)");
  }
}

}  // namespace b200
}  // namespace desklm

#endif  // DESKLM_B200_TRAITS_HPP
