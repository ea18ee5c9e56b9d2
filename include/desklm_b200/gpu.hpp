// desklm_b200/gpu.hpp -- header-only C++ host API over the C ABI
// (include/desklm_cuda.h) for users of the desklm reference library.
//
// Mirrors the reference's public training / scoring interface
// (/root/reference/proj/include/desklm):
//   RnnParams<float> + StandardAdapter   rnn.hpp:61-84, :179-259 -> b200::Model
//   bptt_run (softmax mode)              backprop.hpp:76-222     -> b200::bptt_run
//   rmsprop_update                       rmsprop.hpp:113-133     -> b200::rmsprop_update
//   sharded_perplexity / rnn_perplexity  eval.hpp:84-222          -> b200::sharded_perplexity ...
//   TrainConfig / EpochLog / Trainer     trainer.hpp:43-476       -> b200::Trainer
//   RNLM / ROPT / RTRN                   rnn.hpp:263, rmsprop.hpp:137, trainer.hpp:274
//
// The reference's own types plug in unchanged: every function taking
// parameters, windows, id streams or configs is a template over the
// reference's field names (RnnParams::{v,h,act,w_in,w_rec,w_out} with
// Mat::a storage, WindowBatch::{T,B,inputs,targets,weights},
// IdStream::ids, TrainConfig's fields), so
//
//   desklm::TrainConfig cfg;  desklm::RnnParams<float> p(V, H);  ...
//   desklm::b200::Trainer tr(cfg, p, vocab.words(), train, valid);
//   tr.train(&std::cerr);  tr.save_checkpoint(path);
//
// compiles against either the reference headers or the minimal stand-in
// types at the bottom of this file.  Errors follow the reference:
// std::invalid_argument for usage errors, b200::DataError for data errors.
#ifndef DESKLM_B200_GPU_HPP
#define DESKLM_B200_GPU_HPP

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <ostream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../desklm_cuda.h"

namespace desklm {
namespace b200 {

class DataError : public std::runtime_error {
 public:
  explicit DataError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int rc, const dl_ctx* ctx = nullptr) {
  if (rc == DL_OK) return;
  const std::string m = dl_last_error(ctx) ? dl_last_error(ctx) : "";
  if (rc == DL_EINVAL) throw std::invalid_argument(m);
  if (rc == DL_EDATA) throw DataError(m);
  throw std::runtime_error("desklm_cuda: " + m);
}

enum class Precision : int { kFp32 = DL_FP32, kBf16 = DL_BF16 };

struct BpttResult {
  double loss = 0.0;
  std::size_t positions = 0;
};

struct PerplexityResult {
  double perplexity = 0.0;
  double total_logprob = 0.0;
  std::size_t predicted = 0;
};

// Device-resident model + optimiser state (one GPU).
class Model {
 public:
  Model(std::int64_t V, std::int64_t H, int act = DL_SIGMOID, Precision p = Precision::kBf16,
        int device = 0)
      : v_(V), h_(H) {
    check(dl_create(&ctx_, device, V, H, act, static_cast<int>(p)));
  }
  template <class Params>
  explicit Model(const Params& params, Precision p = Precision::kBf16, int device = 0)
      : Model(params.v, params.h, static_cast<int>(params.act), p, device) {
    upload(params);
  }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;
  ~Model() { dl_destroy(ctx_); }

  dl_ctx* get() const { return ctx_; }
  std::int64_t vocab() const { return v_; }
  std::int64_t hidden() const { return h_; }

  template <class Params>
  void upload(const Params& p) {
    check(dl_set_params(ctx_, p.w_in.a.data(), p.w_rec.a.data(), p.w_out.a.data()), ctx_);
  }
  template <class Params>
  void download(Params& p) const {
    check(dl_get_params(ctx_, p.w_in.a.data(), p.w_rec.a.data(), p.w_out.a.data()), ctx_);
  }
  void set_opt(const float* m_rec, const float* m_in, const float* m_out, double rho,
               double eps) {
    check(dl_set_opt(ctx_, m_rec, m_in, m_out, rho, eps), ctx_);
  }
  void get_opt(float* m_rec, float* m_in, float* m_out) const {
    check(dl_get_opt(ctx_, m_rec, m_in, m_out), ctx_);
  }

 private:
  dl_ctx* ctx_ = nullptr;
  std::int64_t v_, h_;
};

// bptt_run (backprop.hpp:76-222), softmax mode; gradients stay on the device.
template <class WindowBatch, class MatF>
BpttResult bptt_run(Model& m, const WindowBatch& wb, const MatF& h0, MatF* h_final,
                    double loss_scale, float clip, bool compute_grads = true) {
  BpttResult r;
  std::uint64_t pos = 0;
  if (h_final) h_final->a.resize(static_cast<std::size_t>(wb.B * m.hidden()));
  check(dl_window(m.get(), wb.T, wb.B, wb.inputs.data(), wb.targets.data(), wb.weights.data(),
                  h0.a.data(), h_final ? h_final->a.data() : nullptr, loss_scale, clip,
                  compute_grads ? 1 : 0, &r.loss, &pos),
        m.get());
  r.positions = pos;
  return r;
}

// rmsprop_update (rmsprop.hpp:113-133): false = rejected non-finite gradient.
inline bool rmsprop_update(Model& m, double eta) {
  int applied = 0;
  check(dl_rmsprop(m.get(), eta, &applied), m.get());
  return applied != 0;
}

template <class IdStream>
PerplexityResult sharded_perplexity(Model& m, const IdStream& s, int shards,
                                    std::uint32_t bos = 1) {
  PerplexityResult r;
  std::uint64_t pred = 0;
  check(dl_sharded_perplexity(m.get(), s.ids.data(), static_cast<std::int64_t>(s.ids.size()),
                              shards, bos, &r.total_logprob, &pred, &r.perplexity),
        m.get());
  r.predicted = pred;
  return r;
}

template <class IdStream>
PerplexityResult rnn_perplexity(Model& m, const IdStream& s, std::uint32_t bos = 1) {
  PerplexityResult r;
  std::uint64_t pred = 0;
  check(dl_rnn_perplexity(m.get(), s.ids.data(), static_cast<std::int64_t>(s.ids.size()), bos,
                          &r.total_logprob, &pred, &r.perplexity),
        m.get());
  r.predicted = pred;
  return r;
}

// ----------------------------------------------- bottleneck model
// BottleneckParams<float> + BottleneckAdapter on the device (compress.hpp:
// 38-415).  Params: any type with v, h, p, act and Mat-like e, u, w_rec, d
// (desklm::BottleneckParams<float> fits).
inline void check_bn(int rc, const dl_bn* ctx) {
  if (rc == DL_OK) return;
  const std::string msg = dl_bn_last_error(ctx);
  if (rc == DL_EINVAL) throw std::invalid_argument(msg);
  if (rc == DL_EDATA) throw DataError(msg);
  throw std::runtime_error(msg);
}

class BottleneckModel {
 public:
  BottleneckModel(std::int64_t V, std::int64_t H, std::int64_t P, int act = DL_SIGMOID,
                  Precision prec = Precision::kBf16, int device = 0)
      : v_(V), h_(H), p_(P) {
    check_bn(dl_bn_create(&ctx_, device, V, H, P, act, static_cast<int>(prec)), nullptr);
  }
  template <class Params>
  explicit BottleneckModel(const Params& params, Precision prec = Precision::kBf16,
                           int device = 0)
      : BottleneckModel(params.v, params.h, params.p, static_cast<int>(params.act), prec,
                        device) {
    upload(params);
  }
  BottleneckModel(const BottleneckModel&) = delete;
  BottleneckModel& operator=(const BottleneckModel&) = delete;
  ~BottleneckModel() { dl_bn_destroy(ctx_); }

  dl_bn* get() const { return ctx_; }
  std::int64_t vocab() const { return v_; }
  std::int64_t hidden() const { return h_; }
  std::int64_t proj() const { return p_; }

  template <class Params>
  void upload(const Params& p) {
    check_bn(dl_bn_set_params(ctx_, p.e.a.data(), p.u.a.data(), p.w_rec.a.data(), p.d.a.data()),
             ctx_);
  }
  template <class Params>
  void download(Params& p) const {
    check_bn(dl_bn_get_params(ctx_, p.e.a.data(), p.u.a.data(), p.w_rec.a.data(), p.d.a.data()),
             ctx_);
  }
  void set_opt(const float* m_e, const float* m_u, const float* m_rec, const float* m_d,
               double rho, double eps) {
    check_bn(dl_bn_set_opt(ctx_, m_e, m_u, m_rec, m_d, rho, eps), ctx_);
  }

 private:
  dl_bn* ctx_ = nullptr;
  std::int64_t v_, h_, p_;
};

// bptt_run over the bottleneck adapter (softmax mode unless
// dl_bn_set_loss_mode switched the context to NCE).
template <class WindowBatch, class MatF>
BpttResult bptt_run(BottleneckModel& m, const WindowBatch& wb, const MatF& h0, MatF* h_final,
                    double loss_scale, float clip, bool compute_grads = true) {
  BpttResult r;
  std::uint64_t pos = 0;
  if (h_final) h_final->a.resize(static_cast<std::size_t>(wb.B * m.hidden()));
  check_bn(dl_bn_window(m.get(), wb.T, wb.B, wb.inputs.data(), wb.targets.data(),
                        wb.weights.data(), h0.a.data(), h_final ? h_final->a.data() : nullptr,
                        loss_scale, clip, compute_grads ? 1 : 0, &r.loss, &pos),
           m.get());
  r.positions = pos;
  return r;
}

// bottleneck_update (compress.hpp:296-309): false = rejected non-finite gradient.
inline bool bottleneck_update(BottleneckModel& m, double eta) {
  int applied = 0;
  check_bn(dl_bn_rmsprop(m.get(), eta, &applied), m.get());
  return applied != 0;
}

template <class IdStream>
PerplexityResult sharded_perplexity(BottleneckModel& m, const IdStream& s, int shards,
                                    std::uint32_t bos = 1) {
  PerplexityResult r;
  std::uint64_t pred = 0;
  check_bn(dl_bn_sharded_perplexity(m.get(), s.ids.data(),
                                    static_cast<std::int64_t>(s.ids.size()), shards, bos,
                                    &r.total_logprob, &pred, &r.perplexity),
           m.get());
  r.predicted = pred;
  return r;
}

// ln_z_samples (eval.hpp:805-857) for the standard model.
template <class IdStream>
std::vector<double> ln_z_samples(Model& m, const IdStream& s, std::size_t count) {
  std::vector<double> out(count);
  std::int64_t n = 0;
  check(dl_ln_z_samples(m.get(), s.ids.data(), static_cast<std::int64_t>(s.ids.size()),
                        static_cast<std::int64_t>(count), out.data(), &n),
        m.get());
  out.resize(static_cast<std::size_t>(n));
  return out;
}

// ----------------------------------------------------- binary primitives
namespace io {
inline void u8(std::ostream& o, std::uint8_t v) { o.put(static_cast<char>(v)); }
inline void u32(std::ostream& o, std::uint32_t v) {
  char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  o.write(b, 4);
}
inline void u64(std::ostream& o, std::uint64_t v) {
  char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<char>((v >> (8 * i)) & 0xff);
  o.write(b, 8);
}
inline void f32(std::ostream& o, float v) {
  std::uint32_t u;
  std::memcpy(&u, &v, 4);
  u32(o, u);
}
inline void f64(std::ostream& o, double v) {
  std::uint64_t u;
  std::memcpy(&u, &v, 8);
  u64(o, u);
}
inline void str(std::ostream& o, const std::string& s) {
  u64(o, s.size());
  o.write(s.data(), static_cast<std::streamsize>(s.size()));
}
// little-endian readers (util.hpp:115-162); short reads are DataError
inline void need(std::istream& is, const char* what) {
  if (!is) throw DataError(std::string("truncated input: ") + what);
}
inline std::uint8_t get_u8(std::istream& is) {
  char c = 0;
  is.get(c);
  need(is, "u8");
  return static_cast<std::uint8_t>(c);
}
inline std::uint32_t get_u32(std::istream& is) {
  unsigned char b[4];
  is.read(reinterpret_cast<char*>(b), 4);
  need(is, "u32");
  std::uint32_t v = 0;
  for (int i = 3; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
inline std::uint64_t get_u64(std::istream& is) {
  unsigned char b[8];
  is.read(reinterpret_cast<char*>(b), 8);
  need(is, "u64");
  std::uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
inline float get_f32(std::istream& is) {
  const std::uint32_t u = get_u32(is);
  float v;
  std::memcpy(&v, &u, 4);
  return v;
}
inline double get_f64(std::istream& is) {
  const std::uint64_t u = get_u64(is);
  double v;
  std::memcpy(&v, &u, 8);
  return v;
}
inline std::string get_str(std::istream& is) {
  const std::uint64_t n = get_u64(is);
  if (n > (1ull << 30)) throw DataError("implausible string length");
  std::string s(static_cast<std::size_t>(n), '\0');
  is.read(&s[0], static_cast<std::streamsize>(n));
  need(is, "string");
  return s;
}
inline void magic(std::istream& is, const char* m, const char* what) {
  char b[4];
  is.read(b, 4);
  if (!is || std::memcmp(b, m, 4) != 0) throw DataError(std::string(what) + ": bad magic");
}
}  // namespace io

// RNLM (rnn.hpp:263-285): W_out stored H x V.
inline void write_params(std::ostream& os, std::int64_t V, std::int64_t H, int act,
                         const float* w_in, const float* w_rec, const float* w_out,
                         const std::vector<std::string>& words) {
  os.write("RNLM", 4);
  io::u32(os, 1);
  io::u64(os, static_cast<std::uint64_t>(V));
  io::u64(os, static_cast<std::uint64_t>(H));
  io::u8(os, static_cast<std::uint8_t>(act));
  for (std::int64_t i = 0; i < V * H; ++i) io::f32(os, w_in[i]);
  for (std::int64_t i = 0; i < H * H; ++i) io::f32(os, w_rec[i]);
  for (std::int64_t i = 0; i < H; ++i)
    for (std::int64_t w = 0; w < V; ++w) io::f32(os, w_out[w * H + i]);
  io::u64(os, words.size());
  for (const auto& w : words) io::str(os, w);
}

// ROPT (rmsprop.hpp:139-149).
inline void write_rmsprop(std::ostream& os, std::int64_t V, std::int64_t H, double rho,
                          double eps, const float* m_rec, const float* m_in,
                          const float* m_out) {
  os.write("ROPT", 4);
  io::u32(os, 1);
  io::u64(os, static_cast<std::uint64_t>(V));
  io::u64(os, static_cast<std::uint64_t>(H));
  io::f64(os, rho);
  io::f64(os, eps);
  for (std::int64_t i = 0; i < H * H; ++i) io::f32(os, m_rec[i]);
  for (std::int64_t i = 0; i < V; ++i) io::f32(os, m_in[i]);
  for (std::int64_t i = 0; i < V; ++i) io::f32(os, m_out[i]);
}

struct EpochLog {
  int epoch = 0;
  double train_loss = 0.0;
  double valid_ppl = 0.0;
  double eta = 0.0;
  double seconds = 0.0;
  double tokens_per_sec = 0.0;
  std::size_t skipped_updates = 0;
};

namespace detail {
inline std::vector<std::string> words_of(std::vector<std::string> w) { return w; }
template <class Vocab>
auto words_of(const Vocab& v) -> decltype(v.words(), std::vector<std::string>()) {
  return std::vector<std::string>(v.words().begin(), v.words().end());
}
}  // namespace detail

// Trainer<StandardTraits> (trainer.hpp:171-476) with the epoch loop on the
// device (window build, bptt, rmsprop, hidden carry, wrap reset in one CUDA
// graph per window), softmax or NCE (TrainConfig::mode).  Cfg is the
// reference's TrainConfig (or any struct with its field names); the
// vocabulary is a desklm::Vocabulary (or its word list).  Same public
// interface as the reference's Trainer: train / validate / logs / epoch /
// eta / best_ppl / initial_ppl / config / vocab / params (download) and
// RTRN save_checkpoint / load_checkpoint, byte-compatible.  (For the
// reference's own Trainer class over the device see traits.hpp.)
template <class Cfg>
class Trainer {
 public:
  template <class Params, class IdStream, class Vocab>
  Trainer(const Cfg& cfg, const Params& params, const Vocab& vocab, const IdStream& train,
          const IdStream& valid, Precision prec = Precision::kBf16, int device = 0)
      : cfg_(cfg),
        vocab_(detail::words_of(vocab)),
        train_(train.ids),
        model_(params.v, params.h, static_cast<int>(params.act), prec, device),
        rng_(cfg.seed) {
    cfg_.validate();
    const int mode = static_cast<int>(cfg_.mode);  // LossMode: 0 NCE, 1 softmax
    if (static_cast<std::int64_t>(vocab_.size()) != params.v)
      throw std::invalid_argument("trainer: vocabulary/model size mismatch");
    model_.upload(params);
    model_.set_opt(nullptr, nullptr, nullptr, cfg_.rho, cfg_.eps);
    if (mode == 0) {
      // NoiseModel::from_stream (nce.hpp:69-76, trainer.hpp:207-209); the
      // noise draws come from rng_ (seeded with cfg.seed, trainer.hpp:184)
      std::vector<double> counts(static_cast<std::size_t>(params.v), 0.0);
      for (std::uint32_t id : train_)
        if (id != 1u) counts.at(id) += 1.0;
      check(dl_set_loss_mode(model_.get(), 0), model_.get());
      check(dl_set_noise(model_.get(), counts.data(), params.v, cfg_.nce_k, cfg_.noise_floor),
            model_.get());
      put_rng();
    }
    if (cfg_.valid_limit > 0 && static_cast<std::int64_t>(valid.ids.size()) > cfg_.valid_limit)
      valid_.assign(valid.ids.begin(), valid.ids.begin() + cfg_.valid_limit);
    else
      valid_ = valid.ids;
    if (valid_.size() < 2) throw std::invalid_argument("trainer: validation stream too short");
    check(dl_trainer_init(model_.get(), train_.data(), static_cast<std::int64_t>(train_.size()),
                          cfg_.noffset, cfg_.minibatch, cfg_.unroll, cfg_.clip, 1),
          model_.get());
    eta_ = cfg_.eta;
  }

  const Cfg& config() const { return cfg_; }
  const std::vector<std::string>& vocab() const { return vocab_; }
  // the parameters as the reference's RnnParams<float> (downloaded)
  template <class Params>
  void params(Params& out) const {
    model_.download(out);
  }
  const std::vector<EpochLog>& logs() const { return logs_; }
  int epoch() const { return epoch_; }
  double eta() const { return eta_; }
  double best_ppl() const { return best_ppl_; }
  double initial_ppl() const { return initial_ppl_; }
  Model& model() { return model_; }

  double validate() {
    struct S { const std::vector<std::uint32_t>& ids; } s{valid_};
    return sharded_perplexity(model_, s, cfg_.valid_shards).perplexity;
  }

  // trainer.hpp:233-270
  void train(std::ostream* progress = nullptr) {
    if (initial_ppl_ == 0.0) {
      initial_ppl_ = validate();
      best_ppl_ = initial_ppl_;
      if (progress) *progress << "initial valid ppl " << initial_ppl_ << "\n";
    }
    while (epoch_ < cfg_.max_epochs && bad_epochs_ < 2) {
      const auto t0 = std::chrono::steady_clock::now();
      const std::int64_t L = static_cast<std::int64_t>(train_.size());
      const std::int64_t N = static_cast<std::int64_t>(cfg_.noffset) * cfg_.minibatch;
      const std::int64_t T = cfg_.unroll;
      const std::int64_t rounds = (L + N * T - 1) / (N * T);
      const std::int64_t windows = rounds * cfg_.noffset;
      double loss_sum = 0.0;
      std::uint64_t skipped = 0;
      check(dl_trainer_run(model_.get(), 0, windows, eta_, &loss_sum, &skipped), model_.get());
      const double ppl = validate();
      EpochLog log;
      log.epoch = ++epoch_;
      log.train_loss = windows > 0 ? loss_sum / static_cast<double>(windows) : 0.0;
      log.valid_ppl = ppl;
      log.eta = eta_;
      log.seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      log.tokens_per_sec =
          log.seconds > 0.0 ? static_cast<double>(rounds * N * T) / log.seconds : 0.0;
      log.skipped_updates = skipped;
      logs_.push_back(log);
      if (progress)
        *progress << "epoch " << log.epoch << " loss " << log.train_loss << " valid ppl " << ppl
                  << " eta " << log.eta << "\n";
      if (ppl > cfg_.divergence_factor * initial_ppl_)
        throw DataError("trainer: diverged (validation perplexity " + std::to_string(ppl) +
                        " vs initial " + std::to_string(initial_ppl_) + ")");
      if (ppl < best_ppl_) {
        best_ppl_ = ppl;
        bad_epochs_ = 0;
      } else {
        ++bad_epochs_;
        eta_ *= 0.5;
      }
    }
  }

  // RTRN (trainer.hpp:274-292, config echo :412-432), byte-compatible with
  // the reference's Trainer::save_checkpoint.
  void save_checkpoint(std::ostream& os) const {
    const std::int64_t V = model_.vocab(), H = model_.hidden();
    const std::int64_t N = static_cast<std::int64_t>(cfg_.noffset) * cfg_.minibatch;
    std::vector<std::int64_t> cur(N);
    std::vector<float> hid(N * H);
    check(dl_trainer_get_state(model_.get(), cur.data(), hid.data()), model_.get());
    std::vector<float> w_in(V * H), w_rec(H * H), w_out(V * H), m_rec(H * H), m_in(V), m_out(V);
    check(dl_get_params(model_.get(), w_in.data(), w_rec.data(), w_out.data()), model_.get());
    model_.get_opt(m_rec.data(), m_in.data(), m_out.data());
    os.write("RTRN", 4);
    io::u32(os, 1);
    io::u64(os, static_cast<std::uint64_t>(cfg_.nstate));
    io::u64(os, static_cast<std::uint64_t>(cfg_.nproj));
    io::u32(os, static_cast<std::uint32_t>(cfg_.noffset));
    io::u32(os, static_cast<std::uint32_t>(cfg_.minibatch));
    io::u32(os, static_cast<std::uint32_t>(cfg_.unroll));
    io::f64(os, cfg_.eta);
    io::f64(os, cfg_.rho);
    io::f64(os, cfg_.eps);
    io::f64(os, cfg_.clip);
    io::u8(os, static_cast<std::uint8_t>(cfg_.mode));
    io::u32(os, static_cast<std::uint32_t>(cfg_.nce_k));
    io::f64(os, cfg_.noise_floor);
    io::u32(os, static_cast<std::uint32_t>(cfg_.max_epochs));
    io::u64(os, cfg_.seed);
    io::u8(os, static_cast<std::uint8_t>(cfg_.act));
    io::f64(os, cfg_.divergence_factor);
    io::u64(os, static_cast<std::uint64_t>(cfg_.valid_limit));
    io::u32(os, static_cast<std::uint32_t>(cfg_.valid_shards));
    io::f64(os, cfg_.init_range);
    io::u32(os, static_cast<std::uint32_t>(epoch_));
    io::f64(os, eta_);
    io::f64(os, best_ppl_);
    io::u32(os, static_cast<std::uint32_t>(bad_epochs_));
    io::f64(os, initial_ppl_);
    std::ostringstream rs;
    // NCE draws advanced the library's generator; softmax mode never draws
    // (the freshly seeded one)
    rs << (static_cast<int>(cfg_.mode) == 0 ? library_rng() : rng_);
    io::str(os, rs.str());
    io::u64(os, static_cast<std::uint64_t>(N));
    for (std::int64_t c : cur) io::u64(os, static_cast<std::uint64_t>(c));
    for (float x : hid) io::f32(os, x);
    write_params(os, V, H, static_cast<int>(cfg_.act), w_in.data(), w_rec.data(), w_out.data(),
                 vocab_);
    write_rmsprop(os, V, H, cfg_.rho, cfg_.eps, m_rec.data(), m_in.data(), m_out.data());
    os.write("TEND", 4);
  }

  // trainer.hpp:300-336: a checkpoint written with an identical
  // configuration (max_epochs may differ) and streams; training then
  // continues as if uninterrupted.  DataError on any mismatch.
  void load_checkpoint(std::istream& is) {
    io::magic(is, "RTRN", "trainer checkpoint");
    const std::uint32_t version = io::get_u32(is);
    if (version != 1) throw DataError("trainer checkpoint: unsupported version " +
                                      std::to_string(version));
    const bool ok =
        io::get_u64(is) == static_cast<std::uint64_t>(cfg_.nstate) &&
        io::get_u64(is) == static_cast<std::uint64_t>(cfg_.nproj) &&
        io::get_u32(is) == static_cast<std::uint32_t>(cfg_.noffset) &&
        io::get_u32(is) == static_cast<std::uint32_t>(cfg_.minibatch) &&
        io::get_u32(is) == static_cast<std::uint32_t>(cfg_.unroll) &&
        io::get_f64(is) == cfg_.eta && io::get_f64(is) == cfg_.rho &&
        io::get_f64(is) == cfg_.eps && io::get_f64(is) == cfg_.clip &&
        io::get_u8(is) == static_cast<std::uint8_t>(cfg_.mode) &&
        io::get_u32(is) == static_cast<std::uint32_t>(cfg_.nce_k) &&
        io::get_f64(is) == cfg_.noise_floor && (static_cast<void>(io::get_u32(is)), true) &&
        io::get_u64(is) == static_cast<std::uint64_t>(cfg_.seed) &&
        io::get_u8(is) == static_cast<std::uint8_t>(cfg_.act) &&
        io::get_f64(is) == cfg_.divergence_factor &&
        io::get_u64(is) == static_cast<std::uint64_t>(cfg_.valid_limit) &&
        io::get_u32(is) == static_cast<std::uint32_t>(cfg_.valid_shards) &&
        io::get_f64(is) == cfg_.init_range;
    if (!ok) throw DataError("trainer checkpoint: configuration does not match this run");
    const int epoch = static_cast<int>(io::get_u32(is));
    const double eta = io::get_f64(is), best = io::get_f64(is);
    const int bad = static_cast<int>(io::get_u32(is));
    const double initial = io::get_f64(is);
    std::mt19937_64 rng;
    {
      std::istringstream rs(io::get_str(is));
      rs >> rng;
      if (rs.fail()) throw DataError("trainer checkpoint: bad generator state");
    }
    const std::int64_t V = model_.vocab(), H = model_.hidden();
    const std::int64_t N = static_cast<std::int64_t>(cfg_.noffset) * cfg_.minibatch;
    if (io::get_u64(is) != static_cast<std::uint64_t>(N))
      throw DataError("trainer checkpoint: cursor count mismatch");
    std::vector<std::int64_t> cur(N);
    const std::int64_t L = static_cast<std::int64_t>(train_.size());
    for (auto& c : cur) {
      c = static_cast<std::int64_t>(io::get_u64(is));
      if (c < 0 || c >= L) throw DataError("trainer checkpoint: cursor out of range");
    }
    std::vector<float> hid(N * H);
    for (auto& x : hid) x = io::get_f32(is);
    // RNLM (rnn.hpp:283-308), W_out stored H x V
    io::magic(is, "RNLM", "rnn checkpoint");
    if (io::get_u32(is) != 1) throw DataError("rnn checkpoint: unsupported version");
    const std::int64_t v = static_cast<std::int64_t>(io::get_u64(is));
    const std::int64_t h = static_cast<std::int64_t>(io::get_u64(is));
    if (v != V || h != H) throw DataError("trainer checkpoint: model shape mismatch");
    io::get_u8(is);  // activation (part of the configuration echo)
    std::vector<float> w_in(V * H), w_rec(H * H), w_out(V * H);
    for (auto& x : w_in) x = io::get_f32(is);
    for (auto& x : w_rec) x = io::get_f32(is);
    for (std::int64_t i = 0; i < H; ++i)
      for (std::int64_t w = 0; w < V; ++w) w_out[w * H + i] = io::get_f32(is);
    if (io::get_u64(is) != static_cast<std::uint64_t>(V))
      throw DataError("rnn checkpoint: vocabulary size mismatch");
    for (std::int64_t i = 0; i < V; ++i)
      if (io::get_str(is) != vocab_[static_cast<std::size_t>(i)])
        throw DataError("trainer checkpoint: vocabulary mismatch");
    // ROPT (rmsprop.hpp:151-166)
    io::magic(is, "ROPT", "rmsprop state");
    if (io::get_u32(is) != 1) throw DataError("rmsprop state: unsupported version");
    if (io::get_u64(is) != static_cast<std::uint64_t>(V) ||
        io::get_u64(is) != static_cast<std::uint64_t>(H))
      throw DataError("trainer checkpoint: model shape mismatch");
    const double rho = io::get_f64(is), eps = io::get_f64(is);
    std::vector<float> m_rec(H * H), m_in(V), m_out(V);
    for (auto& x : m_rec) x = io::get_f32(is);
    for (auto& x : m_in) x = io::get_f32(is);
    for (auto& x : m_out) x = io::get_f32(is);
    io::magic(is, "TEND", "trainer checkpoint trailer");
    check(dl_trainer_set_state(model_.get(), cur.data(), hid.data()), model_.get());
    check(dl_set_params(model_.get(), w_in.data(), w_rec.data(), w_out.data()), model_.get());
    model_.set_opt(m_rec.data(), m_in.data(), m_out.data(), rho, eps);
    rng_ = rng;
    if (static_cast<int>(cfg_.mode) == 0) put_rng();
    epoch_ = epoch;
    eta_ = eta;
    best_ppl_ = best;
    bad_epochs_ = bad;
    initial_ppl_ = initial;
  }

  void load_checkpoint(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw DataError("cannot open input file: " + path);
    load_checkpoint(in);
  }

  void save_checkpoint(const std::string& path) const {
    const std::string tmp = path + ".tmp";
    {
      std::ofstream out(tmp, std::ios::binary);
      if (!out) throw DataError("cannot open output file: " + tmp);
      save_checkpoint(out);
      out.flush();
      if (!out) throw DataError("write failed: " + tmp);
    }
    if (std::rename(tmp.c_str(), path.c_str()) != 0) throw DataError("rename failed: " + path);
  }

 private:
  Cfg cfg_;
  std::vector<std::string> vocab_;
  std::vector<std::uint32_t> train_;
  std::vector<std::uint32_t> valid_;
  mutable Model model_;
  std::mt19937_64 rng_;

  // rng_ <-> the library's generator (312 words + position, stream order)
  void put_rng() {
    std::stringstream ss;
    ss << rng_;
    std::uint64_t st[313];
    for (auto& v : st) ss >> v;
    check(dl_set_rng_state(model_.get(), st), model_.get());
  }
  std::mt19937_64 library_rng() const {
    std::uint64_t st[313];
    check(dl_get_rng_state(model_.get(), st), model_.get());
    std::stringstream ss;
    for (auto v : st) ss << v << ' ';
    std::mt19937_64 r;
    ss >> r;
    return r;
  }
  std::vector<EpochLog> logs_;
  int epoch_ = 0;
  int bad_epochs_ = 0;
  double eta_ = 0.0;
  double best_ppl_ = 0.0;
  double initial_ppl_ = 0.0;
};

// ---------------------------------------------------------------------
// Minimal stand-ins with the reference's field names, for programs that do
// not include the reference headers.
namespace lite {
struct MatF {
  std::int64_t rows = 0, cols = 0;
  std::vector<float> a;
  MatF() = default;
  MatF(std::int64_t r, std::int64_t c, float v = 0.f) : rows(r), cols(c), a(r * c, v) {}
};
struct RnnParams {
  std::int64_t v = 0, h = 0;
  int act = 0;
  MatF w_in, w_rec, w_out;
  RnnParams(std::int64_t v_, std::int64_t h_, int a = 0)
      : v(v_), h(h_), act(a), w_in(v_, h_), w_rec(h_, h_), w_out(v_, h_) {}
  // rnn.hpp:79-83 + rng.hpp:37-44
  void init_uniform(std::uint64_t seed, double range = 0.1) {
    std::mt19937_64 rng(seed);
    for (MatF* m : {&w_in, &w_rec, &w_out})
      for (float& x : m->a)
        x = static_cast<float>(-range + 2 * range * (static_cast<double>(rng() >> 11) * 0x1.0p-53));
  }
};
struct IdStream {
  std::vector<std::uint32_t> ids;
};
struct WindowBatch {
  std::int64_t T = 0, B = 0;
  std::vector<std::uint32_t> inputs, targets;
  std::vector<std::uint8_t> weights;
};
struct TrainConfig {  // trainer.hpp:43-93 defaults (mode 0 = LossMode::kNce)
  std::int64_t nstate = 256, nproj = 0;
  int noffset = 128, minibatch = 8, unroll = 16;
  double eta = 1e-3, rho = 0.9995, eps = 1e-6, clip = 1.0;
  int mode = 0, nce_k = 64;
  double noise_floor = 1e-8;
  int max_epochs = 20;
  std::uint64_t seed = 1;
  int act = 0;
  double divergence_factor = 10.0;
  std::int64_t valid_limit = 0;
  int valid_shards = 8;
  double init_range = 0.1;
  int threads = 1;
  void validate() const {
    if (nstate < 1 || noffset < 1 || minibatch < 1 || unroll < 1 || !(eta > 0.0) ||
        !(rho > 0.0 && rho < 1.0) || !(eps > 0.0) || !(clip > 0.0) || max_epochs < 1 ||
        !(divergence_factor > 1.0) || valid_limit < 0 || valid_shards < 1)
      throw std::invalid_argument("config: invalid training configuration");
  }
};
}  // namespace lite

}  // namespace b200
}  // namespace desklm

#endif  // DESKLM_B200_GPU_HPP
