// desklm_b200 -- the reference CLI's training and scoring subcommands
// (tools/desklm.cpp rnn-train :509-592, rnn-ppl :594-608, rescore :717-744)
// on the B200 path, built from the reference's headers (file formats,
// Trainer, readers) plus include/desklm_b200/traits.hpp:
//
//   desklm_b200 rnn-train --train IDS --valid IDS --vocab FILE --out MODEL
//                         [--checkpoint F] [--resume F] [--log CSV] [--nstate H]
//                         [--nproj P] [--noffset N] [--minibatch B] [--unroll T]
//                         [--eta X] [--rho X] [--eps X] [--clip X] [--mode nce|softmax]
//                         [--nce-k K] [--noise-floor X] [--max-epochs E]
//                         [--act sigmoid|tanh] [--divergence-factor X]
//                         [--valid-limit N] [--valid-shards S] [--init-range X]
//   desklm_b200 rnn-ppl   --model MODEL (--ids IDS | --text TXT) [--shards S]
//   desklm_b200 rescore   --nbest FILE --model MODEL [--arpa ARPA] [--out F]
//                         [--lambda X] [--lm-scale X] [--wip X] [--fast]
//   global: --seed N --precision fp32|bf16 --device D --quiet
//
// Models are dispatched on their magic like the reference's with_model
// (RNLM -> the standard device model, RNBL -> the bottleneck device model,
// RNQZ -> dequantised on the device).  rnn-train runs the reference's
// desklm::Trainer<GpuStandardTraits> (or <GpuBottleneckTraits> with --nproj),
// so epochs, schedule, checkpoints and outputs are the reference's.
// Exit codes as the reference's main (:1373-1391): 1 usage, 2 data error.
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>

#include "desklm/arpa.hpp"
#include "desklm/desklm.hpp"
#include "desklm_b200/traits.hpp"

using namespace desklm;
namespace b2 = desklm::b200;

namespace {

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string str(const std::string& k, const std::string& d = "") const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  double num(const std::string& k, double d) const {
    return has(k) ? std::stod(kv.at(k)) : d;
  }
  long long integer(const std::string& k, long long d) const {
    return has(k) ? std::stoll(kv.at(k)) : d;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) throw std::invalid_argument(cmd + ": --" + k + " is required");
    return kv.at(k);
  }
};

Args parse(int argc, char** argv) {
  if (argc < 2) throw std::invalid_argument("usage: desklm_b200 rnn-train|rnn-ppl|rescore ...");
  Args a;
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument: " + k);
    k = k.substr(2);
    if (k == "fast" || k == "quiet") {
      a.kv[k] = "1";
      continue;
    }
    if (i + 1 >= argc) throw std::invalid_argument("--" + k + " needs a value");
    a.kv[k] = argv[++i];
  }
  return a;
}

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open input file: " + path);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void spit(const std::string& path, const std::string& bytes) {
  if (path == "-") {
    std::cout << bytes;
    return;
  }
  atomic_write(path, [&](std::ostream& os) { os << bytes; });
}

b2::Precision precision(const Args& a) {
  const std::string p = a.str("precision", "bf16");
  if (p == "bf16") return b2::Precision::kBf16;
  if (p == "fp32") return b2::Precision::kFp32;
  throw std::invalid_argument("--precision: fp32 or bf16");
}

Vocabulary load_vocab(const std::string& path) {
  std::istringstream is(slurp(path));
  return Vocabulary::read(is);
}

IdStream load_ids(const std::string& path, std::size_t v) {
  std::istringstream is(slurp(path));
  return read_id_stream(is, v);
}

IdStream eval_stream(const Args& a, const Vocabulary& v) {
  if (a.has("ids") == a.has("text"))
    throw std::invalid_argument("exactly one of --ids / --text");
  if (a.has("ids")) return load_ids(a.str("ids"), v.size());
  return encode(normalize_text(slurp(a.str("text"))), v);
}

// ---------------------------------------------------------------- train
template <class Traits, class Host>
void do_train(const Args& a, TrainConfig tc, Host p0) {
  const Vocabulary vocab = load_vocab(a.need("vocab"));
  const IdStream train = load_ids(a.need("train"), vocab.size());
  const IdStream valid = load_ids(a.need("valid"), vocab.size());
  const int dev = static_cast<int>(a.integer("device", 0));
  typename Traits::Params gp(p0, precision(a), dev);
  Trainer<Traits> trainer(tc, std::move(gp), vocab, train, valid);
  if (a.has("resume")) {
    std::istringstream is(slurp(a.str("resume")));
    trainer.load_checkpoint(is);
  }
  trainer.train(a.has("quiet") ? nullptr : &std::cerr);
  {
    std::ostringstream os;
    Traits::write_params(os, trainer.params(), vocab);
    spit(a.need("out"), os.str());
  }
  if (a.has("checkpoint")) {
    std::ostringstream os;
    trainer.save_checkpoint(os);
    spit(a.str("checkpoint"), os.str());
  }
  if (a.has("log")) {
    std::ostringstream os;
    write_epoch_log(os, trainer.logs());
    spit(a.str("log"), os.str());
  }
  if (!a.has("quiet"))
    std::fprintf(stderr, "rnn-train: %d epochs, best valid ppl %.4f (initial %.4f)\n",
                 trainer.epoch(), trainer.best_ppl(), trainer.initial_ppl());
}

void rnn_train(const Args& a) {
  TrainConfig tc;
  tc.nstate = a.integer("nstate", 256);
  tc.nproj = a.integer("nproj", 0);
  tc.noffset = static_cast<int>(a.integer("noffset", 128));
  tc.minibatch = static_cast<int>(a.integer("minibatch", 8));
  tc.unroll = static_cast<int>(a.integer("unroll", 16));
  tc.eta = a.num("eta", 0.1);  // the CLI default (desklm.cpp:460-486)
  tc.rho = a.num("rho", 0.9995);
  tc.eps = a.num("eps", 1e-6);
  tc.clip = a.num("clip", 1.0);
  const std::string mode = a.str("mode", "nce");
  if (mode != "nce" && mode != "softmax") throw std::invalid_argument("--mode: nce or softmax");
  tc.mode = mode == "nce" ? LossMode::kNce : LossMode::kSoftmax;
  tc.nce_k = static_cast<int>(a.integer("nce-k", 64));
  tc.noise_floor = a.num("noise-floor", 1e-8);
  tc.max_epochs = static_cast<int>(a.integer("max-epochs", 20));
  tc.seed = static_cast<std::uint64_t>(a.integer("seed", 1));
  const std::string act = a.str("act", "sigmoid");
  if (act != "sigmoid" && act != "tanh") throw std::invalid_argument("--act: sigmoid or tanh");
  tc.act = act == "sigmoid" ? Activation::kSigmoid : Activation::kTanh;
  tc.divergence_factor = a.num("divergence-factor", 10.0);
  tc.valid_limit = a.integer("valid-limit", 0);
  tc.valid_shards = static_cast<int>(a.integer("valid-shards", 8));
  tc.init_range = a.num("init-range", 0.1);
  const auto v = static_cast<std::int64_t>(load_vocab(a.need("vocab")).size());
  if (tc.nproj > 0) {
    BottleneckParams<float> p(v, tc.nstate, tc.nproj, tc.act);
    p.init_uniform(tc.seed, tc.init_range);
    do_train<b2::GpuBottleneckTraits>(a, tc, p);
  } else {
    RnnParams<float> p(v, tc.nstate, tc.act);
    p.init_uniform(tc.seed, tc.init_range);
    do_train<b2::GpuStandardTraits>(a, tc, p);
  }
}

// ------------------------------------------------------------------ ppl
void rnn_ppl(const Args& a) {
  const int shards = static_cast<int>(a.integer("shards", 1));
  PerplexityResult r;
  b2::with_gpu_model(
      slurp(a.need("model")), precision(a),
      [&](const auto& m, const Vocabulary& v) {
        const IdStream s = eval_stream(a, v);
        r = shards > 1 ? sharded_perplexity(m, s, shards, v.bos_id(), 1)
                       : rnn_perplexity(m, s, v.bos_id(), 1);
      },
      static_cast<int>(a.integer("device", 0)));
  std::printf("%.6f\n", r.perplexity);
  if (!a.has("quiet")) std::fprintf(stderr, "rnn-ppl: %zu predicted tokens\n", r.predicted);
}

// -------------------------------------------------------------- rescore
void rescore(const Args& a) {
  std::istringstream is(slurp(a.need("nbest")));
  std::vector<NBestUtt> utts = read_nbest(is);
  std::optional<NGramModel> ng;
  if (a.has("arpa")) {
    std::istringstream as(slurp(a.str("arpa")));
    ng = read_arpa(as);
  }
  b2::with_gpu_model(
      slurp(a.need("model")), precision(a),
      [&](const auto& m, const Vocabulary& v) {
        RescoreConfig rc;
        rc.lambda = a.num("lambda", 0.5);
        rc.lm_scale = a.num("lm-scale", 1.0);
        rc.wip = a.num("wip", 0.0);
        rc.fast = a.has("fast");
        rescore_nbest(utts, m, v, ng ? &*ng : nullptr, rc);
      },
      static_cast<int>(a.integer("device", 0)));
  std::ostringstream os;
  write_nbest(os, utts);
  spit(a.str("out", "-"), os.str());
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "rnn-train") rnn_train(a);
    else if (a.cmd == "rnn-ppl") rnn_ppl(a);
    else if (a.cmd == "rescore") rescore(a);
    else throw std::invalid_argument("unknown subcommand: " + a.cmd);
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const DataError& e) {
    std::fprintf(stderr, "data error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
  return 0;
}
