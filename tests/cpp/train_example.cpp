// C++ host-API example / test driver: trains the RNNLM through
// include/desklm_b200/gpu.hpp exactly as a reference user would drive
// desklm::Trainer<StandardTraits>, then writes the RTRN checkpoint and the
// epoch log.  Inputs come from files written by tests/test_cpp_api.py.
//
//   train_example DIR V H NOFFSET MINIBATCH UNROLL EPOCHS ETA PRECISION
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "desklm_b200/gpu.hpp"

namespace b2 = desklm::b200;

template <class T>
std::vector<T> slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary | std::ios::ate);
  if (!in) throw std::runtime_error("cannot open " + path);
  const std::size_t n = static_cast<std::size_t>(in.tellg());
  std::vector<T> v(n / sizeof(T));
  in.seekg(0);
  in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n));
  return v;
}

int main(int argc, char** argv) {
  if (argc != 10) {
    std::cerr << "usage: train_example DIR V H NOFFSET MINIBATCH UNROLL EPOCHS ETA fp32|bf16\n";
    return 1;
  }
  try {
    const std::string dir = argv[1];
    const long V = std::stol(argv[2]), H = std::stol(argv[3]);
    b2::lite::TrainConfig cfg;
    cfg.nstate = H;
    cfg.noffset = std::stoi(argv[4]);
    cfg.minibatch = std::stoi(argv[5]);
    cfg.unroll = std::stoi(argv[6]);
    cfg.max_epochs = std::stoi(argv[7]);
    cfg.eta = std::stod(argv[8]);
    cfg.mode = 1;  // exact softmax (the reference default is NCE, trainer.hpp:53)
    const auto prec = std::string(argv[9]) == "bf16" ? b2::Precision::kBf16 : b2::Precision::kFp32;
    b2::lite::RnnParams p(V, H);
    const auto w = slurp<float>(dir + "/params.f32");
    std::copy(w.begin(), w.begin() + V * H, p.w_in.a.begin());
    std::copy(w.begin() + V * H, w.begin() + V * H + H * H, p.w_rec.a.begin());
    std::copy(w.begin() + V * H + H * H, w.end(), p.w_out.a.begin());
    b2::lite::IdStream train{slurp<std::uint32_t>(dir + "/train.u32")};
    b2::lite::IdStream valid{slurp<std::uint32_t>(dir + "/valid.u32")};
    std::vector<std::string> vocab = {"<unk>", "<s>", "</s>"};
    for (long i = 3; i < V; ++i) vocab.push_back("w" + std::to_string(i));
    b2::Trainer<b2::lite::TrainConfig> tr(cfg, p, vocab, train, valid, prec);
    tr.train(&std::cerr);
    tr.save_checkpoint(dir + "/ckpt.rtrn");
    {
      // load_checkpoint (trainer.hpp:300-336) round trip: a fresh trainer
      // restored from the file writes the same bytes
      b2::Trainer<b2::lite::TrainConfig> again(cfg, p, vocab, train, valid, prec);
      again.load_checkpoint(dir + "/ckpt.rtrn");
      again.save_checkpoint(dir + "/ckpt2.rtrn");
    }
    std::ofstream log(dir + "/logs.csv");
    log.precision(17);
    log << tr.initial_ppl() << "\n";
    for (const auto& l : tr.logs())
      log << l.epoch << "," << l.train_loss << "," << l.valid_ppl << "," << l.eta << ","
          << l.skipped_updates << "\n";
    // the free-function API on a fresh model: one window + update + scoring
    b2::Model m(p, prec);
    b2::lite::WindowBatch wb;
    wb.T = cfg.unroll;
    wb.B = cfg.minibatch;
    for (long i = 0; i < wb.T * wb.B; ++i) {
      wb.inputs.push_back(train.ids[i]);
      wb.targets.push_back(train.ids[i + 1]);
      wb.weights.push_back(train.ids[i + 1] == 1 ? 0 : 1);
    }
    b2::lite::MatF h0(wb.B, H, 0.5f), hf;
    const auto r = b2::bptt_run(m, wb, h0, &hf, 1.0 / double(wb.T * wb.B), 1.0f);
    const bool ok = b2::rmsprop_update(m, 0.05);
    const auto pr = b2::sharded_perplexity(m, valid, 8);
    log << r.loss << "," << r.positions << "," << ok << "," << pr.perplexity << ","
        << pr.predicted << "\n";
    return 0;
  } catch (const std::invalid_argument& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  }
}
