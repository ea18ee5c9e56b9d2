// oracle/ref_bench.cpp -- CPU BASELINE TIMER, TEST INFRASTRUCTURE ONLY.
//
// Times the unmodified reference (/root/reference/proj/include, read in
// place with -I, nothing copied) on the bench workloads, in-process, with the
// reference's own build flags (-O3 -march=<the GPU host's ISA>, FMA
// contraction allowed, proj/CMakeLists.txt:12-17) and all host threads:
//
//   train: the body of Trainer::run_epoch per window (trainer.hpp:374-397) --
//          bptt_run(StandardAdapter, softmax) + rmsprop_update on resident
//          RnnParams / StandardGrads / RmspropState, windows cut from a
//          random_stream (tests/oracles/helpers.hpp:36-52) at the offset-
//          stream cursors floor(i*L/N) (trainer.hpp:194-195), hidden carried;
//   score: sharded_perplexity (eval.hpp:151-222) over S slices.
//
// Nothing crosses a process or marshalling boundary inside the timed region.
// Output: one JSON object with the per-step wall times.
//
//   ref_bench train V H T B steps warmup threads
//   ref_bench score V H S steps warmup threads
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "desklm/desklm.hpp"
#include "oracles/helpers.hpp"

using namespace desklm;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

static void print(const char* mode, const std::vector<double>& t, int threads, double setup,
                  double loss) {
  std::printf("{\"mode\": \"%s\", \"threads\": %d, \"setup_s\": %.3f, \"check\": %.9g, "
              "\"step_s\": [", mode, threads, setup, loss);
  for (std::size_t i = 0; i < t.size(); ++i) std::printf("%s%.6f", i ? ", " : "", t[i]);
  std::printf("]}\n");
}

int main(int argc, char** argv) {
  if (argc != 9) {
    std::fprintf(stderr, "usage: ref_bench train|score V H T|S B|- steps warmup threads\n");
    return 1;
  }
  const std::string mode = argv[1];
  const std::int64_t V = std::atoll(argv[2]), H = std::atoll(argv[3]);
  const std::int64_t T = std::atoll(argv[4]);
  const std::int64_t B = mode == "train" ? std::atoll(argv[5]) : 0;
  const int steps = std::atoi(argv[6]), warmup = std::atoi(argv[7]);
  const int threads = std::atoi(argv[8]);
  const auto s0 = Clock::now();
  RnnParams<float> p(V, H, Activation::kSigmoid);
  {
    // random init in init_uniform's range (rnn.hpp:79-83), a cheaper source
    std::mt19937 g(7);
    std::uniform_real_distribution<float> u(-0.1f, 0.1f);
    for (Mat<float>* m : {&p.w_in, &p.w_rec, &p.w_out})
      for (float& x : m->a) x = u(g);
  }
  std::mt19937_64 rng(3001);
  std::vector<double> times;
  if (mode == "train") {
    const std::int64_t N = 8 * B;  // noffset 8 groups of B streams
    const IdStream stream = testutil::random_stream(rng, static_cast<std::size_t>(V),
                                          static_cast<std::size_t>(std::max<std::int64_t>(
                                              N * T * (steps + warmup + 2), 1 << 20)));
    const auto& ids = stream.ids;
    const std::int64_t L = static_cast<std::int64_t>(ids.size());
    std::vector<std::int64_t> cursors(N);
    for (std::int64_t i = 0; i < N; ++i) cursors[i] = i * L / N;
    Mat<float> hidden(N, H);
    hidden.fill(0.5f);
    RmspropState opt(V, H, 0.9995, 1e-6);
    StandardGrads<float> grads;
    WindowBatch wb;
    wb.resize(T, B);
    Mat<float> h0(B, H), h_final;
    BpttOptions<float> o;
    o.mode = LossMode::kSoftmax;
    o.loss_scale = 1.0 / static_cast<double>(B * T);
    o.clip = 1.0f;
    o.threads = threads;
    const double setup = secs(s0, Clock::now());
    double loss = 0.0;
    for (int w = 0; w < steps + warmup; ++w) {
      const std::int64_t g0 = (w % 8) * B;
      for (std::int64_t t = 0; t < T; ++t)
        for (std::int64_t b = 0; b < B; ++b) {
          const std::int64_t pos = cursors[g0 + b] + t;
          const std::size_t i = static_cast<std::size_t>(t * B + b);
          wb.inputs[i] = ids[static_cast<std::size_t>(pos % L)];
          wb.targets[i] = ids[static_cast<std::size_t>((pos + 1) % L)];
          wb.weights[i] = wb.targets[i] == Vocabulary::kBosId ? 0 : 1;
        }
      for (std::int64_t b = 0; b < B; ++b)
        std::copy_n(hidden.row(g0 + b), H, h0.row(b));
      const auto t0 = Clock::now();
      StandardAdapter<float> a(p);
      const BpttResult r = bptt_run(a, wb, h0, &grads, &h_final, o);
      rmsprop_update(p, grads, opt, 1e-3);
      const auto t1 = Clock::now();
      for (std::int64_t b = 0; b < B; ++b) {
        std::copy_n(h_final.row(b), H, hidden.row(g0 + b));
        cursors[g0 + b] = (cursors[g0 + b] + T) % L;
      }
      loss += r.loss;
      if (w >= warmup) times.push_back(secs(t0, t1));
    }
    print("train", times, threads, setup, loss);
  } else {
    // S = T slices; one call per timed step block: sharded_perplexity over
    // S * (k + 1) ids walks k lock-step scoring steps
    const std::int64_t S = T;
    const IdStream stream = testutil::random_stream(rng, static_cast<std::size_t>(V),
                                          static_cast<std::size_t>(S * (steps + warmup + 2)));
    const double setup = secs(s0, Clock::now());
    StandardAdapter<float> a(p);
    auto run = [&](int k) {
      IdStream s;
      s.ids.assign(stream.ids.begin(), stream.ids.begin() + S * (k + 1));
      const auto t0 = Clock::now();
      const PerplexityResult r = sharded_perplexity(a, s, static_cast<int>(S),
                                                    Vocabulary::kBosId, threads);
      return std::make_pair(secs(t0, Clock::now()), r.total_logprob);
    };
    if (warmup > 0) run(warmup);
    const auto [dt, tl] = run(steps);
    for (int i = 0; i < steps; ++i) times.push_back(dt / steps);
    print("score", times, threads, setup, tl);
  }
  return 0;
}
