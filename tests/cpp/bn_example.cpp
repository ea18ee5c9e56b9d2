// Bottleneck model through the C++ host API (include/desklm_b200/gpu.hpp):
// a few windows of bptt_run + bottleneck_update, then sharded perplexity and
// the standard model's ln Z samples.  Reads params / windows written by
// tests/test_cpp_api.py, prints one CSV line per result.
//   bn_example <dir> V H P T B windows eta
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "desklm_b200/gpu.hpp"

namespace b200 = desklm::b200;

template <class T>
static std::vector<T> load(const std::string& path, std::size_t n) {
  std::vector<T> v(n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
  if (!f) throw std::runtime_error("short read: " + path);
  return v;
}

struct BnParams {  // the fields BottleneckModel's templates read
  std::int64_t v, h, p;
  int act = 0;
  b200::lite::MatF e, u, w_rec, d;
};

int main(int argc, char** argv) {
  if (argc != 9) return 2;
  const std::string dir = argv[1];
  const std::int64_t V = std::atoll(argv[2]), H = std::atoll(argv[3]), P = std::atoll(argv[4]);
  const std::int64_t T = std::atoll(argv[5]), B = std::atoll(argv[6]);
  const int windows = std::atoi(argv[7]);
  const double eta = std::atof(argv[8]);
  BnParams p;
  p.v = V;
  p.h = H;
  p.p = P;
  const auto flat = load<float>(dir + "/params.f32", V * P + P * H + H * H + H * P);
  std::size_t o = 0;
  for (auto* m : {&p.e, &p.u, &p.w_rec, &p.d}) {
    const std::size_t n = m == &p.e ? V * P : m == &p.u ? P * H : m == &p.w_rec ? H * H : H * P;
    m->a.assign(flat.begin() + o, flat.begin() + o + n);
    o += n;
  }
  const auto ids = load<std::uint32_t>(dir + "/ids.u32", (windows + 1) * T * B + 1);
  b200::BottleneckModel m(p, b200::Precision::kFp32);
  m.set_opt(nullptr, nullptr, nullptr, nullptr, 0.9995, 1e-6);
  b200::lite::MatF h0, hf;
  h0.a.assign(B * H, 0.5f);
  for (int w = 0; w < windows; ++w) {
    b200::lite::WindowBatch wb;
    wb.T = T;
    wb.B = B;
    for (std::int64_t i = 0; i < T * B; ++i) {
      wb.inputs.push_back(ids[w * T * B + i]);
      wb.targets.push_back(ids[w * T * B + i + 1]);
      wb.weights.push_back(ids[w * T * B + i + 1] == 1 ? 0 : 1);
    }
    const b200::BpttResult r = b200::bptt_run(m, wb, h0, &hf, 1.0 / (T * B), 1.0f);
    const bool ok = b200::bottleneck_update(m, eta);
    std::printf("%.17g,%zu,%d\n", r.loss, r.positions, ok ? 1 : 0);
    h0 = hf;
  }
  b200::lite::IdStream valid;
  valid.ids.assign(ids.begin(), ids.end());
  const b200::PerplexityResult pr = b200::sharded_perplexity(m, valid, 8);
  std::printf("%.17g,%zu\n", pr.perplexity, pr.predicted);
  return 0;
}
