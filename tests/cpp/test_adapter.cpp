// test_adapter.cpp — drives the reference-side binding logic (include/rtn_adapter.hpp,
// the body of INTEGRATION.md's MlpBatchedEval replacement) through the C-ABI and
// checks it against the fp64 oracle (test infrastructure, oracle/).
//
//   ./test_adapter            full checks (needs a B200)
//   ./test_adapter --no-device  only that every device entry fails loudly (RTN_ECUDA) without a GPU
//
// Scenarios, each a bug of the round-1 adapter sketch or a reference test re-expressed:
//   1. one thread interleaves two different models: each call evaluates its own
//      network (the sketch reused one thread_local context for every model);
//   2. a Hessian call after Jacobian calls on the same model (the sketch fixed
//      max_order at the first call);
//   3. a model destroyed and a different one built in its place: no stale
//      weights (the sketch keyed its device cache by object address);
//   4. capacity growth K = 10 -> 5000 -> 10;
//   5. two threads on one model (one context each);
//   6. batch == single bit for bit, order 2, {6,32,32,4}, K = 13
//      (proj/tests/test_neural.cpp:119-145);
//   7. error mapping: feature-dim mismatch -> RTN_EDOMAIN (neural.cpp:230-232),
//      ReLU Hessian -> RTN_EUNSUPPORTED (neural.cpp:176-177).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "resmpc_oracle.h"
#include "rtn_adapter.hpp"

namespace {

int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(c)) {                                                         \
      ++g_fail;                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
    }                                                                   \
  } while (0)

rtn_adapter::ModelDesc Desc(const oracle::MlpModel& m) {
  rtn_adapter::ModelDesc d;
  d.sizes = m.layer_sizes;
  d.activation = static_cast<int>(m.activation);
  for (size_t l = 0; l < m.weights.size(); ++l) {
    d.W.push_back(m.weights[l].data());
    d.b.push_back(m.biases[l].data());
  }
  d.in_mean = m.in_mean.data();
  d.in_scale = m.in_scale.data();
  d.out_mean = m.out_mean.data();
  d.out_scale = m.out_scale.data();
  return d;
}

oracle::MlpModel Net(std::vector<int> sizes, oracle::Activation act, unsigned long long seed, double gain) {
  std::mt19937_64 rng(seed);
  oracle::MlpModel m = oracle::RandomNet(rng, sizes, act, true);
  for (size_t l = 0; l + 1 < m.weights.size(); ++l)
    for (double& w : m.weights[l].v) w *= gain;
  return m;
}

std::vector<double> Rows(long long k, int n, unsigned long long seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  std::vector<double> z(static_cast<size_t>(k) * n);
  for (double& v : z) v = u(rng);
  return z;
}

// ‖a−b‖∞/(1+‖b‖∞) per node block, max over nodes (proj/tests/oracles.hpp:30-32)
double MaxRel(const std::vector<double>& a, const std::vector<double>& b, long long k) {
  const size_t blk = a.size() / static_cast<size_t>(k);
  double worst = 0;
  for (long long i = 0; i < k; ++i) {
    double num = 0, den = 0;
    for (size_t j = 0; j < blk; ++j) {
      num = std::max(num, std::fabs(a[i * blk + j] - b[i * blk + j]));
      den = std::max(den, std::fabs(b[i * blk + j]));
    }
    worst = std::max(worst, num / (1 + den));
  }
  return worst;
}

// One call through the adapter vs the oracle; returns the max error over f, J (, H).
double Compare(rtn_adapter::DeviceModel& dm, const oracle::MlpModel& om, long long k, int order, unsigned long long seed) {
  const int in = om.input_dim(), out = om.output_dim();
  const std::vector<double> z = Rows(k, in, seed);
  std::vector<double> f(k * out), j(k * out * in), h(order == 2 ? k * out * in * in : 0);
  dm.Prepare(z.data(), k, in, order, f.data(), j.data(), order == 2 ? h.data() : nullptr);
  const oracle::BatchEval ref = oracle::MlpBatchedEval(om, z.data(), k,
                                                       order == 2 ? oracle::EvalOrder::kHessian
                                                                  : oracle::EvalOrder::kJacobian, 1);
  double e = std::max(MaxRel(f, ref.values, k), MaxRel(j, ref.jac, k));
  if (order == 2) e = std::max(e, MaxRel(h, ref.hess, k));
  return e;
}

int NoDevice() {
  // Without a B200 every device entry returns RTN_ECUDA: there is no CPU fallback.
  oracle::MlpModel om = Net({6, 32, 32, 4}, oracle::Activation::kTanh, 1, 1.0);
  try {
    rtn_adapter::DeviceModel dm(Desc(om));
    CHECK(false);
  } catch (const rtn_adapter::Status& s) {
    CHECK(s.code == RTN_ECUDA);
  }
  // argument validation still maps the reference's ConfigError before any device work
  oracle::MlpModel bad = om;
  bad.in_scale[0] = 0.0;
  try {
    rtn_adapter::DeviceModel dm(Desc(bad));
    CHECK(false);
  } catch (const rtn_adapter::Status& s) {
    CHECK(s.code == RTN_ECONFIG);
  }
  std::printf("test_adapter --no-device: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--no-device") == 0) return NoDevice();
  using oracle::Activation;
  const double tol = 1e-3;  // TF32 mode on these nets (the adapter default)

  // 1. interleaved models on one thread
  oracle::MlpModel a = Net({17, 64, 64, 6}, Activation::kTanh, 11, 2.0);
  oracle::MlpModel b = Net({17, 128, 128, 128, 6}, Activation::kSilu, 12, 1.5);
  {
    rtn_adapter::DeviceModel da(Desc(a)), db(Desc(b));
    for (int it = 0; it < 3; ++it) {
      CHECK(Compare(da, a, 20, 1, 100 + it) < tol);
      CHECK(Compare(db, b, 20, 1, 200 + it) < tol);
    }
    // 2. Hessians after Jacobians on the same model (and back)
    CHECK(da.max_order() == 2);
    CHECK(Compare(da, a, 20, 2, 300) < tol);
    CHECK(Compare(da, a, 20, 1, 301) < tol);
    // 4. capacity growth
    CHECK(Compare(db, b, 10, 1, 400) < tol);
    CHECK(Compare(db, b, 5000, 1, 401) < tol);
    CHECK(Compare(db, b, 10, 1, 402) < tol);
  }
  // 3. destroy a model, build a different one of the same shape in its place
  for (int gen = 0; gen < 4; ++gen) {
    oracle::MlpModel m = Net({17, 64, 64, 6}, Activation::kTanh, 500 + gen, 2.0);
    auto dm = std::make_unique<rtn_adapter::DeviceModel>(Desc(m));
    CHECK(Compare(*dm, m, 16, 1, 600 + gen) < tol);
  }
  // 5. two threads, one model
  {
    rtn_adapter::DeviceModel db(Desc(b));
    double e[2] = {1, 1};
    std::thread t0([&] { e[0] = Compare(db, b, 257, 1, 700); });
    std::thread t1([&] { e[1] = Compare(db, b, 513, 1, 701); });
    t0.join();
    t1.join();
    CHECK(e[0] < tol && e[1] < tol);
  }
  // 6. batch == single bitwise at order 2 (test_neural.cpp:119-145)
  {
    oracle::MlpModel m = Net({6, 32, 32, 4}, Activation::kTanh, 23, 1.0);
    rtn_adapter::DeviceModel dm(Desc(m));
    const long long k = 13;
    const std::vector<double> z = Rows(k, 6, 23);
    std::vector<double> f(k * 4), j(k * 4 * 6), h(k * 4 * 36);
    dm.Prepare(z.data(), k, 6, 2, f.data(), j.data(), h.data());
    bool same = true;
    for (long long i = 0; i < k; ++i) {
      std::vector<double> f1(4), j1(24), h1(144);
      dm.Prepare(z.data() + i * 6, 1, 6, 2, f1.data(), j1.data(), h1.data());
      same = same && std::memcmp(f1.data(), f.data() + i * 4, 4 * 8) == 0 &&
             std::memcmp(j1.data(), j.data() + i * 24, 24 * 8) == 0 &&
             std::memcmp(h1.data(), h.data() + i * 144, 144 * 8) == 0;
    }
    CHECK(same);
    unsigned long long calls = 0, points = 0;
    dm.Counters(&calls, &points);
    CHECK(calls == 1 + k && points == 2 * k);
  }
  // 7. error mapping
  {
    rtn_adapter::DeviceModel da(Desc(a));
    std::vector<double> z(5 * 16), f(5 * 6), j(5 * 6 * 17);
    try {
      da.Prepare(z.data(), 5, 16, 1, f.data(), j.data(), nullptr);
      CHECK(false);
    } catch (const rtn_adapter::Status& s) {
      CHECK(s.code == RTN_EDOMAIN);
    }
    oracle::MlpModel r = Net({17, 32, 6}, Activation::kRelu, 7, 1.0);
    rtn_adapter::DeviceModel dr(Desc(r));
    CHECK(dr.max_order() == 1);
    std::vector<double> h(5 * 6 * 17 * 17), zr(5 * 17);
    try {
      dr.Prepare(zr.data(), 5, 17, 2, f.data(), j.data(), h.data());
      CHECK(false);
    } catch (const rtn_adapter::Status& s) {
      CHECK(s.code == RTN_EUNSUPPORTED);
    }
  }
  std::printf("test_adapter: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
