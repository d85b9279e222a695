// ORACLE SELF-TEST — pins the restated CPU oracle against the reference's own
// known-answer, finite-difference and contract tests for the hot path:
//   /root/reference/proj/tests/test_neural.cpp:11-152, 231-282
//   /root/reference/proj/tests/test_taylor.cpp:8-135
// with the same seeds, shapes and tolerances, plus SiLU / forward-mode checks
// the reference cannot provide (it has no SiLU). Exit code 0 = all pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "resmpc_oracle.h"

using namespace oracle;
using Vec = std::vector<double>;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                             \
  do {                                                                          \
    ++g_checks;                                                                 \
    if (!(cond)) {                                                              \
      ++g_fail;                                                                 \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                           \
  } while (0)

template <typename E, typename F>
static bool Throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double MaxAbs(const Vec& a) {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::fabs(v));
  return m;
}
static double MaxAbsDiff(const Vec& a, const Vec& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}
// ‖a−b‖∞ / (1 + ‖b‖∞) — proj/tests/oracles.hpp:30-32
static double RelError(const Vec& a, const Vec& b) { return MaxAbsDiff(a, b) / (1.0 + MaxAbs(b)); }
static bool Same(const Vec& a, const Vec& b) { return a.size() == b.size() && MaxAbsDiff(a, b) == 0.0; }

// Central differences, column per input (proj/tests/oracles.hpp:17-28);
// result out x in row-major.
static Vec FdJacobian(const std::function<Vec(const Vec&)>& f, const Vec& x, double h) {
  const Vec f0 = f(x);
  const int out = static_cast<int>(f0.size()), in = static_cast<int>(x.size());
  Vec jac(static_cast<size_t>(out) * in);
  for (int j = 0; j < in; ++j) {
    Vec xp = x, xm = x;
    xp[j] += h;
    xm[j] -= h;
    const Vec a = f(xp), b = f(xm);
    for (int o = 0; o < out; ++o) jac[o * in + j] = (a[o] - b[o]) / (2.0 * h);
  }
  return jac;
}

// A deliberately separate forward pass (plain loops, no shared kernels),
// the role of oracles::NaiveMlpForward (proj/tests/oracles.hpp:57-73).
static Vec NaiveForward(const MlpModel& m, const Vec& z) {
  Vec x(z.size());
  for (size_t k = 0; k < z.size(); ++k) x[k] = (z[k] - m.in_mean[k]) / m.in_scale[k];
  for (size_t l = 0; l < m.weights.size(); ++l) {
    const Mat& w = m.weights[l];
    Vec y(static_cast<size_t>(w.rows));
    for (int j = 0; j < w.rows; ++j) {
      double s = 0.0;
      for (int i = 0; i < w.cols; ++i) s += w(j, i) * x[i];
      y[j] = s + m.biases[l][j];
      if (l + 1 < m.weights.size()) {
        if (m.activation == Activation::kTanh) y[j] = std::tanh(y[j]);
        else if (m.activation == Activation::kRelu) y[j] = std::max(0.0, y[j]);
        else y[j] = y[j] / (1.0 + std::exp(-y[j]));
      }
    }
    x = y;
  }
  for (size_t o = 0; o < x.size(); ++o) x[o] = m.out_scale[o] * x[o] + m.out_mean[o];
  return x;
}

static Vec Normalized(Vec v) {
  double n = 0.0;
  for (double e : v) n += e * e;
  n = std::sqrt(n);
  for (double& e : v) e /= n;
  return v;
}

// ------------------------------------------------------------------- neural

static void TestLinearLayer() {  // test_neural.cpp:11-20
  MlpModel m = MakeMlp({3, 2}, Activation::kTanh, "full", 1);
  m.weights[0].v = {1.0, -2.0, 0.5, 0.0, 3.0, 1.0};
  m.biases[0] = {0.25, -1.0};
  const Vec z = {0.3, -0.7, 2.0};
  const Vec y = MlpForward(m, z);
  const Vec expect = {1.0 * 0.3 - 2.0 * -0.7 + 0.5 * 2.0 + 0.25, 3.0 * -0.7 + 1.0 * 2.0 - 1.0};
  CHECK(MaxAbsDiff(y, expect) < 1e-15);
  CHECK(Same(MlpJacobian(m, z), m.weights[0].v));
}

static void TestZeroWeights() {  // test_neural.cpp:22-32
  MlpModel m = MakeMlp({4, 8, 8, 3}, Activation::kTanh, "full", 2);
  for (auto& w : m.weights) std::fill(w.v.begin(), w.v.end(), 0.0);
  for (auto& b : m.biases) std::fill(b.begin(), b.end(), 0.0);
  std::mt19937_64 rng(5);
  for (int i = 0; i < 10; ++i) {
    const Vec z = RandomVector(rng, 4, -3.0, 3.0);
    CHECK(MaxAbs(MlpForward(m, z)) == 0.0);
    CHECK(MaxAbs(MlpJacobian(m, z)) == 0.0);
  }
}

static void TestForwardVsNaive(Activation act, double tol) {  // test_neural.cpp:34-43
  std::mt19937_64 rng(42);
  for (int t = 0; t < 20; ++t) {
    const MlpModel m = RandomNet(rng, {5, 16, 16, 3}, act);
    const Vec z = RandomVector(rng, 5, -2.0, 2.0);
    CHECK(MaxAbsDiff(MlpForward(m, z), NaiveForward(m, z)) < tol);
  }
}

static void TestJacobianFd(Activation act) {  // test_neural.cpp:45-57
  std::mt19937_64 rng(7);
  double worst = 0.0;
  for (int t = 0; t < 100; ++t) {
    const MlpModel m = RandomNet(rng, {4, 12, 12, 2}, act);
    const Vec z = RandomVector(rng, 4, -1.5, 1.5);
    const Vec fd = FdJacobian([&](const Vec& v) { return MlpForward(m, v); }, z, 1e-5);
    worst = std::max(worst, RelError(MlpJacobian(m, z), fd));
  }
  CHECK(worst < 1e-5);
}

static void TestReluJacobianFd() {  // test_neural.cpp:59-68
  std::mt19937_64 rng(19);
  for (int t = 0; t < 20; ++t) {
    const MlpModel m = RandomNet(rng, {3, 10, 2}, Activation::kRelu);
    const Vec z = RandomVector(rng, 3, -1.0, 1.0);
    const Vec fd = FdJacobian([&](const Vec& v) { return MlpForward(m, v); }, z, 1e-7);
    CHECK(RelError(MlpJacobian(m, z), fd) < 1e-4);
  }
}

static void TestHessians(Activation act) {  // test_neural.cpp:70-117
  {  // linear layer → zero
    MlpModel m = MakeMlp({3, 2}, act, "full", 3);
    CHECK(MaxAbs(MlpHessian(m, {1, 2, 3})) == 0.0);
  }
  {  // scalar closed form: y'' = w2 w1² σ''(pre)
    MlpModel m = MakeMlp({1, 1, 1}, act, "full", 4);
    const double w1 = 0.8, b1 = -0.3, w2 = 1.7, z = 0.45;
    m.weights[0].v = {w1};
    m.biases[0] = {b1};
    m.weights[1].v = {w2};
    const double pre = w1 * z + b1;
    double spp;
    if (act == Activation::kTanh) {
      const double t = std::tanh(pre);
      spp = -2.0 * t * (1.0 - t * t);
    } else {
      const double s = 1.0 / (1.0 + std::exp(-pre));
      spp = s * (1.0 - s) * (2.0 + pre * (1.0 - 2.0 * s));
    }
    const double expected = w2 * w1 * w1 * spp;
    const Vec h = MlpHessian(m, {z});
    CHECK(std::fabs(h[0] - expected) <= 1e-12 * std::max(1.0, std::fabs(expected)));
  }
  {  // random nets: exact symmetry + directional FD of the Jacobian
    std::mt19937_64 rng(31);
    double worst = 0.0;
    for (int t = 0; t < 100; ++t) {
      const MlpModel m = RandomNet(rng, {3, 8, 2}, act);
      const Vec z = RandomVector(rng, 3, -1.0, 1.0);
      const Vec h = MlpHessian(m, z);
      for (int o = 0; o < 2; ++o)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) CHECK(h[(o * 3 + a) * 3 + b] == h[(o * 3 + b) * 3 + a]);
      const Vec dir = Normalized(RandomVector(rng, 3));
      const double step = 1e-5;
      Vec zp = z, zm = z;
      for (int k = 0; k < 3; ++k) {
        zp[k] += step * dir[k];
        zm[k] -= step * dir[k];
      }
      const Vec jp = MlpJacobian(m, zp), jm = MlpJacobian(m, zm);
      for (int o = 0; o < 2; ++o) {
        double num = 0.0, den = 0.0;
        for (int a = 0; a < 3; ++a) {
          double an = 0.0;
          for (int b = 0; b < 3; ++b) an += h[(o * 3 + a) * 3 + b] * dir[b];
          const double fd = (jp[o * 3 + a] - jm[o * 3 + a]) / (2.0 * step);
          num += (an - fd) * (an - fd);
          den += fd * fd;
        }
        worst = std::max(worst, std::sqrt(num) / (1.0 + std::sqrt(den)));
      }
    }
    CHECK(worst < 1e-4);
  }
}

static void TestReluHessianRejected() {  // test_neural.cpp:112-116
  std::mt19937_64 rng(77);
  const MlpModel m = RandomNet(rng, {3, 4, 1}, Activation::kRelu);
  CHECK(Throws<UnsupportedError>([&] { MlpHessian(m, {0, 0, 0}); }));
}

static void TestBatchEqualsSingle(Activation act) {  // test_neural.cpp:119-145
  std::mt19937_64 rng(23);
  const MlpModel m = RandomNet(rng, {6, 32, 32, 4}, act);
  const int k = 13;
  Vec z(static_cast<size_t>(k) * 6);
  for (int i = 0; i < k; ++i) {
    const Vec r = RandomVector(rng, 6, -2.0, 2.0);
    std::copy(r.begin(), r.end(), z.begin() + i * 6);
  }
  std::copy(z.begin(), z.begin() + 6, z.begin() + (k - 1) * 6);
  EvalCounters c;
  const BatchEval b = MlpBatchedEval(m, z.data(), k, 6, EvalOrder::kHessian, 0, &c);
  CHECK(c.batched_calls == 1);
  CHECK(c.batched_points == static_cast<std::uint64_t>(k));
  CHECK(c.value_evals == 0);
  for (int i = 0; i < k; ++i) {
    const Vec zi(z.begin() + i * 6, z.begin() + (i + 1) * 6);
    CHECK(Same(Vec(b.values.begin() + i * 4, b.values.begin() + (i + 1) * 4), MlpForward(m, zi)));
    CHECK(Same(Vec(b.jac.begin() + i * 24, b.jac.begin() + (i + 1) * 24), MlpJacobian(m, zi)));
    CHECK(Same(Vec(b.hess.begin() + i * 144, b.hess.begin() + (i + 1) * 144), MlpHessian(m, zi)));
  }
  CHECK(Same(Vec(b.values.begin(), b.values.begin() + 4),
             Vec(b.values.begin() + (k - 1) * 4, b.values.begin() + k * 4)));
  // pool size does not change the bits (threadpool.hpp:12-15)
  const BatchEval b1 = MlpBatchedEval(m, z.data(), k, 6, EvalOrder::kHessian, 1, nullptr);
  const BatchEval b3 = MlpBatchedEval(m, z.data(), k, 6, EvalOrder::kHessian, 3, nullptr);
  CHECK(Same(b1.values, b3.values) && Same(b1.jac, b3.jac) && Same(b1.hess, b3.hess));
}

static void TestMismatchRejected() {  // test_neural.cpp:147-152
  std::mt19937_64 rng(3);
  const MlpModel m = RandomNet(rng, {4, 8, 2});
  const Vec z(15, 0.0);
  CHECK(Throws<InputDomainError>([&] { MlpBatchedEval(m, z.data(), 3, 5, EvalOrder::kValue); }));
}

static void TestRoundTrip(Activation act) {  // test_neural.cpp:231-257
  std::mt19937_64 rng(55);
  MlpModel m = RandomNet(rng, {7, 10, 3}, act);
  m.input_variant = "a_u";
  m.seed = 1234;
  const std::string path = "/tmp/rtn_oracle_model_" + std::to_string(static_cast<int>(act)) + ".bin";
  SaveModel(m, path);
  const MlpModel r = LoadModel(path);
  CHECK(r.layer_sizes == m.layer_sizes);
  CHECK(r.input_variant == "a_u");
  CHECK(r.seed == 1234);
  CHECK(r.activation == m.activation);
  for (size_t l = 0; l < m.weights.size(); ++l) {
    CHECK(Same(r.weights[l].v, m.weights[l].v));
    CHECK(Same(r.biases[l], m.biases[l]));
  }
  CHECK(Same(r.in_mean, m.in_mean) && Same(r.in_scale, m.in_scale));
  std::mt19937_64 rng2(56);
  for (int i = 0; i < 5; ++i) {
    const Vec z = RandomVector(rng2, 7, -2, 2);
    CHECK(Same(MlpForward(r, z), MlpForward(m, z)));
  }
  std::FILE* side = std::fopen((path + ".json").c_str(), "r");
  CHECK(side != nullptr);
  if (side) std::fclose(side);
}

static void TestArch() {  // test_neural.cpp:277-282
  CHECK(ParseArch("3x32") == std::vector<int>({32, 32, 32}));
  CHECK(ParseArch("18,18") == std::vector<int>({18, 18}));
  CHECK(ParseArch("64") == std::vector<int>({64}));
  CHECK(Throws<ConfigError>([] { ParseArch("0x4"); }));
}

static void TestParamCount() {  // SURVEY §6 note: 12x512, in 17, out 6 → 2,901,510
  std::vector<int> s = {17};
  for (int i = 0; i < 12; ++i) s.push_back(512);
  s.push_back(6);
  const MlpModel m = MakeMlp(s, Activation::kSilu, "full", 12512);
  CHECK(m.ParameterCount() == 2901510);
  CHECK(m.ArchName() == "N-12-512");
}

// New: the forward-mode evaluation (the GPU algorithm) agrees with the
// reverse sweep / forward-over-forward Hessian of the restated reference.
static void TestForwardModeAgrees(Activation act) {
  std::mt19937_64 rng(101);
  double wf = 0, wj = 0, wh = 0;
  for (int t = 0; t < 30; ++t) {
    const MlpModel m = RandomNet(rng, {17, 24, 24, 24, 6}, act);
    const Vec z = RandomVector(rng, 17, -2.0, 2.0);
    Vec f(6), j(6 * 17), h(6 * 17 * 17);
    ForwardModeEval(m, z.data(), f.data(), j.data(), act == Activation::kRelu ? nullptr : h.data());
    wf = std::max(wf, RelError(f, MlpForward(m, z)));
    wj = std::max(wj, RelError(j, MlpJacobian(m, z)));
    if (act != Activation::kRelu) wh = std::max(wh, RelError(h, MlpHessian(m, z)));
  }
  CHECK(wf < 1e-13);
  CHECK(wj < 1e-13);
  CHECK(wh < 1e-12);
}

// New: v1 files stay bit-compatible with the reference's reader semantics
// (tag 0 tanh, anything else relu); SiLU goes to v2 so a v1 reader rejects it.
static void TestFileVersions() {
  MlpModel m = MakeMlp({3, 4, 2}, Activation::kSilu, "full", 9);
  SaveModel(m, "/tmp/rtn_oracle_silu.bin");
  std::FILE* fp = std::fopen("/tmp/rtn_oracle_silu.bin", "rb");
  unsigned char head[9] = {0};
  CHECK(fp && std::fread(head, 1, 9, fp) == 9);
  if (fp) std::fclose(fp);
  CHECK(head[4] == 2 && head[8] == 2);  // version 2, tag 2
  m.activation = Activation::kRelu;
  SaveModel(m, "/tmp/rtn_oracle_relu.bin");
  CHECK(LoadModel("/tmp/rtn_oracle_relu.bin").activation == Activation::kRelu);
}

// ------------------------------------------------------------------- taylor

static void TestPrepareEqualsUnbatched() {  // test_taylor.cpp:8-28
  std::mt19937_64 rng(1);
  const MlpModel m = RandomNet(rng, {4, 16, 3});
  const int n = 10;
  Vec z(static_cast<size_t>(n) * 4);
  for (int k = 0; k < n; ++k) {
    const Vec r = RandomVector(rng, 4, -1, 1);
    std::copy(r.begin(), r.end(), z.begin() + k * 4);
  }
  EvalCounters c;
  const auto a = PrepareNodes(m, z.data(), n, 4, 1, &c);
  CHECK(c.batched_calls == 1 && c.batched_points == 10 && c.value_evals == 0 && c.jacobian_evals == 0);
  CHECK(a.size() == 10);
  for (int k = 0; k < n; ++k) {
    const Vec zk(z.begin() + k * 4, z.begin() + (k + 1) * 4);
    CHECK(a[k].node == k);
    CHECK(Same(a[k].f_bar, MlpForward(m, zk)));
    CHECK(Same(a[k].jac, MlpJacobian(m, zk)));
  }
}

static void TestZeroOutputModel() {  // test_taylor.cpp:30-41
  std::mt19937_64 rng(9);
  MlpModel m = RandomNet(rng, {3, 8, 2}, Activation::kTanh, false);
  std::fill(m.weights.back().v.begin(), m.weights.back().v.end(), 0.0);
  std::fill(m.biases.back().begin(), m.biases.back().end(), 0.0);
  const Vec z = RandomVector(rng, 15, -1, 1);
  for (const auto& a : PrepareNodes(m, z.data(), 5, 3, 1)) {
    CHECK(MaxAbs(a.f_bar) == 0.0);
    CHECK(MaxAbs(a.jac) == 0.0);
  }
}

static void TestIdenticalNodes() {  // test_taylor.cpp:43-56
  std::mt19937_64 rng(2);
  const MlpModel m = RandomNet(rng, {3, 12, 2});
  const Vec row = RandomVector(rng, 3);
  Vec z;
  for (int k = 0; k < 4; ++k) z.insert(z.end(), row.begin(), row.end());
  const auto a = PrepareNodes(m, z.data(), 4, 3, 2);
  for (int k = 1; k < 4; ++k) {
    CHECK(Same(a[k].f_bar, a[0].f_bar));
    CHECK(Same(a[k].jac, a[0].jac));
    CHECK(Same(a[k].hess, a[0].hess));
  }
}

static void TestExpansionPointExact() {  // test_taylor.cpp:58-69
  std::mt19937_64 rng(3);
  const MlpModel m = RandomNet(rng, {4, 10, 2});
  const Vec z = RandomVector(rng, 4);
  for (int order : {1, 2}) {
    const auto a = PrepareNodes(m, z.data(), 1, 4, order);
    Vec y(2), j(8);
    EvalTaylor(4, 2, order, a[0].z0.data(), a[0].f_bar.data(), a[0].jac.data(), a[0].hess.data(), z.data(),
               y.data());
    EvalTaylorJacobian(4, 2, order, a[0].z0.data(), a[0].jac.data(), a[0].hess.data(), z.data(), j.data());
    CHECK(Same(y, a[0].f_bar));
    CHECK(Same(j, a[0].jac));
  }
}

static void TestLinearTaylorExact() {  // test_taylor.cpp:71-85
  MlpModel m = MakeMlp({3, 2}, Activation::kTanh, "full", 7);
  m.weights[0].v = {1.0, 0.5, -2.0, 0.0, 1.5, 0.25};
  m.biases[0] = {-0.5, 2.0};
  std::mt19937_64 rng(4);
  const Vec z0 = RandomVector(rng, 3);
  for (int order : {1, 2}) {
    const auto a = PrepareNodes(m, z0.data(), 1, 3, order);
    for (int t = 0; t < 20; ++t) {
      const Vec z = RandomVector(rng, 3, -4, 4);
      Vec y(2);
      EvalTaylor(3, 2, order, a[0].z0.data(), a[0].f_bar.data(), a[0].jac.data(), a[0].hess.data(), z.data(),
                 y.data());
      CHECK(MaxAbsDiff(y, MlpForward(m, z)) < 1e-12);
    }
  }
}

static void TestOrder2JacobianFd(Activation act) {  // test_taylor.cpp:87-100
  std::mt19937_64 rng(5);
  const MlpModel m = RandomNet(rng, {3, 14, 2}, act);
  const Vec z0 = RandomVector(rng, 3);
  const auto a = PrepareNodes(m, z0.data(), 1, 3, 2);
  for (int t = 0; t < 10; ++t) {
    const Vec d = RandomVector(rng, 3);
    Vec z = z0;
    for (int k = 0; k < 3; ++k) z[k] += 0.3 * d[k];
    Vec j(6);
    EvalTaylorJacobian(3, 2, 2, a[0].z0.data(), a[0].jac.data(), a[0].hess.data(), z.data(), j.data());
    const Vec fd = FdJacobian(
        [&](const Vec& v) {
          Vec y(2);
          EvalTaylor(3, 2, 2, a[0].z0.data(), a[0].f_bar.data(), a[0].jac.data(), a[0].hess.data(), v.data(),
                     y.data());
          return y;
        },
        z, 1e-6);
    CHECK(RelError(j, fd) < 1e-6);
  }
}

static void TestRemainderOrders(Activation act) {  // test_taylor.cpp:102-135
  std::mt19937_64 rng(6);
  std::vector<double> r1s, r2s;
  for (int t = 0; t < 40; ++t) {
    const MlpModel m = RandomNet(rng, {3, 16, 16, 2}, act);
    const Vec z0 = RandomVector(rng, 3, -0.5, 0.5);
    const auto a1 = PrepareNodes(m, z0.data(), 1, 3, 1);
    const auto a2 = PrepareNodes(m, z0.data(), 1, 3, 2);
    const Vec dir = Normalized(RandomVector(rng, 3));
    auto rem = [&](const TaylorApprox& a, double step) {
      Vec z = z0, y(2);
      for (int k = 0; k < 3; ++k) z[k] += step * dir[k];
      EvalTaylor(3, 2, a.order, a.z0.data(), a.f_bar.data(), a.jac.data(), a.hess.data(), z.data(), y.data());
      return MaxAbsDiff(y, MlpForward(m, z));
    };
    const double d = 0.02;
    const double r1f = rem(a1[0], d), r1h = rem(a1[0], d / 2), r2f = rem(a2[0], d), r2h = rem(a2[0], d / 2);
    if (r1h > 1e-12) r1s.push_back(r1f / r1h);
    if (r2h > 1e-12) r2s.push_back(r2f / r2h);
  }
  CHECK(r1s.size() > 20 && r2s.size() > 20);
  if (r1s.size() > 20 && r2s.size() > 20) {
    std::nth_element(r1s.begin(), r1s.begin() + r1s.size() / 2, r1s.end());
    std::nth_element(r2s.begin(), r2s.begin() + r2s.size() / 2, r2s.end());
    const double m1 = r1s[r1s.size() / 2], m2 = r2s[r2s.size() / 2];
    CHECK(m1 > 3.5 && m1 < 4.5);
    CHECK(m2 > 6.5 && m2 < 9.5);
  }
}

int main() {
  TestLinearLayer();
  TestZeroWeights();
  TestForwardVsNaive(Activation::kTanh, 1e-12);
  TestForwardVsNaive(Activation::kSilu, 1e-12);
  TestJacobianFd(Activation::kTanh);
  TestJacobianFd(Activation::kSilu);
  TestReluJacobianFd();
  TestHessians(Activation::kTanh);
  TestHessians(Activation::kSilu);
  TestReluHessianRejected();
  TestBatchEqualsSingle(Activation::kTanh);
  TestBatchEqualsSingle(Activation::kSilu);
  TestMismatchRejected();
  TestRoundTrip(Activation::kTanh);
  TestRoundTrip(Activation::kSilu);
  TestArch();
  TestParamCount();
  TestForwardModeAgrees(Activation::kTanh);
  TestForwardModeAgrees(Activation::kSilu);
  TestForwardModeAgrees(Activation::kRelu);
  TestFileVersions();
  TestPrepareEqualsUnbatched();
  TestZeroOutputModel();
  TestIdenticalNodes();
  TestExpansionPointExact();
  TestLinearTaylorExact();
  TestOrder2JacobianFd(Activation::kTanh);
  TestOrder2JacobianFd(Activation::kSilu);
  TestRemainderOrders(Activation::kTanh);
  TestRemainderOrders(Activation::kSilu);
  std::printf("oracle self-test: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
