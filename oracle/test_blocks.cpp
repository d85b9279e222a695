// ORACLE SELF-TEST — pins the continuity-block restatement (blocks_oracle.cpp)
// against the reference's own tests, same seeds / shapes / tolerances:
//   /root/reference/proj/tests/test_integrator.cpp:35-196
//   /root/reference/proj/tests/test_dynamics.cpp:19-134
//   /root/reference/proj/tests/test_sqp_rti.cpp:77-128 (BuildQp mode equivalence)
// plus quadrotor-'full' checks the reference lacks (rtn == naive for a linear
// residual on the quad, FD of the assembled blocks). Exit code 0 = all pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>

#include "blocks_oracle.h"

using namespace oracle;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
  do {                                                                               \
    ++g_checks;                                                                      \
    if (!(cond)) {                                                                   \
      ++g_fail;                                                                      \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                                \
  } while (0)

namespace {

// doctest::Approx(b).epsilon(e): |a-b| < e * (1 + max(|a|,|b|))
bool Approx(double a, double b, double e) { return std::fabs(a - b) < e * (1.0 + std::max(std::fabs(a), std::fabs(b))); }

double MaxAbs(const Vec& a) {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::fabs(v));
  return m;
}
double MaxAbsDiff(const Vec& a, const Vec& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}
double RelError(const Vec& a, const Vec& b) { return MaxAbsDiff(a, b) / (1.0 + MaxAbs(b)); }
double Norm(const Vec& a) {
  double s = 0.0;
  for (double v : a) s += v * v;
  return std::sqrt(s);
}

// proj/tests/oracles.hpp:17-28, out x in row-major
Vec FdJacobian(const std::function<Vec(const Vec&)>& f, const Vec& x, double h = 1e-5) {
  const Vec f0 = f(x);
  const size_t out = f0.size(), in = x.size();
  Vec jac(out * in);
  for (size_t j = 0; j < in; ++j) {
    Vec xp = x, xm = x;
    xp[j] += h;
    xm[j] -= h;
    const Vec fp = f(xp), fm = f(xm);
    for (size_t i = 0; i < out; ++i) jac[i * in + j] = (fp[i] - fm[i]) / (2.0 * h);
  }
  return jac;
}

Vec Normalized(Vec v) {
  const double n = Norm(v);
  for (double& x : v) x /= n;
  return v;
}

// proj/tests/test_integrator.cpp:24-31
Vec RandomQuadState(std::mt19937_64& rng) {
  Vec x(kQuadNx);
  const Vec p = RandomVector(rng, 3, -2, 2);
  const Vec q = Normalized(RandomVector(rng, 4, -1, 1));
  const Vec v = RandomVector(rng, 3, -4, 4);
  const Vec w = RandomVector(rng, 3, -3, 3);
  std::copy(p.begin(), p.end(), x.begin());
  std::copy(q.begin(), q.end(), x.begin() + kQuatRow);
  std::copy(v.begin(), v.end(), x.begin() + kVelRow);
  std::copy(w.begin(), w.end(), x.begin() + kOmegaRow);
  return x;
}

Vec Hover() {
  Vec x(kQuadNx, 0.0);
  x[kQuatRow] = 1.0;
  return x;
}

const QuadParams kParams{};
DynFn QuadFn() {
  return [](const Vec& x, const Vec& u) { return QuadNominalDynamics(x, u, kParams); };
}
DynJacFn QuadJacFn() {
  return [](const Vec& x, const Vec& u, Mat& fx, Mat& fu) { QuadNominalJacobians(x, u, kParams, fx, fu); };
}

template <typename E, typename F>
bool Throws(F f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// --- test_integrator.cpp ------------------------------------------------------
void Integrator() {
  {  // :35-45 zero dynamics
    FevalCounter c;
    const DynFn zero = [](const Vec& x, const Vec&) { return Vec(x.size(), 0.0); };
    const Vec x = {1, 2, 3};
    const Vec next = Rk4Step(zero, x, Vec{0.0}, 0.1, -1, &c);
    CHECK(MaxAbsDiff(next, x) == 0.0);
    CHECK(c.values == 4);
  }
  {  // :47-61 double integrator analytic
    const DynFn f = [](const Vec& x, const Vec& u) { return Vec{x[1], u[0]}; };
    std::mt19937_64 rng(2);
    for (int t = 0; t < 20; ++t) {
      const Vec x0 = RandomVector(rng, 2, -3, 3);
      const double u = RandomVector(rng, 1, -2, 2)[0];
      const double dt = 0.12;
      const Vec next = Rk4Step(f, x0, Vec{u}, dt);
      CHECK(Approx(next[0], x0[0] + x0[1] * dt + 0.5 * u * dt * dt, 1e-13));
      CHECK(Approx(next[1], x0[1] + u * dt, 1e-13));
    }
  }
  {  // :63-68 hover equilibrium
    const Vec u(4, kParams.HoverThrustPerRotor());
    const Vec next = Rk4Step(QuadFn(), Hover(), u, 0.01, kQuatRow);
    CHECK(MaxAbsDiff(next, Hover()) < 1e-9);
  }
  {  // :70-79 quaternion norm preserved
    std::mt19937_64 rng(8);
    for (int t = 0; t < 10; ++t) {
      Vec x = RandomQuadState(rng);
      const Vec w = RandomVector(rng, 3, -20, 20);
      std::copy(w.begin(), w.end(), x.begin() + kOmegaRow);
      const Vec u = RandomVector(rng, 4, 0, 6);
      const Vec next = Rk4Step(QuadFn(), x, u, 0.05, kQuatRow);
      CHECK(std::abs(Norm(Vec(next.begin() + kQuatRow, next.begin() + kQuatRow + 4)) - 1.0) < 1e-6);
    }
  }
  {  // :81-87 non-finite derivative
    const DynFn bad = [](const Vec& x, const Vec&) {
      Vec r(x.size());
      for (size_t i = 0; i < x.size(); ++i) r[i] = x[i] / 0.0;
      return r;
    };
    CHECK(Throws<std::runtime_error>([&] { Rk4Step(bad, Vec{1, 1}, Vec{0.0}, 0.1); }));
  }
  {  // :89-106 zero-dynamics sensitivities
    const DynFn zero = [](const Vec& x, const Vec&) { return Vec(x.size(), 0.0); };
    const DynJacFn dz = [](const Vec& x, const Vec& u, Mat& fx, Mat& fu) {
      fx = Mat(static_cast<int>(x.size()), static_cast<int>(x.size()));
      fu = Mat(static_cast<int>(x.size()), static_cast<int>(u.size()));
    };
    FevalCounter c;
    const SensitivityResult s = Rk4Sensitivities(zero, dz, Vec{1, 2}, Vec{0.0}, 0.1, -1, &c);
    CHECK(MaxAbsDiff(s.phi_bar, Vec{1, 2}) == 0.0);
    CHECK(s.a(0, 0) == 1.0 && s.a(1, 1) == 1.0 && s.a(0, 1) == 0.0 && s.a(1, 0) == 0.0);
    CHECK(MaxAbs(s.b.v) == 0.0);
    CHECK(c.values == 4 && c.jacobians == 4);
  }
  {  // :108-131 LTI = degree-4 truncated exponential
    std::mt19937_64 rng(21);
    for (int t = 0; t < 10; ++t) {
      const int n = 3;
      Mat f(n, n), g(n, 1);
      for (int i = 0; i < n; ++i) {
        const Vec row = RandomVector(rng, n);
        for (int j = 0; j < n; ++j) f(i, j) = row[j];
        g(i, 0) = RandomVector(rng, 1)[0];
      }
      const DynFn dyn = [&](const Vec& x, const Vec& u) {
        Vec r(n);
        for (int i = 0; i < n; ++i) {
          double s = 0.0;
          for (int j = 0; j < n; ++j) s += f(i, j) * x[j];
          r[i] = s + g(i, 0) * u[0];
        }
        return r;
      };
      const DynJacFn djac = [&](const Vec&, const Vec&, Mat& fx, Mat& fu) {
        fx = f;
        fu = g;
      };
      const double dt = 0.07;
      const Vec x0 = RandomVector(rng, n);
      const Vec u0 = RandomVector(rng, 1);
      const SensitivityResult s = Rk4Sensitivities(dyn, djac, x0, u0, dt);
      // oracles.hpp:155-166
      Mat a(n, n), term(n, n);
      for (int i = 0; i < n; ++i) a(i, i) = term(i, i) = 1.0;
      for (int k = 1; k <= 4; ++k) {
        Mat nt(n, n);
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int m = 0; m < n; ++m) acc += term(i, m) * (f(m, j) * dt);
            nt(i, j) = acc / k;
          }
        term = nt;
        for (size_t e = 0; e < a.v.size(); ++e) a.v[e] += term.v[e];
      }
      CHECK(MaxAbsDiff(s.a.v, a.v) < 1e-13);
    }
  }
  {  // :133-150 nominal Jacobians vs FD
    std::mt19937_64 rng(33);
    double worst = 0.0;
    for (int t = 0; t < 100; ++t) {
      const Vec x = RandomQuadState(rng);
      const Vec u = RandomVector(rng, 4, 0.1, 5.0);
      Mat fx, fu;
      QuadNominalJacobians(x, u, kParams, fx, fu);
      const Vec fdx = FdJacobian([&](const Vec& xs) { return QuadNominalDynamics(xs, u, kParams); }, x);
      const Vec fdu = FdJacobian([&](const Vec& us) { return QuadNominalDynamics(x, us, kParams); }, u);
      worst = std::max({worst, RelError(fx.v, fdx), RelError(fu.v, fdu)});
    }
    CHECK(worst < 1e-6);
  }
  {  // :152-164 structure
    std::mt19937_64 rng(44);
    const Vec x = RandomQuadState(rng);
    const Vec u = RandomVector(rng, 4, 0.5, 4.0);
    Mat fx, fu;
    QuadNominalJacobians(x, u, kParams, fx, fu);
    double d = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) d = std::max(d, std::fabs(fx(i, kVelRow + j) - (i == j ? 1.0 : 0.0)));
    CHECK(d == 0.0);
    double r[9], mix[6][4];
    QuatToRot(&x[kQuatRow], r);
    MixingMatrix(kParams, mix);
    double e = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int c = 0; c < 4; ++c) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += r[3 * i + k] * mix[k][c];
        e = std::max(e, std::fabs(fu(kVelRow + i, c) - s / kParams.mass));
      }
    CHECK(e < 1e-14);
  }
  {  // :166-189 RK4 sensitivities vs FD of the raw map
    std::mt19937_64 rng(55);
    const double dt = 0.02;
    double worst = 0.0;
    for (int t = 0; t < 100; ++t) {
      const Vec x = RandomQuadState(rng);
      const Vec u = RandomVector(rng, 4, 0.5, 5.0);
      const SensitivityResult s = Rk4Sensitivities(QuadFn(), QuadJacFn(), x, u, dt, kQuatRow);
      auto raw = [&](const Vec& xs, const Vec& us) { return Rk4Step(QuadFn(), xs, us, dt, -1); };
      const Vec fda = FdJacobian([&](const Vec& xs) { return raw(xs, u); }, x);
      const Vec fdb = FdJacobian([&](const Vec& us) { return raw(x, us); }, u);
      worst = std::max({worst, RelError(s.a.v, fda), RelError(s.b.v, fdb)});
      const Vec rw = raw(x, u);
      CHECK(std::abs(Norm(Vec(s.phi_bar.begin() + kQuatRow, s.phi_bar.begin() + kQuatRow + 4)) - 1.0) < 1e-12);
      CHECK(s.phi_bar[0] == rw[0] && s.phi_bar[1] == rw[1] && s.phi_bar[2] == rw[2]);
    }
    CHECK(worst < 1e-5);
  }
  {  // :191-196 bit-identical repeats
    std::mt19937_64 rng(66);
    const Vec x = RandomQuadState(rng);
    const Vec u = RandomVector(rng, 4, 0.5, 5.0);
    const SensitivityResult s1 = Rk4Sensitivities(QuadFn(), QuadJacFn(), x, u, 0.01, kQuatRow);
    const SensitivityResult s2 = Rk4Sensitivities(QuadFn(), QuadJacFn(), x, u, 0.01, kQuatRow);
    CHECK(s1.a.v == s2.a.v && s1.b.v == s2.b.v && s1.phi_bar == s2.phi_bar);
  }
}

// --- test_dynamics.cpp -----------------------------------------------------------
void Dynamics() {
  {  // :19-31 axis-angle oracle
    std::mt19937_64 rng(11);
    for (int t = 0; t < 50; ++t) {
      const Vec axis = Normalized(RandomVector(rng, 3));
      const double ang = RandomVector(rng, 1, -3.0, 3.0)[0];
      const double q[4] = {std::cos(ang / 2), std::sin(ang / 2) * axis[0], std::sin(ang / 2) * axis[1],
                           std::sin(ang / 2) * axis[2]};
      // Rodrigues (oracles.hpp:36-42)
      const double k[9] = {0, -axis[2], axis[1], axis[2], 0, -axis[0], -axis[1], axis[0], 0};
      double kk[9], ex[9], r[9];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          double s = 0.0;
          for (int m = 0; m < 3; ++m) s += k[3 * i + m] * k[3 * m + j];
          kk[3 * i + j] = s;
        }
      for (int e = 0; e < 9; ++e) ex[e] = (e % 4 == 0 ? 1.0 : 0.0) + std::sin(ang) * k[e] + (1 - std::cos(ang)) * kk[e];
      QuatToRot(q, r);
      CHECK(MaxAbsDiff(Vec(r, r + 9), Vec(ex, ex + 9)) < 1e-12);
      const Vec v = RandomVector(rng, 3, -2.0, 2.0);
      double rv[3];
      QuatRotate(q, v.data(), rv);
      double d = 0.0;
      for (int i = 0; i < 3; ++i) d += std::pow(rv[i] - (ex[3 * i] * v[0] + ex[3 * i + 1] * v[1] + ex[3 * i + 2] * v[2]), 2);
      CHECK(std::sqrt(d) < 1e-12);
    }
  }
  {  // :33-40 90 degree yaw
    const double s = std::sin(M_PI / 4.0);
    const double q[4] = {std::cos(M_PI / 4.0), 0.0, 0.0, s};
    const double v[3] = {1.0, 0.0, 0.0};
    double vb[3];
    QuatRotateInv(q, v, vb);
    CHECK(Approx(vb[0], 0.0, 1e-12) && Approx(vb[1], -1.0, 1e-12) && Approx(vb[2], 0.0, 1e-12));
  }
  double mix[6][4];
  MixingMatrix(kParams, mix);
  auto wrench = [&](const double* u, double* w) {
    for (int r = 0; r < 6; ++r) {
      double s = 0.0;
      for (int i = 0; i < 4; ++i) s += mix[r][i] * u[i];
      w[r] = s;
    }
  };
  {  // :42-49 equal thrusts
    const double u[4] = {1.3, 1.3, 1.3, 1.3};
    double w[6];
    wrench(u, w);
    CHECK(w[0] == 0.0 && w[1] == 0.0 && Approx(w[2], 4 * 1.3, 1e-5));
    CHECK(std::sqrt(w[3] * w[3] + w[4] * w[4] + w[5] * w[5]) < 1e-14);
  }
  {  // :51-61 single-rotor moment arm
    for (int i = 0; i < 4; ++i) {
      double u[4] = {0, 0, 0, 0}, w[6];
      u[i] = 2.0;
      wrench(u, w);
      const double arm = kParams.arm_length * 2.0 / std::sqrt(2.0);
      CHECK(Approx(std::abs(w[3]), arm, 1e-5) && Approx(std::abs(w[4]), arm, 1e-5));
    }
  }
  {  // :63-71 same-spin pair is pure yaw
    const double u[4] = {1.0, 1.0, 0.0, 0.0};
    double w[6];
    wrench(u, w);
    CHECK(std::abs(w[3]) < 1e-14 && std::abs(w[4]) < 1e-14);
    CHECK(Approx(w[5], kParams.rotor_sign[0] * kParams.torque_coeff * 2.0, 1e-5));
  }
  {  // :73-84 geometry oracle (oracles.hpp:46-56)
    std::mt19937_64 rng(7);
    for (int t = 0; t < 30; ++t) {
      const Vec uv = RandomVector(rng, 4, 0.0, kParams.thrust_max);
      double w[6];
      wrench(uv.data(), w);
      const double d = kParams.arm_length / std::sqrt(2.0);
      const double pos[4][2] = {{d, -d}, {-d, d}, {d, d}, {-d, -d}};
      double tau[3] = {0, 0, 0};
      for (int i = 0; i < 4; ++i) {  // pos × (0,0,T): (y T, -x T, 0)
        tau[0] += pos[i][1] * uv[i];
        tau[1] += -pos[i][0] * uv[i];
        tau[2] += kParams.rotor_sign[i] * kParams.torque_coeff * uv[i];
      }
      CHECK(std::sqrt(std::pow(w[3] - tau[0], 2) + std::pow(w[4] - tau[1], 2) + std::pow(w[5] - tau[2], 2)) < 1e-12);
      CHECK(Approx(w[2], uv[0] + uv[1] + uv[2] + uv[3], 1e-5));
    }
  }
  {  // :101-106 hover cancels gravity
    const Vec u(4, kParams.HoverThrustPerRotor());
    CHECK(MaxAbs(QuadNominalDynamics(Hover(), u, kParams)) < 1e-12);
  }
  {  // :108-112 free fall
    const Vec dx = QuadNominalDynamics(Hover(), Vec(4, 0.0), kParams);
    CHECK(dx[kVelRow] == 0.0 && dx[kVelRow + 1] == 0.0 && Approx(dx[kVelRow + 2], -kGravity, 1e-12));
  }
  {  // :114-126 Euler's equation
    Vec x = Hover();
    x[kOmegaRow] = 0.4;
    x[kOmegaRow + 1] = -0.2;
    x[kOmegaRow + 2] = 1.1;
    const Vec u = {1.0, 0.0, 1.0, 0.0};
    const Vec dx = QuadNominalDynamics(x, u, kParams);
    const double d = kParams.arm_length / std::sqrt(2.0);
    const double pos[4][2] = {{d, -d}, {-d, d}, {d, d}, {-d, -d}};
    double tau[3] = {0, 0, 0};
    for (int i = 0; i < 4; ++i) {
      tau[0] += pos[i][1] * u[i];
      tau[1] += -pos[i][0] * u[i];
      tau[2] += kParams.rotor_sign[i] * kParams.torque_coeff * u[i];
    }
    const double* w = &x[kOmegaRow];
    const double* j = kParams.inertia;
    const double jw[3] = {j[0] * w[0], j[1] * w[1], j[2] * w[2]};
    const double cr[3] = {w[1] * jw[2] - w[2] * jw[1], w[2] * jw[0] - w[0] * jw[2], w[0] * jw[1] - w[1] * jw[0]};
    double e = 0.0;
    for (int i = 0; i < 3; ++i) e += std::pow(dx[kOmegaRow + i] - (tau[i] - cr[i]) / j[i], 2);
    CHECK(std::sqrt(e) < 1e-12);
  }
  {  // :128-133 far-from-unit quaternion
    Vec x = Hover();
    x[kQuatRow] = 2.0;
    CHECK(Throws<InputDomainError>([&] { QuadNominalDynamics(x, Vec(4, 0.0), kParams); }));
  }
}

// --- test_sqp_rti.cpp: BuildQp mode equivalence --------------------------------
OcpConfig DiConfig(int horizon, double dt) {  // test_sqp_rti.cpp:13-22
  OcpConfig c;
  c.horizon = horizon;
  c.dt = dt;
  c.q_diag = {10.0, 1.0};
  c.r_diag = {0.5};
  c.u_min = {-1e9};
  c.u_max = {1e9};
  return c;
}

double MaxQpDiff(const QpData& a, const QpData& b) {  // test_sqp_rti.cpp:31-41
  double d = 0.0;
  for (int k = 0; k < a.horizon; ++k) {
    d = std::max({d, MaxAbsDiff(a.a[k].v, b.a[k].v), MaxAbsDiff(a.b[k].v, b.b[k].v),
                  MaxAbsDiff(a.phi_res[k], b.phi_res[k]), MaxAbsDiff(a.q[k], b.q[k]), MaxAbsDiff(a.r[k], b.r[k])});
  }
  return d;
}

NaiveNet Naive(const MlpModel& m) {
  return NaiveNet{[&m](const Vec& z) { return MlpForward(m, z); }, [&m](const Vec& z) { return MlpJacobian(m, z); }};
}

std::vector<TaylorApprox> Prepare(const Plant& plant, const MlpModel& m, const std::vector<Vec>& xs,
                                  const std::vector<Vec>& us, int order) {
  const int n = static_cast<int>(us.size());
  Vec z;
  for (int k = 0; k < n; ++k) {
    const Vec f = plant.features(xs[k], us[k], Vec());
    z.insert(z.end(), f.begin(), f.end());
  }
  return PrepareNodes(m, z.data(), n, plant.feature_dim, order);
}

void BuildQpTests() {
  {  // :77-101 zero residual: rtn == naive == none
    const Plant plant = MakeDoubleIntegratorPlant();
    const OcpConfig cfg = DiConfig(8, 0.05);
    std::mt19937_64 rng(2);
    std::vector<Vec> rx(cfg.horizon + 1, Vec(2, 0.0)), ru(cfg.horizon, Vec(1, 0.0));
    std::vector<Vec> xs = rx, us = ru;
    xs[0] = RandomVector(rng, 2);
    for (auto& u : us) u = RandomVector(rng, 1);
    MlpModel zero = MakeMlp({3, 16, 16, 2}, Activation::kTanh, "full", 5);  // MakeZeroNetwork(2,16,3,2,5)
    for (double& w : zero.weights.back().v) w = 0.0;
    const auto ap = Prepare(plant, zero, xs, us, 1);
    const NaiveNet nv = Naive(zero);
    const QpData q_rtn = BuildQp(plant, cfg, xs, us, rx, ru, &ap, nullptr);
    const QpData q_naive = BuildQp(plant, cfg, xs, us, rx, ru, nullptr, &nv);
    const QpData q_none = BuildQp(plant, cfg, xs, us, rx, ru, nullptr, nullptr);
    CHECK(MaxQpDiff(q_rtn, q_naive) < 1e-12);
    CHECK(MaxQpDiff(q_rtn, q_none) < 1e-12);
  }
  {  // :103-128 linear residual: rtn == naive
    const Plant plant = MakeDoubleIntegratorPlant();
    const OcpConfig cfg = DiConfig(6, 0.05);
    std::mt19937_64 rng(3);
    std::vector<Vec> rx(cfg.horizon + 1, Vec(2, 0.0)), ru(cfg.horizon, Vec(1, 0.0));
    std::vector<Vec> xs = rx, us = ru;
    xs[0] = RandomVector(rng, 2);
    for (auto& u : us) u = RandomVector(rng, 1);
    MlpModel lin = MakeMlp({3, 2}, Activation::kTanh, "full", 7);
    lin.weights[0].v = {0.2, -0.1, 0.3, 0.05, 0.15, -0.2};
    lin.biases[0] = {0.01, -0.02};
    const auto ap = Prepare(plant, lin, xs, us, 1);
    const NaiveNet nv = Naive(lin);
    const QpData a = BuildQp(plant, cfg, xs, us, rx, ru, &ap, nullptr);
    const QpData b = BuildQp(plant, cfg, xs, us, rx, ru, nullptr, &nv);
    CHECK(MaxQpDiff(a, b) < 1e-10);
  }
  // Quadrotor 'full' (the product's plant): linear residual => Taylor exact => rtn == naive.
  const Plant quad = MakeQuadrotorPlant(kParams, "full");
  OcpConfig qc;
  qc.horizon = 12;
  qc.dt = 0.05;
  qc.q_diag = Vec(13, 1.0);
  qc.r_diag = Vec(4, 0.1);
  qc.u_min = Vec(4, 0.0);
  qc.u_max = Vec(4, kParams.thrust_max);
  std::mt19937_64 rng(2203);
  std::vector<Vec> xs, us, rx, ru;
  for (int k = 0; k <= qc.horizon; ++k) {
    xs.push_back(RandomQuadState(rng));
    rx.push_back(RandomQuadState(rng));
  }
  for (int k = 0; k < qc.horizon; ++k) {
    us.push_back(RandomVector(rng, 4, 0.5, 5.0));
    ru.push_back(RandomVector(rng, 4, 0.5, 5.0));
  }
  {
    MlpModel lin = RandomNet(rng, {17, 6});
    const auto ap = Prepare(quad, lin, xs, us, 1);
    const NaiveNet nv = Naive(lin);
    FevalCounter fc;
    const QpData a = BuildQp(quad, qc, xs, us, rx, ru, &ap, nullptr, &fc);
    const QpData b = BuildQp(quad, qc, xs, us, rx, ru, nullptr, &nv);
    CHECK(MaxQpDiff(a, b) < 1e-10);
    CHECK(fc.values == 4u * qc.horizon && fc.jacobians == 4u * qc.horizon);  // test_sqp_rti.cpp:246-247
    CHECK(a.q.size() == 13u && a.hx_diag.size() == 13u);
  }
  {  // order 2 on a nonlinear net: FD of the assembled raw map around each node
    MlpModel net = RandomNet(rng, {17, 24, 24, 6}, Activation::kSilu);
    for (int order = 1; order <= 2; ++order) {
      const auto ap = Prepare(quad, net, xs, us, order);
      qc.taylor_order = order;
      const QpData a = BuildQp(quad, qc, xs, us, rx, ru, &ap, nullptr);
      double worst = 0.0;
      for (int k = 0; k < qc.horizon; ++k) {
        const TaylorApprox* p = &ap[k];
        const DynFn fk = [&](const Vec& x, const Vec& u) {
          Vec f = QuadNominalDynamics(x, u, kParams);
          Vec z(x);
          z.insert(z.end(), u.begin(), u.end());
          Vec y(6);
          EvalTaylor(17, 6, p->order, p->z0.data(), p->f_bar.data(), p->jac.data(),
                     p->hess.empty() ? nullptr : p->hess.data(), z.data(), y.data());
          for (int i = 0; i < 6; ++i) f[7 + i] += y[i];
          return f;
        };
        const Vec fda = FdJacobian([&](const Vec& x) { return Rk4Step(fk, x, us[k], qc.dt, -1); }, xs[k]);
        const Vec fdb = FdJacobian([&](const Vec& u) { return Rk4Step(fk, xs[k], u, qc.dt, -1); }, us[k]);
        worst = std::max({worst, RelError(a.a[k].v, fda), RelError(a.b[k].v, fdb)});
      }
      CHECK(worst < 1e-6);
    }
  }
  // Every residual variant (dynamics.cpp:95-211, plant.cpp:60-85): rtn == naive for a
  // linear residual (the Taylor model of a linear map is exact in feature space), and
  // FD of the assembled blocks for a nonlinear one (orders 1 and 2).
  for (const char* var : {"a", "a_u", "full", "ground"}) {
    const Plant plant = MakeQuadrotorPlant(kParams, var);
    const int nf = plant.feature_dim, nr = plant.residual_dim;
    std::vector<Vec> aux;
    for (int k = 0; k < qc.horizon; ++k) aux.push_back(RandomVector(rng, 9, -0.2, 0.3));
    const std::vector<Vec>* auxp = std::string(var) == "ground" ? &aux : nullptr;
    auto prepare = [&](const MlpModel& m, int order) {
      Vec z;
      for (int k = 0; k < qc.horizon; ++k) {
        const Vec f = plant.features(xs[k], us[k], auxp ? aux[k] : Vec());
        z.insert(z.end(), f.begin(), f.end());
      }
      return PrepareNodes(m, z.data(), qc.horizon, nf, order);
    };
    {
      MlpModel lin = RandomNet(rng, {nf, nr});
      const auto ap = prepare(lin, 1);
      const NaiveNet nv = Naive(lin);
      qc.taylor_order = 1;
      const QpData a = BuildQp(plant, qc, xs, us, rx, ru, &ap, nullptr, nullptr, auxp);
      const QpData b = BuildQp(plant, qc, xs, us, rx, ru, nullptr, &nv, nullptr, auxp);
      CHECK(MaxQpDiff(a, b) < 1e-10);
    }
    MlpModel net = RandomNet(rng, {nf, 24, 24, nr}, Activation::kSilu);
    for (int order = 1; order <= 2; ++order) {
      const auto ap = prepare(net, order);
      qc.taylor_order = order;
      const QpData a = BuildQp(plant, qc, xs, us, rx, ru, &ap, nullptr, nullptr, auxp);
      double worst = 0.0;
      for (int k = 0; k < qc.horizon; ++k) {
        const TaylorApprox* p = &ap[k];
        const Vec ax = auxp ? aux[k] : Vec();
        const DynFn fk = [&](const Vec& x, const Vec& u) {
          Vec f = QuadNominalDynamics(x, u, kParams);
          const Vec z = plant.features(x, u, ax);
          Vec y(nr);
          EvalTaylor(nf, nr, p->order, p->z0.data(), p->f_bar.data(), p->jac.data(),
                     p->hess.empty() ? nullptr : p->hess.data(), z.data(), y.data());
          for (int i = 0; i < nr; ++i) f[7 + i] += y[i];
          return f;
        };
        const Vec fda = FdJacobian([&](const Vec& x) { return Rk4Step(fk, x, us[k], qc.dt, -1); }, xs[k]);
        const Vec fdb = FdJacobian([&](const Vec& u) { return Rk4Step(fk, xs[k], u, qc.dt, -1); }, us[k]);
        worst = std::max({worst, RelError(a.a[k].v, fda), RelError(a.b[k].v, fdb)});
      }
      CHECK(worst < 1e-6);
    }
  }
  qc.taylor_order = 1;
  {  // errors: quaternion far from unit at node 3 -> "build qp: node 3: quad dynamics: ..."
    std::vector<Vec> bad = xs;
    bad[3][kQuatRow] = 3.0;
    MlpModel lin = RandomNet(rng, {17, 6});
    const auto ap = Prepare(quad, lin, bad, us, 1);
    qc.taylor_order = 1;
    std::string msg;
    try {
      BuildQp(quad, qc, bad, us, rx, ru, &ap, nullptr);
    } catch (const std::runtime_error& e) {
      msg = e.what();
    }
    CHECK(msg == "build qp: node 3: quad dynamics: quaternion norm too far from unit");
  }
}

}  // namespace

int main() {
  Integrator();
  Dynamics();
  BuildQpTests();
  std::printf("test_blocks: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
