// ORACLE SELF-TEST — pins the QP / closed-loop restatement (closedloop_oracle.cpp)
// against the reference's own tests, same seeds / shapes / tolerances:
//   /root/reference/proj/tests/test_qp.cpp:55-221 (condensing, box QP vs exhaustive
//   enumeration + KKT, warm starts, crossed bounds)
// plus closed-loop sanity checks the reference states in SPEC (hover is an
// equilibrium of the loop; rollouts are bit-deterministic; a circle is tracked).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>

#include "closedloop_oracle.h"

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

double MaxAbsDiff(const Vec& a, const Vec& b) {
  double m = 0.0;
  for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::fabs(a[i] - b[i]));
  return m;
}

Vec MatVec(const Mat& m, const Vec& v) {
  Vec o(m.rows, 0.0);
  for (std::int64_t i = 0; i < m.rows; ++i)
    for (std::int64_t j = 0; j < m.cols; ++j) o[i] += m(i, j) * v[j];
  return o;
}

double Dot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// test_qp.cpp:11-37
QpData RandomQpData(std::mt19937_64& rng, int nx, int nu, int horizon) {
  QpData qp;
  qp.nx = nx;
  qp.nu = nu;
  qp.horizon = horizon;
  for (int k = 0; k < horizon; ++k) {
    Mat a(nx, nx), b(nx, nu);
    for (int i = 0; i < nx; ++i) {
      const Vec row = RandomVector(rng, nx);
      for (int j = 0; j < nx; ++j) a(i, j) = 0.3 * row[j];
      a(i, i) += 1.0;
    }
    for (int i = 0; i < nx; ++i) {
      const Vec row = RandomVector(rng, nu);
      for (int j = 0; j < nu; ++j) b(i, j) = row[j];
    }
    qp.a.push_back(a);
    qp.b.push_back(b);
    Vec phi = RandomVector(rng, nx);
    for (double& v : phi) v *= 0.1;
    qp.phi_res.push_back(phi);
    qp.q.push_back(RandomVector(rng, nx));
    qp.r.push_back(RandomVector(rng, nu));
    qp.hx_diag.push_back(RandomVector(rng, nx, 0.5, 2.0));
    qp.hu_diag.push_back(RandomVector(rng, nu, 0.5, 2.0));
    qp.du_lb.push_back(Vec(nu, -1.0));
    qp.du_ub.push_back(Vec(nu, 1.0));
  }
  qp.q.push_back(RandomVector(rng, nx));
  qp.hx_diag.push_back(RandomVector(rng, nx, 0.5, 2.0));
  return qp;
}

// test_qp.cpp:39-52
double FullObjective(const QpData& qp, const Vec& dx0, const Vec& du) {
  double obj = 0.0;
  Vec dx = dx0;
  for (int k = 0; k <= qp.horizon; ++k) {
    for (int i = 0; i < qp.nx; ++i) obj += qp.q[k][i] * dx[i] + 0.5 * dx[i] * qp.hx_diag[k][i] * dx[i];
    if (k < qp.horizon) {
      const Vec duk(du.begin() + k * qp.nu, du.begin() + (k + 1) * qp.nu);
      for (int i = 0; i < qp.nu; ++i) obj += qp.r[k][i] * duk[i] + 0.5 * duk[i] * qp.hu_diag[k][i] * duk[i];
      Vec nx = MatVec(qp.a[k], dx);
      const Vec bu = MatVec(qp.b[k], duk);
      for (int i = 0; i < qp.nx; ++i) nx[i] += bu[i] + qp.phi_res[k][i];
      dx = nx;
    }
  }
  return obj;
}

Mat RandomSpd(std::mt19937_64& rng, int n, double shift) {
  Mat m(n, n), h(n, n);
  for (int i = 0; i < n; ++i) {
    const Vec row = RandomVector(rng, n);
    for (int j = 0; j < n; ++j) m(i, j) = row[j];
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += m(i, k) * m(j, k);
      h(i, j) = s + (i == j ? shift : 0.0);
    }
  return h;
}

// Dense SPD solve by Gaussian elimination (the LDLT of oracles.hpp, restated).
Vec SolveDense(Mat a, Vec b) {
  const int n = static_cast<int>(a.rows);
  for (int c = 0; c < n; ++c)
    for (int r = c + 1; r < n; ++r) {
      const double f = a(r, c) / a(c, c);
      for (int k = c; k < n; ++k) a(r, k) -= f * a(c, k);
      b[r] -= f * b[c];
    }
  Vec x(n);
  for (int r = n - 1; r >= 0; --r) {
    double s = b[r];
    for (int k = r + 1; k < n; ++k) s -= a(r, k) * x[k];
    x[r] = s / a(r, r);
  }
  return x;
}

// oracles.hpp:100-152 BruteForceBoxQp
bool BruteForceBoxQp(const Mat& h, const Vec& g, const Vec& lb, const Vec& ub, Vec* sol) {
  const int n = static_cast<int>(g.size());
  long patterns = 1;
  for (int i = 0; i < n; ++i) patterns *= 3;
  double best = std::numeric_limits<double>::infinity();
  bool found = false;
  for (long p = 0; p < patterns; ++p) {
    long code = p;
    std::vector<int> st(n);
    for (int i = 0; i < n; ++i) {
      st[i] = static_cast<int>(code % 3);
      code /= 3;
    }
    Vec x(n, 0.0);
    std::vector<int> fr;
    for (int i = 0; i < n; ++i) {
      if (st[i] == 1) x[i] = lb[i];
      else if (st[i] == 2) x[i] = ub[i];
      else fr.push_back(i);
    }
    const int nf = static_cast<int>(fr.size());
    if (nf > 0) {
      Mat hff(nf, nf);
      Vec rhs(nf);
      for (int i = 0; i < nf; ++i) {
        rhs[i] = -g[fr[i]];
        for (int j = 0; j < nf; ++j) hff(i, j) = h(fr[i], fr[j]);
        for (int j = 0; j < n; ++j)
          if (st[j] != 0) rhs[i] -= h(fr[i], j) * x[j];
      }
      const Vec xf = SolveDense(hff, rhs);
      for (int i = 0; i < nf; ++i) x[fr[i]] = xf[i];
    }
    bool ok = true;
    for (int i = 0; i < n && ok; ++i) ok = x[i] >= lb[i] - 1e-10 && x[i] <= ub[i] + 1e-10;
    if (!ok) continue;
    Vec grad = MatVec(h, x);
    for (int i = 0; i < n; ++i) grad[i] += g[i];
    for (int i = 0; i < n && ok; ++i) {
      if (st[i] == 0) ok = std::abs(grad[i]) < 1e-8;
      if (st[i] == 1) ok = grad[i] >= -1e-10;
      if (st[i] == 2) ok = grad[i] <= 1e-10;
    }
    if (!ok) continue;
    const double obj = 0.5 * Dot(x, MatVec(h, x)) + Dot(g, x);
    if (obj < best) {
      best = obj;
      *sol = x;
      found = true;
    }
  }
  return found;
}

void QpTests() {
  {  // :55-71 recovery maps satisfy the continuity equalities
    std::mt19937_64 rng(1);
    const QpData qp = RandomQpData(rng, 3, 2, 6);
    const Vec dx0 = RandomVector(rng, 3);
    const CondensedQp c = Condense(qp, dx0);
    for (int t = 0; t < 20; ++t) {
      const Vec du = RandomVector(rng, 12);
      Vec dx = dx0;
      for (int k = 0; k < qp.horizon; ++k) {
        Vec rec = MatVec(c.recover_m[k], du);
        for (int i = 0; i < 3; ++i) rec[i] += c.recover_c[k][i];
        CHECK(MaxAbsDiff(rec, dx) < 1e-10);
        Vec nx = MatVec(qp.a[k], dx);
        const Vec bu = MatVec(qp.b[k], Vec(du.begin() + 2 * k, du.begin() + 2 * k + 2));
        for (int i = 0; i < 3; ++i) nx[i] += bu[i] + qp.phi_res[k][i];
        dx = nx;
      }
      Vec rec = MatVec(c.recover_m[qp.horizon], du);
      for (int i = 0; i < 3; ++i) rec[i] += c.recover_c[qp.horizon][i];
      CHECK(MaxAbsDiff(rec, dx) < 1e-10);
    }
  }
  {  // :73-86 condensed objective == full sparse objective
    std::mt19937_64 rng(2);
    const QpData qp = RandomQpData(rng, 4, 2, 5);
    const Vec dx0 = RandomVector(rng, 4);
    const CondensedQp c = Condense(qp, dx0);
    const double c0 = FullObjective(qp, dx0, Vec(10, 0.0));
    for (int t = 0; t < 50; ++t) {
      const Vec du = RandomVector(rng, 10);
      const double cond = 0.5 * Dot(du, MatVec(c.hessian, du)) + Dot(c.gradient, du) + c0;
      const double full = FullObjective(qp, dx0, du);
      CHECK(std::abs(cond - full) < 1e-9 * (1.0 + std::abs(full)));
    }
  }
  {  // :88-103 N=1 hand-eliminated form
    std::mt19937_64 rng(3);
    const QpData qp = RandomQpData(rng, 2, 1, 1);
    const Vec dx0 = {0.3, -0.1};
    const CondensedQp c = Condense(qp, dx0);
    Vec roll = MatVec(qp.a[0], dx0);
    for (int i = 0; i < 2; ++i) roll[i] += qp.phi_res[0][i];
    double h = qp.hu_diag[0][0], g = qp.r[0][0];
    for (int i = 0; i < 2; ++i) {
      h += qp.b[0](i, 0) * qp.hx_diag[1][i] * qp.b[0](i, 0);
      g += qp.b[0](i, 0) * (qp.q[1][i] + qp.hx_diag[1][i] * roll[i]);
    }
    CHECK(std::abs(c.hessian(0, 0) - h) < 1e-12);
    CHECK(std::abs(c.gradient[0] - g) < 1e-12);
  }
  {  // :105-119 identity A, zero B
    std::mt19937_64 rng(4);
    QpData qp = RandomQpData(rng, 2, 1, 3);
    for (int k = 0; k < 3; ++k) {
      qp.a[k] = Mat(2, 2);
      qp.a[k](0, 0) = qp.a[k](1, 1) = 1.0;
      qp.b[k] = Mat(2, 1);
      qp.phi_res[k] = Vec(2, 0.0);
    }
    const CondensedQp c = Condense(qp, Vec(2, 0.0));
    for (int k = 0; k < 3; ++k) {
      CHECK(c.gradient[k] == qp.r[k][0]);
      CHECK(std::abs(c.hessian(k, k) - qp.hu_diag[k][0]) < 1e-12);
    }
  }
  {  // :128-144 unconstrained box QP solves the normal equations
    std::mt19937_64 rng(6);
    for (int t = 0; t < 10; ++t) {
      CondensedQp qp;
      qp.hessian = RandomSpd(rng, 5, 1.0);
      qp.gradient = RandomVector(rng, 5);
      qp.lb.assign(5, -std::numeric_limits<double>::infinity());
      qp.ub.assign(5, std::numeric_limits<double>::infinity());
      const BoxQpResult r = SolveBoxQp(qp);
      CHECK(r.status == QpStatus::kOptimal);
      Vec ng = qp.gradient;
      for (double& v : ng) v = -v;
      CHECK(MaxAbsDiff(r.x, SolveDense(qp.hessian, ng)) < 1e-9);
    }
  }
  {  // :146-157 1-D binding upper bound
    CondensedQp qp;
    qp.hessian = Mat(1, 1);
    qp.hessian(0, 0) = 2.0;
    qp.gradient = {-10.0};
    qp.lb = {-1.0};
    qp.ub = {1.0};
    const BoxQpResult r = SolveBoxQp(qp);
    CHECK(r.status == QpStatus::kOptimal);
    CHECK(r.x[0] == 1.0);
    CHECK(std::abs(r.lam_ub[0] - 8.0) < 1e-12);
    CHECK(r.lam_lb[0] == 0.0);
  }
  {  // :159-193 random box QPs vs exhaustive enumeration + KKT
    std::mt19937_64 rng(7);
    for (int t = 0; t < 200; ++t) {
      const int n = 2 + static_cast<int>(RandomVector(rng, 1, 0, 6.99)[0]);
      CondensedQp qp;
      qp.hessian = RandomSpd(rng, n, 0.3);
      qp.gradient = RandomVector(rng, n);
      for (double& v : qp.gradient) v *= 2.0;
      qp.lb.resize(n);
      qp.ub.resize(n);
      for (int i = 0; i < n; ++i) {
        const double a = RandomVector(rng, 1)[0], b = RandomVector(rng, 1)[0];
        qp.lb[i] = std::min(a, b);
        qp.ub[i] = std::max(a, b) + 0.05;
      }
      Vec expected;
      const bool found = BruteForceBoxQp(qp.hessian, qp.gradient, qp.lb, qp.ub, &expected);
      CHECK(found);
      const BoxQpResult r = SolveBoxQp(qp);
      CHECK(r.status == QpStatus::kOptimal);
      if (found) CHECK(MaxAbsDiff(r.x, expected) < 1e-9);
      Vec stat = MatVec(qp.hessian, r.x);
      for (int i = 0; i < n; ++i) stat[i] += qp.gradient[i] - r.lam_lb[i] + r.lam_ub[i];
      CHECK(MaxAbsDiff(stat, Vec(n, 0.0)) < 1e-8);
      for (int i = 0; i < n; ++i) {
        CHECK(r.x[i] >= qp.lb[i] && r.x[i] <= qp.ub[i]);
        CHECK(std::abs(r.lam_lb[i] * (r.x[i] - qp.lb[i])) < 1e-8);
        CHECK(std::abs(r.lam_ub[i] * (r.x[i] - qp.ub[i])) < 1e-8);
        CHECK(r.lam_lb[i] >= 0.0 && r.lam_ub[i] >= 0.0);
      }
    }
  }
  {  // :195-213 warm starts / identical inputs
    std::mt19937_64 rng(8);
    CondensedQp qp;
    qp.hessian = RandomSpd(rng, 6, 0.5);
    qp.gradient = RandomVector(rng, 6);
    for (double& v : qp.gradient) v *= 3.0;
    qp.lb.assign(6, -0.4);
    qp.ub.assign(6, 0.4);
    const BoxQpResult r1 = SolveBoxQp(qp), r2 = SolveBoxQp(qp);
    CHECK(r1.iterations == r2.iterations && r1.x == r2.x);
    const BoxQpResult r3 = SolveBoxQp(qp, &r1.active);
    CHECK(r3.iterations <= 2);
    CHECK(MaxAbsDiff(r3.x, r1.x) < 1e-12);
  }
  {  // :215-221 crossed bounds
    CondensedQp qp;
    qp.hessian = Mat(2, 2);
    qp.hessian(0, 0) = qp.hessian(1, 1) = 1.0;
    qp.gradient = {0.0, 0.0};
    qp.lb = {1.0, 1.0};
    qp.ub = {-1.0, -1.0};
    bool threw = false;
    try {
      SolveBoxQp(qp);
    } catch (const ConfigError&) {
      threw = true;
    }
    CHECK(threw);
  }
}

void ClosedLoopTests() {
  const QuadParams qp{};
  OcpConfig cfg;
  cfg.horizon = 20;
  cfg.dt = 0.05;
  cfg.q_diag = {10, 10, 10, 1, 1, 1, 1, 1, 1, 1, 0.1, 0.1, 0.1};
  cfg.r_diag = Vec(4, 0.1);
  cfg.u_min = Vec(4, 0.0);
  cfg.u_max = Vec(4, qp.thrust_max);
  // zero residual: the loop runs on the nominal model plus an exactly-zero Taylor term
  const PrepareFn zero = [](const Vec& z, int k, int order) {
    std::vector<TaylorApprox> out(k);
    for (int i = 0; i < k; ++i) {
      out[i].order = order;
      out[i].z0.assign(z.begin() + i * 17, z.begin() + (i + 1) * 17);
      out[i].f_bar.assign(6, 0.0);
      out[i].jac.assign(6 * 17, 0.0);
      if (order == 2) out[i].hess.assign(6 * 17 * 17, 0.0);
    }
    return out;
  };
  {  // hover reference (zero speed is not allowed, so a tiny circle): commands stay near hover
    TrajectoryCfg tc;
    tc.scale = 1e-3;
    tc.speed = 1e-4;
    SimConfig sc;
    sc.noise_ft_sigma = 0.0;
    sc.motor_noise_coeff = 0.0;
    sc.drag[0] = sc.drag[1] = sc.drag[2] = 0.0;
    RtiController ctrl(qp, cfg, zero);
    QuadSim sim(qp, sc);
    ReferenceGenerator refs(tc, qp);
    const Rollout r = RunClosedLoop(ctrl, sim, refs, cfg, 0.2, 0);
    CHECK(!r.failed && r.states.size() == 20u);
    double dev = 0.0;
    for (const Vec& u : r.commands)
      for (double v : u) dev = std::max(dev, std::fabs(v - qp.HoverThrustPerRotor()));
    CHECK(dev < 1e-3);
  }
  {  // circle tracking with drag + noise: bit-deterministic, tracks within 0.5 m over 1 s
    TrajectoryCfg tc;
    SimConfig sc;
    auto run = [&]() {
      RtiController ctrl(qp, cfg, zero);
      QuadSim sim(qp, sc);
      ReferenceGenerator refs(tc, qp);
      return RunClosedLoop(ctrl, sim, refs, cfg, 1.0, 7);
    };
    const Rollout a = run(), b = run();
    CHECK(!a.failed && a.states.size() == 100u);
    bool same = a.states.size() == b.states.size();
    for (size_t k = 0; same && k < a.states.size(); ++k) same = a.states[k] == b.states[k] && a.commands[k] == b.commands[k];
    CHECK(same);
    ReferenceGenerator refs(tc, qp);
    double worst = 0.0;
    for (size_t k = 0; k < a.states.size(); ++k) {
      Vec rx, ru;
      refs.At(0.01 * k, rx, ru);
      worst = std::max(worst, std::sqrt(std::pow(a.states[k][0] - rx[0], 2) + std::pow(a.states[k][1] - rx[1], 2) +
                                        std::pow(a.states[k][2] - rx[2], 2)));
    }
    CHECK(worst < 0.5);
    int ok = 0;
    for (int v : a.ok) ok += v;
    CHECK(ok == 100);
  }
}

}  // namespace

int main() {
  QpTests();
  ClosedLoopTests();
  std::printf("test_closedloop: %d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
