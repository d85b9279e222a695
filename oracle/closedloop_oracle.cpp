// ORACLE — TEST INFRASTRUCTURE ONLY. See closedloop_oracle.h for scope and
// parity status. Line references are to /root/reference/proj.
#include "closedloop_oracle.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>
#include <string>

namespace oracle {

namespace {

double Norm(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i] * v[i];
  return std::sqrt(s);
}

bool AllFinite(const Vec& v) {
  for (double x : v)
    if (!std::isfinite(x)) return false;
  return true;
}

// Eigen::LLT semantics: fails on a non-positive pivot (LLT.h, "x <= 0").
bool Cholesky(const Mat& a, Mat& l) {
  const std::int64_t n = a.rows;
  l = Mat(n, n);
  for (std::int64_t j = 0; j < n; ++j) {
    double d = a(j, j);
    for (std::int64_t k = 0; k < j; ++k) d -= l(j, k) * l(j, k);
    if (d <= 0.0) return false;
    const double ljj = std::sqrt(d);
    l(j, j) = ljj;
    for (std::int64_t i = j + 1; i < n; ++i) {
      double s = a(i, j);
      for (std::int64_t k = 0; k < j; ++k) s -= l(i, k) * l(j, k);
      l(i, j) = s / ljj;
    }
  }
  return true;
}

Vec CholSolve(const Mat& l, const Vec& b) {
  const std::int64_t n = l.rows;
  Vec y(b);
  for (std::int64_t i = 0; i < n; ++i) {
    for (std::int64_t k = 0; k < i; ++k) y[i] -= l(i, k) * y[k];
    y[i] /= l(i, i);
  }
  for (std::int64_t i = n - 1; i >= 0; --i) {
    for (std::int64_t k = i + 1; k < n; ++k) y[i] -= l(k, i) * y[k];
    y[i] /= l(i, i);
  }
  return y;
}

// qp.cpp:10-31 (QpData::Validate; general rows are not represented here)
void ValidateQp(const QpData& qp) {
  if (qp.horizon < 1 || qp.nx < 1 || qp.nu < 1) throw ConfigError("qp data: bad dimensions");
  const size_t n = static_cast<size_t>(qp.horizon);
  if (qp.a.size() != n || qp.b.size() != n || qp.phi_res.size() != n || qp.q.size() != n + 1 ||
      qp.r.size() != n || qp.hx_diag.size() != n + 1 || qp.hu_diag.size() != n || qp.du_lb.size() != n ||
      qp.du_ub.size() != n)
    throw ConfigError("qp data: inconsistent block counts");
  for (size_t k = 0; k < n; ++k) {
    if (qp.a[k].rows != qp.nx || qp.a[k].cols != qp.nx || qp.b[k].rows != qp.nx || qp.b[k].cols != qp.nu)
      throw ConfigError("qp data: continuity block shape mismatch at node " + std::to_string(k));
    for (int i = 0; i < qp.nu; ++i)
      if (qp.du_lb[k][i] > qp.du_ub[k][i])
        throw ConfigError("qp data: crossed input bounds at node " + std::to_string(k));
  }
}

// qp.cpp:77-102
Vec SolveFreeSubproblem(const Mat& h, const Vec& g, const Vec& x, const std::vector<std::int8_t>& active,
                        const std::vector<int>& free_idx, bool* regularized) {
  const int nf = static_cast<int>(free_idx.size());
  Mat hff(nf, nf);
  Vec rhs(nf);
  for (int i = 0; i < nf; ++i) {
    rhs[i] = -g[free_idx[i]];
    for (int j = 0; j < nf; ++j) hff(i, j) = h(free_idx[i], free_idx[j]);
  }
  for (int i = 0; i < nf; ++i) {
    double dot = 0.0;
    for (std::int64_t j = 0; j < h.cols; ++j)
      if (active[j] != 0) dot += h(free_idx[i], j) * x[j];
    rhs[i] -= dot;
  }
  Mat l;
  if (!Cholesky(hff, l)) {
    double tr = 0.0;
    for (int i = 0; i < nf; ++i) tr += hff(i, i);
    const double bump = 1e-9 * std::max(1.0, tr / std::max(1, nf));
    for (int i = 0; i < nf; ++i) hff(i, i) += bump;
    if (regularized != nullptr) *regularized = true;
    if (!Cholesky(hff, l)) throw std::runtime_error("box qp: Hessian not positive definite even after regularization");
  }
  return CholSolve(l, rhs);
}

// ---- simharness.cpp:41-64 ramps
double Ramp(double t, double rt) {
  if (rt <= 0.0 || t >= rt) return 1.0;
  const double s = std::max(0.0, t / rt);
  return s * s * (3.0 - 2.0 * s);
}
double RampIntegral(double t, double rt) {
  if (rt <= 0.0) return std::max(0.0, t);
  if (t <= 0.0) return 0.0;
  if (t >= rt) return 0.5 * rt + (t - rt);
  const double s = t / rt;
  return rt * (s * s * s - 0.5 * s * s * s * s);
}
double RampDerivative(double t, double rt) {
  if (rt <= 0.0 || t <= 0.0 || t >= rt) return 0.0;
  const double s = t / rt;
  return (6.0 * s - 6.0 * s * s) / rt;
}

void QuatMul(const double a[4], const double b[4], double o[4]) {  // quat.hpp:20-25
  o[0] = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
  o[1] = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
  o[2] = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
  o[3] = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
}

void RotToQuat(const double r[9], double q[4]) {  // quat.hpp:77-99 (Shepperd)
  auto R = [&](int i, int j) { return r[3 * i + j]; };
  const double tr = R(0, 0) + R(1, 1) + R(2, 2);
  if (tr > 0.0) {
    const double s = std::sqrt(tr + 1.0) * 2.0;
    q[0] = 0.25 * s; q[1] = (R(2, 1) - R(1, 2)) / s; q[2] = (R(0, 2) - R(2, 0)) / s; q[3] = (R(1, 0) - R(0, 1)) / s;
  } else if (R(0, 0) > R(1, 1) && R(0, 0) > R(2, 2)) {
    const double s = std::sqrt(1.0 + R(0, 0) - R(1, 1) - R(2, 2)) * 2.0;
    q[0] = (R(2, 1) - R(1, 2)) / s; q[1] = 0.25 * s; q[2] = (R(0, 1) + R(1, 0)) / s; q[3] = (R(0, 2) + R(2, 0)) / s;
  } else if (R(1, 1) > R(2, 2)) {
    const double s = std::sqrt(1.0 + R(1, 1) - R(0, 0) - R(2, 2)) * 2.0;
    q[0] = (R(0, 2) - R(2, 0)) / s; q[1] = (R(0, 1) + R(1, 0)) / s; q[2] = 0.25 * s; q[3] = (R(1, 2) + R(2, 1)) / s;
  } else {
    const double s = std::sqrt(1.0 + R(2, 2) - R(0, 0) - R(1, 1)) * 2.0;
    q[0] = (R(1, 0) - R(0, 1)) / s; q[1] = (R(0, 2) + R(2, 0)) / s; q[2] = (R(1, 2) + R(2, 1)) / s; q[3] = 0.25 * s;
  }
  if (q[0] < 0.0)
    for (int i = 0; i < 4; ++i) q[i] = -q[i];
  const double n = Norm(q, 4);
  for (int i = 0; i < 4; ++i) q[i] /= n;
}

void Cross(const double a[3], const double b[3], double o[3]) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

// ---- qp.cpp:33-73 -------------------------------------------------------------
CondensedQp Condense(const QpData& qp, const Vec& dx0) {
  ValidateQp(qp);
  if (static_cast<int>(dx0.size()) != qp.nx) throw ConfigError("condense: dx0 has wrong dimension");
  const int n = qp.horizon, nx = qp.nx, nu = qp.nu, nv = n * nu;
  CondensedQp c;
  c.nu = nu;
  c.recover_m.assign(n + 1, Mat(nx, nv));
  c.recover_c.assign(n + 1, Vec(nx, 0.0));
  c.recover_c[0] = dx0;
  for (int k = 0; k < n; ++k) {
    Mat& mk1 = c.recover_m[k + 1];
    const Mat& mk = c.recover_m[k];
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nv; ++j) {
        double s = 0.0;
        for (int m = 0; m < nx; ++m) s += qp.a[k](i, m) * mk(m, j);
        mk1(i, j) = s;
      }
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nu; ++j) mk1(i, k * nu + j) += qp.b[k](i, j);
    for (int i = 0; i < nx; ++i) {
      double s = 0.0;
      for (int m = 0; m < nx; ++m) s += qp.a[k](i, m) * c.recover_c[k][m];
      c.recover_c[k + 1][i] = s + qp.phi_res[k][i];
    }
  }
  c.hessian = Mat(nv, nv);
  c.gradient.assign(nv, 0.0);
  for (int k = 0; k <= n; ++k) {
    const Mat& m = c.recover_m[k];
    for (int i = 0; i < nv; ++i)
      for (int j = 0; j < nv; ++j) {
        double s = 0.0;
        for (int r = 0; r < nx; ++r) s += m(r, i) * (qp.hx_diag[k][r] * m(r, j));
        c.hessian(i, j) += s;
      }
    for (int i = 0; i < nv; ++i) {
      double s = 0.0;
      for (int r = 0; r < nx; ++r) s += m(r, i) * (qp.q[k][r] + qp.hx_diag[k][r] * c.recover_c[k][r]);
      c.gradient[i] += s;
    }
  }
  c.lb.assign(nv, 0.0);
  c.ub.assign(nv, 0.0);
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < nu; ++j) {
      c.hessian(k * nu + j, k * nu + j) += qp.hu_diag[k][j];
      c.gradient[k * nu + j] += qp.r[k][j];
      c.lb[k * nu + j] = qp.du_lb[k][j];
      c.ub[k * nu + j] = qp.du_ub[k][j];
    }
  Mat h = c.hessian;  // keep it exactly symmetric against accumulation drift
  for (int i = 0; i < nv; ++i)
    for (int j = 0; j < nv; ++j) c.hessian(i, j) = 0.5 * (h(i, j) + h(j, i));
  return c;
}

// ---- qp.cpp:104-208 -----------------------------------------------------------
BoxQpResult SolveBoxQp(const CondensedQp& qp, const std::vector<std::int8_t>* warm_start, int max_iterations) {
  const int n = static_cast<int>(qp.gradient.size());
  for (int i = 0; i < n; ++i)
    if (qp.lb[i] > qp.ub[i]) throw ConfigError("box qp: crossed bounds");
  BoxQpResult res;
  res.active.assign(n, 0);
  Vec x(n, 0.0);
  if (warm_start != nullptr && static_cast<int>(warm_start->size()) == n) res.active = *warm_start;
  for (int i = 0; i < n; ++i) {
    if (res.active[i] < 0 && !std::isfinite(qp.lb[i])) res.active[i] = 0;
    if (res.active[i] > 0 && !std::isfinite(qp.ub[i])) res.active[i] = 0;
    if (res.active[i] < 0) x[i] = qp.lb[i];
    if (res.active[i] > 0) x[i] = qp.ub[i];
    if (res.active[i] == 0) x[i] = std::clamp(0.0, qp.lb[i], qp.ub[i]);
  }
  auto grad_at = [&](const Vec& xv) {
    Vec g(n);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < n; ++j) s += qp.hessian(i, j) * xv[j];
      g[i] = s + qp.gradient[i];
    }
    return g;
  };
  constexpr double kTol = 1e-11;
  for (res.iterations = 0; res.iterations < max_iterations; ++res.iterations) {
    std::vector<int> free_idx;
    for (int i = 0; i < n; ++i)
      if (res.active[i] == 0) free_idx.push_back(i);
    bool at_opt = true;
    if (!free_idx.empty()) {
      const Vec xf = SolveFreeSubproblem(qp.hessian, qp.gradient, x, res.active, free_idx, &res.regularized);
      double alpha = 1.0;
      int blocking = -1;
      std::int8_t side = 0;
      for (size_t i = 0; i < free_idx.size(); ++i) {
        const int idx = free_idx[i];
        const double step = xf[i] - x[idx];
        if (step > kTol && std::isfinite(qp.ub[idx])) {
          const double a = (qp.ub[idx] - x[idx]) / step;
          if (a < alpha - kTol) {
            alpha = a;
            blocking = idx;
            side = 1;
          }
        } else if (step < -kTol && std::isfinite(qp.lb[idx])) {
          const double a = (qp.lb[idx] - x[idx]) / step;
          if (a < alpha - kTol) {
            alpha = a;
            blocking = idx;
            side = -1;
          }
        }
      }
      for (size_t i = 0; i < free_idx.size(); ++i) {
        const int idx = free_idx[i];
        x[idx] += alpha * (xf[i] - x[idx]);
      }
      if (blocking >= 0) {
        res.active[blocking] = side;
        x[blocking] = side > 0 ? qp.ub[blocking] : qp.lb[blocking];
        at_opt = false;
      }
    }
    if (at_opt) {
      const Vec grad = grad_at(x);
      int worst = -1;
      double worst_val = -1e-10;
      for (int i = 0; i < n; ++i) {
        if (res.active[i] == 0) continue;
        const double lam = res.active[i] < 0 ? grad[i] : -grad[i];
        if (lam < worst_val) {
          worst_val = lam;
          worst = i;
        }
      }
      if (worst < 0) {
        res.lam_lb.assign(n, 0.0);
        res.lam_ub.assign(n, 0.0);
        for (int i = 0; i < n; ++i) {
          if (res.active[i] < 0) res.lam_lb[i] = std::max(0.0, grad[i]);
          if (res.active[i] > 0) res.lam_ub[i] = std::max(0.0, -grad[i]);
        }
        res.x = x;
        res.status = QpStatus::kOptimal;
        ++res.iterations;
        return res;
      }
      res.active[worst] = 0;
    }
  }
  const Vec grad = grad_at(x);
  res.lam_lb.assign(n, 0.0);
  res.lam_ub.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    if (res.active[i] < 0) res.lam_lb[i] = std::max(0.0, grad[i]);
    if (res.active[i] > 0) res.lam_ub[i] = std::max(0.0, -grad[i]);
  }
  res.x = x;
  res.status = QpStatus::kMaxIter;
  return res;
}

// ---- sqp_rti.cpp:157-180 ------------------------------------------------------
FeedbackResult SolveFeedback(const QpData& qp, const Vec& x_measured, const std::vector<Vec>& xs,
                             const std::vector<Vec>& us, std::vector<std::int8_t>* warm_active) {
  if (!AllFinite(x_measured)) throw std::runtime_error("feedback: non-finite measured state");
  Vec dx0(x_measured.size());
  for (size_t i = 0; i < dx0.size(); ++i) dx0[i] = x_measured[i] - xs[0][i];
  const CondensedQp cqp = Condense(qp, dx0);
  const BoxQpResult sol = SolveBoxQp(cqp, warm_active != nullptr && !warm_active->empty() ? warm_active : nullptr);
  if (warm_active != nullptr) *warm_active = sol.active;
  FeedbackResult fb;
  fb.qp_iterations = sol.iterations;
  fb.regularized = sol.regularized;
  fb.status = sol.status;
  const int n = qp.horizon, nx = qp.nx, nu = qp.nu, nv = n * nu;
  fb.dxs.resize(n + 1);
  for (int k = 0; k <= n; ++k) {
    fb.dxs[k].assign(nx, 0.0);
    for (int i = 0; i < nx; ++i) {
      double s = 0.0;
      for (int j = 0; j < nv; ++j) s += cqp.recover_m[k](i, j) * sol.x[j];
      fb.dxs[k][i] = s + cqp.recover_c[k][i];
    }
  }
  fb.dus.resize(n);
  for (int k = 0; k < n; ++k) fb.dus[k].assign(sol.x.begin() + k * nu, sol.x.begin() + (k + 1) * nu);
  fb.u_command.resize(nu);
  for (int i = 0; i < nu; ++i) fb.u_command[i] = us[0][i] + fb.dus[0][i];
  if (!AllFinite(sol.x) || !AllFinite(fb.u_command)) throw std::runtime_error("feedback: non-finite QP solution");
  return fb;
}

// ---- sqp_rti.cpp:44-57, 182-280 ---------------------------------------------
RtiController::RtiController(const QuadParams& params, const OcpConfig& cfg, PrepareFn prepare, BuildFn build)
    : params_(params), plant_(MakeQuadrotorPlant(params, "full")), cfg_(cfg), prepare_(std::move(prepare)),
      build_(std::move(build)) {
  cfg_.Validate(plant_.nx, plant_.nu);
  last_command_.assign(plant_.nu, 0.0);
}

void RtiController::Initialize(const Vec& x0, const std::vector<Vec>& rxs, const std::vector<Vec>&) {
  xs_ = rxs;  // InitIterate: states from the window, head replaced by x0, hover inputs
  xs_[0] = x0;
  us_.assign(cfg_.horizon, Vec(plant_.nu, params_.HoverThrustPerRotor()));
  last_command_ = us_[0];
  warm_.clear();
}

Vec RtiController::Cycle(const Vec& x_measured, const std::vector<Vec>& rxs, const std::vector<Vec>& rus) {
  const int n = cfg_.horizon;
  QpData qp;
  bool ok = true;
  if (build_) {  // phases 1+2 together (device fused cycle)
    try {
      qp = build_(xs_, us_, rxs, rus);
    } catch (const std::exception&) {
      ok = false;
    }
  } else {
    Vec z;
    for (int k = 0; k < n; ++k) {
      const Vec f = plant_.features(xs_[k], us_[k], Vec());
      z.insert(z.end(), f.begin(), f.end());
    }
    const std::vector<TaylorApprox> approxes = prepare_(z, n, cfg_.taylor_order);  // phase 1 propagates
    try {
      qp = BuildQp(plant_, cfg_, xs_, us_, rxs, rus, &approxes, nullptr);
    } catch (const std::exception&) {
      ok = false;
    }
  }
  if (ok) {
    FeedbackResult fb;
    try {
      fb = SolveFeedback(qp, x_measured, xs_, us_, &warm_);
      ok = fb.status == QpStatus::kOptimal;
    } catch (const std::exception&) {
      ok = false;
    }
    if (ok) {
      for (int k = 0; k <= n; ++k) {
        for (int i = 0; i < plant_.nx; ++i) xs_[k][i] += fb.dxs[k][i];
        double* q = &xs_[k][kQuatRow];
        const double nq = Norm(q, 4);
        if (nq > 0.0)
          for (int i = 0; i < 4; ++i) q[i] /= nq;
      }
      for (int k = 0; k < n; ++k)
        for (int i = 0; i < plant_.nu; ++i) us_[k][i] += fb.dus[k][i];
      last_command_ = us_[0];
      for (int k = 0; k < n; ++k) xs_[k] = xs_[k + 1];
      for (int k = 0; k + 1 < n; ++k) us_[k] = us_[k + 1];
    }
  }
  ok_ = ok;
  return last_command_;
}

// ---- simharness.cpp:70-158 ----------------------------------------------------
ReferenceGenerator::ReferenceGenerator(const TrajectoryCfg& traj, const QuadParams& params) : traj_(traj) {
  if (!(traj.speed > 0.0)) throw ConfigError("trajectory: speed must be positive");
  if (!(traj.scale > 0.0)) throw ConfigError("trajectory: scale must be positive");
  if (!(traj.duration > 0.0) || traj.ramp_time < 0.0) throw ConfigError("trajectory: bad duration or ramp time");
  params.Validate();
  hover_ = params.HoverThrustPerRotor();
  const int n = 20000;
  const double h = 2.0 * M_PI / n;
  auto speed_at = [this](double th) {
    const double eps = 1e-6;
    double a[3], b[3], d[3];
    Pos(th + eps, a);
    Pos(th - eps, b);
    for (int i = 0; i < 3; ++i) d[i] = (a[i] - b[i]) / (2.0 * eps);
    return Norm(d, 3);
  };
  double sum = speed_at(0.0) + speed_at(2.0 * M_PI);
  for (int i = 1; i < n; ++i) sum += speed_at(i * h) * (i % 2 == 1 ? 4.0 : 2.0);
  lap_ = sum * h / 3.0;
  omega_rate_ = 2.0 * M_PI * traj_.speed / lap_;
}

void ReferenceGenerator::Pos(double theta, double p[3]) const {
  const double a = traj_.scale;
  if (traj_.kind == 0) {
    p[0] = a * std::cos(theta);
    p[1] = a * std::sin(theta);
  } else {
    const double s = std::sin(theta), c = std::cos(theta), d = 1.0 + s * s;
    p[0] = a * c / d;
    p[1] = a * s * c / d;
  }
  p[2] = traj_.z0;
}

void ReferenceGenerator::Eval(double t, Vec& x, Vec& u) const {
  const double theta = omega_rate_ * RampIntegral(t, traj_.ramp_time);
  const double theta_dot = omega_rate_ * Ramp(t, traj_.ramp_time);
  const double theta_ddot = omega_rate_ * RampDerivative(t, traj_.ramp_time);
  const double h = 1e-5;
  double p[3], pp[3], pm[3], dp[3], ddp[3], vel[3], acc[3];
  Pos(theta, p);
  Pos(theta + h, pp);
  Pos(theta - h, pm);
  for (int i = 0; i < 3; ++i) {
    dp[i] = (pp[i] - pm[i]) / (2.0 * h);
    ddp[i] = (pp[i] - 2.0 * p[i] + pm[i]) / (h * h);
    vel[i] = dp[i] * theta_dot;
    acc[i] = ddp[i] * theta_dot * theta_dot + dp[i] * theta_ddot;
  }
  double zb[3] = {acc[0], acc[1], acc[2] + kGravity};
  const double nz = Norm(zb, 3);
  for (double& v : zb) v /= nz;
  const double xc[3] = {1.0, 0.0, 0.0};
  double yb[3], xb[3];
  Cross(zb, xc, yb);
  const double ny = Norm(yb, 3);
  for (double& v : yb) v /= ny;
  Cross(yb, zb, xb);
  const double r[9] = {xb[0], yb[0], zb[0], xb[1], yb[1], zb[1], xb[2], yb[2], zb[2]};
  x.assign(kQuadNx, 0.0);
  for (int i = 0; i < 3; ++i) {
    x[i] = p[i];
    x[kVelRow + i] = vel[i];
  }
  RotToQuat(r, &x[kQuatRow]);
  u.assign(kQuadNu, hover_);
}

void ReferenceGenerator::At(double t, Vec& x, Vec& u) const {
  if (t < 0.0 || t > traj_.duration) throw InputDomainError("reference: t outside [0, duration]");
  Eval(t, x, u);
  const double h = 5e-4;
  const double t0 = std::max(0.0, t - h), t1 = std::min(traj_.duration, t + h);
  Vec x0, x1, dummy;
  Eval(t0, x0, dummy);
  Eval(t1, x1, dummy);
  double q0[4], q1[4], q[4];
  for (int i = 0; i < 4; ++i) {
    q0[i] = x0[kQuatRow + i];
    q1[i] = x1[kQuatRow + i];
    q[i] = x[kQuatRow + i];
  }
  double d0 = 0.0, d1 = 0.0;
  for (int i = 0; i < 4; ++i) {
    d0 += q0[i] * q[i];
    d1 += q1[i] * q[i];
  }
  if (d0 < 0.0)
    for (double& v : q0) v = -v;
  if (d1 < 0.0)
    for (double& v : q1) v = -v;
  double qd[4], qc[4] = {q[0], -q[1], -q[2], -q[3]}, w[4];
  for (int i = 0; i < 4; ++i) qd[i] = (q1[i] - q0[i]) / (t1 - t0);
  QuatMul(qc, qd, w);
  for (int i = 0; i < 3; ++i) x[kOmegaRow + i] = 2.0 * w[1 + i];
}

void ReferenceGenerator::Window(double t, int horizon, double dt, std::vector<Vec>& xs, std::vector<Vec>& us) const {
  xs.clear();
  us.clear();
  for (int k = 0; k <= horizon; ++k) {
    const double tk = std::clamp(t + k * dt, 0.0, traj_.duration);
    Vec x, u;
    At(tk, x, u);
    xs.push_back(x);
    if (k < horizon) us.push_back(u);
  }
}

// ---- simharness.cpp:163-213 ---------------------------------------------------
QuadSim::QuadSim(const QuadParams& params, const SimConfig& cfg) : params_(params), cfg_(cfg) {
  params_.Validate();
  if (!(cfg_.sim_dt > 0.0) || !(cfg_.control_rate_hz > 0.0))
    throw ConfigError("sim config: sim_dt and control_rate_hz must be positive");
  if (cfg_.sim_dt > 1.0 / cfg_.control_rate_hz + 1e-12)
    throw ConfigError("sim config: sim_dt must not exceed the control period");
  Reset(cfg_.seed);
}

void QuadSim::Reset(std::uint64_t seed) {
  rng_.seed(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  const double f_sigma = cfg_.noise_ft_sigma * params_.mass * kGravity;
  const double t_sigma = cfg_.noise_ft_sigma * params_.mass * kGravity * params_.arm_length;
  for (int i = 0; i < 3; ++i) accel_noise_[i] = dist(rng_) * f_sigma / params_.mass;
  for (int i = 0; i < 3; ++i) torque_noise_[i] = dist(rng_) * t_sigma;
}

Vec QuadSim::Derivative(const Vec& x, const Vec& u) const {
  Vec f = QuadNominalDynamics(x, u, params_);
  const double* q = &x[kQuatRow];
  double vb[3], dv[3], da[3];
  QuatRotateInv(q, &x[kVelRow], vb);
  for (int i = 0; i < 3; ++i) dv[i] = cfg_.drag[i] * vb[i];
  QuatRotate(q, dv, da);
  for (int i = 0; i < 3; ++i) {
    f[kVelRow + i] += (-da[i] + accel_noise_[i]) + 0.0;  // + const_accel_disturbance (zero)
    f[kOmegaRow + i] += torque_noise_[i] / params_.inertia[i];
  }
  return f;
}

Vec QuadSim::Step(const Vec& x, const Vec& u_cmd, double dt_ctrl) {
  std::normal_distribution<double> dist(0.0, 1.0);
  if (cfg_.per_step_noise) {
    const double f_sigma = cfg_.noise_ft_sigma * params_.mass * kGravity;
    const double t_sigma = f_sigma * params_.arm_length;
    for (int i = 0; i < 3; ++i) accel_noise_[i] = dist(rng_) * f_sigma / params_.mass;
    for (int i = 0; i < 3; ++i) torque_noise_[i] = dist(rng_) * t_sigma;
  }
  Vec u = u_cmd;
  for (size_t i = 0; i < u.size(); ++i) {
    const double sigma = cfg_.motor_noise_coeff * std::sqrt(std::max(0.0, u_cmd[i]));
    u[i] = std::clamp(u_cmd[i] + sigma * dist(rng_), 0.0, params_.thrust_max);
  }
  const DynFn f = [this](const Vec& xs, const Vec& us) { return Derivative(xs, us); };
  const int substeps = std::max(1, static_cast<int>(std::lround(dt_ctrl / cfg_.sim_dt)));
  const double h = dt_ctrl / substeps;
  Vec state = x;
  for (int s = 0; s < substeps; ++s) state = Rk4Step(f, state, u, h, kQuatRow);
  return state;
}

// ---- simharness.cpp:218-267 ---------------------------------------------------
Rollout RunClosedLoop(RtiController& ctrl, QuadSim& sim, const ReferenceGenerator& refs, const OcpConfig& cfg,
                      double duration, std::uint64_t seed) {
  const double period = 1.0 / sim.config().control_rate_hz;
  const int steps = static_cast<int>(std::floor(duration / period));
  sim.Reset(seed);
  Vec x, u0;
  refs.At(0.0, x, u0);
  std::vector<Vec> wx, wu;
  refs.Window(0.0, cfg.horizon, cfg.dt, wx, wu);
  ctrl.Initialize(x, wx, wu);
  Rollout log;
  for (int k = 0; k < steps; ++k) {
    const double t = k * period;
    Vec u;
    refs.Window(t, cfg.horizon, cfg.dt, wx, wu);
    try {
      u = ctrl.Cycle(x, wx, wu);
    } catch (const std::exception&) {
      log.failed = true;
      break;
    }
    log.states.push_back(x);
    log.commands.push_back(u);
    log.ok.push_back(ctrl.last_ok() ? 1 : 0);
    Vec rx, ru;
    refs.At(t, rx, ru);
    try {
      x = sim.Step(x, u, period);
    } catch (const std::exception&) {
      log.failed = true;
      break;
    }
    double dp[3] = {x[0] - rx[0], x[1] - rx[1], x[2] - rx[2]};
    if (!AllFinite(x) || Norm(dp, 3) > 50.0) {
      log.failed = true;
      break;
    }
  }
  return log;
}

}  // namespace oracle

// ---------------------------------------------------------------------------
// C entry point (ctypes): one closed-loop rollout of the quadrotor with the
// 'full' residual in rtn mode. Phase 1 comes from `prep` (NULL = the oracle's
// own PrepareNodes on `model`); phases 1+2 from `blocks` when it is non-NULL.
//   params[11] QuadParams; cfg[39] = dt, q13, r4, qf13, umin4, umax4
//   traj[6] = kind, scale, speed, duration, z0, ramp_time
//   sim[7]  = drag3, noise_ft_sigma, motor_noise_coeff, sim_dt, control_rate_hz
extern "C" {

typedef int (*oracle_prep_cb)(const double* z, int k, int order, double* f, double* jac, double* hess, void* user);
typedef int (*oracle_blocks_cb)(const double* xs, const double* us, const double* rxs, const double* rus, int n,
                                double* a, double* b, double* phi, double* q, double* r, double* hx, double* hu,
                                double* lb, double* ub, void* user);

static thread_local std::string g_cl_err;
const char* oracle_closed_loop_last_error() { return g_cl_err.c_str(); }

int oracle_closed_loop(const void* model, const double* params, const double* cfgv, int horizon, int has_qf,
                       int order, const double* traj, const double* simv, int per_step_noise, double duration,
                       unsigned long long seed, oracle_prep_cb prep, oracle_blocks_cb blocks, void* user,
                       double* states, double* commands, int* ok, int max_steps, int* n_steps, int* failed) {
  using namespace oracle;
  try {
    QuadParams qp;
    qp.mass = params[0];
    for (int i = 0; i < 3; ++i) qp.inertia[i] = params[1 + i];
    qp.arm_length = params[4];
    qp.torque_coeff = params[5];
    qp.thrust_max = params[6];
    for (int i = 0; i < 4; ++i) qp.rotor_sign[i] = params[7 + i];
    OcpConfig cfg;
    cfg.horizon = horizon;
    cfg.dt = cfgv[0];
    cfg.q_diag.assign(cfgv + 1, cfgv + 14);
    cfg.r_diag.assign(cfgv + 14, cfgv + 18);
    if (has_qf) cfg.q_terminal.assign(cfgv + 18, cfgv + 31);
    cfg.u_min.assign(cfgv + 31, cfgv + 35);
    cfg.u_max.assign(cfgv + 35, cfgv + 39);
    cfg.taylor_order = order;
    const int n = horizon, nf = 17, nr = 6;
    PrepareFn pf;
    const MlpModel* m = static_cast<const MlpModel*>(model);
    if (prep == nullptr) {
      if (m == nullptr && blocks == nullptr)
        throw ConfigError("closed loop: need a model, a prepare callback or a blocks callback");
      if (m != nullptr) pf = [m](const Vec& z, int k, int ord) { return PrepareNodes(*m, z.data(), k, 17, ord); };
    } else {
      pf = [prep, user, nf, nr](const Vec& z, int k, int ord) {
        Vec f(static_cast<size_t>(k) * nr), j(static_cast<size_t>(k) * nr * nf), h;
        if (ord == 2) h.resize(static_cast<size_t>(k) * nr * nf * nf);
        if (prep(z.data(), k, ord, f.data(), j.data(), ord == 2 ? h.data() : nullptr, user) != 0)
          throw std::runtime_error("closed loop: prepare callback failed");
        std::vector<TaylorApprox> out(k);
        for (int i = 0; i < k; ++i) {
          out[i].node = i;
          out[i].order = ord;
          out[i].z0.assign(z.begin() + i * nf, z.begin() + (i + 1) * nf);
          out[i].f_bar.assign(f.begin() + i * nr, f.begin() + (i + 1) * nr);
          out[i].jac.assign(j.begin() + static_cast<size_t>(i) * nr * nf, j.begin() + static_cast<size_t>(i + 1) * nr * nf);
          if (ord == 2)
            out[i].hess.assign(h.begin() + static_cast<size_t>(i) * nr * nf * nf,
                               h.begin() + static_cast<size_t>(i + 1) * nr * nf * nf);
        }
        return out;
      };
    }
    BuildFn bf;
    if (blocks != nullptr) {
      bf = [blocks, user, n](const std::vector<Vec>& xs, const std::vector<Vec>& us, const std::vector<Vec>& rxs,
                             const std::vector<Vec>& rus) {
        Vec fx, fu, frx, fru;
        for (const auto& v : xs) fx.insert(fx.end(), v.begin(), v.end());
        for (const auto& v : us) fu.insert(fu.end(), v.begin(), v.end());
        for (const auto& v : rxs) frx.insert(frx.end(), v.begin(), v.end());
        for (const auto& v : rus) fru.insert(fru.end(), v.begin(), v.end());
        Vec a(n * 169), b(n * 52), phi(n * 13), q((n + 1) * 13), r(n * 4), hx((n + 1) * 13), hu(n * 4), lb(n * 4),
            ub(n * 4);
        if (blocks(fx.data(), fu.data(), frx.data(), fru.data(), n, a.data(), b.data(), phi.data(), q.data(), r.data(),
                   hx.data(), hu.data(), lb.data(), ub.data(), user) != 0)
          throw std::runtime_error("closed loop: blocks callback failed");
        QpData d;
        d.nx = 13;
        d.nu = 4;
        d.horizon = n;
        for (int k = 0; k < n; ++k) {
          Mat ak(13, 13), bk(13, 4);
          std::copy(a.begin() + k * 169, a.begin() + (k + 1) * 169, ak.v.begin());
          std::copy(b.begin() + k * 52, b.begin() + (k + 1) * 52, bk.v.begin());
          d.a.push_back(ak);
          d.b.push_back(bk);
          d.phi_res.emplace_back(phi.begin() + k * 13, phi.begin() + (k + 1) * 13);
          d.r.emplace_back(r.begin() + k * 4, r.begin() + (k + 1) * 4);
          d.hu_diag.emplace_back(hu.begin() + k * 4, hu.begin() + (k + 1) * 4);
          d.du_lb.emplace_back(lb.begin() + k * 4, lb.begin() + (k + 1) * 4);
          d.du_ub.emplace_back(ub.begin() + k * 4, ub.begin() + (k + 1) * 4);
        }
        for (int k = 0; k <= n; ++k) {
          d.q.emplace_back(q.begin() + k * 13, q.begin() + (k + 1) * 13);
          d.hx_diag.emplace_back(hx.begin() + k * 13, hx.begin() + (k + 1) * 13);
        }
        return d;
      };
    }
    TrajectoryCfg tc;
    tc.kind = static_cast<int>(traj[0]);
    tc.scale = traj[1];
    tc.speed = traj[2];
    tc.duration = traj[3];
    tc.z0 = traj[4];
    tc.ramp_time = traj[5];
    SimConfig sc;
    for (int i = 0; i < 3; ++i) sc.drag[i] = simv[i];
    sc.noise_ft_sigma = simv[3];
    sc.motor_noise_coeff = simv[4];
    sc.sim_dt = simv[5];
    sc.control_rate_hz = simv[6];
    sc.per_step_noise = per_step_noise != 0;
    sc.seed = seed;
    RtiController ctrl(qp, cfg, pf, bf);
    QuadSim sim(qp, sc);
    ReferenceGenerator refs(tc, qp);
    const Rollout r = RunClosedLoop(ctrl, sim, refs, cfg, duration, seed);
    const int steps = std::min<int>(static_cast<int>(r.states.size()), max_steps);
    for (int k = 0; k < steps; ++k) {
      std::copy(r.states[k].begin(), r.states[k].end(), states + k * 13);
      std::copy(r.commands[k].begin(), r.commands[k].end(), commands + k * 4);
      ok[k] = r.ok[k];
    }
    *n_steps = steps;
    *failed = r.failed ? 1 : 0;
    return 0;
  } catch (const oracle::ConfigError& e) {
    g_cl_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_cl_err = e.what();
    return 6;
  }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// SolveFeedback (sqp_rti.cpp:157-180) for a batch of instances (QpData arrays
// in the C-ABI layout of rtn_qp_blocks), the checker of rtn_solve_feedback.
extern "C" {

int oracle_solve_feedback(int horizon, long long n_inst, const double* a, const double* b, const double* phi,
                          const double* q, const double* r, const double* hx, const double* hu, const double* lb,
                          const double* ub, const double* x_meas, const double* xs, const double* us,
                          signed char* warm /* n_inst x N*4, in/out, may be null */, double* dxs, double* dus,
                          double* u_cmd, int* status, int* iterations) {
  using namespace oracle;
  try {
    const int n = horizon, nx = 13, nu = 4, nv = n * nu;
    for (long long i = 0; i < n_inst; ++i) {
      QpData d;
      d.nx = nx;
      d.nu = nu;
      d.horizon = n;
      for (int k = 0; k < n; ++k) {
        const long long row = i * n + k;
        Mat ak(nx, nx), bk(nx, nu);
        std::copy(a + row * 169, a + (row + 1) * 169, ak.v.begin());
        std::copy(b + row * 52, b + (row + 1) * 52, bk.v.begin());
        d.a.push_back(ak);
        d.b.push_back(bk);
        d.phi_res.emplace_back(phi + row * nx, phi + (row + 1) * nx);
        d.r.emplace_back(r + row * nu, r + (row + 1) * nu);
        d.hu_diag.emplace_back(hu + row * nu, hu + (row + 1) * nu);
        d.du_lb.emplace_back(lb + row * nu, lb + (row + 1) * nu);
        d.du_ub.emplace_back(ub + row * nu, ub + (row + 1) * nu);
      }
      for (int k = 0; k <= n; ++k) {
        const long long row = i * (n + 1) + k;
        d.q.emplace_back(q + row * nx, q + (row + 1) * nx);
        d.hx_diag.emplace_back(hx + row * nx, hx + (row + 1) * nx);
      }
      std::vector<Vec> vx, vu;
      for (int k = 0; k <= n; ++k) vx.emplace_back(xs + (i * (n + 1) + k) * nx, xs + (i * (n + 1) + k + 1) * nx);
      for (int k = 0; k < n; ++k) vu.emplace_back(us + (i * n + k) * nu, us + (i * n + k + 1) * nu);
      std::vector<std::int8_t> w;
      if (warm) w.assign(warm + i * nv, warm + (i + 1) * nv);
      bool all_free = true;
      for (auto v : w) all_free = all_free && v == 0;
      if (all_free) w.clear();  // an all-zero hint is "no warm start" on both sides
      FeedbackResult fb;
      int st = 0;
      try {
        fb = SolveFeedback(d, Vec(x_meas + i * nx, x_meas + (i + 1) * nx), vx, vu, &w);
        st = fb.status == QpStatus::kOptimal ? 0 : 1;
      } catch (const std::exception&) {
        st = 2;
      }
      status[i] = st;
      iterations[i] = st == 2 ? 0 : fb.qp_iterations;
      if (st == 2) continue;
      if (warm)
        for (int j = 0; j < nv; ++j) warm[i * nv + j] = static_cast<signed char>(w.empty() ? 0 : w[j]);
      for (int k = 0; k <= n; ++k) std::copy(fb.dxs[k].begin(), fb.dxs[k].end(), dxs + (i * (n + 1) + k) * nx);
      for (int k = 0; k < n; ++k) std::copy(fb.dus[k].begin(), fb.dus[k].end(), dus + (i * n + k) * nu);
      std::copy(fb.u_command.begin(), fb.u_command.end(), u_cmd + i * nu);
    }
    return 0;
  } catch (const oracle::ConfigError& e) {
    g_cl_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_cl_err = e.what();
    return 6;
  }
}

}  // extern "C"
