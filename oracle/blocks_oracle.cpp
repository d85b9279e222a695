// ORACLE — TEST INFRASTRUCTURE ONLY. See blocks_oracle.h for scope and parity
// status. Each function cites the reference lines it restates; products are
// plain ascending-index loops (the reference routes them through Eigen).
#include "blocks_oracle.h"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>

namespace oracle {

namespace {

Mat Identity(int n) {
  Mat m(n, n);
  for (int i = 0; i < n; ++i) m(i, i) = 1.0;
  return m;
}

Mat MatMul(const Mat& a, const Mat& b) {
  Mat c(a.rows, b.cols);
  for (std::int64_t i = 0; i < a.rows; ++i)
    for (std::int64_t j = 0; j < b.cols; ++j) {
      double s = 0.0;
      for (std::int64_t k = 0; k < a.cols; ++k) s += a(i, k) * b(k, j);
      c(i, j) = s;
    }
  return c;
}

Mat Scaled(const Mat& a, double s) {
  Mat c = a;
  for (double& v : c.v) v *= s;
  return c;
}

Mat Plus(const Mat& a, const Mat& b) {
  Mat c = a;
  for (size_t i = 0; i < c.v.size(); ++i) c.v[i] += b.v[i];
  return c;
}

Vec Axpy(const Vec& x, double a, const Vec& y) {  // x + a*y
  Vec r(x.size());
  for (size_t i = 0; i < x.size(); ++i) r[i] = x[i] + a * y[i];
  return r;
}

void CheckFinite(const Vec& k, const char* stage) {  // integrator.cpp:12-15
  for (double v : k)
    if (!std::isfinite(v)) throw std::runtime_error(std::string("rk4: non-finite derivative at stage ") + stage);
}

void RenormalizeQuat(Vec& x, int quat_row) {  // integrator.cpp:17-20
  if (quat_row < 0) return;
  double n2 = 0.0;
  for (int i = 0; i < 4; ++i) n2 += x[quat_row + i] * x[quat_row + i];
  const double n = std::sqrt(n2);
  for (int i = 0; i < 4; ++i) x[quat_row + i] /= n;
}

}  // namespace

// ---- quat.hpp ---------------------------------------------------------------
void QuatToRot(const double q[4], double r[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  r[0] = 1.0 - 2.0 * (y * y + z * z);
  r[1] = 2.0 * (x * y - w * z);
  r[2] = 2.0 * (x * z + w * y);
  r[3] = 2.0 * (x * y + w * z);
  r[4] = 1.0 - 2.0 * (x * x + z * z);
  r[5] = 2.0 * (y * z - w * x);
  r[6] = 2.0 * (x * z - w * y);
  r[7] = 2.0 * (y * z + w * x);
  r[8] = 1.0 - 2.0 * (x * x + y * y);
}

void QuatRotDerivatives(const double q[4], double out[4][9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double d0[9] = {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0};
  const double d1[9] = {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x};
  const double d2[9] = {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y};
  const double d3[9] = {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0};
  for (int i = 0; i < 9; ++i) {
    out[0][i] = d0[i];
    out[1][i] = d1[i];
    out[2][i] = d2[i];
    out[3][i] = d3[i];
  }
}

void QuatRotate(const double q[4], const double v[3], double out[3]) {
  double r[9];
  QuatToRot(q, r);
  for (int i = 0; i < 3; ++i) out[i] = r[3 * i] * v[0] + r[3 * i + 1] * v[1] + r[3 * i + 2] * v[2];
}

void QuatRotateInv(const double q[4], const double v[3], double out[3]) {
  double r[9];
  QuatToRot(q, r);
  for (int i = 0; i < 3; ++i) out[i] = r[i] * v[0] + r[3 + i] * v[1] + r[6 + i] * v[2];
}

void QuatKinematics(const double q[4], const double w[3], double out[4]) {
  // 0.5 * QuatMul(q, (0, w)) — quat.hpp:20-25, 107-109
  const double b[4] = {0.0, w[0], w[1], w[2]};
  const double m[4] = {q[0] * b[0] - q[1] * b[1] - q[2] * b[2] - q[3] * b[3],
                       q[0] * b[1] + q[1] * b[0] + q[2] * b[3] - q[3] * b[2],
                       q[0] * b[2] - q[1] * b[3] + q[2] * b[0] + q[3] * b[1],
                       q[0] * b[3] + q[1] * b[2] - q[2] * b[1] + q[3] * b[0]};
  for (int i = 0; i < 4; ++i) out[i] = 0.5 * m[i];
}

// ---- dynamics.cpp -----------------------------------------------------------
void QuadParams::Validate() const {
  if (!(mass > 0.0) || !(arm_length > 0.0) || !(torque_coeff > 0.0) || !(thrust_max > 0.0))
    throw ConfigError("quad params: mass, arm_length, torque_coeff, thrust_max must be positive");
  if (!(std::min(inertia[0], std::min(inertia[1], inertia[2])) > 0.0))
    throw ConfigError("quad params: inertia must be positive");
  double sum = 0.0;
  for (int i = 0; i < 4; ++i) {
    if (rotor_sign[i] != 1.0 && rotor_sign[i] != -1.0)
      throw ConfigError("quad params: rotor_sign entries must be +1 or -1");
    sum += rotor_sign[i];
  }
  if (sum != 0.0) throw ConfigError("quad params: need two rotors of each spin direction");
}

void MixingMatrix(const QuadParams& p, double m[6][4]) {
  const double d = p.arm_length / std::sqrt(2.0);
  const double rx[4] = {d, -d, d, -d};
  const double ry[4] = {-d, d, d, -d};
  for (int r = 0; r < 6; ++r)
    for (int i = 0; i < 4; ++i) m[r][i] = 0.0;
  for (int i = 0; i < 4; ++i) {
    m[2][i] = 1.0;
    m[3][i] = ry[i];
    m[4][i] = -rx[i];
    m[5][i] = p.rotor_sign[i] * p.torque_coeff;
  }
}

Vec QuadNominalDynamics(const Vec& x, const Vec& u, const QuadParams& p) {
  if (x.size() != kQuadNx || u.size() != kQuadNu)
    throw InputDomainError("quad dynamics: bad state/input size");
  const double* q = &x[kQuatRow];
  const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  if (std::abs(qn - 1.0) > 0.25) throw InputDomainError("quad dynamics: quaternion norm too far from unit");
  const double* v = &x[kVelRow];
  const double* w = &x[kOmegaRow];
  double mix[6][4];
  MixingMatrix(p, mix);
  double wrench[6];
  for (int r = 0; r < 6; ++r) {
    double s = 0.0;
    for (int i = 0; i < 4; ++i) s += mix[r][i] * u[i];
    wrench[r] = s;
  }
  const double* t_b = wrench;
  const double* tau = wrench + 3;
  const double* j = p.inertia;
  Vec dx(kQuadNx);
  for (int i = 0; i < 3; ++i) dx[i] = v[i];
  QuatKinematics(q, w, &dx[kQuatRow]);
  double rt[3];
  QuatRotate(q, t_b, rt);
  const double g_w[3] = {0.0, 0.0, -kGravity};
  for (int i = 0; i < 3; ++i) dx[kVelRow + i] = rt[i] / p.mass + g_w[i];
  const double jw[3] = {j[0] * w[0], j[1] * w[1], j[2] * w[2]};
  const double cr[3] = {w[1] * jw[2] - w[2] * jw[1], w[2] * jw[0] - w[0] * jw[2], w[0] * jw[1] - w[1] * jw[0]};
  for (int i = 0; i < 3; ++i) dx[kOmegaRow + i] = (tau[i] - cr[i]) / j[i];
  return dx;
}

// integrator.cpp:91-123
void QuadNominalJacobians(const Vec& x, const Vec& u, const QuadParams& p, Mat& fx, Mat& fu) {
  const double* q = &x[kQuatRow];
  const double* w = &x[kOmegaRow];
  double mix[6][4];
  MixingMatrix(p, mix);
  double t_b[3];
  for (int r = 0; r < 3; ++r) {
    double s = 0.0;
    for (int i = 0; i < 4; ++i) s += mix[r][i] * u[i];
    t_b[r] = s;
  }
  const double* j = p.inertia;
  fx = Mat(kQuadNx, kQuadNx);
  fu = Mat(kQuadNx, kQuadNu);
  for (int i = 0; i < 3; ++i) fx(i, kVelRow + i) = 1.0;
  // ∂q̇/∂q (quat.hpp:112-119) and ∂q̇/∂ω (quat.hpp:122-130)
  const double jq[4][4] = {{0, -w[0], -w[1], -w[2]}, {w[0], 0, w[2], -w[1]}, {w[1], -w[2], 0, w[0]},
                           {w[2], w[1], -w[0], 0}};
  const double jw_[4][3] = {{-q[1], -q[2], -q[3]}, {q[0], -q[3], q[2]}, {q[3], q[0], -q[1]}, {-q[2], q[1], q[0]}};
  for (int r = 0; r < 4; ++r) {
    for (int c = 0; c < 4; ++c) fx(kQuatRow + r, kQuatRow + c) = 0.5 * jq[r][c];
    for (int c = 0; c < 3; ++c) fx(kQuatRow + r, kOmegaRow + c) = 0.5 * jw_[r][c];
  }
  // v̇ = R(q)·T_B/m + g
  double dr[4][9];
  QuatRotDerivatives(q, dr);
  for (int c = 0; c < 4; ++c)
    for (int r = 0; r < 3; ++r)
      fx(kVelRow + r, kQuatRow + c) =
          (dr[c][3 * r] * t_b[0] + dr[c][3 * r + 1] * t_b[1] + dr[c][3 * r + 2] * t_b[2]) / p.mass;
  double rot[9];
  QuatToRot(q, rot);
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 4; ++c)
      fu(kVelRow + r, c) = (rot[3 * r] * mix[0][c] + rot[3 * r + 1] * mix[1][c] + rot[3 * r + 2] * mix[2][c]) / p.mass;
  // ω̇ = J⁻¹(τ − ω × Jω)
  const double jwv[3] = {j[0] * w[0], j[1] * w[1], j[2] * w[2]};
  const double sw[9] = {0.0, -w[2], w[1], w[2], 0.0, -w[0], -w[1], w[0], 0.0};
  const double sjw[9] = {0.0, -jwv[2], jwv[1], jwv[2], 0.0, -jwv[0], -jwv[1], jwv[0], 0.0};
  for (int r = 0; r < 3; ++r) {
    const double inv = 1.0 / j[r];
    for (int c = 0; c < 3; ++c) {
      const double dcross = sw[3 * r + c] * j[c] - sjw[3 * r + c];
      fx(kOmegaRow + r, kOmegaRow + c) = inv * (-dcross);
    }
    for (int c = 0; c < 4; ++c) fu(kOmegaRow + r, c) = inv * mix[3 + r][c];
  }
}

// ---- integrator.cpp ---------------------------------------------------------
Vec Rk4Step(const DynFn& f, const Vec& x, const Vec& u, double dt, int quat_row, FevalCounter* counter) {
  if (!(dt > 0.0)) throw std::invalid_argument("rk4: dt must be positive");
  const Vec k1 = f(x, u);
  CheckFinite(k1, "1");
  const Vec k2 = f(Axpy(x, 0.5 * dt, k1), u);
  CheckFinite(k2, "2");
  const Vec k3 = f(Axpy(x, 0.5 * dt, k2), u);
  CheckFinite(k3, "3");
  const Vec k4 = f(Axpy(x, dt, k3), u);
  CheckFinite(k4, "4");
  if (counter != nullptr) counter->values += 4;
  Vec next(x.size());
  for (size_t i = 0; i < x.size(); ++i)
    next[i] = x[i] + (dt / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  RenormalizeQuat(next, quat_row);
  return next;
}

SensitivityResult Rk4Sensitivities(const DynFn& f, const DynJacFn& df, const Vec& x, const Vec& u, double dt,
                                   int quat_row, FevalCounter* counter) {
  if (!(dt > 0.0)) throw std::invalid_argument("rk4: dt must be positive");
  const int nx = static_cast<int>(x.size());
  const Mat eye = Identity(nx);
  Mat jx, ju;

  const Vec k1 = f(x, u);
  CheckFinite(k1, "1");
  df(x, u, jx, ju);
  const Mat dk1_dx = jx, dk1_du = ju;

  const Vec x2 = Axpy(x, 0.5 * dt, k1);
  const Vec k2 = f(x2, u);
  CheckFinite(k2, "2");
  df(x2, u, jx, ju);
  const Mat dk2_dx = MatMul(jx, Plus(eye, Scaled(dk1_dx, 0.5 * dt)));
  const Mat dk2_du = Plus(MatMul(jx, Scaled(dk1_du, 0.5 * dt)), ju);

  const Vec x3 = Axpy(x, 0.5 * dt, k2);
  const Vec k3 = f(x3, u);
  CheckFinite(k3, "3");
  df(x3, u, jx, ju);
  const Mat dk3_dx = MatMul(jx, Plus(eye, Scaled(dk2_dx, 0.5 * dt)));
  const Mat dk3_du = Plus(MatMul(jx, Scaled(dk2_du, 0.5 * dt)), ju);

  const Vec x4 = Axpy(x, dt, k3);
  const Vec k4 = f(x4, u);
  CheckFinite(k4, "4");
  df(x4, u, jx, ju);
  const Mat dk4_dx = MatMul(jx, Plus(eye, Scaled(dk3_dx, dt)));
  const Mat dk4_du = Plus(MatMul(jx, Scaled(dk3_du, dt)), ju);

  if (counter != nullptr) {
    counter->values += 4;
    counter->jacobians += 4;
  }
  SensitivityResult res;
  res.phi_bar.resize(nx);
  for (int i = 0; i < nx; ++i) res.phi_bar[i] = x[i] + (dt / 6.0) * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  RenormalizeQuat(res.phi_bar, quat_row);
  res.a = Mat(nx, nx);
  for (size_t e = 0; e < res.a.v.size(); ++e)
    res.a.v[e] = eye.v[e] + (dt / 6.0) * (dk1_dx.v[e] + 2.0 * dk2_dx.v[e] + 2.0 * dk3_dx.v[e] + dk4_dx.v[e]);
  res.b = Mat(dk1_du.rows, dk1_du.cols);
  for (size_t e = 0; e < res.b.v.size(); ++e)
    res.b.v[e] = (dt / 6.0) * (dk1_du.v[e] + 2.0 * dk2_du.v[e] + 2.0 * dk3_du.v[e] + dk4_du.v[e]);
  return res;
}

// ---- plant.cpp --------------------------------------------------------------
Plant MakeDoubleIntegratorPlant() {
  Plant p;
  p.name = "double_integrator";
  p.nx = 2;
  p.nu = 1;
  p.f = [](const Vec& x, const Vec& u) { return Vec{x[1], u[0]}; };
  p.df = [](const Vec&, const Vec&, Mat& fx, Mat& fu) {
    fx = Mat(2, 2);
    fx(0, 1) = 1.0;
    fu = Mat(2, 1);
    fu(1, 0) = 1.0;
  };
  p.feature_dim = 3;
  p.residual_dim = 2;
  p.features = [](const Vec& x, const Vec& u, const Vec&) { return Vec{x[0], x[1], u[0]}; };
  p.features_jac = [](const Vec&, const Vec&) { return Identity(3); };
  p.embed = Identity(2);
  return p;
}

Plant MakeQuadrotorPlant(const QuadParams& params, const std::string& variant) {
  params.Validate();
  if (variant != "a" && variant != "a_u" && variant != "full" && variant != "ground")
    throw ConfigError("unknown residual variant '" + variant + "' (expected a, a_u, full, ground)");
  Plant p;
  p.name = "quadrotor";
  p.nx = kQuadNx;
  p.nu = kQuadNu;
  p.quat_row = kQuatRow;
  p.f = [params](const Vec& x, const Vec& u) { return QuadNominalDynamics(x, u, params); };
  p.df = [params](const Vec& x, const Vec& u, Mat& fx, Mat& fu) { QuadNominalJacobians(x, u, params, fx, fu); };
  p.variant_tag = variant;
  const bool full = variant == "full", au = variant == "a_u", ground = variant == "ground";
  p.feature_dim = full ? 17 : (au ? 7 : (ground ? 26 : 3));  // dynamics.cpp:110-118
  p.residual_dim = full ? 6 : 3;
  // dynamics.cpp:125-152 (ResidualInput), plant.cpp:60-73 (ground: x, u, z_WB·1 − patch)
  p.features = [full, au, ground](const Vec& x, const Vec& u, const Vec& aux) {
    if (full || ground) {
      Vec z(x);
      z.insert(z.end(), u.begin(), u.end());
      if (ground) {
        if (aux.size() != 9) throw InputDomainError("quadrotor plant: ground features need a 9-entry patch aux");
        for (int i = 0; i < 9; ++i) z.push_back(x[2] - aux[i]);
      }
      return z;
    }
    Vec z(3);
    QuatRotateInv(&x[kQuatRow], &x[kVelRow], z.data());
    if (au) z.insert(z.end(), u.begin(), u.end());
    return z;
  };
  const int nf = p.feature_dim;
  // dynamics.cpp:154-180 (ResidualInputJacobian)
  p.features_jac = [full, au, ground, nf](const Vec& x, const Vec&) {
    Mat jz(nf, kQuadNx + kQuadNu);
    if (full) return Identity(17);
    if (ground) {
      for (int i = 0; i < 17; ++i) jz(i, i) = 1.0;
      for (int i = 17; i < 26; ++i) jz(i, 2) = 1.0;
      return jz;
    }
    const double* q = &x[kQuatRow];
    const double* v = &x[kVelRow];
    double dr[4][9], r[9];
    QuatRotDerivatives(q, dr);
    QuatToRot(q, r);
    for (int c = 0; c < 4; ++c)
      for (int i = 0; i < 3; ++i)  // dr[c]^T v
        jz(i, kQuatRow + c) = dr[c][i] * v[0] + dr[c][3 + i] * v[1] + dr[c][6 + i] * v[2];
    for (int i = 0; i < 3; ++i)
      for (int c = 0; c < 3; ++c) jz(i, kVelRow + c) = r[3 * c + i];
    if (au)
      for (int i = 0; i < 4; ++i) jz(3 + i, kQuadNx + i) = 1.0;
    return jz;
  };
  p.embed = Mat(kQuadNx, p.residual_dim);
  for (int i = 0; i < 3; ++i) p.embed(kVelRow + i, i) = 1.0;
  if (full)
    for (int i = 0; i < 3; ++i) p.embed(kOmegaRow + i, 3 + i) = 1.0;
  return p;
}

// ---- sqp_rti.cpp ------------------------------------------------------------
void OcpConfig::Validate(int nx, int nu) const {
  if (horizon < 1) throw ConfigError("ocp config: horizon must be >= 1");
  if (!(dt > 0.0)) throw ConfigError("ocp config: dt must be positive");
  if (static_cast<int>(q_diag.size()) != nx || static_cast<int>(r_diag.size()) != nu)
    throw ConfigError("ocp config: weight dimensions do not match the plant");
  if (!q_terminal.empty() && static_cast<int>(q_terminal.size()) != nx)
    throw ConfigError("ocp config: terminal weight dimension mismatch");
  for (double v : q_diag)
    if (v < 0.0) throw ConfigError("ocp config: weights must be nonnegative");
  for (double v : r_diag)
    if (v < 0.0) throw ConfigError("ocp config: weights must be nonnegative");
  if (static_cast<int>(u_min.size()) != nu || static_cast<int>(u_max.size()) != nu)
    throw ConfigError("ocp config: input bound dimensions do not match the plant");
  for (int i = 0; i < nu; ++i)
    if (u_min[i] >= u_max[i]) throw ConfigError("ocp config: u_min must be below u_max");
  if (taylor_order != 1 && taylor_order != 2) throw ConfigError("ocp config: taylor_order must be 1 or 2");
}

QpData BuildQp(const Plant& plant, const OcpConfig& cfg, const std::vector<Vec>& xs, const std::vector<Vec>& us,
               const std::vector<Vec>& ref_xs, const std::vector<Vec>& ref_us,
               const std::vector<TaylorApprox>* approxes, const NaiveNet* naive, FevalCounter* f_counters,
               const std::vector<Vec>* node_aux) {
  cfg.Validate(plant.nx, plant.nu);
  const int n = cfg.horizon;
  if (static_cast<int>(xs.size()) != n + 1 || static_cast<int>(us.size()) != n)
    throw ConfigError("build qp: iterate size mismatch");
  if (static_cast<int>(ref_xs.size()) != n + 1 || static_cast<int>(ref_us.size()) != n)
    throw ConfigError("build qp: reference window size mismatch");
  if (approxes != nullptr && static_cast<int>(approxes->size()) != n)
    throw ConfigError("build qp: need one prepared approximation per shooting node");
  const int nx = plant.nx, nu = plant.nu, nf = plant.feature_dim, nr = plant.residual_dim;

  QpData qp;
  qp.nx = nx;
  qp.nu = nu;
  qp.horizon = n;
  for (int k = 0; k < n; ++k) {
    DynFn fk = plant.f;
    DynJacFn dfk = plant.df;
    const Vec aux = node_aux != nullptr ? (*node_aux)[k] : Vec();  // plant.NodeAux(xs[k]) (sqp_rti.cpp:91)
    if (approxes != nullptr || naive != nullptr) {
      const TaylorApprox* ap = approxes ? &(*approxes)[k] : nullptr;
      // residual value r(z) and Jacobian jn(z) (nr x nf) at feature vector z
      auto rval = [ap, naive, nf, nr](const Vec& z) {
        if (ap == nullptr) return naive->value(z);
        Vec y(nr);
        EvalTaylor(nf, nr, ap->order, ap->z0.data(), ap->f_bar.data(), ap->jac.data(),
                   ap->hess.empty() ? nullptr : ap->hess.data(), z.data(), y.data());
        return y;
      };
      auto rjac = [ap, naive, nf, nr](const Vec& z) {
        if (ap == nullptr) return naive->jacobian(z);
        Vec j(static_cast<size_t>(nr) * nf);
        EvalTaylorJacobian(nf, nr, ap->order, ap->z0.data(), ap->jac.data(),
                           ap->hess.empty() ? nullptr : ap->hess.data(), z.data(), j.data());
        return j;
      };
      fk = [&plant, rval, nx, nr, aux](const Vec& x, const Vec& u) {
        Vec f = plant.f(x, u);
        const Vec r = rval(plant.features(x, u, aux));
        for (int i = 0; i < nx; ++i) {
          double s = 0.0;
          for (int c = 0; c < nr; ++c) s += plant.embed(i, c) * r[c];
          f[i] += s;
        }
        return f;
      };
      dfk = [&plant, rjac, nx, nu, nf, nr, aux](const Vec& x, const Vec& u, Mat& fx, Mat& fu) {
        plant.df(x, u, fx, fu);
        const Vec jn = rjac(plant.features(x, u, aux));
        const Mat jz = plant.features_jac(x, u);
        Mat chain(nx, nf);  // embed * jn
        for (int i = 0; i < nx; ++i)
          for (int c = 0; c < nf; ++c) {
            double s = 0.0;
            for (int o = 0; o < nr; ++o) s += plant.embed(i, o) * jn[static_cast<size_t>(o) * nf + c];
            chain(i, c) = s;
          }
        for (int i = 0; i < nx; ++i) {
          for (int c = 0; c < nx; ++c) {
            double s = 0.0;
            for (int m = 0; m < nf; ++m) s += chain(i, m) * jz(m, c);
            fx(i, c) += s;
          }
          for (int c = 0; c < nu; ++c) {
            double s = 0.0;
            for (int m = 0; m < nf; ++m) s += chain(i, m) * jz(m, nx + c);
            fu(i, c) += s;
          }
        }
      };
    }
    SensitivityResult sens;
    try {
      sens = Rk4Sensitivities(fk, dfk, xs[k], us[k], cfg.dt, plant.quat_row, f_counters);
    } catch (const std::exception& e) {
      throw std::runtime_error("build qp: node " + std::to_string(k) + ": " + e.what());
    }
    qp.a.push_back(sens.a);
    qp.b.push_back(sens.b);
    Vec phi(nx), q(nx), r(nu), hx(nx), hu(nu), lb(nu), ub(nu);
    for (int i = 0; i < nx; ++i) {
      phi[i] = sens.phi_bar[i] - xs[k + 1][i];
      q[i] = 2.0 * (cfg.q_diag[i] * (xs[k][i] - ref_xs[k][i]));
      hx[i] = 2.0 * cfg.q_diag[i];
    }
    for (int i = 0; i < nu; ++i) {
      r[i] = 2.0 * (cfg.r_diag[i] * (us[k][i] - ref_us[k][i]));
      hu[i] = 2.0 * cfg.r_diag[i];
      lb[i] = cfg.u_min[i] - us[k][i];
      ub[i] = cfg.u_max[i] - us[k][i];
    }
    qp.phi_res.push_back(phi);
    qp.q.push_back(q);
    qp.r.push_back(r);
    qp.hx_diag.push_back(hx);
    qp.hu_diag.push_back(hu);
    qp.du_lb.push_back(lb);
    qp.du_ub.push_back(ub);
  }
  const Vec& qf = cfg.TerminalWeight();
  Vec q(nx), hx(nx);
  for (int i = 0; i < nx; ++i) {
    q[i] = 2.0 * (qf[i] * (xs[n][i] - ref_xs[n][i]));
    hx[i] = 2.0 * qf[i];
  }
  qp.q.push_back(q);
  qp.hx_diag.push_back(hx);
  return qp;
}

}  // namespace oracle

// ---------------------------------------------------------------------------
// C entry points for the test harness (ctypes). Flat layouts match the
// product C-ABI (include/rtn_mpc.h, rtn_build_qp):
//   params[11] = mass, inertia[3], arm_length, torque_coeff, thrust_max, rotor_sign[4]
//   cfg[39]    = dt, q_diag[13], r_diag[4], q_terminal[13], u_min[4], u_max[4]
//   per instance: xs (N+1)x13, us Nx4, ref_xs (N+1)x13, ref_us Nx4,
//   approximation rows z0 Nx17, f_bar Nx6, jac Nx6x17, hess Nx6x17x17 (order 2)
//   out a Nx13x13, b Nx13x4, phi_res/q... as QpData (q and hx have N+1 rows).
extern "C" {

static thread_local std::string g_blocks_err;
const char* oracle_blocks_last_error() { return g_blocks_err.c_str(); }

static oracle::QuadParams ParamsFrom(const double* p) {
  oracle::QuadParams q;
  q.mass = p[0];
  for (int i = 0; i < 3; ++i) q.inertia[i] = p[1 + i];
  q.arm_length = p[4];
  q.torque_coeff = p[5];
  q.thrust_max = p[6];
  for (int i = 0; i < 4; ++i) q.rotor_sign[i] = p[7 + i];
  return q;
}

// variant: 0 a, 1 a_u, 2 full, 3 ground (aux: n_inst x N x 9 height patches, ground only)
int oracle_build_qp_quad(const double* params, const double* cfgv, int horizon, int has_qf, int order,
                         long long n_inst, const double* xs, const double* us, const double* rxs,
                         const double* rus, const double* z0, const double* fbar, const double* jac,
                         const double* hess, double* a, double* b, double* phi, double* q, double* r,
                         double* hx, double* hu, double* lb, double* ub, unsigned long long* fevals, int variant,
                         const double* aux) {
  using namespace oracle;
  try {
    const QuadParams qp = ParamsFrom(params);
    static const char* kVariants[4] = {"a", "a_u", "full", "ground"};
    if (variant < 0 || variant > 3) throw ConfigError("unknown residual variant");
    const Plant plant = MakeQuadrotorPlant(qp, kVariants[variant]);
    OcpConfig cfg;
    cfg.horizon = horizon;
    cfg.dt = cfgv[0];
    cfg.q_diag.assign(cfgv + 1, cfgv + 14);
    cfg.r_diag.assign(cfgv + 14, cfgv + 18);
    if (has_qf) cfg.q_terminal.assign(cfgv + 18, cfgv + 31);
    cfg.u_min.assign(cfgv + 31, cfgv + 35);
    cfg.u_max.assign(cfgv + 35, cfgv + 39);
    cfg.taylor_order = order;
    const int n = horizon, nx = kQuadNx, nu = kQuadNu, nf = plant.feature_dim, nr = plant.residual_dim;
    FevalCounter fc;
    for (long long i = 0; i < n_inst; ++i) {
      std::vector<Vec> vx, vu, vrx, vru;
      for (int k = 0; k <= n; ++k) {
        vx.emplace_back(xs + (i * (n + 1) + k) * nx, xs + (i * (n + 1) + k + 1) * nx);
        vrx.emplace_back(rxs + (i * (n + 1) + k) * nx, rxs + (i * (n + 1) + k + 1) * nx);
      }
      for (int k = 0; k < n; ++k) {
        vu.emplace_back(us + (i * n + k) * nu, us + (i * n + k + 1) * nu);
        vru.emplace_back(rus + (i * n + k) * nu, rus + (i * n + k + 1) * nu);
      }
      std::vector<TaylorApprox> ap(n);
      for (int k = 0; k < n; ++k) {
        const long long row = i * n + k;
        ap[k].node = k;
        ap[k].order = order;
        ap[k].z0.assign(z0 + row * nf, z0 + (row + 1) * nf);
        ap[k].f_bar.assign(fbar + row * nr, fbar + (row + 1) * nr);
        ap[k].jac.assign(jac + row * nr * nf, jac + (row + 1) * nr * nf);
        if (order == 2) ap[k].hess.assign(hess + row * nr * nf * nf, hess + (row + 1) * nr * nf * nf);
      }
      std::vector<Vec> vaux;
      if (variant == 3)
        for (int k = 0; k < n; ++k) vaux.emplace_back(aux + (i * n + k) * 9, aux + (i * n + k + 1) * 9);
      QpData d;
      try {
        d = BuildQp(plant, cfg, vx, vu, vrx, vru, &ap, nullptr, &fc, variant == 3 ? &vaux : nullptr);
      } catch (const ConfigError&) {
        throw;
      } catch (const std::exception& e) {
        throw std::runtime_error(n_inst == 1 ? std::string(e.what())
                                             : "instance " + std::to_string(i) + ": " + e.what());
      }
      for (int k = 0; k < n; ++k) {
        const long long row = i * n + k;
        std::copy(d.a[k].v.begin(), d.a[k].v.end(), a + row * nx * nx);
        std::copy(d.b[k].v.begin(), d.b[k].v.end(), b + row * nx * nu);
        std::copy(d.phi_res[k].begin(), d.phi_res[k].end(), phi + row * nx);
        std::copy(d.r[k].begin(), d.r[k].end(), r + row * nu);
        std::copy(d.hu_diag[k].begin(), d.hu_diag[k].end(), hu + row * nu);
        std::copy(d.du_lb[k].begin(), d.du_lb[k].end(), lb + row * nu);
        std::copy(d.du_ub[k].begin(), d.du_ub[k].end(), ub + row * nu);
      }
      for (int k = 0; k <= n; ++k) {
        std::copy(d.q[k].begin(), d.q[k].end(), q + (i * (n + 1) + k) * nx);
        std::copy(d.hx_diag[k].begin(), d.hx_diag[k].end(), hx + (i * (n + 1) + k) * nx);
      }
    }
    if (fevals != nullptr) {
      fevals[0] = fc.values;
      fevals[1] = fc.jacobians;
    }
    return 0;
  } catch (const oracle::ConfigError& e) {
    g_blocks_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_blocks_err = e.what();
    return 6;
  }
}

// Nominal quadrotor derivative and its Jacobians (dynamics.cpp:64-86,
// integrator.cpp:91-123) — exposed for the FD / structure tests.
int oracle_quad_dynamics(const double* params, const double* x, const double* u, double* dx, double* fx,
                         double* fu) {
  using namespace oracle;
  try {
    const QuadParams qp = ParamsFrom(params);
    const Vec vx(x, x + kQuadNx), vu(u, u + kQuadNu);
    const Vec d = QuadNominalDynamics(vx, vu, qp);
    std::copy(d.begin(), d.end(), dx);
    Mat mx, mu;
    QuadNominalJacobians(vx, vu, qp, mx, mu);
    std::copy(mx.v.begin(), mx.v.end(), fx);
    std::copy(mu.v.begin(), mu.v.end(), fu);
    return 0;
  } catch (const std::exception& e) {
    g_blocks_err = e.what();
    return 2;
  }
}

}  // extern "C"
