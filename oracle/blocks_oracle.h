// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free fp64 CPU restatement of the step AFTER the approximation path
// (SURVEY.md §8f rank 1): the RK4 continuity-block builder that consumes the
// per-node (f, A, B[, H]) approximations. It follows:
//   quaternion helpers       /root/reference/proj/include/resmpc/quat.hpp:13-133
//   quadrotor dynamics       /root/reference/proj/src/dynamics.cpp:10-92, 125-211
//   RK4 + sensitivities      /root/reference/proj/src/integrator.cpp:10-123
//   plants                   /root/reference/proj/src/plant.cpp:7-87
//   QP block assembly        /root/reference/proj/src/sqp_rti.cpp:27-150
// Only tests/, bench.py's cpu_baseline leg and __graft_entry__.smoke() may load
// it, and only as the checker — the product path is csrc/rtn_blocks.cu.
//
// Parity status: pinned by tolerance against the reference's own known-answer
// and finite-difference tests (re-expressed in oracle/test_blocks.cpp:
// test_integrator.cpp, test_dynamics.cpp:19-134, test_sqp_rti.cpp:77-150).
// The reference builds every product through Eigen (unbuildable here, no
// Eigen3), so no bitwise pin to reference outputs exists.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "resmpc_oracle.h"

namespace oracle {

using Vec = std::vector<double>;

// ---- quat.hpp ---------------------------------------------------------------
void QuatToRot(const double q[4], double r[9]);                 // quat.hpp:36-44
void QuatRotDerivatives(const double q[4], double out[4][9]);   // quat.hpp:57-74
void QuatRotate(const double q[4], const double v[3], double out[3]);
void QuatRotateInv(const double q[4], const double v[3], double out[3]);
void QuatKinematics(const double q[4], const double w[3], double out[4]);  // quat.hpp:107-109

// ---- dynamics.hpp / dynamics.cpp -------------------------------------------
constexpr int kQuadNx = 13, kQuadNu = 4, kQuatRow = 3, kVelRow = 7, kOmegaRow = 10;
constexpr double kGravity = 9.81;

struct QuadParams {  // dynamics.hpp:50-62
  double mass = 0.75;
  double inertia[3] = {2.5e-3, 2.5e-3, 4.3e-3};
  double arm_length = 0.14;
  double torque_coeff = 0.016;
  double thrust_max = 6.0;
  double rotor_sign[4] = {1.0, 1.0, -1.0, -1.0};
  void Validate() const;  // dynamics.cpp:29-40
  double HoverThrustPerRotor() const { return mass * kGravity / 4.0; }
};

void MixingMatrix(const QuadParams& p, double m[6][4]);  // dynamics.cpp:42-55
Vec QuadNominalDynamics(const Vec& x, const Vec& u, const QuadParams& p);  // dynamics.cpp:64-86
void QuadNominalJacobians(const Vec& x, const Vec& u, const QuadParams& p, Mat& fx,
                          Mat& fu);  // integrator.cpp:91-123

// ---- integrator -------------------------------------------------------------
using DynFn = std::function<Vec(const Vec&, const Vec&)>;
using DynJacFn = std::function<void(const Vec&, const Vec&, Mat&, Mat&)>;
struct FevalCounter {
  std::uint64_t values = 0, jacobians = 0;
};
Vec Rk4Step(const DynFn& f, const Vec& x, const Vec& u, double dt, int quat_row = -1,
            FevalCounter* counter = nullptr);  // integrator.cpp:24-39
struct SensitivityResult {
  Vec phi_bar;
  Mat a, b;
};
SensitivityResult Rk4Sensitivities(const DynFn& f, const DynJacFn& df, const Vec& x, const Vec& u,
                                   double dt, int quat_row = -1,
                                   FevalCounter* counter = nullptr);  // integrator.cpp:41-89

// ---- plant ------------------------------------------------------------------
struct Plant {  // plant.hpp:19-39 (the ground variant's height-map patch arrives as per-node aux)
  std::string name;
  int nx = 0, nu = 0;
  DynFn f;
  DynJacFn df;
  int quat_row = -1;
  std::string variant_tag = "full";
  int feature_dim = 0, residual_dim = 0;
  std::function<Vec(const Vec&, const Vec&, const Vec&)> features;  // (x, u, aux) -> z (plant.hpp:33-36)
  std::function<Mat(const Vec&, const Vec&)> features_jac;  // feature_dim x (nx+nu)
  Mat embed;                                                // nx x residual_dim
};
Plant MakeDoubleIntegratorPlant();                                            // plant.cpp:7-32
// variants a, a_u, full, ground (ground: aux = the node's 3x3 height patch, row-major)
Plant MakeQuadrotorPlant(const QuadParams& p, const std::string& variant);    // plant.cpp:34-85

// ---- sqp_rti ----------------------------------------------------------------
struct OcpConfig {  // sqp_rti.hpp:22-34
  int horizon = 10;
  double dt = 0.1;
  Vec q_diag, r_diag, q_terminal, u_min, u_max;
  int taylor_order = 1;
  void Validate(int nx, int nu) const;  // sqp_rti.cpp:27-42
  const Vec& TerminalWeight() const { return q_terminal.empty() ? q_diag : q_terminal; }
};
struct QpData {  // qp.hpp:13-28
  int nx = 0, nu = 0, horizon = 0;
  std::vector<Mat> a, b;
  std::vector<Vec> phi_res, q, r, hx_diag, hu_diag, du_lb, du_ub;
};
// naive mode: the network is evaluated exactly inside every RK4 stage.
struct NaiveNet {
  std::function<Vec(const Vec&)> value;
  std::function<Vec(const Vec&)> jacobian;  // out x in, row-major
};
// sqp_rti.cpp:59-150. approxes: one TaylorApprox per node (rtn mode), or
// naive != nullptr, or neither (nominal model only). node_aux: per-node
// residual aux (Plant::NodeAux, frozen at the expansion point; ground patch).
QpData BuildQp(const Plant& plant, const OcpConfig& cfg, const std::vector<Vec>& xs,
               const std::vector<Vec>& us, const std::vector<Vec>& ref_xs,
               const std::vector<Vec>& ref_us, const std::vector<TaylorApprox>* approxes,
               const NaiveNet* naive, FevalCounter* f_counters = nullptr,
               const std::vector<Vec>* node_aux = nullptr);

}  // namespace oracle
