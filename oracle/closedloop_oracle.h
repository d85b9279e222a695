// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Closed-loop trajectory check (north star: "the check covers f, A, B, and the
// closed-loop state trajectory over a fixed rollout"). Eigen-free restatement
// of the reference's RTI loop around the approximation path:
//   condensing + box QP       /root/reference/proj/src/qp.cpp:33-208
//   SolveFeedback, RTI cycle  /root/reference/proj/src/sqp_rti.cpp:44-57, 157-280
//   references + simulator    /root/reference/proj/src/simharness.cpp:15-267
// The data-driven preparation (phase 1, PrepareNodes) and optionally phase 2
// (BuildQp's node loop) are pluggable, so the same rollout can run on the
// oracle's fp64 approximations or on the device path's (through its C-ABI),
// and the state trajectories compared. Parity status: the QP solver and the
// simulator follow the reference line by line (Cholesky written out; Eigen's
// LLT is unbuildable here); pinned by the reference's QP / controller tests
// re-expressed in oracle/test_closedloop.cpp.
#pragma once

#include <cstdint>
#include <functional>
#include <random>
#include <vector>

#include "blocks_oracle.h"

namespace oracle {

// ---- qp.hpp / qp.cpp ----------------------------------------------------------
struct CondensedQp {
  Mat hessian;
  Vec gradient, lb, ub;
  std::vector<Mat> recover_m;
  std::vector<Vec> recover_c;
  int nu = 0;
};
CondensedQp Condense(const QpData& qp, const Vec& dx0);  // qp.cpp:33-73

enum class QpStatus { kOptimal, kMaxIter };
struct BoxQpResult {
  Vec x, lam_lb, lam_ub;
  QpStatus status = QpStatus::kOptimal;
  int iterations = 0;
  bool regularized = false;
  std::vector<std::int8_t> active;
};
BoxQpResult SolveBoxQp(const CondensedQp& qp, const std::vector<std::int8_t>* warm_start = nullptr,
                       int max_iterations = 200);  // qp.cpp:104-208

struct FeedbackResult {
  std::vector<Vec> dxs, dus;
  Vec u_command;
  int qp_iterations = 0;
  bool regularized = false;
  QpStatus status = QpStatus::kOptimal;
};
FeedbackResult SolveFeedback(const QpData& qp, const Vec& x_measured, const std::vector<Vec>& xs,
                             const std::vector<Vec>& us, std::vector<std::int8_t>* warm_active);  // sqp_rti.cpp:157-180

// ---- the RTI controller (rtn mode, quadrotor 'full') ------------------------
// Phase 1 provider: fills one TaylorApprox per node from the K x 17 feature rows.
using PrepareFn = std::function<std::vector<TaylorApprox>(const Vec& z_rows, int k, int order)>;
// Optional phase 1+2 provider: returns QpData for (iterate, reference window).
using BuildFn = std::function<QpData(const std::vector<Vec>& xs, const std::vector<Vec>& us,
                                     const std::vector<Vec>& rxs, const std::vector<Vec>& rus)>;

class RtiController {  // sqp_rti.cpp:182-280
 public:
  RtiController(const QuadParams& params, const OcpConfig& cfg, PrepareFn prepare, BuildFn build = nullptr);
  void Initialize(const Vec& x0, const std::vector<Vec>& rxs, const std::vector<Vec>& rus);
  Vec Cycle(const Vec& x_measured, const std::vector<Vec>& rxs, const std::vector<Vec>& rus);
  bool last_ok() const { return ok_; }
  const std::vector<Vec>& xs() const { return xs_; }
  const std::vector<Vec>& us() const { return us_; }

 private:
  QuadParams params_;
  Plant plant_;
  OcpConfig cfg_;
  PrepareFn prepare_;
  BuildFn build_;
  std::vector<Vec> xs_, us_;
  std::vector<std::int8_t> warm_;
  Vec last_command_;
  bool ok_ = true;
};

// ---- simharness -----------------------------------------------------------------
struct TrajectoryCfg {  // simharness.hpp:34-46
  int kind = 0;  // 0 circle, 1 lemniscate
  double scale = 5.0, speed = 2.0, duration = 20.0, z0 = 1.5, ramp_time = 3.0;
};
class ReferenceGenerator {  // simharness.cpp:70-158
 public:
  ReferenceGenerator(const TrajectoryCfg& traj, const QuadParams& params);
  void At(double t, Vec& x, Vec& u) const;
  void Window(double t, int horizon, double dt, std::vector<Vec>& xs, std::vector<Vec>& us) const;

 private:
  void Pos(double theta, double p[3]) const;
  void Eval(double t, Vec& x, Vec& u) const;
  TrajectoryCfg traj_;
  double hover_ = 0.0, omega_rate_ = 0.0, lap_ = 0.0;
};

struct SimConfig {  // simharness.hpp:19-30
  double drag[3] = {0.3, 0.3, 0.15};
  double noise_ft_sigma = 0.005, motor_noise_coeff = 0.02;
  bool per_step_noise = false;
  double sim_dt = 1e-3, control_rate_hz = 100.0;
  std::uint64_t seed = 0;
};
class QuadSim {  // simharness.cpp:163-213
 public:
  QuadSim(const QuadParams& params, const SimConfig& cfg);
  void Reset(std::uint64_t seed);
  Vec Step(const Vec& x, const Vec& u_cmd, double dt_ctrl);
  const SimConfig& config() const { return cfg_; }

 private:
  Vec Derivative(const Vec& x, const Vec& u) const;
  QuadParams params_;
  SimConfig cfg_;
  std::mt19937_64 rng_;
  double accel_noise_[3] = {0, 0, 0}, torque_noise_[3] = {0, 0, 0};
};

struct Rollout {
  std::vector<Vec> states, commands;
  std::vector<int> ok;
  bool failed = false;
};
// simharness.cpp:218-267 (telemetry columns the check does not need are dropped)
Rollout RunClosedLoop(RtiController& ctrl, QuadSim& sim, const ReferenceGenerator& refs, const OcpConfig& cfg,
                      double duration, std::uint64_t seed);

}  // namespace oracle
