// rtn_blocks.h — batched continuity-block builder:
// RK4 sensitivities of f_F + embed·Taylor per shooting node, i.e. the body of
// resmpc::BuildQp's node loop (/root/reference/proj/src/sqp_rti.cpp:86-149)
// for the quadrotor plant with the 'full' residual variant
// (proj/src/plant.cpp:34-85, proj/src/dynamics.cpp:125-190).
#pragma once

#include <cuda_runtime.h>

namespace rtn {

constexpr int kQNx = 13, kQNu = 4, kQNf = 17, kQNr = 6;

// Error word: min over failing nodes of (node << 8 | code); code 10+s = the
// quaternion-domain check of QuadNominalDynamics at RK4 stage s
// (dynamics.cpp:70-73), 20+s = CheckFinite at stage s (integrator.cpp:12-15).
constexpr unsigned long long kNoError = ~0ull;

struct BlkParams {
  // inputs (device): instance-major, node-major rows
  const double* xs;    // n_inst x (N+1) x 13   Iterate::xs
  const double* us;    // n_inst x N x 4        Iterate::us
  const double* rxs;   // n_inst x (N+1) x 13   ReferenceWindow::xs
  const double* rus;   // n_inst x N x 4        ReferenceWindow::us
  const double* z0;    // K x 17 TaylorApprox::z0, or null = [x_k; u_k]
  const double* fbar;  // K x 6
  const double* jac;   // K x 6 x 17
  const double* hess;  // K x 6 x 17 x 17 (order 2) or null
  // outputs (device; any may be null): QpData rows
  double *a, *b, *phi, *q, *r, *hx, *hu, *lb, *ub;
  unsigned long long* first_bad;  // atomic error word (may be null), or
  unsigned char* status;          // per-node status byte, 0 = ok (may be null; zero-copy latency mode)
  long long n_inst;
  int N, order;
  double dt, mass;
  double inertia[3];
  double inv_mass, inv_inertia[3];  // 1/m, 1/J_i in fp64 (multiplies replace the reference's divisions)
  double mix[6][4];  // MixingMatrix (dynamics.cpp:42-55), built on the host in fp64
  double qd[13], rd[4], qf[13], umin[4], umax[4];
};

cudaError_t LaunchQpBlocks(const BlkParams& p, cudaStream_t s);
}  // namespace rtn
