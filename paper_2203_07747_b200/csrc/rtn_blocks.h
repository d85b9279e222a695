// rtn_blocks.h — batched continuity-block builder:
// RK4 sensitivities of f_F + embed·Taylor per shooting node, i.e. the body of
// resmpc::BuildQp's node loop (/root/reference/proj/src/sqp_rti.cpp:86-149)
// for the quadrotor plant with the 'full' residual variant
// (proj/src/plant.cpp:34-85, proj/src/dynamics.cpp:125-190).
#pragma once

#include <cuda_runtime.h>

namespace rtn {

constexpr int kQNx = 13, kQNu = 4, kQNf = 17, kQNr = 6;
// Residual variants (proj/include/resmpc/dynamics.hpp:95-131; codes of rtn_ocp_config::variant):
// full z = [x; u] (17 -> 6), a z = v_B (3 -> 3), a_u z = [v_B; u] (7 -> 3),
// ground z = [x; u; z_WB·1 − patch] (26 -> 3, patch = per-node aux).
enum { kVarFull = 0, kVarA = 1, kVarAU = 2, kVarGround = 3 };
__host__ __device__ constexpr int VarNf(int v) { return v == kVarFull ? 17 : v == kVarA ? 3 : v == kVarAU ? 7 : 26; }
__host__ __device__ constexpr int VarNr(int v) { return v == kVarFull ? 6 : 3; }

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
  const double* z0;    // K x n_f TaylorApprox::z0, or null = features(x_k, u_k, aux_k)
  const double* fbar;  // K x n_r
  const double* jac;   // K x n_r x n_f
  const double* hess;  // K x n_r x n_f x n_f (order 2) or null
  const double* aux;   // K x 9 height patches (ground) or null
  // outputs (device; any may be null): QpData rows
  double *a, *b, *phi, *q, *r, *hx, *hu, *lb, *ub;
  unsigned long long* first_bad;  // atomic error word (may be null), or
  unsigned char* status;          // per-node status byte, 0 = ok (may be null; zero-copy latency mode)
  long long n_inst;
  int N, order, variant;
  double dt, mass;
  double inertia[3];
  double inv_mass, inv_inertia[3];  // 1/m, 1/J_i in fp64 (multiplies replace the reference's divisions)
  double mix[6][4];  // MixingMatrix (dynamics.cpp:42-55), built on the host in fp64
  double qd[13], rd[4], qf[13], umin[4], umax[4];
};

// pdl: launch as a programmatic dependent of the preceding kernel on `s` (the
// fused cycle's MLP kernel): the prologue overlaps that kernel's tail.
cudaError_t LaunchQpBlocks(const BlkParams& p, cudaStream_t s, bool pdl = false);
// z_k = features(x_k, u_k, aux_k) (K x n_f) for the non-'full' variants of the fused cycle.
cudaError_t LaunchFeatures(int variant, const double* xs, const double* us, const double* aux, long long n_inst,
                           int N, double* z, cudaStream_t s);
}  // namespace rtn
