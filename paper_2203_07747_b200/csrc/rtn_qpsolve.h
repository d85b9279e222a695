// rtn_qpsolve.h — batched feedback solve: condensing +
// primal active-set box QP + state recovery per MPC instance, i.e.
// resmpc::SolveFeedback (/root/reference/proj/src/sqp_rti.cpp:157-180,
// proj/src/qp.cpp:33-208) for the quadrotor (nx = 13, nu = 4).
#pragma once

#include <cuda_runtime.h>

namespace rtn {

// Per-instance status: 0 optimal, 1 iteration cap (QpStatus::kMaxIter),
// 2 SolveFeedback threw (non-finite state or solution, crossed bounds),
// 3 Hessian not positive definite even after regularisation (qp.cpp:99-100).
struct FbParams {
  // QpData rows (device), instance-major (rtn_qp_blocks layout)
  const double *a, *b, *phi, *q, *r, *hx, *hu, *lb, *ub;
  const double* x_meas;  // n_inst x 13
  const double* xs;      // n_inst x (N+1) x 13 (the iterate: dx0 = x_meas − xs[0])
  const double* us;      // n_inst x N x 4
  signed char* active;   // n_inst x N·4 working-set hint in / final set out (may be null)
  double *dxs, *dus, *u_cmd;
  int *status, *iterations;
  double* work;          // gridDim.x x FeedbackWorkPerCta(N)
  long long n_inst;
  int N;
};

// Workspace doubles per CTA: condensed Hessian + Cholesky factor (nv x nv each)
// + 7 vectors of nv (nv = 4·N).
__host__ __device__ inline long long FeedbackWorkPerCta(int N) {
  const long long nv = static_cast<long long>(N) * 4;
  return 2 * nv * nv + 7 * nv;
}
size_t FeedbackSmemBytes(int N);
cudaError_t LaunchFeedback(const FbParams& p, int grid, cudaStream_t s);

}  // namespace rtn
