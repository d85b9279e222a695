// rtn_blocks.cu — batched continuity-block builder (fp64, sm_100a).
//
// One warp per shooting node. The RK4 value chain (k1..k4 and the stage
// states) is computed cooperatively, one lane per state row. The sensitivity
// recursion (proj/src/integrator.cpp:41-89)
//     dk_s = J_s · (I + c_s · dk_{s-1})   (x columns)
//     dk_s = J_s · (c_s · dk_{s-1}) + Ju_s (u columns)
// is separable by column, so lane j < 17 carries column j of [A | B] through
// the four stages in registers. The per-stage 13x13 / 13x4 Jacobians
// (nominal + embed·EvalTaylorJacobian, sqp_rti.cpp:100-111) sit in per-warp
// shared memory and are read as broadcasts. Roofline: HBM (≈2.6 KB of fp64 in
// + out per node at order 1); the arithmetic is ~15 kFLOP fp64 per node.
#include <cmath>

#include "rtn_blocks.h"

namespace rtn {
namespace {

constexpr int kWarps = 8;

struct WarpSmem {
  double jx[kQNx * kQNx];   // stage Jacobian wrt x, row-major
  double ju[kQNx * kQNu];   // stage Jacobian wrt u
  double jac[kQNr * kQNf];  // TaylorApprox::jac
  double jn[kQNr * kQNf];   // EvalTaylorJacobian at the stage point
  double g[kQNr * kQNf];    // H_o · dz (order 2)
  double x[kQNx], xs[kQNx], u[kQNu], z0[kQNf], dz[kQNf], fb[kQNr], y[kQNr];
  double k[4][kQNx];
  double phi[kQNx];
};

__device__ __forceinline__ void Report(unsigned long long* w, long long node, int code) {
  atomicMin(w, (static_cast<unsigned long long>(node) << 8) | static_cast<unsigned long long>(code));
}

// Row i of QuadNominalDynamics (dynamics.cpp:64-86) at state X, with the
// body wrench (t_b, tau) already mixed.
__device__ __forceinline__ double NominalRow(int i, const double* X, const double* tb, const double* tau,
                                             const BlkParams& p) {
  const double qw = X[3], qx = X[4], qy = X[5], qz = X[6];
  const double w0 = X[10], w1 = X[11], w2 = X[12];
  if (i < 3) return X[7 + i];
  if (i < 7) {  // 0.5 * QuatMul(q, (0, ω)) (quat.hpp:20-25, 107-109)
    double m;
    if (i == 3) m = qw * 0.0 - qx * w0 - qy * w1 - qz * w2;
    else if (i == 4) m = qw * w0 + qx * 0.0 + qy * w2 - qz * w1;
    else if (i == 5) m = qw * w1 - qx * w2 + qy * 0.0 + qz * w0;
    else m = qw * w2 + qx * w1 - qy * w0 + qz * 0.0;
    return 0.5 * m;
  }
  if (i < 10) {  // R(q)·T_B / m + g_W (quat.hpp:36-49)
    const int r = i - 7;
    double r0, r1, r2;
    if (r == 0) {
      r0 = 1.0 - 2.0 * (qy * qy + qz * qz); r1 = 2.0 * (qx * qy - qw * qz); r2 = 2.0 * (qx * qz + qw * qy);
    } else if (r == 1) {
      r0 = 2.0 * (qx * qy + qw * qz); r1 = 1.0 - 2.0 * (qx * qx + qz * qz); r2 = 2.0 * (qy * qz - qw * qx);
    } else {
      r0 = 2.0 * (qx * qz - qw * qy); r1 = 2.0 * (qy * qz + qw * qx); r2 = 1.0 - 2.0 * (qx * qx + qy * qy);
    }
    const double g = r == 2 ? -9.81 : 0.0;
    return (r0 * tb[0] + r1 * tb[1] + r2 * tb[2]) / p.mass + g;
  }
  // J⁻¹(τ − ω × Jω)
  const int r = i - 10;
  const double jw0 = p.inertia[0] * w0, jw1 = p.inertia[1] * w1, jw2 = p.inertia[2] * w2;
  const double cr = r == 0 ? w1 * jw2 - w2 * jw1 : (r == 1 ? w2 * jw0 - w0 * jw2 : w0 * jw1 - w1 * jw0);
  const double tr = r == 0 ? tau[0] : (r == 1 ? tau[1] : tau[2]);
  const double jr = r == 0 ? p.inertia[0] : (r == 1 ? p.inertia[1] : p.inertia[2]);
  return (tr - cr) / jr;
}

// Row i of QuadNominalJacobians (integrator.cpp:91-123) plus the embedded
// residual Jacobian row (embed·jn·I for the 'full' variant), written to smem.
__device__ __forceinline__ void JacobianRow(int i, const double* X, const double* tb, const BlkParams& p,
                                            WarpSmem& S) {
  double* fx = S.jx + i * kQNx;
  double* fu = S.ju + i * kQNu;
#pragma unroll
  for (int c = 0; c < kQNx; ++c) fx[c] = 0.0;
#pragma unroll
  for (int c = 0; c < kQNu; ++c) fu[c] = 0.0;
  const double qw = X[3], qx = X[4], qy = X[5], qz = X[6];
  const double w0 = X[10], w1 = X[11], w2 = X[12];
  if (i < 3) {
    fx[7 + i] = 1.0;
  } else if (i < 7) {
    // QuatKinematicsJacQ(ω) row r and QuatKinematicsJacOmega(q) row r (quat.hpp:112-130)
    double a0, a1, a2, a3, o0, o1, o2;
    switch (i - 3) {
      case 0: a0 = 0; a1 = -w0; a2 = -w1; a3 = -w2; o0 = -qx; o1 = -qy; o2 = -qz; break;
      case 1: a0 = w0; a1 = 0; a2 = w2; a3 = -w1; o0 = qw; o1 = -qz; o2 = qy; break;
      case 2: a0 = w1; a1 = -w2; a2 = 0; a3 = w0; o0 = qz; o1 = qw; o2 = -qx; break;
      default: a0 = w2; a1 = w1; a2 = -w0; a3 = 0; o0 = -qy; o1 = qx; o2 = qw; break;
    }
    fx[3] = 0.5 * a0;
    fx[4] = 0.5 * a1;
    fx[5] = 0.5 * a2;
    fx[6] = 0.5 * a3;
    fx[10] = 0.5 * o0;
    fx[11] = 0.5 * o1;
    fx[12] = 0.5 * o2;
  } else if (i < 10) {
    const int r = i - 7;
    // dR/dq_c row r (QuatRotDerivatives, quat.hpp:57-74) · t_b / m
    double d[4][3];
    if (r == 0) {
      d[0][0] = 0; d[0][1] = -2 * qz; d[0][2] = 2 * qy;
      d[1][0] = 0; d[1][1] = 2 * qy; d[1][2] = 2 * qz;
      d[2][0] = -4 * qy; d[2][1] = 2 * qx; d[2][2] = 2 * qw;
      d[3][0] = -4 * qz; d[3][1] = -2 * qw; d[3][2] = 2 * qx;
    } else if (r == 1) {
      d[0][0] = 2 * qz; d[0][1] = 0; d[0][2] = -2 * qx;
      d[1][0] = 2 * qy; d[1][1] = -4 * qx; d[1][2] = -2 * qw;
      d[2][0] = 2 * qx; d[2][1] = 0; d[2][2] = 2 * qz;
      d[3][0] = 2 * qw; d[3][1] = -4 * qz; d[3][2] = 2 * qy;
    } else {
      d[0][0] = -2 * qy; d[0][1] = 2 * qx; d[0][2] = 0;
      d[1][0] = 2 * qz; d[1][1] = 2 * qw; d[1][2] = -4 * qx;
      d[2][0] = -2 * qw; d[2][1] = 2 * qz; d[2][2] = -4 * qy;
      d[3][0] = 2 * qx; d[3][1] = 2 * qy; d[3][2] = 0;
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) fx[3 + c] = (d[c][0] * tb[0] + d[c][1] * tb[1] + d[c][2] * tb[2]) / p.mass;
    double r0, r1, r2;
    if (r == 0) {
      r0 = 1.0 - 2.0 * (qy * qy + qz * qz); r1 = 2.0 * (qx * qy - qw * qz); r2 = 2.0 * (qx * qz + qw * qy);
    } else if (r == 1) {
      r0 = 2.0 * (qx * qy + qw * qz); r1 = 1.0 - 2.0 * (qx * qx + qz * qz); r2 = 2.0 * (qy * qz - qw * qx);
    } else {
      r0 = 2.0 * (qx * qz - qw * qy); r1 = 2.0 * (qy * qz + qw * qx); r2 = 1.0 - 2.0 * (qx * qx + qy * qy);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) fu[c] = (r0 * p.mix[0][c] + r1 * p.mix[1][c] + r2 * p.mix[2][c]) / p.mass;
  } else {
    const int r = i - 10;
    // J⁻¹ (−(S(ω)·diag(J) − S(Jω))) row r; S(v) rows (quat.hpp:27-31)
    const double j0 = p.inertia[0], j1 = p.inertia[1], j2 = p.inertia[2];
    const double jw0 = j0 * w0, jw1 = j1 * w1, jw2 = j2 * w2;
    double s0, s1, s2, t0, t1, t2, jr;
    switch (r) {
      case 0: s0 = 0.0; s1 = -w2; s2 = w1; t0 = 0.0; t1 = -jw2; t2 = jw1; jr = j0; break;
      case 1: s0 = w2; s1 = 0.0; s2 = -w0; t0 = jw2; t1 = 0.0; t2 = -jw0; jr = j1; break;
      default: s0 = -w1; s1 = w0; s2 = 0.0; t0 = -jw1; t1 = jw0; t2 = 0.0; jr = j2; break;
    }
    const double inv = 1.0 / jr;
    fx[10] = inv * (-(s0 * j0 - t0));
    fx[11] = inv * (-(s1 * j1 - t1));
    fx[12] = inv * (-(s2 * j2 - t2));
#pragma unroll
    for (int c = 0; c < 4; ++c) fu[c] = inv * (r == 0 ? p.mix[3][c] : (r == 1 ? p.mix[4][c] : p.mix[5][c]));
  }
  if (i >= 7) {  // fx += embed·jn·jz (jz = I for 'full'): rows 7..12 take jn rows 0..5
    const double* jn = S.jn + (i - 7) * kQNf;
#pragma unroll
    for (int c = 0; c < kQNx; ++c) fx[c] += jn[c];
#pragma unroll
    for (int c = 0; c < kQNu; ++c) fu[c] += jn[kQNx + c];
  }
}

__global__ void __launch_bounds__(kWarps * 32) QpBlocksKernel(const BlkParams p) {
  __shared__ WarpSmem smem[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long node = static_cast<long long>(blockIdx.x) * kWarps + warp;
  if (node >= p.n_inst * p.N) return;  // whole warps only: no CTA-wide barriers below
  WarpSmem& S = smem[warp];
  const long long inst = node / p.N;
  const int n = static_cast<int>(node - inst * p.N);
  const long long xrow = inst * (p.N + 1) + n;
  const double dt = p.dt;

  if (lane < kQNx) S.x[lane] = p.xs[xrow * kQNx + lane];
  if (lane < kQNu) S.u[lane] = p.us[node * kQNu + lane];
  if (lane < kQNr) S.fb[lane] = p.fbar[node * kQNr + lane];
  for (int e = lane; e < kQNr * kQNf; e += 32) {
    const double v = p.jac[node * (kQNr * kQNf) + e];
    S.jac[e] = v;
    S.jn[e] = v;  // order 1: EvalTaylorJacobian == jac at every stage (taylor.cpp:67)
  }
  __syncwarp();
  if (lane < kQNf) S.z0[lane] = p.z0 ? p.z0[node * kQNf + lane] : (lane < kQNx ? S.x[lane] : S.u[lane - kQNx]);
  // body wrench = mix · u (MixThrustTorque, dynamics.cpp:57-62)
  double tb[3], tau[3];
#pragma unroll
  for (int r = 0; r < 6; ++r) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) s += p.mix[r][c] * S.u[c];
    if (r < 3) tb[r] = s; else tau[r - 3] = s;
  }

  double dk[kQNx], acc[kQNx];
  const int j = lane;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const double cs = s == 0 ? 0.0 : (s == 3 ? dt : 0.5 * dt);
    // stage state x_s = x + c_s·k_{s-1} (integrator.cpp:57, 65, 73)
    if (lane < kQNx) S.xs[lane] = s == 0 ? S.x[lane] : S.x[lane] + cs * S.k[s - 1][lane];
    __syncwarp();
    if (lane < kQNf) S.dz[lane] = (lane < kQNx ? S.xs[lane] : S.u[lane - kQNx]) - S.z0[lane];
    __syncwarp();
    if (p.order == 2) {  // jn = jac + H·dz, g = H·dz (taylor.cpp:57-74)
      if (lane < kQNf) {
        for (int o = 0; o < kQNr; ++o) {
          const double* h = p.hess + ((node * kQNr + o) * kQNf + lane) * kQNf;
          double g = 0.0;
#pragma unroll
          for (int b = 0; b < kQNf; ++b) g += h[b] * S.dz[b];
          S.g[o * kQNf + lane] = g;
          S.jn[o * kQNf + lane] = S.jac[o * kQNf + lane] + g;
        }
      }
      __syncwarp();
    }
    if (lane < kQNr) {  // EvalTaylor: f_bar + jac·dz (+ ½ dzᵀ H dz)
      double a1 = 0.0;
#pragma unroll
      for (int c = 0; c < kQNf; ++c) a1 += S.jac[lane * kQNf + c] * S.dz[c];
      double y = S.fb[lane] + a1;
      if (p.order == 2) {
        double qv = 0.0;
#pragma unroll
        for (int c = 0; c < kQNf; ++c) qv += S.dz[c] * S.g[lane * kQNf + c];
        y += 0.5 * qv;
      }
      S.y[lane] = y;
    }
    __syncwarp();
    const double* X = S.xs;
    const double qn = sqrt(X[3] * X[3] + X[4] * X[4] + X[5] * X[5] + X[6] * X[6]);
    if (fabs(qn - 1.0) > 0.25) {  // InputDomainError inside f (dynamics.cpp:70-73)
      if (lane == 0) Report(p.first_bad, node, 10 + s + 1);
      return;
    }
    if (lane < kQNx) S.k[s][lane] = NominalRow(lane, X, tb, tau, p) + (lane >= 7 ? S.y[lane - 7] : 0.0);
    __syncwarp();
    const bool bad = lane < kQNx && !isfinite(S.k[s][lane]);
    if (__any_sync(0xffffffffu, bad)) {  // CheckFinite (integrator.cpp:12-15)
      if (lane == 0) Report(p.first_bad, node, 20 + s + 1);
      return;
    }
    if (lane < kQNx) JacobianRow(lane, X, tb, p, S);
    __syncwarp();
    if (j < kQNf) {
      double nd[kQNx];
      if (s == 0) {
#pragma unroll
        for (int i = 0; i < kQNx; ++i) nd[i] = j < kQNx ? S.jx[i * kQNx + j] : S.ju[i * kQNu + (j - kQNx)];
      } else {
        double w[kQNx];
#pragma unroll
        for (int m = 0; m < kQNx; ++m) w[m] = (j == m ? 1.0 : 0.0) + cs * dk[m];
        if (j >= kQNx) {
#pragma unroll
          for (int m = 0; m < kQNx; ++m) w[m] = cs * dk[m];
        }
#pragma unroll
        for (int i = 0; i < kQNx; ++i) {
          double t = 0.0;
#pragma unroll
          for (int m = 0; m < kQNx; ++m) t += S.jx[i * kQNx + m] * w[m];
          nd[i] = j < kQNx ? t : t + S.ju[i * kQNu + (j - kQNx)];
        }
      }
      // dk1 + 2·dk2 + 2·dk3 + dk4, left to right (integrator.cpp:84-88)
#pragma unroll
      for (int i = 0; i < kQNx; ++i) {
        acc[i] = s == 0 ? nd[i] : acc[i] + (s == 3 ? nd[i] : 2.0 * nd[i]);
        dk[i] = nd[i];
      }
    }
    __syncwarp();  // the next stage rewrites S.jx / S.ju
  }

  const double h6 = dt / 6.0;
  if (j < kQNx && p.a) {
#pragma unroll
    for (int i = 0; i < kQNx; ++i) p.a[node * (kQNx * kQNx) + i * kQNx + j] = (i == j ? 1.0 : 0.0) + h6 * acc[i];
  } else if (j >= kQNx && j < kQNf && p.b) {
#pragma unroll
    for (int i = 0; i < kQNx; ++i) p.b[node * (kQNx * kQNu) + i * kQNu + (j - kQNx)] = h6 * acc[i];
  }
  // φ̄ = x + dt/6 (k1 + 2k2 + 2k3 + k4), quaternion renormalised (integrator.cpp:84-86)
  if (lane < kQNx)
    S.phi[lane] = S.x[lane] + h6 * (S.k[0][lane] + 2.0 * S.k[1][lane] + 2.0 * S.k[2][lane] + S.k[3][lane]);
  __syncwarp();
  if (lane < kQNx) {
    double v = S.phi[lane];
    if (lane >= 3 && lane < 7)
      v /= sqrt(S.phi[3] * S.phi[3] + S.phi[4] * S.phi[4] + S.phi[5] * S.phi[5] + S.phi[6] * S.phi[6]);
    const double xn = p.xs[(xrow + 1) * kQNx + lane];
    if (p.phi) p.phi[node * kQNx + lane] = v - xn;  // phi_res = φ̄ − x_{k+1} (sqp_rti.cpp:141)
    // cost terms (sqp_rti.cpp:143-148) and the terminal ones (:150-153)
    if (p.q) p.q[xrow * kQNx + lane] = 2.0 * (p.qd[lane] * (S.x[lane] - p.rxs[xrow * kQNx + lane]));
    if (p.hx) p.hx[xrow * kQNx + lane] = 2.0 * p.qd[lane];
    if (n == p.N - 1) {
      if (p.q) p.q[(xrow + 1) * kQNx + lane] = 2.0 * (p.qf[lane] * (xn - p.rxs[(xrow + 1) * kQNx + lane]));
      if (p.hx) p.hx[(xrow + 1) * kQNx + lane] = 2.0 * p.qf[lane];
    }
  }
  if (lane < kQNu) {
    const double u = S.u[lane];
    if (p.r) p.r[node * kQNu + lane] = 2.0 * (p.rd[lane] * (u - p.rus[node * kQNu + lane]));
    if (p.hu) p.hu[node * kQNu + lane] = 2.0 * p.rd[lane];
    if (p.lb) p.lb[node * kQNu + lane] = p.umin[lane] - u;
    if (p.ub) p.ub[node * kQNu + lane] = p.umax[lane] - u;
  }
}

__global__ void FeaturesFullKernel(const double* __restrict__ xs, const double* __restrict__ us, long long n_inst,
                                   int N, double* __restrict__ z) {
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long K = n_inst * N;
  if (e >= K * kQNf) return;
  const long long node = e / kQNf;
  const int c = static_cast<int>(e - node * kQNf);
  const long long inst = node / N;
  const long long xrow = inst * (N + 1) + (node - inst * N);
  z[e] = c < kQNx ? xs[xrow * kQNx + c] : us[node * kQNu + (c - kQNx)];
}

}  // namespace

cudaError_t LaunchQpBlocks(const BlkParams& p, cudaStream_t s) {
  const long long K = p.n_inst * p.N;
  if (K <= 0) return cudaSuccess;
  const long long grid = (K + kWarps - 1) / kWarps;
  QpBlocksKernel<<<static_cast<unsigned>(grid), kWarps * 32, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t LaunchFeaturesFull(const double* xs, const double* us, long long n_inst, int N, double* z,
                               cudaStream_t s) {
  const long long total = n_inst * N * kQNf;
  if (total <= 0) return cudaSuccess;
  FeaturesFullKernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(xs, us, n_inst, N, z);
  return cudaGetLastError();
}

}  // namespace rtn
