// rtn_blocks.cu — batched continuity-block builder (fp64, sm_100a).
//
// Two shooting nodes per warp, one per half-warp; lane r < 13 of a half owns
// state row r. Per RK4 stage s (proj/src/integrator.cpp:41-89) lane r
//   - forms row r of the stage derivative k_s (nominal quadrotor row +
//     embedded Taylor value, lanes 7..12 evaluate their residual row),
//   - builds row r of the stage Jacobian [J_x | J_u] in registers (nominal
//     row of QuadNominalJacobians + embed·EvalTaylorJacobian row),
//   - computes row r of the sensitivity update
//         dk_s = J_x · (I + c_s·dk_{s-1})  (x columns),  J_x · (c_s·dk_{s-1}) + J_u  (u columns)
//     reading dk_{s-1} from double-buffered shared memory as 16-byte
//     broadcasts (every lane of the half reads the same address),
//   - accumulates dk1 + 2dk2 + 2dk3 + dk4 for its row of [A | B].
// The final A and B blocks are staged in shared memory and written with
// coalesced stores. Roofline: HBM — ≈3.5 KB of fp64 in + out per node at
// order 1; the fp64 arithmetic is ~8 kFLOP per node.
#include <cmath>
#include <cstdlib>

#include "rtn_blocks.h"
#include "rtn_launch.h"

namespace rtn {
namespace {

constexpr int kWarps = 4;          // 8 nodes per CTA
constexpr int kDkStride = 18;      // dk row stride (doubles): 16-byte aligned pairs
constexpr int kDk = kQNx * kDkStride;

constexpr int kMaxNf = 26;
constexpr long long kLatencyMaxNodes = 4096;  // batches up to this size take the HS variant

// Per-node scratch, ≡ 64 (mod 128) bytes: the two nodes of a warp sit in
// disjoint banks, so their broadcast loads do not conflict.
struct NodeSmem {
  double dk[2][kDk];  // dk_{s-1} / dk_s rows, then the A|B staging area
  double x[kQNx], xs[kQNx], u[kQNu], z0[kMaxNf], dz[kMaxNf], k[4][kQNx], phi[kQNx], aux[9];
  double g[kQNr * kQNf];  // H_o·dz at the stage point (order 2); n_r·n_f <= 102 for every variant
  double pad[2];
};
static_assert(sizeof(NodeSmem) % 128 == 64, "node stride must split the banks");

__device__ __forceinline__ void Report(unsigned long long* w, long long node, int code) {
  atomicMin(w, (static_cast<unsigned long long>(node) << 8) | static_cast<unsigned long long>(code));
}

// Column c of R(q) (QuatToRot, quat.hpp:36-44).
__device__ __forceinline__ void RotCol(int c, double qw, double qx, double qy, double qz, double& r0, double& r1,
                                       double& r2) {
  if (c == 0) {
    r0 = 1.0 - 2.0 * (qy * qy + qz * qz); r1 = 2.0 * (qx * qy + qw * qz); r2 = 2.0 * (qx * qz - qw * qy);
  } else if (c == 1) {
    r0 = 2.0 * (qx * qy - qw * qz); r1 = 1.0 - 2.0 * (qx * qx + qz * qz); r2 = 2.0 * (qy * qz + qw * qx);
  } else {
    r0 = 2.0 * (qx * qz + qw * qy); r1 = 2.0 * (qy * qz - qw * qx); r2 = 1.0 - 2.0 * (qx * qx + qy * qy);
  }
}

// Feature c of the residual input at (x, u, aux): ResidualInput (dynamics.cpp:125-152)
// and the ground layout of plant.cpp:60-73.
template <int VAR>
__device__ __forceinline__ double Feature(int c, const double* X, const double* U, const double* aux) {
  if (VAR == kVarFull) return c < kQNx ? X[c] : U[c - kQNx];
  if (VAR == kVarGround) return c < kQNx ? X[c] : (c < kQNf ? U[c - kQNx] : X[2] - aux[c - kQNf]);
  if (c >= 3) return U[c - 3];  // a_u: [v_B; u]
  double r0, r1, r2;            // v_B = R(q)ᵀ v_W (QuatRotateInv)
  RotCol(c, X[3], X[4], X[5], X[6], r0, r1, r2);
  return r0 * X[7] + r1 * X[8] + r2 * X[9];
}

// Row o of embed·jn·jz (sqp_rti.cpp:104-111) with jz = ResidualInputJacobian at the
// stage state (dynamics.cpp:154-180): the residual row's derivative wrt (x, u).
template <int VAR>
__device__ __forceinline__ void ChainRow(const double (&jn)[VarNf(VAR)], const double* X, double (&jc)[kQNf]) {
  if (VAR == kVarFull) {
#pragma unroll
    for (int c = 0; c < kQNf; ++c) jc[c] = jn[c];
  } else if (VAR == kVarGround) {
#pragma unroll
    for (int c = 0; c < kQNf; ++c) jc[c] = jn[c];
    double s = 0.0;  // ∂(z_WB·1 − patch)/∂p_z = 1
#pragma unroll
    for (int m = kQNf; m < 26; ++m) s += jn[m];
    jc[2] += s;
  } else {
#pragma unroll
    for (int c = 0; c < kQNf; ++c) jc[c] = 0.0;
    const double qw = X[3], qx = X[4], qy = X[5], qz = X[6], v0 = X[7], v1 = X[8], v2 = X[9];
    // ∂v_B/∂q_c = dR_cᵀ v (QuatRotateInvJacQ, quat.hpp:88-96; dR_c rows from quat.hpp:57-74)
    const double d[4][3][3] = {{{0, -2 * qz, 2 * qy}, {2 * qz, 0, -2 * qx}, {-2 * qy, 2 * qx, 0}},
                               {{0, 2 * qy, 2 * qz}, {2 * qy, -4 * qx, -2 * qw}, {2 * qz, 2 * qw, -4 * qx}},
                               {{-4 * qy, 2 * qx, 2 * qw}, {2 * qx, 0, 2 * qz}, {-2 * qw, 2 * qz, -4 * qy}},
                               {{-4 * qz, -2 * qw, 2 * qx}, {2 * qw, -4 * qz, 2 * qy}, {2 * qx, 2 * qy, 0}}};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) s += jn[m] * (d[c][0][m] * v0 + d[c][1][m] * v1 + d[c][2][m] * v2);
      jc[3 + c] = s;
    }
    double rc[3][3];  // rc[i][j] = R(i, j)
    RotCol(0, qw, qx, qy, qz, rc[0][0], rc[1][0], rc[2][0]);
    RotCol(1, qw, qx, qy, qz, rc[0][1], rc[1][1], rc[2][1]);
    RotCol(2, qw, qx, qy, qz, rc[0][2], rc[1][2], rc[2][2]);
#pragma unroll
    for (int c = 0; c < 3; ++c)  // ∂v_B/∂v_W = Rᵀ: entry (m, c) = R(c, m)
      jc[7 + c] = jn[0] * rc[c][0] + jn[1] * rc[c][1] + jn[2] * rc[c][2];
    if (VAR == kVarAU) {
#pragma unroll
      for (int i = 0; i < kQNu; ++i) jc[kQNx + i] = jn[3 + i];
    }
  }
}

// Row i of QuadNominalDynamics (dynamics.cpp:64-86) AND of QuadNominalJacobians
// (integrator.cpp:91-123) in one branch per row group (one divergent region
// per stage), plus the embedded residual Jacobian row jn (rows 7..12:
// fx += embed·jn·I for the 'full' variant). Returns the nominal derivative.
__device__ __forceinline__ double NominalRowAndJacobian(int i, const double* X, const double* tb,
                                                       const double* tau, const BlkParams& p,
                                                       const double (&jn)[kQNf], double (&fx)[kQNx],
                                                       double (&fu)[kQNu]) {
  const double qw = X[3], qx = X[4], qy = X[5], qz = X[6];
  const double w0 = X[10], w1 = X[11], w2 = X[12];
#pragma unroll
  for (int c = 0; c < kQNx; ++c) fx[c] = 0.0;
#pragma unroll
  for (int c = 0; c < kQNu; ++c) fu[c] = 0.0;
  double f;
  if (i < 3) {  // ṗ = v
    f = i == 0 ? X[7] : (i == 1 ? X[8] : X[9]);
#pragma unroll
    for (int c = 0; c < 3; ++c) fx[7 + c] = c == i ? 1.0 : 0.0;
  } else if (i < 7) {
    // q̇ = ½ q ⊗ (0, ω) (quat.hpp:20-25, 107-109); QuatKinematicsJacQ / JacOmega rows (quat.hpp:112-130)
    double m, a0, a1, a2, a3, o0, o1, o2;
    switch (i - 3) {
      case 0:
        m = qw * 0.0 - qx * w0 - qy * w1 - qz * w2;
        a0 = 0; a1 = -w0; a2 = -w1; a3 = -w2; o0 = -qx; o1 = -qy; o2 = -qz;
        break;
      case 1:
        m = qw * w0 + qx * 0.0 + qy * w2 - qz * w1;
        a0 = w0; a1 = 0; a2 = w2; a3 = -w1; o0 = qw; o1 = -qz; o2 = qy;
        break;
      case 2:
        m = qw * w1 - qx * w2 + qy * 0.0 + qz * w0;
        a0 = w1; a1 = -w2; a2 = 0; a3 = w0; o0 = qz; o1 = qw; o2 = -qx;
        break;
      default:
        m = qw * w2 + qx * w1 - qy * w0 + qz * 0.0;
        a0 = w2; a1 = w1; a2 = -w0; a3 = 0; o0 = -qy; o1 = qx; o2 = qw;
        break;
    }
    f = 0.5 * m;
    fx[3] = 0.5 * a0;
    fx[4] = 0.5 * a1;
    fx[5] = 0.5 * a2;
    fx[6] = 0.5 * a3;
    fx[10] = 0.5 * o0;
    fx[11] = 0.5 * o1;
    fx[12] = 0.5 * o2;
  } else if (i < 10) {
    // v̇ = R(q)·T_B/m + g (quat.hpp:36-49); dR/dq_c row (QuatRotDerivatives, quat.hpp:57-74)
    const int r = i - 7;
    double d0[3], d1[3], d2[3], d3[3], r0, r1, r2;
    if (r == 0) {
      d0[0] = 0; d0[1] = -2 * qz; d0[2] = 2 * qy;
      d1[0] = 0; d1[1] = 2 * qy; d1[2] = 2 * qz;
      d2[0] = -4 * qy; d2[1] = 2 * qx; d2[2] = 2 * qw;
      d3[0] = -4 * qz; d3[1] = -2 * qw; d3[2] = 2 * qx;
      r0 = 1.0 - 2.0 * (qy * qy + qz * qz); r1 = 2.0 * (qx * qy - qw * qz); r2 = 2.0 * (qx * qz + qw * qy);
    } else if (r == 1) {
      d0[0] = 2 * qz; d0[1] = 0; d0[2] = -2 * qx;
      d1[0] = 2 * qy; d1[1] = -4 * qx; d1[2] = -2 * qw;
      d2[0] = 2 * qx; d2[1] = 0; d2[2] = 2 * qz;
      d3[0] = 2 * qw; d3[1] = -4 * qz; d3[2] = 2 * qy;
      r0 = 2.0 * (qx * qy + qw * qz); r1 = 1.0 - 2.0 * (qx * qx + qz * qz); r2 = 2.0 * (qy * qz - qw * qx);
    } else {
      d0[0] = -2 * qy; d0[1] = 2 * qx; d0[2] = 0;
      d1[0] = 2 * qz; d1[1] = 2 * qw; d1[2] = -4 * qx;
      d2[0] = -2 * qw; d2[1] = 2 * qz; d2[2] = -4 * qy;
      d3[0] = 2 * qx; d3[1] = 2 * qy; d3[2] = 0;
      r0 = 2.0 * (qx * qz - qw * qy); r1 = 2.0 * (qy * qz + qw * qx); r2 = 1.0 - 2.0 * (qx * qx + qy * qy);
    }
    f = (r0 * tb[0] + r1 * tb[1] + r2 * tb[2]) * p.inv_mass + (r == 2 ? -9.81 : 0.0);
    fx[3] = (d0[0] * tb[0] + d0[1] * tb[1] + d0[2] * tb[2]) * p.inv_mass;
    fx[4] = (d1[0] * tb[0] + d1[1] * tb[1] + d1[2] * tb[2]) * p.inv_mass;
    fx[5] = (d2[0] * tb[0] + d2[1] * tb[1] + d2[2] * tb[2]) * p.inv_mass;
    fx[6] = (d3[0] * tb[0] + d3[1] * tb[1] + d3[2] * tb[2]) * p.inv_mass;
#pragma unroll
    for (int c = 0; c < 4; ++c) fu[c] = (r0 * p.mix[0][c] + r1 * p.mix[1][c] + r2 * p.mix[2][c]) * p.inv_mass;
  } else {
    // ω̇ = J⁻¹(τ − ω × Jω); row of J⁻¹(−(S(ω)·diag(J) − S(Jω))) (quat.hpp:27-31)
    const int r = i - 10;
    const double j0 = p.inertia[0], j1 = p.inertia[1], j2 = p.inertia[2];
    const double jw0 = j0 * w0, jw1 = j1 * w1, jw2 = j2 * w2;
    double s0, s1, s2, t0, t1, t2, inv, cr, tr;
    switch (r) {
      case 0:
        s0 = 0.0; s1 = -w2; s2 = w1; t0 = 0.0; t1 = -jw2; t2 = jw1; inv = p.inv_inertia[0];
        cr = w1 * jw2 - w2 * jw1; tr = tau[0];
        break;
      case 1:
        s0 = w2; s1 = 0.0; s2 = -w0; t0 = jw2; t1 = 0.0; t2 = -jw0; inv = p.inv_inertia[1];
        cr = w2 * jw0 - w0 * jw2; tr = tau[1];
        break;
      default:
        s0 = -w1; s1 = w0; s2 = 0.0; t0 = -jw1; t1 = jw0; t2 = 0.0; inv = p.inv_inertia[2];
        cr = w0 * jw1 - w1 * jw0; tr = tau[2];
        break;
    }
    f = (tr - cr) * inv;
    fx[10] = inv * (-(s0 * j0 - t0));
    fx[11] = inv * (-(s1 * j1 - t1));
    fx[12] = inv * (-(s2 * j2 - t2));
#pragma unroll
    for (int c = 0; c < 4; ++c) fu[c] = inv * (r == 0 ? p.mix[3][c] : (r == 1 ? p.mix[4][c] : p.mix[5][c]));
  }
  if (i >= 7) {
#pragma unroll
    for (int c = 0; c < kQNx; ++c) fx[c] += jn[c];
#pragma unroll
    for (int c = 0; c < kQNu; ++c) fu[c] += jn[kQNx + c];
  }
  return f;
}

// HS (latency-sized batches): the kernel is a chain of dependent fp64 steps
// (~6,000 warp-instructions per node at order 2, ~9 cycles each), so a node
// gets a whole warp: both halves run the same rows, half h computes the
// sensitivity columns [8h, 8h + 10) (selects, no divergence), and the order-2
// H·dz rows and the feature/Hessian loads spread over 32 lanes. One CTA per SM
// (no register cap; the 4-CTA variant spills 56-184 bytes per thread at 128
// registers), and at order 2 the node's Hessian rows are copied into shared
// memory once (cp.async, all issued up front) instead of being re-read from L2
// at every RK4 stage. Large batches keep the half-warp L2 variant, 4 CTAs per SM.
template <int ORDER, int VAR, bool HS>
__global__ void __launch_bounds__(kWarps * 32, HS ? 1 : 4) QpBlocksKernel(const BlkParams p) {
  constexpr int NF = VarNf(VAR), NR = VarNr(VAR), NH = NR * NF * NF;
  __shared__ __align__(128) NodeSmem smem[kWarps * 2];
  extern __shared__ __align__(16) double hsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = lane >> 4, r = lane & 15;
  const unsigned half_mask = half ? 0xffff0000u : 0x0000ffffu;
  const long long K = p.n_inst * p.N;
  constexpr int kStep = HS ? 32 : 16;  // lanes per node
  const int nl = HS ? lane : r;         // lane index inside the node's lanes
  const int slot = HS ? warp : warp * 2 + half;
  const long long raw = HS ? static_cast<long long>(blockIdx.x) * kWarps + warp
                           : (static_cast<long long>(blockIdx.x) * kWarps + warp) * 2 + half;
  if ((HS ? raw : (raw & ~1ll)) >= K) return;  // the whole warp is past the end
  const bool valid = raw < K;                  // a past-the-end half shadows its partner's node
  const long long node = valid ? raw : raw - 1;
  const bool writer = !HS || half == 0;        // HS: half 0 stores the row outputs
  NodeSmem& S = smem[slot];
  const long long inst = node / p.N;
  const int n = static_cast<int>(node - inst * p.N);
  const long long xrow = inst * (p.N + 1) + n;
  const double dt = p.dt;
  const bool row = r < kQNx;
  const bool res_row = r >= 7 && r < 7 + NR;  // rows carrying the residual (embed: v̇ [, ω̇])

  if (row) S.x[r] = p.xs[xrow * kQNx + r];
  if (r < kQNu) S.u[r] = p.us[node * kQNu + r];
  if (VAR == kVarGround && r < 9) S.aux[r] = p.aux[node * 9 + r];
  // the tail's inputs from the iterate, loaded up front (host-mapped in latency
  // mode: each is a PCIe round trip that would otherwise follow the RK4 stages)
  double xn = 0.0, rx = 0.0, rxn = 0.0, ru = 0.0;
  if (row) {
    xn = p.xs[(xrow + 1) * kQNx + r];
    if (p.q) rx = p.rxs[xrow * kQNx + r];
    if (p.q && n == p.N - 1) rxn = p.rxs[(xrow + 1) * kQNx + r];
  }
  if (r < kQNu && p.r) ru = p.rus[node * kQNu + r];
  // Programmatic dependent launch (fused cycle): everything above reads only
  // the caller's iterate; the MLP kernel's outputs (and a feature kernel's z0)
  // are read after its grid has completed. A no-op without the launch attribute.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const double* hn = ORDER == 2 ? p.hess + node * NH : nullptr;
  if (ORDER == 2 && HS) {
    double* hs = hsm + slot * NH;
    const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(hs));
    for (int i = nl; i < NH; i += kStep)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8u * i), "l"(hn + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    hn = hs;
  }
  __syncwarp();
  for (int c = nl; c < NF; c += kStep) S.z0[c] = p.z0 ? p.z0[node * NF + c] : Feature<VAR>(c, S.x, S.u, S.aux);
  // Taylor rows: lane 7+o evaluates residual row o (TaylorApprox, taylor.hpp:13-24)
  const int o = res_row ? r - 7 : 0;
  const double* jrow_g = p.jac + (node * NR + o) * NF;
  const double fbo = res_row ? p.fbar[node * NR + o] : 0.0;
  double jn0[NF];  // HS: this lane's Jacobian row, loaded once instead of at every stage
  if (HS) {
#pragma unroll
    for (int c = 0; c < NF; ++c) jn0[c] = res_row ? __ldg(jrow_g + c) : 0.0;
  }
  // body wrench = mix · u (MixThrustTorque, dynamics.cpp:57-62)
  double tb[3], tau[3];
#pragma unroll
  for (int rr = 0; rr < 6; ++rr) {
    double sum = 0.0;
#pragma unroll
    for (int c = 0; c < 4; ++c) sum += p.mix[rr][c] * S.u[c];
    if (rr < 3) tb[rr] = sum; else tau[rr - 3] = sum;
  }

  int failed = 0;
  // sensitivity columns of this lane: all kQNf (+1 pad), or (HS) 10 from jo
  constexpr int kJ = HS ? 10 : kQNf + 1;
  const int jo = HS ? 8 * half : 0;
  double acc[kJ];
#pragma unroll 1
  for (int s = 0; s < 4; ++s) {
    const double cs = s == 0 ? 0.0 : (s == 3 ? dt : 0.5 * dt);
    // stage state x_s = x + c_s·k_{s-1} (integrator.cpp:57, 65, 73)
    if (row) S.xs[r] = s == 0 ? S.x[r] : S.x[r] + cs * S.k[s - 1][r];
    __syncwarp();
    // dz = features(x_s, u, aux) − z0 (the EvalTaylor argument, sqp_rti.cpp:96-99)
    for (int c = nl; c < NF; c += kStep) S.dz[c] = Feature<VAR>(c, S.xs, S.u, S.aux) - S.z0[c];
    __syncwarp();
    if (ORDER == 2) {  // G[o][a] = Σ_b H_o(a,b)·dz_b, n_r·n_f rows spread over the half-warp
      if (HS && s == 0) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
      }
      auto g_row = [&](int e) {
        const double* h = hn + e * NF;
        double g = 0.0;
#pragma unroll
        for (int b = 0; b < NF; ++b) g += (HS ? h[b] : __ldg(h + b)) * S.dz[b];
        S.g[e] = g;
      };
      if constexpr (HS) {  // shared-memory rows, unrolled: the lane's FMA chains interleave
        constexpr int kRowsPerLane = (NR * NF + 31) / 32;
#pragma unroll
        for (int i = 0; i < kRowsPerLane; ++i)
          if (lane + 32 * i < NR * NF) g_row(lane + 32 * i);
      } else {
        for (int e = r; e < NR * NF; e += 16) g_row(e);
      }
      __syncwarp();
    }
    const double* X = S.xs;
    // stage Jacobian row: nominal + embed·EvalTaylorJacobian (taylor.cpp:66-74)
    double fx[kQNx], fu[kQNu], y = 0.0, fnom;
    {
      double jn[NF], jc[kQNf];
#pragma unroll
      for (int c = 0; c < NF; ++c) jn[c] = HS ? jn0[c] : (res_row ? __ldg(jrow_g + c) : 0.0);
      if (res_row) {  // EvalTaylor row o: f_bar + jac·dz (+ ½ dzᵀ H_o dz) (taylor.cpp:57-64)
        double a1 = 0.0;
#pragma unroll
        for (int c = 0; c < NF; ++c) a1 += jn[c] * S.dz[c];
        y = fbo + a1;
        if (ORDER == 2) {  // jn row o += H_o·dz (EvalTaylorJacobian, taylor.cpp:66-74)
          const double* G = S.g + o * NF;
          double qv = 0.0;
#pragma unroll
          for (int a = 0; a < NF; ++a) qv += S.dz[a] * G[a];
#pragma unroll
          for (int c = 0; c < NF; ++c) jn[c] += G[c];
          y += 0.5 * qv;
        }
      }
      ChainRow<VAR>(jn, X, jc);  // zero unless res_row (jn is zero there)
      fnom = NominalRowAndJacobian(row ? r : 0, X, tb, tau, p, jc, fx, fu);
    }
    const double qn = sqrt(X[3] * X[3] + X[4] * X[4] + X[5] * X[5] + X[6] * X[6]);
    if (!failed && fabs(qn - 1.0) > 0.25) failed = 10 + s + 1;  // InputDomainError in f (dynamics.cpp:70-73)
    double kr = 0.0;
    if (row) {
      kr = fnom + (res_row ? y : 0.0);
      S.k[s][r] = kr;
    }
    const unsigned nonfinite = __ballot_sync(0xffffffffu, row && !isfinite(kr)) & half_mask;
    if (!failed && nonfinite) failed = 20 + s + 1;  // CheckFinite (integrator.cpp:12-15)

    // row r of dk_s: x columns jx[j] + Σ_m (c·jx[m]) dk[m][j]; u columns ju[j] + Σ_m (c·jx[m]) dk[m][j]
    auto jcol = [&](int c) { return c < kQNx ? fx[c] : (c < kQNf ? fu[c - kQNx] : 0.0); };  // c compile-time
    double nd[kJ];
#pragma unroll
    for (int j = 0; j < kJ; ++j) nd[j] = HS ? (half ? jcol(8 + j) : jcol(j)) : jcol(j);
    if (s > 0) {
      const double* dkp = S.dk[(s - 1) & 1] + jo;
#pragma unroll
      for (int m = 0; m < kQNx; ++m) {
        const double a = cs * fx[m];
#pragma unroll
        for (int j = 0; j < kJ; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(dkp + m * kDkStride + j);
          nd[j] += a * v.x;
          nd[j + 1] += a * v.y;
        }
      }
    }
    // dk1 + 2·dk2 + 2·dk3 + dk4, left to right (integrator.cpp:84-88)
    const double wgt = s == 3 ? 1.0 : 2.0;
#pragma unroll
    for (int j = 0; j < kJ; ++j) acc[j] = s == 0 ? nd[j] : acc[j] + wgt * nd[j];
    if (s < 3 && row) {  // (HS: columns 8, 9 are written by both halves, with the same bits)
      double* dkn = S.dk[s & 1] + r * kDkStride + jo;
#pragma unroll
      for (int j = 0; j < kJ; j += 2) *reinterpret_cast<double2*>(dkn + j) = make_double2(nd[j], nd[j + 1]);
    }
    __syncwarp();
  }
  if (failed) {
    if (valid && r == 0 && writer) {
      if (p.first_bad) Report(p.first_bad, node, failed);
      if (p.status) p.status[node] = static_cast<unsigned char>(failed);
    }
    return;  // per-lane exit: no warp-wide barrier follows
  }

  const double h6 = dt / 6.0;
  // stage A | B rows in the free dk buffer (dk[1] was last read at stage 2), then coalesced stores
  double* stage = S.dk[1];
  if (row) {
#pragma unroll
    for (int j = 0; j < kJ; ++j) {
      const int c = jo + j;
      if (c < kQNx) stage[r * kQNx + c] = (r == c ? 1.0 : 0.0) + h6 * acc[j];
      else if (c < kQNf) stage[kQNx * kQNx + r * kQNu + (c - kQNx)] = h6 * acc[j];
    }
    // φ̄ = x + dt/6 (k1 + 2k2 + 2k3 + k4) (integrator.cpp:84-86)
    S.phi[r] = S.x[r] + h6 * (S.k[0][r] + 2.0 * S.k[1][r] + 2.0 * S.k[2][r] + S.k[3][r]);
  }
  __syncwarp(HS ? 0xffffffffu : half_mask);
  if (!valid) return;
  if (p.status && r == 0 && writer) p.status[node] = 0;
  if (p.a)
    for (int e = nl; e < kQNx * kQNx; e += kStep) p.a[node * (kQNx * kQNx) + e] = stage[e];
  if (p.b)
    for (int e = nl; e < kQNx * kQNu; e += kStep) p.b[node * (kQNx * kQNu) + e] = stage[kQNx * kQNx + e];
  if (row && writer) {
    double v = S.phi[r];
    if (r >= 3 && r < 7)  // quaternion renormalised (RenormalizeQuat, integrator.cpp:17-20)
      v /= sqrt(S.phi[3] * S.phi[3] + S.phi[4] * S.phi[4] + S.phi[5] * S.phi[5] + S.phi[6] * S.phi[6]);
    if (p.phi) p.phi[node * kQNx + r] = v - xn;  // phi_res = φ̄ − x_{k+1} (sqp_rti.cpp:141)
    // cost terms (sqp_rti.cpp:143-148) and the terminal ones (:150-153)
    if (p.q) p.q[xrow * kQNx + r] = 2.0 * (p.qd[r] * (S.x[r] - rx));
    if (p.hx) p.hx[xrow * kQNx + r] = 2.0 * p.qd[r];
    if (n == p.N - 1) {
      if (p.q) p.q[(xrow + 1) * kQNx + r] = 2.0 * (p.qf[r] * (xn - rxn));
      if (p.hx) p.hx[(xrow + 1) * kQNx + r] = 2.0 * p.qf[r];
    }
  }
  if (r < kQNu && writer) {
    const double u = S.u[r];
    if (p.r) p.r[node * kQNu + r] = 2.0 * (p.rd[r] * (u - ru));
    if (p.hu) p.hu[node * kQNu + r] = 2.0 * p.rd[r];
    if (p.lb) p.lb[node * kQNu + r] = p.umin[r] - u;
    if (p.ub) p.ub[node * kQNu + r] = p.umax[r] - u;
  }
}

template <int VAR>
__global__ void FeaturesKernel(const double* __restrict__ xs, const double* __restrict__ us,
                               const double* __restrict__ aux, long long n_inst, int N, double* __restrict__ z) {
  constexpr int NF = VarNf(VAR);
  const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long K = n_inst * N;
  if (e >= K * NF) return;
  const long long node = e / NF;
  const int c = static_cast<int>(e - node * NF);
  const double* x = xs + (node + node / N) * kQNx;  // inst·(N+1) + n
  z[e] = Feature<VAR>(c, x, us + node * kQNu, aux ? aux + node * 9 : nullptr);
}

}  // namespace

cudaError_t LaunchFeatures(int variant, const double* xs, const double* us, const double* aux, long long n_inst,
                           int N, double* z, cudaStream_t s) {
  const long long total = n_inst * N * VarNf(variant);
  if (total <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>((total + 255) / 256);
  switch (variant) {
    case kVarA: FeaturesKernel<kVarA><<<grid, 256, 0, s>>>(xs, us, aux, n_inst, N, z); break;
    case kVarAU: FeaturesKernel<kVarAU><<<grid, 256, 0, s>>>(xs, us, aux, n_inst, N, z); break;
    case kVarGround: FeaturesKernel<kVarGround><<<grid, 256, 0, s>>>(xs, us, aux, n_inst, N, z); break;
    default: FeaturesKernel<kVarFull><<<grid, 256, 0, s>>>(xs, us, aux, n_inst, N, z); break;
  }
  return cudaGetLastError();
}

template <int ORDER, int VAR, bool HS>
static cudaError_t LaunchBlk(const BlkParams& p, unsigned g, cudaStream_t s, bool pdl) {
  const int dyn = HS && ORDER == 2 ? kWarps * VarNr(VAR) * VarNf(VAR) * VarNf(VAR) * static_cast<int>(sizeof(double)) : 0;
  if (dyn > 0) {
    const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(QpBlocksKernel<ORDER, VAR, HS>), dyn);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(g);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.dynamicSmemBytes = static_cast<size_t>(dyn);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, QpBlocksKernel<ORDER, VAR, HS>, p);
}

cudaError_t LaunchQpBlocks(const BlkParams& p, cudaStream_t s, bool pdl) {
  const long long K = p.n_inst * p.N;
  if (K <= 0) return cudaSuccess;
  const char* e = std::getenv("RTN_BLK_HS");  // A/B aid: 0 forces the 4-CTA variant
  const bool hs = K <= kLatencyMaxNodes && !(e && e[0] == '0');  // latency-sized batches
  const long long per_cta = hs ? kWarps : 2 * kWarps;            // nodes per CTA
  const unsigned g = static_cast<unsigned>((K + per_cta - 1) / per_cta);
#define RTN_BLK(O, V) return hs ? LaunchBlk<O, V, true>(p, g, s, pdl) : LaunchBlk<O, V, false>(p, g, s, pdl)
  switch (p.variant * 2 + (p.order == 2 ? 1 : 0)) {
    case kVarFull * 2: RTN_BLK(1, kVarFull);
    case kVarFull * 2 + 1: RTN_BLK(2, kVarFull);
    case kVarA * 2: RTN_BLK(1, kVarA);
    case kVarA * 2 + 1: RTN_BLK(2, kVarA);
    case kVarAU * 2: RTN_BLK(1, kVarAU);
    case kVarAU * 2 + 1: RTN_BLK(2, kVarAU);
    case kVarGround * 2: RTN_BLK(1, kVarGround);
    default: RTN_BLK(2, kVarGround);
  }
#undef RTN_BLK
}

}  // namespace rtn
