// rtn_qpsolve.cu — batched feedback solve, fp64, sm_100a.
//
// resmpc::SolveFeedback (proj/src/sqp_rti.cpp:157-180) for many independent MPC
// instances: condensing (proj/src/qp.cpp:33-73) and the primal active-set box QP
// (proj/src/qp.cpp:77-208), then the state recovery dx_k = M_k·du + c_k. One CTA
// per instance (grid-stride over instances), each CTA with a global-memory
// workspace for the condensed Hessian and the Cholesky factor of the free
// subproblem (N·nu <= 256). The recovery maps M_k (13 x N·nu) live in shared
// memory, one stage at a time: H accumulates M_kᵀ·diag(hx_k)·M_k as k advances,
// skipping the exactly-zero blocks (M_k has no columns >= k·nu). Scalar decisions
// of the active-set method (ratio test, worst multiplier, lowest index first) run
// on one thread in the reference's order; the dense algebra is CTA-parallel.
#include <cmath>

#include "rtn_qpsolve.h"

namespace rtn {
namespace {

constexpr int kT = 256;  // threads per CTA
constexpr int kNx = 13, kNu = 4;
constexpr double kTol = 1e-11;  // qp.cpp:138

struct Shared {
  int nf, blocking, worst, fail;
  double alpha, trace;
  signed char side;
};

// Recovery-map recursion M_{k+1} = A_k·M_k (+ B_k into column block k), c_{k+1} = A_k·c_k + φ_k
// (qp.cpp:42-48). Only columns < (k+1)·nu are non-zero.
__device__ void AdvanceRecovery(const FbParams& p, long long inst, int k, int nv, const double* M, double* Mn,
                                const double* c, double* cn) {
  const long long row = inst * p.N + k;
  const double* A = p.a + row * (kNx * kNx);
  const double* B = p.b + row * (kNx * kNu);
  const int lim = (k + 1) * kNu;
  for (int e = threadIdx.x; e < kNx * nv; e += kT) {
    const int i = e / nv, j = e - i * nv;
    double s = 0.0;
    if (j < k * kNu) {
#pragma unroll
      for (int m = 0; m < kNx; ++m) s += A[i * kNx + m] * M[m * nv + j];
    }
    if (j >= k * kNu && j < lim) s += B[i * kNu + (j - k * kNu)];  // 0 + B (the A·M part is exactly zero)
    Mn[e] = s;
  }
  if (threadIdx.x < kNx) {
    const int i = threadIdx.x;
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < kNx; ++m) s += A[i * kNx + m] * c[m];
    cn[i] = s + p.phi[row * kNx + i];
  }
}

// Element (i, j), j <= i, of the free-subproblem factor: full rows of stride
// ld (PACKED = false) or the packed lower triangle, row i at i(i+1)/2 (only the
// lower triangle is ever read, so N = 50's 200 x 200 factor fits shared memory).
template <bool PACKED>
__device__ __forceinline__ int Lx(int i, int j, int ld) {
  return PACKED ? ((i * (i + 1)) >> 1) + j : i * ld + j;
}

// Cholesky of the nf x nf matrix in L, in place, right-looking in panels of
// four columns: the panel is factored column by column, then the trailing
// matrix takes the panel's rank-4 update with one read-modify-write per
// element. Every element still sees a(i,j) − l(i,0)l(j,0) − l(i,1)l(j,1) − …
// in ascending k, the operation sequence of qp.cpp's left-looking LLT, but the
// work per column is spread over the CTA and the trailing matrix's shared-
// memory traffic is a quarter of the unblocked form's (profiles/r01_ncu_feedback_n50.txt).
// Returns false (for every thread) on a non-positive pivot.
template <bool PACKED>
__device__ bool Cholesky(double* L, int nf, int ld, Shared&) {
  constexpr int kPw = 4;
  for (int j0 = 0; j0 < nf; j0 += kPw) {
    const int jw = min(kPw, nf - j0), pe = j0 + jw;
    for (int j = j0; j < pe; ++j) {  // panel column j
      const double d = L[Lx<PACKED>(j, j, ld)];
      if (d <= 0.0) return false;  // every thread read the same pivot
      const double ljj = sqrt(d);
      for (int i = j + 1 + threadIdx.x; i < nf; i += kT) L[Lx<PACKED>(i, j, ld)] /= ljj;
      __syncthreads();
      if (threadIdx.x == 0) L[Lx<PACKED>(j, j, ld)] = ljj;  // all threads have read the pivot
      const int nm = pe - (j + 1);  // panel columns right of j
      if (nm > 0) {
        for (int e = threadIdx.x; e < (nf - j - 1) * nm; e += kT) {
          const int i = j + 1 + e / nm, m = j + 1 + e % nm;
          if (i >= m) L[Lx<PACKED>(i, m, ld)] -= L[Lx<PACKED>(i, j, ld)] * L[Lx<PACKED>(m, j, ld)];
        }
      }
      __syncthreads();
    }
    if (pe < nf) {  // trailing update, rows i >= m >= pe
      for (int i = pe + (threadIdx.x >> 3); i < nf; i += kT / 8) {
        double li[kPw];
#pragma unroll
        for (int t = 0; t < kPw; ++t) li[t] = t < jw ? L[Lx<PACKED>(i, j0 + t, ld)] : 0.0;
        double* row = L + Lx<PACKED>(i, 0, ld);
        for (int m = pe + (threadIdx.x & 7); m <= i; m += 8) {
          const double* lm = L + Lx<PACKED>(m, j0, ld);
          double s = row[m];
#pragma unroll
          for (int t = 0; t < kPw; ++t)
            if (t < jw) s -= li[t] * lm[t];
          row[m] = s;
        }
      }
      __syncthreads();
    }
  }
  return true;
}

// Solve L·Lᵀ·y = b in place (column-oriented substitutions) on warp 0; the
// rest of the CTA waits at the closing barrier.
template <bool PACKED>
__device__ void CholSolve(const double* L, int nf, int ld, double* y) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = 0; i < nf; ++i) {
      if (lane == 0) y[i] /= L[Lx<PACKED>(i, i, ld)];
      __syncwarp();
      const double yi = y[i];
      for (int m = i + 1 + lane; m < nf; m += 32) y[m] -= L[Lx<PACKED>(m, i, ld)] * yi;
      __syncwarp();
    }
    for (int i = nf - 1; i >= 0; --i) {
      if (lane == 0) y[i] /= L[Lx<PACKED>(i, i, ld)];
      __syncwarp();
      const double yi = y[i];
      for (int m = lane; m < i; m += 32) y[m] -= L[Lx<PACKED>(i, m, ld)] * yi;
      __syncwarp();
    }
  }
  __syncthreads();
}

// LMODE: where the Cholesky factor of the free subproblem lives — 0 global
// workspace, 1 shared memory (full rows, N <= 36), 2 shared memory (packed
// lower triangle, N <= 51). Shared memory removes its O(nf³) inner-product
// traffic from L2.
template <int LMODE>
__global__ void __launch_bounds__(kT) FeedbackKernel(const FbParams p) {
  constexpr bool SMEM_L = LMODE != 0, PACKED = LMODE == 2;
  extern __shared__ double dyn[];
  const int N = p.N, nv = N * kNu;
  double* M = dyn;              // 13 x nv
  double* Mn = M + kNx * nv;    // 13 x nv
  double* c = Mn + kNx * nv;    // 13
  double* cn = c + 16;          // 13
  double* g = cn + 16;          // the QP vectors (gradient, iterate, subproblem rhs/solution,
  double* x = g + nv;           // bounds, full gradient) in shared memory: the scalar pivot
  double* y = x + nv;           // loops of the active-set method run on one thread and were
  double* lb = y + nv;          // latency-bound on L2 reads
  double* ub = lb + nv;
  double* grad = ub + nv;
  double* Ls = grad + nv;       // nv x nv, or nv(nv+1)/2 packed (SMEM_L)
  int* fidx = reinterpret_cast<int*>(Ls + (SMEM_L ? (PACKED ? (nv * (nv + 1)) / 2 : nv * nv) : 0));  // nv
  signed char* act = reinterpret_cast<signed char*>(fidx + nv);      // nv
  __shared__ Shared sh;
  double* W = p.work + static_cast<long long>(blockIdx.x) * FeedbackWorkPerCta(N);
  double* H = W;               // nv x nv
  double* L = SMEM_L ? Ls : H + nv * nv;  // nv x nv (free subproblem, row stride nv)

  for (long long inst = blockIdx.x; inst < p.n_inst; inst += gridDim.x) {
    // ---------------- condensing (qp.cpp:33-73) ----------------
    for (int e = threadIdx.x; e < nv * nv; e += kT) H[e] = 0.0;
    for (int e = threadIdx.x; e < kNx * nv; e += kT) M[e] = 0.0;
    for (int i = threadIdx.x; i < nv; i += kT) g[i] = 0.0;
    if (threadIdx.x < kNx) c[threadIdx.x] = p.x_meas[inst * kNx + threadIdx.x] - p.xs[inst * (N + 1) * kNx + threadIdx.x];
    __syncthreads();
    for (int k = 0; k <= N; ++k) {
      const long long xrow = inst * (N + 1) + k;
      const double* hxk = p.hx + xrow * kNx;
      const double* qk = p.q + xrow * kNx;
      const int lim = k * kNu;  // M_k is zero in columns >= k·nu
      for (int e = threadIdx.x; e < lim * lim; e += kT) {
        const int i = e / lim, j = e - i * lim;
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < kNx; ++r) s += M[r * nv + i] * (hxk[r] * M[r * nv + j]);
        H[i * nv + j] += s;
      }
      for (int i = threadIdx.x; i < lim; i += kT) {
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < kNx; ++r) s += M[r * nv + i] * (qk[r] + hxk[r] * c[r]);
        g[i] += s;
      }
      __syncthreads();
      if (k < N) {
        AdvanceRecovery(p, inst, k, nv, M, Mn, c, cn);
        __syncthreads();
        for (int e = threadIdx.x; e < kNx * nv; e += kT) M[e] = Mn[e];
        if (threadIdx.x < kNx) c[threadIdx.x] = cn[threadIdx.x];
        __syncthreads();
      }
    }
    for (int e = threadIdx.x; e < nv; e += kT) {
      const long long row = inst * N + e / kNu;
      const int j = e % kNu;
      H[e * nv + e] += p.hu[row * kNu + j];
      g[e] += p.r[row * kNu + j];
      lb[e] = p.lb[row * kNu + j];
      ub[e] = p.ub[row * kNu + j];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nv * nv; e += kT) {  // exact symmetry (qp.cpp:71)
      const int i = e / nv, j = e - i * nv;
      if (i < j) {
        const double v = 0.5 * (H[i * nv + j] + H[j * nv + i]);
        H[i * nv + j] = v;
        H[j * nv + i] = v;
      } else if (i == j) {
        H[e] = 0.5 * (H[e] + H[e]);
      }
    }
    // ---------------- box QP (qp.cpp:104-208) ----------------
    if (threadIdx.x == 0) {  // SolveFeedback / SolveBoxQp input checks (sqp_rti.cpp:159-160, qp.cpp:107-108)
      int bad = 0;
      for (int i = 0; i < kNx; ++i) bad |= !isfinite(p.x_meas[inst * kNx + i]);
      for (int i = 0; i < nv; ++i) bad |= lb[i] > ub[i];
      sh.fail = bad;
    }
    __syncthreads();
    int status = sh.fail ? 2 : 0, iters = 0;
    for (int i = threadIdx.x; i < nv; i += kT) {
      signed char a = p.active ? p.active[inst * nv + i] : 0;
      if (a < 0 && !isfinite(lb[i])) a = 0;
      if (a > 0 && !isfinite(ub[i])) a = 0;
      act[i] = a;
      x[i] = a < 0 ? lb[i] : (a > 0 ? ub[i] : fmin(fmax(0.0, lb[i]), ub[i]));  // std::clamp(0, lb, ub)
    }
    __syncthreads();
    if (threadIdx.x == 0) sh.fail = 0;
    __syncthreads();
    bool done = false;
    for (iters = 0; status == 0 && iters < 200 && !done; ++iters) {
      if (threadIdx.x == 0) {  // free set in index order
        int nf = 0;
        for (int i = 0; i < nv; ++i)
          if (act[i] == 0) fidx[nf++] = i;
        sh.nf = nf;
      }
      __syncthreads();
      const int nf = sh.nf;
      bool at_opt = true;
      if (nf > 0) {
        // hff and rhs = −g_f − Σ_{j active} H(f, j)·x_j (qp.cpp:77-92)
        for (int e = threadIdx.x; e < nf * nf; e += kT) {
          const int a = e / nf, b = e - a * nf;
          if (b <= a) L[Lx<PACKED>(a, b, nv)] = H[fidx[a] * nv + fidx[b]];
        }
        for (int a = threadIdx.x; a < nf; a += kT) {
          double dot = 0.0;
          for (int j = 0; j < nv; ++j)
            if (act[j] != 0) dot += H[fidx[a] * nv + j] * x[j];
          y[a] = -g[fidx[a]] - dot;
        }
        if (threadIdx.x == 0) sh.fail = 0;
        __syncthreads();
        if (!Cholesky<PACKED>(L, nf, nv, sh)) {  // regularise once (qp.cpp:94-100)
          if (threadIdx.x == 0) {
            double tr = 0.0;
            for (int a = 0; a < nf; ++a) tr += H[fidx[a] * nv + fidx[a]];
            sh.trace = 1e-9 * fmax(1.0, tr / (nf > 1 ? nf : 1));
            sh.fail = 0;
          }
          __syncthreads();
          for (int e = threadIdx.x; e < nf * nf; e += kT) {
            const int a = e / nf, b = e - a * nf;
            if (b <= a) L[Lx<PACKED>(a, b, nv)] = H[fidx[a] * nv + fidx[b]] + (a == b ? sh.trace : 0.0);
          }
          __syncthreads();
          if (!Cholesky<PACKED>(L, nf, nv, sh)) {
            status = 3;  // not positive definite even after regularisation
            break;
          }
        }
        CholSolve<PACKED>(L, nf, nv, y);
        if (threadIdx.x == 0) {  // ratio test toward the subproblem solution (qp.cpp:150-170)
          double alpha = 1.0;
          int blocking = -1;
          signed char side = 0;
          for (int a = 0; a < nf; ++a) {
            const int idx = fidx[a];
            const double step = y[a] - x[idx];
            if (step > kTol && isfinite(ub[idx])) {
              const double al = (ub[idx] - x[idx]) / step;
              if (al < alpha - kTol) {
                alpha = al;
                blocking = idx;
                side = 1;
              }
            } else if (step < -kTol && isfinite(lb[idx])) {
              const double al = (lb[idx] - x[idx]) / step;
              if (al < alpha - kTol) {
                alpha = al;
                blocking = idx;
                side = -1;
              }
            }
          }
          sh.alpha = alpha;
          sh.blocking = blocking;
          sh.side = side;
        }
        __syncthreads();
        const double alpha = sh.alpha;
        for (int a = threadIdx.x; a < nf; a += kT) {
          const int idx = fidx[a];
          x[idx] += alpha * (y[a] - x[idx]);
        }
        __syncthreads();
        if (sh.blocking >= 0) {
          if (threadIdx.x == 0) {
            act[sh.blocking] = sh.side;
            x[sh.blocking] = sh.side > 0 ? ub[sh.blocking] : lb[sh.blocking];
          }
          at_opt = false;
        }
        __syncthreads();
      }
      if (at_opt) {  // multipliers of the working set; release the worst violator (qp.cpp:172-196)
        for (int i = threadIdx.x; i < nv; i += kT) {
          double s = 0.0;
          for (int j = 0; j < nv; ++j) s += H[i * nv + j] * x[j];
          grad[i] = s + g[i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          int worst = -1;
          double worst_val = -1e-10;
          for (int i = 0; i < nv; ++i) {
            if (act[i] == 0) continue;
            const double lam = act[i] < 0 ? grad[i] : -grad[i];
            if (lam < worst_val) {
              worst_val = lam;
              worst = i;
            }
          }
          sh.worst = worst;
          if (worst >= 0) act[worst] = 0;
        }
        __syncthreads();
        if (sh.worst < 0) done = true;
      }
    }
    // iters = passes run: on success the final pass counts (qp.cpp:193), at the cap it is 200
    if (status == 0 && !done) status = 1;  // kMaxIter (qp.cpp:199-207)
    __syncthreads();
    // ---------------- recovery and outputs (sqp_rti.cpp:168-178) ----------------
    if (status < 2) {
      for (int e = threadIdx.x; e < kNx * nv; e += kT) M[e] = 0.0;
      if (threadIdx.x < kNx) c[threadIdx.x] = p.x_meas[inst * kNx + threadIdx.x] - p.xs[inst * (N + 1) * kNx + threadIdx.x];
      __syncthreads();
      for (int k = 0; k <= N; ++k) {
        if (threadIdx.x < kNx) {
          const int i = threadIdx.x;
          double s = 0.0;
          for (int j = 0; j < k * kNu; ++j) s += M[i * nv + j] * x[j];
          p.dxs[(inst * (N + 1) + k) * kNx + i] = s + c[i];
        }
        __syncthreads();
        if (k < N) {
          AdvanceRecovery(p, inst, k, nv, M, Mn, c, cn);
          __syncthreads();
          for (int e = threadIdx.x; e < kNx * nv; e += kT) M[e] = Mn[e];
          if (threadIdx.x < kNx) c[threadIdx.x] = cn[threadIdx.x];
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < nv; i += kT) p.dus[inst * nv + i] = x[i];
      if (p.active)
        for (int i = threadIdx.x; i < nv; i += kT) p.active[inst * nv + i] = act[i];
      if (threadIdx.x < kNu) p.u_cmd[inst * kNu + threadIdx.x] = p.us[inst * N * kNu + threadIdx.x] + x[threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      bool finite = status < 2;
      for (int i = 0; finite && i < nv; ++i) finite = isfinite(x[i]);
      for (int i = 0; finite && i < kNu; ++i) finite = isfinite(p.u_cmd[inst * kNu + i]);
      // non-finite solution, or a failed factorisation: SolveFeedback throws (sqp_rti.cpp:176-178)
      p.status[inst] = finite ? status : (status == 3 ? 3 : 2);
      p.iterations[inst] = finite ? iters : 0;
    }
    __syncthreads();
  }
}

}  // namespace

size_t FeedbackSmemBytes(int N) {
  const size_t nv = static_cast<size_t>(N) * kNu;
  return sizeof(double) * (2 * kNx * nv + 32 + 6 * nv) + sizeof(int) * nv + nv + 16;
}

cudaError_t LaunchFeedback(const FbParams& p, int grid, cudaStream_t s) {
  if (p.n_inst <= 0) return cudaSuccess;
  const size_t nv = static_cast<size_t>(p.N) * kNu;
  const size_t base = FeedbackSmemBytes(p.N);
  const size_t full = base + sizeof(double) * nv * nv, packed = base + sizeof(double) * (nv * (nv + 1) / 2);
  constexpr size_t kCap = 220 * 1024;
  const int mode = full <= kCap ? 1 : (packed <= kCap ? 2 : 0);
  const size_t smem = mode == 1 ? full : (mode == 2 ? packed : base);
  static size_t attr[3] = {0, 0, 0};
  auto kern = mode == 1 ? FeedbackKernel<1> : (mode == 2 ? FeedbackKernel<2> : FeedbackKernel<0>);
  if (smem > attr[mode]) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[mode] = smem;
  }
  kern<<<grid, kT, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rtn
