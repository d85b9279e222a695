// rtn_launch.h — host-side launchers of the pair kernel, one translation unit
// per precision mode (rtn_pair_{tf32,3xtf32,bf16x3,order2}.cu) so they compile
// in parallel; rtn_mpc.cu dispatches.
#pragma once
#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <utility>

#include "rtn_kernel.cuh"

namespace rtn {

// cudaFuncSetAttribute applies per device: remember every (kernel, device)
// pair it was set for (a process may drive several devices through the C-ABI's
// `device` argument, from several threads).
inline cudaError_t EnsureSmem(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kern, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kern, dev});
  return e;
}

struct PairGeom {
  int P;        // nodes per CTA
  int ntc_max;  // NTC template (row stride per CTA)
};

// Tile geometry of the pair kernel for a mode / width / batch regime.
PairGeom PairGeometry(int mode, int wp, bool latency, int n_in);

// Launch status: cudaSuccess or the launch error.
cudaError_t LaunchPairTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                           int grid, cudaStream_t st);
cudaError_t LaunchPair3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                             int grid, cudaStream_t st);
cudaError_t LaunchPairBF16x3(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                             int grid, cudaStream_t st);
cudaError_t LaunchPairBF16(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                           int grid, cudaStream_t st);

// Latency kernel on 4-CTA clusters (rtn_quad.cuh): width 512, order <= 1,
// one node per CTA side, grid = 4 x ceil(K / 2).
cudaError_t LaunchQuadTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st);
cudaError_t LaunchQuadBF16x3(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st);
cudaError_t LaunchQuad3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st);
cudaError_t LaunchQuadBF16(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st);

// Width-256 throughput kernel with the activations as the A operand in TMEM
// (rtn_rows.cuh): TF32, order <= 1, 7 <= n_in <= 31, prm.P = 128 / (1 + n_in)
// nodes per CTA, grid = 2 x pairs.
cudaError_t LaunchRowsTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st);
constexpr int kRowsMinIn = 7, kRowsMaxInHost = 31, kRowsMaxMmaHost = 11, kRbMinInHost = 15;
constexpr int kRevMaxInHost = 24;  // reverse mode: W0' (512 x n_in) staged in shared memory
// TF32 width-512 throughput, activations split between TMEM and shared memory
// (rtn_split.cuh); th = the hidden pack in 64-row boxes. Same row geometry as the
// rows kernel (7 <= n_in <= 31).
cudaError_t LaunchSplitTF32(const KParams& prm, const CUtensorMap& th64, const CUtensorMap& tl, int grid,
                            cudaStream_t st);
// Reverse mode (TF32, width 512; rtn_reverse.cuh): pass 0 = values + σ' scratch
// (ta = hidden pack 64-row boxes, tb = output pack), pass 1 = adjoints + J
// (ta = transposed hidden pack, tb = W0' input-major padded to 32 rows).
cudaError_t LaunchReverse(int pass, const KParams& prm, const CUtensorMap& ta, const CUtensorMap& tb, int grid,
                          cudaStream_t st);
// Reverse mode on the pair kernel (3xTF32 / bf16x3, width 256 or 512; rtn_pair.cuh
// variants 3 = values, 4 = adjoints): th = hidden pack (pass 0) or its transpose
// (pass 1), tl = output pack (pass 0) or W0' padded to 32 rows (pass 1).
cudaError_t LaunchPairReverse(int mode, int wp, int pass, const KParams& prm, const CUtensorMap& th,
                              const CUtensorMap& tl, int grid, cudaStream_t st);
// rows per CTA side of the pair reverse passes
inline int PairReverseNtc(int mode, int wp, int pass) {
  if (mode == k3xTF32 && wp == 512) {
    static const bool adj24 = std::getenv("RTN_REV_ADJ24") != nullptr;  // A/B switch
    return pass == 1 && !adj24 ? 40 : 24;
  }
  return 80;
}
// BF16 width-512 throughput, the whole layer input as the A operand in TMEM
// (rtn_rowsb.cuh); 15 <= n_in <= 31.
cudaError_t LaunchRowsBF16(const KParams& prm, const CUtensorMap& th64, const CUtensorMap& tl, int grid,
                           cudaStream_t st);


// Order 2 (value + Jacobian + Hessian), n_in <= kMaxIn2. Order2Ntc picks the
// tile (rows per CTA side): 48 for the quadrotor's 17 inputs in TF32/bf16x3
// (compile-time slot tables), else 24 (n_in <= 23; 3xTF32 then rotates over 4
// main accumulators) or 40. Launch with prm.nt = that value and
// prm.ord2_g = ord2_tiles(n_in, nt) pair tiles per node (prm.num_tiles = g·K).
int Order2Ntc(int mode, int n_in);
cudaError_t LaunchPairOrder2(int mode, const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp,
                             int grid, cudaStream_t st);

}  // namespace rtn
