// rtn_launch.h — host-side launchers of the pair kernel, one translation unit
// per precision mode (rtn_pair_{tf32,3xtf32,bf16x3}.cu) so they compile in
// parallel; rtn_mpc.cu dispatches.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "rtn_kernel.cuh"

namespace rtn {

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

// Latency kernel on 4-CTA clusters (rtn_quad.cuh): TF32, width 512, order <= 1,
// one node per CTA side, grid = 4 x ceil(K / 2).
cudaError_t LaunchQuadTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st);
cudaError_t LaunchQuadBF16x3(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st);
cudaError_t LaunchQuad3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st);

// Width-256 throughput kernel with two tiles in flight per CTA pair
// (rtn_pingpong.cuh): TF32, order <= 1, P = 4 nodes per CTA side.
cudaError_t LaunchPingPongTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                               cudaStream_t st);

// Width-256 throughput kernel with the activations as the A operand in TMEM
// (rtn_rows.cuh): TF32, order <= 1, 7 <= n_in <= 31, prm.P = 128 / (1 + n_in)
// nodes per CTA, grid = 2 x pairs.
cudaError_t LaunchRowsTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st);
constexpr int kRowsMinIn = 7, kRowsMaxInHost = 31, kRowsMaxMmaHost = 11;

// Order 2 (value + Jacobian + Hessian; n_in = 17): two pair-tiles per node.
cudaError_t LaunchPairOrder2(int mode, const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp,
                             int grid, cudaStream_t st);

}  // namespace rtn
