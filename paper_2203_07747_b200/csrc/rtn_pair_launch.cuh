// rtn_pair_launch.cuh — template launch helpers shared by the per-mode
// translation units.
#pragma once

#include "rtn_launch.h"
#include "rtn_pair.cuh"
#include "rtn_quad.cuh"

namespace rtn {

template <int WP, int NS, int P, int NTC, int MODE, int ORD2 = 0>
cudaError_t LaunchPairT(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  using Cfg = PairCfg<WP, NS, P, NTC, MODE, ORD2>;
  auto kern = rtn_pair_kernel<WP, NS, P, NTC, MODE, ORD2>;
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

template <int NS, int NTC, int MODE>
cudaError_t LaunchQuadT(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  using Cfg = PairCfg<512, NS, 1, NTC, MODE, 0>;
  auto kern = rtn_quad_kernel<NS, NTC, MODE>;
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

}  // namespace rtn
