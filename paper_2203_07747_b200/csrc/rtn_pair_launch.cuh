// rtn_pair_launch.cuh — template launch helpers shared by the per-mode
// translation units.
#pragma once

#include "rtn_launch.h"
#include "rtn_pair.cuh"

namespace rtn {

template <int WP, int NS, int P, int NTC, int MODE, bool ORD2 = false>
cudaError_t LaunchPairT(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  using Cfg = PairCfg<WP, NS, P, NTC, MODE, ORD2>;
  auto kern = rtn_pair_kernel<WP, NS, P, NTC, MODE, ORD2>;
  static bool attr_set = false;  // per instantiation, per process
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

}  // namespace rtn
