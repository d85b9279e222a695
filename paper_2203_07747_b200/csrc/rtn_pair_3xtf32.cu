// Pair-kernel instantiations, 3xTF32 mode (split hi/lo tf32 operands, 3 passes).
#include "rtn_pair_launch.cuh"
#include "rtn_quad.cuh"

namespace rtn {

cudaError_t LaunchPair3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                             int grid, cudaStream_t st) {
  if (latency) {
    return wp == 256 ? LaunchPairT<256, 8, 1, 24, k3xTF32>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, 24, k3xTF32>(prm, th, tl, grid, st);
  }
  if (wp == 256) {
    switch (prm.P) {
      case 1: return LaunchPairT<256, 4, 1, 80, k3xTF32>(prm, th, tl, grid, st);
      case 2: return LaunchPairT<256, 4, 2, 80, k3xTF32>(prm, th, tl, grid, st);
      default: return LaunchPairT<256, 4, 4, 80, k3xTF32>(prm, th, tl, grid, st);
    }
  }
  switch (prm.P) {
    case 1: return LaunchPairT<512, 4, 1, 40, k3xTF32>(prm, th, tl, grid, st);
    default: return LaunchPairT<512, 4, 2, 40, k3xTF32>(prm, th, tl, grid, st);
  }
}

cudaError_t LaunchQuad3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st) {
  using Cfg = PairCfg<512, 8, 1, 24, k3xTF32, false>;
  auto kern = rtn_quad_kernel<8, 24, k3xTF32>;
  static bool attr_set = false;
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

}  // namespace rtn
