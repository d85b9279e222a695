// Pair-kernel instantiations, BF16x3 mode (split hi/lo bf16 operands, 3 kind::f16 passes).
#include "rtn_pair_launch.cuh"
#include "rtn_quad.cuh"

namespace rtn {

cudaError_t LaunchPairBF16x3(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                             int grid, cudaStream_t st) {
  if (latency) {
    return wp == 256 ? LaunchPairT<256, 8, 1, 24, kBF16x3>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, 24, kBF16x3>(prm, th, tl, grid, st);
  }
  if (wp == 256) {
    switch (prm.P) {
      case 1: return LaunchPairT<256, 8, 1, 80, kBF16x3>(prm, th, tl, grid, st);
      case 2: return LaunchPairT<256, 8, 2, 80, kBF16x3>(prm, th, tl, grid, st);
      default: return LaunchPairT<256, 8, 4, 80, kBF16x3>(prm, th, tl, grid, st);
    }
  }
  switch (prm.P) {
    case 1: return LaunchPairT<512, 4, 1, 80, kBF16x3>(prm, th, tl, grid, st);
    case 2: return LaunchPairT<512, 4, 2, 80, kBF16x3>(prm, th, tl, grid, st);
    default: return LaunchPairT<512, 4, 4, 80, kBF16x3>(prm, th, tl, grid, st);
  }
}

cudaError_t LaunchQuadBF16x3(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st) {
  return LaunchQuadT<8, 24, kBF16x3>(prm, th, tl, grid, st);
}

}  // namespace rtn
