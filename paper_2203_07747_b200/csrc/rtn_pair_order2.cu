// Pair-kernel instantiations for second order (Hessian rows), all precision modes.
#include "rtn_pair_launch.cuh"

namespace rtn {

cudaError_t LaunchPairOrder2(int mode, const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp,
                             int grid, cudaStream_t st) {
  if (mode == kTF32)
    return wp == 256 ? LaunchPairT<256, 8, 1, kNtc2, kTF32, true>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, kNtc2, kTF32, true>(prm, th, tl, grid, st);
  if (mode == kBF16x3)
    return wp == 256 ? LaunchPairT<256, 8, 1, kNtc2, kBF16x3, true>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, kNtc2, kBF16x3, true>(prm, th, tl, grid, st);
  return wp == 256 ? LaunchPairT<256, 4, 1, kNtc2, k3xTF32, true>(prm, th, tl, grid, st)
                   : LaunchPairT<512, 2, 1, kNtc2, k3xTF32, true>(prm, th, tl, grid, st);
}

}  // namespace rtn
