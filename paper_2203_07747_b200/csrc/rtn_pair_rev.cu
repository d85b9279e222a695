// Reverse-mode variants of the pair kernel (rtn_pair.cuh, ORD2 = 3 value pass,
// 4 adjoint pass) for the split-precision modes; the same tile geometry as
// their forward-mode throughput instantiations.
#include "rtn_pair_launch.cuh"

namespace rtn {

cudaError_t LaunchPairReverse(int mode, int wp, int pass, const KParams& prm, const CUtensorMap& th,
                              const CUtensorMap& tl, int grid, cudaStream_t st) {
  if (mode == k3xTF32) {
    if (wp == 512)
      return pass == 0 ? LaunchPairT<512, 8, 1, 24, k3xTF32, 3>(prm, th, tl, grid, st)
                       : (prm.nt == 40 ? LaunchPairT<512, 4, 1, 40, k3xTF32, 4>(prm, th, tl, grid, st)
                                       : LaunchPairT<512, 8, 1, 24, k3xTF32, 4>(prm, th, tl, grid, st));
    return pass == 0 ? LaunchPairT<256, 4, 1, 80, k3xTF32, 3>(prm, th, tl, grid, st)
                     : LaunchPairT<256, 4, 1, 80, k3xTF32, 4>(prm, th, tl, grid, st);
  }
  if (wp == 512)
    return pass == 0 ? LaunchPairT<512, 4, 1, 80, kBF16x3, 3>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 4, 1, 80, kBF16x3, 4>(prm, th, tl, grid, st);
  return pass == 0 ? LaunchPairT<256, 8, 1, 80, kBF16x3, 3>(prm, th, tl, grid, st)
                   : LaunchPairT<256, 8, 1, 80, kBF16x3, 4>(prm, th, tl, grid, st);
}

}  // namespace rtn
