// Pair-kernel instantiations, single-pass BF16 mode (one kind::f16 pass on
// bf16 operands: half the operand bytes of tf32 and twice its MMA rate).
// Width 256 has 4 chunks of 64 k per block: 4 weight stages.
#include "rtn_pair_launch.cuh"
#include "rtn_quad.cuh"

namespace rtn {

cudaError_t LaunchPairBF16(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                           int grid, cudaStream_t st) {
  if (latency) {
    return wp == 256 ? LaunchPairT<256, 4, 1, 24, kBF16>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, 24, kBF16>(prm, th, tl, grid, st);
  }
  if (wp == 256) {
    switch (prm.P) {
      case 1: return LaunchPairT<256, 4, 1, 80, kBF16>(prm, th, tl, grid, st);
      case 2: return LaunchPairT<256, 4, 2, 80, kBF16>(prm, th, tl, grid, st);
      case 4: return LaunchPairT<256, 4, 4, 80, kBF16>(prm, th, tl, grid, st);
      case 8: return LaunchPairT<256, 4, 8, 80, kBF16>(prm, th, tl, grid, st);
      default: return LaunchPairT<256, 4, 16, 80, kBF16>(prm, th, tl, grid, st);
    }
  }
  switch (prm.P) {
    case 1: return LaunchPairT<512, 8, 1, 80, kBF16>(prm, th, tl, grid, st);
    case 2: return LaunchPairT<512, 8, 2, 80, kBF16>(prm, th, tl, grid, st);
    case 4: return LaunchPairT<512, 8, 4, 80, kBF16>(prm, th, tl, grid, st);
    case 8: return LaunchPairT<512, 8, 8, 80, kBF16>(prm, th, tl, grid, st);
    default: return LaunchPairT<512, 8, 16, 80, kBF16>(prm, th, tl, grid, st);
  }
}

cudaError_t LaunchQuadBF16(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  return LaunchQuadT<8, 24, kBF16>(prm, th, tl, grid, st);
}

}  // namespace rtn
