// Pair-kernel instantiations, 3xTF32 mode (split hi/lo tf32 operands, 3 passes,
// main pass rotating over PairCfg::kChains accumulators).
#include "rtn_pair_launch.cuh"
#include "rtn_quad.cuh"

namespace rtn {

cudaError_t LaunchPair3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                             int grid, cudaStream_t st) {
  if (wp == 512) return LaunchPairT<512, 8, 1, 24, k3xTF32>(prm, th, tl, grid, st);  // PairGeometry: P = 1
  if (latency) return LaunchPairT<256, 8, 1, 24, k3xTF32>(prm, th, tl, grid, st);
  switch (prm.P) {
    case 1: return LaunchPairT<256, 4, 1, 80, k3xTF32>(prm, th, tl, grid, st);
    case 2: return LaunchPairT<256, 4, 2, 80, k3xTF32>(prm, th, tl, grid, st);
    default: return LaunchPairT<256, 4, 4, 80, k3xTF32>(prm, th, tl, grid, st);
  }
}

cudaError_t LaunchQuad3xTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                             cudaStream_t st) {
  return LaunchQuadT<8, 24, k3xTF32>(prm, th, tl, grid, st);
}

}  // namespace rtn
