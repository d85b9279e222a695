// Pair-kernel instantiations for second order (Hessian rows), all precision
// modes: the quadrotor tiles (n_in = 17, NTC = 48, ORD2 = 1) for TF32 and
// bf16x3, and the generic tiles (any n_in <= 31, NTC = 24 or 40, ORD2 = 2).
// Stage counts keep each configuration inside the shared-memory budget
// (generic tiles add 33 KB of per-thread tangent rows and the slot table).
#include "rtn_pair_launch.cuh"

namespace rtn {

int Order2Ntc(int mode, int n_in) {
  if (n_in == kNin2 && mode != k3xTF32) return kNtc2;
  return 1 + n_in <= 24 ? 24 : 40;
}

template <int WP>
static cudaError_t LaunchOrder2W(int mode, const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                                 cudaStream_t st) {
  if (prm.nt == kNtc2) {
    if (mode == kTF32) return LaunchPairT<WP, 8, 1, kNtc2, kTF32, 1>(prm, th, tl, grid, st);
    if (mode == kBF16) return LaunchPairT<WP, (WP == 256 ? 4 : 8), 1, kNtc2, kBF16, 1>(prm, th, tl, grid, st);
    return LaunchPairT<WP, 8, 1, kNtc2, kBF16x3, 1>(prm, th, tl, grid, st);
  }
  if (prm.nt == 24) {
    if (mode == kTF32) return LaunchPairT<WP, 8, 1, 24, kTF32, 2>(prm, th, tl, grid, st);
    if (mode == kBF16) return LaunchPairT<WP, (WP == 256 ? 4 : 8), 1, 24, kBF16, 2>(prm, th, tl, grid, st);
    if (mode == kBF16x3) return LaunchPairT<WP, 8, 1, 24, kBF16x3, 2>(prm, th, tl, grid, st);
    return LaunchPairT<WP, 4, 1, 24, k3xTF32, 2>(prm, th, tl, grid, st);
  }
  if (mode == kTF32) return LaunchPairT<WP, 4, 1, 40, kTF32, 2>(prm, th, tl, grid, st);
  if (mode == kBF16) return LaunchPairT<WP, 4, 1, 40, kBF16, 2>(prm, th, tl, grid, st);
  if (mode == kBF16x3) return LaunchPairT<WP, 4, 1, 40, kBF16x3, 2>(prm, th, tl, grid, st);
  return LaunchPairT<WP, 2, 1, 40, k3xTF32, 2>(prm, th, tl, grid, st);
}

cudaError_t LaunchPairOrder2(int mode, const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp,
                             int grid, cudaStream_t st) {
  return wp == 256 ? LaunchOrder2W<256>(mode, prm, th, tl, grid, st) : LaunchOrder2W<512>(mode, prm, th, tl, grid, st);
}

}  // namespace rtn
