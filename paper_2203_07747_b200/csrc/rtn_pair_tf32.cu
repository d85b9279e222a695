// Pair-kernel instantiations, TF32 mode (one kind::tf32 pass), plus the TF32
// quad (latency) and rows (width-256 throughput) kernels.
#include "rtn_pair_launch.cuh"
#include "rtn_quad.cuh"
#include "rtn_rows.cuh"

namespace rtn {

cudaError_t LaunchPairTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int wp, bool latency,
                           int grid, cudaStream_t st) {
  if (latency) {
    return wp == 256 ? LaunchPairT<256, 8, 1, 24, kTF32>(prm, th, tl, grid, st)
                     : LaunchPairT<512, 8, 1, 24, kTF32>(prm, th, tl, grid, st);
  }
  if (wp == 256) {
    switch (prm.P) {
      case 1: return LaunchPairT<256, 8, 1, 80, kTF32>(prm, th, tl, grid, st);
      case 2: return LaunchPairT<256, 8, 2, 80, kTF32>(prm, th, tl, grid, st);
      case 4: return LaunchPairT<256, 8, 4, 80, kTF32>(prm, th, tl, grid, st);
      case 8: return LaunchPairT<256, 8, 8, 80, kTF32>(prm, th, tl, grid, st);
      default: return LaunchPairT<256, 8, 16, 80, kTF32>(prm, th, tl, grid, st);
    }
  }
  switch (prm.P) {
    case 1: return LaunchPairT<512, 4, 1, 80, kTF32>(prm, th, tl, grid, st);
    case 2: return LaunchPairT<512, 4, 2, 80, kTF32>(prm, th, tl, grid, st);
    case 4: return LaunchPairT<512, 4, 4, 80, kTF32>(prm, th, tl, grid, st);
    case 8: return LaunchPairT<512, 4, 8, 80, kTF32>(prm, th, tl, grid, st);
    default: return LaunchPairT<512, 4, 16, 80, kTF32>(prm, th, tl, grid, st);
  }
}

cudaError_t LaunchQuadTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  return LaunchQuadT<8, 24, kTF32>(prm, th, tl, grid, st);
}

cudaError_t LaunchRowsTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  using Cfg = RowsCfg<6>;
  auto kern = prm.act == 0 ? rtn_rows_kernel<6, 0> : (prm.act == 1 ? rtn_rows_kernel<6, 1> : rtn_rows_kernel<6, 2>);
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

// Geometry for every mode lives here (host-only logic). 3xTF32 at width 512
// always takes the 24-row tile: its TMEM fits four main accumulators per
// 256-neuron block (rtn_pair.cuh, kChains), which keeps the mode within 1e-5.
PairGeom PairGeometry(int mode, int wp, bool latency, int n_in) {
  if (latency || (mode == k3xTF32 && wp == 512)) return {1, 24};
  const int ntc = 80;
  int p = (mode == kTF32 || mode == kBF16) ? 16 : 4;
  while (p > 1 && p * (1 + n_in) > ntc) p >>= 1;
  return {p, ntc};
}

}  // namespace rtn
