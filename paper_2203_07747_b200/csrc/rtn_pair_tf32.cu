// Pair-kernel instantiations, TF32 mode (one kind::tf32 pass).
#include "rtn_pair_launch.cuh"
#include "rtn_pingpong.cuh"
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
  using Cfg = PairCfg<512, 8, 1, 24, kTF32, false>;
  auto kern = rtn_quad_kernel<8, 24>;
  static bool attr_set = false;
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

cudaError_t LaunchPingPongTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid,
                               cudaStream_t st) {
  using Cfg = PingCfg<4, 4, 80>;
  auto kern = rtn_pingpong_kernel<4, 4, 80>;
  static bool attr_set = false;
  if (!attr_set) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

cudaError_t LaunchRowsTF32(const KParams& prm, const CUtensorMap& th, const CUtensorMap& tl, int grid, cudaStream_t st) {
  using Cfg = RowsCfg<6>;
  auto kern = prm.act == 0 ? rtn_rows_kernel<6, 0> : (prm.act == 1 ? rtn_rows_kernel<6, 1> : rtn_rows_kernel<6, 2>);
  static bool attr_set[3] = {false, false, false};
  const int a = prm.act < 0 || prm.act > 2 ? 2 : prm.act;
  if (!attr_set[a]) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set[a] = true;
  }
  kern<<<grid, kThreads, Cfg::kSmemBytes, st>>>(prm, th, tl);
  return cudaGetLastError();
}

// Geometry for every mode lives here (host-only logic).
PairGeom PairGeometry(int mode, int wp, bool latency, int n_in) {
  if (latency) return {1, 24};
  const int ntc = (mode == k3xTF32 && wp == 512) ? 40 : 80;
  int p = mode == kTF32 ? 16 : 4;
  while (p > 1 && p * (1 + n_in) > ntc) p >>= 1;
  return {p, ntc};
}

}  // namespace rtn
