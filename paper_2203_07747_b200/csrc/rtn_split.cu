// Split-kernel instantiations (TF32, width 512; rtn_split.cuh), one
// translation unit so it compiles in parallel with the pair kernels.
#include <cstdio>

#include "rtn_launch.h"
// #define RTN_SPLIT_DEBUG 1  // bounded waits + progress stamps (RTN_TRACE_HOST) for hang hunting
#include "rtn_reverse.cuh"
#include "rtn_rowsb.cuh"
#include "rtn_split.cuh"

#ifndef SPLIT_NS
#define SPLIT_NS 4
#endif

namespace rtn {

cudaError_t LaunchSplitTF32(const KParams& prm, const CUtensorMap& th64, const CUtensorMap& tl, int grid,
                            cudaStream_t st) {
  using Cfg = SplitCfg<SPLIT_NS>;
  auto kern = prm.act == 0 ? rtn_split_kernel<SPLIT_NS, 0> : (prm.act == 1 ? rtn_split_kernel<SPLIT_NS, 1> : rtn_split_kernel<SPLIT_NS, 2>);
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kSplitThreads, Cfg::kSmemBytes, st>>>(prm, th64, tl);
  return cudaGetLastError();
}

cudaError_t LaunchReverse(int pass, const KParams& prm, const CUtensorMap& ta, const CUtensorMap& tb, int grid,
                          cudaStream_t st) {
  using Cfg = RevCfg<4>;
  auto pick = [&](auto k0, auto k1, auto k2) { return prm.act == 0 ? k0 : (prm.act == 1 ? k1 : k2); };
  auto kern = pass == 0 ? pick(rtn_rev_kernel<4, 0, 0>, rtn_rev_kernel<4, 1, 0>, rtn_rev_kernel<4, 2, 0>)
                        : pick(rtn_rev_kernel<4, 0, 1>, rtn_rev_kernel<4, 1, 1>, rtn_rev_kernel<4, 2, 1>);
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kRevThreads, Cfg::kSmemBytes, st>>>(prm, ta, tb);
  return cudaGetLastError();
}

cudaError_t LaunchRowsBF16(const KParams& prm, const CUtensorMap& th64, const CUtensorMap& tl, int grid,
                           cudaStream_t st) {
  using Cfg = RowsBCfg<8>;
  auto kern = prm.act == 0 ? rtn_rowsb_kernel<8, 0> : (prm.act == 1 ? rtn_rowsb_kernel<8, 1> : rtn_rowsb_kernel<8, 2>);
  const cudaError_t e = EnsureSmem(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, kRbThreads, Cfg::kSmemBytes, st>>>(prm, th64, tl);
  return cudaGetLastError();
}

}  // namespace rtn
