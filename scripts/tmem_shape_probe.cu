// Probe (not product): which TMEM (lane, column) each thread receives from
// tcgen05.ld.16x256b.x1 (4 regs) — layout check for the rows kernel's value-row reads.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_07747_b200/csrc scripts/tmem_shape_probe.cu -o scripts/tmem_shape_probe
#include <cstdio>
#include "rtn_kernel.cuh"
using namespace rtn;
__global__ void k(float* out) {
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  float v[8];
  for (int c = 0; c < 8; ++c) v[c] = t * 1000.0f + c;  // lane t (warp w -> lanes 32w..)
  tmem_st8(tb + (static_cast<uint32_t>(warp * 32) << 16), v);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(tb));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[t * 4 + 0] = __uint_as_float(r0); out[t * 4 + 1] = __uint_as_float(r1);
    out[t * 4 + 2] = __uint_as_float(r2); out[t * 4 + 3] = __uint_as_float(r3);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 32); }
}
int main() {
  float* d; cudaMalloc(&d, 128 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
  float h[128]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  for (int t = 0; t < 32; ++t) printf("t%2d: %6.0f %6.0f %6.0f %6.0f\n", t, h[t*4], h[t*4+1], h[t*4+2], h[t*4+3]);
  return 0;
}
