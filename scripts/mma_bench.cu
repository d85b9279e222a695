// Microbenchmarks for the design decisions of the fused kernel (not product):
//  (1) raw tcgen05 kind::tf32 rate, operands resident in smem, per N
//  (2) TMA-bulk-fed pipeline: producer streams 16 KB weight blocks from an
//      L2-resident buffer into NSTAGE stages, MMA warp consumes (4 MMAs per
//      stage), no epilogue — cycles per stage vs NSTAGE and N.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_07747_b200/csrc scripts/mma_bench.cu -o mma_bench
#include <cstdio>
#include <vector>

#include "rtn_kernel.cuh"

using namespace rtn;

__global__ void __launch_bounds__(128, 1) raw_mma(int n, int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 256 * 128);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (16384 + 256 * 128) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (threadIdx.x < 32) tmem_alloc(slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  if (threadIdx.x < 32) {
    const uint64_t a = sw128_desc(smem_u32(sm));
    const uint64_t b = sw128_desc(smem_u32(sm + 16384));
    const uint32_t id = idesc_tf32(128, n);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_tf32_warp(tm, a + 2 * kk, b + 2 * kk, id, 1);
    mma_commit_warp(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

template <int NS>
__global__ void __launch_bounds__(128, 1) pipe_mma(const uint8_t* w, int nblocks_total, int n, int stages_to_run,
                                                   unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act = sm;                       // 256 rows x 128 B
  uint8_t* st = sm + 256 * 128;            // NS x 16 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(st + NS * kStageBytes);
  uint64_t* empty = full + NS;
  uint64_t* done = empty + NS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<float*>(act)[i] = 0.0f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_alloc(slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *slot;
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = l2_evict_last_policy();
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_to_run; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      const int blk = (blockIdx.x * 7 + i) % nblocks_total;
      bulk_g2s_warp(st + s * kStageBytes, w + static_cast<size_t>(blk) * kStageBytes, kStageBytes, &full[s], pol);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    const uint32_t id = idesc_tf32(128, n);
    const uint64_t b = sw128_desc(smem_u32(act));
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_to_run; ++i) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const uint64_t a = sw128_desc(smem_u32(st + s * kStageBytes));
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_tf32_warp(tm, a + 2 * kk, b + 2 * kk, id, 1);
      mma_commit_warp(&empty[s]);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    mma_commit_warp(done);
    mbar_wait(done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tm, 512); }
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int NS>
int run_pipe(const uint8_t* w, int nblk, int n, int grid, unsigned long long* d_cyc) {
  const int smem = 1024 + 256 * 128 + NS * kStageBytes + 256;
  if (smem > 232448) return 0;
  CK(cudaFuncSetAttribute(pipe_mma<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int stages = 4000;
  pipe_mma<NS><<<grid, 128, smem>>>(w, nblk, n, stages, d_cyc);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned long long> c(grid);
  CK(cudaMemcpy(c.data(), d_cyc, grid * 8, cudaMemcpyDeviceToHost));
  double avg = 0; for (auto v : c) avg += v; avg /= grid;
  const double ideal = 4.0 * (128.0 * n / 256.0);
  printf("pipe NS=%d N=%3d grid=%3d: %7.1f cyc/stage (ideal %5.1f) -> %5.1f%% of MMA floor\n", NS, n, grid,
         avg / stages, ideal, 100.0 * ideal / (avg / stages));
  return 0;
}

int main() {
  unsigned long long* d_cyc;
  CK(cudaMalloc(&d_cyc, 148 * 8));
  const int smem = 1024 + 16384 + 256 * 128 + 64;
  CK(cudaFuncSetAttribute(raw_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int n : {16, 32, 64, 72, 80, 128, 144, 192, 256}) {
    const int iters = 2000;
    raw_mma<<<148, 128, smem>>>(n, iters, d_cyc);
    CK(cudaDeviceSynchronize());
    unsigned long long c;
    CK(cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost));
    const double per = double(c) / (iters * 4);
    printf("raw tf32 M=128 N=%3d: %6.1f cyc/MMA (floor %5.1f) -> %5.1f%%  (%.0f MAC/cyc/SM)\n", n, per,
           128.0 * n / 256.0, 100.0 * (128.0 * n / 256.0) / per, 128.0 * n * 8 / per);
  }
  const int nblk = 704;  // 11.5 MB of weights, L2 resident
  uint8_t* w;
  CK(cudaMalloc(&w, static_cast<size_t>(nblk) * kStageBytes));
  CK(cudaMemset(w, 0, static_cast<size_t>(nblk) * kStageBytes));
  for (int n : {72, 144}) {
    run_pipe<2>(w, nblk, n, 148, d_cyc);
    run_pipe<3>(w, nblk, n, 148, d_cyc);
    run_pipe<4>(w, nblk, n, 148, d_cyc);
    run_pipe<6>(w, nblk, n, 148, d_cyc);
    run_pipe<8>(w, nblk, n, 148, d_cyc);
    run_pipe<10>(w, nblk, n, 148, d_cyc);
    run_pipe<3>(w, nblk, n, 1, d_cyc);
    run_pipe<8>(w, nblk, n, 1, d_cyc);
  }
  return 0;
}
