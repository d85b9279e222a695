// Microbenchmarks for the design decisions of the fused kernel (not product):
//  (1) raw tcgen05 kind::tf32 rate, operands resident in smem, per N
//  (2) TMA-bulk-fed pipeline: producer streams 16 KB weight blocks from an
//      L2-resident buffer into NSTAGE stages, MMA warp consumes (4 MMAs per
//      stage), no epilogue — cycles per stage vs NSTAGE and N.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_07747_b200/csrc scripts/mma_bench.cu -o mma_bench
#include <cstdio>
#include <vector>
#include <cstdlib>

#include <cuda.h>
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

// (3) TMA-only stream: no MMA, consumer just frees stages. Bytes/cycle/SM ingress.
template <int NS>
__global__ void __launch_bounds__(64, 1) tma_only(const uint8_t* w, int nblk, int stages, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * kStageBytes);
  uint64_t* empty = full + NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = l2_evict_last_policy();
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      const int blk = (blockIdx.x * 7 + i) % nblk;
      bulk_g2s_warp(sm + s * kStageBytes, w + static_cast<size_t>(blk) * kStageBytes, kStageBytes, &full[s], pol);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&full[s], ph);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      __syncwarp();
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
  }
}

// (4) TMA tensor-map tile loads (2-D, box 32 x 128 fp32, SWIZZLE_128B), 1-SM.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], 16384;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;\n\t}"
      ::"r"(smem_u32(dst)), "l"(tmap), "r"(smem_u32(bar)), "r"(x), "r"(y), "l"(pol) : "memory");
}
template <int NS>
__global__ void __launch_bounds__(64, 1) tma_tensor_only(const __grid_constant__ CUtensorMap tm, int nrowblk, int stages,
                                                        unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NS * kStageBytes);
  uint64_t* empty = full + NS;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = l2_evict_last_policy();
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      const int blk = (blockIdx.x * 7 + i) % (nrowblk * 16);
      tma_load_2d(sm + s * kStageBytes, &tm, (blk % 16) * 32, (blk / 16) * 128, &full[s], pol);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else {
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&full[s], ph);
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      __syncwarp();
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x] = t1 - t0;
  }
}

// (5) CTA-pair stream: 2-SM TMA (each CTA its 128-row half) + leader pair MMAs,
//     N = 2 x rows_per_cta, no epilogue. Cycles per 16 KB/CTA stage.
template <int NS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    pair_pipe(const __grid_constant__ CUtensorMap tm, int rows_per_cta, int stages, unsigned long long* cyc, int lockstep, int variant = 0) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act = sm;  // 80 rows x 128 B
  uint8_t* st = sm + 80 * 128 + 6144;
  st = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(st) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + NS * kStageBytes);
  uint64_t* empty = full + NS;
  uint64_t* done = empty + NS;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 80 * 128 / 4; i += blockDim.x) reinterpret_cast<float*>(act)[i] = 0.0f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_alloc_pair(slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmb = *slot;
  const int warp = threadIdx.x >> 5;
  long long t0 = clock64();
  if (warp == 0) {
    const uint64_t pol = l2_evict_last_policy();
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&empty[s], ph ^ 1);
      if (rank == 0) mbar_expect_tx_elect(&full[s], 2 * kStageBytes);
      const int blk = ((lockstep ? 0 : (blockIdx.x >> 1) * 7) + i) % (22 * 16);
      // variant bit 1: real-kernel walk (layer, 256-block, k chunk) over 11 x 512 rows
      const int c = i % 16, mb = (i / 16) % 2, l = (i / 32) % 11;
      if (variant & 1) tma_load_2sm(st + s * kStageBytes, &tm, c * 32, l * 512 + mb * 256 + rank * 128, &full[s], pol);
      else tma_load_2sm(st + s * kStageBytes, &tm, (blk % 16) * 32, (blk / 16) * 256 + rank * 128, &full[s], pol);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
  } else if (warp == 1 && rank == 0) {
    const uint32_t id = idesc_tf32(256, 2 * rows_per_cta);
    const uint64_t b = sw128_desc(smem_u32(act));
    int s = 0; uint32_t ph = 0;
    for (int i = 0; i < stages; ++i) {
      mbar_wait(&full[s], ph);
      tc_fence_after();
      const int c = i % 16, mb = (i / 16) % 2;
      const uint32_t d = (variant & 2) ? tmb + mb * 160 : tmb;       // bit 2: alternate TMEM regions
      const uint32_t acc = (variant & 4) ? (c != 0) : 1;              // bit 4: accumulate reset per block
      mma4_tf32_pair_commit(d, sw128_desc(smem_u32(st + s * kStageBytes)), b, id, acc, smem_u32(&empty[s]), 0);
      if (++s == NS) { s = 0; ph ^= 1; }
    }
    mma_commit_pair(done);
    mbar_wait(done, 0);
    long long t1 = clock64();
    if (threadIdx.x == 32) cyc[blockIdx.x >> 1] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) { tc_fence_after(); tmem_dealloc_pair(tmb, 512); }
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
  const int fill = getenv("BENCH_FILL") ? atoi(getenv("BENCH_FILL")) : 0;
  CK(cudaMemset(w, fill, static_cast<size_t>(nblk) * kStageBytes));
  printf("weight buffer byte fill 0x%02x\n", fill);
  for (int grid : {1, 20, 74, 148}) {
    constexpr int NS = 8;
    const int smem = 1024 + NS * kStageBytes + 256;
    CK(cudaFuncSetAttribute(tma_only<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int stages = 4000;
    tma_only<NS><<<grid, 64, smem>>>(w, nblk, stages, d_cyc);
    CK(cudaDeviceSynchronize());
    std::vector<unsigned long long> c(grid);
    CK(cudaMemcpy(c.data(), d_cyc, grid * 8, cudaMemcpyDeviceToHost));
    double avg = 0; for (auto v : c) avg += v; avg /= grid;
    printf("tma-only NS=%d grid=%3d: %6.1f cyc per 16 KB stage = %5.1f B/cyc/SM\n", NS, grid, avg / stages,
           16384.0 / (avg / stages));
  }
  {
    // tensor map over the same 11.5 MB buffer viewed as [44*128 rows x 512 fp32]
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    CUtensorMap tm{};
    const cuuint64_t dims[2] = {512, 44 * 128};
    const cuuint64_t str[1] = {512 * 4};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t es[2] = {1, 1};
    for (auto l2 : {CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_L2_PROMOTION_NONE}) {
      reinterpret_cast<Fn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int grid : {1, 20, 148}) {
        constexpr int NS = 8;
        const int smem = 1024 + NS * kStageBytes + 256;
        CK(cudaFuncSetAttribute(tma_tensor_only<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        tma_tensor_only<NS><<<grid, 64, smem>>>(tm, 44, 4000, d_cyc);
        CK(cudaDeviceSynchronize());
        std::vector<unsigned long long> c(grid);
        CK(cudaMemcpy(c.data(), d_cyc, grid * 8, cudaMemcpyDeviceToHost));
        double avg = 0; for (auto v : c) avg += v; avg /= grid;
        printf("tma-tensor(32x128 fp32 sw128, l2promo %d) NS=8 grid=%3d: %6.1f cyc/16KB = %5.1f B/cyc/SM\n", (int)l2, grid,
               avg / 4000, 16384.0 / (avg / 4000));
      }
    }
  }
  {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    CUtensorMap tm{};
    const cuuint64_t dims[2] = {512, 44 * 128};
    const cuuint64_t str[1] = {512 * 4};
    const cuuint32_t box[2] = {32, 128};
    const cuuint32_t es[2] = {1, 1};
    reinterpret_cast<Fn>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, w, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int threads = 384;
    const int lockstep = 1;
    for (int variant : {0, 1, 2, 4, 7})
    for (int rows : {24}) {
      for (int grid : {20}) {
        auto run = [&](auto kern, int ns) -> int {
          const int smem = 1024 + 80 * 128 + 6144 + 1024 + ns * kStageBytes + 256;
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          kern<<<grid, threads, smem>>>(tm, rows, 4000, d_cyc, lockstep, variant);
          CK(cudaDeviceSynchronize());
          std::vector<unsigned long long> c(grid / 2);
          CK(cudaMemcpy(c.data(), d_cyc, (grid / 2) * 8, cudaMemcpyDeviceToHost));
          double avg = 0; for (auto v : c) avg += v; avg /= (grid / 2);
          const double floor = 4.0 * 256.0 * 2 * rows / 512.0;
          printf("variant %d ", variant);
          printf("pair-pipe rows/cta=%2d (N=%3d) NS=%d grid=%3d: %6.1f cyc/stage (math floor %5.1f, smem floor %5.1f)\n",
                 rows, 2 * rows, ns, grid, avg / 4000, floor, 4.0 * (4096 + 32.0 * rows) / 128);
          return 0;
        };
        run(pair_pipe<8>, 8);
      }
    }
  }
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
