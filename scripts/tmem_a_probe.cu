// Probe (not product): pair tcgen05.mma kind::tf32 with the A operand in TMEM
// (rows = TMEM lanes, k = columns) and B (weights, K-major SW128) in shared
// memory. Checks the layout against a CPU product and compares the MMA rate
// with the A-from-shared-memory form, for the "activations as A in TMEM"
// kernel design.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2203_07747_b200/csrc \
//        scripts/tmem_a_probe.cu -o scripts/tmem_a_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rtn_kernel.cuh"

using namespace rtn;

__host__ __device__ inline float aval(int row, int k) { return static_cast<float>((row * 7 + k * 3) % 11 - 5) * 0.25f; }
__host__ __device__ inline float bval(int n, int k) { return static_cast<float>((n * 5 + k * 13) % 9 - 4) * 0.5f; }

__device__ __forceinline__ void mma_tf32_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mode 0: A from TMEM; mode 1: A from smem. reps: K=32 passes accumulated. n: MMA N (per pair).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(int mode, int reps, int n, float* out, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bs = sm;           // 128 neurons x 32 k (16 KB)
  uint8_t* as = sm + 16384;   // 128 rows x 32 k (16 KB), mode 1
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 32768);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 32768 + 64);
  const uint32_t rank = cluster_rank();
  const int t = threadIdx.x, warp = t >> 5;
  if (t == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_pair(slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *slot;
  const int row = static_cast<int>(rank) * 128 + t;
  // A: lane t, columns 256 + k (and the same values in smem for mode 1)
  float a[32];
  for (int k = 0; k < 32; ++k) a[k] = aval(row, k);
  const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
  for (int k = 0; k < 32; k += 8) tmem_st8(tbase + lane_off + 256 + k, a + k);
  tmem_st_wait();
  for (int k = 0; k < 32; ++k) {
    *reinterpret_cast<float*>(as + sw128_offset(t, k, 0)) = a[k];
    *reinterpret_cast<float*>(bs + sw128_offset(t, k, 0)) = bval(static_cast<int>(rank) * 128 + t, k);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  unsigned long long t0 = clock64();
  if (rank == 0 && warp == 0) {
    const uint32_t id = idesc_tf32(256, n);
    const uint64_t bd = sw128_desc(smem_u32(bs)), ad = sw128_desc(smem_u32(as));
    if ((t & 31) == 0) {
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          if (mode == 0) mma_tf32_pair_ts(tbase, tbase + 256 + 8 * ks, bd + 2 * ks, id, (r | ks) != 0);
          else mma_tf32_pair_ss(tbase, ad + 2 * ks, bd + 2 * ks, id, (r | ks) != 0);
        }
    }
    __syncwarp();
    mma_commit_pair(bar);
  }
  mbar_wait(bar, 0);
  tc_fence_after();
  unsigned long long t1 = clock64();
  if (t == 0) cyc[rank] = t1 - t0;
  for (int c = 0; c < n; c += 8) {
    float v[8];
    tmem_ld8(tbase + lane_off + c, v);
    tmem_ld_wait();
    for (int i = 0; i < 8; ++i) out[static_cast<size_t>(row) * 256 + c + i] = v[i];
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc_pair(tbase, 512);
  }
}

int main() {
  float* d_out;
  unsigned long long* d_cyc;
  cudaMalloc(&d_out, 256 * 256 * sizeof(float));
  cudaMalloc(&d_cyc, 2 * sizeof(unsigned long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  std::vector<float> h(256 * 256);
  for (int n : {256, 128}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int reps : {1, 2000}) {
        cudaMemset(d_out, 0, 256 * 256 * sizeof(float));
        probe<<<2, 128, 40 * 1024>>>(mode, reps, n, d_out, d_cyc);
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("mode %d reps %d: %s\n", mode, reps, cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h.data(), d_out, h.size() * sizeof(float), cudaMemcpyDeviceToHost);
        unsigned long long cyc[2];
        cudaMemcpy(cyc, d_cyc, sizeof(cyc), cudaMemcpyDeviceToHost);
        double maxerr = 0.0;
        int bad = 0;
        for (int m = 0; m < 256; ++m)
          for (int j = 0; j < n; ++j) {
            // B columns 0..n/2-1 come from CTA 0's smem, n/2..n-1 from CTA 1's
            const int ng = j < n / 2 ? j : 128 + (j - n / 2);
            double s = 0.0;
            for (int k = 0; k < 32; ++k) s += static_cast<double>(aval(m, k)) * bval(ng, k);
            s *= reps;
            const double err = std::abs(s - h[m * 256 + j]);
            if (err > maxerr) maxerr = err;
            if (err > 1e-3 && bad++ < 3) printf("  mismatch D[%d][%d] = %g, want %g\n", m, j, h[m * 256 + j], s);
          }
        const double per_k8 = static_cast<double>(cyc[0]) / (4.0 * reps);
        printf("N=%d %s reps %4d: max err %.3g, %llu cycles (%.1f per K=8 MMA; floor M*N/256/2 = %d)\n", n,
               mode == 0 ? "A=TMEM" : "A=SMEM", reps, maxerr, cyc[0], per_k8, 128 * n / 256);
      }
    }
  }
  return 0;
}
