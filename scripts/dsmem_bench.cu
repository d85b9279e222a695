// dsmem_bench.cu — throughput of the ways an epilogue can move a tile of
// activations into the peer CTA's shared memory (design evidence for the pair
// kernel's epilogue, rtn_pair.cuh): 256 threads of each CTA of a 2-CTA cluster
// write `bytes` into the peer's smem as
//   0: st.shared::cluster.f32   (32 lanes -> 128 contiguous bytes, the kernel's pattern)
//   1: st.shared::cluster.v4.f32 (32 lanes -> 512 contiguous bytes)
//   2: st.shared.f32 into local staging, then one cp.async.bulk.shared::cluster.shared::cta
//   3: st.shared.f32 local only (reference)
//   4/5: st.async(.v4).b32 to the peer, completion counted on the peer's mbarrier
// and report cycles per KB (max over the two CTAs, median over clusters).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

constexpr int kBytes = 36 * 1024;  // one 4-chunk group of 72 rows (the pair kernel's remote share per block)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024, 1) bench(int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* dst = smem;               // the peer writes here
  uint8_t* stage = smem + kBytes;    // local staging (mode 2)
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * kBytes);
  const uint32_t rank = cluster_rank(), peer = rank ^ 1;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync();
  const uint32_t rdst = mapa(smem_u32(dst), peer);
  const float v = threadIdx.x * 1.0f;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (mode == 0) {
      for (int off = threadIdx.x * 4; off < kBytes; off += blockDim.x * 4)
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(rdst + off), "f"(v) : "memory");
      asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
    } else if (mode == 1) {
      for (int off = threadIdx.x * 16; off < kBytes; off += blockDim.x * 16)
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(rdst + off), "f"(v) : "memory");
      asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
    } else if (mode == 2) {
      for (int off = threadIdx.x * 4; off < kBytes; off += blockDim.x * 4)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_u32(stage) + off), "f"(v) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        // the copy signals complete_tx on the PEER's barrier; the peer waits for its bytes
        const uint32_t rbar = mapa(smem_u32(bar), peer);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         rdst),
                     "r"(smem_u32(stage)), "r"(kBytes), "r"(rbar)
                     : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(kBytes)
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(bar)),
            "r"(r & 1)
            : "memory");
      }
      __syncthreads();
    } else if (mode == 3) {
      for (int off = threadIdx.x * 4; off < kBytes; off += blockDim.x * 4)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(smem_u32(dst) + off), "f"(v) : "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    } else {
      // st.async: remote stores completing on the PEER's mbarrier (complete_tx)
      const uint32_t rbar = mapa(smem_u32(bar), peer);
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(kBytes)
                     : "memory");
      if (mode == 4) {
        for (int off = threadIdx.x * 4; off < kBytes; off += blockDim.x * 4)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(rdst + off),
                       "r"(__float_as_uint(v)), "r"(rbar)
                       : "memory");
      } else {
        for (int off = threadIdx.x * 16; off < kBytes; off += blockDim.x * 16)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(
                           rdst + off),
                       "r"(__float_as_uint(v)), "r"(rbar)
                       : "memory");
      }
      if (threadIdx.x == 0)
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                smem_u32(bar)),
            "r"(r & 1)
            : "memory");
      __syncthreads();
    }
    cluster_sync();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  const int clusters = 74, reps = 200;
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 2 * clusters);
  const int smem = 2 * kBytes + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"st.shared::cluster.f32", "st.shared::cluster.v4.f32", "local st + cp.async.bulk to peer",
                         "st.shared.f32 local only", "st.async.b32 (complete_tx)", "st.async.v4.b32 (complete_tx)"};
  for (int threads : {256, 512})
  for (int mode = 0; mode < 6; ++mode) {
    bench<<<2 * clusters, threads, smem>>>(mode, reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<long long> h(2 * clusters);
    cudaMemcpy(h.data(), d, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost);
    std::vector<long long> mx(clusters);
    for (int c = 0; c < clusters; ++c) mx[c] = std::max(h[2 * c], h[2 * c + 1]);
    std::sort(mx.begin(), mx.end());
    const double cyc = static_cast<double>(mx[clusters / 2]);
    std::printf("%4d threads %-36s %8.0f cycles per %d KB (incl. cluster barrier)  %6.1f B/clk\n", threads, names[mode], cyc,
                kBytes / 1024, kBytes / cyc);
  }
  return 0;
}
