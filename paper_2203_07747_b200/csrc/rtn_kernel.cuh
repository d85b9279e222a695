// rtn_kernel.cuh — fused forward-mode linearisation kernel for sm_100a.
//
// What it computes (per node = one shooting node of one MPC instance):
//   f = out_scale ⊙ net((z − in_mean) ⊘ in_scale) + out_mean,   J = ∂f/∂z
// i.e. the reference's BatchedCore value + Jacobian
// (/root/reference/proj/src/neural.cpp:227-255), but by forward-mode tangent
// propagation instead of the reference's stacked reverse sweep (:132-163):
// every node carries 1 value row + n_in tangent rows through the network, and
// because all nodes share the weights, each hidden layer is ONE dense GEMM
//   D[neuron, row] = Σ_k W[neuron, k] · X[row, k]
// over (nodes × (1+n_in)) rows, on tcgen05 tensor cores (kind::tf32).
//
// Orientation ("swap-AB"): A = weights (M = 128 neurons per block, streamed by
// the TMA bulk engine from a pre-swizzled device pack), B = activations
// (N = tile rows, resident in shared memory for the whole network), D in TMEM
// (lane = neuron, column = row). The epilogue owns one neuron per thread and
// all rows of a tile, so the activation slope scaling of the tangent rows
// (t' = σ'(pre_value)·t) is thread-local. Activations never leave the SM:
// layer l+1 reads what layer l's epilogue wrote back into shared memory.
//
// Layer 0 (n_in → width) runs on CUDA cores: its tangent seed is the identity,
// so the tangent rows after layer 0 are σ'(pre)·W0'[:, k] — no GEMM needed.
// The output layer (width → n_out ≤ 16) runs as a second tcgen05 shape
// (M = 128 tile rows, N = 16 outputs, A = activations, B = W_L').
//
// Pipelines (all mbarrier based; one thread issues TMA, one issues MMA):
//   full/empty[s]   producer ↔ MMA over the weight stage ring
//   tmem_full[g]    MMA → epilogue: neuron block g of the layer is accumulated
//   in_free[g]      MMA → epilogue: the layer's last M-block has consumed
//                   input chunk group g, so the epilogue may overwrite it
//   act_ready[g]    epilogue → MMA: next-layer input group g is in smem
//   tmem_last       MMA → epilogue: output layer accumulated
// With this ordering the epilogue of block g overlaps the MMAs of later
// blocks, and the next layer starts on group 0 while group NMB-1 is still
// being written.
#pragma once

#include <cstdint>

namespace rtn {

constexpr int kStageBytes = 16384;  // one weight stage: 128 neurons x 128 bytes of k
constexpr int kThreads = 384;       // 4 control warps + 8 epilogue warps
constexpr int kMaxOut = 16;

// Precision modes (rtn_pair.cuh): tf32, 3xtf32, bf16x3 and single-pass bf16.
enum : int { kTF32 = 0, k3xTF32 = 1, kBF16x3 = 2, kBF16 = 3 };
__host__ __device__ constexpr bool IsBf16Mode(int mode) { return mode == kBF16x3 || mode == kBF16; }
__host__ __device__ constexpr bool IsSplitMode(int mode) { return mode == k3xTF32 || mode == kBF16x3; }

struct KParams {
  const double* z;   // K x n_in
  double* f;         // K x n_out
  double* jac;       // K x n_out x n_in (may be null for order 0)
  double* hess;      // K x n_out x n_in x n_in (order 2 only)
  long long K;
  long long num_tiles;
  int n_in, n_out, n_hidden, act, order;
  int P;             // nodes per tile (power of two)
  int nt;            // tile rows used (= roundup8(P·(1+n_in))), MMA N
  int lo_rows;       // pair kernel split modes: row offset of the lo weight tiles in the stacked map
  int ord2_g;        // order 2: pair tiles per node (Hessian slot groups)
  unsigned long long* trace;  // optional event timestamps (RTN_TRACE), pair 0 only
  int trace_tile;    // which of pair 0's tiles is traced (RTN_TRACE = 1 + index)
  int dbg;           // perf-isolation switches (RTN_DEBUG): 4 = skip epilogue math, 8 = local stores, 128 = stream only
  const double* mu;  // n_in: in_mean, subtracted in fp64 before the fp32 layer 0
  unsigned int* nonfinite;  // host-mapped flag: set when a written f/J/H value is NaN or Inf
  const float* w0;   // WP x n_in   (W0·diag(1/in_scale)), neuron-major (rows kernel staging)
  const float* w0t;  // n_in x WP   the same, input-major: a warp's 32 neurons read 128 contiguous bytes
  const float* b0;   // WP          (the layer-0 bias; the mean is NOT folded in)
  const float* bh;   // (n_hidden-1) x WP
  const float* bl;   // kMaxOut     (out_scale ⊙ b_L + out_mean)
  // Gather mode (rtn_cycle_qp, 'full' variant): when zx != null, row k is the
  // quadrotor feature vector [x_k; u_k] (ResidualInput 'full', dynamics.cpp:137-139)
  // read straight from the iterate: zx = Iterate::xs (n_inst x (N+1) x 13),
  // zu = us (K x 4). Other variants stage their features with FeaturesKernel.
  const double* zx;
  const double* zu;
  int zN;
  // reverse mode (rtn_reverse.cuh): σ'_l of every node, [n_hidden][K][512] fp32,
  // written by the value pass and read by the adjoint pass; W_L' rows (fp32)
  float* rev_s;
  const float* wl;
};

// Layer-0 weight row of neuron j in registers (n_in <= kMaxIn0 for every tile
// shape), from the input-major copy: coalesced across the warp's neurons.
constexpr int kMaxIn0 = 24;
__device__ __forceinline__ void load_w0_row(const float* w0t, int wp, int j, int n_in, float (&w)[kMaxIn0]) {
#pragma unroll
  for (int k = 0; k < kMaxIn0; ++k) w[k] = k < n_in ? __ldg(w0t + k * wp + j) : 0.0f;
}
// pre = b + Σ_k W0'[j,k]·z[k], ascending k (same rounding as the loop it replaces).
__device__ __forceinline__ float layer0_pre(float b, const float (&w)[kMaxIn0], const float* z, int n_in) {
  float pre = b;
#pragma unroll
  for (int k = 0; k < kMaxIn0; ++k)
    if (k < n_in) pre = fmaf(w[k], z[k], pre);
  return pre;
}

// Element k of node row `node` of the MLP input, centred in fp64: z_k − in_mean_k.
// The reference normalises in fp64 before the first layer
// (proj/src/neural.cpp:107-109); folding the mean into the fp32 layer-0 bias
// instead (b0 − W0'·μ) cancels catastrophically for inputs far from zero
// relative to in_scale, so only the 1/in_scale scaling is folded into W0'.
// address of the raw (uncentred) element k of node z
__device__ __forceinline__ const double* z_ptr(const KParams& prm, long long node, int k) {
  if (prm.zx == nullptr) return prm.z + node * prm.n_in + k;
  const long long xrow = node + node / prm.zN;  // inst·(N+1) + n
  return k < 13 ? prm.zx + xrow * 13 + k : prm.zu + node * 4 + (k - 13);
}
__device__ __forceinline__ double load_z_raw(const KParams& prm, long long node, int k) { return *z_ptr(prm, node, k); }
__device__ __forceinline__ double load_z(const KParams& prm, long long node, int k) {
  return load_z_raw(prm, node, k) - __ldg(prm.mu + k);
}

// Per-call NaN/Inf flag: a thread about to write the outputs o[0..n)
// of one row raises the context's flag if any of them is not finite.
__device__ __forceinline__ void note_nonfinite(const KParams& prm, const float* o, int n) {
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kMaxOut; ++i)
    if (i < n) bad |= !isfinite(o[i]);
  if (bad && prm.nonfinite != nullptr) atomicOr(prm.nonfinite, 1u);
}

// ----------------------------------------------------------------------------
// PTX wrappers

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Lets a programmatic dependent launch (the fused cycle's blocks kernel) be
// scheduled now; it still waits for this grid's completion before reading its
// outputs (griddepcontrol.wait). A no-op when nothing was launched that way.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Long-suspend wait for threads with nothing else to do (epilogue warps
// waiting on the tensor core): the hint lets the scheduler park the warp until
// the phase completes instead of re-polling, keeping issue slots free for the
// producer and MMA warps that share the sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

// TMA bulk copy global → shared, completion signalled on an mbarrier;
// weights are re-read by every SM, so keep them resident in L2.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

// D[tmem] (+)= A[smem] · B[smem]ᵀ, both K-major, tf32 in, fp32 accumulate.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Warp-converged variant: every lane computes the (uniform) operands, one
// elected lane issues. Keeping the warp converged lets ptxas hold the
// descriptors in uniform registers instead of wrapping each UTCHMMA in a
// per-lane uniformity loop.
__device__ __forceinline__ void mma_tf32_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
// Warp-converged producer step: one elected lane arms the barrier and issues
// the bulk copy.
__device__ __forceinline__ void bulk_g2s_warp(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n\t}" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Arrives on `bar` once every previously issued tcgen05.mma of this thread
// has completed (implicitly fences before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
// CW-column TMEM access built from x8 pieces (CW ∈ {8, 16}).
template <int CW>
__device__ __forceinline__ void tmem_ld_cw(uint32_t taddr, float* v) {
#pragma unroll
  for (int i = 0; i < CW; i += 8) tmem_ld8(taddr + i, v + i);
}
template <int CW>
__device__ __forceinline__ void tmem_st_cw(uint32_t taddr, const float* v) {
#pragma unroll
  for (int i = 0; i < CW; i += 8) tmem_st8(taddr + i, v + i);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// fp32 → tf32 round-to-nearest (ties away), as cvt.rna.tf32.f32 but in two
// integer ops: the hardware cvt is emulated with an extra Inf/NaN guard the
// epilogue does not need (activations and tangents are finite).
__device__ __forceinline__ float to_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups
// 1024 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;           // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO
  d |= static_cast<uint64_t>(1) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;           // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

// Byte offset of element (row r, k) inside a K-major SW128 operand whose
// 32-wide k chunks are `chunk_stride` bytes apart.
__host__ __device__ __forceinline__ uint32_t sw128_offset(int r, int k, uint32_t chunk_stride) {
  const int c = k >> 5, u = (k >> 2) & 7;
  return static_cast<uint32_t>(c) * chunk_stride + static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128 +
                                                                         ((u ^ (r & 7)) << 4) + ((k & 3) << 2));
}

// Activation value and slope from the pre-activation, fp32
// (tanh/relu: proj/src/neural.cpp:83-93; SiLU: x·σ(x), σ(1 + x(1−σ))).
__device__ __forceinline__ void act_fwd(int act, float pre, float& val, float& sp) {
  if (act == 0) {
    const float t = tanhf(pre);
    val = t;
    sp = 1.0f - t * t;
  } else if (act == 1) {
    val = pre > 0.0f ? pre : 0.0f;
    sp = pre > 0.0f ? 1.0f : 0.0f;
  } else {
    // σ with the accurate expf (the fast __expf's error grows with |x| and is
    // amplified through deep nets; this runs only on value rows) and an IEEE
    // reciprocal; exp(−x) → ∞ for x ≪ 0 gives σ = 0 exactly, matching the limit.
    const float s = __frcp_rn(1.0f + expf(-pre));
    val = pre * s;
    sp = s * (1.0f + pre * (1.0f - s));
  }
}

// act_fwd for the reverse value pass, where every row is a value row and the
// IEEE reciprocal was ~30% of the pass's instructions: the same accurate expf,
// then an approximate division (<= 2 ulp; σ ∈ (0, 1))
__device__ __forceinline__ void act_fwd_rows(int act, float pre, float& val, float& sp) {
  if (act == 2) {
    const float s = __fdividef(1.0f, 1.0f + expf(-pre));
    val = pre * s;
    sp = s * (1.0f + pre * (1.0f - s));
  } else {
    act_fwd(act, pre, val, sp);
  }
}

}  // namespace rtn

// ============================================================================
// CTA-pair (cta_group::2) primitives for the throughput kernel (rtn_pair.cuh)
namespace rtn {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Shared-memory address of the same object in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Arrive (release, cluster scope) on an mbarrier given by its shared::cluster address.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Remote arrive with the default (.release.cta) semantics, as CUTLASS's
// ClusterBarrier::arrive(cta_id): for TMEM reads, which the tcgen05 fences
// around the barrier order, the cluster-scope release (MEMBAR) of
// mbar_arrive_cluster is not needed.
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_cluster() {
  asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

// Pair MMA (issued by the leader CTA only): A is M-split and B is N-split
// across the two CTAs' shared memory at the same offsets; each CTA's TMEM
// receives its 128 rows of D.
__device__ __forceinline__ void mma_tf32_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit to the mbarrier at the same offset in both CTAs of the pair.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 2-SM TMA tile load: lands in this CTA's smem, transaction bytes counted on
// the LEADER CTA's barrier (peer bit of the barrier address cleared).
__device__ __forceinline__ void tma_load_2sm(void* dst, const void* tmap, int x, int y, uint64_t* bar,
                                             uint64_t policy) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;\n\t}" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(mbar), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_elect(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

}  // namespace rtn

namespace rtn {
// One weight stage of a pair MMA layer in a single asm block: 4 K-steps
// (32 B each: tf32 K=8) with one elect, then a multicast commit of the stage's
// empty barrier (and, if `bar2` is non-zero, a second barrier such as in_free
// or tmem_full). Keeping the 4 MMAs + commit together lets ptxas convert the
// operands to uniform registers once per stage instead of once per MMA.
__device__ __forceinline__ void mma4_tf32_pair_commit(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                      uint32_t accumulate, uint32_t bar, uint32_t bar2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a1, b1, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a2, b2, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], a3, b3, %3, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], m;\n\t"
      "and.pred q, q, e;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], m;\n\t}" ::"r"(
          d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar), "r"(bar2)
      : "memory");
}
}  // namespace rtn

namespace rtn {
// mma4_tf32_pair_commit for kind::f16 (bf16 operands, K = 16 per MMA = the
// same 32 bytes of each operand row, so the descriptor steps are identical).
__device__ __forceinline__ void mma4_bf16_pair_commit(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                      uint32_t accumulate, uint32_t bar, uint32_t bar2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "setp.ne.b32 q, %6, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], m;\n\t"
      "and.pred q, q, e;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], m;\n\t}" ::"r"(
          d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar), "r"(bar2)
      : "memory");
}

// Split-operand pair MMA step (3xTF32 / BF16x3): with A = A_hi + A_lo and
// B = B_hi + B_lo, D += A_hi·B_hi and D2 += A_hi·B_lo + A_lo·B_hi (the lo·lo
// term is below the representation error). 3 passes x 4 K-steps of 32 bytes,
// one elect, then multicast commits of the two weight stages (and bar2 if set).
// `accumulate`: bit 0 for D's first K-step, bit 1 for D2's (set both when
// D2 == D, which folds the correction into the main accumulator: bf16x3). A separate
// D2 (3xTF32) keeps the ~2^-11-sized corrections from being added to the large
// running sum: the tensor core's fp32 accumulation drops up to an ulp of the
// running sum per MMA, and 128 correction MMAs per 512-deep layer made that the
// dominant error; the epilogue adds D + D2 once in fp32.
#define RTN_MMA12(KIND)                                                                                              \
  asm volatile(                                                                                                    \
      "{\n\t.reg .pred p, e, t, q, c;\n\t.reg .b64 x, y;\n\t.reg .b16 m;\n\t.reg .b32 r;\n\t"                     \
      "mov.b16 m, 3;\n\tand.b32 r, %7, 1;\n\tsetp.ne.b32 p, r, 0;\n\tand.b32 r, %7, 2;\n\tsetp.ne.b32 c, r, 0;\n\t" \
      "setp.eq.b32 t, 0, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t"                                                    \
      "elect.sync _|e, 0xffffffff;\n\t"                                                                           \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], %1, %3, %6, p;\n\t"                                      \
      "add.s64 x, %1, 2;\n\tadd.s64 y, %3, 2;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], x, y, %6, t;\n\t" \
      "add.s64 x, %1, 4;\n\tadd.s64 y, %3, 4;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], x, y, %6, t;\n\t" \
      "add.s64 x, %1, 6;\n\tadd.s64 y, %3, 6;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%0], x, y, %6, t;\n\t" \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], %1, %4, %6, c;\n\t"                                      \
      "add.s64 x, %1, 2;\n\tadd.s64 y, %4, 2;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "add.s64 x, %1, 4;\n\tadd.s64 y, %4, 4;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "add.s64 x, %1, 6;\n\tadd.s64 y, %4, 6;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], %2, %3, %6, t;\n\t"                                      \
      "add.s64 x, %2, 2;\n\tadd.s64 y, %3, 2;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "add.s64 x, %2, 4;\n\tadd.s64 y, %3, 4;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "add.s64 x, %2, 6;\n\tadd.s64 y, %3, 6;\n\t@e tcgen05.mma.cta_group::2.kind::" KIND " [%5], x, y, %6, t;\n\t" \
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], m;\n\t"  \
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%9], m;\n\t"  \
      "and.pred q, q, e;\n\t"                                                                                     \
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%10], m;\n\t}" \
      ::"r"(d_tmem), "l"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(d2_tmem), "r"(idesc), "r"(accumulate), "r"(bar0),     \
      "r"(bar1), "r"(bar2)                                                                                       \
      : "memory")

__device__ __forceinline__ void mma12_tf32_pair_commit(uint32_t d_tmem, uint32_t d2_tmem, uint64_t a_hi, uint64_t a_lo,
                                                       uint64_t b_hi, uint64_t b_lo, uint32_t idesc, uint32_t accumulate,
                                                       uint32_t bar0, uint32_t bar1, uint32_t bar2) {
  RTN_MMA12("tf32");
}
__device__ __forceinline__ void mma12_bf16_pair_commit(uint32_t d_tmem, uint32_t d2_tmem, uint64_t a_hi, uint64_t a_lo,
                                                       uint64_t b_hi, uint64_t b_lo, uint32_t idesc, uint32_t accumulate,
                                                       uint32_t bar0, uint32_t bar1, uint32_t bar2) {
  RTN_MMA12("f16");
}
#undef RTN_MMA12

// Instruction descriptor: D f32, A/B bf16, both K-major (kind::f16).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void st_shared_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u16(uint32_t addr, uint16_t v) {
  asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
// bf16 round-to-nearest-even of a finite fp32, and back.
__device__ __forceinline__ uint16_t bf16_rn_bits(float x) {
  const uint32_t u = __float_as_uint(x);
  return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}
__device__ __forceinline__ float bf16_to_f32(uint16_t h) { return __uint_as_float(static_cast<uint32_t>(h) << 16); }
}  // namespace rtn

namespace rtn {
// ---- second order (Hessian rows) -------------------------------------------
// Packed upper-triangle index p of the pair (a, b), a ≤ b, over n inputs:
// p = 0 → (0,0), 1 → (0,1), …, n-1 → (0,n-1), n → (1,1), …
struct PairAB {
  int a, b;
};
__host__ __device__ constexpr PairAB pair_ab(int p, int n) {
  int a = 0;
  while (p >= n - a) {
    p -= n - a;
    ++a;
  }
  return PairAB{a, a + p};
}
constexpr int kMaxIn2 = 31;                       // order 2, generic tiles: 1 + n_in carrier rows <= 32
constexpr int kNin2 = 17;                         // order-2 specialised tiles: quadrotor inputs
constexpr int kPairs2 = kNin2 * (kNin2 + 1) / 2;  // 153 packed Hessian rows per node
constexpr int kCarrier2 = 1 + kNin2;              // value + tangent rows carried by every tile
constexpr int kNtc2 = 48;                         // rows per CTA side in order-2 tiles
constexpr int kSlots2 = 2 * kNtc2 - kCarrier2;    // 78 Hessian rows per tile → 2 tiles per node

// Order-2 tile plan for n_in inputs and NTC rows per CTA side: the carrier
// (value + n_in tangents) sits in side-0 rows [0, 1+n_in); the other
// 2·NTC − (1+n_in) rows are Hessian slots; a node takes ceil(pairs / slots) tiles.
__host__ __device__ constexpr int ord2_slots(int n_in, int ntc) { return 2 * ntc - (1 + n_in); }
__host__ __device__ constexpr int ord2_tiles(int n_in, int ntc) {
  return (n_in * (n_in + 1) / 2 + ord2_slots(n_in, ntc) - 1) / ord2_slots(n_in, ntc);
}

// Activation value, slope and curvature (second-order tangents need σ'').
__device__ __forceinline__ void act_fwd2(int act, float pre, float& val, float& sp, float& spp) {
  if (act == 0) {
    const float t = tanhf(pre);
    val = t;
    sp = 1.0f - t * t;
    spp = -2.0f * t * sp;
  } else {
    const float s = __frcp_rn(1.0f + expf(-pre));
    val = pre * s;
    sp = s * (1.0f + pre * (1.0f - s));
    spp = s * (1.0f - s) * (2.0f + pre * (1.0f - 2.0f * s));
  }
}
}  // namespace rtn

#include <utility>

namespace rtn {
// Second-order epilogue rows with compile-time (a, b): h' = σ'·h + σ''·T_a·T_b
// (hidden layers, T = pre-activation tangents) or h = σ''·T_a·T_b (layer 0,
// where the incoming second-order tangents are zero). P2 ≥ 153 is padding.
template <int P2>
__device__ __forceinline__ float hrow(float h, const float* T, float sp, float spp) {
  if constexpr (P2 < kPairs2) {
    constexpr PairAB ab = pair_ab(P2, kNin2);
    return fmaf(spp, T[ab.a] * T[ab.b], sp * h);
  } else {
    return 0.0f;
  }
}
template <int P2>
__device__ __forceinline__ float hrow0(const float* T, float spp) {
  if constexpr (P2 < kPairs2) {
    constexpr PairAB ab = pair_ab(P2, kNin2);
    return spp * (T[ab.a] * T[ab.b]);
  } else {
    return 0.0f;
  }
}
// v[OFF + s] for s in S...: pair index BASE + s.
template <int BASE, int OFF, int... S>
__device__ __forceinline__ void hrows(float* v, const float* T, float sp, float spp, std::integer_sequence<int, S...>) {
  ((v[OFF + S] = hrow<BASE + S>(v[OFF + S], T, sp, spp)), ...);
}
template <int BASE, int OFF, int... S>
__device__ __forceinline__ void hrows0(float* v, const float* T, float spp, std::integer_sequence<int, S...>) {
  ((v[OFF + S] = hrow0<BASE + S>(T, spp)), ...);
}
}  // namespace rtn
