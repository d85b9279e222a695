// rtn_quad.cuh — latency kernel on 4-CTA clusters (two CTA pairs), order 1,
// TF32, bf16x3 or 3xTF32 (MODE; hi/lo operand split as in rtn_pair.cuh, 3
// passes; 3xTF32 with the main pass rotating over PairCfg::kChains = 4
// accumulators by K-chunk and the corrections in a fifth, rtn_pair.cuh).
//
// Why: at one MPC step (K = N nodes) the pair kernel gives each 2-node
// cluster the WHOLE weight stream; every SM pushes ~5.8 MB of 12x512 weights
// through its shared-memory port twice (TMA write + MMA read), which sets the
// per-step latency. Here a cluster of four CTAs holds the same two nodes:
//   pair p = ranks {2p, 2p+1} computes 256-neuron block p of every hidden
//   layer (M = 256 pair MMA, N = 2 x 24 rows), so each SM streams half the
//   weights and runs one epilogue block per layer instead of two.
// Activations: CTA c produces next-layer K-group c (neurons 128c..128c+127)
// and its epilogue half h writes node h's rows into BOTH CTAs holding node h
// (ranks h and h+2; one of them may be itself), i.e. an all-to-all over DSMEM.
// Synchronisation (all mbarriers):
//   full/empty[s]  per pair: TMA bytes on the pair leader, empty multicast to the pair
//   act_ready[g]   at both leaders (ranks 0, 2): 8 warp arrivals from CTA g per layer
//   in_free[g]     at all four CTAs: one commit from EACH pair's leader (count 2)
//   tmem_full      the pair's own block accumulated (multicast to the pair)
//   tmem_last      pair 0's output layer accumulated
// Pair p walks the K-groups starting at its own (2p, 2p+1), so its first
// act_ready wait also proves its TMEM block was drained by its epilogue.
// One tile (2 nodes) per cluster: used for K <= 2 * (#SMs / 4).
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"
#include "rtn_pair.cuh"

namespace rtn {

// 4 tf32 K-steps + multicast commit of `bar` to `mask` (+ `bar2` to `mask2` if non-zero).
__device__ __forceinline__ void mma4_tf32_pair_commit_m(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                        uint32_t accumulate, uint32_t bar, uint32_t mask,
                                                        uint32_t bar2, uint32_t mask2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b16 m, m2;\n\t"
      "cvt.u16.u32 m, %7;\n\tcvt.u16.u32 m2, %8;\n\t"
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
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], m2;\n\t}" ::"r"(
          d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar), "r"(bar2), "r"(mask), "r"(mask2)
      : "memory");
}
// The same for kind::f16 (single-pass bf16; K = 16 per MMA, same descriptor steps).
__device__ __forceinline__ void mma4_bf16_pair_commit_m(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                                        uint32_t accumulate, uint32_t bar, uint32_t mask,
                                                        uint32_t bar2, uint32_t mask2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t.reg .b16 m, m2;\n\t"
      "cvt.u16.u32 m, %7;\n\tcvt.u16.u32 m2, %8;\n\t"
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
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%6], m2;\n\t}" ::"r"(
          d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar), "r"(bar2), "r"(mask), "r"(mask2)
      : "memory");
}
// bf16x3 chunk (rtn_pair.cuh RTN_MMA12 with D2 == D) with masked multicast commits:
// the two weight stages' empty barriers to `mask`, and `bar2` (if non-zero) to `mask2`.
__device__ __forceinline__ void mma12_bf16_pair_commit_m(uint32_t d, uint64_t a_hi, uint64_t a_lo, uint64_t b_hi,
                                                         uint64_t b_lo, uint32_t idesc, uint32_t accumulate,
                                                         uint32_t bar0, uint32_t bar1, uint32_t mask, uint32_t bar2,
                                                         uint32_t mask2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q;\n\t.reg .b64 x, y;\n\t.reg .b16 m, m2;\n\t"
      "cvt.u16.u32 m, %9;\n\tcvt.u16.u32 m2, %11;\n\t"
      "setp.ne.b32 p, %6, 0;\n\tsetp.eq.b32 t, 0, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %5, p;\n\t"
      "add.s64 x, %1, 2;\n\tadd.s64 y, %3, 2;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %1, 4;\n\tadd.s64 y, %3, 4;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %1, 6;\n\tadd.s64 y, %3, 6;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %4, %5, t;\n\t"
      "add.s64 x, %1, 2;\n\tadd.s64 y, %4, 2;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %1, 4;\n\tadd.s64 y, %4, 4;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %1, 6;\n\tadd.s64 y, %4, 6;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, t;\n\t"
      "add.s64 x, %2, 2;\n\tadd.s64 y, %3, 2;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %2, 4;\n\tadd.s64 y, %3, 4;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "add.s64 x, %2, 6;\n\tadd.s64 y, %3, 6;\n\t@e tcgen05.mma.cta_group::2.kind::f16 [%0], x, y, %5, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%7], m;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], m;\n\t"
      "and.pred q, q, e;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%10], m2;\n\t}" ::"r"(d),
      "l"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accumulate), "r"(bar0), "r"(bar1), "r"(mask),
      "r"(bar2), "r"(mask2)
      : "memory");
}

// 3xTF32 chunk with separate accumulators (rtn_pair.cuh RTN_MMA12): hi·hi into
// d, hi·lo + lo·hi into d2; `accumulate` bit 0 = d's first K-step accumulates,
// bit 1 = d2's. Masked multicast commits as mma12_bf16_pair_commit_m.
__device__ __forceinline__ void mma12_tf32_pair_commit_m(uint32_t d, uint32_t d2, uint64_t a_hi, uint64_t a_lo,
                                                         uint64_t b_hi, uint64_t b_lo, uint32_t idesc,
                                                         uint32_t accumulate, uint32_t bar0, uint32_t bar1,
                                                         uint32_t mask, uint32_t bar2, uint32_t mask2) {
  asm volatile(
      "{\n\t.reg .pred p, e, t, q, c;\n\t.reg .b64 x, y;\n\t.reg .b16 m, m2;\n\t.reg .b32 r;\n\t"
      "cvt.u16.u32 m, %10;\n\tcvt.u16.u32 m2, %12;\n\t"
      "and.b32 r, %7, 1;\n\tsetp.ne.b32 p, r, 0;\n\tand.b32 r, %7, 2;\n\tsetp.ne.b32 c, r, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\tsetp.ne.b32 q, %11, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %2, %4, %6, p;\n\t"
      "add.s64 x, %2, 2;\n\tadd.s64 y, %4, 2;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%0], x, y, %6, t;\n\t"
      "add.s64 x, %2, 4;\n\tadd.s64 y, %4, 4;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%0], x, y, %6, t;\n\t"
      "add.s64 x, %2, 6;\n\tadd.s64 y, %4, 6;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%0], x, y, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], %2, %5, %6, c;\n\t"
      "add.s64 x, %2, 2;\n\tadd.s64 y, %5, 2;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "add.s64 x, %2, 4;\n\tadd.s64 y, %5, 4;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "add.s64 x, %2, 6;\n\tadd.s64 y, %5, 6;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%1], %3, %4, %6, t;\n\t"
      "add.s64 x, %3, 2;\n\tadd.s64 y, %4, 2;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "add.s64 x, %3, 4;\n\tadd.s64 y, %4, 4;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "add.s64 x, %3, 6;\n\tadd.s64 y, %4, 6;\n\t@e tcgen05.mma.cta_group::2.kind::tf32 [%1], x, y, %6, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%8], m;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%9], m;\n\t"
      "and.pred q, q, e;\n\t"
      "@q tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%11], m2;\n\t}" ::"r"(d),
      "r"(d2), "l"(a_hi), "l"(a_lo), "l"(b_hi), "l"(b_lo), "r"(idesc), "r"(accumulate), "r"(bar0), "r"(bar1),
      "r"(mask), "r"(bar2), "r"(mask2)
      : "memory");
}

__device__ __forceinline__ void mma_commit_mask(uint64_t* bar, uint32_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b16 m;\n\t"
      "cvt.u16.u32 m, %1;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(mask)
      : "memory");
}

template <int NSTAGE, int NTC, int MODE = kTF32>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreads, 1)
    rtn_quad_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                    const __grid_constant__ CUtensorMap tmap_l) {
  constexpr int WP = 512, P = 1;
  using C = PairCfg<WP, NSTAGE, P, NTC, MODE, 0>;
  // one 256-neuron block per CTA: main chains at c·kN, corrections at kCorrOff (< 256 columns)
  static_assert((C::kChains + (C::kCorr ? 1 : 0)) * C::kN <= 256, "quad TMEM allocation");
  // tf32: 16 chunks of 32 k, 4 per group; bf16: 8 chunks of 64 k, 2 per group; 4 groups
  constexpr int NKC = C::kNKC, CPG = C::kCPG, NG = C::kNG, SPLIT = C::kSplit, EB = C::kEB;
  static_assert(NG == 4 && (NKC * SPLIT) % NSTAGE == 0, "quad kernel: width 512, whole stage rings per layer");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act_s = smem;
  uint8_t* stage_s = smem + C::kStageOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act_ready = bars + 2 * NSTAGE;
  uint64_t* in_free = act_ready + 4;
  uint64_t* tmem_full = in_free + 4;
  uint64_t* tmem_last = tmem_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pr = static_cast<int>(rank) >> 1;    // pair index = 256-neuron block
  const int sub = static_cast<int>(rank) & 1;    // half of the pair's M
  const bool leader = sub == 0;
  const uint32_t pair_mask = 3u << (2 * pr);
  const int n_in = prm.n_in, ntc = prm.nt;
  const int n_mma_layers = prm.n_hidden - 1;
  const long long node0 = static_cast<long long>(blockIdx.x >> 2) * 2;
  // this epilogue thread's input element, read before the setup (a PCIe round
  // trip with zero-copy latency calls; it overlaps barrier init, TMEM
  // allocation and the cluster barrier)
  double z_first = 0.0;
  if (threadIdx.x >= 128 && static_cast<int>(threadIdx.x) - 128 < 2 * n_in) {
    const int e = static_cast<int>(threadIdx.x) - 128, p = e / n_in;
    if (node0 + p < prm.K) z_first = load_z(prm, node0 + p, e - p * n_in);
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int g = 0; g < 4; ++g) {
      mbar_init(&act_ready[g], 8);  // one elected arrive per epilogue warp of CTA g
      mbar_init(&in_free[g], 2);    // one commit from each pair
      mbar_init(&tmem_full[g], 1);
    }
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_h);
    prefetch_tmap(&tmap_l);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 256);
  pdl_launch_dependents();
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer: this CTA's 128 rows of block pr ====
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    // split modes stream the hi tile then the lo tile of each chunk (lo rows at prm.lo_rows)
    for (int l = 0; l < n_mma_layers; ++l) {
      const int y = l * WP + pr * 256 + sub * 128;
#pragma unroll
      for (int i = 0; i < NKC * SPLIT; ++i) {
        const int c = (i / SPLIT + 2 * pr * CPG) % NKC, sp = i % SPLIT, st = i % NSTAGE;  // rotated K order
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * kStageBytes);
        tma_load_2sm(stage_s + st * kStageBytes, &tmap_h, c * C::kCK, y + sp * prm.lo_rows, &full[st], pol);
        if (st == NSTAGE - 1) ph ^= 1;
      }
    }
    if (pr == 0) {
#pragma unroll
      for (int i = 0; i < NKC * SPLIT; ++i) {
        const int c = i / SPLIT, sp = i % SPLIT, st = i % NSTAGE;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * kLastHalfBytes);
        tma_load_2sm(stage_s + st * kStageBytes, &tmap_l, c * C::kCK, sp * 16 + sub * 8, &full[st], pol);
        if (st == NSTAGE - 1) ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (pair leaders: ranks 0 and 2) ======
    if (leader) {
      const uint32_t idesc_h = IsBf16Mode(MODE) ? idesc_bf16(256, 2 * ntc) : idesc_tf32(256, 2 * ntc);
      const uint32_t idesc_o = IsBf16Mode(MODE) ? idesc_bf16(256, kMaxOut) : idesc_tf32(256, kMaxOut);
      const uint64_t a0 = sw128_desc(smem_u32(stage_s));
      const uint64_t b0 = sw128_desc(smem_u32(act_s));
      constexpr uint32_t kStageD = kStageBytes >> 4, kChunkD = C::kChunkStride >> 4, kSplitD = C::kSplitStride >> 4;
      uint32_t ph = 0, ar = 0;
      // one chunk: weights from stage st0 (hi) [and st0 + 1 (lo)], activations chunk c (hi [, lo])
      // i: position of the chunk in this layer's issue order (split accumulators, 3xTF32)
      auto chunk = [&](int st0, int c, int i, uint32_t idesc, uint32_t acc, uint32_t bar2, uint32_t mask2,
                       bool weights_are_a) {
        const uint64_t wa = a0 + st0 * kStageD, xa = b0 + c * kChunkD;
        if constexpr (MODE == k3xTF32) {
          const uint64_t wb = wa + kStageD, xb = xa + kSplitD;
          // hidden layers: chains c·kN, corrections kCorrOff; output layer: 16·c, 16·kChains
          const uint32_t cs = weights_are_a ? C::kN : 16u, co = weights_are_a ? C::kCorrOff : 16u * C::kChains;
          const uint32_t dm = tmem_base + (i % C::kChains) * cs;
          const uint32_t flags = (i >= C::kChains ? 1u : 0u) | (i != 0 ? 2u : 0u);
          (void)acc;
          if (weights_are_a)
            mma12_tf32_pair_commit_m(dm, tmem_base + co, wa, wb, xa, xb, idesc, flags, smem_u32(&empty[st0]),
                                     smem_u32(&empty[st0 + 1]), pair_mask, bar2, mask2);
          else
            mma12_tf32_pair_commit_m(dm, tmem_base + co, xa, xb, wa, wb, idesc, flags, smem_u32(&empty[st0]),
                                     smem_u32(&empty[st0 + 1]), pair_mask, bar2, mask2);
        } else if constexpr (MODE == kTF32) {
          if (weights_are_a)
            mma4_tf32_pair_commit_m(tmem_base, wa, xa, idesc, acc, smem_u32(&empty[st0]), pair_mask, bar2, mask2);
          else
            mma4_tf32_pair_commit_m(tmem_base, xa, wa, idesc, acc, smem_u32(&empty[st0]), pair_mask, bar2, mask2);
        } else if constexpr (MODE == kBF16) {
          if (weights_are_a)
            mma4_bf16_pair_commit_m(tmem_base, wa, xa, idesc, acc, smem_u32(&empty[st0]), pair_mask, bar2, mask2);
          else
            mma4_bf16_pair_commit_m(tmem_base, xa, wa, idesc, acc, smem_u32(&empty[st0]), pair_mask, bar2, mask2);
        } else {
          const uint64_t wb = wa + kStageD, xb = xa + kSplitD;
          if (weights_are_a)
            mma12_bf16_pair_commit_m(tmem_base, wa, wb, xa, xb, idesc, acc, smem_u32(&empty[st0]),
                                     smem_u32(&empty[st0 + 1]), pair_mask, bar2, mask2);
          else
            mma12_bf16_pair_commit_m(tmem_base, xa, xb, wa, wb, idesc, acc, smem_u32(&empty[st0]),
                                     smem_u32(&empty[st0 + 1]), pair_mask, bar2, mask2);
        }
      };
      for (int l = 0; l < n_mma_layers; ++l) {
#pragma unroll
        for (int i = 0; i < NKC; ++i) {
          const int c = (i + 2 * pr * CPG) % NKC, st = (i * SPLIT) % NSTAGE, g = c / CPG;
          if (i == 0) {  // own groups first: inputs ready AND this pair's TMEM block drained
            mbar_wait_cluster(&act_ready[2 * pr], ar & 1);
            mbar_wait_cluster(&act_ready[2 * pr + 1], ar & 1);
            tc_fence_after();
          } else if ((i % CPG) == 0 && g != 2 * pr + 1) {
            mbar_wait_cluster(&act_ready[g], ar & 1);
            tc_fence_after();
          }
          mbar_wait(&full[st], ph);
          if constexpr (SPLIT == 2) mbar_wait(&full[st + 1], ph);
          tc_fence_after();
          const bool last_of_group = (c % CPG) == CPG - 1;
          chunk(st, c, i, idesc_h, i != 0, last_of_group ? smem_u32(&in_free[g]) : 0u, 0xFu, true);
          if (st + SPLIT - 1 == NSTAGE - 1) ph ^= 1;
        }
        mma_commit_mask(&tmem_full[0], pair_mask);
        ++ar;
      }
      if (pr == 0) {  // output layer: D[row, o] = Σ_k X[row, k]·W_L'[o, k]; M = 2 x 128 rows, N = 16
#pragma unroll
        for (int i = 0; i < NKC; ++i) {
          const int st = (i * SPLIT) % NSTAGE;
          if ((i % CPG) == 0) {
            mbar_wait_cluster(&act_ready[i / CPG], ar & 1);
            tc_fence_after();
          }
          mbar_wait(&full[st], ph);
          if constexpr (SPLIT == 2) mbar_wait(&full[st + 1], ph);
          tc_fence_after();
          chunk(st, i, i, idesc_o, i != 0, 0u, 0u, false);
          if (st + SPLIT - 1 == NSTAGE - 1) ph ^= 1;
        }
        mma_commit_mask(tmem_last, pair_mask);
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: 8 warps, half h = node h's rows ==========
    const int half = (warp - 4) >> 2;
    const int q = warp & 3;
    const int tid_h = q * 32 + lane;
    const int etid = threadIdx.x - 128;
    const int act = prm.act;
    const int rows_used = P * (1 + n_in);
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const int u = ((tid_h * EB) >> 4) & 7;
    int swz[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) swz[i] = ((u ^ i) - u) * 16 + i * 128;
    // node h lives in ranks h and h + 2
    const uint32_t act_local = smem_u32(act_s);
    const uint32_t dst0 = mapa(act_local, static_cast<uint32_t>(half));
    const uint32_t dst1 = mapa(act_local, static_cast<uint32_t>(half + 2));
    const uint32_t ready0 = mapa(smem_u32(&act_ready[rank]), 0), ready2 = mapa(smem_u32(&act_ready[rank]), 2);
    const int grp = static_cast<int>(rank);  // K-group this CTA produces

    auto store_side = [&](const float* v, int j) {
      const uint32_t off = (j / C::kCK) * C::kChunkStride + (((j % C::kCK) * EB) >> 4 << 4) + ((j * EB) & 15);
#pragma unroll
      for (int i = 0; i < NTC; ++i) {
        if ((i & ~7) >= ntc) continue;
        const uint32_t a = off + (i >> 3) * 1024 + swz[i & 7];
        if constexpr (MODE == kTF32) {
          const float h = to_tf32(v[i]);
          st_cluster_f32(dst0 + a, h);
          st_cluster_f32(dst1 + a, h);
        } else if constexpr (MODE == kBF16) {
          const uint16_t h = bf16_rn_bits(v[i]);
          st_cluster_u16(dst0 + a, h);
          st_cluster_u16(dst1 + a, h);
        } else if constexpr (MODE == k3xTF32) {  // tf32 hi and lo
          const float h = to_tf32(v[i]), lo = to_tf32(v[i] - h);
          st_cluster_f32(dst0 + a, h);
          st_cluster_f32(dst1 + a, h);
          st_cluster_f32(dst0 + a + C::kSplitStride, lo);
          st_cluster_f32(dst1 + a + C::kSplitStride, lo);
        } else {  // bf16 hi and lo (rtn_pair.cuh store_side)
          const uint16_t h = bf16_rn_bits(v[i]);
          const uint16_t lo = bf16_rn_bits(v[i] - bf16_to_f32(h));
          st_cluster_u16(dst0 + a, h);
          st_cluster_u16(dst1 + a, h);
          st_cluster_u16(dst0 + a + C::kSplitStride, lo);
          st_cluster_u16(dst1 + a + C::kSplitStride, lo);
        }
      }
    };
    auto publish = [&]() {
      fence_proxy_async_cluster();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive_cluster(ready0);
        mbar_arrive_cluster(ready2);
      }
    };
    const long long node = node0 + half;
    if (etid < 2 * n_in) {
      const int p = etid / n_in;
      zs[etid] = node0 + p < prm.K ? static_cast<float>(z_first) : 0.0f;
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    // ---- layer 0 (CUDA cores): this CTA produces K-group `rank` for both nodes
    {
      const int j = grp * 128 + tid_h;
      float w0[kMaxIn0];
      load_w0_row(prm.w0t, WP, j, n_in, w0);
      float val, sp;
      act_fwd(act, layer0_pre(__ldg(prm.b0 + j), w0, zs + half * n_in, n_in), val, sp);
      float v[NTC];
#pragma unroll
      for (int i = 0; i < NTC; ++i) v[i] = i == 0 ? val : (i < rows_used ? sp * w0[(i - 1) % kMaxIn0] : 0.0f);
      store_side(v, j);
      publish();
    }
    // ---- hidden layers: one block per CTA per layer
    for (int l = 0; l < n_mma_layers; ++l) {
      const int j = pr * 256 + sub * 128 + tid_h;  // == grp * 128 + tid_h
      const float bj = __ldg(prm.bh + l * WP + j);
      mbar_wait_sleep(&tmem_full[0], l & 1);
      tc_fence_after();
      float v[NTC];
      tmem_read_acc<C, NTC>(tmem_base + lane_base + half * ntc, v, ntc, C::kN, C::kCorrOff);
      tc_fence_before();
      float val, sp;
      act_fwd(act, v[0] + bj, val, sp);
      v[0] = val;
#pragma unroll
      for (int i = 1; i < NTC; ++i) v[i] = i < rows_used ? v[i] * sp : 0.0f;
      mbar_wait_sleep(&in_free[grp], l & 1);  // both pairs consumed group grp of this layer's input
      store_side(v, j);
      publish();
    }
    // ---- output layer (pair 0): row r of this CTA's side in TMEM lane r, outputs in columns 0..15
    if (pr == 0 && half == 0) {
      mbar_wait_sleep(tmem_last, 0);
      tc_fence_after();
      float o[16];
      tmem_read_acc<C, 16>(tmem_base + lane_base, o, 16, 16u, 16u * C::kChains);
      const int r = tid_h, n_out = prm.n_out;
      const long long nd = node0 + sub;
      if (nd < prm.K) {
        note_nonfinite(prm, o, n_out);
        if (r == 0) {
          for (int oo = 0; oo < n_out; ++oo) prm.f[nd * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
        } else if (r < rows_used && prm.jac != nullptr) {
          for (int oo = 0; oo < n_out; ++oo) prm.jac[(nd * n_out + oo) * n_in + (r - 1)] = static_cast<double>(o[oo]);
        }
      }
      tc_fence_before();
    }
    (void)node;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 256);
  }
}

}  // namespace rtn
