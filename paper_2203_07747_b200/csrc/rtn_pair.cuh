// rtn_pair.cuh — throughput / latency kernel on CTA pairs (cta_group::2).
//
// Why pairs: a tcgen05 tf32 MMA with both operands in shared memory reads
// them at ~128 B/clk/SM, so M = 128 × N = 72 runs at 72 % of the math floor
// and, once the TMA weight stream shares the SMEM port, at ~62 %; N ≥ 128 is
// needed to be math-bound (scripts/mma_bench.cu). Fp32 activations for a
// 512-wide layer cap a single CTA at ~80 rows of smem, so the N = 144 tile is
// split over two CTAs of a cluster: one pair MMA (M = 256 neurons, N = 2·72
// rows) takes A (weights) half from each CTA and B (activations) half from
// each CTA; each CTA's TMEM receives its 128 neurons for all 144 rows.
//
// Precision modes (MODE):
//   kTF32   : one kind::tf32 pass; operands rounded to tf32 (RNA).
//   k3xTF32 : A = A_hi + A_lo, B = B_hi + B_lo (both tf32), three kind::tf32
//             passes hi·hi + hi·lo + lo·hi; fp32-grade (1e-5 class).
//   kBF16x3 : same split in bf16 (8+8 mantissa bits), three kind::f16 passes
//             at twice the tf32 rate; operand bytes equal to tf32 mode.
//   kBF16   : one kind::f16 pass on bf16 operands (8-bit mantissa): half the
//             operand bytes and twice the MMA rate of tf32, ~8x its error.
//
// 3xTF32 accumulation (PairCfg::kChains): the tensor core adds each K = 8 MMA
// into its fp32 accumulator with an error proportional to the running sum's
// ulp, so the error of a 512-deep layer grows with the number of MMAs that
// land in one accumulator (measured on B200: 192 → 64 → 32 MMAs per chain gave
// 7e-5 → 2.4e-5 → 1.2e-5 at 12x512, gain 2.5). The hi·hi pass therefore
// rotates over kChains accumulators by K-chunk (4 where TMEM allows: 16 MMAs
// per chain), the small hi·lo + lo·hi corrections go to their own accumulator,
// and the epilogue adds them once in fp32: D0 + ((D1 + D2 + D3) + Dcorr).
//
// Variant (ORD2): 0 = order 1; 1, 2 = order 2 (below); 3, 4 = the value and
// adjoint passes of reverse mode (the reference's own algorithm: rtn_reverse.cuh
// describes it; here for the split-precision and BF16 modes, whose operands do
// not fit the split kernel's TMEM/shared-memory layout).
// Order 2 (ORD2): 1 = quadrotor tiles (n_in = 17, compile-time Hessian slot
// tables, NTC = 48); 2 = generic tiles for any n_in <= 31 (runtime slot table
// in shared memory). Both carry the node's value + tangent rows (the
// "carrier") in side-0 rows [0, 1+n_in) and packed Hessian rows (a <= b) in
// every other row: h' = σ'·(W h)_ab + σ''·(W t_a)(W t_b).
//
// Data movement per layer:
//   weights    : 2-SM TMA tile loads (tensor map, SWIZZLE_128B), each CTA its
//                128-neuron half (hi and lo tiles in split modes), bytes
//                counted on the leader's barrier
//   activations: the epilogue of CTA r owns next-layer K-group q = 2·mb + r
//                and writes its rows into BOTH CTAs' operand buffers (the
//                peer's half through DSMEM, st.shared::cluster)
//   barriers   : full[s] (leader); act_ready[c] per 32-k (tf32) chunk of the
//                next layer's input (leader; one arrival per epilogue warp
//                that wrote it), so the next layer's MMAs start on a chunk as
//                soon as it is stored; tmem_empty[mb] (leader; every epilogue
//                warp of both CTAs, right after its TMEM reads), so a TMEM
//                block is reused without waiting for the stores; empty /
//                in_free / tmem_full / tmem_last multicast by the leader's
//                tcgen05.commit to both CTAs.
//   DSMEM      : the peer-side stores (~13.5 B/clk against ~40 B/clk local,
//                scripts/dsmem_bench.cu) are issued one warp after another
//                (named-barrier chain), so the first chunks of a group complete
//                early and the MMA of the next layer resumes on them while the
//                rest is in flight.
#pragma once
#include <type_traits>

#include <cuda.h>

#include "rtn_kernel.cuh"

namespace rtn {

constexpr int kLastHalfBytes = 1024;  // output layer: 8 of the 16 output rows x 128 B

// NTC = operand row stride per CTA (max rows per CTA): 80 for throughput
// tiles (P = 4 quadrotor nodes = 72 rows), 24 for latency tiles (P = 1) and
// for 3xTF32 at width 512, 48 / 24 / 40 for order-2 tiles.
template <int WP, int NSTAGE, int P, int NTC, int MODE, int ORD2 = 0>
struct PairCfg {
  static constexpr int kEB = IsBf16Mode(MODE) ? 2 : 4;  // operand element bytes
  static constexpr int kCK = 128 / kEB;                // k per 128-byte chunk row
  static constexpr int kNKC = WP / kCK;                // chunks per layer input
  static constexpr int kSplit = IsSplitMode(MODE) ? 2 : 1;  // operand buffers (hi[, lo])
  static constexpr int kCPG = 128 / kCK;               // chunks per 128-neuron K-group
  static constexpr int kNMB = WP / 256;                // 256-neuron blocks (pair M)
  static constexpr int kNG = WP / 128;                 // 128-neuron K-groups
  static constexpr int kStagesPerMB = kNKC * kSplit;
  static constexpr uint32_t kChunkStride = NTC * 128;
  static constexpr uint32_t kSplitStride = kNKC * kChunkStride;
  static constexpr uint32_t kActBytes = kSplit * kSplitStride;
  static constexpr uint32_t kStageOff = kActBytes;
  static constexpr uint32_t kBarOff = kStageOff + NSTAGE * kStageBytes;
  // full/empty[NSTAGE], act_ready[16] (per K-chunk), tmem_empty[2], in_free[4], tmem_full[2], tmem_last
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 25;
  static constexpr int kWarpsPerChunk = 2 * (kCK / 32);  // both halves of the owning CTA
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kZsOff = kMiscOff + 16;
  // generic order 2: per-thread tangent rows T_a (2 halves x 32 x 128 fp32) and the slot → (a, b) table
  static constexpr uint32_t kTsOff = (kZsOff + 2 * NTC * 4 + 15) & ~15u;
  static constexpr uint32_t kTsBytes = ORD2 == 2 ? 2 * 32 * 128 * 4 : 0;
  static constexpr uint32_t kAbOff = kTsOff + kTsBytes;
  static constexpr uint32_t kAbBytes = ORD2 == 2 ? 512 * 2 : 0;
  static constexpr uint32_t kSmemBytes = kAbOff + kAbBytes + 1024;
  // TMEM: 256-neuron block mb at column mb·kBlkCols; inside it kChains main
  // accumulators of kN = 2·NTC columns, then (3xTF32) the correction accumulator.
  static constexpr int kN = 2 * NTC;
  static constexpr bool kCorr = MODE == k3xTF32;
  static constexpr int kBlkCols = 512 / kNMB;
  static constexpr int kChains = !kCorr ? 1 : (5 * kN <= kBlkCols ? 4 : (3 * kN <= kBlkCols ? 2 : 1));
  static constexpr int kCorrOff = kChains * kN;
  static_assert(kNMB >= 1 && kNMB <= 2, "pair kernel handles 256 or 512 padded width");
  static_assert(kN % 16 == 0 && kN <= 256, "pair MMA N");
  static_assert((kChains + (kCorr ? 1 : 0)) * kN <= kBlkCols, "TMEM capacity");
  static constexpr int kOutN = ORD2 == 4 ? 32 : kMaxOut;  // output MMA N (reverse adjoint pass: J over 32 inputs)
  static_assert((kChains + (kCorr ? 1 : 0)) * kOutN <= kBlkCols, "output-layer accumulators");
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static_assert(kStagesPerMB % NSTAGE == 0, "every 256-block starts at stage 0 (static stage indices)");
  // the output layer's M = 128-row A reads run past the last chunk into the stage ring
  static_assert((128 - NTC) * 128 <= NSTAGE * kStageBytes, "A-operand overrun must stay in smem");
};

// v[0..N) = this lane's accumulator columns [t, t + N) summed over the main
// chains (t + c·kN) and the 3xTF32 correction accumulator (t + kCorrOff) —
// v = D0 + ((D1 + D2 + D3) + Dcorr) — 16 columns per round trip; columns
// >= lim are not read. `stride` is kN for hidden blocks, 16 for the output layer.
template <class C, int N>
__device__ __forceinline__ void tmem_read_acc(uint32_t t, float* v, int lim, uint32_t stride, uint32_t corr_off) {
#pragma unroll
  for (int c0 = 0; c0 < N; c0 += 8)
    if (c0 < lim) tmem_ld8(t + c0, v + c0);
  tmem_ld_wait();
  constexpr int kExtra = C::kChains - 1 + (C::kCorr ? 1 : 0);
  if constexpr (kExtra > 0) {
#pragma unroll
    for (int c0 = 0; c0 < N; c0 += 16) {
      if (c0 >= lim) break;
      float x[kExtra][16];
#pragma unroll
      for (int e = 0; e < kExtra; ++e) {
        const uint32_t te = t + (e < C::kChains - 1 ? (e + 1) * stride : corr_off) + c0;
        tmem_ld8(te, x[e]);
        if (c0 + 8 < N && c0 + 8 < lim) tmem_ld8(te + 8, x[e] + 8);
      }
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (c0 + i < N && c0 + i < lim) {
          float s = x[0][i];
#pragma unroll
          for (int e = 1; e < kExtra; ++e) s += x[e][i];
          v[c0 + i] += s;
        }
      }
    }
  }
}

__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int WP, int NSTAGE, int P, int NTC, int MODE, int ORD2 = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    rtn_pair_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                    const __grid_constant__ CUtensorMap tmap_l) {
  using C = PairCfg<WP, NSTAGE, P, NTC, MODE, ORD2>;
  static_assert(ORD2 != 1 || NTC == kNtc2, "quadrotor order-2 tiles are 2 x 48 rows");
  constexpr int NMB = C::kNMB, NKC = C::kNKC, NG = C::kNG, SPLIT = C::kSplit, CPG = C::kCPG;
  static_assert(NKC <= 16, "act_ready barriers");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act_s = smem;
  uint8_t* stage_s = smem + C::kStageOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act_ready = bars + 2 * NSTAGE;  // [16]
  uint64_t* tmem_empty = act_ready + 16;    // [2]
  uint64_t* in_free = tmem_empty + 2;       // [4]
  uint64_t* tmem_full = in_free + 4;        // [2]
  uint64_t* tmem_last = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, ntc = prm.nt;  // rows per CTA
  const int n_mma_layers = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  // This epilogue thread's element of the first tile's inputs, read before the
  // setup below: with zero-copy latency calls it is a PCIe round trip, which
  // then overlaps barrier init, TMEM allocation and the cluster barrier.
  // Order 1: raw z (centred later); order 2: centred (load_z).
  double z_first = 0.0;
  if (threadIdx.x >= 128 && pair < prm.num_tiles) {
    const int e = static_cast<int>(threadIdx.x) - 128;
    if constexpr (ORD2 != 0) {
      const long long node0 = pair / (ORD2 == 1 ? 2 : prm.ord2_g);
      if (e < n_in && node0 < prm.K) z_first = load_z(prm, node0, e);
    } else if (e < 2 * P * n_in) {
      const int zp = e / n_in, zk = e - zp * n_in;
      const long long node0 = pair * (2 * P) + zp;
      if (node0 < prm.K)
        z_first = prm.zx == nullptr ? prm.z[node0 * n_in + zk]
                                    : (zk < 13 ? prm.zx[(node0 + node0 / prm.zN) * 13 + zk]
                                               : prm.zu[node0 * 4 + (zk - 13)]);
      else
        z_first = __ldg(prm.mu + zk);
    }
  }

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < 16; ++c) mbar_init(&act_ready[c], C::kWarpsPerChunk);
    for (int mb = 0; mb < 2; ++mb) {
      mbar_init(&tmem_empty[mb], 16);  // 8 epilogue warps x 2 CTAs
      mbar_init(&tmem_full[mb], 1);
    }
    for (int g = 0; g < 4; ++g) mbar_init(&in_free[g], 1);
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_h);
    prefetch_tmap(&tmap_l);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  pdl_launch_dependents();
  if constexpr (ORD2 == 2) {  // slot → (a, b) table of the packed upper triangle
    uint16_t* ab = reinterpret_cast<uint16_t*>(smem + C::kAbOff);
    const int np = n_in * (n_in + 1) / 2;
    for (int p = threadIdx.x; p < np; p += blockDim.x) {
      const PairAB q = pair_ab(p, n_in);
      ab[p] = static_cast<uint16_t>(q.a | (q.b << 8));
    }
    __syncthreads();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const bool tr_pair = prm.trace && pair == 0;
  if (tr_pair && threadIdx.x == 0) {
    prm.trace[196 + rank] = globaltimer();
    prm.trace[250 + rank] = clock64();
  }

  if (warp == 0) {
    // ===================== weight producer: 2-SM TMA, own 128-neuron half ====
    // Chunk loops are fully unrolled: stage indices, phases and coordinates
    // are compile-time, so this single warp is not instruction-latency bound
    // at small N (scripts/mma_bench.cu variants). Split modes stream the hi
    // tile then the lo tile of each chunk (lo rows start at prm.lo_rows).
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    const int yr = static_cast<int>(rank) * 128;
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
      for (int l = 0; l < n_mma_layers; ++l)
        for (int mb = 0; mb < NMB; ++mb) {
          const int wl = ORD2 == 4 ? n_mma_layers - 1 - l : l;  // the adjoint pass walks the layers backwards
          const int y = wl * WP + mb * 256 + yr;
#pragma unroll
          for (int i = 0; i < NKC * SPLIT; ++i) {
            const int c = i / SPLIT, sp = i % SPLIT, st = i % NSTAGE;
            mbar_wait(&empty[st], ph ^ 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kStageBytes);
            tma_load_2sm(stage_s + st * kStageBytes, &tmap_h, c * C::kCK, y + sp * prm.lo_rows, &full[st], pol);
            if (st == NSTAGE - 1) ph ^= 1;
          }
        }
#pragma unroll
      for (int i = 0; i < NKC * SPLIT; ++i) {
        const int c = i / SPLIT, sp = i % SPLIT, st = i % NSTAGE;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * (C::kOutN / 2) * 128);
        tma_load_2sm(stage_s + st * kStageBytes, &tmap_l, c * C::kCK, sp * C::kOutN + static_cast<int>(rank) * (C::kOutN / 2),
                     &full[st], pol);
        if (st == NSTAGE - 1) ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) ======================
    if (leader) {
      const uint32_t idesc_h = IsBf16Mode(MODE) ? idesc_bf16(256, 2 * ntc) : idesc_tf32(256, 2 * ntc);
      const uint32_t idesc_o = IsBf16Mode(MODE) ? idesc_bf16(256, C::kOutN) : idesc_tf32(256, C::kOutN);
      // descriptors advance by (bytes >> 4) in the start-address field
      const uint64_t a0 = sw128_desc(smem_u32(stage_s));
      const uint64_t b0 = sw128_desc(smem_u32(act_s));
      constexpr uint32_t kStageD = kStageBytes >> 4, kChunkD = C::kChunkStride >> 4, kSplitD = C::kSplitStride >> 4;
      const bool stream_only = prm.dbg & 128;  // dbg 128: weight stream + MMAs only (timing)
      uint32_t ph = 0, ar = 0, use0 = 0, use1 = 0;
      // TMEM block mb is about to be overwritten: both CTAs' epilogues must have
      // read its previous contents (tmem_empty, one phase per use of the block).
      auto claim_tmem = [&](int mb) {
        const uint32_t u = mb ? use1 : use0;
        if (!stream_only && u > 0) mbar_wait(&tmem_empty[mb], (u - 1) & 1);
        if (mb) ++use1;
        else ++use0;
        tc_fence_after();
      };
      // input chunk c of the current activation production is in both CTAs' smem
      auto wait_chunk = [&](int c) {
        if (stream_only) return;
        mbar_wait_cluster(&act_ready[c], ar & 1);
        tc_fence_after();
      };
      // One chunk: weights from stage(s) st0[/st1], activations chunk (hi[, lo]).
      auto chunk_mma = [&](uint32_t d, uint32_t d2, uint64_t wa, uint64_t wb, int st0, int st1, uint64_t xa,
                           uint64_t xb, uint32_t idesc, uint32_t acc, uint32_t bar2, bool weights_are_a) {
        if constexpr (MODE == kTF32) {
          if (weights_are_a)
            mma4_tf32_pair_commit(d, wa, xa, idesc, acc, smem_u32(&empty[st0]), bar2);
          else
            mma4_tf32_pair_commit(d, xa, wa, idesc, acc, smem_u32(&empty[st0]), bar2);
        } else if constexpr (MODE == kBF16) {
          if (weights_are_a)
            mma4_bf16_pair_commit(d, wa, xa, idesc, acc, smem_u32(&empty[st0]), bar2);
          else
            mma4_bf16_pair_commit(d, xa, wa, idesc, acc, smem_u32(&empty[st0]), bar2);
        } else {
          const uint64_t ah = weights_are_a ? wa : xa, al = weights_are_a ? wb : xb;
          const uint64_t bh = weights_are_a ? xa : wa, bl = weights_are_a ? xb : wb;
          if constexpr (MODE == k3xTF32)
            mma12_tf32_pair_commit(d, d2, ah, al, bh, bl, idesc, acc, smem_u32(&empty[st0]), smem_u32(&empty[st1]),
                                   bar2);
          else
            mma12_bf16_pair_commit(d, d, ah, al, bh, bl, idesc, (acc & 1u) | 2u, smem_u32(&empty[st0]),
                                   smem_u32(&empty[st1]), bar2);
        }
      };
      // main-pass accumulator of chunk c (rotating over kChains), and the
      // accumulate flags (TF32: a bool; split modes: bit 0 main, bit 1 correction)
      auto chain_acc = [&](int c) -> uint32_t {
        if constexpr (!IsSplitMode(MODE)) return c != 0;
        else return (c >= C::kChains ? 1u : 0u) | (c != 0 ? 2u : 0u);
      };
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
        const bool tr = tr_pair && tile == pair + prm.trace_tile * npairs && lane == 0;
        for (int l = 0; l < n_mma_layers; ++l) {
#pragma unroll 1
          for (int mb = 0; mb < NMB; ++mb) {
            const uint32_t d = tmem_base + mb * C::kBlkCols;
            const uint32_t d2 = C::kCorr ? d + C::kCorrOff : d;
            if (tr) prm.trace[(l * 2 + mb) * 2] = globaltimer();
            claim_tmem(mb);
#pragma unroll
            for (int c = 0; c < NKC; ++c) {
              const int st0 = (c * SPLIT) % NSTAGE, st1 = (c * SPLIT + SPLIT - 1) % NSTAGE;
              if (mb == 0) wait_chunk(c);
              mbar_wait(&full[st0], ph);
              if constexpr (SPLIT == 2) mbar_wait(&full[st1], ph);
              tc_fence_after();
              // extra commit: in_free after the last block consumed K-group c/CPG
              const uint32_t bar2 = (mb == NMB - 1 && (c % CPG) == CPG - 1) ? smem_u32(&in_free[c / CPG]) : 0u;
              chunk_mma(d + (c % C::kChains) * C::kN, d2, a0 + st0 * kStageD, a0 + st1 * kStageD, st0, st1,
                        b0 + c * kChunkD, b0 + kSplitD + c * kChunkD, idesc_h, chain_acc(c), bar2, true);
              if (st1 == NSTAGE - 1) ph ^= 1;
            }
            mma_commit_pair(&tmem_full[mb]);
            if (tr) prm.trace[(l * 2 + mb) * 2 + 1] = globaltimer();
          }
          ++ar;
        }
        // output layer: D[row, o] = Σ_k X[row, k] · W_L'[o, k]; M = 2 x 128 rows, N = 16;
        // main chains at columns 16·c of block 0, the correction accumulator at 16·kChains
        claim_tmem(0);
#pragma unroll
        for (int c = 0; c < NKC; ++c) {
          const int st0 = (c * SPLIT) % NSTAGE, st1 = (c * SPLIT + SPLIT - 1) % NSTAGE;
          wait_chunk(c);
          mbar_wait(&full[st0], ph);
          if constexpr (SPLIT == 2) mbar_wait(&full[st1], ph);
          tc_fence_after();
          chunk_mma(tmem_base + (c % C::kChains) * C::kOutN, C::kCorr ? tmem_base + C::kOutN * C::kChains : tmem_base,
                    a0 + st0 * kStageD, a0 + st1 * kStageD, st0, st1, b0 + c * kChunkD, b0 + kSplitD + c * kChunkD,
                    idesc_o, chain_acc(c), 0u, false);
          if (st1 == NSTAGE - 1) ph ^= 1;
        }
        mma_commit_pair(tmem_last);
        if (tr) prm.trace[44] = globaltimer();
        ++ar;
      }
    }
  } else if (warp >= 4 && !(prm.dbg & 128)) {
    // ===================== epilogue (8 warps per CTA) ========================
    // Thread = one neuron (TMEM lane) of this CTA's 128-neuron half of a
    // 256-block; warp half h owns the rows of side h (the nodes whose operand
    // rows live in CTA h), i.e. TMEM columns [h·ntc, (h+1)·ntc). Results stay
    // in registers until the layer's last block has consumed the input group
    // they overwrite (in_free), then go straight to the owning CTA's shared
    // memory (DSMEM for the peer side), and each warp publishes its chunk.
    const int half = (warp - 4) >> 2;
    const int q = warp & 3;
    const int tid_h = q * 32 + lane;
    const int etid = threadIdx.x - 128;
    const int act = prm.act;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    // Row r of a K-major SW128 operand lives at  col + (r/8)·1024 + (r%8)·128
    // + ((u ^ r%8) − u)·16  relative to row 0 of this thread's neuron column,
    // with u the neuron's 16-byte unit inside its 128-byte chunk row.
    const int u = ((tid_h * C::kEB) >> 4) & 7;
    int swz[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) swz[i] = ((u ^ i) - u) * 16 + i * 128;
    const uint32_t act_local = smem_u32(act_s);
    const bool local_side = half == static_cast<int>(rank) || (prm.dbg & 8);  // dbg 8: timing only
    const uint32_t side_base = local_side ? act_local : mapa(act_local, static_cast<uint32_t>(half));
    const uint32_t ready_cl0 = mapa(smem_u32(&act_ready[0]), 0);
    const uint32_t empty_cl0 = mapa(smem_u32(&tmem_empty[0]), 0);
    uint32_t hl = 0, tiles_done = 0;
    auto trace_on = [&]() {
      return tr_pair && tiles_done == static_cast<uint32_t>(prm.trace_tile) && warp == 4 && lane == 0;
    };

    // Store one neuron column (rows 0..ntc-1) of one side into its operand
    // buffer(s), rounding / splitting per precision mode. row(i) yields the
    // value of row i (an array read, or generated on the fly at layer 0).
    auto store_to = [&](auto&& row, int j, uint32_t buf, bool local) {
      const uint32_t base =
          buf + (j / C::kCK) * C::kChunkStride + ((((j % C::kCK) * C::kEB) >> 4) << 4) + ((j * C::kEB) & 15);
#pragma unroll
      for (int i = 0; i < NTC; ++i) {
        if ((i & ~7) >= ntc) continue;
        const uint32_t a = base + (i >> 3) * 1024 + swz[i & 7];
        const float x = row(i);
        if constexpr (MODE == kTF32) {
          const float h = to_tf32(x);
          if (local) st_shared_f32(a, h);
          else st_cluster_f32(a, h);
        } else if constexpr (MODE == kBF16) {
          const uint16_t h = bf16_rn_bits(x);
          if (local) st_shared_u16(a, h);
          else st_cluster_u16(a, h);
        } else if constexpr (MODE == k3xTF32) {
          const float h = to_tf32(x);
          const float lo = to_tf32(x - h);
          if (local) {
            st_shared_f32(a, h);
            st_shared_f32(a + C::kSplitStride, lo);
          } else {
            st_cluster_f32(a, h);
            st_cluster_f32(a + C::kSplitStride, lo);
          }
        } else {
          const uint16_t h = bf16_rn_bits(x);
          const uint16_t lo = bf16_rn_bits(x - bf16_to_f32(h));
          if (local) {
            st_shared_u16(a, h);
            st_shared_u16(a + C::kSplitStride, lo);
          } else {
            st_cluster_u16(a, h);
            st_cluster_u16(a + C::kSplitStride, lo);
          }
        }
      }
    };
    auto store_side = [&](auto&& row, int j) { store_to(row, j, side_base, local_side); };
    // publishes this warp's chunk of K-group g: its stores are made visible to
    // the async proxy (the tensor core) — a CTA-scope proxy fence when they all
    // went to this CTA's shared memory, cluster scope for DSMEM stores — and
    // the leader's barrier is released at cluster scope
    auto publish_chunk = [&](int g, bool all_local) {
      if (all_local) fence_proxy_async_smem();
      else fence_proxy_async_cluster();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ready_cl0 + 8 * ((g * 128 + q * 32) / C::kCK));
    };
    // Stores, then publishes this warp's chunk of K-group g. The peer-side
    // half issues its DSMEM stores one warp after another (q = 0, 1, 2, 3
    // through a chain of named barriers), so chunk by chunk they complete
    // early instead of all at the end of the shared transfer.
    auto store_publish = [&](auto&& row, int j, int g) {
      const int c = (g * 128 + q * 32) / C::kCK;
      if (!local_side && (prm.dbg & 16)) {  // dbg 16: chain the peer-side warps (experiment)
        if (q > 0) named_bar_sync(2 + half * 3 + (q - 1), 64);
        store_side(row, j);
        if (q < 3) named_bar_arrive(2 + half * 3 + q, 64);
      } else {
        store_side(row, j);
      }
      (void)c;
      publish_chunk(g, local_side);
    };
    // this warp has read TMEM block mb (all lanes' loads complete)
    auto tmem_release = [&](int mb) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(empty_cl0 + 8 * mb);
    };
    // output-layer accumulator of this lane (row), columns = outputs
    auto read_out = [&](float* o) {
      tmem_read_acc<C, 16>(tmem_base + lane_base, o, 16, 16u, 16u * C::kChains);
    };

   if constexpr (ORD2 == 1) {
    // ===================== order-2 epilogue, quadrotor tiles ===================
    // Pair-tile t holds node t/2, Hessian group g = t%2: side 0 rows 0..17 are
    // the carrier (value + 17 tangents), side-0 rows 18..47 and side-1 rows
    // 0..47 are packed Hessian rows g·78 + slot. Every thread sees all 96
    // columns of its neuron in TMEM, so the carrier's pre-activations (value,
    // tangents T_a) are at hand for h' = σ'·H + σ''·T_a·T_b.
    using Seq0 = std::make_integer_sequence<int, kNtc2 - kCarrier2>;  // side-0 Hessian slots
    using Seq1 = std::make_integer_sequence<int, kNtc2>;              // side-1 Hessian slots
    // v: this half's 48 rows; T: carrier tangents (pre-activation); hg: Hessian group.
    auto epi_rows = [&](float* v, const float* T, float val, float sp, float spp, int hg) {
      if (half == 0) {
        v[0] = val;
#pragma unroll
        for (int a = 0; a < kNin2; ++a) v[1 + a] = sp * T[a];
        if (hg == 0) hrows<0, kCarrier2>(v, T, sp, spp, Seq0{});
        else hrows<kSlots2, kCarrier2>(v, T, sp, spp, Seq0{});
      } else {
        if (hg == 0) hrows<kNtc2 - kCarrier2, 0>(v, T, sp, spp, Seq1{});
        else hrows<kSlots2 + kNtc2 - kCarrier2, 0>(v, T, sp, spp, Seq1{});
      }
    };
    auto do_block = [&](int mb, int l, int hg) {
      const int grp = 2 * mb + static_cast<int>(rank);
      const int j = mb * 256 + static_cast<int>(rank) * 128 + tid_h;
      const float bj = __ldg(prm.bh + l * WP + j);
      const uint32_t tb = tmem_base + lane_base + mb * C::kBlkCols;
      mbar_wait_sleep(&tmem_full[mb], hl & 1);
      tc_fence_after();
      const bool tr = trace_on();
      unsigned long long* tp = tr ? prm.trace + 48 + rank * 66 + (l * 2 + mb) * 3 : nullptr;
      if (tr) tp[0] = globaltimer();
      float v[kNtc2], car[24];
      tmem_read_acc<C, kNtc2>(tb + half * kNtc2, v, kNtc2, C::kN, C::kCorrOff);
      tmem_read_acc<C, 24>(tb, car, 24, C::kN, C::kCorrOff);
      tmem_release(mb);
      float val, sp, spp;
      act_fwd2(act, car[0] + bj, val, sp, spp);
      epi_rows(v, car + 1, val, sp, spp, hg);
      mbar_wait_sleep(&in_free[grp], hl & 1);
      if (tr) tp[1] = globaltimer();
      store_publish([&](int i) { return v[i]; }, j, grp);
      if (tr) tp[2] = globaltimer();
    };

    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node = tile >> 1;
      const int hg = static_cast<int>(tile & 1);
      if (tiles_done > 0) {  // the previous tile's output MMAs have read the activation buffer
        mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
      }
      if (etid < kNin2)
        zs[etid] = node < prm.K ? static_cast<float>(tiles_done == 0 ? z_first : load_z(prm, node, etid)) : 0.0f;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // ---- layer 0: v = σ(pre), t_a = σ'·W0'[:,a], h_ab = σ''·W0'[:,a]·W0'[:,b]
      for (int g = static_cast<int>(rank); g < NG; g += 2) {
        const int j = g * 128 + tid_h;
        float w[kNin2];
        float pre = __ldg(prm.b0 + j);
#pragma unroll
        for (int k = 0; k < kNin2; ++k) {
          w[k] = __ldg(prm.w0t + k * WP + j);
          pre = fmaf(w[k], zs[k], pre);
        }
        float val, sp, spp;
        act_fwd2(act, pre, val, sp, spp);
        float v[kNtc2];
        if (half == 0) {
          v[0] = val;
#pragma unroll
          for (int a = 0; a < kNin2; ++a) v[1 + a] = sp * w[a];
          if (hg == 0) hrows0<0, kCarrier2>(v, w, spp, Seq0{});
          else hrows0<kSlots2, kCarrier2>(v, w, spp, Seq0{});
        } else {
          if (hg == 0) hrows0<kNtc2 - kCarrier2, 0>(v, w, spp, Seq1{});
          else hrows0<kSlots2 + kNtc2 - kCarrier2, 0>(v, w, spp, Seq1{});
        }
        store_publish([&](int i) { return v[i]; }, j, g);
      }
      for (int l = 0; l < n_mma_layers; ++l, ++hl)
        for (int mb = 0; mb < NMB; ++mb) do_block(mb, l, hg);
      // ---- output layer: lane = this CTA side's row; columns = outputs
      mbar_wait_sleep(tmem_last, tiles_done & 1);
      tc_fence_after();
      float o[16];
      if (half == 0) read_out(o);
      tmem_release(0);
      if (half == 0) {
        const int r = tid_h, n_out = prm.n_out;
        if (node < prm.K && r < kNtc2) {
          note_nonfinite(prm, o, n_out);
          if (rank == 0 && r < kCarrier2) {
            if (hg == 0) {
              if (r == 0)
                for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
              else
                for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * kNin2 + (r - 1)] = static_cast<double>(o[oo]);
            }
          } else {
            const int slot = rank == 0 ? r - kCarrier2 : (kNtc2 - kCarrier2) + r;
            const int p2 = hg * kSlots2 + slot;
            if (p2 < kPairs2 && prm.hess != nullptr) {
              const PairAB ab = pair_ab(p2, kNin2);
              for (int oo = 0; oo < n_out; ++oo) {
                double* h = prm.hess + (node * n_out + oo) * kNin2 * kNin2;
                h[ab.a * kNin2 + ab.b] = static_cast<double>(o[oo]);
                h[ab.b * kNin2 + ab.a] = static_cast<double>(o[oo]);
              }
            }
          }
        }
      }
    }
   } else if constexpr (ORD2 == 2) {
    // ===================== order-2 epilogue, generic tiles (n_in <= 31) ========
    // Same recurrence with the slot → (a, b) map read from the shared table and
    // the carrier tangents T_a parked in this thread's private shared-memory
    // column (Ts[half][a][tid_h]; registers cannot be indexed at run time).
    constexpr int kCar = NTC < 32 ? NTC : 32;  // carrier columns read (1 + n_in <= kCar)
    const uint16_t* ab_s = reinterpret_cast<const uint16_t*>(smem + C::kAbOff);
    float* ts = reinterpret_cast<float*>(smem + C::kTsOff) + half * 32 * 128 + tid_h;  // ts[a·128]
    const int car_rows = 1 + n_in, slots = 2 * NTC - car_rows, np = n_in * (n_in + 1) / 2;
    const int G = prm.ord2_g;
    // packed pair of row i of this half in group hg (-1: carrier row or padding)
    auto pair_of = [&](int i, int hg) -> int {
      const int s = half == 0 ? i - car_rows : NTC - car_rows + i;
      const int p = hg * slots + s;
      return (s >= 0 && p < np) ? p : -1;
    };
    // rows of this half: carrier (half 0) from (val, sp·t), Hessian rows
    // h' = σ'·h + σ''·T_a·T_b (h = 0 and T = W0' columns at layer 0)
    auto epi_rows = [&](float* v, const float* tcar, float val, float sp, float spp, int hg, bool first) {
#pragma unroll
      for (int i = 0; i < NTC; ++i) {
        if (half == 0 && i < car_rows) {
          constexpr int kLast = kCar - 2;  // car_rows <= kCar: tcar index i - 1 <= kCar - 2
          const int ti = i == 0 ? 0 : (i - 1 < kLast ? i - 1 : kLast);  // compile-time once unrolled
          v[i] = i == 0 ? val : sp * tcar[ti];
        } else {
          const int p = pair_of(i, hg);
          if (p >= 0) {
            const uint32_t abv = ab_s[p];
            const float t2 = ts[(abv & 0xff) * 128] * ts[(abv >> 8) * 128];
            v[i] = first ? spp * t2 : fmaf(spp, t2, sp * v[i]);
          } else {
            v[i] = 0.0f;
          }
        }
      }
    };
    auto do_block = [&](int mb, int l, int hg) {
      const int grp = 2 * mb + static_cast<int>(rank);
      const int j = mb * 256 + static_cast<int>(rank) * 128 + tid_h;
      const float bj = __ldg(prm.bh + l * WP + j);
      const uint32_t tb = tmem_base + lane_base + mb * C::kBlkCols;
      mbar_wait_sleep(&tmem_full[mb], hl & 1);
      tc_fence_after();
      float v[NTC], car[kCar];
      tmem_read_acc<C, NTC>(tb + half * NTC, v, NTC, C::kN, C::kCorrOff);
      tmem_read_acc<C, kCar>(tb, car, car_rows, C::kN, C::kCorrOff);
      tmem_release(mb);
      float val, sp, spp;
      act_fwd2(act, car[0] + bj, val, sp, spp);
#pragma unroll
      for (int a = 0; a + 1 < kCar; ++a)
        if (a < n_in) ts[a * 128] = car[1 + a];
      epi_rows(v, car + 1, val, sp, spp, hg, false);
      mbar_wait_sleep(&in_free[grp], hl & 1);
      store_publish([&](int i) { return v[i]; }, j, grp);
    };

    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node = tile / G;
      const int hg = static_cast<int>(tile - node * G);
      if (tiles_done > 0) {  // the previous tile's output MMAs have read the activation buffer
        mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
      }
      if (etid < n_in)
        zs[etid] = node < prm.K ? static_cast<float>(tiles_done == 0 ? z_first : load_z(prm, node, etid)) : 0.0f;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // ---- layer 0: v = σ(pre), t_a = σ'·W0'[:,a], h_ab = σ''·W0'[:,a]·W0'[:,b]
      for (int g = static_cast<int>(rank); g < NG; g += 2) {
        const int j = g * 128 + tid_h;
        float w[kCar];
        float pre = __ldg(prm.b0 + j);
#pragma unroll
        for (int k = 0; k < kCar; ++k) {
          w[k] = k < n_in ? __ldg(prm.w0t + k * WP + j) : 0.0f;
          if (k < n_in) {
            pre = fmaf(w[k], zs[k], pre);
            ts[k * 128] = w[k];
          }
        }
        float val, sp, spp;
        act_fwd2(act, pre, val, sp, spp);
        float v[NTC];
        epi_rows(v, w, val, sp, spp, hg, true);
        store_publish([&](int i) { return v[i]; }, j, g);
      }
      for (int l = 0; l < n_mma_layers; ++l, ++hl)
        for (int mb = 0; mb < NMB; ++mb) do_block(mb, l, hg);
      // ---- output layer: lane = this CTA side's row; columns = outputs
      mbar_wait_sleep(tmem_last, tiles_done & 1);
      tc_fence_after();
      float o[16];
      if (half == 0) read_out(o);
      tmem_release(0);
      if (half == 0) {
        const int r = tid_h, n_out = prm.n_out;
        if (node < prm.K && r < NTC) {
          note_nonfinite(prm, o, n_out);
          if (rank == 0 && r < car_rows) {
            if (hg == 0) {
              if (r == 0)
                for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
              else
                for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + (r - 1)] = static_cast<double>(o[oo]);
            }
          } else {
            const int s = rank == 0 ? r - car_rows : NTC - car_rows + r;
            const int p = hg * slots + s;
            if (p < np && prm.hess != nullptr) {
              const uint32_t abv = ab_s[p];
              const int a = abv & 0xff, b = abv >> 8;
              for (int oo = 0; oo < n_out; ++oo) {
                double* h = prm.hess + (node * n_out + oo) * n_in * n_in;
                h[a * n_in + b] = static_cast<double>(o[oo]);
                h[b * n_in + a] = static_cast<double>(o[oo]);
              }
            }
          }
        }
      }
    }
   } else if constexpr (ORD2 >= 3) {
    // ===================== reverse mode: value (3) / adjoint (4) pass ========
    // Rows: value pass = nodes (pn = prm.P per side); adjoint pass = node-major
    // (node, output o) rows, kRevOut = 6 outputs (the quadrotor residual; the
    // host refuses other n_out), pn nodes x 6 rows per side. Slopes σ'_l of
    // every node go to / come from prm.rev_s, [n_hidden][K][WP] fp32 (thread =
    // neuron: a warp's 32 neurons of one node are one 128-byte line).
    constexpr bool kAdj = ORD2 == 4;
    constexpr int kRevOut = 6;
    constexpr int kAdjNodes = (NTC + kRevOut - 1) / kRevOut;  // adjoint pass: the side's nodes
    const int n_out = prm.n_out, pn = prm.P;
    const int rows_used = kAdj ? pn * kRevOut : pn;
    const long long K = prm.K;
    const int n_mma = n_mma_layers;
    float* const rs = prm.rev_s;
    auto slope = [&](int li, long long node, int j) -> float* { return rs + (static_cast<long long>(li) * K + node) * WP + j; };
    constexpr int kG0 = NG / 2;
    // first production of a tile: value pass = layer 0 (CUDA cores, fp32; z from
    // global, read by every thread: L1 broadcasts), adjoint pass = W_L'[o, j]·σ'_H;
    // each CTA writes every K-group for its OWN side's rows (local stores only)
    // one element (row i of neuron column j) into this CTA's operand buffer
    auto store_row = [&](int i, int j, float x) {
      const uint32_t a = act_local + (j / C::kCK) * C::kChunkStride + ((((j % C::kCK) * C::kEB) >> 4) << 4) +
                         ((j * C::kEB) & 15) + (i >> 3) * 1024 + ((((((j * C::kEB) >> 4) & 7) ^ (i & 7)) -
                                                                    (((j * C::kEB) >> 4) & 7)) * 16 + (i & 7) * 128);
      if constexpr (MODE == k3xTF32) {
        const float h = to_tf32(x);
        st_shared_f32(a, h);
        st_shared_f32(a + C::kSplitStride, to_tf32(x - h));
      } else {  // bf16x3 (the pair reverse variants are the split-precision modes)
        const uint16_t h = bf16_rn_bits(x);
        st_shared_u16(a, h);
        st_shared_u16(a + C::kSplitStride, bf16_rn_bits(x - bf16_to_f32(h)));
      }
    };
    // first production of a tile: value pass = layer 0 (CUDA cores, fp32), adjoint
    // pass = W_L'[o, j]·σ'_H; each CTA writes every K-group for its OWN side's rows
    // (local stores only). Rolled loops over the rows (one element each) keep the
    // code (and the compile) small; this runs once per tile.
    // value pass: z rows of this CTA's nodes of `tile` into L1 (thread = row
    // end: the first and last element's lines)
    auto prefetch_z = [&](long long tile) {
      if constexpr (!kAdj) {
        const int t = half * 128 + tid_h, i = t >> 1;
        const long long node = tile * (2 * pn) + static_cast<long long>(rank) * pn + i;
        if (tile < prm.num_tiles && i < rows_used && node < K)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(z_ptr(prm, node, (t & 1) ? n_in - 1 : 0)));
      }
    };
    auto first_store = [&](long long tile) {
      const long long nb = tile * (2 * pn) + static_cast<long long>(rank) * pn;
      if constexpr (!kAdj) {
        // this thread's neurons j = g·128 + tid_h of the groups g = half + 2·gi;
        // rows two at a time: 2·kG0 independent fma chains per shuffle of z
        float w[kG0][kMaxIn2], bj[kG0];
#pragma unroll
        for (int gi = 0; gi < kG0; ++gi) {
          const int j = (half + 2 * gi) * 128 + tid_h;
#pragma unroll
          for (int k = 0; k < kMaxIn2; ++k) w[gi][k] = k < n_in ? __ldg(prm.w0t + k * WP + j) : 0.0f;
          bj[gi] = __ldg(prm.b0 + j);
        }
        // lane k holds z[node][k] (one coalesced load per row, raw and centred at
        // use, the next row pair's loads in flight); the warp broadcasts it by
        // shuffle. The rows were prefetched into L1 (prefetch_z): a cold z row
        // costs ~1.5 us under the weight stream, once per row pair otherwise.
        const double mu_l = lane < n_in ? __ldg(prm.mu + lane) : 0.0;
        auto zlane = [&](int i) -> double {  // unconditional load (pads read μ)
          const long long node = nb + i;
          return *((lane < n_in && i < rows_used && node < K) ? z_ptr(prm, node, lane)
                                                              : prm.mu + (lane < n_in ? lane : 0));
        };
        double zr0 = zlane(0), zr1 = zlane(1);
        static_assert(NTC % 2 == 0, "rows in pairs");
#pragma unroll 1
        for (int i = 0; i < ntc; i += 2) {
          const double zn0 = zlane(i + 2), zn1 = zlane(i + 3);
          const float zk0 = static_cast<float>(zr0 - mu_l), zk1 = static_cast<float>(zr1 - mu_l);
          float pre[2][kG0];
#pragma unroll
          for (int gi = 0; gi < kG0; ++gi) pre[0][gi] = pre[1][gi] = bj[gi];
#pragma unroll
          for (int k = 0; k < kMaxIn2; ++k) {
            const float a0 = __shfl_sync(0xffffffffu, zk0, k), a1 = __shfl_sync(0xffffffffu, zk1, k);
#pragma unroll
            for (int gi = 0; gi < kG0; ++gi) {
              pre[0][gi] = fmaf(w[gi][k], a0, pre[0][gi]);
              pre[1][gi] = fmaf(w[gi][k], a1, pre[1][gi]);
            }
          }
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const long long node = nb + i + r;
            const bool live = i + r < rows_used && node < K;
#pragma unroll
            for (int gi = 0; gi < kG0; ++gi) {
              const int j = (half + 2 * gi) * 128 + tid_h;
              float val = 0.0f, sp;
              if (live) {
                act_fwd_rows(act, pre[r][gi], val, sp);
                *slope(0, node, j) = sp;
              }
              store_row(i + r, j, val);
            }
          }
          zr0 = zn0;
          zr1 = zn1;
        }
#pragma unroll
        for (int gi = 0; gi < kG0; ++gi) publish_chunk(half + 2 * gi, true);
      } else {
        // row (node p, output o) = W_L'[o, j]·σ'_H[node p, j]: the 6 weights and the
        // side's slopes are loaded up front (one round trip, not one per row)
#pragma unroll 1
        for (int gi = 0; gi < kG0; ++gi) {
          const int g = half + 2 * gi;
          const int j = g * 128 + tid_h;
          float wlo[kRevOut], sl[kAdjNodes];
#pragma unroll
          for (int o = 0; o < kRevOut; ++o) wlo[o] = __ldg(prm.wl + o * WP + j);
#pragma unroll
          for (int p = 0; p < kAdjNodes; ++p) sl[p] = (p < pn && nb + p < K) ? __ldg(slope(n_mma, nb + p, j)) : 0.0f;
#pragma unroll
          for (int i = 0; i < NTC; ++i) {
            if ((i & ~7) >= ntc) continue;
            store_row(i, j, i < rows_used ? wlo[i % kRevOut] * sl[i / kRevOut] : 0.0f);
          }
          publish_chunk(g, true);
        }
      }
    };
    // hidden block mb of MMA layer l: value pass y = σ(d + b) and σ' to the
    // scratch; adjoint pass y = d·σ' (slopes of the side's nodes loaded before
    // the accumulator wait)
    auto do_block = [&](int mb, int l, long long tile) {
      const int grp = 2 * mb + static_cast<int>(rank);
      const int j = mb * 256 + static_cast<int>(rank) * 128 + tid_h;
      const int li = kAdj ? n_mma - 1 - l : l + 1;
      const long long nb = tile * (2 * pn) + static_cast<long long>(half) * pn;  // side `half`'s nodes
      const uint32_t tsd = tmem_base + lane_base + mb * C::kBlkCols + half * ntc;
      float sn[kAdj ? kAdjNodes : 1];
      if constexpr (kAdj) {
#pragma unroll
        for (int p = 0; p < kAdjNodes; ++p) sn[p] = (p < pn && nb + p < K) ? __ldg(slope(li, nb + p, j)) : 0.0f;
      }
      const float bj = kAdj ? 0.0f : __ldg(prm.bh + l * WP + j);
      mbar_wait_sleep(&tmem_full[mb], hl & 1);
      tc_fence_after();
      const bool tr = trace_on();
      unsigned long long* tp = tr ? prm.trace + 48 + rank * 66 + (l * 2 + mb) * 3 : nullptr;
      if (tr) tp[0] = globaltimer();
      float v[NTC];
      tmem_read_acc<C, NTC>(tsd, v, ntc, C::kN, C::kCorrOff);
      tmem_release(mb);
      if constexpr (!kAdj) {
        // unrolled over the rows (v stays in registers: a rolled loop would index
        // it dynamically, i.e. put it in local memory, which spills to L2 with
        // the shared-memory carve-out) with the activation switch hoisted
        auto act_rows = [&](auto kact) {
          constexpr int kAct = decltype(kact)::value;
          float* sl = slope(li, nb, j);
#pragma unroll
          for (int i = 0; i < NTC; ++i) {
            float val = 0.0f, sp;
            if (i < rows_used) {
              act_fwd_rows(kAct, v[i] + bj, val, sp);
              if (nb + i < K) sl[i * WP] = sp;
            }
            v[i] = val;
          }
        };
        if (act == 0) act_rows(std::integral_constant<int, 0>{});
        else if (act == 1) act_rows(std::integral_constant<int, 1>{});
        else act_rows(std::integral_constant<int, 2>{});
      } else {
#pragma unroll
        for (int i = 0; i < NTC; ++i) v[i] = i < rows_used ? v[i] * sn[i / kRevOut] : 0.0f;
      }
      if (tr) tp[1] = globaltimer();
      mbar_wait_sleep(&in_free[grp], hl & 1);
      store_publish([&](int i) { return v[i]; }, j, grp);
      if (tr) tp[2] = globaltimer();
    };
    // outputs of a finished tile: this CTA's rows in its TMEM lanes
    auto write_out = [&](long long tile) {
      float o[C::kOutN];
      tmem_read_acc<C, C::kOutN>(tmem_base + lane_base, o, C::kOutN, static_cast<uint32_t>(C::kOutN),
                                 static_cast<uint32_t>(C::kOutN * C::kChains));
      const int r = tid_h;
      const long long nb = tile * (2 * pn) + static_cast<long long>(rank) * pn;
      if (r < rows_used) {
        if constexpr (!kAdj) {
          const long long node = nb + r;
          if (node < K) {
            note_nonfinite(prm, o, n_out);
            for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
          }
        } else {
          const int p = r / kRevOut, oo = r - p * kRevOut;
          const long long node = nb + p;
          if (node < K) {
            note_nonfinite(prm, o, n_in);
            double* jr = prm.jac + (node * kRevOut + oo) * n_in;
            for (int i = 0; i < n_in; ++i) jr[i] = static_cast<double>(o[i]);
          }
        }
      }
    };
    long long prev_tile = -1;
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      if (tiles_done > 0) {  // the previous tile's output MMAs have read the activation buffer
        mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
        if (half == 0) write_out(prev_tile);
        tmem_release(0);
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (trace_on()) prm.trace[192 + rank] = globaltimer();
      if (tiles_done == 0) prefetch_z(tile);
      first_store(tile);
      if (trace_on()) prm.trace[194 + rank] = globaltimer();
      for (int l = 0; l < n_mma_layers; ++l, ++hl) {
        if (l == n_mma_layers - 1) prefetch_z(tile + npairs);  // the next tile's z, a layer ahead
        for (int mb = 0; mb < NMB; ++mb) do_block(mb, l, tile);
      }
      prev_tile = tile;
    }
    if (tiles_done > 0) {
      mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
      tc_fence_after();
      if (half == 0) write_out(prev_tile);
    }
   } else {
    // ===================== order-1 epilogue ===================================
    const int rows_used = P * (1 + n_in);   // rows per side
    const bool no_pad = rows_used == ntc;

    // Activation epilogue on one side's rows (fp32): value rows → σ(pre+b),
    // tangent rows → σ'(pre)·t, padding → 0.
    auto scale_side = [&](float* v, float bj) {
      float val[P], sp[P];
#pragma unroll
      for (int p = 0; p < P; ++p) act_fwd(act, v[p] + bj, val[p], sp[p]);
#pragma unroll
      for (int p = 0; p < P; ++p) v[p] = val[p];
      if (no_pad) {
#pragma unroll
        for (int i = P; i < NTC; ++i) v[i] = v[i] * sp[i % P];
      } else {
#pragma unroll
        for (int i = P; i < NTC; ++i) v[i] = i < rows_used ? v[i] * sp[i % P] : 0.0f;
      }
    };
    // Hidden block mb: TMEM (this CTA's 128 neurons, this half's side) →
    // registers → epilogue → operand buffer of K-group 2·mb + rank.
    auto do_block = [&](int mb, int l) {
      const int grp = 2 * mb + static_cast<int>(rank);
      const int j = mb * 256 + static_cast<int>(rank) * 128 + tid_h;
      const float bj = __ldg(prm.bh + l * WP + j);
      const uint32_t tsd = tmem_base + lane_base + mb * C::kBlkCols + half * ntc;
      mbar_wait_sleep(&tmem_full[mb], hl & 1);
      tc_fence_after();
      const bool tr = trace_on();
      unsigned long long* tp = tr ? prm.trace + 48 + rank * 66 + (l * 2 + mb) * 3 : nullptr;
      if (tr) tp[0] = globaltimer();
      float v[NTC];
      if (prm.dbg & 4) {  // dbg 4: no epilogue math or stores (timing)
        tmem_release(mb);
        mbar_wait_sleep(&in_free[grp], hl & 1);
        fence_proxy_async_cluster();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(ready_cl0 + 8 * ((grp * 128 + q * 32) / C::kCK));
        return;
      }
      tmem_read_acc<C, NTC>(tsd, v, ntc, C::kN, C::kCorrOff);
      tmem_release(mb);
      scale_side(v, bj);
      mbar_wait_sleep(&in_free[grp], hl & 1);
      if (tr) tp[1] = globaltimer();
      store_publish([&](int i) { return v[i]; }, j, grp);
      if (tr) tp[2] = globaltimer();
    };
    // Layer 0 (CUDA cores): σ, σ' of pre = b0 + W0'·(z − μ); the tangent rows
    // are σ'·W0'[:, k] (the seed is the identity). Layer 0 needs no TMEM, so
    // each CTA computes EVERY K-group for its OWN side's nodes (warp half h:
    // groups h, h + 2, ...) and all its stores are local: twice the CUDA-core
    // math of an owner-computes split, but none of the DSMEM traffic, which
    // runs at a third of the local store rate (scripts/dsmem_bench.cu).
    constexpr int kG0 = NG / 2;  // K-groups per warp half
    constexpr bool kMayBeWide = P < 4 && NTC / P - 1 > kMaxIn0;  // small-P tiles may see > kMaxIn0 inputs
    float val0[kG0][P], sp0[kG0][P];
    auto layer0_math = [&]() {
      const float* zside = zs + static_cast<int>(rank) * P * n_in;  // this CTA's nodes
#pragma unroll
      for (int gi = 0; gi < kG0; ++gi) {
        const int j = (half + 2 * gi) * 128 + tid_h;
        const float bj = __ldg(prm.b0 + j);
        if (!kMayBeWide || n_in <= kMaxIn0) {
          float w0[kMaxIn0];
          load_w0_row(prm.w0t, WP, j, n_in, w0);
#pragma unroll
          for (int p = 0; p < P; ++p)
            act_fwd(act, layer0_pre(bj, w0, zside + p * n_in, n_in), val0[gi][p], sp0[gi][p]);
        } else {
#pragma unroll
          for (int p = 0; p < P; ++p) {
            float pre = bj;
            for (int k = 0; k < n_in; ++k) pre = fmaf(__ldg(prm.w0t + k * WP + j), zside[p * n_in + k], pre);
            act_fwd(act, pre, val0[gi][p], sp0[gi][p]);
          }
        }
      }
    };
    auto layer0_store = [&]() {
#pragma unroll
      for (int gi = 0; gi < kG0; ++gi) {
        const int g = half + 2 * gi;
        const int j = g * 128 + tid_h;
        // rows: value rows σ(pre), tangent row (k, p) σ'_p·W0'[j, k], padding 0
        if (!kMayBeWide || n_in <= kMaxIn0) {
          float w0[kMaxIn0];
          load_w0_row(prm.w0t, WP, j, n_in, w0);
          store_to([&](int i) {
            return i < P ? val0[gi][i % P] : (i < rows_used ? sp0[gi][i % P] * w0[((i - P) / P) % kMaxIn0] : 0.0f);
          }, j, act_local, true);
        } else {
          store_to([&](int i) {
            return i < P ? val0[gi][i % P]
                         : (i < rows_used ? sp0[gi][i % P] * __ldg(prm.w0t + ((i - P) / P) * WP + j) : 0.0f);
          }, j, act_local, true);
        }
        publish_chunk(g, true);
      }
    };
    // z of the tile's 2P nodes, one element per thread, fetched one tile ahead
    // (registers) so its global-load latency hides behind the hidden layers
    // (the raw fp64 element only: no arithmetic on it until the next tile's staging,
    // so the load is not waited for here)
    const bool zown = etid < 2 * P * n_in;
    const int zp = zown ? etid / n_in : 0, zk = zown ? etid - zp * n_in : 0;
    const double mu_k = __ldg(prm.mu + zk);
    auto fetch_z = [&](long long tile) -> double {
      const long long node = tile * (2 * P) + zp;
      if (!(zown && tile < prm.num_tiles && node < prm.K)) return mu_k;  // stages as 0
      if (prm.zx == nullptr) return prm.z[node * n_in + zk];
      const long long xrow = node + node / prm.zN;  // gather mode: [x_k; u_k] from the iterate
      return zk < 13 ? prm.zx[xrow * 13 + zk] : prm.zu[node * 4 + (zk - 13)];
    };
    // outputs of a finished tile (this CTA's rows in its TMEM lanes, outputs in columns 0..15)
    auto write_out = [&](const float* o, long long node0) {
      const int r = tid_h;
      const int n_out = prm.n_out;
      const long long nbase = node0 + static_cast<long long>(rank) * P;
      if (r < P) {
        const long long node = nbase + r;
        if (node < prm.K) {
          note_nonfinite(prm, o, n_out);
          for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
        }
      } else if (r < rows_used && prm.jac != nullptr) {
        const int k = (r - P) / P, p = (r - P) % P;
        const long long node = nbase + p;
        if (node < prm.K) {
          note_nonfinite(prm, o, n_out);
          for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + k] = static_cast<double>(o[oo]);
        }
      }
    };

    double znext = z_first;  // fetch_z(pair), issued before the setup
    float o[16];
    long long prev_node0 = -1;
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node0 = tile * (2 * P);
      // ---- tile boundary: layer-0 math of this tile overlaps the previous
      // tile's output layer; its stores wait for the output MMAs (which read
      // the activation buffer)
      const bool trb = trace_on();
      unsigned long long* tb = trb ? prm.trace + 180 + rank * 6 : nullptr;
      if (trb) tb[0] = globaltimer();
      if (zown) zs[etid] = static_cast<float>(znext - mu_k);  // centred in fp64 (rtn_kernel.cuh load_z)
      asm volatile("bar.sync 1, 256;" ::: "memory");
      znext = fetch_z(tile + npairs);
      layer0_math();
      if (trb) tb[1] = globaltimer();
      if (tiles_done > 0) {
        mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
        if (trb) tb[2] = globaltimer();
        if (half == 0) read_out(o);
        tmem_release(0);
      }
      if (trb) tb[3] = globaltimer();
      layer0_store();
      if (trace_on()) prm.trace[192 + rank] = globaltimer();
      // the previous tile's outputs go out after the layer-0 publications (a
      // publication's proxy fence would otherwise wait for these global stores)
      if (tiles_done > 0 && half == 0) write_out(o, prev_node0);
      // ---- hidden layers
      for (int l = 0; l < n_mma_layers; ++l, ++hl)
        for (int mb = 0; mb < NMB; ++mb) do_block(mb, l);
      prev_node0 = node0;
      if (trace_on()) prm.trace[194 + rank] = globaltimer();
    }
    if (tiles_done > 0) {  // the last tile's outputs
      mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
      tc_fence_after();
      if (half == 0) {
        read_out(o);
        write_out(o, prev_node0);
      }
    }
   }
  }
  if (tr_pair && threadIdx.x == 0) {
    prm.trace[252 + rank] = globaltimer();
    prm.trace[254 + rank] = clock64();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace rtn
