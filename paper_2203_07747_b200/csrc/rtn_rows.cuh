// rtn_rows.cuh — throughput kernel for padded width 256, TF32, order 1, with
// the activations as the MMA's A operand in TENSOR MEMORY ("rows" orientation).
//
// Why: the pair kernel (rtn_pair.cuh) keeps the activations in shared memory
// as the B operand (lane = neuron). Its epilogue therefore writes every
// activation back through the SMEM port (half of it over DSMEM to the peer
// CTA) while the MMAs and the weight TMA saturate that port, and at width 256
// one M-block per layer leaves nothing to overlap the epilogue with (the
// ping-pong kernel reached 0.43 of the TF32 peak). Here:
//   D[row, neuron] = Σ_k A[row, k] · W[neuron, k]
// with M = 256 tile rows (128 per CTA = TMEM lanes), N = 256 neurons (each
// CTA holds 128 weight rows of the 2-SM TMA tile, as before) and A read from
// TMEM (tcgen05.mma ... [d], [a_tmem], b_desc). TMEM holds two 256-column
// regions R0/R1: layer l reads A from R_{l%2} and accumulates into
// R_{(l+1)%2}; the epilogue rewrites that region in place (tcgen05.ld → σ/σ'
// → tf32 → tcgen05.st), and it becomes layer l+1's A. A CTA's rows are its own
// TMEM lanes, so nothing crosses to the peer, and nothing goes through shared
// memory except small per-node σ/σ' tables. The MMA of layer l+1 starts on
// K-group 0 (columns 0..63) as soon as that group is rewritten, while the
// epilogue finishes groups 1..3 (scripts/tmem_a_probe.cu: A from TMEM runs
// N = 256 pair MMAs at 93 % of the tf32 floor, A from SMEM at 75 %).
//
// Rows: NPC = 128 / (1 + n_in) nodes per CTA (7 for the quadrotor's 17
// inputs), 2·NPC per pair tile. Row p < NPC is the value row of node p; row
// NPC + p·n_in + k the tangent for input k of node p. All value rows sit in
// TMEM lanes 0..NPC-1, so only the lane-quadrant-0 warps read them out for the
// σ tables: TMEM reads run at ~64-128 B/clk per SM (B300_MICROARCH.md), and a
// full second pass over the 128 KB accumulator cost ~1.3 K cycles per layer.
//
// Epilogue (8 warps; warp w reads TMEM lanes 32·(w%4).., warp half h owns
// columns [128h, 128h + 128) as two 64-column groups):
//   value rows publish pre = d + b to smem; the 128 threads of the half then
//   evaluate σ, σ' for all (node, neuron) pairs of the group (≈4 each instead
//   of 64 per value lane); every row reads its node's σ (value) or σ'
//   (tangent: t' = σ'·d) back.
// Layer 0 (n_in → 256, CUDA cores) is the same table trick with W0' staged in
// shared memory once per CTA: tangent row k gets σ'(pre)·W0'[:, k].
// The output layer (256 → n_out ≤ 16) is one more pair MMA, N = 16.
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"

namespace rtn {

constexpr int kRowsMaxIn = 31;     // R = 1 + n_in <= 32 → NPC >= 4
constexpr int kRowsMaxNodes = 16;  // table capacity: R >= 8 → n_in >= 7
constexpr int kRowsTabStride = 260;  // floats per node row of the σ/σ' tables (bank spread)
constexpr int kRowsMaxMma = 11;      // hidden→hidden layers whose biases fit the smem copy

template <int NSTAGE>
struct RowsCfg {
  static constexpr int kWP = 256, kNKC = 8;
  static constexpr uint32_t kStageOff = 0;
  static constexpr uint32_t kW0Off = kStageOff + NSTAGE * kStageBytes;        // 256 x n_in fp32
  static constexpr uint32_t kPreOff = kW0Off + 256 * kRowsMaxIn * 4;                     // [16][260] pre
  static constexpr uint32_t kTabOff = kPreOff + kRowsMaxNodes * kRowsTabStride * 4;      // [16][2][260] σ, σ'
  static constexpr uint32_t kTab0Off = kTabOff + kRowsMaxNodes * 2 * kRowsTabStride * 4; // [16][2][260] layer-0 σ, σ'
  static constexpr uint32_t kZsOff = kTab0Off + kRowsMaxNodes * 2 * kRowsTabStride * 4;  // [16][32] z
  static constexpr uint32_t kBhOff = kZsOff + kRowsMaxNodes * 32 * 4;                      // [11][256] hidden biases
  static constexpr uint32_t kBarOff = kBhOff + kRowsMaxMma * 256 * 4;
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 16 + 2;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kSmemBytes = kMiscOff + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// Four K=8 pair MMAs with A in TMEM (columns a, a+8, a+16, a+24) and B from a
// 32-k SW128 weight stage, one elect, then a multicast commit of the stage's
// empty barrier.
__device__ __forceinline__ void mma4_tf32_pair_ts_commit(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                         uint32_t accumulate, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a1], b1, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a2], b2, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [a3], b3, %3, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], m;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])));
}

// Activation for the rows kernel (TF32 mode only): SiLU through ex2.approx and
// rcp.approx (~2 ulp in fp32, far below the 2^-11 tf32 operand rounding that
// follows); tanh/relu as act_fwd.
template <int ACT>
__device__ __forceinline__ void act_rows(float pre, float& val, float& sp) {
  if constexpr (ACT == 2) {
    float e, s;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(pre * -1.4426950408889634f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(1.0f + e));
    val = pre * s;
    sp = s * (1.0f + pre * (1.0f - s));
  } else {
    act_fwd(ACT, pre, val, sp);
  }
}

// tcgen05.ld.16x256b.x8: TMEM lanes [0, 16) of the warp's quadrant x 64 columns.
__device__ __forceinline__ void tmem_ld_16x256b_x8(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// tcgen05.ld.16x256b.x4: TMEM lanes [0, 16) of the warp's quadrant x 32 columns.
__device__ __forceinline__ void tmem_ld_16x256b_x4(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// ACT is the activation as a template argument (0 tanh, 1 relu, 2 SiLU): one
// inlined activation path keeps the epilogue loop small enough for the
// instruction cache (the runtime switch tripled its code).
template <int NSTAGE, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    rtn_rows_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                    const __grid_constant__ CUtensorMap tmap_l) {
  using C = RowsCfg<NSTAGE>;
  constexpr int NKC = C::kNKC;
  extern __shared__ uint8_t smem_raw[];
  // 1 KB-aligned base as an offset from smem_raw, so every table pointer stays in
  // the shared address space (LDS/STS rather than generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage_s = smem + C::kStageOff;
  float* w0s = reinterpret_cast<float*>(smem + C::kW0Off);
  float* pre_t = reinterpret_cast<float*>(smem + C::kPreOff);
  float* tab = reinterpret_cast<float*>(smem + C::kTabOff);
  float* tab0 = reinterpret_cast<float*>(smem + C::kTab0Off);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);
  float* bhs = reinterpret_cast<float*>(smem + C::kBhOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  // act[s][c]: K-chunk c (32 columns) of A production k is in TMEM, s = k & 1.
  // Two sets so that the next tile's layer 0, published while the MMA warp may
  // still be waiting on the output layer's chunks, never laps a waiter.
  uint64_t* act = bars + 2 * NSTAGE;
  uint64_t* tmem_full = act + 16;
  uint64_t* tmem_last = tmem_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, npc = prm.P;  // inputs, nodes per CTA
  const int n_mma = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int g = 0; g < 16; ++g) mbar_init(&act[g], 16);  // 8 epilogue warps x 2 CTAs
    mbar_init(tmem_full, 1);
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_h);
    prefetch_tmap(&tmap_l);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  pdl_launch_dependents();
  // layer-0 weights (normalisation folded) stay in shared memory for the whole kernel
  for (int i = threadIdx.x; i < 256 * n_in; i += blockDim.x) w0s[i] = __ldg(prm.w0 + i);
  for (int i = threadIdx.x; i < 256 * n_mma; i += blockDim.x) bhs[i] = __ldg(prm.bh + i);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer (2-SM TMA, own 128-neuron half) =====
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    int st = 0;
    const int yr = static_cast<int>(rank) * 128;
    auto next = [&]() {
      if (++st == NSTAGE) {
        st = 0;
        ph ^= 1;
      }
    };
    // K-chunk order: the first MMA layer of a tile (the consumer of layer 0)
    // takes chunks 1..7 then 0, because chunk 0 shares columns with the
    // previous tile's output-layer accumulator (see the epilogue)
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
      for (int l = 0; l < n_mma; ++l)
        for (int i = 0; i < NKC; ++i) {
          const int c = l == 0 ? (i + 1) & (NKC - 1) : i;
          mbar_wait(&empty[st], ph ^ 1);
          if (leader) mbar_expect_tx_elect(&full[st], 2 * kStageBytes);
          tma_load_2sm(stage_s + st * kStageBytes, &tmap_h, c * 32, l * 256 + yr, &full[st], pol);
          next();
        }
      for (int i = 0; i < NKC; ++i) {
        const int c = n_mma == 0 ? (i + 1) & (NKC - 1) : i;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * 1024);
        tma_load_2sm(stage_s + st * kStageBytes, &tmap_l, c * 32, static_cast<int>(rank) * 8, &full[st], pol);
        next();
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) =======================
    if (leader) {
      const uint32_t idesc_h = idesc_tf32(256, 256), idesc_o = idesc_tf32(256, kMaxOut);
      const uint64_t b0 = sw128_desc(smem_u32(stage_s));
      constexpr uint32_t kStageD = kStageBytes >> 4;
      uint32_t ph = 0, cons = 0;
      int st = 0;
      long long tix = 0;
      auto layer = [&](uint32_t a_reg, uint32_t d_reg, uint32_t idesc, int li, bool first) {
        unsigned long long* tp = (prm.trace && pair == 0 && tix < 2 && li < 8 && lane == 0) ? prm.trace + tix * 24 + li * 3 : nullptr;
        if (tp) tp[0] = globaltimer();
        uint64_t* a_set = act + 8 * (cons & 1);
        const uint32_t par = (cons >> 1) & 1;
#pragma unroll 1
        for (int i = 0; i < NKC; ++i) {
          const int c = first ? (i + 1) & (NKC - 1) : i;
          if (!(prm.dbg & 128)) mbar_wait(&a_set[c], par);  // dbg 128: weight stream + MMAs only
          tc_fence_after();
          if (tp && i == 0) tp[1] = globaltimer();
          mbar_wait(&full[st], ph);
          tc_fence_after();
          mma4_tf32_pair_ts_commit(d_reg, a_reg + 32 * c, b0 + st * kStageD, idesc, i != 0, smem_u32(&empty[st]));
          if (++st == NSTAGE) {
            st = 0;
            ph ^= 1;
          }
        }
        if (tp) tp[2] = globaltimer();
        ++cons;
      };
      // Region of a tile's layer-0 output alternates: the next tile's layer 0 is
      // written into the region that holds this tile's output-layer accumulator.
      int b = 0;
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tix) {
        for (int l = 0; l < n_mma; ++l) {
          layer(tmem_base + ((b + l) & 1) * 256, tmem_base + ((b + l + 1) & 1) * 256, idesc_h, l, l == 0);
          mma_commit_pair(tmem_full);
        }
        layer(tmem_base + ((b + n_mma) & 1) * 256, tmem_base + ((b + n_mma + 1) & 1) * 256, idesc_o, n_mma, n_mma == 0);
        mma_commit_pair(tmem_last);
        b = (b + n_mma + 1) & 1;
      }
    }
  } else if (warp >= 4 && (prm.dbg & 128)) {
    // timing aid: drain the MMA completions only (outputs are not written)
    for (long long tile = pair, td = 0, hl = 0; tile < prm.num_tiles; tile += npairs, ++td) {
      for (int l = 0; l < n_mma; ++l, ++hl) mbar_wait(tmem_full, hl & 1);
      mbar_wait(tmem_last, td & 1);
    }
  } else if (warp >= 4) {
    // ===================== epilogue (8 warps per CTA) ==========================
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int etid = threadIdx.x - 128;
    const int r = q * 32 + lane;  // TMEM lane = tile row of this CTA
    const bool is_val = r < npc;
    const int tr = r - npc, tp = tr / n_in;
    const int p = is_val ? r : tp;                 // node (>= npc: padding row)
    const int j = is_val ? 0 : 1 + (tr - tp * n_in);  // 0 value, 1 + k tangent k
    const bool valid = p < npc;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t act_cl = mapa(smem_u32(act), 0);
    const int tab_row = (valid ? p : 0) * 2 * kRowsTabStride + (j == 0 ? 0 : kRowsTabStride);
    const float* my_tab = tab + tab_row;
    const float* my_tab0 = tab0 + tab_row;
    uint32_t hl = 0, tiles_done = 0;

    // RTN_TRACE fine stamps (clock64) of one layer's epilogue: pair 0, tile 1, layer 1 (warps 4 and 8)
    auto fine = [&](int l, int gg, int e) {
      if (prm.trace && pair == 0 && tiles_done == 1 && l == 1 && gg == 0 && q == 0 && lane == 0 && rank == 0)
        prm.trace[216 + h * 12 + e] = clock64();
    };
    int fl = -1;
    // RTN_TRACE: pair 0, tiles 0-1, lane 0 of warps 4 and 8: per layer L (0 = layer 0)
    // [tmem_full seen, chunk 0 published, last chunk published] at 64 + (((rank·2 + h)·2 + t)·6 + L)·3
    auto trace = [&](int L, int e) {
      if (prm.trace && pair == 0 && tiles_done < 2 && L < 6 && q == 0 && lane == 0)
        prm.trace[64 + (((rank * 2 + h) * 2 + tiles_done) * 6 + L) * 3 + e] = globaltimer();
    };
    uint32_t prod = 0;  // A productions published (layer 0 and every hidden layer)
    auto signal = [&](int c) {
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(act_cl + 8 * (8 * (prod & 1) + c));
    };
    // Rewrite 16 columns [c0, c0 + 16) of region `reg` for this thread's row:
    // value rows σ(tab), tangent rows σ'(tab)·m with m the accumulator (hidden
    // layers) or W0'[:, j−1] (layer 0). Padding rows (p >= npc) read node 0's
    // table: finite, and rows are independent through every MMA, so they never
    // reach a stored output.
    // m: the accumulator columns, loaded (tcgen05.ld, asynchronous) by the caller.
    auto finish16 = [&](uint32_t reg, int c0, const float (&m)[16]) {
      float t[16];
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(t + i) = *reinterpret_cast<const float4*>(my_tab + c0 + i);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 16; ++i) t[i] = to_tf32(j == 0 ? t[i] : t[i] * m[i]);
      tmem_st16(reg + lane_base + c0, t);
    };
    auto rewrite16_layer0 = [&](uint32_t reg, int c0) {
      float t[16], m[16];
      const int jw = j > 0 ? j - 1 : 0;
#pragma unroll
      for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(t + i) = *reinterpret_cast<const float4*>(my_tab0 + c0 + i);
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = w0s[(c0 + i) * n_in + jw];
#pragma unroll
      for (int i = 0; i < 16; ++i) t[i] = to_tf32(j == 0 ? t[i] : t[i] * m[i]);
      tmem_st16(reg + lane_base + c0, t);
    };
    // K-chunks c in [c_lo, c_hi) in MMA order: warp half h takes columns
    // 32c + 16h .. + 16 of every chunk, then the chunk is published.
    auto rewrite_chunks0 = [&](uint32_t reg, int c_lo, int c_hi, int L) {
#pragma unroll 1
      for (int c = c_lo; c < c_hi; ++c) {
        rewrite16_layer0(reg, 32 * c + 16 * h);
        signal(c);
        if (c == 0) trace(L, 1);
        if (c == c_hi - 1) trace(L, 2);
      }
    };
    // σ, σ' of nodes [0, npc) for columns [n_lo, n_lo + n_cnt) into the tables,
    // thread = (column, 4-node pass); pre = accumulator + bias (hidden layers).
    auto sigma_cols = [&](int n_lo, int n_cnt, const float* bias) {
      for (int w = etid; w < n_cnt * ((npc + 3) >> 2); w += 256) {
        const int n = n_lo + w % n_cnt, p0 = 4 * (w / n_cnt);
        const float bj = bias[n];
        float pv[4], val[4], sp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = pre_t[(p0 + u) * kRowsTabStride + n] + bj;
#pragma unroll
        for (int u = 0; u < 4; ++u) act_rows<ACT>(pv[u], val[u], sp[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          tab[(p0 + u) * 2 * kRowsTabStride + n] = val[u];
          tab[(p0 + u) * 2 * kRowsTabStride + kRowsTabStride + n] = sp[u];
        }
      }
    };
    // Value rows (TMEM lanes 0..npc-1, quadrant 0) of columns [n_lo, n_lo + 32·x4)
    // to pre_t. The 16x256b shape reads only lanes 0..15 (half the bytes of a
    // 32-lane load; TMEM reads run at ~64 B/clk per SM): thread t gets lanes
    // t/4 and t/4 + 8, columns 8i + 2(t%4) + {0, 1} (scripts/tmem_shape_probe.cu).
    auto publish_values = [&](uint32_t reg, int n_lo, int n_cnt) {
      if (q != 0) return;
      const int a = lane >> 2, cc = 2 * (lane & 3);
      float* d0 = pre_t + a * kRowsTabStride + cc;
      float* d1 = d0 + 8 * kRowsTabStride;
#pragma unroll 1
      for (int s = n_lo; s < n_lo + n_cnt; s += 64) {
        uint32_t v[32];
        tmem_ld_16x256b_x8(reg + s, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (a < npc) *reinterpret_cast<float2*>(d0 + s + 8 * i) = make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
          if (a + 8 < npc)
            *reinterpret_cast<float2*>(d1 + s + 8 * i) = make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
    };

    // z element (node zp, input zk) of this thread (npc·n_in <= 256): loaded one
    // tile ahead into a register so its global latency hides behind the hidden layers
    const int zp = etid / n_in, zk = etid - zp * n_in;
    const bool zown = etid < npc * n_in;
    auto fetch_z = [&](long long tile) -> float {
      const long long node = tile * (2 * npc) + static_cast<long long>(rank) * npc + zp;
      return (zown && tile < prm.num_tiles && node < prm.K) ? static_cast<float>(load_z(prm, node, zk)) : 0.0f;
    };
    // Layer-0 σ, σ' tables of `tile` into tab0 (z staged from the register
    // prefetch). Runs while the tensor core works on the previous tile's output
    // layer, so the next tile's first K-chunk follows its output epilogue directly.
    float znext = fetch_z(pair);
    auto layer0_tables = [&](long long tile) {
      if (zown) zs[zp * 32 + zk] = znext;
      named_bar(3, 256);
      znext = fetch_z(tile + npairs);
      const int n = etid;  // neuron
      const float bj = __ldg(prm.b0 + n);
      float w[kRowsMaxIn];
#pragma unroll
      for (int k = 0; k < kRowsMaxIn; ++k) w[k] = k < n_in ? w0s[n * n_in + k] : 0.0f;
#pragma unroll 1
      for (int p0 = 0; p0 < npc; p0 += 4) {  // four independent chains per pass
        float pre[4], val[4], sp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pre[u] = bj;
#pragma unroll
        for (int k = 0; k < kRowsMaxIn; ++k)
          if (k < n_in) {
#pragma unroll
            for (int u = 0; u < 4; ++u) pre[u] = fmaf(w[k], zs[(p0 + u) * 32 + k], pre[u]);
          }
#pragma unroll
        for (int u = 0; u < 4; ++u) act_rows<ACT>(pre[u], val[u], sp[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          tab0[(p0 + u) * 2 * kRowsTabStride + n] = val[u];
          tab0[(p0 + u) * 2 * kRowsTabStride + kRowsTabStride + n] = sp[u];
        }
      }
      named_bar(3, 256);
    };
    // Tables (values → σ, σ') of the hidden-layer columns [n_lo, n_lo + n_cnt)
    // (n_cnt = 64 or 192; the value-row loads split over both halves' quadrant-0 warps).
    auto table_stage = [&](uint32_t reg, int n_lo, int n_cnt, const float* bias) {
      if (n_cnt == 64) {
        if (h == 0) publish_values(reg, n_lo, 64);
      } else {
        if (h == 0) publish_values(reg, n_lo, 64);
        else publish_values(reg, n_lo + 64, n_cnt - 64);
      }
      named_bar(3, 256);
      sigma_cols(n_lo, n_cnt, bias);
      named_bar(3, 256);
    };
    layer0_tables(pair);
    rewrite_chunks0(tmem_base, 1, 8, 0);
    rewrite_chunks0(tmem_base, 0, 1, 0);
    ++prod;
    int b = 0;  // region of this tile's layer-0 output (the MMA warp tracks the same)
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node0 = tile * (2 * npc) + static_cast<long long>(rank) * npc;
      trace(0, 0);
      // ---- hidden layers: D in R_{(b+l+1)%2}, rewritten in place. The tables of
      // K-chunks c+2, c+3 are built while chunk c+1's accumulator load is in flight.
      for (int l = 0; l < n_mma; ++l, ++hl) {
        const uint32_t reg = tmem_base + ((b + l + 1) & 1) * 256;
        mbar_wait(tmem_full, hl & 1);
        tc_fence_after();
        trace(l + 1, 0);
        fl = l + 1;
        fine(fl, 0, 0);
        const float* bias = bhs + l * 256;
        // stage 0: tables of K-chunks 0..3; the MMAs of chunks 0..2 then cover the
        // second stage (chunks 4..7), while chunk 3's accumulator load is in flight
        table_stage(reg, 0, 128, bias);
        fine(fl, 0, 1);
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          const int c0 = 32 * c + 16 * h;
          float m[16];
          tmem_ld16(reg + lane_base + c0, m);
          if (c == 3) table_stage(reg, 128, 128, bias);
          finish16(reg, c0, m);
          signal(c);
          if (c == 0) {
            trace(l + 1, 1);
            fine(fl, 0, 2);
          }
        }
        ++prod;
        trace(l + 1, 2);
        // the next tile's layer-0 tables fill the wait for this layer's successor
        // (tab0 and zs are free once this tile's layer 0 was rewritten)
        if (l == 0 && tile + npairs < prm.num_tiles) layer0_tables(tile + npairs);
        fine(fl, 0, 3);
      }
      // ---- tile boundary. The output layer accumulates into columns 0..15 of
      // R_nb (the last hidden layer's A region, free once that layer's MMAs
      // completed); the next tile's layer 0 goes to the same region: its
      // K-chunks 1..7 now, while the tensor core runs the output layer, and
      // chunk 0 (columns 0..31) after the output accumulator has been read.
      const int nb = (b + n_mma + 1) & 1;
      const uint32_t reg_next = tmem_base + nb * 256;
      const bool more = tile + npairs < prm.num_tiles;
      if (more) {
        if (n_mma == 0) layer0_tables(tile + npairs);
        rewrite_chunks0(reg_next, 1, 8, 0);
      }
      mbar_wait(tmem_last, tiles_done & 1);
      tc_fence_after();
      if (h == 0) {
        float o[16];
        tmem_ld16(reg_next + lane_base, o);
        tmem_ld_wait();
        const long long node = node0 + p;
        const int n_out = prm.n_out;
        if (valid && node < prm.K) {
          note_nonfinite(prm, o, n_out);
          if (j == 0) {
            for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
          } else if (prm.jac != nullptr) {
            for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + (j - 1)] = static_cast<double>(o[oo]);
          }
        }
      }
      tc_fence_before();
      if (more) {
        named_bar(3, 256);  // the output accumulator has been read by both halves' rows
        rewrite_chunks0(reg_next, 0, 1, 0);
        ++prod;
      }
      b = nb;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace rtn
