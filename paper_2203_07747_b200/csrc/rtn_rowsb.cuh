// rtn_rowsb.cuh — throughput kernel for padded width 512 in single-pass BF16
// mode, order 1, with the whole layer input as the MMA's A operand in TENSOR
// memory.
//
// A bf16 activation row of width 512 packs two k per 32-bit TMEM column, so a
// layer's input (128 rows x 512 k per CTA) takes 256 of the 512 columns — the
// rows-orientation kernel that cannot exist at width 512 in TF32 (rtn_split.cuh
// header) fits here, with no activation ever written to shared memory:
//   D[row, neuron] = Σ_k A[row, k] · W[neuron, k],  M = 256 tile rows (128 per
//   CTA = TMEM lanes), N = 128 neurons per block, 4 blocks per layer,
//   kind::f16 with A from TMEM (TS form), W from 2-SM TMA tiles (64 neurons
//   x 64 k bf16 per CTA).
// TMEM: A in columns [0, 256) (64-k chunk c at 32c), accumulators Da = 256,
// Db = 384. Per layer: B0 → Da, B1 → Db, B2 → Da, B3 → Db; the epilogue
// drains each accumulator into registers as packed bf16 (32 words per thread
// and block: σ for value rows, σ'·d for tangent rows) and hands the region
// back; when B3 is done A is dead, and Y0, Y1, Y2 go into it straight from
// registers (tcgen05.st), then Y3 once Db is drained. The weight stream is the
// only shared-memory traffic (4 KB per K = 16 step per SM: 64 B/clk against a
// 64-cycle MMA floor).
//
// Rows and tables as rtn_rows.cuh / rtn_split.cuh (NPC = 128 / (1 + n_in),
// here <= 8, i.e. n_in >= 15: the next tile's layer-0 σ/σ' tables are
// precomputed in the first hidden layers' idle windows).
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"
#include "rtn_rows.cuh"
#include "rtn_split.cuh"

namespace rtn {

constexpr int kRbThreads = 320;
constexpr int kRbStage = 8192;  // one weight stage per CTA: 64 neurons x 64 k bf16
constexpr int kRbMinIn = 15;    // NPC <= 8

template <int NSTAGE>
struct RowsBCfg {
  static constexpr uint32_t kStageOff = 0;
  static constexpr uint32_t kPreOff = kStageOff + NSTAGE * kRbStage;                  // [16][132] value-row pre
  static constexpr uint32_t kTabOff = kPreOff + kSplitMaxNodes * kSplitTab * 4;       // [16][2][132] σ, σ'
  static constexpr uint32_t kZsOff = kTabOff + kSplitMaxNodes * 2 * kSplitTab * 4;    // [16][32] z
  static constexpr uint32_t kTab0Off = kZsOff + kSplitMaxNodes * 32 * 4;             // [8][2][516] layer-0 σ, σ'
  static constexpr uint32_t kBarOff = kTab0Off + kSplitTab0Nodes * 2 * kSplitTab0 * 4;
  // full/empty[NSTAGE], act[2][8], tmem_full[2], reg_free[2], tmem_last
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 16 + 5;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kSmemBytes = kMiscOff + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// Four K = 16 bf16 pair MMAs with A in TMEM (columns a, a+8, a+16, a+24: two k
// per column) and B from a 64-k SW128 weight stage, then a multicast commit of
// the stage's empty barrier.
__device__ __forceinline__ void mma4_bf16_pair_ts_commit(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                                         uint32_t accumulate, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p, e, t;\n\t.reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t.reg .b16 m;\n\t"
      "mov.b16 m, 3;\n\t"
      "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], b2, %3, t;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a3], b3, %3, t;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], m;\n\t}" ::"r"(
          d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// Two floats as a bf16x2 word (round to nearest even): lo in bits 0..15 (the even k).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

template <int NSTAGE, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kRbThreads, 1)
    rtn_rowsb_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                     const __grid_constant__ CUtensorMap tmap_l) {
  using C = RowsBCfg<NSTAGE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stage_s = smem + C::kStageOff;
  float* pre_t = reinterpret_cast<float*>(smem + C::kPreOff);
  float* tab = reinterpret_cast<float*>(smem + C::kTabOff);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);
  float* tab0 = reinterpret_cast<float*>(smem + C::kTab0Off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act = bars + 2 * NSTAGE;  // [2][8]: 64-k chunk c of production n in set n & 1
  uint64_t* tmem_full = act + 16;     // [2]: Da / Db accumulated
  uint64_t* reg_free = tmem_full + 2; // [2]: Da / Db drained by the epilogue
  uint64_t* tmem_last = reg_free + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, npc = prm.P;
  const int n_mma = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr uint32_t kDa = 256, kDb = 384;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < 16; ++c) mbar_init(&act[c], 16);  // 8 epilogue warps x 2 CTAs
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&reg_free[i], 16);
    }
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_h);
    prefetch_tmap(&tmap_l);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer (2-SM TMA, 64 neurons per CTA) ====
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    int st = 0;
    auto next = [&]() {
      if (++st == NSTAGE) {
        st = 0;
        ph ^= 1;
      }
    };
    const int yr = static_cast<int>(rank) * 64;
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
      for (int l = 0; l < n_mma; ++l)
        for (int b = 0; b < 4; ++b)
          for (int c = 0; c < 8; ++c) {
            mbar_wait(&empty[st], ph ^ 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kRbStage);
            tma_load_2sm(stage_s + st * kRbStage, &tmap_h, c * 64, l * 512 + b * 128 + yr, &full[st], pol);
            next();
          }
      for (int c = 0; c < 8; ++c) {
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * 1024);
        tma_load_2sm(stage_s + st * kRbStage, &tmap_l, c * 64, static_cast<int>(rank) * 8, &full[st], pol);
        next();
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) =======================
    if (leader) {
      const uint32_t idesc_h = idesc_bf16(256, 128), idesc_o = idesc_bf16(256, kMaxOut);
      const uint64_t w0d = sw128_desc(smem_u32(stage_s));
      constexpr uint32_t kStageD = kRbStage >> 4;
      uint32_t ph = 0, prod = 0, uses[2] = {0, 0};
      int st = 0;
      // accumulator region r is about to be overwritten: its previous contents were drained
      auto claim = [&](int r) {
        if (uses[r] > 0) mbar_wait_cluster(&reg_free[r], (uses[r] - 1) & 1);
        ++uses[r];
        tc_fence_after();
      };
      auto block = [&](uint32_t d, uint32_t idesc, bool wait_input) {
        uint64_t* a_set = act + 8 * (prod & 1);
        const uint32_t par = (prod >> 1) & 1;
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
          if (wait_input) mbar_wait_cluster(&a_set[c], par);
          mbar_wait(&full[st], ph);
          tc_fence_after();
          mma4_bf16_pair_ts_commit(d, tmem_base + 32 * c, w0d + st * kStageD, idesc, c != 0, smem_u32(&empty[st]));
          if (++st == NSTAGE) {
            st = 0;
            ph ^= 1;
          }
        }
      };
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
        for (int l = 0; l < n_mma; ++l) {
#pragma unroll 1
          for (int b = 0; b < 4; ++b) {
            claim(b & 1);
            block(tmem_base + ((b & 1) ? kDb : kDa), idesc_h, b == 0);
            mma_commit_pair(&tmem_full[b & 1]);
          }
          ++prod;
        }
        claim(0);  // output layer (N = 16) into columns 0..15 of Da
        block(tmem_base + kDa, idesc_o, true);
        mma_commit_pair(tmem_last);
        ++prod;
      }
    }
  } else if (warp >= 2) {
    // ===================== epilogue (8 warps per CTA) ==========================
    const int q4 = warp & 3, h = (warp - 2) >> 2;
    const int etid = threadIdx.x - 64;
    const int r = q4 * 32 + lane;  // TMEM lane = tile row of this CTA
    const bool is_val = r < npc;
    const int tr = r - npc, tp = tr / n_in;
    const int p = is_val ? r : tp;
    const int j = is_val ? 0 : 1 + (tr - tp * n_in);  // 0 value, 1 + k tangent k
    const bool valid = p < npc;
    const uint32_t lane_base = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t act_cl = mapa(smem_u32(act), 0);
    const uint32_t rf_cl = mapa(smem_u32(reg_free), 0);
    const float* my_tab = tab + (valid ? p : 0) * 2 * kSplitTab + (j == 0 ? 0 : kSplitTab);
    const float* my_tab0 = tab0 + ((valid ? p : 0) * 2 + (j == 0 ? 0 : 1)) * kSplitTab0;
    uint32_t prod = 0, tf_use[2] = {0, 0}, tiles_done = 0;

    auto signal = [&](int c) {  // 64-k chunk c of the current production is in TMEM (this warp's rows)
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(act_cl + 8 * (8 * (prod & 1) + c));
    };
    auto drained = [&](int rg) {  // this warp has read accumulator region rg
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(rf_cl + 8 * rg);
    };
    // value rows (TMEM lanes 0..npc-1, quadrant 0) of a 128-column region → pre_t
    auto publish_values = [&](uint32_t reg) {
      if (q4 != 0) return;
      const int a = lane >> 2, cc = 2 * (lane & 3);
      float* d0 = pre_t + a * kSplitTab + cc;
#pragma unroll 1
      for (int s = 64 * h; s < 64 * h + 64; s += 32) {
        uint32_t v[16];
        tmem_ld_16x256b_x4(reg + s, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (a < npc) *reinterpret_cast<float2*>(d0 + s + 8 * i) = make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
      }
    };
    auto sigma_cols = [&](const float* bias) {
      for (int w = etid; w < 128 * ((npc + 3) >> 2); w += 256) {
        const int n = w & 127, p0 = 4 * (w >> 7);
        const float bj = __ldg(bias + n);
        float pv[4], val[4], sp[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pv[u] = pre_t[(p0 + u) * kSplitTab + n] + bj;
#pragma unroll
        for (int u = 0; u < 4; ++u) act_rows<ACT>(pv[u], val[u], sp[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          tab[(p0 + u) * 2 * kSplitTab + n] = val[u];
          tab[(p0 + u) * 2 * kSplitTab + kSplitTab + n] = sp[u];
        }
      }
    };
    auto tables = [&](uint32_t reg, const float* bias) {
      publish_values(reg);
      named_bar(3, 256);
      sigma_cols(bias);
      named_bar(3, 256);
    };
    // this thread's 64 neurons of a 128-column accumulator as 32 packed bf16x2
    // words: neurons 64cc + 32h + i (cc < 2, i < 32), word 16cc + i/2
    auto read_block = [&](uint32_t reg, uint32_t (&y)[32]) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c0 = 64 * cc + 32 * h + 16 * e;
          float m[16], t[16];
          tmem_ld16(reg + lane_base + c0, m);
#pragma unroll
          for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(t + i) = *reinterpret_cast<const float4*>(my_tab + c0 + i);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; i += 2)
            y[16 * cc + 8 * e + i / 2] =
                pack_bf16x2(j == 0 ? t[i] : t[i] * m[i], j == 0 ? t[i + 1] : t[i + 1] * m[i + 1]);
        }
      }
    };
    // 32 packed words → quarter q of A (64-k chunks 2q, 2q+1; this half's 16 columns of each)
    auto store_a = [&](const uint32_t (&y)[32], int q) {
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        tmem_st16u(tmem_base + lane_base + 32 * (2 * q + cc) + 16 * h, y + 16 * cc);
        signal(2 * q + cc);
      }
    };

    // ---- layer 0: the next tile's σ, σ' tables are computed one quarter per
    // idle window of the first hidden layers (rtn_split.cuh), the tile boundary
    // only forms σ / σ'·W0'[n, k] and stores into A
    const int zp = etid / n_in, zk = etid - zp * n_in;
    const bool zown = etid < npc * n_in;
    auto fetch_z = [&](long long tile) -> float {
      const long long node = tile * (2 * npc) + static_cast<long long>(rank) * npc + zp;
      return (zown && tile < prm.num_tiles && node < prm.K) ? static_cast<float>(load_z(prm, node, zk)) : 0.0f;
    };
    float znext = fetch_z(pair);
    auto layer0_tables = [&](long long tile, int q) {
      if (q == 0) {
        if (zown) zs[zp * 32 + zk] = znext;
        named_bar(3, 256);
        znext = fetch_z(tile + npairs);
      }
      for (int w = etid; w < 128 * ((npc + 3) >> 2); w += 256) {
        const int n = 128 * q + (w & 127), p0 = 4 * (w >> 7);
        float pre[4], wk[kRowsMaxIn];
        const float bj = __ldg(prm.b0 + n);
#pragma unroll
        for (int k = 0; k < kRowsMaxIn; ++k) wk[k] = k < n_in ? __ldg(prm.w0t + k * 512 + n) : 0.0f;
#pragma unroll
        for (int u = 0; u < 4; ++u) pre[u] = bj;
#pragma unroll
        for (int k = 0; k < kRowsMaxIn; ++k) {
          if (k < n_in) {
#pragma unroll
            for (int u = 0; u < 4; ++u) pre[u] = fmaf(wk[k], zs[(p0 + u) * 32 + k], pre[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (p0 + u < kSplitTab0Nodes) {
            float val, sp;
            act_rows<ACT>(pre[u], val, sp);
            tab0[((p0 + u) * 2) * kSplitTab0 + n] = val;
            tab0[((p0 + u) * 2 + 1) * kSplitTab0 + n] = sp;
          }
        }
      }
    };
    auto layer0_store = [&]() {
      const int jw = j > 0 ? j - 1 : 0;
#pragma unroll 1
      for (int q = 0; q < 4; ++q) {
        uint32_t y[32];
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int c0 = 64 * cc + 32 * h;  // 32 neurons of this half in the quarter's 64-k chunk cc
          const float* w0r = prm.w0 + (128 * q + c0) * n_in + jw;
          float wv[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) wv[i] = __ldg(w0r + i * n_in);
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float t0 = my_tab0[128 * q + c0 + i], t1 = my_tab0[128 * q + c0 + i + 1];
            y[16 * cc + i / 2] = pack_bf16x2(j == 0 ? t0 : t0 * wv[i], j == 0 ? t1 : t1 * wv[i + 1]);
          }
        }
        store_a(y, q);
      }
      ++prod;
    };

    for (int q = 0; q < 4; ++q) layer0_tables(pair, q);
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node0 = tile * (2 * npc) + static_cast<long long>(rank) * npc;
      for (int q = n_mma < 4 ? n_mma : 4; q < 4 && tiles_done > 0; ++q) layer0_tables(tile, q);  // short nets
      named_bar(3, 256);  // tab0 complete
      layer0_store();
      for (int l = 0; l < n_mma; ++l) {
        const float* bias = prm.bh + l * 512;
        uint32_t y0[32], y1[32], y2[32];
        mbar_wait_sleep(&tmem_full[0], tf_use[0]++ & 1);  // B0 (Da)
        tc_fence_after();
        tables(tmem_base + kDa, bias);
        read_block(tmem_base + kDa, y0);
        drained(0);
        if (l < 4 && tile + npairs < prm.num_tiles) layer0_tables(tile + npairs, l);
        mbar_wait_sleep(&tmem_full[1], tf_use[1]++ & 1);  // B1 (Db)
        tc_fence_after();
        tables(tmem_base + kDb, bias + 128);
        read_block(tmem_base + kDb, y1);
        drained(1);
        mbar_wait_sleep(&tmem_full[0], tf_use[0]++ & 1);  // B2 (Da)
        tc_fence_after();
        tables(tmem_base + kDa, bias + 256);
        read_block(tmem_base + kDa, y2);
        drained(0);
        mbar_wait_sleep(&tmem_full[1], tf_use[1]++ & 1);  // B3 (Db): A is dead
        tc_fence_after();
        store_a(y0, 0);
        store_a(y1, 1);
        store_a(y2, 2);
        tables(tmem_base + kDb, bias + 384);
        read_block(tmem_base + kDb, y0);
        drained(1);
        store_a(y0, 3);
        ++prod;
      }
      // ---- output layer: columns 0..15 of Da, lane = row
      mbar_wait_sleep(tmem_last, tiles_done & 1);
      tc_fence_after();
      if (h == 0) {
        float o[16];
        tmem_ld16(tmem_base + kDa + lane_base, o);
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
      drained(0);
      named_bar(3, 256);  // the output accumulator has been read before the next tile's layer 0
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
