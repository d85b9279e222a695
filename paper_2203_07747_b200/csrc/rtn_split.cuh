// rtn_split.cuh — throughput kernel for padded width 512, TF32, order 1, with
// the activations as the MMA's A operand, SPLIT between tensor memory and
// shared memory.
//
// Why: the pair kernel (rtn_pair.cuh) keeps the activations in shared memory
// as the B operand (lane = neuron), so every block's outputs go back through
// the shared-memory port — half of them over DSMEM to the peer CTA at ~13 B/clk
// (scripts/dsmem_bench.cu) — while the weight stream already takes ~80 of the
// port's 128 B/clk at N = 144. The rows kernel (rtn_rows.cuh) removes that
// traffic at width 256 by reading A from TMEM (lane = row), but at width 512
// one layer's input alone (128 rows x 512 k fp32) fills all 512 TMEM columns.
// Here:
//   D[row, neuron] = Σ_k A[row, k] · W[neuron, k],  M = 256 tile rows (128 per
//   CTA = TMEM lanes), N = 128 neurons per block, 4 blocks per layer,
// and the layer input is stored as four 128-k quarters: quarters 0 and 1 in
// shared memory (S, 128 KB, K-major SW128: the SS MMA form) and quarters 2 and
// 3 in two 128-column TMEM regions (the TS form). The other two TMEM regions
// (F0, F1) take the accumulators. Per layer (T = the regions of quarters 2, 3):
//   B0 → F0, B1 → F1: the epilogue reads them out into registers (Y0, Y1; 64
//        values per thread each) and hands the regions back;
//   B2 → F0: rewritten in place (σ / σ'·d, tf32) — next layer's quarter 2;
//   B3 → F1: reads S first; when its S half is done (s_free) the epilogue
//        stores Y0, Y1 into S (next layer's quarters 0, 1), and when B3 is
//        done F1 is rewritten in place (quarter 3). T becomes the next F.
// Every activation stays on its SM (no DSMEM), the shared-memory port carries
// the weight tiles (8 KB/CTA per 32-k chunk), the S half of the A reads and
// 128 KB of epilogue stores per layer, and the MMA is math-bound
// (M·N/512 = 64 cycles per K = 8 step). Every block reads its K-chunks in the
// order S then T, so the next layer's B0 starts on the S quarters while the
// epilogue still rewrites F1.
//
// Rows (as rtn_rows.cuh): NPC = 128 / (1 + n_in) nodes per CTA, value row p <
// NPC, tangent row NPC + p·n_in + k; σ/σ' tables from the value rows (TMEM
// lanes 0..15, 16x256b loads) per 128-neuron block.
// Warps: 0 TMA producer, 1 MMA issuer (leader CTA), 2..9 epilogue (warp w
// reads TMEM lanes 32·(w%4).., warp half h = (w−2)/4 owns columns 16h..16h+15
// of every 32-column chunk) — 320 threads, so the two held blocks fit in
// registers (204 per thread).
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"
#include "rtn_rows.cuh"

namespace rtn {

constexpr int kSplitThreads = 320;
constexpr int kSplitStage = 8192;  // one weight stage per CTA: 64 neurons x 32 k fp32
constexpr int kSplitTab = 132;     // floats per node row of the σ/σ' tables (bank spread)
constexpr int kSplitMaxNodes = 16;
constexpr int kSplitTab0Nodes = 8;   // next tile's layer-0 σ/σ' tables precomputed when NPC <= 8 (n_in >= 15)
constexpr int kSplitTab0 = 516;      // floats per (node, σ|σ') row of those tables

#ifdef RTN_SPLIT_DEBUG
// bounded wait: reports which barrier a thread is stuck on, then traps
__device__ __forceinline__ void split_wait(uint64_t* bar, uint32_t parity, int tag, bool cl) {
  for (long long i = 0; i < (1ll << 24); ++i) {
    uint32_t ok;
    if (cl)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    else
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
  }
  printf("split hang: tag %d block %d thread %d parity %u\n", tag, blockIdx.x, threadIdx.x, parity);
  __trap();
}
#define SPW(bar, par, tag) split_wait(bar, par, tag, false)
#define SPT(i, v)                                                                                \
  do {                                                                                           \
    if (prm.trace) *reinterpret_cast<volatile unsigned long long*>(prm.trace + (i)) = (v);       \
  } while (0)
#define SPWC(bar, par, tag) split_wait(bar, par, tag, true)
#else
#define SPW(bar, par, tag) mbar_wait(bar, par)
#define SPT(i, v) \
  do {            \
  } while (0)
#define SPWC(bar, par, tag) mbar_wait_cluster(bar, par)
#endif

// K-chunk order of a block: the first block of a layer (and the output layer)
// takes the quarters in the order the epilogue finishes them — 2 (chunks 8..11,
// rewritten in place while the previous layer's B3 still ran), 0 (stored into
// S while B3 read T: those stores need the shared-memory port that S-operand
// MMAs saturate), 3 (rewritten once B3 is done), 1 (stored last); the other
// blocks S then T, so B3 frees S at its midpoint.
__host__ __device__ constexpr int split_quarter(int qi, bool first) { return first ? (0x1302 >> (4 * qi)) & 15 : qi; }
__host__ __device__ constexpr int split_chunk(int i, bool first) { return 4 * split_quarter(i >> 2, first) + (i & 3); }

template <int NSTAGE>
struct SplitCfg {
  static constexpr uint32_t kSOff = 0;                                    // 8 chunks x 16 KB (quarters 0, 1)
  static constexpr uint32_t kStageOff = kSOff + 8 * 16384;
  static constexpr uint32_t kPreOff = kStageOff + NSTAGE * kSplitStage;   // [16][132] value-row pre
  static constexpr uint32_t kTabOff = kPreOff + kSplitMaxNodes * kSplitTab * 4;      // [16][2][132] σ, σ'
  static constexpr uint32_t kZsOff = kTabOff + kSplitMaxNodes * 2 * kSplitTab * 4;   // [16][32] z
  static constexpr uint32_t kTab0Off = kZsOff + kSplitMaxNodes * 32 * 4;                // [8][2][516] layer-0 σ, σ'
  static constexpr uint32_t kBarOff = kTab0Off + kSplitTab0Nodes * 2 * kSplitTab0 * 4;
  // full/empty[NSTAGE], act[2][16], tmem_full[2], reg_free[2], s_free, tmem_last
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 32 + 6;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kSmemBytes = kMiscOff + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

template <int NSTAGE, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSplitThreads, 1)
    rtn_split_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                     const __grid_constant__ CUtensorMap tmap_l) {
  using C = SplitCfg<NSTAGE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* s_act = smem + C::kSOff;
  uint8_t* stage_s = smem + C::kStageOff;
  float* pre_t = reinterpret_cast<float*>(smem + C::kPreOff);
  float* tab = reinterpret_cast<float*>(smem + C::kTabOff);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);
  float* tab0 = reinterpret_cast<float*>(smem + C::kTab0Off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act = bars + 2 * NSTAGE;  // [2][16]: K-chunk c of production n in set n & 1
  uint64_t* tmem_full = act + 32;     // [2]: blocks 0, 2 / blocks 1, 3
  uint64_t* reg_free = tmem_full + 2; // [2]: the epilogue has drained F0 / F1
  uint64_t* s_free = reg_free + 2;    // B3's shared-memory half is done
  uint64_t* tmem_last = s_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, npc = prm.P;
  const int n_mma = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < 32; ++c) mbar_init(&act[c], 16);  // 8 epilogue warps x 2 CTAs
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&reg_free[i], 16);
    }
    mbar_init(s_free, 1);
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
          for (int i = 0; i < 16; ++i) {
            const int c = split_chunk(i, b == 0);
            if (lane == 0) SPT(rank, (tile << 32) | (l << 16) | (b << 8) | c);
            SPW(&empty[st], ph ^ 1, 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kSplitStage);
            tma_load_2sm(stage_s + st * kSplitStage, &tmap_h, c * 32, l * 512 + b * 128 + yr, &full[st], pol);
            next();
          }
      for (int i = 0; i < 16; ++i) {
        const int c = split_chunk(i, true);
        SPW(&empty[st], ph ^ 1, 2);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * 1024);
        tma_load_2sm(stage_s + st * kSplitStage, &tmap_l, c * 32, static_cast<int>(rank) * 8, &full[st], pol);
        next();
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) =======================
    if (leader) {
      const uint32_t idesc_h = idesc_tf32(256, 128), idesc_o = idesc_tf32(256, kMaxOut);
      const uint64_t w0d = sw128_desc(smem_u32(stage_s));
      const uint64_t s0d = sw128_desc(smem_u32(s_act));
      constexpr uint32_t kStageD = kSplitStage >> 4, kChunkD = 16384 >> 4;
      uint32_t ph = 0, prod = 0, layers = 0, tf_use[2] = {0, 0};
      int st = 0;
      int T0 = 0, T1 = 1, F0 = 2, F1 = 3;  // TMEM regions: quarters 2, 3 / accumulators
      (void)tf_use;
      // one 128-neuron block (or the output layer), K-chunks in split_chunk order
      const bool stream_only = prm.dbg & 128;  // dbg 128: weight stream + MMAs only (timing)
      const bool tr_pair = prm.trace && pair == 0 && !(prm.dbg & 256);
      long long tix = 0;
      unsigned long long* tchunk = nullptr;  // RTN_TRACE: per-chunk issue times of one B0 (layer 5)
      auto block = [&](uint32_t d, uint32_t idesc, bool wait_input, uint32_t sbar, bool first) {
        wait_input = wait_input && !stream_only;
        uint64_t* a_set = act + 16 * (prod & 1);
        const uint32_t par = (prod >> 1) & 1;
#pragma unroll 1
        for (int i = 0; i < 16; ++i) {
          const int c = split_chunk(i, first);
          if (lane == 0) SPT(2, (static_cast<unsigned long long>(prod) << 32) | (wait_input << 16) | c);
          // S quarters are published whole (one proxy fence per warp and quarter):
          // their barrier is the one of the quarter's first chunk
          if (wait_input && (c >= 8 || (c & 3) == 0)) SPWC(&a_set[c], par, 100 + c);
          if (lane == 0) SPT(3, (static_cast<unsigned long long>(prod) << 32) | c);
          if (tchunk) tchunk[2 * i] = globaltimer();
          SPW(&full[st], ph, 3);
          tc_fence_after();
          if (tchunk) tchunk[2 * i + 1] = globaltimer();
          const uint64_t wd = w0d + st * kStageD;
          // dbg 512 / 1024 (with 128; timing only): every chunk's A from S / from T
          const bool from_s = (prm.dbg & 512) ? true : ((prm.dbg & 1024) ? false : c < 8);
          if (from_s) {
            mma4_tf32_pair_commit(d, s0d + (c & 7) * kChunkD, wd, idesc, i != 0, smem_u32(&empty[st]),
                                  c == 7 ? sbar : 0u);
          } else {
            const uint32_t treg = tmem_base + ((c & 7) < 4 ? T0 : T1) * 128 + (c & 3) * 32;
            mma4_tf32_pair_ts_commit(d, treg, wd, idesc, i != 0, smem_u32(&empty[st]));
            if (c == 7 && sbar) mma_commit_pair(s_free);  // dbg 1024 only: S is never read
          }
          if (++st == NSTAGE) {
            st = 0;
            ph ^= 1;
          }
        }
      };
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tix) {
        const bool tr = tr_pair && tix == prm.trace_tile && lane == 0;
        for (int l = 0; l < n_mma; ++l, ++layers) {
          if (tr && l < 11) prm.trace[l * 5] = globaltimer();
          tchunk = (tr && l == 4) ? prm.trace + 200 : nullptr;
          block(tmem_base + F0 * 128, idesc_h, true, 0u, true);
          tchunk = nullptr;
          mma_commit_pair(&tmem_full[0]);
          if (tr && l < 11) prm.trace[l * 5 + 1] = globaltimer();
          block(tmem_base + F1 * 128, idesc_h, false, 0u, false);
          mma_commit_pair(&tmem_full[1]);
          if (tr && l < 11) prm.trace[l * 5 + 2] = globaltimer();
          if (!stream_only) SPWC(&reg_free[0], layers & 1, 4);  // Y0 read out of F0
          tc_fence_after();
          block(tmem_base + F0 * 128, idesc_h, false, 0u, false);
          mma_commit_pair(&tmem_full[0]);
          if (tr && l < 11) prm.trace[l * 5 + 3] = globaltimer();
          if (!stream_only) SPWC(&reg_free[1], layers & 1, 5);  // Y1 read out of F1
          tc_fence_after();
          block(tmem_base + F1 * 128, idesc_h, false, smem_u32(s_free), false);
          mma_commit_pair(&tmem_full[1]);
          if (tr && l < 11) prm.trace[l * 5 + 4] = globaltimer();
          ++prod;
          const int t0 = T0, t1 = T1;  // quarters 2, 3 of the next layer are F0, F1 (in place)
          T0 = F0;
          T1 = F1;
          F0 = t0;
          F1 = t1;
        }
        // output layer (N = 16) into columns 0..15 of F0
        block(tmem_base + F0 * 128, idesc_o, true, 0u, true);
        mma_commit_pair(tmem_last);
        ++prod;
      }
    }
  } else if (warp >= 2 && (prm.dbg & 128)) {
    // timing aid: drain the MMA completions only (outputs are not written)
    uint32_t u0 = 0, u1 = 0, ly = 0;
    for (long long tile = pair, td = 0; tile < prm.num_tiles; tile += npairs, ++td) {
      for (int l = 0; l < n_mma; ++l, ++ly) {
        mbar_wait_sleep(&tmem_full[0], u0++ & 1);
        mbar_wait_sleep(&tmem_full[1], u1++ & 1);
        mbar_wait_sleep(&tmem_full[0], u0++ & 1);
        mbar_wait_sleep(s_free, ly & 1);
        mbar_wait_sleep(&tmem_full[1], u1++ & 1);
      }
      mbar_wait_sleep(tmem_last, td & 1);
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
    const uint32_t s_base = smem_u32(s_act);
    uint32_t prod = 0, layers = 0, tf_use[2] = {0, 0}, tiles_done = 0;
    int T0 = 0, T1 = 1, F0 = 2, F1 = 3;

    // chunk c of the current production is complete in this warp's rows
    auto mark = [&](unsigned long long code) {
      if (lane == 0) SPT(8 + rank * 8 + (warp - 2), code);
    };
    (void)mark;
    auto signal_tmem = [&](int c) {
      mark(1000000ull + prod * 100 + c);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(act_cl + 8 * (16 * (prod & 1) + c));
    };
    auto signal_smem = [&](int c) {
      mark(2000000ull + prod * 100 + c);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(act_cl + 8 * (16 * (prod & 1) + c));
    };
    // value rows (TMEM lanes 0..npc-1, quadrant 0) of a 128-column region → pre_t
    auto publish_values = [&](uint32_t reg) {
      if (q4 != 0) return;
      const int a = lane >> 2, cc = 2 * (lane & 3);
      float* d0 = pre_t + a * kSplitTab + cc;
      float* d1 = d0 + 8 * kSplitTab;
#pragma unroll 1
      for (int s = 64 * h; s < 64 * h + 64; s += 32) {  // warp 4 (h = 0): columns 0..63, warp 8: 64..127
        uint32_t v[16];
        tmem_ld_16x256b_x4(reg + s, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (a < npc) *reinterpret_cast<float2*>(d0 + s + 8 * i) = make_float2(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]));
          if (a + 8 < npc)
            *reinterpret_cast<float2*>(d1 + s + 8 * i) = make_float2(__uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
        }
      }
    };
    // σ, σ' of nodes [0, npc) x the block's 128 columns into tab (bias: 128 floats)
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
    // this thread's 64 values of a 128-column accumulator region: columns
    // 32c + 16h + i, c < 4, as σ (value row) or σ'·d (tangent row), tf32
    auto read_block = [&](uint32_t reg, float (&y)[64]) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // 8-column pieces (the other held block is live)
        const int c0 = 32 * (c >> 1) + 16 * h + 8 * (c & 1);
        float m[8], t[8];
        tmem_ld8(reg + lane_base + c0, m);
        *reinterpret_cast<float4*>(t) = *reinterpret_cast<const float4*>(my_tab + c0);
        *reinterpret_cast<float4*>(t + 4) = *reinterpret_cast<const float4*>(my_tab + c0 + 4);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) y[8 * c + i] = to_tf32(j == 0 ? t[i] : t[i] * m[i]);
      }
    };
    // in-place rewrite of an accumulator region (next layer's quarter q), chunk by chunk
    auto rewrite_block = [&](uint32_t reg, int q) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // 8-column pieces: few live registers next to the held blocks
          const int c0 = 32 * c + 16 * h + 8 * e;
          float m[8], t[8];
          tmem_ld8(reg + lane_base + c0, m);
          *reinterpret_cast<float4*>(t) = *reinterpret_cast<const float4*>(my_tab + c0);
          *reinterpret_cast<float4*>(t + 4) = *reinterpret_cast<const float4*>(my_tab + c0 + 4);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 8; ++i) t[i] = to_tf32(j == 0 ? t[i] : t[i] * m[i]);
          tmem_st8(reg + lane_base + c0, t);
        }
        signal_tmem(4 * q + c);
      }
    };
    // 64 held values → quarter q (0 or 1) of S (SW128, row r), published whole:
    // the proxy fence + cluster-release arrive cost ~1 K cycles per warp, so
    // once per quarter instead of once per chunk
    auto store_s = [&](const float (&y)[64], int q) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t chunk = s_base + (4 * q + c) * 16384 + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {  // 16-byte units 4h + u4 of the 128-byte row
          const int u = 4 * h + u4;
          const uint32_t a = chunk + ((u ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(y[16 * c + 4 * u4]),
                       "f"(y[16 * c + 4 * u4 + 1]), "f"(y[16 * c + 4 * u4 + 2]), "f"(y[16 * c + 4 * u4 + 3])
                       : "memory");
        }
      }
      signal_smem(4 * q);
    };
    // ---- layer 0 (CUDA cores), quarter by quarter: σ, σ' tables of its 128
    // neurons, then this thread's 64 columns: σ (value row) or σ'·W0'[n, k]
    const int zp = etid / n_in, zk = etid - zp * n_in;
    const bool zown = etid < npc * n_in;
    auto fetch_z = [&](long long tile) -> float {
      const long long node = tile * (2 * npc) + static_cast<long long>(rank) * npc + zp;
      return (zown && tile < prm.num_tiles && node < prm.K) ? static_cast<float>(load_z(prm, node, zk)) : 0.0f;
    };
    float znext = fetch_z(pair);
    // RTN_TRACE tile-boundary events: CTA 0 of pair 0, warp 2 lane 0, the tile after trace_tile
    auto tb = [&](int e) {
      if (prm.trace && pair == 0 && rank == 0 && warp == 2 && lane == 0 &&
          tiles_done == static_cast<uint32_t>(prm.trace_tile) + 1)
        prm.trace[180 + e] = globaltimer();
    };
    // ---- layer 0 with precomputed tables (npc <= 8): the σ, σ' of all 512
    // neurons for the next tile are computed in the epilogue's idle time of the
    // current tile's first hidden layer, so the tile boundary only stores.
    const bool pre0 = npc <= kSplitTab0Nodes;
    const float* my_tab0 = tab0 + ((valid ? p : 0) * 2 + (j == 0 ? 0 : 1)) * kSplitTab0;
    // quarter q of the tables (q = 0 first stages z of `tile` from znext and
    // prefetches the tile after); one quarter per idle window
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
    // this thread's 64 values of quarter q from tab0: W0'[n, k] loads first
    auto layer0_quarter = [&](int q, float (&y)[64]) {
      const int jw = j > 0 ? j - 1 : 0;
      const float* w0r = prm.w0 + (128 * q + 16 * h) * n_in + jw;
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 16; ++i) y[16 * c + i] = __ldg(w0r + (32 * c + i) * n_in);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int c0 = 128 * q + 32 * c + 16 * h;
        float t[16];
#pragma unroll
        for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(t + i) = *reinterpret_cast<const float4*>(my_tab0 + c0 + i);
#pragma unroll
        for (int i = 0; i < 16; ++i) y[16 * c + i] = to_tf32(j == 0 ? t[i] : t[i] * y[16 * c + i]);
      }
    };
    auto layer0_pre = [&]() {
#pragma unroll 1
      for (int qi = 0; qi < 4; ++qi) {
        const int q = split_quarter(qi, true);  // the order the first block reads them
        float y[64];
        layer0_quarter(q, y);
        if (q < 2) {
          store_s(y, q);
        } else {
          const uint32_t reg = tmem_base + (q == 2 ? T0 : T1) * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_st16(reg + lane_base + 32 * c + 16 * h, y + 16 * c);
            signal_tmem(4 * q + c);
          }
        }
        tb(3 + 2 * qi);
        tb(4 + 2 * qi);
      }
      ++prod;
    };
    auto layer0 = [&](long long tile) {
      mark(1);
      tb(2);
      if (zown) zs[zp * 32 + zk] = znext;
      named_bar(3, 256);
      mark(2);
      znext = fetch_z(tile + npairs);
      const int jw = j > 0 ? j - 1 : 0;
#pragma unroll 1
      for (int qi = 0; qi < 4; ++qi) {
        const int q = split_quarter(qi, true);  // the order the first block reads them
        mark(10 + q);
        // tables: thread = (neuron n of the quarter, 4-node group); the W0' column
        // loads are all issued before the FMAs (one L2 round trip, not n_in)
        for (int w = etid; w < 128 * ((npc + 3) >> 2); w += 256) {
          const int n = w & 127, p0 = 4 * (w >> 7), ng = 128 * q + n;
          float pre[4], wk[kRowsMaxIn];
          const float bj = __ldg(prm.b0 + ng);
#pragma unroll
          for (int k = 0; k < kRowsMaxIn; ++k) wk[k] = k < n_in ? __ldg(prm.w0t + k * 512 + ng) : 0.0f;
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
            float val, sp;
            act_rows<ACT>(pre[u], val, sp);
            tab[(p0 + u) * 2 * kSplitTab + n] = val;
            tab[(p0 + u) * 2 * kSplitTab + kSplitTab + n] = sp;
          }
        }
        named_bar(3, 256);
        tb(3 + 2 * qi);
        // W0'[n, k] of this tangent row from the neuron-major copy: a warp's rows
        // are consecutive inputs k of one or two nodes, so each load is coalesced;
        // all 64 are issued before use (one L1/L2 round trip)
        float y[64];
        const float* w0r = prm.w0 + (128 * q + 16 * h) * n_in + jw;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) y[16 * c + i] = __ldg(w0r + (32 * c + i) * n_in);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int c0 = 32 * c + 16 * h;
          float t[16];
#pragma unroll
          for (int i = 0; i < 16; i += 4) *reinterpret_cast<float4*>(t + i) = *reinterpret_cast<const float4*>(my_tab + c0 + i);
#pragma unroll
          for (int i = 0; i < 16; ++i) y[16 * c + i] = to_tf32(j == 0 ? t[i] : t[i] * y[16 * c + i]);
        }
        if (q < 2) {
          store_s(y, q);
        } else {
          const uint32_t reg = tmem_base + (q == 2 ? T0 : T1) * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_st16(reg + lane_base + 32 * c + 16 * h, y + 16 * c);
            signal_tmem(4 * q + c);
          }
        }
        tb(4 + 2 * qi);
        named_bar(3, 256);  // tab is rewritten by the next quarter
      }
      ++prod;
    };

    if (pre0)  // the first tile's; later ones during the previous tile's first hidden layers
      for (int q = 0; q < 4; ++q) layer0_tables(pair, q);
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node0 = tile * (2 * npc) + static_cast<long long>(rank) * npc;
      tb(2);
      if (pre0) {
        for (int q = n_mma < 4 ? n_mma : 4; q < 4 && tiles_done > 0; ++q) layer0_tables(tile, q);  // short nets
        named_bar(3, 256);  // tab0 complete
        layer0_pre();
      } else {
        layer0(tile);
      }
      for (int l = 0; l < n_mma; ++l, ++layers) {
        const float* bias = prm.bh + l * 512;
        // RTN_TRACE: CTA 0 of pair 0, warp 2 lane 0, tile trace_tile: 10 events per layer at 64 + 10·l
        unsigned long long* te = (prm.trace && pair == 0 && rank == 0 && warp == 2 && lane == 0 &&
                                  tiles_done == static_cast<uint32_t>(prm.trace_tile) && l < 11)
                                     ? prm.trace + 64 + 10 * l
                                     : nullptr;
        auto ev = [&](int e) {
          if (te) te[e] = globaltimer();
        };
        float y0[64], y1[64];
        // B0 (F0) → registers
        SPW(&tmem_full[0], tf_use[0]++ & 1, 10);
        tc_fence_after();
        ev(0);
        tables(tmem_base + F0 * 128, bias);
        read_block(tmem_base + F0 * 128, y0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(rf_cl);
        // the next tile's layer-0 tables fill the wait for B1 (tab0 and zs are
        // free: this tile's layer 0 has been stored)
        if (pre0 && l < 4 && tile + npairs < prm.num_tiles) layer0_tables(tile + npairs, l);
        ev(1);
        // B1 (F1) → registers
        SPW(&tmem_full[1], tf_use[1]++ & 1, 11);
        tc_fence_after();
        ev(2);
        tables(tmem_base + F1 * 128, bias + 128);
        read_block(tmem_base + F1 * 128, y1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(rf_cl + 8);
        ev(3);
        // B2 (F0) rewritten in place: next layer's quarter 2
        SPW(&tmem_full[0], tf_use[0]++ & 1, 12);
        tc_fence_after();
        ev(4);
        tables(tmem_base + F0 * 128, bias + 256);
        rewrite_block(tmem_base + F0 * 128, 2);
        ev(5);
        // B3 has read S: the held blocks become quarters 0 and 1
        SPW(s_free, layers & 1, 13);
        ev(6);
        store_s(y0, 0);
        ev(7);
        // B3 (F1) rewritten in place: quarter 3
        SPW(&tmem_full[1], tf_use[1]++ & 1, 14);
        tc_fence_after();
        ev(8);
        tables(tmem_base + F1 * 128, bias + 384);
        rewrite_block(tmem_base + F1 * 128, 3);
        store_s(y1, 1);
        ev(9);
        ++prod;
        const int t0 = T0, t1 = T1;
        T0 = F0;
        T1 = F1;
        F0 = t0;
        F1 = t1;
      }
      // ---- output layer: columns 0..15 of F0, lane = row
      mark(3);
      SPW(tmem_last, tiles_done & 1, 15);
      mark(4);
      if (prm.trace && pair == 0 && rank == 0 && warp == 2 && lane == 0 &&
          tiles_done == static_cast<uint32_t>(prm.trace_tile))
        prm.trace[180] = globaltimer();
      tc_fence_after();
      if (h == 0) {
        float o[16];
        tmem_ld16(tmem_base + F0 * 128 + lane_base, o);
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
      named_bar(3, 256);  // the output accumulator has been read before the next tile's layer 0
      if (prm.trace && pair == 0 && rank == 0 && warp == 2 && lane == 0 &&
          tiles_done == static_cast<uint32_t>(prm.trace_tile))
        prm.trace[181] = globaltimer();
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
