// rtn_reverse.cuh — reverse-mode (adjoint) Jacobians for TF32 width-512
// models: an additional throughput mode beside the forward-mode kernels.
//
// The reference computes J with a stacked reverse sweep (BatchedCore →
// RunReverse, /root/reference/proj/src/neural.cpp:132-163): one value row
// forward, then one adjoint row per output backward — 1 + n_out = 7 MMA rows
// per node instead of forward mode's 1 + n_in = 18 (2.57x fewer FLOPs at the
// quadrotor's 17 inputs and 6 outputs). Here that is two launches of the
// split-kernel schedule (rtn_split.cuh: A = activations split between TMEM
// quarters 2-3 and shared-memory quarters 0-1, N = 128-neuron blocks into
// rotating TMEM regions, no DSMEM):
//   PASS 0 (values): rows = nodes (128 per CTA). Layer 0 on CUDA cores (fp32,
//     W0' staged in shared memory), hidden layers y = σ(d + b); every layer's
//     σ'(pre) goes to an HBM scratch [n_hidden][K][512] (the reverse sweep's
//     stored activations: 1 KB per node and layer, fp16); the output layer gives f.
//   PASS 1 (adjoints): rows = (node, output o), n_out per node. The rows start
//     as W_L'[o, :] ⊙ σ'_{H−1} (CUDA cores), each backward step is
//     y[row, k] = (Σ_n G[row, n] W_l[n, k]) · σ'_{l−1}[node, k] — an MMA with
//     the TRANSPOSED hidden pack as B — and the last one multiplies by W0'
//     (input-major copy, zero-padded to 32 rows: N = 32) to give J[o, :].
// Roofline: 2·(1 + n_out)·P_W FLOP per node (bench.py `reverse_mode`).
// The slopes are stored as fp16: σ' of tanh / SiLU / ReLU lies in [-0.1, 1.1],
// where fp16's 11 significant bits round exactly like the tf32 operands the
// adjoint MMAs consume anyway, at half the scratch traffic (the value pass
// spent 20% of its time on fp32 slope stores).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

#include "rtn_kernel.cuh"
#include "rtn_rows.cuh"
#include "rtn_split.cuh"

namespace rtn {

constexpr int kRevThreads = 320;
constexpr int kRevMaxIn = 24;       // PASS 0 stages W0' (512 x n_in fp32) in shared memory
constexpr int kRevStageNodes = 32;  // PASS 1 stages σ' blocks (nodes x 128 fp32, double-buffered) when NPC <= 32

template <int NSTAGE>
struct RevCfg {
  static constexpr uint32_t kSOff = 0;                                    // 8 chunks x 16 KB (quarters 0, 1)
  static constexpr uint32_t kStageOff = kSOff + 8 * 16384;
  static constexpr uint32_t kW0Off = kStageOff + NSTAGE * kSplitStage;    // [512][n_in] W0' (PASS 0)
  static constexpr uint32_t kZsOff = kW0Off + 512 * kRevMaxIn * 4;        // [128][kRevMaxIn] z (PASS 0)
  static constexpr uint32_t kBarOff = kZsOff + 128 * kRevMaxIn * 4;
  // full/empty[NSTAGE], act[2][16], tmem_full[2], reg_free[2], s_free, tmem_last
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 32 + 6;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kSmemBytes = kMiscOff + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
};

// PASS 0: tmap_a = the hidden pack (64-row boxes), tmap_b = the output pack (N = 16).
// PASS 1: tmap_a = the transposed hidden pack (64-row boxes), tmap_b = W0' input-major,
//         zero-padded to 32 rows (N = 32).
template <int NSTAGE, int ACT, int PASS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kRevThreads, 1)
    rtn_rev_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b) {
  using C = RevCfg<NSTAGE>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* s_act = smem + C::kSOff;
  uint8_t* stage_s = smem + C::kStageOff;
  float* w0s = reinterpret_cast<float*>(smem + C::kW0Off);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act = bars + 2 * NSTAGE;
  uint64_t* tmem_full = act + 32;
  uint64_t* reg_free = tmem_full + 2;
  uint64_t* s_free = reg_free + 2;
  uint64_t* tmem_last = s_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kMiscOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, n_out = prm.n_out, npc = prm.P;  // nodes per CTA (PASS 0: 128)
  const int n_mma = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  constexpr int kOutN = PASS == 0 ? kMaxOut : 32;           // output MMA N
  constexpr uint32_t kOutStage = PASS == 0 ? 1024 : 2048;   // its B tile per CTA

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < 32; ++c) mbar_init(&act[c], 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tmem_full[i], 1);
      mbar_init(&reg_free[i], 16);
    }
    mbar_init(s_free, 1);
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_a);
    prefetch_tmap(&tmap_b);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  if constexpr (PASS == 0)  // W0' (neuron-major) for the CUDA-core layer 0
    for (int i = threadIdx.x; i < 512 * n_in; i += blockDim.x) w0s[i] = __ldg(prm.w0 + i);
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
      for (int l = 0; l < n_mma; ++l) {
        const int wl = PASS == 0 ? l : n_mma - 1 - l;  // PASS 1 walks the layers backwards
        for (int b = 0; b < 4; ++b)
          for (int i = 0; i < 16; ++i) {
            const int c = split_chunk(i, b == 0);
            mbar_wait(&empty[st], ph ^ 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kSplitStage);
            tma_load_2sm(stage_s + st * kSplitStage, &tmap_a, c * 32, wl * 512 + b * 128 + yr, &full[st], pol);
            next();
          }
      }
      for (int i = 0; i < 16; ++i) {
        const int c = split_chunk(i, true);
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * kOutStage);
        tma_load_2sm(stage_s + st * kSplitStage, &tmap_b, c * 32, static_cast<int>(rank) * (kOutN / 2), &full[st], pol);
        next();
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) =======================
    if (leader) {
      const uint32_t idesc_h = idesc_tf32(256, 128), idesc_o = idesc_tf32(256, kOutN);
      const uint64_t w0d = sw128_desc(smem_u32(stage_s));
      const uint64_t s0d = sw128_desc(smem_u32(s_act));
      constexpr uint32_t kStageD = kSplitStage >> 4, kChunkD = 16384 >> 4;
      uint32_t ph = 0, prod = 0, layers = 0;
      int st = 0;
      int T0 = 0, T1 = 1, F0 = 2, F1 = 3;
      auto block = [&](uint32_t d, uint32_t idesc, bool wait_input, uint32_t sbar, bool first) {
        uint64_t* a_set = act + 16 * (prod & 1);
        const uint32_t par = (prod >> 1) & 1;
#pragma unroll 1
        for (int i = 0; i < 16; ++i) {
          const int c = split_chunk(i, first);
          if (wait_input && (c >= 8 || (c & 3) == 0)) mbar_wait_cluster(&a_set[c], par);
          mbar_wait(&full[st], ph);
          tc_fence_after();
          const uint64_t wd = w0d + st * kStageD;
          if (c < 8) {
            mma4_tf32_pair_commit(d, s0d + c * kChunkD, wd, idesc, i != 0, smem_u32(&empty[st]), c == 7 ? sbar : 0u);
          } else {
            const uint32_t treg = tmem_base + (c < 12 ? T0 : T1) * 128 + (c & 3) * 32;
            mma4_tf32_pair_ts_commit(d, treg, wd, idesc, i != 0, smem_u32(&empty[st]));
          }
          if (++st == NSTAGE) {
            st = 0;
            ph ^= 1;
          }
        }
      };
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
        for (int l = 0; l < n_mma; ++l, ++layers) {
          block(tmem_base + F0 * 128, idesc_h, true, 0u, true);
          mma_commit_pair(&tmem_full[0]);
          block(tmem_base + F1 * 128, idesc_h, false, 0u, false);
          mma_commit_pair(&tmem_full[1]);
          mbar_wait_cluster(&reg_free[0], layers & 1);
          tc_fence_after();
          block(tmem_base + F0 * 128, idesc_h, false, 0u, false);
          mma_commit_pair(&tmem_full[0]);
          mbar_wait_cluster(&reg_free[1], layers & 1);
          tc_fence_after();
          block(tmem_base + F1 * 128, idesc_h, false, smem_u32(s_free), false);
          mma_commit_pair(&tmem_full[1]);
          ++prod;
          const int t0 = T0, t1 = T1;
          T0 = F0;
          T1 = F1;
          F0 = t0;
          F1 = t1;
        }
        block(tmem_base + F0 * 128, idesc_o, true, 0u, true);  // output: f (PASS 0) or J (PASS 1)
        mma_commit_pair(tmem_last);
        ++prod;
      }
    }
  } else if (warp >= 2) {
    // ===================== epilogue (8 warps per CTA) ==========================
    const int q4 = warp & 3, h = (warp - 2) >> 2;
    const int r = q4 * 32 + lane;  // TMEM lane = tile row of this CTA
    // PASS 0: row = node r. PASS 1: row = (node r / n_out, output r % n_out).
    const int p = PASS == 0 ? r : r / n_out;
    const int o = PASS == 0 ? 0 : r - p * n_out;
    const bool valid = p < npc;
    const uint32_t lane_base = static_cast<uint32_t>(q4 * 32) << 16;
    const uint32_t act_cl = mapa(smem_u32(act), 0);
    const uint32_t rf_cl = mapa(smem_u32(reg_free), 0);
    const uint32_t s_base = smem_u32(s_act);
    uint32_t prod = 0, layers = 0, tf_use[2] = {0, 0}, tiles_done = 0;
    int T0 = 0, T1 = 1, F0 = 2, F1 = 3;
    long long node = 0;  // this row's node in the chunk (the scratch index)

    auto signal_tmem = [&](int c) {
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(act_cl + 8 * (16 * (prod & 1) + c));
    };
    auto signal_smem = [&](int c) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(act_cl + 8 * (16 * (prod & 1) + c));
    };
    // σ' row (fp16) of this thread's node for layer li (PASS 1 reads, PASS 0 writes)
    uint16_t* const rs = reinterpret_cast<uint16_t*>(prm.rev_s);
    auto srow = [&](int li) -> uint16_t* {
      const long long nd = node < prm.K ? node : 0;
      return rs + (static_cast<long long>(li) * prm.K + nd) * 512;
    };
    auto pack8 = [](const float* v) {  // 8 floats → 8 fp16 (16 bytes)
      uint4 u;
      __half2 h;
      h = __floats2half2_rn(v[0], v[1]);
      u.x = *reinterpret_cast<uint32_t*>(&h);
      h = __floats2half2_rn(v[2], v[3]);
      u.y = *reinterpret_cast<uint32_t*>(&h);
      h = __floats2half2_rn(v[4], v[5]);
      u.z = *reinterpret_cast<uint32_t*>(&h);
      h = __floats2half2_rn(v[6], v[7]);
      u.w = *reinterpret_cast<uint32_t*>(&h);
      return u;
    };
    auto unpack8 = [](uint4 u, float* v) {
      uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 f = __half22float2(*reinterpret_cast<__half2*>(&w[i]));
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      }
    };
    // PASS 1: σ'_li of the CTA's nodes for one 128-column block, staged in shared
    // memory (the W0' area) one block ahead by cp.async — per-piece global loads
    // left the adjoint epilogue waiting on HBM (ncu: 70% long-scoreboard stalls)
    const int etid = threadIdx.x - 64;
    const bool stage_sp = PASS == 1 && npc <= kRevStageNodes;
    uint16_t* sbuf = reinterpret_cast<uint16_t*>(w0s);
    uint32_t pf = 0, pc = 0;  // σ' blocks prefetched / consumed
    long long node0 = 0;      // the CTA's first node of the tile
    auto sp_prefetch = [&](int li, int b) {
      uint16_t* dst = sbuf + (pf & 1) * kRevStageNodes * 128;
      for (int ch = etid; ch < npc * 16; ch += 256) {  // 16-byte pieces: 8 slopes
        const int pn = ch >> 4, cq = ch & 15;
        const long long nd = node0 + pn < prm.K ? node0 + pn : 0;
        const uint16_t* src = rs + (static_cast<long long>(li) * prm.K + nd) * 512 + 128 * b + 8 * cq;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + pn * 128 + 8 * cq)), "l"(src)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++pf;
    };
    // the next block's σ' in flight, this block's complete and visible to every epilogue thread
    auto sp_ready = [&](bool more, int li_next, int b_next) {
      named_bar(3, 256);  // every thread is done with the buffer the next prefetch overwrites
      if (more) {
        sp_prefetch(li_next, b_next);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      named_bar(3, 256);
    };
    // 8 accumulator columns c0.. of region reg → σ (PASS 0, σ' to the scratch) or
    // d·σ' (PASS 1), tf32; n0 = the neuron index of column c0 in the layer
    auto finish8 = [&](uint32_t reg, int c0, int n0, int li, const float* bias, float* y) {
      float m[8];
      tmem_ld8(reg + lane_base + c0, m);
      if constexpr (PASS == 0) {
        tmem_ld_wait();
        const bool st = valid && node < prm.K && !(prm.dbg & 2);  // dbg 2: no slope stores (timing only)
        float spv[8];
#pragma unroll
        for (int hq = 0; hq < 2; ++hq) {  // 4 columns at a time: few live registers next to the held blocks
          const float4 b4 = *reinterpret_cast<const float4*>(bias + n0 + 4 * hq);
          const float b[4] = {b4.x, b4.y, b4.z, b4.w};
          float* sp = spv + 4 * hq;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float val;
            if (prm.dbg & 4) {  // dbg 4: no activation math (timing only)
              val = m[4 * hq + i] + b[i];
              sp[i] = val;
            } else {
              act_rows<ACT>(m[4 * hq + i] + b[i], val, sp[i]);
            }
            y[4 * hq + i] = to_tf32(val);
          }
        }
        if (st) *reinterpret_cast<uint4*>(srow(li) + n0) = pack8(spv);
      } else {
        float sp[8];
        if (stage_sp)
          unpack8(*reinterpret_cast<const uint4*>(sbuf + (pc & 1) * kRevStageNodes * 128 + (valid ? p : 0) * 128 + c0), sp);
        else
          unpack8(__ldg(reinterpret_cast<const uint4*>(srow(li) + n0)), sp);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = to_tf32(m[i] * sp[i]);
      }
    };
    // this thread's 64 values of block b: columns 32c + 16h + (0..15), c < 4
    auto read_block = [&](uint32_t reg, int b, int li, const float* bias, float (&y)[64]) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int c0 = 32 * (c >> 1) + 16 * h + 8 * (c & 1);
        finish8(reg, c0, 128 * b + c0, li, bias, y + 8 * c);
      }
    };
    auto rewrite_block = [&](uint32_t reg, int b, int li, const float* bias, int q) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c0 = 32 * c + 16 * h + 8 * e;
          float t[8];
          finish8(reg, c0, 128 * b + c0, li, bias, t);
          tmem_st8(reg + lane_base + c0, t);
        }
        signal_tmem(4 * q + c);
      }
    };
    auto store_s = [&](const float (&y)[64], int q) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t chunk = s_base + (4 * q + c) * 16384 + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
          const int u = 4 * h + u4;
          const uint32_t a = chunk + ((u ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(y[16 * c + 4 * u4]),
                       "f"(y[16 * c + 4 * u4 + 1]), "f"(y[16 * c + 4 * u4 + 2]), "f"(y[16 * c + 4 * u4 + 3])
                       : "memory");
        }
      }
      signal_smem(4 * q);
    };
    // layer 0 / adjoint init: 16 values of chunk c of quarter q into A (S
    // quarters are published whole by the caller after their 4th chunk)
    auto put16 = [&](const float* y, int q, int c) {
      if (q < 2) {
        const uint32_t chunk = s_base + (4 * q + c) * 16384 + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
          const uint32_t a = chunk + (((4 * h + u4) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(y[4 * u4]), "f"(y[4 * u4 + 1]),
                       "f"(y[4 * u4 + 2]), "f"(y[4 * u4 + 3])
                       : "memory");
        }
        if (c == 3) signal_smem(4 * q);
      } else {
        tmem_st16(tmem_base + (q == 2 ? T0 : T1) * 128 + lane_base + 32 * c + 16 * h, y);
        signal_tmem(4 * q + c);
      }
    };
    // ---- the first production of a tile
    auto first_layer = [&](long long tile) {
      if constexpr (PASS == 0) {
        // layer 0 (CUDA cores, fp32): this row's node, W0' from shared memory
        const long long nd = tile * (2 * npc) + static_cast<long long>(rank) * npc + r;
        float z[kRevMaxIn];
#pragma unroll
        for (int k = 0; k < kRevMaxIn; ++k) z[k] = (k < n_in && nd < prm.K) ? static_cast<float>(load_z(prm, nd, k)) : 0.0f;
#pragma unroll 1
        for (int qi = 0; qi < 4; ++qi) {
          const int q = split_quarter(qi, true);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            const int n0 = 128 * q + 32 * c + 16 * h;
            float y[16], sp[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float* w = w0s + (n0 + i) * n_in;
              float pre = __ldg(prm.b0 + n0 + i);
#pragma unroll
              for (int k = 0; k < kRevMaxIn; ++k)
                if (k < n_in) pre = fmaf(w[k], z[k], pre);
              float val;
              act_rows<ACT>(pre, val, sp[i]);
              y[i] = to_tf32(val);
            }
            if (valid && node < prm.K) {
              uint16_t* dst = srow(0) + n0;
              *reinterpret_cast<uint4*>(dst) = pack8(sp);
              *reinterpret_cast<uint4*>(dst + 8) = pack8(sp + 8);
            }
            put16(y, q, c);
          }
        }
      } else {
        // adjoint rows W_L'[o, :] ⊙ σ'_{H-1} (the last hidden layer's slopes)
        const uint16_t* src = srow(n_mma);
        const float* wlr = prm.wl + (o < n_out ? o : 0) * 512;
#pragma unroll 1
        for (int qi = 0; qi < 4; ++qi) {
          const int q = split_quarter(qi, true);
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            const int n0 = 128 * q + 32 * c + 16 * h;
            float y[16], sv[16];
            unpack8(__ldg(reinterpret_cast<const uint4*>(src + n0)), sv);
            unpack8(__ldg(reinterpret_cast<const uint4*>(src + n0 + 8)), sv + 8);
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              const float4 w4 = __ldg(reinterpret_cast<const float4*>(wlr + n0 + i));
              y[i] = to_tf32(sv[i] * w4.x);
              y[i + 1] = to_tf32(sv[i + 1] * w4.y);
              y[i + 2] = to_tf32(sv[i + 2] * w4.z);
              y[i + 3] = to_tf32(sv[i + 3] * w4.w);
            }
            put16(y, q, c);
          }
        }
      }
      ++prod;
    };

    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      node0 = tile * (2 * npc) + static_cast<long long>(rank) * npc;
      node = node0 + p;
      if (stage_sp && n_mma > 0) sp_prefetch(n_mma - 1, 0);  // the first backward step's first block
      first_layer(tile);
      for (int l = 0; l < n_mma; ++l, ++layers) {
        // PASS 0: hidden layer l produces σ'_{l+1}; PASS 1: backward step l multiplies by σ'_{n_mma-1-l}
        const int li = PASS == 0 ? l + 1 : n_mma - 1 - l;
        const float* bias = prm.bh + l * 512;
        if constexpr (PASS == 0) {  // the layer's biases in shared memory (zs area), by layer parity
          float* bs = zs + (l & 1) * 512;
          bs[etid] = __ldg(bias + etid);
          bs[etid + 256] = __ldg(bias + etid + 256);
          named_bar(3, 256);
          bias = bs;
        }
        // PASS 1: make block b's σ' ready, prefetch the next one (the next step's block 0 after block 3)
        auto sp_next = [&](int b) {  // block #pc uses prefetch #pc (buffer pc & 1)
          if (!stage_sp) return;
          const bool more = b < 3 || l + 1 < n_mma;
          sp_ready(more, b < 3 ? li : li - 1, b < 3 ? b + 1 : 0);
        };
        float y0[64], y1[64];
        mbar_wait_sleep(&tmem_full[0], tf_use[0]++ & 1);
        tc_fence_after();
        sp_next(0);
        read_block(tmem_base + F0 * 128, 0, li, bias, y0);
        ++pc;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(rf_cl);
        mbar_wait_sleep(&tmem_full[1], tf_use[1]++ & 1);
        tc_fence_after();
        sp_next(1);
        read_block(tmem_base + F1 * 128, 1, li, bias, y1);
        ++pc;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(rf_cl + 8);
        mbar_wait_sleep(&tmem_full[0], tf_use[0]++ & 1);
        tc_fence_after();
        sp_next(2);
        rewrite_block(tmem_base + F0 * 128, 2, li, bias, 2);
        ++pc;
        mbar_wait_sleep(s_free, layers & 1);
        store_s(y0, 0);
        mbar_wait_sleep(&tmem_full[1], tf_use[1]++ & 1);
        tc_fence_after();
        sp_next(3);
        rewrite_block(tmem_base + F1 * 128, 3, li, bias, 3);
        ++pc;
        store_s(y1, 1);
        ++prod;
        const int t0 = T0, t1 = T1;
        T0 = F0;
        T1 = F1;
        F0 = t0;
        F1 = t1;
      }
      // ---- output: f (PASS 0, N = 16) or J (PASS 1, N = 32 over the inputs), lane = row
      mbar_wait_sleep(tmem_last, tiles_done & 1);
      tc_fence_after();
      if (h == 0) {
        float v[32];
        tmem_ld16(tmem_base + F0 * 128 + lane_base, v);
        if constexpr (PASS == 1) tmem_ld16(tmem_base + F0 * 128 + lane_base + 16, v + 16);
        tmem_ld_wait();
        if (valid && node < prm.K) {
          if constexpr (PASS == 0) {
            note_nonfinite(prm, v, n_out);
#pragma unroll
            for (int oo = 0; oo < kMaxOut; ++oo)
              if (oo < n_out) prm.f[node * n_out + oo] = static_cast<double>(v[oo] + __ldg(prm.bl + oo));
          } else if (o < n_out) {
            note_nonfinite(prm, v, n_in);
            double* jr = prm.jac + (node * n_out + o) * n_in;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < n_in) jr[i] = static_cast<double>(v[i]);
          }
        }
      }
      tc_fence_before();
      named_bar(3, 256);  // the output accumulator and the activations are free for the next tile
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
