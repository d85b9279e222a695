// rtn_rowsa.cuh — throughput kernel for padded width 512, TF32, order 1, with
// the activations as the MMA's A operand in SHARED memory ("rows" orientation,
// M = 128 pair MMAs): no DSMEM traffic at all.
//
// Why: the CTA-pair kernel (rtn_pair.cuh) splits a 512-wide layer's neurons
// over the two CTAs (M = 256 = 2 x 128 neurons) and the node rows over their
// shared memories, so half of every layer's output crosses to the peer CTA.
// Distributed shared memory moves ~13 B/clk per SM whatever the instruction
// (st.shared::cluster scalar or v4, st.async, cp.async.bulk; 128 to 1024
// threads: scripts/dsmem_bench.cu), a third of local stores, so at 12x512 the
// 72 KB per CTA and layer that cross set the layer period (8.6 µs against
// 5.2 µs for the weight stream + MMAs alone, scripts/trace_tput.py).
// Here the roles swap:
//   D[row, neuron] = Σ_k A[row, k] · W[neuron, k]
// M = 128 rows per pair (64 per CTA, each CTA's own rows as the A operand in
// its shared memory), N = 256 neurons (each CTA loads 128 weight rows of the
// 2-SM TMA tile, the B operand). With 64 rows per SM the accumulator uses the
// "2x2" TMEM layout: lanes 0-63 hold the rows x neurons 0..127 of the block,
// lanes 64-127 the same rows x neurons 128..255, each block 128 columns. Every
// CTA's D holds its own rows x all 256 neurons, so the epilogue writes only its
// own shared memory.
//
// Rows: NPC = 64 / (1 + n_in) nodes per CTA (3 for the quadrotor's 17 inputs,
// 84 % of the rows), row p < NPC the value row of node p, row NPC + k·NPC + p
// its tangent for input k. σ/σ' of a (node, neuron) come from the value rows
// through small shared tables (as rtn_rows.cuh): value lanes publish their
// pre-activations, the 256 epilogue threads evaluate σ, σ' per neuron, every
// row reads its node's entry back.
//
// Epilogue: 8 warps; warp e reads TMEM lane quadrant q = e % 4 (rows
// 32·(q%2)..+31, neuron half q/2) and columns [64·(e/4), +64) of the block, and
// writes those 64 neurons of its rows as tf32 with 16-byte stores into the
// SW128 K-major A buffer (two 32-k chunks, each published on its own barrier).
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"
#include "rtn_pair.cuh"
#include "rtn_rows.cuh"

namespace rtn {

constexpr int kRowsAMaxNodes = 8;  // table capacity: 1 + n_in >= 8 → n_in >= 7

template <int NSTAGE>
struct RowsACfg {
  static constexpr int kWP = 512, kNKC = 16, kNMB = 2, kRows = 64;
  static constexpr uint32_t kChunkBytes = kRows * 128;                          // one 32-k chunk of 64 rows
  static constexpr uint32_t kActOff = 0;                                        // 16 chunks: 128 KB
  static constexpr uint32_t kStageOff = kActOff + kNKC * kChunkBytes;
  static constexpr uint32_t kPreOff = kStageOff + NSTAGE * kStageBytes;         // [8][256] value-row pre
  static constexpr uint32_t kTabOff = kPreOff + kRowsAMaxNodes * 256 * 4;       // [8][2][256] σ, σ'
  static constexpr uint32_t kZsOff = kTabOff + kRowsAMaxNodes * 2 * 256 * 4;    // [8][32] z
  static constexpr uint32_t kBarOff = kZsOff + kRowsAMaxNodes * 32 * 4;
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 25;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kSmemBytes = kMiscOff + 16 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static_assert((kNKC % NSTAGE) == 0, "static stage indices per block");
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// ACT as a template argument (0 tanh, 1 relu, 2 SiLU), as rtn_rows.cuh.
template <int NSTAGE, int ACT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    rtn_rowsa_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                     const __grid_constant__ CUtensorMap tmap_l) {
  using C = RowsACfg<NSTAGE>;
  constexpr int NKC = C::kNKC, NMB = C::kNMB, CPG = 4, WP = C::kWP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* act_s = smem + C::kActOff;
  uint8_t* stage_s = smem + C::kStageOff;
  float* pre_t = reinterpret_cast<float*>(smem + C::kPreOff);
  float* tab = reinterpret_cast<float*>(smem + C::kTabOff);
  float* zs = reinterpret_cast<float*>(smem + C::kZsOff);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* act_ready = bars + 2 * NSTAGE;  // [16]
  uint64_t* tmem_empty = act_ready + 16;    // [2]
  uint64_t* in_free = tmem_empty + 2;       // [4]
  uint64_t* tmem_full = in_free + 4;        // [2]
  uint64_t* tmem_last = tmem_full + 2;
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
    for (int c = 0; c < 16; ++c) mbar_init(&act_ready[c], 4);  // 2 warps (row halves) x 2 CTAs
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
  if (warp == 1) tmem_alloc_pair(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer (2-SM TMA, own 128-neuron half) =====
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    const int yr = static_cast<int>(rank) * 128;
    for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
      for (int l = 0; l < n_mma; ++l)
        for (int mb = 0; mb < NMB; ++mb) {
          const int y = l * WP + mb * 256 + yr;
#pragma unroll
          for (int c = 0; c < NKC; ++c) {
            const int st = c % NSTAGE;
            mbar_wait(&empty[st], ph ^ 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kStageBytes);
            tma_load_2sm(stage_s + st * kStageBytes, &tmap_h, c * 32, y, &full[st], pol);
            if (st == NSTAGE - 1) ph ^= 1;
          }
        }
#pragma unroll
      for (int c = 0; c < NKC; ++c) {
        const int st = c % NSTAGE;
        mbar_wait(&empty[st], ph ^ 1);
        if (leader) mbar_expect_tx_elect(&full[st], 2 * kLastHalfBytes);
        tma_load_2sm(stage_s + st * kStageBytes, &tmap_l, c * 32, static_cast<int>(rank) * 8, &full[st], pol);
        if (st == NSTAGE - 1) ph ^= 1;
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) =======================
    if (leader) {
      const uint32_t idesc_h = idesc_tf32(128, 256), idesc_o = idesc_tf32(128, kMaxOut);
      const uint64_t wdesc = sw128_desc(smem_u32(stage_s));
      const uint64_t adesc = sw128_desc(smem_u32(act_s));
      constexpr uint32_t kStageD = kStageBytes >> 4, kChunkD = C::kChunkBytes >> 4;
      const bool stream_only = prm.dbg & 128;
      uint32_t ph = 0, ar = 0, use0 = 0, use1 = 0;
      auto claim_tmem = [&](int mb) {
        const uint32_t u = mb ? use1 : use0;
        if (!stream_only && u > 0) mbar_wait(&tmem_empty[mb], (u - 1) & 1);
        if (mb) ++use1;
        else ++use0;
        tc_fence_after();
      };
      auto wait_chunk = [&](int c) {
        if (stream_only) return;
        mbar_wait_cluster(&act_ready[c], ar & 1);
        tc_fence_after();
      };
      for (long long tile = pair; tile < prm.num_tiles; tile += npairs) {
        const bool tr = prm.trace && pair == 0 && tile == pair + prm.trace_tile * npairs && lane == 0;
        for (int l = 0; l < n_mma; ++l) {
#pragma unroll 1
          for (int mb = 0; mb < NMB; ++mb) {
            if (tr) prm.trace[(l * 2 + mb) * 2] = globaltimer();
            claim_tmem(mb);
            const uint32_t d = tmem_base + mb * 128;
#pragma unroll
            for (int c = 0; c < NKC; ++c) {
              const int st = c % NSTAGE;
              if (mb == 0) wait_chunk(c);
              mbar_wait(&full[st], ph);
              tc_fence_after();
              const uint32_t bar2 = (mb == NMB - 1 && (c % CPG) == CPG - 1) ? smem_u32(&in_free[c / CPG]) : 0u;
              mma4_tf32_pair_commit(d, adesc + c * kChunkD, wdesc + st * kStageD, idesc_h, c != 0,
                                    smem_u32(&empty[st]), bar2);
              if (st == NSTAGE - 1) ph ^= 1;
            }
            mma_commit_pair(&tmem_full[mb]);
            if (tr) prm.trace[(l * 2 + mb) * 2 + 1] = globaltimer();
          }
          ++ar;
        }
        // output layer: D[row, o] = Σ_k A[row, k] · W_L'[o, k] (N = 16: lanes 0-63
        // hold outputs 0..7 in columns 0..7 of block 0's region)
        claim_tmem(0);
#pragma unroll
        for (int c = 0; c < NKC; ++c) {
          const int st = c % NSTAGE;
          wait_chunk(c);
          mbar_wait(&full[st], ph);
          tc_fence_after();
          mma4_tf32_pair_commit(tmem_base, adesc + c * kChunkD, wdesc + st * kStageD, idesc_o, c != 0,
                                smem_u32(&empty[st]), 0u);
          if (st == NSTAGE - 1) ph ^= 1;
        }
        mma_commit_pair(tmem_last);
        ++ar;
      }
    }
  } else if (warp >= 4 && !(prm.dbg & 128)) {
    // ===================== epilogue (8 warps per CTA) ==========================
    const int e = warp - 4, q = warp & 3, sub = e >> 2;
    const int etid = threadIdx.x - 128;
    const int r = ((q & 1) << 5) + lane;      // this thread's row (TMEM lane within the half)
    const int nh = q >> 1;                    // neuron half of the block
    const int nb0 = nh * 128 + sub * 64;      // first of this thread's 64 neurons in the block
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t col0 = static_cast<uint32_t>(sub * 64);  // TMEM column of nb0 within the block region
    const bool is_val = r < npc;
    const int tr = r - npc, tk = tr >= 0 ? tr / npc : 0;
    const int p = is_val ? r : (tr >= 0 ? tr - tk * npc : 0);  // node of this row
    const int rows_used = npc * (1 + n_in);
    const bool valid = r < rows_used;
    const float* my_tab = tab + (valid ? p : 0) * 512 + (is_val ? 0 : 256);
    const uint32_t act_base = smem_u32(act_s);
    const uint32_t row_off = static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128);
    const uint32_t ready_cl0 = mapa(smem_u32(&act_ready[0]), 0);
    const uint32_t empty_cl0 = mapa(smem_u32(&tmem_empty[0]), 0);
    uint32_t hl = 0, tiles_done = 0;

    auto tmem_release = [&](int mb) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(empty_cl0 + 8 * mb);
    };
    auto publish = [&](int c) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ready_cl0 + 8 * c);
    };
    // 16 consecutive neurons [k0, k0 + 16) of this row (tf32-rounded) into the A buffer
    auto store16 = [&](int k0, const float* v) {
#pragma unroll
      for (int i = 0; i < 16; i += 4) {
        const int k = k0 + i;
        const uint32_t u = static_cast<uint32_t>((k >> 2) & 7);
        const uint32_t a = act_base + (k >> 5) * C::kChunkBytes + row_off + ((u ^ (r & 7)) << 4);
        st_shared_v4(a, to_tf32(v[i]), to_tf32(v[i + 1]), to_tf32(v[i + 2]), to_tf32(v[i + 3]));
      }
    };
    // σ, σ' of the block's 256 neurons for this CTA's nodes from pre_t (+ bias)
    auto sigma_tables = [&](const float* bias) {
      const int n = etid;  // neuron of the block
      const float bj = __ldg(bias + n);
#pragma unroll 1
      for (int pp = 0; pp < npc; ++pp) {
        float val, sp;
        act_rows<ACT>(pre_t[pp * 256 + n] + bj, val, sp);
        tab[pp * 512 + n] = val;
        tab[pp * 512 + 256 + n] = sp;
      }
    };
    // Hidden block mb of layer l: tables, then every row rewrites its 64 neurons.
    auto do_block = [&](int mb, int l) {
      const uint32_t reg = tmem_base + lane_base + mb * 128 + col0;
      mbar_wait_sleep(&tmem_full[mb], hl & 1);
      tc_fence_after();
      const bool tr = prm.trace && pair == 0 && tiles_done == static_cast<uint32_t>(prm.trace_tile) && warp == 4 && lane == 0;
      unsigned long long* tp = tr ? prm.trace + 48 + rank * 66 + (l * 2 + mb) * 3 : nullptr;
      if (tr) tp[0] = globaltimer();
      // value rows (lanes 0..npc-1 of quadrants 0 and 2) publish their pre-activations
      if ((q & 1) == 0) {
#pragma unroll
        for (int c0 = 0; c0 < 64; c0 += 16) {
          float v[16];
          tmem_ld16(reg + c0, v);
          tmem_ld_wait();
          if (is_val) {
#pragma unroll
            for (int i = 0; i < 16; i += 4)
              *reinterpret_cast<float4*>(pre_t + r * 256 + nb0 + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          }
        }
      }
      named_bar_sync(1, 256);
      sigma_tables(prm.bh + l * WP + mb * 256);
      named_bar_sync(1, 256);
      if (tr) tp[1] = globaltimer();
      // rows: value σ, tangent σ'·d, padding 0; two 32-neuron chunks, each published
      const int g = mb * 2 + nh;  // K-group of the next layer's input these neurons form
      float v[64];
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 16) tmem_ld16(reg + c0, v + c0);
      tmem_ld_wait();
      tmem_release(mb);
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float t = my_tab[nb0 + i];
        v[i] = !valid ? 0.0f : (is_val ? t : t * v[i]);
      }
      mbar_wait_sleep(&in_free[g], hl & 1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k0 = mb * 256 + nb0 + h * 32;
        store16(k0, v + h * 32);
        store16(k0 + 16, v + h * 32 + 16);
        publish(k0 >> 5);
      }
      if (tr) tp[2] = globaltimer();
    };
    // Layer 0 for one 256-neuron half mb: σ, σ' of pre = b0 + W0'·(z − μ) per
    // (node, neuron), then value rows σ, tangent row (k, p) σ'_p·W0'[j, k].
    auto layer0_half = [&](int mb) {
      {
        const int j = mb * 256 + etid;
        const float bj = __ldg(prm.b0 + j);
#pragma unroll 1
        for (int pp = 0; pp < npc; ++pp) {
          float pre = bj;
          for (int k = 0; k < n_in; ++k) pre = fmaf(__ldg(prm.w0t + k * WP + j), zs[pp * 32 + k], pre);
          float val, sp;
          act_rows<ACT>(pre, val, sp);
          tab[pp * 512 + etid] = val;
          tab[pp * 512 + 256 + etid] = sp;
        }
      }
      named_bar_sync(1, 256);
      const float* w = prm.w0t + tk * WP + mb * 256 + nb0;  // W0'[:, k] of this tangent row's input
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 t = *reinterpret_cast<const float4*>(my_tab + nb0 + h * 32 + i);
          float4 ww = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid && !is_val) ww = __ldg(reinterpret_cast<const float4*>(w + h * 32 + i));
          v[i] = !valid ? 0.0f : (is_val ? t.x : t.x * ww.x);
          v[i + 1] = !valid ? 0.0f : (is_val ? t.y : t.y * ww.y);
          v[i + 2] = !valid ? 0.0f : (is_val ? t.z : t.z * ww.z);
          v[i + 3] = !valid ? 0.0f : (is_val ? t.w : t.w * ww.w);
        }
        const int k0 = mb * 256 + nb0 + h * 32;
        store16(k0, v);
        store16(k0 + 16, v + 16);
        publish(k0 >> 5);
      }
      named_bar_sync(1, 256);  // the tables are rebuilt for the next half
    };

    for (long long tile = pair; tile < prm.num_tiles; tile += npairs, ++tiles_done) {
      const long long node0 = tile * (2 * npc) + static_cast<long long>(rank) * npc;
      // z of this CTA's nodes (centred in fp64, rtn_kernel.cuh load_z)
      if (etid < npc * n_in) {
        const int zp = etid / n_in, zk = etid - zp * n_in;
        const long long node = node0 + zp;
        zs[zp * 32 + zk] = node < prm.K ? static_cast<float>(load_z(prm, node, zk)) : 0.0f;
      }
      if (tiles_done > 0) {  // the previous tile's output MMAs have read the A buffer
        mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
        // outputs of the previous tile: rows in lanes 0..63 (quadrants 0, 1), outputs in columns 0..7
        if (q < 2 && sub == 0) {
          float o[16];
          tmem_ld16(tmem_base + lane_base, o);
          tmem_ld_wait();
          const long long pnode0 = node0 - npairs * 2 * npc;
          const int n_out = prm.n_out;
          if (valid && pnode0 + p < prm.K) {
            note_nonfinite(prm, o, n_out);
            const long long node = pnode0 + p;
            if (is_val)
              for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
            else if (prm.jac != nullptr)
              for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + tk] = static_cast<double>(o[oo]);
          }
        }
        tmem_release(0);
      }
      named_bar_sync(1, 256);  // zs staged
      const bool trb = prm.trace && pair == 0 && tiles_done == static_cast<uint32_t>(prm.trace_tile) && warp == 4 && lane == 0;
      if (trb) prm.trace[180 + rank * 6] = globaltimer();
      layer0_half(0);
      layer0_half(1);
      if (trb) prm.trace[192 + rank] = globaltimer();
      for (int l = 0; l < n_mma; ++l, ++hl)
        for (int mb = 0; mb < NMB; ++mb) do_block(mb, l);
    }
    if (tiles_done > 0) {  // the last tile's outputs
      mbar_wait_sleep(tmem_last, (tiles_done - 1) & 1);
      tc_fence_after();
      if (q < 2 && sub == 0) {
        float o[16];
        tmem_ld16(tmem_base + lane_base, o);
        tmem_ld_wait();
        const long long last_tile = pair + static_cast<long long>(tiles_done - 1) * npairs;
        const long long pnode0 = last_tile * (2 * npc) + static_cast<long long>(rank) * npc;
        const int n_out = prm.n_out;
        if (valid && pnode0 + p < prm.K) {
          note_nonfinite(prm, o, n_out);
          const long long node = pnode0 + p;
          if (is_val)
            for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
          else if (prm.jac != nullptr)
            for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + tk] = static_cast<double>(o[oo]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 256);
  }
}

}  // namespace rtn
