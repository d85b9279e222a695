// rtn_pingpong.cuh — throughput kernel for padded width 256 (one 256-neuron
// block per layer), TF32, order 1.
//
// Why: with a single M-block per layer the pair kernel has nothing to run on
// the tensor core while the epilogue turns layer l's accumulators into layer
// l+1's operands, so the whole epilogue is exposed at every layer boundary
// (5x256 ran at ~29 % of the TF32 peak). Here each CTA pair keeps TWO tiles in
// flight (slots 0 and 1: separate activation buffers, TMEM regions and
// barriers). The MMA warp issues layer l of slot 0, then layer l of slot 1;
// the epilogue of slot 0 overlaps the MMAs of slot 1 and vice versa. Weights
// are streamed once per (layer, slot). Shared memory: 2 x 80 KB activations
// + 4 x 16 KB weight stages.
#pragma once

#include <cuda.h>

#include "rtn_kernel.cuh"
#include "rtn_pair.cuh"

namespace rtn {

template <int NSTAGE, int P, int NTC>
struct PingCfg {
  using B = PairCfg<256, NSTAGE, P, NTC, kTF32, false>;
  static constexpr uint32_t kActBytes = B::kActBytes;  // one slot
  static constexpr uint32_t kStageOff = 2 * kActBytes;
  static constexpr uint32_t kBarOff = kStageOff + NSTAGE * kStageBytes;
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 2 * 6;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kZsOff = kMiscOff + 16;
  static constexpr uint32_t kSmemBytes = kZsOff + 2 * 2 * P * 24 * 4 + 1024;
  static_assert(kSmemBytes <= 232448, "shared memory budget");
  static_assert((B::kNKC % NSTAGE) == 0, "every (layer, slot) block starts at stage 0");
  static_assert((128 - NTC) * 128 <= NSTAGE * kStageBytes, "output-layer A overrun must stay in smem");
};

template <int NSTAGE, int P, int NTC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    rtn_pingpong_kernel(const KParams prm, const __grid_constant__ CUtensorMap tmap_h,
                        const __grid_constant__ CUtensorMap tmap_l) {
  constexpr int WP = 256;
  using PC = PingCfg<NSTAGE, P, NTC>;
  using C = typename PC::B;
  constexpr int NKC = C::kNKC, CPG = C::kCPG;  // 8 chunks, 4 per K-group, 2 K-groups
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* act_s = smem;  // slot s at + s * kActBytes
  uint8_t* stage_s = smem + PC::kStageOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PC::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  uint64_t* sb = bars + 2 * NSTAGE;  // per slot s: act_ready[2], in_free[2], tmem_full, tmem_last
  auto act_ready = [&](int s, int g) { return sb + s * 6 + g; };
  auto in_free = [&](int s, int g) { return sb + s * 6 + 2 + g; };
  auto tmem_full = [&](int s) { return sb + s * 6 + 4; };
  auto tmem_last = [&](int s) { return sb + s * 6 + 5; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + PC::kMiscOff);
  float* zs = reinterpret_cast<float*>(smem + PC::kZsOff);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int n_in = prm.n_in, ntc = prm.nt;
  const int n_mma_layers = prm.n_hidden - 1;
  const long long pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const long long num_tp = (prm.num_tiles + 1) / 2;  // tile pairs

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      for (int g = 0; g < 2; ++g) {
        mbar_init(act_ready(s, g), 8);
        mbar_init(in_free(s, g), 1);
      }
      mbar_init(tmem_full(s), 1);
      mbar_init(tmem_last(s), 1);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    prefetch_tmap(&tmap_h);
    prefetch_tmap(&tmap_l);
  }
  if (warp == 1) tmem_alloc_pair(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer: each (layer, slot) streams the layer ==
    const uint64_t pol = l2_evict_last_policy();
    uint32_t ph = 0;
    const int yr = static_cast<int>(rank) * 128;
    for (long long tp = pair; tp < num_tp; tp += npairs) {
      for (int l = 0; l < n_mma_layers; ++l)
        for (int s = 0; s < 2; ++s) {
          const int y = l * WP + yr;
#pragma unroll
          for (int i = 0; i < NKC; ++i) {
            const int st = i % NSTAGE;
            mbar_wait(&empty[st], ph ^ 1);
            if (leader) mbar_expect_tx_elect(&full[st], 2 * kStageBytes);
            tma_load_2sm(stage_s + st * kStageBytes, &tmap_h, i * C::kCK, y, &full[st], pol);
            if (st == NSTAGE - 1) ph ^= 1;
          }
        }
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int i = 0; i < NKC; ++i) {
          const int st = i % NSTAGE;
          mbar_wait(&empty[st], ph ^ 1);
          if (leader) mbar_expect_tx_elect(&full[st], 2 * kLastHalfBytes);
          tma_load_2sm(stage_s + st * kStageBytes, &tmap_l, i * C::kCK, static_cast<int>(rank) * 8, &full[st], pol);
          if (st == NSTAGE - 1) ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ===================== pair MMA issuer (leader CTA) ======================
    if (leader) {
      const uint32_t idesc_h = idesc_tf32(256, 2 * ntc);
      const uint32_t idesc_o = idesc_tf32(256, kMaxOut);
      const uint64_t a0 = sw128_desc(smem_u32(stage_s));
      constexpr uint32_t kStageD = kStageBytes >> 4, kChunkD = C::kChunkStride >> 4;
      uint32_t ph = 0, ar[2] = {0, 0};
      for (long long tp = pair; tp < num_tp; tp += npairs) {
        for (int l = 0; l < n_mma_layers; ++l)
          for (int s = 0; s < 2; ++s) {
            const uint64_t b0 = sw128_desc(smem_u32(act_s + s * PC::kActBytes));
            const uint32_t d = tmem_base + s * kTmemStride2;
#pragma unroll
            for (int c = 0; c < NKC; ++c) {
              const int st = c % NSTAGE;
              if (c == 0) {  // both groups: inputs ready and this slot's TMEM drained by both CTAs
                mbar_wait_cluster(act_ready(s, 0), ar[s] & 1);
                mbar_wait_cluster(act_ready(s, 1), ar[s] & 1);
                tc_fence_after();
              }
              mbar_wait(&full[st], ph);
              tc_fence_after();
              const uint32_t bar2 = (c % CPG) == CPG - 1 ? smem_u32(in_free(s, c / CPG)) : 0u;
              mma4_tf32_pair_commit(d, a0 + st * kStageD, b0 + c * kChunkD, idesc_h, c != 0, smem_u32(&empty[st]),
                                    bar2);
              if (st == NSTAGE - 1) ph ^= 1;
            }
            mma_commit_pair(tmem_full(s));
            ++ar[s];
          }
        for (int s = 0; s < 2; ++s) {  // output layer: D[row, o], M = 2 x 128 rows, N = 16
          const uint64_t b0 = sw128_desc(smem_u32(act_s + s * PC::kActBytes));
          const uint32_t d = tmem_base + s * kTmemStride2;
#pragma unroll
          for (int c = 0; c < NKC; ++c) {
            const int st = c % NSTAGE;
            if (c == 0) {
              mbar_wait_cluster(act_ready(s, 0), ar[s] & 1);
              mbar_wait_cluster(act_ready(s, 1), ar[s] & 1);
              tc_fence_after();
            }
            mbar_wait(&full[st], ph);
            tc_fence_after();
            mma4_tf32_pair_commit(d, b0 + c * kChunkD, a0 + st * kStageD, idesc_o, c != 0, smem_u32(&empty[st]), 0u);
            if (st == NSTAGE - 1) ph ^= 1;
          }
          mma_commit_pair(tmem_last(s));
          ++ar[s];
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: half h = side h; K-group g = rank =========
    const int half = (warp - 4) >> 2;
    const int q = warp & 3;
    const int tid_h = q * 32 + lane;
    const int etid = threadIdx.x - 128;
    const int act = prm.act;
    const int rows_used = P * (1 + n_in);
    const bool no_pad = rows_used == ntc;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    const int u = ((tid_h * 4) >> 4) & 7;
    int swz[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) swz[i] = ((u ^ i) - u) * 16 + i * 128;
    const uint32_t act_local = smem_u32(act_s);
    const bool local_side = half == static_cast<int>(rank);
    const uint32_t side_base = local_side ? act_local : mapa(act_local, static_cast<uint32_t>(half));
    uint32_t ready_cl[2][2];
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int g = 0; g < 2; ++g) ready_cl[s][g] = mapa(smem_u32(act_ready(s, g)), 0);
    const int grp = static_cast<int>(rank);
    uint32_t tpd = 0;  // tile pairs done

    auto store_side = [&](const float* v, int j, int s) {
      const uint32_t base = side_base + s * PC::kActBytes + (j / C::kCK) * C::kChunkStride +
                            (((j % C::kCK) * 4) >> 4 << 4) + ((j * 4) & 15);
#pragma unroll
      for (int i = 0; i < NTC; ++i) {
        if ((i & ~7) >= ntc) continue;
        const uint32_t a = base + (i >> 3) * 1024 + swz[i & 7];
        const float h = to_tf32(v[i]);
        if (local_side) st_shared_f32(a, h);
        else st_cluster_f32(a, h);
      }
    };
    auto publish = [&](int s) {
      fence_proxy_async_cluster();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(ready_cl[s][grp]);
    };

    for (long long tp = pair; tp < num_tp; tp += npairs, ++tpd) {
      // ---- layer 0 for both slots (CUDA cores)
      for (int s = 0; s < 2; ++s) {
        const long long node0 = (2 * tp + s) * (2 * P);
        if (tpd > 0) {
          mbar_wait_sleep(tmem_last(s), (tpd - 1) & 1);
          tc_fence_after();
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");  // zs reuse
        if (etid < 2 * P * n_in) {
          const int p = etid / n_in, k = etid - p * n_in;
          const long long node = node0 + p;
          zs[etid] = node < prm.K ? static_cast<float>(load_z(prm, node, k)) : 0.0f;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const int j = grp * 128 + tid_h;
        float w0[kMaxIn0];
        load_w0_row(prm.w0 + j * n_in, n_in, w0);
        const float bj = __ldg(prm.b0 + j);
        float val[P], sp[P];
#pragma unroll
        for (int p = 0; p < P; ++p) act_fwd(act, layer0_pre(bj, w0, zs + (half * P + p) * n_in, n_in), val[p], sp[p]);
        float v[NTC];
#pragma unroll
        for (int i = 0; i < NTC; ++i) {
          if (i < P) v[i] = val[i];
          else v[i] = i < rows_used ? sp[i % P] * w0[((i - P) / P) % kMaxIn0] : 0.0f;
        }
        store_side(v, j, s);
        publish(s);
      }
      // ---- hidden layers: slot 0 then slot 1 each layer
      for (int l = 0; l < n_mma_layers; ++l)
        for (int s = 0; s < 2; ++s) {
          const int j = grp * 128 + tid_h;
          const float bj = __ldg(prm.bh + l * WP + j);
          const uint32_t hphase = (tpd * n_mma_layers + l) & 1;
          mbar_wait_sleep(tmem_full(s), hphase);
          tc_fence_after();
          float v[NTC];
#pragma unroll
          for (int c0 = 0; c0 < NTC; c0 += 8)
            if (c0 < ntc) tmem_ld8(tmem_base + lane_base + s * kTmemStride2 + half * ntc + c0, v + c0);
          tmem_ld_wait();
          tc_fence_before();
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
          mbar_wait_sleep(in_free(s, grp), hphase);
          store_side(v, j, s);
          publish(s);
        }
      // ---- output layer per slot: this CTA's rows in its TMEM lanes, outputs in columns 0..15
      for (int s = 0; s < 2; ++s) {
        mbar_wait_sleep(tmem_last(s), tpd & 1);
        tc_fence_after();
        if (half == 0) {
          float o[16];
          tmem_ld16(tmem_base + lane_base + s * kTmemStride2, o);
          tmem_ld_wait();
          const int r = tid_h, n_out = prm.n_out;
          const long long nbase = (2 * tp + s) * (2 * P) + static_cast<long long>(rank) * P;
          if (r < P) {
            const long long node = nbase + r;
            if (node < prm.K)
              for (int oo = 0; oo < n_out; ++oo)
                prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
          } else if (r < rows_used && prm.jac != nullptr) {
            const int k = (r - P) / P, p = (r - P) % P;
            const long long node = nbase + p;
            if (node < prm.K)
              for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + k] = static_cast<double>(o[oo]);
          }
        }
        tc_fence_before();
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, 512);
  }
}

}  // namespace rtn
