// rtn_fused.cuh — the persistent fused kernel (see rtn_kernel.cuh for the
// design). One CTA per SM; each CTA loops over tiles of P nodes.
#pragma once

#include "rtn_kernel.cuh"

namespace rtn {

template <int WP, int NSTAGE, int P>
struct FusedCfg {
  static constexpr int kNMB = WP / 128;  // neuron blocks (M = 128)
  static constexpr int kNKC = WP / 32;   // 32-wide k chunks (one SW128 atom row)
  static constexpr uint32_t kChunkStride = kNT * 128;
  static constexpr uint32_t kActBytes = kNKC * kChunkStride;
  static constexpr uint32_t kStageOff = kActBytes;
  static constexpr uint32_t kBarOff = kStageOff + NSTAGE * kStageBytes;
  // full[NSTAGE], empty[NSTAGE], act_ready[4], in_free[4], tmem_full[4], tmem_last
  static constexpr uint32_t kNumBars = 2 * NSTAGE + 13;
  static constexpr uint32_t kMiscOff = kBarOff + kNumBars * 8;
  static constexpr uint32_t kZsOff = kMiscOff + 16;
  static constexpr uint32_t kSmemBytes = kZsOff + kNT * 4 + 1024;  // + alignment slack
  static_assert(kNMB <= 4, "at most 4 neuron blocks");
  static_assert(kNMB * kTmemStride <= 512, "TMEM capacity");
};

template <int WP, int NSTAGE, int P>
__global__ void __launch_bounds__(kThreads, 1) rtn_fused_kernel(const KParams prm) {
  using C = FusedCfg<WP, NSTAGE, P>;
  constexpr int NMB = C::kNMB, NKC = C::kNKC;
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
  const int n_in = prm.n_in, nt = prm.nt;
  const int n_mma_layers = prm.n_hidden - 1;  // hidden → hidden layers on tensor cores

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int g = 0; g < 4; ++g) {
      mbar_init(&act_ready[g], 256);
      mbar_init(&in_free[g], 1);
      mbar_init(&tmem_full[g], 1);
    }
    mbar_init(tmem_last, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== weight producer (TMA bulk engine) ==================
    // Whole warp runs the loop (converged); one elected lane issues.
    const uint64_t pol = l2_evict_last_policy();
    int s = 0;
    uint32_t ph = 0;
    for (long long tile = blockIdx.x; tile < prm.num_tiles; tile += gridDim.x) {
      const uint8_t* src = prm.w_hidden;
      for (int b = 0; b < n_mma_layers * NMB * NKC; ++b, src += kStageBytes) {
        mbar_wait(&empty[s], ph ^ 1);
        bulk_g2s_warp(stage_s + s * kStageBytes, src, (prm.dbg & 2) ? 1024u : kStageBytes, &full[s], pol);
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
      for (int c = 0; c < NKC; ++c) {
        mbar_wait(&empty[s], ph ^ 1);
        bulk_g2s_warp(stage_s + s * kStageBytes, prm.w_last + c * kLastBlockBytes, kLastBlockBytes, &full[s], pol);
        if (++s == NSTAGE) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (converged warp, elected lane issues) ===
    {
      const uint32_t idesc_h = idesc_tf32(128, nt);
      const uint32_t idesc_o = idesc_tf32(128, kMaxOut);
      const uint32_t act_addr = smem_u32(act_s);
      const uint32_t stage_addr = smem_u32(stage_s);
      int s = 0;
      uint32_t ph = 0, ar = 0;
      for (long long tile = blockIdx.x; tile < prm.num_tiles; tile += gridDim.x) {
        for (int l = 0; l < n_mma_layers; ++l) {
#pragma unroll 1
          for (int mb = 0; mb < NMB; ++mb) {
#pragma unroll 1
            for (int c = 0; c < NKC; ++c) {
              if (mb == 0 && (c & 3) == 0 && !(prm.dbg & 1)) {
                mbar_wait(&act_ready[c >> 2], ar & 1);
                tc_fence_after();
              }
              mbar_wait(&full[s], ph);
              tc_fence_after();
              const uint64_t a = sw128_desc(stage_addr + s * kStageBytes);
              const uint64_t b = sw128_desc(act_addr + c * C::kChunkStride);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_tf32_warp(tmem_base + mb * kTmemStride, a + 2 * kk, b + 2 * kk, idesc_h, (c | kk) != 0);
              mma_commit_warp(&empty[s]);
              if (mb == NMB - 1 && (c & 3) == 3) mma_commit_warp(&in_free[c >> 2]);
              if (++s == NSTAGE) { s = 0; ph ^= 1; }
            }
            mma_commit_warp(&tmem_full[mb]);
          }
          ++ar;
        }
        // output layer: D[row, o] = Σ_k X[row, k] · W_L'[o, k]
#pragma unroll 1
        for (int c = 0; c < NKC; ++c) {
          if ((c & 3) == 0 && !(prm.dbg & 1)) {
            mbar_wait(&act_ready[c >> 2], ar & 1);
            tc_fence_after();
          }
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t a = sw128_desc(act_addr + c * C::kChunkStride);
          const uint64_t b = sw128_desc(stage_addr + s * kStageBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_tf32_warp(tmem_base, a + 2 * kk, b + 2 * kk, idesc_o, (c | kk) != 0);
          mma_commit_warp(&empty[s]);
          if (++s == NSTAGE) { s = 0; ph ^= 1; }
        }
        mma_commit_warp(tmem_last);
        ++ar;
      }
    }
  } else if (warp >= 4 && !(prm.dbg & 1)) {
    // ===================== epilogue (8 warps) =================================
    // Thread = one neuron of a 128-neuron block (TMEM lane); the two warp
    // halves split the tile rows into interleaved CW-column chunks. For each
    // block g the math is done in place in TMEM as soon as tmem_full[g] fires;
    // the copy into shared memory waits for in_free[g] (the layer's last block
    // has consumed input group g), so math never blocks on the in-place hazard.
    constexpr int CW = P > 8 ? P : 8;   // chunk width; multiple of P → static (c−P) mod P
    const int half = (warp - 4) >> 2;
    const int q = warp & 3;             // TMEM lane quadrant
    const int tid_h = q * 32 + lane;    // neuron within a 128-block / row of the output tile
    const int etid = threadIdx.x - 128;
    const int act = prm.act;
    const int rows_used = P * (1 + n_in);
    const int nch = (nt + CW - 1) / CW;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    uint32_t hl = 0;  // hidden layers processed (parity source)
    uint32_t tiles_done = 0;

    // Row r of a K-major SW128 operand lives at  col + (r/8)·1024 + (r%8)·128
    // + ((u ^ r%8) − u)·16  relative to row 0 of this thread's neuron column
    // (u = (j/4) mod 8 is the same for every block g). Precompute the XOR term.
    int swz[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) swz[i] = ((((tid_h >> 2) & 7) ^ i) - ((tid_h >> 2) & 7)) * 16 + i * 128;
    const int full_chunks = rows_used / CW;  // chunks with no padding rows

    // In-place TMEM pass for block g: v = act(pre + b) on value rows,
    // t = σ'(pre)·t on tangent rows, 0 on padding; tf32-rounded.
    auto compute_block = [&](int g, int l) {
      const int j = g * 128 + tid_h;
      const float bj = __ldg(prm.bh + l * WP + j);
      const uint32_t tb = tmem_base + lane_base + g * kTmemStride;
      mbar_wait(&tmem_full[g], hl & 1);
      tc_fence_after();
      if (prm.dbg & 4) return;
      float head[CW];
      tmem_ld_cw<CW>(tb, head);
      tmem_ld_wait();
      float val[P], sp[P];
#pragma unroll
      for (int p = 0; p < P; ++p) act_fwd(act, head[p] + bj, val[p], sp[p]);
      if (half == 0) {  // chunk 0: value rows [0, P) then tangent rows
#pragma unroll
        for (int i = 0; i < CW; ++i)
          head[i] = i < P ? to_tf32(val[i]) : (i < rows_used ? to_tf32(head[i] * sp[i % P]) : 0.0f);
        tmem_st_cw<CW>(tb, head);
      }
      for (int ch = (half == 0 ? 2 : 1); ch < nch; ch += 2) {
        float v[CW];
        tmem_ld_cw<CW>(tb + ch * CW, v);
        tmem_ld_wait();
        if (ch < full_chunks) {
#pragma unroll
          for (int i = 0; i < CW; ++i) v[i] = to_tf32(v[i] * sp[i % P]);
        } else {
#pragma unroll
          for (int i = 0; i < CW; ++i) v[i] = ch * CW + i < rows_used ? to_tf32(v[i] * sp[i % P]) : 0.0f;
        }
        tmem_st_cw<CW>(tb + ch * CW, v);
      }
      tmem_st_wait();
    };
    // Copy block g's results (TMEM) into next-layer input group g (smem).
    auto write_block = [&](int g) {
      const int j = g * 128 + tid_h;
      const uint32_t tb = tmem_base + lane_base + g * kTmemStride;
      mbar_wait(&in_free[g], hl & 1);
      uint8_t* col = act_s + sw128_offset(0, j, C::kChunkStride);
      for (int ch = half; ch < nch && !(prm.dbg & 4); ch += 2) {
        float v[CW];
        tmem_ld_cw<CW>(tb + ch * CW, v);
        tmem_ld_wait();
        uint8_t* base = col + (ch * CW / 8) * 1024;
#pragma unroll
        for (int i = 0; i < CW; ++i) *reinterpret_cast<float*>(base + (i >> 3) * 1024 + swz[i & 7]) = v[i];
      }
      tc_fence_before();
      fence_proxy_async_smem();
      mbar_arrive(&act_ready[g]);
    };

    for (long long tile = blockIdx.x; tile < prm.num_tiles; tile += gridDim.x, ++tiles_done) {
      const long long node0 = tile * P;
      // ---- previous tile's output layer must have consumed the activations
      if (tiles_done > 0) {
        mbar_wait(tmem_last, (tiles_done - 1) & 1);
        tc_fence_after();
      }
      // ---- stage this tile's z rows (fp32) for layer 0
      if (etid < P * n_in) {
        const int p = etid / n_in, k = etid - p * n_in;
        const long long node = node0 + p;
        zs[etid] = node < prm.K ? static_cast<float>(load_z(prm, node, k)) : 0.0f;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      // ---- layer 0 on CUDA cores: value rows + tangent rows σ'(pre)·W0'[:, k]
      for (int g = 0; g < NMB; ++g) {
        const int j = g * 128 + tid_h;
        const float* w0r = prm.w0 + j * n_in;
        const float bj = __ldg(prm.b0 + j);
        float val[P], sp[P];
#pragma unroll
        for (int p = 0; p < P; ++p) {
          float pre = bj;
          for (int k = 0; k < n_in; ++k) pre = fmaf(__ldg(w0r + k), zs[p * n_in + k], pre);
          act_fwd(act, pre, val[p], sp[p]);
        }
        uint8_t* col = act_s + sw128_offset(0, j, C::kChunkStride);
        for (int ch = half; ch < nch; ch += 2) {
          uint8_t* base = col + (ch * CW / 8) * 1024;
#pragma unroll
          for (int i = 0; i < CW; ++i) {
            const int c = ch * CW + i;
            float v;
            if (ch == 0 && i < P) v = val[i];
            else if (c < rows_used) v = sp[i % P] * __ldg(w0r + (c - P) / P);
            else v = 0.0f;
            *reinterpret_cast<float*>(base + (i >> 3) * 1024 + swz[i & 7]) = to_tf32(v);
          }
        }
        fence_proxy_async_smem();
        mbar_arrive(&act_ready[g]);
      }
      // ---- hidden layers on tensor cores
      for (int l = 0; l < n_mma_layers; ++l, ++hl) {
        for (int g = 0; g + 1 < NMB; ++g) compute_block(g, l);
        for (int g = 0; g + 1 < NMB; ++g) write_block(g);
        compute_block(NMB - 1, l);
        write_block(NMB - 1);
      }
      // ---- output layer epilogue: lane = tile row, column = output
      mbar_wait(tmem_last, tiles_done & 1);
      tc_fence_after();
      if (half == 0) {
        float o[16];
        tmem_ld16(tmem_base + lane_base, o);
        tmem_ld_wait();
        const int r = tid_h;
        const int n_out = prm.n_out;
        if (r < P) {
          const long long node = node0 + r;
          if (node < prm.K)
            for (int oo = 0; oo < n_out; ++oo) prm.f[node * n_out + oo] = static_cast<double>(o[oo] + __ldg(prm.bl + oo));
        } else if (r < rows_used && prm.jac != nullptr) {
          const int k = (r - P) / P, p = (r - P) % P;
          const long long node = node0 + p;
          if (node < prm.K)
            for (int oo = 0; oo < n_out; ++oo) prm.jac[(node * n_out + oo) * n_in + k] = static_cast<double>(o[oo]);
        }
      }
      tc_fence_before();
    }
  }
  // warps 2-3 idle
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace rtn
