// rtn_mpc.cu — C-ABI (include/rtn_mpc.h): model loader/packer, contexts and
// the PrepareNodes/MlpBatchedEval-equivalent entry points. Every compute call
// runs the sm_100a kernels (rtn_pair.cuh, rtn_quad.cuh, rtn_rows.cuh,
// rtn_blocks.cu, rtn_qpsolve.cu); there is no CPU fallback.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/rtn_mpc.h"
#include "rtn_blocks.h"
#include "rtn_internal.h"
#include "rtn_launch.h"
#include "rtn_qpsolve.h"

namespace rtn_host {
thread_local std::string g_err;
}  // namespace rtn_host
using namespace rtn_host;

namespace {

// Host-side copy of resmpc::MlpModel (proj/include/resmpc/neural.hpp:19-34).
struct HostModel {
  std::vector<int> sizes;
  int act = 0;
  std::vector<std::vector<double>> W, b;
  std::vector<double> in_mean, in_scale, out_mean, out_scale;
};

// MlpModel::Validate (proj/src/neural.cpp:283-298) → RTN_ECONFIG.
void Validate(const HostModel& m) {
  if (m.sizes.size() < 2) throw Error(RTN_ECONFIG, "mlp: need at least input and output layers");
  for (int s : m.sizes)
    if (s < 1) throw Error(RTN_ECONFIG, "mlp: layer sizes must be positive");
  if (m.W.size() != m.sizes.size() - 1 || m.b.size() != m.W.size())
    throw Error(RTN_ECONFIG, "mlp: weight/bias count does not match layer sizes");
  for (size_t l = 0; l < m.W.size(); ++l) {
    if (m.W[l].size() != static_cast<size_t>(m.sizes[l + 1]) * m.sizes[l])
      throw Error(RTN_ECONFIG, "mlp: layer " + std::to_string(l) + " has incompatible shape");
    if (m.b[l].size() != static_cast<size_t>(m.sizes[l + 1]))
      throw Error(RTN_ECONFIG, "mlp: bias " + std::to_string(l) + " has incompatible shape");
  }
  const size_t in = m.sizes.front(), out = m.sizes.back();
  if (m.in_mean.size() != in || m.in_scale.size() != in || m.out_mean.size() != out || m.out_scale.size() != out)
    throw Error(RTN_ECONFIG, "mlp: normalization vectors do not match layer sizes");
  for (double s : m.in_scale)
    if (!(s > 0.0)) throw Error(RTN_ECONFIG, "mlp: normalization scales must be strictly positive");
  for (double s : m.out_scale)
    if (!(s > 0.0)) throw Error(RTN_ECONFIG, "mlp: normalization scales must be strictly positive");
  if (m.act < 0 || m.act > 2) throw Error(RTN_ECONFIG, "mlp: unknown activation");
}

// Round an fp32 to tf32 (round-to-nearest, ties away), as cvt.rna.tf32.f32.
float RoundTf32(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Round an fp32 to bf16 (round-to-nearest-even), kept as fp32 / as bits.
float RoundBf16(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
uint16_t Bf16Bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return static_cast<uint16_t>(u >> 16);
}

}  // namespace

namespace rtn_host {

unsigned long long* trace_buf = nullptr;  // RTN_TRACE device buffer
void* trace_host = nullptr;               // RTN_TRACE_HOST: the same buffer, host-mapped
constexpr long long kGraphMaxRows = 4096;     // latency mode: graph-captured steps up to this K
constexpr long long kChunkMinRows = 1 << 17;  // chunk only batches this large

// Latency mode: kernels access the pinned staging in place (RTN_ZEROCOPY=0 restores memcpy nodes).
bool ZeroCopy() {
  static const bool on = [] {
    const char* e = std::getenv("RTN_ZEROCOPY");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Fused cycle: the blocks kernel is a programmatic dependent of the MLP kernel
// (launch + prologue overlap its tail; RTN_PDL=0 disables).
bool PdlEnabled() {
  static const bool on = [] {
    const char* e = std::getenv("RTN_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Hidden widths are zero-padded to the kernels' 256- or 512-neuron layouts
// (any width in (256, 512] pads to 512; > 512 is rejected by the caller).
int PaddedWidth(const std::vector<int>& sizes) {
  int w = 0;
  for (size_t l = 1; l + 1 < sizes.size(); ++l) w = std::max(w, sizes[l]);
  return w <= 256 ? 256 : (w <= 512 ? 512 : ((w + 255) / 256) * 256);
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn GetEncodeTiled() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(RTN_ECUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D row-major [rows x cols] map (fp32 or bf16) with a {128 B, box_rows}
// box and the 128-byte swizzle the UMMA descriptors expect.
CUtensorMap MakeTmap(void* base, uint64_t rows, uint64_t cols, uint32_t box_rows, bool bf16) {
  CUtensorMap m{};
  const uint32_t eb = bf16 ? 2 : 4;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * eb};
  const cuuint32_t box[2] = {128 / eb, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = GetEncodeTiled()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                                      base, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(RTN_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

// The device layout of a model as host arrays: everything BuildModel uploads.
// Written to / read from the packed-layout cache file (PackCache) unchanged.
struct Packed {
  int32_t mode = 0, n_in = 0, n_out = 0, n_layers = 0, act = 0, pwp = 0, split = 1, bf16 = 0;
  std::vector<double> mu;                  // in_mean (fp64)
  std::vector<float> w0, w0t, b0, bl, bh;  // layer 0 (neuron- and input-major), biases
  std::vector<uint8_t> th, tl;             // hidden / output operand copies (fp32 or bf16 bytes)
};

// Folds the normalisation into the first/last layer in fp64
// (proj/include/resmpc/neural.hpp:14-18: y = out_scale ⊙ net((z−μ)⊘s) + out_mean):
//   W0' = W0·diag(1/s)   (μ is subtracted from z in fp64 by the kernels, load_z),
//   WL' = diag(out_scale)·WL,  bL' = out_scale ⊙ bL + out_mean,
// and packs the hidden and output layers as row-major operand copies for the
// TMA tensor maps (hi/lo stacked in the split precision modes).
Packed PackModel(const HostModel& hm, rtn_precision prec) {
  Validate(hm);
  if (prec != RTN_TF32 && prec != RTN_3XTF32 && prec != RTN_BF16X3 && prec != RTN_BF16)
    throw Error(RTN_ECONFIG, "unknown precision mode");
  Packed pk;
  pk.mode = prec == RTN_TF32     ? rtn::kTF32
            : prec == RTN_3XTF32 ? rtn::k3xTF32
            : prec == RTN_BF16X3 ? rtn::kBF16x3
                                 : rtn::kBF16;
  const int L = static_cast<int>(hm.sizes.size()) - 1;
  const int n_in = hm.sizes.front(), n_out = hm.sizes.back();
  if (L < 2) throw Error(RTN_EUNSUPPORTED, "device path needs at least one hidden layer");
  const int pwp = PaddedWidth(hm.sizes);
  if (pwp > 512) throw Error(RTN_EUNSUPPORTED, "hidden width > 512 not supported by the device kernels");
  if (n_out > rtn::kMaxOut) throw Error(RTN_EUNSUPPORTED, "n_out > 16 not supported");
  if (n_in > 79) throw Error(RTN_EUNSUPPORTED, "n_in > 79 not supported");
  const int H = L - 1;  // hidden layers (each followed by the activation)
  pk.n_in = n_in;
  pk.n_out = n_out;
  pk.n_layers = L;
  pk.act = hm.act;
  pk.pwp = pwp;
  pk.mu = hm.in_mean;
  // layer 0 (CUDA cores, fp32): W0' = W0·diag(1/in_scale); the bias stays b0
  pk.w0.assign(static_cast<size_t>(pwp) * n_in, 0.0f);
  pk.w0t.assign(static_cast<size_t>(pwp) * n_in, 0.0f);
  pk.b0.assign(pwp, 0.0f);
  for (int j = 0; j < hm.sizes[1]; ++j) {
    for (int k = 0; k < n_in; ++k) {
      const float w = static_cast<float>(hm.W[0][static_cast<size_t>(j) * n_in + k] / hm.in_scale[k]);
      pk.w0[static_cast<size_t>(j) * n_in + k] = w;
      pk.w0t[static_cast<size_t>(k) * pwp + j] = w;
    }
    pk.b0[j] = static_cast<float>(hm.b[0][j]);
  }
  pk.bl.assign(rtn::kMaxOut, 0.0f);
  for (int o = 0; o < n_out; ++o) pk.bl[o] = static_cast<float>(hm.out_scale[o] * hm.b[L - 1][o] + hm.out_mean[o]);
  pk.bh.assign(static_cast<size_t>(std::max(H - 1, 1)) * pwp, 0.0f);
  for (int l = 1; l < H; ++l)
    for (int j = 0; j < hm.sizes[l + 1]; ++j) pk.bh[static_cast<size_t>(l - 1) * pwp + j] = static_cast<float>(hm.b[l][j]);
  // Row-major operand copies for the TMA maps: [hi; lo] stacked (split modes),
  // tf32-rounded fp32 or bf16.
  const int wp = pwp;
  pk.split = rtn::IsSplitMode(pk.mode) ? 2 : 1;
  pk.bf16 = rtn::IsBf16Mode(pk.mode);
  const int split = pk.split;
  const bool bf16 = pk.bf16;
  const size_t hid_rows = static_cast<size_t>(std::max(H - 1, 1)) * wp;
  std::vector<float> th(split * hid_rows * wp, 0.0f), tl(static_cast<size_t>(split) * 16 * wp, 0.0f);
  auto put = [&](std::vector<float>& dst, size_t row, size_t col, double w) {
    // hi part, then the residual in the second half of the stack
    if (bf16) {
      const float h = RoundBf16(static_cast<float>(w));
      dst[row * wp + col] = h;
      if (split == 2) dst[(row + dst.size() / (2 * wp)) * wp + col] = RoundBf16(static_cast<float>(w - h));
    } else {
      const float h = RoundTf32(static_cast<float>(w));
      dst[row * wp + col] = h;
      if (split == 2) dst[(row + dst.size() / (2 * wp)) * wp + col] = RoundTf32(static_cast<float>(w - h));
    }
  };
  for (int l = 1; l < H; ++l) {
    const int rows = hm.sizes[l + 1], cols = hm.sizes[l];
    for (int j = 0; j < rows; ++j)
      for (int k = 0; k < cols; ++k) put(th, static_cast<size_t>(l - 1) * wp + j, k, hm.W[l][static_cast<size_t>(j) * cols + k]);
  }
  {
    const int cols = hm.sizes[L - 1];
    for (int o = 0; o < n_out; ++o)
      for (int k = 0; k < cols; ++k) put(tl, o, k, hm.out_scale[o] * hm.W[L - 1][static_cast<size_t>(o) * cols + k]);
  }
  auto bytes = [&](const std::vector<float>& v, std::vector<uint8_t>& out) {
    if (bf16) {
      out.resize(v.size() * 2);
      for (size_t i = 0; i < v.size(); ++i) {
        const uint16_t h = Bf16Bits(v[i]);
        std::memcpy(out.data() + 2 * i, &h, 2);
      }
    } else {
      out.resize(v.size() * 4);
      std::memcpy(out.data(), v.data(), out.size());
    }
  };
  bytes(th, pk.th);
  bytes(tl, pk.tl);
  return pk;
}

rtn_model* UploadModel(const Packed& pk, int device) {
  int ndev = 0;
  CUDA_CHECK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw Error(RTN_ECUDA, "invalid device ordinal");
  cudaDeviceProp prop{};
  CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) throw Error(RTN_ECUDA, "device is not sm_100 (Blackwell B200)");
  CUDA_CHECK(cudaSetDevice(device));
  std::unique_ptr<rtn_model> m(new rtn_model());
  m->device = device;
  m->prec = pk.mode == rtn::kTF32 ? RTN_TF32 : pk.mode == rtn::k3xTF32 ? RTN_3XTF32 : pk.mode == rtn::kBF16x3 ? RTN_BF16X3 : RTN_BF16;
  m->n_in = pk.n_in;
  m->n_out = pk.n_out;
  m->n_layers = pk.n_layers;
  m->n_hidden = pk.n_layers - 1;
  m->act = pk.act;
  m->wp = pk.pwp;
  m->pair_wp = pk.pwp;
  m->pair_mode = pk.mode;
  auto up = [](void** d, const void* h, size_t n) {
    CUDA_CHECK(cudaMalloc(d, std::max<size_t>(n, 16)));
    if (n) CUDA_CHECK(cudaMemcpy(*d, h, n, cudaMemcpyHostToDevice));
  };
  up(reinterpret_cast<void**>(&m->d_mu), pk.mu.data(), pk.mu.size() * 8);
  up(reinterpret_cast<void**>(&m->d_w0), pk.w0.data(), pk.w0.size() * 4);
  up(reinterpret_cast<void**>(&m->d_w0t), pk.w0t.data(), pk.w0t.size() * 4);
  up(reinterpret_cast<void**>(&m->d_b0), pk.b0.data(), pk.b0.size() * 4);
  up(reinterpret_cast<void**>(&m->d_bl), pk.bl.data(), pk.bl.size() * 4);
  up(reinterpret_cast<void**>(&m->d_bh_pair), pk.bh.data(), pk.bh.size() * 4);
  up(&m->d_wt_hidden, pk.th.data(), pk.th.size());
  up(&m->d_wt_last, pk.tl.data(), pk.tl.size());
  const size_t hid_rows = static_cast<size_t>(std::max(pk.n_layers - 2, 1)) * pk.pwp;
  m->tmap_h = MakeTmap(m->d_wt_hidden, pk.split * hid_rows, pk.pwp, 128, pk.bf16);
  m->tmap_l = MakeTmap(m->d_wt_last, static_cast<uint64_t>(pk.split) * 16, pk.pwp, 8, pk.bf16);
  if (pk.pwp == 512 && pk.split == 1) m->tmap_h64 = MakeTmap(m->d_wt_hidden, hid_rows, pk.pwp, 64, pk.bf16);
  // reverse mode (rtn_ctx_set_jacobian_mode): the hidden packs transposed (W_l^T,
  // [k][n], per split half, in the mode's element type), W0' input-major padded
  // to 32 rows as the J output pack ([hi; lo] in the split modes), and W_L' in
  // fp32 (the pack's hi + lo) for the adjoint rows' start. TF32 width 512 runs
  // on the split-schedule kernels (64-row boxes); every other mode of width 256
  // or 512 on the pair kernel's reverse variants (quadrotor outputs: n_out = 6).
  if ((pk.pwp == 512 || pk.pwp == 256) && pk.n_in <= rtn::kRevMaxInHost && pk.n_in <= rtn::kMaxIn2 &&
      pk.n_layers >= 2) {
    const int nh = std::max(pk.n_layers - 2, 1), wpp = pk.pwp, eb = pk.bf16 ? 2 : 4, sp = pk.split;
    std::vector<uint8_t> tt(pk.th.size());
    for (int h = 0; h < sp; ++h)
      for (int l = 0; l < nh; ++l) {
        const size_t blk = (static_cast<size_t>(h) * nh + l) * wpp;  // first row of layer l in split half h
        for (int k = 0; k < wpp; ++k)
          for (int n = 0; n < wpp; ++n)
            std::memcpy(&tt[((blk + k) * wpp + n) * eb], &pk.th[((blk + n) * wpp + k) * eb], eb);
      }
    std::vector<uint8_t> w0p(static_cast<size_t>(sp) * 32 * wpp * eb, 0);
    for (int i = 0; i < pk.n_in; ++i)
      for (int n = 0; n < wpp; ++n) {
        const float w = pk.w0t[static_cast<size_t>(i) * wpp + n];
        const float hi = pk.bf16 ? RoundBf16(w) : RoundTf32(w);
        const float lo = pk.bf16 ? RoundBf16(w - hi) : RoundTf32(w - hi);
        for (int h = 0; h < sp; ++h) {
          const float v = h == 0 ? hi : lo;
          uint8_t* dst = &w0p[((static_cast<size_t>(h) * 32 + i) * wpp + n) * eb];
          if (pk.bf16) {
            const uint16_t b = Bf16Bits(v);
            std::memcpy(dst, &b, 2);
          } else {
            std::memcpy(dst, &v, 4);
          }
        }
      }
    std::vector<float> wl(static_cast<size_t>(rtn::kMaxOut) * wpp, 0.0f);
    for (int o = 0; o < rtn::kMaxOut; ++o)
      for (int n = 0; n < wpp; ++n)
        for (int h = 0; h < sp; ++h) {
          const size_t idx = (static_cast<size_t>(h) * 16 + o) * wpp + n;
          float v;
          if (pk.bf16) {
            uint16_t b;
            std::memcpy(&b, &pk.tl[idx * 2], 2);
            const uint32_t u = static_cast<uint32_t>(b) << 16;
            std::memcpy(&v, &u, 4);
          } else {
            std::memcpy(&v, &pk.tl[idx * 4], 4);
          }
          wl[static_cast<size_t>(o) * wpp + n] += v;
        }
    up(&m->d_wt_hidden_t, tt.data(), tt.size());
    up(reinterpret_cast<void**>(&m->d_w0t_pad), w0p.data(), w0p.size());
    up(reinterpret_cast<void**>(&m->d_wl32), wl.data(), wl.size() * 4);
    m->tmap_ht = MakeTmap(m->d_wt_hidden_t, sp * hid_rows, wpp, 128, pk.bf16);
    m->tmap_w0p = MakeTmap(m->d_w0t_pad, static_cast<uint64_t>(sp) * 32, wpp, 16, pk.bf16);
    if (pk.mode == rtn::kTF32 && wpp == 512) {
      m->tmap_ht64 = MakeTmap(m->d_wt_hidden_t, hid_rows, wpp, 64, false);
      m->reverse_ok = true;  // split-schedule kernels (rtn_reverse.cuh)
    } else if (pk.n_out == 6 && rtn::IsSplitMode(pk.mode)) {
      m->reverse_pair_ok = true;  // pair-kernel variants (rtn_pair.cuh ORD2 = 3, 4)
    }
  }
  m->lo_rows = static_cast<int>(hid_rows);
  return m.release();
}

rtn_model* BuildModel(const HostModel& hm, int device, rtn_precision prec) {
  return UploadModel(PackModel(hm, prec), device);
}

// ---- digest-keyed packed-layout cache -------------------
// FNV-1a 64 of the RMLP file bytes, the reference's manifest digest
// (/root/reference/proj/src/io.cpp:10-26, Fnv1a64File).
uint64_t Fnv1a64(const std::vector<char>& bytes) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (char c : bytes) {
    h ^= static_cast<unsigned char>(c);
    h *= 0x100000001b3ULL;
  }
  return h;
}

std::string Hex16(uint64_t v) {
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(v));
  return buf;
}

// On-disk copy of a Packed layout ("RTNP" v1): header, then the arrays. Keyed by
// the source file's digest and the precision, so a changed model never matches.
constexpr uint32_t kPackVersion = 1;
bool WritePacked(const std::string& path, uint64_t digest, const Packed& pk) {
  std::ofstream out(path + ".tmp", std::ios::binary);
  if (!out) return false;
  auto w = [&](const void* p, size_t n) { out.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
  auto wv = [&](const auto& v) {
    const uint64_t n = v.size();
    w(&n, 8);
    w(v.data(), n * sizeof(v[0]));
  };
  w("RTNP", 4);
  w(&kPackVersion, 4);
  w(&digest, 8);
  const int32_t hdr[8] = {pk.mode, pk.n_in, pk.n_out, pk.n_layers, pk.act, pk.pwp, pk.split, pk.bf16};
  w(hdr, sizeof(hdr));
  wv(pk.mu);
  wv(pk.w0);
  wv(pk.w0t);
  wv(pk.b0);
  wv(pk.bl);
  wv(pk.bh);
  wv(pk.th);
  wv(pk.tl);
  out.close();
  if (!out) return false;
  return std::rename((path + ".tmp").c_str(), path.c_str()) == 0;
}

bool ReadPacked(const std::string& path, uint64_t digest, int mode, Packed* pk) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return false;
  auto r = [&](void* p, size_t n) {
    in.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    return static_cast<bool>(in);
  };
  auto rv = [&](auto& v) {
    uint64_t n = 0;
    if (!r(&n, 8) || n > (1ull << 32)) return false;
    v.resize(n);
    return r(v.data(), n * sizeof(v[0]));
  };
  char magic[4];
  uint32_t ver = 0;
  uint64_t dg = 0;
  int32_t hdr[8];
  if (!r(magic, 4) || std::memcmp(magic, "RTNP", 4) != 0 || !r(&ver, 4) || ver != kPackVersion || !r(&dg, 8) ||
      dg != digest || !r(hdr, sizeof(hdr)) || hdr[0] != mode)
    return false;
  pk->mode = hdr[0];
  pk->n_in = hdr[1];
  pk->n_out = hdr[2];
  pk->n_layers = hdr[3];
  pk->act = hdr[4];
  pk->pwp = hdr[5];
  pk->split = hdr[6];
  pk->bf16 = hdr[7];
  return rv(pk->mu) && rv(pk->w0) && rv(pk->w0t) && rv(pk->b0) && rv(pk->bl) && rv(pk->bh) && rv(pk->th) &&
         rv(pk->tl);
}

// In-process cache: one packed device model per (file digest, device,
// precision), shared by every rtn_model_load_rmlp of identical bytes and freed
// with its last handle.
struct CacheKey {
  uint64_t digest;
  int device, prec;
  bool operator<(const CacheKey& o) const {
    return std::tie(digest, device, prec) < std::tie(o.digest, o.device, o.prec);
  }
};
std::mutex g_cache_mu;
std::map<CacheKey, rtn_model*> g_cache;

// RMLP v1/v2 parser of a file's bytes (proj/src/neural.cpp:720-755; v2 adds activation tag 2).
HostModel ParseRmlp(const std::vector<char>& bytes) {
  size_t pos = 0;
  auto rd = [&](void* p, size_t n) {
    if (n > bytes.size() - pos) throw Error(RTN_ECONFIG, "unexpected end of file");
    std::memcpy(p, bytes.data() + pos, n);
    pos += n;
  };
  char magic[4];
  rd(magic, 4);
  if (std::memcmp(magic, "RMLP", 4) != 0) throw Error(RTN_ECONFIG, "model: not a model file");
  uint32_t version;
  rd(&version, 4);
  if (version != 1 && version != 2) throw Error(RTN_ECONFIG, "model: unsupported version");
  uint8_t tag;
  rd(&tag, 1);
  HostModel m;
  if (version == 1) m.act = tag == 0 ? 0 : 1;
  else if (tag <= 2) m.act = tag;
  else throw Error(RTN_ECONFIG, "model: unknown activation tag");
  uint32_t n;
  rd(&n, 4);
  std::string variant(n, '\0');
  if (n) rd(&variant[0], n);
  uint64_t seed;
  rd(&seed, 8);
  uint32_t ns;
  rd(&ns, 4);
  if (ns < 2 || ns > 4096) throw Error(RTN_ECONFIG, "mlp: need at least input and output layers");
  m.sizes.resize(ns);
  for (auto& s : m.sizes) {
    uint32_t v;
    rd(&v, 4);
    s = static_cast<int>(v);
  }
  const int in_d = m.sizes.front(), out_d = m.sizes.back();
  m.in_mean.resize(in_d);
  m.in_scale.resize(in_d);
  m.out_mean.resize(out_d);
  m.out_scale.resize(out_d);
  rd(m.in_mean.data(), 8 * in_d);
  rd(m.in_scale.data(), 8 * in_d);
  rd(m.out_mean.data(), 8 * out_d);
  rd(m.out_scale.data(), 8 * out_d);
  for (size_t l = 0; l + 1 < m.sizes.size(); ++l) {
    m.W.emplace_back(static_cast<size_t>(m.sizes[l + 1]) * m.sizes[l]);
    m.b.emplace_back(static_cast<size_t>(m.sizes[l + 1]));
    rd(m.W.back().data(), 8 * m.W.back().size());
    rd(m.b.back().data(), 8 * m.b.back().size());
  }
  return m;
}

// Kernel choice (RTN_KERNEL=pair|latency|quad|rows|split|rowsb forces one where it applies):
//   quad    : width 512, order <= 1, K <= 2·(#SMs/4) — 4-CTA clusters, each
//             CTA pair computes one 256-neuron block (rtn_quad.cuh): one MPC step;
//   latency : pair kernel with one node per CTA side, K <= #SMs;
//   rows    : TF32 width-256 throughput batches, activations as the A operand
//             in TMEM (rtn_rows.cuh);
//   split   : TF32 width-512 throughput batches, the A operand split between
//             TMEM and shared memory (rtn_split.cuh);
//   rowsb   : BF16 width-512 throughput batches (n_in >= 15), the whole layer
//             input as the A operand in TMEM (rtn_rowsb.cuh);
//   pair    : pair-kernel throughput tiles (rtn_pair.cuh).
enum class Kern { kPair, kLatency, kQuad, kRows, kSplit, kRowsB };
Kern Choose(const rtn_model* m, long long K, int num_sms) {
  const bool lat_ok = m->n_in + 1 <= 24;
  const bool quad_ok = lat_ok && m->pair_wp == 512 && m->n_in <= rtn::kMaxIn0 && K <= 2 * (num_sms / 4);
  const bool rows_geom = m->pair_mode == rtn::kTF32 && m->n_in >= rtn::kRowsMinIn && m->n_in <= rtn::kRowsMaxInHost;
  const bool rows_ok = rows_geom && m->pair_wp == 256 && m->n_hidden - 1 <= rtn::kRowsMaxMmaHost;
  const bool split_ok = rows_geom && m->pair_wp == 512;
  const bool rowsb_ok = m->pair_mode == rtn::kBF16 && m->pair_wp == 512 && m->n_in >= rtn::kRbMinInHost &&
                        m->n_in <= rtn::kRowsMaxInHost;
  if (const char* e = std::getenv("RTN_KERNEL")) {
    if (std::strcmp(e, "quad") == 0 && quad_ok) return Kern::kQuad;
    if (std::strcmp(e, "rows") == 0 && rows_ok) return Kern::kRows;
    if (std::strcmp(e, "split") == 0 && split_ok) return Kern::kSplit;
    if (std::strcmp(e, "rowsb") == 0 && rowsb_ok) return Kern::kRowsB;
    if (std::strcmp(e, "latency") == 0 && lat_ok) return Kern::kLatency;
    if (std::strcmp(e, "pair") == 0) return Kern::kPair;
    // a kernel that does not apply to this model: the default choice below
  }
  const char* q = std::getenv("RTN_QUAD");
  if (quad_ok && !(q && q[0] == '0')) return Kern::kQuad;
  if (lat_ok && K <= num_sms) return Kern::kLatency;
  const char* r = std::getenv("RTN_ROWS");
  if (rows_ok && !(r && r[0] == '0')) return Kern::kRows;
  const char* sp = std::getenv("RTN_SPLIT");
  if (split_ok && !(sp && sp[0] == '0')) return Kern::kSplit;
  const char* rb = std::getenv("RTN_ROWSB");
  if (rowsb_ok && !(rb && rb[0] == '0')) return Kern::kRowsB;
  return Kern::kPair;
}

// Reverse mode (rtn_reverse.cuh, rtn_pair.cuh ORD2 3/4): per chunk of nodes,
// the value pass (f and the σ' scratch) then the adjoint pass (J). Chunks are
// as large as a kRevScratchBytes scratch allows and of equal size (no short
// last chunk leaving most CTA pairs idle).
constexpr size_t kRevScratchBytes = size_t{2} << 30;
void EnqueueReverse(rtn_ctx* c, const rtn::KParams& base, long long K) {
  const rtn_model* m = c->model;
  const bool split_sched = m->reverse_ok;  // TF32 width 512; else the pair-kernel variants
  // scratch: fp16 slopes (split schedule) / fp32 slopes (pair variants: the split-precision modes)
  const size_t per_node = static_cast<size_t>(m->n_hidden) * m->pair_wp * (split_sched ? 2 : 4);
  long long r_max = std::max<long long>(1024, static_cast<long long>(kRevScratchBytes / per_node));
  if (const char* ch = std::getenv("RTN_REV_CHUNK")) r_max = std::max(1LL, std::atoll(ch));  // tests: force chunking
  const long long n_chunks = (K + r_max - 1) / r_max;
  const long long R = (K + n_chunks - 1) / n_chunks;
  const size_t need = per_node * static_cast<size_t>(R);
  if (need > c->rev_s_cap) {
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    cudaFree(c->d_rev_s);
    c->d_rev_s = nullptr;
    c->rev_s_cap = 0;
    CUDA_CHECK(cudaMalloc(&c->d_rev_s, need));
    c->rev_s_cap = need;
  }
  const int n_in = m->n_in, n_out = m->n_out;
  const int ntc = rtn::PairReverseNtc(m->pair_mode, m->pair_wp, 0), ntc1 = rtn::PairReverseNtc(m->pair_mode, m->pair_wp, 1);
  for (long long lo = 0; lo < K; lo += R) {
    const long long n = std::min(R, K - lo);
    rtn::KParams p = base;
    p.z = base.z + lo * n_in;
    p.f = base.f + lo * n_out;
    p.jac = base.jac + lo * n_out * n_in;
    p.K = n;
    p.rev_s = c->d_rev_s;
    p.wl = m->d_wl32;
    cudaError_t e;
    if (split_sched) {
      p.nt = 128;
      p.P = 128;  // pass 0: one row per node
      p.num_tiles = (n + 255) / 256;
      int grid = 2 * static_cast<int>(std::min<long long>(p.num_tiles, c->num_sms / 2));
      e = rtn::LaunchReverse(0, p, m->tmap_h64, m->tmap_l, grid, c->stream);
      if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("reverse value pass: ") + cudaGetErrorString(e));
      p.P = 128 / n_out;  // pass 1: n_out adjoint rows per node
      p.num_tiles = (n + 2 * p.P - 1) / (2 * p.P);
      grid = 2 * static_cast<int>(std::min<long long>(p.num_tiles, c->num_sms / 2));
      e = rtn::LaunchReverse(1, p, m->tmap_ht64, m->tmap_w0p, grid, c->stream);
      if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("reverse adjoint pass: ") + cudaGetErrorString(e));
    } else {
      p.lo_rows = m->lo_rows;
      const char* tp = std::getenv("RTN_TRACE_PASS");  // profiling aid: trace only this pass
      const int trace_pass = tp ? std::atoi(tp) : 1;
      unsigned long long* const trace = p.trace;
      p.trace = trace_pass == 0 ? trace : nullptr;
      p.P = ntc;  // pass 0: one row per node, ntc nodes per CTA side
      p.nt = ntc;
      p.num_tiles = (n + 2 * ntc - 1) / (2 * ntc);
      int grid = 2 * static_cast<int>(std::min<long long>(p.num_tiles, c->num_sms / 2));
      e = rtn::LaunchPairReverse(m->pair_mode, m->pair_wp, 0, p, m->tmap_h, m->tmap_l, grid, c->stream);
      if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("reverse value pass: ") + cudaGetErrorString(e));
      p.trace = trace_pass == 1 ? trace : nullptr;
      p.P = ntc1 / 6;  // pass 1: 6 adjoint rows per node
      p.nt = ntc1;
      p.num_tiles = (n + 2 * p.P - 1) / (2 * p.P);
      grid = 2 * static_cast<int>(std::min<long long>(p.num_tiles, c->num_sms / 2));
      e = rtn::LaunchPairReverse(m->pair_mode, m->pair_wp, 1, p, m->tmap_ht, m->tmap_w0p, grid, c->stream);
      if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("reverse adjoint pass: ") + cudaGetErrorString(e));
    }
    c->launches += 2;
  }
}

// d_zx/d_zu (optional): gather the quadrotor rows [x_k; u_k] from an iterate
// (n_inst x (N+1) x 13 states, K x 4 inputs) instead of reading d_z.
void Enqueue(rtn_ctx* c, const double* d_z, long long K, int order, double* d_f, double* d_jac, double* d_hess,
             const double* d_zx, const double* d_zu, int zN) {
  const rtn_model* m = c->model;
  if (K == 0) return;
  rtn::KParams prm{};
  prm.z = d_z;
  prm.zx = d_zx;
  prm.zu = d_zu;
  prm.zN = zN;
  prm.f = d_f;
  prm.jac = order >= 1 ? d_jac : nullptr;
  prm.hess = nullptr;
  prm.K = K;
  prm.n_in = m->n_in;
  prm.n_out = m->n_out;
  prm.n_hidden = m->n_hidden;
  prm.act = m->act;
  prm.order = order;
  prm.lo_rows = m->lo_rows;
  prm.mu = m->d_mu;
  prm.nonfinite = c->h_nonfinite;
  prm.w0 = m->d_w0;
  prm.w0t = m->d_w0t;
  prm.b0 = m->d_b0;
  prm.bh = m->d_bh_pair;
  prm.bl = m->d_bl;
  if (const char* d = std::getenv("RTN_DEBUG")) prm.dbg = std::atoi(d);
  if (const char* tr = std::getenv("RTN_TRACE")) {  // per-event timestamps of pair 0 (profiling aid)
    prm.trace_tile = std::max(0, std::atoi(tr) - 1);
    if (!trace_buf) {
      if (std::getenv("RTN_TRACE_HOST")) {  // host-mapped: readable while a kernel hangs (debug aid)
        CUDA_CHECK(cudaHostAlloc(&trace_host, 256 * 8, cudaHostAllocMapped));
        CUDA_CHECK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&trace_buf), trace_host, 0));
      } else {
        CUDA_CHECK(cudaMalloc(&trace_buf, 256 * 8));
      }
    }
    CUDA_CHECK(cudaMemsetAsync(trace_buf, 0, 256 * 8, c->stream));
    prm.trace = trace_buf;
  }
  cudaError_t e;
  if (order == 1 && c->jac_mode == 1 && (m->reverse_ok || m->reverse_pair_ok) && prm.jac != nullptr &&
      d_zx == nullptr) {
    EnqueueReverse(c, prm, K);
    return;
  }
  if (order == 2) {
    // pair tiles of the node's carrier (value + tangents) plus Hessian slots
    prm.P = 1;
    prm.nt = rtn::Order2Ntc(m->pair_mode, m->n_in);
    if (const char* o2 = std::getenv("RTN_ORD2_NTC")) {  // A/B aid: the generic tiles' heights
      const int v = std::atoi(o2);
      if ((v == 24 || v == 40) && 1 + m->n_in <= v) prm.nt = v;
    }
    prm.ord2_g = rtn::ord2_tiles(m->n_in, prm.nt);
    prm.hess = d_hess;
    prm.num_tiles = static_cast<long long>(prm.ord2_g) * K;
    const int grid = 2 * static_cast<int>(std::min<long long>(prm.num_tiles, c->num_sms / 2));
    e = rtn::LaunchPairOrder2(m->pair_mode, prm, m->tmap_h, m->tmap_l, m->pair_wp, grid, c->stream);
    if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("order-2 kernel launch: ") + cudaGetErrorString(e));
    c->launches += 1;
    return;
  }
  const Kern kern = Choose(m, K, c->num_sms);
  if (kern == Kern::kQuad) {
    prm.P = 1;
    prm.nt = ((1 + m->n_in + 7) / 8) * 8;
    prm.num_tiles = (K + 1) / 2;
    const int g4 = static_cast<int>(4 * prm.num_tiles);
    e = m->pair_mode == rtn::kBF16x3  ? rtn::LaunchQuadBF16x3(prm, m->tmap_h, m->tmap_l, g4, c->stream)
        : m->pair_mode == rtn::kBF16   ? rtn::LaunchQuadBF16(prm, m->tmap_h, m->tmap_l, g4, c->stream)
        : m->pair_mode == rtn::k3xTF32 ? rtn::LaunchQuad3xTF32(prm, m->tmap_h, m->tmap_l, g4, c->stream)
                                       : rtn::LaunchQuadTF32(prm, m->tmap_h, m->tmap_l, g4, c->stream);
    if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("quad kernel launch: ") + cudaGetErrorString(e));
    c->launches += 1;
    return;
  }
  if (kern == Kern::kRowsB) {
    // BF16 width 512: the whole layer input as the A operand in TMEM (rtn_rowsb.cuh)
    prm.P = 128 / (1 + m->n_in);
    prm.nt = 128;
    prm.num_tiles = (K + 2 * prm.P - 1) / (2 * prm.P);
    const int g6 = 2 * static_cast<int>(std::min<long long>(prm.num_tiles, c->num_sms / 2));
    e = rtn::LaunchRowsBF16(prm, m->tmap_h64, m->tmap_l, g6, c->stream);
    if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("rowsb kernel launch: ") + cudaGetErrorString(e));
    c->launches += 1;
    return;
  }
  if (kern == Kern::kSplit) {
    // width 512: activations split between TMEM and shared memory (rtn_split.cuh), 128 rows per CTA
    prm.P = 128 / (1 + m->n_in);
    prm.nt = 128;
    prm.num_tiles = (K + 2 * prm.P - 1) / (2 * prm.P);
    const int g5 = 2 * static_cast<int>(std::min<long long>(prm.num_tiles, c->num_sms / 2));
    e = rtn::LaunchSplitTF32(prm, m->tmap_h64, m->tmap_l, g5, c->stream);
    if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("split kernel launch: ") + cudaGetErrorString(e));
    c->launches += 1;
    return;
  }
  if (kern == Kern::kRows) {
    // width 256: activations as the A operand in TMEM (rtn_rows.cuh), 128 rows per CTA
    prm.P = 128 / (1 + m->n_in);
    prm.nt = 128;
    prm.num_tiles = (K + 2 * prm.P - 1) / (2 * prm.P);
    const int g3 = 2 * static_cast<int>(std::min<long long>(prm.num_tiles, c->num_sms / 2));
    e = rtn::LaunchRowsTF32(prm, m->tmap_h, m->tmap_l, g3, c->stream);
    if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("rows kernel launch: ") + cudaGetErrorString(e));
    c->launches += 1;
    return;
  }
  const bool lat = kern == Kern::kLatency;
  const rtn::PairGeom g = rtn::PairGeometry(m->pair_mode, m->pair_wp, lat, m->n_in);
  prm.P = g.P;
  prm.nt = ((g.P * (1 + m->n_in) + 7) / 8) * 8;
  if (prm.nt > g.ntc_max) throw Error(RTN_EUNSUPPORTED, "node rows exceed the pair tile");
  prm.num_tiles = (K + 2 * prm.P - 1) / (2 * prm.P);  // pair tiles of 2P nodes
  const int grid = 2 * static_cast<int>(std::min<long long>(prm.num_tiles, c->num_sms / 2));
  if (m->pair_mode == rtn::kTF32)
    e = rtn::LaunchPairTF32(prm, m->tmap_h, m->tmap_l, m->pair_wp, lat, grid, c->stream);
  else if (m->pair_mode == rtn::k3xTF32)
    e = rtn::LaunchPair3xTF32(prm, m->tmap_h, m->tmap_l, m->pair_wp, lat, grid, c->stream);
  else if (m->pair_mode == rtn::kBF16)
    e = rtn::LaunchPairBF16(prm, m->tmap_h, m->tmap_l, m->pair_wp, lat, grid, c->stream);
  else
    e = rtn::LaunchPairBF16x3(prm, m->tmap_h, m->tmap_l, m->pair_wp, lat, grid, c->stream);
  if (e != cudaSuccess) throw Error(RTN_ECUDA, std::string("pair kernel launch: ") + cudaGetErrorString(e));
  c->launches += 1;
}

}  // namespace rtn_host

// ----------------------------------------------------------------------------
extern "C" {

const char* rtn_last_error(void) { return g_err.c_str(); }

// Profiling aid (not part of the C-ABI contract): copies the RTN_TRACE buffer
// (256 globaltimer stamps of pair 0's first tile) after a synchronised call.
int rtn_debug_trace(unsigned long long* out, int n) {
  if (!trace_buf || n > 256) return 1;
  if (trace_host) {  // no CUDA call: works while the traced kernel is still running
    std::memcpy(out, trace_host, sizeof(unsigned long long) * n);
    return 0;
  }
  return cudaMemcpy(out, trace_buf, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : 1;
}

rtn_status rtn_model_load_rmlp(const char* path, int device, rtn_precision p, rtn_model** out) {
  return Guard([&] {
    if (!path || !out) throw Error(RTN_ECONFIG, "null argument");
    std::vector<char> bytes;
    {
      std::ifstream in(path, std::ios::binary);
      if (!in) throw Error(RTN_ECONFIG, std::string("model: cannot open '") + path + "'");
      bytes.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    }
    const uint64_t digest = Fnv1a64(bytes);
    const CacheKey key{digest, device, static_cast<int>(p)};
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      auto it = g_cache.find(key);
      if (it != g_cache.end()) {  // identical bytes already on this device in this precision
        ++it->second->refs;
        *out = it->second;
        return;
      }
    }
    // RTN_PACK_CACHE=<dir>: the packed device layout on disk, keyed by the digest
    const char* dir = std::getenv("RTN_PACK_CACHE");
    const int mode = p == RTN_TF32 ? rtn::kTF32 : p == RTN_3XTF32 ? rtn::k3xTF32 : p == RTN_BF16X3 ? rtn::kBF16x3 : rtn::kBF16;
    const std::string pack_path = dir ? std::string(dir) + "/" + Hex16(digest) + "-p" + std::to_string(p) + ".rtnp" : "";
    Packed pk;
    bool from_pack = !pack_path.empty() && ReadPacked(pack_path, digest, mode, &pk);
    if (!from_pack) {
      pk = PackModel(ParseRmlp(bytes), p);
      if (!pack_path.empty()) WritePacked(pack_path, digest, pk);
    }
    rtn_model* m = UploadModel(pk, device);
    m->digest = digest;
    m->from_pack = from_pack;
    m->cached = true;
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      auto it = g_cache.find(key);
      if (it != g_cache.end()) {  // another thread loaded it meanwhile
        ++it->second->refs;
        *out = it->second;
        m->cached = false;
        delete m;
        return;
      }
      g_cache[key] = m;
    }
    *out = m;
  });
}

// FNV-1a 64 digest (hex) of the RMLP file a model was loaded from ("" for models
// built from arrays) and whether its packed layout came from the on-disk cache.
rtn_status rtn_model_digest(const rtn_model* m, char out[17], int* from_pack_cache) {
  return Guard([&] {
    if (!m || !out) throw Error(RTN_ECONFIG, "null argument");
    const std::string h = m->cached || m->digest ? Hex16(m->digest) : std::string();
    std::memcpy(out, h.c_str(), h.size() + 1);
    if (from_pack_cache) *from_pack_cache = m->from_pack ? 1 : 0;
  });
}

rtn_status rtn_model_from_arrays(const int* sizes, int n_sizes, int activation, const double* const* W,
                                 const double* const* b, const double* in_mean, const double* in_scale,
                                 const double* out_mean, const double* out_scale, int device, rtn_precision p,
                                 rtn_model** out) {
  return Guard([&] {
    if (!sizes || !W || !b || !in_mean || !in_scale || !out_mean || !out_scale || !out || n_sizes < 2)
      throw Error(RTN_ECONFIG, "mlp: need at least input and output layers");
    HostModel hm;
    hm.sizes.assign(sizes, sizes + n_sizes);
    for (int s : hm.sizes)
      if (s < 1) throw Error(RTN_ECONFIG, "mlp: layer sizes must be positive");
    hm.act = activation;
    for (int l = 0; l + 1 < n_sizes; ++l) {
      if (!W[l] || !b[l]) throw Error(RTN_ECONFIG, "null layer");
      hm.W.emplace_back(W[l], W[l] + static_cast<size_t>(sizes[l + 1]) * sizes[l]);
      hm.b.emplace_back(b[l], b[l] + sizes[l + 1]);
    }
    hm.in_mean.assign(in_mean, in_mean + sizes[0]);
    hm.in_scale.assign(in_scale, in_scale + sizes[0]);
    hm.out_mean.assign(out_mean, out_mean + sizes[n_sizes - 1]);
    hm.out_scale.assign(out_scale, out_scale + sizes[n_sizes - 1]);
    *out = BuildModel(hm, device, p);
  });
}

void rtn_model_free(rtn_model* m) {
  if (!m) return;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (m->cached) {
      if (--m->refs > 0) return;
      g_cache.erase(CacheKey{m->digest, m->device, static_cast<int>(m->prec)});
    }
  }
  delete m;
}

rtn_status rtn_model_info(const rtn_model* m, int* n_in, int* n_out, int* n_layers, int* activation,
                          int* padded_width) {
  return Guard([&] {
    if (!m) throw Error(RTN_ECONFIG, "null model");
    if (n_in) *n_in = m->n_in;
    if (n_out) *n_out = m->n_out;
    if (n_layers) *n_layers = m->n_layers;
    if (activation) *activation = m->act;
    if (padded_width) *padded_width = m->wp;
  });
}

rtn_status rtn_ctx_create(const rtn_model* m, long long max_rows, int max_order, int latency_mode, rtn_ctx** out) {
  return Guard([&] {
    if (!m || !out) throw Error(RTN_ECONFIG, "null argument");
    if (max_rows < 1) throw Error(RTN_EDOMAIN, "max_rows must be positive");
    if (max_order < 0 || max_order > 2) throw Error(RTN_ECONFIG, "order must be 0, 1 or 2");
    if (max_order == 2) {
      if (m->act == RTN_ACT_RELU)
        throw Error(RTN_EUNSUPPORTED, "mlp hessian: relu networks are not twice differentiable");
      if (m->n_in > rtn::kMaxIn2)
        throw Error(RTN_EUNSUPPORTED, "second-order device path supports at most 31 inputs (1 + n_in carrier rows <= 32)");
    }
    CUDA_CHECK(cudaSetDevice(m->device));
    std::unique_ptr<rtn_ctx> c(new rtn_ctx());
    c->model = m;
    c->max_rows = max_rows;
    c->max_order = max_order;
    c->latency_mode = latency_mode;
    CUDA_CHECK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, m->device));
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking));
    c->ev_in.resize(kMaxChunks);
    c->ev_k.resize(kMaxChunks);
    for (int i = 0; i < kMaxChunks; ++i) {
      CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming));
    }
    c->stream = c->own_stream;
    CUDA_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&c->h_nonfinite), sizeof(unsigned int), cudaHostAllocMapped));
    *c->h_nonfinite = 0;
    const size_t zb = sizeof(double) * max_rows * m->n_in, fb = sizeof(double) * max_rows * m->n_out,
                 jb = fb * m->n_in;
    CUDA_CHECK(cudaMalloc(&c->d_z, zb));
    CUDA_CHECK(cudaMalloc(&c->d_f, fb));
    if (max_order >= 1) CUDA_CHECK(cudaMalloc(&c->d_jac, jb));
    if (max_order >= 2) CUDA_CHECK(cudaMalloc(&c->d_hess, jb * m->n_in));
    // pinned staging for pageable caller buffers is allocated on first use
    *out = c.release();
  });
}

void rtn_ctx_free(rtn_ctx* c) { delete c; }

rtn_status rtn_ctx_set_stream(rtn_ctx* c, void* s) {
  return Guard([&] {
    if (!c) throw Error(RTN_ECONFIG, "null context");
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
  });
}

rtn_status rtn_ctx_synchronize(rtn_ctx* c) {
  return Guard([&] {
    if (!c) throw Error(RTN_ECONFIG, "null context");
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

rtn_status rtn_ctx_set_jacobian_mode(rtn_ctx* c, int mode) {
  return Guard([&] {
    if (!c) throw Error(RTN_ECONFIG, "null context");
    if (mode != 0 && mode != 1) throw Error(RTN_ECONFIG, "jacobian mode must be 0 (forward) or 1 (reverse)");
    if (mode == 1 && !c->model->reverse_ok && !c->model->reverse_pair_ok)
      throw Error(RTN_EUNSUPPORTED,
                  "reverse mode needs n_in <= 24 and a TF32 model of padded width 512, or a 3xTF32 / bf16x3 model "
                  "of padded width 256 or 512 with 6 outputs");
    if (mode != c->jac_mode) {  // captured latency graphs hold the other mode's kernels
      for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
      c->graphs.clear();
    }
    c->jac_mode = mode;
  });
}

rtn_status rtn_ctx_nonfinite(rtn_ctx* c, int* flag, int reset) {
  return Guard([&] {
    if (!c || !flag) throw Error(RTN_ECONFIG, "null argument");
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    *flag = *c->h_nonfinite ? 1 : 0;
    if (reset) *c->h_nonfinite = 0;
  });
}

rtn_status rtn_ctx_counters(const rtn_ctx* c, unsigned long long* calls, unsigned long long* points,
                            unsigned long long* launches) {
  return Guard([&] {
    if (!c) throw Error(RTN_ECONFIG, "null context");
    if (calls) *calls = c->calls;
    if (points) *points = c->points;
    if (launches) *launches = c->launches;
  });
}

}  // extern "C"

namespace rtn_host {
void EnsureStaging(rtn_ctx* c) {
  if (c->h_z) return;
  const rtn_model* m = c->model;
  const size_t zr = sizeof(double) * m->n_in, fr = sizeof(double) * m->n_out, jr = fr * m->n_in;
  CUDA_CHECK(cudaMallocHost(&c->h_z, zr * c->max_rows));
  CUDA_CHECK(cudaMallocHost(&c->h_f, fr * c->max_rows));
  if (c->max_order >= 1) CUDA_CHECK(cudaMallocHost(&c->h_jac, jr * c->max_rows));
  if (c->max_order >= 2) CUDA_CHECK(cudaMallocHost(&c->h_hess, jr * m->n_in * c->max_rows));
}

bool IsPinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void CheckCall(const rtn_ctx* c, long long K, int order) {
  if (!c) throw Error(RTN_ECONFIG, "null context");
  if (order < 0 || order > 2) throw Error(RTN_ECONFIG, "prepare nodes: order must be 0, 1 or 2");
  if (order == 2 && c->model->act == RTN_ACT_RELU)
    throw Error(RTN_EUNSUPPORTED, "mlp hessian: relu networks are not twice differentiable");
  if (order > c->max_order) throw Error(RTN_EUNSUPPORTED, "order exceeds the context's max_order");
  if (K < 0 || K > c->max_rows) throw Error(RTN_EDOMAIN, "K outside [0, max_rows]");
}
}  // namespace rtn_host

extern "C" {

rtn_status rtn_prepare(rtn_ctx* c, const double* z, long long K, int n_cols, int order, double* f, double* jac,
                       double* hess) {
  NvtxRange nvtx("rtn_prepare");
  return Guard([&] {
    CheckCall(c, K, order);
    *c->h_nonfinite = 0;  // per-call flag (the call is blocking: no kernel of this context is in flight)
    const rtn_model* m = c->model;
    if (n_cols != m->n_in)
      throw Error(RTN_EDOMAIN, "mlp eval: feature dim " + std::to_string(n_cols) + " does not match model input " +
                                   std::to_string(m->n_in));
    if (hess != nullptr && order != 2) throw Error(RTN_ECONFIG, "hess must be NULL unless order == 2");
    if (K > 0 && (!z || !f || (order >= 1 && !jac) || (order == 2 && !hess))) throw Error(RTN_ECONFIG, "null buffer");
    c->calls += 1;
    c->points += static_cast<unsigned long long>(K);
    if (K == 0) return;
    CUDA_CHECK(cudaSetDevice(m->device));
    const size_t zr = sizeof(double) * m->n_in, fr = sizeof(double) * m->n_out, jr = fr * m->n_in, hr = jr * m->n_in;
    if (c->latency_mode && K <= kGraphMaxRows && ZeroCopy() && IsPinned(z) && IsPinned(f) &&
        (order < 1 || IsPinned(jac)) && (order < 2 || IsPinned(hess))) {
      // One MPC step on page-locked caller buffers: the kernel reads z and
      // writes f/J/H in place (unified addressing); one graph per buffer set.
      double* jj = order >= 1 ? jac : nullptr;
      double* hh = order == 2 ? hess : nullptr;
      cudaGraphExec_t exec = nullptr;
      for (auto& g : c->graphs)
        if (g.K == K && g.order == order && g.io[0] == z && g.io[1] == f && g.io[2] == jj && g.io[3] == hh)
          exec = g.exec;
      if (!exec) {
        Enqueue(c, z, K, order, f, jj, hh);  // first launch outside capture
        CUDA_CHECK(cudaStreamSynchronize(c->stream));
        cudaGraph_t graph;
        CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        Enqueue(c, z, K, order, f, jj, hh);
        CUDA_CHECK(cudaStreamEndCapture(c->stream, &graph));
        CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
        CUDA_CHECK(cudaGraphDestroy(graph));
        c->launches -= 1;  // the capture pass launched nothing
        if (c->graphs.size() >= 64) {  // bounded cache of buffer sets
          cudaGraphExecDestroy(c->graphs.front().exec);
          c->graphs.erase(c->graphs.begin());
        }
        c->graphs.push_back({K, order, exec, {z, f, jj, hh}});
        return;
      }
      c->launches += 1;
      CUDA_CHECK(cudaGraphLaunch(exec, c->stream));
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
      return;
    }
    if (c->latency_mode && K <= kGraphMaxRows) {
      // One MPC step: pinned staging + a CUDA graph of H2D → kernel → D2H
      // (or the kernel alone on the staging, zero-copy), so the call costs
      // one graph launch and one synchronisation.
      EnsureStaging(c);
      std::memcpy(c->h_z, z, zr * K);
      cudaGraphExec_t exec = nullptr;
      for (auto& g : c->graphs)
        if (g.K == K && g.order == order && g.io[0] == nullptr) exec = g.exec;
      if (!exec) {
        Enqueue(c, c->d_z, K, order, c->d_f, c->d_jac, c->d_hess);  // first launch outside capture (attributes, checks)
        CUDA_CHECK(cudaStreamSynchronize(c->stream));
        cudaGraph_t graph;
        CUDA_CHECK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        if (ZeroCopy()) {
          // The kernel reads z from and writes f/J/H to the pinned staging
          // directly (unified addressing): the graph is the kernel alone.
          Enqueue(c, c->h_z, K, order, c->h_f, order >= 1 ? c->h_jac : nullptr, order == 2 ? c->h_hess : nullptr);
        } else {
          CUDA_CHECK(cudaMemcpyAsync(c->d_z, c->h_z, zr * K, cudaMemcpyHostToDevice, c->stream));
          Enqueue(c, c->d_z, K, order, c->d_f, order >= 1 ? c->d_jac : nullptr, order == 2 ? c->d_hess : nullptr);
          CUDA_CHECK(cudaMemcpyAsync(c->h_f, c->d_f, fr * K, cudaMemcpyDeviceToHost, c->stream));
          if (order >= 1) CUDA_CHECK(cudaMemcpyAsync(c->h_jac, c->d_jac, jr * K, cudaMemcpyDeviceToHost, c->stream));
          if (order == 2) CUDA_CHECK(cudaMemcpyAsync(c->h_hess, c->d_hess, hr * K, cudaMemcpyDeviceToHost, c->stream));
        }
        CUDA_CHECK(cudaStreamEndCapture(c->stream, &graph));
        CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
        CUDA_CHECK(cudaGraphDestroy(graph));
        c->graphs.push_back({K, order, exec, {nullptr, nullptr, nullptr, nullptr}});
      } else {
        c->launches += 1;  // the graph's kernel node
      }
      CUDA_CHECK(cudaGraphLaunch(exec, c->stream));
      CUDA_CHECK(cudaStreamSynchronize(c->stream));
      std::memcpy(f, c->h_f, fr * K);
      if (order >= 1) std::memcpy(jac, c->h_jac, jr * K);
      if (order == 2) std::memcpy(hess, c->h_hess, hr * K);
      return;
    }
    // Page-locked caller buffers are DMA'd directly; pageable ones go through
    // the context's pinned staging.
    const bool pinned = IsPinned(z) && IsPinned(f) && (order < 1 || IsPinned(jac)) && (order < 2 || IsPinned(hess));
    const double* hz = z;
    double* hf = f;
    double* hj = jac;
    double* hh = hess;
    if (!pinned) {
      EnsureStaging(c);
      std::memcpy(c->h_z, z, zr * K);
      hz = c->h_z;
      hf = c->h_f;
      hj = c->h_jac;
      hh = c->h_hess;
    }
    // Large batches: chunk so H2D(i+1) and D2H(i−1) overlap kernel(i).
    const int chunks = K >= kChunkMinRows ? kMaxChunks : 1;
    const long long per = (K + chunks - 1) / chunks;
    CUDA_CHECK(cudaEventRecord(c->ev_in[0], c->stream));  // order after prior work on the compute stream
    CUDA_CHECK(cudaStreamWaitEvent(c->s_in, c->ev_in[0], 0));
    for (int i = 0; i < chunks; ++i) {
      const long long r0 = i * per, n = std::min(per, K - r0);
      if (n <= 0) break;
      CUDA_CHECK(cudaMemcpyAsync(c->d_z + r0 * m->n_in, hz + r0 * m->n_in, zr * n, cudaMemcpyHostToDevice, c->s_in));
      CUDA_CHECK(cudaEventRecord(c->ev_in[i], c->s_in));
      CUDA_CHECK(cudaStreamWaitEvent(c->stream, c->ev_in[i], 0));
      const long long nh = static_cast<long long>(m->n_out) * m->n_in * m->n_in;
      Enqueue(c, c->d_z + r0 * m->n_in, n, order, c->d_f + r0 * m->n_out,
              order >= 1 ? c->d_jac + r0 * m->n_out * m->n_in : nullptr, order == 2 ? c->d_hess + r0 * nh : nullptr);
      CUDA_CHECK(cudaEventRecord(c->ev_k[i], c->stream));
      CUDA_CHECK(cudaStreamWaitEvent(c->s_out, c->ev_k[i], 0));
      CUDA_CHECK(cudaMemcpyAsync(hf + r0 * m->n_out, c->d_f + r0 * m->n_out, fr * n, cudaMemcpyDeviceToHost, c->s_out));
      if (order >= 1)
        CUDA_CHECK(cudaMemcpyAsync(hj + r0 * m->n_out * m->n_in, c->d_jac + r0 * m->n_out * m->n_in, jr * n,
                                   cudaMemcpyDeviceToHost, c->s_out));
      if (order == 2)
        CUDA_CHECK(cudaMemcpyAsync(hh + r0 * nh, c->d_hess + r0 * nh, hr * n, cudaMemcpyDeviceToHost, c->s_out));
    }
    CUDA_CHECK(cudaStreamSynchronize(c->s_out));
    if (!pinned) {
      std::memcpy(f, c->h_f, fr * K);
      if (order >= 1) std::memcpy(jac, c->h_jac, jr * K);
      if (order == 2) std::memcpy(hess, c->h_hess, hr * K);
    }
  });
}

rtn_status rtn_prepare_device(rtn_ctx* c, const double* d_z, long long K, int order, double* d_f, double* d_jac,
                              double* d_hess) {
  NvtxRange nvtx("rtn_prepare_device");
  return Guard([&] {
    CheckCall(c, K, order);
    if (d_hess != nullptr && order != 2) throw Error(RTN_ECONFIG, "hess must be NULL unless order == 2");
    if (K > 0 && (!d_z || !d_f || (order >= 1 && !d_jac) || (order == 2 && !d_hess)))
      throw Error(RTN_ECONFIG, "null buffer");
    c->calls += 1;
    c->points += static_cast<unsigned long long>(K);
    CUDA_CHECK(cudaSetDevice(c->model->device));
    Enqueue(c, d_z, K, order, d_f, d_jac, d_hess);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Continuity-block builder host side (resmpc::BuildQp, sqp_rti.cpp:59-155).
namespace {

constexpr int kNx = 13, kNu = 4;

// QuadParams::Validate (proj/src/dynamics.cpp:29-40), same messages.
void ValidateQuad(const rtn_quad_params& p) {
  if (!(p.mass > 0.0) || !(p.arm_length > 0.0) || !(p.torque_coeff > 0.0) || !(p.thrust_max > 0.0))
    throw Error(RTN_ECONFIG, "quad params: mass, arm_length, torque_coeff, thrust_max must be positive");
  if (!(std::min(p.inertia[0], std::min(p.inertia[1], p.inertia[2])) > 0.0))
    throw Error(RTN_ECONFIG, "quad params: inertia must be positive");
  double sum = 0.0;
  for (int i = 0; i < 4; ++i) {
    if (p.rotor_sign[i] != 1.0 && p.rotor_sign[i] != -1.0)
      throw Error(RTN_ECONFIG, "quad params: rotor_sign entries must be +1 or -1");
    sum += p.rotor_sign[i];
  }
  if (sum != 0.0) throw Error(RTN_ECONFIG, "quad params: need two rotors of each spin direction");
}

// OcpConfig::Validate(13, 4) (proj/src/sqp_rti.cpp:27-42), same messages.
void ValidateCfg(const rtn_ocp_config& c) {
  if (c.horizon < 1) throw Error(RTN_ECONFIG, "ocp config: horizon must be >= 1");
  if (!(c.dt > 0.0)) throw Error(RTN_ECONFIG, "ocp config: dt must be positive");
  for (double v : c.q_diag)
    if (v < 0.0) throw Error(RTN_ECONFIG, "ocp config: weights must be nonnegative");
  for (double v : c.r_diag)
    if (v < 0.0) throw Error(RTN_ECONFIG, "ocp config: weights must be nonnegative");
  for (int i = 0; i < kNu; ++i)
    if (c.u_min[i] >= c.u_max[i]) throw Error(RTN_ECONFIG, "ocp config: u_min must be below u_max");
  if (c.taylor_order != 1 && c.taylor_order != 2) throw Error(RTN_ECONFIG, "ocp config: taylor_order must be 1 or 2");
  if (c.variant < 0 || c.variant > 3)
    throw Error(RTN_ECONFIG, "unknown residual variant code " + std::to_string(c.variant) +
                                 " (expected full, a, a_u, ground)");
}

rtn::BlkParams MakeBlk(const rtn_quad_params& p, const rtn_ocp_config& c, long long n_inst) {
  rtn::BlkParams b;
  std::memset(&b, 0, sizeof b);  // padding too: the struct is compared bytewise as a graph-cache key
  b.n_inst = n_inst;
  b.N = c.horizon;
  b.order = c.taylor_order;
  b.variant = c.variant;
  b.dt = c.dt;
  b.mass = p.mass;
  b.inv_mass = 1.0 / p.mass;
  for (int i = 0; i < 3; ++i) {
    b.inertia[i] = p.inertia[i];
    b.inv_inertia[i] = 1.0 / p.inertia[i];
  }
  // MixingMatrix (proj/src/dynamics.cpp:42-55), fp64 on the host
  const double d = p.arm_length / std::sqrt(2.0);
  const double rx[4] = {d, -d, d, -d}, ry[4] = {-d, d, d, -d};
  for (int i = 0; i < 4; ++i) {
    b.mix[0][i] = 0.0;
    b.mix[1][i] = 0.0;
    b.mix[2][i] = 1.0;
    b.mix[3][i] = ry[i];
    b.mix[4][i] = -rx[i];
    b.mix[5][i] = p.rotor_sign[i] * p.torque_coeff;
  }
  for (int i = 0; i < kNx; ++i) {
    b.qd[i] = c.q_diag[i];
    b.qf[i] = c.has_q_terminal ? c.q_terminal[i] : c.q_diag[i];
  }
  for (int i = 0; i < kNu; ++i) {
    b.rd[i] = c.r_diag[i];
    b.umin[i] = c.u_min[i];
    b.umax[i] = c.u_max[i];
  }
  return b;
}

// One host array <-> one slice of the contiguous device area.
struct Slice {
  const double* src;  // host input (nullptr for outputs)
  double* dst;        // host output (nullptr for inputs)
  size_t off, n;      // doubles
};

struct QpPlan {
  std::vector<Slice> in, out;
  size_t in_total = 0, out_total = 0;
  size_t add_in(const double* h, size_t n) {
    in.push_back({h, nullptr, in_total, n});
    in_total += n;
    return in.back().off;
  }
  size_t add_out(double* h, size_t n) {  // null host pointer: not wanted
    if (!h) return SIZE_MAX;
    out.push_back({nullptr, h, out_total, n});
    out_total += n;
    return out.back().off;
  }
};

void Grow(double** d, size_t* cap, size_t need, bool pinned) {
  if (need <= *cap) return;
  if (pinned) {
    cudaFreeHost(*d);
    *d = nullptr;
    *cap = 0;
    CUDA_CHECK(cudaMallocHost(d, need * sizeof(double)));
  } else {
    cudaFree(*d);
    *d = nullptr;
    *cap = 0;
    CUDA_CHECK(cudaMalloc(d, need * sizeof(double)));
  }
  *cap = need;
}

std::string QpErrorMessage(unsigned long long w, int N, long long n_inst) {
  const long long node = static_cast<long long>(w >> 8);
  const int code = static_cast<int>(w & 0xff);
  const long long inst = node / N, k = node % N;
  std::string what = code / 10 == 1 ? "quad dynamics: quaternion norm too far from unit"
                                     : "rk4: non-finite derivative at stage " + std::to_string(code % 10);
  std::string msg = "build qp: node " + std::to_string(k) + ": " + what;
  if (n_inst > 1) msg = "instance " + std::to_string(inst) + ": " + msg;
  return msg;
}

bool AllPinned(const QpPlan& plan) {
  for (const Slice& s : plan.in)
    if (!IsPinned(s.src)) return false;
  for (const Slice& s : plan.out)
    if (!IsPinned(s.dst)) return false;
  return true;
}

// Shared driver of rtn_build_qp (approximations given) and rtn_cycle_qp
// (approximations computed on the device from z_k = [x_k; u_k]).
void RunQp(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst, const rtn_iterate* it,
           const rtn_approx* ap, rtn_qp_blocks* out, bool cycle, double* f, double* jac, double* hess) {
  if (!p || !cfg) throw Error(RTN_ECONFIG, "null argument");
  ValidateQuad(*p);  // configuration errors first, as BuildQp validates before any work
  ValidateCfg(*cfg);
  if (!c || !it || !out || (!cycle && !ap)) throw Error(RTN_ECONFIG, "null argument");
  const int N = cfg->horizon, order = cfg->taylor_order, var = cfg->variant;
  const int nf = rtn::VarNf(var), nr = rtn::VarNr(var);
  if (n_inst < 0) throw Error(RTN_EDOMAIN, "n_inst must be >= 0");
  const long long K = n_inst * N;
  if (K > c->max_rows) throw Error(RTN_EDOMAIN, "n_inst * horizon exceeds the context's max_rows");
  const rtn_model* m = c->model;
  if (cycle) {
    if (m->n_in != nf || m->n_out != nr)  // sqp_rti.cpp:196-197
      throw Error(RTN_ECONFIG, "controller: model dimensions do not match the plant's residual wiring (model " +
                                   std::to_string(m->n_in) + " -> " + std::to_string(m->n_out) + ", variant needs " +
                                   std::to_string(nf) + " -> " + std::to_string(nr) + ")");
    if (order > c->max_order) throw Error(RTN_EUNSUPPORTED, "taylor_order exceeds the context's max_order");
    if (order == 2 && m->act == RTN_ACT_RELU)
      throw Error(RTN_EUNSUPPORTED, "mlp hessian: relu networks are not twice differentiable");
  }
  if (K > 0 && (!it->xs || !it->us || !it->ref_xs || !it->ref_us)) throw Error(RTN_ECONFIG, "null iterate buffer");
  if (K > 0 && var == rtn::kVarGround && !it->aux)
    throw Error(RTN_EDOMAIN, "quadrotor plant: ground features need a 9-entry patch aux per node");
  if (!cycle && K > 0 && (!ap->z0 || !ap->f_bar || !ap->jac || (order == 2 && !ap->hess)))
    throw Error(RTN_ECONFIG, "null approximation buffer");
  if (cycle) {
    c->calls += 1;  // one batched model call per cycle (SPEC; test_sqp_rti.cpp:246-247)
    c->points += static_cast<unsigned long long>(K);
  }
  if (K == 0) return;
  CUDA_CHECK(cudaSetDevice(m->device));

  const size_t X = static_cast<size_t>(n_inst) * (N + 1) * kNx, U = static_cast<size_t>(K) * kNu,
               Kz = static_cast<size_t>(K);
  QpPlan plan;
  const size_t o_xs = plan.add_in(it->xs, X), o_us = plan.add_in(it->us, U), o_rxs = plan.add_in(it->ref_xs, X),
               o_rus = plan.add_in(it->ref_us, U);
  const size_t o_aux = var == rtn::kVarGround ? plan.add_in(it->aux, Kz * 9) : 0;
  size_t o_z0 = 0, o_fb = 0, o_jac = 0, o_hess = 0;
  if (!cycle) {
    o_z0 = plan.add_in(ap->z0, Kz * nf);
    o_fb = plan.add_in(ap->f_bar, Kz * nr);
    o_jac = plan.add_in(ap->jac, Kz * nr * nf);
    if (order == 2) o_hess = plan.add_in(ap->hess, Kz * nr * nf * nf);
  }
  const size_t o_a = plan.add_out(out->a, Kz * kNx * kNx), o_b = plan.add_out(out->b, Kz * kNx * kNu),
               o_phi = plan.add_out(out->phi_res, Kz * kNx), o_q = plan.add_out(out->q, X),
               o_r = plan.add_out(out->r, U), o_hx = plan.add_out(out->hx_diag, X), o_hu = plan.add_out(out->hu_diag, U),
               o_lb = plan.add_out(out->du_lb, U), o_ub = plan.add_out(out->du_ub, U);
  // device-side approximations of the cycle are copied out like the blocks
  Slice sf{nullptr, f, 0, Kz * nr}, sj{nullptr, jac, 0, Kz * nr * nf}, sh{nullptr, hess, 0, Kz * nr * nf * nf};

  Grow(&c->d_qin, &c->qin_cap, plan.in_total, false);
  Grow(&c->d_qout, &c->qout_cap, std::max<size_t>(plan.out_total, 1), false);
  if (!c->d_bad) {
    CUDA_CHECK(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
    CUDA_CHECK(cudaMallocHost(&c->h_bad, sizeof(unsigned long long)));
  }
  double* din = c->d_qin;
  double* dout = c->d_qout;
  rtn::BlkParams b = MakeBlk(*p, *cfg, n_inst);
  b.xs = din + o_xs;
  b.us = din + o_us;
  b.rxs = din + o_rxs;
  b.rus = din + o_rus;
  b.aux = var == rtn::kVarGround ? din + o_aux : nullptr;
  if (cycle) {
    b.z0 = nullptr;  // z0 = [x_k; u_k], the point PrepareNodes was evaluated at
    b.fbar = c->d_f;
    b.jac = c->d_jac;
    b.hess = order == 2 ? c->d_hess : nullptr;
  } else {
    b.z0 = din + o_z0;
    b.fbar = din + o_fb;
    b.jac = din + o_jac;
    b.hess = order == 2 ? din + o_hess : nullptr;
  }
  auto outp = [dout](size_t off) { return off == SIZE_MAX ? nullptr : dout + off; };
  b.a = outp(o_a);
  b.b = outp(o_b);
  b.phi = outp(o_phi);
  b.q = outp(o_q);
  b.r = outp(o_r);
  b.hx = outp(o_hx);
  b.hu = outp(o_hu);
  b.lb = outp(o_lb);
  b.ub = outp(o_ub);
  b.first_bad = c->d_bad;

  auto enqueue_compute = [&](cudaStream_t s) {
    if (b.first_bad) CUDA_CHECK(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), s));
    if (cycle && var == rtn::kVarFull) {  // PrepareNodes at z_k = [x_k; u_k], gathered inside layer 0
      Enqueue(c, nullptr, K, order, c->d_f, c->d_jac, order == 2 ? c->d_hess : nullptr, b.xs, b.us, N);
    } else if (cycle) {  // other variants: stage z_k = features(x_k, u_k, aux_k) first
      CUDA_CHECK(rtn::LaunchFeatures(var, b.xs, b.us, b.aux, n_inst, N, c->d_z, s));
      c->launches += 1;
      Enqueue(c, c->d_z, K, order, c->d_f, c->d_jac, order == 2 ? c->d_hess : nullptr);
    }
    CUDA_CHECK(rtn::LaunchQpBlocks(b, s, cycle && PdlEnabled()));
    c->launches += 1;
  };
  const unsigned mask = (out->a ? 1u : 0) | (out->b ? 2u : 0) | (out->phi_res ? 4u : 0) | (out->q ? 8u : 0) |
                        (out->r ? 16u : 0) | (out->hx_diag ? 32u : 0) | (out->hu_diag ? 64u : 0) |
                        (out->du_lb ? 128u : 0) | (out->du_ub ? 256u : 0) | (f ? 512u : 0) | (jac ? 1024u : 0) |
                        (hess ? 2048u : 0);
  const bool staged = c->latency_mode || !AllPinned(plan) || (f && !IsPinned(f)) || (jac && !IsPinned(jac)) ||
                      (hess && !IsPinned(hess));
  cudaStream_t s = c->stream;
  if (staged) {
    // Pack everything through contiguous pinned staging: one H2D, one D2H.
    size_t extra = 0;
    if (cycle) extra = (f ? sf.n : 0) + (jac ? sj.n : 0) + (hess ? sh.n : 0);
    Grow(&c->h_qin, &c->hqin_cap, plan.in_total, true);
    Grow(&c->h_qout, &c->hqout_cap, plan.out_total + extra + 1, true);
    for (const Slice& sl : plan.in) std::memcpy(c->h_qin + sl.off, sl.src, sl.n * sizeof(double));
    size_t eo = plan.out_total;
    const size_t o_f = f ? eo : 0;
    eo += f ? sf.n : 0;
    const size_t o_j = jac ? eo : 0;
    eo += jac ? sj.n : 0;
    const size_t o_h = hess ? eo : 0;
    const bool zc = c->latency_mode && K <= kGraphMaxRows && ZeroCopy();
    if (zc) {
      // Zero-copy: the kernels read the iterate from and write QpData to the
      // pinned staging in place (unified addressing); errors come back as
      // per-node status bytes, so the graph holds the two kernels only.
      if (c->status_cap < K) {
        cudaFreeHost(c->h_status);
        c->h_status = nullptr;
        c->status_cap = 0;
        CUDA_CHECK(cudaMallocHost(&c->h_status, static_cast<size_t>(K)));
        c->status_cap = K;
      }
      const double* hin = c->h_qin;
      double* hout = c->h_qout;
      b.xs = hin + o_xs;
      b.us = hin + o_us;
      b.rxs = hin + o_rxs;
      b.rus = hin + o_rus;
      b.aux = var == rtn::kVarGround ? hin + o_aux : nullptr;
      if (!cycle) {
        b.z0 = hin + o_z0;
        b.fbar = hin + o_fb;
        b.jac = hin + o_jac;
        b.hess = order == 2 ? hin + o_hess : nullptr;
      }
      auto houtp = [hout](size_t off) { return off == SIZE_MAX ? nullptr : hout + off; };
      b.a = houtp(o_a);
      b.b = houtp(o_b);
      b.phi = houtp(o_phi);
      b.q = houtp(o_q);
      b.r = houtp(o_r);
      b.hx = houtp(o_hx);
      b.hu = houtp(o_hu);
      b.lb = houtp(o_lb);
      b.ub = houtp(o_ub);
      b.first_bad = nullptr;
      b.status = c->h_status;
    }
    auto body = [&](cudaStream_t st) {
      if (!zc) CUDA_CHECK(cudaMemcpyAsync(din, c->h_qin, plan.in_total * sizeof(double), cudaMemcpyHostToDevice, st));
      enqueue_compute(st);
      if (plan.out_total && !zc)
        CUDA_CHECK(cudaMemcpyAsync(c->h_qout, dout, plan.out_total * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (cycle && f) CUDA_CHECK(cudaMemcpyAsync(c->h_qout + o_f, c->d_f, sf.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (cycle && jac)
        CUDA_CHECK(cudaMemcpyAsync(c->h_qout + o_j, c->d_jac, sj.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (cycle && hess)
        CUDA_CHECK(cudaMemcpyAsync(c->h_qout + o_h, c->d_hess, sh.n * sizeof(double), cudaMemcpyDeviceToHost, st));
      if (!zc) CUDA_CHECK(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    };
    if (c->latency_mode && K <= kGraphMaxRows) {
      const unsigned key = mask | (cycle ? 1u << 31 : 0) | (zc ? 1u << 30 : 0);
      const void* bufs[4] = {c->h_qin, c->h_qout, c->d_qin, c->d_qout};
      const rtn_ctx::QpGraph* g = nullptr;
      for (const auto& e : c->qp_graphs)
        if (e.n_inst == n_inst && e.N == N && e.order == order && e.mask == key &&
            std::memcmp(&e.blk, &b, sizeof b) == 0 && std::memcmp(e.bufs, bufs, sizeof bufs) == 0)
          g = &e;
      if (!g) {
        body(s);  // first run outside capture (kernel attributes, lazy loading)
        CUDA_CHECK(cudaStreamSynchronize(s));
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        const unsigned long long l0 = c->launches;
        CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        body(s);
        CUDA_CHECK(cudaStreamEndCapture(s, &graph));
        const unsigned long long per = c->launches - l0;
        c->launches = l0;  // the capture pass launched nothing
        CUDA_CHECK(cudaGraphInstantiate(&exec, graph, 0));
        CUDA_CHECK(cudaGraphDestroy(graph));
        if (c->qp_graphs.size() >= 64) {  // bounded cache
          cudaGraphExecDestroy(c->qp_graphs.front().exec);
          c->qp_graphs.erase(c->qp_graphs.begin());
        }
        rtn_ctx::QpGraph qg{};
        qg.n_inst = n_inst;
        qg.N = N;
        qg.order = order;
        qg.mask = key;
        std::memcpy(&qg.blk, &b, sizeof b);
        std::memcpy(qg.bufs, bufs, sizeof bufs);
        qg.exec = exec;
        qg.kernels = per;
        c->qp_graphs.push_back(qg);
      } else {
        CUDA_CHECK(cudaGraphLaunch(g->exec, s));
        c->launches += g->kernels;
      }
    } else {
      body(s);
    }
    CUDA_CHECK(cudaStreamSynchronize(s));
    if (zc) {
      for (long long i = 0; i < K; ++i)
        if (c->h_status[i]) throw Error(RTN_ERUNTIME, QpErrorMessage((static_cast<unsigned long long>(i) << 8) |
                                                                         c->h_status[i], N, n_inst));
    } else if (*c->h_bad != rtn::kNoError) {
      throw Error(RTN_ERUNTIME, QpErrorMessage(*c->h_bad, N, n_inst));
    }
    for (const Slice& sl : plan.out) std::memcpy(sl.dst, c->h_qout + sl.off, sl.n * sizeof(double));
    if (cycle && f) std::memcpy(f, c->h_qout + o_f, sf.n * sizeof(double));
    if (cycle && jac) std::memcpy(jac, c->h_qout + o_j, sj.n * sizeof(double));
    if (cycle && hess) std::memcpy(hess, c->h_qout + o_h, sh.n * sizeof(double));
    return;
  }
  // Caller buffers are page-locked: DMA each array directly.
  for (const Slice& sl : plan.in)
    CUDA_CHECK(cudaMemcpyAsync(din + sl.off, sl.src, sl.n * sizeof(double), cudaMemcpyHostToDevice, s));
  enqueue_compute(s);
  CUDA_CHECK(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  for (const Slice& sl : plan.out)
    CUDA_CHECK(cudaMemcpyAsync(sl.dst, dout + sl.off, sl.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (cycle && f) CUDA_CHECK(cudaMemcpyAsync(f, c->d_f, sf.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (cycle && jac) CUDA_CHECK(cudaMemcpyAsync(jac, c->d_jac, sj.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (cycle && hess) CUDA_CHECK(cudaMemcpyAsync(hess, c->d_hess, sh.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  CUDA_CHECK(cudaStreamSynchronize(s));
  if (*c->h_bad != rtn::kNoError) throw Error(RTN_ERUNTIME, QpErrorMessage(*c->h_bad, N, n_inst));
}

}  // namespace

extern "C" {

rtn_status rtn_build_qp(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst,
                        const rtn_iterate* it, const rtn_approx* ap, rtn_qp_blocks* out, unsigned long long* fevals) {
  NvtxRange nvtx("rtn_build_qp");
  return Guard([&] {
    RunQp(c, p, cfg, n_inst, it, ap, out, false, nullptr, nullptr, nullptr);
    if (fevals) {  // FevalCounter: 4 values + 4 Jacobians per node (integrator.cpp:79-82)
      fevals[0] = 4ull * static_cast<unsigned long long>(n_inst * cfg->horizon);
      fevals[1] = fevals[0];
    }
  });
}

rtn_status rtn_build_qp_device(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst,
                               const rtn_iterate* it, const rtn_approx* ap, rtn_qp_blocks* out) {
  NvtxRange nvtx("rtn_build_qp_device");
  return Guard([&] {
    if (!c || !p || !cfg || !it || !ap || !out) throw Error(RTN_ECONFIG, "null argument");
    ValidateQuad(*p);
    ValidateCfg(*cfg);
    if (n_inst < 0) throw Error(RTN_EDOMAIN, "n_inst must be >= 0");
    const long long K = n_inst * cfg->horizon;
    if (K == 0) return;
    CUDA_CHECK(cudaSetDevice(c->model->device));
    if (!c->d_bad) {
      CUDA_CHECK(cudaMalloc(&c->d_bad, sizeof(unsigned long long)));
      CUDA_CHECK(cudaMallocHost(&c->h_bad, sizeof(unsigned long long)));
    }
    rtn::BlkParams b = MakeBlk(*p, *cfg, n_inst);
    b.xs = it->xs;
    b.us = it->us;
    b.rxs = it->ref_xs;
    b.rus = it->ref_us;
    b.z0 = ap->z0;
    b.fbar = ap->f_bar;
    b.jac = ap->jac;
    b.hess = cfg->taylor_order == 2 ? ap->hess : nullptr;
    b.aux = cfg->variant == rtn::kVarGround ? it->aux : nullptr;
    if (!b.xs || !b.us || !b.rxs || !b.rus || !b.fbar || !b.jac || (cfg->taylor_order == 2 && !b.hess) ||
        (cfg->variant == rtn::kVarGround && !b.aux))
      throw Error(RTN_ECONFIG, "null device buffer");
    b.a = out->a;
    b.b = out->b;
    b.phi = out->phi_res;
    b.q = out->q;
    b.r = out->r;
    b.hx = out->hx_diag;
    b.hu = out->hu_diag;
    b.lb = out->du_lb;
    b.ub = out->du_ub;
    b.first_bad = c->d_bad;
    CUDA_CHECK(cudaMemsetAsync(c->d_bad, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_CHECK(rtn::LaunchQpBlocks(b, c->stream));
    c->launches += 1;
    CUDA_CHECK(cudaMemcpyAsync(c->h_bad, c->d_bad, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
    if (*c->h_bad != rtn::kNoError) throw Error(RTN_ERUNTIME, QpErrorMessage(*c->h_bad, cfg->horizon, n_inst));
  });
}

rtn_status rtn_cycle_qp(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst,
                        const rtn_iterate* it, rtn_qp_blocks* out, double* f, double* jac, double* hess) {
  NvtxRange nvtx("rtn_cycle_qp");
  return Guard([&] {
    if (hess && cfg && cfg->taylor_order != 2) throw Error(RTN_ECONFIG, "hess must be NULL unless taylor_order == 2");
    if (c) *c->h_nonfinite = 0;
    RunQp(c, p, cfg, n_inst, it, nullptr, out, true, f, jac, hess);
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Batched feedback solve (resmpc::SolveFeedback, sqp_rti.cpp:157-180).
extern "C" rtn_status rtn_solve_feedback(rtn_ctx* c, const rtn_ocp_config* cfg, long long n_inst,
                                         const rtn_qp_blocks* qp, const double* x_measured, const rtn_iterate* it,
                                         rtn_feedback* out) {
  NvtxRange nvtx("rtn_solve_feedback");
  return Guard([&] {
    if (!cfg) throw Error(RTN_ECONFIG, "null argument");
    if (cfg->horizon < 1) throw Error(RTN_ECONFIG, "qp data: bad dimensions");
    if (cfg->horizon > 64) throw Error(RTN_EUNSUPPORTED, "feedback solve: horizon above 64 (N·nu > 256)");
    if (!c || !qp || !x_measured || !it || !out) throw Error(RTN_ECONFIG, "null argument");
    if (n_inst < 0) throw Error(RTN_EDOMAIN, "n_inst must be >= 0");
    const int N = cfg->horizon, nv = 4 * N;
    if (n_inst == 0) return;
    if (!qp->a || !qp->b || !qp->phi_res || !qp->q || !qp->r || !qp->hx_diag || !qp->hu_diag || !qp->du_lb ||
        !qp->du_ub || !it->xs || !it->us || !out->dxs || !out->dus || !out->u_command || !out->status)
      throw Error(RTN_ECONFIG, "null buffer");
    CUDA_CHECK(cudaSetDevice(c->model->device));
    const size_t K = static_cast<size_t>(n_inst) * N, X = static_cast<size_t>(n_inst) * (N + 1) * 13;
    QpPlan plan;  // doubles in, doubles out; ints/chars travel separately
    const size_t o_a = plan.add_in(qp->a, K * 169), o_b = plan.add_in(qp->b, K * 52),
                 o_phi = plan.add_in(qp->phi_res, K * 13), o_q = plan.add_in(qp->q, X), o_r = plan.add_in(qp->r, K * 4),
                 o_hx = plan.add_in(qp->hx_diag, X), o_hu = plan.add_in(qp->hu_diag, K * 4),
                 o_lb = plan.add_in(qp->du_lb, K * 4), o_ub = plan.add_in(qp->du_ub, K * 4),
                 o_xm = plan.add_in(x_measured, static_cast<size_t>(n_inst) * 13), o_xs = plan.add_in(it->xs, X),
                 o_us = plan.add_in(it->us, K * 4);
    const size_t o_dxs = plan.add_out(out->dxs, X), o_dus = plan.add_out(out->dus, K * 4),
                 o_u = plan.add_out(out->u_command, static_cast<size_t>(n_inst) * 4);
    const int grid = static_cast<int>(std::min<long long>(n_inst, 2LL * c->num_sms));
    const size_t work = static_cast<size_t>(grid) * static_cast<size_t>(rtn::FeedbackWorkPerCta(N));
    Grow(&c->d_fb, &c->fb_cap, plan.in_total + plan.out_total + work, false);
    const size_t small = static_cast<size_t>(n_inst) * (2 * sizeof(int) + nv);
    if (small > c->fb_small_cap) {
      cudaFree(c->d_fb_small);
      c->d_fb_small = nullptr;
      c->fb_small_cap = 0;
      CUDA_CHECK(cudaMalloc(&c->d_fb_small, small));
      c->fb_small_cap = small;
    }
    Grow(&c->h_qin, &c->hqin_cap, plan.in_total, true);
    Grow(&c->h_qout, &c->hqout_cap, plan.out_total + 1, true);
    for (const Slice& sl : plan.in) std::memcpy(c->h_qin + sl.off, sl.src, sl.n * sizeof(double));
    double* din = c->d_fb;
    double* dout = din + plan.in_total;
    int* d_status = reinterpret_cast<int*>(c->d_fb_small);
    int* d_iters = d_status + n_inst;
    signed char* d_act = reinterpret_cast<signed char*>(d_iters + n_inst);
    cudaStream_t s = c->stream;
    CUDA_CHECK(cudaMemcpyAsync(din, c->h_qin, plan.in_total * sizeof(double), cudaMemcpyHostToDevice, s));
    if (out->active)
      CUDA_CHECK(cudaMemcpyAsync(d_act, out->active, static_cast<size_t>(n_inst) * nv, cudaMemcpyHostToDevice, s));
    rtn::FbParams p{};
    p.a = din + o_a;
    p.b = din + o_b;
    p.phi = din + o_phi;
    p.q = din + o_q;
    p.r = din + o_r;
    p.hx = din + o_hx;
    p.hu = din + o_hu;
    p.lb = din + o_lb;
    p.ub = din + o_ub;
    p.x_meas = din + o_xm;
    p.xs = din + o_xs;
    p.us = din + o_us;
    p.active = out->active ? d_act : nullptr;
    p.dxs = dout + o_dxs;
    p.dus = dout + o_dus;
    p.u_cmd = dout + o_u;
    p.status = d_status;
    p.iterations = d_iters;
    p.work = dout + plan.out_total;
    p.n_inst = n_inst;
    p.N = N;
    CUDA_CHECK(rtn::LaunchFeedback(p, grid, s));
    c->launches += 1;
    CUDA_CHECK(cudaMemcpyAsync(c->h_qout, dout, plan.out_total * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaMemcpyAsync(out->status, d_status, static_cast<size_t>(n_inst) * sizeof(int), cudaMemcpyDeviceToHost, s));
    if (out->iterations)
      CUDA_CHECK(cudaMemcpyAsync(out->iterations, d_iters, static_cast<size_t>(n_inst) * sizeof(int),
                                 cudaMemcpyDeviceToHost, s));
    if (out->active)
      CUDA_CHECK(cudaMemcpyAsync(out->active, d_act, static_cast<size_t>(n_inst) * nv, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    for (const Slice& sl : plan.out) std::memcpy(sl.dst, c->h_qout + sl.off, sl.n * sizeof(double));
  });
}
