// tc_emulate.cpp — CPU emulation of the device path's numerics (forward-mode
// rows through tf32 / 3xTF32 tensor-core MMAs with a model of the tensor
// core's fp32 accumulation), to choose the 3xTF32 accumulation scheme before
// building it. Not part of the product; the oracle supplies the fp64 truth.
//
//   g++ -O2 -std=c++17 -I oracle scripts/tc_emulate.cpp oracle/resmpc_oracle.cpp -o /tmp/tc_emulate
//   /tmp/tc_emulate <depth> <width> <gain> <nodes> <mode> <chains> <corr> <drain> <gbits> <rn> <fp64mean>
//
// Tensor-core accumulation model (one kind::tf32 MMA = 8 exact products added
// to the accumulator): every term (accumulator + 8 products) is aligned to the
// largest exponent and truncated to 24 + gbits bits, summed exactly, then
// rounded to fp32 (rn = 1: to nearest, 0: toward zero).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "resmpc_oracle.h"

extern "C" void oracle_quad_nodes(unsigned long long seed, long long k, double* out);

static float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  u = (u + 0x1000u) & 0xffffe000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

static int G_BITS = 0, G_RN = 0;

// fp32 rounding of an exact double
static double to_f32(double s) {
  if (G_RN) return static_cast<double>(static_cast<float>(s));
  if (s == 0.0) return 0.0;
  int e;
  const double m = std::frexp(s, &e);
  return std::ldexp(std::trunc(std::ldexp(m, 24)), e - 24);
}

// one MMA step: acc + sum_{i<8} a[i]*b[i]
static double mma8(double acc, const float* a, const float* b) {
  double t[9];
  t[0] = acc;
  for (int i = 0; i < 8; ++i) t[i + 1] = static_cast<double>(a[i]) * static_cast<double>(b[i]);
  int emax = -10000;
  for (double v : t)
    if (v != 0.0) {
      int e;
      std::frexp(v, &e);
      emax = std::max(emax, e);
    }
  if (emax == -10000) return 0.0;
  const double q = std::ldexp(1.0, emax - 24 - G_BITS);
  double s = 0.0;
  for (double v : t) s += std::trunc(v / q) * q;
  return to_f32(s);
}

struct Cfg {
  int mode;    // 0 tf32, 1 3xtf32
  int chains;  // main accumulators, interleaved by chunk (32 k)
  int corr;    // 1: corrections in their own accumulator
  int drain;   // >0: every `drain` chunks the partials are added (fp32 RN) into a register sum
  int fp64mean;
};

// y[j] = sum_k W[j][k] x[k] for one row, emulating the chunked MMA stream.
static float dot_tc(const Cfg& c, const float* whi, const float* wlo, const float* xhi, const float* xlo, int K) {
  const int nch = K / 32;
  double acc[8] = {0}, corr = 0;
  float reg = 0.0f;
  int in_group = 0;
  for (int ch = 0; ch < nch; ++ch) {
    const int a = ch % c.chains;
    for (int s = 0; s < 4; ++s) {
      const int k0 = ch * 32 + s * 8;
      acc[a] = mma8(acc[a], whi + k0, xhi + k0);
    }
    if (c.mode == 1) {
      double& d2 = c.corr ? corr : acc[a];
      for (int s = 0; s < 4; ++s) d2 = mma8(d2, whi + ch * 32 + s * 8, xlo + ch * 32 + s * 8);
      for (int s = 0; s < 4; ++s) d2 = mma8(d2, wlo + ch * 32 + s * 8, xhi + ch * 32 + s * 8);
    }
    if (c.drain && ++in_group == c.drain) {
      float part = 0.0f;
      for (int i = 0; i < c.chains; ++i) part += static_cast<float>(acc[i]), acc[i] = 0;
      reg += part;
      in_group = 0;
    }
  }
  float v = reg;
  float rest = 0.0f;
  for (int i = c.chains - 1; i >= 1; --i) rest += static_cast<float>(acc[i]);
  rest += static_cast<float>(corr);
  return v + (static_cast<float>(acc[0]) + rest);
}

int main(int argc, char** argv) {
  if (argc < 12) {
    std::fprintf(stderr, "usage: depth width gain nodes mode chains corr drain gbits rn fp64mean\n");
    return 2;
  }
  const int depth = std::atoi(argv[1]), width = std::atoi(argv[2]);
  const double gain = std::atof(argv[3]);
  const int nodes = std::atoi(argv[4]);
  Cfg c{std::atoi(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]), std::atoi(argv[8]), std::atoi(argv[11])};
  G_BITS = std::atoi(argv[9]);
  G_RN = std::atoi(argv[10]);
  std::vector<int> sizes{17};
  for (int i = 0; i < depth; ++i) sizes.push_back(width);
  sizes.push_back(6);
  std::mt19937_64 rng(11);
  oracle::MlpModel m = oracle::RandomNet(rng, sizes, oracle::Activation::kSilu, true);
  for (int l = 0; l + 2 < static_cast<int>(sizes.size()); ++l)
    for (double& w : m.weights[l].v) w *= gain;
  std::vector<double> z(static_cast<size_t>(nodes) * 17);
  oracle_quad_nodes(2203, nodes, z.data());
  const oracle::BatchEval ref = oracle::MlpBatchedEval(m, z.data(), nodes, oracle::EvalOrder::kJacobian, 1);

  const int L = static_cast<int>(sizes.size()) - 1, W = width, R = 18;
  auto split = [&](double w, float& hi, float& lo) {
    hi = tf32_rna(static_cast<float>(w));
    lo = c.mode == 1 ? tf32_rna(static_cast<float>(w - hi)) : 0.0f;
  };
  // packed operands (normalisation folded as in BuildModel)
  std::vector<std::vector<float>> whi(L), wlo(L);
  for (int l = 1; l < L; ++l) {
    const int rows = sizes[l + 1], cols = sizes[l];
    whi[l].assign(static_cast<size_t>(rows) * cols, 0.f);
    wlo[l].assign(static_cast<size_t>(rows) * cols, 0.f);
    for (int j = 0; j < rows; ++j)
      for (int k = 0; k < cols; ++k) {
        double w = m.weights[l](j, k);
        if (l == L - 1) w *= m.out_scale[j];
        split(w, whi[l][static_cast<size_t>(j) * cols + k], wlo[l][static_cast<size_t>(j) * cols + k]);
      }
  }
  double err[3] = {0, 0, 0};
  for (int n = 0; n < nodes; ++n) {
    // layer 0 on CUDA cores (fp32)
    std::vector<float> act(static_cast<size_t>(R) * W), pre_s(W);
    for (int j = 0; j < W; ++j) {
      double accd = m.biases[0][j];
      float w0[17];
      for (int k = 0; k < 17; ++k) {
        const double w = m.weights[0](j, k) / m.in_scale[k];
        w0[k] = static_cast<float>(w);
        if (!c.fp64mean) accd -= w * m.in_mean[k];
      }
      float pre = static_cast<float>(accd);
      for (int k = 0; k < 17; ++k) {
        const double zk = c.fp64mean ? z[n * 17 + k] - m.in_mean[k] : z[n * 17 + k];
        pre = std::fma(w0[k], static_cast<float>(zk), pre);
      }
      const float s = 1.0f / (1.0f + std::exp(-pre));
      act[j] = pre * s;
      const float sp = s * (1.0f + pre * (1.0f - s));
      for (int k = 0; k < 17; ++k) act[static_cast<size_t>(1 + k) * W + j] = sp * w0[k];
    }
    std::vector<float> out(static_cast<size_t>(R) * 6);
    for (int l = 1; l < L; ++l) {
      const int rows = sizes[l + 1];
      const bool last = l == L - 1;
      std::vector<float> xhi(static_cast<size_t>(R) * W), xlo(static_cast<size_t>(R) * W), d(static_cast<size_t>(R) * rows);
      for (size_t i = 0; i < xhi.size(); ++i) {
        xhi[i] = tf32_rna(act[i]);
        xlo[i] = c.mode == 1 ? tf32_rna(act[i] - xhi[i]) : 0.f;
      }
      for (int r = 0; r < R; ++r)
        for (int j = 0; j < rows; ++j)
          d[static_cast<size_t>(r) * rows + j] = dot_tc(c, &whi[l][static_cast<size_t>(j) * W], &wlo[l][static_cast<size_t>(j) * W],
                                                        &xhi[static_cast<size_t>(r) * W], &xlo[static_cast<size_t>(r) * W], W);
      if (last) {
        for (int r = 0; r < R; ++r)
          for (int o = 0; o < 6; ++o) {
            float v = d[static_cast<size_t>(r) * 6 + o];
            if (r == 0) v += static_cast<float>(m.out_scale[o] * m.biases[l][o] + m.out_mean[o]);
            out[static_cast<size_t>(r) * 6 + o] = v;
          }
      } else {
        for (int j = 0; j < rows; ++j) {
          const float pre = d[j] + static_cast<float>(m.biases[l][j]);
          const float s = 1.0f / (1.0f + std::exp(-pre));
          act[j] = pre * s;
          const float sp = s * (1.0f + pre * (1.0f - s));
          for (int r = 1; r < R; ++r) act[static_cast<size_t>(r) * W + j] = d[static_cast<size_t>(r) * rows + j] * sp;
        }
      }
    }
    // per-node block errors (oracles.hpp:30-32)
    auto blk = [&](int which) {
      double num = 0, den = 0;
      for (int o = 0; o < 6; ++o) {
        if (which == 0) {
          num = std::max(num, std::fabs(out[o] - ref.values[n * 6 + o]));
          den = std::max(den, std::fabs(ref.values[n * 6 + o]));
        } else {
          const int k0 = which == 1 ? 0 : 13, k1 = which == 1 ? 13 : 17;
          for (int k = k0; k < k1; ++k) {
            const double rv = ref.jac[(static_cast<size_t>(n) * 6 + o) * 17 + k];
            num = std::max(num, std::fabs(out[static_cast<size_t>(1 + k) * 6 + o] - rv));
            den = std::max(den, std::fabs(rv));
          }
        }
      }
      return num / (1.0 + den);
    };
    for (int b = 0; b < 3; ++b) err[b] = std::max(err[b], blk(b));
  }
  std::printf("depth %d width %d gain %.2f nodes %d mode %d chains %d corr %d drain %d gbits %d rn %d fp64mean %d: "
              "f %.2e A %.2e B %.2e max %.2e\n",
              depth, width, gain, nodes, c.mode, c.chains, c.corr, c.drain, G_BITS, G_RN, c.fp64mean, err[0], err[1],
              err[2], std::max(err[0], std::max(err[1], err[2])));
  return 0;
}
