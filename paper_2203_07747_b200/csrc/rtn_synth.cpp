// rtn_synth.cpp — synthetic workload generators exported by librtn_mpc.so so
// that benches and users can build the BASELINE configurations without the
// test oracle:
//   * rtn_make_mlp: resmpc::MakeMlp semantics (proj/src/neural.cpp:465-489):
//     std::mt19937_64(seed), W ~ U(±1/√fan_in) drawn row-major layer by
//     layer, zero biases, identity normalisation.
//   * rtn_synth_quad_nodes: quadrotor node rows z = [p q v ω u] drawn in the
//     order of RandomQuadState (proj/tests/test_integrator.cpp:24-31) with
//     u ~ U(0.5, 5)^4 (:168), one mt19937_64 stream, instance → node → field.
#include <cmath>
#include <cstdint>
#include <random>

extern "C" {

// W[l] must hold sizes[l+1]*sizes[l] doubles, b[l] sizes[l+1].
int rtn_make_mlp(const int* sizes, int n_sizes, unsigned long long seed, double* const* W, double* const* b) {
  if (!sizes || n_sizes < 2 || !W || !b) return 1;
  std::mt19937_64 rng(seed);
  for (int l = 0; l + 1 < n_sizes; ++l) {
    if (sizes[l] < 1 || sizes[l + 1] < 1) return 1;
    const double bound = 1.0 / std::sqrt(static_cast<double>(sizes[l]));
    std::uniform_real_distribution<double> dist(-bound, bound);
    const long long n = static_cast<long long>(sizes[l + 1]) * sizes[l];
    for (long long i = 0; i < n; ++i) W[l][i] = dist(rng);
    for (int j = 0; j < sizes[l + 1]; ++j) b[l][j] = 0.0;
  }
  return 0;
}

void rtn_synth_quad_nodes(unsigned long long seed, long long k, double* z) {
  std::mt19937_64 rng(seed);
  auto draw = [&](double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(rng); };
  for (long long s = 0; s < k; ++s) {
    double* r = z + s * 17;
    for (int i = 0; i < 3; ++i) r[i] = draw(-2, 2);
    double q[4], n2 = 0.0;
    for (int i = 0; i < 4; ++i) {
      q[i] = draw(-1, 1);
      n2 += q[i] * q[i];
    }
    const double n = std::sqrt(n2);
    for (int i = 0; i < 4; ++i) r[3 + i] = q[i] / n;
    for (int i = 0; i < 3; ++i) r[7 + i] = draw(-4, 4);
    for (int i = 0; i < 3; ++i) r[10 + i] = draw(-3, 3);
    for (int i = 0; i < 4; ++i) r[13 + i] = draw(0.5, 5.0);
  }
}

}  // extern "C"
