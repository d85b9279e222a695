// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Eigen-free fp64 CPU restatement of the reference's per-node MLP
// approximation path (/root/reference/proj/src/neural.cpp:21-327,
// proj/src/taylor.cpp:37-74, proj/include/resmpc/threadpool.hpp), extended
// with a SiLU activation the reference lacks. Only tests/, bench.py's
// cpu_baseline / --impl reference leg and __graft_entry__.smoke() may load it,
// and only as the checker / CPU baseline — never as the product path.
//
// Parity status: pinned by tolerance against the reference's own known-answer
// and finite-difference tests (re-expressed in oracle/test_oracle.cpp). The
// reference itself needs Eigen3 + yaml-cpp (proj/CMakeLists.txt:12-14), which
// are absent, so it cannot be built here; no bitwise pin to reference outputs
// exists. SiLU is pinned only by closed-form and finite-difference checks.
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

// proj/include/resmpc/neural.hpp:10 (kTanh, kRelu) + kSilu (new).
enum class Activation : int { kTanh = 0, kRelu = 1, kSilu = 2 };

// proj/include/resmpc/errors.hpp:9-22
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct InputDomainError : std::invalid_argument {
  explicit InputDomainError(const std::string& w) : std::invalid_argument(w) {}
};
struct UnsupportedError : std::runtime_error {
  explicit UnsupportedError(const std::string& w) : std::runtime_error(w) {}
};

// Row-major dense matrix (the reference's RowMatrixXd, neural.hpp:12).
struct Mat {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> v;
  Mat() = default;
  Mat(std::int64_t r, std::int64_t c) : rows(r), cols(c), v(static_cast<size_t>(r * c), 0.0) {}
  double& operator()(std::int64_t r, std::int64_t c) { return v[static_cast<size_t>(r * cols + c)]; }
  double operator()(std::int64_t r, std::int64_t c) const {
    return v[static_cast<size_t>(r * cols + c)];
  }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
};

// proj/include/resmpc/neural.hpp:19-34
struct MlpModel {
  std::vector<int> layer_sizes;
  std::vector<Mat> weights;                 // weights[l]: sizes[l+1] x sizes[l], row-major
  std::vector<std::vector<double>> biases;  // biases[l]: sizes[l+1]
  Activation activation = Activation::kTanh;
  std::string input_variant = "full";
  std::vector<double> in_mean, in_scale, out_mean, out_scale;
  std::uint64_t seed = 0;

  int input_dim() const { return layer_sizes.front(); }
  int output_dim() const { return layer_sizes.back(); }
  int hidden_layers() const { return static_cast<int>(layer_sizes.size()) - 2; }
  std::int64_t ParameterCount() const;
  std::string ArchName() const;
  void Validate() const;
};

// proj/include/resmpc/neural.hpp:38-44
struct EvalCounters {
  std::uint64_t value_evals = 0, jacobian_evals = 0, hessian_evals = 0;
  std::uint64_t batched_calls = 0, batched_points = 0;
};

enum class EvalOrder { kValue, kJacobian, kHessian };

// Flat result of a batched call (the reference keeps K separate Eigen
// matrices, neural.hpp:59-63; the layout here is the C-ABI one):
//   values[K*out], jac[K*out*in] (o-major, then input), hess[K*out*in*in].
struct BatchEval {
  std::int64_t samples = 0;
  std::vector<double> values, jac, hess;
};

// proj/include/resmpc/threadpool.hpp:16-104 — same contiguous chunking
// (one chunk per participant = workers + caller).
class ThreadPool;

// z_rows: K x in, row-major. threads <= 0 → RESMPC_THREADS / hardware.
BatchEval MlpBatchedEval(const MlpModel& m, const double* z_rows, std::int64_t k, EvalOrder order,
                         int threads = 0, EvalCounters* counters = nullptr);
// Same, with the caller's column count checked against the model input
// (proj/src/neural.cpp:230-232 → InputDomainError).
BatchEval MlpBatchedEval(const MlpModel& m, const double* z_rows, std::int64_t k, int cols,
                         EvalOrder order, int threads = 0, EvalCounters* counters = nullptr);
std::vector<double> MlpForward(const MlpModel& m, const std::vector<double>& z,
                               EvalCounters* counters = nullptr);
std::vector<double> MlpJacobian(const MlpModel& m, const std::vector<double>& z,
                                EvalCounters* counters = nullptr);  // out x in row-major
std::vector<double> MlpHessian(const MlpModel& m, const std::vector<double>& z,
                               EvalCounters* counters = nullptr);   // out x in x in

// Independent forward-mode (tangent-propagation) fp64 implementation; the
// cross-check for the reverse sweep and the algorithm the GPU path uses.
void ForwardModeEval(const MlpModel& m, const double* z, double* f, double* jac, double* hess);

// proj/src/neural.cpp:465-489 and proj/tests/oracles.hpp:166-192
MlpModel MakeMlp(const std::vector<int>& sizes, Activation act, const std::string& variant,
                 std::uint64_t seed);
MlpModel RandomNet(std::mt19937_64& rng, const std::vector<int>& sizes,
                   Activation act = Activation::kTanh, bool random_normalization = true);
std::vector<double> RandomVector(std::mt19937_64& rng, int n, double lo = -1.0, double hi = 1.0);

// proj/src/neural.cpp:685-755 (RMLP v1; v2 = same layout with activation tag
// 2 for SiLU — the v1 reader would silently read tag 2 as ReLU, :729).
void SaveModel(const MlpModel& m, const std::string& path);
MlpModel LoadModel(const std::string& path);
std::vector<int> ParseArch(const std::string& arch);  // proj/src/neural.cpp:757-776

// proj/include/resmpc/taylor.hpp:13-29, proj/src/taylor.cpp:9-55
struct TaylorApprox {
  int node = 0, order = 1;
  std::vector<double> z0, f_bar, jac, hess;  // jac out x in; hess out x in x in (order 2)
};
std::vector<TaylorApprox> PrepareNodes(const MlpModel& m, const double* node_features, std::int64_t k,
                                       int cols, int order, EvalCounters* counters = nullptr);

// proj/src/taylor.cpp:57-74 on the flat layout (one node).
void EvalTaylor(int in, int out, int order, const double* z0, const double* f_bar,
                const double* jac, const double* hess, const double* z, double* y);
void EvalTaylorJacobian(int in, int out, int order, const double* z0, const double* jac,
                        const double* hess, const double* z, double* j);

}  // namespace oracle
