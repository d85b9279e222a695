// ORACLE — TEST INFRASTRUCTURE ONLY (see resmpc_oracle.h for the contract).
//
// Restates the reference's batched evaluation core with the same loop nests
// and the same std::fma accumulation order, so that within this build a batch
// row is bit-identical to the single-sample call (proj/src/neural.cpp:21-26).
#include "resmpc_oracle.h"

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>

namespace oracle {

// ---------------------------------------------------------------------------
// Fork/join pool: proj/include/resmpc/threadpool.hpp:16-104. One contiguous
// chunk per participant (workers + caller), so disjoint-output bodies are
// independent of the pool size.
class ThreadPool {
 public:
  explicit ThreadPool(int workers) {
    for (int i = 0; i < std::max(0, workers); ++i)
      threads_.emplace_back([this, i] { Loop(i + 1); });
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    wake_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int participants() const { return static_cast<int>(threads_.size()) + 1; }

  void ParallelFor(std::int64_t n, const std::function<void(std::int64_t, std::int64_t)>& body) {
    if (n <= 0) return;
    const int parts = participants();
    if (parts == 1 || n == 1) {
      body(0, n);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &body;
      n_ = n;
      parts_ = parts;
      pending_ = static_cast<int>(threads_.size());
      ++gen_;
    }
    wake_.notify_all();
    Chunk(0, body);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void Chunk(int part, const std::function<void(std::int64_t, std::int64_t)>& body) {
    const std::int64_t chunk = (n_ + parts_ - 1) / parts_;
    const std::int64_t b = part * chunk;
    const std::int64_t e = std::min<std::int64_t>(n_, b + chunk);
    if (b < e) body(b, e);
  }
  void Loop(int part) {
    std::uint64_t seen = 0;
    for (;;) {
      const std::function<void(std::int64_t, std::int64_t)>* job = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        wake_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      if (job != nullptr) Chunk(part, *job);
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable wake_, done_;
  const std::function<void(std::int64_t, std::int64_t)>* job_ = nullptr;
  std::int64_t n_ = 0;
  int parts_ = 1, pending_ = 0;
  std::uint64_t gen_ = 0;
  bool stop_ = false;
};

namespace {

// Pool sizing follows ThreadPool::Global (proj/src/neural.cpp:259-268):
// RESMPC_THREADS, else hardware_concurrency. An explicit thread count wins.
ThreadPool& PoolFor(int threads) {
  static std::mutex mu;
  static std::unique_ptr<ThreadPool> pool;
  static int size = -1;
  int want = threads;
  if (want <= 0) {
    want = std::max(1, static_cast<int>(std::thread::hardware_concurrency()));
    if (const char* env = std::getenv("RESMPC_THREADS")) {
      const int n = std::atoi(env);
      if (n >= 1) want = n;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  if (!pool || size != want) {
    pool.reset();
    pool = std::make_unique<ThreadPool>(want - 1);
    size = want;
  }
  return *pool;
}

// Column-major K x n buffer (the reference's Eigen::MatrixXd activations).
struct ColMat {
  std::int64_t rows = 0, cols = 0;
  std::vector<double> v;
  void resize(std::int64_t r, std::int64_t c) {
    rows = r;
    cols = c;
    v.assign(static_cast<size_t>(r * c), 0.0);
  }
  double& at(std::int64_t r, std::int64_t c) { return v[static_cast<size_t>(c * rows + r)]; }
  double at(std::int64_t r, std::int64_t c) const { return v[static_cast<size_t>(c * rows + r)]; }
};

// OUT(s, j) = b[j] + Σ_k W(j, k) · X(s, k), fma over ascending k, parallel
// over j (proj/src/neural.cpp:29-55).
void DenseForward(const Mat& w, const std::vector<double>& b, const ColMat& x, ColMat& out,
                  ThreadPool* pool) {
  const std::int64_t kc = w.cols, m = w.rows, samples = x.rows;
  out.resize(samples, m);
  const double* xd = x.v.data();
  double* od = out.v.data();
  auto body = [&](std::int64_t j0, std::int64_t j1) {
    for (std::int64_t j = j0; j < j1; ++j) {
      double* oj = od + j * samples;
      const double* wrow = w.data() + j * kc;
      const double bj = b[static_cast<size_t>(j)];
      for (std::int64_t s = 0; s < samples; ++s) oj[s] = bj;
      for (std::int64_t k = 0; k < kc; ++k) {
        const double wk = wrow[k];
        const double* xk = xd + k * samples;
        for (std::int64_t s = 0; s < samples; ++s) oj[s] = std::fma(wk, xk[s], oj[s]);
      }
    }
  };
  if (pool) pool->ParallelFor(m, body);
  else body(0, m);
}

// OUT(r, :) = Σ_i G(r, i) · W(i, :), row-major (proj/src/neural.cpp:58-81).
void DenseReverse(const Mat& g, const Mat& w, Mat& out, ThreadPool* pool) {
  const std::int64_t rows = g.rows, m = w.rows, n = w.cols;
  out = Mat(rows, n);
  auto body = [&](std::int64_t r0, std::int64_t r1) {
    for (std::int64_t r = r0; r < r1; ++r) {
      double* orow = out.data() + r * n;
      const double* grow = g.data() + r * m;
      for (std::int64_t k = 0; k < n; ++k) orow[k] = 0.0;
      for (std::int64_t i = 0; i < m; ++i) {
        const double gi = grow[i];
        const double* wrow = w.data() + i * n;
        for (std::int64_t k = 0; k < n; ++k) orow[k] = std::fma(gi, wrow[k], orow[k]);
      }
    }
  };
  if (pool) pool->ParallelFor(rows, body);
  else body(0, rows);
}

inline double Sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }

// proj/src/neural.cpp:83-85 (+ SiLU: x·σ(x)).
inline double ActValue(Activation a, double x) {
  switch (a) {
    case Activation::kTanh: return std::tanh(x);
    case Activation::kRelu: return x > 0.0 ? x : 0.0;
    default: return x * Sigmoid(x);
  }
}

// proj/src/neural.cpp:87-93 (+ SiLU: σ(1 + x(1−σ))).
inline double ActSlopeFromPre(Activation a, double pre) {
  switch (a) {
    case Activation::kTanh: {
      const double t = std::tanh(pre);
      return 1.0 - t * t;
    }
    case Activation::kRelu: return pre > 0.0 ? 1.0 : 0.0;
    default: {
      const double s = Sigmoid(pre);
      return s * (1.0 + pre * (1.0 - s));
    }
  }
}

// Slope and curvature from the pre-activation; tanh follows the reference's
// σ' = 1 − t², σ'' = −2 t σ' (proj/src/neural.cpp:197-199); SiLU's curvature
// is σ(1−σ)(2 + x(1−2σ)).
inline void ActDerivs(Activation a, double pre, double* val, double* sp, double* spp) {
  if (a == Activation::kTanh) {
    const double t = std::tanh(pre);
    *val = t;
    *sp = 1.0 - t * t;
    *spp = -2.0 * t * *sp;
  } else {
    const double s = Sigmoid(pre);
    *val = pre * s;
    *sp = s * (1.0 + pre * (1.0 - s));
    *spp = s * (1.0 - s) * (2.0 + pre * (1.0 - 2.0 * s));
  }
}

struct ForwardPass {
  std::vector<ColMat> pre, act;
};

// proj/src/neural.cpp:101-121
ForwardPass RunForward(const MlpModel& m, const double* z, std::int64_t samples, ThreadPool* pool) {
  const int layers = static_cast<int>(m.weights.size());
  const int in = m.input_dim();
  ForwardPass fp;
  fp.pre.resize(layers);
  fp.act.resize(layers);
  ColMat x;
  x.resize(samples, in);
  for (int k = 0; k < in; ++k)
    for (std::int64_t s = 0; s < samples; ++s)
      x.at(s, k) = (z[s * in + k] - m.in_mean[k]) / m.in_scale[k];
  for (int l = 0; l < layers; ++l) {
    DenseForward(m.weights[l], m.biases[l], x, fp.pre[l], pool);
    if (l + 1 < layers) {
      fp.act[l] = fp.pre[l];
      for (double& v : fp.act[l].v) v = ActValue(m.activation, v);
      x = fp.act[l];
    } else {
      fp.act[l] = fp.pre[l];  // identity output layer
    }
  }
  return fp;
}

// Stacked reverse sweep, (K·out) x in (proj/src/neural.cpp:132-163).
Mat RunReverse(const MlpModel& m, const ForwardPass& fp, ThreadPool* pool) {
  const int layers = static_cast<int>(m.weights.size());
  const std::int64_t samples = fp.pre[0].rows;
  const int out = m.output_dim();
  const std::int64_t rows = samples * out;
  const Mat& wl = m.weights[layers - 1];
  Mat g(rows, m.layer_sizes[layers - 1]);
  for (std::int64_t s = 0; s < samples; ++s)
    for (int o = 0; o < out; ++o)
      std::memcpy(g.data() + (s * out + o) * g.cols, wl.data() + o * wl.cols,
                  sizeof(double) * static_cast<size_t>(wl.cols));
  Mat next;
  for (int l = layers - 2; l >= 0; --l) {
    const ColMat& pre = fp.pre[l];
    const std::int64_t width = pre.cols;
    auto scale = [&](std::int64_t r0, std::int64_t r1) {
      for (std::int64_t r = r0; r < r1; ++r) {
        const std::int64_t s = r / out;
        double* grow = g.data() + r * width;
        for (std::int64_t i = 0; i < width; ++i) grow[i] *= ActSlopeFromPre(m.activation, pre.at(s, i));
      }
    };
    if (pool) pool->ParallelFor(rows, scale);
    else scale(0, rows);
    DenseReverse(g, m.weights[l], next, pool);
    std::swap(g, next);
  }
  return g;
}

// Per-sample forward-over-forward Hessian (proj/src/neural.cpp:175-225),
// generalised from tanh to SiLU. Plain loops replace Eigen's products, so the
// rounding differs from the reference at the ulp level (tolerance parity).
void HessianSingle(const MlpModel& m, const double* z, double* result /* out x in x in */) {
  if (m.activation == Activation::kRelu)
    throw UnsupportedError("mlp hessian: only tanh/silu networks are twice differentiable here");
  const int in = m.input_dim();
  const int layers = static_cast<int>(m.weights.size());
  std::vector<double> x(in);
  for (int k = 0; k < in; ++k) x[k] = (z[k] - m.in_mean[k]) / m.in_scale[k];
  std::vector<double> jac(static_cast<size_t>(in) * in, 0.0);  // width x in
  for (int k = 0; k < in; ++k) jac[static_cast<size_t>(k) * in + k] = 1.0;
  std::vector<double> hess(static_cast<size_t>(in) * in * in, 0.0);  // width x (in x in)
  const size_t hsz = static_cast<size_t>(in) * in;
  for (int l = 0; l < layers; ++l) {
    const Mat& w = m.weights[l];
    const int width = static_cast<int>(w.rows), cols = static_cast<int>(w.cols);
    std::vector<double> pre(width), jn(static_cast<size_t>(width) * in, 0.0),
        hn(static_cast<size_t>(width) * hsz, 0.0);
    for (int j = 0; j < width; ++j) {
      double acc = m.biases[l][j];
      for (int i = 0; i < cols; ++i) acc += w(j, i) * x[i];
      pre[j] = acc;
      for (int i = 0; i < cols; ++i) {
        const double wji = w(j, i);
        if (wji == 0.0) continue;  // the reference skips zero weights (:193)
        for (int a = 0; a < in; ++a) jn[static_cast<size_t>(j) * in + a] += wji * jac[static_cast<size_t>(i) * in + a];
        double* hj = &hn[static_cast<size_t>(j) * hsz];
        const double* hi = &hess[static_cast<size_t>(i) * hsz];
        for (size_t e = 0; e < hsz; ++e) hj[e] += wji * hi[e];
      }
    }
    x.assign(width, 0.0);
    if (l + 1 < layers) {
      for (int j = 0; j < width; ++j) {
        double v, sp, spp;
        ActDerivs(m.activation, pre[j], &v, &sp, &spp);
        x[j] = v;
        double* hj = &hn[static_cast<size_t>(j) * hsz];
        const double* jr = &jn[static_cast<size_t>(j) * in];
        for (int a = 0; a < in; ++a)
          for (int b = 0; b < in; ++b) hj[a * in + b] = sp * hj[a * in + b] + spp * (jr[a] * jr[b]);
        for (int a = 0; a < in; ++a) jn[static_cast<size_t>(j) * in + a] *= sp;
      }
    } else {
      x = pre;
    }
    jac.swap(jn);
    hess.swap(hn);
  }
  // Denormalise and mirror the upper triangle (proj/src/neural.cpp:210-223).
  for (int o = 0; o < m.output_dim(); ++o) {
    const double* h = &hess[static_cast<size_t>(o) * hsz];
    double* r = result + static_cast<size_t>(o) * hsz;
    for (int a = 0; a < in; ++a)
      for (int b = a; b < in; ++b) {
        const double v = m.out_scale[o] * ((1.0 / m.in_scale[a]) * (1.0 / m.in_scale[b])) * h[a * in + b];
        r[a * in + b] = v;
        r[b * in + a] = v;
      }
  }
}

// proj/src/neural.cpp:227-255
BatchEval BatchedCore(const MlpModel& m, const double* z, std::int64_t samples, EvalOrder order,
                      ThreadPool* pool) {
  m.Validate();
  const int in = m.input_dim(), out = m.output_dim();
  BatchEval r;
  r.samples = samples;
  if (samples == 0) return r;
  const ForwardPass fp = RunForward(m, z, samples, pool);
  r.values.resize(static_cast<size_t>(samples * out));
  for (int o = 0; o < out; ++o)  // DenormalizeOutputs (:123-128)
    for (std::int64_t s = 0; s < samples; ++s)
      r.values[static_cast<size_t>(s * out + o)] = fp.act.back().at(s, o) * m.out_scale[o] + m.out_mean[o];
  if (order == EvalOrder::kValue) return r;

  const Mat g = RunReverse(m, fp, pool);
  r.jac.resize(static_cast<size_t>(samples * out * in));
  for (std::int64_t s = 0; s < samples; ++s)  // ExtractJacobian (:165-173)
    for (int o = 0; o < out; ++o)
      for (int k = 0; k < in; ++k)
        r.jac[static_cast<size_t>((s * out + o) * in + k)] = m.out_scale[o] * g(s * out + o, k) / m.in_scale[k];
  if (order == EvalOrder::kJacobian) return r;

  r.hess.resize(static_cast<size_t>(samples * out * in * in));
  auto body = [&](std::int64_t s0, std::int64_t s1) {
    for (std::int64_t s = s0; s < s1; ++s)
      HessianSingle(m, z + s * in, r.hess.data() + static_cast<size_t>(s * out * in * in));
  };
  if (pool) pool->ParallelFor(samples, body);
  else body(0, samples);
  return r;
}

}  // namespace

// ---------------------------------------------------------------------------
// Model: proj/src/neural.cpp:270-298

std::int64_t MlpModel::ParameterCount() const {
  std::int64_t n = 0;
  for (size_t l = 0; l + 1 < layer_sizes.size(); ++l)
    n += static_cast<std::int64_t>(layer_sizes[l + 1]) * (layer_sizes[l] + 1);
  return n;
}

std::string MlpModel::ArchName() const {
  std::ostringstream os;
  os << "N-" << hidden_layers() << "-" << (hidden_layers() > 0 ? layer_sizes[1] : 0);
  return os.str();
}

void MlpModel::Validate() const {
  if (layer_sizes.size() < 2) throw ConfigError("mlp: need at least input and output layers");
  if (weights.size() != layer_sizes.size() - 1 || biases.size() != weights.size())
    throw ConfigError("mlp: weight/bias count does not match layer sizes");
  for (size_t l = 0; l < weights.size(); ++l) {
    if (weights[l].rows != layer_sizes[l + 1] || weights[l].cols != layer_sizes[l])
      throw ConfigError("mlp: layer " + std::to_string(l) + " has incompatible shape");
    if (static_cast<int>(biases[l].size()) != layer_sizes[l + 1])
      throw ConfigError("mlp: bias " + std::to_string(l) + " has incompatible shape");
  }
  if (static_cast<int>(in_mean.size()) != input_dim() || static_cast<int>(in_scale.size()) != input_dim() ||
      static_cast<int>(out_mean.size()) != output_dim() || static_cast<int>(out_scale.size()) != output_dim())
    throw ConfigError("mlp: normalization vectors do not match layer sizes");
  for (double s : in_scale)
    if (!(s > 0.0)) throw ConfigError("mlp: normalization scales must be strictly positive");
  for (double s : out_scale)
    if (!(s > 0.0)) throw ConfigError("mlp: normalization scales must be strictly positive");
}

// ---------------------------------------------------------------------------
// Entry points: proj/src/neural.cpp:300-327

BatchEval MlpBatchedEval(const MlpModel& m, const double* z_rows, std::int64_t k, EvalOrder order,
                         int threads, EvalCounters* counters) {
  if (counters) {
    ++counters->batched_calls;
    counters->batched_points += static_cast<std::uint64_t>(k);
  }
  return BatchedCore(m, z_rows, k, order, &PoolFor(threads));
}

BatchEval MlpBatchedEval(const MlpModel& m, const double* z_rows, std::int64_t k, int cols,
                         EvalOrder order, int threads, EvalCounters* counters) {
  if (cols != m.input_dim())
    throw InputDomainError("mlp eval: feature dim " + std::to_string(cols) +
                           " does not match model input " + std::to_string(m.input_dim()));
  return MlpBatchedEval(m, z_rows, k, order, threads, counters);
}

std::vector<TaylorApprox> PrepareNodes(const MlpModel& m, const double* z, std::int64_t k, int cols,
                                       int order, EvalCounters* counters) {
  if (order != 1 && order != 2) throw ConfigError("prepare nodes: order must be 1 or 2");
  const BatchEval b = MlpBatchedEval(m, z, k, cols, order == 2 ? EvalOrder::kHessian : EvalOrder::kJacobian,
                                     0, counters);
  const int in = m.input_dim(), out = m.output_dim();
  std::vector<TaylorApprox> r(static_cast<size_t>(k));
  for (std::int64_t s = 0; s < k; ++s) {
    TaylorApprox& a = r[static_cast<size_t>(s)];
    a.node = static_cast<int>(s);
    a.order = order;
    a.z0.assign(z + s * in, z + (s + 1) * in);
    a.f_bar.assign(b.values.begin() + s * out, b.values.begin() + (s + 1) * out);
    a.jac.assign(b.jac.begin() + s * out * in, b.jac.begin() + (s + 1) * out * in);
    if (order == 2)
      a.hess.assign(b.hess.begin() + s * out * in * in, b.hess.begin() + (s + 1) * out * in * in);
  }
  return r;
}

std::vector<double> MlpForward(const MlpModel& m, const std::vector<double>& z, EvalCounters* c) {
  if (c) ++c->value_evals;
  if (static_cast<int>(z.size()) != m.input_dim())
    throw InputDomainError("mlp eval: feature dim does not match model input");
  return BatchedCore(m, z.data(), 1, EvalOrder::kValue, nullptr).values;
}

std::vector<double> MlpJacobian(const MlpModel& m, const std::vector<double>& z, EvalCounters* c) {
  if (c) ++c->jacobian_evals;
  if (static_cast<int>(z.size()) != m.input_dim())
    throw InputDomainError("mlp eval: feature dim does not match model input");
  return BatchedCore(m, z.data(), 1, EvalOrder::kJacobian, nullptr).jac;
}

std::vector<double> MlpHessian(const MlpModel& m, const std::vector<double>& z, EvalCounters* c) {
  if (c) ++c->hessian_evals;
  m.Validate();
  if (static_cast<int>(z.size()) != m.input_dim())
    throw InputDomainError("mlp hessian: feature dim mismatch");
  std::vector<double> h(static_cast<size_t>(m.output_dim()) * m.input_dim() * m.input_dim());
  HessianSingle(m, z.data(), h.data());
  return h;
}

// ---------------------------------------------------------------------------
// Forward-mode (tangent) evaluation. Independent of the reverse sweep: rows
// per node = value, n_in tangents, and (optionally) the packed upper triangle
// of second-order tangents, pushed layer by layer. This is the math the GPU
// kernel performs: per hidden layer
//   v' = σ(W v + b),  t'_a = σ'(pre)·(W t_a),  h'_ab = σ'(pre)·(W h_ab) + σ''(pre)·(W t_a)(W t_b).
void ForwardModeEval(const MlpModel& m, const double* z, double* f, double* jac, double* hess) {
  m.Validate();
  const int in = m.input_dim(), out = m.output_dim();
  const int layers = static_cast<int>(m.weights.size());
  const bool second = hess != nullptr;
  if (second && m.activation == Activation::kRelu)
    throw UnsupportedError("forward-mode hessian: relu is not twice differentiable");
  const int npairs = in * (in + 1) / 2;
  // normalised input and its tangent seed diag(1/in_scale)
  std::vector<double> v(in), t(static_cast<size_t>(in) * in, 0.0), h;
  for (int k = 0; k < in; ++k) {
    v[k] = (z[k] - m.in_mean[k]) / m.in_scale[k];
    t[static_cast<size_t>(k) * in + k] = 1.0 / m.in_scale[k];  // t[a][k]: tangent a, component k
  }
  if (second) h.assign(static_cast<size_t>(npairs) * in, 0.0);
  for (int l = 0; l < layers; ++l) {
    const Mat& w = m.weights[l];
    const int n1 = static_cast<int>(w.rows), n0 = static_cast<int>(w.cols);
    std::vector<double> pv(n1), pt(static_cast<size_t>(in) * n1), ph;
    if (second) ph.assign(static_cast<size_t>(npairs) * n1, 0.0);
    for (int j = 0; j < n1; ++j) {
      double acc = m.biases[l][j];
      for (int i = 0; i < n0; ++i) acc += w(j, i) * v[i];
      pv[j] = acc;
      for (int a = 0; a < in; ++a) {
        double s = 0.0;
        for (int i = 0; i < n0; ++i) s += w(j, i) * t[static_cast<size_t>(a) * n0 + i];
        pt[static_cast<size_t>(a) * n1 + j] = s;
      }
      if (second)
        for (int p = 0; p < npairs; ++p) {
          double s = 0.0;
          for (int i = 0; i < n0; ++i) s += w(j, i) * h[static_cast<size_t>(p) * n0 + i];
          ph[static_cast<size_t>(p) * n1 + j] = s;
        }
    }
    if (l + 1 < layers) {
      for (int j = 0; j < n1; ++j) {
        double val, sp, spp;
        if (m.activation == Activation::kRelu) {
          val = pv[j] > 0.0 ? pv[j] : 0.0;
          sp = pv[j] > 0.0 ? 1.0 : 0.0;
          spp = 0.0;
        } else {
          ActDerivs(m.activation, pv[j], &val, &sp, &spp);
        }
        if (second) {
          int p = 0;
          for (int a = 0; a < in; ++a)
            for (int b = a; b < in; ++b, ++p) {
              double& e = ph[static_cast<size_t>(p) * n1 + j];
              e = sp * e + spp * pt[static_cast<size_t>(a) * n1 + j] * pt[static_cast<size_t>(b) * n1 + j];
            }
        }
        for (int a = 0; a < in; ++a) pt[static_cast<size_t>(a) * n1 + j] *= sp;
        pv[j] = val;
      }
    }
    v.swap(pv);
    t.swap(pt);
    if (second) h.swap(ph);
  }
  for (int o = 0; o < out; ++o) {
    f[o] = m.out_scale[o] * v[o] + m.out_mean[o];
    if (jac)
      for (int a = 0; a < in; ++a) jac[o * in + a] = m.out_scale[o] * t[static_cast<size_t>(a) * out + o];
    if (second) {
      int p = 0;
      for (int a = 0; a < in; ++a)
        for (int b = a; b < in; ++b, ++p) {
          const double e = m.out_scale[o] * h[static_cast<size_t>(p) * out + o];
          hess[(static_cast<size_t>(o) * in + a) * in + b] = e;
          hess[(static_cast<size_t>(o) * in + b) * in + a] = e;
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Init: proj/src/neural.cpp:465-489; test nets: proj/tests/oracles.hpp:166-192

MlpModel MakeMlp(const std::vector<int>& sizes, Activation act, const std::string& variant,
                 std::uint64_t seed) {
  if (sizes.size() < 2) throw ConfigError("mlp: need at least input and output layers");
  MlpModel m;
  m.layer_sizes = sizes;
  m.activation = act;
  m.input_variant = variant;
  m.seed = seed;
  std::mt19937_64 rng(seed);
  for (size_t l = 0; l + 1 < sizes.size(); ++l) {
    const double bound = 1.0 / std::sqrt(static_cast<double>(sizes[l]));
    std::uniform_real_distribution<double> dist(-bound, bound);
    Mat w(sizes[l + 1], sizes[l]);
    for (double& e : w.v) e = dist(rng);  // row-major fill order, as Eigen RowMajor data()
    m.weights.push_back(std::move(w));
    m.biases.emplace_back(static_cast<size_t>(sizes[l + 1]), 0.0);
  }
  m.in_mean.assign(sizes.front(), 0.0);
  m.in_scale.assign(sizes.front(), 1.0);
  m.out_mean.assign(sizes.back(), 0.0);
  m.out_scale.assign(sizes.back(), 1.0);
  m.Validate();
  return m;
}

std::vector<double> RandomVector(std::mt19937_64& rng, int n, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  std::vector<double> v(n);
  for (int i = 0; i < n; ++i) v[i] = d(rng);
  return v;
}

MlpModel RandomNet(std::mt19937_64& rng, const std::vector<int>& sizes, Activation act,
                   bool random_normalization) {
  MlpModel m = MakeMlp(sizes, act, "full", rng());
  if (random_normalization) {
    std::uniform_real_distribution<double> mean_d(-0.5, 0.5), scale_d(0.5, 2.0);
    for (size_t i = 0; i < m.in_mean.size(); ++i) {
      m.in_mean[i] = mean_d(rng);
      m.in_scale[i] = scale_d(rng);
    }
    for (size_t i = 0; i < m.out_mean.size(); ++i) {
      m.out_mean[i] = mean_d(rng);
      m.out_scale[i] = scale_d(rng);
    }
  }
  return m;
}

// ---------------------------------------------------------------------------
// RMLP files: proj/src/neural.cpp:685-755

namespace {
template <typename T>
void Put(std::ofstream& o, const T& v) { o.write(reinterpret_cast<const char*>(&v), sizeof(T)); }
template <typename T>
T Get(std::ifstream& i) {
  T v{};
  i.read(reinterpret_cast<char*>(&v), sizeof(T));
  if (!i) throw ConfigError("unexpected end of file");
  return v;
}
void PutVec(std::ofstream& o, const std::vector<double>& v) {
  o.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
}
void GetVec(std::ifstream& i, std::vector<double>& v) {
  i.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
  if (!i) throw ConfigError("unexpected end of file");
}
const char* ActName(Activation a) {
  return a == Activation::kTanh ? "tanh" : (a == Activation::kRelu ? "relu" : "silu");
}
}  // namespace

void SaveModel(const MlpModel& m, const std::string& path) {
  m.Validate();
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ConfigError("model: cannot write '" + path + "'");
  const bool v2 = m.activation == Activation::kSilu;
  out.write("RMLP", 4);
  Put<std::uint32_t>(out, v2 ? 2u : 1u);
  Put<std::uint8_t>(out, static_cast<std::uint8_t>(m.activation));
  Put<std::uint32_t>(out, static_cast<std::uint32_t>(m.input_variant.size()));
  out.write(m.input_variant.data(), static_cast<std::streamsize>(m.input_variant.size()));
  Put<std::uint64_t>(out, m.seed);
  Put<std::uint32_t>(out, static_cast<std::uint32_t>(m.layer_sizes.size()));
  for (int s : m.layer_sizes) Put<std::uint32_t>(out, static_cast<std::uint32_t>(s));
  PutVec(out, m.in_mean);
  PutVec(out, m.in_scale);
  PutVec(out, m.out_mean);
  PutVec(out, m.out_scale);
  for (size_t l = 0; l < m.weights.size(); ++l) {
    PutVec(out, m.weights[l].v);
    PutVec(out, m.biases[l]);
  }
  if (!out) throw ConfigError("model: write failed for '" + path + "'");
  out.close();
  std::ofstream side(path + ".json");
  side << "{\n  \"format\": \"RMLP\",\n  \"version\": " << (v2 ? 2 : 1) << ",\n  \"activation\": \""
       << ActName(m.activation) << "\",\n  \"input_variant\": \"" << m.input_variant
       << "\",\n  \"layer_sizes\": [";
  for (size_t i = 0; i < m.layer_sizes.size(); ++i) side << (i ? ", " : "") << m.layer_sizes[i];
  side << "],\n  \"arch\": \"" << m.ArchName() << "\",\n  \"parameter_count\": " << m.ParameterCount()
       << ",\n  \"seed\": " << m.seed << "\n}\n";
}

MlpModel LoadModel(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ConfigError("model: cannot open '" + path + "'");
  char magic[4];
  in.read(magic, 4);
  if (!in || std::memcmp(magic, "RMLP", 4) != 0) throw ConfigError("model: '" + path + "' is not a model file");
  const auto version = Get<std::uint32_t>(in);
  if (version != 1 && version != 2) throw ConfigError("model: unsupported version");
  MlpModel m;
  const auto tag = Get<std::uint8_t>(in);
  if (version == 1) m.activation = tag == 0 ? Activation::kTanh : Activation::kRelu;  // :729
  else if (tag <= 2) m.activation = static_cast<Activation>(tag);
  else throw ConfigError("model: unknown activation tag");
  const auto n = Get<std::uint32_t>(in);
  m.input_variant.assign(n, '\0');
  in.read(m.input_variant.data(), n);
  if (!in) throw ConfigError("unexpected end of file");
  m.seed = Get<std::uint64_t>(in);
  const auto ns = Get<std::uint32_t>(in);
  m.layer_sizes.resize(ns);
  for (auto& s : m.layer_sizes) s = static_cast<int>(Get<std::uint32_t>(in));
  if (m.layer_sizes.size() < 2) throw ConfigError("mlp: need at least input and output layers");
  m.in_mean.resize(m.input_dim());
  m.in_scale.resize(m.input_dim());
  m.out_mean.resize(m.output_dim());
  m.out_scale.resize(m.output_dim());
  GetVec(in, m.in_mean);
  GetVec(in, m.in_scale);
  GetVec(in, m.out_mean);
  GetVec(in, m.out_scale);
  for (size_t l = 0; l + 1 < m.layer_sizes.size(); ++l) {
    Mat w(m.layer_sizes[l + 1], m.layer_sizes[l]);
    GetVec(in, w.v);
    std::vector<double> b(static_cast<size_t>(m.layer_sizes[l + 1]));
    GetVec(in, b);
    m.weights.push_back(std::move(w));
    m.biases.push_back(std::move(b));
  }
  m.Validate();
  return m;
}

std::vector<int> ParseArch(const std::string& arch) {
  std::vector<int> sizes;
  const auto x = arch.find('x');
  if (x != std::string::npos && arch.find(',') == std::string::npos) {
    const int depth = std::stoi(arch.substr(0, x));
    const int width = std::stoi(arch.substr(x + 1));
    if (depth < 1 || width < 1) throw ConfigError("arch: bad depth/width in '" + arch + "'");
    sizes.assign(depth, width);
    return sizes;
  }
  std::istringstream is(arch);
  std::string tok;
  while (std::getline(is, tok, ',')) {
    const int w = std::stoi(tok);
    if (w < 1) throw ConfigError("arch: bad width in '" + arch + "'");
    sizes.push_back(w);
  }
  if (sizes.empty()) throw ConfigError("arch: empty spec '" + arch + "'");
  return sizes;
}

// ---------------------------------------------------------------------------
// Taylor consumers: proj/src/taylor.cpp:57-74

void EvalTaylor(int in, int out, int order, const double* z0, const double* f_bar, const double* jac,
                const double* hess, const double* z, double* y) {
  std::vector<double> dz(in);
  for (int k = 0; k < in; ++k) dz[k] = z[k] - z0[k];
  for (int o = 0; o < out; ++o) {
    double acc = 0.0;
    for (int k = 0; k < in; ++k) acc += jac[o * in + k] * dz[k];
    y[o] = f_bar[o] + acc;
    if (order == 2) {
      double q = 0.0;
      for (int a = 0; a < in; ++a) {
        double r = 0.0;
        for (int b = 0; b < in; ++b) r += hess[(static_cast<size_t>(o) * in + a) * in + b] * dz[b];
        q += dz[a] * r;
      }
      y[o] += 0.5 * q;
    }
  }
}

void EvalTaylorJacobian(int in, int out, int order, const double* z0, const double* jac,
                        const double* hess, const double* z, double* j) {
  for (int e = 0; e < out * in; ++e) j[e] = jac[e];
  if (order == 1) return;
  std::vector<double> dz(in);
  for (int k = 0; k < in; ++k) dz[k] = z[k] - z0[k];
  for (int o = 0; o < out; ++o)
    for (int a = 0; a < in; ++a) {
      double r = 0.0;
      for (int b = 0; b < in; ++b) r += hess[(static_cast<size_t>(o) * in + a) * in + b] * dz[b];
      j[o * in + a] += r;
    }
}

}  // namespace oracle

// ---------------------------------------------------------------------------
// C entry points for the test harness (ctypes) and the CPU baseline.
extern "C" {

struct oracle_model;  // opaque: oracle::MlpModel

static thread_local std::string g_oracle_err;

const char* oracle_last_error() { return g_oracle_err.c_str(); }

#define ORACLE_GUARD(...)                                   \
  try {                                                     \
    __VA_ARGS__;                                                \
    return 0;                                               \
  } catch (const oracle::ConfigError& e) {                  \
    g_oracle_err = e.what();                                \
    return 1;                                               \
  } catch (const oracle::InputDomainError& e) {             \
    g_oracle_err = e.what();                                \
    return 2;                                               \
  } catch (const oracle::UnsupportedError& e) {             \
    g_oracle_err = e.what();                                \
    return 3;                                               \
  } catch (const std::exception& e) {                       \
    g_oracle_err = e.what();                                \
    return 9;                                               \
  }

// MakeMlp with seed; act 0 tanh 1 relu 2 silu.
int oracle_make_mlp(const int* sizes, int n, int act, unsigned long long seed, oracle_model** out) {
  ORACLE_GUARD({
    auto* m = new oracle::MlpModel(oracle::MakeMlp(std::vector<int>(sizes, sizes + n),
                                                   static_cast<oracle::Activation>(act), "full", seed));
    *out = reinterpret_cast<oracle_model*>(m);
  })
}

// RandomNet drawn from a fresh mt19937_64(rng_seed) stream (oracles.hpp:176-192).
int oracle_random_net(const int* sizes, int n, int act, unsigned long long rng_seed, int random_norm,
                      oracle_model** out) {
  ORACLE_GUARD({
    std::mt19937_64 rng(rng_seed);
    auto* m = new oracle::MlpModel(oracle::RandomNet(rng, std::vector<int>(sizes, sizes + n),
                                                     static_cast<oracle::Activation>(act), random_norm != 0));
    *out = reinterpret_cast<oracle_model*>(m);
  })
}

int oracle_load_model(const char* path, oracle_model** out) {
  ORACLE_GUARD({ *out = reinterpret_cast<oracle_model*>(new oracle::MlpModel(oracle::LoadModel(path))); })
}

int oracle_save_model(const oracle_model* h, const char* path) {
  ORACLE_GUARD({ oracle::SaveModel(*reinterpret_cast<const oracle::MlpModel*>(h), path); })
}

void oracle_free_model(oracle_model* h) { delete reinterpret_cast<oracle::MlpModel*>(h); }

int oracle_model_info(const oracle_model* h, int* n_sizes, int* sizes, int* act) {
  const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
  if (sizes)
    for (size_t i = 0; i < m->layer_sizes.size(); ++i) sizes[i] = m->layer_sizes[i];
  *n_sizes = static_cast<int>(m->layer_sizes.size());
  *act = static_cast<int>(m->activation);
  return 0;
}

// Copies out layer l's weights (rows x cols row-major) and bias.
int oracle_get_layer(const oracle_model* h, int l, double* w, double* b) {
  const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
  if (l < 0 || l >= static_cast<int>(m->weights.size())) return 1;
  std::memcpy(w, m->weights[l].data(), sizeof(double) * m->weights[l].v.size());
  std::memcpy(b, m->biases[l].data(), sizeof(double) * m->biases[l].size());
  return 0;
}

int oracle_set_layer(oracle_model* h, int l, const double* w, const double* b) {
  auto* m = reinterpret_cast<oracle::MlpModel*>(h);
  if (l < 0 || l >= static_cast<int>(m->weights.size())) return 1;
  std::memcpy(m->weights[l].data(), w, sizeof(double) * m->weights[l].v.size());
  std::memcpy(m->biases[l].data(), b, sizeof(double) * m->biases[l].size());
  return 0;
}

int oracle_get_norm(const oracle_model* h, double* in_mean, double* in_scale, double* out_mean,
                    double* out_scale) {
  const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
  std::memcpy(in_mean, m->in_mean.data(), sizeof(double) * m->in_mean.size());
  std::memcpy(in_scale, m->in_scale.data(), sizeof(double) * m->in_scale.size());
  std::memcpy(out_mean, m->out_mean.data(), sizeof(double) * m->out_mean.size());
  std::memcpy(out_scale, m->out_scale.data(), sizeof(double) * m->out_scale.size());
  return 0;
}

int oracle_set_norm(oracle_model* h, const double* in_mean, const double* in_scale, const double* out_mean,
                    const double* out_scale) {
  auto* m = reinterpret_cast<oracle::MlpModel*>(h);
  std::memcpy(m->in_mean.data(), in_mean, sizeof(double) * m->in_mean.size());
  std::memcpy(m->in_scale.data(), in_scale, sizeof(double) * m->in_scale.size());
  std::memcpy(m->out_mean.data(), out_mean, sizeof(double) * m->out_mean.size());
  std::memcpy(m->out_scale.data(), out_scale, sizeof(double) * m->out_scale.size());
  return 0;
}

// Reverse-mode batched core (the reference algorithm). order 0/1/2. Any of
// f/jac/hess may be NULL when not requested.
int oracle_batched_eval(const oracle_model* h, const double* z, long long k, int order, int threads,
                        double* f, double* jac, double* hess) {
  ORACLE_GUARD({
    const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
    const auto r = oracle::MlpBatchedEval(*m, z, k, static_cast<oracle::EvalOrder>(order), threads, nullptr);
    if (f) std::memcpy(f, r.values.data(), sizeof(double) * r.values.size());
    if (jac && order >= 1) std::memcpy(jac, r.jac.data(), sizeof(double) * r.jac.size());
    if (hess && order >= 2) std::memcpy(hess, r.hess.data(), sizeof(double) * r.hess.size());
  })
}

// Independent forward-mode evaluation, one node at a time.
int oracle_forward_mode(const oracle_model* h, const double* z, long long k, int order, double* f,
                        double* jac, double* hess) {
  ORACLE_GUARD({
    const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
    const int in = m->input_dim(), out = m->output_dim();
    for (long long s = 0; s < k; ++s)
      oracle::ForwardModeEval(*m, z + s * in, f + s * out, order >= 1 ? jac + s * out * in : nullptr,
                              order >= 2 ? hess + s * out * in * in : nullptr);
  })
}

int oracle_single(const oracle_model* h, const double* z, int which, double* out) {
  ORACLE_GUARD({
    const auto* m = reinterpret_cast<const oracle::MlpModel*>(h);
    std::vector<double> zz(z, z + m->input_dim()), r;
    if (which == 0) r = oracle::MlpForward(*m, zz);
    else if (which == 1) r = oracle::MlpJacobian(*m, zz);
    else r = oracle::MlpHessian(*m, zz);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
  })
}

// Node rows for the synthetic quadrotor workload: mt19937_64
// stream, per node p~U(-2,2)^3, q=normalise(U(-1,1)^4), v~U(-4,4)^3,
// ω~U(-3,3)^3, u~U(0.5,5)^4 (proj/tests/test_integrator.cpp:24-31,168).
void oracle_quad_nodes(unsigned long long seed, long long k, double* z) {
  std::mt19937_64 rng(seed);
  for (long long s = 0; s < k; ++s) {
    double* r = z + s * 17;
    auto p = oracle::RandomVector(rng, 3, -2, 2);
    auto q = oracle::RandomVector(rng, 4, -1, 1);
    auto v = oracle::RandomVector(rng, 3, -4, 4);
    auto w = oracle::RandomVector(rng, 3, -3, 3);
    auto u = oracle::RandomVector(rng, 4, 0.5, 5.0);
    double n2 = 0.0;
    for (double e : q) n2 += e * e;
    const double n = std::sqrt(n2);
    for (int i = 0; i < 3; ++i) r[i] = p[i];
    for (int i = 0; i < 4; ++i) r[3 + i] = q[i] / n;
    for (int i = 0; i < 3; ++i) r[7 + i] = v[i];
    for (int i = 0; i < 3; ++i) r[10 + i] = w[i];
    for (int i = 0; i < 4; ++i) r[13 + i] = u[i];
  }
}

void oracle_random_vector(unsigned long long seed, int n, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  auto v = oracle::RandomVector(rng, n, lo, hi);
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

int oracle_eval_taylor(int in, int out, int order, const double* z0, const double* f_bar, const double* jac,
                       const double* hess, const double* z, double* y) {
  oracle::EvalTaylor(in, out, order, z0, f_bar, jac, hess, z, y);
  return 0;
}

int oracle_eval_taylor_jacobian(int in, int out, int order, const double* z0, const double* jac,
                                const double* hess, const double* z, double* j) {
  oracle::EvalTaylorJacobian(in, out, order, z0, jac, hess, z, j);
  return 0;
}

}  // extern "C"
