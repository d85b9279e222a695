/*
 * rtn_adapter.hpp — header-only C++ layer over the C-ABI (rtn_mpc.h) for the
 * reference-side binding of MlpBatchedEval / PrepareNodes
 * (/root/reference/proj/include/resmpc/neural.hpp:65-69,
 *  /root/reference/proj/include/resmpc/taylor.hpp:27-29). Eigen-free: the
 * binding in INTEGRATION.md only converts Eigen <-> row-major arrays around it,
 * and tests/cpp/test_adapter.cpp drives exactly this logic.
 *
 * Ownership (fixes of the round-1 sketch):
 *   - a DeviceModel is owned by the host model object it was built from (the
 *     binding keeps it in a shared_ptr member of MlpModel), so its identity IS
 *     the model's identity: no cache keyed by object address, nothing stale
 *     after a model is destroyed and another one lands at the same address;
 *   - contexts are per (DeviceModel, thread), so one thread may interleave
 *     calls on different models, each on its own packed weights;
 *   - every context is created with the highest order the model supports (2
 *     unless ReLU or n_in > 31), so a Hessian call after Jacobian calls works;
 *     capacity grows on demand (contexts are recreated for a larger K).
 */
#ifndef RTN_ADAPTER_HPP_
#define RTN_ADAPTER_HPP_

#include <algorithm>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "rtn_mpc.h"

namespace rtn_adapter {

// A C-ABI failure: status code + rtn_last_error(). The binding maps the code to
// the reference's exception classes (errors.hpp:9-22).
struct Status : std::runtime_error {
  rtn_status code;
  Status(rtn_status c, const std::string& what) : std::runtime_error(what), code(c) {}
};

inline void Check(rtn_status s) {
  if (s != RTN_OK) throw Status(s, rtn_last_error());
}

// The MlpModel fields (neural.hpp:19-34) as plain arrays; W[l] row-major sizes[l+1] x sizes[l].
struct ModelDesc {
  std::vector<int> sizes;
  int activation = RTN_ACT_TANH;  // rtn_activation
  std::vector<const double*> W, b;
  const double* in_mean = nullptr;
  const double* in_scale = nullptr;
  const double* out_mean = nullptr;
  const double* out_scale = nullptr;
};

class DeviceModel {
 public:
  DeviceModel(const ModelDesc& d, int device = 0, rtn_precision precision = RTN_TF32, int latency_mode = 1)
      : latency_mode_(latency_mode) {
    Check(rtn_model_from_arrays(d.sizes.data(), static_cast<int>(d.sizes.size()), d.activation, d.W.data(),
                                d.b.data(), d.in_mean, d.in_scale, d.out_mean, d.out_scale, device, precision, &m_));
    int n_in = 0, n_out = 0, layers = 0, act = 0, wp = 0;
    Check(rtn_model_info(m_, &n_in, &n_out, &layers, &act, &wp));
    n_in_ = n_in;
    n_out_ = n_out;
    max_order_ = (act == RTN_ACT_RELU || n_in > 31) ? 1 : 2;
  }
  DeviceModel(const DeviceModel&) = delete;
  DeviceModel& operator=(const DeviceModel&) = delete;
  ~DeviceModel() {
    for (auto& kv : ctx_) rtn_ctx_free(kv.second.c);
    rtn_model_free(m_);
  }

  int n_in() const { return n_in_; }
  int n_out() const { return n_out_; }
  int max_order() const { return max_order_; }

  // MlpBatchedEval body on row-major buffers: z K x n_cols; f K x n_out;
  // jac K x n_out x n_in (order >= 1); hess K x n_out x n_in x n_in (order 2).
  // Order 2 on a ReLU model (or n_in > 31) returns RTN_EUNSUPPORTED, like the
  // reference's HessianSingle (neural.cpp:176-177).
  void Prepare(const double* z, long long K, int n_cols, int order, double* f, double* jac, double* hess) {
    Check(rtn_prepare(Context(K), z, K, n_cols, order, f, order >= 1 ? jac : nullptr, order == 2 ? hess : nullptr));
  }

  // Calls and points this thread's context has seen (EvalCounters::batched_*).
  void Counters(unsigned long long* calls, unsigned long long* points) {
    unsigned long long launches = 0;
    Check(rtn_ctx_counters(Context(1), calls, points, &launches));
  }

 private:
  struct Ctx {
    rtn_ctx* c = nullptr;
    long long cap = 0;
  };
  // This thread's context, with capacity for K rows.
  rtn_ctx* Context(long long K) {
    std::lock_guard<std::mutex> lk(mu_);
    Ctx& e = ctx_[std::this_thread::get_id()];
    if (!e.c || K > e.cap) {
      const long long cap = std::max<long long>({K, 2 * e.cap, 1024});
      rtn_ctx* c = nullptr;
      Check(rtn_ctx_create(m_, cap, max_order_, latency_mode_, &c));
      if (e.c) rtn_ctx_free(e.c);
      e.c = c;
      e.cap = cap;
    }
    return e.c;
  }

  rtn_model* m_ = nullptr;
  int n_in_ = 0, n_out_ = 0, max_order_ = 1, latency_mode_ = 1;
  std::mutex mu_;
  std::unordered_map<std::thread::id, Ctx> ctx_;
};

}  // namespace rtn_adapter

#endif  // RTN_ADAPTER_HPP_
