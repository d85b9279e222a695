// rtn_internal.h — host-side internals shared by the C-ABI translation units
// (rtn_mpc.cu: models, contexts, PrepareNodes / BuildQp / feedback entry
// points; rtn_comm.cu: the partitioned multi-GPU entry). Not installed.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rtn_mpc.h"
#include "rtn_blocks.h"
#include "rtn_launch.h"

namespace rtn_host {

extern thread_local std::string g_err;  // rtn_last_error()

struct Error : std::runtime_error {
  rtn_status code;
  Error(rtn_status c, const std::string& w) : std::runtime_error(w), code(c) {}
};

#define CUDA_CHECK(x)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess)                                                                         \
      throw ::rtn_host::Error(RTN_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
  } while (0)

// Runs f and maps every exception to a status code + thread-local message:
// no entry point throws or aborts.
template <typename F>
rtn_status Guard(F&& f) {
  try {
    f();
    return RTN_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return RTN_ECONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RTN_ECONFIG;
  }
}

}  // namespace rtn_host

struct rtn_model {
  int device = 0;
  rtn_precision prec = RTN_TF32;
  int n_in = 0, n_out = 0, n_layers = 0, n_hidden = 0, act = 0, wp = 0;
  int pair_wp = 0;            // padded width of the packs (256 or 512)
  float* d_bh_pair = nullptr; // hidden biases with pair_wp stride
  double* d_mu = nullptr;     // in_mean (fp64, subtracted before layer 0)
  float* d_w0 = nullptr;
  float* d_w0t = nullptr;     // input-major copy of W0' (n_in x pair_wp)
  float* d_b0 = nullptr;
  float* d_bl = nullptr;
  // pair (cta_group::2) kernel: plain row-major tf32 weights behind TMA maps
  void* d_wt_hidden = nullptr;  // split x (n_hidden-1)·wp rows x wp cols (fp32 or bf16)
  void* d_wt_last = nullptr;    // split x 16 rows x wp cols
  CUtensorMap tmap_h{}, tmap_l{};
  CUtensorMap tmap_h64{};  // width 512, TF32 / BF16: the same hidden pack in 64-row boxes (split / rowsb kernels)
  // reverse mode (TF32, width 512; rtn_reverse.cuh): the hidden layers transposed
  // (W_l^T, [k][n]) and W0' input-major zero-padded to 32 rows, both tf32-rounded
  void* d_wt_hidden_t = nullptr;
  void* d_w0t_pad = nullptr;
  float* d_wl32 = nullptr;  // W_L' (fp32: the output pack's hi + lo)
  CUtensorMap tmap_ht64{}, tmap_ht{}, tmap_w0p{};
  bool reverse_ok = false;       // TF32 width 512: split-schedule reverse kernels
  bool reverse_pair_ok = false;  // other modes / width 256: pair-kernel reverse variants
  int pair_mode = 0;   // rtn::kTF32 / k3xTF32 / kBF16x3 / kBF16
  // rtn_model_load_rmlp's digest-keyed cache: shared handles are reference counted
  int refs = 1;
  uint64_t digest = 0;     // FNV-1a 64 of the RMLP file bytes
  bool cached = false;     // registered in the in-process cache
  bool from_pack = false;  // packed layout read from RTN_PACK_CACHE
  int lo_rows = 0;     // row offset of the lo tiles in the stacked hidden map
  ~rtn_model() {
    int prev;
    if (cudaGetDevice(&prev) == cudaSuccess) {
      cudaSetDevice(device);
      cudaFree(d_mu);
      cudaFree(d_w0);
      cudaFree(d_w0t);
      cudaFree(d_b0);
      cudaFree(d_bl);
      cudaFree(d_wt_hidden);
      cudaFree(d_wt_last);
      cudaFree(d_bh_pair);
      cudaFree(d_wt_hidden_t);
      cudaFree(d_w0t_pad);
      cudaFree(d_wl32);
      cudaSetDevice(prev);
    }
  }
};

struct rtn_ctx {
  const rtn_model* model = nullptr;
  long long max_rows = 0;
  int max_order = 1;
  int latency_mode = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  double* d_z = nullptr;
  double* d_f = nullptr;
  double* d_jac = nullptr;
  double* d_hess = nullptr;
  double* h_hess = nullptr;
  double* h_z = nullptr;  // pinned staging
  double* h_f = nullptr;
  double* h_jac = nullptr;
  int num_sms = 148;
  unsigned long long calls = 0, points = 0, launches = 0;
  unsigned int* h_nonfinite = nullptr;  // host-mapped NaN/Inf flag the output epilogues raise
  int jac_mode = 0;                     // 0 forward mode, 1 reverse mode (rtn_ctx_set_jacobian_mode)
  float* d_rev_s = nullptr;             // reverse mode: σ' scratch [n_hidden][chunk][512]
  size_t rev_s_cap = 0;                 // floats
  // end-to-end pipeline: copy-in / copy-out streams and per-chunk events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_k;
  // latency mode: one captured graph (H2D, kernel, D2H) per (K, order)
  struct Graph {
    long long K;
    int order;
    cudaGraphExec_t exec;
    const void* io[4];  // caller buffers of a direct (zero-copy) graph; null = staged
  };
  std::vector<Graph> graphs;
  // continuity-block builder: contiguous device in/out areas and pinned
  // staging, grown on demand; the per-call error word; cycle graphs.
  double* d_qin = nullptr;
  double* d_qout = nullptr;
  double* h_qin = nullptr;
  double* h_qout = nullptr;
  size_t qin_cap = 0, qout_cap = 0, hqin_cap = 0, hqout_cap = 0;  // doubles
  unsigned long long* d_bad = nullptr;
  unsigned long long* h_bad = nullptr;
  // feedback solve workspace (grown on demand)
  double* d_fb = nullptr;
  size_t fb_cap = 0;  // doubles
  char* d_fb_small = nullptr;
  size_t fb_small_cap = 0;  // bytes (status, iterations, active)
  unsigned char* h_status = nullptr;  // zero-copy latency mode: per-node status bytes
  long long status_cap = 0;
  // A captured cycle / BuildQp graph bakes in the kernel arguments (every
  // BlkParams field: dt, weights, bounds, quad parameters, variant, buffer
  // pointers) and the staging buffers its copies use; a replay is only valid
  // for the identical set, so all of it is the cache key.
  struct QpGraph {
    long long n_inst;
    int N, order;
    unsigned mask;
    rtn::BlkParams blk;
    const void* bufs[4];  // h_qin, h_qout, d_qin, d_qout at capture
    cudaGraphExec_t exec;
    unsigned long long kernels;  // kernel nodes per replay
  };
  std::vector<QpGraph> qp_graphs;
  ~rtn_ctx() {
    int prev;
    if (cudaGetDevice(&prev) == cudaSuccess) {
      cudaSetDevice(model->device);
      cudaFree(d_z);
      cudaFree(d_f);
      cudaFree(d_jac);
      cudaFree(d_hess);
      cudaFreeHost(h_hess);
      cudaFreeHost(h_z);
      cudaFreeHost(h_f);
      cudaFreeHost(h_jac);
      if (own_stream) cudaStreamDestroy(own_stream);
      if (s_in) cudaStreamDestroy(s_in);
      if (s_out) cudaStreamDestroy(s_out);
      for (auto e : ev_in) cudaEventDestroy(e);
      for (auto e : ev_k) cudaEventDestroy(e);
      for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
      for (auto& g : qp_graphs) cudaGraphExecDestroy(g.exec);
      cudaFree(d_qin);
      cudaFree(d_qout);
      cudaFreeHost(h_qin);
      cudaFreeHost(h_qout);
      cudaFree(d_bad);
      cudaFreeHost(h_bad);
      cudaFree(d_fb);
      cudaFree(d_fb_small);
      cudaFreeHost(h_status);
      cudaFreeHost(h_nonfinite);
      cudaFree(d_rev_s);
      cudaSetDevice(prev);
    }
  }
};

namespace rtn_host {

// NVTX range over one C-ABI call (visible in Nsight Systems / ncu --nvtx).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr int kMaxChunks = 8;  // end-to-end pipeline depth (chunks per call)

// Enqueues one PrepareNodes launch on the context stream (kernel choice,
// tile geometry; rtn_mpc.cu). d_zx/d_zu: gather [x_k; u_k] from an iterate.
void Enqueue(rtn_ctx* c, const double* d_z, long long K, int order, double* d_f, double* d_jac,
             double* d_hess = nullptr, const double* d_zx = nullptr, const double* d_zu = nullptr, int zN = 0);
bool IsPinned(const void* p);
void EnsureStaging(rtn_ctx* c);
void CheckCall(const rtn_ctx* c, long long K, int order);

}  // namespace rtn_host
