// rtn_comm.cu — the multi-GPU entry of the C-ABI: instances
// are independent, so every rank (one process or thread per GPU, each with
// its own context on its own device) evaluates its contiguous block of node
// rows, and the path's one exchange step is the gather of the (f, A, B)
// blocks to the consumer rank over NCCL (NVLink 5 / NVSwitch on a B200 box).
// The rank's rows are processed in chunks; chunk i's grouped ncclSend (and,
// at the root, the ncclRecvs from every rank) run on the communicator's stream
// while chunk i+1's kernel runs on the context stream.
//
// This replaces the reference's process-global fork/join pool
// (/root/reference/proj/include/resmpc/threadpool.hpp:41-62, used by
// BatchedCore through ThreadPool::Global(), proj/src/neural.cpp:259-268),
// which is the only parallelism the reference has.
//
// Peer-store gather (rtn_comm_bind_root_outputs + rtn_prepare_partitioned_p2p):
// the root's output buffers are mapped into every rank (CUDA IPC, or the raw
// pointer when the ranks are threads of one process), and each rank's kernel
// stores its (f, A, B) rows straight into them over NVLink as its tiles
// finish: the gather IS the kernel's output stores, overlapped tile by tile
// with the math, with no staging copy and no NCCL data transfer. A one-element
// NCCL all-reduce after the kernel is the completion barrier.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the library loads and
// every single-GPU entry works without it; a missing NCCL or any NCCL failure
// returns RTN_ENCCL with NCCL's message.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "rtn_internal.h"

using namespace rtn_host;

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  std::string why;  // empty when loaded
};

const NcclApi& Nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](const char* n) {
      void* p = dlsym(h, n);
      if (!p && a.why.empty()) a.why = std::string("libnccl lacks ") + n;
      return p;
    };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.why.empty()) throw Error(RTN_ENCCL, api.why);
  return api;
}

#define NCCL_CHECK(x)                                                                                  \
  do {                                                                                                 \
    const ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess) throw Error(RTN_ENCCL, std::string(#x) + ": " + Nccl().GetErrorString(r_)); \
  } while (0)

// Row ranges [lo, hi) of `chunks` near-equal pieces (paper_2203_07747_b200/sharding.py chunk_bounds).
std::vector<std::pair<long long, long long>> ChunkBounds(long long rows, int chunks) {
  std::vector<std::pair<long long, long long>> b;
  if (rows <= 0) return b;
  const long long c = std::max<long long>(1, std::min<long long>(chunks, rows));
  const long long per = (rows + c - 1) / c;
  for (long long lo = 0; lo < rows; lo += per) b.push_back({lo, std::min(rows, lo + per)});
  return b;
}

// ---- CUDA IPC export / import of device buffers (any pointer inside an allocation)
constexpr int kIpcBytes = 72;  // cudaIpcMemHandle_t (64) + byte offset of the pointer in its allocation (8)

void* AllocationBase(const void* p, size_t* offset) {
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRange>(f);
  }();
  if (!fn) throw Error(RTN_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
    throw Error(RTN_ECONFIG, "ipc export: not a device allocation");
  *offset = static_cast<size_t>(reinterpret_cast<CUdeviceptr>(p) - base);
  return reinterpret_cast<void*>(base);
}

void IpcExport(const void* p, unsigned char out[kIpcBytes]) {
  size_t off = 0;
  void* base = AllocationBase(p, &off);
  cudaIpcMemHandle_t h;
  CUDA_CHECK(cudaIpcGetMemHandle(&h, base));
  std::memcpy(out, &h, sizeof(h));
  const unsigned long long o = off;
  std::memcpy(out + 64, &o, 8);
}

// imported pointer -> the mapping's base (cudaIpcCloseMemHandle takes the base)
std::mutex g_ipc_mu;
std::map<void*, void*> g_ipc_base;

void* IpcImport(const unsigned char in[kIpcBytes], int device) {
  cudaIpcMemHandle_t h;
  std::memcpy(&h, in, sizeof(h));
  unsigned long long off = 0;
  std::memcpy(&off, in + 64, 8);
  CUDA_CHECK(cudaSetDevice(device));
  void* base = nullptr;
  CUDA_CHECK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  void* p = static_cast<unsigned char*>(base) + off;
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  g_ipc_base[p] = base;
  return p;
}

void IpcRelease(void* p) {
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_ipc_mu);
    auto it = g_ipc_base.find(p);
    if (it == g_ipc_base.end()) throw Error(RTN_ECONFIG, "ipc release: pointer was not imported");
    base = it->second;
    g_ipc_base.erase(it);
  }
  CUDA_CHECK(cudaIpcCloseMemHandle(base));
}

}  // namespace

struct rtn_comm {
  int nranks = 0, rank = 0, device = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  long long* d_counts = nullptr;  // [nranks + 1]: the gathered row counts, then this rank's own
  long long* h_counts = nullptr;  // pinned
  cudaEvent_t ev_done = nullptr;
  std::vector<cudaEvent_t> ev_chunk;
  // root: gathered outputs of the host entry (grown on demand)
  double* d_f_all = nullptr;
  double* d_jac_all = nullptr;
  long long all_cap = 0;  // rows
  // peer-store gather: the root's outputs as addressable from this rank
  int p2p_root = -1;
  long long p2p_rows = 0;
  double* p2p_f = nullptr;
  double* p2p_jac = nullptr;
  bool p2p_imported = false;      // p2p_f / p2p_jac are IPC mappings to release
  unsigned char* d_bind = nullptr;  // handle exchange (device, pinned host)
  unsigned char* h_bind = nullptr;
  float* d_flag = nullptr;          // completion all-reduce
  void Unbind() {
    if (p2p_imported) {
      try {
        if (p2p_f) IpcRelease(p2p_f);
        if (p2p_jac) IpcRelease(p2p_jac);
      } catch (...) {
      }
    }
    p2p_root = -1;
    p2p_rows = 0;
    p2p_f = p2p_jac = nullptr;
    p2p_imported = false;
  }
  ~rtn_comm() {
    int prev;
    if (cudaGetDevice(&prev) == cudaSuccess) {
      cudaSetDevice(device);
      Unbind();
      cudaFree(d_bind);
      cudaFreeHost(h_bind);
      cudaFree(d_flag);
      if (comm) Nccl().CommDestroy(comm);
      if (stream) cudaStreamDestroy(stream);
      cudaFree(d_counts);
      cudaFreeHost(h_counts);
      if (ev_done) cudaEventDestroy(ev_done);
      for (auto e : ev_chunk) cudaEventDestroy(e);
      cudaFree(d_f_all);
      cudaFree(d_jac_all);
      cudaSetDevice(prev);
    }
  }
};

namespace {

// Every rank's row count (8 bytes each over NCCL): the root places the blocks with them.
std::vector<long long> ExchangeCounts(rtn_comm* cm, long long K) {
  const NcclApi& nc = Nccl();
  CUDA_CHECK(cudaMemcpyAsync(cm->d_counts + cm->nranks, &K, sizeof(long long), cudaMemcpyHostToDevice, cm->stream));
  NCCL_CHECK(nc.AllGather(cm->d_counts + cm->nranks, cm->d_counts, 1, ncclInt64, cm->comm, cm->stream));
  CUDA_CHECK(cudaMemcpyAsync(cm->h_counts, cm->d_counts, sizeof(long long) * cm->nranks, cudaMemcpyDeviceToHost,
                             cm->stream));
  CUDA_CHECK(cudaStreamSynchronize(cm->stream));
  return std::vector<long long>(cm->h_counts, cm->h_counts + cm->nranks);
}

// Enqueues the partitioned step on the context and communicator streams.
void PartitionedEnqueue(rtn_ctx* c, rtn_comm* cm, const double* d_z, long long K, int order, double* d_f,
                        double* d_jac, int root, double* d_f_all, double* d_jac_all, int chunks,
                        const std::vector<long long>& counts) {
  const NcclApi& nc = Nccl();
  const rtn_model* m = c->model;
  const int n_in = m->n_in, n_out = m->n_out;
  const long long jrow = static_cast<long long>(n_out) * n_in;
  if (counts[cm->rank] != K) throw Error(RTN_ECONFIG, "row count changed between exchange and launch");
  // the communicator stream starts after all prior work of the context (its
  // buffers may be read by an earlier consumer)
  CUDA_CHECK(cudaEventRecord(cm->ev_done, c->stream));
  CUDA_CHECK(cudaStreamWaitEvent(cm->stream, cm->ev_done, 0));
  std::vector<long long> offs(cm->nranks, 0);
  for (int r = 1; r < cm->nranks; ++r) offs[r] = offs[r - 1] + counts[r - 1];
  std::vector<std::vector<std::pair<long long, long long>>> bounds(cm->nranks);
  size_t max_chunks = 0;
  for (int r = 0; r < cm->nranks; ++r) {
    bounds[r] = ChunkBounds(counts[r], chunks);
    max_chunks = std::max(max_chunks, bounds[r].size());
  }
  const bool is_root = cm->rank == root;
  if (is_root && (!d_f_all || (order >= 1 && !d_jac_all))) throw Error(RTN_ECONFIG, "root needs the gather buffers");
  while (cm->ev_chunk.size() < max_chunks) {
    cudaEvent_t e;
    CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cm->ev_chunk.push_back(e);
  }
  // 2. chunk i: kernel on the context stream, then (communicator stream, after
  //    the kernel) the grouped send to the root and, at the root, the receives
  //    of every rank's chunk i — the transfer overlaps chunk i+1's kernel
  const auto& mine = bounds[cm->rank];
  for (size_t i = 0; i < max_chunks; ++i) {
    if (i < mine.size()) {
      const long long lo = mine[i].first, n = mine[i].second - mine[i].first;
      Enqueue(c, d_z + lo * n_in, n, order, d_f + lo * n_out, order >= 1 ? d_jac + lo * jrow : nullptr);
      CUDA_CHECK(cudaEventRecord(cm->ev_chunk[i], c->stream));
      CUDA_CHECK(cudaStreamWaitEvent(cm->stream, cm->ev_chunk[i], 0));
    }
    NCCL_CHECK(nc.GroupStart());
    if (i < mine.size()) {
      const long long lo = mine[i].first, n = mine[i].second - mine[i].first;
      NCCL_CHECK(nc.Send(d_f + lo * n_out, static_cast<size_t>(n * n_out), ncclFloat64, root, cm->comm, cm->stream));
      if (order >= 1)
        NCCL_CHECK(nc.Send(d_jac + lo * jrow, static_cast<size_t>(n * jrow), ncclFloat64, root, cm->comm, cm->stream));
    }
    if (is_root) {
      for (int r = 0; r < cm->nranks; ++r) {
        if (i >= bounds[r].size()) continue;
        const long long lo = bounds[r][i].first, n = bounds[r][i].second - bounds[r][i].first;
        const long long row = offs[r] + lo;
        NCCL_CHECK(nc.Recv(d_f_all + row * n_out, static_cast<size_t>(n * n_out), ncclFloat64, r, cm->comm, cm->stream));
        if (order >= 1)
          NCCL_CHECK(
              nc.Recv(d_jac_all + row * jrow, static_cast<size_t>(n * jrow), ncclFloat64, r, cm->comm, cm->stream));
      }
    }
    NCCL_CHECK(nc.GroupEnd());
  }
  // 3. the call's work completes on the context stream
  CUDA_CHECK(cudaEventRecord(cm->ev_done, cm->stream));
  CUDA_CHECK(cudaStreamWaitEvent(c->stream, cm->ev_done, 0));
}

void CheckPartitioned(rtn_ctx* c, rtn_comm* cm, long long K, int order, int root) {
  if (!c || !cm) throw Error(RTN_ECONFIG, "null argument");
  if (root < 0 || root >= cm->nranks) throw Error(RTN_ECONFIG, "root outside [0, nranks)");
  if (c->model->device != cm->device) throw Error(RTN_ECONFIG, "context and communicator are on different devices");
  if (order == 2)
    throw Error(RTN_EUNSUPPORTED,
                "partitioned prepare gathers f and J only (order <= 1); Hessians stay on their rank (rtn_prepare)");
  CheckCall(c, K, order);
}

}  // namespace

extern "C" {

rtn_status rtn_comm_unique_id(unsigned char id[128]) {
  return Guard([&] {
    if (!id) throw Error(RTN_ECONFIG, "null argument");
    ncclUniqueId u;
    NCCL_CHECK(Nccl().GetUniqueId(&u));
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

rtn_status rtn_comm_create(const unsigned char id[128], int nranks, int rank, int device, rtn_comm** out) {
  return Guard([&] {
    if (!id || !out) throw Error(RTN_ECONFIG, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error(RTN_ECONFIG, "rank outside [0, nranks)");
    const NcclApi& nc = Nccl();
    CUDA_CHECK(cudaSetDevice(device));
    std::unique_ptr<rtn_comm> cm(new rtn_comm());
    cm->nranks = nranks;
    cm->rank = rank;
    cm->device = device;
    CUDA_CHECK(cudaStreamCreateWithFlags(&cm->stream, cudaStreamNonBlocking));
    CUDA_CHECK(cudaMalloc(&cm->d_counts, sizeof(long long) * (nranks + 1)));
    CUDA_CHECK(cudaMallocHost(&cm->h_counts, sizeof(long long) * nranks));
    CUDA_CHECK(cudaEventCreateWithFlags(&cm->ev_done, cudaEventDisableTiming));
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    NCCL_CHECK(nc.CommInitRank(&cm->comm, nranks, u, rank));
    *out = cm.release();
  });
}

void rtn_comm_free(rtn_comm* cm) {
  try {
    delete cm;
  } catch (...) {
  }
}

rtn_status rtn_prepare_partitioned_device(rtn_ctx* c, rtn_comm* cm, const double* d_z, long long K_local, int order,
                                          double* d_f, double* d_jac, int root, double* d_f_all, double* d_jac_all,
                                          int chunks) {
  NvtxRange nvtx("rtn_prepare_partitioned_device");
  return Guard([&] {
    CheckPartitioned(c, cm, K_local, order, root);
    if (K_local > 0 && (!d_z || !d_f || (order >= 1 && !d_jac))) throw Error(RTN_ECONFIG, "null buffer");
    CUDA_CHECK(cudaSetDevice(cm->device));
    c->calls += 1;
    c->points += static_cast<unsigned long long>(K_local);
    const std::vector<long long> counts = ExchangeCounts(cm, K_local);
    PartitionedEnqueue(c, cm, d_z, K_local, order, d_f, d_jac, root, d_f_all, d_jac_all, std::max(1, chunks), counts);
  });
}

rtn_status rtn_ipc_export(const void* d_ptr, unsigned char out[72]) {
  return Guard([&] {
    if (!d_ptr || !out) throw Error(RTN_ECONFIG, "null argument");
    IpcExport(d_ptr, out);
  });
}

rtn_status rtn_ipc_import(const unsigned char handle[72], int device, void** d_ptr) {
  return Guard([&] {
    if (!handle || !d_ptr) throw Error(RTN_ECONFIG, "null argument");
    *d_ptr = IpcImport(handle, device);
  });
}

rtn_status rtn_ipc_release(void* d_ptr) {
  return Guard([&] {
    if (!d_ptr) throw Error(RTN_ECONFIG, "null argument");
    IpcRelease(d_ptr);
  });
}

// Packet broadcast by the root: [0,72) f handle, [72,144) jac handle, then
// rows_total, the raw f / jac pointers, the root's pid and device.
constexpr int kBindBytes = 192;

rtn_status rtn_comm_bind_root_outputs(rtn_comm* cm, int root, double* d_f_all, double* d_jac_all,
                                      long long rows_total) {
  NvtxRange nvtx("rtn_comm_bind_root_outputs");
  return Guard([&] {
    if (!cm) throw Error(RTN_ECONFIG, "null argument");
    if (root < 0 || root >= cm->nranks) throw Error(RTN_ECONFIG, "root outside [0, nranks)");
    const bool is_root = cm->rank == root;
    if (is_root && (!d_f_all || rows_total < 0)) throw Error(RTN_ECONFIG, "root needs f_all (and rows_total >= 0)");
    const NcclApi& nc = Nccl();
    CUDA_CHECK(cudaSetDevice(cm->device));
    cm->Unbind();
    if (!cm->d_bind) {
      CUDA_CHECK(cudaMalloc(&cm->d_bind, kBindBytes));
      CUDA_CHECK(cudaMallocHost(&cm->h_bind, kBindBytes));
      CUDA_CHECK(cudaMalloc(&cm->d_flag, sizeof(float)));
      CUDA_CHECK(cudaMemset(cm->d_flag, 0, sizeof(float)));
    }
    unsigned char* pk = cm->h_bind;
    std::memset(pk, 0, kBindBytes);
    if (is_root) {
      IpcExport(d_f_all, pk);
      if (d_jac_all) IpcExport(d_jac_all, pk + 72);
      const long long pid = static_cast<long long>(getpid()), dev = cm->device;
      const unsigned long long fp = reinterpret_cast<unsigned long long>(d_f_all),
                               jp = reinterpret_cast<unsigned long long>(d_jac_all);
      std::memcpy(pk + 144, &rows_total, 8);
      std::memcpy(pk + 152, &fp, 8);
      std::memcpy(pk + 160, &jp, 8);
      std::memcpy(pk + 168, &pid, 8);
      std::memcpy(pk + 176, &dev, 8);
    }
    CUDA_CHECK(cudaMemcpyAsync(cm->d_bind, pk, kBindBytes, cudaMemcpyHostToDevice, cm->stream));
    NCCL_CHECK(nc.Broadcast(cm->d_bind, cm->d_bind, kBindBytes, ncclUint8, root, cm->comm, cm->stream));
    CUDA_CHECK(cudaMemcpyAsync(pk, cm->d_bind, kBindBytes, cudaMemcpyDeviceToHost, cm->stream));
    CUDA_CHECK(cudaStreamSynchronize(cm->stream));
    long long rows = 0, pid = 0, rdev = 0;
    unsigned long long fp = 0, jp = 0;
    std::memcpy(&rows, pk + 144, 8);
    std::memcpy(&fp, pk + 152, 8);
    std::memcpy(&jp, pk + 160, 8);
    std::memcpy(&pid, pk + 168, 8);
    std::memcpy(&rdev, pk + 176, 8);
    if (is_root) {
      cm->p2p_f = d_f_all;
      cm->p2p_jac = d_jac_all;
    } else if (pid == static_cast<long long>(getpid())) {  // ranks are threads of one process: UVA pointers
      if (rdev != cm->device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(static_cast<int>(rdev), 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_CHECK(e);
        cudaGetLastError();
      }
      cm->p2p_f = reinterpret_cast<double*>(fp);
      cm->p2p_jac = reinterpret_cast<double*>(jp);
    } else {
      cm->p2p_f = static_cast<double*>(IpcImport(pk, cm->device));
      cm->p2p_imported = true;
      if (jp) cm->p2p_jac = static_cast<double*>(IpcImport(pk + 72, cm->device));
    }
    cm->p2p_rows = rows;
    cm->p2p_root = root;
  });
}

rtn_status rtn_prepare_partitioned_p2p(rtn_ctx* c, rtn_comm* cm, const double* d_z, long long K_local, int order) {
  NvtxRange nvtx("rtn_prepare_partitioned_p2p");
  return Guard([&] {
    if (!cm) throw Error(RTN_ECONFIG, "null argument");
    if (cm->p2p_root < 0) throw Error(RTN_ECONFIG, "bind the root's outputs first (rtn_comm_bind_root_outputs)");
    CheckPartitioned(c, cm, K_local, order, cm->p2p_root);
    if (K_local > 0 && !d_z) throw Error(RTN_ECONFIG, "null buffer");
    if (order >= 1 && !cm->p2p_jac) throw Error(RTN_ECONFIG, "order 1 needs the root's jac_all bound");
    const NcclApi& nc = Nccl();
    CUDA_CHECK(cudaSetDevice(cm->device));
    c->calls += 1;
    c->points += static_cast<unsigned long long>(K_local);
    const std::vector<long long> counts = ExchangeCounts(cm, K_local);
    long long off = 0, total = 0;
    for (int r = 0; r < cm->nranks; ++r) {
      if (r < cm->rank) off += counts[r];
      total += counts[r];
    }
    if (total > cm->p2p_rows) throw Error(RTN_ECONFIG, "rows exceed the bound root outputs");
    const rtn_model* m = c->model;
    const long long jrow = static_cast<long long>(m->n_out) * m->n_in;
    // one launch: every tile's output stores land in the root's buffers
    Enqueue(c, d_z, K_local, order, cm->p2p_f + off * m->n_out, order >= 1 ? cm->p2p_jac + off * jrow : nullptr);
    // completion barrier: each rank's all-reduce follows its kernel, so the
    // root's completes after every rank's stores
    CUDA_CHECK(cudaEventRecord(cm->ev_done, c->stream));
    CUDA_CHECK(cudaStreamWaitEvent(cm->stream, cm->ev_done, 0));
    NCCL_CHECK(nc.AllReduce(cm->d_flag, cm->d_flag, 1, ncclFloat32, ncclSum, cm->comm, cm->stream));
    CUDA_CHECK(cudaEventRecord(cm->ev_done, cm->stream));
    CUDA_CHECK(cudaStreamWaitEvent(c->stream, cm->ev_done, 0));
  });
}

rtn_status rtn_prepare_partitioned(rtn_ctx* c, rtn_comm* cm, const double* z_local, long long K_local, int n_cols,
                                   int order, int root, double* f_all, double* jac_all) {
  NvtxRange nvtx("rtn_prepare_partitioned");
  return Guard([&] {
    CheckPartitioned(c, cm, K_local, order, root);
    const rtn_model* m = c->model;
    if (n_cols != m->n_in)
      throw Error(RTN_EDOMAIN, "mlp eval: feature dim " + std::to_string(n_cols) + " does not match model input " +
                                   std::to_string(m->n_in));
    if (K_local > 0 && !z_local) throw Error(RTN_ECONFIG, "null buffer");
    const bool is_root = cm->rank == root;
    if (is_root && (!f_all || (order >= 1 && !jac_all))) throw Error(RTN_ECONFIG, "root needs f_all (and jac_all)");
    CUDA_CHECK(cudaSetDevice(cm->device));
    c->calls += 1;
    c->points += static_cast<unsigned long long>(K_local);
    const size_t zr = sizeof(double) * m->n_in;
    if (K_local > 0) CUDA_CHECK(cudaMemcpyAsync(c->d_z, z_local, zr * K_local, cudaMemcpyHostToDevice, c->stream));
    // the root's receive buffers hold every rank's rows: sized from the exchanged counts
    const std::vector<long long> counts = ExchangeCounts(cm, K_local);
    long long total = 0;
    for (long long n : counts) total += n;
    if (is_root && total > cm->all_cap) {
      cudaFree(cm->d_f_all);
      cudaFree(cm->d_jac_all);
      cm->d_f_all = cm->d_jac_all = nullptr;
      cm->all_cap = 0;
      CUDA_CHECK(cudaMalloc(&cm->d_f_all, sizeof(double) * total * m->n_out));
      CUDA_CHECK(cudaMalloc(&cm->d_jac_all, sizeof(double) * total * m->n_out * m->n_in));
      cm->all_cap = total;
    }
    PartitionedEnqueue(c, cm, c->d_z, K_local, order, c->d_f, c->d_jac, root, is_root ? cm->d_f_all : nullptr,
                       is_root ? cm->d_jac_all : nullptr, kMaxChunks / 2, counts);
    if (is_root && total > 0) {
      CUDA_CHECK(cudaMemcpyAsync(f_all, cm->d_f_all, sizeof(double) * total * m->n_out, cudaMemcpyDeviceToHost, c->stream));
      if (order >= 1)
        CUDA_CHECK(cudaMemcpyAsync(jac_all, cm->d_jac_all, sizeof(double) * total * m->n_out * m->n_in,
                                   cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_CHECK(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
