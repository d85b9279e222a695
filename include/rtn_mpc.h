/*
 * rtn_mpc.h — C-ABI of the B200-native per-node MLP approximation path
 * (Real-time Neural MPC, arXiv 2203.07747).
 *
 * This is the drop-in boundary for the reference's approximation interface:
 *
 *   std::vector<TaylorApprox> resmpc::PrepareNodes(const MlpModel&,
 *       const Eigen::MatrixXd& node_features, int order, EvalCounters*);
 *       -- /root/reference/proj/include/resmpc/taylor.hpp:27-29
 *          /root/reference/proj/src/taylor.cpp:37-55
 *   BatchEval resmpc::MlpBatchedEval(const MlpModel&, const Eigen::MatrixXd& z_rows,
 *       EvalOrder, EvalCounters*);
 *       -- /root/reference/proj/include/resmpc/neural.hpp:65-69
 *          /root/reference/proj/src/neural.cpp:320-327
 *
 * The reference throws C++ exceptions; here each maps to one status code:
 *   ConfigError      (proj/include/resmpc/errors.hpp:9-12)  -> RTN_ECONFIG
 *   InputDomainError (proj/include/resmpc/errors.hpp:15-17) -> RTN_EDOMAIN
 *   UnsupportedError (proj/include/resmpc/errors.hpp:20-22) -> RTN_EUNSUPPORTED
 * No entry point aborts or throws; rtn_last_error() holds a thread-local message.
 *
 * Ownership/threading: a model handle is immutable and may be shared by any
 * number of contexts (the reference's "immutable after loading; evaluation is
 * reentrant", proj/include/resmpc/neural.hpp:17-18). A context owns one CUDA
 * stream, its device workspace and pinned staging; it is single-threaded.
 * Concurrent contexts are safe. The caller owns every host buffer.
 *
 * Layouts (row-major, fp64 on the host side, like the reference):
 *   z    : K x n_in                     (row k = node k)
 *   f    : K x n_out                    (BatchEval::values)
 *   jac  : K x n_out x n_in             (BatchEval::jacobians[k](o, i))
 *   hess : K x n_out x n_in x n_in      (BatchEval::hessians[k][o](a, b))
 */
#ifndef RTN_MPC_H_
#define RTN_MPC_H_

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rtn_model rtn_model; /* opaque, immutable, device-resident packed weights */
typedef struct rtn_ctx rtn_ctx;     /* opaque, one stream + workspace */

typedef enum {
  RTN_OK = 0,
  RTN_ECONFIG = 1,      /* ConfigError: bad shapes, file, order */
  RTN_EDOMAIN = 2,      /* InputDomainError: feature dim mismatch, K out of range */
  RTN_EUNSUPPORTED = 3, /* UnsupportedError: e.g. Hessians of a relu net */
  RTN_ECUDA = 4,        /* CUDA runtime failure (or no sm_100 device) */
  RTN_ENCCL = 5,        /* NCCL unavailable or failed (multi-GPU entry, rtn_comm_*) */
  RTN_ERUNTIME = 6      /* std::runtime_error of BuildQp: "build qp: node k: ..." (sqp_rti.cpp:134-138) */
} rtn_status;

typedef enum {
  RTN_TF32 = 0,   /* one tcgen05 kind::tf32 pass, fp32 accumulate               */
  RTN_3XTF32 = 1, /* tf32 hi/lo split operands, 3 kind::tf32 passes (1e-5 class) */
  RTN_BF16 = 2,   /* one kind::f16 pass on bf16 operands: 2x the tf32 MMA rate, ~8x its error
                     (SURVEY.md §8b's RTN_BF16) */
  RTN_BF16X3 = 3  /* bf16 hi/lo split operands, 3 kind::f16 passes (1e-4 class) */
} rtn_precision;

typedef enum { RTN_ACT_TANH = 0, RTN_ACT_RELU = 1, RTN_ACT_SILU = 2 } rtn_activation;

/* Loads an RMLP v1 (proj/src/neural.cpp:685-755) or v2 (SiLU tag 2) file,
 * folds the normalisation into the first/last layer and packs the weights
 * into the device layout. Replaces resmpc::LoadModel (neural.hpp:117).
 * Digest-keyed (FNV-1a 64 of the file bytes, proj/src/io.cpp:10-26): loading
 * identical bytes again on the same device and precision returns the same
 * shared, reference-counted handle (free each one with rtn_model_free); with
 * RTN_PACK_CACHE=<dir> the packed device layout is also kept on disk as
 * <dir>/<digest>-p<precision>.rtnp and reused by later processes. */
rtn_status rtn_model_load_rmlp(const char* path, int device, rtn_precision p, rtn_model** out);

/* The FNV-1a 64 digest (16 hex digits + NUL) of the RMLP file a model was
 * loaded from ("" for rtn_model_from_arrays), and whether its packed layout
 * came from the RTN_PACK_CACHE file. */
rtn_status rtn_model_digest(const rtn_model* m, char out[17], int* from_pack_cache);

/* Same from in-memory arrays (resmpc::MlpModel fields, neural.hpp:19-34).
 * W[l] is row-major sizes[l+1] x sizes[l]; b[l] has sizes[l+1] entries. */
rtn_status rtn_model_from_arrays(const int* sizes, int n_sizes, int activation,
                                 const double* const* W, const double* const* b,
                                 const double* in_mean, const double* in_scale,
                                 const double* out_mean, const double* out_scale, int device,
                                 rtn_precision p, rtn_model** out);
void rtn_model_free(rtn_model* m);

/* n_in, n_out, number of weight layers, activation, padded hidden width. */
rtn_status rtn_model_info(const rtn_model* m, int* n_in, int* n_out, int* n_layers,
                          int* activation, int* padded_width);

/* max_rows bounds K per call (device workspace is sized for it); max_order in
 * {0,1,2}. latency_mode != 0 captures the launch in a CUDA graph per K. */
rtn_status rtn_ctx_create(const rtn_model* m, long long max_rows, int max_order, int latency_mode,
                          rtn_ctx** out);
void rtn_ctx_free(rtn_ctx* c);

/* The PrepareNodes / MlpBatchedEval equivalent: host z in, host f/jac(/hess)
 * out, blocking. order 0 = value, 1 = + Jacobian, 2 = + Hessian. jac may be
 * NULL for order 0; hess must be NULL unless order == 2. Each call counts as
 * one batched call of K points (proj/src/neural.cpp:322-326). */
rtn_status rtn_prepare(rtn_ctx* c, const double* z, long long K, int n_cols, int order, double* f,
                       double* jac, double* hess);

/* Device-resident variant: all pointers are device pointers on the context's
 * device; enqueued on the context stream, returns without synchronising. */
rtn_status rtn_prepare_device(rtn_ctx* c, const double* d_z, long long K, int order, double* d_f,
                              double* d_jac, double* d_hess);

/* Run the context's work on a caller-provided cudaStream_t (NULL = own). */
rtn_status rtn_ctx_set_stream(rtn_ctx* c, void* cuda_stream);
rtn_status rtn_ctx_synchronize(rtn_ctx* c);

/* NaN/Inf flag (failure detection): 1 if an output value written by
 * the context's kernels since the last reset is not finite. Every blocking
 * call (rtn_prepare, rtn_cycle_qp) resets it first, so after one it describes
 * that call; after device-pointer calls it accumulates until reset. The
 * reference's controller policy on a bad cycle (reuse the last command,
 * sqp_rti.cpp:233-267) stays with the caller. Synchronises the context stream. */
rtn_status rtn_ctx_nonfinite(rtn_ctx* c, int* flag, int reset);
/* Jacobian algorithm for order-1 calls: 0 = forward mode (default; one pass,
 * 1 + n_in rows per node), 1 = reverse mode (the reference's own adjoint sweep,
 * neural.cpp:132-163: a value pass that keeps every layer's slope in an HBM
 * scratch, then 1 adjoint row per output: 1 + n_out rows per node). Reverse
 * mode needs n_in <= 24 and either a TF32 model of padded width 512, or a
 * 3xTF32 / bf16x3 model of padded width 256 or 512 with n_out = 6
 * (RTN_EUNSUPPORTED otherwise); order 0 and 2 calls are unaffected. */
rtn_status rtn_ctx_set_jacobian_mode(rtn_ctx* c, int mode);

/* Counters (EvalCounters::batched_calls / batched_points, neural.hpp:38-44)
 * and the number of device kernel launches this context has issued. */
rtn_status rtn_ctx_counters(const rtn_ctx* c, unsigned long long* batched_calls,
                            unsigned long long* batched_points, unsigned long long* kernel_launches);

const char* rtn_last_error(void);

/* ---------------------------------------------------------------------------
 * Multi-GPU entry: MPC instances are independent, so each rank
 * (one process or thread per GPU, with its own model + context on its device)
 * evaluates its contiguous block of node rows, and the one exchange step is the
 * gather of the (f, A, B) blocks to the consumer rank over NCCL (NVLink /
 * NVSwitch). Replaces the reference's process-global fork/join pool
 * (/root/reference/proj/include/resmpc/threadpool.hpp:41-62) as the path's
 * parallel backend. NCCL is loaded at run time; failures -> RTN_ENCCL.
 * ------------------------------------------------------------------------- */
typedef struct rtn_comm rtn_comm; /* opaque: one NCCL communicator + stream per rank */

/* 128-byte NCCL unique id, created on one rank and sent to the others by the caller. */
rtn_status rtn_comm_unique_id(unsigned char id[128]);
/* Collective over the nranks ranks: every rank calls it with the same id. */
rtn_status rtn_comm_create(const unsigned char id[128], int nranks, int rank, int device, rtn_comm** out);
void rtn_comm_free(rtn_comm* comm);

/* Instance-partitioned PrepareNodes (order 0 or 1; Hessians stay on their rank):
 * every rank passes its own K_local node rows (host, row-major K_local x n_in);
 * the root receives all ranks' rows concatenated in rank order into f_all
 * (sum K x n_out) and jac_all (sum K x n_out x n_in) — host buffers, NULL on the
 * other ranks. Collective and blocking; counts one batched call of K_local points. */
rtn_status rtn_prepare_partitioned(rtn_ctx* c, rtn_comm* comm, const double* z_local, long long K_local, int n_cols,
                                   int order, int root, double* f_all, double* jac_all);
/* Device-pointer variant, enqueued on the context stream: the rank's rows are
 * evaluated in `chunks` pieces and piece i's NCCL transfer to the root overlaps
 * piece i+1's kernel. d_f_all / d_jac_all: the root's device receive buffers. */
rtn_status rtn_prepare_partitioned_device(rtn_ctx* c, rtn_comm* comm, const double* d_z, long long K_local, int order,
                                          double* d_f, double* d_jac, int root, double* d_f_all, double* d_jac_all,
                                          int chunks);

/* Peer-store gather. The root's device output buffers (f_all: rows_total x n_out,
 * jac_all: rows_total x n_out x n_in, NULL for order 0) are bound to the
 * communicator once (collective; other ranks pass NULL): they are mapped into
 * every rank by CUDA IPC (or used directly when the ranks are threads of one
 * process). rtn_prepare_partitioned_p2p then runs one kernel per rank whose
 * output stores go straight into the root's rows for that rank over NVLink --
 * the gather is the kernel's own stores, overlapped tile by tile with the math --
 * followed by a one-element all-reduce as the completion barrier. Enqueued on
 * the context stream; on the root, the buffers are complete once it is done. */
rtn_status rtn_comm_bind_root_outputs(rtn_comm* comm, int root, double* d_f_all, double* d_jac_all,
                                      long long rows_total);
rtn_status rtn_prepare_partitioned_p2p(rtn_ctx* c, rtn_comm* comm, const double* d_z, long long K_local, int order);

/* CUDA IPC of a device buffer between processes (any pointer inside an
 * allocation): 72 bytes = the allocation's cudaIpcMemHandle_t + the pointer's
 * byte offset in it. rtn_ipc_import maps it on `device` (peer access enabled
 * lazily); rtn_ipc_release unmaps a pointer rtn_ipc_import returned. */
rtn_status rtn_ipc_export(const void* d_ptr, unsigned char out[72]);
rtn_status rtn_ipc_import(const unsigned char handle[72], int device, void** d_ptr);
rtn_status rtn_ipc_release(void* d_ptr);

/* ---------------------------------------------------------------------------
 * Continuity-block builder (the step after PrepareNodes).
 * Replaces the node loop of
 *   QpData resmpc::BuildQp(const Plant&, const OcpConfig&, const Iterate&,
 *       const ReferenceWindow&, const std::vector<TaylorApprox>* approxes, ...)
 *       -- /root/reference/proj/include/resmpc/sqp_rti.hpp:56-59
 *          /root/reference/proj/src/sqp_rti.cpp:59-155
 * for the quadrotor plant (MakeQuadrotorPlant, proj/src/plant.cpp:34-85) with
 * any residual variant (rtn_variant; the features and their Jacobian are
 * re-evaluated at every RK4 stage), in rtn mode, batched over
 * n_inst independent MPC instances of horizon N. All arithmetic is fp64.
 * Per node: RK4 sensitivities of f_F + embed·EvalTaylor (integrator.cpp:41-89).
 * Errors: ConfigError -> RTN_ECONFIG (same messages as QuadParams::Validate,
 * OcpConfig::Validate); a quaternion-domain or non-finite stage derivative at
 * any node -> RTN_ERUNTIME with the reference's message for the lowest failing
 * node ("build qp: node k: ..."; "instance i: " prefixed when n_inst > 1).
 * ------------------------------------------------------------------------- */
typedef struct { /* resmpc::QuadParams, proj/include/resmpc/dynamics.hpp:50-62 */
  double mass;
  double inertia[3];
  double arm_length;
  double torque_coeff;
  double thrust_max;
  double rotor_sign[4];
} rtn_quad_params;

/* Residual variant of the quadrotor plant (ResidualVariant, dynamics.hpp:95-131;
 * MakeQuadrotorPlant, plant.cpp:34-85): the network's features z and outputs.
 *   FULL   z = [x; u]                    17 -> 6 (v̇, ω̇ rows)
 *   A      z = v_B = R(q)ᵀ v_W            3 -> 3 (v̇ rows)
 *   AU     z = [v_B; u]                   7 -> 3
 *   GROUND z = [x; u; z_WB·1 − patch]    26 -> 3 (patch: per-node 3x3 height map aux) */
typedef enum { RTN_VARIANT_FULL = 0, RTN_VARIANT_A = 1, RTN_VARIANT_AU = 2, RTN_VARIANT_GROUND = 3 } rtn_variant;

typedef struct { /* resmpc::OcpConfig at quadrotor dims, sqp_rti.hpp:22-34 */
  int horizon; /* N */
  double dt;
  double q_diag[13];
  double r_diag[4];
  int has_q_terminal; /* 0: TerminalWeight() = q_diag */
  double q_terminal[13];
  double u_min[4];
  double u_max[4];
  int taylor_order; /* 1 or 2 */
  int variant;      /* rtn_variant (0 = FULL) */
} rtn_ocp_config;

typedef struct { /* Iterate + ReferenceWindow, row-major, instance-major */
  const double* xs;     /* n_inst x (N+1) x 13 */
  const double* us;     /* n_inst x N x 4 */
  const double* ref_xs; /* n_inst x (N+1) x 13 */
  const double* ref_us; /* n_inst x N x 4 */
  const double* aux;    /* n_inst x N x 9 height patches (Plant::NodeAux, row-major), GROUND only */
} rtn_iterate;

typedef struct { /* one TaylorApprox per node, K = n_inst*N rows (taylor.hpp:13-24); n_f/n_r per variant */
  const double* z0;    /* K x n_f */
  const double* f_bar; /* K x n_r */
  const double* jac;   /* K x n_r x n_f */
  const double* hess;  /* K x n_r x n_f x n_f, taylor_order 2 only (else NULL) */
} rtn_approx;

typedef struct { /* QpData (proj/include/resmpc/qp.hpp:13-28); any pointer may be NULL = not wanted */
  double* a;       /* K x 13 x 13 */
  double* b;       /* K x 13 x 4 */
  double* phi_res; /* K x 13 */
  double* q;       /* n_inst x (N+1) x 13 */
  double* r;       /* K x 4 */
  double* hx_diag; /* n_inst x (N+1) x 13 */
  double* hu_diag; /* K x 4 */
  double* du_lb;   /* K x 4 */
  double* du_ub;   /* K x 4 */
} rtn_qp_blocks;

/* BuildQp from prepared approximations (host buffers, blocking). fevals, if
 * non-NULL, receives FevalCounter {values, jacobians} (+= 4 each per node). */
rtn_status rtn_build_qp(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst,
                        const rtn_iterate* it, const rtn_approx* ap, rtn_qp_blocks* out,
                        unsigned long long* fevals);

/* Same with device pointers; enqueued on the context stream, then waits for
 * the error word only (one 8-byte read) so errors surface like the reference. */
rtn_status rtn_build_qp_device(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg,
                               long long n_inst, const rtn_iterate* d_it, const rtn_approx* d_ap,
                               rtn_qp_blocks* d_out);

/* Phases 1+2 of RtiController::Cycle fused on the device (sqp_rti.cpp:219-231):
 * features z_k = features(x_k, u_k, aux_k) (the MLP's layer 0 gathers them from
 * the iterate) -> PrepareNodes(order = cfg->taylor_order) -> BuildQp. The
 * context's model must be n_f -> n_r of cfg->variant. The approximations are returned too
 * if f/jac/hess are non-NULL. Counts one batched call of K points. */
rtn_status rtn_cycle_qp(rtn_ctx* c, const rtn_quad_params* p, const rtn_ocp_config* cfg, long long n_inst,
                        const rtn_iterate* it, rtn_qp_blocks* out, double* f, double* jac, double* hess);

/* ---------------------------------------------------------------------------
 * Batched feedback solve: resmpc::SolveFeedback
 * (/root/reference/proj/src/sqp_rti.cpp:157-180) per MPC instance — condensing
 * (proj/src/qp.cpp:33-73), the primal active-set box QP with the reference's
 * pivot rules and regularisation (qp.cpp:77-208), and the state recovery
 * dx_k = M_k·du + c_k. Quadrotor dims (nx 13, nu 4), N <= 64. Per-instance
 * status instead of exceptions (RtiController::Cycle turns a throw into
 * ok = false, sqp_rti.cpp:247-252):
 *   0 optimal, 1 iteration cap (QpStatus::kMaxIter), 2 SolveFeedback threw
 *   (non-finite measured state or solution, crossed bounds), 3 Hessian not
 *   positive definite after regularisation.
 * ------------------------------------------------------------------------- */
typedef struct {
  double* dxs;         /* n_inst x (N+1) x 13  FeedbackResult::dxs */
  double* dus;         /* n_inst x N x 4       FeedbackResult::dus */
  double* u_command;   /* n_inst x 4           iterate head input + its step */
  int* status;         /* n_inst */
  int* iterations;     /* n_inst, may be NULL */
  signed char* active; /* n_inst x 4N working set: warm-start hint in, final set out; may be NULL */
} rtn_feedback;

/* qp: QpData as rtn_build_qp returns it; it->xs / it->us: the iterate (dx0 =
 * x_measured − xs[0]); x_measured: n_inst x 13. Host buffers, blocking. */
rtn_status rtn_solve_feedback(rtn_ctx* c, const rtn_ocp_config* cfg, long long n_inst, const rtn_qp_blocks* qp,
                              const double* x_measured, const rtn_iterate* it, rtn_feedback* out);

#ifdef __cplusplus
}
#endif

#endif /* RTN_MPC_H_ */
