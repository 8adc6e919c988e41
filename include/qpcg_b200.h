/*
 * qpcg_b200.h — C-ABI of the B200-native ADMM/PCG QP engine.
 *
 * This is the drop-in boundary for the reference's solve path
 * (reference: /root/reference/proj/include/qpcg/solver.hpp:386-541,
 * `qpcg::solve(const QpProblem<T>&, const Settings<T>&, const WarmStart<T>*,
 * SolveDiagnostics<T>*)`).  The reference exposes only a C++ template API
 * (SURVEY.md F4); the OSQP-style split named by the north star
 * (setup / warm_start / update_rho / update_vectors / solve / cleanup) is
 * mapped onto the reference's phases as follows:
 *
 *   qpcg_fXX_setup          solver.hpp:390-433  validate, symmetrize_upper,
 *                           transpose_csr, Ruiz (scaling.hpp:92-187) or
 *                           identity scaling, ReducedKktOperator + Jacobi
 *                           (linsys.hpp:39-61, :137-148), zero state.
 *   qpcg_fXX_warm_start     solver.hpp:413-428 (x_s = D^-1 x, z_s = E z,
 *                           y_s = c E^-1 y, pcg_warm = x_s).
 *   qpcg_fXX_update_rho     linsys.hpp:153-157 (+ st.rho_bar, solver.hpp:511).
 *   qpcg_fXX_update_vectors NOT in the reference; rescales
 *                           q, l, u with the existing D, E, c.
 *   qpcg_fXX_solve          solver.hpp:434-540 (loop + unscale + objective).
 *   qpcg_fXX_solve_problem  the whole of solver.hpp:386-541 in one call
 *                           (setup + solve + cleanup; runtime_seconds spans
 *                           setup through objective exactly as :392/:537).
 *   qpcg_fXX_cleanup        (destructor)
 *
 * Error codes map 1:1 onto the reference's exception classes:
 *   QPCG_ERR_INVALID  <- std::invalid_argument (problem.hpp:47-92,
 *                        settings.hpp:45-75, sparse.hpp:75-152, linsys.hpp:47-58,
 *                        solver.hpp:414-421)
 *   QPCG_ERR_NOT_PD   <- qpcg::NotPositiveDefiniteError (types.hpp:35-39,
 *                        raised by pcg_solve linsys.hpp:246-250)
 * Non-convergence and infeasibility are statuses, not errors (solver.hpp:57-62).
 *
 * All matrices are CSR with uint32 row_ptr / col_indices (types.hpp:26,
 * sparse.hpp:47-56); P is passed upper-triangular (problem.hpp:56-62).
 * fp32 and fp64 are separate symbol sets (the reference's `T`).
 * Every workspace owns its device, stream and buffers: calls on distinct
 * workspaces are re-entrant (runner.hpp:115-131 calls solve concurrently).
 */
#ifndef QPCG_B200_H
#define QPCG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
#define QPCG_OK 0
#define QPCG_ERR_INVALID 1 /* std::invalid_argument */
#define QPCG_ERR_NOT_PD 2  /* qpcg::NotPositiveDefiniteError */
#define QPCG_ERR_CUDA 3
#define QPCG_ERR_NCCL 4
#define QPCG_ERR_OOM 5
#define QPCG_ERR_RUNTIME 6 /* any other std::runtime_error */

/* ---- SolveStatus, same order as solver.hpp:57-62 ----------------------- */
#define QPCG_STATUS_SOLVED 0
#define QPCG_STATUS_PRIMAL_INFEASIBLE 1
#define QPCG_STATUS_DUAL_INFEASIBLE 2
#define QPCG_STATUS_MAX_ITER_REACHED 3

/* ---- CSR views (sparse.hpp:47-56) -------------------------------------- */
typedef struct {
  uint32_t rows, cols, nnz;
  const double* values;         /* [nnz] */
  const uint32_t* row_ptr;      /* [rows + 1] */
  const uint32_t* col_indices;  /* [nnz] */
} qpcg_csr_f64;

typedef struct {
  uint32_t rows, cols, nnz;
  const float* values;
  const uint32_t* row_ptr;
  const uint32_t* col_indices;
} qpcg_csr_f32;

/* ---- Settings<T> mirror, field for field (settings.hpp:25-42) ----------
 * Values are carried as double for both precisions; the f32 entry points
 * convert each to float exactly as `T(1.6)` etc. would.
 * precision_note (informational only) is not carried. */
typedef struct {
  double alpha;         /* 1.6   relaxation, (0, 2) */
  double sigma;         /* 1e-6  proximal regularization, > 0 */
  double rho_bar_init;  /* 0.1 */
  double eps_abs;       /* 1e-3 */
  double eps_rel;       /* 1e-3 */
  double eps_pinf;      /* 1e-4 */
  double eps_dinf;      /* 1e-4 */
  uint32_t max_admm_iter;       /* 50000 */
  uint32_t check_interval;      /* 5 */
  uint32_t rho_update_interval; /* 10 */
  uint32_t scaling_enabled;     /* 1 (bool) */
  double lambda_pcg;    /* 0.15, (0, 1) */
  double eps_pcg_min;   /* 1e-7 */
  double eps_equil;     /* 1e-3 */
  uint32_t equil_max_passes;    /* 10 */
  uint32_t reserved_;
} qpcg_settings;

/* ---- SolveOutcome<T> scalars (solver.hpp:75-94) + engine timing --------- */
typedef struct {
  int32_t status;                /* QPCG_STATUS_* */
  uint32_t iterations;
  uint64_t pcg_iterations_total;
  double objective;              /* +inf / -inf when infeasible */
  double r_prim_inf;             /* unscaled residual norms at exit */
  double r_dual_inf;
  double runtime_seconds;        /* setup -> objective, as solver.hpp:392/:537 */
  uint32_t equil_passes;
  uint32_t rho_update_count;
  double equil_residual;
  double rho_final;
  uint32_t certificate_valid;    /* 1 when a certificate was written */
  uint32_t n, m;
  uint32_t engine_flags;         /* QPCG_ENGINE_*: which engine paths ran */
  /* engine-side measurements (device-timed with CUDA events) */
  double setup_seconds;          /* device setup: symmetrize/transpose/Ruiz/operator */
  double solve_seconds;          /* ADMM loop + unscale + objective */
  double h2d_seconds;            /* host->device upload inside setup (0 if device input) */
  double d2h_seconds;            /* result download inside solve */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint64_t kernel_launches;      /* launches of the engine's own kernels (setup
                                    counted on the first solve of a workspace) */
} qpcg_info;

/* ---- per-ADMM-iteration diagnostics (SolveDiagnostics, solver.hpp:148-167) */
typedef struct {
  uint32_t admm_iter;      /* 1-based */
  uint32_t iterations;     /* PCG iterations of this call */
  double eps;              /* tolerance handed to PCG */
  double r_prim_scaled_inf;
  double r_dual_scaled_inf;
  int32_t converged;
  int32_t reserved_;
} qpcg_pcg_call;

typedef struct {
  uint32_t admm_iter;
  uint32_t reserved_;
  double rho_before;
  double rho_after;
} qpcg_rho_update;

/* ---- engine options (not part of the reference's Settings) ------------- */
/* qpcg_info.engine_flags */
#define QPCG_ENGINE_ONE_PASS_OPERATOR 1u /* PCG operator apply with A streamed
                                            once (csrc/gram.cuh) */
#define QPCG_ENGINE_PERSISTENT 2u        /* the whole loop as one kernel */
#define QPCG_ENGINE_CARRIED_PRODUCTS 4u  /* z~ = A x~ and r0's A^T (rho z~) carried
                                            through PCG instead of recomputed every
                                            ADMM step (QPCG_ZT_RECUR=0
                                            turns it off) */

#define QPCG_MEM_HOST 0   /* caller arrays are host memory (copied in setup) */
#define QPCG_MEM_DEVICE 1 /* caller arrays are device memory on `device` */

#define QPCG_MODE_GRAPH 0 /* device-resident control flow: CUDA graph with
                             conditional while/if nodes (default) */
#define QPCG_MODE_EAGER 1 /* host-driven loop with a sync per decision (debug) */
#define QPCG_MODE_PERSISTENT 2 /* the whole loop in one kernel: one block (its
                                  L1 holding the matrices) while nnz(A) +
                                  nnz(P) <= 1200 (env QPCG_BLOCK_MAX_NNZ), one
                                  thread-block cluster (hardware barriers)
                                  while <= 1e4 (QPCG_CLUSTER_MAX_NNZ), else a
                                  cooperative grid.  GRAPH picks it by itself
                                  while nnz(A) + nnz(P) <= 2e6 (env
                                  QPCG_PERSIST_MAX_NNZ).  All modes give
                                  bitwise-identical results. */

/* Per-iteration observer (solver.hpp:132-145 IterationView): iter is the
 * 1-based ADMM iteration; x (n), z (m), y (m) the scaled iterates and l, u (m)
 * the scaled bounds, all host arrays of the workspace's precision (float or
 * double), valid only during the call. */
typedef void (*qpcg_iteration_cb)(void* user, uint32_t iter, const void* x, const void* z,
                                  const void* y, const void* l, const void* u, uint32_t n,
                                  uint32_t m);

/* Row sharding.  A is cut into G = virtual_shards x
 * nccl_ranks contiguous nnz-balanced row blocks (qpcg_shard_cuts); every
 * block keeps its own A_g^T, P and the n-vectors are replicated, and the A^T
 * partials are summed across blocks once per operator apply.  Every rank
 * passes the FULL problem (it uploads only its blocks) and receives the full
 * x, z, y.  Loop driver: QPCG_MODE_GRAPH with the peer transport (or
 * virtual blocks only) runs the whole sharded loop as one CUDA graph with
 * conditional nodes (every collective is a kernel); with the NCCL transport,
 * or in QPCG_MODE_EAGER / QPCG_MODE_PERSISTENT, the loop is host-driven (one
 * control-block read per decision). */
typedef struct {
  int32_t device;          /* CUDA ordinal, -1 = current */
  int32_t input_memory;    /* QPCG_MEM_HOST / QPCG_MEM_DEVICE */
  int32_t mode;            /* QPCG_MODE_* */
  int32_t record_diagnostics; /* 1: keep per-PCG-call records */
  int32_t virtual_shards;  /* >1: this process holds that many row blocks on
                              its device, combined in block order */
  int32_t nccl_rank;       /* rank of this process in the NCCL group */
  int32_t nccl_ranks;      /* processes (one per GPU) in the NCCL group */
  int32_t sm_budget;       /* 0: the persistent driver may use the whole
                              device.  k > 0: at most k SMs (a cooperative
                              grid of k SMs, one 16-SM cluster, or one block),
                              so that many small solves share one GPU
                              (batching); results are unchanged */
  void* stream;            /* cudaStream_t to run on (NULL: the workspace
                              creates its own non-blocking stream) */
  const void* nccl_id;     /* NULL: no NCCL.  Else the QPCG_NCCL_ID_BYTES-byte
                              id from qpcg_nccl_unique_id on rank 0, shared by
                              all ranks (e.g. a torch.distributed broadcast) */
  int32_t transport;       /* QPCG_TRANSPORT_*: how the ranks' row blocks are
                              combined */
  int32_t reserved2_;
  const char* rendezvous_dir; /* QPCG_TRANSPORT_PEER without an NCCL id: a
                              directory shared by the ranks (fresh per group)
                              through which they exchange their IPC handles */
  qpcg_iteration_cb on_iteration; /* SolveDiagnostics::on_iteration
                              (solver.hpp:166, :451-454): when set, the solve
                              runs the host-driven loop and calls it after
                              every ADMM step with the SCALED iterates (one
                              device->host copy of x, z, y per iteration: an
                              instrumented mode, not a fast path).  Unsharded
                              workspaces only. */
  void* on_iteration_user;  /* passed back as the callback's first argument */
} qpcg_options;

/* NCCL collectives (default), or stores into every peer's memory (CUDA IPC /
 * NVLink P2P) with device-side barriers: the ranks' partials are summed in
 * block order, bitwise identical to a one-process run with the same number
 * of virtual blocks.  nccl_rank / nccl_ranks give the rank and group size
 * for both transports. */
#define QPCG_TRANSPORT_NCCL 0
#define QPCG_TRANSPORT_PEER 1

#define QPCG_NCCL_ID_BYTES 128

typedef struct qpcg_workspace qpcg_workspace;

/* defaults exactly as settings.hpp:25-42 */
void qpcg_default_settings(qpcg_settings* s);
void qpcg_default_options(qpcg_options* o);
/* settings.hpp:44-75; returns QPCG_OK or QPCG_ERR_INVALID (message via msg) */
int qpcg_validate_settings(const qpcg_settings* s, char* msg, size_t msg_len);
const char* qpcg_version(void);

/* ---- fp64 ---------------------------------------------------------------- */
int qpcg_f64_setup(qpcg_workspace** ws, const qpcg_csr_f64* p_upper,
                   const double* q, const qpcg_csr_f64* a, const double* l,
                   const double* u, const qpcg_settings* settings,
                   const qpcg_options* options);
int qpcg_f64_warm_start(qpcg_workspace* ws, const double* x, const double* z,
                        const double* y);
int qpcg_f64_update_rho(qpcg_workspace* ws, double rho);
int qpcg_f64_update_vectors(qpcg_workspace* ws, const double* q,
                            const double* l, const double* u);
/* x[n], z[m], y[m] and cert (n or m; pass max(n, m)) may be NULL; they are
 * host pointers unless options.input_memory == QPCG_MEM_DEVICE. */
int qpcg_f64_solve(qpcg_workspace* ws, qpcg_info* info, double* x, double* z,
                   double* y, double* cert);
int qpcg_f64_solve_problem(const qpcg_csr_f64* p_upper, const double* q,
                           const qpcg_csr_f64* a, const double* l,
                           const double* u, const qpcg_settings* settings,
                           const qpcg_options* options, const double* warm_x,
                           const double* warm_z, const double* warm_y,
                           qpcg_info* info, double* x, double* z, double* y,
                           double* cert, char* msg, size_t msg_len);

/* ---- fp32 ---------------------------------------------------------------- */
int qpcg_f32_setup(qpcg_workspace** ws, const qpcg_csr_f32* p_upper,
                   const float* q, const qpcg_csr_f32* a, const float* l,
                   const float* u, const qpcg_settings* settings,
                   const qpcg_options* options);
int qpcg_f32_warm_start(qpcg_workspace* ws, const float* x, const float* z,
                        const float* y);
int qpcg_f32_update_rho(qpcg_workspace* ws, double rho);
int qpcg_f32_update_vectors(qpcg_workspace* ws, const float* q, const float* l,
                            const float* u);
int qpcg_f32_solve(qpcg_workspace* ws, qpcg_info* info, float* x, float* z,
                   float* y, float* cert);
int qpcg_f32_solve_problem(const qpcg_csr_f32* p_upper, const float* q,
                           const qpcg_csr_f32* a, const float* l,
                           const float* u, const qpcg_settings* settings,
                           const qpcg_options* options, const float* warm_x,
                           const float* warm_z, const float* warm_y,
                           qpcg_info* info, float* x, float* z, float* y,
                           float* cert, char* msg, size_t msg_len);

/* ---- row sharding --------------------------------------------------------
 * nnz-balanced contiguous row cuts of a CSR row_ptr (host memory) into G
 * blocks: block g owns rows [cuts[g], cuts[g+1]) with cuts[g] the first row
 * whose row_ptr >= g*nnz/G.  Returns 1, or 0 when row_ptr is invalid (then
 * every row is on block 0 and setup reports the reference's error). */
int qpcg_shard_cuts(const uint32_t* row_ptr, uint32_t rows, uint32_t nnz,
                    uint32_t blocks, uint32_t* cuts);
/* writes QPCG_NCCL_ID_BYTES bytes (ncclGetUniqueId); QPCG_ERR_NCCL if NCCL
 * cannot be loaded */
int qpcg_nccl_unique_id(void* out);

/* ---- common to both precisions ------------------------------------------ */
void qpcg_cleanup(qpcg_workspace* ws);
/* Hands the engine's idle device memory back to the driver: the process-wide
 * cache of released workspace blocks (at most QPCG_CACHE_MAX_GB, default 32)
 * and the unused part of the engine's own per-device memory pools (the
 * devices' default pools are never modified).  Live workspaces keep theirs.
 * Synchronises every device the engine has used.  No reference counterpart
 * (the reference frees its std::vectors on return). */
void qpcg_release_cached_memory(void);
const char* qpcg_last_error(const qpcg_workspace* ws);
/* copies up to `cap` records; returns the total number recorded */
uint32_t qpcg_get_pcg_calls(const qpcg_workspace* ws, qpcg_pcg_call* out,
                            uint32_t cap);
uint32_t qpcg_get_rho_updates(const qpcg_workspace* ws, qpcg_rho_update* out,
                              uint32_t cap);
uint32_t qpcg_get_check_iterations(const qpcg_workspace* ws, uint32_t* out,
                                   uint32_t cap);

#ifdef __cplusplus
}
#endif

#endif /* QPCG_B200_H */
