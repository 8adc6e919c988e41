#pragma once
// workspace.cuh — the B200 ADMM/PCG workspace (one device, one stream, all buffers).
//
// Drop-in for qpcg::solve (solver.hpp:386-541).  One workspace = one device,
// one stream, all buffers; calls on distinct workspaces are re-entrant.
//
// Per ADMM step (SURVEY.md §7 hard part 4b):
//   A^T pass  [rhs = A^T(rho z - y) + (sigma x - q) ; r0 = K x~ - rhs]   2 cols
//   k_pcg_init
//   while PCG: A pass [t = rho A p] ; A^T pass [Kp = P p + sigma p + A^T t] ;
//              k_pcg_dot ; k_pcg_update ; k_pcg_pupdate
//   k_pcg_fin
//   A pass    [z~ = A x~, m-side relax/project/dual update (; A x_new on
//             check iterations: 2 cols, else 1 col)]
//   k_xupdate
//   if check: A^T pass [A^T y, P x, r_dual] ; k_residuals
//             if not optimal: A_o^T, P_o, A_o passes ; k_infeas
//   if rho:   k_rho ; k_precond
// The matrix streams are A and A^T once per PCG iteration plus once each per
// ADMM step (the reference streams 4 A-sized matrices + P per step).
//
// Three drivers run this sequence with bitwise-identical results: a CUDA
// graph with conditional WHILE/IF nodes (default), the persistent kernel of
// persist.cuh (one block / one cluster / a cooperative grid; picked by the
// graph mode for small problems) and a host-driven eager loop.  The row-
// sharded engine (shard.cuh) drives one Workspace per row block.  Setup
// allocations go through the workspace's arena (common.cuh).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/qpcg_b200.h"
#include "../../include/qpcg_b200_ops.h"
#include "admm.cuh"
#include "comm.cuh"
#include "gram.cuh"
#include "persist.cuh"
#include "setup.cuh"
#include "upload.cuh"

namespace qpcg_b200 {

template <typename T>
struct HostCsr {
  uint32_t rows, cols, nnz;
  const T* values;
  const uint32_t* row_ptr;
  const uint32_t* col_indices;
};

inline double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// ------------------------------------------------------------ setup kernels
// act: this pass runs (device flag); act_next (nullable): written with
// whether the next pass runs, (more && deviation > eps) — the loop test of
// scaling.hpp:116 decided on the device, so the passes need no host sync
template <typename T>
__global__ void __launch_bounds__(kThreads) k_ruiz_delta(const T* pn, const T* atn, uint32_t n,
                                                        const T* an, uint32_t m, T* dx, T* dz,
                                                        T* d, T* e, T* q, T* part,
                                                        uint32_t* counter, T* dev_out,
                                                        const uint32_t* act, uint32_t* act_next,
                                                        uint32_t more, T eps) {
  // scaling.hpp:125-138: delta = 1/sqrt(col norm) (1 for empty), D *= dx, E *= dz,
  // q *= dx; deviation = |1 - delta|_inf (:163-165)
  if (act && !*act) return;
  T v[1] = {T(0)};
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T cn = smax(pn[i], atn[i]);
    const T di = cn > T(0) ? T(1) / t_sqrt(cn) : T(1);
    dx[i] = di;
    d[i] *= di;
    q[i] *= di;
    v[0] = smax(v[0], tabs(T(1) - di));
  }
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const T a = an[j];
    const T dj = a > T(0) ? T(1) / t_sqrt(a) : T(1);
    dz[j] = dj;
    e[j] *= dj;
    v[0] = smax(v[0], tabs(T(1) - dj));
  }
  T tot[1];
  if (!grid_reduce<T, 1>(v, 0x1u, part, counter, tot)) return;
  if (threadIdx.x == 0) {
    *dev_out = tot[0];
    if (act_next) *act_next = (more && tot[0] > eps) ? 1u : 0u;
  }
}

// gamma = 1/max(mean, |q|_inf) (1 if 0); c *= gamma  (scaling.hpp:159-162)
template <typename T>
__global__ void k_ruiz_gamma(const T* mean, const T* qinf, T* gamma, T* c, const uint32_t* act) {
  if (act && !*act) return;
  const T denom = smax(*mean, *qinf);
  const T g = denom > T(0) ? T(1) / denom : T(1);
  *gamma = g;
  *c *= g;
}

template <typename T>
__global__ void k_scale_by(T* v, uint32_t n, const T* g, const uint32_t* act) {
  if (act && !*act) return;
  const T s = *g;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v[i] *= s;
}

// =====================================================================
// What the C-ABI (engine.cu) sees of an engine: the single-device Workspace
// below or the row-sharded Sharded (shard.cuh).  engine.cu instantiates no
// kernel; each precision is compiled in its own TU (engine_f64.cu /
// engine_f32.cu) behind make_engine<T>.
template <typename T>
struct IEngine {
  using value_type = T;
  virtual ~IEngine() = default;
  virtual void setup(const HostCsr<T>& Pu, const T* q, const HostCsr<T>& A, const T* l,
                     const T* u, const qpcg_settings& st, const qpcg_options& op) = 0;
  virtual void warm_start(const T* x, const T* z, const T* y) = 0;
  virtual void update_rho(T rho) = 0;
  virtual void update_vectors(const T* q, const T* l, const T* u) = 0;
  virtual void solve(qpcg_info* info, T* x, T* z, T* y, T* cert) = 0;
  // diagnostics / debug / kernel timing (the first row block when sharded)
  virtual uint32_t pcg_calls(qpcg_pcg_call* out, uint32_t cap) = 0;
  virtual uint32_t rho_updates(qpcg_rho_update* out, uint32_t cap) = 0;
  virtual uint32_t check_iterations(uint32_t* out, uint32_t cap) = 0;
  virtual void dims(uint64_t* d) = 0;
  virtual void debug_scaled(T* pv, uint32_t* prp, uint32_t* pci, T* q, T* av, T* atv,
                            uint32_t* atrp, uint32_t* atci, T* l, T* u, T* d, T* e,
                            double* scal) = 0;
  virtual void debug_operator(const T* x, T* kx, T* dinv) = 0;
  virtual void bench_kernels(uint32_t reps, double* out) = 0;
};
template <typename T>
IEngine<T>* make_engine(bool sharded);             // engine_fXX.cu
template <typename T>
void validate_settings_in(const qpcg_settings& s);  // engine_fXX.cu (settings.hpp:44-75 in T)
template <typename T>
void op_spmv(const HostCsr<T>& m, const T* x, T* y, int device);  // engine_fXX.cu
template <typename T>
void op_pcg(const HostCsr<T>& pf, const HostCsr<T>& a, const HostCsr<T>& at, T sigma, T rho,
            const T* b, const T* warm, T eps, uint32_t max_iter, T* x, double* res,
            int device);  // engine_fXX.cu

// =====================================================================
template <typename T>
class Workspace : public IEngine<T> {
 public:
  int device = 0;
  cudaStream_t s = nullptr;
  CubTemp tmp;
  Dev<T> D{};
  Ctl<T> hc{};
  qpcg_settings set{};
  qpcg_options opt{};
  std::vector<void*> allocs;
  uint32_t* permA = nullptr;  // transpose permutation of A
  WinPlan winA;               // its windowed-gather plan (setup only)
  uint32_t* p_rows = nullptr;  // rows of P_full with entries (ordered mean)
  uint32_t n_prows = 0;
  T* ruiz_scal = nullptr;      // [mean, qinf, gamma, c, dev]
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double setup_seconds = 0, h2d_seconds = 0, setup_wall = 0;
  uint64_t h2d_bytes = 0;
  std::string err;
  bool have_solved = false;
  bool own_stream = true;
  uint64_t setup_launches = 0;
  bool have_counted_setup = false;
  bool ran_persistent = false;

  ~Workspace() {
    if (up_thread.joinable()) up_thread.join();  // (a setup that failed before wait_values)
    if (s_up) {
      cudaStreamSynchronize(s_up);
      cudaStreamDestroy(s_up);
    }
    if (ev_vals) cudaEventDestroy(ev_vals);
    if (s_side) {
      cudaStreamSynchronize(s_side);
      cudaStreamDestroy(s_side);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    {
      AllocScope scope(s, &arena);
      if (s) cudaStreamSynchronize(s);  // every stream that used the buffers is idle now
      for (void* p : allocs) dfree(p);  // arena blocks: back to the arena; others: the pool
      for (SpmvPlan<T>* p : {&D.pP, &D.pA, &D.pAT, &gLo, &gHi}) plan_free(*p);
      if (tmp.ptr) dfree(tmp.ptr);
      tmp.ptr = nullptr;
      tmp.bytes = 0;
      if (s) cudaStreamSynchronize(s);
      arena.return_all();
    }
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (s && own_stream) cudaStreamDestroy(s);
  }

  Arena arena;  // see common.cuh
  template <typename U>
  U* alloc(size_t count) {
    void* p = nullptr;
    AllocScope scope(s, &arena);
    CK(dmalloc(&p, sizeof(U) * (count ? count : 1)));
    allocs.push_back(p);
    return static_cast<U*>(p);
  }
  T* vec(size_t count, bool zero = true) {
    T* p = alloc<T>(count);
    if (zero) CK(cudaMemsetAsync(p, 0, sizeof(T) * (count ? count : 1), s));
    return p;
  }
  void upload(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (opt.input_memory == QPCG_MEM_HOST) {
      CK(h2d(dst, src, bytes, s, device));  // pageable sources through the pinned stager
      h2d_bytes += bytes;
    } else {
      CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  void download(void* dst, const void* src, size_t bytes) {
    if (bytes == 0 || dst == nullptr) return;
    const bool host = opt.input_memory == QPCG_MEM_HOST;
    CK(cudaMemcpyAsync(dst, src, bytes, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s));
  }
  void fill(T* p, uint32_t n, T v) {
    for_n(n, [=] __device__(uint32_t i) { p[i] = v; }, s);
  }
  T read_scalar(const T* p) {
    T v;
    CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
  }
  void pull_ctl() {
    CK(cudaMemcpyAsync(&hc, D.ctl, sizeof(Ctl<T>), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  void push_ctl() { CK(cudaMemcpyAsync(D.ctl, &hc, sizeof(Ctl<T>), cudaMemcpyHostToDevice, s)); }

  // ------------------------------------------------------------- setup
  // The single-device setup; the sharded path (shard.cuh) runs the same
  // phases per row block with its collectives in between.
  void setup(const HostCsr<T>& Pu, const T* q, const HostCsr<T>& A, const T* l, const T* u,
             const qpcg_settings& st, const qpcg_options& op) override {
    const double w0 = now_s();
    const uint64_t l0 = g_launches;
    begin(st, op, nullptr);
    AllocScope scope(s, &arena);
    CK(cudaEventRecord(ev0, s));
    // host input: A's values (2/3 of the upload) come in on a side stream
    // while the structural setup (validation of the rows, plans, symmetrize,
    // the transpose structure, the compressed index) runs on the main one
    {
      const char* e = std::getenv("QPCG_NO_DEFER");
      defer_values = op.input_memory == QPCG_MEM_HOST && !(e && e[0] == '1');
    }
    // QPCG_SETUP_TRACE=1: host time at each phase boundary (stream synced)
    static const bool trace = [] {
      const char* e = std::getenv("QPCG_SETUP_TRACE");
      return e && e[0] == '1';
    }();
    auto mark = [&](const char* what) {
      if (!trace) return;
      CK(cudaStreamSynchronize(s));
      std::fprintf(stderr, "[setup] %-16s %8.3f ms  launches %llu\n", what, (now_s() - w0) * 1e3,
                   (unsigned long long)(g_launches - l0));
    };
    trace_t0 = trace ? w0 : 0.0;
    load(Pu, q, A, l, u, 0, A.rows, false);
    mark("load");
    ValKeys k = validate_keys();
    raise_first(k);
    mark("validate");
    build_structures();
    mark("structures");
    uint32_t passes = 0;
    T deviation = T(0);
    if (set.scaling_enabled) {
      // every pass enqueued at once: pass p's kernels run iff rz_act[p]
      // (k_ruiz_delta of pass p - 1 decides), one synchronisation at the end
      ruiz_prepare();
      tmark("ruiz prepare");
      const uint32_t P = set.equil_max_passes;
      rz_act = alloc<uint32_t>(size_t(P) + 1);
      rz_dev = vec(size_t(P) + 1, true);
      CK(cudaMemsetAsync(rz_act, 0, sizeof(uint32_t) * (size_t(P) + 1), s));
      const uint32_t one = 1u;
      CK(cudaMemcpyAsync(rz_act, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
      for (uint32_t p = 0; p < P; ++p) {
        ruiz_norms(int(p));
        ruiz_delta(int(p));
        ruiz_scale(int(p));
        if (p < 2) tmark(p == 0 ? "ruiz pass 0" : "ruiz pass 1");
      }
      std::vector<uint32_t> act(size_t(P) + 1);
      std::vector<T> dev(size_t(P) + 1);
      CK(cudaMemcpyAsync(act.data(), rz_act, sizeof(uint32_t) * (size_t(P) + 1),
                         cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(dev.data(), rz_dev, sizeof(T) * (size_t(P) + 1), cudaMemcpyDeviceToHost,
                         s));
      CK(cudaStreamSynchronize(s));
      while (passes < P && act[passes]) ++passes;
      deviation = passes ? dev[passes - 1] : T(1);
    }
    mark("ruiz");
    finish_scaling(passes, deviation);
    diag_ata_kernel<T><<<grid_for(uint64_t(D.n) * 32), kThreads, 0, s>>>(D.AT, D.diag_ata, nullptr);
    CK_LAUNCH();
    mark("finish_scaling");
    finish_setup();
    mark("finish_setup");
    build_gram();
    mark("gram");
    CK(cudaEventRecord(ev1, s));
    CK(cudaEventSynchronize(ev1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    setup_seconds = ms * 1e-3;
    setup_wall = now_s() - w0;
    setup_launches = g_launches - l0;
  }

  uint32_t equil_passes = 0;
  T equil_residual = T(0);

  // setup-phase state
  uint32_t *pu_rp = nullptr, *pu_ci = nullptr, *a_rp = nullptr, *a_ci = nullptr;
  T *pu_v = nullptr, *a_v = nullptr;
  uint32_t pu_nnz = 0, pu_cols = 0, a_cols = 0;
  uint32_t row0 = 0;  // first global row of this block of A (sharded path)
  uint32_t nnz0 = 0;  // first global entry of this block
  bool p_square = true, a_cols_ok = true;
  T *rz_dx = nullptr, *rz_dz = nullptr, *rz_pn = nullptr, *rz_atn = nullptr, *rz_an = nullptr;

  // settings, device, stream, pool, events
  void begin(const qpcg_settings& st, const qpcg_options& op, cudaStream_t shared) {
    set = st;
    opt = op;
    validate_settings(st);
    device = op.device;
    if (device < 0) CK(cudaGetDevice(&device));
    CK(cudaSetDevice(device));
    if (shared != nullptr) {
      s = shared;
      own_stream = false;
    } else if (op.stream != nullptr) {
      s = static_cast<cudaStream_t>(op.stream);
      own_stream = false;
    } else {
      CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    configure_pool(device);
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
  }

  // Upload P (upper), q and the row block [r0, r1) of A, l, u — the only
  // host->device traffic of a solve.  slice == false: A as given (rows 0..m).
  void load(const HostCsr<T>& Pu, const T* q, const HostCsr<T>& A, const T* l, const T* u,
            uint32_t r0, uint32_t r1, bool slice) {
    const double th = now_s();
    const uint32_t n = Pu.rows, m = r1 - r0;
    p_square = Pu.rows == Pu.cols;
    a_cols_ok = A.cols == Pu.cols;
    pu_nnz = Pu.nnz;
    pu_cols = Pu.cols;
    a_cols = A.cols;
    D.n = n;
    D.m = m;
    uint32_t e0 = 0, e1 = A.nnz;
    if (slice) {  // row_ptr is valid here (shard_cuts checked it on the host)
      e0 = host_rp(A, r0);
      e1 = host_rp(A, r1);
    }
    row0 = r0;
    nnz0 = e0;
    const uint32_t annz = e1 - e0;
    pu_rp = alloc<uint32_t>(n + 1);
    pu_ci = alloc<uint32_t>(Pu.nnz);
    pu_v = alloc<T>(Pu.nnz);
    a_rp = alloc<uint32_t>(m + 1);
    a_ci = alloc<uint32_t>(annz);
    a_v = alloc<T>(annz);
    D.q_o = alloc<T>(n);
    D.l_o = alloc<T>(m);
    D.u_o = alloc<T>(m);
    upload(pu_rp, Pu.row_ptr, sizeof(uint32_t) * (n + 1));
    upload(pu_ci, Pu.col_indices, sizeof(uint32_t) * Pu.nnz);
    upload(pu_v, Pu.values, sizeof(T) * Pu.nnz);
    upload(a_rp, A.row_ptr + r0, sizeof(uint32_t) * (m + 1));
    upload(a_ci, A.col_indices + e0, sizeof(uint32_t) * annz);
    if (defer_values && annz) {
      if (!s_up) {
        CK(cudaStreamCreateWithFlags(&s_up, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_vals, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(ev_vals, s));  // a_v is allocated on s
      CK(cudaStreamWaitEvent(s_up, ev_vals, 0));
      // a background host thread feeds the copy (a pageable source is staged
      // by host threads; cudaMemcpyAsync would block this thread until done)
      // while this one enqueues the structural setup
      const void* src = A.values + e0;
      const size_t nb = sizeof(T) * annz;
      T* dst = a_v;
      const int dev = device;
      cudaStream_t su = s_up;
      cudaEvent_t ev = ev_vals;
      up_err = cudaSuccess;
      up_thread = std::thread([this, src, nb, dst, dev, su, ev] {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = h2d(dst, src, nb, su, dev);
        if (e == cudaSuccess) e = cudaEventRecord(ev, su);
        up_err = e;
      });
      h2d_bytes += nb;
      values_pending = true;
    } else {
      upload(a_v, A.values + e0, sizeof(T) * annz);
    }
    upload(D.q_o, q, sizeof(T) * n);
    upload(D.l_o, l + r0, sizeof(T) * m);
    upload(D.u_o, u + r0, sizeof(T) * m);
    if (slice && e0 != 0) {
      uint32_t* rp = a_rp;
      for_n(m + 1, [=] __device__(uint32_t i) { rp[i] -= e0; }, s);
    }
    D.A = DevCsr<T>{m, A.cols, annz, a_v, a_rp, a_ci};
    h2d_t0 = th;
    if (opt.input_memory == QPCG_MEM_HOST && !values_pending) {
      CK(cudaStreamSynchronize(s));
      h2d_seconds = now_s() - th;
    }
  }
  // deferred-values bookkeeping (single-device host-input setup)
  bool defer_values = false, values_pending = false;
  cudaStream_t s_up = nullptr;
  cudaEvent_t ev_vals = nullptr;
  double h2d_t0 = 0;
  std::thread up_thread;
  cudaError_t up_err = cudaSuccess;
  void wait_values() {
    if (!values_pending) return;
    if (up_thread.joinable()) up_thread.join();
    CK(up_err);
    CK(cudaStreamWaitEvent(s, ev_vals, 0));
    CK(cudaEventSynchronize(ev_vals));
    h2d_seconds = now_s() - h2d_t0;  // upload wall time, overlapped with the structural setup
    values_pending = false;
  }
  uint32_t host_rp(const HostCsr<T>& A, uint32_t r) {
    if (opt.input_memory == QPCG_MEM_HOST) return A.row_ptr[r];
    uint32_t v = 0;
    CK(cudaMemcpyAsync(&v, A.row_ptr + r, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return v;
  }

  // Validation (problem.hpp:46-92, sparse.hpp:98-124): three stage keys, each
  // the minimum (category, global index, position) found; raise_first applies
  // the reference's check order.  Keys of row blocks combine by min.
  struct ValKeys {
    unsigned long long k[3];  // P rows, A rows, values/bounds
    uint32_t ends[4];         // P row_ptr ends, A row_ptr ends (block-local)
  };
  ValKeys validate_keys() {
    const uint32_t n = D.n, m = D.m;
    ValKeys v;
    CK(cudaMemcpyAsync(v.ends + 0, pu_rp, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v.ends + 1, pu_rp + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v.ends + 2, a_rp, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v.ends + 3, a_rp + m, 4, cudaMemcpyDeviceToHost, s));
    unsigned long long* key = alloc<unsigned long long>(3);
    CK(cudaMemsetAsync(key, 0xff, 24, s));
    CK(cudaStreamSynchronize(s));
    const bool p_ok = v.ends[0] == 0 && v.ends[1] == pu_nnz;
    const bool a_ok = v.ends[2] == 0 && v.ends[3] == D.A.nnz;
    if (p_ok) {
      validate_csr_rows_kernel<<<grid_for(n), kThreads, 0, s>>>(pu_rp, pu_ci, n, pu_cols, kValPRowPtr,
                                                               p_square ? 1 : 0, key, 0);
      CK_LAUNCH();
    }
    if (a_ok) {
      validate_csr_rows_kernel<<<grid_for(m), kThreads, 0, s>>>(a_rp, a_ci, m, a_cols, kValARowPtr, 0,
                                                               key + 1, row0);
      CK_LAUNCH();
      if (!values_pending) launch_value_checks(key + 2);
    }
    CK(cudaMemcpyAsync(v.k, key, 24, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (values_pending) value_key = key + 2;  // checked once the values have arrived
    return v;
  }
  unsigned long long* value_key = nullptr;
  void launch_value_checks(unsigned long long* key) {
    const uint32_t n = D.n, m = D.m;
    validate_values_kernel<T><<<grid_for(pu_nnz), kThreads, 0, s>>>(pu_v, pu_nnz, kValPFinite, key, 0);
    validate_values_kernel<T><<<grid_for(D.A.nnz), kThreads, 0, s>>>(a_v, D.A.nnz, kValAFinite, key, nnz0);
    validate_values_kernel<T><<<grid_for(n), kThreads, 0, s>>>(D.q_o, n, kValQFinite, key, 0);
    validate_bounds_kernel<T><<<grid_for(m), kThreads, 0, s>>>(D.l_o, D.u_o, m, key, row0);
    CK_LAUNCH();
  }
  // the values' checks (problem.hpp:75-91, the last in the reference's order)
  // after a deferred upload
  void check_values_late() {
    if (!value_key) return;
    wait_values();
    launch_value_checks(value_key);
    unsigned long long k = 0;
    CK(cudaMemcpyAsync(&k, value_key, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    value_key = nullptr;
    if (k != ~0ull) throw InvalidArgument(validation_message(k));
  }
  void raise_first(const ValKeys& v) const {
    if (v.ends[0] != 0 || v.ends[1] != pu_nnz)
      throw InvalidArgument("csr: row_ptr must start at 0 and end at nnz");
    if ((v.k[0] >> 56) == kValPRowPtr) throw InvalidArgument(validation_message(v.k[0]));
    if (v.ends[2] != 0 || v.ends[3] != D.A.nnz)
      throw InvalidArgument("csr: row_ptr must start at 0 and end at nnz");
    if ((v.k[1] >> 56) == kValARowPtr) throw InvalidArgument(validation_message(v.k[1]));
    if (!p_square) throw InvalidArgument("problem: P must be square");
    if (D.n == 0) throw InvalidArgument("problem: at least one variable required");
    if ((v.k[0] >> 56) == kValPBelow) throw InvalidArgument(validation_message(v.k[0]));
    if (!a_cols_ok) throw InvalidArgument("problem: A column count must equal n");
    if (v.k[2] != ~0ull) throw InvalidArgument(validation_message(v.k[2]));
  }

  static bool compress_indices() {  // QPCG_COMPRESS=0: uint32 column streams
    const char* e = std::getenv("QPCG_COMPRESS");
    return !(e && e[0] == '0');
  }

  // symmetrize_upper, transpose_csr, plans, the original and scaled copies
  // QPCG_SETUP_TRACE=1: finer marks inside build_structures (stream synced)
  double trace_t0 = 0.0;
  void tmark(const char* what) {
    if (trace_t0 == 0.0) return;
    CK(cudaStreamSynchronize(s));
    std::fprintf(stderr, "[setup]   %-20s %8.3f ms\n", what, (now_s() - trace_t0) * 1e3);
  }
  void build_structures() {
    // this workspace's stream and arena for the transient buffers too (the
    // helpers free them stream-ordered, without a synchronisation)
    AllocScope scope(s, &arena);
    const uint32_t n = D.n, m = D.m, annz = D.A.nnz;
    DevCsr<T> Pup{n, n, pu_nnz, pu_v, pu_rp, pu_ci};
    SpmvPlan<T> pPu = plan_build<T>(pu_rp, n, pu_nnz, tmp, s);
    D.pA = plan_build<T>(a_rp, m, annz, tmp, s);
    uint32_t* row_of = alloc<uint32_t>(std::max(pu_nnz, annz));
    plan_visit(Pup, pPu, RowOfFn{row_of}, s);
    // symmetrize_upper (solver.hpp:397)
    DevCsr<T> Pfull;
    symmetrize_upper_dev(Pup, row_of, Pfull, tmp, s);
    allocs.push_back(Pfull.rp);
    allocs.push_back(Pfull.ci);
    allocs.push_back(Pfull.val);
    plan_free(pPu);
    D.pP = plan_build<T>(Pfull.rp, n, Pfull.nnz, tmp, s);
    D.Po = Pfull;
    tmark("plans A, P + symm.");
    // transpose_csr (solver.hpp:398)
    plan_visit(D.A, D.pA, RowOfFn{row_of}, s);
    uint32_t* at_rp = alloc<uint32_t>(n + 1);
    uint32_t* at_ci = alloc<uint32_t>(annz);
    permA = alloc<uint32_t>(annz);
    transpose_structure(a_ci, row_of, n, annz, at_rp, at_ci, permA, tmp, s, &winA);
    tmark("transpose struct");
    D.pAT = plan_build<T>(at_rp, n, annz, tmp, s);
    tmark("plan A^T");
    if (compress_indices()) {  // 16-bit column offsets for the A / A^T streams
      plan_compress(D.pA, a_ci, annz, n, tmp, s);
      plan_compress(D.pAT, at_ci, annz, m, tmp, s);
    }
    tmark("compress");
    // ---- from here on A's values are needed
    check_values_late();
    tmark("values");
    T* ato_v = alloc<T>(annz);
    gather_windowed(a_v, permA, at_rp, annz, winA, ato_v, s);
    tmark("A_orig^T gather");
    D.Ao = DevCsr<T>{m, n, annz, a_v, a_rp, a_ci};
    D.ATo = DevCsr<T>{n, m, annz, ato_v, at_rp, at_ci};
    D.pPo = D.pP;
    D.pAo = D.pA;
    D.pATo = D.pAT;
    // ---- control block + reductions
    D.ctl = alloc<Ctl<T>>(1);
    D.red = alloc<T>(kRedBlocks * kMaxQ);
    CK(cudaMemsetAsync(D.ctl, 0, sizeof(Ctl<T>), s));
    ruiz_scal = vec(8);
    // q_inf_orig (solver.hpp:399)
    k_infnorm<T><<<red_grid<T>(n), kThreads, 0, s>>>(D.q_o, n, D.red, &D.ctl->red_counter,
                                                      ruiz_scal + 5);
    CK_LAUNCH();
    // ---- scaled copies
    D.P = DevCsr<T>{n, n, Pfull.nnz, alloc<T>(Pfull.nnz), Pfull.rp, Pfull.ci};
    D.A = DevCsr<T>{m, n, annz, alloc<T>(annz), a_rp, a_ci};
    D.AT = DevCsr<T>{n, m, annz, alloc<T>(annz), at_rp, at_ci};
    CK(cudaMemcpyAsync(D.P.val, Pfull.val, sizeof(T) * Pfull.nnz, cudaMemcpyDeviceToDevice, s));
    // with scaling, the first Ruiz pass writes the scaled A and A^T straight
    // from the originals (ruiz_scale), so they are not copied here
    if (!set.scaling_enabled) {
      CK(cudaMemcpyAsync(D.A.val, a_v, sizeof(T) * annz, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(D.AT.val, ato_v, sizeof(T) * annz, cudaMemcpyDeviceToDevice, s));
    }
    D.q = vec(n, false);
    CK(cudaMemcpyAsync(D.q, D.q_o, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
    D.d = vec(n, false);
    D.e = vec(m, false);
    D.d_inv = vec(n, false);
    D.e_inv = vec(m, false);
    D.l = vec(m, false);
    D.u = vec(m, false);
    fill(D.d, n, T(1));
    fill(D.e, m, T(1));
    const T c = T(1);
    CK(cudaMemcpyAsync(ruiz_scal + 3, &c, sizeof(T), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }

  // modified Ruiz equilibration (scaling.hpp:92-187), bit-exact, one pass per
  // ruiz_norms / ruiz_delta / ruiz_scale; ruiz_scal[4] = the pass deviation.
  // Row blocks combine rz_atn (max) and the deviation (max) in between: both
  // maxima are order-free, so the sharded scaling is bit-identical too.
  void ruiz_prepare() {
    const uint32_t n = D.n, m = D.m;
    rz_norms_fresh = false;
    rz_dx = vec(n, false);
    rz_dz = vec(m, false);
    rz_pn = vec(n, false);
    rz_atn = vec(n, false);
    rz_an = vec(m, false);
    // rows of P_full with entries, for the ordered mean (structure is fixed)
    uint32_t* flags = alloc<uint32_t>(n + 1);
    uint32_t* pos = alloc<uint32_t>(n + 1);
    p_rows = alloc<uint32_t>(n + 1);
    nonempty_flags_kernel<<<grid_for(n), kThreads, 0, s>>>(D.P.rp, n, flags);
    CK_LAUNCH();
    exclusive_scan_u32(flags, pos, n, tmp, s);
    n_prows = scan_total(flags, pos, n, s);
    compact_kernel<<<grid_for(n), kThreads, 0, s>>>(flags, pos, n, p_rows);
    CK_LAUNCH();
    rz_packed = vec(size_t(n_prows) + 1, false);
  }
  T* rz_packed = nullptr;  // P's row norms of the nonempty rows, packed for the ordered mean
  // the A / A^T row norms of the current values: computed here in the first
  // pass, afterwards by the previous pass's fused scaling visit
  bool rz_norms_fresh = false;
  // rz_act[p]: pass p runs (device flags; the unsharded setup enqueues every
  // pass without a host synchronisation and k_ruiz_delta decides the next);
  // rz_dev[p]: pass p's deviation
  uint32_t* rz_act = nullptr;
  T* rz_dev = nullptr;
  const uint32_t* act_of(int pass) const { return pass < 0 ? nullptr : rz_act + pass; }
  void ruiz_norms(int pass = -1) {
    const uint32_t* act = act_of(pass);
    row_inf_norms(D.P, D.pP, rz_pn, s, act);
    if (D.m == 0 || D.AT.nnz == 0)  // empty block: no column contributes
      CK(cudaMemsetAsync(rz_atn, 0, sizeof(T) * D.n, s));
    else if (!rz_norms_fresh)  // (first pass: the scaled copies are not written yet)
      row_inf_norms(D.ATo, D.pAT, rz_atn, s, act);
    if (!rz_norms_fresh) row_inf_norms(D.Ao, D.pA, rz_an, s, act);
  }
  void ruiz_delta(int pass = -1) {
    const uint32_t n = D.n, m = D.m;
    const bool dev_loop = pass >= 0;
    k_ruiz_delta<T><<<red_grid<T>(std::max(n, m)), kThreads, 0, s>>>(
        rz_pn, rz_atn, n, rz_an, m, rz_dx, rz_dz, D.d, D.e, D.q, D.red, &D.ctl->red_counter,
        dev_loop ? rz_dev + pass : ruiz_scal + 4, act_of(pass),
        dev_loop ? rz_act + pass + 1 : nullptr,
        dev_loop && uint32_t(pass + 1) < set.equil_max_passes ? 1u : 0u, T(set.eps_equil));
    CK_LAUNCH();
  }
  // The cost scaling (the sequential mean of P's row norms, |q|, gamma, P and
  // q *= gamma) only depends on P and q: it runs on a side stream while the
  // main stream scales A and A^T (the mean is a latency-bound dependent chain).
  cudaStream_t s_side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void ruiz_scale(int pass = -1) {
    const uint32_t n = D.n;
    const uint32_t* act = act_of(pass);
    if (!s_side) {
      // high priority: the side stream's one-block sequential mean must get an
      // SM as soon as one frees up, not after the main stream's full-grid
      // scaling visits (it is a ~0.5 ms dependent chain at config 2)
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CK(cudaStreamCreateWithPriority(&s_side, cudaStreamNonBlocking, hi));
      CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    plan_visit(D.P, D.pP, ScaleRowColFn<T>{D.P.val, D.P.ci, rz_dx, rz_dx}, s, act);
    row_inf_norms(D.P, D.pP, rz_pn, s, act);
    static const bool serial = [] {
      const char* e = std::getenv("QPCG_RUIZ_SERIAL");
      return e && e[0] == '1';
    }();
    cudaStream_t s_side = serial ? s : this->s_side;
    CK(cudaEventRecord(ev_fork, s));
    CK(cudaStreamWaitEvent(s_side, ev_fork, 0));
    // cost scaling (scaling.hpp:156-162), side stream
    T* mean = ruiz_scal + 0;
    T* qinf = ruiz_scal + 1;
    T* gamma = ruiz_scal + 2;
    T* cc = ruiz_scal + 3;
    if (n_prows) {
      pack_list_kernel<T><<<grid_for(n_prows), kThreads, 0, s_side>>>(rz_pn, p_rows, n_prows,
                                                                      rz_packed, act);
      CK_LAUNCH();
    }
    ordered_mean_kernel<T><<<1, 256, 0, s_side>>>(rz_packed, nullptr, n_prows, n, mean, act);
    CK_LAUNCH();
    k_infnorm<T><<<red_grid<T>(n), kThreads, 0, s_side>>>(D.q, n, D.red, &D.ctl->red_counter, qinf,
                                                          act);
    CK_LAUNCH();
    k_ruiz_gamma<T><<<1, 1, 0, s_side>>>(mean, qinf, gamma, cc, act);
    CK_LAUNCH();
    k_scale_by<T><<<grid_for(D.P.nnz), kThreads, 0, s_side>>>(D.P.val, D.P.nnz, gamma, act);
    k_scale_by<T><<<grid_for(n), kThreads, 0, s_side>>>(D.q, n, gamma, act);
    CK_LAUNCH();
    CK(cudaEventRecord(ev_join, s_side));
    // main stream meanwhile: A rows (dz) then cols (dx); A^T rows (dx) then cols (dz)
    // (+ the row norms of the scaled values for the next pass)
    // first pass: read the originals, write the scaled copies
    scale_and_norms(D.A, D.pA, rz_norms_fresh ? D.A.val : D.Ao.val, rz_dz, rz_dx, rz_an, s, act);
    scale_and_norms(D.AT, D.pAT, rz_norms_fresh ? D.AT.val : D.ATo.val, rz_dx, rz_dz, rz_atn, s,
                    act);
    rz_norms_fresh = true;
    CK(cudaStreamWaitEvent(s, ev_join, 0));
  }

  // scaling.hpp:166-176 (A^T re-derived from the scaled A, reciprocals, l, u),
  // q_inf_scaled, diag(P)
  void finish_scaling(uint32_t passes, T deviation) {
    const uint32_t n = D.n, m = D.m;
    equil_passes = passes;
    equil_residual = deviation;
    if (set.scaling_enabled) gather_windowed(D.A.val, permA, D.AT.rp, D.A.nnz, winA, D.AT.val, s);
    winA.release();  // (the transpose permutation's last use)
    {
      T *d = D.d, *e = D.e, *di = D.d_inv, *ei = D.e_inv, *lo = D.l_o, *uo = D.u_o, *ls = D.l,
        *us = D.u;
      for_n(n, [=] __device__(uint32_t i) { di[i] = T(1) / d[i]; }, s);
      for_n(m, [=] __device__(uint32_t j) {
        ei[j] = T(1) / e[j];
        ls[j] = e[j] * lo[j];
        us[j] = e[j] * uo[j];
      }, s);
    }
    if (!set.scaling_enabled) {  // identity_scaled_problem (scaling.hpp:190-205): l, u copied
      CK(cudaMemcpyAsync(D.l, D.l_o, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(D.u, D.u_o, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
    }
    // q_inf_scaled (solver.hpp:407)
    k_infnorm<T><<<red_grid<T>(n), kThreads, 0, s>>>(D.q, n, D.red, &D.ctl->red_counter,
                                                      ruiz_scal + 6);
    CK_LAUNCH();
    // ---- operator caches + Jacobi (linsys.hpp:59-60, 137-148)
    D.diag_p = vec(n, false);
    D.diag_ata = vec(n, false);
    D.dinv = vec(n, false);
    extract_diag_kernel<T><<<grid_for(n), kThreads, 0, s>>>(D.P, D.diag_p);
    CK_LAUNCH();
  }

  // state and workspace vectors, the control block, the Jacobi diagonal
  void finish_setup() {
    const uint32_t n = D.n, m = D.m;
    D.x = vec(n); D.xt = vec(n); D.dx = vec(n); D.b = vec(n); D.r = vec(n); D.p = vec(n);
    D.kp = vec(n); D.best = vec(n); D.px = vec(n); D.aty = vec(n); D.rdual = vec(n);
    D.xo = vec(n); D.pxo = vec(n);
    D.z = vec(m); D.y = vec(m); D.zt = vec(m); D.dy = vec(m); D.t = vec(m); D.ax = vec(m);
    D.zo = vec(m); D.yo = vec(m); D.ap = vec(m);
    if (!D.split) {  // the carried w (the row-sharded rhs pass keeps its two columns)
      D.atp = vec(n);
      D.w = vec(n);
      D.g1m = vec(m);
    }
    D.cert = vec(std::max(n, m));
    D.g2m = alloc<pair_t<T>>(m);
    D.g2n = alloc<pair_t<T>>(n);
    if (D.split) {
      D.part = vec(2 * size_t(n));
      D.shsc = vec(kShScal);
    }
    const uint32_t cap = opt.record_diagnostics ? set.max_admm_iter : 0u;
    D.calls = alloc<DiagRec<T>>(cap);
    D.checks = alloc<uint32_t>(cap);
    D.rhos = alloc<RhoRec<T>>(cap);
    // ---- control block
    T hs[8];
    CK(cudaMemcpyAsync(hs, ruiz_scal, sizeof(T) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const qpcg_settings& st = set;
    std::memset(&hc, 0, sizeof(hc));
    hc.alpha = T(st.alpha);
    hc.sigma = T(st.sigma);
    hc.eps_abs = T(st.eps_abs);
    hc.eps_rel = T(st.eps_rel);
    hc.eps_pinf = T(st.eps_pinf);
    hc.eps_dinf = T(st.eps_dinf);
    hc.lambda = T(st.lambda_pcg);
    hc.eps_min = T(st.eps_pcg_min);
    hc.max_iter = st.max_admm_iter;
    hc.check_interval = st.check_interval;
    hc.rho_interval = st.rho_update_interval;
    hc.pcg_cap = pcg_cap(n);
    const T c = hs[3];
    hc.c = c;
    hc.c_inv = T(1) / c;
    hc.q_inf_orig = hs[5];
    hc.q_inf_scaled = hs[6];
    hc.rho = T(st.rho_bar_init);
    hc.status = QPCG_STATUS_MAX_ITER_REACHED;
    hc.diag_cap = cap;
    hc.zt_recur = zt_recur_enabled();
    hc.w_recur = hc.zt_recur && !D.split;
    {  // break-even PCG count: one A pass vs (3 m-vector accesses + ~8 MB of
       // tail latency at the HBM rate) per carried iteration
      const double pass = plan_stream_bytes(D.A, D.pA) + double(n) * sizeof(T);
      const double per_it = 3.0 * double(m) * sizeof(T) + 8e6;
      hc.zt_kmax = uint32_t(std::min(pass / per_it, 1e9));
      if (const char* e = std::getenv("QPCG_ZT_KMAX"))  // (tests: force the carry on small problems)
        hc.zt_kmax = uint32_t(std::strtoul(e, nullptr, 10));
    }
    push_ctl();
    k_precond<T><<<grid_for(n), kThreads, 0, s>>>(D, 1);
    CK_LAUNCH();
  }

  static uint32_t pcg_cap(uint32_t n) {  // solver.hpp:330-334, evaluated in T
    const uint32_t by_dim = (uint32_t)std::ceil(T(20) * std::sqrt(static_cast<T>(n)));
    return std::max<uint32_t>(20, std::min<uint32_t>(by_dim, n));
  }

  static void validate_settings(const qpcg_settings& s) {  // settings.hpp:44-75 in T
    auto bad = [](const char* m) { throw InvalidArgument(m); };
    const T alpha = T(s.alpha);
    if (!(alpha > T(0)) || !(alpha < T(2))) bad("settings: alpha must be in (0, 2)");
    if (!(T(s.sigma) > T(0))) bad("settings: sigma must be positive");
    if (!(T(s.rho_bar_init) > T(0))) bad("settings: rho_bar_init must be positive");
    if (T(s.eps_abs) < T(0) || T(s.eps_rel) < T(0)) bad("settings: tolerances must be >= 0");
    if (!(T(s.eps_pinf) > T(0)) || !(T(s.eps_dinf) > T(0)))
      bad("settings: infeasibility tolerances must be positive");
    if (s.max_admm_iter < 1 || s.check_interval < 1 || s.rho_update_interval < 1)
      bad("settings: iteration counts must be >= 1");
    if (!(T(s.lambda_pcg) > T(0)) || !(T(s.lambda_pcg) < T(1)))
      bad("settings: lambda_pcg must be in (0, 1)");
    if (!(T(s.eps_pcg_min) > T(0))) bad("settings: eps_pcg_min must be positive");
    if (!(T(s.eps_equil) > T(0)) || s.equil_max_passes < 1)
      bad("settings: bad equilibration parameters");
  }

  // ------------------------------------------------ one-pass operator apply
  // (gram.cuh): K p with A streamed once; built at the end of setup when A
  // has a dense column window, else the two-pass SpMV path runs.
  GramDev<T> gram{};
  bool gram_on = false;
  size_t gram_smem = 0;
  uint32_t gram_threads = 0;
  DevCsr<T> atLo{}, atHi{};  // row-range views of A^T outside the window
  SpmvPlan<T> gLo{}, gHi{};
  uint32_t gram_hi0 = 0;
  uint64_t gram_nnz_g = 0;  // padded in-window entries of the row-pass rows
  uint32_t gram_nnz_out = 0, gram_ng = 0, gram_nthin = 0, gram_thin_nnz = 0;
  static constexpr size_t kGramSmemBudget = 225u << 10;

  void enq_gram_kernel_only() {
    k_gram<T><<<gram.G, gram_threads, gram_smem, s>>>(D, gram);
    CK_LAUNCH();
  }
  void enq_gram() {
    enq_gram_kernel_only();
    if (gram.n_trows) {
      k_gram_thin<T><<<grid_for(gram.n_trows), kThreads, 0, s>>>(D, gram);
      CK_LAUNCH();
    }
    k_gram_reduce<T><<<ceil_div(gram.W, 32u), 32 * kGramRedGroups, 0, s>>>(D, gram);
    CK_LAUNCH();
    if (gLo.grid())
      launch_spmv<T, 1, SumOp>(atLo, gLo, GatherVec<T>{D.t}, EpiKpOff<T>{D, T(0), 0u}, s);
    if (gHi.grid())
      launch_spmv<T, 1, SumOp>(atHi, gHi, GatherVec<T>{D.t}, EpiKpOff<T>{D, T(0), gram_hi0}, s);
  }

  void build_gram() {
    // opt-in (QPCG_GRAM=1): measured slower than the two-pass SpMV on B200 at
    // every eligible BASELINE config (profiles/r02_gram_experiment.txt)
    const char* env = std::getenv("QPCG_GRAM");
    const bool force = env && env[0] == '1';
    if (!force || D.split || D.A.nnz == 0 || D.n == 0 || D.m == 0) return;
    const uint32_t n = D.n, m = D.m, nnz = D.A.nnz;
    // the dense column window from the column counts (A^T's row_ptr): the
    // smallest range holding every column with >= min(512, max count / 4)
    // entries (a column with fewer is cheaper through the A^T stream than as
    // G partial slots)
    std::vector<uint32_t> rp(size_t(n) + 1);
    CK(cudaMemcpyAsync(rp.data(), D.AT.rp, sizeof(uint32_t) * (size_t(n) + 1),
                       cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint32_t maxcnt = 0;
    for (uint32_t c = 0; c < n; ++c) maxcnt = std::max(maxcnt, rp[c + 1] - rp[c]);
    const uint32_t thr = std::min(512u, std::max(2u, maxcnt / 4));
    uint32_t a = n, b = 0;
    for (uint32_t c = 0; c < n; ++c)
      if (rp[c + 1] - rp[c] >= thr) {
        a = std::min(a, c);
        b = c;
      }
    if (a == n) return;
    const uint32_t W = b - a + 1;
    // shared memory: p's window and the accumulator (W each) + the ring
    const size_t acc_bytes = 2 * size_t((W + 15u) & ~15u) * sizeof(T);
    if (W > 65536u || acc_bytes > kGramSmemBudget * 3 / 4) return;
    if (!force && double(rp[b + 1] - rp[a]) < 0.75 * double(nnz)) return;
    // per row: entries inside / outside the window
    uint32_t *cin, *cout, *rp_out, *isg, *pos;
    unsigned int* mx;
    CK(dmalloc(&cin, sizeof(uint32_t) * (size_t(m) + 1)));
    CK(dmalloc(&cout, sizeof(uint32_t) * (size_t(m) + 1)));
    CK(dmalloc(&isg, sizeof(uint32_t) * (size_t(m) + 1)));
    CK(dmalloc(&pos, sizeof(uint32_t) * (size_t(m) + 1)));
    CK(dmalloc(&mx, sizeof(unsigned int)));
    auto release = [&] {
      for (void* q : {(void*)cin, (void*)cout, (void*)isg, (void*)pos, (void*)mx}) CK(dfree(q));
    };
    rp_out = alloc<uint32_t>(size_t(m) + 1);
    CK(cudaMemsetAsync(cout + m, 0, sizeof(uint32_t), s));
    CK(cudaMemsetAsync(mx, 0, sizeof(unsigned int), s));
    gram_count_kernel<<<grid_for(uint64_t(m) * 32), kThreads, 0, s>>>(D.A.rp, D.A.ci, m, a, W, cin,
                                                                      cout, mx);
    CK_LAUNCH();
    exclusive_scan_u32(cout, rp_out, m + 1, tmp, s);
    // the row-pass rows (>= kGramThin in-window entries) and the thin rows
    gram_isg_kernel<<<grid_for(uint64_t(m) + 1), kThreads, 0, s>>>(cin, m, isg);
    CK_LAUNCH();
    exclusive_scan_u32(isg, pos, m + 1, tmp, s);
    uint32_t h[3];
    CK(cudaMemcpyAsync(h, pos + m, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h + 1, rp_out + m, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h + 2, mx, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint32_t ng = h[0];
    gram_nnz_out = h[1];
    const uint32_t slot_len = (h[2] + 7u) & ~7u;  // the longest row, padded
    if (ng == 0 || h[2] > kGramMaxRowLen) {
      release();
      return;
    }
    // shared memory: the window accumulator + NS ring slots; NS - 2 consumers
    const size_t slot_bytes = size_t(slot_len) * (sizeof(T) + sizeof(uint16_t));
    const uint32_t NS = uint32_t(
        std::min<size_t>(16, (kGramSmemBudget - acc_bytes - 256) / slot_bytes));
    if (NS < 3) {
      release();
      return;
    }
    gram.NS = NS;
    gram.slot_len = slot_len;
    gram.C = std::min<uint32_t>(8, NS - 1);
    gram_threads = 32 * (1 + gram.C);
    gram_smem = acc_bytes + size_t(NS) * slot_bytes + 2 * NS * sizeof(uint64_t);
    uint32_t* grows = alloc<uint32_t>(size_t(ng) + 1);
    uint32_t* trows = alloc<uint32_t>(size_t(m - ng) + 1);
    uint8_t* thin = alloc<uint8_t>(size_t(m) + 1);
    gram_split_kernel<<<grid_for(m), kThreads, 0, s>>>(cin, pos, m, grows, trows, thin);
    CK_LAUNCH();
    // padded storage of the row-pass rows' in-window entries
    uint32_t* glen = alloc<uint32_t>(size_t(ng) + 1);
    uint32_t* gstart = alloc<uint32_t>(size_t(ng) + 1);
    gram_plen_kernel<<<grid_for(uint64_t(ng) + 1), kThreads, 0, s>>>(grows, ng, cin, isg, glen);
    CK_LAUNCH();
    exclusive_scan_u32(isg, gstart, ng + 1, tmp, s);
    uint32_t tot_g = 0;
    CK(cudaMemcpyAsync(&tot_g, gstart + ng, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    gram_nnz_g = tot_g;
    uint32_t* din = pos;  // (pos is no longer needed)
    CK(cudaMemsetAsync(din, 0xff, sizeof(uint32_t) * m, s));
    gram_din_kernel<<<grid_for(ng), kThreads, 0, s>>>(grows, ng, gstart, din);
    CK_LAUNCH();
    uint16_t* off_g = alloc<uint16_t>(size_t(tot_g) + 8);
    T* val_g = alloc<T>(size_t(tot_g) + 8);
    CK(cudaMemsetAsync(off_g, 0, sizeof(uint16_t) * (size_t(tot_g) + 8), s));
    CK(cudaMemsetAsync(val_g, 0, sizeof(T) * (size_t(tot_g) + 8), s));
    uint32_t* col_out = alloc<uint32_t>(size_t(gram_nnz_out) + 1);
    T* val_out = alloc<T>(size_t(gram_nnz_out) + 1);
    gram_fill_kernel<T><<<grid_for(uint64_t(m) * 32), kThreads, 0, s>>>(
        D.A.rp, D.A.ci, D.A.val, m, a, W, din, rp_out, off_g, val_g, col_out, val_out);
    CK_LAUNCH();
    // cost-balanced CTA ranges over the row-pass rows
    gram_weight_kernel<<<grid_for(uint64_t(ng) + 1), kThreads, 0, s>>>(grows, ng, cin, cout, isg);
    CK_LAUNCH();
    uint32_t* wpre = alloc<uint32_t>(size_t(ng) + 1);
    exclusive_scan_u32(isg, wpre, ng + 1, tmp, s);
    // A_thin^T over the window columns
    uint32_t* tcnt = cin;  // (cin is no longer needed: W + 1 <= m + 1 is not guaranteed)
    if (W + 1 > m + 1) CK(dmalloc(&tcnt, sizeof(uint32_t) * (size_t(W) + 1)));
    CK(cudaMemsetAsync(tcnt + W, 0, 4, s));
    gram_thin_t_kernel<T><<<grid_for(uint64_t(W) * 32), kThreads, 0, s>>>(
        D.AT.rp, D.AT.ci, D.AT.val, a, W, thin, tcnt, nullptr, nullptr, nullptr, 0);
    CK_LAUNCH();
    uint32_t* rp_thin = alloc<uint32_t>(size_t(W) + 1);
    exclusive_scan_u32(tcnt, rp_thin, W + 1, tmp, s);
    uint32_t nthin = 0, wtot = 0;
    CK(cudaMemcpyAsync(&nthin, rp_thin + W, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&wtot, wpre + ng, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (tcnt != cin) CK(dfree(tcnt));
    gram_nthin = nthin;
    gram_thin_nnz = nnz - (wtot - kGramRowCost * ng);  // entries of the thin rows
    uint32_t* col_thin = alloc<uint32_t>(size_t(nthin) + 1);
    T* val_thin = alloc<T>(size_t(nthin) + 1);
    gram_thin_t_kernel<T><<<grid_for(uint64_t(W) * 32), kThreads, 0, s>>>(
        D.AT.rp, D.AT.ci, D.AT.val, a, W, thin, nullptr, rp_thin, col_thin, val_thin, 1);
    CK_LAUNCH();
    release();
    // grid: as many CTAs as fit
    int sms = 0, nb = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaFuncSetAttribute(k_gram<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gram_smem)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_gram<T>, int(gram_threads), gram_smem));
    if (nb <= 0) return;
    gram.G = std::min<uint32_t>(uint32_t(sms) * uint32_t(nb), ng);
    uint32_t* cut = alloc<uint32_t>(size_t(gram.G) + 1);
    gram_cut_kernel<<<ceil_div(gram.G + 1, 256u), 256, 0, s>>>(wpre, ng, gram.G, cut);
    CK_LAUNCH();
    gram.w0 = a;
    gram.W = W;
    gram.cut = cut;
    gram.rows = grows;
    gram.gstart = gstart;
    gram.glen = glen;
    gram.off_g = off_g;
    gram.val_g = val_g;
    gram.trows = trows;
    gram.n_trows = m - ng;
    gram.rp_thin = rp_thin;
    gram.col_thin = col_thin;
    gram.val_thin = val_thin;
    gram.rp_out = rp_out;
    gram.col_out = col_out;
    gram.val_out = val_out;
    gram.part = alloc<T>(size_t(gram.G) * W);
    gram_ng = ng;
    if (const char* dg = std::getenv("QPCG_GRAM_DEBUG")) gram.dbg = uint32_t(std::atoi(dg));
    // A^T rows outside the window: [0, a) and [b + 1, n)
    if (a > 0) {
      atLo = D.AT;
      atLo.rows = a;
      gLo = plan_build<T>(atLo.rp, a, rp[a], tmp, s);
    }
    if (b + 1 < n) {
      atHi = D.AT;
      atHi.rp = D.AT.rp + (b + 1);
      atHi.rows = n - (b + 1);
      gram_hi0 = b + 1;
      gHi = plan_build<T>(atHi.rp, n - (b + 1), rp[n] - rp[b + 1], tmp, s);
    }
    gram_on = true;
    hc.zt_recur = 0;  // the one-pass apply forms A p inside the Gram product, not kept
    hc.w_recur = 0;
    push_ctl();
    if (const char* tr = std::getenv("QPCG_GRAM_TRACE"); tr && tr[0] == '1')
      std::fprintf(stderr,
                   "[gram] window [%u, %u) W=%u, row-pass rows %u (max %u entries, slot %u), thin "
                   "rows %u (A_thin^T %u), out-of-window entries %u; ring %u slots, %u consumer "
                   "warps, smem %zu B, G=%u (%d per SM)\n",
                   a, b + 1, W, ng, h[2], slot_len, m - ng, nthin, gram_nnz_out, NS, gram.C,
                   gram_smem, gram.G, nb);
  }
  // bytes one operator apply streams on the one-pass path (k_gram + reduce +
  // the out-of-window A^T rows; P, p and the vectors as in §8(d))
  double gram_stream_bytes() const {
    const double S = sizeof(T), m = D.m;
    // row pass (padded in-window entries, out-of-window entries, the row
    // descriptors), t, the partial windows written and read, the thin rows'
    // entries (k_gram_thin) and A_thin^T
    double b = double(gram_nnz_g) * (S + 2) + double(gram_nnz_out) * (S + 4) +
               8.0 * (double(gram_ng) + 1) + 8.0 * (m + 1) + S * m +
               2.0 * S * double(gram.G) * gram.W + double(gram_thin_nnz) * (S + 4) +
               double(gram_nthin) * (S + 4);
    if (gLo.grid()) b += plan_stream_bytes(atLo, gLo);
    if (gHi.grid()) b += plan_stream_bytes(atHi, gHi);
    return b;
  }

  // ------------------------------------------------------ enqueue helpers
  // rhs + r0: the 2-column pass, or 1 column when r0's A^T (rho z~) is the
  // carried w (admm.cuh rhs_one; decided on the device, one launch)
  void enq_rhs(const Handles&) {
    k_pack_rhs<T><<<grid_for(D.m), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    launch_spmv_select<T, 1, GatherVec<T>, EpiRhs1<T>, 2, GatherRhs<T>, EpiRhs<T>>(
        D.AT, D.pAT, GatherVec<T>{D.g1m}, EpiRhs1<T>{D, T(0)}, GatherRhs<T>{D.g2m},
        EpiRhs<T>{D, T(0)}, s);
  }
  void enq_pcg_init(const Handles& H) {
    k_pcg_init<T><<<red_grid<T>(D.n), kThreads, 0, s>>>(D, H);
    CK_LAUNCH();
  }
  void enq_pcg_iter(const Handles& H) {
    if (gram_on) {
      enq_gram();
    } else {
      launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.p}, EpiAp<T>{D.t, D.ap, D.ctl}, s);
      launch_spmv<T, 1, SumOp>(D.AT, D.pAT, GatherVec<T>{D.t}, EpiKp<T>{D, T(0)}, s);
    }
    if (coop_pcg_ok()) {
      Dev<T> d = D;
      Handles h = H;
      void* args[] = {&d, &h};
      CK(cudaLaunchCooperativeKernel((const void*)k_pcg_step<T>, dim3(red_grid<T>(D.n)),
                                     dim3(kThreads), args, 0, s));
      CK_LAUNCH();
      return;
    }
    k_pcg_dot<T><<<red_grid<T>(D.n), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    k_pcg_update<T><<<red_grid<T>(D.n), kThreads, 0, s>>>(D, H);
    CK_LAUNCH();
    k_pcg_pupdate<T><<<grid_for(D.n), kThreads, 0, s>>>(D);
    CK_LAUNCH();
  }
  // k_pcg_step (opt-in, QPCG_COOP_PCG=1): needs cooperative launches to
  // capture into CUDA graphs on this driver (probed once per process) and a
  // co-resident grid.  Measured at config 2: 378.3 / 378.6 ms per solve with
  // the three kernels vs 379.6 / 380.2 ms fused (inside the graph the two
  // launches it saves cost ~1 us each; svm's PCG iteration 750 vs 749 us), so
  // the separate kernels stay the default; the results are identical.
  bool coop_pcg_ok() {
    static const bool env_on = [] {
      const char* e = std::getenv("QPCG_COOP_PCG");
      return e && e[0] == '1';
    }();
    if (!env_on) return false;
    if (coop_state == 0) {
      int nb = 0, sms = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg_step<T>, kThreads, 0);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
      const bool fits = uint64_t(nb) * uint64_t(sms) >= red_grid<T>(D.n);
      coop_state = (fits && coop_capture_probe()) ? 1 : 2;
    }
    return coop_state == 1;
  }
  int coop_state = 0;  // 0 unknown, 1 on, 2 off
  // z~ carried through PCG (admm.cuh zt_pass); QPCG_ZT_RECUR=0 runs the z~
  // pass after every PCG solve as the reference does
  static uint32_t zt_recur_enabled() {
    static const uint32_t on = [] {
      const char* e = std::getenv("QPCG_ZT_RECUR");
      return (e && e[0] == '0') ? 0u : 1u;
    }();
    return on;
  }
  // After PCG: k_pcg_fin, the z~ pass (skipped on the device when z~ was
  // carried, admm.cuh zt_pass; in the graph it sits in an IF node, so a
  // skipped pass launches nothing), the m-side update, the n-side update.
  void enq_post_pcg(const Handles& H) {
    enq_pcg_fin(H);
    enq_zt_pass();
    enq_post_zt(H);
  }
  void enq_pcg_fin(const Handles& H) {
    k_pcg_fin<T><<<grid_for(D.n), kThreads, 0, s>>>(D, H);
    CK_LAUNCH();
  }
  // z~ = A x~ with the m-side update: the 2-column build on check iterations
  // (col 1 = A x_new), else the 1-column one; one launch
  void enq_zt_pass() {
    if (D.pA.u8)  // short rows: the m-side update as a row-parallel pass (EpiAdmmStore)
      launch_spmv_select<T, 1, GatherVec<T>, EpiAdmmStore<T, 1>, 2, GatherAdmm<T>,
                         EpiAdmmStore<T, 2>>(D.A, D.pA, GatherVec<T>{D.xt}, EpiAdmmStore<T, 1>{D},
                                             GatherAdmm<T>{D.g2n}, EpiAdmmStore<T, 2>{D}, s);
    else
      launch_spmv_select<T, 1, GatherVec<T>, EpiAdmm<T, 1>, 2, GatherAdmm<T>, EpiAdmm<T, 2>>(
          D.A, D.pA, GatherVec<T>{D.xt}, EpiAdmm<T, 1>{D, T(0), T(0), T(0), false},
          GatherAdmm<T>{D.g2n}, EpiAdmm<T, 2>{D, T(0), T(0), T(0), false}, s);
  }
  void enq_post_zt(const Handles& H) {
    // short-row plans: always (EpiAdmmStore only stored z~); else only when
    // the z~ pass was skipped (its fused epilogue did not run)
    k_admm_mside<T><<<grid_for(D.m), kThreads, 0, s>>>(D, D.pA.u8 != 0);
    CK_LAUNCH();
    k_xupdate<T><<<grid_for(D.n), kThreads, 0, s>>>(D, H);
    CK_LAUNCH();
  }
  void enq_check(const Handles& H, int mode) {
    launch_spmv<T, 1, SumOp>(D.AT, D.pAT, GatherVec<T>{D.y}, EpiDual<T>{D}, s);
    k_residuals<T><<<red_grid<T>(std::max(D.n, D.m)), kThreads, 0, s>>>(D, mode, H);
    CK_LAUNCH();
  }
  void enq_infeas(const Handles&) {
    k_infeas_vec<T><<<red_grid<T>(std::max(D.n, D.m)), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    launch_spmv<T, 1, SumOp>(
        D.ATo, D.pATo, GatherCertY<T>{D.e, D.dy, D.ctl, T(0), T(0)},
        EpiNormMax<T>{&D.ctl->atv_inf_bits, &D.ctl->need_pinf}, s);
    launch_spmv<T, 1, SumOp>(D.Po, D.pPo, GatherCertX<T>{D.d, D.dx, D.ctl, T(0)},
                             EpiNormMax<T>{&D.ctl->pv_inf_bits, &D.ctl->need_dinf}, s);
    k_infeas_mid<T><<<1, 1, 0, s>>>(D);
    CK_LAUNCH();
    launch_spmv<T, 1, SumOp>(
        D.Ao, D.pAo, GatherCertX<T>{D.d, D.dx, D.ctl, T(0)},
        EpiDualRows<T>{D.l_o, D.u_o, &D.ctl->dinf_bad, &D.ctl->need_dinf, T(0), D.ctl}, s);
    k_infeas<T><<<1, 1, 0, s>>>(D);
    CK_LAUNCH();
  }
  void enq_rho_flag(const Handles& H) {
    k_rho_flag<T><<<1, 1, 0, s>>>(D, H);
    CK_LAUNCH();
  }
  void enq_rho(const Handles&) {
    k_rho<T><<<red_grid<T>(D.m), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    k_precond<T><<<grid_for(D.n), kThreads, 0, s>>>(D, 0);
    CK_LAUNCH();
  }
  void enq_admm_cond(const Handles& H) {
    k_admm_cond<T><<<1, 1, 0, s>>>(D, H);
    CK_LAUNCH();
  }
  // residuals at the current iterates (solver.hpp:436, :517)
  void enq_residuals_fresh(int mode) {
    launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.x}, EpiStore<T>{D.ax}, s);
    enq_check(Handles{}, mode);
  }

  // ------------------------------------------------------- graph build
  cudaGraph_t add_cond_in_capture(cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
    CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
    return cp.conditional.phGraph_out[0];
  }

  uint64_t body_kernels[6] = {};  // per execution: ADMM step, PCG iteration, check, infeas, rho, z~ pass
  void build_graph() {
    CK(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h_admm, h_pcg, h_chk, h_inf, h_rho, h_zt;
    CK(cudaGraphConditionalHandleCreate(&h_admm, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_admm;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t n_admm;
    CK(cudaGraphAddNode(&n_admm, graph, nullptr, 0, &cp));
    cudaGraph_t b_admm = cp.conditional.phGraph_out[0];
    CK(cudaGraphConditionalHandleCreate(&h_pcg, b_admm, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&h_chk, b_admm, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&h_rho, b_admm, 0, cudaGraphCondAssignDefault));
    CK(cudaGraphConditionalHandleCreate(&h_zt, b_admm, 0, cudaGraphCondAssignDefault));
    Handles H;
    H.zt = (unsigned long long)h_zt;
    H.admm = (unsigned long long)h_admm;
    H.pcg = (unsigned long long)h_pcg;
    H.chk = (unsigned long long)h_chk;
    H.rho = (unsigned long long)h_rho;
    cudaGraph_t b_pcg, b_chk, b_rho, b_inf, b_zt, g_out;
    // kernels per execution of each body, counted as they are captured
    // (the solve's launch count multiplies them by the executions)
    uint64_t c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_admm, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_rhs(H);
    enq_pcg_init(H);
    b_pcg = add_cond_in_capture(h_pcg, cudaGraphCondTypeWhile);
    enq_pcg_fin(H);
    b_zt = add_cond_in_capture(h_zt, cudaGraphCondTypeIf);
    enq_post_zt(H);
    b_chk = add_cond_in_capture(h_chk, cudaGraphCondTypeIf);
    enq_rho_flag(H);
    b_rho = add_cond_in_capture(h_rho, cudaGraphCondTypeIf);
    enq_admm_cond(H);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[0] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_pcg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_pcg_iter(H);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[1] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_zt, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_zt_pass();
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[5] = g_launches - c0;
    CK(cudaGraphConditionalHandleCreate(&h_inf, b_chk, 0, cudaGraphCondAssignDefault));
    H.inf = (unsigned long long)h_inf;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_chk, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_check(H, 0);
    b_inf = add_cond_in_capture(h_inf, cudaGraphCondTypeIf);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[2] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_inf, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_infeas(H);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[3] = g_launches - c0;
    c0 = g_launches;
    CK(cudaStreamBeginCaptureToGraph(s, b_rho, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    enq_rho(H);
    CK(cudaStreamEndCapture(s, &g_out));
    body_kernels[4] = g_launches - c0;
    CK(cudaGraphInstantiate(&exec, graph, 0));
  }

  // ------------------------------------------------- persistent loop
  // The small-problem path (persist.cuh): the whole loop in one cooperative
  // kernel.  Chosen automatically in graph mode while A fits the L2 budget.
  T* persist_part = nullptr;
  static uint64_t persist_max_nnz() {
    const char* e = std::getenv("QPCG_PERSIST_MAX_NNZ");
    return e ? std::strtoull(e, nullptr, 10) : 2000000ull;
  }
  bool use_persistent() const {
    if (D.split) return false;
    if (opt.mode == QPCG_MODE_PERSISTENT) return true;
    return opt.mode == QPCG_MODE_GRAPH && uint64_t(D.A.nnz) + D.P.nnz <= persist_max_nnz();
  }
  static uint64_t block_max_nnz() {
    const char* e = std::getenv("QPCG_BLOCK_MAX_NNZ");
    return e ? std::strtoull(e, nullptr, 10) : 1200ull;
  }
  static uint64_t cluster_max_nnz() {
    const char* e = std::getenv("QPCG_CLUSTER_MAX_NNZ");
    return e ? std::strtoull(e, nullptr, 10) : 10000ull;
  }
  void run_persistent() {
    if (!persist_part) persist_part = alloc<T>(2 * kMaxQ * kMaxVirtual);
    PersistBufs<T> B{persist_part, D.ctl};
    void* args[] = {(void*)&D, (void*)&B};
    const uint64_t work = uint64_t(D.A.nnz) + D.P.nnz;
    // largest cluster the kernel can run as (same device model); thread-safe
    // one-time probe (solve_batch runs workspaces from several threads)
    static const int cluster = [] {
      int c_ok = 0;
      auto* kc = k_admm_persistent<T, ClusterSync>;
      if (cudaFuncSetAttribute(kc, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        for (int c : {16, 8}) {
          cudaLaunchConfig_t cfg = {};
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = c;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.gridDim = dim3(c);
          cfg.blockDim = dim3(kThreads);
          cfg.attrs = at;
          cfg.numAttrs = 1;
          int nc = 0;
          if (cudaOccupancyMaxActiveClusters(&nc, kc, &cfg) == cudaSuccess && nc > 0) {
            c_ok = c;
            break;
          }
        }
      }
      cudaGetLastError();
      return c_ok;
    }();
    const int budget = std::max(0, opt.sm_budget);  // SMs this solve may hold (0: all)
    if (work <= block_max_nnz() || budget == 1) {
      // tiny problem (or a one-SM budget): one block, __syncthreads barriers,
      // matrices held in its L1
      k_admm_persistent<T, BlockSync><<<1, kThreads, 0, s>>>(D, B);
      CK_LAUNCH();
      return;
    }
    if (cluster > 0 && (work <= cluster_max_nnz() || (budget >= cluster && budget < 2 * cluster))) {
      // tiny problem: one cluster, hardware barriers
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cluster;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(cluster);
      cfg.blockDim = dim3(kThreads);
      cfg.stream = s;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      // (the attribute is per device: set it for this one too)
      CK(cudaFuncSetAttribute(k_admm_persistent<T, ClusterSync>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      CK(cudaLaunchKernelExC(&cfg, (const void*)k_admm_persistent<T, ClusterSync>, args));
      CK_LAUNCH();
      return;
    }
    // co-resident blocks (same device model; thread-safe one-time probe)
    static const int grid_per_sm = [] {
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_admm_persistent<T, GridSync>,
                                                       kThreads, 0));
      return std::max(1, per_sm);
    }();
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int max_grid = grid_per_sm * sms;
    // measured: more co-resident blocks is faster at every size; a budget
    // caps the grid (the reductions emulate a fixed geometry, so any grid
    // gives the same bits)
    const int grid = budget > 0 ? std::min(max_grid, grid_per_sm * budget) : max_grid;
    CK(cudaLaunchCooperativeKernel((const void*)k_admm_persistent<T, GridSync>, dim3(grid),
                                   dim3(kThreads), args, 0, s));
    CK_LAUNCH();
  }

  // ------------------------------------------------------- eager loop
  void run_eager() {
    Handles H{};
    // SolveDiagnostics::on_iteration (solver.hpp:451-454): the scaled
    // iterates after every ADMM step, before the check; bounds once
    std::vector<T> hx, hz, hy, hl, hu;
    if (opt.on_iteration) {
      hx.resize(D.n);
      hz.resize(D.m);
      hy.resize(D.m);
      hl.resize(D.m);
      hu.resize(D.m);
      if (D.m) {
        CK(cudaMemcpyAsync(hl.data(), D.l, sizeof(T) * D.m, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hu.data(), D.u, sizeof(T) * D.m, cudaMemcpyDeviceToHost, s));
      }
    }
    for (;;) {
      pull_ctl();
      if (hc.done || hc.error || hc.iter >= hc.max_iter) break;
      enq_rhs(H);
      enq_pcg_init(H);
      pull_ctl();
      while (hc.pcg_active && !hc.error) {
        enq_pcg_iter(H);
        pull_ctl();
      }
      enq_post_pcg(H);
      pull_ctl();
      if (opt.on_iteration && !hc.error) {
        CK(cudaMemcpyAsync(hx.data(), D.x, sizeof(T) * D.n, cudaMemcpyDeviceToHost, s));
        if (D.m) {
          CK(cudaMemcpyAsync(hz.data(), D.z, sizeof(T) * D.m, cudaMemcpyDeviceToHost, s));
          CK(cudaMemcpyAsync(hy.data(), D.y, sizeof(T) * D.m, cudaMemcpyDeviceToHost, s));
        }
        CK(cudaStreamSynchronize(s));
        opt.on_iteration(opt.on_iteration_user, hc.iter, hx.data(), hz.data(), hy.data(),
                         hl.data(), hu.data(), D.n, D.m);
      }
      if (hc.is_check && !hc.error) {
        enq_check(H, 0);
        pull_ctl();
        if (hc.inf_branch) enq_infeas(H);
      }
      enq_rho_flag(H);
      enq_rho(H);
    }
  }

  // ------------------------------------------------------------ solve
  // reset the per-solve state (solver.hpp:412, :430-443)
  void reset_solve_state() {
    pull_ctl();
    hc.iter = 0;
    hc.done = 0;
    hc.error = 0;
    hc.status = QPCG_STATUS_MAX_ITER_REACHED;
    hc.pcg_total = 0;
    hc.rho_update_count = 0;
    hc.n_calls = hc.n_checks = hc.n_rho = 0;
    hc.pcg_active = 0;
    hc.red_counter = 0;
    hc.n_inf = 0;
    hc.n_rho_branch = 0;
    hc.n_zt = 0;
    hc.k_last = 0;  // the first PCG solve carries z~ (a fresh workspace's state)
    hc.w_valid = 0;  // and the first rhs pass forms both columns
    push_ctl();
  }
  void raise_device_error() {
    if (hc.error == kErrNotPD)
      throw NotPositiveDefinite("pcg: encountered direction of nonpositive curvature");
    if (hc.error == kErrRho) throw InvalidArgument("kkt operator: rho must be positive");
    if (hc.error == kErrInvalid) throw InvalidArgument("pcg: warm start must be finite");
  }
  void fill_info(qpcg_info* info, double solve_s, double d2h, uint32_t n, uint32_t m) const {
    const bool has_cert = hc.status == 1 || hc.status == 2;
    std::memset(info, 0, sizeof(*info));
    info->status = int32_t(hc.status);
    info->iterations = hc.iter;
    info->pcg_iterations_total = hc.pcg_total;
    info->objective = double(hc.objective);
    info->r_prim_inf = double(hc.rp_o);
    info->r_dual_inf = double(hc.rd_o);
    info->equil_passes = equil_passes;
    info->rho_update_count = hc.rho_update_count;
    info->equil_residual = double(equil_residual);
    info->rho_final = double(hc.rho);
    info->certificate_valid = has_cert;
    info->n = n;
    info->m = m;
    info->engine_flags = (gram_on ? QPCG_ENGINE_ONE_PASS_OPERATOR : 0u) |
                         (ran_persistent ? QPCG_ENGINE_PERSISTENT : 0u) |
                         (hc.zt_recur ? QPCG_ENGINE_CARRIED_PRODUCTS : 0u);
    info->setup_seconds = setup_seconds;
    info->solve_seconds = solve_s;
    info->h2d_seconds = h2d_seconds;
    info->d2h_seconds = opt.input_memory == QPCG_MEM_HOST ? d2h : 0.0;
    info->h2d_bytes = h2d_bytes;
    info->d2h_bytes = opt.input_memory == QPCG_MEM_HOST
                          ? sizeof(T) * (uint64_t(n) + 2ull * m) +
                                (has_cert ? sizeof(T) * (hc.status == 1 ? m : n) : 0)
                          : 0;
  }

  void solve(qpcg_info* info, T* x, T* z, T* y, T* cert) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    const double w0 = now_s();
    CK(cudaEventRecord(ev0, s));
    reset_solve_state();
    uint64_t graph_build = 0;
    const uint64_t l0 = g_launches;
    // initial residuals and PCG tolerance (solver.hpp:436-441)
    enq_residuals_fresh(1);
    if (opt.mode == QPCG_MODE_EAGER || opt.on_iteration) {
      run_eager();
    } else if (use_persistent()) {
      ran_persistent = true;
      run_persistent();
    } else {
      if (!exec) {
        const uint64_t b0 = g_launches;
        build_graph();
        graph_build = g_launches - b0;
      }
      CK(cudaGraphLaunch(exec, s));
    }
    pull_ctl();
    raise_device_error();
    if (!hc.residuals_current) enq_residuals_fresh(2);
    k_unscale<T><<<grid_for(std::max(D.n, D.m)), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    if (hc.status != 1 && hc.status != 2)
      launch_spmv<T, 1, SumOp>(D.Po, D.pPo, GatherVec<T>{D.xo}, EpiStore<T>{D.pxo}, s);
    k_objective<T><<<red_grid<T>(D.n), kThreads, 0, s>>>(D);
    CK_LAUNCH();
    CK(cudaEventRecord(ev1, s));
    pull_ctl();
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, ev0, ev1));
    const double td = now_s();
    download(x, D.xo, sizeof(T) * D.n);
    download(z, D.zo, sizeof(T) * D.m);
    download(y, D.yo, sizeof(T) * D.m);
    const bool has_cert = hc.status == 1 || hc.status == 2;
    uint64_t launches = g_launches - l0 - graph_build;
    if (opt.mode != QPCG_MODE_EAGER && !use_persistent())  // kernels executed inside the graph
      launches += body_kernels[0] * hc.iter + body_kernels[1] * hc.pcg_total +
                  body_kernels[2] * hc.n_checks + body_kernels[3] * hc.n_inf +
                  body_kernels[4] * hc.n_rho_branch + body_kernels[5] * hc.n_zt;
    if (has_cert) download(cert, D.cert, sizeof(T) * (hc.status == 1 ? D.m : D.n));
    CK(cudaStreamSynchronize(s));
    const double d2h = now_s() - td;
    have_solved = true;
    if (info) {
      fill_info(info, ms * 1e-3, d2h, D.n, D.m);
      info->runtime_seconds = now_s() - w0;
      info->kernel_launches = launches + (have_counted_setup ? 0 : setup_launches);
    }
    have_counted_setup = true;
  }

  // ------------------------------------------------- OSQP-style updates
  void warm_start(const T* x, const T* z, const T* y) override {  // solver.hpp:413-428
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    if (warm_stage(x, z, y) != ~0ull) throw InvalidArgument("solve: warm start must be finite");
    warm_apply();
  }
  // upload + finiteness key (~0 = all finite); the sharded path combines the
  // keys of its row blocks before anyone throws
  T *w_tx = nullptr, *w_tz = nullptr, *w_ty = nullptr;
  unsigned long long warm_stage(const T* x, const T* z, const T* y) {
    const uint32_t n = D.n, m = D.m;
    w_tx = vec(n, false);
    w_tz = vec(m, false);
    w_ty = vec(m, false);
    upload(w_tx, x, sizeof(T) * n);
    upload(w_tz, z, sizeof(T) * m);
    upload(w_ty, y, sizeof(T) * m);
    unsigned long long* key = alloc<unsigned long long>(1);
    CK(cudaMemsetAsync(key, 0xff, 8, s));
    validate_values_kernel<T><<<grid_for(n), kThreads, 0, s>>>(w_tx, n, 1, key);
    validate_values_kernel<T><<<grid_for(m), kThreads, 0, s>>>(w_tz, m, 1, key);
    validate_values_kernel<T><<<grid_for(m), kThreads, 0, s>>>(w_ty, m, 1, key);
    CK_LAUNCH();
    unsigned long long k;
    CK(cudaMemcpyAsync(&k, key, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return k;
  }
  void warm_apply() {
    const uint32_t n = D.n, m = D.m;
    const T c = hc.c;
    T *X = D.x, *XT = D.xt, *Z = D.z, *Y = D.y, *di = D.d_inv, *e = D.e, *ei = D.e_inv;
    const T *tx = w_tx, *tz = w_tz, *ty = w_ty;
    for_n(n, [=] __device__(uint32_t i) {
      const T v = di[i] * tx[i];
      X[i] = v;
      XT[i] = v;
    }, s);
    for_n(m, [=] __device__(uint32_t j) {
      Z[j] = e[j] * tz[j];
      Y[j] = (ei[j] * ty[j]) * c;
    }, s);
    // keep the invariant zt == A x~ used by the fused r0 (pcg_warm = x)
    launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.xt}, EpiStore<T>{D.zt}, s);
    CK(cudaStreamSynchronize(s));
  }

  void update_rho(T rho) override {  // linsys.hpp:153-157
    if (!(rho > T(0))) throw InvalidArgument("kkt operator: rho must be positive");
    CK(cudaSetDevice(device));
    pull_ctl();
    hc.rho = rho;
    hc.w_valid = 0;
    push_ctl();
    k_precond<T><<<grid_for(D.n), kThreads, 0, s>>>(D, 1);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
  }

  // ----------------------------------------------------- debug / bench
  void debug_scaled(T* pv, uint32_t* prp, uint32_t* pci, T* q, T* av, T* atv, uint32_t* atrp,
                    uint32_t* atci, T* l, T* u, T* d, T* e, double* scal) override {
    CK(cudaSetDevice(device));
    auto dl = [&](void* dst, const void* src, size_t b) {
      if (dst) CK(cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, s));
    };
    dl(pv, D.P.val, sizeof(T) * D.P.nnz);
    dl(prp, D.P.rp, 4 * (size_t(D.n) + 1));
    dl(pci, D.P.ci, 4 * size_t(D.P.nnz));
    dl(q, D.q, sizeof(T) * D.n);
    dl(av, D.A.val, sizeof(T) * D.A.nnz);
    dl(atv, D.AT.val, sizeof(T) * D.AT.nnz);
    dl(atrp, D.AT.rp, 4 * (size_t(D.n) + 1));
    dl(atci, D.AT.ci, 4 * size_t(D.AT.nnz));
    dl(l, D.l, sizeof(T) * D.m);
    dl(u, D.u, sizeof(T) * D.m);
    dl(d, D.d, sizeof(T) * D.n);
    dl(e, D.e, sizeof(T) * D.m);
    CK(cudaStreamSynchronize(s));
    if (scal) {
      scal[0] = double(hc.c);
      scal[1] = double(hc.c_inv);
      scal[2] = double(equil_passes);
      scal[3] = double(equil_residual);
    }
  }

  void debug_operator(const T* x, T* kx, T* dinv) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    pull_ctl();
    const Ctl<T> saved = hc;
    hc.pcg_active = 1;
    hc.error = 0;
    push_ctl();
    CK(cudaMemcpyAsync(D.p, x, sizeof(T) * D.n, cudaMemcpyHostToDevice, s));
    launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.p}, EpiAp<T>{D.t, D.ap, D.ctl}, s);
    launch_spmv<T, 1, SumOp>(D.AT, D.pAT, GatherVec<T>{D.t}, EpiKp<T>{D, T(0)}, s);
    if (kx) CK(cudaMemcpyAsync(kx, D.kp, sizeof(T) * D.n, cudaMemcpyDeviceToHost, s));
    if (dinv) CK(cudaMemcpyAsync(dinv, D.dinv, sizeof(T) * D.n, cudaMemcpyDeviceToHost, s));
    hc = saved;
    push_ctl();
    CK(cudaStreamSynchronize(s));
  }

  // CUDA-event timing of the PCG-iteration kernels (bench.py roofline)
  void bench_kernels(uint32_t reps, double* out) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    pull_ctl();
    const Ctl<T> saved = hc;
    Ctl<T> run = hc;
    run.pcg_active = 1;
    run.error = 0;
    run.done = 0;
    run.rm = T(1);
    run.thr = T(0);
    run.best_norm = (T)INFINITY;
    run.pcg_cap = 0xffffffffu;
    run.k = 0;
    fill(D.p, D.n, T(1));
    fill(D.r, D.n, T(1));
    std::vector<cudaEvent_t> ev(2 * reps);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[4] = {0, 0, 0, 0};
    for (int which = 0; which < 4; ++which) {
      if (which == 3 && !gram_on) break;
      for (uint32_t i = 0; i < reps; ++i) {
        hc = run;
        push_ctl();
        CK(cudaEventRecord(ev[2 * i], s));
        if (which == 0)
          launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.p}, EpiAp<T>{D.t, D.ap, D.ctl}, s);
        else if (which == 1)
          launch_spmv<T, 1, SumOp>(D.AT, D.pAT, GatherVec<T>{D.t}, EpiKp<T>{D, T(0)}, s);
        else if (which == 2)
          enq_pcg_iter(Handles{});
        else
          enq_gram_kernel_only();
        CK(cudaEventRecord(ev[2 * i + 1], s));
      }
      CK(cudaStreamSynchronize(s));
      double tot = 0;
      for (uint32_t i = 0; i < reps; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        tot += ms;
      }
      acc[which] = tot / reps;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    hc = saved;
    push_ctl();
    CK(cudaStreamSynchronize(s));
    const double S = sizeof(T);
    auto mb = [&](const DevCsr<T>& M) { return double(M.nnz) * (S + 4) + (double(M.rows) + 1) * 4; };
    const double n = D.n, m = D.m;
    out[0] = acc[0];
    out[1] = acc[1];
    out[2] = acc[2];
    out[3] = mb(D.A) + S * n + S * m;                    // read A, p; write t
    out[4] = mb(D.AT) + mb(D.P) + S * m + 2 * S * n;     // read A^T, P, t, p; write Kp
    out[5] = mb(D.A) + mb(D.AT) + mb(D.P) + S * (2 * m + 11 * n);
    // the same with the bytes of the formats actually streamed (compressed
    // column offsets where the plan has them)
    const double fa = plan_stream_bytes(D.A, D.pA), fat = plan_stream_bytes(D.AT, D.pAT);
    out[6] = fa + S * n + S * m;
    out[7] = fat + mb(D.P) + S * m + 2 * S * n;
    out[8] = fa + fat + mb(D.P) + S * (2 * m + 11 * n);
    // one-pass operator apply (gram.cuh): k_gram alone, its bytes (A's
    // in-window + out-of-window entries, row pointers, t, the partial windows
    // written), the whole PCG iteration's bytes on that path
    out[9] = acc[3];
    out[10] = gram_on ? double(gram_nnz_g) * (S + 2) + double(gram_nnz_out) * (S + 4) +
                            8.0 * (double(gram_ng) + 1) + 8.0 * (m + 1) + S * m + S * n +
                            S * double(gram.G) * gram.W
                      : 0.0;
    out[11] = gram_on ? gram_stream_bytes() + mb(D.P) + S * (11 * n) : 0.0;
  }

  // ------------------------------------- operator-level PCG (ops C-ABI)
  // ReducedKktOperator (linsys.hpp:39-61) + Jacobi (:137-148) on caller
  // matrices (P full, A, A^T), then pcg_solve (linsys.hpp:190-276) run by the
  // same kernels as the ADMM loop (k_pcg_init / the two SpMV passes /
  // k_pcg_dot / k_pcg_update / k_pcg_pupdate / k_pcg_fin).
  void setup_operator(const HostCsr<T>& Pf, const HostCsr<T>& A, const HostCsr<T>& AT, T sigma,
                      T rho, int dev) {
    if (!(sigma > T(0)) || !(rho > T(0)))
      throw InvalidArgument("kkt operator: sigma and rho must be positive");
    if (Pf.rows != Pf.cols || A.cols != Pf.cols || AT.rows != A.cols || AT.cols != A.rows)
      throw InvalidArgument("kkt operator: dimension mismatch");
    qpcg_settings st;
    std::memset(&st, 0, sizeof(st));
    st.alpha = 1.6;
    st.sigma = double(sigma);
    st.rho_bar_init = double(rho);
    st.eps_abs = st.eps_rel = 1e-3;
    st.eps_pinf = st.eps_dinf = 1e-4;
    st.max_admm_iter = st.check_interval = st.rho_update_interval = 1;
    st.lambda_pcg = 0.15;
    st.eps_pcg_min = 1e-7;
    st.eps_equil = 1e-3;
    st.equil_max_passes = 1;
    qpcg_options op;
    std::memset(&op, 0, sizeof(op));
    op.device = dev;
    op.input_memory = QPCG_MEM_HOST;
    op.mode = QPCG_MODE_EAGER;
    begin(st, op, nullptr);
    AllocScope scope(s, &arena);
    const uint32_t n = Pf.rows, m = A.rows;
    D.n = n;
    D.m = m;
    auto up = [&](const HostCsr<T>& H) {
      DevCsr<T> M{H.rows, H.cols, H.nnz, alloc<T>(H.nnz), alloc<uint32_t>(size_t(H.rows) + 1),
                  alloc<uint32_t>(H.nnz)};
      upload(M.val, H.values, sizeof(T) * H.nnz);
      upload(M.rp, H.row_ptr, 4 * (size_t(H.rows) + 1));
      upload(M.ci, H.col_indices, 4 * size_t(H.nnz));
      return M;
    };
    D.P = up(Pf);
    D.A = up(A);
    D.AT = up(AT);
    D.pP = plan_build<T>(D.P.rp, n, D.P.nnz, tmp, s);
    D.pA = plan_build<T>(D.A.rp, m, D.A.nnz, tmp, s);
    D.pAT = plan_build<T>(D.AT.rp, n, D.AT.nnz, tmp, s);
    // linsys.hpp:54-58: a_t must be transpose_csr(a) bit for bit
    {
      uint32_t* row_of = alloc<uint32_t>(A.nnz);
      plan_visit(D.A, D.pA, RowOfFn{row_of}, s);
      uint32_t* trp = alloc<uint32_t>(size_t(n) + 1);
      uint32_t* tci = alloc<uint32_t>(A.nnz);
      uint32_t* perm = alloc<uint32_t>(A.nnz);
      transpose_structure(D.A.ci, row_of, n, A.nnz, trp, tci, perm, tmp, s);
      uint32_t* bad = alloc<uint32_t>(1);
      CK(cudaMemsetAsync(bad, 0, 4, s));
      const uint32_t *atrp = D.AT.rp, *atci = D.AT.ci, *pm = perm;
      const T *av = D.A.val, *atv = D.AT.val;
      const uint32_t annz = A.nnz, AT_nnz = AT.nnz;
      if (AT_nnz != annz) {
        CK(cudaMemsetAsync(bad, 1, 1, s));
      } else {
        for_n(n + 1, [=] __device__(uint32_t i) { if (trp[i] != atrp[i]) *bad = 1u; }, s);
        for_n(annz, [=] __device__(uint32_t i) {
          // bitwise value comparison (the reference compares std::vector<T>)
          if (tci[i] != atci[i] || !(av[pm[i]] == atv[i] || (av[pm[i]] != av[pm[i]] && atv[i] != atv[i])))
            *bad = 1u;
        }, s);
      }
      uint32_t hb = 0;
      CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (hb) throw InvalidArgument("kkt operator: a_t is not the transpose of a");
    }
    if (compress_indices()) {
      plan_compress(D.pA, D.A.ci, A.nnz, n, tmp, s);
      plan_compress(D.pAT, D.AT.ci, AT.nnz, m, tmp, s);
    }
    D.ctl = alloc<Ctl<T>>(1);
    D.red = alloc<T>(kRedBlocks * kMaxQ);
    CK(cudaMemsetAsync(D.ctl, 0, sizeof(Ctl<T>), s));
    D.diag_p = vec(n, false);
    D.diag_ata = vec(n, false);
    D.dinv = vec(n, false);
    extract_diag_kernel<T><<<grid_for(n), kThreads, 0, s>>>(D.P, D.diag_p);
    CK_LAUNCH();
    diag_ata_kernel<T><<<grid_for(uint64_t(n) * 32), kThreads, 0, s>>>(D.AT, D.diag_ata, nullptr);
    CK_LAUNCH();
    D.x = vec(n); D.xt = vec(n); D.b = vec(n); D.r = vec(n); D.p = vec(n); D.kp = vec(n);
    D.best = vec(n);
    D.t = vec(m);
    D.g2n = alloc<pair_t<T>>(n);
    std::memset(&hc, 0, sizeof(hc));
    hc.alpha = T(1.6);
    hc.sigma = sigma;
    hc.rho = rho;
    hc.check_interval = 1;
    push_ctl();
    k_precond<T><<<grid_for(n), kThreads, 0, s>>>(D, 1);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
  }

  void op_pcg(const T* b, const T* warm, T eps, uint32_t max_iter, T* x, double* res) {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    if (!(eps > T(0))) throw InvalidArgument("pcg: eps must be positive");
    const uint32_t n = D.n;
    upload(D.b, b, sizeof(T) * n);
    upload(D.xt, warm, sizeof(T) * n);
    pull_ctl();
    hc.error = 0;
    hc.done = 0;
    hc.pcg_eps = eps;
    hc.pcg_cap = max_iter;
    hc.pcg_active = 1;  // enables the operator passes below
    hc.iter = 0;
    push_ctl();
    // r0 = K x0 - b (linsys.hpp:219-220): the passes read p
    CK(cudaMemcpyAsync(D.p, D.xt, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
    launch_spmv<T, 1, SumOp>(D.A, D.pA, GatherVec<T>{D.p}, EpiAp<T>{D.t, D.ap, D.ctl}, s);
    launch_spmv<T, 1, SumOp>(D.AT, D.pAT, GatherVec<T>{D.t}, EpiKp<T>{D, T(0)}, s);
    {
      T *r = D.r, *kp = D.kp;
      const T* bb = D.b;
      for_n(n, [=] __device__(uint32_t i) { r[i] = kp[i] - bb[i]; }, s);
    }
    enq_pcg_init(Handles{});
    pull_ctl();
    if (hc.pcg_active && hc.pcg_cap == 0) {  // linsys.hpp:235-241 before any iteration
      hc.pcg_active = 0;
      hc.pcg_exit = kPcgCap;
      push_ctl();
    }
    while (hc.pcg_active && !hc.error) {
      enq_pcg_iter(Handles{});
      pull_ctl();
    }
    if (hc.error == kErrNotPD)
      throw NotPositiveDefinite("pcg: encountered direction of nonpositive curvature");
    if (hc.error == kErrRho) throw InvalidArgument("kkt operator: rho must be positive");
    if (hc.error == kErrInvalid) throw InvalidArgument("pcg: warm start must be finite");
    k_pcg_fin<T><<<grid_for(n), kThreads, 0, s>>>(D, Handles{});
    CK_LAUNCH();
    download(x, D.xt, sizeof(T) * n);
    CK(cudaStreamSynchronize(s));
    pull_ctl();
    const bool cap = hc.pcg_exit == kPcgCap, zero = hc.pcg_exit == kPcgZeroRhs;
    res[0] = double(hc.k);
    res[1] = zero ? 0.0 : double(cap ? hc.best_norm : hc.r_norm);
    res[2] = cap ? 0.0 : 1.0;
  }

  // ---------------------------------------------------- diagnostics (C-ABI)
  uint32_t pcg_calls(qpcg_pcg_call* out, uint32_t cap) override {
    const uint32_t n = std::min(hc.n_calls, hc.diag_cap);
    std::vector<DiagRec<T>> recs(n);
    if (n) cudaMemcpy(recs.data(), D.calls, sizeof(DiagRec<T>) * n, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < n && i < cap; ++i) {
      out[i].admm_iter = recs[i].admm_iter;
      out[i].iterations = recs[i].iterations;
      out[i].eps = double(recs[i].eps);
      out[i].r_prim_scaled_inf = double(recs[i].rp);
      out[i].r_dual_scaled_inf = double(recs[i].rd);
      out[i].converged = int32_t(recs[i].converged);
      out[i].reserved_ = 0;
    }
    return n;
  }
  uint32_t rho_updates(qpcg_rho_update* out, uint32_t cap) override {
    const uint32_t n = std::min(hc.n_rho, hc.diag_cap);
    std::vector<RhoRec<T>> recs(n);
    if (n) cudaMemcpy(recs.data(), D.rhos, sizeof(RhoRec<T>) * n, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < n && i < cap; ++i) {
      out[i].admm_iter = recs[i].admm_iter;
      out[i].reserved_ = 0;
      out[i].rho_before = double(recs[i].before);
      out[i].rho_after = double(recs[i].after);
    }
    return n;
  }
  uint32_t check_iterations(uint32_t* out, uint32_t cap) override {
    const uint32_t n = std::min(hc.n_checks, hc.diag_cap);
    std::vector<uint32_t> recs(n);
    if (n) cudaMemcpy(recs.data(), D.checks, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost);
    for (uint32_t i = 0; i < n && i < cap; ++i) out[i] = recs[i];
    return n;
  }
  void dims(uint64_t* d) override {
    d[0] = D.n;
    d[1] = D.m;
    d[2] = D.P.nnz;
    d[3] = D.A.nnz;
    d[4] = equil_passes;
    d[5] = 0;
  }

  // Not in the reference: rescale with the existing D, E, c.
  void update_vectors(const T* q, const T* l, const T* u) override {
    CK(cudaSetDevice(device));
    AllocScope scope(s, &arena);
    const unsigned long long k = vectors_stage(q, l, u);
    if (k != ~0ull) throw InvalidArgument(validation_message(k));
    vectors_apply();
  }
  // Uploads into scratch (the vectors not given are copied from the current
  // data) and validates there: a rejected update leaves q_o / l_o / u_o and
  // their scaled copies untouched.  The scratch lives until vectors_apply in
  // the caller's AllocScope.
  T *v_q = nullptr, *v_l = nullptr, *v_u = nullptr;
  unsigned long long vectors_stage(const T* q, const T* l, const T* u) {
    const uint32_t n = D.n, m = D.m;
    v_q = vec(n, false);
    v_l = vec(m, false);
    v_u = vec(m, false);
    auto stage = [&](T* dst, const T* src, const T* cur, uint32_t len) {
      if (src) upload(dst, src, sizeof(T) * len);
      else if (len) CK(cudaMemcpyAsync(dst, cur, sizeof(T) * len, cudaMemcpyDeviceToDevice, s));
    };
    stage(v_q, q, D.q_o, n);
    stage(v_l, l, D.l_o, m);
    stage(v_u, u, D.u_o, m);
    unsigned long long* key = alloc<unsigned long long>(1);
    CK(cudaMemsetAsync(key, 0xff, 8, s));
    validate_values_kernel<T><<<grid_for(n), kThreads, 0, s>>>(v_q, n, kValQFinite, key);
    validate_bounds_kernel<T><<<grid_for(m), kThreads, 0, s>>>(v_l, v_u, m, key, row0);
    CK_LAUNCH();
    unsigned long long k;
    CK(cudaMemcpyAsync(&k, key, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return k;
  }
  void vectors_apply() {
    const uint32_t n = D.n, m = D.m;
    const T c = hc.c;
    if (n) CK(cudaMemcpyAsync(D.q_o, v_q, sizeof(T) * n, cudaMemcpyDeviceToDevice, s));
    if (m) CK(cudaMemcpyAsync(D.l_o, v_l, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
    if (m) CK(cudaMemcpyAsync(D.u_o, v_u, sizeof(T) * m, cudaMemcpyDeviceToDevice, s));
    T *qs = D.q, *qo = D.q_o, *d = D.d, *e = D.e, *ls = D.l, *us = D.u, *lo = D.l_o, *uo = D.u_o;
    for_n(n, [=] __device__(uint32_t i) { qs[i] = c * (d[i] * qo[i]); }, s);
    for_n(m, [=] __device__(uint32_t j) {
      ls[j] = e[j] * lo[j];
      us[j] = e[j] * uo[j];
    }, s);
    k_infnorm<T><<<red_grid<T>(n), kThreads, 0, s>>>(D.q_o, n, D.red, &D.ctl->red_counter,
                                                      &D.ctl->q_inf_orig);
    k_infnorm<T><<<red_grid<T>(n), kThreads, 0, s>>>(D.q, n, D.red, &D.ctl->red_counter,
                                                      &D.ctl->q_inf_scaled);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s));
    pull_ctl();
  }
};

}  // namespace qpcg_b200
