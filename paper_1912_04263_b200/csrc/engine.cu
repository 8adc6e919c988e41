// engine.cu — the C-ABI (include/qpcg_b200.h, include/qpcg_b200_ops.h) over
// the B200 ADMM/PCG workspace (workspace.cuh) and its row-sharded variant
// (shard.cuh).  See workspace.cuh for the per-step kernel sequence.
#include "workspace.cuh"

#include "shard.cuh"

// =====================================================================
// C-ABI
// =====================================================================
using namespace qpcg_b200;

struct qpcg_workspace {
  int precision = 64;
  std::unique_ptr<IEngine<double>> e64;  // Workspace<double> or Sharded<double>
  std::unique_ptr<IEngine<float>> e32;
  std::string err;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(qpcg_workspace* ws, F&& f) {
  std::string* msg = ws ? &ws->err : &g_last_error;
  try {
    f();
    return QPCG_OK;
  } catch (const InvalidArgument& e) {
    *msg = e.what();
    return QPCG_ERR_INVALID;
  } catch (const NotPositiveDefinite& e) {
    *msg = e.what();
    return QPCG_ERR_NOT_PD;
  } catch (const OutOfMemory& e) {
    *msg = e.what();
    return QPCG_ERR_OOM;
  } catch (const CudaError& e) {
    *msg = e.what();
    return QPCG_ERR_CUDA;
  } catch (const NcclError& e) {
    *msg = e.what();
    return QPCG_ERR_NCCL;
  } catch (const std::exception& e) {
    *msg = e.what();
    return QPCG_ERR_RUNTIME;
  }
}

template <typename T, typename CsrT>
HostCsr<T> host_csr(const CsrT* c) {
  return HostCsr<T>{c->rows, c->cols, c->nnz, c->values, c->row_ptr, c->col_indices};
}

template <typename T>
std::unique_ptr<IEngine<T>>& slot(qpcg_workspace* ws);
template <>
std::unique_ptr<IEngine<double>>& slot<double>(qpcg_workspace* ws) { return ws->e64; }
template <>
std::unique_ptr<IEngine<float>>& slot<float>(qpcg_workspace* ws) { return ws->e32; }

bool is_sharded(const qpcg_options& o) {
  return o.virtual_shards > 1 || o.nccl_id != nullptr || o.transport == QPCG_TRANSPORT_PEER;
}

template <typename T, typename CsrT>
int setup_impl(qpcg_workspace** out, const CsrT* p, const T* q, const CsrT* a, const T* l,
               const T* u, const qpcg_settings* s, const qpcg_options* o) {
  if (out == nullptr || p == nullptr || a == nullptr || q == nullptr || l == nullptr ||
      u == nullptr) {
    g_last_error = "setup: null argument";
    return QPCG_ERR_INVALID;
  }
  auto* ws = new qpcg_workspace();
  ws->precision = sizeof(T) * 8;
  qpcg_settings st;
  qpcg_default_settings(&st);
  if (s) st = *s;
  qpcg_options op;
  qpcg_default_options(&op);
  if (o) op = *o;
  const int rc = guarded(ws, [&] {
    slot<T>(ws).reset(make_engine<T>(is_sharded(op)));
    slot<T>(ws)->setup(host_csr<T>(p), q, host_csr<T>(a), l, u, st, op);
  });
  if (rc != QPCG_OK) {
    g_last_error = ws->err;
    delete ws;
    *out = nullptr;
    return rc;
  }
  *out = ws;
  return rc;
}

template <typename T>
IEngine<T>* get(const qpcg_workspace* w) {
  auto* ws = const_cast<qpcg_workspace*>(w);
  if (ws == nullptr || !slot<T>(ws)) throw InvalidArgument("workspace: wrong precision or null");
  return slot<T>(ws).get();
}

template <typename T, typename CsrT>
int solve_problem_impl(const CsrT* p, const T* q, const CsrT* a, const T* l, const T* u,
                       const qpcg_settings* s, const qpcg_options* o, const T* wx, const T* wz,
                       const T* wy, qpcg_info* info, T* x, T* z, T* y, T* cert, char* msg,
                       size_t msg_len) {
  const double t0 = now_s();
  qpcg_workspace* ws = nullptr;
  int rc = setup_impl<T>(&ws, p, q, a, l, u, s, o);
  if (rc == QPCG_OK && wx != nullptr) rc = guarded(ws, [&] { get<T>(ws)->warm_start(wx, wz, wy); });
  if (rc == QPCG_OK) rc = guarded(ws, [&] { get<T>(ws)->solve(info, x, z, y, cert); });
  if (rc == QPCG_OK && info) info->runtime_seconds = now_s() - t0;  // solver.hpp:392 -> :537
  if (rc != QPCG_OK && msg && msg_len) {
    const std::string& e = ws ? ws->err : g_last_error;
    std::snprintf(msg, msg_len, "%s", e.c_str());
  }
  delete ws;
  return rc;
}

// f(engine) on whichever precision the workspace holds
template <typename F>
int either(const qpcg_workspace* w, F&& f) {
  auto* ws = const_cast<qpcg_workspace*>(w);
  return guarded(ws, [&] {
    if (ws && ws->e64)
      f(*ws->e64);
    else if (ws && ws->e32)
      f(*ws->e32);
    else
      throw InvalidArgument("workspace: null");
  });
}

}  // namespace

extern "C" {

void qpcg_default_settings(qpcg_settings* s) {
  std::memset(s, 0, sizeof(*s));
  s->alpha = 1.6;
  s->sigma = 1e-6;
  s->rho_bar_init = 0.1;
  s->eps_abs = 1e-3;
  s->eps_rel = 1e-3;
  s->eps_pinf = 1e-4;
  s->eps_dinf = 1e-4;
  s->max_admm_iter = 50000;
  s->check_interval = 5;
  s->rho_update_interval = 10;
  s->scaling_enabled = 1;
  s->lambda_pcg = 0.15;
  s->eps_pcg_min = 1e-7;
  s->eps_equil = 1e-3;
  s->equil_max_passes = 10;
}

void qpcg_default_options(qpcg_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->device = -1;
  o->input_memory = QPCG_MEM_HOST;
  o->mode = QPCG_MODE_GRAPH;
  o->record_diagnostics = 0;
  o->virtual_shards = 1;
}

int qpcg_validate_settings(const qpcg_settings* s, char* msg, size_t msg_len) {
  try {
    validate_settings_in<double>(*s);
    return QPCG_OK;
  } catch (const std::exception& e) {
    if (msg && msg_len) std::snprintf(msg, msg_len, "%s", e.what());
    return QPCG_ERR_INVALID;
  }
}

const char* qpcg_version(void) { return "qpcg-b200 0.1 (sm_100a)"; }

int qpcg_f64_setup(qpcg_workspace** ws, const qpcg_csr_f64* p, const double* q,
                   const qpcg_csr_f64* a, const double* l, const double* u,
                   const qpcg_settings* s, const qpcg_options* o) {
  return setup_impl<double>(ws, p, q, a, l, u, s, o);
}
int qpcg_f32_setup(qpcg_workspace** ws, const qpcg_csr_f32* p, const float* q,
                   const qpcg_csr_f32* a, const float* l, const float* u, const qpcg_settings* s,
                   const qpcg_options* o) {
  return setup_impl<float>(ws, p, q, a, l, u, s, o);
}
int qpcg_f64_warm_start(qpcg_workspace* ws, const double* x, const double* z, const double* y) {
  return guarded(ws, [&] { get<double>(ws)->warm_start(x, z, y); });
}
int qpcg_f32_warm_start(qpcg_workspace* ws, const float* x, const float* z, const float* y) {
  return guarded(ws, [&] { get<float>(ws)->warm_start(x, z, y); });
}
int qpcg_f64_update_rho(qpcg_workspace* ws, double rho) {
  return guarded(ws, [&] { get<double>(ws)->update_rho(rho); });
}
int qpcg_f32_update_rho(qpcg_workspace* ws, double rho) {
  return guarded(ws, [&] { get<float>(ws)->update_rho(float(rho)); });
}
int qpcg_f64_update_vectors(qpcg_workspace* ws, const double* q, const double* l, const double* u) {
  return guarded(ws, [&] { get<double>(ws)->update_vectors(q, l, u); });
}
int qpcg_f32_update_vectors(qpcg_workspace* ws, const float* q, const float* l, const float* u) {
  return guarded(ws, [&] { get<float>(ws)->update_vectors(q, l, u); });
}
int qpcg_f64_solve(qpcg_workspace* ws, qpcg_info* info, double* x, double* z, double* y,
                   double* cert) {
  return guarded(ws, [&] { get<double>(ws)->solve(info, x, z, y, cert); });
}
int qpcg_f32_solve(qpcg_workspace* ws, qpcg_info* info, float* x, float* z, float* y,
                   float* cert) {
  return guarded(ws, [&] { get<float>(ws)->solve(info, x, z, y, cert); });
}
int qpcg_f64_solve_problem(const qpcg_csr_f64* p, const double* q, const qpcg_csr_f64* a,
                           const double* l, const double* u, const qpcg_settings* s,
                           const qpcg_options* o, const double* wx, const double* wz,
                           const double* wy, qpcg_info* info, double* x, double* z, double* y,
                           double* cert, char* msg, size_t msg_len) {
  return solve_problem_impl<double>(p, q, a, l, u, s, o, wx, wz, wy, info, x, z, y, cert, msg,
                                    msg_len);
}
int qpcg_f32_solve_problem(const qpcg_csr_f32* p, const float* q, const qpcg_csr_f32* a,
                           const float* l, const float* u, const qpcg_settings* s,
                           const qpcg_options* o, const float* wx, const float* wz,
                           const float* wy, qpcg_info* info, float* x, float* z, float* y,
                           float* cert, char* msg, size_t msg_len) {
  return solve_problem_impl<float>(p, q, a, l, u, s, o, wx, wz, wy, info, x, z, y, cert, msg,
                                   msg_len);
}
void qpcg_cleanup(qpcg_workspace* ws) { delete ws; }
void qpcg_release_cached_memory(void) { release_cached_memory(); }

int qpcg_shard_cuts(const uint32_t* row_ptr, uint32_t rows, uint32_t nnz, uint32_t blocks,
                    uint32_t* cuts) {
  if (row_ptr == nullptr || cuts == nullptr || blocks == 0) return 0;
  return shard_cuts(row_ptr, rows, nnz, blocks, cuts) ? 1 : 0;
}

int qpcg_nccl_unique_id(void* out) {
  return guarded(nullptr, [&] {
    if (out == nullptr) throw InvalidArgument("nccl: null id buffer");
    ncclUniqueId id;
    nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == QPCG_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(out, &id, sizeof(id));
  });
}
const char* qpcg_last_error(const qpcg_workspace* ws) {
  return ws ? ws->err.c_str() : g_last_error.c_str();
}

uint32_t qpcg_get_pcg_calls(const qpcg_workspace* ws, qpcg_pcg_call* out, uint32_t cap) {
  uint32_t k = 0;
  either(ws, [&](auto& e) { k = e.pcg_calls(out, cap); });
  return k;
}
uint32_t qpcg_get_rho_updates(const qpcg_workspace* ws, qpcg_rho_update* out, uint32_t cap) {
  uint32_t k = 0;
  either(ws, [&](auto& e) { k = e.rho_updates(out, cap); });
  return k;
}
uint32_t qpcg_get_check_iterations(const qpcg_workspace* ws, uint32_t* out, uint32_t cap) {
  uint32_t k = 0;
  either(ws, [&](auto& e) { k = e.check_iterations(out, cap); });
  return k;
}

int qpcg_debug_dims(const qpcg_workspace* ws, uint64_t* dims) {
  return either(ws, [&](auto& e) { e.dims(dims); });
}

int qpcg_debug_scaled(const qpcg_workspace* ws, void* pv, uint32_t* prp, uint32_t* pci, void* q,
                      void* av, void* atv, uint32_t* atrp, uint32_t* atci, void* l, void* u,
                      void* d, void* e, double* scal) {
  return either(ws, [&](auto& en) {
    using T = typename std::remove_reference_t<decltype(en)>::value_type;
    en.debug_scaled((T*)pv, prp, pci, (T*)q, (T*)av, (T*)atv, atrp, atci, (T*)l, (T*)u, (T*)d,
                    (T*)e, scal);
  });
}

int qpcg_debug_operator(qpcg_workspace* ws, const void* x, void* kx, void* dinv) {
  return either(ws, [&](auto& en) {
    using T = typename std::remove_reference_t<decltype(en)>::value_type;
    en.debug_operator((const T*)x, (T*)kx, (T*)dinv);
  });
}

int qpcg_bench_kernels(qpcg_workspace* ws, uint32_t reps, double* out) {
  return qpcg_bench_kernels_n(ws, reps, out, 9);  // the round-1 layout: 9 doubles
}
int qpcg_bench_kernels_n(qpcg_workspace* ws, uint32_t reps, double* out, uint32_t cap) {
  double full[QPCG_BENCH_KERNELS_MAX] = {};
  const int rc = either(ws, [&](auto& e) { e.bench_kernels(reps, full); });
  if (rc == QPCG_OK && out != nullptr)
    for (uint32_t i = 0; i < cap && i < QPCG_BENCH_KERNELS_MAX; ++i) out[i] = full[i];
  return rc;
}

}  // extern "C"

template <typename T, typename CsrT>
static int op_spmv_impl(const CsrT* mv, const T* x, T* y, int device) {
  return guarded(nullptr, [&] { op_spmv<T>(host_csr<T>(mv), x, y, device); });
}

extern "C" {

int qpcg_f64_op_spmv(const qpcg_csr_f64* m, const double* x, double* y, int device) {
  return op_spmv_impl<double>(m, x, y, device);
}
int qpcg_f32_op_spmv(const qpcg_csr_f32* m, const float* x, float* y, int device) {
  return op_spmv_impl<float>(m, x, y, device);
}

int qpcg_f64_op_pcg(const qpcg_csr_f64* p_full, const qpcg_csr_f64* a, const qpcg_csr_f64* a_t,
                    double sigma, double rho, const double* b, const double* warm, double eps,
                    uint32_t max_iter, double* x, double* res, int device) {
  return guarded(nullptr, [&] {
    op_pcg<double>(host_csr<double>(p_full), host_csr<double>(a), host_csr<double>(a_t), sigma, rho,
                   b, warm, eps, max_iter, x, res, device);
  });
}
int qpcg_f32_op_pcg(const qpcg_csr_f32* p_full, const qpcg_csr_f32* a, const qpcg_csr_f32* a_t,
                    double sigma, double rho, const float* b, const float* warm, double eps,
                    uint32_t max_iter, float* x, double* res, int device) {
  return guarded(nullptr, [&] {
    op_pcg<float>(host_csr<float>(p_full), host_csr<float>(a), host_csr<float>(a_t), float(sigma),
                  float(rho), b, warm, float(eps), max_iter, x, res, device);
  });
}

}  // extern "C"
