// qpcg_b200_adapter.hpp — drop-in C++ front end for the reference's API.
//
// Include AFTER the reference's own headers (it uses qpcg::QpProblem,
// qpcg::Settings, qpcg::WarmStart, qpcg::SolveDiagnostics, qpcg::SolveOutcome
// from solver.hpp) and link libqpcg_b200.so.  It provides
//
//   template <typename T>
//   qpcg::SolveOutcome<T> qpcg::b200::solve(const QpProblem<T>&, const Settings<T>&,
//                                           const WarmStart<T>* = nullptr,
//                                           SolveDiagnostics<T>* = nullptr);
//
// with the exact signature and semantics of qpcg::solve (solver.hpp:386-389)
// and the same exception classes (std::invalid_argument,
// qpcg::NotPositiveDefiniteError, std::runtime_error), so the reference's
// bench runner swaps with one line at runner.hpp:84:
//
//   const SolveOutcome<T> out = qpcg::b200::solve(p, settings);
//
// SolveDiagnostics: pcg_calls, check_iterations and rho_updates are filled
// after the solve; a set on_iteration (solver.hpp:166, :451-454) switches the
// engine to its host-driven loop and is called after every ADMM step with the
// scaled iterates (qpcg_options.on_iteration: one device->host copy per
// iteration, an instrumented mode).  Unlike the reference, pcg_calls is not
// yet appended while the callback runs.
#ifndef QPCG_B200_ADAPTER_HPP
#define QPCG_B200_ADAPTER_HPP

#include <chrono>
#include <functional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qpcg_b200.h"

namespace qpcg::b200 {

namespace adapter_detail {

inline qpcg_csr_f64 view(const qpcg::CsrMatrix<double>& m) {
  return qpcg_csr_f64{m.rows, m.cols, m.nnz(), m.values.data(), m.row_ptr.data(),
                      m.col_indices.data()};
}
inline qpcg_csr_f32 view(const qpcg::CsrMatrix<float>& m) {
  return qpcg_csr_f32{m.rows, m.cols, m.nnz(), m.values.data(), m.row_ptr.data(),
                      m.col_indices.data()};
}

template <typename T>
qpcg_settings settings(const qpcg::Settings<T>& s) {
  qpcg_settings c;
  qpcg_default_settings(&c);
  c.alpha = double(s.alpha);
  c.sigma = double(s.sigma);
  c.rho_bar_init = double(s.rho_bar_init);
  c.eps_abs = double(s.eps_abs);
  c.eps_rel = double(s.eps_rel);
  c.eps_pinf = double(s.eps_pinf);
  c.eps_dinf = double(s.eps_dinf);
  c.max_admm_iter = s.max_admm_iter;
  c.check_interval = s.check_interval;
  c.rho_update_interval = s.rho_update_interval;
  c.scaling_enabled = s.scaling_enabled ? 1u : 0u;
  c.lambda_pcg = double(s.lambda_pcg);
  c.eps_pcg_min = double(s.eps_pcg_min);
  c.eps_equil = double(s.eps_equil);
  c.equil_max_passes = s.equil_max_passes;
  return c;
}

[[noreturn]] inline void rethrow(int rc, const std::string& msg) {
  if (rc == QPCG_ERR_INVALID) throw std::invalid_argument(msg);
  if (rc == QPCG_ERR_NOT_PD) throw qpcg::NotPositiveDefiniteError(msg);
  throw std::runtime_error(msg);
}

template <typename T>
struct Api;
template <>
struct Api<double> {
  static int setup(qpcg_workspace** w, const qpcg_csr_f64* p, const double* q,
                   const qpcg_csr_f64* a, const double* l, const double* u,
                   const qpcg_settings* s, const qpcg_options* o) {
    return qpcg_f64_setup(w, p, q, a, l, u, s, o);
  }
  static int warm(qpcg_workspace* w, const double* x, const double* z, const double* y) {
    return qpcg_f64_warm_start(w, x, z, y);
  }
  static int solve(qpcg_workspace* w, qpcg_info* i, double* x, double* z, double* y,
                   double* c) {
    return qpcg_f64_solve(w, i, x, z, y, c);
  }
};
template <>
struct Api<float> {
  static int setup(qpcg_workspace** w, const qpcg_csr_f32* p, const float* q,
                   const qpcg_csr_f32* a, const float* l, const float* u,
                   const qpcg_settings* s, const qpcg_options* o) {
    return qpcg_f32_setup(w, p, q, a, l, u, s, o);
  }
  static int warm(qpcg_workspace* w, const float* x, const float* z, const float* y) {
    return qpcg_f32_warm_start(w, x, z, y);
  }
  static int solve(qpcg_workspace* w, qpcg_info* i, float* x, float* z, float* y, float* c) {
    return qpcg_f32_solve(w, i, x, z, y, c);
  }
};

// appends this solve's PCG records not yet in diag (base: the size diag had
// when the solve started; the reference only ever appends to it)
template <typename T>
void append_pcg_calls(qpcg_workspace* w, qpcg::SolveDiagnostics<T>* diag, size_t base) {
  const uint32_t k = qpcg_get_pcg_calls(w, nullptr, 0);
  const size_t have = diag->pcg_calls.size() - base;
  if (k <= have) return;
  std::vector<qpcg_pcg_call> calls(k);
  qpcg_get_pcg_calls(w, calls.data(), k);
  for (size_t i = have; i < calls.size(); ++i) {
    const auto& c = calls[i];
    diag->pcg_calls.push_back({c.admm_iter, T(c.eps), T(c.r_prim_scaled_inf),
                               T(c.r_dual_scaled_inf), c.iterations, c.converged != 0});
  }
}

// qpcg_iteration_cb -> std::function<void(const IterationView<T>&)>; like the
// reference (solver.hpp:446-454) the iteration's PcgCall is appended to
// diag->pcg_calls before the callback runs
template <typename T>
struct IterTrampoline {
  const std::function<void(const qpcg::IterationView<T>&)>* fn;
  std::vector<T> x, z, y, l, u;
  qpcg_workspace* w = nullptr;
  qpcg::SolveDiagnostics<T>* diag = nullptr;
  size_t base = 0;
  static void call(void* user, uint32_t iter, const void* xp, const void* zp, const void* yp,
                   const void* lp, const void* up, uint32_t n, uint32_t m) {
    auto* t = static_cast<IterTrampoline*>(user);
    if (t->w && t->diag) append_pcg_calls(t->w, t->diag, t->base);
    auto fill = [](std::vector<T>& v, const void* p, uint32_t k) {
      const T* a = static_cast<const T*>(p);
      v.assign(a, a + k);
    };
    fill(t->x, xp, n);
    fill(t->z, zp, m);
    fill(t->y, yp, m);
    if (t->l.size() != m) {  // bounds do not change during a solve
      fill(t->l, lp, m);
      fill(t->u, up, m);
    }
    (*t->fn)(qpcg::IterationView<T>{iter, t->x, t->z, t->y, t->l, t->u});
  }
};

struct WsGuard {
  qpcg_workspace* w = nullptr;
  ~WsGuard() { qpcg_cleanup(w); }
};

}  // namespace adapter_detail

// solver.hpp:386-541, on the B200
template <typename T>
qpcg::SolveOutcome<T> solve(const qpcg::QpProblem<T>& p, const qpcg::Settings<T>& s,
                            std::type_identity_t<const qpcg::WarmStart<T>*> initial = nullptr,
                            std::type_identity_t<qpcg::SolveDiagnostics<T>*> diag = nullptr) {
  using namespace adapter_detail;
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>);
  const auto pv = view(p.p_upper);
  const auto av = view(p.a);
  const qpcg_settings cs = settings(s);
  qpcg_options opt;
  qpcg_default_options(&opt);
  opt.record_diagnostics = diag != nullptr ? 1 : 0;
  IterTrampoline<T> tramp{diag != nullptr ? &diag->on_iteration : nullptr, {}, {}, {}, {}, {},
                          nullptr, diag, diag != nullptr ? diag->pcg_calls.size() : 0};
  if (diag != nullptr && diag->on_iteration) {
    opt.on_iteration = &IterTrampoline<T>::call;
    opt.on_iteration_user = &tramp;
  }
  if (p.q.size() != p.p_upper.rows) throw std::invalid_argument("problem: q length must equal n");
  if (p.l.size() != p.a.rows || p.u.size() != p.a.rows)
    throw std::invalid_argument("problem: bound lengths must equal m");
  const auto t_start = std::chrono::steady_clock::now();  // solver.hpp:392
  WsGuard g;
  int rc = Api<T>::setup(&g.w, &pv, p.q.data(), &av, p.l.data(), p.u.data(), &cs, &opt);
  if (rc != QPCG_OK) rethrow(rc, qpcg_last_error(nullptr));
  tramp.w = g.w;
  const size_t n = p.p_upper.rows, m = p.a.rows;
  if (initial != nullptr) {
    if (initial->x.size() != n || initial->z.size() != m || initial->y.size() != m)
      throw std::invalid_argument("solve: warm start dimension mismatch");
    rc = Api<T>::warm(g.w, initial->x.data(), initial->z.data(), initial->y.data());
    if (rc != QPCG_OK) rethrow(rc, qpcg_last_error(g.w));
  }
  qpcg::SolveOutcome<T> out;
  out.x.resize(n);
  out.z.resize(m);
  out.y.resize(m);
  std::vector<T> cert(n > m ? n : m);
  qpcg_info info;
  rc = Api<T>::solve(g.w, &info, out.x.data(), out.z.data(), out.y.data(), cert.data());
  if (rc != QPCG_OK) rethrow(rc, qpcg_last_error(g.w));
  out.status = static_cast<qpcg::SolveStatus>(info.status);
  if (info.certificate_valid)
    out.certificate.assign(cert.begin(),
                           cert.begin() + (info.status == QPCG_STATUS_PRIMAL_INFEASIBLE ? m : n));
  out.objective = T(info.objective);
  out.iterations = info.iterations;
  out.pcg_iterations_total = info.pcg_iterations_total;
  out.r_prim_inf = T(info.r_prim_inf);
  out.r_dual_inf = T(info.r_dual_inf);
  out.runtime_seconds =  // solver.hpp:537-539: setup through objective
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  out.equil_passes = info.equil_passes;
  out.equil_residual = T(info.equil_residual);
  out.rho_final = T(info.rho_final);
  out.rho_update_count = info.rho_update_count;
  if (diag != nullptr) {
    append_pcg_calls(g.w, diag, tramp.base);  // (on_iteration may have appended some)
    std::vector<uint32_t> checks(qpcg_get_check_iterations(g.w, nullptr, 0));
    qpcg_get_check_iterations(g.w, checks.data(), uint32_t(checks.size()));
    for (auto it : checks) diag->check_iterations.push_back(it);
    std::vector<qpcg_rho_update> rho(qpcg_get_rho_updates(g.w, nullptr, 0));
    qpcg_get_rho_updates(g.w, rho.data(), uint32_t(rho.size()));
    for (const auto& r : rho)
      diag->rho_updates.push_back({r.admm_iter, T(r.rho_before), T(r.rho_after)});
  }
  return out;
}

}  // namespace qpcg::b200

#endif  // QPCG_B200_ADAPTER_HPP
