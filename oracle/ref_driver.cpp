// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim around the UNMODIFIED reference headers
// (/root/reference/proj/include/qpcg/*.hpp, included in place via -I; no
// reference source is copied into this repository).  Built by
// oracle/Makefile into oracle/_ref/libqpcg_ref.so, it is the pinned parity
// oracle and the CPU baseline ("kind": "reference").  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load it.
//
// Exposed:
//   * problem generation through the reference's own RNG + recipes
//     (bench/generators.hpp), both by (class, scale, seed) and with the
//     explicit sizes of SURVEY.md §8(d) (scale tag 100);
//   * qpcg::solve (solver.hpp:386-541) with Settings/WarmStart/Diagnostics;
//   * the hot-path building blocks (spmv, transpose_csr, symmetrize_upper,
//     ruiz_equilibrate, ReducedKktOperator::apply, build_preconditioner,
//     pcg_solve, adaptive_eps, diag_ata, extract_diagonal) for kernel-level
//     parity tests;
//   * timing helpers for the bounded CPU baseline sample.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "qpcg/bench/generators.hpp"
#include "qpcg/bench/runner.hpp"
#include "qpcg/linsys.hpp"
#include "qpcg/scaling.hpp"
#include "qpcg/solver.hpp"
#include "qpcg/sparse.hpp"

#include "qpcg_b200.h"  // shared C structs (settings / info / csr views)

namespace {

using qpcg::index_t;
namespace qb = qpcg::bench;
namespace qbd = qpcg::bench::detail;

thread_local std::string g_err;

template <typename T>
struct CsrView {
  uint32_t rows, cols, nnz;
  const T* values;
  const uint32_t* row_ptr;
  const uint32_t* col_indices;
};

template <typename T>
qpcg::CsrMatrix<T> to_csr(const void* view) {
  const auto* v = static_cast<const CsrView<T>*>(view);
  qpcg::CsrMatrix<T> m;
  m.rows = v->rows;
  m.cols = v->cols;
  m.values.assign(v->values, v->values + v->nnz);
  m.row_ptr.assign(v->row_ptr, v->row_ptr + v->rows + 1);
  m.col_indices.assign(v->col_indices, v->col_indices + v->nnz);
  return m;
}

template <typename T>
qpcg::Settings<T> to_settings(const qpcg_settings* s) {
  qpcg::Settings<T> o;
  if (s == nullptr) return o;
  o.alpha = T(s->alpha);
  o.sigma = T(s->sigma);
  o.rho_bar_init = T(s->rho_bar_init);
  o.eps_abs = T(s->eps_abs);
  o.eps_rel = T(s->eps_rel);
  o.eps_pinf = T(s->eps_pinf);
  o.eps_dinf = T(s->eps_dinf);
  o.max_admm_iter = s->max_admm_iter;
  o.check_interval = s->check_interval;
  o.rho_update_interval = s->rho_update_interval;
  o.lambda_pcg = T(s->lambda_pcg);
  o.eps_pcg_min = T(s->eps_pcg_min);
  o.scaling_enabled = s->scaling_enabled != 0;
  o.eps_equil = T(s->eps_equil);
  o.equil_max_passes = s->equil_max_passes;
  return o;
}

template <typename T>
std::vector<T> vec(const T* p, size_t n) {
  return std::vector<T>(p, p + n);
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return QPCG_OK;
  } catch (const qpcg::NotPositiveDefiniteError& e) {
    g_err = e.what();
    return QPCG_ERR_NOT_PD;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return QPCG_ERR_INVALID;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QPCG_ERR_RUNTIME;
  }
}

// ---------------------------------------------------------------------------
// Explicit-size instances; each follows the draw order of
// the corresponding gen_* in generators.hpp with the sizes made explicit and
// the key derived as derive_key({class, 100, seed}).
// ---------------------------------------------------------------------------
qb::CounterRng rng_explicit(qb::ProblemClass c, uint64_t seed) {
  return qb::CounterRng(
      qb::derive_key({static_cast<uint64_t>(c), uint64_t(100), seed}));
}

qpcg::QpProblem<double> gen_random_explicit(index_t n, index_t m,
                                            index_t p_per_row, uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kRandom, seed);  // gen_random_qp
  qpcg::QpProblem<double> p;
  p.p_upper = qbd::gram_psd_upper(rng, n, n, p_per_row, 0.1);
  p.q.resize(n);
  for (double& v : p.q) v = rng.normal();
  p.a = qbd::sample_sparse(rng, m, n, 0.15);
  std::vector<double> x0(n);
  for (double& v : x0) v = rng.normal();
  const std::vector<double> ax0 = qpcg::spmv(p.a, x0);
  p.l.resize(m);
  p.u.resize(m);
  for (index_t i = 0; i < m; ++i) {
    p.l[i] = ax0[i] - rng.uniform(0.05, 1.05);
    p.u[i] = ax0[i] + rng.uniform(0.05, 1.05);
  }
  return p;
}

qpcg::QpProblem<double> gen_lasso_explicit(index_t n, index_t md,
                                           uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kLasso, seed);  // gen_lasso
  auto a_data = qbd::sample_sparse(rng, md, n, 0.15);
  std::vector<double> x_true(n, 0.0);
  for (double& v : x_true) {
    if (rng.bernoulli(0.1)) v = rng.normal();
  }
  std::vector<double> b = qpcg::spmv(a_data, x_true);
  for (double& v : b) v += 0.01 * rng.normal();
  const auto a_t = qpcg::transpose_csr(a_data);
  const double lambda = qpcg::inf_norm(qpcg::spmv(a_t, b)) / 5.0;
  return qb::make_lasso_qp(a_data, b, lambda);
}

qpcg::QpProblem<double> gen_huber_explicit(index_t n, index_t md,
                                           uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kHuber, seed);  // gen_huber
  auto a_data = qbd::sample_sparse(rng, md, n, 0.15);
  std::vector<double> x_true(n);
  for (double& v : x_true) v = rng.normal();
  std::vector<double> b = qpcg::spmv(a_data, x_true);
  for (double& v : b) v += 0.01 * rng.normal();
  for (double& v : b) {
    if (rng.bernoulli(0.1)) {
      v += (rng.bernoulli(0.5) ? 1.0 : -1.0) * rng.uniform(5.0, 10.0);
    }
  }
  return qb::make_huber_qp(a_data, b, 1.0);
}

qpcg::QpProblem<double> gen_svm_explicit(index_t n, index_t md, uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kSvm, seed);  // gen_svm
  const double shift = 1.0 / std::sqrt(0.15 * double(n));
  std::vector<double> labels(md);
  std::vector<qbd::Triplet> t;
  for (index_t i = 0; i < md; ++i) {
    labels[i] = i < md / 2 ? 1.0 : -1.0;
    for (index_t c = 0; c < n; ++c) {
      if (rng.bernoulli(0.15)) t.push_back({i, c, labels[i] * shift + rng.normal()});
    }
  }
  const auto a_data = qbd::csr_from_triplets(md, n, t);
  return qb::make_svm_qp(a_data, labels, 1.0);
}

qpcg::QpProblem<double> gen_portfolio_explicit(index_t n, index_t k,
                                               uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kPortfolio, seed);  // gen_portfolio
  auto f_t = qbd::sample_sparse(rng, k, n, 0.5);
  std::vector<double> d_diag(n), mu(n);
  for (double& v : d_diag) v = rng.uniform(0.0, std::sqrt(double(k)));
  for (double& v : mu) v = rng.normal();
  return qb::make_portfolio_qp(f_t, d_diag, mu, 1.0);
}

qpcg::QpProblem<double> gen_equality_explicit(index_t n, index_t rows,
                                              uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kEquality, seed);  // gen_equality
  auto p_upper = qbd::gram_psd_upper(rng, n, n, 3, 0.1);
  std::vector<double> q(n);
  for (double& v : q) v = rng.normal();
  auto a = qbd::sample_sparse(rng, rows, n, 0.15);
  std::vector<double> x0(n);
  for (double& v : x0) v = rng.normal();
  const std::vector<double> b = qpcg::spmv(a, x0);
  return qb::make_equality_qp(p_upper, q, a, b);
}

qpcg::QpProblem<double> gen_control_explicit(index_t nx, index_t nu,
                                             index_t horizon, uint64_t seed) {
  auto rng = rng_explicit(qb::ProblemClass::kControl, seed);  // gen_control
  std::vector<double> a_dyn(static_cast<size_t>(nx) * nx);
  for (double& v : a_dyn) v = rng.normal();
  double row_sum_norm = 0.0;
  for (index_t i = 0; i < nx; ++i) {
    double s = 0.0;
    for (index_t j = 0; j < nx; ++j) s += std::abs(a_dyn[size_t(i) * nx + j]);
    row_sum_norm = std::max(row_sum_norm, s);
  }
  if (row_sum_norm > 0.0) {
    for (double& v : a_dyn) v *= 0.95 / row_sum_norm;
  }
  std::vector<double> b_in(static_cast<size_t>(nx) * nu);
  for (double& v : b_in) v = rng.normal();
  std::vector<double> q_diag(nx), qt_diag(nx), r_diag(nu), x_init(nx);
  for (double& v : q_diag) v = rng.uniform(0.1, 2.0);
  for (double& v : qt_diag) v = rng.uniform(0.1, 2.0);
  for (double& v : r_diag) v = rng.uniform(0.1, 1.0);
  const double x_bound = rng.uniform(1.0, 3.0);
  const double u_bound = rng.uniform(0.5, 2.0);
  for (double& v : x_init) v = rng.uniform(-0.5, 0.5) * x_bound;
  return qb::make_control_qp(a_dyn, b_in, q_diag, r_diag, qt_diag, x_init,
                             x_bound, u_bound, horizon);
}

// Diagnostics of the last solve on this thread.
struct LastDiag {
  std::vector<qpcg_pcg_call> calls;
  std::vector<qpcg_rho_update> rho;
  std::vector<uint32_t> checks;
};
thread_local LastDiag g_diag;

template <typename T>
int solve_impl(const void* pv, const T* q, const void* av, const T* l,
               const T* u, const qpcg_settings* sp, const T* wx, const T* wz,
               const T* wy, qpcg_info* info, T* x, T* z, T* y, T* cert,
               int record_diag) {
  return guarded([&] {
    qpcg::QpProblem<T> p;
    p.p_upper = to_csr<T>(pv);
    p.a = to_csr<T>(av);
    const size_t n = p.p_upper.rows, m = p.a.rows;
    p.q = vec(q, n);
    p.l = vec(l, m);
    p.u = vec(u, m);
    const qpcg::Settings<T> s = to_settings<T>(sp);
    qpcg::WarmStart<T> ws;
    const qpcg::WarmStart<T>* wsp = nullptr;
    if (wx != nullptr) {
      ws.x = vec(wx, n);
      ws.z = vec(wz, m);
      ws.y = vec(wy, m);
      wsp = &ws;
    }
    qpcg::SolveDiagnostics<T> diag;
    g_diag = LastDiag{};
    const auto out = qpcg::solve(p, s, wsp, record_diag ? &diag : nullptr);
    if (record_diag) {
      for (const auto& c : diag.pcg_calls) {
        qpcg_pcg_call r{};
        r.admm_iter = c.admm_iter;
        r.iterations = c.iterations;
        r.eps = double(c.eps);
        r.r_prim_scaled_inf = double(c.r_prim_scaled_inf);
        r.r_dual_scaled_inf = double(c.r_dual_scaled_inf);
        r.converged = c.converged ? 1 : 0;
        g_diag.calls.push_back(r);
      }
      for (const auto& c : diag.rho_updates) {
        qpcg_rho_update r{};
        r.admm_iter = c.admm_iter;
        r.rho_before = double(c.rho_before);
        r.rho_after = double(c.rho_after);
        g_diag.rho.push_back(r);
      }
      for (auto it : diag.check_iterations) g_diag.checks.push_back(it);
    }
    if (info != nullptr) {
      std::memset(info, 0, sizeof(*info));
      info->status = static_cast<int32_t>(out.status);
      info->iterations = out.iterations;
      info->pcg_iterations_total = out.pcg_iterations_total;
      info->objective = double(out.objective);
      info->r_prim_inf = double(out.r_prim_inf);
      info->r_dual_inf = double(out.r_dual_inf);
      info->runtime_seconds = out.runtime_seconds;
      info->equil_passes = out.equil_passes;
      info->equil_residual = double(out.equil_residual);
      info->rho_final = double(out.rho_final);
      info->rho_update_count = out.rho_update_count;
      info->certificate_valid = out.certificate.empty() ? 0 : 1;
      info->n = uint32_t(n);
      info->m = uint32_t(m);
    }
    if (x != nullptr) std::copy(out.x.begin(), out.x.end(), x);
    if (z != nullptr) std::copy(out.z.begin(), out.z.end(), z);
    if (y != nullptr) std::copy(out.y.begin(), out.y.end(), y);
    if (cert != nullptr && !out.certificate.empty()) {
      std::copy(out.certificate.begin(), out.certificate.end(), cert);
    }
  });
}

template <typename T>
void copy_csr_out(const qpcg::CsrMatrix<T>& m, T* vals, uint32_t* rp,
                  uint32_t* ci) {
  if (vals) std::copy(m.values.begin(), m.values.end(), vals);
  if (rp) std::copy(m.row_ptr.begin(), m.row_ptr.end(), rp);
  if (ci) std::copy(m.col_indices.begin(), m.col_indices.end(), ci);
}

double now_s() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

const char* qref_last_error() { return g_err.c_str(); }

// ---- problem generation (double data, as every gen_* draws in double) ------
void* qref_gen_class(int cls, uint32_t scale, uint64_t seed) {
  try {
    qb::BenchSpec spec;
    spec.problem_class = static_cast<qb::ProblemClass>(cls);
    spec.scale_index = scale;
    spec.seed = seed;
    return new qpcg::QpProblem<double>(qb::generate<double>(spec));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

// kind: 0 random(a=n, b=m, c=p_per_row), 1 lasso(a=n, b=md),
// 2 huber(a=n, b=md), 3 svm(a=n, b=md), 4 portfolio(a=n, b=k),
// 5 equality(a=n, b=rows), 6 control(a=nx, b=nu, c=horizon)
void* qref_gen_explicit(int kind, uint32_t a, uint32_t b, uint32_t c,
                        uint64_t seed) {
  try {
    switch (kind) {
      case 0: return new qpcg::QpProblem<double>(gen_random_explicit(a, b, c, seed));
      case 1: return new qpcg::QpProblem<double>(gen_lasso_explicit(a, b, seed));
      case 2: return new qpcg::QpProblem<double>(gen_huber_explicit(a, b, seed));
      case 3: return new qpcg::QpProblem<double>(gen_svm_explicit(a, b, seed));
      case 4: return new qpcg::QpProblem<double>(gen_portfolio_explicit(a, b, seed));
      case 5: return new qpcg::QpProblem<double>(gen_equality_explicit(a, b, seed));
      case 6: return new qpcg::QpProblem<double>(gen_control_explicit(a, b, c, seed));
      default: g_err = "unknown kind"; return nullptr;
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

uint64_t qref_target_nnz(uint32_t scale) { return qb::target_nnz(scale); }

// dims[0..3] = n, m, nnz(P_upper), nnz(A)
void qref_problem_dims(const void* h, uint64_t* dims) {
  const auto* p = static_cast<const qpcg::QpProblem<double>*>(h);
  dims[0] = p->num_vars();
  dims[1] = p->num_constraints();
  dims[2] = p->p_upper.nnz();
  dims[3] = p->a.nnz();
}

void qref_problem_export(const void* h, double* pv, uint32_t* prp, uint32_t* pci,
                         double* q, double* av, uint32_t* arp, uint32_t* aci,
                         double* l, double* u) {
  const auto* p = static_cast<const qpcg::QpProblem<double>*>(h);
  copy_csr_out(p->p_upper, pv, prp, pci);
  copy_csr_out(p->a, av, arp, aci);
  std::copy(p->q.begin(), p->q.end(), q);
  std::copy(p->l.begin(), p->l.end(), l);
  std::copy(p->u.begin(), p->u.end(), u);
}

void qref_problem_free(void* h) { delete static_cast<qpcg::QpProblem<double>*>(h); }

// ---- full solve (solver.hpp:386-541) ---------------------------------------
int qref_solve_f64(const qpcg_csr_f64* p, const double* q, const qpcg_csr_f64* a,
                   const double* l, const double* u, const qpcg_settings* s,
                   const double* wx, const double* wz, const double* wy,
                   qpcg_info* info, double* x, double* z, double* y,
                   double* cert, int record_diag) {
  return solve_impl<double>(p, q, a, l, u, s, wx, wz, wy, info, x, z, y, cert,
                            record_diag);
}
int qref_solve_f32(const qpcg_csr_f32* p, const float* q, const qpcg_csr_f32* a,
                   const float* l, const float* u, const qpcg_settings* s,
                   const float* wx, const float* wz, const float* wy,
                   qpcg_info* info, float* x, float* z, float* y, float* cert,
                   int record_diag) {
  return solve_impl<float>(p, q, a, l, u, s, wx, wz, wy, info, x, z, y, cert,
                           record_diag);
}

uint32_t qref_diag_pcg_calls(qpcg_pcg_call* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_diag.calls.size(); ++i) out[i] = g_diag.calls[i];
  return uint32_t(g_diag.calls.size());
}
uint32_t qref_diag_rho_updates(qpcg_rho_update* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_diag.rho.size(); ++i) out[i] = g_diag.rho[i];
  return uint32_t(g_diag.rho.size());
}
uint32_t qref_diag_checks(uint32_t* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_diag.checks.size(); ++i) out[i] = g_diag.checks[i];
  return uint32_t(g_diag.checks.size());
}

// ---- building blocks --------------------------------------------------------
int qref_spmv_f64(const qpcg_csr_f64* m, const double* x, double* y) {
  return guarded([&] {
    const auto mm = to_csr<double>(m);
    const auto r = qpcg::spmv(mm, vec(x, mm.cols));
    std::copy(r.begin(), r.end(), y);
  });
}
int qref_spmv_f32(const qpcg_csr_f32* m, const float* x, float* y) {
  return guarded([&] {
    const auto mm = to_csr<float>(m);
    const auto r = qpcg::spmv(mm, vec(x, mm.cols));
    std::copy(r.begin(), r.end(), y);
  });
}

// out arrays sized nnz / cols+1 by the caller (transpose keeps nnz)
int qref_transpose_f64(const qpcg_csr_f64* m, double* vals, uint32_t* rp,
                       uint32_t* ci) {
  return guarded([&] { copy_csr_out(qpcg::transpose_csr(to_csr<double>(m)), vals, rp, ci); });
}

// two-phase: call with vals == NULL to get the output nnz
int64_t qref_symmetrize_f64(const qpcg_csr_f64* m, double* vals, uint32_t* rp,
                            uint32_t* ci) {
  int64_t nnz = -1;
  const int rc = guarded([&] {
    const auto full = qpcg::symmetrize_upper(to_csr<double>(m));
    nnz = full.nnz();
    if (vals != nullptr) copy_csr_out(full, vals, rp, ci);
  });
  return rc == QPCG_OK ? nnz : -int64_t(rc);
}

int qref_row_inf_norms_f64(const qpcg_csr_f64* m, double* out) {
  return guarded([&] {
    const auto r = qpcg::row_inf_norms(to_csr<double>(m));
    std::copy(r.begin(), r.end(), out);
  });
}

int qref_diag_ata_f64(const qpcg_csr_f64* a, double* out) {
  return guarded([&] {
    const auto r = qpcg::diag_ata(to_csr<double>(a));
    std::copy(r.begin(), r.end(), out);
  });
}

int qref_extract_diagonal_f64(const qpcg_csr_f64* m, double* out) {
  return guarded([&] {
    const auto r = qpcg::extract_diagonal(to_csr<double>(m));
    std::copy(r.begin(), r.end(), out);
  });
}

// Ruiz on (p_full, q, a, l, u).  Outputs (caller-sized): p_full values [nnzP],
// q_s [n], a values [nnzA], a_t values [nnzA] + a_t structure, l_s/u_s [m],
// d/e/d_inv/e_inv, scal[0..3] = c, c_inv, passes_used, final deviation.
}  // extern "C"
namespace {
template <typename T>
int ruiz_impl(const void* pf, const T* q, const void* a, const T* l, const T* u,
              double eps_equil, uint32_t passes, T* pv, T* qs, T* av, T* atv,
              uint32_t* atrp, uint32_t* atci, T* ls, T* us, T* d, T* e,
              T* dinv, T* einv, double* scal) {
  return guarded([&] {
    const auto P = to_csr<T>(pf);
    const auto A = to_csr<T>(a);
    const auto sp = qpcg::ruiz_equilibrate(P, vec(q, P.rows), A, vec(l, A.rows),
                                           vec(u, A.rows), T(eps_equil), passes);
    std::copy(sp.p_full.values.begin(), sp.p_full.values.end(), pv);
    std::copy(sp.q.begin(), sp.q.end(), qs);
    std::copy(sp.a.values.begin(), sp.a.values.end(), av);
    copy_csr_out(sp.a_t, atv, atrp, atci);
    std::copy(sp.l.begin(), sp.l.end(), ls);
    std::copy(sp.u.begin(), sp.u.end(), us);
    std::copy(sp.scaling.d.begin(), sp.scaling.d.end(), d);
    std::copy(sp.scaling.e.begin(), sp.scaling.e.end(), e);
    std::copy(sp.scaling.d_inv.begin(), sp.scaling.d_inv.end(), dinv);
    std::copy(sp.scaling.e_inv.begin(), sp.scaling.e_inv.end(), einv);
    scal[0] = double(sp.scaling.c);
    scal[1] = double(sp.scaling.c_inv);
    scal[2] = double(sp.passes_used);
    scal[3] = double(sp.final_delta_deviation);
  });
}
}  // namespace
extern "C" {
int qref_ruiz_f64(const qpcg_csr_f64* pf, const double* q, const qpcg_csr_f64* a,
                  const double* l, const double* u, double eps_equil,
                  uint32_t passes, double* pv, double* qs, double* av,
                  double* atv, uint32_t* atrp, uint32_t* atci, double* ls,
                  double* us, double* d, double* e, double* dinv, double* einv,
                  double* scal) {
  return ruiz_impl<double>(pf, q, a, l, u, eps_equil, passes, pv, qs, av, atv,
                           atrp, atci, ls, us, d, e, dinv, einv, scal);
}
int qref_ruiz_f32(const qpcg_csr_f32* pf, const float* q, const qpcg_csr_f32* a,
                  const float* l, const float* u, double eps_equil,
                  uint32_t passes, float* pv, float* qs, float* av, float* atv,
                  uint32_t* atrp, uint32_t* atci, float* ls, float* us, float* d,
                  float* e, float* dinv, float* einv, double* scal) {
  return ruiz_impl<float>(pf, q, a, l, u, eps_equil, passes, pv, qs, av, atv,
                          atrp, atci, ls, us, d, e, dinv, einv, scal);
}

// K x with K = P + sigma I + rho A'A (linsys.hpp:80-90); also returns the
// Jacobi diagonal (linsys.hpp:137-148) in diag_m (may be NULL).
int qref_kkt_apply_f64(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                       const qpcg_csr_f64* at, double sigma, double rho,
                       const double* x, double* out, double* diag_m) {
  return guarded([&] {
    qpcg::ReducedKktOperator<double> op(to_csr<double>(pf), to_csr<double>(a),
                                        to_csr<double>(at), sigma, rho);
    const auto r = op.apply(vec(x, op.dim()));
    std::copy(r.begin(), r.end(), out);
    if (diag_m != nullptr) {
      const auto pre = qpcg::build_preconditioner(op);
      std::copy(pre.diag_m.begin(), pre.diag_m.end(), diag_m);
    }
  });
}

// pcg_solve (linsys.hpp:190-276); res[0] = iterations, res[1] = final
// residual norm, res[2] = converged
int qref_pcg_f64(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                 const qpcg_csr_f64* at, double sigma, double rho,
                 const double* b, const double* warm, double eps,
                 uint32_t max_iter, double* x, double* res) {
  return guarded([&] {
    qpcg::ReducedKktOperator<double> op(to_csr<double>(pf), to_csr<double>(a),
                                        to_csr<double>(at), sigma, rho);
    const auto pre = qpcg::build_preconditioner(op);
    const auto r = qpcg::pcg_solve(op, pre, vec(b, op.dim()),
                                   vec(warm, op.dim()), eps, max_iter);
    std::copy(r.solution.begin(), r.solution.end(), x);
    res[0] = r.iterations;
    res[1] = r.final_residual_norm;
    res[2] = r.converged ? 1.0 : 0.0;
  });
}

int qref_adaptive_eps_f64(double rp, double rd, double lambda, double eps_min,
                          double* out) {
  return guarded([&] { *out = qpcg::adaptive_eps(rp, rd, lambda, eps_min); });
}

uint32_t qref_pcg_cap_f64(uint32_t n) { return qpcg::detail::pcg_iteration_cap<double>(n); }
uint32_t qref_pcg_cap_f32(uint32_t n) { return qpcg::detail::pcg_iteration_cap<float>(n); }

// ---- bounded CPU-baseline sample --------------------------------------------
// Times the reference's own setup phases and hot-path operators on a problem:
// out[0] symmetrize_upper (solver.hpp:397), out[1] transpose_csr (:398),
// out[2] ruiz_equilibrate with max_passes = 1 (scaling.hpp:92-187; includes its
// copies and two transposes), out[3] ReducedKktOperator construction
// (linsys.hpp:39-61), out[4] one K-apply (linsys.hpp:80-90), out[5] one A^T
// spmv (admm_step rhs, solver.hpp:352), out[6] one A spmv (z~ = A x~,
// solver.hpp:360), out[7] compute_residuals (solver.hpp:191-208), out[8] total
// seconds spent in this call.  Operator timings are means over `reps`.
int qref_time_components_f64(const qpcg_csr_f64* p, const double* q,
                             const qpcg_csr_f64* a, const double* l,
                             const double* u, uint32_t reps, double* out) {
  return guarded([&] {
    const double t0 = now_s();
    const auto pu = to_csr<double>(p);
    const auto A = to_csr<double>(a);
    const size_t n = pu.rows, m = A.rows;
    double t = now_s();
    const auto pf = qpcg::symmetrize_upper(pu);
    out[0] = now_s() - t;
    t = now_s();
    const auto at = qpcg::transpose_csr(A);
    out[1] = now_s() - t;
    t = now_s();
    const auto sp = qpcg::ruiz_equilibrate(pf, vec(q, n), A, vec(l, m), vec(u, m),
                                           1e-3, 1);
    out[2] = now_s() - t;
    t = now_s();
    qpcg::ReducedKktOperator<double> op(sp.p_full, sp.a, sp.a_t, 1e-6, 0.1);
    out[3] = now_s() - t;
    std::vector<double> x(n, 1.0), o, zt(m, 1.0), yv(m, 0.5), ax;
    t = now_s();
    for (uint32_t r = 0; r < reps; ++r) op.apply(x, o);
    out[4] = (now_s() - t) / reps;
    t = now_s();
    for (uint32_t r = 0; r < reps; ++r) qpcg::spmv(sp.a_t, zt, o);
    out[5] = (now_s() - t) / reps;
    t = now_s();
    for (uint32_t r = 0; r < reps; ++r) qpcg::spmv(sp.a, x, ax);
    out[6] = (now_s() - t) / reps;
    t = now_s();
    for (uint32_t r = 0; r < reps; ++r) (void)qpcg::compute_residuals(sp, x, zt, yv);
    out[7] = (now_s() - t) / reps;
    out[8] = now_s() - t0;
  });
}

// ---- bench/runner.hpp sweep (the reference's own CSV, runtime included) -----
// Writes run_benchmark + write_csv into out (NUL-terminated, truncated to
// cap); returns the full length or -1 on error.
int64_t qref_run_benchmark_csv(const int* classes, uint32_t n_classes, const uint32_t* scales,
                               uint32_t n_scales, uint32_t instances, uint64_t base_seed,
                               uint32_t threads, const qpcg_settings* s, char* out, size_t cap) {
  try {
    qb::SweepOptions o;
    for (uint32_t i = 0; i < n_classes; ++i) o.classes.push_back(static_cast<qb::ProblemClass>(classes[i]));
    for (uint32_t i = 0; i < n_scales; ++i) o.scales.push_back(scales[i]);
    o.instances_per_size = instances;
    o.base_seed = base_seed;
    o.threads = threads;
    std::ostringstream os;
    qb::write_csv(os, qb::run_benchmark<double>(o, to_settings<double>(s)));
    const std::string csv = os.str();
    if (out && cap) {
      const size_t k = std::min(cap - 1, csv.size());
      std::memcpy(out, csv.data(), k);
      out[k] = 0;
    }
    return int64_t(csv.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
