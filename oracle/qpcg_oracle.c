/*
 * oracle/qpcg_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker / CPU
 * baseline "port").  Plain-C restatement of the reference solve path; see
 * qpcg_oracle.h for the pinning status and the usage restriction.
 * The precision-generic body lives in qpcg_oracle_body.inc.
 */
#define _POSIX_C_SOURCE 199309L
#include "qpcg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];

static int fail_code(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
static int fail(const char* msg) { return fail_code(QPCG_ERR_INVALID, msg); }

const char* oracle_last_error(void) { return g_err; }

static void* xcalloc(size_t n, size_t sz) {
  void* p = calloc(n, sz);
  if (p == NULL) {
    fprintf(stderr, "oracle: out of memory\n");
    abort();
  }
  return p;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* settings.hpp:25-42 defaults */
static void qpcg_default_settings_local(qpcg_settings* s) {
  memset(s, 0, sizeof(*s));
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

/* ---- SolveDiagnostics (solver.hpp:148-167) of the last solve ---------- */
static _Thread_local qpcg_pcg_call* g_calls;
static _Thread_local uint32_t g_ncalls, g_capcalls;
static _Thread_local qpcg_rho_update* g_rho;
static _Thread_local uint32_t g_nrho, g_caprho;
static _Thread_local uint32_t* g_checks;
static _Thread_local uint32_t g_nchecks, g_capchecks;

static void diag_reset(void) { g_ncalls = g_nrho = g_nchecks = 0; }

#define DIAG_PUSH(arr, n, cap, type, val)                               \
  do {                                                                  \
    if ((n) == (cap)) {                                                 \
      (cap) = (cap) ? 2 * (cap) : 256;                                  \
      (arr) = (type*)realloc((arr), sizeof(type) * (cap));              \
    }                                                                   \
    (arr)[(n)++] = (val);                                               \
  } while (0)

static void diag_pcg_call(uint32_t it, uint32_t pit, double eps, double rp,
                          double rd, int conv) {
  qpcg_pcg_call c;
  memset(&c, 0, sizeof(c));
  c.admm_iter = it;
  c.iterations = pit;
  c.eps = eps;
  c.r_prim_scaled_inf = rp;
  c.r_dual_scaled_inf = rd;
  c.converged = conv;
  DIAG_PUSH(g_calls, g_ncalls, g_capcalls, qpcg_pcg_call, c);
}
static void diag_check(uint32_t it) {
  DIAG_PUSH(g_checks, g_nchecks, g_capchecks, uint32_t, it);
}
static void diag_rho(uint32_t it, double before, double after) {
  qpcg_rho_update r;
  memset(&r, 0, sizeof(r));
  r.admm_iter = it;
  r.rho_before = before;
  r.rho_after = after;
  DIAG_PUSH(g_rho, g_nrho, g_caprho, qpcg_rho_update, r);
}

uint32_t oracle_diag_pcg_calls(qpcg_pcg_call* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_ncalls; ++i) out[i] = g_calls[i];
  return g_ncalls;
}
uint32_t oracle_diag_rho_updates(qpcg_rho_update* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_nrho; ++i) out[i] = g_rho[i];
  return g_nrho;
}
uint32_t oracle_diag_checks(uint32_t* out, uint32_t cap) {
  for (uint32_t i = 0; i < cap && i < g_nchecks; ++i) out[i] = g_checks[i];
  return g_nchecks;
}

/* ---- instantiate the body for double and float ------------------------ */
#define T double
#define S(name) f64_##name
#define SQRT sqrt
#define FABS fabs
#define CEIL ceil
typedef qpcg_csr_f64 f64_view;
#include "qpcg_oracle_body.inc"
#undef T
#undef S
#undef SQRT
#undef FABS
#undef CEIL

#define T float
#define S(name) f32_##name
#define SQRT sqrtf
#define FABS fabsf
#define CEIL ceilf
typedef qpcg_csr_f32 f32_view;
#include "qpcg_oracle_body.inc"
#undef T
#undef S
#undef SQRT
#undef FABS
#undef CEIL

/* ---- exported entry points -------------------------------------------- */
int oracle_f64_solve(const qpcg_csr_f64* p, const double* q, const qpcg_csr_f64* a,
                     const double* l, const double* u, const qpcg_settings* s,
                     const double* wx, const double* wz, const double* wy,
                     qpcg_info* info, double* x, double* z, double* y,
                     double* cert, int record_diag) {
  return f64_solve(p, q, a, l, u, s, wx, wz, wy, info, x, z, y, cert, record_diag);
}
int oracle_f32_solve(const qpcg_csr_f32* p, const float* q, const qpcg_csr_f32* a,
                     const float* l, const float* u, const qpcg_settings* s,
                     const float* wx, const float* wz, const float* wy,
                     qpcg_info* info, float* x, float* z, float* y, float* cert,
                     int record_diag) {
  return f32_solve(p, q, a, l, u, s, wx, wz, wy, info, x, z, y, cert, record_diag);
}

int oracle_f64_spmv(const qpcg_csr_f64* v, const double* x, double* y) {
  f64_csr m;
  f64_csr_from_view(&m, v);
  f64_spmv(&m, x, y);
  f64_csr_free(&m);
  return QPCG_OK;
}
int oracle_f32_spmv(const qpcg_csr_f32* v, const float* x, float* y) {
  f32_csr m;
  f32_csr_from_view(&m, v);
  f32_spmv(&m, x, y);
  f32_csr_free(&m);
  return QPCG_OK;
}

static void out_csr_f64(const f64_csr* m, double* vals, uint32_t* rp, uint32_t* ci) {
  if (vals) memcpy(vals, m->values, sizeof(double) * m->nnz);
  if (rp) memcpy(rp, m->row_ptr, sizeof(uint32_t) * ((size_t)m->rows + 1));
  if (ci) memcpy(ci, m->col, sizeof(uint32_t) * m->nnz);
}
static void out_csr_f32(const f32_csr* m, float* vals, uint32_t* rp, uint32_t* ci) {
  if (vals) memcpy(vals, m->values, sizeof(float) * m->nnz);
  if (rp) memcpy(rp, m->row_ptr, sizeof(uint32_t) * ((size_t)m->rows + 1));
  if (ci) memcpy(ci, m->col, sizeof(uint32_t) * m->nnz);
}

int oracle_f64_transpose(const qpcg_csr_f64* v, double* vals, uint32_t* rp,
                         uint32_t* ci) {
  f64_csr m, t;
  f64_csr_from_view(&m, v);
  f64_transpose(&m, &t);
  out_csr_f64(&t, vals, rp, ci);
  f64_csr_free(&m);
  f64_csr_free(&t);
  return QPCG_OK;
}

int64_t oracle_f64_symmetrize(const qpcg_csr_f64* v, double* vals, uint32_t* rp,
                              uint32_t* ci) {
  f64_csr m, f;
  f64_csr_from_view(&m, v);
  int rc = f64_symmetrize_upper(&m, &f);
  f64_csr_free(&m);
  if (rc != QPCG_OK) return -(int64_t)rc;
  int64_t nnz = f.nnz;
  if (vals) out_csr_f64(&f, vals, rp, ci);
  f64_csr_free(&f);
  return nnz;
}

#define RUIZ_EXPORT(SUF, TT, OUTCSR)                                            \
  int oracle_##SUF##_ruiz(const qpcg_csr_##SUF* pf, const TT* q,                \
                          const qpcg_csr_##SUF* a, const TT* l, const TT* u,    \
                          double eps_equil, uint32_t passes, TT* pv, TT* qs,    \
                          TT* av, TT* atv, uint32_t* atrp, uint32_t* atci,      \
                          TT* ls, TT* us, TT* d, TT* e, TT* dinv, TT* einv,     \
                          double* scal) {                                       \
    SUF##_csr P, A;                                                             \
    SUF##_scaled sp;                                                            \
    SUF##_csr_from_view(&P, pf);                                                \
    SUF##_csr_from_view(&A, a);                                                 \
    int rc = SUF##_ruiz(&P, q, &A, l, u, (TT)eps_equil, passes, &sp);           \
    if (rc == QPCG_OK) {                                                        \
      const uint32_t n = P.rows, m = A.rows;                                    \
      memcpy(pv, sp.p_full.values, sizeof(TT) * sp.p_full.nnz);                 \
      memcpy(qs, sp.q, sizeof(TT) * n);                                         \
      memcpy(av, sp.a.values, sizeof(TT) * sp.a.nnz);                           \
      OUTCSR(&sp.a_t, atv, atrp, atci);                                         \
      memcpy(ls, sp.l, sizeof(TT) * m);                                         \
      memcpy(us, sp.u, sizeof(TT) * m);                                         \
      memcpy(d, sp.d, sizeof(TT) * n);                                          \
      memcpy(e, sp.e, sizeof(TT) * m);                                          \
      memcpy(dinv, sp.d_inv, sizeof(TT) * n);                                   \
      memcpy(einv, sp.e_inv, sizeof(TT) * m);                                   \
      scal[0] = (double)sp.c;                                                   \
      scal[1] = (double)sp.c_inv;                                               \
      scal[2] = (double)sp.passes_used;                                         \
      scal[3] = (double)sp.final_delta_deviation;                               \
      SUF##_scaled_free(&sp);                                                   \
    }                                                                           \
    SUF##_csr_free(&P);                                                         \
    SUF##_csr_free(&A);                                                         \
    return rc;                                                                  \
  }
RUIZ_EXPORT(f64, double, out_csr_f64)
RUIZ_EXPORT(f32, float, out_csr_f32)

int oracle_f64_kkt_apply(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                         const qpcg_csr_f64* at, double sigma, double rho,
                         const double* x, double* out, double* diag_m) {
  f64_csr P, A, AT;
  f64_op op;
  f64_csr_from_view(&P, pf);
  f64_csr_from_view(&A, a);
  f64_csr_from_view(&AT, at);
  int rc = f64_op_init(&op, &P, &A, &AT, sigma, rho);
  if (rc == QPCG_OK) {
    f64_op_apply(&op, x, out);
    if (diag_m) memcpy(diag_m, op.diag_m, sizeof(double) * P.rows);
    f64_op_free(&op);
  }
  f64_csr_free(&P);
  f64_csr_free(&A);
  f64_csr_free(&AT);
  return rc;
}

int oracle_f64_pcg(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                   const qpcg_csr_f64* at, double sigma, double rho,
                   const double* b, const double* warm, double eps,
                   uint32_t max_iter, double* x, double* res) {
  f64_csr P, A, AT;
  f64_op op;
  f64_csr_from_view(&P, pf);
  f64_csr_from_view(&A, a);
  f64_csr_from_view(&AT, at);
  int rc = f64_op_init(&op, &P, &A, &AT, sigma, rho);
  if (rc == QPCG_OK) {
    uint32_t it = 0;
    double fn = 0;
    int conv = 0;
    memcpy(x, warm, sizeof(double) * P.rows);
    rc = f64_pcg(&op, b, x, eps, max_iter, &it, &fn, &conv);
    res[0] = it;
    res[1] = fn;
    res[2] = conv;
    f64_op_free(&op);
  }
  f64_csr_free(&P);
  f64_csr_free(&A);
  f64_csr_free(&AT);
  return rc;
}

int oracle_f64_adaptive_eps(double rp, double rd, double lambda, double eps_min,
                            double* out) {
  return f64_adaptive_eps(rp, rd, lambda, eps_min, out);
}

uint32_t oracle_pcg_cap_f64(uint32_t n) { return f64_pcg_cap(n); }
uint32_t oracle_pcg_cap_f32(uint32_t n) { return f32_pcg_cap(n); }
