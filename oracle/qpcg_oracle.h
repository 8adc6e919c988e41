/*
 * oracle/qpcg_oracle.h — TEST INFRASTRUCTURE ONLY (parity checker).
 *
 * Plain-C restatement of the reference's ADMM/PCG solve path
 * (/root/reference/proj/include/qpcg/{sparse,scaling,linsys,solver}.hpp).
 * Parity status: PINNED — tests/test_oracle_pin.py checks it bit-for-bit
 * against the reference itself (oracle/_ref/libqpcg_ref.so, built from the
 * unmodified reference headers) and against the SPEC.md known-answer tests.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker / CPU baseline — never as the
 * product path.
 */
#ifndef QPCG_ORACLE_H
#define QPCG_ORACLE_H

#include <stdint.h>

#include "qpcg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* oracle_last_error(void);

/* full solve, solver.hpp:386-541; same argument meaning as qpcg_fXX_solve_problem */
int oracle_f64_solve(const qpcg_csr_f64* p_upper, const double* q,
                     const qpcg_csr_f64* a, const double* l, const double* u,
                     const qpcg_settings* s, const double* wx, const double* wz,
                     const double* wy, qpcg_info* info, double* x, double* z,
                     double* y, double* cert, int record_diag);
int oracle_f32_solve(const qpcg_csr_f32* p_upper, const float* q,
                     const qpcg_csr_f32* a, const float* l, const float* u,
                     const qpcg_settings* s, const float* wx, const float* wz,
                     const float* wy, qpcg_info* info, float* x, float* z,
                     float* y, float* cert, int record_diag);
uint32_t oracle_diag_pcg_calls(qpcg_pcg_call* out, uint32_t cap);
uint32_t oracle_diag_rho_updates(qpcg_rho_update* out, uint32_t cap);
uint32_t oracle_diag_checks(uint32_t* out, uint32_t cap);

/* building blocks */
int oracle_f64_spmv(const qpcg_csr_f64* m, const double* x, double* y);
int oracle_f32_spmv(const qpcg_csr_f32* m, const float* x, float* y);
int oracle_f64_transpose(const qpcg_csr_f64* m, double* vals, uint32_t* rp,
                         uint32_t* ci);
int64_t oracle_f64_symmetrize(const qpcg_csr_f64* m, double* vals,
                              uint32_t* rp, uint32_t* ci);
int oracle_f64_ruiz(const qpcg_csr_f64* pf, const double* q,
                    const qpcg_csr_f64* a, const double* l, const double* u,
                    double eps_equil, uint32_t passes, double* pv, double* qs,
                    double* av, double* atv, uint32_t* atrp, uint32_t* atci,
                    double* ls, double* us, double* d, double* e, double* dinv,
                    double* einv, double* scal);
int oracle_f32_ruiz(const qpcg_csr_f32* pf, const float* q,
                    const qpcg_csr_f32* a, const float* l, const float* u,
                    double eps_equil, uint32_t passes, float* pv, float* qs,
                    float* av, float* atv, uint32_t* atrp, uint32_t* atci,
                    float* ls, float* us, float* d, float* e, float* dinv,
                    float* einv, double* scal);
int oracle_f64_kkt_apply(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                         const qpcg_csr_f64* at, double sigma, double rho,
                         const double* x, double* out, double* diag_m);
int oracle_f64_pcg(const qpcg_csr_f64* pf, const qpcg_csr_f64* a,
                   const qpcg_csr_f64* at, double sigma, double rho,
                   const double* b, const double* warm, double eps,
                   uint32_t max_iter, double* x, double* res);
int oracle_f64_adaptive_eps(double rp, double rd, double lambda,
                            double eps_min, double* out);
uint32_t oracle_pcg_cap_f64(uint32_t n);
uint32_t oracle_pcg_cap_f32(uint32_t n);

#ifdef __cplusplus
}
#endif

#endif /* QPCG_ORACLE_H */
