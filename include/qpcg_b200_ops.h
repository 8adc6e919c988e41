/*
 * qpcg_b200_ops.h — operator-level C-ABI of the B200 engine.
 *
 * Mirrors the reference's operator-level sub-API that SPEC.md and its tests
 * exercise: spmv (sparse.hpp:283-303), the scaled problem
 * produced by setup (symmetrize_upper sparse.hpp:237-281, transpose_csr
 * :207-232, ruiz_equilibrate scaling.hpp:92-187), the reduced-KKT operator
 * (ReducedKktOperator::apply linsys.hpp:80-90) and its Jacobi diagonal
 * (build_preconditioner linsys.hpp:137-148).  Used by the parity tests and by
 * bench.py's kernel timing; host pointers throughout.
 */
#ifndef QPCG_B200_OPS_H
#define QPCG_B200_OPS_H

#include "qpcg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* y = M x on the device (plan-driven SpMV kernel), host arrays in/out */
int qpcg_f64_op_spmv(const qpcg_csr_f64* m, const double* x, double* y, int device);
int qpcg_f32_op_spmv(const qpcg_csr_f32* m, const float* x, float* y, int device);

/* pcg_solve (linsys.hpp:190-276) on the ReducedKktOperator built from
 * (p_full, a, a_t, sigma, rho) (linsys.hpp:39-61; a_t must equal
 * transpose_csr(a) bit for bit) with its Jacobi preconditioner
 * (linsys.hpp:137-148), run by the engine's own PCG kernels.  x[n] receives
 * the solution; res[0..2] = iterations, final residual norm (the best one on
 * an iteration-cap exit), converged (0/1).  QPCG_ERR_NOT_PD on a direction
 * of nonpositive curvature; QPCG_ERR_INVALID on the reference's argument
 * errors (eps <= 0, dimensions, non-finite warm start, a_t mismatch). */
int qpcg_f64_op_pcg(const qpcg_csr_f64* p_full, const qpcg_csr_f64* a, const qpcg_csr_f64* a_t,
                    double sigma, double rho, const double* b, const double* warm, double eps,
                    uint32_t max_iter, double* x, double* res, int device);
int qpcg_f32_op_pcg(const qpcg_csr_f32* p_full, const qpcg_csr_f32* a, const qpcg_csr_f32* a_t,
                    double sigma, double rho, const float* b, const float* warm, double eps,
                    uint32_t max_iter, float* x, double* res, int device);

/* dims[0..5] = n, m, nnz(P full), nnz(A), equil passes, 0 */
int qpcg_debug_dims(const qpcg_workspace* ws, uint64_t* dims);

/* The scaled problem held by the workspace (ScaledProblem, scaling.hpp:57-68)
 * plus the structures built at setup.  Arrays sized by qpcg_debug_dims;
 * scal[0..3] = c, c_inv, passes_used, final deviation.  Any pointer may be
 * NULL.  Values are T (double for f64 workspaces, float for f32). */
int qpcg_debug_scaled(const qpcg_workspace* ws, void* p_values, uint32_t* p_row_ptr,
                      uint32_t* p_col, void* q, void* a_values, void* at_values,
                      uint32_t* at_row_ptr, uint32_t* at_col, void* l, void* u, void* d,
                      void* e, double* scal);

/* K x with the workspace's current rho (linsys.hpp:80-90) and the Jacobi
 * inverse diagonal (linsys.hpp:145) */
int qpcg_debug_operator(qpcg_workspace* ws, const void* x, void* kx, void* diag_m_inv);

/* Times `reps` launches each of the PCG-iteration kernels on the workspace's
 * stream with CUDA events.  out[0] ms per A pass (t = rho A p), out[1] ms per
 * A^T pass (Kp = P p + sigma p + A^T t), out[2] ms per whole PCG iteration
 * (the path the solve uses), out[3..5] algorithmic bytes of each (SURVEY
 * §8(d): 4-byte column indices), out[6..8] the same with the bytes of the
 * matrix formats actually streamed (16-bit compressed column offsets where
 * used).  qpcg_bench_kernels writes these 9 doubles; qpcg_bench_kernels_n
 * writes min(cap, QPCG_BENCH_KERNELS_MAX) and adds out[9] ms per one-pass
 * kernel k_gram (csrc/gram.cuh, opt-in; 0 when off), out[10] its bytes,
 * out[11] the bytes of a whole PCG iteration on that path. */
#define QPCG_BENCH_KERNELS_MAX 12
int qpcg_bench_kernels(qpcg_workspace* ws, uint32_t reps, double* out);
int qpcg_bench_kernels_n(qpcg_workspace* ws, uint32_t reps, double* out, uint32_t cap);

#ifdef __cplusplus
}
#endif

#endif /* QPCG_B200_OPS_H */
