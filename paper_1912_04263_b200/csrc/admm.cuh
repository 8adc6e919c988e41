// admm.cuh — device control block, deterministic grid reductions and the
// fused ADMM/PCG vector + SpMV-epilogue kernels.
//
// Every scalar decision of the reference loop (solver.hpp:444-514 and
// pcg_solve linsys.hpp:233-269) is taken on the device by the last block of a
// reduction kernel, so the loops run without host synchronisation: in graph
// mode the same kernels also drive CUDA-graph conditional nodes.
#pragma once

#include <cooperative_groups.h>

#include "spmv.cuh"
#include "comm.cuh"

namespace qpcg_b200 {

enum PcgExit : uint32_t { kPcgConverged = 0, kPcgCap = 1, kPcgZeroRhs = 2 };
enum ErrCode : uint32_t { kErrNone = 0, kErrInvalid = 1, kErrNotPD = 2, kErrRho = 3 };

// Device-resident control block (one per workspace).
template <typename T>
struct Ctl {
  // settings (settings.hpp:25-42, in T)
  T alpha, sigma, eps_abs, eps_rel, eps_pinf, eps_dinf, lambda, eps_min;
  uint32_t max_iter, check_interval, rho_interval, pcg_cap;
  // scaling scalars (scaling.hpp:43-56)
  T c, c_inv, q_inf_orig, q_inf_scaled;
  // ADMM state (SolverState, solver.hpp:103-134)
  T rho, pcg_eps, last_rp, last_rd;
  uint32_t iter, done, status, error;
  uint32_t rho_update_count, residuals_current, is_check, admm_continue;
  unsigned long long pcg_total;
  // PCG (linsys.hpp:207-275)
  T b_norm, thr, r_norm, best_norm, rm, alpha_cg, beta, curv;
  uint32_t k, pcg_active, pcg_exit, improved;
  // residual norms: scaled and unscaled (solver.hpp:460-475)
  T rp_s, rd_s, ax_s, z_s, px_s, aty_s;
  T rp_o, rd_o, ax_o, z_o, px_o, aty_o;
  // certificates (solver.hpp:236-297, 318-325)
  T dx_norm, dy_norm, support, qv;
  uint32_t need_pinf, need_dinf, pinf_bad, dinf_bad;
  unsigned long long atv_inf_bits, pv_inf_bits;
  // objective (solver.hpp:525-532)
  T objective;
  // reductions / diagnostics
  uint32_t red_counter, n_calls, n_checks, n_rho;
  uint32_t inf_branch, rho_branch, diag_cap, n_inf, n_rho_branch;
  // z~ = A x~ carried through PCG as z~ += alpha_k (A p_k) (see zt_pass):
  // zt_recur enables it; zt_acc: this PCG solve carries it (decided at its
  // start: the previous solve took <= zt_kmax iterations); k_last: that count
  uint32_t zt_recur, zt_acc, zt_kmax, k_last;
  uint32_t n_zt;  // z~ passes run (graph launch accounting)
  // w = A^T (rho z~) carried alongside z~ (w += alpha_k A^T t_k): w_recur
  // enables it; w_valid: the next rhs pass may take r0's column from w
  uint32_t w_recur, w_valid;
};

// diagnostics records (device side, converted to qpcg_pcg_call on the host)
template <typename T>
struct DiagRec {
  uint32_t admm_iter, iterations;
  T eps, rp, rd;
  uint32_t converged, pad;
};
template <typename T>
struct RhoRec {
  uint32_t admm_iter, pad;
  T before, after;
};

// Handles of the CUDA-graph conditional nodes (0 in eager mode).
struct Handles {
  unsigned long long admm = 0, pcg = 0, chk = 0, inf = 0, rho = 0, zt = 0;
};

__device__ __forceinline__ void set_cond(unsigned long long h, unsigned int v) {
  if (h != 0ull) cudaGraphSetConditional((cudaGraphConditionalHandle)h, v);
}

// Device view of every workspace buffer.
template <typename T>
struct Dev {
  uint32_t n, m;
  Ctl<T>* ctl;
  T* red;  // [kRedBlocks * kMaxQ] reduction partials
  // scaled problem (ScaledProblem, scaling.hpp:57-68)
  DevCsr<T> P, A, AT;
  SpmvPlan<T> pP, pA, pAT;
  T *q, *l, *u, *d, *e, *d_inv, *e_inv;
  // original problem (for infeasibility tests and the objective)
  DevCsr<T> Po, Ao, ATo;
  SpmvPlan<T> pPo, pAo, pATo;
  T *q_o, *l_o, *u_o;
  // iterates
  T *x, *z, *y, *xt, *zt, *dx, *dy;
  // PCG workspace
  T *b, *r, *p, *kp, *best, *dinv, *t, *diag_p, *diag_ata;
  T* ap;  // [m] A p of the current PCG iteration (unscaled by rho), for the z~ recurrence
  T *atp, *w;  // [n] A^T t of the current PCG iteration; carried A^T (rho z~)
  T* g1m;      // [m] rho z - y (the one-column rhs pass's gather)
  // residual workspace (ResidualData, solver.hpp:181-188)
  T *ax, *px, *aty, *rdual;
  // outputs (unscaled)
  T *xo, *zo, *yo, *cert, *pxo;
  // interleaved gather operands of the two-column passes
  pair_t<T>* g2m;  // [m] {rho z - y, rho z~}
  pair_t<T>* g2n;  // [n] {x~, alpha x~ + (1 - alpha) x}
  // diagnostics
  DiagRec<T>* calls;
  uint32_t* checks;
  RhoRec<T>* rhos;
  // row sharding.  split == 0: the fused single-device
  // path.  split == 1: this Dev is one row block of A; the A^T passes write
  // n-partials into `part` and the m-side scalar reductions into `shsc`, the
  // comm combines them across shards, and the *_finish / *_decide kernels
  // consume the combined values (identical on every shard).
  uint32_t split, sh_index, sh_count, pad_sh;
  T* part;  // [2n]
  T* shsc;  // [kShScal]
};

constexpr int kShScal = 16;

constexpr int kMaxQ = 16;

template <typename T>
__host__ __device__ inline uint32_t red_grid(uint32_t len) {
  uint32_t g = (len + kThreads - 1) / kThreads;
  if (g > (uint32_t)kRedBlocks) g = kRedBlocks;
  return g == 0 ? 1u : g;
}

// Grid-stride loop whose loads are issued kLoadAhead strides ahead of their
// use.  The reduction kernels run on the fixed kRedBlocks x kThreads grid
// (deterministic partials), i.e. ~76k threads; with one load per thread in
// flight a 1e6-element vector streams at well under 1 TB/s (svm: 92 us of
// vector kernels per PCG iteration).  ld(i) loads element i's operands, use(i,
// v) consumes them; elements are consumed in exactly the plain loop's order,
// so every result is bitwise unchanged (the persistent driver, which calls
// the same *_elems bodies, stays identical too).
constexpr int kLoadAhead = 4;
template <class Ld, class Use>
__device__ __forceinline__ void strided(uint32_t t0, uint32_t stride, uint32_t n, Ld ld, Use use) {
  uint64_t i = t0;
  const uint64_t st = stride;
  for (; i + (kLoadAhead - 1) * st < n; i += kLoadAhead * st) {
    decltype(ld(0u)) v[kLoadAhead];
#pragma unroll
    for (int u = 0; u < kLoadAhead; ++u) v[u] = ld(uint32_t(i + u * st));
#pragma unroll
    for (int u = 0; u < kLoadAhead; ++u) use(uint32_t(i + u * st), v[u]);
  }
  for (; i < n; i += st) use(uint32_t(i), ld(uint32_t(i)));
}
template <typename T>
struct V2 {
  T a, b;
};
template <typename T>
struct V3 {
  T a, b, c;
};
template <typename T>
struct V4 {
  T a, b, c, d;
};

// Block all-reduce (result in every thread), fixed tree.
template <typename T, bool MAX>
__device__ __forceinline__ T block_allreduce(T v, T* sm) {
  v = MAX ? warp_max(v) : warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  if (w == 0) {
    T r = (l < kWarpsPerBlock) ? sm[l] : T(0);
    r = MAX ? warp_max(r) : warp_sum(r);
    if (l == 0) sm[32] = r;
  }
  __syncthreads();
  return sm[32];
}

// Deterministic grid reduction of NQ quantities (mask bit q set = max, else
// sum).  Returns true in every thread of the last block to arrive, with the
// totals in tot[].  Partials are combined in block-index order.
template <typename T, int NQ>
__device__ bool grid_reduce(const T (&vals)[NQ], uint32_t max_mask, T* part, uint32_t* counter,
                            T (&tot)[NQ]) {
  __shared__ T sm[33];
  __shared__ bool is_last;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool mx = (max_mask >> q) & 1u;
    const T b = mx ? block_allreduce<T, true>(vals[q], sm) : block_allreduce<T, false>(vals[q], sm);
    if (threadIdx.x == 0) part[q * gridDim.x + blockIdx.x] = b;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(counter, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool mx = (max_mask >> q) & 1u;
    T a = T(0);
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      const T v = __ldcg(part + q * gridDim.x + i);
      a = mx ? smax(a, v) : a + v;
    }
    tot[q] = mx ? block_allreduce<T, true>(a, sm) : block_allreduce<T, false>(a, sm);
  }
  if (threadIdx.x == 0) *counter = 0u;
  return true;
}

template <typename T>
__device__ __forceinline__ T tabs(T v) {
  return v < T(0) ? -v : v;
}

// atomicMax over non-negative floating values through their bit patterns
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, double v) {
  atomicMax(a, (unsigned long long)__double_as_longlong(v));
}
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* a, float v) {
  atomicMax(a, (unsigned long long)__float_as_uint(v));
}
__host__ __device__ inline double bits_to_value(unsigned long long b, double) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)b);
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
__host__ __device__ inline float bits_to_value(unsigned long long b, float) {
  const uint32_t u = (uint32_t)b;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}

// Sequential dot of P row r with gathered vector x (spmv of P, one row, in
// stored order: bit-identical to sparse.hpp:289-295 for that row).
template <typename T>
__device__ __forceinline__ T prow_dot(const DevCsr<T>& P, uint32_t r, const T* x) {
  T s = T(0);
  const uint32_t b = P.rp[r], e = P.rp[r + 1];
  for (uint32_t k = b; k < e; ++k) s += P.val[k] * x[P.ci[k]];
  return s;
}

// =====================================================================
// SpMV gathers and epilogues of the loop
// =====================================================================

// rhs pass over A^T (admm_step, solver.hpp:351-355) fused with the PCG r0
// operator apply (linsys.hpp:218-219, 80-90): col0 = rho z - y, col1 = rho z~
// (A x~_prev == z~ from the previous step, reused bit-exactly).
// The two gathered columns are packed by k_pack_rhs into one interleaved
// array so each nnz costs a single 16-byte gather (one L2 sector) instead of
// three scattered 8-byte ones.
template <typename T, bool NC = true>
struct GatherRhs {
  const pair_t<T>* g2;
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ void operator()(uint32_t c, T (&g)[2]) const {
    const pair_t<T> v = ldv<NC>(g2 + c);
    g[0] = v.x;
    g[1] = v.y;
  }
};
// {rho z - y, rho z~} (solver.hpp:351; linsys.hpp:84-85 with A x~ = z~)
// (rhs_one: only rho z - y, the r0 column comes from the carried w)
template <typename T>
__device__ __forceinline__ bool rhs_one(const Ctl<T>* C) {
  return C->w_recur != 0 && C->w_valid != 0;
}
template <typename T>
__device__ __forceinline__ void pack_rhs_elems(const Dev<T>& D, uint32_t t0, uint32_t stride) {
  const T rho = D.ctl->rho;
  if (rhs_one(D.ctl)) {
    for (uint32_t i = t0; i < D.m; i += stride) D.g1m[i] = rho * D.z[i] - D.y[i];
    return;
  }
  for (uint32_t i = t0; i < D.m; i += stride) {
    pair_t<T> v;
    v.x = rho * D.z[i] - D.y[i];
    v.y = rho * D.zt[i];
    D.g2m[i] = v;
  }
}
template <typename T>
__global__ void k_pack_rhs(Dev<T> D) {
  if (D.ctl->error) return;
  pack_rhs_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
template <typename T>
__device__ __forceinline__ void rhs_row(const Dev<T>& D, T sigma, uint32_t r, T s0, T s1) {
  const T rhs = s0 + (sigma * D.x[r] - D.q[r]);
  const T xt = D.xt[r];
  const T kx = (prow_dot(D.P, r, D.xt) + sigma * xt) + s1;
  D.b[r] = rhs;
  D.r[r] = kx - rhs;
}
// two columns: rhs and r0's A^T (rho z~), which also (re)starts the carried w
template <typename T>
struct EpiRhs {
  Dev<T> D;
  T sigma;
  bool keep = false;
  __device__ __forceinline__ bool init() {
    sigma = D.ctl->sigma;
    keep = D.ctl->w_recur != 0;
    return D.ctl->error == 0 && !rhs_one(D.ctl);
  }
  __device__ __forceinline__ void prefetch(uint32_t r) const {
    prefetch_l1(D.x + r);
    prefetch_l1(D.q + r);
    prefetch_l1(D.xt + r);
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[2]) const {
    rhs_row(D, sigma, r, s[0], s[1]);
    if (keep) D.w[r] = s[1];
  }
};
// one column (rho z - y): r0's A^T (rho z~) is the carried w (see zt_pass)
template <typename T>
struct EpiRhs1 {
  Dev<T> D;
  T sigma;
  __device__ __forceinline__ bool init() {
    sigma = D.ctl->sigma;
    return D.ctl->error == 0 && rhs_one(D.ctl);
  }
  __device__ __forceinline__ void prefetch(uint32_t r) const {
    prefetch_l1(D.x + r);
    prefetch_l1(D.q + r);
    prefetch_l1(D.xt + r);
    prefetch_l1(D.w + r);
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const {
    rhs_row(D, sigma, r, s[0], D.w[r]);
  }
};

// t = rho (A p)   (linsys.hpp:84-85); with the z~ recurrence on, A p itself
// is kept as well (ap, read by k_pcg_update once alpha_k is known)
template <typename T>
struct EpiAp {
  T* t;
  T* ap;  // nullptr: not kept
  const Ctl<T>* ctl;
  T rho = T(0);
  bool keep = false;
  __device__ __forceinline__ bool init() {
    rho = ctl->rho;
    keep = ap != nullptr && ctl->zt_acc != 0;
    return ctl->pcg_active != 0 && ctl->error == 0;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const {
    t[r] = s[0] * rho;
    if (keep) ap[r] = s[0];
  }
};

// Kp = (P p + sigma p) + A^T t   (linsys.hpp:86-89)
template <typename T>
__device__ __forceinline__ T kp_row(const Dev<T>& D, T sigma, uint32_t r, T s) {
  return (prow_dot(D.P, r, D.p) + sigma * D.p[r]) + s;
}
template <typename T>
struct EpiKp {
  Dev<T> D;
  T sigma;
  bool keep = false;  // A^T t kept for the carried w
  __device__ __forceinline__ bool init() {
    sigma = D.ctl->sigma;
    keep = D.ctl->w_recur != 0 && D.ctl->zt_acc != 0;
    return D.ctl->pcg_active != 0 && D.ctl->error == 0;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const {
    D.kp[r] = kp_row(D, sigma, r, s[0]);
    if (keep) D.atp[r] = s[0];
  }
};

// Whether the ADMM step needs the z~ pass (z~ = A x~, solver.hpp:359) after
// this PCG solve.  With the recurrence on (Ctl::zt_recur), z~ is carried
// through PCG by linearity: the warm start is the previous x~ whose A x~ is
// the previous z~, and every x_{k+1} = x_k + alpha_k p_k adds alpha_k (A p_k),
// which the PCG A pass has just computed (EpiAp keeps it), so the full
// matrix read of the z~ pass is skipped.  It still runs (and overwrites the
// carried z~ with the directly computed product) on check iterations, where
// the 2-column pass also forms A x_new for the residuals (which therefore stay
// the reference's direct products, and the carried rounding restarts every
// check_interval steps), and when PCG did not return its last iterate (cap:
// best iterate; b == 0: zero).  Carrying costs three m-vector accesses per
// PCG iteration against one A pass per ADMM step, so a solve carries it only
// when the previous solve took at most zt_kmax iterations (the break-even
// count from the sizes, set on the host): the PCG-heavy portfolio steps
// (~120 iterations each) run the pass instead.
template <typename T>
__device__ __forceinline__ bool zt_pass(const Ctl<T>* C) {
  return C->zt_acc == 0 || C->pcg_exit != kPcgConverged ||
         ((C->iter + 1) % C->check_interval) == 0;
}

// z~ = A x~ with the whole m-side ADMM update fused (solver.hpp:360-378);
// col1 (check iterations only) = A x_new with x_new formed on the fly exactly
// as solver.hpp:366-367 forms it, feeding compute_residuals' A x (:196).
template <typename T, bool NC = true>
struct GatherAdmm {  // {x~, x_new} packed by k_pcg_fin
  const pair_t<T>* g2;
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ void operator()(uint32_t c, T (&g)[2]) const {
    const pair_t<T> v = ldv<NC>(g2 + c);
    g[0] = v.x;
    g[1] = v.y;
  }
};
// NCOL 2 on check iterations (col 1 = A x_new for the residuals), NCOL 1 (x~
// only, an 8-byte gather) otherwise.  init() is true only for the build this
// iteration needs: the stand-alone path runs both in one launch
// (spmv_select_kernel), the persistent loop calls both phases.
template <typename T, int NCOL = 2>
struct EpiAdmm {
  Dev<T> D;
  T alpha, one_m_alpha, rho;
  bool two;
  __device__ __forceinline__ bool init() {
    alpha = D.ctl->alpha;
    one_m_alpha = T(1) - alpha;
    rho = D.ctl->rho;
    two = ((D.ctl->iter + 1) % D.ctl->check_interval) == 0;
    return D.ctl->error == 0 && two == (NCOL == 2) && zt_pass(D.ctl);
  }
  __device__ __forceinline__ void prefetch(uint32_t r) const {
    prefetch_l1(D.z + r);
    prefetch_l1(D.y + r);
    prefetch_l1(D.l + r);
    prefetch_l1(D.u + r);
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[NCOL]) const {
    mside(D, alpha, one_m_alpha, rho, r, s[0]);
    if constexpr (NCOL == 2) D.ax[r] = s[1];
  }
  // the m-side update of row r (solver.hpp:369-376) from its z~
  static __device__ __forceinline__ void mside(const Dev<T>& D, T alpha, T one_m_alpha, T rho,
                                               uint32_t r, T zt) {
    const T zp = D.z[r], yp = D.y[r];
    const T w = alpha * zt + one_m_alpha * zp + yp / rho;
    const T zn = smin(smax(w, D.l[r]), D.u[r]);
    const T yn = rho * (w - zn);
    D.zt[r] = zt;
    D.z[r] = zn;
    D.y[r] = yn;
    D.dy[r] = yn - yp;
  }
};

// Plans of short rows (svm's A: 1e6 rows of ~151 entries) run the m-side
// update as a separate row-parallel pass instead of in the SpMV epilogue: the
// epilogue of a warp-per-row item executes on one lane, so 1e6 of them (with
// their IEEE division and 8 scattered accesses) cost ~200 us of issue slots,
// while a thread per row does the same arithmetic coalesced.  The z~ pass
// then only stores z~ (and A x on check iterations); same values, same bits.
template <typename T, int NCOL = 2>
struct EpiAdmmStore {
  Dev<T> D;
  __device__ __forceinline__ bool init() {
    const bool two = ((D.ctl->iter + 1) % D.ctl->check_interval) == 0;
    return D.ctl->error == 0 && two == (NCOL == 2) && zt_pass(D.ctl);
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[NCOL]) const {
    D.zt[r] = s[0];
    if constexpr (NCOL == 2) D.ax[r] = s[1];
  }
};
// always: after an EpiAdmmStore pass (short-row plans); else only when the
// z~ pass was skipped (the fused EpiAdmm epilogue did not run)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_admm_mside(Dev<T> D, bool always) {
  const Ctl<T>* C = D.ctl;
  if (C->error || (!always && zt_pass(C))) return;
  const T alpha = C->alpha, oma = T(1) - alpha, rho = C->rho;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < D.m; j += gridDim.x * blockDim.x)
    EpiAdmm<T, 1>::mside(D, alpha, oma, rho, j, D.zt[j]);
}

// plain store (A x for the initial / final residuals)
template <typename T>
struct EpiStore {
  T* out;
  __device__ __forceinline__ bool init() { return true; }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const { out[r] = s[0]; }
};

// A^T y with P x and r_dual fused (compute_residuals, solver.hpp:197-204)
template <typename T>
__device__ __forceinline__ void dual_row(const Dev<T>& D, uint32_t r, T s) {
  const T px = prow_dot(D.P, r, D.x);
  D.aty[r] = s;
  D.px[r] = px;
  D.rdual[r] = px + D.q[r] + s;
}
template <typename T>
struct EpiDual {
  Dev<T> D;
  __device__ __forceinline__ bool init() { return D.ctl->error == 0; }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const { dual_row(D, r, s[0]); }
};

// certificate vectors formed on the fly (certificate_vectors, solver.hpp:318-325,
// then normalised: check_primal/dual_infeasible :240-243, :275-278)
template <typename T, bool NC = true>
struct GatherCertY {  // v_i = ((e_i dy_i) c_inv) * (1/|dy|)
  const T *e, *dy;
  const Ctl<T>* ctl;
  T c_inv, s;
  __device__ __forceinline__ void init() {
    c_inv = ctl->c_inv;
    s = T(1) / ctl->dy_norm;
  }
  __device__ __forceinline__ void operator()(uint32_t c, T (&g)[1]) const {
    g[0] = ((__ldg(e + c) * ldv<NC>(dy + c)) * c_inv) * s;
  }
};
template <typename T, bool NC = true>
struct GatherCertX {  // v_i = (d_i dx_i) * (1/|dx|)
  const T *d, *dx;
  const Ctl<T>* ctl;
  T s;
  __device__ __forceinline__ void init() { s = T(1) / ctl->dx_norm; }
  __device__ __forceinline__ void operator()(uint32_t c, T (&g)[1]) const {
    g[0] = (__ldg(d + c) * ldv<NC>(dx + c)) * s;
  }
};
template <typename T>
struct EpiNormMax {  // max |row result| into a bits slot (order-free => exact)
  unsigned long long* slot;
  const uint32_t* enable;
  __device__ __forceinline__ bool init() { return *enable != 0; }
  __device__ __forceinline__ void operator()(uint32_t, const T (&s)[1]) const {
    atomic_max_nonneg(slot, tabs(s[0]));
  }
};
template <typename T>
struct EpiDualRows {  // per-row sign tests of check_dual_infeasible (:283-295)
  const T *l, *u;
  uint32_t* bad;
  const uint32_t* enable;
  T eps;
  const Ctl<T>* ctl;
  __device__ __forceinline__ bool init() {
    eps = ctl->eps_dinf;
    return *enable != 0;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const {
    const T li = l[r], ui = u[r], av = s[0];
    const bool lf = li != -(T)INFINITY, uf = ui != (T)INFINITY;
    bool b = false;
    if (lf && uf)
      b = tabs(av) > eps;
    else if (!uf && lf)
      b = av < -eps;
    else if (!lf && uf)
      b = av > eps;
    if (b) atomicOr(bad, 1u);
  }
};

// ---------------------------------------------------------------------
// split (row-sharded) A^T passes: store the shard's n-partials; the comm sums
// them across shards and the finish kernels below apply the epilogue.
// gate: 0 always, 1 while PCG is active, 2 while the primal certificate is
// still possible (need_pinf).
template <typename T, int NCOL>
struct EpiPart {
  T* out;
  const Ctl<T>* ctl;
  uint32_t gate;
  __device__ __forceinline__ bool init() {
    if (ctl->error) return false;
    if (gate == 1) return ctl->pcg_active != 0;
    if (gate == 2) return ctl->inf_branch != 0 && ctl->need_pinf != 0;
    return true;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[NCOL]) const {
#pragma unroll
    for (int j = 0; j < NCOL; ++j) out[(size_t)r * NCOL + j] = s[j];
  }
};

// The fused peer form of EpiPart: the row results go straight into this
// block's slot on EVERY rank (NVLink P2P stores, overlapped with the SpMV),
// so the reduction step is only a barrier and the ordered local sum.
template <typename T, int NCOL>
struct EpiPeer {
  PeerPtrs dst;  // this block's slot (set 0) in every rank's area
  int R;
  const Ctl<T>* ctl;
  uint32_t gate;
  size_t set_bytes;
  const unsigned long long* epoch;  // this rank's barrier epoch: its parity picks the set
  size_t set;
  __device__ __forceinline__ bool init() {
    if (ctl->error) return false;
    set = (p2p_epoch(epoch) & 1ull) * set_bytes;
    if (gate == 1) return ctl->pcg_active != 0;
    return true;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[NCOL]) const {
    for (int q = 0; q < R; ++q) {
      T* o = reinterpret_cast<T*>(dst.p[q] + set) + (size_t)r * NCOL;
#pragma unroll
      for (int j = 0; j < NCOL; ++j) o[j] = s[j];
    }
  }
};

// rhs / r0 from the combined 2-column partials (EpiRhs semantics)
template <typename T>
__global__ void k_rhs_finish(Dev<T> D) {
  const Ctl<T>* C = D.ctl;
  if (C->error) return;
  const T sigma = C->sigma;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x)
    rhs_row(D, sigma, i, D.part[2 * (size_t)i], D.part[2 * (size_t)i + 1]);
}

// A^T y, P x, r_dual from the combined partial (EpiDual semantics)
template <typename T>
__global__ void k_dual_finish(Dev<T> D) {
  if (D.ctl->error) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x)
    dual_row(D, i, D.part[i]);
}

// |A_o^T v|_inf of the combined certificate product (EpiNormMax semantics)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_atv_norm(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (C->error || !C->inf_branch || !C->need_pinf) return;
  T v[1] = {T(0)};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x)
    v[0] = smax(v[0], tabs(D.part[i]));
  T tot[1];
  if (!grid_reduce<T, 1>(v, 0x1u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x == 0) atomic_max_nonneg(&C->atv_inf_bits, tot[0]);
}

// the shard's dual-row flag as a summable scalar
template <typename T>
__global__ void k_flag_to_scal(Dev<T> D) {
  D.shsc[0] = D.ctl->dinf_bad ? T(1) : T(0);
}

// =====================================================================
// vector kernels
//
// Each kernel is an element body (grid-strided from t0 by stride) plus, for
// the reductions, a decision taken by one thread from the reduced totals.
// The stand-alone kernels below wrap them with grid_reduce; the persistent
// loop (persist.cuh) calls the same bodies and decisions between grid
// barriers, so both drivers execute the identical arithmetic.
// =====================================================================

// PCG initialisation (linsys.hpp:203-233) after the fused rhs/r0 pass.
// v: max|b|, max|r|, r.y, #nonfinite(x~)
template <typename T>
__device__ __forceinline__ void pcg_init_elems(const Dev<T>& D, uint32_t t0, uint32_t stride,
                                               T (&v)[4]) {
  strided(t0, stride, D.n,
          [&](uint32_t i) { return V4<T>{D.r[i], D.dinv[i], D.xt[i], D.b[i]}; },
          [&](uint32_t i, const V4<T>& e) {
            const T ri = e.a;
            const T yi = e.b * ri;
            D.p[i] = -yi;
            const T xi = e.c;
            D.best[i] = xi;
            v[0] = smax(v[0], tabs(e.d));
            v[1] = smax(v[1], tabs(ri));
            v[2] += ri * yi;
            if (!isfinite(xi)) v[3] += T(1);
          });
}
template <typename T>
__device__ void pcg_init_decide(Ctl<T>* C, const T (&tot)[4], Handles H) {
  C->k = 0;
  C->improved = 0;
  C->pcg_exit = kPcgConverged;
  C->zt_acc = C->zt_recur != 0 && C->k_last <= C->zt_kmax;
  uint32_t active = 0;
  if (tot[3] != T(0)) {
    C->error = kErrInvalid;  // pcg: warm start must be finite (linsys.hpp:203-205)
    C->done = 1;
  } else if (tot[0] == T(0)) {
    C->pcg_exit = kPcgZeroRhs;  // linsys.hpp:208-213
    C->b_norm = T(0);
  } else {
    C->b_norm = tot[0];
    C->thr = C->pcg_eps * tot[0];
    C->r_norm = tot[1];
    C->best_norm = tot[1];
    C->rm = tot[2];
    active = (C->r_norm > C->thr) && !(C->rm == T(0));
  }
  C->pcg_active = active;
  set_cond(H.pcg, active);
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_init(Dev<T> D, Handles H) {
  Ctl<T>* C = D.ctl;
  if (C->error) return;
  T v[4] = {T(0), T(0), T(0), T(0)};
  pcg_init_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[4];
  if (!grid_reduce<T, 4>(v, 0x3u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  pcg_init_decide(C, tot, H);
}

// curvature p.Kp and step length (linsys.hpp:246-253)
template <typename T>
__device__ __forceinline__ void pcg_dot_elems(const Dev<T>& D, uint32_t t0, uint32_t stride,
                                              T (&v)[1]) {
  if (D.split) {  // Kp = (P p + sigma p) + sum_g A_g^T t_g  (EpiKp semantics)
    const T sigma = D.ctl->sigma;
    for (uint32_t i = t0; i < D.n; i += stride) {
      const T kp = kp_row(D, sigma, i, D.part[i]);
      D.kp[i] = kp;
      v[0] += D.p[i] * kp;
    }
  } else {
    strided(t0, stride, D.n, [&](uint32_t i) { return V2<T>{D.p[i], D.kp[i]}; },
            [&](uint32_t, const V2<T>& e) { v[0] += e.a * e.b; });
  }
}
template <typename T>
__device__ void pcg_dot_decide(Ctl<T>* C, const T (&tot)[1]) {
  C->curv = tot[0];
  if (tot[0] <= T(0)) {
    C->error = kErrNotPD;  // NotPositiveDefiniteError (linsys.hpp:247-250)
    C->done = 1;
    C->pcg_active = 0;
  } else {
    C->alpha_cg = C->rm / tot[0];
  }
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_dot(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (!C->pcg_active || C->error) return;
  T v[1] = {T(0)};
  pcg_dot_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[1];
  if (!grid_reduce<T, 1>(v, 0x0u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  pcg_dot_decide(C, tot);
}

// x += a p; r += a Kp; y = M^-1 r; r.y; |r|  (linsys.hpp:254-263)
template <typename T>
__device__ __forceinline__ void pcg_update_elems(const Dev<T>& D, uint32_t t0, uint32_t stride,
                                                 T (&v)[2]) {
  const T a = D.ctl->alpha_cg;
  strided(t0, stride, D.n,
          [&](uint32_t i) {
            return V4<T>{D.xt[i] + a * D.p[i], D.r[i], D.kp[i], D.dinv[i]};
          },
          [&](uint32_t i, const V4<T>& e) {
            D.xt[i] = e.a;
            const T ri = e.b + a * e.c;
            D.r[i] = ri;
            const T yi = e.d * ri;
            v[0] += ri * yi;
            v[1] = smax(v[1], tabs(ri));
          });
  if (D.ctl->zt_acc) {  // z~ += a (A p)  (zt_pass)
    strided(t0, stride, D.m, [&](uint32_t j) { return V2<T>{D.zt[j], D.ap[j]}; },
            [&](uint32_t j, const V2<T>& e) { D.zt[j] = e.a + a * e.b; });
    if (D.ctl->w_recur)  // w += a (A^T t), i.e. A^T (rho z~) with the same rho
      strided(t0, stride, D.n, [&](uint32_t i) { return V2<T>{D.w[i], D.atp[i]}; },
              [&](uint32_t i, const V2<T>& e) { D.w[i] = e.a + a * e.b; });
  }
}
template <typename T>
__device__ void pcg_update_decide(Ctl<T>* C, const T (&tot)[2], Handles H) {
  const T rm_next = tot[0];
  C->beta = rm_next / C->rm;
  C->rm = rm_next;
  C->k += 1;
  C->r_norm = tot[1];
  C->improved = tot[1] < C->best_norm;
  if (C->improved) C->best_norm = tot[1];
  uint32_t active = C->r_norm > C->thr;
  if (active) {
    if (C->k >= C->pcg_cap) {
      C->pcg_exit = kPcgCap;  // linsys.hpp:235-241: return best iterate
      active = 0;
    } else if (C->rm == T(0)) {
      active = 0;  // linsys.hpp:243
    }
  }
  C->pcg_active = active;
  set_cond(H.pcg, active);
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_update(Dev<T> D, Handles H) {
  Ctl<T>* C = D.ctl;
  if (!C->pcg_active || C->error) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(H.pcg, 0);
    return;
  }
  T v[2] = {T(0), T(0)};
  pcg_update_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[2];
  if (!grid_reduce<T, 2>(v, 0x2u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  pcg_update_decide(C, tot, H);
}

// p = -y + beta p; best-iterate copy (linsys.hpp:259, 264-267)
template <typename T>
__device__ __forceinline__ void pcg_pupdate_elems(const Dev<T>& D, uint32_t t0, uint32_t stride) {
  const Ctl<T>* C = D.ctl;
  if (C->error || C->k == 0) return;  // nothing to do before the first update
  const T beta = C->beta;
  const bool imp = C->improved;
  if (imp) {
    strided(t0, stride, D.n,
            [&](uint32_t i) { return V4<T>{D.dinv[i], D.r[i], D.p[i], D.xt[i]}; },
            [&](uint32_t i, const V4<T>& e) {
              const T yi = e.a * e.b;
              D.p[i] = -yi + beta * e.c;
              D.best[i] = e.d;
            });
  } else {
    strided(t0, stride, D.n, [&](uint32_t i) { return V3<T>{D.dinv[i], D.r[i], D.p[i]}; },
            [&](uint32_t i, const V3<T>& e) {
              const T yi = e.a * e.b;
              D.p[i] = -yi + beta * e.c;
            });
  }
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_pupdate(Dev<T> D) {
  pcg_pupdate_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// The three vector kernels of a PCG iteration (k_pcg_dot, k_pcg_update,
// k_pcg_pupdate) as ONE cooperative kernel on the same fixed reduction grid,
// separated by grid barriers: the same per-thread elements, block trees and
// block-ordered partial sums, so every bit is unchanged (the persistent driver
// and the separate kernels agree with it), minus two launches and two
// last-block round trips per iteration.  Launched cooperatively (all blocks
// co-resident: red_grid() <= 2 per SM), also inside the CUDA graph.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_step(Dev<T> D, Handles H) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  Ctl<T>* C = D.ctl;
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
  if (!C->pcg_active || C->error) {  // (uniform: written by earlier kernels)
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(H.pcg, 0);
    return;
  }
  {  // p . Kp, alpha (k_pcg_dot)
    T v[1] = {T(0)};
    pcg_dot_elems(D, t0, stride, v);
    T tot[1];
    if (grid_reduce<T, 1>(v, 0x0u, D.red, &C->red_counter, tot) && threadIdx.x == 0)
      pcg_dot_decide(C, tot);
  }
  grid.sync();
  if (C->error) {  // NotPositiveDefinite (k_pcg_update's exit)
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(H.pcg, 0);
    return;
  }
  {  // x, r, r.y, |r| (k_pcg_update)
    T v[2] = {T(0), T(0)};
    pcg_update_elems(D, t0, stride, v);
    T tot[2];
    if (grid_reduce<T, 2>(v, 0x2u, D.red, &C->red_counter, tot) && threadIdx.x == 0)
      pcg_update_decide(C, tot, H);
  }
  grid.sync();
  pcg_pupdate_elems(D, t0, stride);  // p, best (k_pcg_pupdate)
}

// PCG exit: x~ = 0 (b == 0) or best iterate (cap); PcgCall record.
// also packs {x~, x_new} for the z~ pass; x_new = alpha x~ + (1 - alpha) x is
// formed exactly as solver.hpp:366-367 (only needed on check iterations).
template <typename T>
__device__ __forceinline__ void pcg_fin_elems(const Dev<T>& D, uint32_t t0, uint32_t stride) {
  const Ctl<T>* C = D.ctl;
  const uint32_t ex = C->pcg_exit;
  const bool two = ((C->iter + 1) % C->check_interval) == 0;
  const T alpha = C->alpha, oma = T(1) - alpha;
  for (uint32_t i = t0; i < D.n; i += stride) {
    T xt = D.xt[i];
    if (ex != kPcgConverged) {
      xt = ex == kPcgZeroRhs ? T(0) : D.best[i];
      D.xt[i] = xt;
    }
    pair_t<T> v;
    v.x = xt;
    v.y = two ? alpha * xt + oma * D.x[i] : T(0);
    D.g2n[i] = v;
  }
}
template <typename T>
__device__ void pcg_fin_book(const Dev<T>& D, bool record) {
  Ctl<T>* C = D.ctl;
  C->pcg_total += C->k;
  C->k_last = C->k;
  const bool pass = zt_pass(C);
  if (pass) C->n_zt += 1;
  // w carried through this whole solve and not restarted by a z~ pass: the
  // next rhs pass takes r0's column from it (a rho change clears it)
  C->w_valid = C->w_recur != 0 && C->zt_acc != 0 && !pass;
  if (record && C->n_calls < C->diag_cap) {
    DiagRec<T> rec;
    rec.admm_iter = C->iter + 1;
    rec.iterations = C->k;
    rec.eps = C->pcg_eps;
    rec.rp = C->last_rp;
    rec.rd = C->last_rd;
    rec.converged = C->pcg_exit != kPcgCap;
    rec.pad = 0;
    D.calls[C->n_calls] = rec;
  }
  C->n_calls += 1;
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_pcg_fin(Dev<T> D, Handles H) {
  if (blockIdx.x == 0 && threadIdx.x == 0)  // the graph's IF node around the z~ pass
    set_cond(H.zt, D.ctl->error == 0 && zt_pass(D.ctl));
  if (D.ctl->error) return;
  pcg_fin_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) pcg_fin_book(D, true);
}

// n-side relaxation (solver.hpp:366-368, 377) and the iteration counter.
template <typename T>
__device__ __forceinline__ void xupdate_elems(const Dev<T>& D, uint32_t t0, uint32_t stride) {
  const T alpha = D.ctl->alpha, oma = T(1) - alpha;
  for (uint32_t i = t0; i < D.n; i += stride) {
    const T xp = D.x[i];
    const T xn = alpha * D.xt[i] + oma * xp;
    D.x[i] = xn;
    D.dx[i] = xn - xp;
  }
}
template <typename T>
__device__ void xupdate_book(Ctl<T>* C, Handles H) {
  const uint32_t it = C->iter + 1;
  C->iter = it;
  C->residuals_current = 0;
  const uint32_t chk = (it % C->check_interval) == 0;
  C->is_check = chk;
  set_cond(H.chk, chk);
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_xupdate(Dev<T> D, Handles H) {
  Ctl<T>* C = D.ctl;
  if (C->error) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(H.chk, 0);
    return;
  }
  xupdate_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
  if (blockIdx.x == 0 && threadIdx.x == 0) xupdate_book(C, H);
}

// Residual bookkeeping, adaptive eps and the termination test from the 14
// reduced norms (solver.hpp:205-206, 222-230, 468-476; linsys.hpp:170-179).
// record: write the check-iteration diagnostics (one writer).
template <typename T>
__device__ void residuals_decide(Dev<T> D, const T (&tot)[14], int mode, Handles H,
                                 bool record = true) {
  Ctl<T>* C = D.ctl;
  const T c_inv = C->c_inv;
  C->rp_s = tot[0];
  C->ax_s = tot[1];
  C->z_s = tot[2];
  C->rd_s = tot[7];
  C->px_s = tot[8];
  C->aty_s = tot[9];
  C->rp_o = tot[3];
  C->ax_o = tot[4];
  C->z_o = tot[5];
  C->rd_o = c_inv * tot[10];
  C->px_o = c_inv * tot[11];
  C->aty_o = c_inv * tot[12];
  C->dy_norm = tot[6];
  C->dx_norm = tot[13];
  C->residuals_current = 1;
  uint32_t inf = 0;
  if (mode != 2) {
    // adaptive_eps (linsys.hpp:170-179)
    const T e = smax(C->lambda * t_sqrt(C->rp_s * C->rd_s), C->eps_min);
    C->pcg_eps = e;
    C->last_rp = C->rp_s;
    C->last_rd = C->rd_s;
  }
  if (mode == 0) {
    if (record && C->n_checks < C->diag_cap) D.checks[C->n_checks] = C->iter;
    C->n_checks += 1;
    // check_optimal (solver.hpp:222-230) on unscaled norms
    const T eps_prim = C->eps_abs + C->eps_rel * smax(C->ax_o, C->z_o);
    const T eps_dual = C->eps_abs + C->eps_rel * smax(smax(C->px_o, C->aty_o), C->q_inf_orig);
    if (C->rp_o <= eps_prim && C->rd_o <= eps_dual) {
      C->status = 0;  // solved
      C->done = 1;
    } else {
      C->need_pinf = C->dy_norm != T(0);
      C->need_dinf = C->dx_norm != T(0);
      C->pinf_bad = 0;
      C->dinf_bad = 0;
      C->atv_inf_bits = 0ull;
      C->pv_inf_bits = 0ull;
      inf = C->need_pinf | C->need_dinf;
    }
  }
  C->inf_branch = inf;
  C->n_inf += inf;
  set_cond(H.inf, inf);
}

// Residual norms (solver.hpp:205-206, 468-475) + termination (:476-495 start).
// mode 0: loop check; mode 1: initial residuals (eps only); mode 2: final.
// v: 0 rp_s 1 ax_s 2 z_s 3 rp_o 4 ax_o 5 z_o 6 dy_norm | 7 rd_s 8 px_s 9 aty_s
//    10 rd_o' 11 px_o' 12 aty_o' 13 dx_norm  (all maxima)
template <typename T>
__device__ __forceinline__ void residuals_elems(const Dev<T>& D, uint32_t t0, uint32_t stride,
                                                T (&v)[14]) {
  const T c_inv = D.ctl->c_inv;
  strided(t0, stride, D.m,
          [&](uint32_t i) {
            return V4<T>{D.ax[i], D.z[i], D.e_inv[i], (D.e[i] * D.dy[i]) * c_inv};
          },
          [&](uint32_t, const V4<T>& e) {
            const T ax = e.a, z = e.b, ei = e.c;
            const T rp = ax - z;
            v[0] = smax(v[0], tabs(rp));
            v[1] = smax(v[1], tabs(ax));
            v[2] = smax(v[2], tabs(z));
            v[3] = smax(v[3], tabs(rp * ei));
            v[4] = smax(v[4], tabs(ax * ei));
            v[5] = smax(v[5], tabs(z * ei));
            v[6] = smax(v[6], tabs(e.d));
          });
  strided(t0, stride, D.n,
          [&](uint32_t i) {
            return V4<T>{D.rdual[i], D.px[i], D.aty[i], D.d[i] * D.dx[i]};
          },
          [&](uint32_t i, const V4<T>& e) {
            const T rd = e.a, px = e.b, aty = e.c, di = D.d_inv[i];
            v[7] = smax(v[7], tabs(rd));
            v[8] = smax(v[8], tabs(px));
            v[9] = smax(v[9], tabs(aty));
            v[10] = smax(v[10], tabs(rd * di));
            v[11] = smax(v[11], tabs(px * di));
            v[12] = smax(v[12], tabs(aty * di));
            v[13] = smax(v[13], tabs(e.d));
          });
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_residuals(Dev<T> D, int mode, Handles H) {
  Ctl<T>* C = D.ctl;
  if (C->error) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_cond(H.inf, 0);
    return;
  }
  T v[14];
#pragma unroll
  for (int q = 0; q < 14; ++q) v[q] = T(0);
  residuals_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[14];
  if (!grid_reduce<T, 14>(v, 0x3fffu, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  if (D.split) {  // shard partials: every entry is a max, combined by the comm
    for (int q = 0; q < 14; ++q) D.shsc[q] = tot[q];
    return;
  }
  residuals_decide(D, tot, mode, H);
}

// split mode: the decision from the combined maxima
template <typename T>
__global__ void k_residuals_decide(Dev<T> D, int mode, Handles H) {
  if (threadIdx.x != 0 || D.ctl->error) return;
  T tot[14];
  for (int q = 0; q < 14; ++q) tot[q] = D.shsc[q];
  residuals_decide(D, tot, mode, H);
}

// Infeasibility tests (solver.hpp:236-297, 481-495).  Both tests are
// conjunctions, so they are evaluated cheapest-first and each A-sized pass
// over the ORIGINAL matrices runs only while its certificate is still
// possible (the SpMV epilogues read need_pinf / need_dinf): same booleans as
// the reference, far fewer matrix streams on ordinary (feasible) solves.
// Stage 1: the vector parts — support sum and infinite-bound tests of the
// primal certificate (:248-263), q'v of the dual one (:281).
// v: support (sum), bad (max; a count across row blocks), q'v (sum)
template <typename T>
__device__ __forceinline__ void infeas_vec_elems(const Dev<T>& D, uint32_t t0, uint32_t stride,
                                                 T (&v)[3]) {
  const Ctl<T>* C = D.ctl;
  const T c_inv = C->c_inv, eps_p = C->eps_pinf;
  const T sy = C->need_pinf ? T(1) / C->dy_norm : T(0);
  const T sx = C->need_dinf ? T(1) / C->dx_norm : T(0);
  if (C->need_pinf) {
    for (uint32_t i = t0; i < D.m; i += stride) {
      const T vi = ((D.e[i] * D.dy[i]) * c_inv) * sy;
      const T neg = smin(vi, T(0)), pos = smax(vi, T(0));
      const T li = D.l_o[i], ui = D.u_o[i];
      if (li == -(T)INFINITY) {
        if (neg < -eps_p) v[1] = T(1);
      } else {
        v[0] += li * neg;
      }
      if (ui == (T)INFINITY) {
        if (pos > eps_p) v[1] = T(1);
      } else {
        v[0] += ui * pos;
      }
    }
  }
  // (n-vectors are replicated across row blocks: block 0 alone sums q'v)
  if (C->need_dinf && (!D.split || D.sh_index == 0)) {
    for (uint32_t i = t0; i < D.n; i += stride) v[2] += D.q_o[i] * ((D.d[i] * D.dx[i]) * sx);
  }
}
template <typename T>
__device__ void infeas_vec_decide(Ctl<T>* C, const T (&tot)[3]) {
  C->support = tot[0];
  C->qv = tot[2];
  if (C->need_pinf && !(tot[1] == T(0) && tot[0] < C->eps_pinf)) C->need_pinf = 0;
  if (C->need_dinf && !(tot[2] < C->eps_dinf)) C->need_dinf = 0;
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_infeas_vec(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (C->error || !C->inf_branch) return;
  T v[3] = {T(0), T(0), T(0)};
  infeas_vec_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[3];
  if (!grid_reduce<T, 3>(v, 0x2u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  if (D.split) {  // partials, combined by a sum (bad: a count, still 0 iff none)
    D.shsc[0] = tot[0];
    D.shsc[1] = tot[1];
    D.shsc[2] = tot[2];
    return;
  }
  infeas_vec_decide(C, tot);
}

template <typename T>
__global__ void k_infeas_vec_decide(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (threadIdx.x != 0 || C->error || !C->inf_branch) return;
  const T tot[3] = {D.shsc[0], D.shsc[1], D.shsc[2]};
  infeas_vec_decide(C, tot);
}

// Stage 2 (after the P_orig pass): |P v| <= eps (:280)
template <typename T>
__device__ void infeas_mid_decide(Ctl<T>* C) {
  if (C->need_dinf && bits_to_value(C->pv_inf_bits, T(0)) > C->eps_dinf) C->need_dinf = 0;
}
template <typename T>
__global__ void k_infeas_mid(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (C->error || !C->inf_branch) return;
  infeas_mid_decide(C);
}

// Stage 3: decision after the A_orig^T (primal) and A_orig (dual) passes
template <typename T>
__device__ void infeas_decide(Ctl<T>* C, bool dual_rows_bad) {
  const bool primal = C->need_pinf && !(bits_to_value(C->atv_inf_bits, T(0)) > C->eps_pinf);
  const bool dual = C->need_dinf && !dual_rows_bad;
  if (primal) {
    C->status = 1;
    C->done = 1;
  } else if (dual) {
    C->status = 2;
    C->done = 1;
  }
}
template <typename T>
__global__ void k_infeas(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (C->error || !C->inf_branch) return;
  infeas_decide(C, D.split ? D.shsc[0] != T(0) : C->dinf_bad != 0);
}

// decides the rho branch (solver.hpp:498)
template <typename T>
__device__ void rho_flag_book(Ctl<T>* C, Handles H) {
  const uint32_t f = !C->error && !C->done && (C->iter % C->rho_interval) == 0;
  C->rho_branch = f;
  C->n_rho_branch += f;
  set_cond(H.rho, f);
}
template <typename T>
__global__ void k_rho_flag(Dev<T> D, Handles H) {
  rho_flag_book(D.ctl, H);
}

// adapt_rho (solver.hpp:302-314) from the last residuals and the current |z|.
// record: write the rho-update diagnostics (one writer).
template <typename T>
__device__ void rho_decide(Dev<T> D, T z_inf, bool record = true) {
  Ctl<T>* C = D.ctl;
  const T fl = T(1e-10);
  const T rel_prim = C->last_rp / smax(smax(C->ax_s, z_inf), fl);
  const T rel_dual = C->last_rd / smax(smax(smax(C->px_s, C->aty_s), C->q_inf_scaled), fl);
  const T rho = C->rho;
  T next;
  if (rel_prim == T(0) && rel_dual == T(0))
    next = rho;
  else if (rel_dual == T(0))
    next = T(1e6);
  else {
    next = rho * t_sqrt(rel_prim / rel_dual);
    if (next < T(1e-6)) next = T(1e-6);
    else if (T(1e6) < next) next = T(1e6);
  }
  if (record && C->n_rho < C->diag_cap) {
    RhoRec<T> rr;
    rr.admm_iter = C->iter;
    rr.pad = 0;
    rr.before = rho;
    rr.after = next;
    D.rhos[C->n_rho] = rr;
  }
  C->n_rho += 1;
  C->w_valid = 0;  // w = A^T (rho z~) holds the old rho
  if (!(next > T(0))) {
    C->error = kErrRho;  // kkt operator: rho must be positive
    C->done = 1;
    return;
  }
  C->rho = next;
  C->rho_update_count += 1;
}
template <typename T>
__device__ __forceinline__ void rho_elems(const Dev<T>& D, uint32_t t0, uint32_t stride, T (&v)[1]) {
  strided(t0, stride, D.m, [&](uint32_t i) { return D.z[i]; },
          [&](uint32_t, T z) { v[0] = smax(v[0], tabs(z)); });
}
template <typename T>
__global__ void __launch_bounds__(kThreads) k_rho(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  if (!C->rho_branch) return;
  T v[1] = {T(0)};
  rho_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, v);
  T tot[1];
  if (!grid_reduce<T, 1>(v, 0x1u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  if (D.split) {  // this block's max |z|, combined by a max
    D.shsc[0] = tot[0];
    return;
  }
  rho_decide(D, tot[0]);
}
template <typename T>
__global__ void k_rho_decide(Dev<T> D) {
  if (threadIdx.x != 0 || !D.ctl->rho_branch) return;
  rho_decide(D, D.shsc[0]);
}

// Jacobi diagonal (linsys.hpp:142-146): (diag_p + sigma) + rho diag_ata
template <typename T>
__device__ __forceinline__ void precond_elems(const Dev<T>& D, uint32_t t0, uint32_t stride) {
  const T sigma = D.ctl->sigma, rho = D.ctl->rho;
  for (uint32_t i = t0; i < D.n; i += stride) {
    const T dm = D.diag_p[i] + sigma + rho * D.diag_ata[i];
    D.dinv[i] = T(1) / dm;
  }
}
template <typename T>
__global__ void k_precond(Dev<T> D, int force) {
  const Ctl<T>* C = D.ctl;
  if (!force && !C->rho_branch) return;
  if (C->error) return;
  precond_elems(D, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// loop condition (solver.hpp:444)
template <typename T>
__device__ __forceinline__ uint32_t admm_go(const Ctl<T>* C) {
  return !C->done && !C->error && C->iter < C->max_iter;
}
template <typename T>
__global__ void k_admm_cond(Dev<T> D, Handles H) {
  Ctl<T>* C = D.ctl;
  const uint32_t go = admm_go(C);
  C->admm_continue = go;
  set_cond(H.admm, go);
}

// unscale_solution (scaling.hpp:209-222) and the certificate (solver.hpp:485, 491)
template <typename T>
__global__ void k_unscale(Dev<T> D) {
  const Ctl<T>* C = D.ctl;
  const T c_inv = C->c_inv;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = t0; i < D.n; i += stride) D.xo[i] = D.d[i] * D.x[i];
  for (uint32_t i = t0; i < D.m; i += stride) {
    D.zo[i] = D.e_inv[i] * D.z[i];
    D.yo[i] = (D.e[i] * D.y[i]) * c_inv;
  }
  if (C->status == 1) {
    const T s = T(1) / C->dy_norm;
    for (uint32_t i = t0; i < D.m; i += stride) D.cert[i] = ((D.e[i] * D.dy[i]) * c_inv) * s;
  } else if (C->status == 2) {
    const T s = T(1) / C->dx_norm;
    for (uint32_t i = t0; i < D.n; i += stride) D.cert[i] = (D.d[i] * D.dx[i]) * s;
  }
}

// objective = 0.5 x'(P x) + q'x on the original data (solver.hpp:530-531)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_objective(Dev<T> D) {
  Ctl<T>* C = D.ctl;
  T v[2] = {T(0), T(0)};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x) {
    v[0] += D.xo[i] * D.pxo[i];
    v[1] += D.q_o[i] * D.xo[i];
  }
  T tot[2];
  if (!grid_reduce<T, 2>(v, 0x0u, D.red, &C->red_counter, tot)) return;
  if (threadIdx.x != 0) return;
  if (C->status == 1)
    C->objective = (T)INFINITY;
  else if (C->status == 2)
    C->objective = -(T)INFINITY;
  else
    C->objective = T(0.5) * tot[0] + tot[1];
}

// max-norm helper (q_inf etc.)
template <typename T>
__global__ void __launch_bounds__(kThreads) k_infnorm(const T* v, uint32_t n, T* part,
                                                     uint32_t* counter, T* out,
                                                     const uint32_t* act = nullptr) {
  if (act && !*act) return;  // (an inactive Ruiz pass)
  T a[1] = {T(0)};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    a[0] = smax(a[0], tabs(v[i]));
  T tot[1];
  if (!grid_reduce<T, 1>(a, 0x1u, part, counter, tot)) return;
  if (threadIdx.x == 0) *out = tot[0];
}

}  // namespace qpcg_b200
