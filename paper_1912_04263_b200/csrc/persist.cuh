// persist.cuh — the whole ADMM/PCG loop (solver.hpp:444-514, pcg_solve
// linsys.hpp:233-269) as ONE cooperative kernel: the small-problem latency
// path.
//
// Below ~1e6 nonzeros a matrix pass reads an L2-resident matrix in a few
// microseconds, so the graph path's ~13 kernels per ADMM step and 5 per PCG
// iteration (each a launch plus a conditional-node round trip) dominate.
// Here one grid of co-resident blocks walks the same phases separated by grid
// barriers:
//   * the phases call the SAME element bodies, SpMV item/row routines and
//     decision functions as the stand-alone kernels (admm.cuh, spmv.cuh);
//   * every reduction emulates the stand-alone launch geometry (virtual
//     blocks of red_grid(len) x kThreads threads, the same per-thread strides,
//     the same block tree and the same in-order combination of the block
//     partials), so the persistent, graph and eager drivers are bitwise
//     identical;
//   * each block keeps its own copy of the control block in shared memory and
//     takes every decision itself from the (identical) reduced totals, so a
//     decision costs no extra barrier; block 0 writes the diagnostics and the
//     final control block back;
//   * gathered vectors are read with coherent loads (they are rewritten
//     between barriers of this kernel); the matrices stay on the read-only
//     streaming path.
#pragma once

#include <cooperative_groups.h>

#include "admm.cuh"

namespace qpcg_b200 {

namespace cgp = cooperative_groups;

template <typename T>
struct PersistBufs {
  T* part;            // [2][kMaxQ * kMaxVirtual] ping-pong reduction partials
  Ctl<T>* gctl;       // the global control block (atomic slots of the infeasibility passes)
};
constexpr uint32_t kMaxVirtual = 2 * kNumSMs;  // red_grid() never exceeds kRedBlocks

// The barrier between phases: the whole grid (cooperative launch, one or two
// blocks per SM) or one thread-block cluster (up to 16 SMs, hardware barrier:
// the tiny-problem variant, where barrier latency is the whole cost).
// rank() / count(): this block among the blocks solving the instance.
// kL1: the matrices are read through the L1 (one SM holds the whole instance,
// so after the first pass they are served on-chip; the grid variants stream
// them past L1 like the stand-alone kernels).
struct GridSync {
  cgp::grid_group g;
  static constexpr bool kL1 = false;
  __device__ GridSync() : g(cgp::this_grid()) {}
  __device__ __forceinline__ void sync() { g.sync(); }
  __device__ __forceinline__ uint32_t rank() const { return blockIdx.x; }
  __device__ __forceinline__ uint32_t count() const { return gridDim.x; }
};
struct ClusterSync {
  static constexpr bool kL1 = false;
  __device__ __forceinline__ void sync() { cgp::this_cluster().sync(); }
  __device__ __forceinline__ uint32_t rank() const { return blockIdx.x; }
  __device__ __forceinline__ uint32_t count() const { return gridDim.x; }
};
// one block = one instance: __syncthreads barriers, L1-resident matrices
struct BlockSync {
  static constexpr bool kL1 = true;
  __device__ __forceinline__ void sync() { __syncthreads(); }
  __device__ __forceinline__ uint32_t rank() const { return 0u; }
  __device__ __forceinline__ uint32_t count() const { return 1u; }
};

// Reduction with the stand-alone kernels' geometry: virtual block vb of
// Gv = red_grid(len) covers threads vb*kThreads + tid with stride Gv*kThreads.
template <typename T, int NQ, typename F, class Sync>
__device__ __forceinline__ void preduce(F&& elems, uint32_t len, uint32_t max_mask, T* part,
                                        Sync& grid, T (&tot)[NQ]) {
  __shared__ T sm[33];
  const uint32_t Gv = red_grid<T>(len);
  for (uint32_t vb = grid.rank(); vb < Gv; vb += grid.count()) {
    T v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = T(0);
    elems(vb * kThreads + threadIdx.x, Gv * kThreads, v);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const bool mx = (max_mask >> q) & 1u;
      const T b = mx ? block_allreduce<T, true>(v[q], sm) : block_allreduce<T, false>(v[q], sm);
      if (threadIdx.x == 0) part[q * Gv + vb] = b;
    }
  }
  grid.sync();
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const bool mx = (max_mask >> q) & 1u;
    T a = T(0);
    for (uint32_t i = threadIdx.x; i < Gv; i += blockDim.x) {
      const T v = __ldcg(part + q * Gv + i);
      a = mx ? smax(a, v) : a + v;
    }
    tot[q] = mx ? block_allreduce<T, true>(a, sm) : block_allreduce<T, false>(a, sm);
  }
}

// One SpMV pass over the plan with the whole grid (warps stride the items,
// threads stride the short rows); same per-item / per-row arithmetic as
// spmv_kernel.
template <typename T, int NCOL, class Op, class Gather, class Epi, class Sync>
__device__ __forceinline__ void spmv_phase(const Sync& sy, const DevCsr<T>& M,
                                           const SpmvPlan<T>& P, Gather gather, Epi epi) {
  if (!epi.init()) return;
  gather.init();
  const uint32_t t0 = sy.rank() * blockDim.x + threadIdx.x, stride = sy.count() * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t it = t0 >> 5; it < P.n_items; it += stride >> 5) {
    if (P.off16 != nullptr)
      spmv_item<T, NCOL, Op, Gather, Epi, 8, true, Sync::kL1>(M, P, gather, epi, it, lane);
    else
      spmv_item<T, NCOL, Op, Gather, Epi, 4, false, Sync::kL1>(M, P, gather, epi, it, lane);
  }
  for (uint32_t idx = t0; idx < P.n_short; idx += stride)
    spmv_short<T, NCOL, Op, Gather, Epi, Sync::kL1>(M, P, gather, epi, idx);
}

template <typename T, class Sync>
__global__ void __launch_bounds__(kThreads, 2) k_admm_persistent(Dev<T> Dg, PersistBufs<T> B) {
  Sync grid;
  __shared__ Ctl<T> sctl;
  if (threadIdx.x == 0) sctl = *Dg.ctl;
  __syncthreads();
  Dev<T> D = Dg;
  D.ctl = &sctl;
  Ctl<T>* C = &sctl;
  const Handles H{};
  const bool rec = grid.rank() == 0;  // the one writer of diagnostics records
  const uint32_t t0 = grid.rank() * blockDim.x + threadIdx.x, stride = grid.count() * blockDim.x;
  uint32_t pp = 0;
  auto part = [&]() { return B.part + (pp++ & 1u) * (kMaxQ * kMaxVirtual); };
  const uint32_t nm = D.n > D.m ? D.n : D.m;

  while (admm_go(C)) {
    // ---- rhs + r0 (solver.hpp:351-355, linsys.hpp:218-219)
    if (!C->error) pack_rhs_elems(D, t0, stride);
    grid.sync();
    spmv_phase<T, 2, SumOp>(grid, D.AT, D.pAT, GatherRhs<T, false>{D.g2m}, EpiRhs<T>{D, T(0)});
    spmv_phase<T, 1, SumOp>(grid, D.AT, D.pAT, GatherVec<T, false>{D.g1m}, EpiRhs1<T>{D, T(0)});
    grid.sync();
    if (!C->error) {  // k_pcg_init
      T tot[4];
      preduce<T, 4>([&](uint32_t a, uint32_t b, T(&v)[4]) { pcg_init_elems(D, a, b, v); }, D.n,
                    0x3u, part(), grid, tot);
      if (threadIdx.x == 0) pcg_init_decide(C, tot, H);
      __syncthreads();
    }
    // ---- PCG iterations
    while (C->pcg_active && !C->error) {
      spmv_phase<T, 1, SumOp>(grid, D.A, D.pA, GatherVec<T, false>{D.p}, EpiAp<T>{D.t, D.ap, C});
      grid.sync();
      spmv_phase<T, 1, SumOp>(grid, D.AT, D.pAT, GatherVec<T, false>{D.t}, EpiKp<T>{D, T(0)});
      grid.sync();
      {
        T tot[1];
        preduce<T, 1>([&](uint32_t a, uint32_t b, T(&v)[1]) { pcg_dot_elems(D, a, b, v); }, D.n,
                      0x0u, part(), grid, tot);
        if (threadIdx.x == 0) pcg_dot_decide(C, tot);
        __syncthreads();
      }
      if (C->pcg_active && !C->error) {
        T tot[2];
        preduce<T, 2>([&](uint32_t a, uint32_t b, T(&v)[2]) { pcg_update_elems(D, a, b, v); },
                      D.n, 0x2u, part(), grid, tot);
        if (threadIdx.x == 0) pcg_update_decide(C, tot, H);
        __syncthreads();
      }
      pcg_pupdate_elems(D, t0, stride);
      grid.sync();
    }
    // ---- exit of PCG, z~ pass with the m-side update, n-side relaxation
    if (!C->error) {
      pcg_fin_elems(D, t0, stride);
      __syncthreads();
      if (threadIdx.x == 0) pcg_fin_book(D, rec);
      __syncthreads();
    }
    grid.sync();
    spmv_phase<T, 2, SumOp>(grid, D.A, D.pA, GatherAdmm<T, false>{D.g2n},
                            EpiAdmm<T, 2>{D, T(0), T(0), T(0), false});
    spmv_phase<T, 1, SumOp>(grid, D.A, D.pA, GatherVec<T, false>{D.xt},
                            EpiAdmm<T, 1>{D, T(0), T(0), T(0), false});
    if (!C->error && !zt_pass(C)) {  // z~ carried through PCG: the m-side update alone
      const T alpha = C->alpha, oma = T(1) - alpha, rho = C->rho;
      for (uint32_t j = t0; j < D.m; j += stride) EpiAdmm<T, 1>::mside(D, alpha, oma, rho, j, D.zt[j]);
    }
    grid.sync();
    if (!C->error) {
      xupdate_elems(D, t0, stride);
      __syncthreads();
      if (threadIdx.x == 0) xupdate_book(C, H);
      __syncthreads();
    }
    grid.sync();
    // ---- termination check (solver.hpp:458-496)
    if (C->is_check && !C->error) {
      spmv_phase<T, 1, SumOp>(grid, D.AT, D.pAT, GatherVec<T, false>{D.y}, EpiDual<T>{D});
      grid.sync();
      {
        T tot[14];
        preduce<T, 14>([&](uint32_t a, uint32_t b, T(&v)[14]) { residuals_elems(D, a, b, v); },
                       nm, 0x3fffu, part(), grid, tot);
        if (threadIdx.x == 0) residuals_decide(D, tot, 0, H, rec);
        __syncthreads();
      }
      if (C->inf_branch) {
        // atomic slots of the certificate passes live in the global block
        if (grid.rank() == 0 && threadIdx.x == 0) {
          B.gctl->atv_inf_bits = 0ull;
          B.gctl->pv_inf_bits = 0ull;
          B.gctl->dinf_bad = 0u;
        }
        {
          T tot[3];
          preduce<T, 3>([&](uint32_t a, uint32_t b, T(&v)[3]) { infeas_vec_elems(D, a, b, v); },
                        nm, 0x2u, part(), grid, tot);
          if (threadIdx.x == 0) infeas_vec_decide(C, tot);
          __syncthreads();
        }
        spmv_phase<T, 1, SumOp>(grid, D.ATo, D.pATo, GatherCertY<T, false>{D.e, D.dy, C, T(0), T(0)},
                                EpiNormMax<T>{&B.gctl->atv_inf_bits, &C->need_pinf});
        spmv_phase<T, 1, SumOp>(grid, D.Po, D.pPo, GatherCertX<T, false>{D.d, D.dx, C, T(0)},
                                EpiNormMax<T>{&B.gctl->pv_inf_bits, &C->need_dinf});
        grid.sync();
        if (threadIdx.x == 0) {
          C->atv_inf_bits = __ldcg(&B.gctl->atv_inf_bits);
          C->pv_inf_bits = __ldcg(&B.gctl->pv_inf_bits);
          infeas_mid_decide(C);
        }
        __syncthreads();
        spmv_phase<T, 1, SumOp>(grid, 
            D.Ao, D.pAo, GatherCertX<T, false>{D.d, D.dx, C, T(0)},
            EpiDualRows<T>{D.l_o, D.u_o, &B.gctl->dinf_bad, &C->need_dinf, T(0), C});
        grid.sync();
        if (threadIdx.x == 0) {
          C->dinf_bad = __ldcg(&B.gctl->dinf_bad);
          infeas_decide(C, C->dinf_bad != 0);
        }
        __syncthreads();
      }
    }
    // ---- rho adaptation (solver.hpp:498-513)
    if (threadIdx.x == 0) rho_flag_book(C, H);
    __syncthreads();
    if (C->rho_branch) {
      T tot[1];
      preduce<T, 1>([&](uint32_t a, uint32_t b, T(&v)[1]) { rho_elems(D, a, b, v); }, D.m, 0x1u,
                    part(), grid, tot);
      if (threadIdx.x == 0) rho_decide(D, tot[0], rec);
      __syncthreads();
      if (!C->error) precond_elems(D, t0, stride);
      grid.sync();
    }
  }
  if (grid.rank() == 0 && threadIdx.x == 0) {
    C->admm_continue = 0;
    *Dg.ctl = sctl;
  }
}

}  // namespace qpcg_b200
