// spmv.cuh — deterministic, skew-robust CSR SpMV for sm_100a.
//
// Reference semantics: `spmv` (sparse.hpp:283-303), y[r] = sum_k val[k] *
// x[col[k]].  The reference sums each row left to right; here:
//   * rows with <= kShortRowMax nnz ("S bin") run one thread per row and sum
//     left to right — bit-identical to the reference for those rows;
//   * longer rows are cut into work items of <= 2^P.chunk_log2 nnz ("W bin"), one
//     warp per item, lanes striding the item with coalesced loads; lanes
//     combine with a fixed xor-butterfly and multi-item rows combine their
//     per-item partials in item order.  The order is fixed per matrix, so
//     results are reproducible run to run.
// The plan (bins + items) is built once on the device at setup from row_ptr
// alone (row-length statistics), so A, A^T and P of any
// skew (portfolio: one 141k-nnz row next to 141k one-nnz rows; svm A^T: 1000
// rows of 151k) are load-balanced by the hardware block scheduler.
//
// The kernel is templated on
//   NCOL   number of gathered vectors sharing one pass over the matrix
//          (e.g. A^T (rho z - y) and A^T (rho z~) in one stream, SURVEY §7
//          hard part 4b),
//   Op     SumOp (dot of row with gathered vectors) or MaxAbsOp (row_inf_norms,
//          sparse.hpp:324-330),
//   Gather functor producing the NCOL gathered values for a column index,
//   Epi    functor consuming (row, sums[NCOL]) — the fused epilogue.
#pragma once

#include <cub/cub.cuh>

#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"

namespace qpcg_b200 {

struct WorkItem {
  uint32_t row, beg, end, lr;  // lr: long-row index, UINT32_MAX if single item
};

template <typename T>
struct SpmvPlan {
  uint32_t n_items = 0, n_short = 0, n_long = 0, n_partials = 0;
  uint32_t nb_items = 0, nb_short = 0;
  WorkItem* items = nullptr;    // [n_items], longest first
  uint32_t* short_rows = nullptr;  // [n_short], increasing row order
  uint2* lrinfo = nullptr;      // [n_long] {partial base, item count}
  T* partials = nullptr;        // [n_partials * kMaxCols]
  uint32_t* counters = nullptr; // [n_long], zero between launches
  // Compressed column indices of the work items (plan_compress).  An item is
  // read by its warp 32 consecutive entries of one row at a time (strictly
  // increasing columns); chunk j of item it has id c0[it] + j and
  //   cbase[id] = first column,  col[k] = cbase[id] + off16[k]   (span < 2^16)
  //   cbase[id] = kWide | w,     col    = wide[32 w + lane]        (otherwise)
  // so the streams carry 2 index bytes per entry instead of 4.  off16 is
  // indexed by entry position; short rows keep the uint32 ci.
  uint16_t* off16 = nullptr;
  uint32_t* cbase = nullptr;
  uint32_t* c0 = nullptr;
  uint32_t* wide = nullptr;
  uint32_t n_chunks = 0, n_wide = 0;
  uint32_t chunk_log2 = 12;  // work items hold <= 2^chunk_log2 nnz (plan_chunk_log2)
  // uncompressed plans whose items average 97..255 entries (svm's A: 151)
  // run the U = 8 build: one predicated round of 8 strides covers an item,
  // where U = 4 needs a full round plus a dependent tail round (same
  // arithmetic, same results)
  uint32_t u8 = 0;
  uint32_t grid() const { return nb_items + nb_short; }
};

constexpr uint32_t kWide = 0x80000000u;
constexpr uint32_t kLongItemMean = 256;  // mean entries per item to compress / unroll 8

constexpr int kMaxCols = 3;

// ------------------------------------------------------------------ ops
struct SumOp {
  template <typename T>
  __device__ __forceinline__ static void acc(T& a, T v, T g) { a += v * g; }
  template <typename T>
  __device__ __forceinline__ static T warp(T a) { return warp_sum(a); }
  template <typename T>
  __device__ __forceinline__ static T join(T a, T b) { return a + b; }
  static constexpr bool kNeedsGather = true;
};
struct MaxAbsOp {
  template <typename T>
  __device__ __forceinline__ static void acc(T& a, T v, T) {
    T x = v < T(0) ? -v : v;
    a = x > a ? x : a;
  }
  template <typename T>
  __device__ __forceinline__ static T warp(T a) { return warp_max(a); }
  template <typename T>
  __device__ __forceinline__ static T join(T a, T b) { return b > a ? b : a; }
  static constexpr bool kNeedsGather = false;
};

// gather helpers
// gathered loads: read-only path (NC) in the stand-alone kernels; plain
// (coherent) loads inside the persistent loop, where the gathered vectors are
// rewritten between grid barriers of the same kernel
template <bool NC, typename V>
__device__ __forceinline__ V ldv(const V* p) {
  if constexpr (NC) return __ldg(p);
  else return *p;
}
template <typename T, bool NC = true>
struct GatherVec {  // x[c]
  const T* __restrict__ x;
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ void operator()(uint32_t c, T (&g)[1]) const { g[0] = ldv<NC>(x + c); }
};
template <typename T, int N>
struct GatherNone {
  __device__ __forceinline__ void init() {}
  __device__ __forceinline__ void operator()(uint32_t, T (&g)[N]) const {
#pragma unroll
    for (int j = 0; j < N; ++j) g[j] = T(0);
  }
};

__device__ __forceinline__ uint16_t ld_stream(const uint16_t* p) {
  unsigned short v;
  asm volatile(QPCG_LD_Q ".u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}

// One warp, one work item: lanes stride the item 32 entries at a time
// (coalesced), U strides in flight; the last < 32U entries in one predicated
// step.  CMP: columns from the compressed index (SpmvPlan::off16).
// L1: read the matrix through the L1 (the one-SM persistent variant, whose
// whole instance stays on-chip); otherwise stream it past L1.
template <bool L1, typename V>
__device__ __forceinline__ V ld_mat(const V* p) {
  if constexpr (L1) return __ldg(p);
  else return ld_stream(p);
}

template <typename T, int NCOL, class Op, class Gather, int U, bool CMP, bool L1 = false>
__device__ __forceinline__ void item_loop(const DevCsr<T>& M, const SpmvPlan<T>& P,
                                          const Gather& gather, const WorkItem& item, uint32_t c0,
                                          uint32_t lane, T (&acc)[NCOL]) {
  const T* __restrict__ val = M.val;
  const uint32_t* __restrict__ ci = M.ci;
  uint32_t k = item.beg + lane;
  const uint32_t end = item.end;
  uint32_t ch = c0;  // chunk id of the entries at k (CMP)
  // column of stride u: plain load, or base (shuffled from lane u) + offset
  auto load_col = [&](uint32_t kk, uint32_t bl, int u, bool ok, uint32_t& c, uint16_t& o,
                      uint32_t& b) {
    if (!CMP) {
      c = ok ? ld_mat<L1>(ci + kk) : 0u;
    } else {
      b = __shfl_sync(0xffffffffu, bl, u);
      o = ok ? ld_mat<L1>(P.off16 + kk) : (uint16_t)0;
    }
  };
  auto col_of = [&](uint32_t c, uint16_t o, uint32_t b) -> uint32_t {
    if (!CMP) return c;
    return (b & kWide) ? __ldg(P.wide + 32u * (b & ~kWide) + lane) : b + o;
  };
  for (; k + 32u * (U - 1) < end; k += 32u * U, ch += U) {
    uint32_t c[U], b[U];
    uint16_t o[U];
    T v[U];
    const uint32_t bl = (CMP && lane < (uint32_t)U) ? __ldg(P.cbase + ch + lane) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = ld_mat<L1>(val + k + 32u * u);
      if (Op::kNeedsGather) load_col(k + 32u * u, bl, u, true, c[u], o[u], b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      T g[NCOL];
      if (Op::kNeedsGather) gather(col_of(c[u], o[u], b[u]), g);
#pragma unroll
      for (int j = 0; j < NCOL; ++j) Op::acc(acc[j], v[u], Op::kNeedsGather ? g[j] : T(0));
    }
  }
  const uint32_t kf = k - lane;  // first entry of the remaining strides
  if (kf < end) {  // the < 32U remaining entries: one predicated step, all loads in flight
    uint32_t c[U], b[U];
    uint16_t o[U];
    T v[U];
    const uint32_t nch = (end - kf + 31u) / 32u;
    const uint32_t bl = (CMP && lane < nch) ? __ldg(P.cbase + ch + lane) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k + 32u * u < end;
      v[u] = ok ? ld_mat<L1>(val + k + 32u * u) : T(0);
      if (Op::kNeedsGather) load_col(k + 32u * u, bl, u, ok, c[u], o[u], b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (k + 32u * u < end) {
        T g[NCOL];
        if (Op::kNeedsGather) gather(col_of(c[u], o[u], b[u]), g);
#pragma unroll
        for (int j = 0; j < NCOL; ++j) Op::acc(acc[j], v[u], Op::kNeedsGather ? g[j] : T(0));
      }
    }
  }
}

// --------------------------------------------------------------- kernel
// End of a work item: warp-reduce the lane sums, then the epilogue (single
// item) or the deterministic combine of a multi-item row.
template <typename T, int NCOL, class Op, class Epi>
__device__ __forceinline__ void item_finish(const DevCsr<T>& M, const SpmvPlan<T>& P, const Epi& epi,
                                            const WorkItem& item, uint32_t lane, T (&acc)[NCOL]) {
#pragma unroll
  for (int j = 0; j < NCOL; ++j) acc[j] = Op::warp(acc[j]);
  if (item.lr == 0xffffffffu) {
    if (lane == 0) epi(item.row, acc);
    return;
  }
  // publish the partial; the release/acquire counter increment orders it
  // before the last arriver's reads
  uint32_t prev = 0;
  const uint2 info = P.lrinfo[item.lr];
  if (lane == 0) {
    const uint32_t chunk = (item.beg - M.rp[item.row]) >> P.chunk_log2;
    T* part = P.partials + (size_t)(info.x + chunk) * kMaxCols;
#pragma unroll
    for (int j = 0; j < NCOL; ++j) part[j] = acc[j];
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                 : "=r"(prev) : "l"(P.counters + item.lr) : "memory");
  }
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != info.y - 1) return;
  __syncwarp();
  // last arriver: the lanes load the partials in parallel, lane 0 joins them
  // in item order (the same order as a sequential loop: bitwise stable)
  T tot[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; ++j) tot[j] = T(0);
  for (uint32_t q0 = 0; q0 < info.y; q0 += 32) {
    T pv[NCOL];
    const uint32_t q = q0 + lane;
    const T* pp = P.partials + (size_t)(info.x + q) * kMaxCols;
#pragma unroll
    for (int j = 0; j < NCOL; ++j) pv[j] = q < info.y ? __ldcg(pp + j) : T(0);
    const uint32_t cnt = min(32u, info.y - q0);
    for (uint32_t t = 0; t < cnt; ++t) {
#pragma unroll
      for (int j = 0; j < NCOL; ++j) {
        const T v = __shfl_sync(0xffffffffu, pv[j], t);
        tot[j] = Op::join(tot[j], v);
      }
    }
  }
  if (lane != 0) return;
  P.counters[item.lr] = 0u;
  epi(item.row, tot);
}

// Epilogues that read per-row operands (the m-side ADMM update, the rhs and
// K p rows) expose prefetch(row): lane 0 of a single-item row issues it at
// the start of the item, so those loads travel while the row streams instead
// of after the warp reduction (svm: 1e6 rows of 151 entries, 4 operand loads
// each).
template <class E, class = void>
struct HasPrefetch : std::false_type {};
template <class E>
struct HasPrefetch<E, std::void_t<decltype(std::declval<const E&>().prefetch(0u))>>
    : std::true_type {};
__device__ __forceinline__ void prefetch_l1(const void* p) {
#ifndef QPCG_NO_PREFETCH
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#else
  (void)p;
#endif
}

// One work item (one warp; lane 0 runs the epilogue).  Multi-item rows
// publish a partial; the last item to arrive combines them in item order
// (deterministic).
template <typename T, int NCOL, class Op, class Gather, class Epi, int U, bool CMP,
          bool L1 = false, bool PF = false>
__device__ __forceinline__ void spmv_item_run(const DevCsr<T>& M, const SpmvPlan<T>& P,
                                              const Gather& gather, const Epi& epi,
                                              const WorkItem& item, uint32_t c0, uint32_t lane) {
  // (PF: stand-alone kernels only; the persistent loop rewrites these vectors
  // between grid barriers and keeps to plain loads)
  if constexpr (PF && HasPrefetch<Epi>::value) {
    if (lane == 0 && item.lr == 0xffffffffu) epi.prefetch(item.row);
  }
  T acc[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; ++j) acc[j] = T(0);
  item_loop<T, NCOL, Op, Gather, U, CMP && Op::kNeedsGather, L1>(M, P, gather, item, c0, lane, acc);
  item_finish<T, NCOL, Op, Epi>(M, P, epi, item, lane, acc);
}
template <typename T, int NCOL, class Op, class Gather, class Epi, int U, bool CMP,
          bool L1 = false, bool PF = false>
__device__ __forceinline__ void spmv_item(const DevCsr<T>& M, const SpmvPlan<T>& P,
                                          const Gather& gather, const Epi& epi, uint32_t it,
                                          uint32_t lane) {
  spmv_item_run<T, NCOL, Op, Gather, Epi, U, CMP, L1, PF>(M, P, gather, epi, P.items[it],
                                                          CMP ? P.c0[it] : 0u, lane);
}

// One short row (<= kShortRowMax nnz), one thread, left to right: bit-exact.
template <typename T, int NCOL, class Op, class Gather, class Epi, bool L1 = false>
__device__ __forceinline__ void spmv_short(const DevCsr<T>& M, const SpmvPlan<T>& P,
                                           const Gather& gather, const Epi& epi, uint32_t idx) {
  const uint32_t r = P.short_rows[idx];
  const uint32_t b = __ldg(M.rp + r), e = __ldg(M.rp + r + 1);
  T acc[NCOL];
#pragma unroll
  for (int j = 0; j < NCOL; ++j) acc[j] = T(0);
  for (uint32_t k = b; k < e; ++k) {
    const T v = ld_mat<L1>(M.val + k);
    T g[NCOL];
    if (Op::kNeedsGather) gather(ld_mat<L1>(M.ci + k), g);
#pragma unroll
    for (int j = 0; j < NCOL; ++j) Op::acc(acc[j], v, Op::kNeedsGather ? g[j] : T(0));
  }
  epi(r, acc);
}

// Two builds of the kernel (registers are per kernel, so they are separate
// kernels rather than branches): U = 8 strides in flight with the compressed
// index for plans of long items (the latency-bound streams of A / A^T), and
// U = 4 with uint32 columns for plans of short items, where occupancy wins.
// One item per warp, blocks handed out in item order by the hardware: a
// grid-stride walk of resident warps over the items (descriptor prefetch)
// measured 1.6x slower on the lasso A pass — the warps drift apart and the
// in-flight rows stop sharing column windows and DRAM pages.
template <typename T, int NCOL, class Op, class Gather, class Epi, int U, bool CMP>
__global__ void __launch_bounds__(kThreads) spmv_kernel(DevCsr<T> M, SpmvPlan<T> P, Gather gather,
                                                       Epi epi) {
  // functors load their device-resident scalars (rho, flags) once per thread;
  // an inactive epilogue (e.g. a skipped certificate pass) exits immediately
  if (!epi.init()) return;
  gather.init();
  if (blockIdx.x < P.nb_items) {
    const uint32_t it = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (it < P.n_items)
      spmv_item<T, NCOL, Op, Gather, Epi, U, CMP, false, true>(M, P, gather, epi, it, threadIdx.x & 31);
  } else {
    const uint32_t idx = (blockIdx.x - P.nb_items) * kThreads + threadIdx.x;
    if (idx < P.n_short) spmv_short<T, NCOL, Op, Gather, Epi>(M, P, gather, epi, idx);
  }
}

// Two passes over the same matrix of which at most one is active per launch
// (an epilogue whose init() is false is inactive), in one kernel: the active
// one runs exactly as in spmv_kernel.  Saves the full-grid launch of the
// inactive pass (~10 us for 12k exiting blocks), e.g. the z~ pass's 1- and
// 2-column builds.
template <typename T, int N1, class G1, class E1, int N2, class G2, class E2, int U, bool CMP>
__global__ void __launch_bounds__(kThreads) spmv_select_kernel(DevCsr<T> M, SpmvPlan<T> P, G1 g1,
                                                              E1 e1, G2 g2, E2 e2) {
  auto run = [&](auto& gather, auto& epi, auto ncol) {
    constexpr int NCOL = decltype(ncol)::value;
    using Gather = std::remove_reference_t<decltype(gather)>;
    using Epi = std::remove_reference_t<decltype(epi)>;
    gather.init();
    if (blockIdx.x < P.nb_items) {
      const uint32_t it = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
      if (it < P.n_items)
        spmv_item<T, NCOL, SumOp, Gather, Epi, U, CMP, false, true>(M, P, gather, epi, it,
                                                                    threadIdx.x & 31);
    } else {
      const uint32_t idx = (blockIdx.x - P.nb_items) * kThreads + threadIdx.x;
      if (idx < P.n_short) spmv_short<T, NCOL, SumOp, Gather, Epi>(M, P, gather, epi, idx);
    }
  };
  if (e2.init()) run(g2, e2, std::integral_constant<int, N2>{});
  else if (e1.init()) run(g1, e1, std::integral_constant<int, N1>{});
}

template <typename T, int N1, class G1, class E1, int N2, class G2, class E2>
void launch_spmv_select(const DevCsr<T>& M, const SpmvPlan<T>& P, const G1& g1, const E1& e1,
                        const G2& g2, const E2& e2, cudaStream_t s) {
  if (P.grid() == 0) return;
  if (P.off16 != nullptr)
    spmv_select_kernel<T, N1, G1, E1, N2, G2, E2, 8, true><<<P.grid(), kThreads, 0, s>>>(M, P, g1, e1,
                                                                                         g2, e2);
  else if (P.u8)
    spmv_select_kernel<T, N1, G1, E1, N2, G2, E2, 8, false><<<P.grid(), kThreads, 0, s>>>(M, P, g1,
                                                                                          e1, g2, e2);
  else
    spmv_select_kernel<T, N1, G1, E1, N2, G2, E2, 4, false><<<P.grid(), kThreads, 0, s>>>(M, P, g1, e1,
                                                                                          g2, e2);
  CK_LAUNCH();
}

template <typename T, int NCOL, class Op, class Gather, class Epi>
void launch_spmv(const DevCsr<T>& M, const SpmvPlan<T>& P, const Gather& g, const Epi& e,
                 cudaStream_t s) {
  if (P.grid() == 0) return;
  if (P.off16 != nullptr)
    spmv_kernel<T, NCOL, Op, Gather, Epi, 8, true><<<P.grid(), kThreads, 0, s>>>(M, P, g, e);
  else if (P.u8)
    spmv_kernel<T, NCOL, Op, Gather, Epi, 8, false><<<P.grid(), kThreads, 0, s>>>(M, P, g, e);
  else
    spmv_kernel<T, NCOL, Op, Gather, Epi, 4, false><<<P.grid(), kThreads, 0, s>>>(M, P, g, e);
  CK_LAUNCH();
}

// ------------------------------------------------------------ plan build
static __global__ void plan_classify_kernel(const uint32_t* __restrict__ rp, uint32_t rows,
                                            uint32_t chunk,
                                     uint32_t* is_short, uint32_t* nch, uint32_t* is_multi,
                                     uint32_t* multi_nch) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const uint32_t len = rp[r + 1] - rp[r];
    const uint32_t s = len <= kShortRowMax;
    const uint32_t c = s ? 0u : ceil_div(len, chunk);
    is_short[r] = s;
    nch[r] = c;
    is_multi[r] = c > 1;
    multi_nch[r] = c > 1 ? c : 0u;
  }
}

static __global__ void plan_emit_kernel(const uint32_t* __restrict__ rp, uint32_t rows,
                                        uint32_t chunk,
                                 const uint32_t* is_short, const uint32_t* short_pos,
                                 const uint32_t* nch, const uint32_t* item_off,
                                 const uint32_t* lr_idx, const uint32_t* pbase,
                                 uint32_t* short_rows, WorkItem* items, uint32_t* item_len,
                                 uint2* lrinfo, int by_chunk) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    if (is_short[r]) {
      short_rows[short_pos[r]] = r;
      continue;
    }
    const uint32_t c = nch[r], b = rp[r], e = rp[r + 1];
    const uint32_t lr = c > 1 ? lr_idx[r] : 0xffffffffu;
    if (c > 1) lrinfo[lr] = make_uint2(pbase[r], c);
    for (uint32_t q = 0; q < c; ++q) {
      WorkItem w;
      w.row = r;
      w.beg = b + q * chunk;
      w.end = min(e, w.beg + chunk);
      w.lr = lr;
      items[item_off[r] + q] = w;
      // sort key.  by_chunk: the q-th chunks of all rows first, in row order,
      // then the (q+1)-th ...: chunk q of a row with sorted columns covers
      // about the same column window in every row of similar density, so the
      // warps resident on an SM gather from one window (L1 reuse).  Else:
      // longest first (balanced tail).
      item_len[item_off[r] + q] = by_chunk ? q : chunk - (w.end - w.beg);
    }
  }
}

static __global__ void iota_kernel(uint32_t* out, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = i;
}

static __global__ void plan_gather_items_kernel(const WorkItem* in, const uint32_t* order, uint32_t n,
                                         WorkItem* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = in[order[i]];
}

// Scratch-backed helpers for cub device calls.
struct CubTemp {
  void* ptr = nullptr;
  size_t bytes = 0;
  void ensure(size_t b) {
    if (b <= bytes) return;
    if (ptr) CK(dfree(ptr));
    CK(dmalloc(&ptr, b));
    bytes = b;
  }
  ~CubTemp() {
    if (ptr) dfree(ptr);  // owners free explicitly inside their AllocScope
  }
};

inline void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint32_t n, CubTemp& tmp,
                               cudaStream_t s) {
  if (n == 0) return;
  size_t b = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, n, s));
  tmp.ensure(b);
  CK(cub::DeviceScan::ExclusiveSum(tmp.ptr, b, in, out, n, s));
}

inline uint32_t grid_for(uint64_t n, int threads = kThreads) {
  uint64_t g = (n + threads - 1) / threads;
  if (g > 8u * kNumSMs * 8u) g = 8u * kNumSMs * 8u;
  return g == 0 ? 1u : uint32_t(g);
}

// Total of an exclusive scan: last exclusive value + last input.
// Totals of K exclusive scans of length n with one stream synchronisation.
template <int K>
inline void scan_totals(const uint32_t* const (&in)[K], const uint32_t* const (&ex)[K], uint32_t n,
                        uint32_t (&out)[K], cudaStream_t s) {
  if (n == 0) {
    for (int i = 0; i < K; ++i) out[i] = 0;
    return;
  }
  uint32_t h[2 * K];
  for (int i = 0; i < K; ++i) {
    CK(cudaMemcpyAsync(h + 2 * i, ex[i] + n - 1, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h + 2 * i + 1, in[i] + n - 1, 4, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < K; ++i) out[i] = h[2 * i] + h[2 * i + 1];
}
inline uint32_t scan_total(const uint32_t* in, const uint32_t* ex, uint32_t n, cudaStream_t s) {
  if (n == 0) return 0;
  uint32_t a = 0, b = 0;
  CK(cudaMemcpyAsync(&a, ex + n - 1, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&b, in + n - 1, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return a + b;
}

// bytes one SumOp pass streams from the matrix in the plan's format (values,
// column indices or compressed offsets + chunk bases + chunk ids, row_ptr)
template <typename T>
double plan_stream_bytes(const DevCsr<T>& M, const SpmvPlan<T>& P) {
  const double idx = P.off16 ? 2.0 * M.nnz + 4.0 * P.n_chunks + 4.0 * P.n_items + 128.0 * P.n_wide
                             : 4.0 * M.nnz;
  return double(sizeof(T)) * M.nnz + idx + 4.0 * (double(M.rows) + 1);
}

template <typename T>
void plan_free(SpmvPlan<T>& P) {
  dfree(P.items);
  dfree(P.short_rows);
  dfree(P.lrinfo);
  dfree(P.partials);
  dfree(P.counters);
  dfree(P.off16);
  dfree(P.cbase);
  dfree(P.c0);
  dfree(P.wide);
  P = SpmvPlan<T>{};
}

static __global__ void chunk_count_kernel(const WorkItem* items, uint32_t n, uint32_t* nch) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    nch[i] = ceil_div(items[i].end - items[i].beg, 32u);
}

// warp per item: classify every 32-entry chunk, write offsets / wide columns.
// fill == 0 only counts the wide chunks (sizing pass).
static __global__ void compress_kernel(const uint32_t* __restrict__ ci, const WorkItem* items, uint32_t n,
                                const uint32_t* c0, uint16_t* off16, uint32_t* cbase,
                                uint32_t* wide, uint32_t* n_wide, int fill) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t it = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n; it += nw) {
    const WorkItem w = items[it];
    uint32_t ch = fill ? c0[it] : 0u;
    for (uint32_t k0 = w.beg; k0 < w.end; k0 += 32u, ++ch) {
      const uint32_t cnt = min(32u, w.end - k0);
      const uint32_t k = k0 + lane;
      const uint32_t c = lane < cnt ? ci[k] : 0u;
      const uint32_t first = __shfl_sync(0xffffffffu, c, 0);
      const uint32_t last = __shfl_sync(0xffffffffu, c, cnt - 1);
      if (last - first < 65536u) {
        if (fill) {
          if (lane < cnt) off16[k] = (uint16_t)(c - first);
          if (lane == 0) cbase[ch] = first;
        }
        continue;
      }
      uint32_t slot = 0;
      if (lane == 0) slot = atomicAdd(n_wide, 1u);
      slot = __shfl_sync(0xffffffffu, slot, 0);
      if (fill) {
        wide[32u * slot + lane] = c;
        if (lane == 0) cbase[ch] = kWide | slot;
      }
    }
  }
}

// Build the compressed index of P's work items over the structure `ci`.
// Columns must stay below 2^31 (the wide flag) or the plan stays uncompressed.
template <typename T>
void plan_compress(SpmvPlan<T>& P, const uint32_t* ci, uint32_t nnz, uint32_t cols, CubTemp& tmp,
                   cudaStream_t s) {
  if (P.n_items == 0 || cols >= kWide) return;
  // only plans of long items: short items keep the high-occupancy kernel
  if (uint64_t(nnz) < uint64_t(kLongItemMean) * P.n_items) return;
  uint32_t* nch;
  CK(dmalloc(&nch, sizeof(uint32_t) * P.n_items));
  CK(dmalloc(&P.c0, sizeof(uint32_t) * P.n_items));
  chunk_count_kernel<<<grid_for(P.n_items), kThreads, 0, s>>>(P.items, P.n_items, nch);
  CK_LAUNCH();
  exclusive_scan_u32(nch, P.c0, P.n_items, tmp, s);
  uint32_t* cnt;
  CK(dmalloc(&cnt, sizeof(uint32_t)));
  CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), s));
  const uint32_t g = grid_for(uint64_t(P.n_items) * 32);
  compress_kernel<<<g, kThreads, 0, s>>>(ci, P.items, P.n_items, P.c0, nullptr, nullptr, nullptr,
                                          cnt, 0);
  CK_LAUNCH();
  // chunk total and wide-chunk count with one synchronisation
  uint32_t h[3];
  CK(cudaMemcpyAsync(h, P.c0 + P.n_items - 1, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + 1, nch + P.n_items - 1, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h + 2, cnt, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(dfree(nch));
  P.n_chunks = h[0] + h[1];
  P.n_wide = h[2];
  // (+32: the per-stride base load of a warp may read up to U - 1 ids past
  // the item's last chunk)
  CK(dmalloc(&P.off16, sizeof(uint16_t) * (size_t(nnz) + 1)));
  CK(dmalloc(&P.cbase, sizeof(uint32_t) * (size_t(P.n_chunks) + 32)));
  CK(dmalloc(&P.wide, sizeof(uint32_t) * 32 * (size_t(P.n_wide) + 1)));
  CK(cudaMemsetAsync(cnt, 0, sizeof(uint32_t), s));
  compress_kernel<<<g, kThreads, 0, s>>>(ci, P.items, P.n_items, P.c0, P.off16, P.cbase, P.wide,
                                          cnt, 1);
  CK_LAUNCH();
  CK(dfree(cnt));
}

// Build the plan for a CSR structure whose row_ptr lives on the device.
template <typename T>
SpmvPlan<T> plan_build(const uint32_t* d_rp, uint32_t rows, uint64_t nnz, CubTemp& tmp,
                       cudaStream_t s) {
  SpmvPlan<T> P;
  P.chunk_log2 = plan_chunk_log2(nnz);
  const char* ord = std::getenv("QPCG_ITEM_ORDER");
  const int by_chunk = !(ord && ord[0] == 'l');  // "len": longest first
  if (rows == 0) return P;
  uint32_t *is_short, *nch, *is_multi, *multi_nch, *short_pos, *item_off, *lr_idx, *pbase;
  const size_t bytes = sizeof(uint32_t) * rows;
  CK(dmalloc(&is_short, bytes));
  CK(dmalloc(&nch, bytes));
  CK(dmalloc(&is_multi, bytes));
  CK(dmalloc(&multi_nch, bytes));
  CK(dmalloc(&short_pos, bytes));
  CK(dmalloc(&item_off, bytes));
  CK(dmalloc(&lr_idx, bytes));
  CK(dmalloc(&pbase, bytes));
  const uint32_t chunk = 1u << P.chunk_log2;
  plan_classify_kernel<<<grid_for(rows), kThreads, 0, s>>>(d_rp, rows, chunk, is_short, nch, is_multi,
                                                          multi_nch);
  CK_LAUNCH();
  exclusive_scan_u32(is_short, short_pos, rows, tmp, s);
  exclusive_scan_u32(nch, item_off, rows, tmp, s);
  exclusive_scan_u32(is_multi, lr_idx, rows, tmp, s);
  exclusive_scan_u32(multi_nch, pbase, rows, tmp, s);
  uint32_t tot[4];
  scan_totals<4>({is_short, nch, is_multi, multi_nch}, {short_pos, item_off, lr_idx, pbase}, rows,
                 tot, s);
  P.n_short = tot[0];
  P.n_items = tot[1];
  P.n_long = tot[2];
  P.n_partials = tot[3];
  CK(dmalloc(&P.short_rows, sizeof(uint32_t) * (P.n_short ? P.n_short : 1)));
  CK(dmalloc(&P.items, sizeof(WorkItem) * (P.n_items ? P.n_items : 1)));
  CK(dmalloc(&P.lrinfo, sizeof(uint2) * (P.n_long ? P.n_long : 1)));
  CK(dmalloc(&P.partials, sizeof(T) * kMaxCols * (P.n_partials ? P.n_partials : 1)));
  CK(dmalloc(&P.counters, sizeof(uint32_t) * (P.n_long ? P.n_long : 1)));
  CK(cudaMemsetAsync(P.counters, 0, sizeof(uint32_t) * (P.n_long ? P.n_long : 1), s));
  WorkItem* items_tmp = nullptr;
  uint32_t *keys = nullptr, *keys_out = nullptr, *order = nullptr, *order_out = nullptr;
  const uint32_t ni = P.n_items ? P.n_items : 1;
  CK(dmalloc(&items_tmp, sizeof(WorkItem) * ni));
  CK(dmalloc(&keys, sizeof(uint32_t) * ni));
  CK(dmalloc(&keys_out, sizeof(uint32_t) * ni));
  CK(dmalloc(&order, sizeof(uint32_t) * ni));
  CK(dmalloc(&order_out, sizeof(uint32_t) * ni));
  plan_emit_kernel<<<grid_for(rows), kThreads, 0, s>>>(d_rp, rows, chunk, is_short, short_pos, nch,
                                                      item_off, lr_idx, pbase, P.short_rows,
                                                      items_tmp, keys, P.lrinfo, by_chunk);
  CK_LAUNCH();
  if (P.n_items > 0) {
    // stable sort of items by length (longest first) for a balanced tail
    iota_kernel<<<grid_for(P.n_items), kThreads, 0, s>>>(order, P.n_items);
    CK_LAUNCH();
    size_t b = 0;
    const int kbits = by_chunk ? 20 : int(P.chunk_log2) + 1;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b, keys, keys_out, order, order_out, P.n_items, 0,
                                       kbits, s));
    tmp.ensure(b);
    CK(cub::DeviceRadixSort::SortPairs(tmp.ptr, b, keys, keys_out, order, order_out, P.n_items, 0,
                                       kbits, s));
    plan_gather_items_kernel<<<grid_for(P.n_items), kThreads, 0, s>>>(items_tmp, order_out,
                                                                     P.n_items, P.items);
    CK_LAUNCH();
  }
  P.nb_items = ceil_div(P.n_items, kWarpsPerBlock);
  P.nb_short = ceil_div(P.n_short, kThreads);
  {  // mean W-bin item length from the totals (row_ptr[rows] - short entries is not
     // known here; the item count and nnz bound it well enough for the choice)
    const char* e = std::getenv("QPCG_U8");
    const uint64_t mean = P.n_items ? nnz / P.n_items : 0;
    P.u8 = e ? (e[0] == '1') : (mean > 96 && mean < kLongItemMean);
  }
  CK(cudaStreamSynchronize(s));
  for (void* p : {(void*)is_short, (void*)nch, (void*)is_multi, (void*)multi_nch, (void*)short_pos,
                  (void*)item_off, (void*)lr_idx, (void*)pbase, (void*)items_tmp, (void*)keys,
                  (void*)keys_out, (void*)order, (void*)order_out})
    CK(dfree(p));
  return P;
}

}  // namespace qpcg_b200
