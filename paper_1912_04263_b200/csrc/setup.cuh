// setup.cuh — device-side setup: validation, symmetrize_upper, transpose_csr,
// modified Ruiz equilibration and the operator's diagonal caches.
//
// Everything here is bit-exact with the reference (SURVEY.md §8(c) parity
// ladder rungs 1-2):
//   * transpose_csr (sparse.hpp:207-232): stable radix sort of entry indices by
//     column => each output row lists source rows in increasing order, exactly
//     the reference's row-major scatter order; the permutation is kept so the
//     scaled A^T can be re-derived from scaled A (scaling.hpp:175) by a gather.
//   * symmetrize_upper (sparse.hpp:237-281): output row j = [mirrored strict-
//     upper entries of column j in source-row order] ++ [input row j].
//   * Ruiz (scaling.hpp:92-187): max-reductions are order-free; scalings are
//     elementwise products in the reference's order ((v*d_row)*d_col); the
//     one sequential sum (mean of P column norms, :156-158) runs as a single
//     ordered chain that skips exact zeros (x + 0 == x for x >= 0).
//   * diag_ata (sparse.hpp:401-408) = per-A^T-row sequential sum of squares;
//     extract_diagonal (sparse.hpp:382-397) = first diagonal match per row.
#pragma once

#include <algorithm>
#include <vector>

#include "spmv.cuh"

namespace qpcg_b200 {

// -------------------------------------------------------- visitor kernels
// Calls f(row, k) for every stored entry, driven by a plan (load balanced).
template <typename T, class F>
__global__ void __launch_bounds__(kThreads) plan_visit_kernel(DevCsr<T> M, SpmvPlan<T> P, F f,
                                                             const uint32_t* act) {
  if (act && !*act) return;  // (an inactive Ruiz pass)
  if (blockIdx.x < P.nb_items) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t it = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (it >= P.n_items) return;
    const WorkItem item = P.items[it];
    for (uint32_t k = item.beg + lane; k < item.end; k += 32) f(item.row, k);
  } else {
    const uint32_t idx = (blockIdx.x - P.nb_items) * kThreads + threadIdx.x;
    if (idx >= P.n_short) return;
    const uint32_t r = P.short_rows[idx];
    for (uint32_t k = M.rp[r]; k < M.rp[r + 1]; ++k) f(r, k);
  }
}
template <typename T, class F>
void plan_visit(const DevCsr<T>& M, const SpmvPlan<T>& P, F f, cudaStream_t s,
                const uint32_t* act = nullptr) {
  if (P.grid() == 0) return;
  plan_visit_kernel<T, F><<<P.grid(), kThreads, 0, s>>>(M, P, f, act);
  CK_LAUNCH();
}

struct RowOfFn {
  uint32_t* row_of;
  __device__ void operator()(uint32_t r, uint32_t k) const { row_of[k] = r; }
};
template <typename T>
struct ScaleRowColFn {  // v = (v * dr[row]) * dc[col]  (scale_rows then scale_columns)
  T* val;
  const uint32_t* ci;
  const T* dr;
  const T* dc;
  __device__ void operator()(uint32_t r, uint32_t k) const { val[k] = (val[k] * dr[r]) * dc[ci[k]]; }
};

template <typename F>
__global__ void for_n_kernel(uint32_t n, F f) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) f(i);
}
template <typename F>
void for_n(uint32_t n, F f, cudaStream_t s) {
  if (n == 0) return;
  for_n_kernel<F><<<grid_for(n), kThreads, 0, s>>>(n, f);
  CK_LAUNCH();
}

// ---------------------------------------------------------- validation
// Error keys: the first violation in the reference's check order wins.
// Key layout (uint64): [category:8][row or index:32][pos:24]
enum ValCat : uint32_t {
  kValPRowPtr = 1,  // P csr row loop
  kValARowPtr = 2,  // A csr row loop
  kValPBelow = 3,   // problem: P has entries below diagonal
  kValPFinite = 4,
  kValAFinite = 5,
  kValQFinite = 6,
  kValBounds = 7,
};

__device__ __forceinline__ void val_report(unsigned long long* key, uint32_t cat, uint32_t idx,
                                           uint32_t pos) {
  const unsigned long long k = ((unsigned long long)cat << 56) |
                               ((unsigned long long)idx << 24) | (pos & 0xffffffu);
  atomicMin(key, k);
}

// sparse.hpp:110-123 per-row checks; pos 0 = nondecreasing, 2j+1 = bound of
// j-th entry, 2j+2 = ordering of j-th entry
// (off: global index of element 0 — a row block of A reports global rows, so
// the minimum over blocks is the unsharded first error)
static __global__ void validate_csr_rows_kernel(const uint32_t* rp, const uint32_t* ci, uint32_t rows,
                                         uint32_t cols, uint32_t cat, int check_upper,
                                         unsigned long long* key, uint32_t off = 0) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    const uint32_t b = rp[r], e = rp[r + 1];
    if (e < b) {
      val_report(key, cat, r + off, 0);
      continue;
    }
    for (uint32_t k = b; k < e; ++k) {
      const uint32_t j = k - b;
      if (ci[k] >= cols) {
        val_report(key, cat, r + off, 2 * j + 1);
        break;
      }
      if (k > b && ci[k] <= ci[k - 1]) {
        val_report(key, cat, r + off, 2 * j + 2);
        break;
      }
    }
    if (check_upper) {
      for (uint32_t k = b; k < e; ++k)
        if (ci[k] < r) {
          val_report(key, kValPBelow, r + off, k - b);
          break;
        }
    }
  }
}

template <typename T>
__global__ void validate_values_kernel(const T* v, uint32_t n, uint32_t cat,
                                       unsigned long long* key, uint32_t off = 0) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (!isfinite(v[i])) val_report(key, cat, i + off, 0);
}

// problem.hpp:86-91 per bound: NaN (pos 0), inf-side (pos 1), l > u (pos 2)
template <typename T>
__global__ void validate_bounds_kernel(const T* l, const T* u, uint32_t m, unsigned long long* key,
                                       uint32_t off = 0) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const T li = l[i], ui = u[i];
    if (isnan(li) || isnan(ui))
      val_report(key, kValBounds, i + off, 0);
    else if (li == (T)INFINITY || ui == -(T)INFINITY)
      val_report(key, kValBounds, i + off, 1);
    else if (li > ui)
      val_report(key, kValBounds, i + off, 2);
  }
}

inline const char* validation_message(unsigned long long key) {
  const uint32_t cat = uint32_t(key >> 56);
  const uint32_t pos = uint32_t(key & 0xffffffu);
  switch (cat) {
    case kValPRowPtr:
    case kValARowPtr:
      if (pos == 0) return "csr: row_ptr must be nondecreasing";
      if (pos & 1u) return "csr: column index out of bounds";
      return "csr: column indices must be strictly increasing within a row";
    case kValPBelow: return "problem: P has entries below diagonal";
    case kValPFinite: return "problem: P not finite";
    case kValAFinite: return "problem: A not finite";
    case kValQFinite: return "problem: q not finite";
    case kValBounds:
      if (pos == 0) return "problem: bounds contain NaN";
      if (pos == 1) return "problem: l must be < +inf and u > -inf";
      return "problem: l must not exceed u";
  }
  return "problem: invalid";
}

// ------------------------------------------------------------ transpose
struct TransposeMap {
  uint32_t* perm = nullptr;  // [nnz] output position -> source entry index
};

// out_rp[c] = first position of the sorted column keys holding a key >= c
// (the transpose's row pointer read off the sort; the per-entry atomic count
// it replaces took 1.6 ms at config 2 on the hot data columns)
static __global__ void rp_from_sorted_kernel(const uint32_t* __restrict__ keys, uint32_t nnz,
                                             uint32_t cols, uint32_t* out_rp) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= cols; c += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = nnz;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (keys[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    out_rp[c] = lo;
  }
}

inline int bits_for(uint32_t n) {
  int b = 1;
  while (b < 32 && (1ull << b) < (unsigned long long)n) ++b;
  return b;
}

// Structure of the transpose of (rows x cols, row_of[], ci[]):
// out_rp [cols+1], out_ci [nnz] (= source rows), perm [nnz].
struct WinPlan;
inline void transpose_structure(const uint32_t* ci, const uint32_t* row_of, uint32_t cols,
                                uint32_t nnz, uint32_t* out_rp, uint32_t* out_ci, uint32_t* perm,
                                CubTemp& tmp, cudaStream_t s, WinPlan* wp = nullptr);

template <typename T>
void gather_values(const T* src, const uint32_t* perm, uint32_t nnz, T* dst, cudaStream_t s) {
  for_n(nnz, [=] __device__(uint32_t i) { dst[i] = src[perm[i]]; }, s);
}

// The same gather, dst[i] = src[perm[i]] for the transpose (dst in A^T order,
// src in A order), in L2-sized WINDOWS of source positions.  A^T row c lists
// its source entries in increasing position (rows increase), so the entries
// of c whose source position lies in window [P_w, P_w+1) are one contiguous
// segment: window by window, a warp per long A^T row copies its next segment
// (a cursor per row), the window's source stays L2-resident while every
// column gathers from it, and the destination is written in contiguous runs.
// The plain gather touches a new 32-byte sector for nearly every 8-byte value
// (lasso: 17.5 GB of DRAM traffic for 3 GB of data,
// profiles/r01_ncu_kernels_config2.md).  A^T rows shorter than kWinLongRow
// are gathered directly (one thread each).  Used for A's values and for the
// source-row array that becomes A^T's column indices.
constexpr uint32_t kWinLongRow = 64;
template <typename T>
__global__ void win_gather_kernel(const T* __restrict__ src, const uint32_t* __restrict__ perm,
                                  const uint32_t* __restrict__ at_rp, const uint32_t* rows,
                                  uint32_t nrows, uint32_t* cur, uint32_t p_end, T* dst) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < nrows; t += nw) {
    const uint32_t c = rows[t];
    uint32_t k = cur[t];
    const uint32_t e = at_rp[c + 1];
    for (;;) {
      const uint32_t kk = k + lane;
      uint32_t sp = 0xffffffffu;
      if (kk < e) sp = perm[kk];
      const bool in = sp < p_end;
      const unsigned bal = __ballot_sync(0xffffffffu, in);
      if (in) dst[kk] = src[sp];
      const uint32_t cnt = __popc(bal);  // a prefix: the source positions increase
      k += cnt;
      if (cnt < 32u) break;
    }
    if (lane == 0) cur[t] = k;
  }
}
template <typename T>
__global__ void short_gather_kernel(const T* __restrict__ src, const uint32_t* __restrict__ perm,
                                    const uint32_t* __restrict__ at_rp, const uint32_t* rows,
                                    uint32_t nrows, T* dst) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nrows; t += gridDim.x * blockDim.x) {
    const uint32_t c = rows[t];
    for (uint32_t k = at_rp[c]; k < at_rp[c + 1]; ++k) dst[k] = src[perm[k]];
  }
}
static __global__ void win_split_kernel(const uint32_t* at_rp, uint32_t n, const uint32_t* pos,
                                        uint32_t* longr, uint32_t* shortr, uint32_t* cur) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x) {
    const bool lg = at_rp[c + 1] - at_rp[c] >= kWinLongRow;
    if (lg) {
      longr[pos[c]] = c;
      cur[pos[c]] = at_rp[c];
    } else {
      shortr[c - pos[c]] = c;
    }
  }
}
static __global__ void win_flag_kernel(const uint32_t* at_rp, uint32_t n, uint32_t* f) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= n; c += gridDim.x * blockDim.x)
    f[c] = c < n && at_rp[c + 1] - at_rp[c] >= kWinLongRow;
}
// the long / short A^T rows and the per-row cursors, shared by every gather
// through one permutation (reset() rewinds the cursors)
struct WinPlan {
  uint32_t n = 0, nl = 0;
  uint32_t *longr = nullptr, *shortr = nullptr, *cur = nullptr, *cur0 = nullptr;
  void build(const uint32_t* at_rp, uint32_t rows, CubTemp& tmp, cudaStream_t s) {
    n = rows;
    uint32_t *f, *pos;
    CK(dmalloc(&f, sizeof(uint32_t) * (size_t(n) + 1)));
    CK(dmalloc(&pos, sizeof(uint32_t) * (size_t(n) + 1)));
    CK(dmalloc(&longr, sizeof(uint32_t) * (size_t(n) + 1)));
    CK(dmalloc(&shortr, sizeof(uint32_t) * (size_t(n) + 1)));
    CK(dmalloc(&cur, sizeof(uint32_t) * (size_t(n) + 1)));
    CK(dmalloc(&cur0, sizeof(uint32_t) * (size_t(n) + 1)));
    win_flag_kernel<<<grid_for(uint64_t(n) + 1), kThreads, 0, s>>>(at_rp, n, f);
    CK_LAUNCH();
    exclusive_scan_u32(f, pos, n + 1, tmp, s);
    win_split_kernel<<<grid_for(n), kThreads, 0, s>>>(at_rp, n, pos, longr, shortr, cur0);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(&nl, pos + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(dfree(f));
    CK(dfree(pos));
  }
  void release() {
    for (void* p : {(void*)longr, (void*)shortr, (void*)cur, (void*)cur0}) CK(dfree(p));
    longr = shortr = cur = cur0 = nullptr;
  }
};
template <typename T>
void gather_windowed(const T* src, const uint32_t* perm, const uint32_t* at_rp, uint32_t nnz,
                     const WinPlan& wp, T* dst, cudaStream_t s) {
  constexpr uint64_t kWindowBytes = 32ull << 20;
  const uint64_t per = std::max<uint64_t>(1, kWindowBytes / sizeof(T));
  const uint32_t nwin = uint32_t((uint64_t(nnz) + per - 1) / per);
  if (nwin <= 1 || wp.n == 0) {  // one window: the plain gather is already L2-resident
    for_n(nnz, [=] __device__(uint32_t i) { dst[i] = src[perm[i]]; }, s);
    return;
  }
  if (wp.n - wp.nl) {
    short_gather_kernel<T><<<grid_for(wp.n - wp.nl), kThreads, 0, s>>>(src, perm, at_rp, wp.shortr,
                                                                        wp.n - wp.nl, dst);
    CK_LAUNCH();
  }
  if (wp.nl) {
    CK(cudaMemcpyAsync(wp.cur, wp.cur0, sizeof(uint32_t) * wp.nl, cudaMemcpyDeviceToDevice, s));
    for (uint32_t w = 0; w < nwin; ++w) {
      const uint32_t p_end = uint32_t(std::min<uint64_t>(nnz, per * (w + 1)));
      win_gather_kernel<T><<<grid_for(uint64_t(wp.nl) * 32), kThreads, 0, s>>>(
          src, perm, at_rp, wp.longr, wp.nl, wp.cur, p_end, dst);
      CK_LAUNCH();
    }
  }
}

inline void transpose_structure(const uint32_t* ci, const uint32_t* row_of, uint32_t cols,
                                uint32_t nnz, uint32_t* out_rp, uint32_t* out_ci, uint32_t* perm,
                                CubTemp& tmp, cudaStream_t s, WinPlan* wp) {
  CK(cudaMemsetAsync(out_rp, 0, sizeof(uint32_t) * (cols + 1), s));
  if (nnz == 0) return;
  uint32_t *keys_out, *idx;
  CK(dmalloc(&keys_out, sizeof(uint32_t) * nnz));
  CK(dmalloc(&idx, sizeof(uint32_t) * nnz));
  iota_kernel<<<grid_for(nnz), kThreads, 0, s>>>(idx, nnz);
  CK_LAUNCH();
  size_t b = 0;
  const int nb = bits_for(cols);
  CK(cub::DeviceRadixSort::SortPairs(nullptr, b, ci, keys_out, idx, perm, nnz, 0, nb, s));
  tmp.ensure(b);
  CK(cub::DeviceRadixSort::SortPairs(tmp.ptr, b, ci, keys_out, idx, perm, nnz, 0, nb, s));
  rp_from_sorted_kernel<<<grid_for(uint64_t(cols) + 1), kThreads, 0, s>>>(keys_out, nnz, cols,
                                                                         out_rp);
  CK_LAUNCH();
  // out_ci[i] = row_of[perm[i]], windowed like the value gathers
  if (wp) {
    wp->build(out_rp, cols, tmp, s);
    gather_windowed(row_of, perm, out_rp, nnz, *wp, out_ci, s);
  } else {
    const uint32_t* perm_c = perm;
    for_n(nnz, [=] __device__(uint32_t i) { out_ci[i] = row_of[perm_c[i]]; }, s);
  }
  // (frees are ordered on s: dmalloc / dfree follow the caller's AllocScope(s))
  CK(dfree(keys_out));
  CK(dfree(idx));
}

// ---------------------------------------------------- symmetrize_upper
// Returns nnz of the full matrix; fills the device arrays of `out` (allocated
// here).  up_row_of is the row of each upper entry.
template <typename T>
uint32_t symmetrize_upper_dev(const DevCsr<T>& up, const uint32_t* up_row_of, DevCsr<T>& out,
                              CubTemp& tmp, cudaStream_t s) {
  const uint32_t n = up.rows, nnz = up.nnz;
  // strict-upper entries, in source order
  uint32_t *flags, *pos, *sel, *sel_cols, *lower_rp, *lower_ci, *lower_perm;
  CK(dmalloc(&flags, sizeof(uint32_t) * (nnz + 1)));
  CK(dmalloc(&pos, sizeof(uint32_t) * (nnz + 1)));
  const uint32_t* ci = up.ci;
  for_n(nnz, [=] __device__(uint32_t k) { flags[k] = ci[k] != up_row_of[k]; }, s);
  exclusive_scan_u32(flags, pos, nnz, tmp, s);
  const uint32_t nstrict = scan_total(flags, pos, nnz, s);
  CK(dmalloc(&sel, sizeof(uint32_t) * (nstrict + 1)));
  CK(dmalloc(&sel_cols, sizeof(uint32_t) * (nstrict + 1)));
  CK(dmalloc(&lower_rp, sizeof(uint32_t) * (n + 1)));
  CK(dmalloc(&lower_ci, sizeof(uint32_t) * (nstrict + 1)));
  CK(dmalloc(&lower_perm, sizeof(uint32_t) * (nstrict + 1)));
  for_n(nnz, [=] __device__(uint32_t k) {
    if (flags[k]) {
      sel[pos[k]] = k;
      sel_cols[pos[k]] = ci[k];
    }
  }, s);
  // lower part = transpose of the strict upper part (rows ordered by source row)
  uint32_t* sel_rows;
  CK(dmalloc(&sel_rows, sizeof(uint32_t) * (nstrict + 1)));
  for_n(nstrict, [=] __device__(uint32_t i) { sel_rows[i] = up_row_of[sel[i]]; }, s);
  transpose_structure(sel_cols, sel_rows, n, nstrict, lower_rp, lower_ci, lower_perm, tmp, s);
  // out row j: lower_cnt(j) + upper_len(j)
  uint32_t *cnt;
  CK(dmalloc(&cnt, sizeof(uint32_t) * (n + 1)));
  const uint32_t* urp = up.rp;
  for_n(n + 1, [=] __device__(uint32_t j) {
    cnt[j] = j < n ? (lower_rp[j + 1] - lower_rp[j]) + (urp[j + 1] - urp[j]) : 0u;
  }, s);
  out.rows = out.cols = n;
  out.nnz = nstrict + nnz;
  CK(dmalloc(&out.rp, sizeof(uint32_t) * (n + 1)));
  CK(dmalloc(&out.ci, sizeof(uint32_t) * (out.nnz + 1)));
  CK(dmalloc(&out.val, sizeof(T) * (out.nnz + 1)));
  exclusive_scan_u32(cnt, out.rp, n + 1, tmp, s);
  uint32_t* orp = out.rp;
  uint32_t* oci = out.ci;
  T* ov = out.val;
  const T* uv = up.val;
  // mirrored entries
  for_n(nstrict, [=] __device__(uint32_t i) {
    const uint32_t j = sel_cols[lower_perm[i]];  // output row (= source column)
    const uint32_t dst = orp[j] + (i - lower_rp[j]);
    oci[dst] = lower_ci[i];
    ov[dst] = uv[sel[lower_perm[i]]];
  }, s);
  // own entries
  for_n(nnz, [=] __device__(uint32_t k) {
    const uint32_t j = up_row_of[k];
    const uint32_t dst = orp[j] + (lower_rp[j + 1] - lower_rp[j]) + (k - urp[j]);
    oci[dst] = ci[k];
    ov[dst] = uv[k];
  }, s);
  for (void* p : {(void*)flags, (void*)pos, (void*)sel, (void*)sel_cols, (void*)lower_rp,
                  (void*)lower_ci, (void*)lower_perm, (void*)sel_rows, (void*)cnt})
    CK(dfree(p));
  return out.nnz;
}

// ------------------------------------------------------- row reductions
template <typename T>
struct StoreEpi {
  T* out;
  const uint32_t* act = nullptr;  // an inactive Ruiz pass: no-op
  __device__ bool init() { return act == nullptr || *act != 0u; }
  __device__ void operator()(uint32_t r, const T (&s)[1]) const { out[r] = s[0]; }
};

template <typename T>
void row_inf_norms(const DevCsr<T>& M, const SpmvPlan<T>& P, T* out, cudaStream_t s,
                   const uint32_t* act = nullptr) {
  if (M.rows == 0) return;
  launch_spmv<T, 1, MaxAbsOp>(M, P, GatherNone<T, 1>{}, StoreEpi<T>{out, act}, s);
}

// One Ruiz scaling visit, v = (v * dr[row]) * dc[col] (scale_rows then
// scale_columns, scaling.hpp:362-380, :333-341), fused with the row
// inf-norms of the scaled values (row_inf_norms, :324-330) that the NEXT
// pass needs: a max is order-free, so the norms are bit-identical to a
// separate pass, which saves one read of the matrix per pass.  Loads are
// issued U strides at a time (the generic plan_visit keeps one in flight).
template <typename T, int U>
__global__ void __launch_bounds__(kThreads) scale_norm_kernel(DevCsr<T> M, SpmvPlan<T> P,
                                                              const T* src,
                                                              const T* __restrict__ dr,
                                                              const T* __restrict__ dc, T* norm,
                                                              const uint32_t* act) {
  if (act && !*act) return;
  if (blockIdx.x < P.nb_items) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t it = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (it >= P.n_items) return;
    const WorkItem item = P.items[it];
    const T r = dr[item.row];
    T acc[1] = {T(0)};
    for (uint32_t k0 = item.beg; k0 < item.end; k0 += 32u * U) {
      T v[U];
      uint32_t c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = k0 + 32u * u + lane;
        const bool ok = k < item.end;
        v[u] = ok ? src[k] : T(0);
        c[u] = ok ? M.ci[k] : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = k0 + 32u * u + lane;
        if (k < item.end) {
          const T x = (v[u] * r) * dc[c[u]];
          M.val[k] = x;
          MaxAbsOp::acc(acc[0], x, T(0));
        }
      }
    }
    item_finish<T, 1, MaxAbsOp, StoreEpi<T>>(M, P, StoreEpi<T>{norm}, item, lane, acc);
  } else {
    const uint32_t idx = (blockIdx.x - P.nb_items) * kThreads + threadIdx.x;
    if (idx >= P.n_short) return;
    const uint32_t row = P.short_rows[idx];
    const T r = dr[row];
    T a = T(0);
    for (uint32_t k = M.rp[row]; k < M.rp[row + 1]; ++k) {
      const T x = (src[k] * r) * dc[M.ci[k]];
      M.val[k] = x;
      MaxAbsOp::acc(a, x, T(0));
    }
    norm[row] = a;
  }
}
// src: the values to scale (M.val in place, or the originals on the first
// pass, which then also initialises M.val)
template <typename T>
void scale_and_norms(const DevCsr<T>& M, const SpmvPlan<T>& P, const T* src, const T* dr,
                     const T* dc, T* norm, cudaStream_t s, const uint32_t* act = nullptr) {
  if (P.grid() == 0) return;
  scale_norm_kernel<T, 4><<<P.grid(), kThreads, 0, s>>>(M, P, src, dr, dc, norm, act);
  CK_LAUNCH();
}

// diag_ata: warp per A^T row, sequential sum of squares in stored order.
// init (nullable): running sums carried in from the row blocks above (the
// sharded chain); out may alias init.
template <typename T>
__global__ void diag_ata_kernel(DevCsr<T> AT, T* out, const T* init) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < AT.rows; r += nwarps) {
    const uint32_t b = AT.rp[r], e = AT.rp[r + 1];
    T s = init ? init[r] : T(0);
    for (uint32_t k0 = b; k0 < e; k0 += 32) {
      const uint32_t k = k0 + lane;
      const T v = k < e ? AT.val[k] : T(0);
      const T sq = v * v;
      const uint32_t cnt = min(32u, e - k0);
      for (uint32_t j = 0; j < cnt; ++j) {
        const T t = __shfl_sync(0xffffffffu, sq, j);
        s += t;
      }
    }
    if (lane == 0) out[r] = s;
  }
}

// extract_diagonal
template <typename T>
__global__ void extract_diag_kernel(DevCsr<T> P, T* out) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < P.rows; r += gridDim.x * blockDim.x) {
    T d = T(0);
    for (uint32_t k = P.rp[r]; k < P.rp[r + 1]; ++k)
      if (P.ci[k] == r) {
        d = P.val[k];
        break;
      }
    out[r] = d;
  }
}

// Sequential sum of v over the rows in `list` (increasing row order), divided
// by n: the mean of scaling.hpp:156-158.  Rows outside the list are empty
// (norm exactly 0) and x + 0 == x for the non-negative running sum, so the
// chain is bit-identical to the reference's sum over all n rows.  One block:
// warp 0 runs the ordered chain on a shared-memory tile while warps 1..7 stage
// the next tile (double buffering hides the gather latency).
constexpr int kMeanTile = 2048;
template <typename T>
__global__ void __launch_bounds__(256) ordered_mean_kernel(const T* __restrict__ v,
                                                          const uint32_t* __restrict__ list,
                                                          uint32_t cnt, uint32_t n, T* out,
                                                          const uint32_t* act = nullptr) {
  if (act && !*act) return;
  __shared__ T buf[2][kMeanTile];
  const uint32_t tid = threadIdx.x;
  // list == nullptr: v is already packed (pack_list_kernel), the tile loads
  // are then coalesced and quick even while the main stream saturates HBM
  for (uint32_t i = tid; i < kMeanTile && i < cnt; i += blockDim.x)
    buf[0][i] = list ? v[list[i]] : v[i];
  __syncthreads();
  T s = T(0);
  for (uint32_t t = 0; uint64_t(t) * kMeanTile < cnt; ++t) {
    const uint32_t cur = t & 1u, nxt = cur ^ 1u;
    const uint64_t base_next = uint64_t(t + 1) * kMeanTile;
    if (tid >= 32) {
      for (uint32_t i = tid - 32; i < kMeanTile && base_next + i < cnt; i += blockDim.x - 32)
        buf[nxt][i] = list ? v[list[base_next + i]] : v[base_next + i];
    } else if (tid == 0) {
      const uint32_t m = uint32_t(min(uint64_t(kMeanTile), uint64_t(cnt) - uint64_t(t) * kMeanTile));
      const T* b = buf[cur];
      uint32_t i = 0;
      for (; i + 8 <= m; i += 8) {
        T r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = b[i + j];
#pragma unroll
        for (int j = 0; j < 8; ++j) s += r[j];
      }
      for (; i < m; ++i) s += b[i];
    }
    __syncthreads();
  }
  if (tid == 0) *out = s / T(n);
}

// packed[i] = v[list[i]] (the ordered mean's operands, gathered in parallel)
template <typename T>
__global__ void pack_list_kernel(const T* __restrict__ v, const uint32_t* __restrict__ list,
                                 uint32_t cnt, T* packed, const uint32_t* act) {
  if (act && !*act) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    packed[i] = v[list[i]];
}

// rows of a CSR structure with at least one stored entry, in increasing order
static __global__ void nonempty_flags_kernel(const uint32_t* rp, uint32_t rows, uint32_t* flags) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    flags[r] = rp[r + 1] > rp[r];
}
static __global__ void compact_kernel(const uint32_t* flags, const uint32_t* pos, uint32_t rows,
                               uint32_t* list) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    if (flags[r]) list[pos[r]] = r;
}

}  // namespace qpcg_b200
