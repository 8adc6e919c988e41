// gram.cuh — the PCG operator apply K p = P p + sigma p + A^T (rho A p)
// (ReducedKktOperator::apply, linsys.hpp:80-90) with A streamed from HBM ONCE.
//
// The reference forms t = rho (A p) with one pass over A and then A^T t with a
// second pass over its explicit transpose (linsys.hpp:84-88); the generic
// engine path does the same (two SpMV launches, ~2 x 1.5 GB per PCG iteration
// at the 1.5e8-nnz configs).  Here one persistent kernel walks A's rows once:
//
//   * a producer warp streams whole rows (their in-window values and 16-bit
//     column offsets, one cp.async.bulk each, rows padded to 8 entries) into
//     a ring of shared-memory slots tracked by mbarriers, so a CTA keeps NS
//     rows in flight independently of its registers;
//   * consumer warps take the rows round-robin: t_j = rho (a_j . p) from the
//     slot (gathering p), then scatter acc[c - w0] += a_jc t_j into a
//     shared-memory accumulator over A's dense column WINDOW [w0, w0 + W)
//     (the data columns of lasso / huber / svm: 1e4, 1e4, 1e3 columns);
//   * the scatters of a CTA happen strictly in row order (a ticket in shared
//     memory), so every acc entry is the sequential sum over the CTA's rows in
//     increasing row index, the order of the reference's A^T row
//     (sparse.hpp:289-295 over A^T entries sorted by source row);
//   * the G per-CTA partial windows are summed in CTA order (= increasing row
//     ranges) by k_gram_reduce, which also forms Kp = (P p + sigma p) + s for
//     the window columns (the EpiKp arithmetic, admm.cuh kp_row);
//   * the few entries outside the window (lasso's residual column, svm's slack
//     column: ~1 per row) are read from global memory for t_j and contribute
//     to A^T t through the ordinary SpMV over the A^T rows outside the window;
//   * "thin" rows (fewer than kGramThin in-window entries: lasso's 2e4 box
//     rows, svm's 1e6 slack rows) are left out of the row pass: one thread
//     per thin row forms its t_j left to right (k_gram_thin, the reference's
//     row order), and their in-window entries reach A^T t through a small
//     transposed copy (A_thin^T, one row per window column) that
//     k_gram_reduce adds after the CTA partials.
//
// Every step is deterministic (static row ranges, ticketed scatter, ordered
// partial sums), so graph / eager runs stay bitwise identical.  The summation
// order of A^T t differs from the two-pass path only in grouping (per-CTA
// partials), i.e. at the ulp level the parity protocol already covers.
//
// OPT-IN (QPCG_GRAM=1).  Measured on B200 (profiles/r02_gram_experiment.txt):
// the row pass alone already runs at 0.54-0.65 ms against 0.28 ms for the
// A pass, and the window scatter costs 0.3-0.6 ms more: every entry needs a
// random 8-byte shared-memory read-modify-write (bank-conflicted wavefronts)
// on top of its gather, so the SM's shared-memory pipe, not HBM, sets the
// pace, and the two-pass SpMV (0.57 ms per operator apply at config 2) stays
// the default.  Kept as a tested, deterministic alternative operator.
//
// Eligibility (Workspace::build_gram): an unsharded workspace, a window of at most 64Ki columns whose accumulator
// takes at most half of the shared-memory budget and holds >= 75 % of A's
// entries, in-window row lengths <= 4096 with at least 4 ring slots.
// With QPCG_GRAM=1 the 75 % share is not required.
#pragma once

#include "admm.cuh"

namespace qpcg_b200 {

constexpr uint32_t kGramMaxRowLen = 4096;
constexpr uint32_t kGramThin = 32;      // rows with fewer in-window entries: thread per row
constexpr uint32_t kGramRowCost = 256;  // per-row cost in entries when balancing the CTAs

template <typename T>
struct GramDev {
  uint32_t w0 = 0, W = 0, G = 0, NS = 0;  // NS: row slots of the shared-memory ring
  uint32_t slot_len = 0, C = 0;           // slot capacity (entries, multiple of 8); consumer warps
  const uint32_t* cut = nullptr;   // [G + 1] ranges of `rows` per CTA (cost-balanced)
  const uint32_t* rows = nullptr;  // the row-pass rows, increasing
  const uint32_t* gstart = nullptr;  // [ng + 1] row-pass row i's entries start at gstart[i]
  const uint32_t* glen = nullptr;    // [ng] its in-window entry count
  const uint16_t* off_g = nullptr;   // in-window entries (col - w0), rows padded to 8 entries
  const T* val_g = nullptr;
  const uint32_t* trows = nullptr; // the thin rows, increasing
  uint32_t n_trows = 0, dbg = 0;   // dbg: QPCG_GRAM_DEBUG (timing experiments): 1 no ticket,
                                   // 3 no ticket and no scatter
  const uint32_t* rp_thin = nullptr;  // [W + 1] A_thin^T: per window column
  const uint32_t* col_thin = nullptr; //   source row of each entry (increasing)
  const T* val_thin = nullptr;
  const uint32_t* rp_out = nullptr;  // [m + 1] out-of-window entries of every row
  const uint32_t* col_out = nullptr;
  const T* val_out = nullptr;
  T* part = nullptr;  // [G * W] per-CTA partial windows
};

// ----------------------------------------------------- mbarrier / bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// One pass over A: t = rho A p (row-pass rows) and the per-CTA partial
// windows of A^T t.  Warp 0 (one lane) is the producer: it streams whole rows
// (values + 16-bit window offsets, one cp.async.bulk each) into a ring of NS
// shared-memory slots, so NS rows per CTA are in flight regardless of
// registers.  Warps 1..C consume rows round-robin: the dot product from the
// slot with p's window staged in shared memory (the gathers never leave the
// SM), t_j, then the scatter into the window accumulator, then the slot is
// released.  The scatter is ordered by row within each of kGramSeg column
// segments of the window (one ticket each): a row's entries are sorted by
// column, so segment s is a contiguous part of the slot, and up to kGramSeg
// rows scatter at once (into different segments) while each accumulator
// entry still sums its rows in increasing order.
//   dynamic shared memory: pw[W] | acc[W] | NS slots of slot_len values |
//   NS slots of slot_len offsets | full[NS], empty[NS] mbarriers
constexpr uint32_t kGramSeg = 4;
template <typename T>
__global__ void k_gram(Dev<T> D, GramDev<T> g) {
  extern __shared__ __align__(128) unsigned char gram_smem[];
  __shared__ volatile uint32_t turn[kGramSeg];
  const Ctl<T>* C = D.ctl;
  if (!C->pcg_active || C->error) return;  // (EpiAp::init)
  const uint32_t Wp = (g.W + 15u) & ~15u;
  T* pw = reinterpret_cast<T*>(gram_smem);
  T* acc = pw + Wp;
  T* sval = acc + Wp;
  uint16_t* soff = reinterpret_cast<uint16_t*>(sval + size_t(g.NS) * g.slot_len);
  uint64_t* full = reinterpret_cast<uint64_t*>(soff + size_t(g.NS) * g.slot_len);
  uint64_t* empty = full + g.NS;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < g.W; i += blockDim.x) {
    acc[i] = T(0);
    pw[i] = D.p[g.w0 + i];
  }
  if (threadIdx.x < kGramSeg) turn[threadIdx.x] = 0u;
  if (threadIdx.x == 0) {
    for (uint32_t q = 0; q < g.NS; ++q) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t i0 = g.cut[blockIdx.x], nrow = g.cut[blockIdx.x + 1] - i0;
  if (warp == 0) {  // ---------------------------------------- producer
    if (lane == 0) {
      for (uint32_t q = 0; q < nrow; ++q) {
        const uint32_t slot = q % g.NS, round = q / g.NS;
        if (round > 0) mbar_wait(empty + slot, (round - 1) & 1u);
        const uint32_t st = __ldg(g.gstart + i0 + q);
        const uint32_t len8 = __ldg(g.gstart + i0 + q + 1) - st;  // padded length
        mbar_expect_tx(full + slot, len8 * uint32_t(sizeof(T) + sizeof(uint16_t)));
        bulk_g2s(sval + size_t(slot) * g.slot_len, g.val_g + st, len8 * uint32_t(sizeof(T)),
                 full + slot);
        bulk_g2s(soff + size_t(slot) * g.slot_len, g.off_g + st, len8 * 2u, full + slot);
      }
    }
  } else {  // ---------------------------------------------- consumers
    const T rho = C->rho;
    const uint32_t seg_w = (g.W + kGramSeg - 1) / kGramSeg;  // columns per segment
    for (uint32_t q = warp - 1; q < nrow; q += g.C) {
      const uint32_t slot = q % g.NS, round = q / g.NS;
      const uint32_t i = i0 + q;
      const uint32_t j = __ldg(g.rows + i), len = __ldg(g.glen + i);
      const uint32_t ob = __ldg(g.rp_out + j), oe = __ldg(g.rp_out + j + 1);
      T s = T(0);
      // out-of-window entries first (global; their loads overlap the wait)
      for (uint32_t k = ob + lane; k < oe; k += 32u) s += g.val_out[k] * __ldg(D.p + g.col_out[k]);
      mbar_wait(full + slot, round & 1u);
      const T* sv = sval + size_t(slot) * g.slot_len;
      const uint16_t* so = soff + size_t(slot) * g.slot_len;
#pragma unroll 4
      for (uint32_t k = lane; k < len; k += 32u) s += sv[k] * pw[so[k]];
      s = warp_sum(s);
      const T tj = s * rho;  // EpiAp: t[r] = s * rho
      // segment boundaries within the slot: lane q < kGramSeg finds the first
      // entry of segment q + 1 (offsets are increasing)
      uint32_t bnd = len;
      if (lane < kGramSeg - 1) {
        const uint32_t key = (lane + 1) * seg_w;
        uint32_t lo = 0, hi = len;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (so[mid] < key) lo = mid + 1;
          else hi = mid;
        }
        bnd = lo;
      }
      if (lane == 0) D.t[j] = tj;
      uint32_t sb = 0;
#pragma unroll
      for (uint32_t sg = 0; sg < kGramSeg; ++sg) {
        const uint32_t se = __shfl_sync(0xffffffffu, bnd, sg);  // end of segment sg
        if (!(g.dbg & 1u)) {
          if (lane == 0) {
            while (turn[sg] != q) __nanosleep(32);
            __threadfence_block();
          }
          __syncwarp();
        }
        if ((g.dbg & 3u) != 3u) {
          for (uint32_t k = sb + lane; k < se; k += 32u) {
            T* a = acc + so[k];
            *a = *a + sv[k] * tj;
          }
        }
        __syncwarp();
        __threadfence_block();
        if (lane == 0) turn[sg] = q + 1u;
        sb = se;
      }
      if (lane == 0) mbar_arrive(empty + slot);  // the slot may be refilled
    }
  }
  __syncthreads();
  T* out = g.part + size_t(blockIdx.x) * g.W;
  for (uint32_t i = threadIdx.x; i < g.W; i += blockDim.x) out[i] = acc[i];
}

// s[c] = sum over CTAs (in CTA order, 8 fixed groups of consecutive CTAs
// combined left to right) of the partial windows; Kp for the window columns.
constexpr uint32_t kGramRedGroups = 8;
template <typename T>
__global__ void __launch_bounds__(32 * kGramRedGroups) k_gram_reduce(Dev<T> D, GramDev<T> g) {
  __shared__ T sm[kGramRedGroups][33];
  const Ctl<T>* C = D.ctl;
  if (!C->pcg_active || C->error) return;
  const uint32_t lane = threadIdx.x & 31u, grp = threadIdx.x >> 5;
  const uint32_t col = blockIdx.x * 32u + lane;
  const uint32_t per = (g.G + kGramRedGroups - 1) / kGramRedGroups;
  const uint32_t c0 = min(g.G, grp * per), c1 = min(g.G, c0 + per);
  T s = T(0);
  if (col < g.W) {
    const T* pp = g.part + col;
    uint32_t c = c0;
    for (; c + 8 <= c1; c += 8) {
      T q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = __ldcg(pp + size_t(c + u) * g.W);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += q[u];
    }
    for (; c < c1; ++c) s += __ldcg(pp + size_t(c) * g.W);
  }
  sm[grp][lane] = s;
  __syncthreads();
  if (grp != 0 || col >= g.W) return;
  T tot = sm[0][lane];
#pragma unroll
  for (uint32_t q = 1; q < kGramRedGroups; ++q) tot = tot + sm[q][lane];
  for (uint32_t k = g.rp_thin[col]; k < g.rp_thin[col + 1]; ++k)  // thin rows, row order
    tot = tot + g.val_thin[k] * D.t[g.col_thin[k]];
  const uint32_t i = g.w0 + col;
  D.kp[i] = kp_row(D, C->sigma, i, tot);
}

// t_j = rho (a_j . p) for the thin rows: one thread per row, left to right
// over the row's CSR entries (the reference's order, sparse.hpp:289-295).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_gram_thin(Dev<T> D, GramDev<T> g) {
  const Ctl<T>* C = D.ctl;
  if (!C->pcg_active || C->error) return;
  const T rho = C->rho;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < g.n_trows;
       i += gridDim.x * blockDim.x) {
    const uint32_t j = g.trows[i];
    T s = T(0);
    for (uint32_t k = D.A.rp[j]; k < D.A.rp[j + 1]; ++k) s += D.A.val[k] * D.p[D.A.ci[k]];
    D.t[j] = s * rho;
  }
}

// Kp = (P p + sigma p) + A^T t for the A^T rows OUTSIDE the window: the
// plan's rows are numbered from `off` (a row-range view of A^T).
template <typename T>
struct EpiKpOff {
  Dev<T> D;
  T sigma;
  uint32_t off;
  __device__ __forceinline__ bool init() {
    sigma = D.ctl->sigma;
    return D.ctl->pcg_active != 0 && D.ctl->error == 0;
  }
  __device__ __forceinline__ void operator()(uint32_t r, const T (&s)[1]) const {
    D.kp[r + off] = kp_row(D, sigma, r + off, s[0]);
  }
};

// ------------------------------------------------------------ setup kernels
// per row: number of entries inside / outside the window
static __global__ void gram_count_kernel(const uint32_t* __restrict__ rp,
                                         const uint32_t* __restrict__ ci, uint32_t rows,
                                         uint32_t w0, uint32_t W, uint32_t* cin, uint32_t* cout,
                                         unsigned int* max_in) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const uint32_t b = rp[r], e = rp[r + 1];
    uint32_t k_in = 0;
    for (uint32_t k = b + lane; k < e; k += 32u) k_in += (ci[k] - w0) < W;
    k_in = warp_sum(k_in);
    if (lane == 0) {
      cin[r] = k_in;
      cout[r] = (e - b) - k_in;
      atomicMax(max_in, k_in);
    }
  }
}

// per row: split the entries (order kept) into the in-window and out-of-window arrays
template <typename T>
__global__ void gram_fill_kernel(const uint32_t* __restrict__ rp, const uint32_t* __restrict__ ci,
                                 const T* __restrict__ val, uint32_t rows, uint32_t w0, uint32_t W,
                                 const uint32_t* din, const uint32_t* rp_out, uint16_t* off_g,
                                 T* val_g, uint32_t* col_out, T* val_out) {
  // din[r]: where row r's in-window entries go (~0: a thin row, not stored)
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += nw) {
    const uint32_t b = rp[r], e = rp[r + 1];
    uint32_t pin = din[r], pout = rp_out[r];
    for (uint32_t k0 = b; k0 < e; k0 += 32u) {
      const uint32_t k = k0 + lane;
      const bool ok = k < e;
      const uint32_t c = ok ? ci[k] : 0u;
      const bool in = ok && (c - w0) < W;
      const unsigned bi = __ballot_sync(0xffffffffu, in);
      const unsigned bo = __ballot_sync(0xffffffffu, ok && !in);
      if (in) {
        if (pin != 0xffffffffu) {
          const uint32_t at = pin + __popc(bi & lt);
          off_g[at] = (uint16_t)(c - w0);
          val_g[at] = val[k];
        }
      } else if (ok) {
        const uint32_t at = pout + __popc(bo & lt);
        col_out[at] = c;
        val_out[at] = val[k];
      }
      if (pin != 0xffffffffu) pin += __popc(bi);
      pout += __popc(bo);
    }
  }
}
// padded in-window length per row-pass row (the ring moves whole 16-byte
// multiples), and the row -> storage map of the fill
static __global__ void gram_plen_kernel(const uint32_t* grows, uint32_t ng, const uint32_t* cin,
                                        uint32_t* plen, uint32_t* glen) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= ng; i += gridDim.x * blockDim.x) {
    const uint32_t c = i < ng ? cin[grows[i]] : 0u;
    plen[i] = (c + 7u) & ~7u;
    if (i < ng) glen[i] = c;
  }
}
static __global__ void gram_din_kernel(const uint32_t* grows, uint32_t ng, const uint32_t* gstart,
                                       uint32_t* din) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x)
    din[grows[i]] = gstart[i];
}

// row lists: the row-pass rows (>= kGramThin in-window entries) and the thin
// rows, both increasing; pos = exclusive scan of is_g
static __global__ void gram_split_kernel(const uint32_t* cin, const uint32_t* pos, uint32_t rows,
                                         uint32_t* grows, uint32_t* trows, uint8_t* thin) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < rows; j += gridDim.x * blockDim.x) {
    const bool big = cin[j] >= kGramThin;
    if (big) grows[pos[j]] = j;
    else trows[j - pos[j]] = j;
    thin[j] = !big;
  }
}
static __global__ void gram_isg_kernel(const uint32_t* cin, uint32_t rows, uint32_t* isg) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= rows; j += gridDim.x * blockDim.x)
    isg[j] = j < rows && cin[j] >= kGramThin;
}
// cost of each row-pass row: its entries plus a fixed per-row latency share
static __global__ void gram_weight_kernel(const uint32_t* grows, uint32_t ng, const uint32_t* cin,
                                          const uint32_t* cout, uint32_t* w) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= ng; i += gridDim.x * blockDim.x)
    w[i] = i < ng ? cin[grows[i]] + cout[grows[i]] + kGramRowCost : 0u;
}
// A_thin^T: per window column c (A^T row w0 + c), its entries whose source
// row is thin; count (fill == 0) or copy in order (fill == 1)
template <typename T>
__global__ void gram_thin_t_kernel(const uint32_t* __restrict__ at_rp,
                                   const uint32_t* __restrict__ at_ci, const T* __restrict__ at_val,
                                   uint32_t w0, uint32_t W, const uint8_t* __restrict__ thin,
                                   uint32_t* cnt, const uint32_t* rp_thin, uint32_t* col_thin,
                                   T* val_thin, int fill) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < W; c += nw) {
    const uint32_t b = at_rp[w0 + c], e = at_rp[w0 + c + 1];
    uint32_t at = fill ? rp_thin[c] : 0u;
    for (uint32_t k0 = b; k0 < e; k0 += 32u) {
      const uint32_t k = k0 + lane;
      const bool ok = k < e;
      const uint32_t src = ok ? at_ci[k] : 0u;
      const bool take = ok && thin[src];
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      if (fill && take) {
        const uint32_t q = at + __popc(bal & lt);
        col_thin[q] = src;
        val_thin[q] = at_val[k];
      }
      at += __popc(bal);
    }
    if (!fill && lane == 0) cnt[c] = at;
  }
}

// cut[g] = first index whose prefix weight >= g * total / G (balanced contiguous ranges)
static __global__ void gram_cut_kernel(const uint32_t* __restrict__ rp, uint32_t rows, uint32_t G,
                                       uint32_t* cut) {
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi > G) return;
  if (gi == 0 || gi == G) {
    cut[gi] = gi == 0 ? 0u : rows;
    return;
  }
  const uint64_t target = uint64_t(rp[rows]) * gi / G;
  uint32_t lo = 0, hi = rows;  // first r in [0, rows] with rp[r] >= target
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (rp[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  cut[gi] = lo;
}

}  // namespace qpcg_b200
