// gen.cpp — host-side problem instances, bit-identical to the reference's
// generators (bench/rng.hpp, bench/generators.hpp), multi-threaded.
//
// The reference draws every instance from a counter-based splitmix64 stream
// (rng.hpp:39-88).  `sample_sparse` (generators.hpp:156-167) walks the rows*cols
// entries in row-major order, drawing one uniform per entry and two more for
// the N(0,1) value of an accepted entry, so the counter position of entry e
// depends on all earlier accept decisions.  Parallel restatement: the counter
// axis is cut into chunks; a walk can only enter a chunk at offset 0, 1 or 2,
// so each chunk is simulated from all three entry phases (which merge after a
// few steps), the phases are resolved by a sequential pass over the chunk
// summaries, and a second parallel pass emits the accepted entries.  The
// draws, and therefore the instance, are identical to the sequential walk
// (tests/test_generators.py checks bit-equality against oracle/_ref).
//
// Instances: generate(class, scale, seed) (generators.hpp:693-705) and the
// explicit sizes of SURVEY.md §8(d) (key derive_key({class, 100, seed})).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using u32 = uint32_t;
using u64 = uint64_t;
constexpr u64 kGolden = 0x9E3779B97F4A7C15ULL;
constexpr double kPi = 3.141592653589793238462643383279502884;

// rng.hpp:39-46
inline u64 mix64(u64 z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
// rng.hpp:48-54
u64 derive_key(std::initializer_list<u64> words) {
  u64 key = 0;
  for (u64 w : words) key = mix64(key ^ (w + kGolden));
  return key;
}
inline double u01_at(u64 key, u64 pos) {
  return static_cast<double>(mix64(key + pos * kGolden) >> 11) * 0x1.0p-53;
}
inline double normal_at(u64 key, u64 pos) {  // rng.hpp:72-77 (draws pos, pos+1)
  const double u1 = 1.0 - u01_at(key, pos);
  const double u2 = u01_at(key, pos + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
}

// rng.hpp:56-88
struct Rng {
  u64 key, counter = 0;
  explicit Rng(u64 k) : key(k) {}
  u64 next_u64() { return mix64(key + (++counter) * kGolden); }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double normal() {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
  }
  u64 next_below(u64 bound) { return next_u64() % bound; }
  bool bernoulli(double p) { return uniform() < p; }
};

struct Csr {
  u32 rows = 0, cols = 0;
  std::vector<double> val;
  std::vector<u32> rp, ci;
  u64 nnz() const { return val.size(); }
};

struct Qp {
  Csr p, a;
  std::vector<double> q, l, u;
};

int g_threads = 0;
int nthreads() {
  if (g_threads > 0) return g_threads;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? int(h) : 4;
}

template <class F>
void parallel_for(u64 n, F f) {
  const int t = int(std::max<u64>(1, std::min<u64>(u64(nthreads()), n)));
  if (t == 1) {
    for (u64 i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<u64> next{0};
  std::vector<std::thread> pool;
  for (int k = 0; k < t; ++k)
    pool.emplace_back([&] {
      for (u64 i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& th : pool) th.join();
}

// ------------------------------------------------- parallel Bernoulli walk
struct ChunkSum {
  u64 steps[3], acc[3];
  u32 exit[3];
};

// Walk `entries` entries from draw rng.counter+1; entry e is accepted iff
// uniform() < density and then consumes a normal.  Fills `ent` (accepted entry
// indices, increasing) and `val[k] = shift(row) + normal` and advances rng.
void bernoulli_walk(Rng& rng, u64 entries, u64 cols, double density,
                    const std::vector<double>* row_shift, std::vector<u64>& ent,
                    std::vector<double>& val) {
  ent.clear();
  val.clear();
  if (entries == 0) return;
  const u64 key = rng.key;
  const u64 start = rng.counter + 1;
  const u64 S = u64(1) << 21;  // counter positions per chunk
  auto accept = [&](u64 pos) { return u01_at(key, pos) < density; };
  std::vector<ChunkSum> sums;
  std::vector<u32> phase;
  std::vector<u64> e0;
  u64 e = 0;
  u32 ph = 0;
  u64 last_chunk = 0;
  bool finished = false;
  while (!finished) {  // pass 1, in batches of chunks
    const u64 base = sums.size();
    // expected counter span = entries * (1 + 2 density); size the batch so
    // small instances do not simulate idle chunks
    const u64 need = u64(double(entries) * (1.0 + 2.0 * density) * 1.02 / double(S)) + 2;
    const u64 batch = std::max<u64>(1, std::min<u64>(std::max<u64>(4 * u64(nthreads()), 32),
                                                     need > base ? need - base : 1));
    sums.resize(base + batch);
    parallel_for(batch, [&](u64 bi) {
      const u64 j = base + bi;
      const u64 lo = start + j * S, hi = lo + S;
      ChunkSum cs;
      u64 p[3] = {lo, lo + 1, lo + 2}, st[3] = {0, 0, 0}, ac[3] = {0, 0, 0};
      bool merged[3] = {true, false, false};
      u64 ds[3] = {0, 0, 0}, da[3] = {0, 0, 0};  // chain k minus chain 0 at the merge
      auto step = [&](int k) {
        const bool a = accept(p[k]);
        p[k] += a ? 3 : 1;
        st[k] += 1;
        ac[k] += a;
      };
      while (!merged[1] || !merged[2]) {  // advance the lowest chain
        int kmin = 0;
        for (int k = 1; k < 3; ++k)
          if (!merged[k] && p[k] < p[kmin]) kmin = k;
        if (p[kmin] >= hi) break;
        step(kmin);
        for (int k = 1; k < 3; ++k)
          if (!merged[k] && p[k] == p[0]) {
            merged[k] = true;
            ds[k] = st[k] - st[0];
            da[k] = ac[k] - ac[0];
          }
      }
      for (int k = 1; k < 3; ++k)
        if (!merged[k]) {
          while (p[k] < hi) step(k);
          cs.steps[k] = st[k];
          cs.acc[k] = ac[k];
          cs.exit[k] = u32(p[k] - hi);
        }
      while (p[0] < hi) step(0);
      cs.steps[0] = st[0];
      cs.acc[0] = ac[0];
      cs.exit[0] = u32(p[0] - hi);
      for (int k = 1; k < 3; ++k)
        if (merged[k]) {
          cs.steps[k] = st[0] + ds[k];
          cs.acc[k] = ac[0] + da[k];
          cs.exit[k] = cs.exit[0];
        }
      sums[j] = cs;
    });
    for (u64 j = base; j < base + batch; ++j) {  // sequential phase resolution
      phase.push_back(ph);
      e0.push_back(e);
      const ChunkSum& cs = sums[j];
      if (e + cs.steps[ph] >= entries) {
        finished = true;
        last_chunk = j;
        break;
      }
      e += cs.steps[ph];
      ph = cs.exit[ph];
    }
  }
  const u64 nch = last_chunk + 1;
  // pass 2a: accepted count and end position per chunk (the last chunk stops
  // at the entry budget)
  std::vector<u64> cnt(nch), endpos(nch);
  auto walk = [&](u64 j, auto&& on_accept) {
    u64 pos = start + j * S + phase[j];
    const u64 hi = start + j * S + S;
    u64 ee = e0[j];
    while (ee < entries && (j == last_chunk || pos < hi)) {
      if (accept(pos)) {
        on_accept(ee, pos);
        pos += 3;
      } else {
        pos += 1;
      }
      ++ee;
    }
    return pos;
  };
  parallel_for(nch, [&](u64 j) {
    u64 c = 0;
    endpos[j] = walk(j, [&](u64, u64) { ++c; });
    cnt[j] = c;
  });
  std::vector<u64> a0(nch);
  u64 total = 0;
  for (u64 j = 0; j < nch; ++j) {
    a0[j] = total;
    total += cnt[j];
  }
  ent.resize(total);
  val.resize(total);
  parallel_for(nch, [&](u64 j) {  // pass 2b: emit
    u64 out = a0[j];
    walk(j, [&](u64 ee, u64 pos) {
      const double nv = normal_at(key, pos + 1);
      ent[out] = ee;
      val[out] = row_shift ? (*row_shift)[ee / cols] + nv : nv;
      ++out;
    });
  });
  rng.counter = endpos[nch - 1] - 1;
}

// generators.hpp:156-167 sample_sparse; with row_shift it is the svm cloud
// loop (generators.hpp:681-688): value = labels[i]*shift + normal.
Csr sample_sparse(Rng& rng, u32 rows, u32 cols, double density,
                  const std::vector<double>* row_shift = nullptr) {
  Csr m;
  m.rows = rows;
  m.cols = cols;
  std::vector<u64> ent;
  bernoulli_walk(rng, u64(rows) * cols, cols, density, row_shift, ent, m.val);
  m.ci.resize(ent.size());
  m.rp.assign(size_t(rows) + 1, 0);
  parallel_for((ent.size() + (1 << 20) - 1) >> 20, [&](u64 b) {
    const u64 lo = b << 20, hi = std::min<u64>(ent.size(), lo + (1 << 20));
    for (u64 k = lo; k < hi; ++k) m.ci[k] = u32(ent[k] % cols);
  });
  for (u64 k = 0; k < ent.size(); ++k) ++m.rp[u32(ent[k] / cols) + 1];
  for (u32 r = 0; r < rows; ++r) m.rp[r + 1] += m.rp[r];
  return m;
}

struct Triplet {
  u32 r, c;
  double v;
};

// generators.hpp:214-245
Csr csr_from_triplets(u32 rows, u32 cols, std::vector<Triplet>& t, bool sum_duplicates) {
  std::stable_sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  });
  if (sum_duplicates) {
    std::vector<Triplet> merged;
    merged.reserve(t.size());
    for (const Triplet& e : t) {
      if (!merged.empty() && merged.back().r == e.r && merged.back().c == e.c)
        merged.back().v += e.v;
      else
        merged.push_back(e);
    }
    t.swap(merged);
  }
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.rp.assign(size_t(rows) + 1, 0);
  m.val.reserve(t.size());
  m.ci.reserve(t.size());
  for (const Triplet& e : t) {
    ++m.rp[e.r + 1];
    m.val.push_back(e.v);
    m.ci.push_back(e.c);
  }
  for (u32 r = 0; r < rows; ++r) m.rp[r + 1] += m.rp[r];
  return m;
}

// generators.hpp:263-295
Csr gram_psd_upper(Rng& rng, u32 n, u32 rows, u32 nnz_per_row, double alpha) {
  std::vector<Triplet> t;
  std::vector<u32> cols(nnz_per_row);
  std::vector<double> vals(nnz_per_row);
  for (u32 r = 0; r < rows; ++r) {
    for (u32 j = 0; j < nnz_per_row; ++j) {
      u32 c;
      bool fresh;
      do {
        c = static_cast<u32>(rng.next_below(n));
        fresh = true;
        for (u32 k = 0; k < j; ++k) fresh = fresh && cols[k] != c;
      } while (!fresh);
      cols[j] = c;
      vals[j] = rng.normal();
    }
    std::vector<u32> order(nnz_per_row);
    for (u32 j = 0; j < nnz_per_row; ++j) order[j] = j;
    std::sort(order.begin(), order.end(), [&](u32 a, u32 b) { return cols[a] < cols[b]; });
    for (u32 a = 0; a < nnz_per_row; ++a)
      for (u32 b = a; b < nnz_per_row; ++b)
        t.push_back({cols[order[a]], cols[order[b]], vals[order[a]] * vals[order[b]]});
  }
  for (u32 i = 0; i < n; ++i) t.push_back({i, i, alpha});
  return csr_from_triplets(n, n, t, true);
}

// sparse.hpp:283-296 (sequential per row; rows in parallel)
std::vector<double> spmv(const Csr& m, const std::vector<double>& x) {
  std::vector<double> y(m.rows);
  parallel_for((u64(m.rows) + 4095) / 4096, [&](u64 b) {
    const u32 lo = u32(b * 4096), hi = u32(std::min<u64>(m.rows, b * 4096 + 4096));
    for (u32 r = lo; r < hi; ++r) {
      double s = 0.0;
      for (u32 k = m.rp[r]; k < m.rp[r + 1]; ++k) s += m.val[k] * x[m.ci[k]];
      y[r] = s;
    }
  });
  return y;
}

// spmv(transpose(m), b): per column, sum in increasing row order
std::vector<double> spmv_transpose(const Csr& m, const std::vector<double>& b) {
  std::vector<double> y(m.cols, 0.0);
  for (u32 r = 0; r < m.rows; ++r)
    for (u32 k = m.rp[r]; k < m.rp[r + 1]; ++k) y[m.ci[k]] += m.val[k] * b[r];
  return y;
}

double inf_norm(const std::vector<double>& v) {
  double m = 0.0;
  for (double x : v) {
    const double a = std::abs(x);
    if (a > m) m = a;
  }
  return m;
}

// Row-wise CSR builder for the reformulations (rows and columns are emitted in
// sorted order, so csr_from_triplets' stable sort would be the identity).
struct RowBuilder {
  Csr m;
  RowBuilder(u32 cols, u64 nnz_hint) {
    m.cols = cols;
    m.rp.push_back(0);
    m.val.reserve(nnz_hint);
    m.ci.reserve(nnz_hint);
  }
  void put(u32 c, double v) {
    m.ci.push_back(c);
    m.val.push_back(v);
  }
  void end_row() {
    m.rp.push_back(u32(m.val.size()));
    m.rows += 1;
  }
};

Csr diag_csr(u32 n, const std::vector<std::pair<u32, double>>& d) {  // sorted diag entries
  Csr m;
  m.rows = m.cols = n;
  m.rp.assign(size_t(n) + 1, 0);
  for (auto& e : d) {
    ++m.rp[e.first + 1];
    m.ci.push_back(e.first);
    m.val.push_back(e.second);
  }
  for (u32 r = 0; r < n; ++r) m.rp[r + 1] += m.rp[r];
  return m;
}

// generators.hpp:392-433
Qp make_lasso(const Csr& a, const std::vector<double>& b, double lambda) {
  const u32 md = a.rows, n = a.cols, nvar = n + md + n, t_off = n + md, m = md + 2 * n;
  Qp p;
  std::vector<std::pair<u32, double>> d;
  for (u32 i = 0; i < md; ++i) d.push_back({n + i, 2.0});
  p.p = diag_csr(nvar, d);
  p.q.assign(nvar, 0.0);
  for (u32 j = 0; j < n; ++j) p.q[t_off + j] = lambda;
  p.l.assign(m, 0.0);
  p.u.assign(m, 0.0);
  RowBuilder A(nvar, a.nnz() + md + 4ull * n);
  for (u32 i = 0; i < md; ++i) {
    for (u32 k = a.rp[i]; k < a.rp[i + 1]; ++k) A.put(a.ci[k], a.val[k]);
    A.put(n + i, -1.0);
    A.end_row();
    p.l[i] = b[i];
    p.u[i] = b[i];
  }
  for (u32 j = 0; j < n; ++j) {
    A.put(j, 1.0);
    A.put(t_off + j, -1.0);
    A.end_row();
    p.l[md + j] = -INFINITY;
    p.u[md + j] = 0.0;
  }
  for (u32 j = 0; j < n; ++j) {
    A.put(j, 1.0);
    A.put(t_off + j, 1.0);
    A.end_row();
    p.l[md + n + j] = 0.0;
    p.u[md + n + j] = INFINITY;
  }
  p.a = std::move(A.m);
  return p;
}

// generators.hpp:346-388
Qp make_huber(const Csr& a, const std::vector<double>& b, double mh) {
  const u32 md = a.rows, n = a.cols, nvar = n + 3 * md;
  Qp p;
  std::vector<std::pair<u32, double>> d;
  for (u32 i = 0; i < md; ++i) d.push_back({n + i, 2.0});
  p.p = diag_csr(nvar, d);
  p.q.assign(nvar, 0.0);
  for (u32 i = 0; i < md; ++i) {
    p.q[n + md + i] = 2.0 * mh;
    p.q[n + 2 * md + i] = 2.0 * mh;
  }
  p.l.assign(3 * size_t(md), 0.0);
  p.u.assign(3 * size_t(md), 0.0);
  RowBuilder A(nvar, a.nnz() + 5ull * md);
  for (u32 i = 0; i < md; ++i) {
    for (u32 k = a.rp[i]; k < a.rp[i + 1]; ++k) A.put(a.ci[k], a.val[k]);
    A.put(n + i, -1.0);
    A.put(n + md + i, -1.0);
    A.put(n + 2 * md + i, 1.0);
    A.end_row();
    p.l[i] = b[i];
    p.u[i] = b[i];
  }
  for (u32 i = 0; i < md; ++i) {
    A.put(n + md + i, 1.0);
    A.end_row();
    p.u[md + i] = INFINITY;
  }
  for (u32 i = 0; i < md; ++i) {
    A.put(n + 2 * md + i, 1.0);
    A.end_row();
    p.u[2 * md + i] = INFINITY;
  }
  p.a = std::move(A.m);
  return p;
}

// generators.hpp:438-476
Qp make_portfolio(const Csr& f_t, const std::vector<double>& dd, const std::vector<double>& mu,
                  double gamma) {
  const u32 k = f_t.rows, n = f_t.cols, nvar = n + k, m = 1 + k + n;
  Qp p;
  std::vector<std::pair<u32, double>> d;
  for (u32 j = 0; j < n; ++j)
    if (dd[j] != 0.0) d.push_back({j, 2.0 * gamma * dd[j]});
  for (u32 i = 0; i < k; ++i) d.push_back({n + i, 2.0 * gamma});
  p.p = diag_csr(nvar, d);
  p.q.assign(nvar, 0.0);
  for (u32 j = 0; j < n; ++j) p.q[j] = -mu[j];
  p.l.assign(m, 0.0);
  p.u.assign(m, 0.0);
  RowBuilder A(nvar, f_t.nnz() + 2ull * n + k);
  for (u32 j = 0; j < n; ++j) A.put(j, 1.0);
  A.end_row();
  p.l[0] = 1.0;
  p.u[0] = 1.0;
  for (u32 i = 0; i < k; ++i) {
    for (u32 kk = f_t.rp[i]; kk < f_t.rp[i + 1]; ++kk) A.put(f_t.ci[kk], f_t.val[kk]);
    A.put(n + i, -1.0);
    A.end_row();
  }
  for (u32 j = 0; j < n; ++j) {
    A.put(j, 1.0);
    A.end_row();
    p.u[1 + k + j] = INFINITY;
  }
  p.a = std::move(A.m);
  return p;
}

// generators.hpp:480-513
Qp make_svm(const Csr& a, const std::vector<double>& labels, double lambda) {
  const u32 md = a.rows, n = a.cols, nvar = n + md, m = 2 * md;
  Qp p;
  std::vector<std::pair<u32, double>> d;
  for (u32 j = 0; j < n; ++j) d.push_back({j, 2.0});
  p.p = diag_csr(nvar, d);
  p.q.assign(nvar, 0.0);
  for (u32 i = 0; i < md; ++i) p.q[n + i] = lambda;
  p.l.assign(m, 0.0);
  p.u.assign(m, 0.0);
  RowBuilder A(nvar, a.nnz() + 2ull * md);
  for (u32 i = 0; i < md; ++i) {
    for (u32 k = a.rp[i]; k < a.rp[i + 1]; ++k) A.put(a.ci[k], labels[i] * a.val[k]);
    A.put(n + i, -1.0);
    A.end_row();
    p.l[i] = -INFINITY;
    p.u[i] = -1.0;
  }
  for (u32 i = 0; i < md; ++i) {
    A.put(n + i, 1.0);
    A.end_row();
    p.u[md + i] = INFINITY;
  }
  p.a = std::move(A.m);
  return p;
}

// generators.hpp:340-328 make_control_qp
Qp make_control(const std::vector<double>& a_dyn, const std::vector<double>& b_in,
                const std::vector<double>& q_diag, const std::vector<double>& r_diag,
                const std::vector<double>& qt_diag, const std::vector<double>& x_init,
                double x_bound, double u_bound, u32 horizon) {
  const u32 nx = u32(q_diag.size()), nu = u32(r_diag.size()), T = horizon;
  const u32 nvar = nx * (T + 1) + nu * T, u_off = nx * (T + 1);
  Qp p;
  std::vector<std::pair<u32, double>> d;
  for (u32 t = 0; t < T; ++t)
    for (u32 i = 0; i < nx; ++i)
      if (q_diag[i] != 0.0) d.push_back({t * nx + i, 2 * q_diag[i]});
  for (u32 i = 0; i < nx; ++i)
    if (qt_diag[i] != 0.0) d.push_back({T * nx + i, 2 * qt_diag[i]});
  for (u32 t = 0; t < T; ++t)
    for (u32 i = 0; i < nu; ++i)
      if (r_diag[i] != 0.0) d.push_back({u_off + t * nu + i, 2 * r_diag[i]});
  p.p = diag_csr(nvar, d);
  p.q.assign(nvar, 0.0);
  RowBuilder A(nvar, u64(T) * nx * (nx + nu + 1) + 2ull * nvar);
  for (u32 i = 0; i < nx; ++i) {
    A.put(i, 1.0);
    A.end_row();
    p.l.push_back(x_init[i]);
    p.u.push_back(x_init[i]);
  }
  for (u32 t = 0; t < T; ++t)
    for (u32 i = 0; i < nx; ++i) {
      for (u32 j = 0; j < nx; ++j) {
        const double v = a_dyn[size_t(i) * nx + j];
        if (v != 0.0) A.put(t * nx + j, v);
      }
      A.put((t + 1) * nx + i, -1.0);
      for (u32 j = 0; j < nu; ++j) {
        const double v = b_in[size_t(i) * nu + j];
        if (v != 0.0) A.put(u_off + t * nu + j, v);
      }
      A.end_row();
      p.l.push_back(0.0);
      p.u.push_back(0.0);
    }
  for (u32 t = 1; t <= T; ++t)
    for (u32 i = 0; i < nx; ++i) {
      A.put(t * nx + i, 1.0);
      A.end_row();
      p.l.push_back(-x_bound);
      p.u.push_back(x_bound);
    }
  for (u32 t = 0; t < T; ++t)
    for (u32 i = 0; i < nu; ++i) {
      A.put(u_off + t * nu + i, 1.0);
      A.end_row();
      p.l.push_back(-u_bound);
      p.u.push_back(u_bound);
    }
  p.a = std::move(A.m);
  return p;
}

// ----------------------------------------------------------- gen_* recipes
enum Cls { kControl = 0, kEquality, kHuber, kLasso, kPortfolio, kRandom, kSvm };

// generators.hpp:643-667 with explicit sizes
Qp gen_random(Rng& rng, u32 n, u32 m, u32 p_per_row) {
  Qp p;
  p.p = gram_psd_upper(rng, n, n, p_per_row, 0.1);
  p.q.resize(n);
  for (double& v : p.q) v = rng.normal();
  p.a = sample_sparse(rng, m, n, 0.15);
  std::vector<double> x0(n);
  for (double& v : x0) v = rng.normal();
  const std::vector<double> ax0 = spmv(p.a, x0);
  p.l.resize(m);
  p.u.resize(m);
  for (u32 i = 0; i < m; ++i) {
    p.l[i] = ax0[i] - rng.uniform(0.05, 1.05);
    p.u[i] = ax0[i] + rng.uniform(0.05, 1.05);
  }
  return p;
}
// generators.hpp:606-625
Qp gen_lasso(Rng& rng, u32 n, u32 md) {
  Csr a = sample_sparse(rng, md, n, 0.15);
  std::vector<double> x_true(n, 0.0);
  for (double& v : x_true)
    if (rng.bernoulli(0.1)) v = rng.normal();
  std::vector<double> b = spmv(a, x_true);
  for (double& v : b) v += 0.01 * rng.normal();
  const double lambda = inf_norm(spmv_transpose(a, b)) / 5.0;
  return make_lasso(a, b, lambda);
}
// generators.hpp:584-603
Qp gen_huber(Rng& rng, u32 n, u32 md) {
  Csr a = sample_sparse(rng, md, n, 0.15);
  std::vector<double> x_true(n);
  for (double& v : x_true) v = rng.normal();
  std::vector<double> b = spmv(a, x_true);
  for (double& v : b) v += 0.01 * rng.normal();
  for (double& v : b)
    if (rng.bernoulli(0.1)) v += (rng.bernoulli(0.5) ? 1.0 : -1.0) * rng.uniform(5.0, 10.0);
  return make_huber(a, b, 1.0);
}
// generators.hpp:670-691
Qp gen_svm(Rng& rng, u32 n, u32 md) {
  const double shift = 1.0 / std::sqrt(0.15 * double(n));
  std::vector<double> labels(md), row_shift(md);
  for (u32 i = 0; i < md; ++i) {
    labels[i] = i < md / 2 ? 1.0 : -1.0;
    row_shift[i] = labels[i] * shift;
  }
  Csr a = sample_sparse(rng, md, n, 0.15, &row_shift);
  return make_svm(a, labels, 1.0);
}
// generators.hpp:628-641
Qp gen_portfolio(Rng& rng, u32 n, u32 k) {
  Csr f_t = sample_sparse(rng, k, n, 0.5);
  std::vector<double> dd(n), mu(n);
  for (double& v : dd) v = rng.uniform(0.0, std::sqrt(double(k)));
  for (double& v : mu) v = rng.normal();
  return make_portfolio(f_t, dd, mu, 1.0);
}
// generators.hpp:564-581
Qp gen_equality(Rng& rng, u32 n, u32 rows) {
  Csr p_upper = gram_psd_upper(rng, n, n, 3, 0.1);
  std::vector<double> q(n);
  for (double& v : q) v = rng.normal();
  Csr a = sample_sparse(rng, rows, n, 0.15);
  std::vector<double> x0(n);
  for (double& v : x0) v = rng.normal();
  const std::vector<double> b = spmv(a, x0);
  Qp p;
  p.p = std::move(p_upper);
  p.q = std::move(q);
  p.a = std::move(a);
  p.l = b;
  p.u = b;
  return p;
}
// generators.hpp:529-561
Qp gen_control(Rng& rng, u32 nx, u32 nu, u32 horizon) {
  std::vector<double> a_dyn(size_t(nx) * nx);
  for (double& v : a_dyn) v = rng.normal();
  double row_sum_norm = 0.0;
  for (u32 i = 0; i < nx; ++i) {
    double s = 0.0;
    for (u32 j = 0; j < nx; ++j) s += std::abs(a_dyn[size_t(i) * nx + j]);
    row_sum_norm = std::max(row_sum_norm, s);
  }
  if (row_sum_norm > 0.0)
    for (double& v : a_dyn) v *= 0.95 / row_sum_norm;
  std::vector<double> b_in(size_t(nx) * nu);
  for (double& v : b_in) v = rng.normal();
  std::vector<double> q_diag(nx), qt_diag(nx), r_diag(nu), x_init(nx);
  for (double& v : q_diag) v = rng.uniform(0.1, 2.0);
  for (double& v : qt_diag) v = rng.uniform(0.1, 2.0);
  for (double& v : r_diag) v = rng.uniform(0.1, 1.0);
  const double x_bound = rng.uniform(1.0, 3.0);
  const double u_bound = rng.uniform(0.5, 2.0);
  for (double& v : x_init) v = rng.uniform(-0.5, 0.5) * x_bound;
  return make_control(a_dyn, b_in, q_diag, r_diag, qt_diag, x_init, x_bound, u_bound, horizon);
}

// generators.hpp:200-204
u64 target_nnz(u32 scale) {
  if (scale == 0) return 300;
  return static_cast<u64>(std::llround(1000.0 * std::pow(10.0, (scale - 1) * 3.0 / 7.0)));
}

// generators.hpp:693-705 (generate<double>(BenchSpec))
Qp generate(int cls, u32 scale, u64 seed) {
  Rng rng(derive_key({u64(cls), u64(scale), seed}));
  const double target = static_cast<double>(target_nnz(scale));
  auto lr = [](double v) { return static_cast<u32>(std::lround(v)); };
  switch (cls) {
    case kControl: {
      const u32 nx = std::max<u32>(2, lr(std::sqrt(target / 15.0)));
      return gen_control(rng, nx, std::max<u32>(1, nx / 2), 10);
    }
    case kEquality: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target / 0.075)));
      return gen_equality(rng, n, std::max<u32>(1, n / 2));
    }
    case kHuber: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target / 0.3)));
      return gen_huber(rng, n, 2 * n);
    }
    case kLasso: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target / 0.3)));
      return gen_lasso(rng, n, 2 * n);
    }
    case kPortfolio: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target * 200.0)));
      return gen_portfolio(rng, n, std::max<u32>(1, n / 100));
    }
    case kRandom: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target / 1.5)));
      return gen_random(rng, n, 10 * n, 3);
    }
    case kSvm: {
      const u32 n = std::max<u32>(4, lr(std::sqrt(target / 0.3)));
      return gen_svm(rng, n, 2 * n);
    }
  }
  throw std::invalid_argument("generate: unknown problem class");
}

// explicit sizes; kinds as oracle/ref_driver.cpp
Qp generate_explicit(int kind, u32 a, u32 b, u32 c, u64 seed) {
  static const int cls_of[] = {kRandom, kLasso, kHuber, kSvm, kPortfolio, kEquality, kControl};
  if (kind < 0 || kind > 6) throw std::invalid_argument("unknown kind");
  Rng rng(derive_key({u64(cls_of[kind]), u64(100), seed}));
  switch (kind) {
    case 0: return gen_random(rng, a, b, c);
    case 1: return gen_lasso(rng, a, b);
    case 2: return gen_huber(rng, a, b);
    case 3: return gen_svm(rng, a, b);
    case 4: return gen_portfolio(rng, a, b);
    case 5: return gen_equality(rng, a, b);
    default: return gen_control(rng, a, b, c);
  }
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* qgen_last_error() { return g_err.c_str(); }
void qgen_set_threads(int t) { g_threads = t; }

void* qgen_class(int cls, uint32_t scale, uint64_t seed) {
  try {
    return new Qp(generate(cls, scale, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* qgen_explicit(int kind, uint32_t a, uint32_t b, uint32_t c, uint64_t seed) {
  try {
    return new Qp(generate_explicit(kind, a, b, c, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

uint64_t qgen_target_nnz(uint32_t scale) { return target_nnz(scale); }

void qgen_dims(const void* h, uint64_t* dims) {
  const Qp* p = static_cast<const Qp*>(h);
  dims[0] = p->p.rows;
  dims[1] = p->a.rows;
  dims[2] = p->p.nnz();
  dims[3] = p->a.nnz();
}

void qgen_export(const void* h, double* pv, uint32_t* prp, uint32_t* pci, double* q, double* av,
                 uint32_t* arp, uint32_t* aci, double* l, double* u) {
  const Qp* p = static_cast<const Qp*>(h);
  auto cp = [](void* dst, const void* src, size_t bytes) {
    if (bytes) std::memcpy(dst, src, bytes);
  };
  cp(pv, p->p.val.data(), 8 * p->p.val.size());
  cp(prp, p->p.rp.data(), 4 * p->p.rp.size());
  cp(pci, p->p.ci.data(), 4 * p->p.ci.size());
  cp(q, p->q.data(), 8 * p->q.size());
  // large arrays copied in parallel slices
  const Csr& A = p->a;
  const u64 nz = A.val.size();
  parallel_for((nz + (1 << 22) - 1) >> 22, [&](u64 b) {
    const u64 lo = b << 22, n = std::min<u64>(nz, lo + (1 << 22)) - lo;
    std::memcpy(av + lo, A.val.data() + lo, 8 * n);
    std::memcpy(aci + lo, A.ci.data() + lo, 4 * n);
  });
  cp(arp, A.rp.data(), 4 * A.rp.size());
  cp(l, p->l.data(), 8 * p->l.size());
  cp(u, p->u.data(), 8 * p->u.size());
}

void qgen_free(void* h) { delete static_cast<Qp*>(h); }

}  // extern "C"
