// textio.cpp — the reference's text problem format (io.hpp:14-19, 86-168),
// read and written natively and in parallel.
//
//   matrix   "rows cols nnz", then nnz lines "row col value", sorted
//            zero-based coordinate order (write_matrix / read_matrix :87-112)
//   vector   one value per line, inf / -inf spelled out (:114-131)
//   problem  "n m", P upper block, q, A block, l, u (:133-156)
//
// Reading follows the reference's std::istream semantics token for token:
// indices are `is >> long long` (skip whitespace, optional sign, digits; a
// negative value or no digits is "io: bad index field", :67-71), scalars are a
// whitespace-delimited token converted by std::stod / std::stof (strtod /
// strtof on the token's prefix: no conversion or ERANGE is "io: cannot parse
// value '<token>'", :46-58), end of input before a token is "io: unexpected
// end of input" (:62-64).  The COO block is then validated like
// validate(CooMatrix) (sparse.hpp:76-96), converted like coo_to_csr
// (:158-173), the header checked (:149-151) and the problem validated like
// validate(QpProblem) (problem.hpp:47-92), with the reference's messages.
// Errors are reported with their kind: 1 = std::runtime_error (io), 2 =
// std::invalid_argument (validation).
//
// A block of a matrix's "row col value" lines is parsed in parallel slices
// when every line of it holds exactly those three fields (the layout the
// writer produces); any other layout is parsed sequentially with the same
// token rules, so the result never depends on the path taken.
//
// Writing reproduces `os << setprecision(max_digits10) << v` (libstdc++
// formats it as printf "%.*g": 17 digits for double, 9 for float) with
// inf / -inf spelled out (:73-82), formatted in parallel slices and written in
// order.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace {

using u32 = uint32_t;
using u64 = uint64_t;

struct IoError {
  int kind;  // 1 runtime_error, 2 invalid_argument
  std::string msg;
};
[[noreturn]] void io_fail(const std::string& m) { throw IoError{1, m}; }
[[noreturn]] void arg_fail(const std::string& m) { throw IoError{2, m}; }

int io_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return h ? int(h) : 1;
}
template <class F>
void parallel_each(u64 n, F f) {  // f(i) for i < n, on up to io_threads() threads
  const u64 t = std::min<u64>(u64(io_threads()), n);
  if (t <= 1) {
    for (u64 i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (u64 w = 0; w < t; ++w)
    th.emplace_back([&, w] {
      for (u64 i = w; i < n; i += t) f(i);
    });
  for (auto& x : th) x.join();
}

inline bool is_ws(char c) {  // std::isspace in the "C" locale
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// istream-like cursor over a NUL-terminated buffer [p, end)
struct Cursor {
  const char* p;
  const char* end;
  void skip_ws() {
    while (p < end && is_ws(*p)) ++p;
  }
  // is >> long long, then the v < 0 check (io.hpp:67-71)
  bool index(u32& out) {
    skip_ws();
    if (p >= end) return false;
    errno = 0;
    char* e = nullptr;
    const long long v = std::strtoll(p, &e, 10);
    if (e == p || errno == ERANGE || v < 0) return false;
    p = e;
    out = static_cast<u32>(v);  // static_cast<index_t>, as the reference (wraps)
    return true;
  }
  u32 next_index() {
    u32 v;
    if (!index(v)) io_fail("io: bad index field");
    return v;
  }
  // is >> token; std::stod / std::stof (io.hpp:46-65)
  template <typename T>
  double next_scalar() {
    skip_ws();
    if (p >= end) io_fail("io: unexpected end of input");
    const char* t = p;
    while (p < end && !is_ws(*p)) ++p;
    errno = 0;
    char* e = nullptr;
    double v;
    if (sizeof(T) == 4) v = double(std::strtof(t, &e));
    else v = std::strtod(t, &e);
    if (e == t || errno == ERANGE) io_fail("io: cannot parse value '" + std::string(t, p) + "'");
    return v;
  }
};

struct Block {  // one matrix in COO order
  u32 rows = 0, cols = 0;
  std::vector<u32> ri, ci;
  std::vector<double> val;
};

// Parse n "r c v" lines starting at cur.p in parallel; false (cursor
// untouched) when the text is not exactly n such lines.
template <typename T>
bool parse_lines_parallel(Cursor& cur, u64 n, Block& b) {
  static const u64 min_n = [] {  // QPCG_IO_PAR_MIN: smallest block parsed in parallel
    const char* e = std::getenv("QPCG_IO_PAR_MIN");
    return e ? std::strtoull(e, nullptr, 10) : u64(1) << 20;
  }();
  if (n < min_n || n == 0) return false;
  // the entries start on the line after the header
  const char* s = cur.p;
  while (s < cur.end && (*s == ' ' || *s == '\t' || *s == '\r')) ++s;
  if (s >= cur.end || *s != '\n') return false;
  ++s;
  // find the end of the n-th line
  const int t = io_threads();
  // cut [s, ...) into slices at newlines, counting lines per slice
  const char* lim = cur.end;
  std::vector<const char*> cut(t + 1);
  cut[0] = s;
  for (int i = 1; i < t; ++i) {
    const char* c = s + (lim - s) * i / t;
    if (c < cut[i - 1]) c = cut[i - 1];
    const char* nl = static_cast<const char*>(std::memchr(c, '\n', size_t(lim - c)));
    cut[i] = nl ? nl + 1 : lim;
  }
  cut[t] = lim;
  std::vector<u64> lines(t, 0);
  parallel_each(u64(t), [&](u64 i) {
    u64 c = 0;
    for (const char* q = cut[i]; q < cut[i + 1];) {
      const char* nl = static_cast<const char*>(std::memchr(q, '\n', size_t(cut[i + 1] - q)));
      if (!nl) break;
      ++c;
      q = nl + 1;
    }
    lines[i] = c;
  });
  // the slice holding line n: the block ends after its n-th newline
  u64 before = 0;
  int last = -1;
  for (int i = 0; i < t; ++i) {
    if (before + lines[i] >= n) {
      last = i;
      break;
    }
    before += lines[i];
  }
  if (last < 0) return false;  // fewer than n full lines: the sequential path reports it
  const char* stop = cut[last];
  for (u64 k = before; k < n; ++k) stop = static_cast<const char*>(std::memchr(stop, '\n', size_t(lim - stop))) + 1;
  // slices over [s, stop) at newlines; each parses its lines into a prefix-summed position
  std::vector<const char*> sl(t + 1);
  sl[0] = s;
  for (int i = 1; i < t; ++i) {
    const char* c = s + (stop - s) * i / t;
    if (c < sl[i - 1]) c = sl[i - 1];
    const char* nl = static_cast<const char*>(std::memchr(c, '\n', size_t(stop - c)));
    sl[i] = nl ? nl + 1 : stop;
  }
  sl[t] = stop;
  std::vector<u64> cnt(t, 0), off(t + 1, 0);
  parallel_each(u64(t), [&](u64 i) {
    u64 c = 0;
    for (const char* q = sl[i]; q < sl[i + 1];) {
      q = static_cast<const char*>(std::memchr(q, '\n', size_t(sl[i + 1] - q))) + 1;
      ++c;
    }
    cnt[i] = c;
  });
  for (int i = 0; i < t; ++i) off[i + 1] = off[i] + cnt[i];
  if (off[t] != n) return false;
  b.ri.resize(n);
  b.ci.resize(n);
  b.val.resize(n);
  std::vector<int> ok(t, 1);
  std::vector<IoError> err(t);
  std::vector<int> has_err(t, 0);
  parallel_each(u64(t), [&](u64 i) {
    {
      Cursor c{sl[i], stop};
      u64 k = off[i];
      try {
        while (c.p < sl[i + 1]) {
          const char* line_end =
              static_cast<const char*>(std::memchr(c.p, '\n', size_t(sl[i + 1] - c.p)));
          // fields must all lie on this line
          u32 r, cc;
          Cursor lc{c.p, line_end};
          lc.skip_ws();
          if (lc.p >= line_end) { ok[i] = 0; return; }
          if (!lc.index(r) || lc.p > line_end) { ok[i] = 0; return; }
          lc.skip_ws();
          if (lc.p >= line_end) { ok[i] = 0; return; }
          if (!lc.index(cc) || lc.p > line_end) { ok[i] = 0; return; }
          lc.skip_ws();
          if (lc.p >= line_end) { ok[i] = 0; return; }
          const char* tk = lc.p;
          while (lc.p < line_end && !is_ws(*lc.p)) ++lc.p;
          errno = 0;
          char* e = nullptr;
          const double v = sizeof(T) == 4 ? double(std::strtof(tk, &e)) : std::strtod(tk, &e);
          if (e == tk || errno == ERANGE) {
            // the token rule decides: report as the sequential reader would
            err[i] = IoError{1, "io: cannot parse value '" + std::string(tk, lc.p) + "'"};
            has_err[i] = 1;
            return;
          }
          lc.skip_ws();
          if (lc.p != line_end) { ok[i] = 0; return; }
          b.ri[k] = r;
          b.ci[k] = cc;
          b.val[k] = v;
          ++k;
          c.p = line_end + 1;
        }
      } catch (...) {
        ok[i] = 0;
      }
    }
  });
  for (int i = 0; i < t; ++i) {
    if (!ok[i]) return false;
  }
  for (int i = 0; i < t; ++i) {
    if (has_err[i]) throw err[i];  // first slice in file order
  }
  cur.p = stop;
  return true;
}

template <typename T>
Block read_block(Cursor& cur) {
  Block b;
  b.rows = cur.next_index();
  b.cols = cur.next_index();
  const u32 nnz = cur.next_index();
  if (!parse_lines_parallel<T>(cur, nnz, b)) {
    b.ri.clear();
    b.ci.clear();
    b.val.clear();
    b.ri.reserve(nnz);
    b.ci.reserve(nnz);
    b.val.reserve(nnz);
    for (u32 k = 0; k < nnz; ++k) {
      b.ri.push_back(cur.next_index());
      b.ci.push_back(cur.next_index());
      b.val.push_back(cur.next_scalar<T>());
    }
  }
  // validate(CooMatrix) (sparse.hpp:76-96)
  const u64 n = b.val.size();
  for (u64 k = 0; k < n; ++k) {
    if (b.ri[k] >= b.rows || b.ci[k] >= b.cols) arg_fail("coo: entry index out of bounds");
    if (k > 0) {
      const bool row_ok = b.ri[k] > b.ri[k - 1];
      const bool col_ok = b.ri[k] == b.ri[k - 1] && b.ci[k] > b.ci[k - 1];
      if (!row_ok && !col_ok)
        arg_fail("coo: entries must be sorted by row then column, without duplicates");
    }
  }
  return b;
}

struct Csr {
  u32 rows = 0, cols = 0;
  std::vector<double> val;
  std::vector<u32> rp, ci;
};
Csr coo_to_csr(Block&& b) {  // sparse.hpp:158-173
  Csr m;
  m.rows = b.rows;
  m.cols = b.cols;
  m.val = std::move(b.val);
  m.ci = std::move(b.ci);
  m.rp.assign(size_t(m.rows) + 1, 0);
  for (u32 r : b.ri) ++m.rp[size_t(r) + 1];
  for (u32 r = 0; r < m.rows; ++r) m.rp[r + 1] += m.rp[r];
  return m;
}

template <typename T>
std::vector<double> read_vec(Cursor& cur, u64 count) {
  std::vector<double> v;
  v.reserve(count);
  for (u64 i = 0; i < count; ++i) v.push_back(cur.next_scalar<T>());
  return v;
}

struct Problem {
  Csr p, a;
  std::vector<double> q, l, u;
};

void validate_problem(const Problem& p) {  // problem.hpp:47-92 (CSR parts hold by construction)
  if (p.p.rows != p.p.cols) arg_fail("problem: P must be square");
  if (p.p.rows == 0) arg_fail("problem: at least one variable required");
  for (u32 r = 0; r < p.p.rows; ++r)
    for (u32 k = p.p.rp[r]; k < p.p.rp[r + 1]; ++k)
      if (p.p.ci[k] < r) arg_fail("problem: P has entries below diagonal");
  if (p.a.cols != p.p.cols) arg_fail("problem: A column count must equal n");
  if (p.q.size() != p.p.rows) arg_fail("problem: q length must equal n");
  if (p.l.size() != p.a.rows || p.u.size() != p.a.rows) arg_fail("problem: bound lengths must equal m");
  for (double v : p.p.val)
    if (!std::isfinite(v)) arg_fail("problem: P not finite");
  for (double v : p.a.val)
    if (!std::isfinite(v)) arg_fail("problem: A not finite");
  for (double v : p.q)
    if (!std::isfinite(v)) arg_fail("problem: q not finite");
  for (u32 i = 0; i < p.a.rows; ++i) {
    if (std::isnan(p.l[i]) || std::isnan(p.u[i])) arg_fail("problem: bounds contain NaN");
    if (p.l[i] == HUGE_VAL || p.u[i] == -HUGE_VAL)
      arg_fail("problem: l must be < +inf and u > -inf");
    if (p.l[i] > p.u[i]) arg_fail("problem: l must not exceed u");
  }
}

template <typename T>
Problem read_problem(const std::string& text) {  // io.hpp:143-156
  Cursor cur{text.c_str(), text.c_str() + text.size()};
  Problem p;
  const u32 n = cur.next_index();
  const u32 m = cur.next_index();
  p.p = coo_to_csr(read_block<T>(cur));
  p.q = read_vec<T>(cur, n);
  p.a = coo_to_csr(read_block<T>(cur));
  p.l = read_vec<T>(cur, m);
  p.u = read_vec<T>(cur, m);
  if (p.p.rows != n || p.a.rows != m) io_fail("io: problem header does not match blocks");
  validate_problem(p);
  return p;
}

// ----------------------------------------------------------------- writing
template <typename T>
inline void put_scalar(std::string& o, double v) {  // io.hpp:73-82
  if (v == HUGE_VAL) {
    o += "inf";
  } else if (v == -HUGE_VAL) {
    o += "-inf";
  } else {
    char buf[48];
    const int k = std::snprintf(buf, sizeof buf, "%.*g", sizeof(T) == 4 ? 9 : 17, v);
    o.append(buf, size_t(k));
  }
}
inline void put_u32(std::string& o, u32 v) {
  char buf[16];
  const int k = std::snprintf(buf, sizeof buf, "%u", v);
  o.append(buf, size_t(k));
}

struct Out {
  std::FILE* f;
  void put(const std::string& s) {
    if (!s.empty() && std::fwrite(s.data(), 1, s.size(), f) != s.size()) io_fail("io: write failed");
  }
};

// validate(CsrMatrix) (sparse.hpp:98-123), as csr_to_coo runs it
void validate_csr(u32 rows, u32 cols, u64 nnz, const u32* rp, const u32* ci) {
  if (rp[0] != 0 || rp[rows] != nnz) arg_fail("csr: row_ptr must start at 0 and end at nnz");
  for (u32 r = 0; r < rows; ++r) {
    if (rp[r + 1] < rp[r]) arg_fail("csr: row_ptr must be nondecreasing");
    for (u32 k = rp[r]; k < rp[r + 1]; ++k) {
      if (ci[k] >= cols) arg_fail("csr: column index out of bounds");
      if (k > rp[r] && ci[k] <= ci[k - 1])
        arg_fail("csr: column indices must be strictly increasing within a row");
    }
  }
}

template <typename T>
void write_matrix(Out& out, u32 rows, u32 cols, u64 nnz, const double* v, const u32* rp,
                  const u32* ci) {  // io.hpp:86-96
  validate_csr(rows, cols, nnz, rp, ci);
  std::string h;
  put_u32(h, rows);
  h += ' ';
  put_u32(h, cols);
  h += ' ';
  h += std::to_string(nnz);
  h += '\n';
  out.put(h);
  // row of every entry, then the lines formatted in parallel slices of rows
  const int t = io_threads();
  const u64 nsl = std::max<u64>(1, std::min<u64>(u64(t) * 8, nnz / 65536 + 1));
  std::vector<std::string> text(nsl);
  // slice s covers rows [r0, r1) with about nnz / nsl entries
  std::vector<u32> rcut(nsl + 1, rows);
  rcut[0] = 0;
  for (u64 s = 1; s < nsl; ++s) {
    const u64 target = nnz * s / nsl;
    u32 lo = rcut[s - 1], hi = rows;  // first row with rp[row] >= target
    while (lo < hi) {
      const u32 mid = lo + (hi - lo) / 2;
      if (rp[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    rcut[s] = lo;
  }
  parallel_each(nsl, [&](u64 s) {
    {
      std::string& o = text[s];
      o.reserve(size_t(rp[rcut[s + 1]] - rp[rcut[s]]) * 36);
      for (u32 r = rcut[s]; r < rcut[s + 1]; ++r)
        for (u32 k = rp[r]; k < rp[r + 1]; ++k) {
          put_u32(o, r);
          o += ' ';
          put_u32(o, ci[k]);
          o += ' ';
          put_scalar<T>(o, v[k]);
          o += '\n';
        }
    }
  });
  for (auto& s : text) out.put(s);
}

template <typename T>
void write_vector(Out& out, const double* v, u64 n) {  // io.hpp:114-120
  std::string o;
  o.reserve(size_t(n) * 26);
  for (u64 i = 0; i < n; ++i) {
    put_scalar<T>(o, v[i]);
    o += '\n';
  }
  out.put(o);
}

thread_local std::string g_err;
thread_local int g_err_kind = 0;

std::string slurp(const char* path) {
  std::FILE* f = std::fopen(path, "rb");
  if (!f) io_fail(std::string("io: cannot open ") + path);
  std::string s;
  if (std::fseek(f, 0, SEEK_END) == 0) {
    const long len = std::ftell(f);
    if (len > 0) {
      s.resize(size_t(len));
      std::rewind(f);
      const size_t got = std::fread(&s[0], 1, size_t(len), f);
      s.resize(got);
    }
  }
  std::fclose(f);
  return s;
}

}  // namespace

extern "C" {

const char* qio_last_error() { return g_err.c_str(); }
int qio_last_error_kind() { return g_err_kind; }

// load_problem<T> (io.hpp:165-170): a handle, or null (qio_last_error*)
void* qio_read_problem(const char* path, int f32) {
  try {
    const std::string text = slurp(path);
    return new Problem(f32 ? read_problem<float>(text) : read_problem<double>(text));
  } catch (const IoError& e) {
    g_err = e.msg;
    g_err_kind = e.kind;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_kind = 1;
  }
  return nullptr;
}

void qio_dims(const void* h, uint64_t* dims) {
  const Problem* p = static_cast<const Problem*>(h);
  dims[0] = p->p.rows;
  dims[1] = p->a.rows;
  dims[2] = p->p.val.size();
  dims[3] = p->a.val.size();
  dims[4] = p->a.cols;
}

void qio_export(const void* h, double* pv, uint32_t* prp, uint32_t* pci, double* q, double* av,
                uint32_t* arp, uint32_t* aci, double* l, double* u) {
  const Problem* p = static_cast<const Problem*>(h);
  auto cp = [](void* dst, const void* src, size_t bytes) {
    if (bytes) std::memcpy(dst, src, bytes);
  };
  cp(pv, p->p.val.data(), 8 * p->p.val.size());
  cp(prp, p->p.rp.data(), 4 * p->p.rp.size());
  cp(pci, p->p.ci.data(), 4 * p->p.ci.size());
  cp(q, p->q.data(), 8 * p->q.size());
  cp(av, p->a.val.data(), 8 * p->a.val.size());
  cp(arp, p->a.rp.data(), 4 * p->a.rp.size());
  cp(aci, p->a.ci.data(), 4 * p->a.ci.size());
  cp(l, p->l.data(), 8 * p->l.size());
  cp(u, p->u.data(), 8 * p->u.size());
}

void qio_free(void* h) { delete static_cast<Problem*>(h); }

// save_problem<T> (io.hpp:133-140, 158-163); values as doubles (a float
// problem's values widen exactly).  0, or -1 (qio_last_error*).
int qio_write_problem(const char* path, int f32, uint32_t n, uint32_t p_cols, uint32_t m,
                      uint32_t a_cols,
                      uint64_t pnnz, const double* pv, const uint32_t* prp, const uint32_t* pci,
                      const double* q, uint64_t annz, const double* av, const uint32_t* arp,
                      const uint32_t* aci, const double* l, const double* u) {
  std::FILE* f = nullptr;
  try {
    f = std::fopen(path, "wb");
    if (!f) io_fail(std::string("io: cannot open ") + path);
    Out out{f};
    std::string h;
    put_u32(h, n);
    h += ' ';
    put_u32(h, m);
    h += '\n';
    out.put(h);
    if (f32) {
      write_matrix<float>(out, n, p_cols, pnnz, pv, prp, pci);
      write_vector<float>(out, q, n);
      write_matrix<float>(out, m, a_cols, annz, av, arp, aci);
      write_vector<float>(out, l, m);
      write_vector<float>(out, u, m);
    } else {
      write_matrix<double>(out, n, p_cols, pnnz, pv, prp, pci);
      write_vector<double>(out, q, n);
      write_matrix<double>(out, m, a_cols, annz, av, arp, aci);
      write_vector<double>(out, l, m);
      write_vector<double>(out, u, m);
    }
    if (std::fclose(f) != 0) {
      f = nullptr;
      io_fail("io: write failed");
    }
    return 0;
  } catch (const IoError& e) {
    g_err = e.msg;
    g_err_kind = e.kind;
  }
  if (f) std::fclose(f);
  return -1;
}

}  // extern "C"
