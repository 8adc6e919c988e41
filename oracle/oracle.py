"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end for the two CPU checkers:

* ``REF``    oracle/_ref/libqpcg_ref.so — the unmodified reference headers
             (solver.hpp / linsys.hpp / scaling.hpp / sparse.hpp / generators.hpp)
             behind ref_driver.cpp; also the reference's problem generators.
* ``ORACLE`` oracle/liboracle.so — the plain-C restatement (qpcg_oracle.c),
             pinned bit-for-bit to REF by tests/test_oracle_pin.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1912_04263_b200 import _abi
from paper_1912_04263_b200.problem import (CsrMatrix, NotPositiveDefiniteError, QpProblem,
                                           Settings, SolveDiagnostics, outcome_from_c)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libqpcg_ref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

# ProblemClass order, generators.hpp:150-158
CLASSES = ["control", "equality", "huber", "lasso", "portfolio", "random", "svm"]


def build() -> None:
    """Compile the oracle (and _ref when /root/reference is present)."""
    subprocess.check_call(["make", "-s", "-C", HERE, "all"])


_libs: dict = {}


def _load(path: str) -> C.CDLL:
    if path not in _libs:
        if not os.path.exists(path):
            build()
        _libs[path] = C.CDLL(path)
    return _libs[path]


def ref_lib() -> C.CDLL:
    lib = _load(REF_SO)
    lib.qref_gen_class.restype = C.c_void_p
    lib.qref_gen_class.argtypes = [C.c_int, C.c_uint32, C.c_uint64]
    lib.qref_gen_explicit.restype = C.c_void_p
    lib.qref_gen_explicit.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
    lib.qref_problem_free.argtypes = [C.c_void_p]
    lib.qref_problem_dims.argtypes = [C.c_void_p, C.c_void_p]
    lib.qref_problem_export.argtypes = [C.c_void_p] + [C.c_void_p] * 9
    lib.qref_last_error.restype = C.c_char_p
    lib.qref_target_nnz.restype = C.c_uint64
    lib.qref_symmetrize_f64.restype = C.c_int64
    lib.qref_pcg_cap_f64.restype = C.c_uint32
    return lib


def oracle_lib() -> C.CDLL:
    lib = _load(ORACLE_SO)
    lib.oracle_last_error.restype = C.c_char_p
    lib.oracle_f64_symmetrize.restype = C.c_int64
    return lib


# ---------------------------------------------------------------- generation
def _export(h) -> QpProblem:
    lib = ref_lib()
    if not h:
        raise RuntimeError(lib.qref_last_error().decode())
    dims = np.zeros(4, np.uint64)
    lib.qref_problem_dims(C.c_void_p(h), dims.ctypes.data)
    n, m, nnzp, nnza = (int(v) for v in dims)
    pv, prp, pci = np.empty(nnzp), np.empty(n + 1, np.uint32), np.empty(nnzp, np.uint32)
    av, arp, aci = np.empty(nnza), np.empty(m + 1, np.uint32), np.empty(nnza, np.uint32)
    q, l, u = np.empty(n), np.empty(m), np.empty(m)
    lib.qref_problem_export(C.c_void_p(h), *[a.ctypes.data for a in (pv, prp, pci, q, av, arp, aci, l, u)])
    lib.qref_problem_free(C.c_void_p(h))
    return QpProblem(CsrMatrix(n, n, pv, prp, pci), q, CsrMatrix(m, n, av, arp, aci), l, u)


def ref_generate(cls: str, scale: int, seed: int = 0) -> QpProblem:
    """bench::generate<double>(BenchSpec{cls, scale, seed}), generators.hpp:693-705."""
    return _export(ref_lib().qref_gen_class(CLASSES.index(cls), scale, seed))


EXPLICIT_KINDS = {"random": 0, "lasso": 1, "huber": 2, "svm": 3, "portfolio": 4,
                  "equality": 5, "control": 6}


def ref_generate_explicit(kind: str, a: int, b: int, c: int = 0, seed: int = 0) -> QpProblem:
    """Explicit-size instances of SURVEY.md §8(d) through the reference's recipes."""
    return _export(ref_lib().qref_gen_explicit(EXPLICIT_KINDS[kind], a, b, c, seed))


# --------------------------------------------------------------------- solve
def _solve(lib, fn, diag_fns, p: QpProblem, settings: Settings | None, warm=None,
           diag: SolveDiagnostics | None = None, err_fn=None):
    dt = p.dtype
    n, m = p.n, p.m
    s = (settings or Settings()).to_c()
    x, z, y = np.zeros(n, dt), np.zeros(m, dt), np.zeros(m, dt)
    cert = np.zeros(max(n, m), dt)
    info = _abi.Info()
    pv, av = p.p_upper.view(), p.a.view()
    w = (None, None, None) if warm is None else tuple(np.ascontiguousarray(v, dt) for v in (warm.x, warm.z, warm.y))
    rc = fn(C.byref(pv), _abi.ptr(p.q), C.byref(av), _abi.ptr(p.l), _abi.ptr(p.u), C.byref(s),
            *[_abi.ptr(v) for v in w], C.byref(info), _abi.ptr(x), _abi.ptr(z), _abi.ptr(y),
            _abi.ptr(cert), 1 if diag is not None else 0)
    if rc != _abi.QPCG_OK:
        msg = err_fn().decode()
        if rc == _abi.QPCG_ERR_NOT_PD:
            raise NotPositiveDefiniteError(msg)
        if rc == _abi.QPCG_ERR_INVALID:
            raise ValueError(msg)
        raise RuntimeError(msg)
    if diag is not None:
        calls_fn, rho_fn, checks_fn = diag_fns
        k = calls_fn(None, 0)
        buf = (_abi.PcgCall * max(k, 1))()
        calls_fn(buf, k)
        diag.pcg_calls = [dict(admm_iter=c.admm_iter, iterations=c.iterations, eps=c.eps,
                               r_prim_scaled_inf=c.r_prim_scaled_inf,
                               r_dual_scaled_inf=c.r_dual_scaled_inf, converged=bool(c.converged))
                          for c in buf[:k]]
        k = rho_fn(None, 0)
        rb = (_abi.RhoUpdate * max(k, 1))()
        rho_fn(rb, k)
        diag.rho_updates = [dict(admm_iter=r.admm_iter, rho_before=r.rho_before,
                                 rho_after=r.rho_after) for r in rb[:k]]
        k = checks_fn(None, 0)
        cb = (C.c_uint32 * max(k, 1))()
        checks_fn(cb, k)
        diag.check_iterations = list(cb[:k])
    return outcome_from_c(info, x, z, y, cert)


def ref_solve(p: QpProblem, settings: Settings | None = None, warm=None, diag=None):
    """qpcg::solve (solver.hpp:386-541) — the reference itself."""
    lib = ref_lib()
    fn = lib.qref_solve_f64 if p.dtype == np.float64 else lib.qref_solve_f32
    return _solve(lib, fn, (lib.qref_diag_pcg_calls, lib.qref_diag_rho_updates, lib.qref_diag_checks),
                  p, settings, warm, diag, lib.qref_last_error)


def oracle_solve(p: QpProblem, settings: Settings | None = None, warm=None, diag=None):
    """The plain-C restatement of qpcg::solve."""
    lib = oracle_lib()
    fn = lib.oracle_f64_solve if p.dtype == np.float64 else lib.oracle_f32_solve
    return _solve(lib, fn, (lib.oracle_diag_pcg_calls, lib.oracle_diag_rho_updates,
                            lib.oracle_diag_checks), p, settings, warm, diag, lib.oracle_last_error)


# ------------------------------------------------------------ building blocks
def _which(kind: str):
    return (ref_lib(), "qref_") if kind == "ref" else (oracle_lib(), "oracle_")


def spmv(m: CsrMatrix, x: np.ndarray, kind: str = "oracle") -> np.ndarray:
    lib, pre = _which(kind)
    dt = m.values.dtype
    suf = "f64" if dt == np.float64 else "f32"
    fn = getattr(lib, f"{pre}{suf}_spmv" if kind == "oracle" else f"qref_spmv_{suf}")
    y = np.zeros(m.rows, dt)
    x = np.ascontiguousarray(x, dt)
    v = m.view()
    fn(C.byref(v), _abi.ptr(x), _abi.ptr(y))
    return y


def transpose(m: CsrMatrix, kind: str = "oracle") -> CsrMatrix:
    lib, _ = _which(kind)
    fn = lib.oracle_f64_transpose if kind == "oracle" else lib.qref_transpose_f64
    vals = np.zeros(m.nnz, np.float64)
    rp, ci = np.zeros(m.cols + 1, np.uint32), np.zeros(m.nnz, np.uint32)
    v = m.astype(np.float64).view()
    fn(C.byref(v), _abi.ptr(vals), _abi.ptr(rp), _abi.ptr(ci))
    return CsrMatrix(m.cols, m.rows, vals.astype(m.values.dtype), rp, ci)


def symmetrize_upper(m: CsrMatrix, kind: str = "oracle") -> CsrMatrix:
    lib, _ = _which(kind)
    fn = lib.oracle_f64_symmetrize if kind == "oracle" else lib.qref_symmetrize_f64
    fn.restype = C.c_int64
    v = m.astype(np.float64).view()
    nnz = fn(C.byref(v), None, None, None)
    if nnz < 0:
        raise ValueError("symmetrize_upper failed")
    vals, rp, ci = np.zeros(nnz), np.zeros(m.rows + 1, np.uint32), np.zeros(nnz, np.uint32)
    fn(C.byref(v), _abi.ptr(vals), _abi.ptr(rp), _abi.ptr(ci))
    return CsrMatrix(m.rows, m.cols, vals.astype(m.values.dtype), rp, ci)


def ruiz(p_full: CsrMatrix, q, a: CsrMatrix, l, u, eps_equil=1e-3, passes=10, kind="oracle"):
    """ruiz_equilibrate (scaling.hpp:92-187); returns a dict of the scaled problem."""
    lib, _ = _which(kind)
    dt = p_full.values.dtype
    suf = "f64" if dt == np.float64 else "f32"
    fn = getattr(lib, f"oracle_{suf}_ruiz" if kind == "oracle" else f"qref_ruiz_{suf}")
    n, m = p_full.rows, a.rows
    out = dict(p_values=np.zeros(p_full.nnz, dt), q=np.zeros(n, dt), a_values=np.zeros(a.nnz, dt),
               at_values=np.zeros(a.nnz, dt), at_row_ptr=np.zeros(n + 1, np.uint32),
               at_col=np.zeros(a.nnz, np.uint32), l=np.zeros(m, dt), u=np.zeros(m, dt),
               d=np.zeros(n, dt), e=np.zeros(m, dt), d_inv=np.zeros(n, dt), e_inv=np.zeros(m, dt))
    scal = np.zeros(4)
    pv, av = p_full.view(), a.view()
    rc = fn(C.byref(pv), _abi.ptr(np.ascontiguousarray(q, dt)), C.byref(av),
            _abi.ptr(np.ascontiguousarray(l, dt)), _abi.ptr(np.ascontiguousarray(u, dt)),
            C.c_double(eps_equil), C.c_uint32(passes),
            *[_abi.ptr(out[k]) for k in ("p_values", "q", "a_values", "at_values", "at_row_ptr",
                                          "at_col", "l", "u", "d", "e", "d_inv", "e_inv")],
            _abi.ptr(scal))
    if rc != 0:
        raise ValueError("ruiz failed")
    out.update(c=scal[0], c_inv=scal[1], passes_used=int(scal[2]), deviation=scal[3])
    return out


def kkt_apply(pf: CsrMatrix, a: CsrMatrix, at: CsrMatrix, sigma, rho, x, kind="oracle"):
    lib, _ = _which(kind)
    fn = lib.oracle_f64_kkt_apply if kind == "oracle" else lib.qref_kkt_apply_f64
    out, dm = np.zeros(pf.rows), np.zeros(pf.rows)
    v1, v2, v3 = pf.view(), a.view(), at.view()
    rc = fn(C.byref(v1), C.byref(v2), C.byref(v3), C.c_double(sigma), C.c_double(rho),
            _abi.ptr(np.ascontiguousarray(x, np.float64)), _abi.ptr(out), _abi.ptr(dm))
    if rc != 0:
        raise ValueError("kkt_apply failed")
    return out, dm


def pcg(pf, a, at, sigma, rho, b, warm, eps, max_iter, kind="oracle"):
    lib, _ = _which(kind)
    fn = lib.oracle_f64_pcg if kind == "oracle" else lib.qref_pcg_f64
    x, res = np.zeros(pf.rows), np.zeros(3)
    v1, v2, v3 = pf.view(), a.view(), at.view()
    rc = fn(C.byref(v1), C.byref(v2), C.byref(v3), C.c_double(sigma), C.c_double(rho),
            _abi.ptr(np.ascontiguousarray(b, np.float64)),
            _abi.ptr(np.ascontiguousarray(warm, np.float64)), C.c_double(eps),
            C.c_uint32(max_iter), _abi.ptr(x), _abi.ptr(res))
    if rc == _abi.QPCG_ERR_NOT_PD:
        raise NotPositiveDefiniteError("pcg")
    if rc != 0:
        raise ValueError("pcg failed")
    return x, int(res[0]), res[1], bool(res[2])


def adaptive_eps(rp, rd, lam, eps_min, kind="oracle"):
    lib, _ = _which(kind)
    fn = lib.oracle_f64_adaptive_eps if kind == "oracle" else lib.qref_adaptive_eps_f64
    out = C.c_double()
    rc = fn(C.c_double(rp), C.c_double(rd), C.c_double(lam), C.c_double(eps_min), C.byref(out))
    if rc != 0:
        raise ValueError("adaptive_eps")
    return out.value


def pcg_cap(n: int, dtype=np.float64, kind="oracle") -> int:
    lib, _ = _which(kind)
    suf = "f64" if dtype == np.float64 else "f32"
    fn = getattr(lib, f"oracle_pcg_cap_{suf}" if kind == "oracle" else f"qref_pcg_cap_{suf}")
    fn.restype = C.c_uint32
    return int(fn(C.c_uint32(n)))
