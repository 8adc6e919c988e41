"""Kernel-level parity: the device setup is bit-exact with the reference
(SURVEY.md §8(c) rungs 1-2), SpMV and the K-apply match within summation-order
rounding."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import _abi, generators as G, solver
from paper_1912_04263_b200.problem import CsrMatrix, Settings
from _util import paper_matrix

pytestmark = pytest.mark.gpu


def scaled_of(ws, dtype):
    lib = solver.load_library()
    dims = np.zeros(6, np.uint64)
    lib.qpcg_debug_dims.argtypes = [C.c_void_p, C.c_void_p]
    assert lib.qpcg_debug_dims(ws.ws, dims.ctypes.data) == 0
    n, m, nnzp, nnza = (int(v) for v in dims[:4])
    out = dict(p_values=np.zeros(nnzp, dtype), p_row_ptr=np.zeros(n + 1, np.uint32),
               p_col=np.zeros(nnzp, np.uint32), q=np.zeros(n, dtype), a_values=np.zeros(nnza, dtype),
               at_values=np.zeros(nnza, dtype), at_row_ptr=np.zeros(n + 1, np.uint32),
               at_col=np.zeros(nnza, np.uint32), l=np.zeros(m, dtype), u=np.zeros(m, dtype),
               d=np.zeros(n, dtype), e=np.zeros(m, dtype))
    scal = np.zeros(4)
    lib.qpcg_debug_scaled.argtypes = [C.c_void_p] + [C.c_void_p] * 13
    rc = lib.qpcg_debug_scaled(ws.ws, *[out[k].ctypes.data for k in (
        "p_values", "p_row_ptr", "p_col", "q", "a_values", "at_values", "at_row_ptr", "at_col",
        "l", "u", "d", "e")], scal.ctypes.data)
    assert rc == 0
    return out, scal


@pytest.mark.parametrize("cls,scale", [(c, s) for c in G.CLASSES for s in (2, 6)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_setup_bit_exact(cls, scale, dtype):
    p = G.generate(cls, scale, 1).astype(dtype)
    with solver.Workspace(p, Settings(), device=0) as ws:
        got, scal = scaled_of(ws, dtype)
    pf = O.symmetrize_upper(p.p_upper.astype(np.float64)).astype(dtype)
    assert np.array_equal(got["p_row_ptr"], pf.row_ptr) and np.array_equal(got["p_col"], pf.col_indices)
    ref = O.ruiz(pf, p.q, p.a, p.l, p.u, 1e-3, 10)
    for k in ("q", "a_values", "at_values", "at_row_ptr", "l", "u", "d", "e"):
        assert np.array_equal(got[k], ref[k]), k
    assert np.array_equal(got["at_col"], ref["at_col"])
    assert np.array_equal(got["p_values"], ref["p_values"])
    assert scal[0] == ref["c"] and scal[2] == ref["passes_used"] and scal[3] == ref["deviation"]


def test_setup_identity_scaling_and_paper_transpose():
    A = paper_matrix()
    P = CsrMatrix.from_dense(np.eye(5))
    from paper_1912_04263_b200.problem import QpProblem
    p = QpProblem(P, np.zeros(5), A, -np.ones(4), np.ones(4))
    with solver.Workspace(p, Settings(scaling_enabled=False), device=0) as ws:
        got, scal = scaled_of(ws, np.float64)
    assert list(got["at_row_ptr"]) == [0, 2, 4, 6, 6, 8]
    assert list(got["at_col"]) == [0, 3, 1, 2, 1, 3, 0, 2]
    assert list(got["at_values"]) == [1, 7, 5, 2, 1, 1, 4, 1]
    assert scal[0] == 1.0 and np.all(got["d"] == 1)


def op_spmv(m: CsrMatrix, x):
    lib = solver.load_library()
    pre = "f64" if m.values.dtype == np.float64 else "f32"
    fn = getattr(lib, f"qpcg_{pre}_op_spmv")
    fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
    y = np.zeros(m.rows, m.values.dtype)
    v = m.view()
    x = np.ascontiguousarray(x, m.values.dtype)
    assert fn(C.addressof(v), x.ctypes.data, y.ctypes.data, 0) == 0
    return y


def skewed(rng, rows, cols):
    """rows of 0..3 nnz, ~200 nnz, and a few 5000-50000-nnz rows (multi-item)."""
    lens = rng.choice([0, 1, 2, 3, 9, 33, 200], size=rows)
    lens[rng.choice(rows, 4, replace=False)] = [5000, 20000, 50000, 2049]
    lens = np.minimum(lens, cols)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    ci = np.concatenate([np.sort(rng.choice(cols, l, replace=False)) for l in lens]).astype(np.uint32)
    vals = rng.standard_normal(int(rp[-1]))
    return CsrMatrix(rows, cols, vals, rp, ci)


@pytest.mark.parametrize("seed", [0, 1])
def test_spmv_against_oracle(seed):
    rng = np.random.default_rng(seed)
    M = skewed(rng, 3000, 60000)
    x = rng.standard_normal(M.cols)
    y = op_spmv(M, x)
    yr = O.spmv(M, x)
    lens = np.diff(M.row_ptr.astype(np.int64))
    short = lens <= 8
    assert np.array_equal(y[short], yr[short])  # thread-per-row: reference order
    bound = 1e-13 * (np.abs(M.to_scipy()) @ np.abs(x)) + 1e-300
    assert np.all(np.abs(y - yr) <= bound)
    M32 = M.astype(np.float32)
    y32 = op_spmv(M32, x.astype(np.float32))
    assert np.allclose(y32, yr, rtol=0, atol=float(np.max(1e-4 * (np.abs(M.to_scipy()) @ np.abs(x)))))


def test_spmv_paper_and_empty():
    A = paper_matrix()
    assert list(op_spmv(A, np.ones(5))) == [5, 6, 3, 8]
    assert list(op_spmv(A, np.array([1.0, 0, 0, 0, 0]))) == [1, 0, 0, 7]
    E = CsrMatrix(3, 4, np.zeros(0), np.zeros(4, np.uint32), np.zeros(0, np.uint32))
    assert list(op_spmv(E, np.ones(4))) == [0, 0, 0]


@pytest.mark.parametrize("cls", ["lasso", "portfolio", "svm", "random"])
def test_operator_apply(cls):
    p = G.generate(cls, 5, 0)
    with solver.Workspace(p, Settings(), device=0) as ws:
        got, _ = scaled_of(ws, np.float64)
        x = np.random.default_rng(0).standard_normal(p.n)
        kx, dinv = np.zeros(p.n), np.zeros(p.n)
        lib = solver.load_library()
        lib.qpcg_debug_operator.argtypes = [C.c_void_p] * 4
        assert lib.qpcg_debug_operator(ws.ws, x.ctypes.data, kx.ctypes.data, dinv.ctypes.data) == 0
    n = p.n
    pf = CsrMatrix(n, n, got["p_values"], got["p_row_ptr"], got["p_col"])
    a = CsrMatrix(p.m, n, got["a_values"], p.a.row_ptr, p.a.col_indices)
    at = CsrMatrix(n, p.m, got["at_values"], got["at_row_ptr"], got["at_col"])
    kr, dm = O.kkt_apply(pf, a, at, 1e-6, 0.1, x)
    assert np.array_equal(dinv, 1.0 / dm)  # Jacobi diagonal bit-exact (linsys.hpp:142-146)
    scale = np.abs(pf.to_scipy()) @ np.abs(x) + 0.1 * (np.abs(at.to_scipy()) @ (np.abs(a.to_scipy()) @ np.abs(x))) + 1e-6 * np.abs(x)
    assert np.all(np.abs(kx - kr) <= 1e-12 * scale + 1e-300)
