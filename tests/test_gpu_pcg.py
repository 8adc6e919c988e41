"""Operator-level pcg_solve (linsys.hpp:190-276) through the ops C-ABI, run by
the engine's own PCG kernels: SPEC acceptance 2 (200 random SPD systems,
eps = 1e-10, solution within 1e-6 of a dense solve), the reference's edge
behaviour (zero rhs, iteration cap returning the best iterate, nonpositive
curvature, argument errors) and agreement with the oracle's PCG."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import solver
from paper_1912_04263_b200.problem import CsrMatrix, NotPositiveDefiniteError

pytestmark = pytest.mark.gpu


def csr(M):
    rows, cols = M.shape
    rp, ci, v = [0], [], []
    for r in range(rows):
        nz = np.nonzero(M[r])[0]
        ci.extend(nz)
        v.extend(M[r, nz])
        rp.append(len(ci))
    return CsrMatrix(rows, cols, np.array(v, np.float64), np.array(rp, np.uint32),
                     np.array(ci, np.uint32))


def op_pcg(pf, a, at, sigma, rho, b, warm, eps, max_iter, dtype=np.float64):
    lib = solver.load_library()
    pre = "f64" if dtype == np.float64 else "f32"
    fn = getattr(lib, f"qpcg_{pre}_op_pcg")
    fn.argtypes = [C.c_void_p] * 3 + [C.c_double, C.c_double, C.c_void_p, C.c_void_p, C.c_double,
                                      C.c_uint32, C.c_void_p, C.c_void_p, C.c_int]
    views = [m.astype(dtype).view() for m in (pf, a, at)]
    b = np.ascontiguousarray(b, dtype)
    warm = np.ascontiguousarray(warm, dtype)
    x = np.zeros(pf.rows, dtype)
    res = np.zeros(3)
    rc = fn(*[C.addressof(v) for v in views], sigma, rho, b.ctypes.data, warm.ctypes.data, eps,
            max_iter, x.ctypes.data, res.ctypes.data, 0)
    if rc != 0:
        msg = lib.qpcg_last_error(None).decode()
        if rc == 2:
            raise NotPositiveDefiniteError(msg)
        raise ValueError(msg)
    return x, int(res[0]), res[1], bool(res[2])


def system(rng, n, m, dens=0.3):
    L = rng.standard_normal((n, n)) * (rng.random((n, n)) < dens)
    Pf = L @ L.T
    Pf[np.abs(Pf) < 1e-13] = 0
    A = rng.standard_normal((m, n)) * (rng.random((m, n)) < dens)
    return csr(Pf), csr(A), O.transpose(csr(A)), Pf, A


def test_spec_acceptance_200_random_spd():
    rng = np.random.default_rng(2024)
    worst = 0.0
    for i in range(200):
        n, m = int(rng.integers(2, 40)), int(rng.integers(0, 40))
        pf, a, at, Pf, A = system(rng, n, m)
        sigma, rho = 10.0 ** rng.uniform(-6, -2), 10.0 ** rng.uniform(-2, 1)
        K = Pf + sigma * np.eye(n) + rho * A.T @ A
        b = rng.standard_normal(n)
        x, k, rn, conv = op_pcg(pf, a, at, sigma, rho, b, np.zeros(n), 1e-10, 10 * n + 20)
        xd = np.linalg.solve(K, b)
        err = np.max(np.abs(x - xd)) / max(1.0, np.max(np.abs(xd)))
        worst = max(worst, err)
        assert conv and err <= 1e-6, (i, n, m, err, k)
        xo, ko, rno, convo = O.pcg(pf, a, at, sigma, rho, b, np.zeros(n), 1e-10, 10 * n + 20)
        assert convo and abs(k - ko) <= 2, (k, ko)
    print("worst relative error vs dense:", worst)


def test_warm_start_cap_and_best_iterate_match_oracle():
    rng = np.random.default_rng(7)
    pf, a, at, _, _ = system(rng, 60, 80, 0.2)
    b, warm = rng.standard_normal(60), rng.standard_normal(60)
    for cap in (0, 1, 3, 7):
        x, k, rn, conv = op_pcg(pf, a, at, 1e-6, 0.1, b, warm, 1e-12, cap)
        xo, ko, rno, convo = O.pcg(pf, a, at, 1e-6, 0.1, b, warm, 1e-12, cap)
        assert (k, conv) == (ko, convo) == (cap, False)
        assert rn == pytest.approx(rno, rel=1e-9)
        assert np.allclose(x, xo, rtol=1e-9, atol=1e-12)


def test_zero_rhs_and_errors():
    rng = np.random.default_rng(3)
    pf, a, at, _, _ = system(rng, 10, 12)
    x, k, rn, conv = op_pcg(pf, a, at, 1e-6, 0.1, np.zeros(10), rng.standard_normal(10), 1e-8, 50)
    assert conv and k == 0 and rn == 0.0 and np.all(x == 0)  # linsys.hpp:208-213
    with pytest.raises(ValueError, match="eps must be positive"):
        op_pcg(pf, a, at, 1e-6, 0.1, np.ones(10), np.zeros(10), 0.0, 50)
    with pytest.raises(ValueError, match="warm start must be finite"):
        op_pcg(pf, a, at, 1e-6, 0.1, np.ones(10), np.full(10, np.nan), 1e-8, 50)
    with pytest.raises(ValueError, match="sigma and rho must be positive"):
        op_pcg(pf, a, at, 0.0, 0.1, np.ones(10), np.zeros(10), 1e-8, 50)
    bad = CsrMatrix(at.rows, at.cols, at.values * 2.0, at.row_ptr, at.col_indices)
    with pytest.raises(ValueError, match="a_t is not the transpose of a"):
        op_pcg(pf, a, bad, 1e-6, 0.1, np.ones(10), np.zeros(10), 1e-8, 50)
    neg = csr(-np.eye(10) * 5.0)
    with pytest.raises(NotPositiveDefiniteError):
        op_pcg(neg, csr(np.zeros((1, 10))), O.transpose(csr(np.zeros((1, 10)))), 1e-6, 0.1,
               np.ones(10), np.zeros(10), 1e-8, 50)


def test_f32_pcg():
    rng = np.random.default_rng(11)
    pf, a, at, Pf, A = system(rng, 30, 40)
    K = Pf + 1e-3 * np.eye(30) + 0.5 * A.T @ A
    b = rng.standard_normal(30)
    x, k, rn, conv = op_pcg(pf, a, at, 1e-3, 0.5, b, np.zeros(30), 1e-5, 500, np.float32)
    xd = np.linalg.solve(K, b)
    assert np.max(np.abs(x - xd)) <= 1e-3 * max(1.0, np.max(np.abs(xd)))
