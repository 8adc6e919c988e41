"""Pins the plain-C oracle (oracle/liboracle.so) bit-for-bit to the reference
itself (oracle/_ref, the unmodified headers) — CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200.problem import CsrMatrix, NotPositiveDefiniteError, Settings, WarmStart, SolveDiagnostics
from _util import kat_problems

S = Settings(lambda_pcg=0.01)


def same_outcome(a, b):
    assert a.status == b.status
    assert a.iterations == b.iterations
    assert a.pcg_iterations_total == b.pcg_iterations_total
    assert a.rho_update_count == b.rho_update_count and a.rho_final == b.rho_final
    assert a.equil_passes == b.equil_passes and a.equil_residual == b.equil_residual
    for k in ("x", "z", "y", "certificate"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.objective == b.objective or (np.isinf(a.objective) and a.objective == b.objective)
    assert a.r_prim_inf == b.r_prim_inf and a.r_dual_inf == b.r_dual_inf


@pytest.mark.parametrize("cls", O.CLASSES)
@pytest.mark.parametrize("scale", [0, 2, 4])
@pytest.mark.parametrize("seed", [0, 1])
def test_solve_bit_exact_f64(cls, scale, seed):
    p = O.ref_generate(cls, scale, seed)
    da, db = SolveDiagnostics(), SolveDiagnostics()
    same_outcome(O.oracle_solve(p, S, diag=da), O.ref_solve(p, S, diag=db))
    assert da.pcg_calls == db.pcg_calls
    assert da.check_iterations == db.check_iterations
    assert da.rho_updates == db.rho_updates


@pytest.mark.parametrize("cls", O.CLASSES)
def test_solve_bit_exact_defaults_and_f32(cls):
    p = O.ref_generate(cls, 3, 0)
    same_outcome(O.oracle_solve(p, Settings(max_admm_iter=400)),
                 O.ref_solve(p, Settings(max_admm_iter=400)))
    p32 = p.astype(np.float32)
    same_outcome(O.oracle_solve(p32, S), O.ref_solve(p32, S))


@pytest.mark.parametrize("name", list(kat_problems()))
def test_kat_problems_bit_exact(name):
    p = kat_problems()[name]
    same_outcome(O.oracle_solve(p, Settings()), O.ref_solve(p, Settings()))


def test_settings_variants_and_warm_start():
    p = O.ref_generate("huber", 2, 3)
    for s in (Settings(lambda_pcg=0.01, scaling_enabled=False),
              Settings(lambda_pcg=0.05, check_interval=3, rho_update_interval=7, alpha=1.2),
              Settings(lambda_pcg=0.01, equil_max_passes=2, max_admm_iter=37)):
        same_outcome(O.oracle_solve(p, s), O.ref_solve(p, s))
    r = O.ref_solve(p, S)
    w = WarmStart(r.x * 0.9, r.z, r.y)
    same_outcome(O.oracle_solve(p, S, warm=w), O.ref_solve(p, S, warm=w))


def _rand_csr(rng, rows, cols, density, square_upper=False):
    d = (rng.random((rows, cols)) < density) * rng.standard_normal((rows, cols))
    if square_upper:
        d = np.triu(d)
    return CsrMatrix.from_dense(d)


@pytest.mark.parametrize("seed", range(6))
def test_building_blocks_bit_exact(seed):
    rng = np.random.default_rng(seed)
    A = _rand_csr(rng, 13, 9, 0.3)
    x = rng.standard_normal(9)
    assert np.array_equal(O.spmv(A, x), O.spmv(A, x, kind="ref"))
    for kind in ("oracle", "ref"):
        t = O.transpose(A, kind=kind)
        tt = O.transpose(t, kind=kind)
        assert np.array_equal(tt.values, A.values) and np.array_equal(tt.col_indices, A.col_indices)
    t1, t2 = O.transpose(A), O.transpose(A, kind="ref")
    assert all(np.array_equal(getattr(t1, k), getattr(t2, k)) for k in ("values", "row_ptr", "col_indices"))
    U = _rand_csr(rng, 9, 9, 0.4, square_upper=True)
    s1, s2 = O.symmetrize_upper(U), O.symmetrize_upper(U, kind="ref")
    assert all(np.array_equal(getattr(s1, k), getattr(s2, k)) for k in ("values", "row_ptr", "col_indices"))
    dense = s1.to_scipy().toarray()
    assert np.array_equal(dense, dense.T)
    q, l = rng.standard_normal(9), -rng.random(13)
    u = rng.random(13)
    r1, r2 = O.ruiz(s1, q, A, l, u), O.ruiz(s1, q, A, l, u, kind="ref")
    for k in r1:
        assert np.array_equal(np.asarray(r1[k]), np.asarray(r2[k])), k
    at = O.transpose(A)
    k1, d1 = O.kkt_apply(s1, A, at, 1e-6, 0.3, x)
    k2, d2 = O.kkt_apply(s1, A, at, 1e-6, 0.3, x, kind="ref")
    assert np.array_equal(k1, k2) and np.array_equal(d1, d2)
    b = rng.standard_normal(9)
    # P + sigma I + rho A'A may be indefinite for a random P: both must agree on that too
    res = []
    for kind in ("oracle", "ref"):
        try:
            res.append(O.pcg(s1, A, at, 1e-6, 0.3, b, np.zeros(9), 1e-10, 50, kind=kind))
        except NotPositiveDefiniteError:
            res.append("notpd")
    if res[0] == "notpd":
        assert res[1] == "notpd"
    else:
        assert np.array_equal(res[0][0], res[1][0]) and res[0][1:] == res[1][1:]


def test_pcg_cap_and_adaptive_eps():
    for n in (1, 5, 19, 20, 400, 401, 1000, 120000, 1001000):
        for dt in (np.float64, np.float32):
            assert O.pcg_cap(n, dt) == O.pcg_cap(n, dt, kind="ref")
    for rp, rd in ((1e-2, 1e-4), (0.0, 0.0), (1.0, 1.0), (3.7, 1e-9)):
        assert O.adaptive_eps(rp, rd, 0.15, 1e-7) == O.adaptive_eps(rp, rd, 0.15, 1e-7, kind="ref")


def test_validation_messages_match():
    base = kat_problems()["two_var"]
    bad = []
    p = kat_problems()["two_var"]
    p.l = p.l.copy(); p.l[0] = 5.0; p.u = p.u.copy(); p.u[0] = 1.0
    bad.append(p)
    p = kat_problems()["two_var"]
    p.q = p.q.copy(); p.q[1] = np.nan
    bad.append(p)
    p = kat_problems()["two_var"]
    p.a.col_indices = p.a.col_indices[::-1].copy()
    bad.append(p)
    for p in bad:
        msgs = []
        for fn in (O.oracle_solve, O.ref_solve):
            with pytest.raises(ValueError) as e:
                fn(p, Settings())
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1]
    for s in (Settings(alpha=2.0), Settings(lambda_pcg=1.0), Settings(check_interval=0)):
        msgs = []
        for fn in (O.oracle_solve, O.ref_solve):
            with pytest.raises(ValueError) as e:
                fn(base, s)
            msgs.append(str(e.value))
        assert msgs[0] == msgs[1]
