"""Property tests (SURVEY.md §4 builder plan (ii)): random small QPs with
empty rows and columns, +-inf bounds, m = 0, duplicate-free ragged CSR.
For every drawn instance:
  * the device setup (symmetrize, transpose, all Ruiz passes) is bit-exact
    with the reference (oracle restatement pinned to it);
  * the graph, persistent and eager drivers are bitwise identical;
  * the status agrees with the oracle when the oracle solves or proves
    infeasibility, the solution passes the independent KKT re-check, and the
    iterates satisfy l <= z <= u (SPEC acceptance 8) up to the unscaling
    rounding.
Hypothesis runs derandomized (a fixed example set), so the suite is
deterministic like the engine."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from oracle import oracle as O
from paper_1912_04263_b200 import solver
from paper_1912_04263_b200.problem import CsrMatrix, QpProblem, Settings
from _util import kkt_ok
from test_gpu_kernels import op_spmv, scaled_of
from test_gpu_persistent import same

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01, max_admm_iter=400)


def csr_from_dense(M):
    rows, cols = M.shape
    rp, ci, v = [0], [], []
    for r in range(rows):
        nz = np.nonzero(M[r])[0]
        ci.extend(nz)
        v.extend(M[r, nz])
        rp.append(len(ci))
    return CsrMatrix(rows, cols, np.array(v, np.float64), np.array(rp, np.uint32),
                     np.array(ci, np.uint32))


@st.composite
def qps(draw):
    n = draw(st.integers(1, 24))
    m = draw(st.integers(0, 30))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    # P = L L^T with L sparse (empty rows/cols allowed) -> convex; upper triangle
    L = rng.standard_normal((n, n)) * (rng.random((n, n)) < draw(st.sampled_from([0.0, 0.1, 0.4])))
    Pf = L @ L.T
    Pf[np.abs(Pf) < 1e-12] = 0.0
    A = rng.standard_normal((m, n)) * (rng.random((m, n)) < draw(st.sampled_from([0.05, 0.3, 1.0])))
    x0 = rng.standard_normal(n)
    ax = A @ x0
    lo = ax - rng.uniform(0.1, 1.0, m)
    hi = ax + rng.uniform(0.1, 1.0, m)
    kind = rng.integers(0, 4, m)  # 0 box, 1 l=-inf, 2 u=+inf, 3 equality
    lo[kind == 1] = -np.inf
    hi[kind == 2] = np.inf
    hi[kind == 3] = lo[kind == 3]
    q = rng.standard_normal(n) * draw(st.sampled_from([0.0, 1.0]))
    return QpProblem(csr_from_dense(np.triu(Pf)), q, csr_from_dense(A), lo, hi)


PROP = settings(max_examples=60, deadline=None, derandomize=True,
                suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])


@PROP
@given(qps())
def test_random_qp_setup_bit_exact(p):
    with solver.Workspace(p, Settings(), device=0) as ws:
        got, scal = scaled_of(ws, np.float64)
    pf = O.symmetrize_upper(p.p_upper)
    ref = O.ruiz(pf, p.q, p.a, p.l, p.u, 1e-3, 10)
    for k in ("q", "a_values", "at_values", "at_row_ptr", "at_col", "l", "u", "d", "e", "p_values"):
        assert np.array_equal(got[k], ref[k], equal_nan=True), k
    assert scal[0] == ref["c"] and scal[2] == ref["passes_used"]


@PROP
@given(qps())
def test_random_qp_drivers_and_parity(p):
    g = solver.solve(p, S, device=0, mode="graph")
    e = solver.solve(p, S, device=0, mode="eager")
    same(g, e)
    same(g, solver.solve(p, S, device=0, mode="persistent"))
    o = O.oracle_solve(p, S)
    if o.status in ("solved", "primal_infeasible", "dual_infeasible"):
        assert g.status == o.status, (g.status, o.status, g.iterations, o.iterations)
    if g.status == "solved":
        assert kkt_ok(p, g, S, 1.0 + 1e-9)
        tol = 1e-9 * (1.0 + np.abs(g.z))
        assert np.all(g.z >= p.l - tol) and np.all(g.z <= p.u + tol)


@pytest.mark.parametrize("cols", [60000, 200000])
def test_compressed_spmv_with_wide_chunks(cols):
    """The 16-bit compressed columns, including chunks whose 32 entries span
    >= 65536 columns (the wide fallback), against the oracle."""
    rng = np.random.default_rng(cols)
    rows = 600
    lens = rng.choice([0, 5, 300, 2100, 9000], size=rows)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    ci = np.concatenate([np.sort(rng.choice(cols, l, replace=False)) for l in lens]).astype(np.uint32)
    M = CsrMatrix(rows, cols, rng.standard_normal(int(rp[-1])), rp, ci)
    x = rng.standard_normal(cols)
    y, yr = op_spmv(M, x), O.spmv(M, x)
    bound = 1e-13 * (np.abs(M.to_scipy()) @ np.abs(x)) + 1e-300
    assert np.all(np.abs(y - yr) <= bound)
