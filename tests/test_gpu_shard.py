"""Row-sharded engine on the B200: A held as G nnz-balanced
row blocks (virtual shards on one device; the NCCL path with one rank), the
A^T partials combined per operator apply.  Same parity protocol as the
unsharded engine (tests/test_gpu_parity.py), plus the sharded-specific
invariants: identical setup (Ruiz / Jacobi are bit-exact under sharding),
identical statuses and error messages, deterministic runs."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import QpProblem, Settings, SolveDiagnostics, WarmStart
from _util import kat_problems, kkt_ok, rel
from test_gpu_parity import check_parity

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


@pytest.mark.parametrize("cls", G.CLASSES)
@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_classes_parity(cls, shards):
    for scale in (3, 6):
        p = G.generate(cls, scale, 0)
        g = solver.solve(p, S, device=0, shards=shards)
        o = O.oracle_solve(p, S)
        check_parity(p, S, g, o)
        one = solver.solve(p, S, device=0)
        assert g.status == one.status
        assert g.equil_passes == one.equil_passes  # Ruiz is bit-exact under sharding
        assert abs(g.iterations - one.iterations) <= 50


def test_sharded_first_pcg_call_matches_unsharded():
    """Ruiz, the Jacobi diagonal (diag(A^T A) chain) and the initial residuals
    are bit-exact under sharding, so the first adaptive tolerance is too."""
    p = G.generate("lasso", 5, 1)
    d1, d4 = SolveDiagnostics(), SolveDiagnostics()
    a = solver.solve(p, S, diag=d1, device=0)
    b = solver.solve(p, S, diag=d4, device=0, shards=4)
    assert d1.pcg_calls[0]["eps"] == d4.pcg_calls[0]["eps"]
    assert d1.pcg_calls[0]["r_prim_scaled_inf"] == d4.pcg_calls[0]["r_prim_scaled_inf"]
    assert a.status == b.status == "solved"
    k = min(10, len(d1.pcg_calls), len(d4.pcg_calls))
    assert [c["iterations"] for c in d1.pcg_calls[:k]] == [c["iterations"] for c in d4.pcg_calls[:k]]


def test_sharded_deterministic_and_more_shards_than_rows():
    p = G.generate("portfolio", 5, 0)
    a = solver.solve(p, S, device=0, shards=4)
    b = solver.solve(p, S, device=0, shards=4)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.z, b.z) and a.iterations == b.iterations
    k = kat_problems()["two_var"]  # m = 1 < 3 blocks: two blocks are empty
    g = solver.solve(k, Settings(), device=0, shards=3)
    one = solver.solve(k, Settings(), device=0)
    assert g.status == one.status == "solved" and np.allclose(g.x, one.x, rtol=1e-9)


@pytest.mark.parametrize("name", list(kat_problems()))
def test_sharded_kats(name):
    p = kat_problems()[name]
    g = solver.solve(p, Settings(), device=0, shards=2)
    one = solver.solve(p, Settings(), device=0)
    assert g.status == one.status and g.iterations == one.iterations
    assert np.allclose(g.x, one.x, rtol=1e-9, atol=1e-12)
    if one.certificate is not None and len(one.certificate):
        assert np.allclose(g.certificate, one.certificate, atol=1e-12)
        assert g.objective == one.objective


def test_sharded_errors_match_unsharded():
    from paper_1912_04263_b200.problem import CsrMatrix
    base = G.generate("lasso", 3, 0)
    cases = []
    p = G.generate("lasso", 3, 0); p.l = p.l.copy(); p.u = p.u.copy()
    p.l[-1], p.u[-1] = 5.0, 1.0; cases.append(p)                      # l > u in the last block
    p = G.generate("lasso", 3, 0); p.a.values = p.a.values.copy()
    p.a.values[-3] = np.nan; cases.append(p)                            # NaN in the last block
    p = G.generate("lasso", 3, 0); ci = p.a.col_indices.copy()
    e = int(p.a.row_ptr[-2]); ci[e], ci[e + 1] = ci[e + 1], ci[e]
    p.a.col_indices = ci; cases.append(p)                               # unsorted row, last block
    p = G.generate("lasso", 3, 0); rp = p.a.row_ptr.copy().astype(np.int64)
    rp[5] = rp[7]; p.a.row_ptr = rp.astype(np.uint32); cases.append(p)  # decreasing row_ptr
    for p in cases:
        with pytest.raises(ValueError) as e1:
            solver.solve(p, S, device=0)
        with pytest.raises(ValueError) as e3:
            solver.solve(p, S, device=0, shards=3)
        assert str(e3.value) == str(e1.value)
    assert base is not None


def test_sharded_workspace_updates():
    p = G.generate("control", 4, 0)
    with solver.Workspace(p, S, device=0, shards=2) as ws, solver.Workspace(p, S, device=0) as w1:
        a, a1 = ws.solve(), w1.solve()
        assert a.status == a1.status == "solved"
        ws.warm_start(a.x, a.z, a.y)
        b = ws.solve()
        assert b.status == "solved" and b.iterations <= a.iterations
        ws.update_rho(1.0)
        l2, u2 = p.l * 0.9, p.u * 0.9
        ws.update_vectors(l=l2, u=u2)
        c = ws.solve()
        p2 = QpProblem(p.p_upper, p.q, p.a, l2, u2)
        assert c.status == "solved" and kkt_ok(p2, c, S)
        bad = l2.copy(); bad[-1] = np.inf
        with pytest.raises(ValueError, match="l must be < \\+inf"):
            ws.update_vectors(l=bad)
        with pytest.raises(ValueError, match="warm start must be finite"):
            z = a.z.copy(); z[-1] = np.nan
            ws.warm_start(a.x, z, a.y)


def test_sharded_nccl_single_rank():
    """The NCCL code path (dlopen'd libnccl, ncclCommInitRank, allreduce,
    chain, block gather) with one rank holding two virtual blocks."""
    uid = solver.nccl_unique_id()
    assert len(uid) == 128
    p = G.generate("huber", 5, 0)
    g = solver.solve(p, S, device=0, shards=2, nccl=(0, 1, uid))
    v = solver.solve(p, S, device=0, shards=2)
    o = O.oracle_solve(p, S)
    check_parity(p, S, g, o)
    assert g.status == v.status and abs(g.iterations - v.iterations) <= 10


@pytest.mark.parametrize("cls", ["svm", "lasso", "huber"])
def test_sharded_f32(cls):
    """fp32 row-sharded engine against the fp32 oracle under the §8(c)
    protocol (1e-3 objective and x, or 2x the oracle's reorder noise)."""
    p = G.generate(cls, 5, 0).astype(np.float32)
    g = solver.solve(p, S, device=0, shards=2)
    o = O.oracle_solve(p, S)
    check_parity(p, S, g, o)


def test_sharded_warm_start_matches_oracle():
    p = G.generate("huber", 4, 2)
    o = O.oracle_solve(p, S)
    w = WarmStart(o.x * 0.95, o.z, o.y * 1.05)
    g = solver.solve(p, S, initial=w, device=0, shards=3)
    ow = O.oracle_solve(p, S, warm=w)
    assert g.status == ow.status == "solved"
    assert rel(g.objective, ow.objective) < 1e-3


@pytest.mark.parametrize("cls", ["lasso", "huber", "portfolio"])
def test_sharded_graph_equals_host_loop(cls):
    """The device-driven sharded loop (one CUDA graph, conditional nodes) is
    bitwise identical to the host-driven one."""
    p = G.generate(cls, 5, 0)
    a = solver.solve(p, S, device=0, shards=3, mode="graph")
    b = solver.solve(p, S, device=0, shards=3, mode="eager")
    assert a.status == b.status and a.iterations == b.iterations
    assert a.pcg_iterations_total == b.pcg_iterations_total
    assert np.array_equal(a.x, b.x) and np.array_equal(a.z, b.z) and np.array_equal(a.y, b.y)


def test_peer_transport_nccl_bootstrap_single_rank():
    """The peer transport bootstrapped over NCCL (ncclAllGather of the IPC
    handles), one rank x 2 blocks: bitwise equal to the 2 virtual blocks."""
    uid = solver.nccl_unique_id()
    p = G.generate("control", 5, 0)
    g = solver.solve(p, S, device=0, shards=2, nccl=(0, 1, uid), peer=(0, 1, None))
    v = solver.solve(p, S, device=0, shards=2)
    assert g.status == v.status and g.iterations == v.iterations
    assert np.array_equal(g.x, v.x) and np.array_equal(g.z, v.z)
