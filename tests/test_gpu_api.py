"""The OSQP-style workspace API and error behaviour through the C-ABI."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import NotPositiveDefiniteError, Settings, WarmStart
from _util import dense_qp, kat_problems, kkt_ok, rel

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


def test_warm_start_matches_oracle():
    p = G.generate("huber", 4, 2)
    o = O.oracle_solve(p, S)
    w = WarmStart(o.x * 0.95, o.z, o.y * 1.05)
    g = solver.solve(p, S, initial=w, device=0)
    ow = O.oracle_solve(p, S, warm=w)
    assert g.status == ow.status == "solved"
    assert rel(g.objective, ow.objective) < 1e-3


def test_warm_start_from_solution_converges_fast():
    p = G.generate("lasso", 5, 0)
    with solver.Workspace(p, S, device=0) as ws:
        a = ws.solve()
        ws.warm_start(a.x, a.z, a.y)
        b = ws.solve()
    assert b.status == "solved" and b.iterations <= a.iterations


def test_repeated_solve_continues_from_state():
    p = G.generate("svm", 4, 0)
    with solver.Workspace(p, S, device=0) as ws:
        a = ws.solve()
        b = ws.solve()  # OSQP semantics: iterates and rho persist
    assert b.status == "solved" and b.iterations <= a.iterations


def test_update_rho_and_vectors():
    p = G.generate("control", 4, 0)
    # eps = 1e-5 so that "equals a fresh solve within KKT tolerance" (SURVEY
    # §8(f) rank 1: the update is not bit-equal to a fresh solve, Ruiz's gamma
    # depends on q) is held to the north star's 1e-3
    S5 = Settings(lambda_pcg=0.01, eps_abs=1e-5, eps_rel=1e-5)
    with solver.Workspace(p, S5, device=0) as ws:
        a = ws.solve()
        ws.update_rho(1.0)
        b = ws.solve()
        assert b.status == "solved" and kkt_ok(p, b, S5)
        # receding-horizon style update of the bounds
        l2, u2 = p.l * 0.9, p.u * 0.9
        ws.update_vectors(l=l2, u=u2)
        c = ws.solve()
    from paper_1912_04263_b200.problem import QpProblem
    p2 = QpProblem(p.p_upper, p.q, p.a, l2, u2)
    assert c.status == "solved" and kkt_ok(p2, c, S5)
    fresh = O.oracle_solve(p2, S5)
    assert rel(c.objective, fresh.objective) < 1e-3
    scale = max(1.0, float(np.max(np.abs(fresh.x))))
    assert float(np.max(np.abs(c.x - fresh.x))) / scale < 1e-3
    with pytest.raises(ValueError, match="rho must be positive"):
        with solver.Workspace(p, S, device=0) as ws:
            ws.update_rho(-1.0)


def test_invalid_problems_raise_reference_messages():
    k = kat_problems()
    cases = []
    p = k["two_var"]; p.l = np.array([5.0]); p.u = np.array([1.0]); cases.append(p)
    p = kat_problems()["two_var"]; p.q = np.array([0.0, np.inf]); cases.append(p)
    p = kat_problems()["two_var"]; p.a.col_indices = p.a.col_indices[::-1].copy(); cases.append(p)
    from paper_1912_04263_b200.problem import CsrMatrix, QpProblem
    below = CsrMatrix(2, 2, np.array([1.0, 1.0, 1.0]), np.array([0, 1, 3], np.uint32),
                      np.array([0, 0, 1], np.uint32))  # (1,0) is below the diagonal
    cases.append(QpProblem(below, np.zeros(2), CsrMatrix.from_dense([[1.0, 1.0]]), np.zeros(1), np.ones(1)))
    for p in cases:
        with pytest.raises(ValueError) as eo:
            O.oracle_solve(p, Settings())
        with pytest.raises(ValueError) as eg:
            solver.solve(p, Settings(), device=0)
        assert str(eg.value) == str(eo.value)
    with pytest.raises(ValueError, match="alpha"):
        solver.solve(k["two_var"], Settings(alpha=2.5), device=0)


def test_not_positive_definite():
    p = dense_qp([[-5.0, 0.0], [0.0, -5.0]], [1.0, 1.0], [[1.0, 0.0]], [-1.0], [1.0])
    with pytest.raises(NotPositiveDefiniteError):
        O.oracle_solve(p, Settings())
    with pytest.raises(NotPositiveDefiniteError):
        solver.solve(p, Settings(), device=0)


def test_max_iter_status():
    p = G.generate("portfolio", 4, 0)
    s = Settings(lambda_pcg=0.01, max_admm_iter=7)
    g = solver.solve(p, s, device=0)
    o = O.oracle_solve(p, s)
    assert g.status == o.status == "max_iter_reached" and g.iterations == o.iterations == 7


def test_reentrant_workspaces():
    p1, p2 = G.generate("lasso", 4, 0), G.generate("svm", 4, 1)
    w1, w2 = solver.Workspace(p1, S, device=0), solver.Workspace(p2, S, device=0)
    a, b = w1.solve(), w2.solve()
    a2 = solver.solve(p1, S, device=0)
    assert np.array_equal(a.x, a2.x) and b.status == "solved"
    w1.close(); w2.close()


def test_rejected_update_vectors_leaves_the_workspace_unchanged():
    """A rejected update (l > u) must not leak into the original-data
    buffers: the next solve equals one on the untouched workspace bit for bit,
    and a later valid q-only update is accepted."""
    p = G.generate("control", 4, 0)
    with solver.Workspace(p, S, device=0) as ws:
        ws.solve()
        bad_l = p.u + 1.0
        with pytest.raises(ValueError, match="l must not exceed u"):
            ws.update_vectors(l=bad_l)
        b1 = ws.solve()
        ws.update_vectors(q=p.q * 1.0)
        c1 = ws.solve()
    with solver.Workspace(p, S, device=0) as ws:
        ws.solve()
        b2 = ws.solve()
        ws.update_vectors(q=p.q * 1.0)
        c2 = ws.solve()
    assert np.array_equal(b1.x, b2.x) and b1.objective == b2.objective
    assert np.array_equal(c1.x, c2.x) and c1.status == c2.status


def test_update_vectors_length_checked():
    p = G.generate("lasso", 3, 0)
    with solver.Workspace(p, S, device=0) as ws:
        with pytest.raises(ValueError, match="q length must equal n"):
            ws.update_vectors(q=np.zeros(p.n + 1))
        with pytest.raises(ValueError, match="bound lengths must equal m"):
            ws.update_vectors(u=np.zeros(p.m - 1))
        with pytest.raises(ValueError, match="warm start dimension mismatch"):
            ws.warm_start(np.zeros(p.n), np.zeros(p.m), np.zeros(p.m + 2))
        assert ws.solve().status == "solved"


def test_release_cached_memory_returns_device_memory():
    import torch
    p = G.config("1")
    solver.solve(p, S, device=0)
    solver.release_cached_memory()
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info(0)
    for _ in range(2):
        solver.solve(p, S, device=0)
    free1, _ = torch.cuda.mem_get_info(0)
    solver.release_cached_memory()
    free2, _ = torch.cuda.mem_get_info(0)
    print(f"free: after a release {free0 >> 20} MiB, after two solves {free1 >> 20} MiB, "
          f"after a release {free2 >> 20} MiB")
    assert free2 >= free1
    assert free2 >= free0 - (64 << 20)  # nothing of the finished solves is kept


def test_on_iteration_observer():
    """SolveDiagnostics.on_iteration (solver.hpp:166, :451-454): one call per
    ADMM iteration with the scaled iterates; the instrumented (host-driven)
    loop gives bitwise the same solve as the graph driver."""
    from paper_1912_04263_b200.problem import SolveDiagnostics
    p = G.generate("huber", 4, 1)
    views, seen = [], []
    d = SolveDiagnostics()
    d.on_iteration = lambda v: (views.append(v), seen.append(
        bool(d.pcg_calls) and d.pcg_calls[-1]["admm_iter"] == v.iter))
    g = solver.solve(p, S, diag=d, device=0)
    ref = solver.solve(p, S, device=0)
    assert [v.iter for v in views] == list(range(1, g.iterations + 1))
    assert np.array_equal(g.x, ref.x) and g.iterations == ref.iterations
    last = views[-1]
    assert last.x.shape == (p.n,) and last.z.shape == (p.m,) and last.l.shape == (p.m,)
    assert np.all(last.l <= last.z) and np.all(last.z <= last.u)  # z = proj_[l,u](w), scaled
    assert len(d.pcg_calls) == g.iterations
    assert all(seen)  # each iteration's PcgCall is recorded before the callback


def test_nccl_before_torch_import():
    """The engine loads NCCL lazily; when that happens before `import torch` it
    must map the same NCCL torch will (the pip copy, QPCG_NCCL_LIB), or the
    later import clashes with an older system libnccl.so.2."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1912_04263_b200 import solver\n"
            "solver.nccl_unique_id()\n"
            "import torch\n"
            "print('ok', torch.cuda.mem_get_info(0)[0] > 0)\n") % (
        __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok True" in r.stdout, r.stderr[-2000:]


def test_bench_kernels_output_sizes():
    """qpcg_bench_kernels writes exactly its documented 9 doubles (callers size
    their buffers for it); qpcg_bench_kernels_n writes at most `cap`."""
    import ctypes as C
    lib = solver.load_library()
    lib.qpcg_bench_kernels.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
    lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
    p = G.generate("lasso", 4, 0)
    with solver.Workspace(p, S, device=0) as ws:
        out = np.full(16, -7.0)
        assert lib.qpcg_bench_kernels(ws.ws, 2, out.ctypes.data) == 0
        assert np.all(out[9:] == -7.0) and np.all(out[:3] > 0)
        out = np.full(16, -7.0)
        assert lib.qpcg_bench_kernels_n(ws.ws, 2, out.ctypes.data, 5) == 0
        assert np.all(out[5:] == -7.0)
        out = np.full(16, -7.0)
        assert lib.qpcg_bench_kernels_n(ws.ws, 2, out.ctypes.data, 16) == 0
        assert np.all(out[12:] == -7.0)
