"""The small-problem path: the whole ADMM/PCG loop in one cooperative kernel
(csrc/persist.cuh).  Its reductions emulate the
stand-alone kernels' launch geometry, so it must be BITWISE identical to the
graph and eager drivers; on top of that the usual oracle parity."""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import NotPositiveDefiniteError, Settings, SolveDiagnostics
from _util import dense_qp, kat_problems
from test_gpu_parity import check_parity

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


def graph_only(p, s, **kw):
    old = os.environ.get("QPCG_PERSIST_MAX_NNZ")
    os.environ["QPCG_PERSIST_MAX_NNZ"] = "0"
    try:
        return solver.solve(p, s, device=0, mode="graph", **kw)
    finally:
        if old is None:
            del os.environ["QPCG_PERSIST_MAX_NNZ"]
        else:
            os.environ["QPCG_PERSIST_MAX_NNZ"] = old


def same(a, b):
    assert a.status == b.status
    assert a.iterations == b.iterations and a.pcg_iterations_total == b.pcg_iterations_total
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and np.array_equal(a.z, b.z)
    assert a.objective == b.objective or (np.isnan(a.objective) and np.isnan(b.objective))
    assert a.rho_final == b.rho_final
    assert np.array_equal(a.certificate, b.certificate)


@pytest.mark.parametrize("cls", G.CLASSES)
def test_persistent_bitwise_equals_graph_and_eager(cls):
    p = G.generate(cls, 5, 1)
    a = solver.solve(p, S, device=0, mode="persistent")
    b = graph_only(p, S)
    c = solver.solve(p, S, device=0, mode="eager")
    same(a, b)
    same(a, c)
    check_parity(p, S, a, O.oracle_solve(p, S))


@pytest.mark.parametrize("name", list(kat_problems()))
def test_persistent_kats_and_certificates(name):
    p = kat_problems()[name]
    a = solver.solve(p, Settings(), device=0, mode="persistent")
    b = solver.solve(p, Settings(), device=0, mode="eager")
    same(a, b)


def test_persistent_diagnostics_match_eager():
    p = G.generate("lasso", 4, 0)
    d1, d2 = SolveDiagnostics(), SolveDiagnostics()
    solver.solve(p, S, diag=d1, device=0, mode="persistent")
    solver.solve(p, S, diag=d2, device=0, mode="eager")
    assert d1.pcg_calls == d2.pcg_calls
    assert d1.rho_updates == d2.rho_updates
    assert d1.check_iterations == d2.check_iterations


def test_persistent_errors_and_limits():
    p = dense_qp([[-5.0, 0.0], [0.0, -5.0]], [1.0, 1.0], [[1.0, 0.0]], [-1.0], [1.0])
    with pytest.raises(NotPositiveDefiniteError):
        solver.solve(p, Settings(), device=0, mode="persistent")
    p = G.generate("portfolio", 4, 0)
    s = Settings(lambda_pcg=0.01, max_admm_iter=7)
    a = solver.solve(p, s, device=0, mode="persistent")
    assert a.status == "max_iter_reached" and a.iterations == 7
    same(a, solver.solve(p, s, device=0, mode="eager"))


def test_persistent_workspace_reuse_and_f32():
    p = G.generate("control", 4, 0)
    with solver.Workspace(p, S, device=0, mode="persistent") as ws, \
            solver.Workspace(p, S, device=0, mode="eager") as we:
        for w in (ws, we):
            w.solve()
            w.update_rho(1.0)
            w.update_vectors(l=p.l * 0.9, u=p.u * 0.9)
        same(ws.solve(), we.solve())
    p32 = G.generate("svm", 5, 0).astype(np.float32)
    s32 = Settings(lambda_pcg=0.01, eps_abs=3e-3, eps_rel=3e-3)
    same(solver.solve(p32, s32, device=0, mode="persistent"),
         solver.solve(p32, s32, device=0, mode="eager"))


@pytest.mark.parametrize("cfg", ["1", "1p"])
def test_persistent_config1(cfg):
    p = G.config(cfg)
    a = solver.solve(p, S, device=0, mode="persistent")
    same(a, graph_only(p, S))
