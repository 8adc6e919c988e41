"""SPEC.md known-answer tests and the committed golden fixtures, on the oracle."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200.problem import CsrMatrix, Settings
from _util import kat_problems, paper_matrix

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.json")))


def test_paper_matrix_kats():
    A = paper_matrix()
    t = O.transpose(A)
    # A^T as CSR equals the paper's CSC arrays
    assert list(t.row_ptr) == [0, 2, 4, 6, 6, 8]
    assert list(t.col_indices) == [0, 3, 1, 2, 1, 3, 0, 2]
    assert list(t.values) == [1, 7, 5, 2, 1, 1, 4, 1]
    assert list(O.spmv(A, np.array([1.0, 0, 0, 0, 0]))) == [1, 0, 0, 7]
    assert list(O.spmv(A, np.ones(5))) == [5, 6, 3, 8]


def test_operator_and_jacobi_kats():
    pf = CsrMatrix.from_dense(np.diag([1.0, 2.0]))
    a1 = CsrMatrix.from_dense(np.array([[1.0, 1.0]]))
    kx, _ = O.kkt_apply(pf, a1, O.transpose(a1), 0.001, 0.5, np.array([1.0, 0.0]))
    assert np.allclose(kx, [1.501, 0.5], rtol=0, atol=1e-15)
    _, dm = O.kkt_apply(pf, a1, O.transpose(a1), 1e-6, 0.1, np.array([1.0, 0.0]))
    assert np.allclose(dm, [1.100001, 2.100001], rtol=1e-15)
    assert O.adaptive_eps(1e-2, 1e-4, 0.15, 1e-7) == pytest.approx(1.5e-4, rel=1e-15)


def test_solve_kats():
    k = kat_problems()
    r = O.oracle_solve(k["n1_equality"], Settings())
    assert r.status == "solved" and abs(r.x[0] - 1.0003) < 1e-3 and abs(r.objective - 0.5003) < 1e-3
    r = O.oracle_solve(k["unconstrained"], Settings())
    assert r.status == "solved" and abs(r.x[0] + 2.0) < 1e-3 and abs(r.objective + 2.0) < 1e-3
    r = O.oracle_solve(k["two_var"], Settings())
    assert r.status == "solved" and np.allclose(r.x, 0.5001, atol=1e-3)
    r = O.oracle_solve(k["primal_infeasible"], Settings())
    assert r.status == "primal_infeasible" and r.iterations == 5
    assert np.allclose(r.certificate, [1.0, -1.0])
    r = O.oracle_solve(k["dual_infeasible"], Settings())
    assert r.status == "dual_infeasible" and r.iterations == 5
    assert np.allclose(r.certificate, [1.0])


def test_golden_fixtures_match_oracle():
    A = paper_matrix()
    t = O.transpose(A)
    g = GOLD["kat"]
    assert [int(v) for v in t.row_ptr] == g["paper_transpose"]["row_ptr"]
    assert list(t.values) == g["paper_transpose"]["values"]
    for name, p in kat_problems().items():
        r = O.oracle_solve(p, Settings())
        gg = GOLD["solves"][name]
        assert (r.status, r.iterations, r.pcg_iterations_total) == (gg["status"], gg["iterations"], gg["pcg"])
        assert list(r.x) == gg["x"]
    for cls in O.CLASSES:
        r = O.oracle_solve(O.ref_generate(cls, 2, 0), Settings(lambda_pcg=0.01))
        gg = GOLD["solves"][f"{cls}_s2"]
        assert (r.status, r.iterations, r.pcg_iterations_total, r.objective) == \
            (gg["status"], gg["iterations"], gg["pcg"], gg["objective"])
