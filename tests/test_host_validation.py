"""Host-side argument checks of the Python mirror (no GPU needed: every case
raises before a pointer crosses the C-ABI).  Messages are the reference's:
problem.hpp:47-70, sparse.hpp:100-106, solver.hpp:414-417, io.hpp:175-205 and
settings.hpp:44-75."""
import numpy as np
import pytest

from paper_1912_04263_b200 import solver
from paper_1912_04263_b200.problem import CsrMatrix, QpProblem, Settings, WarmStart


def two_var():
    P = CsrMatrix(2, 2, np.array([4.0, 1.0, 2.0]), np.array([0, 2, 3], np.uint32),
                  np.array([0, 1, 1], np.uint32))
    A = CsrMatrix.from_dense([[1.0, 1.0], [1.0, 0.0], [0.0, 1.0]])
    return QpProblem(P, np.array([1.0, 1.0]), A, np.array([1.0, 0.0, 0.0]),
                     np.array([1.0, 0.7, 0.7]))


@pytest.mark.parametrize("mutate,msg", [
    (lambda p: setattr(p, "q", np.zeros(3)), "problem: q length must equal n"),
    (lambda p: setattr(p, "q", np.zeros(1)), "problem: q length must equal n"),
    (lambda p: setattr(p, "l", np.zeros(2)), "problem: bound lengths must equal m"),
    (lambda p: setattr(p, "u", np.ones(5)), "problem: bound lengths must equal m"),
    (lambda p: setattr(p.a, "row_ptr", np.array([0, 2, 3], np.uint32)),
     "csr: row_ptr must have rows + 1 entries"),
    (lambda p: setattr(p.a, "values", p.a.values[:-1]), "csr: col_indices/value length mismatch"),
    (lambda p: setattr(p.p_upper, "col_indices", np.array([0, 1], np.uint32)),
     "csr: col_indices/value length mismatch"),
])
def test_lengths_rejected_before_the_abi(mutate, msg):
    p = two_var()
    mutate(p)
    import re
    with pytest.raises(ValueError, match=re.escape(msg)):
        solver.solve(p, Settings())
    with pytest.raises(ValueError, match=re.escape(msg)):
        solver.Workspace(p, Settings())


def test_warm_start_dimension_mismatch():
    p = two_var()
    w = WarmStart(np.zeros(3), np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError, match="solve: warm start dimension mismatch"):
        solver.solve(p, Settings(), initial=w)


def test_reassigned_arrays_are_coerced_to_the_problem_dtype():
    p = two_var().astype(np.float32)
    p.q = np.array([1.0, 2.0])            # float64 assigned after construction
    p.a.values = p.a.values.astype(np.float64)
    c = p.checked()
    assert c.q.dtype == c.a.values.dtype == c.l.dtype == np.float32
    assert c.q.flags.c_contiguous and list(c.q) == [1.0, 2.0]


def test_settings_from_json_converts_and_validates():
    s = Settings.from_json('{"lambda_pcg": 0.01, "max_admm_iter": 10.7, "alpha": 1}')
    assert s.lambda_pcg == 0.01 and s.max_admm_iter == 10 and isinstance(s.alpha, float)
    with pytest.raises(ValueError, match="settings: alpha must be in \\(0, 2\\)"):
        Settings.from_json('{"alpha": 3}')
    with pytest.raises(ValueError, match="lambda_pcg must be in \\(0, 1\\)"):
        Settings.from_json('{"lambda_pcg": 1.5}')
    with pytest.raises(RuntimeError, match="type must be number, but is string"):
        Settings.from_json('{"lambda_pcg": "0.01"}')
    with pytest.raises(RuntimeError, match="type must be boolean, but is number"):
        Settings.from_json('{"scaling_enabled": 1}')
    with pytest.raises(RuntimeError, match="type must be number, but is boolean"):
        Settings.from_json('{"max_admm_iter": true}')
    with pytest.raises(RuntimeError, match="settings: unknown key 'lambda'"):
        Settings.from_json('{"lambda": 0.01}')
    # a negative index wraps like static_cast<uint32_t>, then validate accepts it
    assert Settings.from_json('{"check_interval": -1}').check_interval == 0xFFFFFFFF


def test_release_cached_memory_is_exported():
    assert hasattr(solver.load_library(), "qpcg_release_cached_memory")
