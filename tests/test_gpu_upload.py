"""Host input through the pinned staging ring (csrc/upload.cuh): a problem
whose arrays are pageable (numpy) and the same problem in pinned memory give
bitwise-identical solves; A's values here exceed the staging threshold
(8 MB), so the pageable run takes the staged path with the background feed."""
import numpy as np
import pytest
import torch

from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import CsrMatrix, QpProblem, Settings

pytestmark = pytest.mark.gpu


def _pinned(p: QpProblem) -> QpProblem:
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    m = lambda c: CsrMatrix(c.rows, c.cols, pin(c.values), pin(c.row_ptr), pin(c.col_indices))  # noqa: E731
    return QpProblem(m(p.p_upper), pin(p.q), m(p.a), pin(p.l), pin(p.u))


def test_pageable_and_pinned_inputs_agree():
    p = G.generate_explicit("lasso", 1000, 20000, 0, 3)  # 3e6 nnz: 24 MB of values
    assert p.a.values.nbytes >= 8 << 20
    s = Settings(lambda_pcg=0.01, max_admm_iter=200)
    a = solver.solve(p, s, device=0)
    b = solver.solve(_pinned(p), s, device=0)
    assert (a.status, a.iterations, a.pcg_iterations_total) == \
        (b.status, b.iterations, b.pcg_iterations_total)
    for f in ("x", "y", "z"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert a.info["h2d_bytes"] == b.info["h2d_bytes"] > 0
