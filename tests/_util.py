"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import math

import numpy as np

from paper_1912_04263_b200.problem import CsrMatrix, QpProblem, Settings

INF = math.inf


def paper_matrix(dtype=np.float64) -> CsrMatrix:
    """The 4x5 example of PAPER.md:575-608."""
    return CsrMatrix(4, 5, np.array([1, 4, 5, 1, 2, 1, 7, 1], dtype),
                     np.array([0, 2, 4, 6, 8], np.uint32),
                     np.array([0, 4, 1, 2, 1, 4, 0, 2], np.uint32))


def dense_qp(P_upper, q, A, l, u, dtype=np.float64) -> QpProblem:
    return QpProblem(CsrMatrix.from_dense(np.triu(np.asarray(P_upper, float)), dtype),
                     np.asarray(q, dtype), CsrMatrix.from_dense(np.asarray(A, float), dtype),
                     np.asarray(l, dtype), np.asarray(u, dtype))


def kat_problems(dtype=np.float64) -> dict:
    """SPEC.md:376-378 (solve examples) and :421/:430/:597 (infeasibility)."""
    return {
        "n1_equality": dense_qp([[1.0]], [0.0], [[1.0]], [1.0], [1.0], dtype),
        "unconstrained": dense_qp([[1.0]], [2.0], [[1.0]], [-INF], [INF], dtype),
        "two_var": dense_qp(np.eye(2), [-1.0, -1.0], [[1.0, 1.0]], [-INF], [1.0], dtype),
        "primal_infeasible": dense_qp([[1.0]], [0.0], [[1.0], [1.0]], [-INF, 1.0], [-1.0, INF],
                                      dtype),
        "dual_infeasible": QpProblem(CsrMatrix(1, 1, np.zeros(0, dtype), np.zeros(2, np.uint32),
                                               np.zeros(0, np.uint32)),
                                     np.array([-1.0], dtype), CsrMatrix.from_dense([[1.0]], dtype),
                                     np.array([-INF], dtype), np.array([INF], dtype)),
    }


def kkt_residuals(p: QpProblem, x, z, y):
    """Independent residuals on the ORIGINAL data (SPEC acceptance 3; Eq. 6)."""
    P = p.p_upper.to_scipy().astype(np.float64)
    Pf = P + P.T - __import__("scipy.sparse", fromlist=["diags"]).diags(P.diagonal())
    A = p.a.to_scipy().astype(np.float64)
    x, z, y = (np.asarray(v, np.float64) for v in (x, z, y))
    ax = A @ x
    px = Pf @ x
    aty = A.T @ y
    q = p.q.astype(np.float64)
    rp = np.max(np.abs(ax - z)) if p.m else 0.0
    rd = np.max(np.abs(px + q + aty)) if p.n else 0.0
    norms = dict(ax=np.max(np.abs(ax)) if p.m else 0.0, z=np.max(np.abs(z)) if p.m else 0.0,
                 px=np.max(np.abs(px)), aty=np.max(np.abs(aty)), q=np.max(np.abs(q)))
    return rp, rd, norms


def kkt_ok(p: QpProblem, out, settings: Settings, slack: float = 1.0) -> bool:
    rp, rd, nm = kkt_residuals(p, out.x, out.z, out.y)
    eps_p = settings.eps_abs + settings.eps_rel * max(nm["ax"], nm["z"])
    eps_d = settings.eps_abs + settings.eps_rel * max(nm["px"], nm["aty"], nm["q"])
    return rp <= slack * eps_p and rd <= slack * eps_d


def reversed_twin(p: QpProblem) -> QpProblem:
    """The same QP with A's rows (and l, u) reversed: only summation order changes
    (SURVEY.md §8(c) reorder-noise protocol)."""
    A = p.a
    rows = A.rows
    rp = A.row_ptr.astype(np.int64)
    order = np.arange(rows)[::-1]
    vals, cols, nrp = [], [], [0]
    for r in order:
        vals.append(A.values[rp[r]:rp[r + 1]])
        cols.append(A.col_indices[rp[r]:rp[r + 1]])
        nrp.append(nrp[-1] + rp[r + 1] - rp[r])
    a2 = CsrMatrix(rows, A.cols, np.concatenate(vals) if vals else A.values[:0],
                   np.array(nrp, np.uint32), np.concatenate(cols) if cols else A.col_indices[:0])
    return QpProblem(p.p_upper, p.q, a2, p.l[::-1].copy(), p.u[::-1].copy())


def rel(a, b) -> float:
    return abs(a - b) / max(1.0, abs(b))


def xrel(x, xr) -> float:
    return float(np.max(np.abs(np.asarray(x, float) - xr)) / max(1.0, np.max(np.abs(xr)))) if len(xr) else 0.0
