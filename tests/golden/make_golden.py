"""Regenerate tests/golden/*.json from the REFERENCE itself (oracle/_ref, built from
the unmodified /root/reference headers).  Run in the build container:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from _util import kat_problems, paper_matrix  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1912_04263_b200.problem import CsrMatrix, Settings  # noqa: E402


def f(v):
    return [float(x) for x in np.asarray(v).ravel()]


def main():
    out = {"source": "oracle/_ref (unmodified reference headers)", "kat": {}, "solves": {}}
    A = paper_matrix()
    at = O.transpose(A, kind="ref")
    out["kat"]["paper_transpose"] = dict(row_ptr=[int(v) for v in at.row_ptr],
                                         col=[int(v) for v in at.col_indices], values=f(at.values))
    out["kat"]["paper_spmv_e0"] = f(O.spmv(A, np.array([1.0, 0, 0, 0, 0]), kind="ref"))
    out["kat"]["paper_spmv_ones"] = f(O.spmv(A, np.ones(5), kind="ref"))
    pf = CsrMatrix.from_dense(np.diag([1.0, 2.0]))
    a1 = CsrMatrix.from_dense(np.array([[1.0, 1.0]]))
    kx, _ = O.kkt_apply(pf, a1, O.transpose(a1, kind="ref"), 0.001, 0.5, np.array([1.0, 0.0]), kind="ref")
    _, dm = O.kkt_apply(pf, a1, O.transpose(a1, kind="ref"), 1e-6, 0.1, np.array([1.0, 0.0]), kind="ref")
    out["kat"]["operator_k10"] = f(kx)
    out["kat"]["jacobi_diag"] = f(dm)
    out["kat"]["adaptive_eps"] = O.adaptive_eps(1e-2, 1e-4, 0.15, 1e-7, kind="ref")
    for name, p in kat_problems().items():
        r = O.ref_solve(p, Settings())
        out["solves"][name] = dict(status=r.status, iterations=r.iterations,
                                   pcg=r.pcg_iterations_total, objective=r.objective,
                                   x=f(r.x), z=f(r.z), y=f(r.y), certificate=f(r.certificate))
    for cls in O.CLASSES:
        p = O.ref_generate(cls, 2, 0)
        r = O.ref_solve(p, Settings(lambda_pcg=0.01))
        out["solves"][f"{cls}_s2"] = dict(status=r.status, iterations=r.iterations,
                                          pcg=r.pcg_iterations_total, objective=r.objective,
                                          x=f(r.x))
    with open(os.path.join(HERE, "reference_outputs.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "reference_outputs.json"))


if __name__ == "__main__":
    main()
