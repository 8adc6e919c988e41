"""z~ recurrence A/B (admm.cuh zt_pass): run with QPCG_ZT_RECUR=0 and =1 in two
processes and compare trajectories (iteration counts, PCG counts per call,
residuals at the checks) on the given instances and drivers.
usage: QPCG_ZT_RECUR=1 python scripts/zt_recur_check.py out.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04263_b200 import generators as G, solver  # noqa: E402
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics  # noqa: E402

CASES = [("random", 4, Settings(max_admm_iter=20000)), ("lasso", 4, Settings(max_admm_iter=2000)),
         ("svm", 4, Settings(max_admm_iter=2000)), ("control", 4, Settings(max_admm_iter=2000)),
         ("random", 6, Settings(max_admm_iter=20000)), ("huber", 5, Settings(lambda_pcg=0.01)),
         ("portfolio", 5, Settings(lambda_pcg=0.01))]
out = []
for cls, sc, s in CASES:
    p = G.generate(cls, sc, 0)
    for mode in ("graph", "eager"):
        d = SolveDiagnostics()
        g = solver.solve(p, s, device=0, mode=mode, diag=d)
        out.append(dict(cls=cls, scale=sc, mode=mode, status=g.status, iterations=g.iterations,
                        pcg=g.pcg_iterations_total, objective=g.objective,
                        calls=[c["iterations"] for c in d.pcg_calls][:400],
                        rp=[c["r_prim_scaled_inf"] for c in d.pcg_calls][:400]))
        print(cls, sc, mode, g.status, g.iterations, g.pcg_iterations_total, g.objective, flush=True)
json.dump(out, open(sys.argv[1], "w"))
