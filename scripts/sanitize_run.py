"""Small solves through every driver, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck):
    compute-sanitizer --tool memcheck python scripts/sanitize_run.py"""
import sys

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np

from _util import kat_problems
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

S = Settings(lambda_pcg=0.01, max_admm_iter=60)
probs = [G.generate("lasso", 3, 0), G.generate("portfolio", 3, 0), G.generate("svm", 2, 1),
         kat_problems()["primal_infeasible"], kat_problems()["dual_infeasible"]]
for p in probs:
    for mode in ("eager", "graph", "persistent"):
        r = solver.solve(p, S, device=0, mode=mode)
        print(mode, p.n, p.m, r.status, r.iterations, flush=True)
    r = solver.solve(p, S, device=0, shards=2)
    print("sharded", p.n, p.m, r.status, r.iterations, flush=True)
    with solver.Workspace(p, S, device=0, mode="eager") as ws:
        a = ws.solve()
        ws.warm_start(a.x, a.z, a.y)
        ws.update_rho(0.5)
        ws.update_vectors(q=p.q * 1.0)
        ws.solve()
print("done")
