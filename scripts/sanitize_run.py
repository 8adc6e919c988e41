"""Small solves through every driver (plus one staged-upload solve and a
solve_batch), for compute-sanitizer (memcheck /
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
# round 2: the on_iteration observer (host-driven loop), the opt-in one-pass
# operator (gram.cuh), a rejected update_vectors, the memory release
import os
from paper_1912_04263_b200.problem import SolveDiagnostics
views = []
r = solver.solve(probs[0], S, device=0, diag=SolveDiagnostics(on_iteration=views.append))
print("on_iteration", len(views), r.iterations, flush=True)
os.environ["QPCG_GRAM"] = "1"
for p in ((G.generate("lasso", 4, 0), G.generate("svm", 3, 0))
          if os.environ.get("SANITIZE_GRAM", "1") == "1" else ()):
    r = solver.solve(p, S, device=0, mode="eager")
    print("gram", p.n, p.m, r.status, r.iterations, r.info["engine_flags"], flush=True)
del os.environ["QPCG_GRAM"]
with solver.Workspace(probs[0], S, device=0) as ws:
    ws.solve()
    try:
        ws.update_vectors(l=probs[0].u + 1.0)
    except ValueError as e:
        print("rejected update:", e, flush=True)
    ws.solve()
print("after the rejected update", flush=True)
# staged pageable upload (A's values > 8 MB) with the background feed
big = G.generate_explicit("lasso", 1000, 20000, 0, 3)  # 24 MB of values: staged
r = solver.solve(big, S, device=0)
print("staged", big.a.nnz, r.status, r.iterations, flush=True)
# many small solves side by side with a capped persistent driver
outs = solver.solve_batch([G.generate("random", 2, s) for s in range(4)], S, device=0,
                          concurrency=2)
print("batch", [o.iterations for o in outs], flush=True)
print("done", flush=True)
solver.release_cached_memory()
print("released", flush=True)
