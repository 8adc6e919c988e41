"""Device solve time of the loop drivers on small / medium problems:
graph (conditional nodes), persistent (one cooperative kernel), eager.
    python scripts/mode_sweep.py"""
import os
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

S = Settings(lambda_pcg=1e-3)
cases = [("config", "1"), ("config", "1p")] + [(c, s) for c in ("lasso", "huber", "svm", "portfolio", "control") for s in (5, 7, 8, 9)]
for kind, arg in cases:
    p = G.config(arg) if kind == "config" else G.generate(kind, arg, 0)
    row = []
    for mode, env in (("graph", "0"), ("persistent", None)):
        if env is not None:
            os.environ["QPCG_PERSIST_MAX_NNZ"] = env
        else:
            os.environ.pop("QPCG_PERSIST_MAX_NNZ", None)
        ts = []
        for _ in range(3):
            g = solver.solve(p, S, device=0, mode=mode)
            ts.append(g.info["solve_seconds"])
        row.append((mode, min(ts), g.iterations, g.pcg_iterations_total, g.info["setup_seconds"]))
    os.environ.pop("QPCG_PERSIST_MAX_NNZ", None)
    print(f"{kind}:{arg} n={p.n} m={p.m} nnzA={p.a.nnz} " + " | ".join(
        f"{m}: loop {t*1e3:8.2f} ms ({it}/{pcg})" for m, t, it, pcg, _ in row)
        + f" | setup {row[0][4]*1e3:.2f} ms | speedup {row[0][1]/row[1][1]:.2f}x", flush=True)
