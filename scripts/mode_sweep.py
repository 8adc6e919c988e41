"""Device solve time of the loop drivers on small / medium problems:
graph (conditional nodes), persistent grid (one cooperative kernel), persistent
cluster (one thread-block cluster, hardware barriers).
    python scripts/mode_sweep.py"""
import os
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

S = Settings(lambda_pcg=1e-3)
MODES = (("graph", "graph", {"QPCG_PERSIST_MAX_NNZ": "0"}),
         ("grid", "persistent", {"QPCG_CLUSTER_MAX_NNZ": "0", "QPCG_BLOCK_MAX_NNZ": "0"}),
         ("cluster", "persistent", {"QPCG_CLUSTER_MAX_NNZ": "100000000", "QPCG_BLOCK_MAX_NNZ": "0"}),
         ("block", "persistent", {"QPCG_BLOCK_MAX_NNZ": "100000000"}))
cases = [(c, s) for c in ("lasso", "huber", "svm", "random", "control", "portfolio", "equality")
         for s in (0, 1, 2, 3, 4, 5)]
for kind, arg in cases:
    p = G.config(arg) if kind == "config" else G.generate(kind, arg, 0)
    row = []
    for name, mode, env in MODES:
        for k in ("QPCG_PERSIST_MAX_NNZ", "QPCG_CLUSTER_MAX_NNZ", "QPCG_BLOCK_MAX_NNZ"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ts = [solver.solve(p, S, device=0, mode=mode) for _ in range(3)]
        row.append((name, min(t.info["solve_seconds"] for t in ts), ts[-1]))
    for k in ("QPCG_PERSIST_MAX_NNZ", "QPCG_CLUSTER_MAX_NNZ", "QPCG_BLOCK_MAX_NNZ"):
        os.environ.pop(k, None)
    g = row[0][2]
    same = all(r[2].iterations == g.iterations and (r[2].x == g.x).all() for r in row)
    print(f"{kind}:{arg} N={p.a.nnz + p.p_upper.nnz} it={g.iterations}/{g.pcg_iterations_total} "
          + " | ".join(f"{n} {t*1e3:8.2f} ms" for n, t, _ in row) + f" | bitwise-same={same}",
          flush=True)
