"""Loop time of the persistent driver's barrier variants (one block / one
16-SM cluster / cooperative grid) on tiny instances: python scripts/persist_variants.py"""
import os, sys
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
S = Settings(lambda_pcg=0.01)
MODES = (("cluster", {"QPCG_CLUSTER_MAX_NNZ": "100000000", "QPCG_BLOCK_MAX_NNZ": "0"}),
         ("block", {"QPCG_BLOCK_MAX_NNZ": "100000000"}),
         ("grid", {"QPCG_CLUSTER_MAX_NNZ": "0", "QPCG_BLOCK_MAX_NNZ": "0"}))
for kind, scale in (("lasso", 0), ("lasso", 1), ("lasso", 2), ("huber", 2), ("svm", 2), ("random", 2), ("lasso", 3)):
    p = G.generate(kind, scale, 0)
    row = []
    for name, env in MODES:
        for k in ("QPCG_CLUSTER_MAX_NNZ", "QPCG_BLOCK_MAX_NNZ"):
            os.environ.pop(k, None)
        os.environ.update(env)
        ts = [solver.solve(p, S, device=0, mode="persistent") for _ in range(3)]
        t = min(x.info["solve_seconds"] for x in ts)
        it = ts[-1].iterations + ts[-1].pcg_iterations_total
        row.append(f"{name} {t*1e3:7.2f} ms ({t*1e6/it:5.1f} us/it)")
    print(f"{kind}:{scale} N={p.a.nnz + p.p_upper.nnz} | " + " | ".join(row), flush=True)
