"""Sharded solve under compute-sanitizer synccheck (scripts/sync_shard.py <mode>)."""
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

mode = sys.argv[1] if len(sys.argv) > 1 else "graph"
p = G.generate("lasso", 3, 0)
r = solver.solve(p, Settings(lambda_pcg=0.01, max_admm_iter=60), device=0, shards=2, mode=mode)
print("sharded", mode, r.status, r.iterations, flush=True)
