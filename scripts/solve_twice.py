"""Solve a BASELINE config twice in one process (for warm-cache launch lists:
ncu --cache-control none --launch-skip <launches of one solve> ...)."""
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
mode = sys.argv[2] if len(sys.argv) > 2 else "graph"
p = G.config(cfg)
for _ in range(2):
    out = solver.solve(p, Settings(lambda_pcg=1e-3), device=0, mode=mode)
    print(out.status, out.iterations, out.pcg_iterations_total, out.runtime_seconds, flush=True)
