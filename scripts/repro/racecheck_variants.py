"""One solve of the staged-upload lasso instance (3e6 nnz) in a chosen driver,
for bisecting a compute-sanitizer racecheck crash:
    compute-sanitizer --tool racecheck python scripts/repro/racecheck_variants.py MODE ITERS"""
import sys
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
mode, it = sys.argv[1], int(sys.argv[2])
p = G.generate_explicit("lasso", 1000, 20000, 0, 3)
r = solver.solve(p, Settings(lambda_pcg=0.01, max_admm_iter=it), device=0, mode=mode)
print(mode, it, "ok", r.status, r.iterations, flush=True)
