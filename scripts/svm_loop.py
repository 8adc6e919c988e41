"""svm (config 4) with the loop capped: per-iteration cost of the whole ADMM
loop (graph driver).   python scripts/svm_loop.py [ITERS]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
it = int(sys.argv[1]) if len(sys.argv) > 1 else 200
p = G.config("4")
for k in range(2):
    g = solver.solve(p, Settings(lambda_pcg=1e-3, max_admm_iter=it), device=0)
print("svm", g.status, g.iterations, g.pcg_iterations_total, "setup %.1f ms loop %.1f ms" % (
    g.info["setup_seconds"] * 1e3, g.info["solve_seconds"] * 1e3), flush=True)
