"""One solve of a BASELINE config (for ncu launch lists / captures)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
mode = sys.argv[2] if len(sys.argv) > 2 else "eager"
lam = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
p = G.config(cfg)
g = solver.solve(p, Settings(lambda_pcg=lam), device=0, mode=mode)
print(f"config {cfg}: {g.status} iters={g.iterations} pcg={g.pcg_iterations_total} launches={g.info['kernel_launches']}")
