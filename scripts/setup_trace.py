"""Setup phase timeline of one config (QPCG_SETUP_TRACE=1 prints it):
    QPCG_SETUP_TRACE=1 python scripts/setup_trace.py 2"""
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

p = G.config(sys.argv[1] if len(sys.argv) > 1 else "2")
for _ in range(3):
    o = solver.solve(p, Settings(lambda_pcg=1e-3), device=0)
    print(f"setup {o.info['setup_seconds']*1e3:.2f} ms loop {o.info['solve_seconds']*1e3:.2f} ms",
          file=sys.stderr, flush=True)
