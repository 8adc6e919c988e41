"""Setup phase trace of a tiny instance (lasso scale 2):
    QPCG_SETUP_TRACE=1 python scripts/tiny_setup_trace.py"""
import sys, os
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
p = G.generate("lasso", 2, 0)
for i in range(3):
    o = solver.solve(p, Settings(lambda_pcg=0.01), device=0)
    print("setup", o.info["setup_seconds"]*1e3, "loop", o.info["solve_seconds"]*1e3, "total", o.runtime_seconds*1e3, file=sys.stderr)
