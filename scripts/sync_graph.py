"""Unsharded conditional-graph solve (persistent driver disabled) for synccheck."""
import os
import sys

os.environ["QPCG_PERSIST_MAX_NNZ"] = "0"
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

p = G.generate("lasso", 3, 0)
r = solver.solve(p, Settings(lambda_pcg=0.01, max_admm_iter=60), device=0, mode="graph")
print("graph", r.status, r.iterations, flush=True)
