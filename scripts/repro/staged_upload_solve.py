import sys
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
S = Settings(lambda_pcg=0.01, max_admm_iter=60)
big = G.generate_explicit("lasso", 1000, 20000, 0, 3)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    r = solver.solve(big, S, device=0)
print("staged", big.a.nnz, r.status, r.iterations, flush=True)
