"""Run the REFERENCE (oracle/_ref, unmodified headers, 1 thread) to completion on
a BASELINE config and store its outcome under profiles/ (parity anchor + measured
CPU time).  Usage: python scripts/ref_solve_config.py CONFIG LAMBDA [MAXIT]"""
import json, os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import oracle as O
from paper_1912_04263_b200 import generators as G
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
cfg, lam = sys.argv[1], float(sys.argv[2])
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
p = G.config(cfg)
d = SolveDiagnostics()
t = time.time()
r = O.ref_solve(p, Settings(lambda_pcg=lam, max_admm_iter=maxit), diag=d)
wall = time.time() - t
out = dict(config=cfg, lambda_pcg=lam, status=r.status, iterations=r.iterations,
           pcg_iterations_total=r.pcg_iterations_total, objective=r.objective,
           r_prim_inf=r.r_prim_inf, r_dual_inf=r.r_dual_inf, runtime_seconds=r.runtime_seconds,
           wall_seconds=wall, equil_passes=r.equil_passes, rho_final=r.rho_final,
           pcg_per_call=[c["iterations"] for c in d.pcg_calls],
           host=os.uname().nodename, nproc=os.cpu_count(), threads_used=1,
           x_inf=float(np.max(np.abs(r.x))))
os.makedirs("/root/repo/profiles", exist_ok=True)
fn = f"/root/repo/profiles/ref_solve_config{cfg}_lam{lam:g}.json"
json.dump(out, open(fn, "w"), indent=1)
np.save(f"/tmp/ref_x_config{cfg}_lam{lam:g}.npy", r.x)
print(json.dumps({k: v for k, v in out.items() if k != "pcg_per_call"}))
