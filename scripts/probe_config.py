"""One diagnosed solve of a BASELINE config on the GPU (progress + timings)."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 50000
t = time.time(); p = G.config(cfg); print(f"gen {time.time()-t:.1f}s n={p.n} m={p.m} nnzA={p.a.nnz}", flush=True)
d = SolveDiagnostics()
t = time.time()
g = solver.solve(p, Settings(lambda_pcg=0.01, max_admm_iter=maxit), diag=d, device=0)
print(f"status={g.status} iters={g.iterations} pcg={g.pcg_iterations_total} obj={g.objective:.10g} "
      f"setup={g.info['setup_seconds']:.3f} solve={g.info['solve_seconds']:.3f} wall={time.time()-t:.2f} "
      f"rho_final={g.rho_final:.4g} rp={g.r_prim_inf:.3e} rd={g.r_dual_inf:.3e} launches={g.info['kernel_launches']}", flush=True)
its = [c["iterations"] for c in d.pcg_calls]
print("pcg per admm (first 20):", its[:20])
print("pcg per admm (last 20):", its[-20:])
print("eps (every 50th):", [f"{c['eps']:.2e}" for c in d.pcg_calls[::50]])
print("rho updates (first/last 5):", [(r['admm_iter'], round(r['rho_after'],5)) for r in d.rho_updates[:5]], [(r['admm_iter'], round(r['rho_after'],5)) for r in d.rho_updates[-5:]])
