"""The REFERENCE (oracle/_ref, 1 thread) at PURE DEFAULT settings on a full-size
BASELINE config, with the ADMM loop capped at MAXIT (the uncapped run is
50 000 iterations of a diverging loop: days on one core).  Stores the status
and the per-PCG-call trajectory (eps, scaled residuals, PCG iterations) as a
golden anchor for tests/test_gpu_parity.py::test_full_size_defaults_against_reference.

    python scripts/ref_defaults_trajectory.py CONFIG [MAXIT]   (CPU, minutes)
"""
import json, os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import oracle as O
from paper_1912_04263_b200 import generators as G
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
cfg = sys.argv[1]
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 100
p = G.config(cfg)
d = SolveDiagnostics()
t = time.time()
r = O.ref_solve(p, Settings(max_admm_iter=maxit), diag=d)
wall = time.time() - t
out = dict(config=cfg, settings="defaults", max_admm_iter=maxit, status=r.status,
           iterations=r.iterations, pcg_iterations_total=r.pcg_iterations_total,
           objective=r.objective, r_prim_inf=r.r_prim_inf, r_dual_inf=r.r_dual_inf,
           rho_final=r.rho_final, runtime_seconds=r.runtime_seconds, wall_seconds=wall,
           pcg_calls=d.pcg_calls, rho_updates=d.rho_updates,
           note=f"reference qpcg::solve (oracle/_ref, unmodified headers, 1 thread), pure "
                f"default settings except max_admm_iter={maxit}; scripts/ref_defaults_trajectory.py")
json.dump(out, open(f"/root/repo/tests/golden/config{cfg}_reference_defaults.json", "w"))
print(json.dumps({k: v for k, v in out.items() if k not in ("pcg_calls", "rho_updates")}))
