"""Quick GPU check: engine vs oracle on small reference-generated problems."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import oracle as O
from paper_1912_04263_b200 import solver
from paper_1912_04263_b200.problem import Settings

mode = sys.argv[1] if len(sys.argv) > 1 else "eager"
S = Settings(lambda_pcg=0.01)
for cls in O.CLASSES:
    for scale in (1, 3, 5):
        p = O.ref_generate(cls, scale, 0)
        t = time.time(); o = O.oracle_solve(p, S); to = time.time() - t
        try:
            t = time.time(); g = solver.solve(p, S, mode=mode); tg = time.time() - t
        except Exception as e:
            print(cls, scale, "ERROR", repr(e)); continue
        rel = abs(g.objective - o.objective) / max(1.0, abs(o.objective))
        dx = np.max(np.abs(g.x - o.x)) / max(1.0, np.max(np.abs(o.x)))
        print(f"{cls:9s} {scale} n={p.n:6d} m={p.m:6d} ref:{o.status}/{o.iterations}/{o.pcg_iterations_total} "
              f"gpu:{g.status}/{g.iterations}/{g.pcg_iterations_total} obj_rel={rel:.2e} x_rel={dx:.2e} "
              f"t_cpu={to:.3f} t_gpu={tg:.3f} setup={g.info['setup_seconds']:.4f} solve={g.info['solve_seconds']:.4f}", flush=True)
