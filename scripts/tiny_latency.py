"""Setup vs loop time of tiny instances (default graph mode, which picks the
persistent drivers): python scripts/tiny_latency.py"""
import sys

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

S = Settings(lambda_pcg=0.01)
for kind in ("lasso", "huber", "svm", "random", "control", "portfolio", "equality"):
    for scale in (2, 4):
        p = G.generate(kind, scale, 0)
        ts = [solver.solve(p, S, device=0) for _ in range(4)]
        t = min(ts[1:], key=lambda o: o.runtime_seconds)
        pcg = max(t.pcg_iterations_total, 1)
        print(f"{kind}:{scale} N={p.a.nnz + p.p_upper.nnz} it={t.iterations}/{t.pcg_iterations_total} "
              f"total {t.runtime_seconds*1e3:7.2f} ms setup {t.info['setup_seconds']*1e3:6.2f} ms "
              f"loop {t.info['solve_seconds']*1e3:7.2f} ms = {t.info['solve_seconds']*1e6/(pcg + t.iterations):6.2f} us/(pcg+admm it)",
              flush=True)
