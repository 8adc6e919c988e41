"""Many small instances per GPU: wall time of solving a batch of instances with
k concurrent workspaces (one stream each, host threads), k = 1, 2, 4, 8, 16.
    python scripts/batch_throughput.py [class] [scale] [count]"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

cls = sys.argv[1] if len(sys.argv) > 1 else "lasso"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 2
count = int(sys.argv[3]) if len(sys.argv) > 3 else 64
S = Settings(lambda_pcg=0.01)
probs = [G.generate(cls, scale, s) for s in range(count)]
solver.solve(probs[0], S, device=0)  # warm up the context
ref = [solver.solve(p, S, device=0) for p in probs]
for k in (1, 2, 4, 8, 16):
    for how in ("threads", "solve_batch"):
        t = time.time()
        if how == "threads":
            with ThreadPoolExecutor(max_workers=k) as ex:
                outs = list(ex.map(lambda p: solver.solve(p, S, device=0), probs))
        else:
            outs = solver.solve_batch(probs, S, device=0, concurrency=k, small_nnz=10**9)
        dt = time.time() - t
        same = all((o.x == r.x).all() and o.iterations == r.iterations for o, r in zip(outs, ref))
        print(f"{cls}:{scale} x{count} {how:11s} k={k:2d} wall {dt*1e3:8.1f} ms  "
              f"{count/dt:7.1f} solves/s  bitwise-same={same}", flush=True)
    continue
    same = all((o.x == r.x).all() and o.iterations == r.iterations for o, r in zip(outs, ref))
    print(f"{cls}:{scale} x{count} threads={k:2d} wall {dt*1e3:8.1f} ms  {count/dt:7.1f} solves/s  "
          f"bitwise-same={same}", flush=True)
