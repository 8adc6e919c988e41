"""Sweep lambda_pcg on a BASELINE config (GPU) + kernel timing at full size."""
import ctypes as C, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
cfg = sys.argv[1]
lams = [float(v) for v in sys.argv[2].split(",")]
maxit = int(sys.argv[3])
t = time.time(); p = G.config(cfg); print(f"[{cfg}] gen {time.time()-t:.1f}s n={p.n} m={p.m} nnzA={p.a.nnz}", flush=True)
for lam in lams:
    d = SolveDiagnostics()
    g = solver.solve(p, Settings(lambda_pcg=lam, max_admm_iter=maxit), diag=d, device=0)
    its = [c["iterations"] for c in d.pcg_calls]
    print(f"[{cfg}] lam={lam:g}: {g.status} iters={g.iterations} pcg={g.pcg_iterations_total} obj={g.objective:.8g} "
          f"setup={g.info['setup_seconds']:.3f}s loop={g.info['solve_seconds']:.3f}s rp={g.r_prim_inf:.2e} rd={g.r_dual_inf:.2e} "
          f"pcg[:12]={its[:12]} zero_pcg={sum(1 for i in its if i == 0)}", flush=True)
lib = solver.load_library()
with solver.Workspace(p, Settings(lambda_pcg=lams[0]), device=0) as ws:
    out = np.zeros(9)
    lib.qpcg_bench_kernels.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
    lib.qpcg_bench_kernels(ws.ws, 20, out.ctypes.data)
print(f"[{cfg}] kernels: A {out[0]:.4f} ms ({out[3]/out[0]/1e6:.0f} GB/s), A^T {out[1]:.4f} ms ({out[4]/out[1]/1e6:.0f} GB/s), "
      f"PCG iter {out[2]:.4f} ms ({out[5]/out[2]/1e6:.0f} GB/s)", flush=True)
