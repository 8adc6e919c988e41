"""Time the PCG-iteration kernels (CUDA events, qpcg_bench_kernels) on the
BASELINE configs without solving: python scripts/kernel_sweep.py 2,3,4 [reps]"""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import numpy as np

from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lib = solver.load_library()
lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
for cfg in cfgs:
    p = G.config(cfg)
    with solver.Workspace(p, Settings(lambda_pcg=1e-3), device=0) as ws:
        out = np.zeros(12)
        lib.qpcg_bench_kernels_n(ws.ws, reps, out.ctypes.data, 12)
        lib.qpcg_bench_kernels_n(ws.ws, reps, out.ctypes.data, 12)
    print(f"[{cfg}] A {out[0]*1e3:7.1f} us {out[3]/out[0]/1e6:6.0f} GB/s | A^T {out[1]*1e3:7.1f} us "
          f"{out[4]/out[1]/1e6:6.0f} GB/s | PCG iter {out[2]*1e3:7.1f} us {out[5]/out[2]/1e6:6.0f} GB/s"
          f" (format bytes: {out[8]/out[2]/1e6:6.0f} GB/s)",
          flush=True)
