"""fp32 kernel timing on the BASELINE configs (see kernel_sweep.py)."""
import ctypes as C
import sys

sys.path.insert(0, "/root/repo")
import numpy as np

from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

lib = solver.load_library()
lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
for cfg in sys.argv[1].split(","):
    p = G.config(cfg).astype(np.float32)
    with solver.Workspace(p, Settings(lambda_pcg=1e-3), device=0) as ws:
        out = np.zeros(12)
        lib.qpcg_bench_kernels_n(ws.ws, 20, out.ctypes.data, 12)
        lib.qpcg_bench_kernels_n(ws.ws, 20, out.ctypes.data, 12)
    print(f"[{cfg} f32] A {out[0]*1e3:7.1f} us | A^T {out[1]*1e3:7.1f} us | PCG iter {out[2]*1e3:7.1f} us "
          f"({out[8]/out[2]/1e6:6.0f} GB/s format bytes)", flush=True)
