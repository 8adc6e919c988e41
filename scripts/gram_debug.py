"""k_gram timing variants (QPCG_GRAM_DEBUG: 0 normal, 1 no ticket, 3 no
ticket and no scatter) on one config.   python scripts/gram_debug.py [CFG]"""
import ctypes as C
import os
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
lib = solver.load_library()
lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
p = G.config(cfg)
for dbg in ("0", "1", "3"):
    os.environ["QPCG_GRAM_DEBUG"] = dbg
    os.environ["QPCG_GRAM_TRACE"] = "1"
    with solver.Workspace(p, Settings(lambda_pcg=1e-3), device=0) as ws:
        out = np.zeros(12)
        lib.qpcg_bench_kernels_n(ws.ws, 10, out.ctypes.data, 12)
    print(f"dbg={dbg}: k_gram {out[9]:.4f} ms, pcg iteration {out[2]:.4f} ms, "
          f"A {out[0]:.4f} A^T {out[1]:.4f}", flush=True)
