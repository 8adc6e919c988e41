"""One-pass vs two-pass PCG operator apply on full-size BASELINE configs:
solve time, iterations, objective and the per-iteration kernel timings
(qpcg_bench_kernels) with QPCG_GRAM=1 / 0.
    python scripts/gram_check.py [CONFIGS...]   (GPU)"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

S = Settings(lambda_pcg=1e-3)
lib = solver.load_library()
lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
for cfg in sys.argv[1:] or ["2", "3", "4"]:
    p = G.config(cfg)
    if cfg == "4":
        S.max_admm_iter = 300
    for gram in ("1", "0"):
        os.environ["QPCG_GRAM"] = gram
        with solver.Workspace(p, S, device=0) as ws:
            r = ws.solve()
            out = np.zeros(12)
            lib.qpcg_bench_kernels_n(ws.ws, 20, out.ctypes.data, 12)
        t = time.time()
        r2 = solver.solve(p, S, device=0)
        print(json.dumps({"config": cfg, "gram": gram, "status": r.status,
                          "iterations": r.iterations, "pcg": r.pcg_iterations_total,
                          "engine_flags": r.info.get("engine_flags"),
                          "objective": r.objective, "setup_s": r.info["setup_seconds"],
                          "loop_s": r.info["solve_seconds"], "resolve_wall": time.time() - t,
                          "a_ms": out[0], "at_ms": out[1], "pcg_iter_ms": out[2],
                          "k_gram_ms": out[9], "k_gram_bytes": out[10],
                          "pcg_iter_bytes_gram": out[11]}), flush=True)
    S.max_admm_iter = 50000
