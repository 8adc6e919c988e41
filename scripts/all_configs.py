"""Solve every BASELINE config on the GPU once (graph mode) and KKT-check the
answer on the ORIGINAL data with scipy (independent of engine and oracle).

    python scripts/all_configs.py [lambda] [configs,comma,sep] [max_iter]

Writes one JSON line per config to stdout (collected into profiles/)."""
import json
import sys
import time

sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import ctypes as C

import numpy as np

from _util import kkt_residuals
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

lam = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "1p", "2", "3", "4", "5a", "5b"]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 50000
for cfg in cfgs:
    t = time.time()
    p = G.config(cfg)
    gen = time.time() - t
    s = Settings(lambda_pcg=lam, max_admm_iter=maxit)
    t = time.time()
    g = solver.solve(p, s, device=0)
    wall = time.time() - t
    rp, rd, nm = kkt_residuals(p, g.x, g.z, g.y)
    eps_p = s.eps_abs + s.eps_rel * max(nm["ax"], nm["z"])
    eps_d = s.eps_abs + s.eps_rel * max(nm["px"], nm["aty"], nm["q"])
    lib = solver.load_library()
    with solver.Workspace(p, s, device=0) as ws:
        out = np.zeros(9)
        lib.qpcg_bench_kernels.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p]
        lib.qpcg_bench_kernels(ws.ws, 10, out.ctypes.data)
    rec = dict(config=cfg, n=p.n, m=p.m, nnz_A=int(p.a.nnz), nnz_P_upper=int(p.p_upper.nnz),
               lambda_pcg=lam, status=g.status, iterations=g.iterations,
               pcg_iterations_total=g.pcg_iterations_total, objective=g.objective,
               setup_s=g.info["setup_seconds"], loop_s=g.info["solve_seconds"], wall_s=wall,
               gen_s=gen, kkt_rp=rp, kkt_rd=rd, kkt_eps_p=eps_p, kkt_eps_d=eps_d,
               kkt_ok=bool(rp <= eps_p and rd <= eps_d),
               a_pass_ms=out[0], at_pass_ms=out[1], pcg_iter_ms=out[2],
               a_pass_gbs=out[3] / out[0] / 1e6, at_pass_gbs=out[4] / out[1] / 1e6,
               pcg_iter_gbs=out[5] / out[2] / 1e6, launches=g.info["kernel_launches"])
    print(json.dumps(rec), flush=True)
