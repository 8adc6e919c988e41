"""e2e (host-array) solve timing breakdown: python scripts/e2e_dbg.py"""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_1912_04263_b200 import generators
from paper_1912_04263_b200.problem import Settings
p = generators.config("2")
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    eng = bench.Engine(p, Settings(lambda_pcg=1e-3), 0, st.cuda_stream, np.float64, "graph")
    for k in range(5):
        for mem in ("host", "device"):
            torch.cuda.synchronize(); t = time.time()
            info = eng.solve(mem)
            torch.cuda.synchronize()
            print(mem, f"wall={time.time()-t:.3f} setup={info.setup_seconds:.3f} h2d={info.h2d_seconds:.3f} loop={info.solve_seconds:.3f} d2h={info.d2h_seconds:.3f} runtime={info.runtime_seconds:.3f}", flush=True)
