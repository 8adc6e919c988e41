"""One solve of a BASELINE config with the ADMM loop capped, for ncu captures
of the loop kernels (svm never converges: the cap keeps the capture bounded).

    python scripts/ncu_capture.py CONFIG [f64|f32] [MAXIT] [LAMBDA] [MODE]

Typical capture (one GPU; skips setup's Ruiz SpMV launches):
    ncu --set full --clock-control none --import-source on \
        -k regex:'spmv_kernel|spmv_select_kernel|k_pcg' --launch-skip 60 --launch-count 40 \
        -o gpurun_out/ncu_cfg4 python scripts/ncu_capture.py 4 f64 12
"""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
cfg = sys.argv[1] if len(sys.argv) > 1 else "2"
dt = np.float32 if (len(sys.argv) > 2 and sys.argv[2] == "f32") else np.float64
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 20
lam = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-3
mode = sys.argv[5] if len(sys.argv) > 5 else "eager"
p = G.config(cfg, dtype=dt)
g = solver.solve(p, Settings(lambda_pcg=lam, max_admm_iter=maxit), device=0, mode=mode)
print(f"config {cfg} {dt.__name__}: {g.status} iters={g.iterations} pcg={g.pcg_iterations_total} "
      f"launches={g.info['kernel_launches']}")
