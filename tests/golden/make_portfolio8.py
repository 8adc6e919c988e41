"""Golden fixture for tests/test_gpu_parity.py::test_portfolio_scale8_eps1e5 (VERDICT r01:
"a portfolio scale-8 comparison at eps = 1e-5"): the oracle's solve of
generate("portfolio", 8, 0) at eps_abs = eps_rel = 1e-5 (lambda_pcg 0.01) and of
its row-reversed twin (the oracle's own reorder noise at that tolerance).
    python tests/golden/make_portfolio8.py   (CPU, ~5 minutes)"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1912_04263_b200 import generators as G  # noqa: E402
from paper_1912_04263_b200.problem import Settings  # noqa: E402
from _util import reversed_twin  # noqa: E402

S = Settings(lambda_pcg=0.01, eps_abs=1e-5, eps_rel=1e-5, max_admm_iter=20000)
p = G.generate("portfolio", 8, 0)
o = O.oracle_solve(p, S)
t = O.oracle_solve(reversed_twin(p), S)
xs = max(1.0, float(np.max(np.abs(o.x))))
out = {"class": "portfolio", "scale": 8, "seed": 0, "settings": "lambda_pcg 0.01, eps 1e-5",
       "status": o.status, "iterations": o.iterations, "objective": o.objective,
       "x": [float(v) for v in o.x],
       "twin_status": t.status, "twin_iterations": t.iterations,
       "noise_rel_obj": abs(t.objective - o.objective) / max(1.0, abs(o.objective)),
       "noise_x": float(np.max(np.abs(t.x - o.x))) / xs,
       "note": "oracle (plain-C restatement, pinned to the reference) — make_portfolio8.py"}
json.dump(out, open(os.path.join(HERE, "portfolio8_eps1e-5.json"), "w"))
print({k: v for k, v in out.items() if k != "x"})
