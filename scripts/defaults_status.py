"""Every BASELINE config at full size at PURE DEFAULT settings
on the engine, uncapped (max_admm_iter = 50 000), beside the reference's capped
trajectory (tests/golden/config*_reference_defaults.json).  One JSON line per
config -> stdout.   python scripts/defaults_status.py [CONFIGS...]"""
import json, os, sys, time
sys.path.insert(0, "/root/repo")
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
cfgs = sys.argv[1:] or ["1", "1p", "2", "3", "4", "5a", "5b"]
for c in cfgs:
    p = G.config(c)
    t = time.time()
    d = SolveDiagnostics()
    g = solver.solve(p, Settings(), device=0, diag=d)
    wall = time.time() - t
    gold = os.path.join("/root/repo/tests/golden", f"config{c}_reference_defaults.json")
    ref = json.load(open(gold)) if os.path.exists(gold) else None
    zero = sum(1 for x in d.pcg_calls if x["iterations"] == 0)
    print(json.dumps({"config": c, "settings": "defaults (lambda_pcg 0.15, max_admm_iter 50000)",
                      "status": g.status, "iterations": g.iterations,
                      "pcg_iterations_total": g.pcg_iterations_total,
                      "pcg_calls_with_0_iterations": zero, "r_prim_inf": g.r_prim_inf,
                      "r_dual_inf": g.r_dual_inf, "rho_final": g.rho_final, "wall_s": wall,
                      "reference_capped": None if ref is None else
                      {k: ref[k] for k in ("max_admm_iter", "status", "iterations",
                                           "pcg_iterations_total", "r_dual_inf")}}), flush=True)
