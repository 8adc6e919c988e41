"""The reference's own summation-order noise on a full-size BASELINE config
(SURVEY.md §8(c) parity protocol, step 3): the reference (oracle/_ref, 1
thread) solves the row-reversed twin of the instance (same QP, A's rows and
l, u reversed) and the objective / x differences against its solve of the
original (tests/golden/config<C>_reference_solve.json, full x from
/tmp/ref_x_config<C>_lam<L>.npy written by scripts/ref_solve_config.py) are
stored in that golden file as noise_rel_obj / noise_x.
    python scripts/ref_noise_config.py CONFIG LAMBDA [f64|f32]   (CPU, minutes)"""
import json, sys, time
sys.path.insert(0, "/root/repo")
sys.path.insert(0, "/root/repo/tests")
import numpy as np
from oracle import oracle as O
from paper_1912_04263_b200 import generators as G
from paper_1912_04263_b200.problem import Settings
from _util import reversed_twin

cfg, lam = sys.argv[1], float(sys.argv[2])
f32 = len(sys.argv) > 3 and sys.argv[3] == "f32"
sfx = "_f32" if f32 else ""
gold_fn = f"/root/repo/tests/golden/config{cfg}{sfx}_reference_solve.json"
gold = json.load(open(gold_fn))
x0 = np.load(f"/tmp/ref_x_config{cfg}{sfx}_lam{lam:g}.npy").astype(np.float64)
p = G.config(cfg, dtype=np.float32 if f32 else np.float64)
tw = reversed_twin(p)
t = time.time()
r = O.ref_solve(tw, Settings(lambda_pcg=lam))
gold["noise_status"] = r.status
gold["noise_iterations"] = r.iterations
gold["noise_rel_obj"] = abs(r.objective - gold["objective"]) / max(1.0, abs(gold["objective"]))
gold["noise_x"] = float(np.max(np.abs(r.x.astype(np.float64) - x0)) / max(1.0, np.max(np.abs(x0))))
gold["noise_note"] = ("reference solve of the row-reversed twin (scripts/ref_noise_config.py): "
                      "the reference's own summation-order noise on this instance")
json.dump(gold, open(gold_fn, "w"))
print(json.dumps({k: gold[k] for k in ("noise_status", "noise_iterations", "noise_rel_obj",
                                        "noise_x")}), f"{time.time() - t:.0f}s")
