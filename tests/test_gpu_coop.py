"""The opt-in cooperative PCG vector step (k_pcg_step, QPCG_COOP_PCG=1) is
bitwise identical to the three separate kernels, in the graph and eager
drivers (subprocess: the switch is read once per process)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import json, sys, hashlib
sys.path.insert(0, %r)
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
S = Settings(lambda_pcg=0.01)
out = {}
for cls, sc in (("lasso", 6), ("svm", 5), ("portfolio", 5)):
    p = G.generate(cls, sc, 0)
    for mode in ("graph", "eager"):
        r = solver.solve(p, S, device=0, mode=mode)
        out[f"{cls}-{mode}"] = [r.iterations, r.pcg_iterations_total,
                                hashlib.sha1(r.x.tobytes() + r.y.tobytes()).hexdigest()]
print(json.dumps(out))
"""


def run(env):
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], capture_output=True, text=True,
                       env=dict(os.environ, QPCG_PERSIST_MAX_NNZ="0", **env), timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_cooperative_pcg_step_bitwise():
    a = run({"QPCG_COOP_PCG": "0"})
    b = run({"QPCG_COOP_PCG": "1"})
    assert a == b
