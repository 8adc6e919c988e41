"""The one-pass PCG operator apply (csrc/gram.cuh: K p with A streamed once,
the A^T side accumulated per CTA over A's dense column window).  An opt-in
path (QPCG_GRAM=1; measured slower than the two-pass SpMV on B200, DESIGN.md
§4), forced here on small instances and compared with the two-pass path and
the oracle; graph vs eager bitwise with the path on (subprocess: the
persistent driver, which small graph-mode solves would take, is switched off
there)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
from test_gpu_parity import check_parity

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _solve(p, gram, mode="eager", diag=None):
    old = os.environ.get("QPCG_GRAM")
    os.environ["QPCG_GRAM"] = "1" if gram else "0"
    try:
        return solver.solve(p, S, device=0, mode=mode, diag=diag)
    finally:
        if old is None:
            del os.environ["QPCG_GRAM"]
        else:
            os.environ["QPCG_GRAM"] = old


@pytest.mark.parametrize("cls,scale", [("lasso", 5), ("huber", 5), ("svm", 5), ("lasso", 7),
                                       ("random", 4), ("control", 4), ("portfolio", 4)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gram_matches_two_pass_and_oracle(cls, scale, dtype):
    p = G.generate(cls, scale, 0).astype(dtype)
    dg, d2 = SolveDiagnostics(), SolveDiagnostics()
    g = _solve(p, True, diag=dg)
    t = _solve(p, False, diag=d2)
    o = O.oracle_solve(p, S)
    check_parity(p, S, g, o)
    assert g.status == t.status
    # the operator differs from the two-pass one only in the grouping of the
    # A^T sums: the first PCG calls take the same iteration counts within the
    # summation-order noise (portfolio is chaotic; fp32 noisier)
    k = min(5, len(dg.pcg_calls), len(d2.pcg_calls))
    band = 2 if dtype == np.float64 else 4
    for a, b in zip(dg.pcg_calls[:k], d2.pcg_calls[:k]):
        assert abs(a["iterations"] - b["iterations"]) <= band


SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, %r)
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
S = Settings(lambda_pcg=0.01)
out = {}
for cls in ("lasso", "svm", "huber"):
    p = G.generate(cls, 6, 1)
    a = solver.solve(p, S, device=0, mode="graph")
    b = solver.solve(p, S, device=0, mode="eager")
    c = solver.solve(p, S, device=0, mode="graph")
    out[cls] = dict(it=[a.iterations, b.iterations, c.iterations],
                    same=bool(np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y)
                              and np.array_equal(a.x, c.x) and a.objective == b.objective),
                    launches=int(a.info["kernel_launches"]))
print(json.dumps(out))
"""


def test_gram_graph_eager_bitwise_and_repeatable():
    env = dict(os.environ, QPCG_GRAM="1", QPCG_PERSIST_MAX_NNZ="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT % ROOT], capture_output=True, text=True,
                       env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    for cls, v in out.items():
        assert v["same"], (cls, v)
        assert len(set(v["it"])) == 1, (cls, v)
