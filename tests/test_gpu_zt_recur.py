"""z~ and r0's A^T (rho z~) carried through PCG (csrc/admm.cuh zt_pass,
rhs_one) against the reference's per-step z~ = A x~ pass (solver.hpp:359) and
two-column rhs/r0 pass (solver.hpp:351-355, linsys.hpp:218-219), selected per
process by QPCG_ZT_RECUR: the same solve in two processes must give the same
status and iteration count and agree to rounding noise (the carried products
differ from the direct ones in the last bits only; both restart from direct
products after every check iteration)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import json, sys
import numpy as np
sys.path.insert(0, %r)
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings
out = []
for cls, sc in (("lasso", 5), ("huber", 5), ("svm", 4), ("control", 5)):
    for mode in ("graph", "eager"):
        g = solver.solve(G.generate(cls, sc, 0), Settings(lambda_pcg=0.01), device=0, mode=mode)
        out.append([cls, mode, g.status, g.iterations, g.objective, g.x.tolist()])
print(json.dumps(out))
""" % ROOT


def run(flag):
    env = dict(os.environ, QPCG_ZT_RECUR=flag)
    r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_carried_z_tilde_matches_the_per_step_pass():
    import numpy as np
    a, b = run("0"), run("1")
    for (cls, mode, st0, it0, ob0, x0), (_, _, st1, it1, ob1, x1) in zip(a, b):
        assert st0 == st1 and it0 == it1, (cls, mode, it0, it1)
        assert abs(ob0 - ob1) <= 1e-9 * max(1.0, abs(ob0)), (cls, mode, ob0, ob1)
        x0, x1 = np.array(x0), np.array(x1)
        assert np.max(np.abs(x0 - x1)) <= 1e-8 * max(1.0, np.max(np.abs(x0))), cls
    # graph and eager stay bitwise identical with the carried z~
    for i in range(0, len(b), 2):
        assert b[i][3:] == b[i + 1][3:]


@pytest.fixture
def carry_always():
    """The break-even gate keeps the carry off on small problems (one A pass
    costs less than the per-iteration carry there); force it on so the carried
    paths of all three drivers run on every PCG solve."""
    old = os.environ.get("QPCG_ZT_KMAX")
    os.environ["QPCG_ZT_KMAX"] = "1000000"
    yield
    if old is None:
        del os.environ["QPCG_ZT_KMAX"]
    else:
        os.environ["QPCG_ZT_KMAX"] = old


@pytest.mark.parametrize("cls", ["control", "equality", "huber", "lasso", "portfolio", "random",
                                 "svm"])
def test_carried_paths_bitwise_across_drivers_and_parity(cls, carry_always):
    from oracle import oracle as O
    from paper_1912_04263_b200 import generators as G, solver
    from paper_1912_04263_b200.problem import Settings
    from test_gpu_parity import check_parity
    from test_gpu_persistent import graph_only, same
    s = Settings(lambda_pcg=0.01)
    p = G.generate(cls, 5, 1)
    a = solver.solve(p, s, device=0, mode="persistent")
    b = graph_only(p, s)
    c = solver.solve(p, s, device=0, mode="eager")
    same(a, b)
    same(a, c)
    check_parity(p, s, a, O.oracle_solve(p, s))


def test_forced_carry_skips_z_tilde_passes(carry_always):
    """With the carry forced on, the graph launches fewer z~ passes (IF node)."""
    from paper_1912_04263_b200 import generators as G
    from paper_1912_04263_b200.problem import Settings
    from test_gpu_persistent import graph_only
    s = Settings(lambda_pcg=0.01)
    p = G.generate("lasso", 5, 1)
    on = graph_only(p, s)
    os.environ["QPCG_ZT_KMAX"] = "0"  # carry only after PCG solves of 0 iterations
    off = graph_only(p, s)
    assert on.iterations == off.iterations
    assert on.info["kernel_launches"] < off.info["kernel_launches"]
    assert on.info["engine_flags"] & 4  # QPCG_ENGINE_CARRIED_PRODUCTS
