"""Many small solves on one GPU (solve_batch / sm_budget, SURVEY.md §8(f)
rank 3): capping the persistent driver's SMs and running solves side by side
changes no bit of any outcome."""
import numpy as np
import pytest

from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


def _eq(a, b):
    return (a.status == b.status and a.iterations == b.iterations
            and a.pcg_iterations_total == b.pcg_iterations_total
            and np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and np.array_equal(a.z, b.z))


@pytest.mark.parametrize("budget", [1, 5, 16, 24, 40])
def test_sm_budget_is_bitwise_neutral(budget):
    # block / cluster / grid regimes of the persistent driver
    for cls, scale in (("lasso", 1), ("huber", 3), ("portfolio", 4), ("svm", 5)):
        p = G.generate(cls, scale, 1)
        assert _eq(solver.solve(p, S, device=0, sm_budget=budget), solver.solve(p, S, device=0)), \
            (cls, scale, budget)


def test_solve_batch_matches_individual_solves():
    probs = [G.generate(c, s, seed) for c in ("lasso", "random", "control", "equality")
             for s in (2, 4) for seed in (0, 1)]
    ref = [solver.solve(p, S, device=0) for p in probs]
    for k in (1, 4, 9):
        outs = solver.solve_batch(probs, S, device=0, concurrency=k)
        assert all(_eq(o, r) for o, r in zip(outs, ref)), k
