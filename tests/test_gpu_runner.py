"""The runner on the B200 engine: same CSV rows as the reference's
bench/runner.hpp sweep (statuses equal, iteration counts within the parity
band; runtime is the engine's own)."""
import io

import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import runner
from paper_1912_04263_b200.problem import Settings
from test_runner import reference_csv

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


def test_runner_b200_against_reference_sweep():
    classes, scales = ["control", "lasso", "random", "svm"], [1, 3]
    ref = [r.split(",") for r in reference_csv(classes, scales, 3, S).strip().splitlines()[1:]]
    recs = runner.run_benchmark(classes, scales, S, instances_per_size=3, threads=2)
    assert len(recs) == len(ref)
    for r, x in zip(recs, ref):
        assert (r.class_name, str(r.N), str(r.n), str(r.m)) == tuple(x[:4])
        assert r.status == x[4]
        assert abs(r.iterations - int(x[5])) <= 25
        assert r.runtime_seconds > 0
    f = io.StringIO()
    runner.write_csv(recs, f, compare=[runner.BenchRecord(r.class_name, status=r.status,
                                                          runtime_seconds=1.0) for r in recs])
    assert f.getvalue().splitlines()[0] == runner.HEADER + runner.COMPARE_HEADER
