"""The sweep runner reproduces the reference's bench/runner.hpp CSV: same
rows, order, mean records and number formatting (runtime_seconds is a timing
and is compared only for presence)."""
import ctypes as C
import io

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import _abi, generators as G, runner
from paper_1912_04263_b200.problem import Settings

CLASSES = ["lasso", "svm", "random", "equality"]
SCALES = [1, 2]
S = Settings(lambda_pcg=0.01)


def reference_csv(classes, scales, instances, settings):
    lib = O.ref_lib()
    fn = lib.qref_run_benchmark_csv
    fn.restype = C.c_int64
    fn.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64,
                   C.c_uint32, C.c_void_p, C.c_char_p, C.c_size_t]
    cls = (C.c_int * len(classes))(*[G.CLASSES.index(c) for c in classes])
    sc = (C.c_uint32 * len(scales))(*scales)
    st = settings.to_c()
    buf = C.create_string_buffer(1 << 20)
    k = fn(C.cast(cls, C.c_void_p), len(classes), C.cast(sc, C.c_void_p), len(scales), instances,
           0, 1, C.cast(C.pointer(st), C.c_void_p), buf, 1 << 20)
    assert k > 0, lib.qref_last_error()
    return buf.value.decode()


def strip_runtime(csv_text, col=7):
    rows = [r.split(",") for r in csv_text.strip().splitlines()]
    for r in rows[1:]:
        assert r[col] != ""
        r[col] = "<t>"
    return rows


def test_runner_matches_reference_csv():
    ref = reference_csv(CLASSES, SCALES, 3, S)
    recs = runner.run_benchmark(CLASSES, SCALES, S, instances_per_size=3,
                                solve_fn=lambda p, s: O.ref_solve(p, s))
    f = io.StringIO()
    runner.write_csv(recs, f)
    mine = f.getvalue()
    assert mine.splitlines()[0] == ref.splitlines()[0] == runner.HEADER
    a, b = strip_runtime(mine), strip_runtime(ref)
    assert len(a) == len(b) == 1 + len(CLASSES) * len(SCALES) * 4
    assert a == b


def test_runner_threads_keep_order_and_errors_are_records():
    def flaky(p, s):
        if p.n % 2:
            raise ValueError("boom")
        return O.oracle_solve(p, s)
    r1 = runner.run_benchmark(["lasso", "svm"], [1], S, 4, solve_fn=flaky, threads=1)
    r4 = runner.run_benchmark(["lasso", "svm"], [1], S, 4, solve_fn=flaky, threads=4)
    assert [(r.class_name, r.N, r.status, r.iterations) for r in r1] == \
        [(r.class_name, r.N, r.status, r.iterations) for r in r4]
    assert any(r.status == "error" for r in r1) or all(r.n % 2 == 0 for r in r1)
    assert [r.status for r in r1][4] == "mean" and [r.status for r in r1][9] == "mean"


def test_number_format_matches_ostream():
    assert runner._g10(0.1) == "0.1"
    assert runner._g10(1e-05) == "1e-05"
    assert runner._g10(123456.78901234) == "123456.789"
    assert runner._g10(float("inf")) == "inf"
    assert runner._llround(2.5) == 3 and runner._llround(3.5) == 4 and runner._llround(2.4999) == 2
