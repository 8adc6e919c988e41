"""Benchmark sweep with the reference's CSV schema (bench/runner.hpp:39-174),
solved by the B200 engine.

Mirrors ``run_benchmark`` / ``write_csv``: instances are generated with the
reference's recipes (bench/generators.hpp, native restatement in
``generators``), solved, and emitted one record per instance plus a "mean"
record per (class, scale) group, in (class, scale, instance) order whatever
the completion order of the worker pool.  ``runtime_seconds`` is the solve
call's own figure (setup through objective, solver.hpp:392/:537; generation
excluded, runner.hpp:14-16).

The solve function is pluggable (``solve_fn(problem, settings) -> outcome``);
the default is the B200 engine.  ``compare`` rows add the same instance solved
by a second function (bench.py --sweep passes the reference CPU solver there),
giving the paper's Figs. 2-3 style GPU-vs-CPU sweep in one CSV.

    python -m paper_1912_04263_b200.runner --classes lasso,svm --scales 1,3,5 \\
        --instances 10 [--threads 4] [--settings '{"lambda_pcg": 0.01}']
"""
from __future__ import annotations

import argparse
import dataclasses
import math
import sys
from concurrent.futures import ThreadPoolExecutor
from typing import Callable, Sequence

from . import generators
from .problem import Settings

HEADER = ("class_name,N,n,m,status,iterations,pcg_total,runtime_seconds,"
          "r_prim_inf,r_dual_inf")  # runner.hpp:52-55
COMPARE_HEADER = ",ref_status,ref_iterations,ref_pcg_total,ref_runtime_seconds,speedup"


@dataclasses.dataclass
class BenchRecord:  # runner.hpp:39-50
    class_name: str
    N: int = 0  # nnz(P upper) + nnz(A)
    n: int = 0
    m: int = 0
    status: str = ""
    iterations: int = 0
    pcg_total: int = 0
    runtime_seconds: float = 0.0
    r_prim_inf: float = 0.0
    r_dual_inf: float = 0.0


def _g10(v: float) -> str:
    """std::ostream << setprecision(10) << v (default float field)."""
    if math.isnan(v):
        return "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return format(v, ".10g")


def to_csv_row(r: BenchRecord) -> str:  # runner.hpp:57-65
    return (f"{r.class_name},{r.N},{r.n},{r.m},{r.status},{r.iterations},{r.pcg_total},"
            f"{_g10(r.runtime_seconds)},{_g10(r.r_prim_inf)},{_g10(r.r_dual_inf)}")


def _llround(x: float) -> int:  # std::llround: half away from zero
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def b200_solve(device: int = 0, mode: str = "graph") -> Callable:
    from . import solver

    def solve(p, s):
        return solver.solve(p, s, device=device, mode=mode)
    return solve


def solve_one(cls: str, scale: int, seed: int, settings: Settings,
              solve_fn: Callable) -> BenchRecord:  # runner.hpp:76-97
    rec = BenchRecord(class_name=cls)
    try:
        p = generators.generate(cls, scale, seed)
        rec.N = int(p.p_upper.nnz) + int(p.a.nnz)
        rec.n, rec.m = p.n, p.m
        out = solve_fn(p, settings)
        rec.status = out.status
        rec.iterations = int(out.iterations)
        rec.pcg_total = int(out.pcg_iterations_total)
        rec.runtime_seconds = float(out.runtime_seconds)
        rec.r_prim_inf = float(out.r_prim_inf)
        rec.r_dual_inf = float(out.r_dual_inf)
    except Exception:  # the reference records any std::exception as "error"
        rec.status = "error"
    return rec


def run_benchmark(classes: Sequence[str], scales: Sequence[int], settings: Settings,
                  instances_per_size: int = 10, base_seed: int = 0, threads: int = 1,
                  solve_fn: Callable | None = None) -> list[BenchRecord]:
    """runner.hpp:99-166: records in (class, scale, instance) order with a
    "mean" record after each group."""
    solve_fn = solve_fn or b200_solve()
    tasks = [(c, s, base_seed + i) for c in classes for s in scales
             for i in range(instances_per_size)]
    if threads <= 1:
        results = [solve_one(c, s, seed, settings, solve_fn) for c, s, seed in tasks]
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            results = list(ex.map(lambda t: solve_one(*t, settings, solve_fn), tasks))
    out: list[BenchRecord] = []
    idx = 0
    k = float(instances_per_size)
    for c in classes:
        for _ in scales:
            mean = BenchRecord(class_name=c, status="mean")
            n_sum = m_sum = big_n_sum = iter_sum = pcg_sum = 0.0
            for _i in range(instances_per_size):
                r = results[idx]
                idx += 1
                out.append(r)
                big_n_sum += float(r.N)
                n_sum += r.n
                m_sum += r.m
                iter_sum += r.iterations
                pcg_sum += float(r.pcg_total)
                mean.runtime_seconds += r.runtime_seconds
                mean.r_prim_inf += r.r_prim_inf
                mean.r_dual_inf += r.r_dual_inf
            mean.N = _llround(big_n_sum / k)
            mean.n = _llround(n_sum / k)
            mean.m = _llround(m_sum / k)
            mean.iterations = _llround(iter_sum / k)
            mean.pcg_total = _llround(pcg_sum / k)
            mean.runtime_seconds /= k
            mean.r_prim_inf /= k
            mean.r_dual_inf /= k
            out.append(mean)
    return out


def write_csv(recs: Sequence[BenchRecord], f=sys.stdout,
              compare: Sequence[BenchRecord] | None = None) -> None:
    """runner.hpp:168-171; with `compare`, each row gains the second solver's
    status / iterations / runtime and the speed-up (its runtime / ours)."""
    f.write(HEADER + (COMPARE_HEADER if compare is not None else "") + "\n")
    for i, r in enumerate(recs):
        row = to_csv_row(r)
        if compare is not None:
            c = compare[i]
            sp = c.runtime_seconds / r.runtime_seconds if r.runtime_seconds > 0 else float("nan")
            row += f",{c.status},{c.iterations},{c.pcg_total},{_g10(c.runtime_seconds)},{_g10(sp)}"
        f.write(row + "\n")


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--classes", default="all")
    ap.add_argument("--scales", default="1,2,3")
    ap.add_argument("--instances", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--settings", default="{}", help="JSON with Settings keys (io.hpp rules)")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--mode", default="graph", choices=["graph", "eager", "persistent"])
    a = ap.parse_args(argv)
    classes = generators.CLASSES if a.classes == "all" else a.classes.split(",")
    scales = [int(v) for v in a.scales.split(",")]
    recs = run_benchmark(classes, scales, Settings.from_json(a.settings), a.instances, a.seed,
                         a.threads, b200_solve(a.device, a.mode))
    write_csv(recs)


if __name__ == "__main__":
    main()
