"""End-to-end parity of the B200 engine with the oracle (SURVEY.md §8(c)
protocol): same status; both solutions pass an independent KKT check on the
ORIGINAL data; objective and x within 1e-3 relative OR within 2x the oracle's
own reorder noise (oracle on the row-reversed twin); iteration counts reported."""
import dataclasses
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings, SolveDiagnostics
from _util import kat_problems, kkt_ok, rel, reversed_twin, xrel

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_outputs.json")))


def check_parity(p, s, g, o, tol=1e-3):
    assert g.status == o.status, (g.status, o.status)
    if o.status == "solved":
        slack = 1.0 if p.dtype == np.float64 else 2.0
        assert kkt_ok(p, g, s, slack), "engine solution fails the KKT re-check on original data"
        assert kkt_ok(p, o, s, slack)
        ro, rx = rel(g.objective, o.objective), xrel(g.x, o.x)
        if ro > tol or rx > tol:
            tw = O.oracle_solve(reversed_twin(p), s)  # oracle's own reorder noise
            assert tw.status == o.status
            no, nx = rel(tw.objective, o.objective), xrel(tw.x, o.x)
            if ro <= max(tol, 2 * no) and rx <= max(tol, 2 * nx):
                return
            # classes whose eps=1e-3 answer is chaotic
            # (portfolio, huber; F3) are compared again at eps = 1e-5, where the
            # 1e-3 objective and solution criteria apply.
            s5 = dataclasses.replace(s, eps_abs=1e-5, eps_rel=1e-5, max_admm_iter=20000)
            g5, o5 = solver.solve(p, s5, device=0), O.oracle_solve(p, s5)
            assert g5.status == o5.status, (g5.status, o5.status, ro, no, rx, nx)
            if o5.status == "solved":
                ro5, rx5 = rel(g5.objective, o5.objective), xrel(g5.x, o5.x)
                if ro5 > tol or rx5 > tol:  # the oracle's own noise at eps = 1e-5
                    t5 = O.oracle_solve(reversed_twin(p), s5)
                    no5, nx5 = rel(t5.objective, o5.objective), xrel(t5.x, o5.x)
                    assert ro5 <= max(tol, 2 * no5), (ro5, no5, ro, no)
                    assert rx5 <= max(tol, 2 * nx5), (rx5, nx5, rx, nx)
    elif o.status in ("primal_infeasible", "dual_infeasible"):
        assert g.objective == o.objective
        assert np.allclose(g.certificate, o.certificate, atol=1e-6)


@pytest.mark.parametrize("cls", G.CLASSES)
@pytest.mark.parametrize("scale", [1, 3, 5, 7])
def test_classes_f64(cls, scale):
    for seed in (0, 1):
        p = G.generate(cls, scale, seed)
        g = solver.solve(p, S, device=0)
        o = O.oracle_solve(p, S)
        check_parity(p, S, g, o)
        assert abs(g.iterations - o.iterations) <= 50  # reported band; parity gate is above


@pytest.mark.parametrize("cls", G.CLASSES)
@pytest.mark.parametrize("scale", [3, 5, 7])
def test_classes_f32(cls, scale):
    """fp32 engine against the fp32 oracle (SPEC acceptance 10; fp32 is
    compared with fp32) under the same protocol as fp64:
    objective and x within 1e-3, or within 2x the fp32 oracle's reorder noise,
    KKT re-check on the original data."""
    p = G.generate(cls, scale, 0).astype(np.float32)
    g = solver.solve(p, S, device=0)
    o = O.oracle_solve(p, S)
    check_parity(p, S, g, o)


@pytest.mark.parametrize("cls", ["lasso", "svm", "random", "control"])
def test_default_settings_status_match(cls):
    p = G.generate(cls, 4, 0)
    # random converges near 2000 iterations, and its count moves by ~25 % under
    # a mere reordering of the same instance (oracle: 1825, reversed twin 1635;
    # seed 1: 2340 vs 1775), so a 2000 cap sits inside its own noise band: it
    # runs to the reference's default cap (settings.hpp:33)
    s = Settings(max_admm_iter=50000 if cls == "random" else 2000)
    g = solver.solve(p, s, device=0)
    o = O.oracle_solve(p, s)
    assert g.status == o.status


@pytest.mark.parametrize("name", list(kat_problems()))
def test_kat_solves(name):
    p = kat_problems()[name]
    g = solver.solve(p, Settings(), device=0)
    gg = GOLD["solves"][name]
    assert g.status == gg["status"]
    assert g.iterations == gg["iterations"]
    assert np.allclose(g.x, gg["x"], rtol=1e-6, atol=1e-9)
    if gg["certificate"]:
        assert np.allclose(g.certificate, gg["certificate"], atol=1e-12)
        assert g.objective == gg["objective"]


@pytest.mark.parametrize("cfg", ["1", "1p"])
def test_config1(cfg):
    p = G.config(cfg)
    g = solver.solve(p, S, device=0)
    o = O.oracle_solve(p, S)
    check_parity(p, S, g, o)


def test_graph_and_eager_are_bitwise_identical():
    p = G.generate("huber", 5, 1)
    a = solver.solve(p, S, device=0, mode="graph")
    b = solver.solve(p, S, device=0, mode="eager")
    assert a.iterations == b.iterations and a.pcg_iterations_total == b.pcg_iterations_total
    assert np.array_equal(a.x, b.x) and np.array_equal(a.y, b.y) and a.objective == b.objective


def test_run_to_run_determinism():
    p = G.generate("portfolio", 5, 0)
    a = solver.solve(p, S, device=0)
    b = solver.solve(p, S, device=0)
    assert np.array_equal(a.x, b.x) and a.iterations == b.iterations


def test_cadence_matches_reference():
    """SPEC acceptance 7: checks every 5, rho every 10, eps from the last residuals."""
    p = G.generate("lasso", 4, 0)
    dg, do = SolveDiagnostics(), SolveDiagnostics()
    g = solver.solve(p, S, diag=dg, device=0)
    o = O.oracle_solve(p, S, diag=do)
    assert dg.check_iterations == list(range(5, g.iterations + 1, 5))
    assert [r["admm_iter"] for r in dg.rho_updates] == \
        [i for i in range(10, g.iterations + 1, 10) if i < g.iterations or g.status != "solved"]
    for c in dg.pcg_calls:
        want = max(0.01 * np.sqrt(c["r_prim_scaled_inf"] * c["r_dual_scaled_inf"]), 1e-7)
        assert c["eps"] == pytest.approx(want, rel=1e-15, abs=0)
    k = min(len(dg.pcg_calls), len(do.pcg_calls), 10)
    assert [c["iterations"] for c in dg.pcg_calls[:k]] == [c["iterations"] for c in do.pcg_calls[:k]]


GOLD_CONFIGS = sorted(f[len("config"):-len("_reference_solve.json")]
                      for f in os.listdir(os.path.join(os.path.dirname(__file__), "golden"))
                      if f.startswith("config") and f.endswith("_reference_solve.json"))


@pytest.mark.parametrize("cfg", GOLD_CONFIGS)
def test_full_size_config_against_reference_run(cfg):
    """BASELINE configs at full size (1.0e8-1.5e8 nnz) against the reference's own
    completed solve of the identical instance (tests/golden/config*_reference_solve.json,
    produced by scripts/ref_solve_config.py: minutes on one CPU core each; the
    _f32 anchors are the reference instantiated with T = float)."""
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                      f"config{cfg}_reference_solve.json")))
    f32 = cfg.endswith("_f32")
    p = G.config(cfg[:-4] if f32 else cfg, dtype=np.float32 if f32 else np.float64)
    s = Settings(lambda_pcg=ref["lambda_pcg"])
    g = solver.solve(p, s, device=0)
    assert g.status == ref["status"] == "solved"
    xs = g.x[::ref["x_sample_stride"]].astype(np.float64)
    xdiff = np.max(np.abs(xs - np.array(ref["x_sample"]))) / max(1.0, ref["x_inf"])
    # north-star tolerance (objective and x within 1e-3), widened to 2x the
    # reference's own reorder noise on this instance where it was measured
    # (scripts/ref_noise_config.py: the reference on the row-reversed twin)
    tol_o = max(1e-3, 2 * ref.get("noise_rel_obj", 0.0))
    tol_x = max(1e-3, 2 * ref.get("noise_x", 0.0))
    print(f"config {cfg}: iterations {g.iterations}/{g.pcg_iterations_total} vs reference "
          f"{ref['iterations']}/{ref['pcg_iterations_total']}, objective rel "
          f"{rel(g.objective, ref['objective']):.2e}, x {xdiff:.2e} (tolerances {tol_o:.1e}, "
          f"{tol_x:.1e})")
    if f32 or cfg == "5a":  # fp32, and portfolio (chaotic at eps = 1e-3)
        assert rel(g.objective, ref["objective"]) < tol_o
        assert xdiff <= tol_x
        assert kkt_ok(p, g, s, 2.0 if f32 else 1.0)
        if not f32:
            assert abs(g.iterations - ref["iterations"]) <= 5
        return
    assert abs(g.iterations - ref["iterations"]) <= 5
    assert rel(g.objective, ref["objective"]) < 1e-6
    assert xdiff <= 1e-4
    assert kkt_ok(p, g, s)


DEFAULT_CONFIGS = sorted(f[len("config"):-len("_reference_defaults.json")]
                         for f in os.listdir(os.path.join(os.path.dirname(__file__), "golden"))
                         if f.startswith("config") and f.endswith("_reference_defaults.json"))


@pytest.mark.parametrize("cfg", DEFAULT_CONFIGS)
def test_full_size_defaults_against_reference(cfg):
    """every config also at PURE DEFAULT settings (lambda_pcg =
    0.15, where the reference diverges), against the reference's own
    run of the identical full-size instance with the loop capped
    (tests/golden/config*_reference_defaults.json, scripts/ref_defaults_trajectory.py):
    same status and iteration count, the same PCG iteration counts for the
    first calls, the same adaptive tolerances until the trajectory turns
    chaotic."""
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                      f"config{cfg}_reference_defaults.json")))
    p = G.config(cfg)
    s = Settings(max_admm_iter=ref["max_admm_iter"])
    d = SolveDiagnostics()
    g = solver.solve(p, s, device=0, diag=d)
    assert g.status == ref["status"]
    assert g.iterations == ref["iterations"]
    rc = ref["pcg_calls"]
    k = min(len(rc), len(d.pcg_calls), 10)
    # the first tolerance comes from the initial residuals (bit-exact setup);
    # the PCG iteration counts agree exactly except for portfolio, whose
    # ~250-iteration solves at the 1e-7 tolerance floor move by a few
    # iterations under reordering (its own reorder noise on this
    # instance is 5e-3 in the objective): a 5 % band there
    assert d.pcg_calls[0]["eps"] == pytest.approx(rc[0]["eps"], rel=1e-9)
    for a, b in zip(d.pcg_calls[:k], rc[:k]):
        band = 0 if cfg != "5a" else max(3, int(0.05 * b["iterations"]))
        assert abs(a["iterations"] - b["iterations"]) <= band, (a, b)
    for a, b in zip(d.pcg_calls[1:3], rc[1:3]):
        assert a["eps"] == pytest.approx(b["eps"], rel=1e-6 if cfg != "5a" else 1e-2)


def test_portfolio_scale8_eps1e5():
    """SURVEY.md §8(c) step 4 at a larger portfolio: at eps = 1e-5 the
    chaotic class is held to the 1e-3 objective and x criteria against the oracle
    (tests/golden/portfolio8_eps1e-5.json, tests/golden/make_portfolio8.py), widened
    only to 2x the oracle's own reorder noise at that tolerance."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                       "portfolio8_eps1e-5.json")))
    p = G.generate("portfolio", 8, 0)
    s = Settings(lambda_pcg=0.01, eps_abs=1e-5, eps_rel=1e-5, max_admm_iter=20000)
    g = solver.solve(p, s, device=0)
    assert g.status == gold["status"] == "solved"
    ro = rel(g.objective, gold["objective"])
    rx = xrel(g.x, np.array(gold["x"]))
    print(f"portfolio 8 @1e-5: iterations {g.iterations} vs {gold['iterations']}, objective {ro:.2e}, "
          f"x {rx:.2e} (oracle twin noise {gold['noise_rel_obj']:.2e}, {gold['noise_x']:.2e})")
    assert ro <= max(1e-3, 2 * gold["noise_rel_obj"])
    assert rx <= max(1e-3, 2 * gold["noise_x"])
    assert kkt_ok(p, g, s)
