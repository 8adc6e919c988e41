"""The reference's text problem format (io.hpp) through textio.py.

Pinned two ways: committed golden outcomes of the reference's own io.hpp
(tests/golden/textio_cases.json and ref_lasso_s1_seed0.txt, made by
tests/golden/make_textio_golden.py with oracle/_ref/ref_io) and, where
oracle/_ref/ref_io is built, live comparisons on generated instances of every
class.  CPU only."""
import hashlib
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1912_04263_b200 import generators as G, textio
from paper_1912_04263_b200.problem import Settings

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from textio_cases import TEXTIO_CASES  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "textio_cases.json")))
REF_IO = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "ref_io")
need_ref = pytest.mark.skipif(not os.path.exists(REF_IO), reason="oracle/_ref/ref_io not built")


def _same(p, g):
    for f in ("values", "row_ptr", "col_indices"):
        assert np.array_equal(getattr(p.p_upper, f), getattr(g.p_upper, f))
        assert np.array_equal(getattr(p.a, f), getattr(g.a, f))
    for v in "qlu":
        assert np.array_equal(getattr(p, v), getattr(g, v))
    assert (p.p_upper.rows, p.p_upper.cols, p.a.rows, p.a.cols) == \
        (g.p_upper.rows, g.p_upper.cols, g.a.rows, g.a.cols)


def _sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("name", sorted(TEXTIO_CASES))
def test_case_matches_reference(tmp_path, name, prec):
    src = tmp_path / "in.txt"
    src.write_bytes(TEXTIO_CASES[name].encode())
    want = GOLD[name][prec]
    dtype = np.float32 if prec == "f32" else np.float64
    if "error" in want:
        exc = ValueError if want["error"] == "invalid" else RuntimeError
        with pytest.raises(exc) as e:
            textio.read_problem(str(src), dtype)
        assert str(e.value) == want["message"]
        return
    p = textio.read_problem(str(src), dtype)
    assert p.dtype == dtype
    out = tmp_path / "out.txt"
    textio.write_problem(str(out), p)
    assert _sha(out) == want["sha256"]


def test_golden_reference_file_reads_as_generated(tmp_path):
    path = os.path.join(HERE, "golden", "ref_lasso_s1_seed0.txt")
    p = textio.read_problem(path)
    _same(p, G.generate("lasso", 1, 0))
    out = tmp_path / "out.txt"
    textio.write_problem(str(out), p)
    assert out.read_bytes() == open(path, "rb").read()


@need_ref
@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("cls", G.CLASSES)
def test_reference_written_instances(tmp_path, cls, prec):
    """save_problem of the reference reads back bit for bit; ours writes the
    same bytes (every class, both precisions)."""
    ref = tmp_path / "ref.txt"
    code = {"control": 0, "equality": 1, "huber": 2, "lasso": 3, "portfolio": 4, "random": 5,
            "svm": 6}[cls]
    subprocess.run([REF_IO, "gen", str(code), "3", "11", str(ref)] + (["f32"] if prec == "f32" else []),
                   check=True)
    dtype = np.float32 if prec == "f32" else np.float64
    p = textio.read_problem(str(ref), dtype)
    _same(p, G.generate(cls, 3, 11, dtype=dtype))
    out = tmp_path / "ours.txt"
    textio.write_problem(str(out), p)
    assert out.read_bytes() == ref.read_bytes()


@need_ref
def test_parallel_block_path_matches_sequential(tmp_path):
    """The parallel "row col value" line parser (forced on small blocks with
    QPCG_IO_PAR_MIN) gives the same problem and the same errors as the
    sequential token reader."""
    ref = tmp_path / "ref.txt"
    subprocess.run([REF_IO, "gen", "3", "5", "2", str(ref)], check=True)
    for name in ("ok_base", "ok_crlf", "ok_two_entries_per_line", "err_alpha_value",
                 "err_unsorted", "err_subnormal_value"):
        (tmp_path / f"{name}.txt").write_bytes(TEXTIO_CASES[name].encode())
    prog = f"""
import sys, hashlib
sys.path.insert(0, {os.path.dirname(HERE)!r})
from paper_1912_04263_b200 import textio
for f in sys.argv[1:]:
    try:
        p = textio.read_problem(f)
        textio.write_problem(f + '.out', p)
        print(f, hashlib.sha256(open(f + '.out', 'rb').read()).hexdigest())
    except Exception as e:
        print(f, type(e).__name__, e)
"""
    files = [str(ref)] + [str(tmp_path / f"{n}.txt") for n in
                          ("ok_base", "ok_crlf", "ok_two_entries_per_line", "err_alpha_value",
                           "err_unsorted", "err_subnormal_value")]
    outs = []
    for par_min in ("1", str(1 << 40)):
        env = dict(os.environ, QPCG_IO_PAR_MIN=par_min)
        r = subprocess.run([sys.executable, "-c", prog, *files], env=env, capture_output=True,
                           text=True, check=True)
        outs.append(r.stdout)
    assert outs[0] == outs[1]
    assert _sha(str(ref) + ".out") == _sha(str(ref))


@need_ref
def test_settings_json_matches_reference(tmp_path):
    cfg = {"alpha": 1.4, "sigma": 1e-5, "lambda_pcg": 0.01, "max_admm_iter": 1234,
           "check_interval": 3, "scaling_enabled": False, "eps_equil": 0.002,
           "precision_note": "fp64"}
    path = tmp_path / "s.json"
    path.write_text(json.dumps(cfg))
    r = subprocess.run([REF_IO, "settings", str(path)], capture_output=True, text=True, check=True)
    ref = dict(line.split("=", 1) for line in r.stdout.split())
    s = textio.load_settings(str(path))
    for k, v in ref.items():
        got = getattr(s, k)
        assert (float(got) if not isinstance(got, bool) else int(got)) == float(v), k
    bad = tmp_path / "bad.json"
    bad.write_text('{"alhpa": 1.0}')
    r = subprocess.run([REF_IO, "settings", str(bad)], capture_output=True, text=True)
    assert r.returncode == 3
    with pytest.raises(RuntimeError) as e:
        textio.load_settings(str(bad))
    assert r.stdout.strip() == f"ERR runtime {e.value}"


def test_missing_file_message(tmp_path):
    with pytest.raises(RuntimeError, match="io: cannot open"):
        textio.read_problem(str(tmp_path / "nope.txt"))
    with pytest.raises(RuntimeError, match="io: cannot open"):
        textio.load_settings(str(tmp_path / "nope.json"))


def test_round_trip_engine_generated(tmp_path):
    """write -> read is the identity on a generated instance (both precisions)."""
    for dtype in (np.float64, np.float32):
        g = G.generate("portfolio", 2, 5, dtype=dtype)
        path = tmp_path / "p.txt"
        textio.write_problem(str(path), g)
        _same(textio.read_problem(str(path), dtype), g)
