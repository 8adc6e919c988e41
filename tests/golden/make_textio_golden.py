"""Golden outcomes of the reference's io.hpp for tests/test_textio.py.

Runs oracle/_ref/ref_io (the unmodified reference io.hpp, built by
oracle/Makefile) on every case of TEXTIO_CASES and records, per precision,
either the error it throws (kind + message) or the sha256 of the file it
writes back (load_problem + save_problem).  Also writes
ref_lasso_s1_seed0.txt: the reference's save_problem of generate(lasso, 1, 0).

    python tests/golden/make_textio_golden.py
"""
import hashlib
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from textio_cases import TEXTIO_CASES  # noqa: E402

REF_IO = os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle", "_ref", "ref_io")


def ref_outcome(text: str, f32: bool) -> dict:
    with tempfile.TemporaryDirectory() as d:
        src, dst = os.path.join(d, "in.txt"), os.path.join(d, "out.txt")
        with open(src, "w", newline="") as f:
            f.write(text)
        args = [REF_IO, "rt", src, dst] + (["f32"] if f32 else [])
        r = subprocess.run(args, capture_output=True, text=True)
        if r.returncode == 3:
            _, kind, msg = r.stdout.rstrip("\n").split(" ", 2)
            return {"error": kind, "message": msg}
        r.check_returncode()
        return {"sha256": hashlib.sha256(open(dst, "rb").read()).hexdigest()}


def main():
    out = {}
    for name, text in TEXTIO_CASES.items():
        out[name] = {"f64": ref_outcome(text, False), "f32": ref_outcome(text, True)}
    with open(os.path.join(HERE, "textio_cases.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    subprocess.run([REF_IO, "gen", "3", "1", "0", os.path.join(HERE, "ref_lasso_s1_seed0.txt")],
                   check=True)


if __name__ == "__main__":
    main()
