"""bench.py's reference arm end to end on the CPU (config 1: seconds) and the
JSON contract of its line; a name check of the whole script so a refactor
cannot leave the GPU arm calling an undefined helper."""
import ast
import builtins
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def test_reference_arm_line():
    r = subprocess.run([sys.executable, BENCH, "--impl", "reference", "--config", "1",
                        "--steps", "3", "--warmup", "2"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "s" and line["value"] > 0
    assert line["steps"] == 1 and line["requested_steps"] == 3
    assert line["solve"]["status"] == "solved"
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["value"] == line["value"]
    cfg = line["config"]
    for k in ("workload", "config_id", "n", "m", "nnz_A", "settings", "parallelism", "l2", "mode"):
        assert k in cfg


def test_every_called_name_is_defined():
    tree = ast.parse(open(BENCH).read())
    defined = set(dir(builtins))
    for node in ast.walk(tree):
        if isinstance(node, (ast.FunctionDef, ast.ClassDef)):
            defined.add(node.name)
        elif isinstance(node, (ast.Import, ast.ImportFrom)):
            defined.update((a.asname or a.name).split(".")[0] for a in node.names)
        elif isinstance(node, ast.Name) and isinstance(node.ctx, ast.Store):
            defined.add(node.id)
        elif isinstance(node, ast.arg):
            defined.add(node.arg)
    called = {n.func.id for n in ast.walk(tree) if isinstance(n, ast.Call)
              and isinstance(n.func, ast.Name)}
    assert not (called - defined), sorted(called - defined)
