"""The C++ drop-in (include/qpcg_b200_adapter.hpp) called from a program built
against the reference's own headers (oracle/_ref/adapter_check)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.gpu
def test_adapter_runs_against_reference_types():
    assert os.path.exists(EXE), "build with make -C oracle adapter (needs /root/reference)"
    out = subprocess.run([EXE, "3"], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count(" OK") == 8  # 7 classes + the on_iteration check
    assert "MISMATCH" not in out.stdout
    assert "invalid_argument" in out.stdout


def test_adapter_binary_links_engine():
    if not os.path.exists(EXE):
        pytest.skip("adapter_check not built (reference headers absent)")
    ldd = subprocess.run(["ldd", EXE], capture_output=True, text=True).stdout
    assert "libqpcg_b200.so" in ldd and "not found" not in ldd
