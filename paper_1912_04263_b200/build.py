"""Build the engine's shared libraries in-tree (they travel with the gpurun snapshot).

    python -m paper_1912_04263_b200.build [--force]

* libqpcg_b200.so : CUDA engine + C-ABI, sm_100a only, --fmad=false (see
                    csrc/common.cuh for why), -lineinfo for ncu source pages.
* libqpcg_gen.so  : host C++ instance generators (counter RNG, parallel) and the
                    reference's text problem format (textio.cpp).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ENGINE_SO = os.path.join(HERE, "libqpcg_b200.so")
GEN_SO = os.path.join(HERE, "libqpcg_gen.so")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "--fmad=false",
              "--extended-lambda", "-std=c++17", "-Xcompiler", "-fPIC",
              f"-I{os.path.join(ROOT, 'include')}"]
# the C-ABI and one translation unit per precision (explicit instantiations of
# Workspace<T> / Sharded<T>), compiled in parallel, linked into one .so
ENGINE_TUS = ["engine.cu", "engine_f64.cu", "engine_f32.cu"]
OBJ_DIR = os.path.join(HERE, "build")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_engine(force: bool = False) -> str:
    deps = glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "qpcg_b200.h"), os.path.join(ROOT, "include", "qpcg_b200_ops.h")]
    if not (force or _stale(ENGINE_SO, deps)):
        return ENGINE_SO
    os.makedirs(OBJ_DIR, exist_ok=True)
    objs, procs = [], []
    for tu in ENGINE_TUS:
        obj = os.path.join(OBJ_DIR, tu.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, "-c", "-o", obj, os.path.join(CSRC, tu)]
        print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    rcs = [p.wait() for p in procs]
    if any(rcs):
        raise subprocess.CalledProcessError(max(rcs), "nvcc")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", ENGINE_SO, *objs]
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return ENGINE_SO


def build_gen(force: bool = False) -> str:
    srcs = [os.path.join(CSRC, f) for f in ("gen.cpp", "textio.cpp")]
    if not os.path.exists(srcs[0]):
        return ""
    if force or _stale(GEN_SO, srcs):
        cmd = ["g++", "-std=c++17", "-O3", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
               "-o", GEN_SO, *srcs]
        print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return GEN_SO


def build(force: bool = False) -> None:
    build_engine(force)
    build_gen(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
