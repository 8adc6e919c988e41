"""Problem instances of the reference's benchmark classes (native, multi-threaded).

Bit-identical to bench::generate (generators.hpp:693-705) and to the explicit
sizes of SURVEY.md §8(d) (checked against oracle/_ref by
tests/test_generators.py).  BASELINE configs:

    config("1")   random n=1000, m=10000 (reference recipe, P 3 nnz/row)
    config("1p")  random n=1000, m=10000, P ~15 % dense (13 nnz/row)
    config("2")   lasso 10^4 features x 10^5 samples, 15 %
    config("3")   huber 10^4 x 10^5, 15 %
    config("4")   svm 10^3 features x 10^6 samples, 15 %
    config("5a")  portfolio N ~ 1e8 (n = 141421 assets, k = 1414 factors)
    config("5b")  control / MPC, gen_control scale 13
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .problem import CsrMatrix, QpProblem

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqpcg_gen.so")
CLASSES = ["control", "equality", "huber", "lasso", "portfolio", "random", "svm"]
KINDS = {"random": 0, "lasso": 1, "huber": 2, "svm": 3, "portfolio": 4, "equality": 5,
         "control": 6}

# name -> (kind, a, b, c) explicit sizes, or ("class", scale)
CONFIGS = {
    "1": ("random", 1000, 10000, 3),
    "1p": ("random", 1000, 10000, 13),
    "2": ("lasso", 10000, 100000, 0),
    "3": ("huber", 10000, 100000, 0),
    "4": ("svm", 1000, 1000000, 0),
    "5a": ("portfolio", 141421, 1414, 0),
    "5b": ("class", "control", 13),
}

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from .build import build_gen
            build_gen()
        lib = C.CDLL(LIB_PATH)
        lib.qgen_class.restype = C.c_void_p
        lib.qgen_class.argtypes = [C.c_int, C.c_uint32, C.c_uint64]
        lib.qgen_explicit.restype = C.c_void_p
        lib.qgen_explicit.argtypes = [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64]
        lib.qgen_dims.argtypes = [C.c_void_p, C.c_void_p]
        lib.qgen_export.argtypes = [C.c_void_p] + [C.c_void_p] * 9
        lib.qgen_free.argtypes = [C.c_void_p]
        lib.qgen_last_error.restype = C.c_char_p
        lib.qgen_target_nnz.restype = C.c_uint64
        lib.qgen_set_threads.argtypes = [C.c_int]
        _lib = lib
    return _lib


def set_threads(t: int) -> None:
    _load().qgen_set_threads(int(t))


def _export(h) -> QpProblem:
    lib = _load()
    if not h:
        raise RuntimeError(lib.qgen_last_error().decode())
    try:
        dims = np.zeros(4, np.uint64)
        lib.qgen_dims(C.c_void_p(h), dims.ctypes.data)
        n, m, nnzp, nnza = (int(v) for v in dims)
        pv, prp, pci = np.empty(nnzp), np.empty(n + 1, np.uint32), np.empty(nnzp, np.uint32)
        av, arp, aci = np.empty(nnza), np.empty(m + 1, np.uint32), np.empty(nnza, np.uint32)
        q, l, u = np.empty(n), np.empty(m), np.empty(m)
        lib.qgen_export(C.c_void_p(h), *[a.ctypes.data for a in (pv, prp, pci, q, av, arp, aci, l, u)])
    finally:
        lib.qgen_free(C.c_void_p(h))
    return QpProblem(CsrMatrix(n, n, pv, prp, pci), q, CsrMatrix(m, n, av, arp, aci), l, u)


def generate(cls: str, scale: int, seed: int = 0, dtype=np.float64) -> QpProblem:
    """bench::generate<T>(BenchSpec{cls, scale, seed})."""
    p = _export(_load().qgen_class(CLASSES.index(cls), scale, seed))
    return p if dtype == np.float64 else p.astype(dtype)


def generate_explicit(kind: str, a: int, b: int, c: int = 0, seed: int = 0,
                      dtype=np.float64) -> QpProblem:
    p = _export(_load().qgen_explicit(KINDS[kind], a, b, c, seed))
    return p if dtype == np.float64 else p.astype(dtype)


def config(name: str, seed: int = 0, dtype=np.float64) -> QpProblem:
    spec = CONFIGS[name]
    if spec[0] == "class":
        return generate(spec[1], spec[2], seed, dtype)
    return generate_explicit(*spec, seed=seed, dtype=dtype)


def target_nnz(scale: int) -> int:
    return int(_load().qgen_target_nnz(scale))
