"""The reference's text problem format and settings JSON (io.hpp), natively.

    read_problem(path, dtype=np.float64) -> QpProblem    load_problem<T>  io.hpp:165-170
    write_problem(path, problem)                           save_problem<T>  io.hpp:158-163
    load_settings(path) -> Settings                        load_settings<T> io.hpp:207-214

The parser and writer live in libqpcg_gen.so (csrc/textio.cpp): files written
by the reference read back bit for bit, files written here are byte-identical
to the reference's, and malformed input fails with the reference's message —
RuntimeError for std::runtime_error (io), ValueError for
std::invalid_argument (validation), the mapping solver.py uses for the engine.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .problem import CsrMatrix, QpProblem, Settings

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libqpcg_gen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from .build import build_gen
            build_gen()
        lib = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        lib.qio_read_problem.restype = vp
        lib.qio_read_problem.argtypes = [C.c_char_p, C.c_int]
        lib.qio_dims.argtypes = [vp, vp]
        lib.qio_export.argtypes = [vp] * 10
        lib.qio_free.argtypes = [vp]
        lib.qio_last_error.restype = C.c_char_p
        lib.qio_last_error_kind.restype = C.c_int
        lib.qio_write_problem.restype = C.c_int
        lib.qio_write_problem.argtypes = [C.c_char_p, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, C.c_uint64, vp, vp, vp, vp, C.c_uint64, vp, vp, vp, vp, vp]
        _lib = lib
    return _lib


def _raise(lib):
    msg = lib.qio_last_error().decode()
    if lib.qio_last_error_kind() == 2:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def read_problem(path: str, dtype=np.float64) -> QpProblem:
    """load_problem<T>: T = float parses with std::stof, double with std::stod."""
    dtype = np.dtype(dtype)
    if dtype not in (np.float64, np.float32):
        raise TypeError("dtype must be float64 or float32")
    lib = _load()
    h = lib.qio_read_problem(os.fsencode(path), int(dtype == np.float32))
    if not h:
        _raise(lib)
    try:
        d = np.zeros(5, np.uint64)
        lib.qio_dims(h, d.ctypes.data)
        n, m, pnnz, annz, acols = (int(v) for v in d)
        pv, pci = np.empty(pnnz), np.empty(pnnz, np.uint32)
        prp = np.empty(n + 1, np.uint32)
        av, aci = np.empty(annz), np.empty(annz, np.uint32)
        arp = np.empty(m + 1, np.uint32)
        q, lo, up = np.empty(n), np.empty(m), np.empty(m)
        lib.qio_export(h, _ptr(pv), _ptr(prp), _ptr(pci), _ptr(q), _ptr(av), _ptr(arp), _ptr(aci),
                       _ptr(lo), _ptr(up))
    finally:
        lib.qio_free(h)
    return QpProblem(CsrMatrix(n, n, pv.astype(dtype), prp, pci), q.astype(dtype),
                     CsrMatrix(m, acols, av.astype(dtype), arp, aci), lo.astype(dtype),
                     up.astype(dtype))


def write_problem(path: str, p: QpProblem) -> None:
    """save_problem<T> with T the problem's dtype (max_digits10: 17 / 9 digits)."""
    lib = _load()
    f32 = p.dtype == np.float32
    w = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731 (exact widening)
    pv, q, av, lo, up = w(p.p_upper.values), w(p.q), w(p.a.values), w(p.l), w(p.u)
    rc = lib.qio_write_problem(
        os.fsencode(path), int(f32), p.p_upper.rows, p.p_upper.cols, p.a.rows, p.a.cols,
        p.p_upper.nnz, _ptr(pv),
        _ptr(p.p_upper.row_ptr), _ptr(p.p_upper.col_indices), _ptr(q), p.a.nnz, _ptr(av),
        _ptr(p.a.row_ptr), _ptr(p.a.col_indices), _ptr(lo), _ptr(up))
    if rc != 0:
        _raise(lib)


def load_settings(path: str) -> Settings:
    """io.hpp:207-214 (+ settings_from_json :175-205 via Settings.from_json)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise RuntimeError(f"io: cannot open {path}") from None
    return Settings.from_json(text)
