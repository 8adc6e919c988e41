"""ctypes mirror of include/qpcg_b200.h (the engine's C-ABI).

Struct layouts are kept field-for-field identical to the header; the
``test_abi`` CPU test checks sizes/offsets against a compiled probe.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

QPCG_OK = 0
QPCG_ERR_INVALID = 1
QPCG_ERR_NOT_PD = 2
QPCG_ERR_CUDA = 3
QPCG_ERR_NCCL = 4
QPCG_ERR_OOM = 5
QPCG_ERR_RUNTIME = 6

STATUS_NAMES = {0: "solved", 1: "primal_infeasible", 2: "dual_infeasible", 3: "max_iter_reached"}

MEM_HOST = 0
MEM_DEVICE = 1
MODE_GRAPH = 0
MODE_EAGER = 1
MODE_PERSISTENT = 2

u32p = C.POINTER(C.c_uint32)


class CsrF64(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("nnz", C.c_uint32),
                ("values", C.c_void_p), ("row_ptr", C.c_void_p), ("col_indices", C.c_void_p)]


CsrF32 = CsrF64  # identical layout (pointer-typed as void*)


class Settings(C.Structure):
    _fields_ = [("alpha", C.c_double), ("sigma", C.c_double), ("rho_bar_init", C.c_double),
                ("eps_abs", C.c_double), ("eps_rel", C.c_double), ("eps_pinf", C.c_double),
                ("eps_dinf", C.c_double), ("max_admm_iter", C.c_uint32),
                ("check_interval", C.c_uint32), ("rho_update_interval", C.c_uint32),
                ("scaling_enabled", C.c_uint32), ("lambda_pcg", C.c_double),
                ("eps_pcg_min", C.c_double), ("eps_equil", C.c_double),
                ("equil_max_passes", C.c_uint32), ("reserved_", C.c_uint32)]


class Info(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_uint32),
                ("pcg_iterations_total", C.c_uint64), ("objective", C.c_double),
                ("r_prim_inf", C.c_double), ("r_dual_inf", C.c_double),
                ("runtime_seconds", C.c_double), ("equil_passes", C.c_uint32),
                ("rho_update_count", C.c_uint32), ("equil_residual", C.c_double),
                ("rho_final", C.c_double), ("certificate_valid", C.c_uint32),
                ("n", C.c_uint32), ("m", C.c_uint32), ("engine_flags", C.c_uint32),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("h2d_seconds", C.c_double), ("d2h_seconds", C.c_double),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("kernel_launches", C.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved_"}


class PcgCall(C.Structure):
    _fields_ = [("admm_iter", C.c_uint32), ("iterations", C.c_uint32), ("eps", C.c_double),
                ("r_prim_scaled_inf", C.c_double), ("r_dual_scaled_inf", C.c_double),
                ("converged", C.c_int32), ("reserved_", C.c_int32)]


class RhoUpdate(C.Structure):
    _fields_ = [("admm_iter", C.c_uint32), ("reserved_", C.c_uint32),
                ("rho_before", C.c_double), ("rho_after", C.c_double)]


class Options(C.Structure):
    _fields_ = [("device", C.c_int32), ("input_memory", C.c_int32), ("mode", C.c_int32),
                ("record_diagnostics", C.c_int32), ("virtual_shards", C.c_int32),
                ("nccl_rank", C.c_int32), ("nccl_ranks", C.c_int32), ("sm_budget", C.c_int32),
                ("stream", C.c_void_p), ("nccl_id", C.c_void_p), ("transport", C.c_int32),
                ("reserved2_", C.c_int32), ("rendezvous_dir", C.c_char_p),
                ("on_iteration", C.c_void_p), ("on_iteration_user", C.c_void_p)]


# qpcg_iteration_cb: (user, iter, x, z, y, l, u, n, m)
ITERATION_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32)


TRANSPORT_NCCL = 0
TRANSPORT_PEER = 1


NCCL_ID_BYTES = 128


def default_settings() -> Settings:
    """settings.hpp:25-42 defaults."""
    s = Settings()
    s.alpha, s.sigma, s.rho_bar_init = 1.6, 1e-6, 0.1
    s.eps_abs, s.eps_rel, s.eps_pinf, s.eps_dinf = 1e-3, 1e-3, 1e-4, 1e-4
    s.max_admm_iter, s.check_interval, s.rho_update_interval = 50000, 5, 10
    s.scaling_enabled = 1
    s.lambda_pcg, s.eps_pcg_min = 0.15, 1e-7
    s.eps_equil, s.equil_max_passes = 1e-3, 10
    return s


def ptr(a: np.ndarray | None) -> C.c_void_p | None:
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "arrays crossing the ABI must be contiguous"
    return C.c_void_p(a.ctypes.data)


def csr_view(values: np.ndarray, row_ptr: np.ndarray, col_indices: np.ndarray,
             rows: int, cols: int) -> CsrF64:
    v = CsrF64()
    v.rows, v.cols, v.nnz = rows, cols, int(values.shape[0])
    v.values, v.row_ptr, v.col_indices = ptr(values), ptr(row_ptr), ptr(col_indices)
    v._keep = (values, row_ptr, col_indices)  # keep arrays alive with the view
    return v


REPO_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
