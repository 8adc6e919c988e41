"""Host-side mirror of the reference's interface types.

* ``CsrMatrix``   <- sparse.hpp:47-56   (uint32 row_ptr / col_indices)
* ``QpProblem``   <- problem.hpp:34-44  (P upper-triangular, q, A, l, u)
* ``Settings``    <- settings.hpp:25-42 (same field names and defaults)
* ``WarmStart``   <- solver.hpp:96-101
* ``SolveOutcome``<- solver.hpp:75-94
* ``SolveDiagnostics`` <- solver.hpp:148-167
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import _abi


class NotPositiveDefiniteError(RuntimeError):
    """qpcg::NotPositiveDefiniteError (types.hpp:35-39)."""


@dataclass
class CsrMatrix:
    rows: int
    cols: int
    values: np.ndarray
    row_ptr: np.ndarray
    col_indices: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.uint32)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.uint32)
        self.values = np.ascontiguousarray(self.values)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def astype(self, dtype) -> "CsrMatrix":
        return CsrMatrix(self.rows, self.cols, self.values.astype(dtype), self.row_ptr,
                         self.col_indices)

    def view(self) -> _abi.CsrF64:
        return _abi.csr_view(self.values, self.row_ptr, self.col_indices, self.rows, self.cols)

    def checked(self, dtype) -> "CsrMatrix":
        """The array-length rules of validate(CsrMatrix) (sparse.hpp:100-106)
        that the C-ABI cannot see (it receives rows / nnz only), with every
        array coerced to its C type right before a call."""
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.uint32)
        ci = np.ascontiguousarray(self.col_indices, dtype=np.uint32)
        v = np.ascontiguousarray(self.values, dtype=dtype)
        if rp.ndim != 1 or rp.shape[0] != int(self.rows) + 1:
            raise ValueError("csr: row_ptr must have rows + 1 entries")
        if ci.ndim != 1 or v.ndim != 1 or ci.shape[0] != v.shape[0]:
            raise ValueError("csr: col_indices/value length mismatch")
        return CsrMatrix(int(self.rows), int(self.cols), v, rp, ci)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values, self.col_indices.astype(np.int64),
                              self.row_ptr.astype(np.int64)), shape=(self.rows, self.cols))

    @staticmethod
    def from_dense(d: np.ndarray, dtype=np.float64) -> "CsrMatrix":
        d = np.asarray(d)
        rows, cols = d.shape
        rp, ci, vals = [0], [], []
        for r in range(rows):
            for c in range(cols):
                if d[r, c] != 0:
                    ci.append(c)
                    vals.append(d[r, c])
            rp.append(len(ci))
        return CsrMatrix(rows, cols, np.array(vals, dtype=dtype), np.array(rp, np.uint32),
                         np.array(ci, np.uint32))


@dataclass
class QpProblem:
    p_upper: CsrMatrix
    q: np.ndarray
    a: CsrMatrix
    l: np.ndarray
    u: np.ndarray

    def __post_init__(self):
        dt = self.p_upper.values.dtype
        self.q = np.ascontiguousarray(self.q, dtype=dt)
        self.l = np.ascontiguousarray(self.l, dtype=dt)
        self.u = np.ascontiguousarray(self.u, dtype=dt)

    @property
    def dtype(self):
        return self.p_upper.values.dtype

    def num_vars(self) -> int:
        return self.p_upper.rows

    def num_constraints(self) -> int:
        return self.a.rows

    @property
    def n(self) -> int:
        return self.p_upper.rows

    @property
    def m(self) -> int:
        return self.a.rows

    def astype(self, dtype) -> "QpProblem":
        """generators.hpp:297-327 cast_problem: elementwise static_cast."""
        return QpProblem(self.p_upper.astype(dtype), self.q.astype(dtype), self.a.astype(dtype),
                         self.l.astype(dtype), self.u.astype(dtype))

    def nnz_total(self) -> int:
        """runner.hpp:81  N = nnz(P upper) + nnz(A)."""
        return self.p_upper.nnz + self.a.nnz

    def checked(self) -> "QpProblem":
        """A copy (views where possible) whose arrays all have the problem's
        dtype and whose lengths satisfy problem.hpp:47-70 / sparse.hpp:100-106,
        in the reference's order, so that the C-ABI (which receives n, m and
        nnz only) never reads past a caller's buffer.  The remaining rules
        (values, bounds, structure) are the engine's and raise the same
        messages there."""
        dt = self.dtype
        if dt not in (np.float64, np.float32):
            raise TypeError(f"unsupported dtype {dt}")
        P = self.p_upper.checked(dt)
        A = self.a.checked(dt)
        q = np.ascontiguousarray(self.q, dtype=dt)
        l = np.ascontiguousarray(self.l, dtype=dt)
        u = np.ascontiguousarray(self.u, dtype=dt)
        if P.rows == P.cols and P.rows > 0 and A.cols == P.cols:
            if q.ndim != 1 or q.shape[0] != P.rows:
                raise ValueError("problem: q length must equal n")
            if l.ndim != 1 or u.ndim != 1 or l.shape[0] != A.rows or u.shape[0] != A.rows:
                raise ValueError("problem: bound lengths must equal m")
        else:  # the engine reports the shape error; keep its reads in bounds
            q = np.resize(q, max(P.rows, 1)).astype(dt)
            l = np.resize(l, max(A.rows, 1)).astype(dt)
            u = np.resize(u, max(A.rows, 1)).astype(dt)
        return QpProblem(P, q, A, l, u)


@dataclass
class Settings:
    alpha: float = 1.6
    sigma: float = 1e-6
    rho_bar_init: float = 0.1
    eps_abs: float = 1e-3
    eps_rel: float = 1e-3
    eps_pinf: float = 1e-4
    eps_dinf: float = 1e-4
    max_admm_iter: int = 50000
    check_interval: int = 5
    rho_update_interval: int = 10
    lambda_pcg: float = 0.15
    eps_pcg_min: float = 1e-7
    scaling_enabled: bool = True
    eps_equil: float = 1e-3
    equil_max_passes: int = 10
    precision_note: str = ""

    _KEYS = ("alpha", "sigma", "rho_bar_init", "eps_abs", "eps_rel", "eps_pinf", "eps_dinf",
             "max_admm_iter", "check_interval", "rho_update_interval", "lambda_pcg",
             "eps_pcg_min", "scaling_enabled", "eps_equil", "equil_max_passes", "precision_note")

    def to_c(self) -> _abi.Settings:
        s = _abi.Settings()
        for f in dataclasses.fields(self):
            if f.name == "precision_note":
                continue
            v = getattr(self, f.name)
            setattr(s, f.name, int(v) if f.name in ("max_admm_iter", "check_interval",
                                                   "rho_update_interval", "equil_max_passes",
                                                   "scaling_enabled") else float(v))
        return s

    _FLOATS = ("alpha", "sigma", "rho_bar_init", "eps_abs", "eps_rel", "eps_pinf", "eps_dinf",
               "lambda_pcg", "eps_pcg_min", "eps_equil")
    _INDICES = ("max_admm_iter", "check_interval", "rho_update_interval", "equil_max_passes")

    def validate(self) -> "Settings":
        """settings.hpp:44-75 (qpcg_validate_settings): ValueError with the
        reference's message."""
        import ctypes as C
        from .solver import load_library
        msg = C.create_string_buffer(256)
        if load_library().qpcg_validate_settings(C.byref(self.to_c()), msg, 256) != _abi.QPCG_OK:
            raise ValueError(msg.value.decode())
        return self

    @staticmethod
    def _json_type(v) -> str:
        if v is None:
            return "null"
        if isinstance(v, bool):
            return "boolean"
        if isinstance(v, (int, float)):
            return "number"
        if isinstance(v, str):
            return "string"
        return "array" if isinstance(v, list) else "object"

    @classmethod
    def from_json(cls, obj) -> "Settings":
        """io.hpp:175-205 settings_from_json: flat keys, an unknown key is an
        error, each value converted as nlohmann's get<T> / get<index_t> /
        get<bool> / get<std::string> does (a wrong JSON type raises its
        type_error text), then validate(s) (:203)."""
        import json
        if isinstance(obj, (str, bytes)):
            obj = json.loads(obj)
        s = cls()
        for k, v in obj.items():
            if k not in cls._KEYS:
                raise RuntimeError(f"settings: unknown key '{k}'")
            t = cls._json_type(v)
            if k in cls._FLOATS or k in cls._INDICES:
                if t != "number":
                    raise RuntimeError(f"[json.exception.type_error.302] type must be number, "
                                       f"but is {t}")
                if k in cls._FLOATS:
                    v = float(v)
                else:  # static_cast<uint32_t> of the stored integer / truncated float
                    v = int(v) & 0xFFFFFFFF
            elif k == "scaling_enabled":
                if t != "boolean":
                    raise RuntimeError(f"[json.exception.type_error.302] type must be boolean, "
                                       f"but is {t}")
            elif t != "string":  # precision_note
                raise RuntimeError(f"[json.exception.type_error.302] type must be string, "
                                   f"but is {t}")
            setattr(s, k, v)
        return s.validate()


@dataclass
class WarmStart:
    x: np.ndarray
    z: np.ndarray
    y: np.ndarray


@dataclass
class IterationView:
    """solver.hpp:135-145: the scaled iterates handed to on_iteration."""
    iter: int
    x: np.ndarray
    z: np.ndarray
    y: np.ndarray
    l: np.ndarray
    u: np.ndarray


@dataclass
class SolveDiagnostics:
    pcg_calls: list = field(default_factory=list)  # dicts: admm_iter, eps, r_prim_scaled_inf, ...
    check_iterations: list = field(default_factory=list)
    rho_updates: list = field(default_factory=list)
    # solver.hpp:166: called after every ADMM step with an IterationView (the
    # engine then runs its host-driven loop: one D2H of x, z, y per iteration)
    on_iteration: object = None


@dataclass
class SolveOutcome:
    status: str
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    certificate: np.ndarray
    objective: float
    iterations: int
    pcg_iterations_total: int
    r_prim_inf: float
    r_dual_inf: float
    runtime_seconds: float
    equil_passes: int
    equil_residual: float
    rho_final: float
    rho_update_count: int
    info: dict = field(default_factory=dict)


def outcome_from_c(info: _abi.Info, x, z, y, cert) -> SolveOutcome:
    st = _abi.STATUS_NAMES[info.status]
    if info.certificate_valid:
        cert = cert[: (info.m if st == "primal_infeasible" else info.n)].copy()
    else:
        cert = np.zeros(0, dtype=x.dtype)
    return SolveOutcome(status=st, x=x, y=y, z=z, certificate=cert, objective=info.objective,
                        iterations=info.iterations, pcg_iterations_total=info.pcg_iterations_total,
                        r_prim_inf=info.r_prim_inf, r_dual_inf=info.r_dual_inf,
                        runtime_seconds=info.runtime_seconds, equil_passes=info.equil_passes,
                        equil_residual=info.equil_residual, rho_final=info.rho_final,
                        rho_update_count=info.rho_update_count, info=info.as_dict())
