"""Host-side mirror of the reference's solve entry point over the C-ABI.

``solve(problem, settings, initial=None, diag=None)`` has the meaning of
``qpcg::solve`` (solver.hpp:386-541) and raises the same error classes
(``ValueError`` for std::invalid_argument, ``NotPositiveDefiniteError``).
``Workspace`` is the OSQP-style split (setup / warm_start / update_rho /
update_vectors / solve) of include/qpcg_b200.h.

There is no CPU fallback: if ``libqpcg_b200.so`` is missing or no CUDA
device is present, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _abi
from .problem import (NotPositiveDefiniteError, QpProblem, Settings, SolveDiagnostics,
                      WarmStart, outcome_from_c)

LIB_PATH = os.environ.get("QPCG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                      "libqpcg_b200.so")

_lib = None


def _point_at_pip_nccl() -> None:
    """QPCG_NCCL_LIB -> the pip NCCL (nvidia-nccl) that torch loads, when it is
    installed and the variable is unset: the engine dlopens NCCL lazily, and
    a system libnccl.so.2 of another version mapped first would clash with a
    later `import torch` (csrc/comm.cuh nccl_api)."""
    if os.environ.get("QPCG_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia")
        for base in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(base, "nccl", "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["QPCG_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def load_library() -> C.CDLL:
    """Load the engine's C-ABI library (never falls back to anything else)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"qpcg-b200: CUDA engine not built ({LIB_PATH} missing); "
                          "run __graft_entry__.build() / python -m paper_1912_04263_b200.build")
    _point_at_pip_nccl()
    lib = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    for pre in ("f64", "f32"):
        getattr(lib, f"qpcg_{pre}_setup").argtypes = [C.POINTER(vp), vp, vp, vp, vp, vp, vp, vp]
        getattr(lib, f"qpcg_{pre}_warm_start").argtypes = [vp, vp, vp, vp]
        getattr(lib, f"qpcg_{pre}_update_rho").argtypes = [vp, C.c_double]
        getattr(lib, f"qpcg_{pre}_update_vectors").argtypes = [vp, vp, vp, vp]
        getattr(lib, f"qpcg_{pre}_solve").argtypes = [vp, vp, vp, vp, vp, vp]
        getattr(lib, f"qpcg_{pre}_solve_problem").argtypes = [vp] * 15 + [C.c_char_p, C.c_size_t]
    lib.qpcg_cleanup.argtypes = [vp]
    lib.qpcg_release_cached_memory.argtypes = []
    lib.qpcg_release_cached_memory.restype = None
    lib.qpcg_last_error.argtypes = [vp]
    lib.qpcg_last_error.restype = C.c_char_p
    lib.qpcg_version.restype = C.c_char_p
    lib.qpcg_get_pcg_calls.argtypes = [vp, vp, C.c_uint32]
    lib.qpcg_get_pcg_calls.restype = C.c_uint32
    lib.qpcg_get_rho_updates.argtypes = [vp, vp, C.c_uint32]
    lib.qpcg_get_rho_updates.restype = C.c_uint32
    lib.qpcg_get_check_iterations.argtypes = [vp, vp, C.c_uint32]
    lib.qpcg_get_check_iterations.restype = C.c_uint32
    lib.qpcg_shard_cuts.argtypes = [vp, C.c_uint32, C.c_uint32, C.c_uint32, vp]
    lib.qpcg_nccl_unique_id.argtypes = [vp]
    _lib = lib
    return lib


def release_cached_memory() -> None:
    """Return the engine's idle device memory (released workspaces' cached
    blocks, unused pool memory) to the driver; live workspaces keep theirs."""
    load_library().qpcg_release_cached_memory()


def _raise(rc: int, msg: str):
    if rc == _abi.QPCG_ERR_INVALID:
        raise ValueError(msg)
    if rc == _abi.QPCG_ERR_NOT_PD:
        raise NotPositiveDefiniteError(msg)
    if rc == _abi.QPCG_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def _pre(dtype) -> str:
    if dtype == np.float64:
        return "f64"
    if dtype == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {dtype}")


def _iteration_trampoline(fn, dtype):
    """qpcg_iteration_cb -> fn(IterationView) with numpy copies."""
    from .problem import IterationView
    ct = C.c_double if dtype == np.float64 else C.c_float

    def cb(_user, it, x, z, y, l, u, n, m):
        def arr(p, k):
            return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (k,)).copy() if k else \
                np.zeros(0, dtype)
        fn(IterationView(int(it), arr(x, n), arr(z, m), arr(y, m), arr(l, m), arr(u, m)))
    return _abi.ITERATION_CB(cb)


def make_options(device: int = -1, mode: str = "graph", record_diagnostics: bool = False,
                 device_memory: bool = False, shards: int = 1,
                 nccl: tuple | None = None, peer: tuple | None = None,
                 sm_budget: int = 0, on_iteration=None, dtype=np.float64) -> _abi.Options:
    """sm_budget: SMs the persistent driver may hold (0: the whole device);
    shards: row blocks of A held on this device (virtual shards);
    nccl: (rank, ranks, id_bytes) to join the row-sharded NCCL group
    (id_bytes from nccl_unique_id() on rank 0);
    peer: (rank, ranks, rendezvous_dir) for the peer-memory transport."""
    o = _abi.Options()
    o.device = device
    o.input_memory = _abi.MEM_DEVICE if device_memory else _abi.MEM_HOST
    o.mode = {"eager": _abi.MODE_EAGER, "persistent": _abi.MODE_PERSISTENT}.get(mode, _abi.MODE_GRAPH)
    o.record_diagnostics = 1 if record_diagnostics else 0
    o.virtual_shards = max(1, int(shards))
    o.sm_budget = max(0, int(sm_budget))
    if on_iteration is not None:
        o._keep_cb = _iteration_trampoline(on_iteration, dtype)  # outlives the workspace
        o.on_iteration = C.cast(o._keep_cb, C.c_void_p)
    if nccl is not None:
        rank, ranks, uid = nccl
        buf = C.create_string_buffer(bytes(uid), _abi.NCCL_ID_BYTES)
        o.nccl_rank, o.nccl_ranks = int(rank), int(ranks)
        o.nccl_id = C.cast(buf, C.c_void_p)
        o._keep_id = buf  # the id must outlive the setup call
    if peer is not None:  # (rank, ranks, rendezvous_dir or None with an NCCL id)
        rank, ranks, rdir = peer
        o.transport = _abi.TRANSPORT_PEER
        o.nccl_rank, o.nccl_ranks = int(rank), int(ranks)
        if rdir is not None:
            o._keep_dir = C.create_string_buffer(str(rdir).encode())
            o.rendezvous_dir = C.cast(o._keep_dir, C.c_char_p)
    return o


def shard_cuts(row_ptr: np.ndarray, nnz: int, blocks: int) -> tuple[np.ndarray, bool]:
    """nnz-balanced contiguous row cuts (qpcg_shard_cuts; host-only, no GPU)."""
    rp = np.ascontiguousarray(row_ptr, np.uint32)
    cuts = np.zeros(blocks + 1, np.uint32)
    ok = load_library().qpcg_shard_cuts(_abi.ptr(rp), len(rp) - 1, int(nnz), int(blocks),
                                        _abi.ptr(cuts))
    return cuts, bool(ok)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (rank 0 creates it and shares it with the group)."""
    lib = load_library()
    buf = C.create_string_buffer(_abi.NCCL_ID_BYTES)
    rc = lib.qpcg_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != _abi.QPCG_OK:
        _raise(rc, lib.qpcg_last_error(None).decode())
    return buf.raw


class Workspace:
    """OSQP-style workspace: setup once, then solve / warm_start / update_*."""

    def __init__(self, problem: QpProblem, settings: Settings | None = None, device: int = -1,
                 mode: str = "graph", record_diagnostics: bool = False, shards: int = 1,
                 nccl: tuple | None = None, peer: tuple | None = None, on_iteration=None):
        self.lib = load_library()
        problem = problem.checked()  # lengths + dtype before any pointer crosses the ABI
        self.problem = problem
        self.dtype = problem.dtype
        self.pre = _pre(self.dtype)
        self.settings = settings or Settings()
        self._opts = make_options(device, mode, record_diagnostics, shards=shards, nccl=nccl,
                                  peer=peer, on_iteration=on_iteration, dtype=problem.dtype)
        self._s = self.settings.to_c()
        self._pv, self._av = problem.p_upper.view(), problem.a.view()
        self.ws = C.c_void_p()
        rc = getattr(self.lib, f"qpcg_{self.pre}_setup")(
            C.byref(self.ws), C.addressof(self._pv), _abi.ptr(problem.q), C.addressof(self._av),
            _abi.ptr(problem.l), _abi.ptr(problem.u), C.addressof(self._s),
            C.addressof(self._opts))
        if rc != _abi.QPCG_OK:
            self.ws = None
            _raise(rc, self.lib.qpcg_last_error(None).decode())

    def _check(self, rc):
        if rc != _abi.QPCG_OK:
            _raise(rc, self.lib.qpcg_last_error(self.ws).decode())

    def warm_start(self, x, z, y):
        a = _warm_arrays(x, z, y, self.problem.n, self.problem.m, self.dtype)
        self._check(getattr(self.lib, f"qpcg_{self.pre}_warm_start")(self.ws, *[_abi.ptr(v) for v in a]))

    def update_rho(self, rho: float):
        self._check(getattr(self.lib, f"qpcg_{self.pre}_update_rho")(self.ws, C.c_double(rho)))

    def update_vectors(self, q=None, l=None, u=None):
        a = [None if v is None else np.ascontiguousarray(v, self.dtype).reshape(-1)
             for v in (q, l, u)]
        if a[0] is not None and a[0].shape[0] != self.problem.n:
            raise ValueError("update_vectors: q length must equal n")
        if any(v is not None and v.shape[0] != self.problem.m for v in a[1:]):
            raise ValueError("update_vectors: bound lengths must equal m")
        self._check(getattr(self.lib, f"qpcg_{self.pre}_update_vectors")(self.ws, *[_abi.ptr(v) for v in a]))

    def solve(self, diag: SolveDiagnostics | None = None):
        n, m = self.problem.n, self.problem.m
        x, z, y = np.zeros(n, self.dtype), np.zeros(m, self.dtype), np.zeros(m, self.dtype)
        cert = np.zeros(max(n, m), self.dtype)
        info = _abi.Info()
        self._check(getattr(self.lib, f"qpcg_{self.pre}_solve")(
            self.ws, C.addressof(info), _abi.ptr(x), _abi.ptr(z), _abi.ptr(y), _abi.ptr(cert)))
        if diag is not None:
            fetch_diagnostics(self.lib, self.ws, diag)
        return outcome_from_c(info, x, z, y, cert)

    def close(self):
        if self.ws:
            self.lib.qpcg_cleanup(self.ws)
            self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _warm_arrays(x, z, y, n: int, m: int, dtype):
    """solver.hpp:414-417: a warm start of the wrong size is rejected before
    any pointer reaches the ABI (finiteness is checked by the engine)."""
    a = [np.ascontiguousarray(v, dtype).reshape(-1) for v in (x, z, y)]
    if a[0].shape[0] != n or a[1].shape[0] != m or a[2].shape[0] != m:
        raise ValueError("solve: warm start dimension mismatch")
    return a


def fetch_diagnostics(lib, ws, diag: SolveDiagnostics):
    k = lib.qpcg_get_pcg_calls(ws, None, 0)
    buf = (_abi.PcgCall * max(k, 1))()
    lib.qpcg_get_pcg_calls(ws, buf, k)
    diag.pcg_calls = [dict(admm_iter=c.admm_iter, iterations=c.iterations, eps=c.eps,
                           r_prim_scaled_inf=c.r_prim_scaled_inf,
                           r_dual_scaled_inf=c.r_dual_scaled_inf, converged=bool(c.converged))
                      for c in buf[:k]]
    k = lib.qpcg_get_rho_updates(ws, None, 0)
    rb = (_abi.RhoUpdate * max(k, 1))()
    lib.qpcg_get_rho_updates(ws, rb, k)
    diag.rho_updates = [dict(admm_iter=r.admm_iter, rho_before=r.rho_before, rho_after=r.rho_after)
                        for r in rb[:k]]
    k = lib.qpcg_get_check_iterations(ws, None, 0)
    cb = (C.c_uint32 * max(k, 1))()
    lib.qpcg_get_check_iterations(ws, cb, k)
    diag.check_iterations = list(cb[:k])


def solve(p: QpProblem, settings: Settings | None = None, initial: WarmStart | None = None,
          diag: SolveDiagnostics | None = None, device: int = -1, mode: str = "graph",
          shards: int = 1, nccl: tuple | None = None, peer: tuple | None = None,
          sm_budget: int = 0):
    """Drop-in for qpcg::solve (solver.hpp:386-541) on the B200 engine.
    shards > 1 / nccl / peer: the row-sharded engine;
    sm_budget: cap on the SMs of the persistent driver (see solve_batch)."""
    if diag is not None:
        fn, holder = diag.on_iteration, {}

        def observed(view):  # solver.hpp:446-454: the PcgCall is recorded first
            if "ws" in holder:
                fetch_diagnostics(holder["ws"].lib, holder["ws"].ws, diag)
            fn(view)
        with Workspace(p, settings, device, mode, record_diagnostics=True, shards=shards,
                       nccl=nccl, peer=peer, on_iteration=observed if fn else None) as ws:
            holder["ws"] = ws
            if initial is not None:
                ws.warm_start(initial.x, initial.z, initial.y)
            return ws.solve(diag)
    lib = load_library()
    p = p.checked()  # lengths + dtype before any pointer crosses the ABI
    pre = _pre(p.dtype)
    n, m = p.n, p.m
    dt = p.dtype
    s = (settings or Settings()).to_c()
    o = make_options(device, mode, shards=shards, nccl=nccl, peer=peer, sm_budget=sm_budget)
    x, z, y = np.zeros(n, dt), np.zeros(m, dt), np.zeros(m, dt)
    cert = np.zeros(max(n, m), dt)
    info = _abi.Info()
    pv, av = p.p_upper.view(), p.a.view()
    w = [None, None, None] if initial is None else _warm_arrays(initial.x, initial.z, initial.y,
                                                                  n, m, dt)
    msg = C.create_string_buffer(512)
    rc = getattr(lib, f"qpcg_{pre}_solve_problem")(
        C.addressof(pv), _abi.ptr(p.q), C.addressof(av), _abi.ptr(p.l), _abi.ptr(p.u),
        C.addressof(s), C.addressof(o), *[_abi.ptr(v) for v in w], C.addressof(info),
        _abi.ptr(x), _abi.ptr(z), _abi.ptr(y), _abi.ptr(cert), msg, 512)
    if rc != _abi.QPCG_OK:
        _raise(rc, msg.value.decode())
    return outcome_from_c(info, x, z, y, cert)


def solve_batch(problems, settings: Settings | None = None, device: int = -1,
                concurrency: int = 8, small_nnz: int = 30000) -> list:
    """Many independent problems on one GPU.
    Problems with nnz(A) + nnz(P_upper) <= small_nnz run `concurrency` at a
    time, each on its own workspace and stream with its persistent driver
    capped at one 16-SM thread-block cluster (sm_budget = 16), so they share
    the GPU instead of each holding all of it; larger problems run one after
    another with the whole device (measured: side-by-side solves only pay off
    below ~3e4 nonzeros, scripts/batch_throughput.py).  Outcomes in input
    order, bitwise equal to solve()."""
    from concurrent.futures import ThreadPoolExecutor
    problems = list(problems)
    out = [None] * len(problems)
    small = [i for i, p in enumerate(problems) if p.nnz_total() <= small_nnz]
    k = max(1, min(int(concurrency), len(small) or 1))
    if small:
        with ThreadPoolExecutor(max_workers=k) as ex:
            budget = 16 if k > 1 else 0
            for i, o in zip(small, ex.map(lambda i: solve(problems[i], settings, device=device,
                                                          sm_budget=budget), small)):
                out[i] = o
    for i, p in enumerate(problems):
        if out[i] is None:
            out[i] = solve(p, settings, device=device)
    return out
