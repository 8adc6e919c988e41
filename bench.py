#!/usr/bin/env python
"""bench.py — B200 ADMM/PCG QP engine on BASELINE.json's headline workload.

Metric (BASELINE.json): "QP solve time to eps=1e-3 (s) and PCG-iteration HBM
GB/s vs roofline".  A *step* is one complete solve — qpcg_f64_solve_problem,
i.e. the reference's `qpcg::solve` timed region (solver.hpp:392 -> :537:
symmetrize, transpose, Ruiz, ADMM/PCG loop, unscale, objective) — of the
workload `config` names (default: BASELINE configs[1], lasso with 10^4
features x 10^5 samples at 15 % density, generated with the reference's own
RNG and recipes; fp64; settings {"lambda_pcg": 1e-3} (0.01, the survey's choice, diverges at this size — DESIGN.md §2).

* value       seconds per solve with the problem already resident in HBM
              (device-pointer inputs), CUDA events on the engine's stream.
* e2e         the same through the reference-facing C-ABI with pinned HOST
              arrays: H2D of P, q, A, l, u and D2H of x, z, y inside the step.
* roofline    the dominant kernel (the A^T SpMV of the PCG operator apply,
              Kp = P p + sigma p + A^T (rho A p)) timed with CUDA events on the
              engine stream right after the timed region; algorithmic bytes per
              SURVEY.md §8(d); peak = MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline  the reference itself (oracle/_ref, unmodified headers) on the
              same instance, 1 core (it is single threaded): its setup
              phases and hot-path operators are timed on a bounded sample and
              the solve time is extrapolated with the REFERENCE's own iteration
              counts (its committed complete solve of the instance).

--impl reference runs only the reference CPU arm (rank 0): the instance built by
the reference's own generators, then ONE complete qpcg::solve of it (minutes on
one core; value = its runtime_seconds), same metric and config dict.
Multi-GPU (torchrun, N > 1): the ROW-SHARDED engine — every
rank holds an nnz-balanced block of A's rows (+ its own A_g^T), and the A^T
partials are combined once per operator apply: by default the SpMV epilogue
stores its rows straight into every peer's memory (NVLink P2P via CUDA IPC)
and a device-side barrier + block-ordered sum follows (--transport nccl: NCCL
allreduce instead); one instance solved by all N GPUs ("strong" scaling),
value = max over ranks of the device-timed solve.  --replicas instead solves an independent instance per rank ("weak").
--shards K (N = 1) runs the sharded engine with K row blocks on one GPU.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QP solve time to eps=1e-3 (s) and PCG-iteration HBM GB/s vs roofline"
WORKLOADS = {
    "1": "random QP n=1000 m=10000 (reference recipe, P 3 nnz/row)",
    "1p": "random QP n=1000 m=10000, P ~15% dense",
    "2": "lasso 1e4 features x 1e5 samples, 15% dense (n=120000, m=120000, nnz(A)=1.5e8)",
    "3": "huber 1e5 x 1e4, 15% dense (n=310000, m=300000, nnz(A)=1.5e8)",
    "4": "svm 1e6 samples x 1e3 features, 15% dense (n=1001000, m=2000000, nnz(A)=1.5e8)",
    "5a": "portfolio N~1e8 (n=142835, m=142836, nnz(A)=1.0e8)",
    "5b": "control/MPC gen_control scale 13 (nnz(A)=1.39e8)",
}


def _json_default(o):
    """numpy scalars / arrays in the bench line -> plain JSON values."""
    if isinstance(o, np.generic):
        return o.item()
    if isinstance(o, np.ndarray):
        return o.tolist()
    raise TypeError(f"not JSON serializable: {type(o).__name__}")


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="2", choices=sorted(WORKLOADS))
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--lambda-pcg", type=float, default=1e-3)
    ap.add_argument("--e2e-steps", type=int, default=0, help="0: same as --steps")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="graph", choices=["graph", "eager"])
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent instance per rank instead of the row-sharded solve")
    ap.add_argument("--shards", type=int, default=1, help="row blocks per GPU (virtual shards)")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="N > 1: combine the ranks' A^T partials by stores into every peer's "
                         "memory fused into the SpMV epilogue (peer) or by NCCL allreduce")
    ap.add_argument("--sweep", default="",
                    help="CLASSES:SCALES[:INSTANCES] (e.g. lasso,svm:1,3,5:10): instead of the "
                         "headline line, print the bench/runner.hpp CSV sweep solved by the engine "
                         "with the reference CPU solver's columns beside it")
    return ap.parse_args()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for l in self.lines:
            p = [x.strip() for x in l.split(",")]
            if len(p) >= 8:
                rows.append(p)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        loaded = [r for r in rows if (num(r[3]) or 0) > 0] or rows
        sm = [num(r[0]) for r in loaded if num(r[0]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(rows[0][1]), "samples": len(rows),
                "samples_under_load": len(loaded), "reasons": reasons}


# ---------------------------------------------------------- engine calls
def _views(arrs, n, m, dev):
    """CSR views (host numpy or device torch tensors) for the C-ABI."""
    from paper_1912_04263_b200 import _abi
    def p(a):
        return C.c_void_p(a.data_ptr() if dev else a.ctypes.data)
    pv, prp, pci, q, av, arp, aci, l, u = arrs
    P = _abi.CsrF64()
    P.rows, P.cols, P.nnz = n, n, int(pv.shape[0])
    P.values, P.row_ptr, P.col_indices = p(pv), p(prp), p(pci)
    A = _abi.CsrF64()
    A.rows, A.cols, A.nnz = m, n, int(av.shape[0])
    A.values, A.row_ptr, A.col_indices = p(av), p(arp), p(aci)
    return P, A, p(q), p(l), p(u)


class Engine:
    def __init__(self, problem, settings, device, stream_ptr, dtype, mode, shards=1, nccl=None,
                 transport="nccl", peer_dir=None):
        import torch
        from paper_1912_04263_b200 import _abi, solver
        self.lib = solver.load_library()
        self.torch = torch
        self.n, self.m = problem.n, problem.m
        self.settings = settings.to_c()
        self.dtype = dtype
        self.pre = "f64" if dtype == np.float64 else "f32"
        tdt = torch.float64 if dtype == np.float64 else torch.float32
        host = [problem.p_upper.values.astype(dtype), problem.p_upper.row_ptr,
                problem.p_upper.col_indices, problem.q.astype(dtype),
                problem.a.values.astype(dtype), problem.a.row_ptr, problem.a.col_indices,
                problem.l.astype(dtype), problem.u.astype(dtype)]
        # pinned host copies (e2e) and HBM-resident copies (value)
        self.host = [torch.from_numpy(np.ascontiguousarray(h)).pin_memory() for h in host]
        self.dev = [t.to(f"cuda:{device}", non_blocking=False) for t in self.host]
        torch.cuda.synchronize()
        self.host_np = [t.numpy() for t in self.host]
        self.out_dev = [torch.empty(k, dtype=tdt, device=f"cuda:{device}")
                        for k in (self.n, self.m, self.m, max(self.n, self.m))]
        self.out_host = [torch.empty(k, dtype=tdt).pin_memory()
                         for k in (self.n, self.m, self.m, max(self.n, self.m))]
        self.bytes_in = sum(int(t.numel() * t.element_size()) for t in self.host)
        self.opts = {}
        for memkind in ("device", "host"):
            o = _abi.Options()
            o.device = device
            o.input_memory = _abi.MEM_DEVICE if memkind == "device" else _abi.MEM_HOST
            o.mode = _abi.MODE_EAGER if mode == "eager" else _abi.MODE_GRAPH
            o.record_diagnostics = 0
            o.virtual_shards = shards
            o.stream = C.c_void_p(stream_ptr)
            if nccl is not None:  # (rank, ranks, id): the row-sharded group
                self._id = C.create_string_buffer(bytes(nccl[2]), _abi.NCCL_ID_BYTES)
                o.nccl_rank, o.nccl_ranks = nccl[0], nccl[1]
                o.nccl_id = C.cast(self._id, C.c_void_p)
                if transport == "peer":  # NCCL only bootstraps the IPC handles
                    o.transport = _abi.TRANSPORT_PEER
            if peer_dir is not None:  # (rank, ranks, rendezvous directory)
                self._dir = C.create_string_buffer(peer_dir[2].encode())
                o.nccl_rank, o.nccl_ranks = peer_dir[0], peer_dir[1]
                o.transport = _abi.TRANSPORT_PEER
                o.rendezvous_dir = C.cast(self._dir, C.c_char_p)
            self.opts[memkind] = o
        self._abi = _abi
        self.msg = C.create_string_buffer(512)

    def solve(self, memkind: str):
        _abi = self._abi
        dev = memkind == "device"
        arrs = self.dev if dev else self.host_np
        P, A, q, l, u = _views(arrs, self.n, self.m, dev)
        outs = self.out_dev if dev else self.out_host
        op = (lambda t: C.c_void_p(t.data_ptr()))
        info = _abi.Info()
        rc = getattr(self.lib, f"qpcg_{self.pre}_solve_problem")(
            C.addressof(P), q, C.addressof(A), l, u, C.addressof(self.settings),
            C.addressof(self.opts[memkind]), None, None, None, C.addressof(info),
            *[op(t) for t in outs], self.msg, 512)
        if rc != 0:
            raise RuntimeError(f"solve failed rc={rc}: {self.msg.value.decode()}")
        return info

    def kernel_timing(self, reps: int):
        """CUDA-event timing of the PCG-iteration kernels on a set-up workspace."""
        _abi = self._abi
        P, A, q, l, u = _views(self.dev, self.n, self.m, True)
        ws = C.c_void_p()
        rc = getattr(self.lib, f"qpcg_{self.pre}_setup")(
            C.byref(ws), C.addressof(P), q, C.addressof(A), l, u, C.addressof(self.settings),
            C.addressof(self.opts["device"]))
        if rc != 0:
            raise RuntimeError(self.lib.qpcg_last_error(None).decode())
        try:
            out = np.zeros(12)
            self.lib.qpcg_bench_kernels_n.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32]
            rc = self.lib.qpcg_bench_kernels_n(ws, reps, out.ctypes.data, 12)
            if rc != 0:
                raise RuntimeError(self.lib.qpcg_last_error(ws).decode())
        finally:
            self.lib.qpcg_cleanup(ws)
        return out

    def resolve_timing(self):
        """The setup / solve split: one workspace, a first
        solve, then the MPC-style re-solve after moving every bound by 1 %
        (qpcg_update_vectors + qpcg_solve, warm from the previous iterates)."""
        _abi = self._abi
        P, A, q, l, u = _views(self.dev, self.n, self.m, True)
        ws = C.c_void_p()
        pre = self.pre
        rc = getattr(self.lib, f"qpcg_{pre}_setup")(
            C.byref(ws), C.addressof(P), q, C.addressof(A), l, u, C.addressof(self.settings),
            C.addressof(self.opts["device"]))
        if rc != 0:
            raise RuntimeError(self.lib.qpcg_last_error(None).decode())
        try:
            op = (lambda t: C.c_void_p(t.data_ptr()))
            solve = getattr(self.lib, f"qpcg_{pre}_solve")
            solve.argtypes = [C.c_void_p] * 6
            first = _abi.Info()
            if solve(ws, C.addressof(first), *[op(t) for t in self.out_dev]) != 0:
                raise RuntimeError(self.lib.qpcg_last_error(ws).decode())
            lo, hi = self.dev[7] * 1.01, self.dev[8] * 1.01
            lo, hi = self.torch.minimum(lo, hi), self.torch.maximum(lo, hi)
            upd = getattr(self.lib, f"qpcg_{pre}_update_vectors")
            upd.argtypes = [C.c_void_p] * 4
            self.torch.cuda.synchronize()
            t0 = time.time()
            if upd(ws, None, op(lo), op(hi)) != 0:
                raise RuntimeError(self.lib.qpcg_last_error(ws).decode())
            second = _abi.Info()
            if solve(ws, C.addressof(second), *[op(t) for t in self.out_dev]) != 0:
                raise RuntimeError(self.lib.qpcg_last_error(ws).decode())
            self.torch.cuda.synchronize()
            wall = time.time() - t0
        finally:
            self.lib.qpcg_cleanup(ws)
        return {"first_solve_s": first.solve_seconds, "first_iterations": int(first.iterations),
                "resolve_s": wall, "resolve_device_s": second.solve_seconds,
                "resolve_iterations": int(second.iterations),
                "resolve_pcg_iterations": int(second.pcg_iterations_total),
                "resolve_status": int(second.status),
                "what": "bounds moved by 1 %, qpcg_update_vectors + qpcg_solve on the set-up "
                        "workspace (no setup, warm iterates)"}


# ------------------------------------------------------------ CPU baseline
def full_reference_seconds(cfg: str, lam: float):
    try:
        with open(os.path.join(ROOT, "profiles", f"ref_solve_config{cfg}_lam{lam:g}.json")) as f:
            return float(json.load(f)["runtime_seconds"])
    except Exception:
        return None


def cpu_baseline(problem, counts: dict, budget_reps: int = 1, cfg: str = "", lam: float = 0.0) -> dict:
    """The reference (oracle/_ref, unmodified headers, 1 core) on a bounded
    sample of the same instance; solve time extrapolated from its measured
    components and the solve's iteration counts."""
    from oracle import oracle as O  # cpu_baseline leg only
    lib = O.ref_lib()
    P, A, q, l, u = _views([problem.p_upper.values, problem.p_upper.row_ptr,
                            problem.p_upper.col_indices, problem.q, problem.a.values,
                            problem.a.row_ptr, problem.a.col_indices, problem.l, problem.u],
                           problem.n, problem.m, False)
    out = np.zeros(9)
    t0 = time.time()
    rc = lib.qref_time_components_f64(C.byref(P), q, C.byref(A), l, u,
                                      C.c_uint32(budget_reps), C.c_void_p(out.ctypes.data))
    if rc != 0:
        raise RuntimeError(lib.qref_last_error().decode())
    wall = time.time() - t0
    t_sym, t_trans, t_ruiz1, t_op, t_k, t_at, t_a, t_res = (float(v) for v in out[:8])
    full = full_reference_seconds(cfg, lam) if cfg else None
    passes = int(counts.get("equil_passes", 10))
    iters = int(counts["iterations"])
    pcg = int(counts["pcg_iterations_total"])
    checks = iters // 5
    # solve() = symmetrize + transpose + Ruiz + operator build + loop.  Ruiz:
    # the measured 1-pass call includes two transposes of A and the copies; each
    # further pass costs the pass body only (estimated as the 1-pass time minus
    # the two transposes).  Loop: per ADMM step the rhs A^T spmv, the PCG r0
    # K-apply and z~ = A x~; one K-apply per PCG iteration; per check the
    # residuals (3 spmv) and, while unsolved, the A^T infeasibility spmv.
    pass_body = max(t_ruiz1 - 2.0 * t_trans, 0.0)
    setup = t_sym + t_trans + t_ruiz1 + (passes - 1) * pass_body + t_op
    # initial residuals; per unsolved check the residuals plus the two
    # certificate products over the original matrices (A_o^T v, A_o v)
    loop = t_res + iters * (t_at + t_k + t_a) + pcg * t_k + checks * (t_res + t_at + t_a)
    return {"value": setup + loop, "unit": "s", "cores": 1, "kind": "reference",
            "sample": (f"oracle/_ref (unmodified reference headers, g++ -O3 -ffp-contract=off, "
                       f"1 thread) on the same instance: symmetrize {t_sym:.2f}s, transpose "
                       f"{t_trans:.2f}s, 1-pass Ruiz {t_ruiz1:.2f}s, operator build {t_op:.2f}s, "
                       f"K-apply {t_k:.3f}s, A^T spmv {t_at:.3f}s, A spmv {t_a:.3f}s, residuals "
                       f"{t_res:.3f}s ({wall:.1f}s of CPU); solve time EXTRAPOLATED to {passes} "
                       f"Ruiz passes, {iters} ADMM / {pcg} PCG iterations, {checks} checks "
                       f"(counts: {counts.get('source', 'given')})"
                       + (f"; the reference's complete solve of this instance took {full:.0f} s on one "
                          f"core of the build container (profiles/ref_solve_config{cfg}_*.json)"
                          if full else "")),
            "extrapolated": True, "nproc": os.cpu_count(),
            "components_s": {"symmetrize": t_sym, "transpose": t_trans, "ruiz_1pass": t_ruiz1,
                             "operator_build": t_op, "k_apply": t_k, "at_spmv": t_at,
                             "a_spmv": t_a, "residuals": t_res, "setup_est": setup,
                             "loop_est": loop}}


def reference_counts(config: str, lam: float):
    """The REFERENCE's own iteration counts for this instance: its complete
    solve, committed as a golden anchor (tests/golden/config*_reference_solve.json,
    scripts/ref_solve_config.py).  None when no such run exists."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", f"config{config}_reference_solve.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    if abs(float(d.get("lambda_pcg", -1.0)) - lam) > 1e-15:
        return None
    return {"iterations": int(d["iterations"]), "pcg_iterations_total": int(d["pcg_iterations_total"]),
            "equil_passes": int(d["equil_passes"]), "runtime_seconds": float(d["runtime_seconds"]),
            "source": f"the reference's complete solve (tests/golden/config{config}_reference_solve.json)"}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


def ncu_traffic(config: str, dtype: str = "f64", kernel: str = "EpiKp"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu capture of this config (profiles/ncu_summary.json, written by
    scripts/ncu_summarize.py; key <config> or <config>_f32)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        rec = d.get(config if dtype == "f64" else f"{config}_f32", {})
        k = rec.get("kernels", {}).get(kernel)
        return k.get("dram_bytes") if k else None
    except Exception:
        return None


def config_dict(args, problem, world: int, sharded: bool) -> dict:
    """The workload description both arms print (identical dicts)."""
    S = 8 if args.dtype == "f64" else 4
    a_bytes = problem.a.nnz * (S + 4) * 2
    return {"workload": WORKLOADS[args.config], "config_id": args.config,
            "n": problem.n, "m": problem.m, "nnz_P_upper": problem.p_upper.nnz,
            "nnz_A": problem.a.nnz, "settings": {"lambda_pcg": args.lambda_pcg},
            "parallelism": (f"rowshard{world}-{args.transport}" if sharded else f"replicas{world}")
                           if world > 1 else
                           ("single" if args.shards <= 1 else f"virtual-rowshard{args.shards}"),
            "l2": ("inputs larger than L2 (A and A^T streams ~%.1f GB per PCG iteration)"
                   % (a_bytes / 1e9)) if a_bytes >= (256 << 20) else
                  "matrices fit in L2: a 512 MB buffer is overwritten before every timed step",
            "mode": args.mode}


def reference_problem(config: str):
    """The instance generated by the REFERENCE's own generators (oracle/_ref:
    bench::detail recipes / bench::generate, generators.hpp) — bit-identical to
    the engine arm's native generator (tests/test_generators.py)."""
    from oracle import oracle as O  # reference arm only
    from paper_1912_04263_b200.generators import CONFIGS
    spec = CONFIGS[config]
    if spec[0] == "class":
        return O.ref_generate(spec[1], spec[2], 0)
    return O.ref_generate_explicit(*spec, seed=0)


# --------------------------------------------------------------- arms
def run_reference(args, rank: int, world: int) -> None:
    """The reference's own CPU implementation of the path: ONE complete
    qpcg::solve (solver.hpp:386-541, oracle/_ref = the unmodified headers) of
    the instance the reference's own generators build.  value = the solve's
    runtime_seconds (its own timed region, solver.hpp:392 -> :539).  A full
    solve of a BASELINE config takes minutes on one core, so exactly one step
    is run whatever --steps / --warmup say (both printed as requested_*)."""
    if rank != 0:
        return
    from oracle import oracle as O  # reference arm only
    from paper_1912_04263_b200.problem import Settings
    tg = time.time()
    problem = reference_problem(args.config)
    if args.dtype == "f32":
        problem = problem.astype(np.float32)
    gen_s = time.time() - tg
    log(f"reference generated config {args.config}: nnz(A)={problem.a.nnz} in {gen_s:.1f}s")
    t0 = time.time()
    r = O.ref_solve(problem, Settings(lambda_pcg=args.lambda_pcg))
    wall = time.time() - t0
    v = float(r.runtime_seconds)
    log(f"reference solve: {r.status} {r.iterations} ADMM / {r.pcg_iterations_total} PCG, "
        f"runtime {v:.1f}s (wall {wall:.1f}s)")
    cb = {"value": v, "unit": "s", "cores": 1, "kind": "reference", "extrapolated": False,
          "sample": (f"one complete qpcg::solve (oracle/_ref: the unmodified reference headers, "
                     f"g++ -O3 -ffp-contract=off, single-threaded as the reference is) of the "
                     f"whole config-{args.config} instance, generated by the reference's own "
                     f"generators; runtime_seconds = its own timed region"),
          "nproc": os.cpu_count(), "wall_s": wall}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
            "steps": 1, "warmup": 0, "requested_steps": args.steps,
            "requested_warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic (reference RNG + recipes, SURVEY.md §8(d))",
            "config": config_dict(args, problem, world, world > 1 and not args.replicas),
            "solve": {"status": r.status, "iterations": int(r.iterations),
                      "pcg_iterations_total": int(r.pcg_iterations_total),
                      "objective": float(r.objective), "r_prim_inf": float(r.r_prim_inf),
                      "r_dual_inf": float(r.r_dual_inf), "equil_passes": int(r.equil_passes)},
            "generation_s": gen_s, "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line, default=_json_default), flush=True)


def run_sweep(args) -> None:
    """runner.hpp-schema CSV: the engine's row + the reference's (oracle/_ref,
    1 core, the cpu_baseline leg) status / iterations / runtime + speed-up."""
    from oracle import oracle as O  # reference columns only
    from paper_1912_04263_b200 import generators, runner
    from paper_1912_04263_b200.problem import Settings
    parts = args.sweep.split(":")
    classes = generators.CLASSES if parts[0] == "all" else parts[0].split(",")
    scales = [int(v) for v in parts[1].split(",")]
    k = int(parts[2]) if len(parts) > 2 else 10
    s = Settings(lambda_pcg=args.lambda_pcg)
    runner.b200_solve(0, args.mode)(generators.generate(classes[0], scales[0], 0), s)  # context warm-up
    mine = runner.run_benchmark(classes, scales, s, k, solve_fn=runner.b200_solve(0, args.mode))
    ref = runner.run_benchmark(classes, scales, s, k, solve_fn=lambda p, st: O.ref_solve(p, st))
    runner.write_csv(mine, sys.stdout, compare=ref)


def main():
    args = parse()
    if args.sweep:
        run_sweep(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    # QPCG_BENCH_SAME_GPU=1: every rank on GPU 0 (a harness dry run of the
    # multi-rank path on a one-GPU box: gloo for the host collectives, the
    # engine's peer transport bootstrapped through a rendezvous directory)
    same_gpu = os.environ.get("QPCG_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        # NCCL's init lines (communicator size and rank per process) let the
        # driver verify that N ranks formed one group
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_1912_04263_b200 import generators, solver
    from paper_1912_04263_b200.problem import Settings
    dtype = np.float64 if args.dtype == "f64" else np.float32
    sharded = world > 1 and not args.replicas
    nccl = None
    rdir = None
    if sharded and same_gpu:  # rendezvous directory instead of an NCCL id
        import tempfile
        obj = [tempfile.mkdtemp(prefix="qpcg_rdv_") if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rdir = obj[0]
    elif sharded:  # one NCCL group for the engine, id shared over torch.distributed
        obj = [solver.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl = (rank, world, obj[0])
    tg = time.time()
    problem = generators.config(args.config, seed=0 if sharded else rank)
    gen_s = time.time() - tg
    log(f"generated config {args.config}: n={problem.n} m={problem.m} nnz(A)={problem.a.nnz} in {gen_s:.1f}s")
    settings = Settings(lambda_pcg=args.lambda_pcg)
    stream = torch.cuda.Stream(device=local)
    with torch.cuda.stream(stream):
        eng = Engine(problem, settings, local, stream.cuda_stream, dtype, args.mode,
                     shards=args.shards, nccl=nccl, transport=args.transport,
                     peer_dir=(rank, world, rdir) if rdir else None)
        for i in range(args.warmup):
            t = time.time()
            info = eng.solve("device")
            log(f"warmup {i}: status={info.status} iters={info.iterations} pcg={info.pcg_iterations_total} "
                f"setup={info.setup_seconds:.3f}s loop={info.solve_seconds:.3f}s wall={time.time() - t:.2f}s")
        def barrier():
            if dist is not None:
                dist.barrier()
        # ---- timed region: K device-resident solves
        barrier()
        torch.cuda.synchronize()
        clocks = ClockSampler(local)
        clocks.start()
        # instances whose matrices fit in L2 (126 MB): overwrite a 512 MB buffer
        # between the timed steps, outside the timed events
        a_bytes = problem.a.nnz * (np.dtype(dtype).itemsize + 4) * 2
        flush = torch.empty(64 << 20, dtype=torch.float64, device=f"cuda:{local}") \
            if a_bytes < (256 << 20) else None
        infos, ms_steps = [], []
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            infos.append(eng.solve("device"))
            e1.record(stream)
            e1.synchronize()
            ms_steps.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        barrier()
        clk = clocks.stop()
        ms = sum(ms_steps) / args.steps
        # ---- e2e: host pinned arrays through the C-ABI
        ke = args.e2e_steps or args.steps
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        einfos = [eng.solve("host") for _ in range(ke)]
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms_e2e = f0.elapsed_time(f1) / ke
        # ---- dominant kernel, CUDA events on the engine stream
        log(f"timed: {ms:.2f} ms/solve, e2e {ms_e2e:.2f} ms/solve")
        kt = eng.kernel_timing(args.kernel_reps)
        log(f"kernels: A {kt[0]:.4f} ms, A^T {kt[1]:.4f} ms, PCG iteration {kt[2]:.4f} ms")
        resolve = eng.resolve_timing()
        log(f"re-solve after a bound update: {resolve['resolve_iterations']} iterations, "
            f"{resolve['resolve_s'] * 1e3:.1f} ms (first solve {resolve['first_solve_s'] * 1e3:.1f} ms)")
    if dist is not None:
        props = torch.cuda.get_device_properties(local)
        log(json.dumps({"rank": rank, "local_rank": local, "device": local,
                        "device_uuid": str(getattr(props, "uuid", "")), "world": world,
                        "ranks_seen": dist.get_world_size(),
                        "transport": (args.transport if sharded else "none (replicas)"),
                        "engine_group": (f"{world} ranks x {args.shards} block(s)"
                                         if sharded else "independent"),
                        "ms_per_solve": ms, "iterations": int(infos[-1].iterations)}))
        t = torch.tensor([ms, ms_e2e], device="cpu" if same_gpu else f"cuda:{local}",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    last = infos[-1]
    pk = peaks()
    S = 8 if dtype == np.float64 else 4
    at_ms, pcg_ms = kt[1], kt[2]
    gram = bool(kt[9] > 0)  # the one-pass operator apply (csrc/gram.cuh) runs the PCG iterations
    hbm = pk["hbm_gbs"]
    rate = lambda b, t_ms: b / (t_ms * 1e-3) / 1e9  # noqa: E731
    if gram:
        # dominant kernel: k_gram (t = rho A p and the partial windows of A^T t
        # in one pass over A).  Algorithmic bytes (§8(d) style, 4-byte
        # indices): MB(A) + S n (p) + S m (t) + S G W (partial windows) =
        # kt[10] with the index bytes at 4 instead of the 2 streamed
        S_ = 8 if dtype == np.float64 else 4
        nnz_a = problem.a.nnz
        alg = kt[10] + 2.0 * nnz_a  # 16-bit in-window offsets counted at 4 bytes
        kern = {"kernel": "k_gram: one pass over A forming t = rho A p and A^T t's window "
                          "partials (PCG operator apply, csrc/gram.cuh)",
                "achieved": rate(alg, kt[9]), "algorithmic_bytes_per_launch": alg,
                "launch_ms": kt[9]}
    else:
        kern = {"kernel": "spmv A^T pass of the PCG operator (Kp = P p + sigma p + A^T t)"
                          + (" on rank 0's row block" if sharded or args.shards > 1 else ""),
                "achieved": rate(kt[4], at_ms), "algorithmic_bytes_per_launch": kt[4],
                "launch_ms": at_ms}
    achieved = kern["achieved"]
    loop_s = last.solve_seconds
    roofline = {"bound": "hbm", **kern, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "peak_source": pk["source"],
                "traffic": None if (sharded or args.shards > 1) else
                           ncu_traffic(args.config, args.dtype, "k_gram" if gram else "EpiKp"),
                "operator_path": "one-pass (k_gram)" if gram else "two-pass (A, A^T SpMV)",
                "a_pass": {"ms": kt[0], "bytes": kt[3], "achieved": rate(kt[3], kt[0])},
                "at_pass": {"ms": at_ms, "bytes": kt[4], "achieved": rate(kt[4], at_ms)},
                # SURVEY §8(d)'s B_pcg counts BOTH matrix streams; on the one-pass
                # path A^T's window rows are never read, so this is an
                # EFFECTIVE rate (it may exceed the peak); format_bytes has the
                # bytes actually streamed
                "pcg_iteration": {"ms": pcg_ms, "bytes": kt[5],
                                  "achieved": rate(kt[5], pcg_ms),
                                  "frac": rate(kt[5], pcg_ms) / hbm,
                                  "effective": gram},
                "format_bytes": {"a_pass": kt[6], "at_pass": kt[7],
                                 "pcg_iteration": kt[11] if gram else kt[8],
                                 "at_pass_frac": rate(kt[7], at_ms) / hbm,
                                 "k_gram": kt[10] if gram else None,
                                 "k_gram_frac": rate(kt[10], kt[9]) / hbm if gram else None,
                                 "pcg_iteration_frac":
                                     rate(kt[11] if gram else kt[8], pcg_ms) / hbm},
                "frac_of_nominal_8TBs": achieved / 8000.0}
    line = {"metric": METRIC, "value": ms * 1e-3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None,
            "dtype": args.dtype, "data": "synthetic (reference RNG + recipes, SURVEY.md §8(d))",
            "config": config_dict(args, problem, world, sharded),
            "solve": {"status": int(last.status), "iterations": int(last.iterations),
                      "pcg_iterations_total": int(last.pcg_iterations_total),
                      "objective": last.objective, "r_prim_inf": last.r_prim_inf,
                      "r_dual_inf": last.r_dual_inf, "equil_passes": int(last.equil_passes),
                      "setup_s": last.setup_seconds, "loop_s": loop_s,
                      "live_pcg_gbs": (kt[5] * last.pcg_iterations_total) / loop_s / 1e9
                      if loop_s > 0 else None},
            "workspace_reuse": resolve,
            "gpu_launches": int(sum(i.kernel_launches for i in infos)),
            "engine_flags": int(last.engine_flags),
            "clocks": clk, "roofline": roofline,
            "e2e": {"value": ms_e2e * 1e-3, "unit": "s",
                    "h2d_bytes_per_step": int(einfos[-1].h2d_bytes),
                    "d2h_bytes_per_step": int(einfos[-1].d2h_bytes)},
            "generation_s": gen_s}
    if not args.no_cpu_baseline:
        try:
            counts = reference_counts(args.config, args.lambda_pcg) or {
                "iterations": int(last.iterations),
                "pcg_iterations_total": int(last.pcg_iterations_total),
                "equil_passes": int(last.equil_passes),
                "source": "this engine's solve (no complete reference solve of this instance "
                          "is committed)"}
            line["cpu_baseline"] = cpu_baseline(problem, counts, cfg=args.config,
                                                lam=args.lambda_pcg)
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"value": None, "error": repr(e)}
    print(json.dumps(line, default=_json_default), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
