"""Row sharding on CPU: the nnz-balanced cuts of the C-ABI,
and the sharded algorithm — block transposes, the A^T-partial allreduce of the
K-apply, the max-combined Ruiz column norms, the diag(A^T A) chain and a full
sharded PCG — run by 2 processes over torch.distributed `gloo` against the
oracle.  The GPU engine runs the same protocol (csrc/shard.cuh); its parity is
checked on the B200 by tests/test_gpu_shard.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import CsrMatrix


def cuts_mirror(rp, nnz, blocks):
    """Python restatement of shard_cuts (csrc/comm.cuh)."""
    rp = np.asarray(rp, np.int64)
    rows = len(rp) - 1
    ok = rp[0] == 0 and rp[-1] == nnz and bool(np.all(np.diff(rp) >= 0))
    if not ok:
        return np.array([0] + [rows] * blocks, np.uint32), False
    c = [0]
    for g in range(1, blocks):
        c.append(max(c[-1], int(np.searchsorted(rp, nnz * g // blocks, side="left"))))
    c.append(rows)
    return np.array(c, np.uint32), True


@pytest.mark.parametrize("cls,scale", [("lasso", 3), ("portfolio", 4), ("svm", 3), ("control", 3),
                                       ("random", 2)])
@pytest.mark.parametrize("blocks", [1, 2, 3, 8])
def test_shard_cuts_match_mirror(cls, scale, blocks):
    p = G.generate(cls, scale, 0)
    cuts, ok = solver.shard_cuts(p.a.row_ptr, p.a.nnz, blocks)
    ref, ok_ref = cuts_mirror(p.a.row_ptr, p.a.nnz, blocks)
    assert ok and ok_ref
    assert np.array_equal(cuts, ref)
    assert cuts[0] == 0 and cuts[-1] == p.m and np.all(np.diff(cuts.astype(np.int64)) >= 0)
    # balance: no block exceeds its share by more than the longest row
    rp = p.a.row_ptr.astype(np.int64)
    per = rp[cuts[1:]] - rp[cuts[:-1]]
    assert per.max() <= p.a.nnz / blocks + np.diff(rp).max() + 1


def test_shard_cuts_edge_cases():
    cuts, ok = solver.shard_cuts(np.array([0, 2, 1, 3], np.uint32), 3, 2)  # decreasing
    assert not ok and list(cuts) == [0, 3, 3]
    cuts, ok = solver.shard_cuts(np.array([0, 1, 2], np.uint32), 5, 2)  # end != nnz
    assert not ok
    cuts, ok = solver.shard_cuts(np.array([0, 4], np.uint32), 4, 4)  # more blocks than rows
    assert ok and list(cuts) == [0, 1, 1, 1, 1]
    cuts, ok = solver.shard_cuts(np.array([0], np.uint32), 0, 3)  # m = 0
    assert ok and list(cuts) == [0, 0, 0, 0]


def row_block(a: CsrMatrix, r0: int, r1: int) -> CsrMatrix:
    e0, e1 = int(a.row_ptr[r0]), int(a.row_ptr[r1])
    return CsrMatrix(r1 - r0, a.cols, a.values[e0:e1].copy(),
                     (a.row_ptr[r0:r1 + 1] - e0).astype(np.uint32), a.col_indices[e0:e1].copy())


def seq_sumsq(vals):
    s = 0.0
    for v in vals:
        s += v * v
    return s


def _worker(rank, world, port, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        p = G.generate("lasso", 3, 1)
        pf = O.symmetrize_upper(p.p_upper)
        a, at = p.a, O.transpose(p.a)
        cuts, ok = solver.shard_cuts(a.row_ptr, a.nnz, world)
        assert ok
        r0, r1 = int(cuts[rank]), int(cuts[rank + 1])
        ag = row_block(a, r0, r1)
        agt = O.transpose(ag)
        # block transpose == the global transpose's entries from this block's rows
        for c in range(p.n):
            b, e = int(at.row_ptr[c]), int(at.row_ptr[c + 1])
            src = at.col_indices[b:e].astype(np.int64)
            sel = (src >= r0) & (src < r1)
            gb, ge = int(agt.row_ptr[c]), int(agt.row_ptr[c + 1])
            assert np.array_equal(agt.col_indices[gb:ge].astype(np.int64), src[sel] - r0)
            assert np.array_equal(agt.values[gb:ge], at.values[b:e][sel])
        sigma, rho = 1e-6, 0.1
        # K-apply: t_g = rho A_g x local; s = sum_g A_g^T t_g (allreduce); Kx = P x + sigma x + s
        x = np.random.default_rng(5).standard_normal(p.n)
        t = O.spmv(ag, x) * rho
        s = torch.from_numpy(O.spmv(agt, t))
        dist.all_reduce(s)
        kx = (O.spmv(pf, x) + sigma * x) + s.numpy()
        ref, _ = O.kkt_apply(pf, a, at, sigma, rho, x)
        assert np.allclose(kx, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
        # Ruiz column norms: max over blocks is exact
        colmax = torch.from_numpy(np.array([np.abs(agt.values[agt.row_ptr[c]:agt.row_ptr[c + 1]]).max(initial=0.0)
                                            for c in range(p.n)]))
        dist.all_reduce(colmax, op=dist.ReduceOp.MAX)
        full = np.array([np.abs(at.values[at.row_ptr[c]:at.row_ptr[c + 1]]).max(initial=0.0)
                         for c in range(p.n)])
        assert np.array_equal(colmax.numpy(), full)
        # diag(A^T A): sequential chain through the blocks in row order (bit-exact)
        acc = torch.zeros(p.n, dtype=torch.float64)
        if rank > 0:
            dist.recv(acc, src=rank - 1)
        av = acc.numpy()
        for c in range(p.n):
            s_ = av[c]
            for v in agt.values[agt.row_ptr[c]:agt.row_ptr[c + 1]]:
                s_ += v * v
            av[c] = s_
        if rank + 1 < world:
            dist.send(acc, dst=rank + 1)
        dist.broadcast(acc, src=world - 1)
        seq = np.array([seq_sumsq(at.values[at.row_ptr[c]:at.row_ptr[c + 1]]) for c in range(p.n)])
        assert np.array_equal(acc.numpy(), seq)
        # sharded PCG (linsys.hpp:190-276 with the A^T partial allreduce) vs the oracle
        diag_p = np.array([next((pf.values[k] for k in range(pf.row_ptr[i], pf.row_ptr[i + 1])
                                 if pf.col_indices[k] == i), 0.0) for i in range(p.n)])
        dinv = 1.0 / ((diag_p + sigma) + rho * seq)

        def K(v):
            sg = torch.from_numpy(O.spmv(agt, O.spmv(ag, v) * rho))
            dist.all_reduce(sg)
            return (O.spmv(pf, v) + sigma * v) + sg.numpy()

        b = np.random.default_rng(9).standard_normal(p.n)
        eps, cap = 1e-10, O.pcg_cap(p.n)
        xk = np.zeros(p.n)
        r = K(xk) - b
        y = dinv * r
        pk = -y
        rm = r @ y
        k = 0
        thr = eps * np.abs(b).max()
        while np.abs(r).max() > thr and k < cap and rm != 0:
            kp = K(pk)
            al = rm / (pk @ kp)
            xk = xk + al * pk
            r = r + al * kp
            y = dinv * r
            rn = r @ y
            pk = -y + (rn / rm) * pk
            rm = rn
            k += 1
        xo, ko, _, conv = O.pcg(pf, a, at, sigma, rho, b, np.zeros(p.n), eps, cap)
        out[rank] = (k, ko, float(np.abs(xk - xo).max() / max(1.0, np.abs(xo).max())), conv)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_algorithm_gloo_world2():
    torch.set_num_threads(1)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in (0, 1):
        k, ko, dx, conv = out[rank]
        assert conv
        assert abs(k - ko) <= 2, (k, ko)
        assert dx < 1e-8, dx
    assert out[0] == out[1]  # identical decisions and values on every rank
