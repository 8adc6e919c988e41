"""The row-sharded engine across PROCESSES over the peer-memory transport
(CUDA IPC mappings + device-side barriers), run here as 2 processes sharing
the one B200 (the same code maps NVLink peers across GPUs).  Each process
holds its rank's row blocks; the partials are summed in block order, so the
result must be bitwise identical to ONE process holding all the blocks as
virtual shards."""
import multiprocessing as mp
import os
import tempfile

import numpy as np
import pytest

from paper_1912_04263_b200 import generators as G, solver
from paper_1912_04263_b200.problem import Settings

pytestmark = pytest.mark.gpu
S = Settings(lambda_pcg=0.01)


def _rank(rank, ranks, local, rdir, cls, scale, q, mode="graph"):
    try:
        p = G.generate(cls, scale, 0)
        r = solver.solve(p, S, device=0, shards=local, peer=(rank, ranks, rdir), mode=mode)
        q.put((rank, r.status, r.iterations, r.pcg_iterations_total, r.x, r.z, r.y, r.objective,
               r.info["kernel_launches"]))
    except Exception as e:  # reported to the parent
        q.put((rank, "exception", repr(e)))


def run_ranks(ranks, local, cls, scale, mode="graph"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as rdir:
        procs = [ctx.Process(target=_rank, args=(r, ranks, local, rdir, cls, scale, q, mode))
                 for r in range(ranks)]
        for pr in procs:
            pr.start()
        out = {}
        try:
            for _ in range(ranks):
                item = q.get(timeout=600)
                out[item[0]] = item
        finally:
            for pr in procs:
                pr.join(timeout=60)
                if pr.is_alive():
                    pr.terminate()
    return out


@pytest.mark.parametrize("cls,scale,ranks,local,mode", [("lasso", 4, 2, 1, "graph"),
                                                        ("huber", 3, 2, 2, "graph"),
                                                        ("svm", 3, 2, 1, "eager")])
def test_peer_transport_two_processes_bitwise_equal_virtual(cls, scale, ranks, local, mode):
    """mode graph: the whole sharded loop as one CUDA graph per process, the
    peer stores / device barriers inside it; eager: the host-driven loop."""
    out = run_ranks(ranks, local, cls, scale, mode)
    for r in range(ranks):
        assert out[r][1] != "exception", out[r]
    p = G.generate(cls, scale, 0)
    v = solver.solve(p, S, device=0, shards=ranks * local)  # one process, virtual blocks
    for r in range(ranks):
        _, status, it, pcg, x, z, y, obj, _ = out[r]
        assert status == v.status and it == v.iterations and pcg == v.pcg_iterations_total
        assert np.array_equal(x, v.x) and np.array_equal(z, v.z) and np.array_equal(y, v.y)
        assert obj == v.objective
