"""N > 1 host logic on CPU (gloo, world size 2): vdmc.count_slices_reduce slices the task list
with the planner's cost-balanced split, counts each slice into a private partial and
reduces to rank 0.  The graph object is duck-typed: plan()/count() are served by the oracle
over root ranges (the counting itself is the GPU's job and is covered by -m gpu), so this
checks the partition bookkeeping, the reduce and the uint64-as-int64 bit handling."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as G


class OracleSliceGraph:
    """plan/count over 'tasks' = roots in original-id order (one task per root)."""

    def __init__(self, g, k):
        import oracle
        from paper_2201_11655_b200 import vdmc
        self.g, self.k, self.oracle, self.vdmc = g, k, oracle, vdmc
        n = g[0]
        deg = np.bincount(np.concatenate([g[1], g[2]]), minlength=n)
        self.prefix = np.cumsum(1 + deg.astype(np.int64) ** 3)

    def plan(self, k, nparts):
        return self.vdmc.split_costs(self.prefix, nparts)

    def count(self, k, work=None, kind="directed"):
        lo, hi = work if work is not None else (0, self.g[0])
        out = self.oracle.count_esu(self.g, k, lo, hi, threads=1)
        return torch.from_numpy(out.view(np.int64).copy())


def _worker(rank, world, port, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_11655_b200 import vdmc
        g = G.make_config("cfg3", scale=0.004)
        sg = OracleSliceGraph(g, k)
        parts = sg.plan(k, world)
        out = vdmc.count_slices_reduce(sg, k)
        if rank == 0:
            q.put((parts, out.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("k", [3, 4])
def test_count_distributed_world2(oracle_mod, k):
    from paper_2201_11655_b200 import build as b
    b.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts, got = q.get(timeout=300)   # drain before join: a large message blocks the writer
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    g = G.make_config("cfg3", scale=0.004)
    assert parts[0][0] == 0 and parts[-1][1] == g[0] and parts[0][1] == parts[1][0]
    assert np.array_equal(got, oracle_mod.count_esu(g, k))
