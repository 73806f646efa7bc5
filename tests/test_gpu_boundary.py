"""GPU tests of the rest of the C-ABI boundary (include/vdmc.h):
vdmc_symmetrize against the paper's worked CSR example, the immutable graph
shared by concurrent counts on two streams, per-call options and timings, root-range
slices, and the NCCL multi-GPU count (vdmc_count_distributed) on a one-rank communicator."""
import os
import socket
import threading

import numpy as np
import pytest

import graphgen as G
from conftest import read_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests need a B200")
    from paper_2201_11655_b200 import build as b
    b.build()
    from paper_2201_11655_b200 import vdmc
    return vdmc


def _dev_graph(vd, g, rank=None):
    import torch
    n, s, d = g
    return vd.Graph(n, torch.from_numpy(np.ascontiguousarray(s, np.int32)).cuda(),
                    torch.from_numpy(np.ascontiguousarray(d, np.int32)).cuda(), rank=rank)


def test_symmetrize_paper_example(vd):
    """arcs 0->1 0->2 0->3 2->0 3->1 3->2; directed Indices [0,3,3,4,6], Neighbors
    [1,2,3,0,1,2]; undirected Indices [0,3,5,7,10], Neighbors [1,2,3,0,3,0,3,0,1,2]."""
    ind, nbr, dirc = vd.symmetrize(4, [0, 3, 3, 4, 6], [1, 2, 3, 0, 1, 2])
    assert ind.tolist() == [0, 3, 5, 7, 10]
    assert nbr.tolist() == [1, 2, 3, 0, 3, 0, 3, 0, 1, 2]
    # codes: bit0 = v -> nbr, bit1 = nbr -> v (0<->2 is the one mutual pair: one entry, code 3)
    assert dirc.tolist() == [1, 3, 1, 2, 2, 3, 2, 2, 1, 1]


def test_symmetrize_golden_file(vd):
    rows = {r[1]: r[2:] for r in read_golden("paper_example.txt") if r[0] == "csr"}
    ind, nbr, dirc = vd.symmetrize(4, [int(x) for x in rows["directed_indices"]],
                                   [int(x) for x in rows["directed_neighbors"]])
    assert ind.tolist() == [int(x) for x in rows["undirected_indices"]]
    assert nbr.tolist() == [int(x) for x in rows["undirected_neighbors"]]


def test_symmetrize_round_trip(vd, oracle_mod):
    """The paper's CSR of random digraphs (with duplicate arcs) -> vdmc_symmetrize ->
    vdmc_build_graph counts exactly what the edge-list build counts."""
    for seed in range(4):
        n, s, d = G.random_small(40, 0.15, 900 + seed)
        s = np.concatenate([s, s[:7]])
        d = np.concatenate([d, d[:7]])
        o = np.lexsort((d, s))
        ind = np.zeros(n + 1, np.int64)
        np.add.at(ind, s[o] + 1, 1)
        ind = np.cumsum(ind)
        sym = vd.symmetrize(n, ind, d[o])
        assert sym[0][-1] == sym[1].size
        for k in (3, 4):
            gr = vd.Graph.from_sym_csr(n, *sym)
            assert np.array_equal(gr.count(k).cpu().numpy().view(np.uint64), oracle_mod.count_esu((n, s, d), k))
            gr.close()


def test_symmetrize_errors(vd):
    with pytest.raises(vd.VdmcError, match="ESELFLOOP"):
        vd.symmetrize(3, [0, 1, 1, 1], [0])
    with pytest.raises(vd.VdmcError, match="ERANGE"):
        vd.symmetrize(3, [0, 1, 1, 1], [9])
    with pytest.raises(vd.VdmcError, match="EINVAL"):
        vd.symmetrize(3, [0, 2, 1, 1], [1, 2])
    ind, nbr, dirc = vd.symmetrize(3, [0, 0, 0, 0], [])
    assert ind.tolist() == [0, 0, 0, 0] and nbr.size == 0 and dirc.size == 0


def test_concurrent_counts_two_streams(vd, oracle_mod):
    """The graph is immutable: counts of k = 3 and k = 4 (and two k = 4 with different path
    options) issued concurrently on two streams from two host threads equal sequential ones."""
    import torch
    g = G.make_config("cfg3", scale=0.03)
    gr = _dev_graph(vd, g)
    want = {3: oracle_mod.count_esu(g, 3), 4: oracle_mod.count_esu(g, 4)}
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = [(4, {}), (3, {}), (4, {"ca_capacity": 5, "star_block": 17}), (4, {"heavy_global": 1})]
    for rep in range(3):
        res = [None] * len(jobs)
        errs = []

        def run(i):
            try:
                k, opt = jobs[i]
                st = streams[i % 2]
                with torch.cuda.stream(st):
                    out = gr.count(k, stream=st, options=opt)
                st.synchronize()
                res[i] = out.cpu().numpy().view(np.uint64)
            except Exception as e:   # surfaced below
                errs.append(e)

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for (k, _), r in zip(jobs, res):
            assert np.array_equal(r, want[k]), (rep, k)
    gr.close()


def test_timings_and_options_validation(vd):
    g = G.make_config("cfg3", scale=0.01)
    gr = _dev_graph(vd, g)
    assert gr.info["build_ms"] > 0
    tm = {}
    gr.count(4, timings=tm)
    assert set(tm) == {"schedule", "enum", "finalize", "count"} and tm["enum"] > 0 and tm["count"] >= tm["enum"]
    for bad in ({"star_block": 2000}, {"cross_block": 5}, {"heavy_global": 2}, {"ca_capacity": -1}):
        with pytest.raises(vd.VdmcError, match="EINVAL"):
            gr.count(4, options=bad)
    with pytest.raises(ValueError):
        gr.count(4, options={"nope": 1})
    gr.close()


def test_root_range_slices(vd, oracle_mod):
    """Root-range slices (vdmc_root_range over order positions) partition the task list;
    their partials sum to the full matrix, and a single root's slice equals the oracle's
    per-root count under the same (identity) order."""
    import torch
    g = G.make_config("cfg3", scale=0.01)
    n = g[0]
    gr = _dev_graph(vd, g, rank=np.arange(n))
    full = gr.count(4).clone()
    cuts = [0, 1, 7, 100, n // 2, n]
    acc = torch.zeros_like(full)
    for a, b in zip(cuts[:-1], cuts[1:]):
        acc += gr.count(4, work=gr.root_range(a, b))
    assert torch.equal(acc, full)
    assert gr.root_range(0, n) == (0, gr.ntasks)
    for r in (0, 3, 50):
        got = gr.count(4, work=gr.root_range(r, r + 1)).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, oracle_mod.count_esu(g, 4, r, r + 1)), r
    gr.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_count_distributed_nccl_one_rank(vd, oracle_mod):
    """vdmc_count_distributed on a one-rank NCCL communicator (the box has one GPU): plan,
    slice count into the class-major partial, ncclReduce, finalise on the root."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = vd.Comm(device=0)
        g = G.make_config("cfg3", scale=0.02)
        gr = _dev_graph(vd, g)
        for k in (3, 4):
            out = vd.count_distributed(gr, k, comm)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle_mod.count_esu(g, k))
        out = vd.count_distributed(gr, 4, comm, kind="undirected")
        assert np.array_equal(out.cpu().numpy().view(np.uint64), oracle_mod.count_undirected(g, 4))
        with pytest.raises(vd.VdmcError, match="EINVAL"):
            vd.count_distributed(gr, 4, comm, root=1)
        gr.close()
        comm.close()
    finally:
        dist.destroy_process_group()
