"""GPU parity of 5-vertex motifs ("appropriate for 5 motifs too") and
of the generic BFS-layer path (layers.cu) at k = 3 / 4: vdmc_count(k = 5) / option layered=1
through the C ABI vs the oracle (brute force / ESU / per-vertex ESU), bit-exact uint64."""
import numpy as np
import pytest

import graphgen as G
from test_gpu_parity import _fixtures

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


def gcount(vd, g, k, rank=None, kind="directed", options=None, work=None):
    import torch
    n, s, d = g
    gr = vd.Graph(n, torch.from_numpy(np.ascontiguousarray(s, np.int32)).cuda(),
                  torch.from_numpy(np.ascontiguousarray(d, np.int32)).cuda(), rank=rank)
    out = gr.count(k, kind=kind, options=options).cpu().numpy().view(np.uint64)
    gr.close()
    return out


def test_small_fixtures_k5_vs_brute_force(vd, oracle_mod):
    for name, g in _fixtures()[::3]:
        if g[0] > 24:
            continue
        assert np.array_equal(gcount(vd, g, 5), oracle_mod.count_brute(g, 5)), name


@pytest.mark.parametrize("k", [3, 4])
def test_layered_path_k34(vd, oracle_mod, k):
    """The generic path at k = 3 / 4 equals the oracle (and so the specialised kernels)."""
    for name, g in _fixtures()[::4]:
        assert np.array_equal(gcount(vd, g, k, options={"layered": 1}), oracle_mod.count_brute(g, k)), name
    g = G.make_config("cfg3", scale=0.01)
    assert np.array_equal(gcount(vd, g, k, options={"layered": 1}), oracle_mod.count_esu(g, k))


def test_single_motif_graphs_k5(vd, oracle_mod):
    """Every one of the 9364 classes as its own 5-vertex component (its canonical matrix), randomly
    relabelled: each member gets exactly 1 in that class."""
    t = oracle_mod.class_table(5)
    ids = t["class_ids"]
    order = [(i, j) for i in range(5) for j in range(5) if i != j]
    src, dst = [], []
    for c, m in enumerate(ids):
        for b, (i, j) in enumerate(order):
            if (int(m) >> (19 - b)) & 1:
                src.append(c * 5 + i)
                dst.append(c * 5 + j)
    n = len(ids) * 5
    perm = np.random.default_rng(55).permutation(n)
    g = G.relabel((n, np.array(src), np.array(dst)), perm)
    import torch
    gr = vd.Graph(n, torch.from_numpy(g[1].astype(np.int32)).cuda(), torch.from_numpy(g[2].astype(np.int32)).cuda())
    out = gr.count(5)                                   # [46820][9364] on the device: compare there
    want_col = np.empty(n, np.int64)
    want_col[perm] = np.repeat(np.arange(len(ids)), 5)  # vertex perm[c*5+i] belongs to component c
    assert torch.equal(out.sum(dim=1).cpu(), torch.ones(n, dtype=torch.int64))
    assert torch.equal(out.argmax(dim=1).cpu(), torch.from_numpy(want_col))
    gr.close()


@pytest.mark.parametrize("name,scale", [("cfg2", 0.05), ("cfg3", 0.002), ("cfg5", 0.0004)])
def test_scaled_configs_k5(vd, oracle_mod, name, scale):
    g = G.make_config(name, scale=scale)
    assert np.array_equal(gcount(vd, g, 5), oracle_mod.count_esu(g, 5))


def test_rank_invariance_and_slices_k5(vd, oracle_mod):
    import torch
    g = G.make_config("cfg3", scale=0.002)
    want = oracle_mod.count_esu(g, 5)
    rank = np.random.default_rng(4).permutation(g[0])
    assert np.array_equal(gcount(vd, g, 5, rank=rank), want)
    n, s, d = g
    gr = vd.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    acc = None
    for sl in gr.plan(4, 3):
        x = gr.count(5, work=sl)
        acc = x.clone() if acc is None else acc + x
    assert np.array_equal(acc.cpu().numpy().view(np.uint64), want)
    gr.close()


def test_undirected_k5(vd, oracle_mod):
    g = G.make_config("cfg3", scale=0.002)
    assert np.array_equal(gcount(vd, g, 5, kind="undirected"), oracle_mod.count_undirected(g, 5))


def test_cfg2_full_size_sampled_rows_k5(vd, oracle_mod):
    """cfg2 at full size (ER n = 20 000, p = 5e-4): sampled rows vs the oracle's per-vertex ESU and
    the k x census invariant over the whole n x 9364 matrix."""
    import torch
    g = G.make_config("cfg2")
    n, s, d = g
    gr = vd.Graph(n, torch.from_numpy(s).cuda(), torch.from_numpy(d).cuda())
    out = gr.count(5)
    assert np.all(out.sum(dim=0).cpu().numpy().view(np.uint64) % np.uint64(5) == 0)
    host = out.cpu().numpy().view(np.uint64)
    gr.close()
    verts = np.random.default_rng(2).choice(n, 24, replace=False).astype(np.int32)
    assert np.array_equal(host[verts], oracle_mod.count_vertex(g, 5, verts))
