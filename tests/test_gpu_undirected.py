"""GPU parity for undirected motifs: libvdmc.so's VDMC_UNDIRECTED kind
(through the C ABI) vs the oracle's count_undirected, bit-exact uint64, on small fixtures, the
heavy/light paths, random orders, slices, and full BASELINE sizes (sampled rows + invariant)."""
import numpy as np
import pytest

import graphgen as G
from test_gpu_parity import _fixtures, _sample_vertices

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


def ucount(vd, g, k, rank=None, options=None):
    import torch
    n, s, d = g
    gr = vd.Graph(n, torch.from_numpy(np.ascontiguousarray(s, np.int32)).cuda(),
                  torch.from_numpy(np.ascontiguousarray(d, np.int32)).cuda(), rank=rank)
    out = gr.count(k, kind="undirected", options=options).cpu().numpy().view(np.uint64)
    gr.close()
    return out


@pytest.mark.parametrize("k", [3, 4])
def test_class_ids(vd, oracle_mod, k):
    assert vd.class_ids(k, "undirected").tolist() == oracle_mod.undirected_class_ids(k).tolist()
    assert vd.num_classes(k, "undirected") == (2 if k == 3 else 6)


@pytest.mark.parametrize("k", [3, 4])
def test_small_fixtures(vd, oracle_mod, k):
    for name, g in _fixtures():
        assert np.array_equal(ucount(vd, g, k), oracle_mod.count_undirected(g, k, method="brute")), name


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("mode", ["smem", "global", "random-rank", "all", "enum"])
def test_heavy_and_light_paths(vd, oracle_mod, k, mode):
    g = G.make_config("cfg3", scale=0.03)
    opts = {"global": {"heavy_global": 1, "force_big": 1},
            "enum": {"star_block": 1023},   # the enumerated heavy path (default: closed form)
            "all": {"star_block": 5, "cross_block": 33, "force_big": 1, "ca_capacity": 7}}.get(mode)
    rank = np.random.default_rng(5).permutation(g[0]) if mode == "random-rank" else None
    assert np.array_equal(ucount(vd, g, k, rank=rank, options=opts), oracle_mod.count_undirected(g, k))


def test_slices_sum_to_full(vd):
    import torch
    g = G.make_config("cfg3", scale=0.01)
    gr = vd.Graph(g[0], torch.from_numpy(g[1]).cuda(), torch.from_numpy(g[2]).cuda())
    full = gr.count(4, kind="undirected").clone()
    acc = torch.zeros_like(full)
    for s in gr.plan(4, 3):
        acc += gr.count(4, work=s, kind="undirected")
    assert torch.equal(acc, full)
    gr.close()


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_configs_full_matrix(vd, oracle_mod, name):
    g = G.make_config(name)
    if name == "cfg3":
        g = G.make_config(name, scale=0.05)
    assert np.array_equal(ucount(vd, g, 4), oracle_mod.count_undirected(g, 4))


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_full_size_sampled_rows(vd, oracle_mod, name):
    import torch
    g = G.make_config(name)
    gr = vd.Graph(g[0], torch.from_numpy(g[1]).cuda(), torch.from_numpy(g[2]).cuda())
    out = gr.count(4, kind="undirected")
    assert np.all(out.sum(dim=0).cpu().numpy().view(np.uint64) % 4 == 0)
    host = out.cpu().numpy().view(np.uint64)
    gr.close()
    verts = _sample_vertices(g, 4, 16, 2e7, seed=11)
    assert np.array_equal(host[verts], oracle_mod.count_vertex_undirected(g, 4, verts))
