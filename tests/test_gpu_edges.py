"""GPU parity of edge-level counts: vdmc_count_edges through the
C ABI vs the oracle's count_edges_{brute,esu}, bit-exact uint64 [edges][C] matrices, rows in the
canonical edge order (vdmc_get_edges = the oracle's edge_list)."""
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


def _graph(vd, g, rank=None):
    import torch
    n, s, d = g
    return vd.Graph(n, torch.from_numpy(np.ascontiguousarray(s, np.int32)).cuda(),
                    torch.from_numpy(np.ascontiguousarray(d, np.int32)).cuda(), rank=rank)


def ecount(vd, g, k, rank=None, kind="directed"):
    gr = _graph(vd, g, rank)
    out = gr.count_edges(k, kind=kind).cpu().numpy().view(np.uint64)
    u, v = gr.edges()
    gr.close()
    return out, u, v


def _undirected_edges(oracle_mod, g, k):
    sym = oracle_mod.symmetrize(g)
    full = oracle_mod.count_edges_esu(sym, k)
    ids = list(oracle_mod.class_table(k)["class_ids"])
    cols = [ids.index(c) for c in oracle_mod.undirected_class_ids(k)]
    return np.ascontiguousarray(full[:, cols])


@pytest.mark.parametrize("k", [3, 4])
def test_small_fixtures_vs_brute_force(vd, oracle_mod, k):
    for name, g in _fixtures():
        got, u, v = ecount(vd, g, k)
        eu, ev = oracle_mod.edge_list(g)
        assert np.array_equal(u, eu) and np.array_equal(v, ev), name
        assert np.array_equal(got, oracle_mod.count_edges_brute(g, k)), name


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("name,scale", [("cfg2", 1.0), ("cfg3", 0.03), ("cfg4", 0.004), ("cfg5", 0.002)])
def test_configs_full_matrix(vd, oracle_mod, name, scale, k):
    """Hubs (lists beyond the shared-memory slots: the global-scratch path) and uniform ER."""
    g = G.make_config(name, scale=scale)
    got, u, v = ecount(vd, g, k)
    eu, ev = oracle_mod.edge_list(g)
    assert np.array_equal(u, eu) and np.array_equal(v, ev)
    assert np.array_equal(got, oracle_mod.count_edges_esu(g, k))


@pytest.mark.parametrize("k", [3, 4])
def test_rank_invariance(vd, oracle_mod, k):
    g = G.make_config("cfg3", scale=0.01)
    want = oracle_mod.count_edges_esu(g, k)
    for seed in range(2):
        rank = np.random.default_rng(seed).permutation(g[0])
        assert np.array_equal(ecount(vd, g, k, rank=rank)[0], want)


@pytest.mark.parametrize("k", [3, 4])
def test_undirected_kind(vd, oracle_mod, k):
    g = G.make_config("cfg3", scale=0.01)
    assert np.array_equal(ecount(vd, g, k, kind="undirected")[0], _undirected_edges(oracle_mod, g, k))


def test_slices_and_census(vd, oracle_mod):
    """Slice partials sum to the full matrix; the census identity against the GPU's own vertex
    counts (sum_e counts_e[e][j] = |E(class j)| x sum_v counts_v[v][j] / k)."""
    import torch
    from test_oracle_edges import _class_edges
    g = G.make_config("cfg3", scale=0.02)
    gr = _graph(vd, g)
    full = gr.count_edges(4).clone()
    acc = torch.zeros_like(full)
    for sl in gr.plan(4, 3):
        acc += gr.count_edges(4, work=sl)
    assert torch.equal(acc, full)
    vx = gr.count(4).cpu().numpy().view(np.uint64)
    census = vx.sum(axis=0, dtype=np.uint64) // np.uint64(4)
    e = full.cpu().numpy().view(np.uint64).sum(axis=0, dtype=np.uint64)
    assert np.array_equal(e, _class_edges(oracle_mod, 4) * census)
    gr.close()


def test_edge_cases(vd):
    import torch
    empty = np.zeros(0, np.int32)
    for n in (0, 1, 3):
        out, u, v = ecount(vd, (n, empty, empty), 4)
        assert out.shape == (0, 199) and u.size == 0
    out, u, v = ecount(vd, (2, np.array([0, 1]), np.array([1, 0])), 3)
    assert out.shape == (1, 13) and not out.any() and u.tolist() == [0] and v.tolist() == [1]
    gr = _graph(vd, G.random_small(10, 0.3, 1))
    tm = {}
    gr.count_edges(4, timings=tm)
    assert tm["enum"] > 0
    with pytest.raises(vd.VdmcError, match="EK"):
        gr.count_edges(5)
    gr.close()
    del torch
