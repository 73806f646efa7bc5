"""Full-size parity on the hub (heavy) path -- the paths the kernel takes only at BASELINE size.

* cfg4 (n = 1M) built with the identity order: preferential-attachment hubs are the low ids,
  so a root's task slice (vdmc_root_range) holds exactly the connected 4-sets whose minimum
  original id is that root -- the oracle's count_esu(g, 4, r, r + 1) (Lemma 1, P:142-146;
  per-member increment P:118).  Roots with forward degree > 1024 run star items over more than
  one 1023-wide b block and cross items over more than 3 position blocks.
* A star centre whose row exceeds 2^32: closed form (every triple of leaves with the centre
  is a connected 4-set; its class depends only on the three leaf codes unless leaf-leaf arcs
  are present, whose triples are enumerated and classified with the oracle's table).
* Rank invariance at full size (Lemma 1 holds for every order): cfg4 and cfg5 counted
  under the default order and under a random order are bit-identical.
"""
import math
import threading
from collections import Counter
from itertools import combinations

import numpy as np
import pytest

import graphgen as G

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


def _forward_degrees(g):
    n, s, d = g
    a = np.minimum(s, d).astype(np.int64)
    b = np.maximum(s, d).astype(np.int64)
    key = np.unique(a * n + b)
    return np.bincount(key // n, minlength=n)


@pytest.mark.slow
def test_cfg4_hub_roots_identity_order(vd, oracle_mod):
    """Three cfg4 roots with forward degree in [1024, 1100] (about 2.7e8 sets each): the GPU's
    task slice of each root vs the oracle's per-root ESU, whole n x 199 partial matrices.  The
    oracle roots run in parallel host threads (ctypes releases the GIL)."""
    g = G.make_config("cfg4")
    fwd = _forward_degrees(g)
    roots = [int(r) for r in np.nonzero((fwd >= 1024) & (fwd <= 1100))[0][-3:]]
    assert len(roots) == 3
    want = {}

    def oracle_root(r):
        want[r] = oracle_mod.count_esu(g, 4, r, r + 1, threads=1)

    th = [threading.Thread(target=oracle_root, args=(r,)) for r in roots]
    for t in th:
        t.start()
    gr = _dev_graph(vd, g, rank=np.arange(g[0], dtype=np.int32))
    got = {}
    for r in roots:
        lo, hi = gr.root_range(r, r + 1)
        assert hi - lo == fwd[r]
        got[r] = gr.count(4, work=(lo, hi)).cpu().numpy().view(np.uint64)
        # the same slice with the forced path options: the enumerated heavy path (every set
        # visited, 1023-wide star blocks; and with every fallback forced) and the closed form with
        # global buffers and per-item flushes: still the same partial
        for opts in ({"star_block": 1023},
                     {"heavy_global": 1, "ca_capacity": 4096, "force_big": 1, "star_block": 300, "cross_block": 100},
                     {"heavy_global": 1, "force_big": 1}):
            alt = gr.count(4, work=(lo, hi), options=opts)
            assert np.array_equal(alt.cpu().numpy().view(np.uint64), got[r]), (r, opts)
    gr.close()
    for t in th:
        t.join()
    for r in roots:
        assert got[r].sum(dtype=np.uint64) > 8 * 10 ** 8   # k x (sets rooted at r), about 4 x 2.5e8
        assert np.array_equal(got[r], want[r]), r


def _star_graph(leaves, extra, seed):
    """Centre 0 and `leaves` leaves with random arc codes (1: 0 -> x, 2: x -> 0, 3: both), plus
    `extra` random leaf-leaf pairs with random codes."""
    rng = np.random.default_rng(seed)
    code = rng.integers(1, 4, leaves)
    src, dst = [], []
    for i, c in enumerate(code.tolist()):
        x = i + 1
        if c & 1:
            src.append(0), dst.append(x)
        if c & 2:
            src.append(x), dst.append(0)
    pairs = set()
    while len(pairs) < extra:
        x, y = sorted(rng.choice(leaves, 2, replace=False).tolist())
        pairs.add((x + 1, y + 1))
    ll = {}
    for (x, y) in sorted(pairs):
        c = int(rng.integers(1, 4))
        ll[(x, y)] = c
        if c & 1:
            src.append(x), dst.append(y)
        if c & 2:
            src.append(y), dst.append(x)
    return (leaves + 1, np.array(src, np.int32), np.array(dst, np.int32)), code, ll


def _col_of(t, arcs):
    """Column of the 4-vertex digraph with arc set `arcs` over vertices 0..3 (paper index
    P:81, Fig. 1, then the oracle's min-isomorph table)."""
    idx = 0
    for i in range(4):
        for j in range(4):
            if i != j:
                idx = (idx << 1) | ((i, j) in arcs)
    return int(t["col"][idx])


def test_star_centre_row_above_2_32(vd, oracle_mod):
    """Centre row of a 6000-leaf star with 300 leaf-leaf pairs: C(6000, 3) = 3.6e10 > 2^32
    connected 4-sets; expected row by closed form over leaf-code multisets, corrected by
    explicit enumeration of the (few) triples that contain a leaf-leaf pair."""
    L, E = 6000, 300
    g, code, ll = _star_graph(L, E, 42)
    t = oracle_mod.class_table(4)

    def arcs_for(codes3, pairs3):
        arcs = set()
        for i, c in enumerate(codes3):
            if c & 1:
                arcs.add((0, i + 1))
            if c & 2:
                arcs.add((i + 1, 0))
        for (i, j), c in pairs3.items():
            if c & 1:
                arcs.add((i + 1, j + 1))
            if c & 2:
                arcs.add((j + 1, i + 1))
        return arcs

    nc = Counter(code.tolist())
    want = np.zeros(len(t["class_ids"]), dtype=object)
    for combo in {tuple(sorted(x)) for x in combinations([1, 1, 1, 2, 2, 2, 3, 3, 3], 3)}:
        cnt = Counter(combo)
        ways = 1
        for c, m in cnt.items():
            ways *= math.comb(nc[c], m)
        want[_col_of(t, arcs_for(combo, {}))] += ways
    # triples containing at least one leaf-leaf pair: move them from the plain star class
    adj = {}
    for (x, y), c in ll.items():
        adj.setdefault(x, {})[y] = c
        adj.setdefault(y, {})[x] = c if c == 3 else 3 - c   # code seen from y
    tri = set()
    for (x, y) in ll:
        for z in range(1, L + 1):
            if z != x and z != y:
                tri.add(tuple(sorted((x, y, z))))
    for tr in tri:
        cs = [int(code[v - 1]) for v in tr]
        pairs3 = {}
        for i, j in ((0, 1), (0, 2), (1, 2)):
            c = adj.get(tr[i], {}).get(tr[j])
            if c:
                pairs3[(i, j)] = c
        want[_col_of(t, arcs_for(cs, {}))] -= 1
        want[_col_of(t, arcs_for(cs, pairs3))] += 1
    want = np.array([int(x) for x in want], dtype=np.uint64)
    assert int(want.sum(dtype=np.uint64)) == math.comb(L, 3) > 2 ** 32
    gr = _dev_graph(vd, g)
    for opts in ({}, {"heavy_global": 1}, {"force_big": 1, "star_block": 257}):
        row = gr.count(4, options=opts)[0].cpu().numpy().view(np.uint64)
        assert np.array_equal(row, want), opts
    # a few leaves (one with a leaf-leaf pair): the oracle's per-vertex ESU
    leaves = np.array([1, 2, next(iter(ll))[0]], np.int32)
    full = gr.count(4).cpu().numpy().view(np.uint64)
    assert np.array_equal(full[leaves], oracle_mod.count_vertex(g, 4, leaves))
    assert np.all(full.sum(axis=0, dtype=np.uint64) % np.uint64(4) == 0)
    gr.close()


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_rank_invariance_full_size(vd, name):
    """Lemma 1: the counts do not depend on the vertex order.  Full-size graph,
    default (degree-descending) order vs a random order: every uint64 entry identical."""
    import torch
    g = G.make_config(name)
    gr = _dev_graph(vd, g)
    a = gr.count(4)
    ha = a.sum(dim=0).cpu()
    gr.close()
    rank = np.random.default_rng(17).permutation(g[0]).astype(np.int32)
    gr = _dev_graph(vd, g, rank=rank)
    b = gr.count(4)
    assert torch.equal(a, b)
    assert torch.equal(b.sum(dim=0).cpu(), ha)
    gr.close()
