"""Pins of the oracle's edge-level counts ("counting motifs
for edges, rather than vertices ... only requires updating edges and not vertices"): every
connected k-set adds one, in its class, to each G_U edge inside it.

Pinned by things other than the oracle itself: a hand-derived golden of the paper's example
graph, closed forms (complete digraphs, stars, directed cycles), a table-free pure-Python brute
force, the census identity sum_e counts[e][j] = edges(class j) x census_j against the (pinned)
vertex counts, and the regular-class degree identity sum_{e ∋ v} counts[e][j] = d x counts[v][j].
"""
import math

import numpy as np
import pytest

import graphgen as G
from conftest import read_golden


def _col(oracle_mod, k, cid):
    return list(oracle_mod.class_table(k)["class_ids"]).index(cid)


def test_edge_list_paper_example(oracle_mod):
    eu, ev = oracle_mod.edge_list(G.paper_example())
    assert list(zip(eu.tolist(), ev.tolist())) == [(0, 1), (0, 2), (0, 3), (1, 3), (2, 3)]


@pytest.mark.parametrize("k", [3, 4])
def test_paper_example_golden(oracle_mod, k):
    g = G.paper_example()
    eu, ev = oracle_mod.edge_list(g)
    rows = {(int(r[1]), int(r[2])): r[3:] for r in read_golden("paper_example_edges.txt") if r[0] == f"k{k}"}
    want = np.zeros((eu.size, oracle_mod.num_classes(k)), np.uint64)
    for i, (u, v) in enumerate(zip(eu.tolist(), ev.tolist())):
        for item in rows[(u, v)]:
            cid, cnt = item.split(":")
            want[i, _col(oracle_mod, k, int(cid))] = int(cnt)
    assert np.array_equal(oracle_mod.count_edges_brute(g, k), want)
    assert np.array_equal(oracle_mod.count_edges_esu(g, k), want)


@pytest.mark.parametrize("k", [3, 4])
def test_closed_forms(oracle_mod, k):
    C = oracle_mod.num_classes(k)
    # complete digraph K_n: every edge lies in C(n-2, k-2) sets, all complete (63 / 4095)
    for n in (5, 7):
        out = oracle_mod.count_edges_esu(G.complete_digraph(n), k)
        want = np.zeros((math.comb(n, 2), C), np.uint64)
        want[:, _col(oracle_mod, k, 63 if k == 3 else 4095)] = math.comb(n - 2, k - 2)
        assert np.array_equal(out, want)
    # out-star / in-star with L leaves: each edge in C(L-1, k-2) sets of the star class
    for L in (6, 9):
        for g, cid in ((G.out_star(L), 3 if k == 3 else 7), (G.in_star(L), 10 if k == 3 else 292)):
            out = oracle_mod.count_edges_brute(g, k)
            want = np.zeros((L, C), np.uint64)
            want[:, _col(oracle_mod, k, cid)] = math.comb(L - 1, k - 2)
            assert np.array_equal(out, want)
    # directed cycle C_n, n > k: the k-sets are the n windows (directed paths 6 / 84); an edge
    # lies in the k - 1 windows that contain both its ends
    for n in (7, 9):
        out = oracle_mod.count_edges_esu(G.directed_cycle(n), k)
        want = np.zeros((n, C), np.uint64)
        want[:, _col(oracle_mod, k, 6 if k == 3 else 84)] = k - 1
        assert np.array_equal(out, want)


def _py_dense(oracle_mod, g, k):
    eu, ev = oracle_mod.edge_list(g)
    idx = {(u, v): i for i, (u, v) in enumerate(zip(eu.tolist(), ev.tolist()))}
    ids = list(oracle_mod.class_table(k)["class_ids"])
    out = np.zeros((eu.size, len(ids)), np.uint64)
    for (e, cid), x in oracle_mod.count_edges_py(g, k).items():
        out[idx[e], ids.index(cid)] = x
    return out


@pytest.mark.parametrize("k", [3, 4])
def test_brute_and_esu_vs_pure_python(oracle_mod, k):
    for seed in range(12):
        g = G.random_small(7 + seed % 4, (0.2, 0.4, 0.6)[seed % 3], 4100 + seed)
        want = _py_dense(oracle_mod, g, k)
        assert np.array_equal(oracle_mod.count_edges_brute(g, k), want), seed
        assert np.array_equal(oracle_mod.count_edges_esu(g, k), want), seed


def _class_edges(oracle_mod, k):
    """Number of G_U edges (unordered pairs with an arc either way) of each class, from its
    canonical paper index (P:81 bit order: pair (i, j), i != j, row-major, MSB first)."""
    pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(pairs)
    out = []
    for cid in oracle_mod.class_table(k)["class_ids"]:
        und = {tuple(sorted(pairs[b])) for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}
        out.append(len(und))
    return np.array(out, np.uint64)


def _class_regular_degree(oracle_mod, k):
    """d if the class's underlying undirected graph is d-regular, else 0."""
    pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(pairs)
    out = []
    for cid in oracle_mod.class_table(k)["class_ids"]:
        deg = [0] * k
        for (i, j) in {tuple(sorted(pairs[b])) for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}:
            deg[i] += 1
            deg[j] += 1
        out.append(deg[0] if len(set(deg)) == 1 else 0)
    return np.array(out, np.uint64)


@pytest.mark.parametrize("k", [3, 4])
def test_census_and_degree_identities(oracle_mod, k):
    """sum_e counts_e[e][j] = |E(class j)| x census_j (census_j = sum_v counts_v[v][j] / k), and for
    d-regular classes sum_{e ∋ v} counts_e[e][j] = d x counts_v[v][j] -- on BA and ER graphs."""
    ce = _class_edges(oracle_mod, k)
    reg = _class_regular_degree(oracle_mod, k)
    assert reg.any()
    for g in (G.make_config("cfg3", scale=0.002), G.gnp_directed(300, 0.03, 12), G.random_small(40, 0.3, 3)):
        ev_ = oracle_mod.count_edges_esu(g, k)
        vx = oracle_mod.count_esu(g, k)
        census = vx.sum(axis=0, dtype=np.uint64) // np.uint64(k)
        assert np.array_equal(ev_.sum(axis=0, dtype=np.uint64), ce * census)
        eu, evv = oracle_mod.edge_list(g)
        inc = np.zeros_like(vx)
        np.add.at(inc, eu, ev_)
        np.add.at(inc, evv, ev_)
        cols = np.nonzero(reg)[0]
        assert np.array_equal(inc[:, cols], vx[:, cols] * reg[cols])


@pytest.mark.parametrize("k", [3, 4])
def test_root_range_partials(oracle_mod, k):
    g = G.make_config("cfg3", scale=0.002)
    n = g[0]
    full = oracle_mod.count_edges_esu(g, k)
    acc = np.zeros_like(full)
    for lo, hi in ((0, 5), (5, 100), (100, n)):
        acc += oracle_mod.count_edges_esu(g, k, lo, hi)
    assert np.array_equal(acc, full)


@pytest.mark.parametrize("k", [3, 4])
def test_edge_rows_match_full(oracle_mod, k):
    """Per-edge rows (the full-size sampling oracle) equal the rows of the full matrix."""
    g = G.make_config("cfg3", scale=0.002)
    full = oracle_mod.count_edges_esu(g, k)
    eu, ev = oracle_mod.edge_list(g)
    pick = np.random.default_rng(k).choice(eu.size, 40, replace=False)
    for a, b in ((eu, ev), (ev, eu)):   # either end may be the ESU root
        assert np.array_equal(oracle_mod.count_edge_rows(g, k, a[pick], b[pick]), full[pick])
