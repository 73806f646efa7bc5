"""Pins of the oracle at k = 5 ("Claims and data structure are
appropriate for 5 motifs too").  The definition is unchanged (P:81 index of the 5 x 5 adjacency
matrix, 20 bits, minimum over the 5! orders; P:118 per-member increment); pinned by textbook
counts (OEIS A003085: 9364 weakly connected digraphs on 5 nodes; A003027: 1,027,080 weakly
connected labelled ones), closed forms whose class ids are re-derived here in pure Python, a
table-free pure-Python brute force, and the k x census invariant."""
import itertools
import math

import numpy as np
import pytest

import graphgen as G

K = 5


def py_class(arcs, verts):
    """Minimum paper index (Fig. 1 bit order: rows, diagonal removed, MSB first) over the
    orders of `verts` -- pure Python, no table."""
    best = None
    for P in itertools.permutations(verts):
        bits = 0
        for i in range(K):
            for j in range(K):
                if i != j:
                    bits = (bits << 1) | ((P[i], P[j]) in arcs)
        best = bits if best is None else min(best, bits)
    return best


def col(oracle_mod, cid):
    return list(oracle_mod.class_table(K)["class_ids"]).index(cid)


def test_class_table_counts(oracle_mod):
    t = oracle_mod.class_table(K)
    assert len(t["class_ids"]) == 9364              # OEIS A003085(5)
    assert int(t["conn"].sum()) == 1027080          # OEIS A003027(5)
    assert t["canon"][(1 << 20) - 1] == (1 << 20) - 1 and not t["conn"][0]
    assert np.all(np.diff(t["class_ids"]) > 0)
    assert oracle_mod.n_iso(K).sum() == 1027080


def test_closed_forms(oracle_mod):
    C = oracle_mod.num_classes(K)
    # complete digraph: every vertex in C(n-1, 4) sets of class 2^20 - 1
    for n in (6, 7):
        out = oracle_mod.count_esu(G.complete_digraph(n), K)
        want = np.zeros((n, C), np.uint64)
        want[:, col(oracle_mod, (1 << 20) - 1)] = math.comb(n - 1, 4)
        assert np.array_equal(out, want)
    # transitive tournament (the "regular DAG" of P:218): C(n-1, 4) sets of the TT5 class
    g = G.transitive_tournament(7)
    arcs = set(zip(g[1].tolist(), g[2].tolist()))
    cid = py_class(arcs, (0, 1, 2, 3, 4))
    want = np.zeros((7, C), np.uint64)
    want[:, col(oracle_mod, cid)] = math.comb(6, 4)
    assert np.array_equal(oracle_mod.count_brute(g, K), want)
    # directed cycle, n > 5: each vertex in the 5 windows containing it, all directed 5-paths
    g = G.directed_cycle(9)
    arcs = set(zip(g[1].tolist(), g[2].tolist()))
    cid = py_class(arcs, (0, 1, 2, 3, 4))
    want = np.zeros((9, C), np.uint64)
    want[:, col(oracle_mod, cid)] = 5
    assert np.array_equal(oracle_mod.count_esu(g, K), want)
    # out-star with 7 leaves: centre C(7, 4), leaf C(6, 3)
    g = G.out_star(7)
    arcs = set(zip(g[1].tolist(), g[2].tolist()))
    cid = py_class(arcs, (0, 1, 2, 3, 4))
    out = oracle_mod.count_brute(g, K)
    j = col(oracle_mod, cid)
    assert out[0, j] == math.comb(7, 4) and np.all(out[1:, j] == math.comb(6, 3)) and out.sum() == 5 * math.comb(7, 4)


def test_brute_esu_vs_pure_python(oracle_mod):
    ids = list(oracle_mod.class_table(K)["class_ids"])
    for seed in range(6):
        g = G.random_small(7 + seed % 2, (0.3, 0.5)[seed % 2], 5100 + seed)
        n = g[0]
        want = np.zeros((n, len(ids)), np.uint64)
        for (v, cid), x in oracle_mod.count_py(g, K).items():
            want[v, ids.index(cid)] = x
        assert np.array_equal(oracle_mod.count_brute(g, K), want), seed
        assert np.array_equal(oracle_mod.count_esu(g, K), want), seed


def test_invariants_and_edges(oracle_mod):
    g = G.make_config("cfg3", scale=0.001)
    v = oracle_mod.count_esu(g, K)
    assert np.all(v.sum(axis=0, dtype=np.uint64) % np.uint64(K) == 0)
    e = oracle_mod.count_edges_esu(g, K)
    from test_oracle_edges import _class_edges
    census = v.sum(axis=0, dtype=np.uint64) // np.uint64(K)
    assert np.array_equal(e.sum(axis=0, dtype=np.uint64), _class_edges(oracle_mod, K) * census)
    small = G.random_small(8, 0.4, 9)
    assert np.array_equal(oracle_mod.count_edges_brute(small, K), oracle_mod.count_edges_esu(small, K))
