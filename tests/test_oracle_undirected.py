"""Undirected motifs in the oracle, pinned to things other than itself:
hand-derived class indices and OEIS counts (tests/golden/undirected_classes.txt), a table-free
pure-Python brute force naming classes by edge count + degree sequence, closed forms, the
direction collapse of the (separately pinned) directed oracle, and Eq. 4 for an undirected
G(n, p) (undirected n_max = C(k, 2))."""
import math

import numpy as np
import pytest

import graphgen as G
from conftest import read_golden


def golden():
    rows = read_golden("undirected_classes.txt")
    d = {"uclasses": {}, "ulabelled": {}, "uclass": {}, "uniso": {}}
    for r in rows:
        if r[0] in ("uclasses", "ulabelled"):
            d[r[0]][int(r[1])] = int(r[2])
        elif r[0] == "uclass":
            d["uclass"].setdefault(int(r[1]), {})[r[2]] = int(r[3])
        elif r[0] == "uniso":
            d["uniso"][int(r[1])] = [int(x) for x in r[2:]]
    return d


GOLD = golden()


@pytest.mark.parametrize("k", [3, 4])
def test_class_ids_and_iso_counts(oracle_mod, k):
    ids = oracle_mod.undirected_class_ids(k)
    assert len(ids) == GOLD["uclasses"][k]
    assert sorted(GOLD["uclass"][k].values()) == ids.tolist()
    iso = oracle_mod.n_iso_undirected(k)
    assert iso.tolist() == GOLD["uniso"][k]
    assert iso.sum() == GOLD["ulabelled"][k]


def _named(oracle_mod, g, k):
    """count_py_undirected as a matrix in the oracle's column order (via the golden names)."""
    ids = oracle_mod.undirected_class_ids(k).tolist()
    out = np.zeros((g[0], len(ids)), np.uint64)
    for (v, name), c in oracle_mod.count_py_undirected(g, k).items():
        out[v, ids.index(GOLD["uclass"][k][name])] = c
    return out


@pytest.mark.parametrize("k", [3, 4])
def test_vs_pure_python_brute_force(oracle_mod, k):
    for seed in range(40):
        n = 5 + seed % 8
        g = G.random_small(n, (0.15, 0.35, 0.6)[seed % 3], 900 + seed)
        want = _named(oracle_mod, g, k)
        assert np.array_equal(oracle_mod.count_undirected(g, k), want), seed
        assert np.array_equal(oracle_mod.count_undirected(g, k, method="brute"), want), seed


@pytest.mark.parametrize("k", [3, 4])
def test_closed_forms(oracle_mod, k):
    ids = oracle_mod.undirected_class_ids(k).tolist()
    col = {name: ids.index(c) for name, c in GOLD["uclass"][k].items()}
    top = "triangle" if k == 3 else "clique"
    # K_n in any orientation (here a transitive tournament): every vertex C(n-1, k-1) cliques
    for n in (5, 7):
        out = oracle_mod.count_undirected(G.transitive_tournament(n), k)
        assert (out[:, col[top]] == math.comb(n - 1, k - 1)).all() and out.sum() == n * math.comb(n - 1, k - 1)
    # star with L leaves (in or out): centre C(L, k-1), leaf C(L-1, k-2) stars
    L = 9
    name = "path" if k == 3 else "star"
    for g in (G.out_star(L), G.in_star(L)):
        out = oracle_mod.count_undirected(g, k)
        assert out[0, col[name]] == math.comb(L, k - 1)
        assert (out[1:, col[name]] == math.comb(L - 1, k - 2)).all()
        assert out.sum() == k * math.comb(L, k - 1)
    # cycle C_n, n > k, any orientation: every vertex lies on k paths of k consecutive vertices
    for g in (G.directed_cycle(8), G.undirected_cycle(8)):
        out = oracle_mod.count_undirected(g, k)
        assert (out[:, col["path"]] == k).all() and out.sum() == 8 * k
    # C_4 itself, k = 4: one 4-cycle per vertex
    if k == 4:
        out = oracle_mod.count_undirected(G.directed_cycle(4), 4)
        assert (out[:, col["cycle"]] == 1).all() and out.sum() == 4


@pytest.mark.parametrize("k", [3, 4])
def test_direction_collapse_of_directed_oracle(oracle_mod, k):
    """Summing the directed columns per underlying undirected class gives the undirected row:
    the class of G_U[S] is the symmetric closure of the directed class's matrix."""
    t = oracle_mod.class_table(k)
    pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(pairs)
    uids = oracle_mod.undirected_class_ids(k).tolist()
    collapse = []
    for cid in t["class_ids"]:
        bits = {pairs[b] for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}
        sym = bits | {(j, i) for (i, j) in bits}
        m = sum(1 << (nb - 1 - b) for b in range(nb) if pairs[b] in sym)
        collapse.append(uids.index(int(t["canon"][m])))
    M = np.zeros((len(t["class_ids"]), len(uids)), np.uint64)
    M[np.arange(len(collapse)), collapse] = 1
    for seed in range(8):
        g = G.random_small(24, 0.2, 4400 + seed)
        d = oracle_mod.count_esu(g, k)
        assert np.array_equal((d @ M).astype(np.uint64), oracle_mod.count_undirected(g, k))


@pytest.mark.parametrize("k", [3, 4])
def test_eq4_undirected_gnp(oracle_mod, k):
    """Eq. 4 at the realised p-hat of an undirected G(n, p), summed over vertices, R seeds:
    |mean - E| <= 4 SE + 1% for classes with E >= 1000 (reading G12: exact expectation)."""
    n, p, R = 300, 0.04, 6
    tot = []
    for rep in range(R):
        g = G.gnp_undirected(n, p, 5100 + rep)
        ph = g[1].size / (n * (n - 1) / 2)
        e = oracle_mod.expected_gnp_undirected(k, n, ph) * n
        tot.append(oracle_mod.count_undirected(g, k).sum(axis=0).astype(float) / e)
    tot = np.array(tot)
    E = oracle_mod.expected_gnp_undirected(k, n, p) * n
    m, se = tot.mean(axis=0), tot.std(axis=0, ddof=1) / np.sqrt(R)
    ok = E >= 1000
    assert ok.sum() >= (1 if k == 3 else 2)
    assert (np.abs(m[ok] - 1.0) <= 4 * se[ok] + 0.01).all(), (m, se, E)
    mid = (E >= 10) & ~ok                 # Poisson-like: 6 SE + 3 sqrt(E / R) / E
    assert (np.abs(m[mid] - 1.0) <= 6 * se[mid] + 3 / np.sqrt(E[mid] * R)).all(), (m, se, E)


@pytest.mark.parametrize("k", [3, 4])
def test_count_vertex_undirected_vs_pure_python(oracle_mod, k):
    """count_vertex_undirected (per-vertex ESU on G_U) pinned to the table-free pure-Python brute
    force on random graphs, and on a star centre to the closed form C(L, k-1)."""
    ids = oracle_mod.undirected_class_ids(k).tolist()
    for seed in range(12):
        n = 6 + seed % 6
        g = G.random_small(n, (0.2, 0.4, 0.6)[seed % 3], 7300 + seed)
        want = _named(oracle_mod, g, k)
        verts = np.array(sorted({0, n // 2, n - 1}), np.int32)
        assert np.array_equal(oracle_mod.count_vertex_undirected(g, k, verts), want[verts]), seed
    L = 11
    row = oracle_mod.count_vertex_undirected(G.out_star(L), k, np.array([0, 3], np.int32))
    col = ids.index(GOLD["uclass"][k]["path" if k == 3 else "star"])
    assert row[0, col] == math.comb(L, k - 1) and row[0].sum() == math.comb(L, k - 1)
    assert row[1, col] == math.comb(L - 1, k - 2) and row[1].sum() == math.comb(L - 1, k - 2)
