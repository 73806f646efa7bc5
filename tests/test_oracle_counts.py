"""Pins for the oracle's count functions, -m "not gpu".

The oracle (brute force = the definition, ESU, and the paper's BFS-shape method)
is pinned against things that do not come from itself:
  * the paper's worked example, counts hand-derived (tests/golden);
  * closed forms for complete digraphs, transitive tournaments ("regular DAGs",
    P:218), directed and mutual cycles, out/in-stars;
  * a pure-Python brute force that canonicalises on the fly (no table);
  * single-motif graphs (each labelled connected motif once);
  * invariants: column sums = k x census, transpose, direction collapse, order
    invariance (Lemma 1), partial sums over root ranges;
  * the textbook k=3 row sum C(d,2) + sum_{u in N(v)} (d_u - 1) - 2 t_v;
  * Eq. 4 on directed G(n, p), statistically.
"""
import itertools
import math

import numpy as np
import pytest

import graphgen as G
from conftest import read_golden, to_dense


def col_of(oracle_mod, k, cid):
    return int(oracle_mod.class_table(k)["col"][cid])


# ------------------------------------------------------------------ golden
def test_paper_csr_example(oracle_mod):
    """directed Indices [0,3,3,4,6], Neighbors [1,2,3,0,1,2]; undirected ones."""
    gold = {r[1]: [int(x) for x in r[2:]] for r in read_golden("paper_example.txt") if r[0] == "csr"}
    oi, on, ui, un = oracle_mod.csr(G.paper_example())
    assert oi.tolist() == gold["directed_indices"]
    assert on.tolist() == gold["directed_neighbors"]
    assert ui.tolist() == gold["undirected_indices"]
    assert un.tolist() == gold["undirected_neighbors"]


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("fn", ["count_brute", "count_esu", "count_bfs"])
def test_paper_example_counts(oracle_mod, k, fn):
    g = G.paper_example()
    want = {}
    for r in read_golden("paper_example.txt"):
        if r[0] == f"k{k}":
            for item in r[2:]:
                c, x = item.split(":")
                want[(int(r[1]), int(c))] = int(x)
    expect = to_dense(want, 4, oracle_mod.class_table(k)["class_ids"])
    assert np.array_equal(getattr(oracle_mod, fn)(g, k), expect)


# -------------------------------------------------------------- closed forms
@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("n", [4, 5, 7])
def test_complete_digraph(oracle_mod, k, n):
    out = oracle_mod.count_esu(G.complete_digraph(n), k)
    want = np.zeros_like(out)
    want[:, col_of(oracle_mod, k, (1 << (k * (k - 1))) - 1)] = math.comb(n - 1, k - 1)
    assert np.array_equal(out, want)
    assert np.array_equal(oracle_mod.count_brute(G.complete_digraph(n), k), want)


@pytest.mark.parametrize("k,cid", [(3, 11), (4, 311)])
@pytest.mark.parametrize("n", [4, 6, 9])
def test_transitive_tournament(oracle_mod, k, cid, n):
    """Regular DAG: every k-set is a transitive tournament."""
    for fn in (oracle_mod.count_esu, oracle_mod.count_bfs, oracle_mod.count_brute):
        out = fn(G.transitive_tournament(n), k)
        want = np.zeros_like(out)
        want[:, col_of(oracle_mod, k, cid)] = math.comb(n - 1, k - 1)
        assert np.array_equal(out, want)


@pytest.mark.parametrize("k,cid", [(3, 6), (4, 84)])
@pytest.mark.parametrize("n", [5, 6, 9])
def test_directed_cycle(oracle_mod, k, cid, n):
    """Directed C_n, n > k: each vertex lies in k consecutive k-sets, all directed paths."""
    for fn in (oracle_mod.count_esu, oracle_mod.count_bfs, oracle_mod.count_brute):
        out = fn(G.directed_cycle(n), k)
        want = np.zeros_like(out)
        want[:, col_of(oracle_mod, k, cid)] = k
        assert np.array_equal(out, want)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("n", [5, 6, 7, 8, 9])
def test_mutual_cycles_lemma4(oracle_mod, k, n):
    """C5..C9 with mutual arcs: the Lemma 4 configuration ('exactly 5')."""
    g = G.undirected_cycle(n)
    want = oracle_mod.count_brute(g, k)
    assert np.array_equal(oracle_mod.count_bfs(g, k), want)
    assert np.array_equal(oracle_mod.count_esu(g, k), want)
    assert np.all(want.sum(axis=1) == k)           # k consecutive sets through each vertex


@pytest.mark.parametrize("k,out_id,in_id", [(3, 3, 10), (4, 7, 292)])
@pytest.mark.parametrize("leaves", [3, 5, 8])
def test_stars(oracle_mod, k, out_id, in_id, leaves):
    for gen, cid in ((G.out_star, out_id), (G.in_star, in_id)):
        out = oracle_mod.count_esu(gen(leaves), k)
        want = np.zeros_like(out)
        c = col_of(oracle_mod, k, cid)
        want[0, c] = math.comb(leaves, k - 1)
        want[1:, c] = math.comb(leaves - 1, k - 2)
        assert np.array_equal(out, want)


# ---------------------------------------------------- independent brute force
@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("seed", range(6))
def test_brute_vs_pure_python(oracle_mod, k, seed):
    n = 7 + seed % 3
    g = G.random_small(n, [0.2, 0.4, 0.7][seed % 3], 100 + seed)
    want = to_dense(oracle_mod.count_py(g, k), n, oracle_mod.class_table(k)["class_ids"])
    assert np.array_equal(oracle_mod.count_brute(g, k), want)


def _fixtures():
    fx = []
    for seed in range(72):
        n = 5 + seed % 26
        for p in (0.1, 0.3, 0.6):
            fx.append((f"rand{seed}-{p}", G.random_small(n, p, 7000 + seed)))
    for n in (4, 5, 6, 7):
        fx.append((f"K{n}", G.complete_digraph(n)))
    for n in (3, 4, 5, 6, 7, 8, 9):
        fx.append((f"C{n}", G.undirected_cycle(n)))
        fx.append((f"dC{n}", G.directed_cycle(n)))
    fx += [("path7", G.directed_path(7)), ("star6", G.out_star(6)), ("instar6", G.in_star(6)),
           ("grid3x3", G.dag_grid(3, 3)), ("grid3x4", G.dag_grid(3, 4)),
           ("paper", G.paper_example())]
    return fx


FIXTURES = _fixtures()


@pytest.mark.parametrize("k", [3, 4])
def test_esu_and_bfs_equal_brute_force(oracle_mod, k):
    """SPEC acceptance 1: >= 200 random digraphs + structured fixtures, each also
    under two random vertex orders for the paper's method (order invariance, Lemma 1)."""
    assert len(FIXTURES) >= 216 + 20
    for name, g in FIXTURES:
        want = oracle_mod.count_brute(g, k)
        assert np.array_equal(oracle_mod.count_esu(g, k), want), name
        assert np.array_equal(oracle_mod.count_bfs(g, k), want), name
        rng = np.random.default_rng(len(name) + g[0])
        for _ in range(2):
            rank = rng.permutation(g[0])
            assert np.array_equal(oracle_mod.count_bfs(g, k, rank=rank), want), name


@pytest.mark.parametrize("k", [3, 4])
def test_single_motif_graphs(oracle_mod, k):
    """Every connected labelled motif (54 / 3834) as its own component, randomly relabelled:
    each of its vertices has exactly 1, in that motif's class, and 0 elsewhere."""
    t = oracle_mod.class_table(k)
    masks = np.nonzero(t["conn"])[0]
    order = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(order)
    src, dst = [], []
    for c, m in enumerate(masks):
        for b, (i, j) in enumerate(order):
            if (int(m) >> (nb - 1 - b)) & 1:
                src.append(c * k + i)
                dst.append(c * k + j)
    n = len(masks) * k
    perm = np.random.default_rng(k).permutation(n)
    g = G.relabel((n, np.array(src), np.array(dst)), perm)
    out = oracle_mod.count_esu(g, k)
    want = np.zeros_like(out)
    for c, m in enumerate(masks):
        for i in range(k):
            want[perm[c * k + i], t["col"][m]] = 1
    assert np.array_equal(out, want)


# --------------------------------------------------------------- invariants
def _transpose_col_map(oracle_mod, k):
    t = oracle_mod.class_table(k)
    order = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(order)
    tau = []
    for cid in t["class_ids"]:
        arcs = {order[b] for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}
        m2 = oracle_mod.paper_index(k, {(j, i) for (i, j) in arcs})
        tau.append(int(t["col"][m2]))
    return np.array(tau)


def _collapse_col_map(oracle_mod, k):
    t = oracle_mod.class_table(k)
    order = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(order)
    out = []
    for cid in t["class_ids"]:
        arcs = {order[b] for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}
        sym = arcs | {(j, i) for (i, j) in arcs}
        out.append(int(t["col"][oracle_mod.paper_index(k, sym)]))
    return np.array(out)


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("seed", range(4))
def test_invariants(oracle_mod, k, seed):
    g = G.make_config("cfg3", rep=seed, scale=0.004) if seed % 2 else \
        G.gnp_directed(300, 0.02, 900 + seed)
    n = g[0]
    full = oracle_mod.count_esu(g, k)
    # (a) each set is counted at k member rows
    assert np.all(full.sum(axis=0) % k == 0)
    out, nsets = oracle_mod.count_esu(g, k, return_sets=True)
    assert int(full.sum()) == k * nsets
    # (b) transpose: counts(G^T)[v][j] = counts(G)[v][tau(j)]
    tau = _transpose_col_map(oracle_mod, k)
    assert np.array_equal(oracle_mod.count_esu(G.transpose(g), k), full[:, tau])
    # (c) direction collapse: sum directed classes per undirected shape
    cmap = _collapse_col_map(oracle_mod, k)
    collapsed = np.zeros_like(full)
    for j in range(full.shape[1]):
        collapsed[:, cmap[j]] += full[:, j]
    assert np.array_equal(oracle_mod.count_esu(G.make_mutual(g), k), collapsed)
    # (d) vertex relabelling moves rows only
    perm = np.random.default_rng(seed).permutation(n)
    assert np.array_equal(oracle_mod.count_esu(G.relabel(g, perm), k)[perm], full)
    # (e) the paper's method under the degree order and a random order
    deg = np.bincount(np.concatenate([g[1], g[2]]), minlength=n)
    rank = np.empty(n, np.int64)
    rank[np.lexsort((np.arange(n), -deg))] = np.arange(n)
    assert np.array_equal(oracle_mod.count_bfs(g, k, rank=rank), full)
    # (f) partials over root ranges sum to the full matrix; sampled rows agree
    cut = n // 3
    parts = oracle_mod.count_esu(g, k, 0, cut) + oracle_mod.count_esu(g, k, cut, n)
    assert np.array_equal(parts, full)
    verts = np.random.default_rng(seed + 1).choice(n, 12, replace=False)
    assert np.array_equal(oracle_mod.count_vertex(g, k, verts), full[verts])


@pytest.mark.parametrize("seed", range(3))
def test_k3_row_sum_textbook(oracle_mod, seed):
    """Connected 3-sets through v: C(d_v,2) + sum_{u~v}(d_u - 1) - 2 t_v (G_U degrees d,
    triangles t_v = (A^2 o A)_vv / 2 ... summed per row)."""
    g = G.gnp_directed(400, 0.015, 40 + seed) if seed != 1 else G.make_config("cfg3", scale=0.005)
    n, s, d = g
    A = np.zeros((n, n), np.int64)
    A[s, d] = 1
    A = ((A + A.T) > 0).astype(np.int64)
    deg = A.sum(1)
    tri = ((A @ A) * A).sum(1) // 2
    want = deg * (deg - 1) // 2 + A @ (deg - 1) - 2 * tri
    got = oracle_mod.count_esu(g, 3).sum(axis=1).astype(np.int64)
    assert np.array_equal(got, want)


def test_eq4_gnp_statistical(oracle_mod):
    """Eq. 4 on directed G(n, p) at the realised p-hat (reading G12/G13):
    totals per class (column sum / k) vs C(n,k) N_Iso p^ne (1-p)^(nmax-ne), over R seeds."""
    for k, n, p, R in ((3, 1000, 0.1, 4), (4, 150, 0.08, 4)):
        tot = []
        phats = []
        for r in range(R):
            g = G.gnp_directed(n, p, 5000 + 17 * r + k)
            tot.append(oracle_mod.count_esu(g, k).sum(axis=0).astype(np.float64) / k)
            phats.append(g[1].size / (n * (n - 1)))
        tot = np.array(tot)
        E = np.mean([oracle_mod.expected_gnp(k, n, ph) * n / k for ph in phats], axis=0)
        mean = tot.mean(0)
        se = tot.std(0, ddof=1) / np.sqrt(R)
        for j in range(len(E)):
            if E[j] >= 1:
                assert abs(mean[j] - E[j]) <= 6 * se[j] + 3 * np.sqrt(E[j] / R) + 1e-9, (k, j)
            else:
                assert tot[:, j].max() <= 10, (k, j)
        # a wrong model (p doubled) must fail on the dominant classes
        E2 = oracle_mod.expected_gnp(k, n, 2 * np.mean(phats)) * n / k
        big = E >= 1000
        assert np.any(np.abs(mean[big] - E2[big]) > 6 * se[big] + 3 * np.sqrt(E2[big] / R))


def test_expected_gnp_closed_forms(oracle_mod):
    # p = 1: complete class gets C(n-1, k-1), every other class 0
    e = oracle_mod.expected_gnp(3, 5, 1.0)
    assert e[-1] == math.comb(4, 2) and np.all(e[:-1] == 0)
    # sum over all classes + disconnected mass = C(n-1,k-1): connected mass < 1 of it
    assert oracle_mod.expected_gnp(4, 50, 0.3).sum() < math.comb(49, 3)


@pytest.mark.parametrize("bad,msg", [((3, np.array([0, 1]), np.array([1, 1])), "self-loop"),
                                     ((3, np.array([0]), np.array([5])), "out of range")])
def test_oracle_rejects_bad_input(oracle_mod, bad, msg):
    with pytest.raises(ValueError, match=msg):
        oracle_mod.count_esu(bad, 3)


def test_empty_and_tiny(oracle_mod):
    for g in ((0, np.zeros(0, np.int32), np.zeros(0, np.int32)),
              (2, np.array([0, 1]), np.array([1, 0])),
              (5, np.zeros(0, np.int32), np.zeros(0, np.int32))):
        for k in (3, 4):
            assert not oracle_mod.count_esu(g, k).any()
            assert not oracle_mod.count_brute(g, k).any()
            assert not oracle_mod.count_bfs(g, k).any()
