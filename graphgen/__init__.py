"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no symmetrisation, ordering,
enumeration or classification).  It only draws directed edge lists
``(n, src, dst)`` with numpy PCG64 from a seed, and builds a few named toy
graphs.  Both sides (``oracle/`` and ``paper_2201_11655_b200``) consume the same
arrays; neither imports the other.

Every generator returns a *simple* directed graph: int32 ``src``/``dst`` arrays,
no self-loops, no duplicated ordered pair (u, v).  A mutual pair is two ordered
edges u->v and v->u.

Recipes (DESIGN.md §"Inputs"):

* ``gnp_directed`` — directed G(n, p) of PAPER.md §"Comparison to Theory"
  ("each pair of vertices is connected with a constant probability p"):
  every ordered pair (u, v), u != v, is an edge independently with probability p
  (reading G13: ordered pairs are independent, n_max = 2*C(k,2)).
  Drawn by geometric skipping over the n(n-1) ordered-pair positions
  (Batagelj & Brandes 2005, "Efficient generation of large random networks").
* ``ba_directed`` — preferential attachment (Barabasi-Albert) via Batagelj &
  Brandes' endpoint-copying algorithm: vertex v adds m endpoints, each copied
  uniformly from the endpoint list built so far (probability proportional to
  degree).  Self-loops and repeated pairs are dropped; each undirected pair is
  made mutual with probability ``rho``, otherwise oriented by a fair coin.  This
  gives heavy-tailed in- and out-degrees (the scale-free workloads of P:175,
  P:243).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "gnp_directed", "gnp_undirected", "ba_directed", "CONFIGS", "make_config", "config_seed",
    "complete_digraph", "transitive_tournament", "directed_cycle", "out_star",
    "in_star", "directed_path", "dag_grid", "undirected_cycle", "paper_example",
    "random_small", "relabel", "transpose", "make_mutual",
]


def _sorted_unique(key: np.ndarray) -> np.ndarray:
    # np.unique is pathologically slow on 1e7+ int64 in this numpy; sort + diff instead
    key = np.sort(key)
    if key.size == 0:
        return key
    keep = np.empty(key.size, dtype=bool)
    keep[0] = True
    np.not_equal(key[1:], key[:-1], out=keep[1:])
    return key[keep]


def _finish(n: int, src: np.ndarray, dst: np.ndarray):
    """Drop self-loops and duplicate ordered pairs; return int32 arrays sorted by (src, dst)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = _sorted_unique(src * np.int64(n) + dst)
    return n, (key // n).astype(np.int32), (key % n).astype(np.int32)


def gnp_directed(n: int, p: float, seed: int):
    """Directed G(n, p): each of the n(n-1) ordered pairs independently with prob. p."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(n)
    if n < 2 or p <= 0.0:
        return n, np.zeros(0, np.int32), np.zeros(0, np.int32)
    total = n * (n - 1)
    if p >= 1.0:
        pos = np.arange(total, dtype=np.int64)
    else:
        chunks = []
        last = -1
        expect = total * p
        while True:
            draw = int(expect * 1.05 + 10 * np.sqrt(expect) + 64)
            gaps = rng.geometric(p, size=draw).astype(np.int64)
            q = last + np.cumsum(gaps)
            q = q[q < total]
            chunks.append(q)
            if q.size < draw:
                break
            last = int(q[-1])
        pos = np.concatenate(chunks)
    u = pos // (n - 1)
    w = pos % (n - 1)
    v = w + (w >= u)
    return _finish(n, u, v)


def gnp_undirected(n: int, p: float, seed: int):
    """Undirected G(n, p): each of the C(n, 2) unordered pairs independently with
    prob. p, emitted as one arc u -> v with u < v (the undirected motif count ignores it)."""
    n, s, d = gnp_directed(n, p, seed)
    keep = s < d                          # an ordered-pair G(n,p) restricted to u < v
    return n, s[keep], d[keep]


def ba_directed(n: int, m: int, seed: int, rho: float = 0.1):
    """Directed preferential-attachment graph (Batagelj-Brandes endpoint copying).

    Seed: a clique on vertices 0..m.  Vertex v > m then adds m endpoints, each a
    uniform copy from the endpoint list of all EARLIER vertices' edges.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    n, m = int(n), int(m)
    m0 = min(m + 1, n)
    cu, cv = np.triu_indices(m0, 1)
    L0 = 2 * cu.size
    vals0 = np.empty(L0, dtype=np.int64)
    vals0[0::2], vals0[1::2] = cu, cv
    nn = max(0, n - m0)
    L = L0 + 2 * nn * m
    # T[p] = the list position whose vertex slot p copies; fixed points hold a vertex
    T = np.arange(L, dtype=np.int64)
    slot = np.arange(nn * m, dtype=np.int64)
    odd = L0 + 2 * slot + 1
    hi = L0 + 2 * (slot // m) * m          # endpoints of vertices before this one
    T[odd] = (rng.random(slot.size) * hi).astype(np.int64)
    while True:                            # pointer jumping until each copy hits a fixed point
        t = T[odd]
        bad = (t >= L0) & ((t - L0) & 1 == 1)
        if not bad.any():
            break
        T[odd] = np.where(bad, T[t], t)
    def vertex_at(p):
        return np.where(p < L0, vals0[np.minimum(p, L0 - 1)], m0 + (p - L0) // 2 // m)
    u = np.concatenate([cu, m0 + slot // m])
    v = np.concatenate([cv, vertex_at(T[odd])])
    keep = u != v
    u, v = u[keep], v[keep]
    a = np.minimum(u, v)
    b = np.maximum(u, v)
    key = _sorted_unique(a * np.int64(n) + b)
    a, b = key // n, key % n
    r = rng.random(a.size)
    flip = rng.random(a.size) < 0.5
    mutual = r < rho
    s1 = np.where(flip, b, a)
    d1 = np.where(flip, a, b)
    src = np.concatenate([s1, d1[mutual]])
    dst = np.concatenate([d1, s1[mutual]])
    return _finish(n, src, dst)


# BASELINE.json configs; seeds are 2201 + 100*cfg.
CONFIGS = {
    "cfg1": dict(kind="gnp", n=1000, p=3.0 / 999.0, k=(3,),
                 desc="directed Erdos-Renyi n=1,000 avg out-degree 3, k=3"),
    "cfg2": dict(kind="gnp", n=20000, p=5e-4, k=(4,),
                 desc="directed Erdos-Renyi n=20,000 p=5e-4, k=4"),
    "cfg3": dict(kind="ba", n=200000, m=10, rho=0.1, k=(3, 4),
                 desc="directed power-law n=200,000 ~2M edges, k=3 and k=4"),
    "cfg4": dict(kind="ba", n=1000000, m=10, rho=0.1, k=(4,),
                 desc="directed power-law n=1M ~10M edges heavy-tailed in/out, k=4"),
    "cfg5": dict(kind="gnp", n=5000000, p=8.0 / 4999999.0, k=(4,),
                 desc="directed Erdos-Renyi n=5M avg out-degree 8 (~40M edges), k=4"),
}


def config_seed(name: str, rep: int = 0) -> int:
    return 2201 + 100 * int(name[3:]) + rep


def make_config(name: str, rep: int = 0, scale: float = 1.0):
    """Generate BASELINE config ``name`` (optionally with n scaled down for tests)."""
    c = CONFIGS[name]
    seed = config_seed(name, rep)
    n = max(8, int(round(c["n"] * scale)))
    if c["kind"] == "gnp":
        avg = c["p"] * (c["n"] - 1)          # keep the average degree when scaling
        return gnp_directed(n, min(1.0, avg / (n - 1)), seed)
    return ba_directed(n, c["m"], seed, c["rho"])


# ---------------------------------------------------------------- toy graphs
def complete_digraph(n: int):
    u, v = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    return _finish(n, u.ravel(), v.ravel())


def transitive_tournament(n: int):
    """u -> v for every u < v (the 'regular DAG' of P:218)."""
    u, v = np.triu_indices(n, 1)
    return _finish(n, u, v)


def directed_cycle(n: int):
    u = np.arange(n)
    return _finish(n, u, (u + 1) % n)


def undirected_cycle(n: int):
    """C_n with every pair mutual."""
    u = np.arange(n)
    return _finish(n, np.concatenate([u, (u + 1) % n]), np.concatenate([(u + 1) % n, u]))


def out_star(leaves: int):
    return _finish(leaves + 1, np.zeros(leaves, np.int64), np.arange(1, leaves + 1))


def in_star(leaves: int):
    return _finish(leaves + 1, np.arange(1, leaves + 1), np.zeros(leaves, np.int64))


def directed_path(n: int):
    u = np.arange(n - 1)
    return _finish(n, u, u + 1)


def dag_grid(rows: int, cols: int):
    """Grid DAG: (i,j) -> (i+1,j) and (i,j) -> (i,j+1)."""
    idx = np.arange(rows * cols).reshape(rows, cols)
    s = np.concatenate([idx[:-1, :].ravel(), idx[:, :-1].ravel()])
    d = np.concatenate([idx[1:, :].ravel(), idx[:, 1:].ravel()])
    return _finish(rows * cols, s, d)


def paper_example():
    """0->1, 0->2, 0->3, 2->0, 3->1, 3->2."""
    return _finish(4, [0, 0, 0, 2, 3, 3], [1, 2, 3, 0, 1, 2])


def random_small(n: int, p: float, seed: int):
    """Tiny directed G(n, p) by explicit coin flips (test fixtures)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    u, v = np.nonzero(a)
    return _finish(n, u, v)


def relabel(g, perm: np.ndarray):
    """Rename vertex x to perm[x]."""
    n, s, d = g
    perm = np.asarray(perm, dtype=np.int64)
    return _finish(n, perm[s], perm[d])


def transpose(g):
    n, s, d = g
    return _finish(n, d, s)


def make_mutual(g):
    """Every edge becomes a mutual pair (G_U with all codes 3)."""
    n, s, d = g
    return _finish(n, np.concatenate([s, d]), np.concatenate([d, s]))
