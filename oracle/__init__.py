"""VDMC CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2201_11655_b200``) never imports it, and the two share no code.

Contents (each function cites the PAPER.md passage it follows; see
``vdmc_oracle.c`` for the C side):

* ``csr``            — the paper's CSR for a directed graph.
* ``class_table``    — motif index -> minimum-isomorph index, connectivity and the
                       ascending column list (Fig. 1).
* ``count_brute``    — the definition written out over all C(n, k) subsets.
* ``count_esu``      — the same matrix via ESU (Wernicke 2006, cited at P:36).
* ``count_vertex``   — rows of sampled vertices (ESU with the vertex forced minimal).
* ``count_bfs``      — the paper's method itself (proper k-BFS, Lemmas 2-4).
* ``count_py``       — a pure-Python brute force with on-the-fly canonicalisation
                       (tiny graphs only; shares nothing with the C file).
* ``expected_gnp``   — Eq. 4, expected per-vertex count in G(n, p).
* ``n_iso``          — N_Iso(m): isomorph count per class.
* ``symmetrize`` / ``undirected_class_ids`` / ``count_undirected`` — undirected motifs
                       (counted "in the undirected graph induced by ignoring the
                       direction of edges", G_U of P:76): the directed definition applied to
                       the all-mutual graph of G_U, columns = the all-mutual classes.
* ``count_py_undirected`` — pure-Python brute force for undirected motifs, classes named by
                       (edge count, degree sequence) (shares nothing with the C file).
* ``expected_gnp_undirected`` — Eq. 4 with the undirected n_max = C(k, 2).
* ``edge_list`` / ``count_edges_brute`` / ``count_edges_esu`` — edge-level counts, the
                       Discussion's extension ("counting motifs for edges ... only requires
                       updating edges and not vertices"): +1 in the set's class for every G_U
                       edge inside the set; rows = G_U edges {u < v} in lexicographic order.
* ``count_edge_rows`` — rows of sampled edges (per-edge ESU), for full-size sampled parity.
* ``count_edges_py`` — pure-Python brute force of the same (tiny graphs; shares nothing with C).

Every function is pinned by ``tests/test_oracle_*.py`` (closed forms, the
hand-worked golden of the paper's example graph, single-motif graphs,
invariants and Eq. 4); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "vdmc_oracle.c")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (-O2 -fopenmp).  Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-march=native", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _edges(g):
    n, s, d = g
    s = np.ascontiguousarray(s, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    return int(n), s, d


_ERR = {-1: "bad argument", -2: "vertex id out of range", -3: "self-loop", -4: "out of memory"}


def _check(rc):
    if rc != 0:
        raise ValueError(f"oracle: {_ERR.get(rc, rc)}")


def num_classes(k: int) -> int:
    return len(class_table(k)["class_ids"])


_TABLES: dict = {}


def class_table(k: int) -> dict:
    """canon[m], conn[m], col[m] for every index m, and the ascending class ids."""
    if k in _TABLES:
        return _TABLES[k]
    lib = _load()
    M = 1 << (k * (k - 1))
    canon = np.zeros(M, np.int32)
    conn = np.zeros(M, np.uint8)
    col = np.zeros(M, np.int32)
    ids = np.zeros(16384, np.int32)
    nc = ctypes.c_int32(0)
    _check(lib.oracle_class_table(ctypes.c_int(k), _p(canon), _p(conn), _p(col), _p(ids),
                                  ctypes.byref(nc)))
    t = dict(canon=canon, conn=conn.astype(bool), col=col, class_ids=ids[: nc.value].copy())
    _TABLES[k] = t
    return t


def n_iso(k: int) -> np.ndarray:
    """N_Iso(m) per column: number of connected indices whose minimum is the class."""
    t = class_table(k)
    c = t["col"][t["conn"]]
    return np.bincount(c, minlength=len(t["class_ids"]))


def n_edges(k: int) -> np.ndarray:
    """n_e(m) per column: number of arcs of the class (popcount of its index)."""
    return np.array([bin(int(x)).count("1") for x in class_table(k)["class_ids"]])


def csr(g):
    """(directed Indices, Neighbors, undirected Indices, Neighbors) as in P:130-133."""
    lib = _load()
    n, s, d = _edges(g)
    m = s.size
    oind = np.zeros(n + 1, np.int64)
    onbr = np.zeros(max(m, 1), np.int32)
    uind = np.zeros(n + 1, np.int64)
    unbr = np.zeros(max(2 * m, 1), np.int32)
    _check(lib.oracle_csr(ctypes.c_int64(n), ctypes.c_int64(m), _p(s), _p(d), _p(oind), _p(onbr),
                          _p(uind), _p(unbr)))
    return oind, onbr[: oind[n]].copy(), uind, unbr[: uind[n]].copy()


def count_brute(g, k: int) -> np.ndarray:
    lib = _load()
    n, s, d = _edges(g)
    out = np.zeros((n, num_classes(k)), np.uint64)
    _check(lib.oracle_count_brute(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d),
                                  ctypes.c_int(k), _p(out)))
    return out


def count_esu(g, k: int, root_lo: int = 0, root_hi: int | None = None, threads: int = 0,
              return_sets: bool = False):
    """Full matrix (or the partial of roots [root_lo, root_hi) in original-id order)."""
    lib = _load()
    n, s, d = _edges(g)
    if root_hi is None:
        root_hi = n
    out = np.zeros((n, num_classes(k)), np.uint64)
    nsets = ctypes.c_uint64(0)
    _check(lib.oracle_count_esu(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d),
                                ctypes.c_int(k), ctypes.c_int64(root_lo), ctypes.c_int64(root_hi),
                                ctypes.c_int(threads), _p(out), ctypes.byref(nsets)))
    return (out, int(nsets.value)) if return_sets else out


def count_vertex(g, k: int, verts, threads: int = 0) -> np.ndarray:
    """Rows counts[v] for the given vertices only."""
    lib = _load()
    n, s, d = _edges(g)
    verts = np.ascontiguousarray(verts, dtype=np.int32)
    out = np.zeros((verts.size, num_classes(k)), np.uint64)
    _check(lib.oracle_count_vertex(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d),
                                   ctypes.c_int(k), ctypes.c_int64(verts.size), _p(verts),
                                   ctypes.c_int(threads), _p(out)))
    return out


def count_bfs(g, k: int, rank=None) -> np.ndarray:
    """The paper's proper k-BFS enumeration; rank[v] = index of v (None = original ids)."""
    lib = _load()
    n, s, d = _edges(g)
    r = None if rank is None else np.ascontiguousarray(rank, dtype=np.int32)
    out = np.zeros((n, num_classes(k)), np.uint64)
    _check(lib.oracle_count_bfs(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d),
                                ctypes.c_int(k), _p(r), _p(out)))
    return out


# ------------------------------------------------------------------ pure Python
def paper_index(k: int, arcs) -> int:
    """Fig. 1: rows of the adjacency matrix, diagonal removed, MSB first."""
    bits = "".join("1" if (i, j) in arcs else "0"
                   for i in range(k) for j in range(k) if i != j)
    return int(bits, 2)


def count_py(g, k: int):
    """Pure-Python brute force for tiny graphs: returns {(v, canonical id): count}."""
    n, s, d = g
    arcs = set(zip(s.tolist(), d.tolist()))
    out: dict = {}
    for S in itertools.combinations(range(n), k):
        # connected in G_U?  (grow a component from S[0])
        comp = {S[0]}
        grew = True
        while grew:
            grew = False
            for x in S:
                if x not in comp and any((x, y) in arcs or (y, x) in arcs for y in comp):
                    comp.add(x)
                    grew = True
        if len(comp) < k:
            continue
        best = min(paper_index(k, {(i, j) for i in range(k) for j in range(k)
                                   if i != j and (P[i], P[j]) in arcs})
                   for P in itertools.permutations(S))
        for v in S:
            out[(v, best)] = out.get((v, best), 0) + 1
    return out


def expected_gnp(k: int, n: int, p: float) -> np.ndarray:
    """Eq. 4: E[X_{k,m}(i)] = C(n-1,k-1) N_Iso(m) p^{n_e} (1-p)^{n_max-n_e},
    directed n_max = 2*C(k,2).  One value per column."""
    ne = n_edges(k)
    nmax = k * (k - 1)
    return math.comb(n - 1, k - 1) * n_iso(k) * p ** ne * (1.0 - p) ** (nmax - ne)


# ------------------------------------------------------------------ undirected motifs
def symmetrize(g):
    """G_U as a directed graph ("ignoring the direction of the edge"): every arc u -> v
    becomes the mutual pair u <-> v (duplicates merged)."""
    n, s, d = g
    s = np.asarray(s, np.int64)
    d = np.asarray(d, np.int64)
    a = np.concatenate([s, d])
    b = np.concatenate([d, s])
    key = np.unique(a * n + b) if a.size else np.zeros(0, np.int64)
    return n, (key // n).astype(np.int32), (key % n).astype(np.int32)


def undirected_class_ids(k: int) -> np.ndarray:
    """Canonical ids of the undirected k-motifs: the paper's index of a symmetric
    adjacency matrix, minimised over vertex orders -- i.e. the connected classes whose
    minimum-index matrix is symmetric (reading G17)."""
    t = class_table(k)
    pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(pairs)
    out = []
    for cid in t["class_ids"]:
        bits = {pairs[b] for b in range(nb) if (int(cid) >> (nb - 1 - b)) & 1}
        if all((j, i) in bits for (i, j) in bits):
            out.append(int(cid))
    return np.array(out, np.int64)


def count_undirected(g, k: int, method: str = "esu") -> np.ndarray:
    """Undirected per-vertex k-motif counts: every connected k-set S, class of the
    G_U-induced subgraph, +1 for every member.  Written as the directed definition on
    symmetrize(g) -- whose induced subgraphs are exactly the symmetric matrices of G_U[S] --
    restricted to the all-mutual columns.  method: "esu" or "brute"."""
    sym = symmetrize(g)
    full = count_esu(sym, k) if method == "esu" else count_brute(sym, k)
    ids = list(class_table(k)["class_ids"])
    cols = [ids.index(c) for c in undirected_class_ids(k)]
    return np.ascontiguousarray(full[:, cols])


def count_vertex_undirected(g, k: int, verts) -> np.ndarray:
    """Rows of sampled vertices of count_undirected (per-vertex ESU on symmetrize(g))."""
    ids = list(class_table(k)["class_ids"])
    cols = [ids.index(c) for c in undirected_class_ids(k)]
    return np.ascontiguousarray(count_vertex(symmetrize(g), k, verts)[:, cols])


# (edge count, sorted degree sequence) names every connected graph on 3 or 4 vertices
UNDIRECTED_NAMES = {
    3: {(2, (1, 1, 2)): "path", (3, (2, 2, 2)): "triangle"},
    4: {(3, (1, 1, 1, 3)): "star", (3, (1, 1, 2, 2)): "path", (4, (1, 2, 2, 3)): "paw",
        (4, (2, 2, 2, 2)): "cycle", (5, (2, 2, 3, 3)): "diamond", (6, (3, 3, 3, 3)): "clique"},
}


def count_py_undirected(g, k: int):
    """Pure-Python brute force: {(v, name): count} over connected k-sets of G_U, the class
    named by its edge count and degree sequence (no index, no table)."""
    n, s, d = g
    und = {frozenset(e) for e in zip(s.tolist(), d.tolist())}
    out: dict = {}
    for S in itertools.combinations(range(n), k):
        es = [(x, y) for x, y in itertools.combinations(S, 2) if frozenset((x, y)) in und]
        comp, grew = {S[0]}, True
        while grew:
            grew = False
            for x, y in es:
                if (x in comp) != (y in comp):
                    comp |= {x, y}
                    grew = True
        if len(comp) < k:
            continue
        deg = tuple(sorted(sum(v in e for e in es) for v in S))
        name = UNDIRECTED_NAMES[k][(len(es), deg)]
        for v in S:
            out[(v, name)] = out.get((v, name), 0) + 1
    return out


def n_iso_undirected(k: int) -> np.ndarray:
    """Labelled undirected graphs per undirected class (the undirected N_Iso of P:187)."""
    return np.array([_n_sym_masks(k, int(c)) for c in undirected_class_ids(k)])


def _n_sym_masks(k: int, cid: int) -> int:
    """Symmetric indices whose minimum over vertex orders is cid (labelled undirected graphs)."""
    t = class_table(k)
    pairs = [(i, j) for i in range(k) for j in range(k) if i != j]
    nb = len(pairs)
    cnt = 0
    for m in range(1 << nb):
        bits = {pairs[b] for b in range(nb) if (m >> (nb - 1 - b)) & 1}
        if all((j, i) in bits for (i, j) in bits) and t["conn"][m] and int(t["canon"][m]) == cid:
            cnt += 1
    return cnt


def expected_gnp_undirected(k: int, n: int, p: float) -> np.ndarray:
    """Eq. 4 for an undirected G(n, p): n_max = C(k, 2), N_Iso the
    labelled undirected graphs of the class, n_e its edge count."""
    ids = undirected_class_ids(k)
    ne = np.array([bin(int(c)).count("1") // 2 for c in ids])
    iso = n_iso_undirected(k)
    nmax = k * (k - 1) // 2
    return math.comb(n - 1, k - 1) * iso * p ** ne * (1.0 - p) ** (nmax - ne)


# ------------------------------------------------------------------ edge-level counts
def edge_list(g):
    """G_U edges (u < v), lexicographic: the row order of every edge-level matrix."""
    lib = _load()
    n, s, d = _edges(g)
    ne = ctypes.c_int64(0)
    _check(lib.oracle_edge_list(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d), None, None,
                                ctypes.byref(ne)))
    eu = np.zeros(max(ne.value, 1), np.int32)
    ev = np.zeros(max(ne.value, 1), np.int32)
    _check(lib.oracle_edge_list(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d), _p(eu), _p(ev),
                                ctypes.byref(ne)))
    return eu[: ne.value].copy(), ev[: ne.value].copy()


def count_edges_brute(g, k: int) -> np.ndarray:
    """[edges][C]: the definition over all C(n, k) subsets, every G_U edge of each connected set."""
    lib = _load()
    n, s, d = _edges(g)
    ne = edge_list(g)[0].size
    out = np.zeros((ne, num_classes(k)), np.uint64)
    _check(lib.oracle_count_edges_brute(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d),
                                        ctypes.c_int(k), _p(out)))
    return out


def count_edges_esu(g, k: int, root_lo: int = 0, root_hi: int | None = None, threads: int = 0) -> np.ndarray:
    """[edges][C] via ESU (sets whose minimum original id is in [root_lo, root_hi))."""
    lib = _load()
    n, s, d = _edges(g)
    if root_hi is None:
        root_hi = n
    ne = edge_list(g)[0].size
    out = np.zeros((ne, num_classes(k)), np.uint64)
    _check(lib.oracle_count_edges_esu(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d), ctypes.c_int(k),
                                      ctypes.c_int64(root_lo), ctypes.c_int64(root_hi), ctypes.c_int(threads),
                                      _p(out)))
    return out


def count_edge_rows(g, k: int, eu, ev, threads: int = 0) -> np.ndarray:
    """Rows of sampled G_U edges {eu[i], ev[i]} of count_edges_* (per-edge ESU: every set containing
    eu[i], kept if it contains ev[i])."""
    lib = _load()
    n, s, d = _edges(g)
    eu = np.ascontiguousarray(eu, dtype=np.int32)
    ev = np.ascontiguousarray(ev, dtype=np.int32)
    out = np.zeros((eu.size, num_classes(k)), np.uint64)
    _check(lib.oracle_count_edge_rows(ctypes.c_int64(n), ctypes.c_int64(s.size), _p(s), _p(d), ctypes.c_int(k),
                                      ctypes.c_int64(eu.size), _p(eu), _p(ev), ctypes.c_int(threads), _p(out)))
    return out


def count_edges_py(g, k: int):
    """Pure-Python brute force, tiny graphs: {((u, v), canonical id): count} with u < v."""
    n, s, d = g
    arcs = set(zip(s.tolist(), d.tolist()))
    out: dict = {}
    for S in itertools.combinations(range(n), k):
        und = {(x, y) for x in S for y in S if x < y and ((x, y) in arcs or (y, x) in arcs)}
        comp = {S[0]}
        grew = True
        while grew:
            grew = False
            for (x, y) in und:
                if (x in comp) != (y in comp):
                    comp |= {x, y}
                    grew = True
        if len(comp) < k:
            continue
        best = min(paper_index(k, {(i, j) for i in range(k) for j in range(k)
                                   if i != j and (P[i], P[j]) in arcs})
                   for P in itertools.permutations(S))
        for e in und:
            out[(e, best)] = out.get((e, best), 0) + 1
    return out
