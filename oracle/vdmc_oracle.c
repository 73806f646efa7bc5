/*
 * vdmc_oracle.c -- plain, slow, obviously-correct CPU oracle for VDMC
 * (Levinas, Scherz, Louzoun, arXiv 2201.11655; /root/reference/PAPER.md = "P:n").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or run this file.  The product
 * path (paper_2201_11655_b200/) never imports, links or calls it, and this file
 * shares no code, header, table or constant generator with it.
 *
 * What it computes (the plain definition the method reaches exactly, Lemma 1,
 * P:142-146): for every k-vertex set S (k in {3,4}) that is connected in the
 * underlying undirected graph G_U,
 *     m   = the paper's motif index of G[S] (Fig. 1),
 *     cls = minimum index over all k! vertex orders,
 *     counts[v][col(cls)] += 1 for every v in S.
 * Columns are the connected classes in ascending canonical index (reading G9).
 *
 * Functions (each cites the passage it follows):
 *   oracle_csr          the paper's directed / undirected CSR
 *   oracle_class_table  index -> min-isomorph index, connectivity, columns
 *   oracle_count_brute  all C(n,k) subsets (the definition written out; Lemma 1 proof P:144)
 *   oracle_count_esu    same result via ESU (Wernicke 2006 "FANMOD", cited P:36), a textbook
 *                       enumeration of connected k-sets with no BFS shapes
 *   oracle_count_vertex per-vertex rows for sampled vertices (ESU with v forced minimal)
 *   oracle_count_bfs    the paper's own method: proper k-BFS(i) per root, BFS depth
 *                       labels, Lemma 3 rules + Lemma 4 correction
 *   oracle_edge_list, oracle_count_edges_brute, oracle_count_edges_esu
 *                       edge-level counts, the Discussion's extension ("counting motifs for
 *                       edges, rather than vertices ... only requires updating edges and not
 *                       vertices once a motif was counted"): for every connected k-set S and every
 *                       G_U edge {x, y} inside S, ecounts[row(x, y)][col] += 1 (reading G18)
 *
 * Pins: tests/test_oracle_*.py (brute force vs closed forms, hand-worked golden,
 * single-motif graphs, invariants, Eq. 4).  No function here is "parity unpinned".
 *
 * Error codes: 0 ok, -1 bad argument, -2 vertex id out of range, -3 self-loop, -4 alloc failure.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define MAXK 5   /* k = 5: SURVEY §8(f) NEXT-3, "appropriate for 5 motifs too" */
#define MAXCLASSES 16384

/* ------------------------------------------------------------------ graph */
typedef struct {
    int64_t n;
    int64_t *oind; int32_t *onbr;   /* directed CSR: out-neighbours, sorted, unique */
    int64_t *uind; int32_t *unbr;   /* G_U CSR: undirected neighbours, sorted, unique */
} ograph;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* CSR from a list of (row, col) pairs: counting sort by row, then sort+dedup each row. */
static int build_csr(int64_t n, int64_t m, const int32_t *row, const int32_t *col,
                     int64_t **ind_out, int32_t **nbr_out) {
    int64_t *ind = calloc((size_t)n + 1, sizeof(int64_t));
    int32_t *nbr = malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    int64_t *fill = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!ind || !nbr || !fill) { free(ind); free(nbr); free(fill); return -4; }
    for (int64_t e = 0; e < m; e++) ind[row[e] + 1]++;
    for (int64_t v = 0; v < n; v++) ind[v + 1] += ind[v];
    for (int64_t v = 0; v < n; v++) fill[v] = ind[v];
    for (int64_t e = 0; e < m; e++) nbr[fill[row[e]]++] = col[e];
    /* sort and dedup each list, compacting in place */
    int64_t w = 0;
    for (int64_t v = 0; v < n; v++) {
        int64_t b = ind[v], e = ind[v + 1];
        qsort(nbr + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
        int64_t start = w;
        for (int64_t i = b; i < e; i++)
            if (i == b || nbr[i] != nbr[i - 1]) nbr[w++] = nbr[i];
        ind[v] = start;
    }
    ind[n] = w;
    free(fill);
    *ind_out = ind; *nbr_out = nbr;
    return 0;
}

static void free_graph(ograph *g) {
    free(g->oind); free(g->onbr); free(g->uind); free(g->unbr);
    memset(g, 0, sizeof(*g));
}

static int make_graph(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, ograph *g) {
    memset(g, 0, sizeof(*g));
    if (n < 0 || m < 0 || (m > 0 && (!src || !dst))) return -1;
    for (int64_t e = 0; e < m; e++) {
        if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n) return -2;
        if (src[e] == dst[e]) return -3;   /* simple graph, no self edges */
    }
    g->n = n;
    int rc = build_csr(n, m, src, dst, &g->oind, &g->onbr);
    if (rc) return rc;
    /* G_U: ignore the direction of every edge */
    int32_t *r2 = malloc((size_t)(2 * m + 1) * sizeof(int32_t));
    int32_t *c2 = malloc((size_t)(2 * m + 1) * sizeof(int32_t));
    if (!r2 || !c2) { free(r2); free(c2); free_graph(g); return -4; }
    for (int64_t e = 0; e < m; e++) {
        r2[2 * e] = src[e]; c2[2 * e] = dst[e];
        r2[2 * e + 1] = dst[e]; c2[2 * e + 1] = src[e];
    }
    rc = build_csr(n, 2 * m, r2, c2, &g->uind, &g->unbr);
    free(r2); free(c2);
    if (rc) free_graph(g);
    return rc;
}

static int in_sorted(const int32_t *a, int64_t len, int32_t x) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo < len && a[lo] == x;
}
static int has_arc(const ograph *g, int32_t x, int32_t y) {      /* x -> y in G */
    return in_sorted(g->onbr + g->oind[x], g->oind[x + 1] - g->oind[x], y);
}
static int adjacent(const ograph *g, int32_t x, int32_t y) {     /* {x,y} in G_U */
    return in_sorted(g->unbr + g->uind[x], g->uind[x + 1] - g->uind[x], y);
}

/* ----------------------------------------------------------- motif index */
/* Paper's index (Fig. 1): the k x k adjacency matrix read by rows with
 * the diagonal removed, first entry = most significant bit.  Bit of ordered pair (i,j): */
static int pair_bit(int k, int i, int j) {
    int idx = i * (k - 1) + (j < i ? j : j - 1);   /* position in the row-major off-diagonal list */
    return k * (k - 1) - 1 - idx;
}

static int index_of_matrix(int k, int a[MAXK][MAXK]) {
    int m = 0;
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++)
            if (i != j && a[i][j]) m |= 1 << pair_bit(k, i, j);
    return m;
}

static void matrix_of_index(int k, int m, int a[MAXK][MAXK]) {
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++)
            a[i][j] = (i != j) && ((m >> pair_bit(k, i, j)) & 1);
}

/* next lexicographic permutation; returns 0 after the last one */
static int next_perm(int *p, int k) {
    int i = k - 2;
    while (i >= 0 && p[i] >= p[i + 1]) i--;
    if (i < 0) return 0;
    int j = k - 1;
    while (p[j] <= p[i]) j--;
    int t = p[i]; p[i] = p[j]; p[j] = t;
    for (int l = i + 1, r = k - 1; l < r; l++, r--) { t = p[l]; p[l] = p[r]; p[r] = t; }
    return 1;
}

static int uf_find(int *par, int x) { while (par[x] != x) x = par[x] = par[par[x]]; return x; }

/* Weakly connected: connected in the underlying undirected graph. */
static int matrix_connected(int k, int a[MAXK][MAXK]) {
    int par[MAXK];
    for (int i = 0; i < k; i++) par[i] = i;
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++)
            if (a[i][j]) par[uf_find(par, i)] = uf_find(par, j);
    for (int i = 1; i < k; i++) if (uf_find(par, i) != uf_find(par, 0)) return 0;
    return 1;
}

typedef struct {
    int k, nbits, nclasses;
    int32_t *canon;      /* [2^nbits] minimum index over all k! orders */
    uint8_t *conn;       /* [2^nbits] weakly connected? */
    int32_t *col;        /* [2^nbits] column of canon (ascending canonical ids), -1 if disconnected */
    int32_t class_ids[MAXCLASSES];   /* 13 / 199 / 9364 for k = 3 / 4 / 5 */
} otable;

static int make_table(int k, otable *t) {
    memset(t, 0, sizeof(*t));
    if (k < 3 || k > MAXK) return -1;
    t->k = k; t->nbits = k * (k - 1);
    int M = 1 << t->nbits;
    t->canon = malloc((size_t)M * sizeof(int32_t));
    t->conn = malloc((size_t)M);
    t->col = malloc((size_t)M * sizeof(int32_t));
    if (!t->canon || !t->conn || !t->col) return -4;
    #pragma omp parallel for schedule(static)
    for (int m = 0; m < M; m++) {
        int a[MAXK][MAXK], b[MAXK][MAXK], p[MAXK];
        matrix_of_index(k, m, a);
        t->conn[m] = (uint8_t)matrix_connected(k, a);
        for (int i = 0; i < k; i++) p[i] = i;
        int best = M;
        do {   /* relabel: new vertex i is old vertex p[i] */
            for (int i = 0; i < k; i++)
                for (int j = 0; j < k; j++) b[i][j] = a[p[i]][p[j]];
            int x = index_of_matrix(k, b);
            if (x < best) best = x;
        } while (next_perm(p, k));
        t->canon[m] = best;
    }
    /* columns: connected canonical ids in ascending order (reading G9) */
    int nc = 0;
    for (int m = 0; m < M; m++)
        if (t->conn[m] && t->canon[m] == m) t->class_ids[nc++] = m;
    t->nclasses = nc;
    for (int m = 0; m < M; m++) {
        t->col[m] = -1;
        if (!t->conn[m]) continue;
        int lo = 0, hi = nc;   /* class_ids ascending: binary search for canon[m] */
        while (lo < hi) { int mid = (lo + hi) / 2; if (t->class_ids[mid] < t->canon[m]) lo = mid + 1; else hi = mid; }
        t->col[m] = lo;
    }
    return 0;
}

static void free_table(otable *t) { free(t->canon); free(t->conn); free(t->col); }

/* classify the set (v[0..k-1]) in this vertex order; returns its column */
static int classify(const ograph *g, const otable *t, const int32_t *v) {
    int a[MAXK][MAXK];
    for (int i = 0; i < t->k; i++)
        for (int j = 0; j < t->k; j++)
            a[i][j] = (i != j) && has_arc(g, v[i], v[j]);
    return t->col[index_of_matrix(t->k, a)];
}

/* +1 in that class for every vertex of the set, root included */
static void add_set(uint64_t *counts, int nc, int k, const int32_t *v, int col) {
    for (int i = 0; i < k; i++) {
        #pragma omp atomic
        counts[(int64_t)v[i] * nc + col] += 1;
    }
}

/* ----------------------------------------------------- edge-level counts */
/* Edge rows: the G_U edges {x < y} in lexicographic order, i.e. the upper entries of the
 * undirected CSR read row by row.  erow[e] = row of the pair of CSR entry e (both
 * entries of a pair get the same row). */
static int64_t *edge_rows(const ograph *g, int64_t *nedges) {
    int64_t nnz = g->uind[g->n];
    int64_t *erow = malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int64_t));
    if (!erow) return NULL;
    int64_t row = 0;
    for (int32_t x = 0; x < g->n; x++)
        for (int64_t e = g->uind[x]; e < g->uind[x + 1]; e++)
            if (g->unbr[e] > x) erow[e] = row++;
    for (int32_t x = 0; x < g->n; x++)
        for (int64_t e = g->uind[x]; e < g->uind[x + 1]; e++) {
            int32_t y = g->unbr[e];
            if (y > x) continue;
            /* the mirror entry x in y's list */
            int64_t lo = g->uind[y], hi = g->uind[y + 1];
            while (lo < hi) { int64_t mid = (lo + hi) / 2; if (g->unbr[mid] < x) lo = mid + 1; else hi = mid; }
            erow[e] = erow[lo];
        }
    *nedges = row;
    return erow;
}

static int64_t edge_row(const ograph *g, const int64_t *erow, int32_t x, int32_t y) {
    int64_t lo = g->uind[x], hi = g->uind[x + 1];
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (g->unbr[mid] < y) lo = mid + 1; else hi = mid; }
    return erow[lo];
}

/* +1 in that class for every G_U edge of the set ("updating edges and not vertices") */
static void add_set_edges(const ograph *g, const int64_t *erow, uint64_t *ecounts, int nc, int k,
                          const int32_t *v, int col) {
    for (int a = 0; a < k; a++)
        for (int b = a + 1; b < k; b++)
            if (adjacent(g, v[a], v[b])) {
                #pragma omp atomic
                ecounts[edge_row(g, erow, v[a], v[b]) * nc + col] += 1;
            }
}

/* ================================================================ exports */

/* The paper's CSR for a directed edge list: directed out-lists and G_U lists. */
int oracle_csr(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
               int64_t *oind, int32_t *onbr, int64_t *undi, int32_t *unbr) {
    ograph g;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    memcpy(oind, g.oind, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(onbr, g.onbr, (size_t)g.oind[n] * sizeof(int32_t));
    memcpy(undi, g.uind, (size_t)(n + 1) * sizeof(int64_t));
    memcpy(unbr, g.unbr, (size_t)g.uind[n] * sizeof(int32_t));
    free_graph(&g);
    return 0;
}

int oracle_class_table(int k, int32_t *canon, uint8_t *conn, int32_t *col,
                       int32_t *class_ids, int32_t *nclasses) {
    otable t;
    int rc = make_table(k, &t);
    if (rc) { if (rc != -1) free_table(&t); return rc; }
    int M = 1 << t.nbits;
    if (canon) memcpy(canon, t.canon, (size_t)M * sizeof(int32_t));
    if (conn) memcpy(conn, t.conn, (size_t)M);
    if (col) memcpy(col, t.col, (size_t)M * sizeof(int32_t));
    if (class_ids) memcpy(class_ids, t.class_ids, (size_t)t.nclasses * sizeof(int32_t));
    if (nclasses) *nclasses = t.nclasses;
    free_table(&t);
    return 0;
}

/* Definition written out: every k-subset, connectivity by union-find on G_U[S]. */
int oracle_count_brute(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                       int k, uint64_t *counts) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    memset(counts, 0, (size_t)n * t.nclasses * sizeof(uint64_t));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i0 = 0; i0 < n; i0++) {
        /* every combination i0 < c[1] < ... < c[k-1] < n, in lexicographic order */
        int64_t c[MAXK];
        c[0] = i0;
        for (int a = 1; a < k; a++) c[a] = i0 + a;
        if (c[k - 1] >= n) continue;
        for (;;) {
            int32_t v[MAXK];
            for (int a = 0; a < k; a++) v[a] = (int32_t)c[a];
            int par[MAXK];
            for (int a = 0; a < k; a++) par[a] = a;
            for (int a = 0; a < k; a++)
                for (int b = a + 1; b < k; b++)
                    if (adjacent(&g, v[a], v[b])) par[uf_find(par, a)] = uf_find(par, b);
            int ok = 1;
            for (int a = 1; a < k; a++) if (uf_find(par, a) != uf_find(par, 0)) ok = 0;
            if (ok) add_set(counts, t.nclasses, k, v, classify(&g, &t, v));
            int a = k - 1;
            while (a >= 1 && c[a] == n - k + a) a--;
            if (a < 1) break;
            c[a]++;
            for (int b = a + 1; b < k; b++) c[b] = c[b - 1] + 1;
        }
    }
    free_table(&t); free_graph(&g);
    return 0;
}

/* ---------------------------------------------------------------- ESU */
/* Wernicke's ESU (FANMOD, cited at P:36) enumerates every connected k-set whose minimum
 * (under the order "allowed") is the root exactly once:
 *   ExtendSubgraph(Vsub, Vext, v):
 *     if |Vsub| = k: output Vsub
 *     while Vext != {}: remove w from Vext;
 *        Vext' = Vext u { u in N_excl(w, Vsub) : u > v };  ExtendSubgraph(Vsub u {w}, Vext', v)
 *   with N_excl(w, Vsub) = N(w) \ (Vsub u N(Vsub)).
 * Per-thread state: nsub[u] = |N(u) n Vsub| (u in N(Vsub) iff nsub[u] > 0), insub[u]. */
typedef struct {
    const ograph *g; const otable *t; uint64_t *counts;
    uint64_t *ecounts; const int64_t *erow;  /* edge-level mode: per G_U edge, else NULL */
    int32_t need; uint64_t *row;             /* edge-row mode: only sets containing `need`, into row */
    int k; int32_t root; int root_is_min;   /* root_is_min: every other vertex is "> root" */
    int32_t *nsub; uint8_t *insub;
    int32_t sub[MAXK];
    uint64_t nsets;
} esu_ctx;

static void esu_push(esu_ctx *c, int32_t w, int s) {
    c->sub[s] = w; c->insub[w] = 1;
    for (int64_t e = c->g->uind[w]; e < c->g->uind[w + 1]; e++) c->nsub[c->g->unbr[e]]++;
}
static void esu_pop(esu_ctx *c, int32_t w) {
    c->insub[w] = 0;
    for (int64_t e = c->g->uind[w]; e < c->g->uind[w + 1]; e++) c->nsub[c->g->unbr[e]]--;
}

static void esu_extend(esu_ctx *c, int s, int32_t *ext, int64_t next) {
    if (s == c->k) {
        if (c->row) {   /* edge-row mode: the root is one end of the edge, `need` the other */
            int has = 0;
            for (int i = 0; i < c->k; i++) has |= c->sub[i] == c->need;
            if (has) c->row[classify(c->g, c->t, c->sub)] += 1;
        } else if (c->ecounts)
            add_set_edges(c->g, c->erow, c->ecounts, c->t->nclasses, c->k, c->sub, classify(c->g, c->t, c->sub));
        else
            add_set(c->counts, c->t->nclasses, c->k, c->sub, classify(c->g, c->t, c->sub));
        c->nsets++;
        return;
    }
    while (next > 0) {
        int32_t w = ext[--next];
        /* Vext' = remaining Vext, then the exclusive neighbours of w (computed vs. Vsub before w) */
        int64_t cap = next + (c->g->uind[w + 1] - c->g->uind[w]);
        int32_t *ext2 = malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int32_t));
        memcpy(ext2, ext, (size_t)next * sizeof(int32_t));
        int64_t n2 = next;
        if (s + 1 < c->k)
            for (int64_t e = c->g->uind[w]; e < c->g->uind[w + 1]; e++) {
                int32_t u = c->g->unbr[e];
                int greater = c->root_is_min ? (u != c->root) : (u > c->root);
                if (greater && !c->insub[u] && c->nsub[u] == 0) ext2[n2++] = u;
            }
        esu_push(c, w, s);
        esu_extend(c, s + 1, ext2, n2);
        esu_pop(c, w);
        free(ext2);
    }
}

static void esu_root(esu_ctx *c) {
    const ograph *g = c->g;
    int32_t v = c->root;
    int64_t deg = g->uind[v + 1] - g->uind[v];
    int32_t *ext = malloc((size_t)(deg > 0 ? deg : 1) * sizeof(int32_t));
    int64_t ne = 0;
    for (int64_t e = g->uind[v]; e < g->uind[v + 1]; e++) {
        int32_t u = g->unbr[e];
        if (c->root_is_min || u > v) ext[ne++] = u;
    }
    esu_push(c, v, 0);
    esu_extend(c, 1, ext, ne);
    esu_pop(c, v);
    free(ext);
}

/* All connected k-sets whose minimum ORIGINAL id lies in [root_lo, root_hi). Summing the
 * results of any cover of [0, n) by disjoint ranges gives the full count matrix. */
int oracle_count_esu(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int k,
                     int64_t root_lo, int64_t root_hi, int nthreads, uint64_t *counts,
                     uint64_t *nsets_out) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    if (root_lo < 0) root_lo = 0;
    if (root_hi > n) root_hi = n;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    memset(counts, 0, (size_t)n * t.nclasses * sizeof(uint64_t));
    if (nthreads > 0) omp_set_num_threads(nthreads);
    uint64_t total = 0;
    #pragma omp parallel reduction(+:total)
    {
        esu_ctx c;
        memset(&c, 0, sizeof(c));
        c.g = &g; c.t = &t; c.counts = counts; c.k = k;
        c.nsub = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
        c.insub = calloc((size_t)(n > 0 ? n : 1), 1);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t r = root_lo; r < root_hi; r++) {
            c.root = (int32_t)r; c.root_is_min = 0;
            esu_root(&c);
        }
        total += c.nsets;
        free(c.nsub); free(c.insub);
    }
    if (nsets_out) *nsets_out = total;
    free_table(&t); free_graph(&g);
    return 0;
}

/* Row of each sampled vertex v: ESU from v with v treated as the minimum of the order, which
 * enumerates every connected k-set containing v exactly once.  rows: [nv][nclasses]. */
int oracle_count_vertex(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int k,
                        int64_t nv, const int32_t *verts, int nthreads, uint64_t *rows) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    for (int64_t i = 0; i < nv; i++) if (verts[i] < 0 || verts[i] >= n) return -2;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    int nc = t.nclasses;
    memset(rows, 0, (size_t)nv * nc * sizeof(uint64_t));
    if (nthreads > 0) omp_set_num_threads(nthreads);
    #pragma omp parallel
    {
        esu_ctx c;
        memset(&c, 0, sizeof(c));
        c.g = &g; c.t = &t; c.k = k;
        c.nsub = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
        c.insub = calloc((size_t)(n > 0 ? n : 1), 1);
        uint64_t *tmp = calloc((size_t)(n > 0 ? n : 1) * nc, sizeof(uint64_t));
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < nv; i++) {
            c.counts = tmp;
            c.root = verts[i]; c.root_is_min = 1;
            esu_root(&c);
            memcpy(rows + i * nc, tmp + (int64_t)verts[i] * nc, (size_t)nc * sizeof(uint64_t));
            memset(tmp, 0, (size_t)n * nc * sizeof(uint64_t));   /* plain and slow, by design */
        }
        free(tmp); free(c.nsub); free(c.insub);
    }
    free_table(&t); free_graph(&g);
    return 0;
}

/* ------------------------------------------------------ the paper's method */
/* VDMC as written: vertices in a given order ("index" = position; rank==NULL
 * means original ids).  For each root i, a BFS in G_U over vertices of higher index gives
 * every vertex its minimal depth.  Proper k-BFS(i) trees are enumerated by
 * shape (Lemma 2): k=3: "2" (avg depth 2/3) and "1+1" (avg depth 1); k=4: "3"
 * (0.75), "2+1" (1), "1+2" (1.25), "1+1+1" (1.5).  Lemma 3: a tree edge never goes
 * from a depth to a lower or equal depth, and same-depth vertices follow index order.
 * Lemma 4: in the 1.5 chain the last vertex is accepted with global label 2
 * or 3 as long as it is not adjacent to the chain's depth-1 vertex (reading G4).  A depth-2
 * vertex adjacent to both depth-1 vertices of a "2+1" tree is taken from the first
 * (lower-index) one only (reading G5).  Vertices are ordered by depth then index before
 * the index is computed; the column does not depend on that order. */
int oracle_count_bfs(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int k,
                     const int32_t *rank, uint64_t *counts) {
    otable t; ograph g;
    if (k != 3 && k != 4) return -1;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    int nc = t.nclasses;
    memset(counts, 0, (size_t)n * nc * sizeof(uint64_t));
    int64_t *idx = malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));   /* index of vertex */
    int32_t *byidx = malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t)); /* vertex at index */
    for (int64_t v = 0; v < n; v++) idx[v] = rank ? rank[v] : v;
    for (int64_t v = 0; v < n; v++) byidx[idx[v]] = (int32_t)v;
    #pragma omp parallel
    {
        int8_t *depth = malloc((size_t)(n > 0 ? n : 1));
        int32_t *queue = malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
        int32_t *touched = malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
        memset(depth, -1, (size_t)(n > 0 ? n : 1));
        #pragma omp for schedule(dynamic, 1)
        for (int64_t ii = 0; ii < n; ii++) {
            int32_t i = byidx[ii];
            /* BFS over vertices with higher index, depth <= k-1 */
            int64_t qh = 0, qt = 0, nt = 0;
            depth[i] = 0; queue[qt++] = i; touched[nt++] = i;
            while (qh < qt) {
                int32_t x = queue[qh++];
                if (depth[x] >= k - 1) continue;
                for (int64_t e = g.uind[x]; e < g.uind[x + 1]; e++) {
                    int32_t y = g.unbr[e];
                    if (idx[y] <= ii || depth[y] >= 0) continue;
                    depth[y] = (int8_t)(depth[x] + 1);
                    queue[qt++] = y; touched[nt++] = y;
                }
            }
            /* depth-1 vertices in index order */
            int64_t n1 = 0;
            for (int64_t e = g.uind[i]; e < g.uind[i + 1]; e++)
                if (depth[g.unbr[e]] == 1) n1++;
            int32_t *d1 = malloc((size_t)(n1 > 0 ? n1 : 1) * sizeof(int32_t));
            n1 = 0;
            for (int64_t e = g.uind[i]; e < g.uind[i + 1]; e++)
                if (depth[g.unbr[e]] == 1) d1[n1++] = g.unbr[e];
            /* sort by index (insertion sort: plain) */
            for (int64_t a = 1; a < n1; a++) {
                int32_t x = d1[a]; int64_t b = a - 1;
                while (b >= 0 && idx[d1[b]] > idx[x]) { d1[b + 1] = d1[b]; b--; }
                d1[b + 1] = x;
            }
            int32_t v[MAXK];
            v[0] = i;
            for (int64_t a = 0; a < n1; a++) {
                int32_t A = d1[a];
                v[1] = A;
                if (k == 3) {
                    /* "2": two depth-1 vertices in index order */
                    for (int64_t b = a + 1; b < n1; b++) {
                        v[2] = d1[b];
                        add_set(counts, nc, 3, v, classify(&g, &t, v));
                    }
                    /* "1+1": a depth-2 child of A (tree edge depth 1 -> 2 only) */
                    for (int64_t e = g.uind[A]; e < g.uind[A + 1]; e++) {
                        int32_t B = g.unbr[e];
                        if (depth[B] != 2) continue;
                        v[2] = B;
                        add_set(counts, nc, 3, v, classify(&g, &t, v));
                    }
                    continue;
                }
                for (int64_t b = a + 1; b < n1; b++) {
                    int32_t B = d1[b];
                    v[2] = B;
                    /* "3": three depth-1 vertices in index order */
                    for (int64_t c = b + 1; c < n1; c++) {
                        v[3] = d1[c];
                        add_set(counts, nc, 4, v, classify(&g, &t, v));
                    }
                    /* "2+1": a depth-2 child of A, or of B when not also a child of A (G5) */
                    for (int64_t e = g.uind[A]; e < g.uind[A + 1]; e++) {
                        int32_t C = g.unbr[e];
                        if (depth[C] != 2) continue;
                        v[3] = C;
                        add_set(counts, nc, 4, v, classify(&g, &t, v));
                    }
                    for (int64_t e = g.uind[B]; e < g.uind[B + 1]; e++) {
                        int32_t C = g.unbr[e];
                        if (depth[C] != 2 || adjacent(&g, A, C)) continue;
                        v[3] = C;
                        add_set(counts, nc, 4, v, classify(&g, &t, v));
                    }
                }
                /* "1+2": two depth-2 children of A in index order */
                for (int64_t e = g.uind[A]; e < g.uind[A + 1]; e++) {
                    int32_t B = g.unbr[e];
                    if (depth[B] != 2) continue;
                    for (int64_t f = g.uind[A]; f < g.uind[A + 1]; f++) {
                        int32_t C = g.unbr[f];
                        if (depth[C] != 2 || idx[C] <= idx[B]) continue;
                        v[2] = B; v[3] = C;
                        add_set(counts, nc, 4, v, classify(&g, &t, v));
                    }
                }
                /* "1+1+1": chain i - A - B - C; B a depth-2 child of A; C a child of B with
                 * label 3, or label 2 but not adjacent to A (Lemma 4 correction) */
                for (int64_t e = g.uind[A]; e < g.uind[A + 1]; e++) {
                    int32_t B = g.unbr[e];
                    if (depth[B] != 2) continue;
                    v[2] = B;
                    for (int64_t f = g.uind[B]; f < g.uind[B + 1]; f++) {
                        int32_t C = g.unbr[f];
                        if (depth[C] == 3 || (depth[C] == 2 && !adjacent(&g, A, C))) {
                            v[3] = C;
                            add_set(counts, nc, 4, v, classify(&g, &t, v));
                        }
                    }
                }
            }
            free(d1);
            for (int64_t q = 0; q < nt; q++) depth[touched[q]] = -1;
        }
        free(depth); free(queue); free(touched);
    }
    free(idx); free(byidx);
    free_table(&t); free_graph(&g);
    return 0;
}

/* ------------------------------------------------------ edge-level exports */
/* The G_U edge rows: eu[r] < ev[r], lexicographic.  eu/ev may be NULL (count only). */
int oracle_edge_list(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                     int32_t *eu, int32_t *ev, int64_t *nedges) {
    ograph g;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    int64_t row = 0;
    for (int32_t x = 0; x < n; x++)
        for (int64_t e = g.uind[x]; e < g.uind[x + 1]; e++)
            if (g.unbr[e] > x) {
                if (eu) eu[row] = x;
                if (ev) ev[row] = g.unbr[e];
                row++;
            }
    *nedges = row;
    free_graph(&g);
    return 0;
}

/* Definition written out for edges: every k-subset connected in G_U, +1 in its class for every
 * G_U edge inside it.  ecounts: [nedges][nclasses], rows as oracle_edge_list. */
int oracle_count_edges_brute(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                             int k, uint64_t *ecounts) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    int64_t ne = 0;
    int64_t *erow = edge_rows(&g, &ne);
    if (!erow) { free_table(&t); free_graph(&g); return -4; }
    memset(ecounts, 0, (size_t)ne * t.nclasses * sizeof(uint64_t));
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i0 = 0; i0 < n; i0++) {
        int64_t c[MAXK];
        c[0] = i0;
        for (int a = 1; a < k; a++) c[a] = i0 + a;
        if (c[k - 1] >= n) continue;
        for (;;) {
            int32_t v[MAXK];
            for (int a = 0; a < k; a++) v[a] = (int32_t)c[a];
            int par[MAXK];
            for (int a = 0; a < k; a++) par[a] = a;
            for (int a = 0; a < k; a++)
                for (int b = a + 1; b < k; b++)
                    if (adjacent(&g, v[a], v[b])) par[uf_find(par, a)] = uf_find(par, b);
            int ok = 1;
            for (int a = 1; a < k; a++) if (uf_find(par, a) != uf_find(par, 0)) ok = 0;
            if (ok) add_set_edges(&g, erow, ecounts, t.nclasses, k, v, classify(&g, &t, v));
            int a = k - 1;
            while (a >= 1 && c[a] == n - k + a) a--;
            if (a < 1) break;
            c[a]++;
            for (int b = a + 1; b < k; b++) c[b] = c[b - 1] + 1;
        }
    }
    free(erow); free_table(&t); free_graph(&g);
    return 0;
}

/* The same via ESU (every connected k-set once, from its minimum id in [root_lo, root_hi)). */
int oracle_count_edges_esu(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int k,
                           int64_t root_lo, int64_t root_hi, int nthreads, uint64_t *ecounts) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    if (root_lo < 0) root_lo = 0;
    if (root_hi > n) root_hi = n;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    int64_t ne = 0;
    int64_t *erow = edge_rows(&g, &ne);
    if (!erow) { free_table(&t); free_graph(&g); return -4; }
    memset(ecounts, 0, (size_t)ne * t.nclasses * sizeof(uint64_t));
    if (nthreads > 0) omp_set_num_threads(nthreads);
    #pragma omp parallel
    {
        esu_ctx c;
        memset(&c, 0, sizeof(c));
        c.g = &g; c.t = &t; c.ecounts = ecounts; c.erow = erow; c.k = k;
        c.nsub = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
        c.insub = calloc((size_t)(n > 0 ? n : 1), 1);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t r = root_lo; r < root_hi; r++) {
            c.root = (int32_t)r; c.root_is_min = 0;
            esu_root(&c);
        }
        free(c.nsub); free(c.insub);
    }
    free(erow); free_table(&t); free_graph(&g);
    return 0;
}

/* Rows of sampled edges {eu[i], ev[i]} (must be G_U edges): every connected k-set containing
 * both ends, per class -- ESU from eu[i] with eu[i] treated as the minimum (every set containing
 * it, once), keeping the sets that contain ev[i].  rows: [ne][nclasses]. */
int oracle_count_edge_rows(int64_t n, int64_t m, const int32_t *src, const int32_t *dst, int k,
                           int64_t ne, const int32_t *eu, const int32_t *ev, int nthreads, uint64_t *rows) {
    otable t; ograph g;
    if (k < 3 || k > MAXK) return -1;
    for (int64_t i = 0; i < ne; i++)
        if (eu[i] < 0 || eu[i] >= n || ev[i] < 0 || ev[i] >= n) return -2;
    int rc = make_graph(n, m, src, dst, &g);
    if (rc) return rc;
    for (int64_t i = 0; i < ne; i++)
        if (!adjacent(&g, eu[i], ev[i])) { free_graph(&g); return -1; }
    if ((rc = make_table(k, &t))) { free_graph(&g); return rc; }
    int nc = t.nclasses;
    memset(rows, 0, (size_t)ne * nc * sizeof(uint64_t));
    if (nthreads > 0) omp_set_num_threads(nthreads);
    #pragma omp parallel
    {
        esu_ctx c;
        memset(&c, 0, sizeof(c));
        c.g = &g; c.t = &t; c.k = k;
        c.nsub = calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
        c.insub = calloc((size_t)(n > 0 ? n : 1), 1);
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < ne; i++) {
            c.row = rows + i * nc;
            c.need = ev[i];
            c.root = eu[i]; c.root_is_min = 1;
            esu_root(&c);
        }
        free(c.nsub); free(c.insub);
    }
    free_table(&t); free_graph(&g);
    return 0;
}
