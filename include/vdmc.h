/*
 * vdmc.h -- C ABI of libvdmc.so, the B200 (sm_100a) implementation of VDMC's hot path:
 * per-vertex counts of every connected directed 3- and 4-vertex motif
 * (Levinas, Scherz, Louzoun, arXiv 2201.11655; "P:n" = line n of the paper's PAPER.md).
 *
 * Problem statement: G = (V, E) is an unweighted directed simple
 * graph.  A k-motif is a set of k vertices connected in the underlying undirected graph G_U
 * (P:76-77).  Its class is the minimum, over all k! vertex orders, of the motif index: the
 * k x k adjacency matrix read by rows with the diagonal removed, first entry = most
 * significant bit (Fig. 1; isomorphs merged to the minimum).
 *
 *   counts[v][j] = number of k-motifs S with v in S whose class is vdmc_class_ids(k)[j]
 *                  (every member counted, root included: P:113)
 *
 * Columns are the connected classes in ascending canonical index: 13 for k = 3, 199 for
 * k = 4.  Rows are ORIGINAL vertex ids.  Counts are uint64 (a hub row exceeds 2^32).
 *
 * Conventions for every function:
 *   - returns vdmc_status; VDMC_OK (0) on success.  On failure vdmc_last_error() returns a
 *     thread-local message naming the offending vertex / argument; outputs are untouched
 *     unless stated.
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA global memory on
 *     the graph's device (e.g. a torch CUDA tensor's data_ptr()).
 *   - stream arguments are a cudaStream_t passed as void* (NULL = the legacy default stream).
 *   - no function keeps a pointer the caller passed in: inputs are copied.
 */
#ifndef VDMC_H
#define VDMC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t vdmc_status;
enum {
    VDMC_OK = 0,
    VDMC_EINVAL = 1,     /* NULL pointer, n < 0 or n >= 2^30, bad indptr, bad enum value   */
    VDMC_ERANGE = 2,     /* a vertex id outside [0, n)                                      */
    VDMC_ESELFLOOP = 3,  /* an arc v -> v (the index removes the diagonal: simple graphs) */
    VDMC_EASYM = 4,      /* symmetric-CSR input whose mirror entry or mirrored code is missing */
    VDMC_EORDER = 5,     /* rank is not a permutation of [0, n)                             */
    VDMC_EK = 6,         /* k not in {3, 4}                                                 */
    VDMC_ENOMEM = 7,     /* device or host allocation failed                                */
    VDMC_ECUDA = 8,      /* a CUDA runtime error (message has cudaGetErrorString)            */
    VDMC_ENODEV = 9      /* no CUDA device / invalid device ordinal                         */
};

typedef struct vdmc_graph vdmc_graph;   /* opaque; immutable after build except for scratch */

/* Motif kind.  VDMC_DIRECTED: the classes above.  VDMC_UNDIRECTED:
 * undirected motifs "in the undirected graph induced by ignoring the direction of edges"
 * (G_U): a connected k-set's class is that of its G_U-induced subgraph, indexed by
 * the paper's index of its symmetric adjacency matrix (reading G17), so the
 * columns are the all-mutual directed classes: k = 3 -> [23, 63] (path, triangle); k = 4 ->
 * [591, 669, 735, 1782, 1791, 4095] (star, path, paw, 4-cycle, diamond, clique). */
enum { VDMC_DIRECTED = 0, VDMC_UNDIRECTED = 1 };

/* A contiguous slice [task_lo, task_hi) of the graph's task list.  A task is one
 * (root r, depth-1 neighbour a) pair with rank(a) > rank(r): the paper's unit of GPU work,
 * "each pair of a vertex and one of its neighbors is computed separately".
 * Tasks are ordered by root rank, then by a's rank. */
typedef struct { int64_t task_lo, task_hi; } vdmc_range;

typedef struct {
    int64_t n;          /* vertices                                                    */
    int64_t nnz;        /* entries of the symmetric G_U CSR (= 2 x undirected edges)   */
    int64_t arcs;       /* directed arcs |E| (a mutual pair counts 2)                  */
    int64_t ntasks;     /* (root, neighbour) tasks = nnz / 2                            */
    int64_t max_degree; /* largest G_U degree                                           */
    int32_t device;
} vdmc_graph_info;

/* Build from a directed edge list: arc src[e] -> dst[e], e in [0, m).
 *   src, dst : int32 [m]; host memory if on_device == 0, device memory (on `device`) if 1.
 *   rank     : NULL = the paper's order, undirected degree descending with ties by ascending
 *              id (reading G2/G3); else a host int32 [n] permutation giving each
 *              vertex its position in the order (the result does not depend on it: Lemma 1).
 *   Duplicate arcs are merged; u->v plus v->u is one G_U edge with both direction bits (S1).
 *   Steps run on the device on `stream`; the call returns after the graph is built.
 *   Errors: VDMC_EINVAL, VDMC_ERANGE (message names the arc), VDMC_ESELFLOOP, VDMC_EORDER,
 *           VDMC_ENOMEM, VDMC_ECUDA, VDMC_ENODEV.  *out is set only on success. */
vdmc_status vdmc_build_graph_edges(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                   int on_device, const int32_t *rank, int device, void *stream,
                                   vdmc_graph **out);

/* Build from the symmetric G_U CSR with direction codes (all host memory):
 *   indptr : int64 [n+1], indptr[0] = 0, nondecreasing
 *   nbr    : int32 [indptr[n]], neighbours of each vertex (any order, 0 <= id < n)
 *   dir    : uint8 [indptr[n]], code in {1,2,3}: bit0 = v -> nbr, bit1 = nbr -> v
 *   The entry (v, u, c) must be mirrored by (u, v, swap(c)) after duplicates are OR-merged,
 *   else VDMC_EASYM.  rank / device / out as above (uses the default stream). */
vdmc_status vdmc_build_graph(int64_t n, const int64_t *indptr, const int32_t *nbr,
                             const uint8_t *dir, const int32_t *rank, int device,
                             vdmc_graph **out);

/* Count k-motifs (k in {3,4}) into counts: device uint64 [n][vdmc_num_classes(k)], row =
 * original vertex id, fully overwritten.  work = NULL counts everything; otherwise only the
 * motifs whose (root, depth-1 neighbour) task lies in *work.  The partials of any set of
 * disjoint slices covering [0, ntasks) sum to the full result bit-exactly (integer adds).
 * Asynchronous on `stream`; valid after the stream synchronises.  The call itself may
 * synchronise `stream` once per graph (first count: schedule lists and the heavy-root pre-pass).
 * Errors: VDMC_EK, VDMC_EINVAL (NULL, bad slice, G_U degree >= 2^21), VDMC_ENOMEM, VDMC_ECUDA. */
vdmc_status vdmc_count(vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                       void *stream);

/* vdmc_count for either motif kind: counts is device uint64 [n][vdmc_num_classes_kind(k, kind)].
 * Same enumeration, slices and semantics as vdmc_count; only the class table differs.
 * Errors: as vdmc_count, plus VDMC_EINVAL for kind not in {VDMC_DIRECTED, VDMC_UNDIRECTED}. */
vdmc_status vdmc_count_kind(vdmc_graph *g, int k, int kind, uint64_t *counts, const vdmc_range *work,
                            void *stream);

/* Cost-balanced split of the task list into nparts contiguous slices:
 * parts[p] for p in [0, nparts).  Uses a per-task cost proxy computed on the device
 * (synchronous).  Errors: VDMC_EK, VDMC_EINVAL (nparts < 1 or parts NULL), VDMC_ECUDA. */
vdmc_status vdmc_plan(vdmc_graph *g, int k, int nparts, vdmc_range *parts);

/* Host-only helper used by vdmc_plan: given inclusive prefix sums of per-task costs
 * (host int64 [ntasks], nondecreasing), slice p = [first task whose prefix exceeds
 * p*total/nparts, ...).  Slices are contiguous, disjoint and cover [0, ntasks). */
vdmc_status vdmc_split_costs(const int64_t *prefix, int64_t ntasks, int nparts, vdmc_range *parts);

/* 13 for k = 3, 199 for k = 4, -1 otherwise. */
int vdmc_num_classes(int k);

/* ids[j] = canonical (minimum) paper index of column j, ascending (reading G9).
 * ids: host uint16 [vdmc_num_classes(k)].  Errors: VDMC_EK, VDMC_EINVAL. */
vdmc_status vdmc_class_ids(int k, uint16_t *ids);

/* Class count / column ids for a motif kind: 13 / 199 (directed), 2 / 6 (undirected); -1 (or
 * VDMC_EK / VDMC_EINVAL) for a bad k or kind. */
int vdmc_num_classes_kind(int k, int kind);
vdmc_status vdmc_class_ids_kind(int k, int kind, uint16_t *ids);

/* Graph facts (host struct). */
vdmc_status vdmc_get_info(const vdmc_graph *g, vdmc_graph_info *info);

/* The vertex order used: order[i] = original id of the vertex at position i (host int32 [n]). */
vdmc_status vdmc_get_order(const vdmc_graph *g, int32_t *order);

/* Device-side timing of the last vdmc_count / build on this graph, filled when profiling is
 * on: ms[0] = build (whole), ms[1] = plan, ms[2] = enumeration kernel, ms[3] = finalize,
 * ms[4] = whole count.  Read after the stream has synchronised.  nms <= 5. */
vdmc_status vdmc_set_profiling(vdmc_graph *g, int on);
vdmc_status vdmc_last_timings(const vdmc_graph *g, float *ms, int nms);

/* Number of kernels this library has launched in this process (all graphs, all devices). */
int64_t vdmc_kernel_launches(void);

/* Free the graph and its device memory (NULL is a no-op).  Large device buffers (>= 4 MiB)
 * return to the library's process-wide block cache, so the next build / count on this device
 * reuses them without page mapping; vdmc_trim releases the idle ones. */
void vdmc_free_graph(vdmc_graph *g);

/* Synchronise `device` and release the library's idle cached device blocks to the driver.
 * Blocks held by live graphs are untouched.  Errors: VDMC_ENODEV (no such device), VDMC_ECUDA. */
vdmc_status vdmc_trim(int device);

/* Thread-local message for the last failing call on this thread ("" if none). */
const char *vdmc_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* VDMC_H */
