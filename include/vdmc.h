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
 *   - a vdmc_graph is immutable once built: every count call takes a const handle and draws
 *     its working memory (accumulator, work counters, scratch) per call, so one graph may be
 *     counted concurrently from several host threads / streams.
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
    VDMC_ENODEV = 9,     /* no CUDA device / invalid device ordinal                         */
    VDMC_ENCCL = 10      /* an NCCL error in the multi-GPU reduce (message has ncclGetErrorString) */
};

typedef struct vdmc_graph vdmc_graph;   /* opaque; immutable after build */

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
 * Tasks are ordered by root rank, then by a's rank; there is one task per G_U edge. */
typedef struct { int64_t task_lo, task_hi; } vdmc_range;

typedef struct {
    int64_t n;          /* vertices                                                    */
    int64_t nnz;        /* entries of the symmetric G_U CSR (= 2 x undirected edges)   */
    int64_t arcs;       /* directed arcs |E| (a mutual pair counts 2)                  */
    int64_t ntasks;     /* (root, neighbour) tasks = nnz / 2 = undirected edges         */
    int64_t max_degree; /* largest G_U degree                                           */
    int32_t device;
    float build_ms;     /* device time of the build (S1 + S2 + the S4 schedule)         */
} vdmc_graph_info;

/* Per-call options of vdmc_count_ex.  Zero-initialise and set what you need; every field's 0
 * means "the default".  All path options are RESULT-PRESERVING: they choose how the same sets
 * are enumerated, never which (tests force each path and compare with the oracle).
 *   kind         VDMC_DIRECTED (0) or VDMC_UNDIRECTED
 *   star_block   0 (default): the heavy "3" sets are counted in closed form per task (key
 *                histograms of N+(r) plus the sets with an induced edge, classified one by one);
 *                in [1, 1023]: they are enumerated instead, in work items of that many b positions
 *   cross_block  R positions per heavy "2+1" work item, in [32, 1023] (default 256)
 *   heavy_global 1 = heavy-task buffers in global memory (the path taken when the largest
 *                degree does not fit shared memory)
 *   force_big    1 = flush the 32-bit per-warp histograms after every work item (the path
 *                taken when the largest degree exceeds 32767)
 *   ca_capacity  entries of the per-CTA scratch holding the R-neighbour lists of a heavy
 *                task's depth-2 vertices (default 65536); a task whose lists do not fit
 *                enumerates its "2+1" sets one depth-2 vertex at a time instead
 *   acc64        1 = 64-bit accumulator words even when 32 bits provably suffice (the library
 *                uses 32-bit words when 6 maxdeg^3 < 2^32 (k = 4) / 2 maxdeg^2 < 2^32 (k = 3):
 *                a bound on the connected sets through one vertex, so no count can wrap)
 *   layered      1 = the generic BFS-layer path (layers.cu; the only path for k = 5) for k = 3 / 4
 *   timings_ms   NULL, or host float[4] filled with device times (schedule + memset, enumerate,
 *                finalise, whole call); the call then synchronises `stream` before returning */
typedef struct {
    int32_t kind;
    int32_t star_block;
    int32_t cross_block;
    int32_t heavy_global;
    int32_t force_big;
    int32_t layered;
    int32_t acc64;
    int32_t reserved0;
    int64_t ca_capacity;
    float *timings_ms;
} vdmc_count_options;

/* Build from a directed edge list: arc src[e] -> dst[e], e in [0, m).
 *   src, dst : int32 [m]; host memory if on_device == 0, device memory (on `device`) if 1.
 *   rank     : NULL = the paper's order, undirected degree descending with ties by ascending
 *              id (reading G2/G3); else a host int32 [n] permutation giving each
 *              vertex its position in the order (the result does not depend on it: Lemma 1).
 *   Duplicate arcs are merged; u->v plus v->u is one G_U edge with both direction bits (S1).
 *   S1, S2, the class tables (S3) and the S4 schedule (heavy/light lists, induced adjacency
 *   of heavy roots) are all built here, on the device, on `stream`; the call returns after
 *   the graph is built.
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

/* The paper's CSR -> the symmetric G_U CSR with direction codes.
 *   in : out_indptr int64 [n+1] and out_nbr int32 [out_indptr[n]]: the paper's directed CSR
 *        ("Indices" / "Neighbors"): the out-neighbours of each vertex.
 *   out: *indptr int64 [n+1], *nbr int32 [nnz], *dir uint8 [nnz]: the undirected CSR of
 *        P:133, each list ascending by neighbour id, one entry per G_U edge end with its
 *        direction code (bit0 = v -> nbr, bit1 = nbr -> v; a mutual pair is ONE entry with
 *        code 3, reading G14).  Example: arcs 0->1 0->2 0->3 2->0 3->1 3->2 give
 *        indptr [0,3,5,7,10], nbr [1,2,3, 0,3, 0,3, 0,1,2], dir [1,3,1, 2,2, 3,2, 2,1,1].
 *   The three outputs are allocated by the library (host); free each with vdmc_free_host.
 *   Runs on `device` (expansion, radix sort and OR-merge are the S1 kernels).  Duplicate arcs
 *   merge.  Errors: VDMC_EINVAL, VDMC_ERANGE, VDMC_ESELFLOOP, VDMC_ENOMEM, VDMC_ECUDA,
 *   VDMC_ENODEV; outputs are set only on success. */
vdmc_status vdmc_symmetrize(int64_t n, const int64_t *out_indptr, const int32_t *out_nbr, int device,
                            int64_t **indptr, int32_t **nbr, uint8_t **dir);

/* Release host memory returned by the library (vdmc_symmetrize).  NULL is a no-op. */
void vdmc_free_host(void *p);

/* 5-vertex motifs ("appropriate for 5 motifs too"): vdmc_count /
 * vdmc_count_kind / vdmc_count_ex accept k = 5 and run the generic BFS-layer path (one set per
 * lane, 16-bit LUT of 2^20 masks); counts is then device uint64 [n][9364] (directed) or [n][21]
 * (undirected).  k = 5 is not available in vdmc_count_edges / vdmc_count_distributed (VDMC_EK).
 *
 * Count k-motifs (k in {3,4}) into counts: device uint64 [n][vdmc_num_classes(k)], row =
 * original vertex id, fully overwritten.  work = NULL counts everything; otherwise only the
 * motifs whose (root, depth-1 neighbour) task lies in *work.  The partials of any set of
 * disjoint slices covering [0, ntasks) sum to the full result bit-exactly (integer adds).
 * Asynchronous on `stream`; valid after the stream synchronises.  Working memory is drawn
 * per call (the graph is not modified).
 * Errors: VDMC_EK, VDMC_EINVAL (NULL, bad slice, G_U degree >= 2^21), VDMC_ENOMEM, VDMC_ECUDA. */
vdmc_status vdmc_count(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                       void *stream);

/* vdmc_count for either motif kind: counts is device uint64 [n][vdmc_num_classes_kind(k, kind)].
 * Same enumeration, slices and semantics as vdmc_count; only the class table differs.
 * Errors: as vdmc_count, plus VDMC_EINVAL for kind not in {VDMC_DIRECTED, VDMC_UNDIRECTED}. */
vdmc_status vdmc_count_kind(const vdmc_graph *g, int k, int kind, uint64_t *counts,
                            const vdmc_range *work, void *stream);

/* vdmc_count with options (NULL = all defaults, directed).  Errors: as vdmc_count_kind, plus
 * VDMC_EINVAL for an option outside its range. */
vdmc_status vdmc_count_ex(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                          const vdmc_count_options *opt, void *stream);

/* Edge-level counts, the Discussion's extension: "counting motifs for
 * edges, rather than vertices ... only requires updating edges and not vertices once a motif
 * was counted".
 *   counts[e][j] = number of connected k-sets S containing both ends of the G_U edge e whose
 *                  class is vdmc_class_ids_kind(k, kind)[j]  (every G_U edge inside S: +1)
 * counts: device uint64 [ntasks][C] (one row per G_U edge; ntasks = edges), rows in the
 * canonical edge order: (u, v) with u < v ORIGINAL ids, lexicographic (vdmc_get_edges lists
 * them).  work / opt / stream as vdmc_count_ex (only opt->kind and opt->timings_ms are used: the
 * edge path enumerates every set explicitly).  Partials of disjoint task slices sum to the full
 * result.  Errors: as vdmc_count_ex, plus VDMC_EINVAL for >= 2^31 edges. */
vdmc_status vdmc_count_edges(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                             const vdmc_count_options *opt, void *stream);

/* The G_U edge of each row of vdmc_count_edges: u[e] < v[e], original ids, lexicographic
 * (host int32 [ntasks] each; synchronous).  Errors: VDMC_EINVAL, VDMC_ECUDA. */
vdmc_status vdmc_get_edges(const vdmc_graph *g, int32_t *u, int32_t *v);

/* Cost-balanced split of the task list into nparts contiguous slices:
 * parts[p] for p in [0, nparts).  Uses a per-task cost proxy of the kernels' work computed on
 * the device (synchronous; nothing is cached in the graph).
 * Errors: VDMC_EK, VDMC_EINVAL (nparts < 1 or parts NULL), VDMC_ECUDA. */
vdmc_status vdmc_plan(const vdmc_graph *g, int k, int nparts, vdmc_range *parts);

/* Host-only helper used by vdmc_plan: given inclusive prefix sums of per-task costs
 * (host int64 [ntasks], nondecreasing), slice p = [first task whose prefix exceeds
 * p*total/nparts, ...).  Slices are contiguous, disjoint and cover [0, ntasks). */
vdmc_status vdmc_split_costs(const int64_t *prefix, int64_t ntasks, int nparts, vdmc_range *parts);

/* The tasks of the roots at order positions [pos_lo, pos_hi) (position = rank, see
 * vdmc_get_order): a root-range work slice (north star: "partitioned by root-vertex ranges").
 * Errors: VDMC_EINVAL (NULL, 0 <= pos_lo <= pos_hi <= n violated), VDMC_ECUDA. */
vdmc_status vdmc_root_range(const vdmc_graph *g, int64_t pos_lo, int64_t pos_hi, vdmc_range *out);

/* 13 for k = 3, 199 for k = 4, 9364 for k = 5, -1 otherwise. */
int vdmc_num_classes(int k);

/* ids[j] = canonical (minimum) paper index of column j, ascending (reading G9).
 * ids: host uint16 [vdmc_num_classes(k)].  Errors: VDMC_EK, VDMC_EINVAL. */
vdmc_status vdmc_class_ids(int k, uint16_t *ids);

/* Class count / column ids for a motif kind: 13 / 199 (directed), 2 / 6 (undirected); -1 (or
 * VDMC_EK / VDMC_EINVAL) for a bad k or kind. */
int vdmc_num_classes_kind(int k, int kind);
vdmc_status vdmc_class_ids_kind(int k, int kind, uint16_t *ids);

/* Column ids for k in {3, 4, 5} (k = 5 indices need 20 bits): ids host uint32 [num_classes].
 * k = 5: 9364 directed classes (OEIS A003085), 21 undirected (A001349).  The first call for
 * k = 5 builds the 2^20-entry table on the host cores (about a second).
 * Errors: VDMC_EK, VDMC_EINVAL. */
vdmc_status vdmc_class_ids32(int k, int kind, uint32_t *ids);

/* Graph facts (host struct). */
vdmc_status vdmc_get_info(const vdmc_graph *g, vdmc_graph_info *info);

/* The vertex order used: order[i] = original id of the vertex at position i (host int32 [n]). */
vdmc_status vdmc_get_order(const vdmc_graph *g, int32_t *order);

/* Number of kernels this library has launched in this process (all graphs, all devices). */
int64_t vdmc_kernel_launches(void);

/* ------------------------------------------------------------------ multi-GPU
 * The paper proposes "sending chunks of vertices in the root of the BFS to different GPUs"
 * (P:312).  One process per GPU; each holds the whole graph (replicated), counts its
 * cost-balanced task slice (vdmc_plan) into a private partial, and one NCCL reduce (sum of
 * uint64) over NVLink gives the root rank the full matrix.  Integer addition is associative,
 * so the result is bit-identical for every number of GPUs.  The communicator is NCCL's own;
 * the caller only moves the 128-byte unique id from rank 0 to the others (e.g. with
 * torch.distributed.broadcast_object_list). */
typedef struct vdmc_comm vdmc_comm;

/* A fresh NCCL unique id (128 bytes, host).  Call on one rank only.  Errors: VDMC_ENCCL. */
vdmc_status vdmc_comm_unique_id(uint8_t id[128]);

/* Join the communicator of `nranks` ranks as `rank`, using `device`.  Collective: every rank
 * calls it with the same id.  Errors: VDMC_EINVAL, VDMC_ENODEV, VDMC_ENCCL. */
vdmc_status vdmc_comm_init(int nranks, int rank, const uint8_t id[128], int device, vdmc_comm **out);

/* Destroy the communicator (NULL is a no-op). */
void vdmc_comm_free(vdmc_comm *c);

/* Collective count: every rank of `comm` calls it with a graph built from the same input and
 * the same k / options.  Rank p counts slice p of vdmc_plan(g, k, nranks) into a private
 * class-major partial; ncclReduce (sum, uint64) of the partials to `root`; root writes the full
 * matrix into counts (device uint64 [n][C], rows = original ids).  counts is ignored on the
 * other ranks (may be NULL).  Asynchronous on `stream` after the (synchronous) plan.
 * Errors: as vdmc_count_ex, plus VDMC_EINVAL (root outside [0, nranks)), VDMC_ENCCL. */
vdmc_status vdmc_count_distributed(const vdmc_graph *g, int k, const vdmc_count_options *opt,
                                   vdmc_comm *comm, int root, uint64_t *counts, void *stream);

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
