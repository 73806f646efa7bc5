// vdmc_internal.cuh -- shared declarations of libvdmc.so (product path; no oracle code here).
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

#include "../../include/vdmc.h"

namespace vdmc {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
vdmc_status fail(vdmc_status st, const char *fmt, ...);
void count_launch(int n = 1);
// Device memory (api.cu): small buffers from the device's default stream-ordered pool; large
// ones from a process-wide cache of blocks that are reused best-fit across calls and graphs
// (no page mapping or pool fragmentation in a step).  Stream-ordered: dfree(p, s) makes the
// block reusable after the work queued on s; a reuse on another stream waits for it.
cudaError_t dalloc(void **p, size_t bytes, cudaStream_t s);
void dfree(void *p, cudaStream_t s);
void trim_cache(int dev);   // release the idle cached blocks of a device
// Host-side trace (VDMC_TRACE=1): prints the host milliseconds since the previous point.
void trace(const char *what);

#define VDMC_CUDA(call)                                                                  \
    do {                                                                                 \
        cudaError_t err_ = (call);                                                       \
        if (err_ != cudaSuccess)                                                         \
            return ::vdmc::fail(err_ == cudaErrorMemoryAllocation ? VDMC_ENOMEM : VDMC_ECUDA, \
                                "%s:%d %s: %s", __FILE__, __LINE__, #call,               \
                                cudaGetErrorString(err_));                               \
    } while (0)

#define VDMC_LAUNCH()                                                                    \
    do {                                                                                 \
        ::vdmc::count_launch();                                                          \
        cudaError_t err_ = cudaGetLastError();                                           \
        if (err_ != cudaSuccess)                                                         \
            return ::vdmc::fail(VDMC_ECUDA, "%s:%d launch: %s", __FILE__, __LINE__,      \
                                cudaGetErrorString(err_));                               \
    } while (0)

// --------------------------------------------------------- motif classes
// Device mask layout ("pair-code-major", any bijection of the paper's index is allowed,
// SURVEY §8(a) S3): vertices in enumeration order (r, a, b, c); pair p of (0,1),(0,2),(0,3),
// (1,2),(1,3),(2,3) [k=4] or (0,1),(0,2),(1,2) [k=3] occupies bits 2p..2p+1 with
//   bit 2p   = first -> second,   bit 2p+1 = second -> first.
// The host LUT maps every such mask to the column of its minimum-isomorph paper index.
// kind 0 = directed motifs, 1 = undirected motifs (classes of the G_U-induced subgraph)
constexpr int kNumClasses3 = 13;
constexpr int kNumClasses4 = 199;
constexpr int kNumClassesU3 = 2;
constexpr int kNumClassesU4 = 6;
constexpr uint8_t kNoClass = 255;

const uint8_t *host_lut(int k, int kind);          // [64] or [4096]
const uint32_t *host_class_ids32(int k, int kind); // k in {3, 4, 5}
const uint16_t *host_class_ids(int k, int kind);   // [13] / [199], undirected [2] / [6]
int num_classes(int k, int kind);

}  // namespace vdmc

// ------------------------------------------------------------ graph handle
// Immutable once vdmc_build_graph* returns: count calls read it and draw their working memory
// (accumulator, work counters, scratch) per call.
struct vdmc_graph {
    int device = 0;
    int64_t n = 0, nnz = 0, arcs = 0, ntasks = 0, max_degree = 0;
    // G_U in rank order.  adj entry = (rank(nbr) << 2) | code, code bit0 = owner -> nbr,
    // bit1 = nbr -> owner; every list sorted ascending (= by rank).
    int64_t *off = nullptr;        // [n+1]
    int64_t *split = nullptr;      // [n]   first entry of v's list with rank > v
    uint32_t *adj = nullptr;       // [nnz]
    int32_t *order = nullptr;      // [n]   order[rank] = original id
    int64_t *tfirst = nullptr;     // [n+1] first task of each root (exclusive scan of forward degrees)
    int32_t *task_root = nullptr;  // [ntasks]
    uint8_t *lut[2][2] = {};       // [kind][k == 4] device class LUTs (S3)
    // S4 schedule: tasks of heavy roots (CTA per task) and light roots (warp per root), both
    // ascending (= rank order, longest first), so a task slice maps to a contiguous sub-list
    int32_t *heavy_task = nullptr; // [nheavy]
    int32_t *light_root = nullptr; // [nlight] light items: root, and the item's first task offset in
    int32_t *light_i0 = nullptr;   // [nlight] the root (a root of D tasks is cut into items of <= 8 tasks)
    int64_t nheavy = 0, nlight = 0;
    // induced adjacency of N+(r) in position space for heavy roots r (S4 pre-pass):
    // entries of the position p of root r: nr_adj[nr_off[hbase[r] + p] .. nr_off[hbase[r] + p + 1])
    int32_t *hroots = nullptr;     // [nhroots] heavy roots, rank order
    int64_t nhroots = 0;
    int64_t hub_tasks = 0;         // heavy tasks of the leading roots of degree > kHubDeg (enum.cu)
    int64_t *hbase = nullptr;      // [n] segment base per heavy root
    int64_t *nr_off = nullptr;     // [sum D+ over heavy roots + 1]
    uint32_t *nr_adj = nullptr;    // position << 2 | code(x, R[position])
    int64_t nr_total = 0;
    float build_ms = 0;
};

namespace vdmc {
struct CountOpts {   // validated vdmc_count_options
    int kind = 0, star_block = 0, cross_block = 0, heavy_global = 0, force_big = 0, layered = 0;
    int acc64 = 0;   // 1 = force the 64-bit accumulator even when 32 bits provably suffice
    int64_t ca_capacity = 0;
    float *timings_ms = nullptr;
};
vdmc_status build_device(int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst,
                         const int32_t *h_rank, int device, cudaStream_t stream, vdmc_graph *g);
// S4 schedule + class LUT upload, run at the end of a build
vdmc_status build_schedule(vdmc_graph *g, cudaStream_t s);
// per-task cost proxy, inclusive prefix (host [ntasks])
vdmc_status plan_prefix(const vdmc_graph *g, int k, int64_t *prefix_host, cudaStream_t s);
// count the slice [lo, hi) into the class-major accumulator acc [C][n] (caller-allocated
// device memory, rank order); no finalise
vdmc_status count_into(const vdmc_graph *g, int k, const CountOpts &o, unsigned long long *acc, int64_t lo,
                       int64_t hi, cudaStream_t s, float *ms3);
// class-major rank-order accumulator -> row-major [original id][C]
vdmc_status finalize(const vdmc_graph *g, int C, const unsigned long long *acc, uint64_t *counts, cudaStream_t s);
// the same with a 32-bit accumulator (enum32.cu), used when every count provably fits 32 bits
vdmc_status count_into32(const vdmc_graph *g, int k, const CountOpts &o, unsigned int *acc, int64_t lo, int64_t hi,
                         cudaStream_t s, float *ms3);
vdmc_status finalize32(const vdmc_graph *g, int C, const unsigned int *acc, uint64_t *counts, cudaStream_t s);
// true if every (vertex, class) count of a k-count fits 32 bits (bound on sets through a vertex)
inline bool counts_fit_u32(const vdmc_graph *g, int k) {
    const double d = (double)g->max_degree;
    return (k == 3 ? 2.0 * d * d : 6.0 * d * d * d) < 4294967296.0;
}
// edge-level counts (edges.cu): counts [edges][C] in the canonical edge order; ms (optional,
// host float[4]) as vdmc_count_options.timings_ms
vdmc_status count_edges_impl(const vdmc_graph *g, int k, int kind, uint64_t *counts, int64_t lo, int64_t hi,
                             cudaStream_t s, float *ms);
vdmc_status edge_list_impl(const vdmc_graph *g, int32_t *u, int32_t *v);
// generic BFS-layer path for k <= 5 (layers.cu); 16-bit class LUT per (device, k, kind)
vdmc_status count_layers_impl(const vdmc_graph *g, int k, int kind, uint64_t *counts, int64_t lo, int64_t hi,
                              cudaStream_t s, float *ms);
vdmc_status device_lut16(int device, int k, int kind, const uint16_t **out);
// S1 only, for vdmc_symmetrize: G_U entries in ORIGINAL ids, sorted by (owner, nbr), OR-merged
vdmc_status symmetrize_device(int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst, cudaStream_t s,
                              int64_t *nnz_out, uint64_t **d_entries, int *vb_out);
}  // namespace vdmc
