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
const uint16_t *host_class_ids(int k, int kind);   // [13] / [199], undirected [2] / [6]
int num_classes(int k, int kind);

}  // namespace vdmc

// ------------------------------------------------------------ graph handle
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
    // scratch owned by the handle (lazily grown)
    uint64_t *acc = nullptr;       // [n][C] accumulator in rank order
    size_t acc_bytes = 0;
    uint32_t *lscratch = nullptr;  // per-warp depth-2 candidate lists
    size_t lscratch_elems = 0;
    unsigned long long *ctr = nullptr;   // work counter(s)
    uint8_t *lut[2][2] = {};        // [kind][k == 4] device class LUTs
    int64_t *cost = nullptr;       // [ntasks] inclusive prefix of the plan's cost proxy
    int cost_k = 0;
    // schedule: tasks of heavy roots (CTA per task) and light roots (warp per root), rank order
    int32_t *heavy_task = nullptr; // [nheavy]
    int32_t *light_root = nullptr; // [nlight]
    int64_t nheavy = 0, nlight = 0;
    int roots_ready = 0;
    // induced adjacency of N+(r) in position space for heavy roots r (S4 pre-pass):
    // entries of the position p of root r: nr_adj[nr_off[hbase[r] + p] .. nr_off[hbase[r] + p + 1])
    int32_t *hroots = nullptr;     // [nhroots] heavy roots, rank order
    int64_t nhroots = 0;
    int64_t *hbase = nullptr;      // [n] segment base per heavy root
    int64_t *nr_off = nullptr;     // [sum D+ over heavy roots + 1]
    uint32_t *nr_adj = nullptr;    // position << 2 | code(x, R[position])
    int64_t nr_total = 0;
    // profiling
    int profiling = 0;
    cudaEvent_t ev[8] = {};
    float last_ms[5] = {0, 0, 0, 0, 0};
    float build_ms = 0;
};

namespace vdmc {
vdmc_status build_device(int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst,
                         const int32_t *h_rank, int device, cudaStream_t stream, vdmc_graph *g);
vdmc_status ensure_acc(vdmc_graph *g, int k, int kind, cudaStream_t s);
vdmc_status ensure_plan(vdmc_graph *g, int k, cudaStream_t stream);
vdmc_status launch_count(vdmc_graph *g, int k, int kind, uint64_t *counts, int64_t lo, int64_t hi,
                         cudaStream_t stream);
}  // namespace vdmc
