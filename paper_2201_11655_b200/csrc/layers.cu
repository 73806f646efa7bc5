// layers.cu -- k-vertex motifs for any k <= 5 by proper BFS layering:
// "Claims and data structure are appropriate for 5 motifs too".
//
// The method generalised from its k = 3 / 4 shapes (Lemma 2; Lemmas 3-4):
// a connected set S with minimum r (Lemma 1) has unique BFS layers D_1, D_2, ... in
// G_U[S] from r; listing S as r, then D_1 by rank, then D_2 by rank, ... gives one sequence
// v_0 = r, v_1, ..., v_{k-1} per set.  A sequence is grown one vertex at a time; if the last
// vertex lies in layer L, the next vertex u (rank > r, u not in S) is either
//   (same layer L)  adjacent to a vertex of layer L-1, to none of layers < L-1, rank(u) > rank(last)
//   (layer L + 1)   adjacent to a vertex of layer L, to none of layers <= L-1
// -- exactly the Lemma 3 rules (no tree edge to a lower or equal depth, same-depth vertices in
// index order) with depths taken inside S (reading G4).  Every connected k-set with minimum r is
// produced once: its own sorted sequence is valid prefix by prefix, and no other sequence has its
// vertex set (the layers of a set are unique).  A candidate reachable from several sources of
// the same layer is taken from the first one only (the "2+1" de-duplication, reading G5).
// Task = (r, v_1 = a): the paper's (vertex, neighbour) unit; a is the lowest-rank vertex
// of D_1.  One warp per task; internal levels walk candidates one at a time (warp-uniform), the
// last level puts one candidate (one set) per lane.  Codes of every pair come from binary searches
// in the sorted G_U lists; the 2k(k-1)/2-bit mask (pair-code-major, as the k = 3 / 4 path) goes
// through a 16-bit class LUT (2^20 entries for k = 5, L2-resident).  Counts: row-major u64
// accumulator [rank][C] (C = 9364 for k = 5: 75 KB per row), lanes with equal classes merged for
// the members shared by the warp.
#include <algorithm>

#include "vdmc_internal.cuh"

namespace vdmc {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kLWarps = 8;
constexpr int kLBlock = kLWarps * 32;
constexpr uint32_t kNoCol = 0xffffu;

struct LDev {
    const int64_t *__restrict__ off;
    const int64_t *__restrict__ split;
    const uint32_t *__restrict__ adj;
    const int64_t *__restrict__ tfirst;
    const int32_t *__restrict__ task_root;
    const uint16_t *__restrict__ lut;       // mask -> column, kNoCol = disconnected
    unsigned long long *__restrict__ acc;   // row-major [rank][C]
    uint32_t C;
    uint32_t *__restrict__ scr;             // per-warp candidate lists of the internal levels
    int64_t per_level;                      // words per level per warp (4 * maxdeg)
};

// code(x, y) with x first (bit0 = x -> y, bit1 = y -> x), 0 if not adjacent: y in x's list
__device__ __forceinline__ uint32_t code_of(const LDev &g, uint32_t x, uint32_t y) {
    int64_t lo = g.off[x], hi = g.off[x + 1];
    const int64_t end = hi;
    const uint32_t key = y << 2;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (g.adj[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < end && (g.adj[lo] >> 2) == y) ? (g.adj[lo] & 3u) : 0u;
}

__device__ __forceinline__ bool adjacent(const LDev &g, uint32_t x, uint32_t y) { return code_of(g, x, y) != 0u; }

// pair index of (i, j), i < j < K, lexicographic: the device mask keeps pair p in bits 2p, 2p+1
template <int K>
__device__ __forceinline__ int pair_index(int i, int j) {
    return i * (2 * K - i - 1) / 2 + (j - i - 1);
}

struct Prefix {          // warp-uniform
    uint32_t v[5];       // v[0] = r
    int layer[5];
    uint32_t mask;       // pair codes among v[0..m)
};

// Is u (rank > r) a valid next vertex after the prefix v[0..m)?  Returns its layer (0 = no).
// src = index of the prefix vertex whose list u came from; the caller walks, for the same layer,
// the lists of layer L-1 vertices (same-layer option) and of layer L vertices (next-layer option).
__device__ __forceinline__ int accept(const LDev &g, const Prefix &P, int m, uint32_t u, int src) {
    const int L = P.layer[m - 1];
    const int ls = P.layer[src];
    int cand;
    if (ls == L - 1) cand = L;            // same layer as the last vertex
    else if (ls == L) cand = L + 1;       // opens the next layer
    else return 0;
    if (cand == L && u <= P.v[m - 1]) return 0;   // same-layer vertices in rank order
    for (int j = 0; j < m; j++)
        if (P.v[j] == u) return 0;
    for (int j = 0; j < m; j++) {
        const int lj = P.layer[j];
        if (lj < cand - 1 || (lj == cand - 1 && j < src)) {   // lower layers; earlier sources
            if (adjacent(g, P.v[j], u)) return 0;
        }
    }
    return cand;
}

// the mask bits of u joining the prefix as vertex m
template <int K>
__device__ __forceinline__ uint32_t join_mask(const LDev &g, const Prefix &P, int m, uint32_t u) {
    uint32_t mk = 0;
    for (int j = 0; j < m; j++) mk |= code_of(g, P.v[j], u) << (2 * pair_index<K>(j, m));
    return mk;
}

// Walk the candidate sources of the prefix v[0..m): the lists of the layer L-1 and layer L
// vertices, 32 entries per step; f(u, layer, lane-valid) is called warp-uniformly per step.
template <typename F>
__device__ __forceinline__ void walk(const LDev &g, const Prefix &P, int m, int lane, F &&f) {
    const int L = P.layer[m - 1];
    const uint32_t r = P.v[0];
    for (int src = 0; src < m; src++) {
        const int ls = P.layer[src];
        if (ls != L - 1 && ls != L) continue;
        const uint32_t x = P.v[src];
        // layer-0 source (r): only its forward list (rank > r)
        const int64_t b0 = src == 0 ? g.split[x] : g.off[x], b1 = g.off[x + 1];
        for (int64_t base = b0; base < b1; base += 32) {
            const int64_t p = base + lane;
            uint32_t u = 0;
            int lay = 0;
            if (p < b1) {
                u = g.adj[p] >> 2;
                if (u > r) lay = accept(g, P, m, u, src);
            }
            f(u, lay);
        }
    }
}

template <int K>
__device__ void leaf(const LDev &g, Prefix &P, int lane) {
    constexpr int m = K - 1;
    walk(g, P, m, lane, [&](uint32_t u, int lay) {
        uint32_t col = kNoCol;
        if (lay) col = g.lut[P.mask | join_mask<K>(g, P, m, u)];
        if (col != kNoCol) atomicAdd(g.acc + (size_t)u * g.C + col, 1ull);
        const unsigned mm = __match_any_sync(kFull, col);
        if (col != kNoCol && lane == __ffs(mm) - 1) {
            const unsigned long long c = __popc(mm);
            for (int j = 0; j < m; j++) atomicAdd(g.acc + (size_t)P.v[j] * g.C + col, c);
        }
    });
}

// internal level m: collect the candidates into the warp's list, then extend by each in turn
template <int K, int M>
__device__ void level(const LDev &g, Prefix &P, uint32_t *lists, int lane) {
    if constexpr (M == K - 1) {
        leaf<K>(g, P, lane);
    } else {
        uint32_t *cand = lists + (M - 2) * g.per_level;
        int nc = 0;
        walk(g, P, M, lane, [&](uint32_t u, int lay) {
            const unsigned bal = __ballot_sync(kFull, lay != 0);
            if (lay) cand[nc + __popc(bal & ((1u << lane) - 1u))] = u << 3 | (uint32_t)lay;
            nc += __popc(bal);
        });
        __syncwarp();
        const uint32_t saved = P.mask;
        for (int q = 0; q < nc; q++) {
            const uint32_t e = cand[q];
            const uint32_t u = e >> 3;
            P.v[M] = u;
            P.layer[M] = (int)(e & 7u);
            P.mask = saved | join_mask<K>(g, P, M, u);
            level<K, M + 1>(g, P, lists, lane);
        }
        P.mask = saved;
        __syncwarp();
    }
}

template <int K>
__global__ void __launch_bounds__(kLBlock) k_layers(LDev g, int64_t lo, int64_t hi, unsigned long long *ctr) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *lists = g.scr + ((int64_t)blockIdx.x * kLWarps + wid) * (K > 3 ? (K - 3) : 1) * g.per_level;
    for (;;) {
        unsigned long long x = 0;
        if (lane == 0) x = atomicAdd(ctr, 1ull);
        const int64_t t = lo + (int64_t)__shfl_sync(kFull, x, 0);
        if (t >= hi) break;
        const uint32_t r = (uint32_t)g.task_root[t];
        const uint32_t ea = g.adj[g.split[r] + (t - g.tfirst[r])];
        Prefix P;
        P.v[0] = r;
        P.layer[0] = 0;
        P.v[1] = ea >> 2;
        P.layer[1] = 1;
        P.mask = ea & 3u;   // pair (0, 1)
        level<K, 2>(g, P, lists, lane);
    }
}

__global__ void k_rows_out(int64_t n, uint32_t C, const int32_t *__restrict__ order,
                           const unsigned long long *__restrict__ acc, unsigned long long *__restrict__ out) {
    for (int64_t v = blockIdx.x; v < n; v += gridDim.x) {
        const unsigned long long *src = acc + (size_t)v * C;
        unsigned long long *dst = out + (size_t)order[v] * C;
        for (uint32_t j = threadIdx.x; j < C; j += blockDim.x) dst[j] = src[j];
    }
}

}  // namespace

vdmc_status count_layers_impl(const vdmc_graph *g, int k, int kind, uint64_t *counts, int64_t lo, int64_t hi,
                              cudaStream_t s, float *ms) {
    const int C = num_classes(k, kind);
    const uint16_t *lut = nullptr;
    vdmc_status st = device_lut16(g->device, k, kind, &lut);
    if (st) return st;
    cudaEvent_t ev[3] = {};
    if (ms) {
        for (auto &e : ev) VDMC_CUDA(cudaEventCreate(&e));
        VDMC_CUDA(cudaEventRecord(ev[0], s));
    }
    int nsm = 0;
    VDMC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    int per_sm = 0;
    auto kern = k == 3 ? k_layers<3> : (k == 4 ? k_layers<4> : k_layers<5>);
    VDMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kLBlock, 0));
    const int grid = std::max(1, nsm * std::max(per_sm, 1));
    const int64_t per_level = 4 * std::max<int64_t>(g->max_degree, 1) + 32;
    const int levels = k > 3 ? k - 3 : 1;
    const size_t accn = (size_t)std::max<int64_t>(g->n, 1) * C;
    unsigned long long *acc = nullptr, *ctr = nullptr;
    uint32_t *scr = nullptr;
    VDMC_CUDA(dalloc((void **)&acc, accn * 8, s));
    VDMC_CUDA(dalloc((void **)&ctr, 8, s));
    VDMC_CUDA(dalloc((void **)&scr, (size_t)grid * kLWarps * levels * per_level * 4, s));
    VDMC_CUDA(cudaMemsetAsync(acc, 0, accn * 8, s));
    VDMC_CUDA(cudaMemsetAsync(ctr, 0, 8, s));
    LDev d{};
    d.off = g->off;
    d.split = g->split;
    d.adj = g->adj;
    d.tfirst = g->tfirst;
    d.task_root = g->task_root;
    d.lut = lut;
    d.acc = acc;
    d.C = (uint32_t)C;
    d.scr = scr;
    d.per_level = per_level;
    if (hi > lo) {
        kern<<<grid, kLBlock, 0, s>>>(d, lo, hi, ctr);
        VDMC_LAUNCH();
    }
    if (ms) VDMC_CUDA(cudaEventRecord(ev[1], s));
    if (g->n > 0) {
        k_rows_out<<<(unsigned)std::min<int64_t>(g->n, (int64_t)nsm * 16), 256, 0, s>>>(
            g->n, (uint32_t)C, g->order, acc, (unsigned long long *)counts);
        VDMC_LAUNCH();
    }
    dfree(acc, s);
    dfree(ctr, s);
    dfree(scr, s);
    if (ms) {
        VDMC_CUDA(cudaEventRecord(ev[2], s));
        VDMC_CUDA(cudaEventSynchronize(ev[2]));
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        ms[0] = 0;
        ms[1] = a;
        ms[2] = b;
        ms[3] = a + b;
        for (auto &e : ev) cudaEventDestroy(e);
    }
    return VDMC_OK;
}

}  // namespace vdmc
