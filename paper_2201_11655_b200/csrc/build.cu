// build.cu -- device graph build: SURVEY §8(a) S1 (ingest + symmetrise) and S2 (order,
// relabel, split), all on the GPU.
//
// S1 ("G_U ... ignoring the direction"; P:81 simple graphs; P:125-134 CSR):
//   every arc u -> v yields two G_U entries, (u, v, code 1) and (v, u, code 2), packed in a
//   64-bit key  owner << (vb + 2) | nbr << 2 | code  (vb = bits of a vertex id; the sorts read
//   only bits [2, 2 vb + 2): 6 radix passes at n = 5M).  One radix sort groups each unordered pair's
//   entries; OR-merging equal (owner, nbr) keys gives ONE entry per G_U edge with both
//   direction bits (a mutual pair is a single entry with code 3 -- reading G14).
// S2: rank = undirected degree descending, ties by ascending id (G2/G3).
//   Entries are relabelled to ranks and sorted again, so each list is ascending in rank and
//   the packed uint32 entry  rank << 2 | code  sorts exactly like the rank.  split[v] = first
//   entry with rank > v: the suffix N+(v) of "higher index" vertices (G7).
// Tasks ("each pair of a vertex and one of its neighbors"): one per forward entry,
//   numbered root-major; tfirst = exclusive scan of the forward degrees.
#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "vdmc_internal.cuh"

namespace vdmc {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(int64_t work) {
    int64_t b = (work + kThreads - 1) / kThreads;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

__global__ void k_arc_keys(int64_t m, int64_t n, int vb, const int32_t *__restrict__ src,
                           const int32_t *__restrict__ dst, uint64_t *__restrict__ keys,
                           unsigned long long *__restrict__ bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = src[e], v = dst[e];
        if (u < 0 || u >= n || v < 0 || v >= n || u == v) {
            // record the first bad arc (smallest index): 2 bits of kind + index
            unsigned long long tag = ((unsigned long long)e << 2) | (u == v ? 1ull : 2ull);
            atomicMin(bad, tag);
            u = 0;
            v = 1;
        }
        keys[2 * e] = ((uint64_t)u << (vb + 2)) | ((uint64_t)v << 2) | 1u;       // owner u, u -> v
        keys[2 * e + 1] = ((uint64_t)v << (vb + 2)) | ((uint64_t)u << 2) | 2u;   // owner v, nbr -> owner
    }
}

// head[i] = 1 if entry i starts a new (owner, nbr) pair
__global__ void k_heads(int64_t len, const uint64_t *__restrict__ keys, int32_t *__restrict__ head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || (keys[i] >> 2) != (keys[i - 1] >> 2)) ? 1 : 0;
}

// merged[pos[i]] = pair key | OR of the run's codes; deg[owner]++
__global__ void k_merge(int64_t len, int vb, const uint64_t *__restrict__ keys, const int32_t *__restrict__ head,
                        const int64_t *__restrict__ pos, uint64_t *__restrict__ merged, int32_t *__restrict__ deg,
                        unsigned long long *__restrict__ arcs) {
    unsigned long long local_arcs = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
        if (!head[i]) continue;
        uint64_t k = keys[i];
        uint64_t code = k & 3;
        for (int64_t j = i + 1; j < len && (keys[j] >> 2) == (k >> 2); j++) code |= keys[j] & 3;
        merged[pos[i]] = (k & ~3ull) | code;
        atomicAdd(&deg[k >> (vb + 2)], 1);
        local_arcs += code & 1;   // count each arc once, from its tail's entry
    }
    atomicAdd(arcs, local_arcs);
}

__global__ void k_rank_keys(int64_t n, const int32_t *__restrict__ deg, uint64_t *__restrict__ keys) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        keys[v] = ((uint64_t)(0x7fffffffu - (uint32_t)deg[v]) << 32) | (uint64_t)v;   // degree desc, id asc
}

__global__ void k_order_from_keys(int64_t n, const uint64_t *__restrict__ keys, int32_t *__restrict__ order,
                                  int32_t *__restrict__ rank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = (int32_t)(keys[i] & 0xffffffffu);
        order[i] = v;
        rank[v] = (int32_t)i;
    }
}

__global__ void k_order_from_rank(int64_t n, const int32_t *__restrict__ rank, int32_t *__restrict__ order) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        order[rank[v]] = (int32_t)v;
}

__global__ void k_relabel(int64_t nnz, int vb, const uint64_t *__restrict__ merged, const int32_t *__restrict__ rank,
                          uint64_t *__restrict__ keys, int32_t *__restrict__ deg_r) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t k = merged[i];
        const uint64_t vmask = (1ull << vb) - 1ull;
        uint64_t ro = (uint64_t)rank[k >> (vb + 2)], rn = (uint64_t)rank[(k >> 2) & vmask];
        keys[i] = (ro << (vb + 2)) | (rn << 2) | (k & 3);
        atomicAdd(&deg_r[ro], 1);
    }
}

__global__ void k_adj(int64_t nnz, int vb, const uint64_t *__restrict__ keys, uint32_t *__restrict__ adj) {
    const uint64_t mask = (1ull << (vb + 2)) - 1ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
        adj[i] = (uint32_t)(keys[i] & mask);   // rank(nbr) << 2 | code  (rank < 2^30)
}

// split[v] = first entry of v's list with rank > v;  fwd[v] = forward degree
__global__ void k_split(int64_t n, const int64_t *__restrict__ off, const uint32_t *__restrict__ adj,
                        int64_t *__restrict__ split, int64_t *__restrict__ fwd) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = off[v], hi = off[v + 1];
        const uint32_t key = (uint32_t)(v + 1) << 2;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < key) lo = mid + 1; else hi = mid;
        }
        split[v] = lo;
        fwd[v] = off[v + 1] - lo;
    }
}

// task_root[t] = r for t in [tfirst[r], tfirst[r+1]); one warp per root
__global__ void k_task_root(int64_t n, const int64_t *__restrict__ tfirst, int32_t *__restrict__ task_root) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
         r += ((int64_t)gridDim.x * blockDim.x) >> 5)
        for (int64_t t = tfirst[r] + lane; t < tfirst[r + 1]; t += 32) task_root[t] = (int32_t)r;
}

struct Tmp {   // stream-ordered temporaries, freed on scope exit
    cudaStream_t s;
    std::vector<void *> ptrs;
    explicit Tmp(cudaStream_t st) : s(st) {}
    ~Tmp() { for (void *p : ptrs) dfree(p, s); }
    template <class T> cudaError_t alloc(T **p, size_t count) {
        cudaError_t e = dalloc((void **)p, std::max<size_t>(1, count) * sizeof(T), s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
};

int bits_for(int64_t x) {   // bits needed to hold values in [0, x)
    int b = 1;
    while ((int64_t(1) << b) < x) b++;
    return b;
}

}  // namespace

// S1 on the device: arcs -> one G_U entry per (owner, nbr) pair with the OR of its direction
// codes, sorted by (owner, nbr) in ORIGINAL ids.  merged (length nnz) is one half of the
// caller's double buffer keys/keys2 [2m]; deg[owner] counts entries (G_U degree).
static vdmc_status s1_entries(int64_t n, int64_t m, int vb, const int32_t *d_src, const int32_t *d_dst,
                              cudaStream_t s, Tmp &tmp, uint64_t *keys, uint64_t *keys2, int32_t *deg,
                              uint64_t **merged_out, int64_t *nnz_out, int64_t *arcs_out) {
    const int64_t L = 2 * m;
    *merged_out = nullptr;
    *nnz_out = 0;
    *arcs_out = 0;
    if (m <= 0) return VDMC_OK;
    int32_t *head = nullptr;
    int64_t *pos = nullptr;
    unsigned long long *flags = nullptr;   // [0] first bad arc, [1] arc count
    VDMC_CUDA(tmp.alloc(&head, L));
    VDMC_CUDA(tmp.alloc(&pos, L));
    VDMC_CUDA(tmp.alloc(&flags, 2));
    VDMC_CUDA(cudaMemsetAsync(flags, 0xff, sizeof(unsigned long long), s));
    VDMC_CUDA(cudaMemsetAsync(flags + 1, 0, sizeof(unsigned long long), s));
    k_arc_keys<<<grid_for(m), kThreads, 0, s>>>(m, n, vb, d_src, d_dst, keys, flags);
    VDMC_LAUNCH();
    size_t tb = 0;
    void *tstore = nullptr;
    cub::DoubleBuffer<uint64_t> db(keys, keys2);
    VDMC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int)L, 2, 2 * vb + 2, s));
    VDMC_CUDA(tmp.alloc((char **)&tstore, tb));
    VDMC_CUDA(cub::DeviceRadixSort::SortKeys(tstore, tb, db, (int)L, 2, 2 * vb + 2, s));
    trace("sort1 enqueued");
    count_launch(2 * ((2 * vb + 7) / 8));
    uint64_t *sorted = db.Current();
    k_heads<<<grid_for(L), kThreads, 0, s>>>(L, sorted, head);
    VDMC_LAUNCH();
    size_t tb2 = 0;
    VDMC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, head, pos, (int)L, s));
    void *tstore2 = nullptr;
    VDMC_CUDA(tmp.alloc((char **)&tstore2, tb2));
    VDMC_CUDA(cub::DeviceScan::ExclusiveSum(tstore2, tb2, head, pos, (int)L, s));
    count_launch(2);
    uint64_t *merged = (sorted == keys) ? keys2 : keys;   // free half of the double buffer
    k_merge<<<grid_for(L), kThreads, 0, s>>>(L, vb, sorted, head, pos, merged, deg, flags + 1);
    VDMC_LAUNCH();
    int64_t last_pos = 0;
    int32_t last_head = 0;
    unsigned long long hf[2];
    VDMC_CUDA(cudaMemcpyAsync(&last_pos, pos + L - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaMemcpyAsync(&last_head, head + L - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaMemcpyAsync(hf, flags, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaStreamSynchronize(s));
    trace("sync after merge");
    if (hf[0] != ~0ull) {
        long long e = (long long)(hf[0] >> 2);
        if ((hf[0] & 3) == 1) return fail(VDMC_ESELFLOOP, "arc %lld is a self-loop", e);
        return fail(VDMC_ERANGE, "arc %lld has a vertex id outside [0, %lld)", e, (long long)n);
    }
    *merged_out = merged;
    *nnz_out = last_pos + last_head;
    *arcs_out = (int64_t)hf[1];
    return VDMC_OK;
}

vdmc_status symmetrize_device(int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst, cudaStream_t s,
                              int64_t *nnz_out, uint64_t **d_entries, int *vb_out) {
    Tmp tmp(s);
    const int vb = bits_for(std::max<int64_t>(n, 2));
    uint64_t *keys = nullptr, *keys2 = nullptr;
    int32_t *deg = nullptr;
    VDMC_CUDA(tmp.alloc(&keys, 2 * m));
    VDMC_CUDA(tmp.alloc(&keys2, 2 * m));
    VDMC_CUDA(tmp.alloc(&deg, n));
    VDMC_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    uint64_t *merged = nullptr;
    int64_t nnz = 0, arcs = 0;
    vdmc_status st = s1_entries(n, m, vb, d_src, d_dst, s, tmp, keys, keys2, deg, &merged, &nnz, &arcs);
    if (st) return st;
    uint64_t *out = nullptr;
    VDMC_CUDA(dalloc((void **)&out, sizeof(uint64_t) * std::max<int64_t>(nnz, 1), s));
    if (nnz) VDMC_CUDA(cudaMemcpyAsync(out, merged, sizeof(uint64_t) * nnz, cudaMemcpyDeviceToDevice, s));
    VDMC_CUDA(cudaStreamSynchronize(s));
    *nnz_out = nnz;
    *d_entries = out;
    *vb_out = vb;
    return VDMC_OK;
}

vdmc_status build_device(int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst, const int32_t *h_rank,
                         int device, cudaStream_t s, vdmc_graph *g) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    VDMC_CUDA(cudaEventCreate(&e0));
    VDMC_CUDA(cudaEventCreate(&e1));
    VDMC_CUDA(cudaEventRecord(e0, s));
    trace("build start");
    g->n = n;
    Tmp tmp(s);
    const int vb = bits_for(std::max<int64_t>(n, 2));
    const int64_t L = 2 * m;
    uint64_t *keys = nullptr, *keys2 = nullptr, *merged = nullptr;
    int32_t *deg = nullptr, *rank = nullptr, *deg_r = nullptr;
    int64_t *fwd = nullptr;
    VDMC_CUDA(tmp.alloc(&keys, L));
    VDMC_CUDA(tmp.alloc(&keys2, L));
    VDMC_CUDA(tmp.alloc(&deg, n));
    VDMC_CUDA(tmp.alloc(&deg_r, n));
    VDMC_CUDA(tmp.alloc(&rank, n));
    VDMC_CUDA(tmp.alloc(&fwd, n));
    VDMC_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    VDMC_CUDA(cudaMemsetAsync(deg_r, 0, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    trace("build allocs+memsets");

    // ---- S1: entries, sort, OR-merge
    {
        vdmc_status st = s1_entries(n, m, vb, d_src, d_dst, s, tmp, keys, keys2, deg, &merged, &g->nnz, &g->arcs);
        if (st) return st;
    }
    const int64_t nnz = g->nnz;

    // ---- S2: order
    VDMC_CUDA(dalloc((void **)&g->order, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    if (n > 0) {
        if (h_rank) {
            VDMC_CUDA(cudaMemcpyAsync(rank, h_rank, sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
            k_order_from_rank<<<grid_for(n), kThreads, 0, s>>>(n, rank, g->order);
            VDMC_LAUNCH();
        } else {
            uint64_t *rk = nullptr, *rk2 = nullptr;
            VDMC_CUDA(tmp.alloc(&rk, n));
            VDMC_CUDA(tmp.alloc(&rk2, n));
            k_rank_keys<<<grid_for(n), kThreads, 0, s>>>(n, deg, rk);
            VDMC_LAUNCH();
            cub::DoubleBuffer<uint64_t> db(rk, rk2);
            size_t tb = 0;
            VDMC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int)n, 0, 64, s));
            void *ts = nullptr;
            VDMC_CUDA(tmp.alloc((char **)&ts, tb));
            VDMC_CUDA(cub::DeviceRadixSort::SortKeys(ts, tb, db, (int)n, 0, 64, s));
            count_launch(16);
            k_order_from_keys<<<grid_for(n), kThreads, 0, s>>>(n, db.Current(), g->order, rank);
            VDMC_LAUNCH();
        }
    }

    trace("order");
    // ---- S2: relabel + sort + CSR
    VDMC_CUDA(dalloc((void **)&g->off, sizeof(int64_t) * (n + 1), s));
    VDMC_CUDA(dalloc((void **)&g->split, sizeof(int64_t) * std::max<int64_t>(n, 1), s));
    VDMC_CUDA(dalloc((void **)&g->adj, sizeof(uint32_t) * std::max<int64_t>(nnz, 1), s));
    VDMC_CUDA(dalloc((void **)&g->tfirst, sizeof(int64_t) * (n + 1), s));
    VDMC_CUDA(cudaMemsetAsync(g->off, 0, sizeof(int64_t) * (n + 1), s));
    VDMC_CUDA(cudaMemsetAsync(g->tfirst, 0, sizeof(int64_t) * (n + 1), s));
    if (nnz > 0) {
        uint64_t *rl = (merged == keys) ? keys2 : keys;
        k_relabel<<<grid_for(nnz), kThreads, 0, s>>>(nnz, vb, merged, rank, rl, deg_r);
        VDMC_LAUNCH();
        cub::DoubleBuffer<uint64_t> db(rl, merged);
        size_t tb = 0;
        VDMC_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int)nnz, 2, 2 * vb + 2, s));
        void *ts = nullptr;
        VDMC_CUDA(tmp.alloc((char **)&ts, tb));
        VDMC_CUDA(cub::DeviceRadixSort::SortKeys(ts, tb, db, (int)nnz, 2, 2 * vb + 2, s));
        count_launch(2 * ((2 * vb + 7) / 8));
        k_adj<<<grid_for(nnz), kThreads, 0, s>>>(nnz, vb, db.Current(), g->adj);
        trace("sort2 enqueued");
        VDMC_LAUNCH();
    }
    if (n > 0) {
        size_t tb = 0;
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, deg_r, g->off + 1, (int)n, s));
        void *ts = nullptr;
        VDMC_CUDA(tmp.alloc((char **)&ts, tb));
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(ts, tb, deg_r, g->off + 1, (int)n, s));
        count_launch(2);
        k_split<<<grid_for(n), kThreads, 0, s>>>(n, g->off, g->adj, g->split, fwd);
        VDMC_LAUNCH();
        size_t tbf = 0;
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tbf, fwd, g->tfirst + 1, (int)n, s));
        void *tsf = nullptr;
        VDMC_CUDA(tmp.alloc((char **)&tsf, tbf));
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(tsf, tbf, fwd, g->tfirst + 1, (int)n, s));
        count_launch(2);
        // max degree
        int32_t *dmax = nullptr;
        VDMC_CUDA(tmp.alloc(&dmax, 1));
        size_t tb3 = 0;
        VDMC_CUDA(cub::DeviceReduce::Max(nullptr, tb3, deg_r, dmax, (int)n, s));
        void *ts3 = nullptr;
        VDMC_CUDA(tmp.alloc((char **)&ts3, tb3));
        VDMC_CUDA(cub::DeviceReduce::Max(ts3, tb3, deg_r, dmax, (int)n, s));
        count_launch(1);
        int32_t hmax = 0;
        VDMC_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        VDMC_CUDA(cudaStreamSynchronize(s));
        g->max_degree = hmax;
        trace("sync max degree");
    }
    g->ntasks = nnz / 2;
    VDMC_CUDA(dalloc((void **)&g->task_root, sizeof(int32_t) * std::max<int64_t>(g->ntasks, 1), s));
    if (g->ntasks > 0) {
        k_task_root<<<grid_for(n * 32), kThreads, 0, s>>>(n, g->tfirst, g->task_root);
        VDMC_LAUNCH();
    }
    {   // S3 device LUTs + S4 schedule (heavy/light lists, induced adjacency of heavy roots)
        vdmc_status st = build_schedule(g, s);
        if (st) return st;
    }
    VDMC_CUDA(cudaEventRecord(e1, s));
    VDMC_CUDA(cudaStreamSynchronize(s));
    VDMC_CUDA(cudaEventElapsedTime(&g->build_ms, e0, e1));
    trace("build end sync");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return VDMC_OK;
}

}  // namespace vdmc
