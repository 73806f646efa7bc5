// api.cu -- the C ABI of libvdmc.so (declared and documented in include/vdmc.h),
// error reporting, and the motif-class lookup table.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "vdmc_internal.cuh"

namespace vdmc {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_err = msg; }

vdmc_status fail(vdmc_status st, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

void count_launch(int n) { g_launches += n; }

void trace(const char *what) {
    static const bool on = [] { const char *e = getenv("VDMC_TRACE"); return e && e[0] == '1'; }();
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[vdmc trace] %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

// Device memory.  Small buffers: stream-ordered allocations from the device's default pool
// (release threshold = max, so freed memory stays mapped).  Buffers >= kBigBytes (count
// matrices, sort keys, scratch): a process-wide cache of cudaMalloc'd blocks, reused best-fit
// across calls and graphs, so a step never pays page mapping for GB-sized buffers and the pool
// never fragments them.  A cached block remembers the stream it was freed on and an event
// recorded there; a reuse on another stream waits for that event (stream-ordered semantics).
namespace {
constexpr size_t kBigBytes = size_t(4) << 20;
constexpr size_t kGrain = size_t(2) << 20;
struct Block {
    void *p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    cudaStream_t last = nullptr;
    cudaEvent_t ready = nullptr;
};
std::mutex g_mem_mu;
std::vector<Block> g_free;                  // cached, idle
std::unordered_map<void *, Block> g_live;   // handed out
bool g_pool_configured[64] = {};
}  // namespace

static cudaError_t configure_pool(int dev) {
    if (dev >= 64 || g_pool_configured[dev]) return cudaSuccess;
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, dev);
    if (e != cudaSuccess) return e;
    uint64_t thr = ~0ull;
    if ((e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess) return e;
    g_pool_configured[dev] = true;
    return cudaSuccess;
}

// free every idle cached block of `dev` (caller holds g_mem_mu)
static void trim_locked(int dev) {
    for (size_t i = 0; i < g_free.size();) {
        if (g_free[i].dev == dev) {
            cudaEventSynchronize(g_free[i].ready);
            cudaFree(g_free[i].p);
            cudaEventDestroy(g_free[i].ready);
            g_free[i] = g_free.back();
            g_free.pop_back();
        } else {
            i++;
        }
    }
}

cudaError_t dalloc(void **p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    if ((e = configure_pool(dev)) != cudaSuccess) return e;
    if (bytes < kBigBytes) return cudaMallocAsync(p, bytes ? bytes : 1, s);
    const size_t need = (bytes + kGrain - 1) / kGrain * kGrain;
    int best = -1;
    for (size_t i = 0; i < g_free.size(); i++) {   // best fit within 25% + one grain
        const Block &b = g_free[i];
        if (b.dev == dev && b.bytes >= need && b.bytes <= need + need / 4 + kGrain &&
            (best < 0 || b.bytes < g_free[best].bytes))
            best = (int)i;
    }
    Block b;
    if (best >= 0) {
        b = g_free[best];
        g_free[best] = g_free.back();
        g_free.pop_back();
        if (b.last != s && (e = cudaStreamWaitEvent(s, b.ready, 0)) != cudaSuccess) return e;
    } else {
        e = cudaMalloc(&b.p, need);
        if (e == cudaErrorMemoryAllocation) {   // give the idle cache back and retry once
            cudaGetLastError();
            trim_locked(dev);
            e = cudaMalloc(&b.p, need);
        }
        if (e != cudaSuccess) return e;
        if ((e = cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming)) != cudaSuccess) {
            cudaFree(b.p);
            return e;
        }
        b.bytes = need;
        b.dev = dev;
    }
    g_live[b.p] = b;
    *p = b.p;
    return cudaSuccess;
}

void dfree(void *p, cudaStream_t s) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_mem_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) {
        cudaFreeAsync(p, s);
        return;
    }
    Block b = it->second;
    g_live.erase(it);
    b.last = s;
    cudaEventRecord(b.ready, s);
    g_free.push_back(b);
}

void trim_cache(int dev) {
    std::lock_guard<std::mutex> lk(g_mem_mu);
    trim_locked(dev);
}

// ------------------------------------------------------------ class table
// Paper index (Fig. 1): the adjacency matrix read row by row without the
// diagonal; the first entry is the most significant bit.  Class = minimum index over all
// k! relabellings.  Connectivity is that of the underlying undirected graph
// (P:77).  Built once per process, for every device mask (layout in vdmc_internal.cuh).
struct ClassTable {
    int k = 0;
    std::vector<uint8_t> lut;        // device mask -> column
    std::vector<uint16_t> ids;       // column -> canonical paper index
};

static int paper_index(int k, const int adj[4][4], const int *perm) {
    // row-major over (i, j), i != j, vertex i of the new order is old vertex perm[i]
    int idx = 0;
    for (int i = 0; i < k; i++)
        for (int j = 0; j < k; j++)
            if (i != j) idx = (idx << 1) | adj[perm[i]][perm[j]];
    return idx;
}

// kind 1 (undirected motifs, "count undirected sub-graph in the undirected graph induced
// by ignoring the direction"; reading G17): a set's class is that of its G_U-induced subgraph,
// i.e. every pair with an arc in either direction is an edge both ways; its index is the
// paper's index of that symmetric adjacency matrix.
static void build_table(int k, int kind, ClassTable &t) {
    static const int P3[3][2] = {{0, 1}, {0, 2}, {1, 2}};
    static const int P4[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    const int npairs = k == 3 ? 3 : 6;
    const int(*pairs)[2] = k == 3 ? P3 : P4;
    const int nmask = 1 << (2 * npairs);
    std::vector<int> canon(nmask);
    std::vector<char> conn(nmask);
    for (int m = 0; m < nmask; m++) {
        int adj[4][4] = {};
        int und[4][4] = {};
        for (int p = 0; p < npairs; p++) {
            int c = (m >> (2 * p)) & 3, x = pairs[p][0], y = pairs[p][1];
            if (kind == 1 && c) c = 3;
            if (c & 1) adj[x][y] = 1;
            if (c & 2) adj[y][x] = 1;
            if (c) und[x][y] = und[y][x] = 1;
        }
        // connectivity by a flood fill from vertex 0
        int seen = 1, grown = 1;
        while (grown) {
            grown = 0;
            for (int x = 0; x < k; x++)
                if (seen >> x & 1)
                    for (int y = 0; y < k; y++)
                        if (und[x][y] && !(seen >> y & 1)) seen |= 1 << y, grown = 1;
        }
        conn[m] = seen == (1 << k) - 1;
        int perm[4] = {0, 1, 2, 3};
        int best = 1 << 30;
        do best = std::min(best, paper_index(k, adj, perm));
        while (std::next_permutation(perm, perm + k));
        canon[m] = best;
    }
    std::vector<int> ids;
    for (int m = 0; m < nmask; m++)
        if (conn[m]) ids.push_back(canon[m]);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    t.k = k;
    t.ids.assign(ids.begin(), ids.end());
    t.lut.assign(nmask, kNoClass);
    for (int m = 0; m < nmask; m++)
        if (conn[m])
            t.lut[m] = (uint8_t)(std::lower_bound(ids.begin(), ids.end(), canon[m]) - ids.begin());
}

static ClassTable g_tab[4];
static std::once_flag g_tab_once;

static const ClassTable &table(int k, int kind) {
    std::call_once(g_tab_once, [] {
        for (int kd = 0; kd < 2; kd++) {
            build_table(3, kd, g_tab[2 * kd]);
            build_table(4, kd, g_tab[2 * kd + 1]);
        }
    });
    return g_tab[2 * kind + (k == 3 ? 0 : 1)];
}

const uint8_t *host_lut(int k, int kind) { return table(k, kind).lut.data(); }
const uint16_t *host_class_ids(int k, int kind) { return table(k, kind).ids.data(); }
int num_classes(int k, int kind) {
    return (k == 3 || k == 4) && (kind == 0 || kind == 1) ? (int)table(k, kind).ids.size() : -1;
}

}  // namespace vdmc

using namespace vdmc;

// ================================================================== C ABI
extern "C" {

const char *vdmc_last_error(void) { return g_err.c_str(); }

int64_t vdmc_kernel_launches(void) { return g_launches.load(); }

int vdmc_num_classes(int k) { return vdmc::num_classes(k, VDMC_DIRECTED); }

int vdmc_num_classes_kind(int k, int kind) { return vdmc::num_classes(k, kind); }

vdmc_status vdmc_class_ids_kind(int k, int kind, uint16_t *ids) {
    if (k != 3 && k != 4) return fail(VDMC_EK, "k=%d not in {3,4}", k);
    if (kind != VDMC_DIRECTED && kind != VDMC_UNDIRECTED) return fail(VDMC_EINVAL, "kind=%d not in {0,1}", kind);
    if (!ids) return fail(VDMC_EINVAL, "ids is NULL");
    memcpy(ids, host_class_ids(k, kind), sizeof(uint16_t) * num_classes(k, kind));
    return VDMC_OK;
}

vdmc_status vdmc_class_ids(int k, uint16_t *ids) { return vdmc_class_ids_kind(k, VDMC_DIRECTED, ids); }

static vdmc_status check_device(int device) {
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
        cudaGetLastError();
        return fail(VDMC_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= nd) return fail(VDMC_ENODEV, "device %d not in [0,%d)", device, nd);
    return VDMC_OK;
}

static vdmc_status check_rank(int64_t n, const int32_t *rank) {
    if (!rank) return VDMC_OK;
    std::vector<char> seen((size_t)n, 0);
    for (int64_t v = 0; v < n; v++) {
        int32_t r = rank[v];
        if (r < 0 || r >= n || seen[r]) return fail(VDMC_EORDER, "rank is not a permutation (vertex %lld)", (long long)v);
        seen[r] = 1;
    }
    return VDMC_OK;
}

vdmc_status vdmc_build_graph_edges(int64_t n, int64_t m, const int32_t *src, const int32_t *dst,
                                   int on_device, const int32_t *rank, int device, void *stream,
                                   vdmc_graph **out) {
    if (!out) return fail(VDMC_EINVAL, "out is NULL");
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(VDMC_EINVAL, "n=%lld outside [0, 2^30)", (long long)n);
    if (m < 0 || (m > 0 && (!src || !dst))) return fail(VDMC_EINVAL, "bad edge arrays (m=%lld)", (long long)m);
    if (on_device != 0 && on_device != 1) return fail(VDMC_EINVAL, "on_device must be 0 or 1");
    if (!on_device) {   // host input: validate here so the message can name the arc
        for (int64_t e = 0; e < m; e++) {
            if (src[e] < 0 || src[e] >= n || dst[e] < 0 || dst[e] >= n)
                return fail(VDMC_ERANGE, "arc %lld (%d -> %d): vertex id outside [0, %lld)", (long long)e,
                            src[e], dst[e], (long long)n);
            if (src[e] == dst[e])
                return fail(VDMC_ESELFLOOP, "arc %lld is a self-loop at vertex %d", (long long)e, src[e]);
        }
    }
    vdmc_status st = check_rank(n, rank);
    if (st) return st;
    if ((st = check_device(device))) return st;
    VDMC_CUDA(cudaSetDevice(device));
    cudaStream_t s = (cudaStream_t)stream;
    vdmc_graph *g = new vdmc_graph();
    g->device = device;
    const int32_t *d_src = src, *d_dst = dst;
    int32_t *tmp = nullptr;
    if (!on_device && m > 0) {
        cudaError_t e1 = dalloc((void **)&tmp, sizeof(int32_t) * 2 * m, s);
        if (e1 != cudaSuccess) { delete g; return fail(VDMC_ENOMEM, "cudaMallocAsync: %s", cudaGetErrorString(e1)); }
        cudaMemcpyAsync(tmp, src, sizeof(int32_t) * m, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(tmp + m, dst, sizeof(int32_t) * m, cudaMemcpyHostToDevice, s);
        d_src = tmp;
        d_dst = tmp + m;
    }
    st = build_device(n, m, d_src, d_dst, rank, device, s, g);
    if (tmp) dfree(tmp, s);
    if (st) { vdmc_free_graph(g); return st; }
    *out = g;
    return VDMC_OK;
}

vdmc_status vdmc_build_graph(int64_t n, const int64_t *indptr, const int32_t *nbr, const uint8_t *dir,
                             const int32_t *rank, int device, vdmc_graph **out) {
    if (!out || !indptr) return fail(VDMC_EINVAL, "NULL argument");
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(VDMC_EINVAL, "n=%lld outside [0, 2^30)", (long long)n);
    if (indptr[0] != 0) return fail(VDMC_EINVAL, "indptr[0] != 0");
    for (int64_t v = 0; v < n; v++)
        if (indptr[v + 1] < indptr[v]) return fail(VDMC_EINVAL, "indptr decreases at vertex %lld", (long long)v);
    const int64_t nnz = indptr[n];
    if (nnz > 0 && (!nbr || !dir)) return fail(VDMC_EINVAL, "NULL nbr/dir");
    // entries (v, u, code) with duplicates OR-merged; check each has its mirror
    std::vector<uint64_t> ent;
    ent.reserve((size_t)nnz);
    for (int64_t v = 0; v < n; v++)
        for (int64_t e = indptr[v]; e < indptr[v + 1]; e++) {
            int32_t u = nbr[e];
            if (u < 0 || u >= n) return fail(VDMC_ERANGE, "vertex %lld: neighbour %d outside [0,%lld)", (long long)v, u, (long long)n);
            if (u == v) return fail(VDMC_ESELFLOOP, "self-loop at vertex %lld", (long long)v);
            if (dir[e] < 1 || dir[e] > 3) return fail(VDMC_EINVAL, "vertex %lld: code %d not in {1,2,3}", (long long)v, dir[e]);
            ent.push_back(((uint64_t)v << 34) | ((uint64_t)u << 2) | dir[e]);
        }
    std::sort(ent.begin(), ent.end());
    std::vector<uint64_t> merged;
    for (size_t i = 0; i < ent.size(); i++) {
        if (!merged.empty() && (merged.back() >> 2) == (ent[i] >> 2)) merged.back() |= ent[i] & 3;
        else merged.push_back(ent[i]);
    }
    std::vector<int32_t> s, d;
    for (uint64_t x : merged) {
        uint64_t v = x >> 34, u = (x >> 2) & ((1ull << 32) - 1), c = x & 3;
        uint64_t cm = ((c & 1) << 1) | (c >> 1);
        uint64_t mirror = (u << 34) | (v << 2) | cm;
        if (!std::binary_search(merged.begin(), merged.end(), mirror))
            return fail(VDMC_EASYM, "entry (%llu, %llu) code %llu has no mirror (%llu, %llu) code %llu",
                        (unsigned long long)v, (unsigned long long)u, (unsigned long long)c,
                        (unsigned long long)u, (unsigned long long)v, (unsigned long long)cm);
        if (c & 1) { s.push_back((int32_t)v); d.push_back((int32_t)u); }
    }
    return vdmc_build_graph_edges(n, (int64_t)s.size(), s.data(), d.data(), 0, rank, device, nullptr, out);
}

vdmc_status vdmc_get_info(const vdmc_graph *g, vdmc_graph_info *info) {
    if (!g || !info) return fail(VDMC_EINVAL, "NULL argument");
    info->n = g->n;
    info->nnz = g->nnz;
    info->arcs = g->arcs;
    info->ntasks = g->ntasks;
    info->max_degree = g->max_degree;
    info->device = g->device;
    return VDMC_OK;
}

vdmc_status vdmc_get_order(const vdmc_graph *g, int32_t *order) {
    if (!g || !order) return fail(VDMC_EINVAL, "NULL argument");
    VDMC_CUDA(cudaSetDevice(g->device));
    if (g->n) VDMC_CUDA(cudaMemcpy(order, g->order, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost));
    return VDMC_OK;
}

vdmc_status vdmc_count_kind(vdmc_graph *g, int k, int kind, uint64_t *counts, const vdmc_range *work, void *stream) {
    if (k != 3 && k != 4) return fail(VDMC_EK, "k=%d not in {3,4}", k);
    if (kind != VDMC_DIRECTED && kind != VDMC_UNDIRECTED) return fail(VDMC_EINVAL, "kind=%d not in {0,1}", kind);
    if (!g) return fail(VDMC_EINVAL, "graph is NULL");
    if (!counts && g->n > 0) return fail(VDMC_EINVAL, "counts is NULL");
    int64_t lo = 0, hi = g->ntasks;
    if (work) {
        if (work->task_lo < 0 || work->task_hi < work->task_lo || work->task_hi > g->ntasks)
            return fail(VDMC_EINVAL, "work slice [%lld,%lld) not inside [0,%lld)", (long long)work->task_lo,
                        (long long)work->task_hi, (long long)g->ntasks);
        lo = work->task_lo;
        hi = work->task_hi;
    }
    VDMC_CUDA(cudaSetDevice(g->device));
    return launch_count(g, k, kind, counts, lo, hi, (cudaStream_t)stream);
}

vdmc_status vdmc_count(vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work, void *stream) {
    return vdmc_count_kind(g, k, VDMC_DIRECTED, counts, work, stream);
}

vdmc_status vdmc_split_costs(const int64_t *prefix, int64_t ntasks, int nparts, vdmc_range *parts) {
    if (nparts < 1 || !parts || ntasks < 0 || (ntasks > 0 && !prefix))
        return fail(VDMC_EINVAL, "bad arguments to vdmc_split_costs");
    const int64_t total = ntasks ? prefix[ntasks - 1] : 0;
    int64_t prev = 0;
    for (int p = 0; p < nparts; p++) {
        int64_t end;
        if (p == nparts - 1) end = ntasks;
        else {
            // first task whose inclusive prefix exceeds the target share ends this slice
            const __int128 target = (__int128)total * (p + 1) / nparts;
            end = std::upper_bound(prefix, prefix + ntasks, (int64_t)target) - prefix;
            end = std::max(end, prev);
        }
        parts[p].task_lo = prev;
        parts[p].task_hi = end;
        prev = end;
    }
    return VDMC_OK;
}

vdmc_status vdmc_plan(vdmc_graph *g, int k, int nparts, vdmc_range *parts) {
    if (k != 3 && k != 4) return fail(VDMC_EK, "k=%d not in {3,4}", k);
    if (!g || nparts < 1 || !parts) return fail(VDMC_EINVAL, "bad arguments to vdmc_plan");
    VDMC_CUDA(cudaSetDevice(g->device));
    vdmc_status st = ensure_plan(g, k, nullptr);
    if (st) return st;
    std::vector<int64_t> prefix((size_t)g->ntasks);
    if (g->ntasks) VDMC_CUDA(cudaMemcpy(prefix.data(), g->cost, sizeof(int64_t) * g->ntasks, cudaMemcpyDeviceToHost));
    return vdmc_split_costs(prefix.data(), g->ntasks, nparts, parts);
}

vdmc_status vdmc_set_profiling(vdmc_graph *g, int on) {
    if (!g) return fail(VDMC_EINVAL, "graph is NULL");
    VDMC_CUDA(cudaSetDevice(g->device));
    if (on && !g->ev[0])
        for (auto &e : g->ev) VDMC_CUDA(cudaEventCreate(&e));
    g->profiling = on ? 1 : 0;
    return VDMC_OK;
}

vdmc_status vdmc_last_timings(const vdmc_graph *g, float *ms, int nms) {
    if (!g || !ms || nms < 0 || nms > 5) return fail(VDMC_EINVAL, "bad arguments to vdmc_last_timings");
    vdmc_graph *gg = const_cast<vdmc_graph *>(g);
    if (g->profiling && g->ev[0]) {
        VDMC_CUDA(cudaSetDevice(g->device));
        // events: 0 count start, 1 plan done, 2 enum done, 3 finalize done
        float t[3];
        VDMC_CUDA(cudaEventElapsedTime(&t[0], g->ev[0], g->ev[1]));
        VDMC_CUDA(cudaEventElapsedTime(&t[1], g->ev[1], g->ev[2]));
        VDMC_CUDA(cudaEventElapsedTime(&t[2], g->ev[2], g->ev[3]));
        gg->last_ms[1] = t[0];
        gg->last_ms[2] = t[1];
        gg->last_ms[3] = t[2];
        gg->last_ms[4] = t[0] + t[1] + t[2];
    }
    gg->last_ms[0] = g->build_ms;
    for (int i = 0; i < nms; i++) ms[i] = g->last_ms[i];
    return VDMC_OK;
}

vdmc_status vdmc_trim(int device) {
    vdmc_status st = check_device(device);
    if (st) return st;
    VDMC_CUDA(cudaSetDevice(device));
    VDMC_CUDA(cudaDeviceSynchronize());
    trim_cache(device);
    return VDMC_OK;
}

void vdmc_free_graph(vdmc_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    cudaDeviceSynchronize();
    void *ptrs[] = {g->off, g->split, g->adj, g->order, g->tfirst, g->task_root, g->acc,
                    g->lscratch, g->ctr, g->lut[0][0], g->lut[0][1], g->lut[1][0], g->lut[1][1], g->cost, g->heavy_task, g->light_root,
                    g->hroots, g->hbase, g->nr_off, g->nr_adj};
    for (void *p : ptrs) dfree(p, nullptr);
    cudaStreamSynchronize(nullptr);
    for (auto &e : g->ev)
        if (e) cudaEventDestroy(e);
    delete g;
}

}  // extern "C"
