// api.cu -- the C ABI of libvdmc.so (declared and documented in include/vdmc.h),
// error reporting, and the motif-class lookup table.
#include <algorithm>
#include <array>
#include <tuple>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <unordered_map>
#include <vector>

#include <nccl.h>

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
// Generic 16-bit tables for k <= 5 (the BFS-layer path, layers.cu): the same
// definition (P:81 index, min over the k! orders, P:95 / P:138) over the pair-code-major device
// mask of k(k-1)/2 pairs in lexicographic order -- for k = 3 / 4 the same layout and columns as
// the 8-bit tables.  k = 5: 2^20 masks x 120 orders, built on all host cores once per process.
struct Table16 {
    std::vector<uint16_t> lut;   // mask -> column, 0xffff = disconnected
    std::vector<uint32_t> ids;   // column -> canonical paper index (20 bits for k = 5)
};

static void build_table16(int k, int kind, Table16 &t) {
    int pairs[10][2], np = 0;
    for (int i = 0; i < k; i++)
        for (int j = i + 1; j < k; j++) pairs[np][0] = i, pairs[np][1] = j, np++;
    const int nmask = 1 << (2 * np);
    std::vector<int32_t> canon(nmask);
    std::vector<char> conn(nmask);
    std::vector<std::array<int, 5>> perms;
    std::array<int, 5> p = {0, 1, 2, 3, 4};
    do perms.push_back(p);
    while (std::next_permutation(p.begin(), p.begin() + k));
    auto work = [&](int m0, int m1) {
        for (int m = m0; m < m1; m++) {
            int adj[5][5] = {}, und[5][5] = {};
            for (int q = 0; q < np; q++) {
                int c = (m >> (2 * q)) & 3;
                const int x = pairs[q][0], y = pairs[q][1];
                if (kind == 1 && c) c = 3;
                if (c & 1) adj[x][y] = 1;
                if (c & 2) adj[y][x] = 1;
                if (c) und[x][y] = und[y][x] = 1;
            }
            int seen = 1, grown = 1;
            while (grown) {
                grown = 0;
                for (int x = 0; x < k; x++)
                    if (seen >> x & 1)
                        for (int y = 0; y < k; y++)
                            if (und[x][y] && !(seen >> y & 1)) seen |= 1 << y, grown = 1;
            }
            conn[m] = seen == (1 << k) - 1;
            int best = 1 << 30;
            for (const auto &pp : perms) {   // new vertex i = old vertex pp[i]; rows, MSB first
                int idx = 0;
                for (int i = 0; i < k; i++)
                    for (int j = 0; j < k; j++)
                        if (i != j) idx = (idx << 1) | adj[pp[i]][pp[j]];
                best = std::min(best, idx);
            }
            canon[m] = best;
        }
    };
    const int nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int q = 0; q < nt; q++) th.emplace_back(work, (int)((int64_t)nmask * q / nt), (int)((int64_t)nmask * (q + 1) / nt));
    for (auto &x : th) x.join();
    std::vector<uint32_t> ids;
    for (int m = 0; m < nmask; m++)
        if (conn[m]) ids.push_back((uint32_t)canon[m]);
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    t.ids = ids;
    t.lut.assign(nmask, 0xffffu);
    for (int m = 0; m < nmask; m++)
        if (conn[m]) t.lut[m] = (uint16_t)(std::lower_bound(ids.begin(), ids.end(), (uint32_t)canon[m]) - ids.begin());
}

static Table16 g_tab16[3][2];   // [k - 3][kind]
static std::once_flag g_tab16_once[3][2];

static const Table16 &table16(int k, int kind) {
    std::call_once(g_tab16_once[k - 3][kind], [k, kind] { build_table16(k, kind, g_tab16[k - 3][kind]); });
    return g_tab16[k - 3][kind];
}

int num_classes(int k, int kind) {
    if (kind != 0 && kind != 1) return -1;
    if (k == 3 || k == 4) return (int)table(k, kind).ids.size();
    if (k == 5) return kind == 0 ? 9364 : 21;   // OEIS A003085(5) / A001349(5); table16 agrees (tests)
    return -1;
}

// the 16-bit LUT of (k, kind) on `device` (uploaded once per process, never freed)
vdmc_status device_lut16(int device, int k, int kind, const uint16_t **out) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, uint16_t *> cache;
    const Table16 &t = table16(k, kind);
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(device, k, kind);
    auto it = cache.find(key);
    if (it == cache.end()) {
        uint16_t *p = nullptr;
        VDMC_CUDA(cudaMalloc((void **)&p, t.lut.size() * sizeof(uint16_t)));
        VDMC_CUDA(cudaMemcpy(p, t.lut.data(), t.lut.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
        it = cache.emplace(key, p).first;
    }
    *out = it->second;
    return VDMC_OK;
}

const uint32_t *host_class_ids32(int k, int kind) { return table16(k, kind).ids.data(); }

}  // namespace vdmc

using namespace vdmc;

// ================================================================== C ABI
extern "C" {

const char *vdmc_last_error(void) { return g_err.c_str(); }

int64_t vdmc_kernel_launches(void) { return g_launches.load(); }

int vdmc_num_classes(int k) { return vdmc::num_classes(k, VDMC_DIRECTED); }

int vdmc_num_classes_kind(int k, int kind) { return vdmc::num_classes(k, kind); }

vdmc_status vdmc_class_ids_kind(int k, int kind, uint16_t *ids) {
    if (k != 3 && k != 4) return fail(VDMC_EK, "k=%d not in {3,4} (k = 5: vdmc_class_ids32)", k);
    if (kind != VDMC_DIRECTED && kind != VDMC_UNDIRECTED) return fail(VDMC_EINVAL, "kind=%d not in {0,1}", kind);
    if (!ids) return fail(VDMC_EINVAL, "ids is NULL");
    memcpy(ids, host_class_ids(k, kind), sizeof(uint16_t) * num_classes(k, kind));
    return VDMC_OK;
}

vdmc_status vdmc_class_ids(int k, uint16_t *ids) { return vdmc_class_ids_kind(k, VDMC_DIRECTED, ids); }

vdmc_status vdmc_class_ids32(int k, int kind, uint32_t *ids) {
    if (k < 3 || k > 5) return fail(VDMC_EK, "k=%d not in {3,4,5}", k);
    if (kind != VDMC_DIRECTED && kind != VDMC_UNDIRECTED) return fail(VDMC_EINVAL, "kind=%d not in {0,1}", kind);
    if (!ids) return fail(VDMC_EINVAL, "ids is NULL");
    const int C = num_classes(k, kind);
    if ((int)vdmc::table16(k, kind).ids.size() != C)
        return fail(VDMC_EINVAL, "class table of k=%d has %d classes, expected %d", k,
                    (int)vdmc::table16(k, kind).ids.size(), C);
    memcpy(ids, host_class_ids32(k, kind), sizeof(uint32_t) * C);
    return VDMC_OK;
}

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

vdmc_status vdmc_symmetrize(int64_t n, const int64_t *out_indptr, const int32_t *out_nbr, int device,
                            int64_t **indptr, int32_t **nbr, uint8_t **dir) {
    if (!out_indptr || !indptr || !nbr || !dir) return fail(VDMC_EINVAL, "NULL argument");
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(VDMC_EINVAL, "n=%lld outside [0, 2^30)", (long long)n);
    if (out_indptr[0] != 0) return fail(VDMC_EINVAL, "Indices[0] != 0");
    for (int64_t v = 0; v < n; v++)
        if (out_indptr[v + 1] < out_indptr[v]) return fail(VDMC_EINVAL, "Indices decreases at vertex %lld", (long long)v);
    const int64_t m = out_indptr[n];
    if (m > 0 && !out_nbr) return fail(VDMC_EINVAL, "Neighbors is NULL");
    // the paper's CSR row v lists the heads of v's arcs: expand to the arc list
    std::vector<int32_t> src((size_t)m), dst((size_t)m);
    for (int64_t v = 0; v < n; v++)
        for (int64_t e = out_indptr[v]; e < out_indptr[v + 1]; e++) {
            const int32_t u = out_nbr[e];
            if (u < 0 || u >= n)
                return fail(VDMC_ERANGE, "vertex %lld: out-neighbour %d outside [0,%lld)", (long long)v, u, (long long)n);
            if (u == v) return fail(VDMC_ESELFLOOP, "self-loop at vertex %lld", (long long)v);
            src[(size_t)e] = (int32_t)v;
            dst[(size_t)e] = u;
        }
    vdmc_status st = check_device(device);
    if (st) return st;
    VDMC_CUDA(cudaSetDevice(device));
    cudaStream_t s = nullptr;
    int32_t *d = nullptr;
    VDMC_CUDA(dalloc((void **)&d, sizeof(int32_t) * 2 * std::max<int64_t>(m, 1), s));
    if (m) {
        VDMC_CUDA(cudaMemcpyAsync(d, src.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
        VDMC_CUDA(cudaMemcpyAsync(d + m, dst.data(), sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
    }
    int64_t nnz = 0;
    uint64_t *ent = nullptr;
    int vb = 0;
    st = symmetrize_device(n, m, d, d + m, s, &nnz, &ent, &vb);
    dfree(d, s);
    if (st) return st;
    std::vector<uint64_t> h((size_t)nnz);
    cudaError_t ce = nnz ? cudaMemcpy(h.data(), ent, sizeof(uint64_t) * nnz, cudaMemcpyDeviceToHost) : cudaSuccess;
    dfree(ent, s);
    VDMC_CUDA(ce);
    int64_t *ip = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
    int32_t *nb = (int32_t *)malloc(sizeof(int32_t) * std::max<int64_t>(nnz, 1));
    uint8_t *dc = (uint8_t *)malloc(std::max<int64_t>(nnz, 1));
    if (!ip || !nb || !dc) {
        free(ip);
        free(nb);
        free(dc);
        return fail(VDMC_ENOMEM, "host allocation of %lld entries failed", (long long)nnz);
    }
    // entries: owner << (vb + 2) | nbr << 2 | code, sorted by (owner, nbr)
    const uint64_t vmask = (1ull << vb) - 1ull;
    for (int64_t v = 0; v <= n; v++) ip[v] = 0;
    for (int64_t e = 0; e < nnz; e++) {
        ip[(h[e] >> (vb + 2)) + 1]++;
        nb[e] = (int32_t)((h[e] >> 2) & vmask);
        dc[e] = (uint8_t)(h[e] & 3u);
    }
    for (int64_t v = 0; v < n; v++) ip[v + 1] += ip[v];
    *indptr = ip;
    *nbr = nb;
    *dir = dc;
    return VDMC_OK;
}

void vdmc_free_host(void *p) { free(p); }

vdmc_status vdmc_get_info(const vdmc_graph *g, vdmc_graph_info *info) {
    if (!g || !info) return fail(VDMC_EINVAL, "NULL argument");
    info->n = g->n;
    info->nnz = g->nnz;
    info->arcs = g->arcs;
    info->ntasks = g->ntasks;
    info->max_degree = g->max_degree;
    info->device = g->device;
    info->build_ms = g->build_ms;
    return VDMC_OK;
}

vdmc_status vdmc_get_order(const vdmc_graph *g, int32_t *order) {
    if (!g || !order) return fail(VDMC_EINVAL, "NULL argument");
    VDMC_CUDA(cudaSetDevice(g->device));
    if (g->n) VDMC_CUDA(cudaMemcpy(order, g->order, sizeof(int32_t) * g->n, cudaMemcpyDeviceToHost));
    return VDMC_OK;
}

static vdmc_status check_opts(int k, const vdmc_count_options *opt, CountOpts &o) {
    if (k < 3 || k > 5) return fail(VDMC_EK, "k=%d not in {3,4,5}", k);
    if (!opt) return VDMC_OK;
    if (opt->kind != VDMC_DIRECTED && opt->kind != VDMC_UNDIRECTED) return fail(VDMC_EINVAL, "kind=%d not in {0,1}", opt->kind);
    if (opt->star_block < 0 || opt->star_block > 1023) return fail(VDMC_EINVAL, "star_block=%d not in [1,1023] (0 = default)", opt->star_block);
    if (opt->cross_block != 0 && (opt->cross_block < 32 || opt->cross_block > 1023))
        return fail(VDMC_EINVAL, "cross_block=%d not in [32,1023] (0 = default)", opt->cross_block);
    if (opt->heavy_global < 0 || opt->heavy_global > 1 || opt->force_big < 0 || opt->force_big > 1)
        return fail(VDMC_EINVAL, "heavy_global / force_big must be 0 or 1");
    if (opt->layered < 0 || opt->layered > 1) return fail(VDMC_EINVAL, "layered must be 0 or 1");
    if (opt->acc64 < 0 || opt->acc64 > 1) return fail(VDMC_EINVAL, "acc64 must be 0 or 1");
    if (opt->ca_capacity < 0 || opt->ca_capacity > (int64_t(1) << 30))
        return fail(VDMC_EINVAL, "ca_capacity=%lld not in [1, 2^30] (0 = default)", (long long)opt->ca_capacity);
    o.kind = opt->kind;
    o.star_block = opt->star_block;
    o.cross_block = opt->cross_block;
    o.heavy_global = opt->heavy_global;
    o.force_big = opt->force_big;
    o.ca_capacity = opt->ca_capacity;
    o.layered = opt->layered;
    o.acc64 = opt->acc64;
    o.timings_ms = opt->timings_ms;
    return VDMC_OK;
}

static vdmc_status check_work(const vdmc_graph *g, const vdmc_range *work, int64_t &lo, int64_t &hi) {
    lo = 0;
    hi = g->ntasks;
    if (work) {
        if (work->task_lo < 0 || work->task_hi < work->task_lo || work->task_hi > g->ntasks)
            return fail(VDMC_EINVAL, "work slice [%lld,%lld) not inside [0,%lld)", (long long)work->task_lo,
                        (long long)work->task_hi, (long long)g->ntasks);
        lo = work->task_lo;
        hi = work->task_hi;
    }
    return VDMC_OK;
}

// one count: per-call class-major accumulator (block cache), enumerate, finalise
static vdmc_status count_impl(const vdmc_graph *g, int k, const CountOpts &o, uint64_t *counts, int64_t lo, int64_t hi,
                              cudaStream_t s) {
    const int C = num_classes(k, o.kind);
    float ms3[2] = {0, 0};
    cudaEvent_t ev[3] = {};
    if (o.timings_ms) {
        for (auto &e : ev) VDMC_CUDA(cudaEventCreate(&e));
        VDMC_CUDA(cudaEventRecord(ev[0], s));
    }
    const bool a32 = !o.acc64 && counts_fit_u32(g, k);   // 32-bit words when no count can exceed 2^32
    void *acc = nullptr;
    VDMC_CUDA(dalloc(&acc, (size_t)std::max<int64_t>(g->n, 1) * C * (a32 ? 4 : 8), s));
    vdmc_status st = a32 ? count_into32(g, k, o, (unsigned int *)acc, lo, hi, s, o.timings_ms ? ms3 : nullptr)
                         : count_into(g, k, o, (unsigned long long *)acc, lo, hi, s, o.timings_ms ? ms3 : nullptr);
    if (st == VDMC_OK) {
        if (o.timings_ms) cudaEventRecord(ev[1], s);
        st = a32 ? finalize32(g, C, (const unsigned int *)acc, counts, s)
                 : finalize(g, C, (const unsigned long long *)acc, counts, s);
        if (o.timings_ms) cudaEventRecord(ev[2], s);
    }
    dfree(acc, s);
    if (o.timings_ms) {
        if (st == VDMC_OK) {
            cudaEventSynchronize(ev[2]);
            float fin = 0, all = 0;
            cudaEventElapsedTime(&fin, ev[1], ev[2]);
            cudaEventElapsedTime(&all, ev[0], ev[2]);
            o.timings_ms[0] = ms3[0];
            o.timings_ms[1] = ms3[1];
            o.timings_ms[2] = fin;
            o.timings_ms[3] = all;
        }
        for (auto &e : ev) cudaEventDestroy(e);
    }
    return st;
}

vdmc_status vdmc_count_ex(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                          const vdmc_count_options *opt, void *stream) {
    CountOpts o;
    vdmc_status st = check_opts(k, opt, o);
    if (st) return st;
    if (!g) return fail(VDMC_EINVAL, "graph is NULL");
    if (!counts && g->n > 0) return fail(VDMC_EINVAL, "counts is NULL");
    int64_t lo, hi;
    if ((st = check_work(g, work, lo, hi))) return st;
    VDMC_CUDA(cudaSetDevice(g->device));
    if (k == 5 || o.layered)   // the generic BFS-layer path (layers.cu)
        return count_layers_impl(g, k, o.kind, counts, lo, hi, (cudaStream_t)stream, o.timings_ms);
    return count_impl(g, k, o, counts, lo, hi, (cudaStream_t)stream);
}

vdmc_status vdmc_count_kind(const vdmc_graph *g, int k, int kind, uint64_t *counts, const vdmc_range *work,
                            void *stream) {
    vdmc_count_options o{};
    o.kind = kind;
    return vdmc_count_ex(g, k, counts, work, &o, stream);
}

vdmc_status vdmc_count(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work, void *stream) {
    return vdmc_count_ex(g, k, counts, work, nullptr, stream);
}

vdmc_status vdmc_count_edges(const vdmc_graph *g, int k, uint64_t *counts, const vdmc_range *work,
                             const vdmc_count_options *opt, void *stream) {
    CountOpts o;
    vdmc_status st = check_opts(k, opt, o);
    if (st) return st;
    if (k == 5) return fail(VDMC_EK, "edge-level counts: k=%d not in {3,4}", k);
    if (!g) return fail(VDMC_EINVAL, "graph is NULL");
    if (!counts && g->ntasks > 0) return fail(VDMC_EINVAL, "counts is NULL");
    int64_t lo, hi;
    if ((st = check_work(g, work, lo, hi))) return st;
    VDMC_CUDA(cudaSetDevice(g->device));
    return count_edges_impl(g, k, o.kind, counts, lo, hi, (cudaStream_t)stream, o.timings_ms);
}

vdmc_status vdmc_get_edges(const vdmc_graph *g, int32_t *u, int32_t *v) {
    if (!g || ((!u || !v) && g->ntasks > 0)) return fail(VDMC_EINVAL, "NULL argument");
    VDMC_CUDA(cudaSetDevice(g->device));
    return edge_list_impl(g, u, v);
}

vdmc_status vdmc_root_range(const vdmc_graph *g, int64_t pos_lo, int64_t pos_hi, vdmc_range *out) {
    if (!g || !out) return fail(VDMC_EINVAL, "NULL argument");
    if (pos_lo < 0 || pos_hi < pos_lo || pos_hi > g->n)
        return fail(VDMC_EINVAL, "positions [%lld,%lld) not inside [0,%lld]", (long long)pos_lo, (long long)pos_hi,
                    (long long)g->n);
    VDMC_CUDA(cudaSetDevice(g->device));
    VDMC_CUDA(cudaMemcpy(&out->task_lo, g->tfirst + pos_lo, sizeof(int64_t), cudaMemcpyDeviceToHost));
    VDMC_CUDA(cudaMemcpy(&out->task_hi, g->tfirst + pos_hi, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return VDMC_OK;
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

vdmc_status vdmc_plan(const vdmc_graph *g, int k, int nparts, vdmc_range *parts) {
    if (k != 3 && k != 4) return fail(VDMC_EK, "k=%d not in {3,4}", k);
    if (!g || nparts < 1 || !parts) return fail(VDMC_EINVAL, "bad arguments to vdmc_plan");
    VDMC_CUDA(cudaSetDevice(g->device));
    std::vector<int64_t> prefix((size_t)g->ntasks);
    vdmc_status st = plan_prefix(g, k, prefix.data(), nullptr);
    if (st) return st;
    return vdmc_split_costs(prefix.data(), g->ntasks, nparts, parts);
}

// ------------------------------------------------------------------ multi-GPU (NCCL)
struct vdmc_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0, rank = 0, device = 0;
};

#define VDMC_NCCL(call)                                                                              \
    do {                                                                                             \
        ncclResult_t r_ = (call);                                                                    \
        if (r_ != ncclSuccess) return fail(VDMC_ENCCL, "%s: %s", #call, ncclGetErrorString(r_));       \
    } while (0)

vdmc_status vdmc_comm_unique_id(uint8_t id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    if (!id) return fail(VDMC_EINVAL, "id is NULL");
    ncclUniqueId u;
    VDMC_NCCL(ncclGetUniqueId(&u));
    memcpy(id, &u, sizeof u);
    return VDMC_OK;
}

vdmc_status vdmc_comm_init(int nranks, int rank, const uint8_t id[128], int device, vdmc_comm **out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(VDMC_EINVAL, "bad arguments to vdmc_comm_init");
    vdmc_status st = check_device(device);
    if (st) return st;
    VDMC_CUDA(cudaSetDevice(device));
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    ncclComm_t c = nullptr;
    VDMC_NCCL(ncclCommInitRank(&c, nranks, u, rank));
    vdmc_comm *h = new vdmc_comm();
    h->comm = c;
    h->nranks = nranks;
    h->rank = rank;
    h->device = device;
    *out = h;
    return VDMC_OK;
}

void vdmc_comm_free(vdmc_comm *c) {
    if (!c) return;
    if (c->comm) ncclCommDestroy(c->comm);
    delete c;
}

vdmc_status vdmc_count_distributed(const vdmc_graph *g, int k, const vdmc_count_options *opt, vdmc_comm *comm,
                                   int root, uint64_t *counts, void *stream) {
    CountOpts o;
    vdmc_status st = check_opts(k, opt, o);
    if (st) return st;
    if (k == 5 || o.layered) return fail(VDMC_EK, "vdmc_count_distributed: k=%d not in {3,4} / layered path", k);
    if (!g || !comm) return fail(VDMC_EINVAL, "NULL graph or communicator");
    if (root < 0 || root >= comm->nranks) return fail(VDMC_EINVAL, "root %d not in [0,%d)", root, comm->nranks);
    if (comm->device != g->device) return fail(VDMC_EINVAL, "graph on device %d, communicator on %d", g->device, comm->device);
    if (comm->rank == root && !counts && g->n > 0) return fail(VDMC_EINVAL, "counts is NULL on the root rank");
    VDMC_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<vdmc_range> parts((size_t)comm->nranks);
    if ((st = vdmc_plan(g, k, comm->nranks, parts.data()))) return st;
    const vdmc_range my = parts[(size_t)comm->rank];
    const int C = num_classes(k, o.kind);
    const size_t elems = (size_t)std::max<int64_t>(g->n, 1) * C;
    const bool a32 = !o.acc64 && counts_fit_u32(g, k);   // the full sums fit 32 bits, so do the partials
    void *acc = nullptr;
    VDMC_CUDA(dalloc(&acc, elems * (a32 ? 4 : 8), s));
    o.timings_ms = nullptr;
    st = a32 ? count_into32(g, k, o, (unsigned int *)acc, my.task_lo, my.task_hi, s, nullptr)
             : count_into(g, k, o, (unsigned long long *)acc, my.task_lo, my.task_hi, s, nullptr);
    if (st == VDMC_OK) {
        // sum of the class-major partials (unsigned wrap-around addition: exact), then the root
        // restores rows in place of original ids
        ncclResult_t r = ncclReduce(acc, acc, elems, a32 ? ncclUint32 : ncclUint64, ncclSum, root, comm->comm, s);
        if (r != ncclSuccess) st = fail(VDMC_ENCCL, "ncclReduce: %s", ncclGetErrorString(r));
        else if (comm->rank == root)
            st = a32 ? finalize32(g, C, (const unsigned int *)acc, counts, s)
                     : finalize(g, C, (const unsigned long long *)acc, counts, s);
    }
    dfree(acc, s);
    return st;
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
    void *ptrs[] = {g->off, g->split, g->adj, g->order, g->tfirst, g->task_root, g->lut[0][0], g->lut[0][1],
                    g->lut[1][0], g->lut[1][1], g->heavy_task, g->light_root, g->light_i0, g->hroots, g->hbase, g->nr_off,
                    g->nr_adj};
    for (void *p : ptrs) dfree(p, nullptr);
    cudaStreamSynchronize(nullptr);
    delete g;
}

}  // extern "C"
