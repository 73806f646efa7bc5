// enum.cu -- SURVEY §8(a) S4-S9 on the device: schedule, enumerate, classify, accumulate,
// finalise.
//
// The method: for every root r, count the proper k-BFS(r) -- the connected
// k-sets whose lowest-index vertex is r (Lemma 1) -- grouped by BFS-level shape
// (Lemma 2), each set once (Lemma 3; Lemma 4).  In rank order
// (vertex id = rank) with N+(x) = {u in N(x) : u > r} and L_x = N+(x) \ N(r) (depth-2
// children of depth-1 vertex x), the S-local shape rules (reading G4/G5) are
//   k = 3:  "2"     a < b in N+(r)
//           "1+1"   a in N+(r), b in L_a
//   k = 4:  "3"     a < b < c in N+(r)
//           "2+1"   a < b in N+(r), c in L_a, or c in L_b \ N(a)
//           "1+2"   a in N+(r), b < c in L_a
//           "1+1+1" a in N+(r), b in L_a, c in N+(b) \ N(r) \ N(a)
// Every connected set with minimum r falls in exactly one case once (its depth-1 set
// S n N(r) has 3, 2 or 1 members).
//
// Work unit: the task (r, a), a in N+(r): one warp; lanes split the inner loops.
// Classification: the pair codes of (r, a, b, c) form a 12-bit (6-bit) mask
// -> shared-memory LUT -> column of the minimum-isomorph class ("in real time").
// Accumulation ("for each vertex"; P:334 atomic add): r and a are fixed per task and
// share one per-warp shared-memory histogram (flushed once per task); b is warp-uniform in
// every inner loop, so equal columns are merged with __match_any_sync and added once; the
// innermost member c (k = 4) or b (k = 3) takes one u64 atomicAdd per set.
#include <algorithm>

#include <cub/cub.cuh>

#include "vdmc_internal.cuh"

namespace vdmc {
namespace {

constexpr int kWarps = 8;
constexpr int kBlock = kWarps * 32;
constexpr unsigned kFull = 0xffffffffu;

struct Dev {
    const int64_t *__restrict__ off;
    const int64_t *__restrict__ split;
    const uint32_t *__restrict__ adj;
    const int64_t *__restrict__ tfirst;
    const int32_t *__restrict__ task_root;
    unsigned long long *__restrict__ acc;   // [n][C], row = rank
};

__device__ __forceinline__ uint32_t swap2(uint32_t c) { return ((c & 1u) << 1) | (c >> 1); }

// first position in [lo, hi) whose entry has rank >= key (entries sort like their rank)
__device__ __forceinline__ int64_t lower_rank(const uint32_t *__restrict__ adj, int64_t lo, int64_t hi,
                                              uint32_t key) {
    const uint32_t k2 = key << 2;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (__ldg(adj + mid) < k2) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// code of y in the list [lo, hi) (owner's perspective), 0 if absent
__device__ __forceinline__ uint32_t code_in(const uint32_t *__restrict__ adj, int64_t lo, int64_t hi, uint32_t y) {
    int64_t p = lower_rank(adj, lo, hi, y);
    if (p < hi) {
        uint32_t e = __ldg(adj + p);
        if ((e >> 2) == y) return e & 3u;
    }
    return 0;
}

// code(x, y): bit0 = x -> y, bit1 = y -> x; searched in the shorter list
__device__ __forceinline__ uint32_t pair_code(const Dev &g, uint32_t x, uint32_t y) {
    const int64_t x0 = __ldg(g.off + x), x1 = __ldg(g.off + x + 1);
    const int64_t y0 = __ldg(g.off + y), y1 = __ldg(g.off + y + 1);
    if (x1 - x0 <= y1 - y0) return code_in(g.adj, x0, x1, y);
    return swap2(code_in(g.adj, y0, y1, x));
}

// r and a of the task: +cnt per column group in the warp's histogram
__device__ __forceinline__ void add_root(unsigned long long *wcnt, int col, int lane) {
    const unsigned m = __match_any_sync(kFull, col);
    if (col != kNoClass && lane == __ffs(m) - 1) wcnt[col] += __popc(m);
}

// r, a (histogram) and the warp-uniform member b (one atomic per column group)
template <int C>
__device__ __forceinline__ void add_root_b(unsigned long long *wcnt, unsigned long long *acc, uint32_t b, int col,
                                           int lane) {
    const unsigned m = __match_any_sync(kFull, col);
    if (col != kNoClass && lane == __ffs(m) - 1) {
        const unsigned cnt = __popc(m);
        wcnt[col] += cnt;
        atomicAdd(acc + (size_t)b * C + col, (unsigned long long)cnt);
    }
}

template <int K>
__global__ void __launch_bounds__(kBlock) k_enum(Dev g, int64_t lo, int64_t hi, unsigned long long *ctr,
                                                  const uint8_t *__restrict__ lut_g, uint32_t *__restrict__ lscr,
                                                  int64_t lcap) {
    constexpr int C = K == 3 ? kNumClasses3 : kNumClasses4;
    constexpr int NM = K == 3 ? 64 : 4096;
    __shared__ uint8_t lut[NM];
    __shared__ unsigned long long wcnt_all[kWarps][C];
    for (int i = threadIdx.x; i < NM; i += kBlock) lut[i] = lut_g[i];
    for (int i = threadIdx.x; i < kWarps * C; i += kBlock) (&wcnt_all[0][0])[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    unsigned long long *wcnt = wcnt_all[wid];
    uint32_t *L = lscr + (blockIdx.x * (int64_t)kWarps + wid) * lcap;
    const uint32_t *__restrict__ adj = g.adj;
    unsigned long long *__restrict__ acc = g.acc;

    for (;;) {
        unsigned long long t0 = 0;
        if (lane == 0) t0 = atomicAdd(ctr, 1ull);
        const int64_t t = lo + (int64_t)__shfl_sync(kFull, t0, 0);
        if (t >= hi) break;
        const uint32_t r = (uint32_t)g.task_root[t];
        const int64_t rs = g.split[r], re = g.off[r + 1];
        const int64_t ia = rs + (t - g.tfirst[r]);   // a's entry in r's list
        const uint32_t ea = adj[ia];
        const uint32_t a = ea >> 2, cra = ea & 3u;
        const int64_t a0 = g.off[a], a1 = g.off[a + 1];
        const int64_t as = lower_rank(adj, a0, a1, r + 1);   // a's entries with rank > r

        if constexpr (K == 3) {
            // "2": b in N+(r) after a.  mask (r,a) | (r,b) << 2 | (a,b) << 4
            for (int64_t base = ia + 1; base < re; base += 32) {
                const int64_t p = base + lane;
                int col = kNoClass;
                if (p < re) {
                    const uint32_t eb = adj[p], b = eb >> 2;
                    col = lut[cra | (eb & 3u) << 2 | pair_code(g, a, b) << 4];
                    atomicAdd(acc + (size_t)b * C + col, 1ull);
                }
                add_root(wcnt, col, lane);
            }
            // "1+1": b in L_a.  (r,b) = 0
            for (int64_t base = as; base < a1; base += 32) {
                const int64_t p = base + lane;
                int col = kNoClass;
                if (p < a1) {
                    const uint32_t eb = adj[p], b = eb >> 2;
                    if (code_in(adj, rs, re, b) == 0) {
                        col = lut[cra | (eb & 3u) << 4];
                        atomicAdd(acc + (size_t)b * C + col, 1ull);
                    }
                }
                add_root(wcnt, col, lane);
            }
        } else {
            // L_a = N+(a) \ N(r): entries of a's list (code (a, x)) kept in the warp's scratch
            int nL = 0;
            for (int64_t base = as; base < a1; base += 32) {
                const int64_t p = base + lane;
                bool keep = false;
                uint32_t e = 0;
                if (p < a1) {
                    e = adj[p];
                    keep = code_in(adj, rs, re, e >> 2) == 0;
                }
                const unsigned bal = __ballot_sync(kFull, keep);
                if (keep) L[nL + __popc(bal & ((1u << lane) - 1u))] = e;
                nL += __popc(bal);
            }
            __syncwarp();
            // mask: (r,a) | (r,b)<<2 | (r,c)<<4 | (a,b)<<6 | (a,c)<<8 | (b,c)<<10
            for (int64_t jb = ia + 1; jb < re; jb++) {           // b in N+(r) after a
                const uint32_t eb = adj[jb], b = eb >> 2;
                const uint32_t mb = cra | (eb & 3u) << 2 | pair_code(g, a, b) << 6;
                // "3": c in N+(r) after b
                for (int64_t base = jb + 1; base < re; base += 32) {
                    const int64_t p = base + lane;
                    int col = kNoClass;
                    if (p < re) {
                        const uint32_t ec = adj[p], c = ec >> 2;
                        col = lut[mb | (ec & 3u) << 4 | pair_code(g, a, c) << 8 | pair_code(g, b, c) << 10];
                        atomicAdd(acc + (size_t)c * C + col, 1ull);
                    }
                    add_root_b<C>(wcnt, acc, b, col, lane);
                }
                // "2+1", c in L_a:  (a,c) from a's list, (b,c) by search
                for (int base = 0; base < nL; base += 32) {
                    const int q = base + lane;
                    int col = kNoClass;
                    if (q < nL) {
                        const uint32_t ec = L[q], c = ec >> 2;
                        col = lut[mb | (ec & 3u) << 8 | pair_code(g, b, c) << 10];
                        atomicAdd(acc + (size_t)c * C + col, 1ull);
                    }
                    add_root_b<C>(wcnt, acc, b, col, lane);
                }
                // "2+1", c in L_b \ N(a):  (b,c) from b's list, (a,c) = 0
                const int64_t b1 = g.off[b + 1];
                const int64_t bs = lower_rank(adj, g.off[b], b1, r + 1);
                for (int64_t base = bs; base < b1; base += 32) {
                    const int64_t p = base + lane;
                    int col = kNoClass;
                    if (p < b1) {
                        const uint32_t ec = adj[p], c = ec >> 2;
                        if (code_in(adj, rs, re, c) == 0 && pair_code(g, a, c) == 0) {
                            col = lut[mb | (ec & 3u) << 10];
                            atomicAdd(acc + (size_t)c * C + col, 1ull);
                        }
                    }
                    add_root_b<C>(wcnt, acc, b, col, lane);
                }
            }
            for (int x = 0; x < nL; x++) {                        // b in L_a
                const uint32_t eb = L[x], b = eb >> 2;
                const uint32_t mb = cra | (eb & 3u) << 6;
                // "1+2": c in L_a after b
                for (int base = x + 1; base < nL; base += 32) {
                    const int q = base + lane;
                    int col = kNoClass;
                    if (q < nL) {
                        const uint32_t ec = L[q], c = ec >> 2;
                        col = lut[mb | (ec & 3u) << 8 | pair_code(g, b, c) << 10];
                        atomicAdd(acc + (size_t)c * C + col, 1ull);
                    }
                    add_root_b<C>(wcnt, acc, b, col, lane);
                }
                // "1+1+1": c in N+(b) \ N(r) \ N(a)  (Lemma 4: c may have global depth 2)
                const int64_t b1 = g.off[b + 1];
                const int64_t bs = lower_rank(adj, g.off[b], b1, r + 1);
                for (int64_t base = bs; base < b1; base += 32) {
                    const int64_t p = base + lane;
                    int col = kNoClass;
                    if (p < b1) {
                        const uint32_t ec = adj[p], c = ec >> 2;
                        if (code_in(adj, rs, re, c) == 0 && pair_code(g, a, c) == 0) {
                            col = lut[mb | (ec & 3u) << 10];
                            atomicAdd(acc + (size_t)c * C + col, 1ull);
                        }
                    }
                    add_root_b<C>(wcnt, acc, b, col, lane);
                }
            }
            __syncwarp();
        }
        // flush the task's histogram into rows r and a
        __syncwarp();
        for (int j = lane; j < C; j += 32) {
            const unsigned long long v = wcnt[j];
            if (v) {
                atomicAdd(acc + (size_t)r * C + j, v);
                atomicAdd(acc + (size_t)a * C + j, v);
                wcnt[j] = 0;
            }
        }
        __syncwarp();
    }
}

// S9: rows from rank order to original ids
template <int C>
__global__ void k_finalize(int64_t n, const int32_t *__restrict__ order, const unsigned long long *__restrict__ acc,
                           unsigned long long *__restrict__ out) {
    const int64_t total = n * C;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = idx / C, j = idx - v * C;
        out[(int64_t)order[v] * C + j] = acc[idx];
    }
}

// S4 cost proxy per task (r, a): sets of shape "3" plus the list lengths the other shapes scan
__global__ void k_cost(int64_t ntasks, int k, const int64_t *__restrict__ off, const int64_t *__restrict__ split,
                       const uint32_t *__restrict__ adj, const int64_t *__restrict__ tfirst,
                       const int32_t *__restrict__ task_root, int64_t *__restrict__ cost) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntasks; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = task_root[t];
        const int64_t rs = split[r], re = off[r + 1];
        const int64_t ia = rs + (t - tfirst[r]);
        const int64_t rem = re - ia - 1;
        const uint32_t a = adj[ia] >> 2;
        const int64_t da = off[a + 1] - off[a];
        cost[t] = k == 3 ? 1 + rem + da : 1 + rem * (rem - 1) / 2 + rem * da + da * da;
    }
}

}  // namespace

vdmc_status ensure_acc(vdmc_graph *g, int k) {
    const int C = num_classes(k);
    const size_t need = (size_t)std::max<int64_t>(g->n, 1) * C * sizeof(uint64_t);
    if (g->acc_bytes < need) {
        if (g->acc) cudaFree(g->acc);
        g->acc = nullptr;
        g->acc_bytes = 0;
        VDMC_CUDA(cudaMalloc(&g->acc, need));
        g->acc_bytes = need;
    }
    if (!g->ctr) VDMC_CUDA(cudaMalloc(&g->ctr, 4 * sizeof(unsigned long long)));
    if (!g->lut3) {
        VDMC_CUDA(cudaMalloc(&g->lut3, 64));
        VDMC_CUDA(cudaMemcpy(g->lut3, host_lut(3), 64, cudaMemcpyHostToDevice));
    }
    if (!g->lut4) {
        VDMC_CUDA(cudaMalloc(&g->lut4, 4096));
        VDMC_CUDA(cudaMemcpy(g->lut4, host_lut(4), 4096, cudaMemcpyHostToDevice));
    }
    return VDMC_OK;
}

vdmc_status ensure_plan(vdmc_graph *g, int k, cudaStream_t s) {
    if (g->cost && g->cost_k == k) return VDMC_OK;
    if (!g->cost) VDMC_CUDA(cudaMalloc(&g->cost, sizeof(int64_t) * std::max<int64_t>(g->ntasks, 1)));
    if (g->ntasks > 0) {
        int64_t *raw = nullptr;
        VDMC_CUDA(cudaMallocAsync(&raw, sizeof(int64_t) * g->ntasks, s));
        k_cost<<<148 * 8, 256, 0, s>>>(g->ntasks, k, g->off, g->split, g->adj, g->tfirst, g->task_root, raw);
        VDMC_LAUNCH();
        size_t tb = 0;
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, raw, g->cost, (int)g->ntasks, s));
        void *ts = nullptr;
        VDMC_CUDA(cudaMallocAsync(&ts, tb, s));
        VDMC_CUDA(cub::DeviceScan::InclusiveSum(ts, tb, raw, g->cost, (int)g->ntasks, s));
        count_launch(2);
        cudaFreeAsync(ts, s);
        cudaFreeAsync(raw, s);
        VDMC_CUDA(cudaStreamSynchronize(s));
    }
    g->cost_k = k;
    return VDMC_OK;
}

template <int K>
static vdmc_status run(vdmc_graph *g, uint64_t *counts, int64_t lo, int64_t hi, cudaStream_t s) {
    constexpr int C = K == 3 ? kNumClasses3 : kNumClasses4;
    int dev = g->device, nsm = 0, per_sm = 0;
    VDMC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    VDMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_enum<K>, kBlock, 0));
    const int grid = std::max(1, nsm * std::max(per_sm, 1));
    const int64_t lcap = std::max<int64_t>(g->max_degree, 1);
    if (K == 4) {
        const size_t need = (size_t)grid * kWarps * lcap;
        if (g->lscratch_elems < need) {
            if (g->lscratch) cudaFree(g->lscratch);
            g->lscratch = nullptr;
            g->lscratch_elems = 0;
            VDMC_CUDA(cudaMalloc(&g->lscratch, need * sizeof(uint32_t)));
            g->lscratch_elems = need;
        }
    }
    if (g->profiling) VDMC_CUDA(cudaEventRecord(g->ev[0], s));
    VDMC_CUDA(cudaMemsetAsync(g->acc, 0, (size_t)std::max<int64_t>(g->n, 1) * C * sizeof(uint64_t), s));
    VDMC_CUDA(cudaMemsetAsync(g->ctr, 0, sizeof(unsigned long long), s));
    if (g->profiling) VDMC_CUDA(cudaEventRecord(g->ev[1], s));
    Dev d{g->off, g->split, g->adj, g->tfirst, g->task_root, (unsigned long long *)g->acc};
    if (hi > lo) {
        k_enum<K><<<grid, kBlock, 0, s>>>(d, lo, hi, g->ctr, K == 3 ? g->lut3 : g->lut4, g->lscratch, lcap);
        VDMC_LAUNCH();
    }
    if (g->profiling) VDMC_CUDA(cudaEventRecord(g->ev[2], s));
    if (g->n > 0) {
        const int64_t total = g->n * C;
        const unsigned fg = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)nsm * 16);
        k_finalize<C><<<fg, 256, 0, s>>>(g->n, g->order, (const unsigned long long *)g->acc,
                                           (unsigned long long *)counts);
        VDMC_LAUNCH();
    }
    if (g->profiling) VDMC_CUDA(cudaEventRecord(g->ev[3], s));
    return VDMC_OK;
}

vdmc_status launch_count(vdmc_graph *g, int k, uint64_t *counts, int64_t lo, int64_t hi, cudaStream_t s) {
    vdmc_status st = ensure_acc(g, k);
    if (st) return st;
    return k == 3 ? run<3>(g, counts, lo, hi, s) : run<4>(g, counts, lo, hi, s);
}

}  // namespace vdmc
