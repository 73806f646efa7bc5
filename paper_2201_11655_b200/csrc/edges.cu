// edges.cu -- edge-level motif counts: the Discussion's extension,
// "counting motifs for edges, rather than vertices.  This change is minimal and only requires
// updating edges and not vertices once a motif was counted".
//
//   ecounts[e][j] = number of connected k-sets S containing both ends of the G_U edge e whose
//                   class is class_ids(k)[j]      (every G_U edge inside S gets +1; reading G18)
//
// The enumeration is the vertex path's proper k-BFS with the same S-local shape
// rules (Lemmas 2-4, reading G4/G5) and the same task unit (r, a), but every set is
// emitted explicitly (one set per lane): the vertex kernel's aggregated star / cross items
// credit members, not the edges between them.  Edge ids: the G_U edge {x < y} (ranks) is the
// task (x, y), id = tfirst[x] + position of y in N+(x) -- so the edge (r, a) of a task is the
// task itself, (r, b) for b = R[j] is tfirst[r] + j, and an edge met while walking a list comes
// from eid[] (per CSR entry, built per call).  Per set, with members r, a (fixed per task), b
// (warp-uniform) and c (per lane):
//   (r, a): warp-private histogram H, flushed once per task into edge t;
//   (r, b), (a, b): warp-uniform, lanes with equal classes merged (__match_any_sync);
//   edges touching c: one u64 atomicAdd per lane.
// Accumulator: class-major [C][ntasks] (u64), restored to rows [edge][C] in the canonical edge
// order (u < v by ORIGINAL id, lexicographic) by the vertex path's k_finalize with an edge
// permutation.
#include <algorithm>

#include <cub/cub.cuh>

#include "vdmc_internal.cuh"

namespace vdmc {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNone = 255;
constexpr int kEWarps = 8;                 // warps per CTA, one task each
constexpr int kEBlock = kEWarps * 32;
constexpr int kSR = 512;                   // R staged in shared memory when |N+(r)| <= kSR
constexpr int kSL = 512;                   // L_a staged in shared memory when deg(a) <= kSL
// per-warp shared words: R[kSR], La[kSL], LaE[kSL], Ba/Bb[kSR/16], Bl[kSL/16]
constexpr int kEWords = kSR + 2 * kSL + 2 * (kSR / 16) + kSL / 16;

struct EDev {
    const int64_t *__restrict__ off;
    const int64_t *__restrict__ split;
    const uint32_t *__restrict__ adj;
    const int64_t *__restrict__ tfirst;
    const int32_t *__restrict__ task_root;
    const uint32_t *__restrict__ eid;     // [nnz] edge id of each CSR entry
    unsigned long long *__restrict__ acc; // class-major [C][ns]
    uint64_t ns;                          // column stride = ntasks
    uint32_t *__restrict__ gscr;          // per-warp global scratch (lists too long for smem)
    int64_t gper;                         // words per warp: R, La, LaE [maxdeg] + 3 bitmaps
    int maxdeg;
};

__device__ __forceinline__ uint32_t get2(const uint32_t *B, int p) { return (B[p >> 4] >> ((p & 15) << 1)) & 3u; }
__device__ __forceinline__ void set2(uint32_t *B, int p, uint32_t code) { atomicOr(B + (p >> 4), code << ((p & 15) << 1)); }

__device__ __forceinline__ int find_rank(const uint32_t *S, int len, uint32_t x) {
    const uint32_t key = x << 2;
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < len && (S[lo] >> 2) == x) ? lo : -1;
}

// edge id of the G_U edge {x, y} (they must be adjacent): y's position in N+(min)
__device__ __forceinline__ uint32_t edge_of(const EDev &g, uint32_t x, uint32_t y) {
    const uint32_t lo_v = min(x, y), hi_v = max(x, y);
    int64_t lo = g.split[lo_v], hi = g.off[lo_v + 1];
    const int64_t s0 = lo;
    const uint32_t key = hi_v << 2;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (g.adj[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)(g.tfirst[lo_v] + (lo - s0));
}

__device__ __forceinline__ unsigned long long *eacc(const EDev &g, uint32_t e, uint32_t col) {
    return g.acc + ((size_t)col * g.ns + e);
}

// the task's (r, a) histogram -> edge t (also mid-task when a task could overflow 32 bits)
template <int C>
__device__ __forceinline__ void flush_h(uint32_t *H, const EDev &g, uint32_t t, int lane) {
    __syncwarp();
    for (int q = lane; q < C; q += 32) {
        const uint32_t v = H[q];
        if (v) {
            atomicAdd(eacc(g, t, q), (unsigned long long)v);
            H[q] = 0;
        }
    }
    __syncwarp();
}

// One set per lane (col = kNone: no set).  H: the task's (r, a) histogram.  eu1/eu2: edges
// that are the same for every lane (~0u = absent); el1..el3: this lane's other edges.
__device__ __forceinline__ void emit(uint32_t *H, const EDev &g, int col, uint32_t eu1, uint32_t eu2, uint32_t el1,
                                     uint32_t el2, uint32_t el3, int lane) {
    const bool v = col != kNone;
    const uint32_t cc = v ? (uint32_t)col : 0u;
    if (v) {
        if (el1 != ~0u) atomicAdd(eacc(g, el1, cc), 1ull);
        if (el2 != ~0u) atomicAdd(eacc(g, el2, cc), 1ull);
        if (el3 != ~0u) atomicAdd(eacc(g, el3, cc), 1ull);
    }
    const unsigned m = __match_any_sync(kFull, col);
    if (v && lane == __ffs(m) - 1) {
        const uint32_t cnt = __popc(m);
        atomicAdd(H + cc, cnt);
        if (eu1 != ~0u) atomicAdd(eacc(g, eu1, cc), (unsigned long long)cnt);
        if (eu2 != ~0u) atomicAdd(eacc(g, eu2, cc), (unsigned long long)cnt);
    }
}

template <int K, int C>
__global__ void __launch_bounds__(kEBlock, 3) k_edges(EDev g, int64_t lo, int64_t hi, unsigned long long *ctr,
                                                   const uint8_t *__restrict__ lut_g) {
    constexpr int NM = K == 3 ? 64 : 4096;
    __shared__ uint8_t lut[NM];
    __shared__ uint32_t hist[kEWarps][C];
    extern __shared__ uint32_t sm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int q = threadIdx.x; q < NM; q += kEBlock) lut[q] = lut_g[q];
    for (int q = threadIdx.x; q < kEWarps * C; q += kEBlock) (&hist[0][0])[q] = 0;
    __syncthreads();
    uint32_t *H = hist[wid];
    uint32_t *ws = sm + wid * kEWords;
    uint32_t *gw = g.gscr + ((int64_t)blockIdx.x * kEWarps + wid) * g.gper;
    const int bwg = (g.maxdeg + 15) / 16;
    for (;;) {
        unsigned long long x = 0;
        if (lane == 0) x = atomicAdd(ctr, 1ull);
        const int64_t t = lo + (int64_t)__shfl_sync(kFull, x, 0);
        if (t >= hi) break;
        const uint32_t r = (uint32_t)g.task_root[t];
        const int64_t rs = g.split[r];
        const int D = (int)(g.off[r + 1] - rs);
        const int i = (int)(t - g.tfirst[r]);
        const uint32_t er = (uint32_t)g.tfirst[r];   // edge id of (r, R[j]) = er + j
        const uint32_t ea = g.adj[rs + i], a = ea >> 2, cra = ea & 3u;
        const int64_t a0 = g.off[a], a1 = g.off[a + 1];
        const int dega = (int)(a1 - a0);
        // buffers: shared memory when both lists fit, else this warp's global scratch
        const bool small = D <= kSR && dega <= kSL;
        uint32_t *R, *La, *LaE, *Ba, *Bb, *Bl;
        if (small) {
            R = ws;
            La = ws + kSR;
            LaE = La + kSL;
            Ba = LaE + kSL;
            Bb = Ba + kSR / 16;
            Bl = Bb + kSR / 16;
            for (int q = lane; q < D; q += 32) R[q] = g.adj[rs + q];
        } else {
            R = const_cast<uint32_t *>(g.adj + rs);
            La = gw;
            LaE = gw + g.maxdeg;
            Ba = gw + 2 * (int64_t)g.maxdeg;
            Bb = Ba + bwg;
            Bl = Bb + bwg;
        }
        for (int q = lane; q < (D + 15) / 16; q += 32) Ba[q] = Bb[q] = 0;
        for (int q = lane; q < (dega + 15) / 16; q += 32) Bl[q] = 0;
        __syncwarp();
        // phase A: code(a, x) for x in R -> Ba; L_a = N(a) n {> r} \ N(r) (sorted) + edge ids
        int nL = 0;
        for (int base = 0; base < dega; base += 32) {
            const int p = base + lane;
            bool keep = false;
            uint32_t e = 0;
            if (p < dega) {
                e = g.adj[a0 + p];
                const uint32_t xv = e >> 2;
                if (xv > r) {
                    const int pos = find_rank(R, D, xv);
                    if (pos >= 0) set2(Ba, pos, e & 3u);
                    else keep = true;
                }
            }
            const unsigned bal = __ballot_sync(kFull, keep);
            if (keep) {
                const int w = nL + __popc(bal & ((1u << lane) - 1u));
                La[w] = e;
                LaE[w] = g.eid[a0 + p];
            }
            nL += __popc(bal);
        }
        __syncwarp();
        const bool bigt = D > 32767 || nL > 32767;   // a task's 32-bit histogram could overflow
        if constexpr (K == 3) {
            // "2": b in R after a: edges (r,a), (r,b), (a,b) if present
            for (int base = i + 1; base < D; base += 32) {
                const int j = base + lane;
                int col = kNone;
                uint32_t erb = ~0u, eab = ~0u;
                if (j < D) {
                    const uint32_t eb = R[j], cab = get2(Ba, j);
                    col = lut[cra | (eb & 3u) << 2 | cab << 4];
                    erb = er + j;
                    if (cab) eab = edge_of(g, a, eb >> 2);
                }
                emit(H, g, col, ~0u, ~0u, erb, eab, ~0u, lane);
            }
            // "1+1": b in L_a: edges (r,a), (a,b)
            for (int base = 0; base < nL; base += 32) {
                const int q = base + lane;
                int col = kNone;
                uint32_t eab = ~0u;
                if (q < nL) {
                    col = lut[cra | (La[q] & 3u) << 4];
                    eab = LaE[q];
                }
                emit(H, g, col, ~0u, ~0u, eab, ~0u, ~0u, lane);
            }
        } else {
            // b in R after a: walk N(b) once ("2+1" with c in L_b \ N(a); scatter Bb, Bl), then
            // "3" (c in R after b) and "2+1" with c in L_a
            for (int j = i + 1; j < D; j++) {
                const uint32_t eb = R[j], b = eb >> 2, crb = eb & 3u, cab = get2(Ba, j);
                const uint32_t mb = cra | crb << 2 | cab << 6;
                const uint32_t erb = er + j, eab = cab ? edge_of(g, a, b) : ~0u;
                const int64_t b0 = g.off[b], b1 = g.off[b + 1];
                bool tb = false, tl = false;
                for (int64_t base = b0; base < b1; base += 32) {
                    const int64_t p = base + lane;
                    int col = kNone;
                    uint32_t ebc = ~0u;
                    if (p < b1) {
                        const uint32_t e = g.adj[p], c = e >> 2;
                        if (c > r) {
                            const int pos = find_rank(R, D, c);
                            if (pos >= 0) {
                                if (pos > j) {
                                    set2(Bb, pos, e & 3u);
                                    tb = true;
                                }
                            } else {
                                const int q = find_rank(La, nL, c);
                                if (q >= 0) {
                                    set2(Bl, q, e & 3u);
                                    tl = true;
                                } else {   // c in L_b \ N(a): edges (r,a) (r,b) (a,b)? (b,c)
                                    col = lut[mb | (e & 3u) << 10];
                                    ebc = g.eid[p];
                                }
                            }
                        }
                    }
                    emit(H, g, col, erb, eab, ebc, ~0u, ~0u, lane);
                }
                __syncwarp();
                const int n3 = D - j - 1;
                for (int base = 0; base < n3 + nL; base += 32) {
                    const int xq = base + lane;
                    int col = kNone;
                    uint32_t e1 = ~0u, e2 = ~0u, e3 = ~0u;
                    if (xq < n3) {   // "3": c = R[p]: edges (r,c), (a,c)?, (b,c)?
                        const int p = j + 1 + xq;
                        const uint32_t ec = R[p], c = ec >> 2, cac = get2(Ba, p), cbc = get2(Bb, p);
                        col = lut[mb | (ec & 3u) << 4 | cac << 8 | cbc << 10];
                        e1 = er + p;
                        if (cac) e2 = edge_of(g, a, c);
                        if (cbc) e3 = edge_of(g, b, c);
                    } else if (xq < n3 + nL) {   // "2+1", c = L_a[q]: edges (a,c), (b,c)?
                        const int q = xq - n3;
                        const uint32_t ec = La[q], c = ec >> 2, cbc = get2(Bl, q);
                        col = lut[mb | (ec & 3u) << 8 | cbc << 10];
                        e1 = LaE[q];
                        if (cbc) e2 = edge_of(g, b, c);
                    }
                    emit(H, g, col, erb, eab, e1, e2, e3, lane);
                }
                __syncwarp();
                if (__any_sync(kFull, tb))
                    for (int q = ((j + 1) >> 4) + lane; q < (D + 15) / 16; q += 32) Bb[q] = 0;
                if (__any_sync(kFull, tl))
                    for (int q = lane; q < (nL + 15) / 16; q += 32) Bl[q] = 0;
                if (bigt) flush_h<C>(H, g, (uint32_t)t, lane);
                __syncwarp();
            }
            // b = L_a[x]: walk N(b) once ("1+1+1"; scatter Bl for "1+2"), then "1+2"
            for (int xb = 0; xb < nL; xb++) {
                const uint32_t eb = La[xb], b = eb >> 2, cab = eb & 3u;
                const uint32_t mb = cra | cab << 6, eab = LaE[xb];
                const int64_t b0 = g.off[b], b1 = g.off[b + 1];
                bool tl = false;
                for (int64_t base = b0; base < b1; base += 32) {
                    const int64_t p = base + lane;
                    int col = kNone;
                    uint32_t ebc = ~0u;
                    if (p < b1) {
                        const uint32_t e = g.adj[p], c = e >> 2;
                        if (c > r && find_rank(R, D, c) < 0) {
                            const int q = find_rank(La, nL, c);
                            if (q >= 0) {
                                if (q > xb) {
                                    set2(Bl, q, e & 3u);
                                    tl = true;
                                }
                            } else {   // "1+1+1": edges (r,a) (a,b) (b,c)
                                col = lut[mb | (e & 3u) << 10];
                                ebc = g.eid[p];
                            }
                        }
                    }
                    emit(H, g, col, eab, ~0u, ebc, ~0u, ~0u, lane);
                }
                __syncwarp();
                for (int base = xb + 1; base < nL; base += 32) {   // "1+2": c = L_a[q], q > xb
                    const int q = base + lane;
                    int col = kNone;
                    uint32_t e1 = ~0u, e2 = ~0u;
                    if (q < nL) {
                        const uint32_t ec = La[q], c = ec >> 2, cbc = get2(Bl, q);
                        col = lut[mb | (ec & 3u) << 8 | cbc << 10];
                        e1 = LaE[q];
                        if (cbc) e2 = edge_of(g, b, c);
                    }
                    emit(H, g, col, eab, ~0u, e1, e2, ~0u, lane);
                }
                __syncwarp();
                if (__any_sync(kFull, tl))
                    for (int q = ((xb + 1) >> 4) + lane; q < (nL + 15) / 16; q += 32) Bl[q] = 0;
                if (bigt) flush_h<C>(H, g, (uint32_t)t, lane);
                __syncwarp();
            }
        }
        flush_h<C>(H, g, (uint32_t)t, lane);   // the task's edge (r, a): the histogram of all its sets
    }
}

// eid[q] for every CSR entry: the edge {owner, nbr} = task (min, max); one warp per vertex
__global__ void k_eid(int64_t n, const int64_t *__restrict__ off, const int64_t *__restrict__ split,
                      const uint32_t *__restrict__ adj, const int64_t *__restrict__ tfirst, uint32_t *__restrict__ eid) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t v0 = off[v], vs = split[v], v1 = off[v + 1];
        for (int64_t q = v0 + lane; q < v1; q += 32) {
            if (q >= vs) {
                eid[q] = (uint32_t)(tfirst[v] + (q - vs));
            } else {   // nbr u < v: v's position in N+(u)
                const uint32_t u = adj[q] >> 2;
                int64_t lo = split[u], hi = off[u + 1];
                const int64_t s0 = lo;
                const uint32_t key = (uint32_t)v << 2;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (adj[mid] < key) lo = mid + 1;
                    else hi = mid;
                }
                eid[q] = (uint32_t)(tfirst[u] + (lo - s0));
            }
        }
    }
}

// per task: canonical key min(orig) << 32 | max(orig), value = task id
__global__ void k_edge_keys(int64_t ntasks, const int32_t *__restrict__ task_root, const int64_t *__restrict__ split,
                            const int64_t *__restrict__ tfirst, const uint32_t *__restrict__ adj,
                            const int32_t *__restrict__ order, uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntasks; t += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = task_root[t];
        const uint32_t a = adj[split[r] + (t - tfirst[r])] >> 2;
        const uint64_t u = (uint32_t)order[r], v = (uint32_t)order[a];
        keys[t] = (min(u, v) << 32) | max(u, v);
        vals[t] = (int32_t)t;
    }
}

__global__ void k_scatter_rows(int64_t ntasks, const int32_t *__restrict__ sorted_t, int32_t *__restrict__ rowof) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ntasks; q += (int64_t)gridDim.x * blockDim.x)
        rowof[sorted_t[q]] = (int32_t)q;
}

__global__ void k_split_keys(int64_t ntasks, const uint64_t *__restrict__ keys, int32_t *__restrict__ u,
                             int32_t *__restrict__ v) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ntasks; q += (int64_t)gridDim.x * blockDim.x) {
        u[q] = (int32_t)(keys[q] >> 32);
        v[q] = (int32_t)(keys[q] & 0xffffffffu);
    }
}

struct Tmp {   // stream-ordered temporaries, freed on scope exit
    cudaStream_t s;
    void *ptrs[16] = {};
    int np = 0;
    explicit Tmp(cudaStream_t st) : s(st) {}
    ~Tmp() {
        for (int q = 0; q < np; q++) dfree(ptrs[q], s);
    }
    template <class T> cudaError_t alloc(T **p, size_t count) {
        cudaError_t e = dalloc((void **)p, std::max<size_t>(1, count) * sizeof(T), s);
        if (e == cudaSuccess) ptrs[np++] = *p;
        return e;
    }
};

// canonical edge order: sorted (key, task) pairs; rowof[t] = row of task t (optional), and the
// sorted keys (optional)
vdmc_status edge_order(const vdmc_graph *g, cudaStream_t s, Tmp &tmp, int32_t **rowof_out, uint64_t **keys_out) {
    const int64_t T = g->ntasks;
    uint64_t *k0 = nullptr, *k1 = nullptr;
    int32_t *v0 = nullptr, *v1 = nullptr, *rowof = nullptr;
    VDMC_CUDA(tmp.alloc(&k0, T));
    VDMC_CUDA(tmp.alloc(&k1, T));
    VDMC_CUDA(tmp.alloc(&v0, T));
    VDMC_CUDA(tmp.alloc(&v1, T));
    VDMC_CUDA(tmp.alloc(&rowof, T));
    k_edge_keys<<<148 * 8, 256, 0, s>>>(T, g->task_root, g->split, g->tfirst, g->adj, g->order, k0, v0);
    VDMC_LAUNCH();
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    cub::DoubleBuffer<int32_t> dv(v0, v1);
    size_t tb = 0;
    VDMC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, (int)T, 0, 64, s));
    void *ts = nullptr;
    VDMC_CUDA(tmp.alloc((char **)&ts, tb));
    VDMC_CUDA(cub::DeviceRadixSort::SortPairs(ts, tb, dk, dv, (int)T, 0, 64, s));
    count_launch(8);
    k_scatter_rows<<<148 * 8, 256, 0, s>>>(T, dv.Current(), rowof);
    VDMC_LAUNCH();
    *rowof_out = rowof;
    if (keys_out) *keys_out = dk.Current();
    return VDMC_OK;
}

template <int K, int C>
vdmc_status run_edges(const vdmc_graph *g, const uint8_t *lut, unsigned long long *acc, const uint32_t *eid,
                      int64_t lo, int64_t hi, cudaStream_t s) {
    int nsm = 0;
    VDMC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    const size_t smem = (size_t)kEWarps * kEWords * 4;
    VDMC_CUDA(cudaFuncSetAttribute(k_edges<K, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    VDMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_edges<K, C>, kEBlock, smem));
    const int grid = std::max(1, nsm * std::max(per_sm, 1));
    const int md = (int)std::max<int64_t>(g->max_degree, 1);
    const int64_t gper = 2 * (int64_t)md + 3 * ((md + 15) / 16) + 1;
    Tmp tmp(s);
    uint32_t *scr = nullptr;
    unsigned long long *ctr = nullptr;
    VDMC_CUDA(tmp.alloc(&scr, (size_t)grid * kEWarps * gper));
    VDMC_CUDA(tmp.alloc(&ctr, 1));
    VDMC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), s));
    EDev d{};
    d.off = g->off;
    d.split = g->split;
    d.adj = g->adj;
    d.tfirst = g->tfirst;
    d.task_root = g->task_root;
    d.eid = eid;
    d.acc = acc;
    d.ns = (uint64_t)std::max<int64_t>(g->ntasks, 1);
    d.gscr = scr;
    d.gper = gper;
    d.maxdeg = md;
    if (hi > lo) {
        k_edges<K, C><<<grid, kEBlock, smem, s>>>(d, lo, hi, ctr, lut);
        VDMC_LAUNCH();
    }
    return VDMC_OK;
}

}  // namespace

vdmc_status count_edges_impl(const vdmc_graph *g, int k, int kind, uint64_t *counts, int64_t lo, int64_t hi,
                             cudaStream_t s, float *ms) {
    const int C = num_classes(k, kind);
    const int64_t T = g->ntasks;
    if (T == 0) return VDMC_OK;
    if (T >= (int64_t(1) << 31)) return fail(VDMC_EINVAL, "%lld edges >= 2^31 are not supported", (long long)T);
    cudaEvent_t ev[3] = {};
    if (ms) {
        for (auto &e : ev) VDMC_CUDA(cudaEventCreate(&e));
        VDMC_CUDA(cudaEventRecord(ev[0], s));
    }
    Tmp tmp(s);
    uint32_t *eid = nullptr;
    unsigned long long *acc = nullptr;
    VDMC_CUDA(tmp.alloc(&eid, g->nnz));
    VDMC_CUDA(tmp.alloc(&acc, (size_t)T * C));
    VDMC_CUDA(cudaMemsetAsync(acc, 0, (size_t)T * C * sizeof(uint64_t), s));
    k_eid<<<148 * 16, 256, 0, s>>>(g->n, g->off, g->split, g->adj, g->tfirst, eid);
    VDMC_LAUNCH();
    const uint8_t *lut = g->lut[kind][k == 4 ? 1 : 0];
    vdmc_status st;
    if (kind == VDMC_UNDIRECTED)
        st = k == 3 ? run_edges<3, kNumClassesU3>(g, lut, acc, eid, lo, hi, s)
                    : run_edges<4, kNumClassesU4>(g, lut, acc, eid, lo, hi, s);
    else
        st = k == 3 ? run_edges<3, kNumClasses3>(g, lut, acc, eid, lo, hi, s)
                    : run_edges<4, kNumClasses4>(g, lut, acc, eid, lo, hi, s);
    if (st) return st;
    if (ms) VDMC_CUDA(cudaEventRecord(ev[1], s));
    int32_t *rowof = nullptr;
    if ((st = edge_order(g, s, tmp, &rowof, nullptr))) return st;
    // rows: task order -> canonical edge order (the vertex finalise with rowof as the permutation)
    vdmc_graph view = *g;
    view.n = T;
    view.order = rowof;
    if ((st = finalize(&view, C, acc, counts, s))) return st;
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

vdmc_status edge_list_impl(const vdmc_graph *g, int32_t *u, int32_t *v) {
    const int64_t T = g->ntasks;
    if (T == 0) return VDMC_OK;
    cudaStream_t s = nullptr;
    Tmp tmp(s);
    int32_t *rowof = nullptr, *du = nullptr, *dv = nullptr;
    uint64_t *keys = nullptr;
    vdmc_status st = edge_order(g, s, tmp, &rowof, &keys);
    if (st) return st;
    VDMC_CUDA(tmp.alloc(&du, T));
    VDMC_CUDA(tmp.alloc(&dv, T));
    k_split_keys<<<148 * 8, 256, 0, s>>>(T, keys, du, dv);
    VDMC_LAUNCH();
    VDMC_CUDA(cudaMemcpyAsync(u, du, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaMemcpyAsync(v, dv, sizeof(int32_t) * T, cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaStreamSynchronize(s));
    return VDMC_OK;
}

}  // namespace vdmc
