// enum.cu -- SURVEY §8(a) S4-S9 on the device: schedule, enumerate, classify, accumulate,
// finalise.
//
// The method: for every root r, count the proper k-BFS(r) -- the connected
// k-sets whose lowest-index vertex is r (Lemma 1) -- grouped by BFS-level shape
// (Lemma 2), each set once (Lemma 3; Lemma 4).  In rank order
// (vertex id = rank) with R = N+(r) = {u in N(r) : u > r} and L_x = N+(x) \ N(r) (the
// depth-2 children of a depth-1 vertex x), the S-local shape rules (readings G4/G5) are
//   k = 3:  "2"     a < b in R
//           "1+1"   a in R, b in L_a
//   k = 4:  "3"     a < b < c in R
//           "2+1"   a < b in R, c in L_a, or c in L_b \ N(a)
//           "1+2"   a in R, b < c in L_a
//           "1+1+1" a in R, b in L_a, c in N+(b) \ N(r) \ N(a)   (Lemma 4: c may be "depth 2")
// Every connected set with minimum r falls in exactly one case, once.
//
// Work unit ("each pair of a vertex and one of its neighbors"): the task (r, a).
//   * heavy roots (deg(r) > kLightDeg): the CTA stages R = N+(r) once per root; a task whose a
//     has a short list (<= kWL) runs on one warp (light_task_hp<HV>, 16 tasks in flight per
//     CTA), the others on the whole CTA (the 16 warps split its items).  R and L_a live in
//     shared memory (global scratch if the graph's degree is too big).
//   * light roots: one warp per item (<= kLightChunk tasks of one root), its tasks in sequence;
//     R, L_a and their staged lists in the warp's smem.
//   One persistent kernel: CTAs drain the heavy task list (ordered by rank = degree
//   descending, then by a's position: longest first), then their warps drain the light
//   items.  Both lists come from a global atomic counter.  k = 4 default: closed forms
//   (DESIGN §3b), the "2+1" R[j] side of heavy roots summed per root by k_rside.
// Membership tests are binary searches in the staged sorted lists (shared memory).  The
// codes (a, x) and (b, x) for x in R or L_a are scattered once into 2-bit-per-position
// bitmaps, so the innermost loops (one set per lane) read only shared memory.
// Classification: the pair codes of (r, a, b, c) form a 12-bit (6-bit) mask ->
// shared-memory LUT -> column of the minimum-isomorph class, "in real time".
// Accumulation (P:334 atomic add): r and a are fixed per task: one warp-private u32
// histogram, flushed per task into rows r and a; b is warp-uniform in every inner loop
// (k = 4): lanes with equal columns are merged by __match_any_sync into one atomic; the
// innermost member (c for k = 4, b for k = 3) takes one u64 atomicAdd per set.
#include <algorithm>

#include <cstdlib>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "vdmc_internal.cuh"

// The accumulator word: u64, or u32 when every count provably fits (enum32.cu compiles this file
// again with VDMC_ACC32 = 1; the host picks it when 6 * maxdeg^3 < 2^32, a bound on the connected
// 4-sets through one vertex, so no (vertex, class) count can wrap).  Halving the n x C matrix
// keeps twice as many of its hot class columns in L2.
#ifndef VDMC_ACC32
#define VDMC_ACC32 0
#endif

namespace vdmc {
namespace {

#if VDMC_ACC32
using AccT = unsigned int;
#else
using AccT = unsigned long long;
#endif

constexpr int kWarps = 16;            // warps per CTA
constexpr int kBlock = kWarps * 32;
constexpr int kLightDeg = 128;        // light root: G_U degree <= this (measured best of 64/128/256)
constexpr unsigned kFull = 0xffffffffu;
constexpr int kNone = 255;
constexpr int kPF = 2;                // light walks: list entries per lane loaded ahead
constexpr int kHChunk = 32;           // heavy tasks fetched per CTA request (<= 32: one warp classifies them)
constexpr int kHubDeg = 1024;         // heavy tasks of the leading roots above this degree (a prefix of the heavy
constexpr int kHubChunk = 16;         // list under the degree order) are fetched kHubChunk per request
constexpr int kWL = 256;              // heavy warp-mode task: a's list length at most this (its L_a slot;
                                      // measured 64 / 128 / 256 / 512: 256 best)
constexpr int kLightChunk = 8;        // light items: at most this many tasks of one root (a root of ~100
                                      // tasks is ~15 ms of one warp: cut, it no longer bounds a slice)

// Profiling switches that DROP work (VDMC_PHASES / VDMC_SKIP / VDMC_MINREM) exist only in the
// profiling build (-DVDMC_PROFILING, tools/build_variant.sh); the product library has none.
#ifdef VDMC_PROFILING
#define VDMC_SKIPF(g) ((g).skip)
#else
#define VDMC_SKIPF(g) 0
#endif

struct Dev {
    const int64_t *__restrict__ off;
    const int64_t *__restrict__ split;
    const uint32_t *__restrict__ adj;
    const int64_t *__restrict__ tfirst;
    const int32_t *__restrict__ task_root;
    const int32_t *__restrict__ heavy_task;   // task ids of heavy roots, rank order
    const int32_t *__restrict__ light_root;   // light items (root, first task offset i0), rank order
    const int32_t *__restrict__ light_i0;
    int64_t nheavy, nlight;
    AccT *__restrict__ acc;                   // accumulator, class-major: element (v = rank, col) at col * ns + v
    uint32_t ns;                              // column stride = n
    uint32_t *__restrict__ gheavy;            // global fallback: per-CTA heavy buffers
    uint32_t *__restrict__ glight;            // global fallback: per-warp oversize L_a + bitmap
    int64_t gheavy_per_cta, glight_per_warp;  // words
    int heavy_in_smem;                        // heavy buffers fit in shared memory
    int big;                                  // flush the u32 histograms per item (degrees > 32767, or forced)
    int maxdeg;
    int off32;                                // n * C < 2^32: 32-bit accumulator offsets
    int fold;                                 // star items: b positions per item (<= kMaxBlock: 10-bit fields);
                                              // 0 = default kMaxBlock
    int xblock;                               // cross items: positions per item (<= kMaxBlock)
#ifdef VDMC_PROFILING
    int skip;                                 // profiling build only: bit0 star3_heavy, bit1 b in R loop, bit2 b in L_a loop, bit3 no cross items (ca_build)
    int minrem;                               // profiling build only: skip heavy tasks with D - i - 1 < minrem
                                              // (minrem < 0: skip those with D - i - 1 >= -minrem)
#endif
    uint32_t *__restrict__ gca;               // per-CTA: c's R-neighbour lists of a heavy task (cross items)
    int64_t gca_per_cta;                      // words: CAbeg[maxdeg], CAlen[maxdeg], CA[ca_cap]
    uint32_t ca_cap;
    const int64_t *__restrict__ hbase;        // heavy root -> segment of nr_off
    const int64_t *__restrict__ nr_off;       // induced adjacency of N+(r), position space
    const uint32_t *__restrict__ nr_adj;
    int64_t hub_tasks;                        // heavy tasks of the leading roots of degree > kHubDeg
    uint32_t *__restrict__ gM;                // closed forms, heavy tasks: M[w] per task at (hbase[r] + i) * 4 + w;
                                              // the "2+1" R[j] side is then added per root by k_rside
};

// shared-memory layout (words), computed on the host
struct Layout {
    int R, La, Ba, Bb, Bl;        // heavy: R[maxdeg], La[maxdeg], Ba[bw], Bb[kWarps][bw], Bl[kWarps][lw]
    int bw, lw;                   // bitmap words for R positions / L positions
    int hist;                     // per-warp u32 histograms [kWarps][C]
    int light;                    // light region: per warp kLightWords
    int total;                    // words
    int T;                        // heavy: bucket index of R (u16 positions, kBuckets + 1 of them), or -1
    int NB;                       // heavy: bit q = position q of R has an induced neighbour (k_nr lists)
    int W, ws, wm;                // heavy: per-warp slots of the warp-mode tasks (overlay La..Bl), stride, enabled
};
constexpr int kLW = kLightDeg;               // light list capacity
constexpr int kLB = (kLightDeg + 15) / 16;   // light bitmap words
// per light warp: R[kLW], La[kLW], Ba[kLB], Bb[kLB], Bl[kLB]
constexpr int kSmax = 64;                    // light: lists staged for at most this many vertices
constexpr int kPool = 896;                   // light: staged list entries, R's lists then L_a's lists
constexpr int kFW = 32;                      // light: 1024-bit membership filters of R and of L_a
constexpr int kRecCap = 128;                 // light: induced-edge records of N+(r) per item (top of the pool)
constexpr int kLightWords = 2 * kLW + 3 * kLB + 2 * (2 * kSmax + 1) + kPool + 2 * kFW + 4;   // + M[4] (closed form)

// accumulator element (v, col) at col * n + v.  Class-major: the updates of one class from many
// sets share sectors with other vertices' updates of the same (hot) class, so a matrix far
// larger than L2 still hits L2 for the few classes that dominate (cfg5: 417 -> 352 ms vs
// row-major, profiles/r01_v8_*); rows are restored by k_finalize.
__device__ __forceinline__ AccT *accp(const Dev &g, uint32_t v, uint32_t col) {
    return g.acc + ((size_t)col * g.ns + v);
}

// Light walks: a 1024-bit one-hash filter of a vertex set (R per root, L_a per task).  A clear
// bit proves the vertex is not in the set, so most list entries skip the binary search (in ER
// graphs nearly every walked entry is in neither); a set bit falls back to the exact search.
__device__ __forceinline__ uint32_t fhash(uint32_t v) { return (v * 0x9E3779B1u) >> 22; }
__device__ __forceinline__ bool fmay(const uint32_t *F, uint32_t v) {
    if (!F) return true;
    const uint32_t h = fhash(v);
    return (F[h >> 5] >> (h & 31u)) & 1u;
}
__device__ __forceinline__ void fadd(uint32_t *F, uint32_t v) {
    const uint32_t h = fhash(v);
    atomicOr(F + (h >> 5), 1u << (h & 31u));
}

__device__ __forceinline__ int find_rank(const uint32_t *S, int len, uint32_t x) {
    // position of vertex x in the sorted entry list S[0..len), or -1
    const uint32_t key = x << 2;
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < len && (S[lo] >> 2) == x) ? lo : -1;
}

// Heavy roots: a bucket index over R's vertex range (R ascends): bucket b holds the positions
// [T[b], T[b + 1]) whose vertex v has (v - lo) >> shift == b; a lookup is one table read plus a
// binary search over ~D / kBuckets entries instead of log2(D) steps over all of R.
constexpr int kBuckets = 4096;
struct RIndex {
    uint32_t lo, hi;   // vertex range of R
    int shift;         // bucket width 2^shift
    const uint16_t *T; // nullptr: plain binary search
};
__device__ __forceinline__ int find_pos(const uint32_t *R, int D, uint32_t x, const RIndex &ix) {
    if (!ix.T) return find_rank(R, D, x);
    if (x < ix.lo || x > ix.hi) return -1;
    const uint32_t b = (x - ix.lo) >> ix.shift;
    int lo = ix.T[b], hi = ix.T[b + 1];
    const uint32_t key = x << 2;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (R[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return (lo < ix.T[b + 1] && (R[lo] >> 2) == x) ? lo : -1;
}
// build T for the staged R (whole CTA; the caller syncs before use).  Returns the index.
__device__ __forceinline__ RIndex build_rindex(const uint32_t *R, int D, uint16_t *T, int tid, int nthreads) {
    RIndex ix{0u, 0u, 0, nullptr};
    if (T == nullptr || D <= 0 || D > 65535) return ix;
    ix.lo = R[0] >> 2;
    ix.hi = R[D - 1] >> 2;
    const uint32_t span = ix.hi - ix.lo;   // buckets 0 .. span >> shift
    const uint32_t nbmax = (uint32_t)min(kBuckets, max(32, 2 * D));   // ~2 buckets per entry: O(D) to build
    int sh = 0;
    while ((span >> sh) >= nbmax) sh++;
    ix.shift = sh;
    const int nb = (int)(span >> sh) + 1;   // <= nbmax; lookups read T[0 .. nb]
    for (int q = tid; q < D; q += nthreads) {   // T[b] = first q with bucket(R[q]) >= b
        const int bq = (int)(((R[q] >> 2) - ix.lo) >> sh);
        const int bp = q > 0 ? (int)(((R[q - 1] >> 2) - ix.lo) >> sh) : -1;
        for (int b = bp + 1; b <= bq; b++) T[b] = (uint16_t)q;
    }
    if (tid == 0) T[nb] = (uint16_t)D;   // end of the last bucket
    ix.T = T;
    return ix;
}

__device__ __forceinline__ uint32_t swap2(uint32_t c) { return ((c & 1u) << 1) | (c >> 1); }
__device__ __forceinline__ uint32_t get2(const uint32_t *B, int p) { return (B[p >> 4] >> ((p & 15) << 1)) & 3u; }
__device__ __forceinline__ void set2(uint32_t *B, int p, uint32_t code) { atomicOr(B + (p >> 4), code << ((p & 15) << 1)); }

// predicated fire-and-forget add (no divergent branch around it in the uniform b loops)
#if !VDMC_ACC32
__device__ __forceinline__ void red_if(bool p, unsigned long long *addr, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.global.add.u64 [%0], %1;\n\t}\n" ::"l"(addr),
        "l"((unsigned long long)v), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ void acc_add(unsigned long long *p, uint32_t v) { atomicAdd(p, (unsigned long long)v); }
#else
__device__ __forceinline__ void red_if(bool p, unsigned int *addr, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.global.add.u32 [%0], %1;\n\t}\n" ::"l"(addr),
        "r"(v), "r"((uint32_t)p)
        : "memory");
}
__device__ __forceinline__ void acc_add(unsigned int *p, uint32_t v) { atomicAdd(p, v); }
#endif

// predicated shared-memory u32 reduction (histograms)
__device__ __forceinline__ void red_shared_if(bool p, uint32_t *addr, uint32_t v) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(addr)),
        "r"(v), "r"((uint32_t)p)
        : "memory");
}

// one set with members r, a (histogram H), b (warp-uniform, merged per column) and c (lane)
template <int C>
__device__ __forceinline__ void emit4(uint32_t *H, const Dev &g, uint32_t b, uint32_t c, int col, int lane) {
    const bool v = col != kNone;
    const uint32_t cc = v ? (uint32_t)col : 0u;
    red_if(v, accp(g, c, cc), 1u);
    const unsigned m = __match_any_sync(kFull, col);
    const bool lead = v && lane == __ffs(m) - 1;   // one lane per distinct column (predicated, no branch)
    const uint32_t cnt = __popc(m);
    red_shared_if(lead, H + cc, cnt);
    red_if(lead, accp(g, b, cc), cnt);
}

// one set with members r, a (histogram H) and b (lane)
template <int C>
__device__ __forceinline__ void emit3(uint32_t *H, const Dev &g, uint32_t b, int col, int lane) {
    const bool v = col != kNone;
    const uint32_t cc = v ? (uint32_t)col : 0u;
    red_if(v, accp(g, b, cc), 1u);
    const unsigned m = __match_any_sync(kFull, col);
    red_shared_if(v && lane == __ffs(m) - 1, H + cc, (uint32_t)__popc(m));
}

__device__ __forceinline__ void acc_addw(AccT *p, AccT v) { atomicAdd(p, v); }   // modular ("-1" = all ones)

// warp-private histogram -> rows r and a (entries are signed 32-bit: |net count| < 2^31 between
// flushes -- per task below degree 32767, per work item above it)
template <int C>
__device__ __forceinline__ void flush_hist(uint32_t *H, const Dev &g, uint32_t r, uint32_t a, int lane) {
    __syncwarp();
    for (int j = lane; j < C; j += 32) {
        const uint32_t v = H[j];
        if (v) {   // signed: the closed forms' take-backs can leave a net negative entry in a warp
            const AccT sv = (AccT)(long long)(int)v;
            acc_addw(accp(g, r, j), sv);
            acc_addw(accp(g, a, j), sv);
            H[j] = 0;
        }
    }
    __syncwarp();
}

__device__ __forceinline__ void clear_words(uint32_t *B, int w0, int w1, int lane) {   // words [w0, w1)
    for (int w = w0 + lane; w < w1; w += 32) B[w] = 0;
}

// A vertex's adjacency list: in global memory, or staged in the warp's shared memory.
struct List {
    const uint32_t *p;
    int len;
};
__device__ __forceinline__ List glist(const Dev &g, uint32_t v) {
    const int64_t o = g.off[v];
    return List{g.adj + o, (int)(g.off[v + 1] - o)};
}

// Copy the lists of the m vertices V[q] >> 2 (q < m) into B (capacity cap), S[q] = start of
// q's list, S[m] = total, O[q] = its global offset.  One flattened pass, every load
// independent (memory-level parallelism instead of one dependent chain per list).
// Returns false (and stages nothing) if m > smax or the lists exceed cap.  One warp.
__device__ __forceinline__ void gather_wait() {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
}
__device__ bool gather_lists(const Dev &g, const uint32_t *V, int m, uint32_t *S, uint32_t *O, int smax, uint32_t *B,
                             int cap, int lane, bool wait = true) {
    if (m > smax) return false;
    int total = 0;
    for (int b0 = 0; b0 < m; b0 += 32) {
        const int q = b0 + lane;
        int len = 0;
        uint32_t o = 0;
        bool big = false;
        if (q < m) {
            const uint32_t v = V[q] >> 2;
            const int64_t x0 = g.off[v];
            o = (uint32_t)x0;
            big = x0 > 0xffffffffll;   // 32-bit staged offsets: graphs past 2^32 entries are not staged
            len = (int)(g.off[v + 1] - x0);
        }
        if (__any_sync(kFull, big)) return false;
        int inc = len;   // inclusive warp scan
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int y = __shfl_up_sync(kFull, inc, d);
            if (lane >= d) inc += y;
        }
        if (q < m) {
            S[q] = (uint32_t)(total + inc - len);
            O[q] = o;
        }
        total += __shfl_sync(kFull, inc, 31);
    }
    __syncwarp();
    if (total > cap) return false;
    if (lane == 0) S[m] = (uint32_t)total;
    __syncwarp();
    // asynchronous global -> shared copies (cp.async): every entry of the gather is in flight at
    // once instead of one dependent load per lane and step.  The list holding entry f: as in
    // flat_walk, 32 consecutive entries per pass, a bitmap of the list starts inside (base,
    // base + 32] and one popc (every staged list is non-empty: its vertex is adjacent to r or a)
    int o = 0;
    for (int base = 0; base < total; base += 32) {
        const int qb = o + 1 + lane;
        const int d = qb < m ? (int)S[qb] - base : 64;
        const unsigned E = __reduce_or_sync(kFull, d >= 1 && d <= 32 ? 1u << (d - 1) : 0u);
        const int own = o + __popc(E & ((1u << lane) - 1u));
        o += __popc(E);
        const int f = base + lane;
        if (f < total) {
            const uint32_t *src = g.adj + ((int64_t)O[own] + (f - (int)S[own]));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((uint32_t)__cvta_generic_to_shared(B + f)),
                         "l"(src)
                         : "memory");
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    if (wait) gather_wait();   // else the caller waits (gather_wait) before reading B
    return true;
}

// Lists staged in a light warp's shared memory (gather_lists), else read from global memory.
struct Staged {
    const uint32_t *RL, *RS;   // lists of the vertices of R     (valid if rok)
    const uint32_t *LL, *LS;   // lists of the vertices of L_a   (valid if lok)
    bool rok, lok;
    const uint32_t *FR, *FL;   // membership filters of R and L_a
};
__device__ __forceinline__ List list_at(const Dev &g, const uint32_t *V, int q, const uint32_t *B, const uint32_t *S,
                                        bool ok) {
    if (ok) return List{B + S[q], (int)(S[q + 1] - S[q])};
    return glist(g, V[q] >> 2);
}

// Phase A of a task: scatter code(a, x) for x in R into Ba; collect L_a (sorted) into La.
// al = a's list.  Run by one warp.  Returns |L_a|.
__device__ int build_a(uint32_t r, List al, const uint32_t *R, int D, uint32_t *Ba, uint32_t *La, int lane,
                       const uint32_t *FR, const RIndex *ix = nullptr) {
    int nL = 0;
    for (int base = 0; base < al.len; base += 32) {
        const int p = base + lane;
        bool keep = false;
        uint32_t e = 0;
        if (p < al.len) {
            e = al.p[p];
            const uint32_t x = e >> 2;
            if (x > r) {
                const int pos = ix ? find_pos(R, D, x, *ix) : (fmay(FR, x) ? find_rank(R, D, x) : -1);
                if (pos >= 0) set2(Ba, pos, e & 3u);
                else keep = true;
            }
        }
        const unsigned bal = __ballot_sync(kFull, keep);
        if (keep) La[nL + __popc(bal & ((1u << lane) - 1u))] = e;
        nL += __popc(bal);
    }
    __syncwarp();
    return nL;
}

// Phase A of a heavy task, by the whole CTA: a's list in 32-entry groups, warp w takes groups
// w, w + NW, ...  Pass 1 scatters code(a, x), x in R, into Ba and records per group the ballot
// of its L_a entries; warp 0 scans the group counts; pass 2 writes La (sorted: list order).
// tmp: 2 * ceil(len / 32) words of scratch.  *s_nL = |L_a|.  Ends with a barrier.
template <int NW>
__device__ void build_a_cta(uint32_t r, List al, const uint32_t *R, int D, uint32_t *Ba, uint32_t *La, uint32_t *tmp,
                            int *s_nL, int wid, int lane, const RIndex &ix) {
    const int G = (al.len + 31) >> 5;
    uint32_t *KM = tmp, *KO = tmp + G;
    for (int gi = wid; gi < G; gi += NW) {
        const int p = gi * 32 + lane;
        bool keep = false;
        if (p < al.len) {
            const uint32_t e = al.p[p], x = e >> 2;
            if (x > r) {
                const int pos = find_pos(R, D, x, ix);
                if (pos >= 0) set2(Ba, pos, e & 3u);
                else keep = true;
            }
        }
        const unsigned km = __ballot_sync(kFull, keep);
        if (lane == 0) KM[gi] = km;
    }
    __syncthreads();
    if (wid == 0) {
        int bk = 0;
        for (int g0 = 0; g0 < G; g0 += 32) {
            const int gi = g0 + lane;
            const int ck = gi < G ? __popc(KM[gi]) : 0;
            int ik = ck;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int yk = __shfl_up_sync(kFull, ik, d);
                if (lane >= d) ik += yk;
            }
            if (gi < G) KO[gi] = (uint32_t)(bk + ik - ck);
            bk += __shfl_sync(kFull, ik, 31);
        }
        if (lane == 0) *s_nL = bk;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    for (int gi = wid; gi < G; gi += NW) {
        const unsigned km = KM[gi];
        if (km >> lane & 1u) La[KO[gi] + __popc(km & lt)] = al.p[gi * 32 + lane];
    }
    __syncthreads();
}

// ------------------------------------------------------------------ shape "3" at heavy roots
// Task (r, a = R[i]); the star sets are {r, a, b = R[j], c = R[p]} with i < j < p.  A chunk
// is W = 32 * kStarM consecutive c positions [cb, ce) (lane l, slot t owns p = cb + 32 t + l);
// the warp walks b = R[j] for j in (i, ce) uniformly, one iteration = the chunk's sets with
// that b.  Per iteration the warp reads R[j] (rank(b) << 2 | code(r, b)); code(a, b) comes
// from codes[j] and code(b, c) from the root's induced adjacency in position space (pre-pass
// k_nr) through a per-c pointer.  A set is "plain" when code(a, b) = code(b, c) = 0 (almost
// every set at a hub: the induced graph of N+(r) has density ~2e-4 in cfg4); its mask, hence
// its class, is then fixed by c's key (code(r, c), code(a, c)) and the iteration's code(r, b):
//   * c side: the plain sets of every c with p > j get +1 in the field code(r, b) of a
//     warp-uniform packed counter U (one add per iteration for the whole chunk); c takes its
//     value when the walk reaches p (snapshot: U counts exactly the b before c), corrected by
//     the per-c deltas of its non-plain sets;
//   * b side: the key lanes (0..11) hold the number of chunk c's after b with their key and
//     add it, in the class lut[key | code(r, b)], to b's row: one atomic per key present;
//   * events (an a-b edge: every set of that b; a b-c edge: that c's set) are classified one
//     by one through the LUT entry of their full mask (star_event).
// Every set is counted once, in the class of its exact mask.  A work item is a chunk x a block
// of at most `fold` (<= 1023: 10-bit fields) consecutive b positions: items of bounded length
// balance a task's warps; at a block's end the c's still ahead take U and every c flushes.
// Counts are packed in 10-bit fields (inc_of), so a block spans at most kMaxBlock = 1023 b's.
constexpr int kStarM = 4;                  // c slots per lane
constexpr int kStarW = 32 * kStarM;        // c positions per star chunk
constexpr uint32_t kInfPos = 0x3fffffffu;

// row offset of vertex v's column col in the accumulator (32-bit when n*C < 2^32)
template <int C, bool OFF32>
__device__ __forceinline__ AccT *acc_at(const Dev &g, uint32_t v, uint32_t col) {
    if (OFF32) return g.acc + (col * g.ns + v);
    return g.acc + ((size_t)col * g.ns + v);
}


// one set in the 10-bit field of code(r, b) in {1, 2, 3}; a block spans <= 1023 b's, so no field
// overflows, and packed corrections (U + d) are exact field by field (final fields in [0, 1023])
__device__ __forceinline__ uint32_t inc_of(uint32_t crb) { return 1u << (crb * 10u - 10u); }
constexpr int kMaxBlock = 1023;   // (enumerated path: star_block <= kMaxBlock, checked by the API)

// c at position p: next entry of its induced list after index q with position < p, else INF
__device__ __forceinline__ void nr_next(const Dev &g, int64_t seg, int p, uint32_t &q, uint32_t &npos) {
    q++;
    npos = kInfPos;
    if ((int64_t)q < g.nr_off[seg + p + 1]) {
        const uint32_t x = g.nr_adj[q] >> 2;
        if ((int)x < p) npos = x;
    }
}

struct StarS {
    uint32_t d[kStarM];                // per c: packed count deltas, then (after its snapshot) its counts
    uint32_t npos[kStarM], q[kStarM];  // next event position of c, index of that induced entry
    uint32_t keys;                     // 4 bits per slot: code(r,c) - 1 + 3 code(a,c); 15 = no c
    uint32_t U;                        // warp-uniform plain counts, 10-bit fields: n(crb=1) | n(crb=2) << 10 | n(crb=3) << 20
    unsigned cntk;                     // key lanes: chunk c's after the current b with this lane's key
    uint32_t cols;                     // key lanes: column of (key | code(r,b)) in byte code(r,b)
};

template <int C>
__device__ __forceinline__ void star_flush_c(const Dev &g, const uint8_t *lut, uint32_t *H, uint32_t cra, uint32_t c,
                                             uint32_t key, uint32_t f) {
    const uint32_t lmask = cra | ((key % 3u) + 1u) << 4 | (key / 3u) << 8;
    const uint32_t n[3] = {f & 0x3ffu, (f >> 10) & 0x3ffu, f >> 20};
#pragma unroll
    for (uint32_t crb = 1; crb <= 3; crb++) {
        if (n[crb - 1]) {
            const int col = lut[lmask | crb << 2];
            acc_add(accp(g, c, col), n[crb - 1]);
            atomicAdd(H + col, n[crb - 1]);
        }
    }
}

// the c at position j (>= cb) takes its snapshot; its key lane stops counting it for b's
__device__ __forceinline__ void star_snapshot(StarS &s, int j, int cb, int lane) {
    const int o = j - cb, owner = o & 31, ts = o >> 5;
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        if (t == ts) {
            if (lane == owner) s.d[t] += s.U;
            const uint32_t kk = __shfl_sync(kFull, (s.keys >> (4 * t)) & 15u, owner);
            if ((uint32_t)lane == kk) s.cntk--;
        }
    }
}

// iteration j with an event: an a-b edge (every set of b is classified alone) and/or b-c
// edges (those c's sets are classified alone); the rest are plain
template <int C>
__device__ __forceinline__ void star_event(const Dev &g, const uint8_t *lut, uint32_t *H, uint32_t cra,
                                           const uint32_t *R, const uint8_t *codes, int64_t seg, StarS &s, int j,
                                           int cb, int ce, int lane) {
    if (j >= cb) star_snapshot(s, j, cb, lane);
    const uint32_t e = R[j], crb = e & 3u, b = e >> 2;
    const uint32_t cab = (uint32_t)codes[j] >> 2;
    const bool aev = cab != 0u;
    unsigned nh = 0;   // key lanes: plain-count correction (hit c's with this key)
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        const int p = cb + 32 * t + lane;
        const bool valid = p < ce && p > j;
        const bool hit = valid && s.npos[t] == (uint32_t)j;
        const bool slow = valid && (aev || hit);
        const uint32_t key = (s.keys >> (4 * t)) & 15u;
        int col = kNone;
        if (slow) {
            const uint32_t cbc = hit ? swap2(g.nr_adj[s.q[t]] & 3u) : 0u;   // the entry holds code(c, b)
            const uint32_t lmask = cra | ((key % 3u) + 1u) << 4 | (key / 3u) << 8;
            col = lut[lmask | crb << 2 | cab << 6 | cbc << 10];
            acc_add(accp(g, R[p] >> 2, col), 1u);
            atomicAdd(H + col, 1u);
            if (!aev) s.d[t] -= inc_of(crb);   // U will count this j for every c: take it back for this one
        }
        const unsigned m = __match_any_sync(kFull, col);
        if (col != kNone && lane == __ffs(m) - 1) acc_add(accp(g, b, col), __popc(m));
        if (!aev) {
            for (unsigned hm = __ballot_sync(kFull, hit); hm; hm &= hm - 1) {
                const uint32_t kk = __shfl_sync(kFull, key, __ffs(hm) - 1);
                if ((uint32_t)lane == kk) nh++;
            }
        }
        if (hit) nr_next(g, seg, p, s.q[t], s.npos[t]);
    }
    if (!aev) {
        s.U += inc_of(crb);
        const unsigned cnt = s.cntk - nh;
        if (cnt) acc_add(accp(g, b, ((s.cols >> (crb << 3)) & 0xffu)), cnt);
    }
}

// event-free iterations [j0, j1): U counts, key lanes add to b's row; TAIL: snapshots
template <int C, bool OFF32, bool TAIL>
__device__ __forceinline__ void star_fast(const Dev &g, const uint32_t *R, StarS &s, int j0, int j1, int cb,
                                          int lane) {
    if (!TAIL) {
#pragma unroll 4
        for (int j = j0; j < j1; j++) {
            const uint32_t e = R[j];   // rank(b) << 2 | code(r, b)
            const uint32_t crb = e & 3u;
            s.U += inc_of(crb);
            red_if(s.cntk != 0u, acc_at<C, OFF32>(g, e >> 2, (s.cols >> (crb << 3)) & 0xffu), s.cntk);
        }
    } else {
#pragma unroll
        for (int t = 0; t < kStarM; t++) {
            const int a0 = max(j0, cb + 32 * t), a1 = min(j1, cb + 32 * t + 32);
            const uint32_t kt = (s.keys >> (4 * t)) & 15u;
            for (int j = a0; j < a1; j++) {
                const int owner = j - cb - 32 * t;
                if (lane == owner) s.d[t] += s.U;
                if ((uint32_t)lane == __shfl_sync(kFull, kt, owner)) s.cntk--;
                const uint32_t e = R[j];
                const uint32_t crb = e & 3u;
                s.U += inc_of(crb);
                red_if(s.cntk != 0u, acc_at<C, OFF32>(g, e >> 2, (s.cols >> (crb << 3)) & 0xffu), s.cntk);
            }
        }
    }
}

template <int C>
__device__ __forceinline__ void star_fast_any(const Dev &g, const uint32_t *R, StarS &s, int j0, int j1, int cb,
                                              int lane) {
    const int f1 = min(j1, cb);
    if (j0 < f1) {
        if (g.off32) star_fast<C, true, false>(g, R, s, j0, f1, cb, lane);
        else star_fast<C, false, false>(g, R, s, j0, f1, cb, lane);
    }
    const int t0 = max(j0, cb);
    if (t0 < j1) {
        if (g.off32) star_fast<C, true, true>(g, R, s, t0, j1, cb, lane);
        else star_fast<C, false, true>(g, R, s, t0, j1, cb, lane);
    }
}

// one set with members r, a (histogram H), b (per lane: the owner of the walked entry) and c (lane):
// b-side atomics merged over the lanes with the same (owner, column)
template <int C>
__device__ __forceinline__ void emit4v(uint32_t *H, const Dev &g, uint32_t b, int owner, uint32_t c, int col,
                                       int lane) {
    const bool v = col != kNone;
    const uint32_t cc = v ? (uint32_t)col : 0u;
    red_if(v, accp(g, c, cc), 1u);
    const unsigned m = __match_any_sync(kFull, v ? ((uint32_t)owner << 8 | cc) : 0xffffffffu);
    const bool lead = v && lane == __ffs(m) - 1;
    const uint32_t cnt = __popc(m);
    red_shared_if(lead, H + cc, cnt);
    red_if(lead, accp(g, b, cc), cnt);
}

// Flattened walk over the staged lists q in [q0, q1) (pool entries [S[q0], S[q1]), every list
// non-empty): 32 consecutive entries per pass whatever the list lengths, so short lists do not
// leave lanes idle.  The owner of entry f is q0 + #{q in (q0, q1) : S[q] <= f}: per pass the
// lanes load the next 32 list starts, and a bitmap of the starts inside (base, base + 32] gives
// each lane its owner with one popc.  fn(owner, entry, valid) is called by every lane.
template <typename Fn>
__device__ __forceinline__ void flat_walk(const uint32_t *pool, const uint32_t *S, int q0, int q1, int lane, Fn fn) {
    const int f1 = (int)S[q1];
    int o = q0;
    for (int base = (int)S[q0]; base < f1; base += 32) {
        const int qb = o + 1 + lane;
        const int d = qb < q1 ? (int)S[qb] - base : 64;   // start of list qb, relative to base
        const unsigned B = __reduce_or_sync(kFull, d >= 1 && d <= 32 ? 1u << (d - 1) : 0u);
        const int owner = o + __popc(B & ((1u << lane) - 1u));
        const int f = base + lane;
        const bool valid = f < f1;
        fn(owner, valid ? pool[f] : 0u, valid);
        o += __popc(B);
    }
}

// ------------------------------------- shapes "3" and "2+1" at heavy roots, counted in closed form
// Task (r, x = R[i]), Y = code(r, x).  The key of a position q != i is codes[q] = x_q | al_q << 2
// with x_q = code(r, R[q]) and al_q = code(x, R[q]); N[k] = #{q > i : key k}, N[16 + k] =
// #{q < i : key k} (counted when codes[] is built), M[w] = #{c in L_x : code(x, c) = w}.
//
// "3" = {r, x, R[j], R[p]}, i < j < p.  A pair (j, p) with no R[j]-R[p] edge has the mask
// Y | x_j << 2 | x_p << 4 | al_j << 6 | al_p << 8: its class cls(k_j, k_p) depends on the two keys
// only and is symmetric in them (exchanging the roles of b and c relabels the same digraph; the
// LUT gives the minimum isomorph).  So
//   * R[q] (q > i) lies in N[k'] - [k_q = k'] - #{induced neighbours of R[q] beyond i with key k'}
//     such sets of class cls(k_q, k') -- one atomic per key present;
//   * r and x lie in N[k] N[k'] (k < k') or C(N[k], 2) (k = k') sets of class cls(k, k');
//   * a pair with an R[j]-R[p] edge (an entry of the root's induced adjacency, k_nr) is an event:
//     classified alone by its full mask (code(R[j], R[p]) in bits 10-11) and taken back from its
//     plain class.
// "2+1" with x as a depth-1 vertex (the partition of the enumerated cross items):
//   PART 1, j > i: {r, a = x, b = R[j], c}, c in L_x, every j:  mask Y | x_j << 2 | al_j << 6 |
//                  w_c << 8 | code(R[j], c) << 10
//   PART 2, j < i: {r, a = R[j], b = x, c}, c in L_x, c not adjacent to R[j]:  mask x_j | Y << 2 |
//                  swap(al_j) << 6 | w_c << 10
// With no R[j]-c edge the class depends on (k_j, w_c, part) only: c lies in N[k] (part 1) /
// N[16 + k] (part 2) sets per key, R[j] in M[w] sets per w, r and x in M[w] N[..k] sets; every
// R[j]-c edge (walked from c's list) is an event of part 1 (classified alone) or removes a part-2
// set, and is taken back from the plain counts.
// The induced graph of N+(r) is sparse (cfg4: 51K edges over all 6585 heavy roots), so a task
// costs O(D + sum of |N(c)| over c in L_x) plus its events instead of O((D - i)^2 + |L_x| D) set
// visits; every set is still counted once, in the class of its exact mask.
// Take-backs make some partial sums negative: the r / x side of the events and take-backs goes to
// the per-CTA histogram Hs of modular 64-bit words, flushed once per task (closed_root).
constexpr int kSPM = 2;                 // positions per lane in one closed-form item
constexpr int kSPW = 32 * kSPM;

__device__ __forceinline__ void hs_add(unsigned long long *Hs, uint32_t col, long long v) {
    atomicAdd(Hs + col, (unsigned long long)v);
}
__device__ __forceinline__ uint32_t star_mask(uint32_t cra, uint32_t kb, uint32_t kc) {   // plain "3" mask
    return cra | (kb & 3u) << 2 | (kc & 3u) << 4 | (kb >> 2) << 6 | (kc >> 2) << 8;
}
__device__ __forceinline__ uint32_t p1_mask(uint32_t cra, uint32_t kj, uint32_t w) {   // plain "2+1" part 1
    return cra | (kj & 3u) << 2 | (kj >> 2) << 6 | w << 8;
}
__device__ __forceinline__ uint32_t p2_mask(uint32_t cra, uint32_t kj, uint32_t w) {   // plain "2+1" part 2
    return (kj & 3u) | cra << 2 | swap2(kj >> 2) << 6 | w << 10;
}

// "3": positions [q0, q0 + kSPW) beyond i, one per lane
template <int C>
__device__ __forceinline__ void star_closed_item(const Dev &g, const uint8_t *lut, unsigned long long *Hs,
                                                 uint32_t cra, int i, const uint32_t *R, int D,
                                                 const uint8_t *codes, const int *sN, uint32_t P, int64_t seg,
                                                 int q0, int lane, const uint32_t *NB) {
#pragma unroll 1
    for (int t = 0; t < kSPM; t++) {
        const int q = q0 + 32 * t + lane;
        if (q >= D) break;   // no warp-collective operations below
        const uint32_t v = R[q] >> 2, kq = codes[q];
        uint64_t corr = 0;   // induced neighbours beyond i with keys 1..3 (al = 0), 21-bit fields
        const bool has = (NB[q >> 5] >> (q & 31)) & 1u;   // most positions have none: no list bounds read
        int64_t e = has ? g.nr_off[seg + q] : 0;
        const int64_t e1 = has ? g.nr_off[seg + q + 1] : 0;
        if (e1 - e > 16) {   // first entry with position > i (the list ascends in position)
            int64_t lo = e, hi = e1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if ((int)(g.nr_adj[mid] >> 2) <= i) lo = mid + 1;
                else hi = mid;
            }
            e = lo;
        }
        for (; e < e1; e++) {
            const uint32_t en = g.nr_adj[e];
            const int p = (int)(en >> 2);
            if (p <= i) continue;
            const uint32_t kp = codes[p];
            const uint32_t mp = star_mask(cra, kq, kp);
            if (kp < 4u) corr += 1ull << (21u * (kp - 1u));
            else acc_addw(accp(g, v, lut[mp]), (AccT)0 - (AccT)1);   // not plain: taken back from below
            if (p > q) {   // the event {r, x, R[q], R[p]}, R[q] in the b slots
                const uint32_t col = lut[mp | (en & 3u) << 10], pl = lut[mp];
                acc_add(accp(g, v, col), 1u);
                acc_add(accp(g, R[p] >> 2, col), 1u);   // (R[p]'s own walk takes it back from its plain sets)
                hs_add(Hs, col, 1);
                hs_add(Hs, pl, -1);
            }
        }
        for (uint32_t m = P; m; m &= m - 1u) {   // plain sets of R[q], per partner key
            const uint32_t k = (uint32_t)__ffs(m) - 1u;
            uint32_t cnt = (uint32_t)sN[k] - (k == kq ? 1u : 0u);
            if (k < 4u) cnt -= (uint32_t)(corr >> (21u * (k - 1u))) & 0x1fffffu;
            if (cnt) acc_add(accp(g, v, lut[star_mask(cra, kq, k)]), cnt);
        }
    }
}

// "2+1", the R[j] side: positions j in [q0, q0 + kSPW), j != i, one per lane: M[w] sets per w
template <int C>
__device__ __forceinline__ void cross_j_closed(const Dev &g, const uint8_t *lut, uint32_t cra, int i,
                                               const uint32_t *R, int D, const uint8_t *codes, const int *sM,
                                               int q0, int lane) {
#pragma unroll 1
    for (int t = 0; t < kSPM; t++) {
        const int j = q0 + 32 * t + lane;
        if (j >= D) break;
        if (j == i) continue;
        const uint32_t y = R[j] >> 2, kj = codes[j];
#pragma unroll
        for (uint32_t w = 1; w <= 3; w++) {
            const uint32_t mw = (uint32_t)sM[w];
            if (mw) acc_add(accp(g, y, lut[j > i ? p1_mask(cra, kj, w) : p2_mask(cra, kj, w)]), mw);
        }
    }
}

// u = L_x[q] (one warp, one walk of u's list) for every shape with a depth-2 vertex:
//   * u as c of "2+1": an entry y = R[j] (j != i) is a part-1 event (j > i: classified alone) or
//     a part-2 removal (j < i: the set belongs to R[j]'s task), both taken back from the plain
//     counts; afterwards u's plain "2+1" sets per (part, key), lane l = (l >> 4, l & 15);
//   * u as b of "1+2" / "1+1+1": an entry y in L_x after u is a "1+2" event (classified alone,
//     taken back); an entry y outside N[r] u N[x], y > r, is a "1+1+1" set {r, x, u, y}, enumerated
//     one per lane; afterwards u's plain "1+2" sets per partner code w2.
// y = x (always in u's list) is in R and tested first, so that the lane holding it does not send
// the whole warp through the binary search.
template <int C>
__device__ __forceinline__ void u_closed(const Dev &g, const uint8_t *lut, unsigned long long *Hs, uint32_t *H,
                                         uint32_t r, uint32_t x, uint32_t cra, int i, const uint32_t *R, int D,
                                         const uint8_t *codes, const uint32_t *La, int nL, const int *sN,
                                         const int *sM, int q, int lane, const RIndex &ix) {
    const uint32_t eu = La[q], u = eu >> 2, w = eu & 3u;
    const uint32_t mb = cra | w << 6;   // u in the b slots of "1+2" / "1+1+1": (a, b) = code(x, u)
    const int64_t u0 = g.off[u], u1 = g.off[u + 1];
    for (int64_t base = u0; base < u1; base += 32 * kPF) {
        uint32_t ev[kPF];
#pragma unroll
        for (int t = 0; t < kPF; t++) {
            const int64_t p = base + 32 * t + lane;
            ev[t] = p < u1 ? g.adj[p] : 0u;
        }
#pragma unroll
        for (int t = 0; t < kPF; t++) {
            if (base + 32 * t >= u1) break;
            const uint32_t e = ev[t], y = e >> 2;
            int col = kNone;
            uint32_t cy = 0;
            if (base + 32 * t + lane < u1 && y > r && y != x) {
                const int pos = find_pos(R, D, y, ix);
                if (pos >= 0) {
                    const uint32_t kj = codes[pos];
                    if (pos > i) {   // part-1 event: code(R[j], u) = swap(code(u, R[j]))
                        const uint32_t mp = p1_mask(cra, kj, w);
                        const uint32_t ce = lut[mp | swap2(e & 3u) << 10], pl = lut[mp];
                        acc_add(accp(g, u, ce), 1u);
                        acc_add(accp(g, y, ce), 1u);
                        acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                        acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                        hs_add(Hs, ce, 1);
                        hs_add(Hs, pl, -1);
                    } else {         // part 2: u ~ R[j], the set belongs to R[j]'s task
                        const uint32_t pl = lut[p2_mask(cra, kj, w)];
                        acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                        acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                        hs_add(Hs, pl, -1);
                    }
                } else {
                    const int qq = find_rank(La, nL, y);
                    if (qq >= 0) {
                        if (qq > q) {   // "1+2" {r, x, u, y} with a u-y edge: event
                            const uint32_t mp = mb | (La[qq] & 3u) << 8;
                            const uint32_t ce = lut[mp | (e & 3u) << 10], pl = lut[mp];
                            acc_add(accp(g, u, ce), 1u);
                            acc_add(accp(g, y, ce), 1u);
                            acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                            acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                            hs_add(Hs, ce, 1);
                            hs_add(Hs, pl, -1);
                        }
                    } else {
                        col = lut[mb | (e & 3u) << 10];   // "1+1+1" {r, x, u, y}
                        cy = y;
                    }
                }
            }
            emit4<C>(H, g, u, cy, col, lane);
        }
    }
    const uint32_t k = (uint32_t)lane & 15u;
    const int n = sN[lane];
    if (n > 0 && (k & 3u)) acc_add(accp(g, u, lut[lane < 16 ? p1_mask(cra, k, w) : p2_mask(cra, k, w)]), (uint32_t)n);
    if (lane >= 1 && lane <= 3) {
        const uint32_t w2 = (uint32_t)lane, cnt = (uint32_t)sM[w2] - (w2 == w ? 1u : 0u);
        if (cnt) acc_add(accp(g, u, lut[cra | w << 6 | w2 << 8]), cnt);
    }
}

// r and x: the plain sets of every key pair ("3"), of every (key, w, part) ("2+1") and of every
// code pair (w1, w2) ("1+2"), and the per-CTA take-back histogram; once per task, after the
// items (threads tid < 256 / 96 / 96..111 / C)
template <int C>
__device__ __forceinline__ void closed_root(const Dev &g, const uint8_t *lut, uint32_t r, uint32_t x, uint32_t cra,
                                            const int *sN, const int *sM, unsigned long long *Hs, int tid) {
    if (tid < 256) {
        const uint32_t k1 = (uint32_t)tid >> 4, k2 = (uint32_t)tid & 15u;
        if (k1 <= k2 && (k1 & 3u) && (k2 & 3u)) {
            const uint64_t n1 = (uint64_t)sN[k1], n2 = (uint64_t)sN[k2];
            const uint64_t pairs = k1 < k2 ? n1 * n2 : n1 * (n1 - (n1 > 0)) / 2;
            if (pairs) {
                const uint32_t col = lut[star_mask(cra, k1, k2)];
                acc_addw(accp(g, r, col), (AccT)pairs);
                acc_addw(accp(g, x, col), (AccT)pairs);
            }
        }
    }
    if (tid < 96) {
        const int part = tid / 48, rest = tid % 48;
        const uint32_t k = (uint32_t)rest / 3u, w = (uint32_t)rest % 3u + 1u;
        const uint64_t n = (uint64_t)sN[16 * part + (int)k] * (uint64_t)sM[w];
        if (n && (k & 3u)) {
            const uint32_t col = lut[part == 0 ? p1_mask(cra, k, w) : p2_mask(cra, k, w)];
            acc_addw(accp(g, r, col), (AccT)n);
            acc_addw(accp(g, x, col), (AccT)n);
        }
    }
    if (tid >= 96 && tid < 112) {   // "1+2": pairs of L_x per (w1 <= w2)
        const uint32_t w1 = (uint32_t)(tid - 96) >> 2, w2 = (uint32_t)(tid - 96) & 3u;
        if (w1 >= 1 && w1 <= w2 && w2 <= 3) {
            const uint64_t m1 = (uint64_t)sM[w1], m2 = (uint64_t)sM[w2];
            const uint64_t n = w1 < w2 ? m1 * m2 : m1 * (m1 - (m1 > 0)) / 2;
            if (n) {
                const uint32_t col = lut[cra | w1 << 6 | w2 << 8];
                acc_addw(accp(g, r, col), (AccT)n);
                acc_addw(accp(g, x, col), (AccT)n);
            }
        }
    }
    if (tid < C) {
        const unsigned long long h = Hs[tid];
        if (h) {
            acc_addw(accp(g, r, tid), (AccT)h);
            acc_addw(accp(g, x, tid), (AccT)h);
            Hs[tid] = 0;
        }
    }
}

// first j' in [j, jend) with an a-b edge (codes[j'] >= 4), else jend
__device__ __forceinline__ int next_a_event(const uint8_t *codes, int j, int jend, int lane) {
    for (int base = j; base < jend; base += 32) {
        const int p = base + lane;
        const unsigned m = __ballot_sync(kFull, p < jend && codes[p] >= 4);
        if (m) return base + __ffs(m) - 1;
    }
    return jend;
}

// star item (k, jb) of the task (r, a = R[i]): c positions [cb, ce) = [max(D - W(k+1), i+2), D - W k)
// (chunk k), b positions [jlo, jhi) = block jb of [i+1, ce) in steps of fold
__device__ __forceinline__ int star_blocks(int D, int i, int k, int S) {
    const int ce = D - kStarW * k;
    return (ce - i - 1 + S - 1) / S;
}

template <int C>
__device__ __forceinline__ void star_item(const Dev &g, const uint8_t *lut, uint32_t r, int i, const uint32_t *R,
                                          int D, const uint32_t *Ba, const uint8_t *codes, uint32_t cra, uint32_t a,
                                          uint32_t *H, int k, int jb, int fold, int lane) {
    const int64_t seg = g.hbase[r];
    const int ce = D - kStarW * k, cb = max(ce - kStarW, i + 2);
    const int jlo = i + 1 + jb * fold, jhi = min(ce, jlo + fold);
    StarS s;
    s.keys = 0;
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        const int p = cb + 32 * t + lane;
        s.d[t] = 0;
        s.npos[t] = kInfPos;
        s.q[t] = 0;
        uint32_t key = 15u;
        if (p < ce && p >= jlo) {   // c's before the block were completed by earlier blocks
            const uint32_t ec = R[p];
            key = (ec & 3u) - 1u + 3u * get2(Ba, p);
            s.q[t] = (uint32_t)g.nr_off[seg + p] - 1u;
            do nr_next(g, seg, p, s.q[t], s.npos[t]);   // first induced neighbour in the block
            while (s.npos[t] < (uint32_t)jlo);
        }
        s.keys |= key << (4 * t);
    }
    s.cntk = 0;
#pragma unroll
    for (uint32_t q = 0; q < 12; q++) {
        unsigned cnt = 0;
#pragma unroll
        for (int t = 0; t < kStarM; t++) cnt += __popc(__ballot_sync(kFull, ((s.keys >> (4 * t)) & 15u) == q));
        if ((uint32_t)lane == q) s.cntk = cnt;
    }
    s.cols = 0;
    if (s.cntk) {
        const uint32_t kmask = cra | ((uint32_t)(lane % 3) + 1u) << 4 | ((uint32_t)(lane / 3) & 3u) << 8;
        s.cols = (uint32_t)lut[kmask | 1u << 2] << 8 | (uint32_t)lut[kmask | 2u << 2] << 16 |
                 (uint32_t)lut[kmask | 3u << 2] << 24;
    }
    s.U = 0;
    int j = jlo;
    int anext = next_a_event(codes, j, jhi, lane);
    while (j < jhi) {
        uint32_t cm = s.npos[0];
#pragma unroll
        for (int t = 1; t < kStarM; t++) cm = min(cm, s.npos[t]);
        const int cev = (int)min(__reduce_min_sync(kFull, cm), kInfPos);
        const int stop = min(jhi, min(anext, cev));
        star_fast_any<C>(g, R, s, j, stop, cb, lane);
        j = stop;
        if (j >= jhi) break;
        star_event<C>(g, lut, H, cra, R, codes, seg, s, j, cb, ce, lane);
        j++;
        if (anext < j) anext = next_a_event(codes, j, jhi, lane);
    }
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        const int p = cb + 32 * t + lane;
        if (p < ce && p >= jlo) {
            if (p >= jhi) s.d[t] += s.U;   // still ahead of the walk: every b of the block precedes it
            star_flush_c<C>(g, lut, H, cra, R[p] >> 2, (s.keys >> (4 * t)) & 15u, s.d[t]);
        }
    }
    if (g.big) flush_hist<C>(H, g, r, a, lane);
    __syncwarp();
}

// b = R[j] (k = 4): walk N(b) once -- c in R after b -> Bb (light tasks only; heavy tasks run
// star_chunk), c in L_a -> Bl, else a "2+1" set with c in L_b \ N(a); then "3" over R (light)
// and "2+1" over L_a.
template <int C, int NW>
__device__ __forceinline__ void item_b_in_R(const Dev &g, const uint8_t *lut, uint32_t r, int i, int j,
                                            const uint32_t *R, int D, const uint32_t *Ba, const uint32_t *La, int nL,
                                            uint32_t *Bb, uint32_t *Bl, uint32_t *H, uint32_t cra, uint32_t a,
                                            List bl, int lane, const uint32_t *FR = nullptr,
                                            const uint32_t *FL = nullptr) {
    const uint32_t eb = R[j], b = eb >> 2;
    const uint32_t mb = cra | (eb & 3u) << 2 | get2(Ba, j) << 6;
    bool tb = false, tl = false;   // this lane set a code in Bb / Bl
    for (int base = 0; base < bl.len; base += 32 * kPF) {
        uint32_t ev[kPF];   // kPF loads in flight per lane (b's list is often in global memory)
#pragma unroll
        for (int u = 0; u < kPF; u++) {
            const int p = base + 32 * u + lane;
            ev[u] = p < bl.len ? bl.p[p] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPF; u++) {
            if (base + 32 * u >= bl.len) break;
            const uint32_t e = ev[u];
            int col = kNone;
            uint32_t c = 0;
            if (base + 32 * u + lane < bl.len) {
                c = e >> 2;
                if (c > r) {
                    const int pos = fmay(FR, c) ? find_rank(R, D, c) : -1;
                    if (pos >= 0) {
                        if (NW == 1 && pos > j) {
                            set2(Bb, pos, e & 3u);
                            tb = true;
                        }
                    } else {
                        const int q = fmay(FL, c) ? find_rank(La, nL, c) : -1;
                        if (q >= 0) {
                            set2(Bl, q, e & 3u);
                            tl = true;
                        } else {
                            col = lut[mb | (e & 3u) << 10];
                        }
                    }
                }
            }
            emit4<C>(H, g, b, c, col, lane);
        }
    }
    const bool anyb = __any_sync(kFull, tb), anyl = __any_sync(kFull, tl);
    // "3" (c in R after b; light tasks) and "2+1" (c in L_a) in one index space, so a warp
    // iteration is filled from both when they are short
    const int n3 = NW == 1 ? D - j - 1 : 0;
    for (int base = 0; base < n3 + nL; base += 32) {
        const int x = base + lane;
        int col = kNone;
        uint32_t c = 0;
        if (x < n3) {
            const int p = j + 1 + x;
            const uint32_t ec = R[p];
            c = ec >> 2;
            col = lut[mb | (ec & 3u) << 4 | get2(Ba, p) << 8 | get2(Bb, p) << 10];
        } else if (x < n3 + nL) {
            const int q = x - n3;
            const uint32_t ec = La[q];
            c = ec >> 2;
            col = lut[mb | (ec & 3u) << 8 | get2(Bl, q) << 10];
        }
        emit4<C>(H, g, b, c, col, lane);
    }
    __syncwarp();
    if (NW == 1 && anyb) clear_words(Bb, (j + 1) >> 4, (D + 15) >> 4, lane);
    if (anyl) clear_words(Bl, 0, (nL + 15) >> 4, lane);
    if (g.big) flush_hist<C>(H, g, r, a, lane);
    __syncwarp();
}

// b = L_a[x] (k = 4): walk N(b) once -- c in R -> skip, c in L_a after b -> Bl ("1+2"), else a
// "1+1+1" set; then "1+2" over L_a after b.
template <int C>
__device__ __forceinline__ void item_b_in_La(const Dev &g, const uint8_t *lut, uint32_t r, int x, const uint32_t *R,
                                             int D, const uint32_t *La, int nL, uint32_t *Bl, uint32_t *H,
                                             uint32_t cra, uint32_t a, List bl, int lane, const uint32_t *FR = nullptr,
                                             const uint32_t *FL = nullptr) {
    const uint32_t eb = La[x], b = eb >> 2;
    const uint32_t mb = cra | (eb & 3u) << 6;
    bool tl = false;
    for (int base = 0; base < bl.len; base += 32 * kPF) {
        uint32_t ev[kPF];
#pragma unroll
        for (int u = 0; u < kPF; u++) {
            const int p = base + 32 * u + lane;
            ev[u] = p < bl.len ? bl.p[p] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kPF; u++) {
            if (base + 32 * u >= bl.len) break;
            const uint32_t e = ev[u];
            int col = kNone;
            uint32_t c = 0;
            if (base + 32 * u + lane < bl.len) {
                c = e >> 2;
                if (c > r && c != a && (!fmay(FR, c) || find_rank(R, D, c) < 0)) {
                    const int q = fmay(FL, c) ? find_rank(La, nL, c) : -1;
                    if (q >= 0) {
                        if (q > x) {
                            set2(Bl, q, e & 3u);
                            tl = true;
                        }
                    } else {
                        col = lut[mb | (e & 3u) << 10];
                    }
                }
            }
            emit4<C>(H, g, b, c, col, lane);
        }
    }
    const bool anyl = __any_sync(kFull, tl);
    for (int base = x + 1; base < nL; base += 32) {
        const int q = base + lane;
        int col = kNone;
        uint32_t c = 0;
        if (q < nL) {
            const uint32_t ec = La[q];
            c = ec >> 2;
            col = lut[mb | (ec & 3u) << 8 | get2(Bl, q) << 10];
        }
        emit4<C>(H, g, b, c, col, lane);
    }
    __syncwarp();
    if (anyl) clear_words(Bl, (x + 1) >> 4, (nL + 15) >> 4, lane);
    if (g.big) flush_hist<C>(H, g, r, a, lane);
    __syncwarp();
}

// ------------------------------------------------------------------ "2+1" at heavy roots
// For the task (r, x = R[i]) both kinds of "2+1" set containing x are enumerated with lanes =
// c in L_x (kStarM per lane: 128-wide chunks of L_x) and a warp-uniform walk over positions j
// of R (one item = a chunk of c's x a block of kCrossBlock positions):
//   PART 2, j < i:  {r, a = R[j], b = x, c}, c in L_b \ N(a)   (only if R[j] is not adjacent to c)
//   PART 1, j > i:  {r, a = x, b = R[j], c}, c in L_a          (every j)
// Together these are exactly the "2+1" sets whose first or second depth-1 vertex is x, each
// once (the set {r, a < b, c} is met in the task of a if c ~ a, else in the task of b).
// code(R[j], c) comes from c's R-neighbour list, built per task in CTA scratch (ca_build).
// As in the star loop, a plain set (no x-R[j] edge and no R[j]-c edge) has its class fixed by
// c's key code(x, c) and the iteration's code(r, R[j]): every c counts it in the warp-uniform
// U, corrected per c at its events; R[j] gets, from key lanes 0..2, the number of the chunk's
// c's with that key; an x-R[j] edge makes every set of that j non-plain (classified alone), an
// R[j]-c edge makes c's PART 1 set non-plain and removes its PART 2 set (c is in N(a)).
constexpr int kCrossBlock = 256;    // default j-block length g.xblock (<= kMaxBlock: the 10-bit count fields)

// c's R-neighbour list pointer: next entry (position of R, code(c, R[pos])) with position < jend
__device__ __forceinline__ void ca_next(const uint32_t *CA, uint32_t q1, uint32_t &q, uint32_t &npos) {
    q++;
    npos = q < q1 ? CA[q] >> 2 : kInfPos;
}

template <int C, int PART>
__device__ __forceinline__ void cross_flush(const Dev &g, const uint8_t *lut, uint32_t *H, uint32_t cra,
                                            const uint32_t *La, int q0, int nL, StarS &s, int lane) {
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        const int q = q0 + 32 * t + lane;
        if (q < nL) {
            const uint32_t ec = La[q], c = ec >> 2, cxc = ec & 3u;
            const uint32_t f = s.d[t] + s.U;
            const uint32_t n[3] = {f & 0x3ffu, (f >> 10) & 0x3ffu, f >> 20};
#pragma unroll
            for (uint32_t crj = 1; crj <= 3; crj++) {
                if (n[crj - 1]) {
                    const int col = PART == 1 ? lut[cra | crj << 2 | cxc << 8] : lut[crj | cra << 2 | cxc << 10];
                    acc_add(accp(g, c, col), n[crj - 1]);
                    atomicAdd(H + col, n[crj - 1]);
                }
            }
        }
        s.d[t] = 0;
    }
    s.U = 0;
}

// positions [j0, j1) of one part (all c's of the chunk valid throughout)
template <int C, int PART>
__device__ __forceinline__ void cross_part(const Dev &g, const uint8_t *lut, uint32_t *H, uint32_t cra,
                                           const uint32_t *R, const uint8_t *codes, const uint32_t *La, int q0,
                                           int nL, const uint32_t *CAbeg, const uint32_t *CAlen, const uint32_t *CA,
                                           StarS &s, int j0, int j1, int lane) {
    if (j0 >= j1) return;
    const uint32_t kc = (uint32_t)lane + 1u;
    s.cols = 0;
    if (s.cntk) {
        s.cols = PART == 1 ? ((uint32_t)lut[cra | 1u << 2 | kc << 8] << 8 | (uint32_t)lut[cra | 2u << 2 | kc << 8] << 16 |
                              (uint32_t)lut[cra | 3u << 2 | kc << 8] << 24)
                           : ((uint32_t)lut[1u | cra << 2 | kc << 10] << 8 | (uint32_t)lut[2u | cra << 2 | kc << 10] << 16 |
                              (uint32_t)lut[3u | cra << 2 | kc << 10] << 24);
    }
    int j = j0;
    int anext = next_a_event(codes, j, j1, lane);
    while (j < j1) {
        uint32_t cm = s.npos[0];
#pragma unroll
        for (int t = 1; t < kStarM; t++) cm = min(cm, s.npos[t]);
        const int cev = (int)min(__reduce_min_sync(kFull, cm), kInfPos);
        const int stop = min(j1, min(anext, cev));
        if (j < stop) {
            if (g.off32) star_fast<C, true, false>(g, R, s, j, stop, 0, lane);
            else star_fast<C, false, false>(g, R, s, j, stop, 0, lane);
        }
        j = stop;
        if (j >= j1) break;
        // event at j
        const uint32_t e = R[j], crj = e & 3u, b = e >> 2;
        const uint32_t cxj = (uint32_t)codes[j] >> 2;   // code(x, R[j])
        const bool aev = cxj != 0u;
        unsigned nh = 0;
#pragma unroll
        for (int t = 0; t < kStarM; t++) {
            const int q = q0 + 32 * t + lane;
            const bool valid = q < nL;
            const bool hit = valid && s.npos[t] == (uint32_t)j;
            int col = kNone;
            uint32_t c = 0;
            const bool slow = PART == 1 ? valid && (aev || hit) : valid && aev && !hit;
            if (slow) {
                const uint32_t ec = La[q], cxc = ec & 3u;
                c = ec >> 2;
                if (PART == 1) {
                    const uint32_t cjc = hit ? swap2(CA[s.q[t]] & 3u) : 0u;   // the entry holds code(c, R[j])
                    col = lut[cra | crj << 2 | cxj << 6 | cxc << 8 | cjc << 10];
                } else {
                    col = lut[crj | cra << 2 | swap2(cxj) << 6 | cxc << 10];
                }
                acc_add(accp(g, c, col), 1u);
                atomicAdd(H + col, 1u);
            }
            if (hit && !aev) s.d[t] -= inc_of(crj);   // U will count this j for every c: take it back
            const unsigned m = __match_any_sync(kFull, col);
            if (col != kNone && lane == __ffs(m) - 1) acc_add(accp(g, b, col), __popc(m));
            if (!aev) {
                const uint32_t key = valid ? (La[q] & 3u) - 1u : 15u;
                for (unsigned hm = __ballot_sync(kFull, hit); hm; hm &= hm - 1) {
                    const uint32_t kk = __shfl_sync(kFull, key, __ffs(hm) - 1);
                    if ((uint32_t)lane == kk) nh++;
                }
            }
            if (hit) ca_next(CA, CAbeg[q] + CAlen[q], s.q[t], s.npos[t]);
        }
        if (!aev) {
            s.U += inc_of(crj);
            const unsigned cnt = s.cntk - nh;
            if (cnt) acc_add(accp(g, b, ((s.cols >> (crj << 3)) & 0xffu)), cnt);
        }
        j++;
        if (anext < j) anext = next_a_event(codes, j, j1, lane);
    }
    cross_flush<C, PART>(g, lut, H, cra, La, q0, nL, s, lane);
}

// item (k, jb): c = L_x[128k .. 128k+127], positions j in block jb of length kCrossBlock
template <int C>
__device__ __forceinline__ void cross_item(const Dev &g, const uint8_t *lut, uint32_t r, int i, const uint32_t *R,
                                           int D, const uint8_t *codes, const uint32_t *La, int nL,
                                           const uint32_t *CAbeg, const uint32_t *CAlen, const uint32_t *CA,
                                           uint32_t cra, uint32_t a, uint32_t *H, int k, int jb, int lane) {
    const int j0 = jb * g.xblock, j1 = min(D, j0 + g.xblock);
    const int q0 = kStarW * k;
    StarS s;
    s.keys = 0;
#pragma unroll
    for (int t = 0; t < kStarM; t++) {
        const int q = q0 + 32 * t + lane;
        s.d[t] = 0;
        s.npos[t] = kInfPos;
        s.q[t] = 0;
        if (q < nL) {   // pointer to c's first R-neighbour at or after j0
            const uint32_t q1 = CAbeg[q] + CAlen[q];
            s.q[t] = CAbeg[q] - 1u;
            do ca_next(CA, q1, s.q[t], s.npos[t]);
            while (s.npos[t] < (uint32_t)j0);
        }
    }
    s.cntk = 0;
#pragma unroll
    for (uint32_t kk = 0; kk < 3; kk++) {
        unsigned cnt = 0;
#pragma unroll
        for (int t = 0; t < kStarM; t++) {
            const int q = q0 + 32 * t + lane;
            cnt += __popc(__ballot_sync(kFull, q < nL && (La[q] & 3u) - 1u == kk));
        }
        if ((uint32_t)lane == kk) s.cntk = cnt;
    }
    s.U = 0;
    cross_part<C, 2>(g, lut, H, cra, R, codes, La, q0, nL, CAbeg, CAlen, CA, s, j0, min(j1, i), lane);
    cross_part<C, 1>(g, lut, H, cra, R, codes, La, q0, nL, CAbeg, CAlen, CA, s, max(j0, i + 1), j1, lane);
    if (g.big) flush_hist<C>(H, g, r, a, lane);
    __syncwarp();
}

// The "2+1" sets of the task (r, x = R[i]) for one c = L_x[q], used when the task's c
// R-neighbour lists do not fit the CA scratch.  It keeps the cross items' partition (a set
// {r, a < b, c} belongs to the task of the depth-1 vertex c hangs off first: a if c ~ a, else
// b), so tasks of one root may mix both paths: one lane per position j of R,
//   PART 1, j > i:  {r, a = x, b = R[j], c}           (every j)
//   PART 2, j < i:  {r, a = R[j], b = x, c}           (only if c is not adjacent to R[j])
// code(c, R[j]) is scattered from c's list into the warp's 2-bit bitmap Bw first.
template <int C>
__device__ __forceinline__ void cross_c_item(const Dev &g, const uint8_t *lut, uint32_t r, int i, const uint32_t *R,
                                             int D, const uint8_t *codes, const uint32_t *La, int q, uint32_t *Bw,
                                             uint32_t *H, uint32_t cra, uint32_t x, int lane) {
    const uint32_t ec = La[q], c = ec >> 2, cxc = ec & 3u;
    const int64_t c0 = g.off[c], c1 = g.off[c + 1];
    bool any = false;
    for (int64_t base = c0; base < c1; base += 32) {
        const int64_t p = base + lane;
        if (p < c1) {
            const uint32_t e = g.adj[p];
            if ((e >> 2) > r) {
                const int pos = find_rank(R, D, e >> 2);
                if (pos >= 0 && pos != i) {
                    set2(Bw, pos, e & 3u);
                    any = true;
                }
            }
        }
    }
    __syncwarp();
    for (int base = 0; base < D; base += 32) {
        const int j = base + lane;
        int col = kNone;
        uint32_t b = 0;
        if (j < D && j != i) {
            const uint32_t e = R[j], crj = e & 3u, cxj = (uint32_t)codes[j] >> 2, ccj = get2(Bw, j);
            b = e >> 2;
            if (j > i) col = lut[cra | crj << 2 | cxj << 6 | cxc << 8 | swap2(ccj) << 10];
            else if (ccj == 0u) col = lut[crj | cra << 2 | swap2(cxj) << 6 | cxc << 10];
        }
        emit4<C>(H, g, c, b, col, lane);   // c warp-uniform, R[j] per lane
    }
    __syncwarp();
    if (__any_sync(kFull, any)) clear_words(Bw, 0, (D + 15) >> 4, lane);
    if (g.big) flush_hist<C>(H, g, r, x, lane);
    __syncwarp();
}

// c's R-neighbour lists (positions ascending, x = R[i] excluded, code(c, R[pos])) for every c
// in L_x, into the CTA scratch; each warp walks the lists of its c's twice (count, write).
// Returns false if they do not fit (the task then runs cross_c_item per c instead).
template <int NW>
__device__ __forceinline__ bool ca_build(const Dev &g, uint32_t r, int i, const uint32_t *R, int D,
                                         const uint32_t *La, int nL, uint32_t *CAbeg, uint32_t *CAlen, uint32_t *CA,
                                         int *s_ca, int w, int lane) {
    for (;;) {   // c's taken from a shared counter (s_ca[1]): a hub c's long list does not stall one warp's share
        int q = 0;
        if (lane == 0) q = atomicAdd(s_ca + 1, 1);
        q = __shfl_sync(kFull, q, 0);
        if (q >= nL) break;
        const uint32_t c = La[q] >> 2;
        const int64_t c0 = g.off[c], c1 = g.off[c + 1];
        int cnt = 0;
        for (int64_t base = c0; base < c1; base += 32) {
            const int64_t p = base + lane;
            bool keep = false;
            if (p < c1) {
                const uint32_t y = g.adj[p] >> 2;
                if (y > r) {
                    const int pos = find_rank(R, D, y);
                    keep = pos >= 0 && pos != i;
                }
            }
            cnt += __popc(__ballot_sync(kFull, keep));
        }
        int beg = 0;
        if (lane == 0) beg = atomicAdd(s_ca, cnt);
        beg = __shfl_sync(kFull, beg, 0);
        if (lane == 0) {
            CAbeg[q] = (uint32_t)beg;
            CAlen[q] = (uint32_t)cnt;
        }
        if (beg + cnt > (int)g.ca_cap) continue;
        int k = 0;
        for (int64_t base = c0; base < c1; base += 32) {
            const int64_t p = base + lane;
            int pos = -1;
            uint32_t e = 0;
            if (p < c1) {
                e = g.adj[p];
                if ((e >> 2) > r) {
                    pos = find_rank(R, D, e >> 2);
                    if (pos == i) pos = -1;
                }
            }
            const unsigned bal = __ballot_sync(kFull, pos >= 0);
            if (pos >= 0) CA[beg + k + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)pos << 2) | (e & 3u);
            k += __popc(bal);
        }
    }
    __syncthreads();
    return *s_ca <= (int)g.ca_cap;
}

// ------------------------------------------------------------- light tasks (k = 4), closed form
// One warp, the task (r, a = R[i]) of a light root, Y = code(r, a).  As at heavy roots: "3" (b, c
// in R beyond i), "2+1" with c in L_a (every b in R beyond i) and "1+2" (b, c in L_a) are counted
// from the key counts N[k] (positions beyond i) and M[w] (|L_a| per code(a, c)), with their
// edge pairs as events (classified alone, taken back from the plain counts); the sets that need
// a walked entry -- "2+1" with c in L_b \ N(a), and "1+1+1" -- are enumerated one per lane as
// before.  The walks of b's list (b in R beyond i, b in L_a) find every event and take-back; when
// the lists are staged they are walked flattened (flat_walk), else list by list.
// N is the warp's 16 words at Bb (unused by this path), M its 4 words after the filters.
// Light k = 4 task (r, x = R[i]) in closed form with the heavy partition of "2+1" (PART 1 / PART 2,
// as at heavy roots): no walk of R's lists per task.  A light root's tasks all take this path, so
// every "2+1" set {r, a < b, c} is counted once, in the task of the first depth-1 vertex c hangs
// off.  Per task: the key counts N (beyond i: slots 0..15, before i: 16..31) and M;
// the "3" take-backs and events from the item's induced-edge records (rec[0..nrec): q | p << 8 |
// code(R[q], R[p]) << 16, both directions, every position > the item's first task; when they did
// not fit, rec == nullptr and R's lists beyond i are walked for their R entries instead); the
// R[j] side of "3" (j > i) and "2+1" (all j != i); the c side of "2+1" / "1+2" for c in L_x; one
// walk per u in L_x (part-1 events and part-2 removals for u ~ R[j], "1+2" events, "1+1+1"
// sets); the plain pairs of r and x.  N: 32 ints, M: 4 ints of the warp's scratch.
// HV: a small task of a heavy root run by one warp (R is the CTA's staged N+(r)): positions by the
// bucket index ix, the "3" induced edges from k_nr's lists (NB: positions that have any), and the
// "2+1" R[j] side left to k_rside (this task's M goes to gMt[0..3]).
template <int C, bool HV = false>
__device__ __forceinline__ void light_task_hp(const Dev &g, const uint8_t *lut, uint32_t r, int i,
                                              const uint32_t *R, int D, const uint32_t *Ba, const uint32_t *La,
                                              int nL, uint32_t *H, int *N, int *M, const Staged *st,
                                              const uint32_t *rec, int nrec, int lane, const RIndex *ix = nullptr,
                                              int64_t seg = 0, const uint32_t *NB = nullptr, uint32_t *gMt = nullptr) {
    const uint32_t Y = R[i] & 3u, x = R[i] >> 2;
    const uint32_t *FR = st->FR, *FL = st->FL;
    auto key = [&](int q) -> uint32_t { return (R[q] & 3u) | get2(Ba, q) << 2; };
    auto rpos = [&](uint32_t y) -> int {   // position of vertex y in R, or -1
        if constexpr (HV) return find_pos(R, D, y, *ix);
        else return fmay(FR, y) ? find_rank(R, D, y) : -1;
    };
    N[lane] = 0;
    if (lane < 4) M[lane] = 0;
    __syncwarp();
    for (int base = 0; base < D; base += 32) {   // one leader per distinct slot: no race
        const int q = base + lane;
        const uint32_t slot = q < D && q != i ? key(q) | (q < i ? 16u : 0u) : 0u;
        const unsigned m = __match_any_sync(kFull, slot);
        if (slot && lane == __ffs(m) - 1) N[slot] += __popc(m);
    }
    for (int base = 0; base < nL; base += 32) {
        const int q = base + lane;
        const uint32_t w = q < nL ? La[q] & 3u : 0u;
        const unsigned m = __match_any_sync(kFull, w);
        if (w && lane == __ffs(m) - 1) M[w] += __popc(m);
    }
    __syncwarp();
    const uint32_t PP = __ballot_sync(kFull, N[lane] > 0);   // slots present (beyond | before << 16)
    const uint32_t P = PP & 0xffffu;
    if (HV && lane < 4) gMt[lane] = (uint32_t)M[lane];
    // "3": an induced edge R[q] - R[p] (q, p > i) is not a plain partner of R[q]; q < p: the event
    // {r, x, R[q], R[p]}, classified by its full mask
    auto rec_act = [&](int q, int p, uint32_t z) {
        const uint32_t kq = key(q), kp = key(p);
        const uint32_t mp = star_mask(Y, kq, kp), pl = lut[mp];
        acc_addw(accp(g, R[q] >> 2, pl), (AccT)0 - (AccT)1);
        if (p > q) {
            const uint32_t ce = lut[mp | z << 10];
            acc_add(accp(g, R[q] >> 2, ce), 1u);
            acc_add(accp(g, R[p] >> 2, ce), 1u);
            atomicAdd(H + ce, 1u);
            atomicAdd(H + pl, 0xffffffffu);
        }
    };
    if constexpr (HV) {
        for (int q = i + 1 + lane; q < D; q += 32) {   // no warp-collective operations inside
            if (!((NB[q >> 5] >> (q & 31)) & 1u)) continue;
            for (int64_t e = g.nr_off[seg + q], e1 = g.nr_off[seg + q + 1]; e < e1; e++) {
                const uint32_t en = g.nr_adj[e];
                const int p = (int)(en >> 2);
                if (p > i) rec_act(q, p, en & 3u);
            }
        }
    } else if (rec) {
        for (int t = lane; t < nrec; t += 32) {
            const uint32_t v = rec[-1 - t];
            const int q = (int)(v & 0xffu), p = (int)((v >> 8) & 0xffu);
            if (q > i && p > i) rec_act(q, p, v >> 16);
        }
    } else if (i + 1 < D) {
        const uint32_t xi = x;
        auto ent = [&](int q, uint32_t e, bool valid) {
            const uint32_t c = e >> 2;
            if (valid && c > xi && fmay(FR, c)) {
                const int p = find_rank(R, D, c);
                if (p >= 0) rec_act(q, p, e & 3u);
            }
        };
        if (st->rok) flat_walk(st->RL, st->RS, i + 1, D, lane, ent);
        else
            for (int q = i + 1; q < D; q++) {
                const List bl = glist(g, R[q] >> 2);
                for (int p = lane; p < bl.len; p += 32) ent(q, bl.p[p], true);
            }
    }
    // R[j] (lanes): plain "3" sets per partner key (j > i), plain "2+1" sets per w (part 1 / 2)
    for (int j = lane; j < D; j += 32) {
        if (j == i) continue;
        const uint32_t b = R[j] >> 2, kb = key(j);
        if (j > i)
            for (uint32_t m = P; m; m &= m - 1u) {
                const uint32_t k = (uint32_t)__ffs(m) - 1u;
                const uint32_t cnt = (uint32_t)N[k] - (k == kb ? 1u : 0u);
                if (cnt) acc_add(accp(g, b, lut[star_mask(Y, kb, k)]), cnt);
            }
        if (!HV)   // (heavy roots: k_rside)
#pragma unroll
            for (uint32_t w = 1; w <= 3; w++)
                if (M[w]) acc_add(accp(g, b, lut[j > i ? p1_mask(Y, kb, w) : p2_mask(Y, kb, w)]), (uint32_t)M[w]);
    }
    // c in L_x (lanes): plain "2+1" sets per (part, key), plain "1+2" sets per partner code
    for (int q = lane; q < nL; q += 32) {
        const uint32_t ec = La[q], c = ec >> 2, w = ec & 3u;
        for (uint32_t m = PP; m; m &= m - 1u) {
            const uint32_t s = (uint32_t)__ffs(m) - 1u, k = s & 15u;
            acc_add(accp(g, c, lut[s < 16 ? p1_mask(Y, k, w) : p2_mask(Y, k, w)]), (uint32_t)N[s]);
        }
#pragma unroll
        for (uint32_t w2 = 1; w2 <= 3; w2++) {
            const uint32_t cnt = (uint32_t)M[w2] - (w2 == w ? 1u : 0u);
            if (cnt) acc_add(accp(g, c, lut[Y | w << 6 | w2 << 8]), cnt);
        }
    }
    if (st->lok) gather_wait();   // the L_x lists' copies (issued before the filter build)
    // an entry e of u = L_x[q]'s list
    auto u_entry = [&](int q, uint32_t e, bool valid, uint32_t &y) -> int {
        y = e >> 2;
        if (!valid || y <= r || y == x) return kNone;
        const uint32_t eu = La[q], u = eu >> 2, w = eu & 3u;
        const int pos = rpos(y);
        if (pos >= 0) {   // u ~ R[j]
            const uint32_t kj = key(pos);
            if (pos > i) {   // part-1 event: code(R[j], u) = swap(code(u, R[j]))
                const uint32_t mp = p1_mask(Y, kj, w);
                const uint32_t ce = lut[mp | swap2(e & 3u) << 10], pl = lut[mp];
                acc_add(accp(g, u, ce), 1u);
                acc_add(accp(g, y, ce), 1u);
                acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                atomicAdd(H + ce, 1u);
                atomicAdd(H + pl, 0xffffffffu);
            } else {         // part 2: the set belongs to R[j]'s task
                const uint32_t pl = lut[p2_mask(Y, kj, w)];
                acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                atomicAdd(H + pl, 0xffffffffu);
            }
            return kNone;
        }
        const uint32_t mb = Y | w << 6;
        const int qq = fmay(FL, y) ? find_rank(La, nL, y) : -1;
        if (qq >= 0) {
            if (qq > q) {   // "1+2" with a u-y edge: event
                const uint32_t mp = mb | (La[qq] & 3u) << 8;
                const uint32_t ce = lut[mp | (e & 3u) << 10], pl = lut[mp];
                acc_add(accp(g, u, ce), 1u);
                acc_add(accp(g, y, ce), 1u);
                acc_addw(accp(g, u, pl), (AccT)0 - (AccT)1);
                acc_addw(accp(g, y, pl), (AccT)0 - (AccT)1);
                atomicAdd(H + ce, 1u);
                atomicAdd(H + pl, 0xffffffffu);
            }
            return kNone;
        }
        return lut[mb | (e & 3u) << 10];   // "1+1+1" {r, x, u, y}
    };
    if (st->lok && nL > 0) {
        flat_walk(st->LL, st->LS, 0, nL, lane, [&](int q, uint32_t e, bool valid) {
            uint32_t y;
            const int col = u_entry(q, e, valid, y);
            emit4v<C>(H, g, La[q] >> 2, q, y, col, lane);
        });
    } else {
        for (int q = 0; q < nL; q++) {
            const List ul = list_at(g, La, q, st->LL, st->LS, st->lok);
            for (int base = 0; base < ul.len; base += 32) {
                const int p = base + lane;
                uint32_t y;
                const int col = u_entry(q, p < ul.len ? ul.p[p] : 0u, p < ul.len, y);
                emit4<C>(H, g, La[q] >> 2, y, col, lane);
            }
            if (g.big) flush_hist<C>(H, g, r, x, lane);
        }
    }
    __syncwarp();
    // r and x: the plain pairs -- "3" per key pair, "2+1" per (part, key, w), "1+2" per w pair
    for (int idx = lane; idx < 256 + 96 + 16; idx += 32) {
        uint64_t cnt = 0;
        uint32_t mask = 0;
        if (idx < 256) {
            const uint32_t k1 = (uint32_t)idx >> 4, k2 = (uint32_t)idx & 15u;
            if (k1 <= k2 && ((P >> k1) & (P >> k2) & 1u)) {
                const uint64_t n1 = (uint64_t)N[k1], n2 = (uint64_t)N[k2];
                cnt = k1 < k2 ? n1 * n2 : n1 * (n1 - 1) / 2;
                mask = star_mask(Y, k1, k2);
            }
        } else if (idx < 256 + 96) {
            const uint32_t part = (uint32_t)(idx - 256) / 48u, rest = (uint32_t)(idx - 256) % 48u;
            const uint32_t k = rest / 3u, w = rest % 3u + 1u;
            if ((PP >> (16u * part + k)) & 1u) {
                cnt = (uint64_t)N[16u * part + k] * (uint64_t)M[w];
                mask = part == 0 ? p1_mask(Y, k, w) : p2_mask(Y, k, w);
            }
        } else {
            const uint32_t w1 = (uint32_t)(idx - 352) >> 2, w2 = (uint32_t)(idx - 352) & 3u;
            if (w1 >= 1 && w1 <= w2 && w2 <= 3) {
                const uint64_t m1 = (uint64_t)M[w1], m2 = (uint64_t)M[w2];
                cnt = w1 < w2 ? m1 * m2 : m1 * (m1 - (m1 > 0)) / 2;
                mask = Y | w1 << 6 | w2 << 8;
            }
        }
        if (cnt) {
            const uint32_t col = lut[mask];
            acc_addw(accp(g, r, col), (AccT)cnt);
            acc_addw(accp(g, x, col), (AccT)cnt);
        }
    }
}

// The task (r, a = R[i]).  Ba/La (phase A) and, for heavy k = 4 tasks, codes must be ready.
// NW == 1: one warp does everything in order.  NW > 1 (heavy): the CTA's warps take work
// items from the shared counter *wctr (star chunks longest first, then b in R, then b in L_a).
// Bb/Bl are this warp's scratch bitmaps (zero on entry and exit), H its histogram.
template <int K, int C, int NW>
__device__ __forceinline__ void task_loops(const Dev &g, const uint8_t *lut, uint32_t r, int i, const uint32_t *R,
                                           int D, const uint32_t *Ba, const uint32_t *La, int nL, uint32_t *Bb,
                                           uint32_t *Bl, uint32_t *H, const uint8_t *codes, int *wctr, uint32_t *ca,
                                           int *s_ca, const Staged *st, int w, int lane, const int *sN = nullptr,
                                           const int *sM = nullptr, unsigned long long *Hs = nullptr,
                                           const RIndex *ix = nullptr, const uint32_t *NB = nullptr) {
    const uint32_t ea = R[i], a = ea >> 2, cra = ea & 3u;
    if constexpr (K == 3) {
        // "2": b in R after a.   mask (r,a) | (r,b) << 2 | (a,b) << 4
        for (int base = i + 1 + w * 32; base < D; base += NW * 32) {
            const int p = base + lane;
            int col = kNone;
            uint32_t b = 0;
            if (p < D) {
                const uint32_t eb = R[p];
                b = eb >> 2;
                col = lut[cra | (eb & 3u) << 2 | get2(Ba, p) << 4];
            }
            emit3<C>(H, g, b, col, lane);
        }
        // "1+1": b in L_a.   (r,b) = 0
        for (int base = w * 32; base < nL; base += NW * 32) {
            const int q = base + lane;
            int col = kNone;
            uint32_t b = 0;
            if (q < nL) {
                const uint32_t eb = La[q];
                b = eb >> 2;
                col = lut[cra | (eb & 3u) << 4];
            }
            emit3<C>(H, g, b, col, lane);
        }
        if (g.big) flush_hist<C>(H, g, r, a, lane);
    } else if constexpr (NW == 1) {
        for (int j = i + 1; !(VDMC_SKIPF(g) & 2) && j < D; j++)
            item_b_in_R<C, 1>(g, lut, r, i, j, R, D, Ba, La, nL, Bb, Bl, H, cra, a,
                              list_at(g, R, j, st->RL, st->RS, st->rok), lane, st->FR, st->FL);
        for (int x = 0; !(VDMC_SKIPF(g) & 4) && x < nL; x++)
            item_b_in_La<C>(g, lut, r, x, R, D, La, nL, Bl, H, cra, a, list_at(g, La, x, st->LL, st->LS, st->lok),
                            lane, st->FR, st->FL);
    } else if (g.fold <= 0) {
        // closed form (default): one walk per u in L_x (the long, uneven items first), then the
        // "3" items (positions beyond i) and the "2+1" R[j]-side items (all positions), which fill
        // the warps' tails
        const int rem = D - i - 1;
        // (measured: batching several u's per item with a flattened walk is slower, 197-277 vs 182 ms
        // on cfg4 -- fewer items balance the warps worse and the per-entry owner shuffles cost more
        // than the idle lanes of short lists)
        const int nu = (VDMC_SKIPF(g) & 4) ? 0 : nL;
        const int nstar = rem >= 2 ? (rem + kSPW - 1) / kSPW : 0;
        const int nj = (VDMC_SKIPF(g) & 2) || nL == 0 || g.gM ? 0 : (D + kSPW - 1) / kSPW;
        const int total = nu + nstar + nj;
        const uint32_t P = __ballot_sync(kFull, lane < 16 && sN[lane] > 0);   // keys present beyond i
        const int64_t seg = g.hbase[r];
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(wctr, 1);
            it = __shfl_sync(kFull, it, 0);
            if (it >= total) break;
            if (it < nu) {
                u_closed<C>(g, lut, Hs, H, r, a, cra, i, R, D, codes, La, nL, sN, sM, it, lane, *ix);
                if (g.big) flush_hist<C>(H, g, r, a, lane);
            } else if (it < nu + nstar) {
                if (!(VDMC_SKIPF(g) & 1))
                    star_closed_item<C>(g, lut, Hs, cra, i, R, D, codes, sN, P, seg, i + 1 + (it - nu) * kSPW, lane,
                                        NB);
            } else {
                cross_j_closed<C>(g, lut, cra, i, R, D, codes, sM, (it - nu - nstar) * kSPW, lane);
            }
            __syncwarp();
        }
    } else {
        // enumerated path (star_block option): star chunk items, cross items over CA lists
        uint32_t *CAbeg = ca, *CAlen = ca + g.maxdeg, *CA = ca + 2 * (int64_t)g.maxdeg;
        const bool cross = !(VDMC_SKIPF(g) & 8) && ca_build<NW>(g, r, i, R, D, La, nL, CAbeg, CAlen, CA, s_ca, w, lane);
        const int fold = g.fold;
        const int nch = D - (i + 2) > 0 ? (D - (i + 2) + kStarW - 1) / kStarW : 0;   // star chunks
        int nstar = 0;
        for (int kk = 0; kk < nch; kk++) nstar += star_blocks(D, i, kk, fold);
        const int nck = (nL + kStarW - 1) / kStarW, njb = (D + g.xblock - 1) / g.xblock;
        const int nB = cross ? nck * njb : nL;                                  // "2+1" items
        const int total = nstar + nB + nL;
        // star items (bounded length), then the "2+1" items, then the b-in-L_a items
        for (;;) {
            int it = 0;
            if (lane == 0) it = atomicAdd(wctr, 1);
            it = __shfl_sync(kFull, it, 0);
            if (it >= total) break;
            int star_k = -1, star_b = 0, b_it = -1;
            if (it < nstar) {
                int rem = it, kk = 0;
                for (;; kk++) {
                    const int nb = star_blocks(D, i, kk, fold);
                    if (rem < nb) break;
                    rem -= nb;
                }
                star_k = kk;
                star_b = rem;
            } else if (it < nstar + nB) {
                b_it = it - nstar;
            }
            if (star_k >= 0) {
                if (!(VDMC_SKIPF(g) & 1)) star_item<C>(g, lut, r, i, R, D, Ba, codes, cra, a, H, star_k, star_b, fold, lane);
            } else if (b_it >= 0) {
                if (VDMC_SKIPF(g) & 2) continue;
                if (cross)
                    cross_item<C>(g, lut, r, i, R, D, codes, La, nL, CAbeg, CAlen, CA, cra, a, H, b_it / njb,
                                  b_it % njb, lane);
                else
                    cross_c_item<C>(g, lut, r, i, R, D, codes, La, b_it, Bl, H, cra, a, lane);
            } else {
                if (!(VDMC_SKIPF(g) & 4))
                    item_b_in_La<C>(g, lut, r, it - nstar - nB, R, D, La, nL, Bl, H, cra, a,
                                    glist(g, La[it - nstar - nB] >> 2), lane);
            }
        }
    }
}

template <int K, int C, bool HSMEM>
__global__ void __launch_bounds__(kBlock, 2) k_enum(Dev g, Layout L, int64_t lo, int64_t hi,
                                                     unsigned long long *ctr, const uint8_t *__restrict__ lut_g) {
    constexpr int NM = K == 3 ? 64 : 4096;
    extern __shared__ uint32_t sm[];
    __shared__ uint8_t lut[NM];
    __shared__ int64_t s_item, s_sub[4];   // s_sub: the slice's heavy_task [h0, h1) and light_root [l0, l1)
    __shared__ int s_nL, s_work, s_ca[2];   // s_ca: CA space used, next c of ca_build
    __shared__ unsigned s_wm;               // heavy: warp-mode tasks of the fetched chunk (bit per task)
    __shared__ int s_cnt;                   // heavy: tasks in the fetched chunk
    __shared__ int32_t s_wr[kHChunk];       // heavy: their roots
    __shared__ int s_N[32], s_M[4];         // closed forms: key counts beyond / before i, |L_x| per code(x, c)
    __shared__ unsigned long long Hs[C];    // closed forms: r / x side of events and take-backs (modular)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int q = tid; q < NM; q += kBlock) lut[q] = lut_g[q];
    if (tid < C) Hs[tid] = 0;
    if (tid < 32) s_N[tid] = 0;
    if (tid < 4) s_M[tid] = 0;
    for (int q = tid; q < L.total; q += kBlock) sm[q] = 0;
    uint32_t *H = sm + L.hist + wid * C;
    if (tid < 4) {   // both lists ascend with the task id, so the slice [lo, hi) is a sub-list of each
        const bool heavy = tid < 2;
        const int64_t key = (tid & 1) ? hi : lo;
        int64_t a = 0, b = heavy ? g.nheavy : g.nlight;
        while (a < b) {   // first entry whose tasks end after key (heavy: task >= key; light: tfirst[r+1] > key
            const int64_t mid = (a + b) >> 1;   // for lo, tfirst[r] >= key for hi)
            bool before;
            if (heavy) before = g.heavy_task[mid] < key;
            else {   // the item's tasks [t0, t1)
                const int64_t r = g.light_root[mid];
                const int64_t t0 = g.tfirst[r] + g.light_i0[mid];
                const int64_t t1 = min(t0 + kLightChunk, g.tfirst[r + 1]);
                before = (tid & 1) ? t0 < key : t1 <= key;
            }
            if (before) a = mid + 1;
            else b = mid;
        }
        s_sub[tid] = a;
    }

    // ---------------- heavy phase: one CTA per task (r, a)
    {
        // HSMEM: the heavy buffers are carved from shared memory (the compiler then emits LDS)
        uint32_t *hb = HSMEM ? sm : g.gheavy + (int64_t)blockIdx.x * g.gheavy_per_cta;
        uint32_t *R = hb + L.R, *La = hb + L.La, *Ba = hb + L.Ba;
        uint32_t *Bl = hb + L.Bl + wid * L.lw;
        uint8_t *codes = reinterpret_cast<uint8_t *>(hb + L.Bb);   // heavy: per-task code bytes
        if (!HSMEM) {   // zero this CTA's global bitmaps once
            for (int q = tid; q < L.Bl + kWarps * L.lw - L.Ba; q += kBlock) hb[L.Ba + q] = 0;
        }
        __syncthreads();
        int64_t staged = -1;
        RIndex rix{0u, 0u, 0, nullptr};
        const bool wmode = HSMEM && K == 4 && L.wm && g.fold <= 0 && g.gM != nullptr;
        int64_t h = 0, hend = 0;
        for (;;) {   // bounds re-read from shared memory (keeps them out of the loop's registers)
            if (h >= hend) {   // kHChunk consecutive tasks per fetch: one R staging for a small root's
                               // tasks, and two barriers per chunk instead of per task
                if (tid == 0) {   // chunk k: kHubChunk tasks over the hub prefix of the slice, then kHChunk
                    const int64_t k = (int64_t)atomicAdd(ctr, 1ull);
                    const int64_t K1 = (g.hub_tasks + kHubChunk - 1) / kHubChunk;
                    s_item = s_sub[0] + (k < K1 ? k * kHubChunk : K1 * kHubChunk + (k - K1) * kHChunk);
                    s_cnt = k < K1 ? kHubChunk : kHChunk;
                }
                __syncthreads();
                h = s_item;
                hend = h + s_cnt;
                if (wmode && wid == 0) {   // warp-mode tasks: a's list fits the warp's slot
                    const int64_t x = h + lane;
                    bool wm = false;
                    int32_t rr = -1;
                    if (x < hend && x < s_sub[1]) {
                        const int64_t t = g.heavy_task[x];
                        rr = g.task_root[t];
                        const int64_t rs = g.split[rr];
                        const uint32_t a = g.adj[rs + (t - g.tfirst[rr])] >> 2;
                        wm = g.off[a + 1] - g.off[a] <= kWL;   // (a positions limit measured slower)
                    }
                    const unsigned m = __ballot_sync(kFull, wm);
                    if (lane < kHChunk) s_wr[lane] = rr;
                    if (lane == 0) s_wm = m;
                }
                __syncthreads();
            }
            if (h >= s_sub[1]) break;
            // stage N+(r) (once per root): R, NB (positions with an induced neighbour), the bucket index
            auto stage = [&](uint32_t r) {
                const int64_t rs = g.split[r];
                const int D = (int)(g.off[r + 1] - rs);
                for (int q = tid; q < D; q += kBlock) R[q] = g.adj[rs + q];
                if (K == 4 && g.fold <= 0) {
                    const int64_t seg = g.hbase[r];
                    for (int base = wid * 32; base < D; base += kBlock) {
                        const int q = base + lane;
                        const unsigned m = __ballot_sync(kFull, q < D && g.nr_off[seg + q + 1] > g.nr_off[seg + q]);
                        if (lane == 0) hb[L.NB + (base >> 5)] = m;
                    }
                }
                staged = r;
                __syncthreads();
                rix = build_rindex(R, D, L.T >= 0 && g.fold <= 0 ? reinterpret_cast<uint16_t *>(hb + L.T) : nullptr,
                                   tid, kBlock);
                __syncthreads();
            };
            if (wmode && ((s_wm >> (int)(h - s_item)) & 1u)) {
                // a run of warp-mode tasks of one root: one warp per task (light_task_hp<HV>), in snake order
                // over the warps (the run's tasks shrink along it)
                const uint32_t r = (uint32_t)s_wr[h - s_item];
                int64_t h2 = h + 1;
                while (h2 < hend && h2 < s_sub[1] && ((s_wm >> (int)(h2 - s_item)) & 1u) &&
                       (uint32_t)s_wr[h2 - s_item] == r)
                    h2++;
                if (staged != r) stage(r);
                const int64_t rs = g.split[r], seg = g.hbase[r], tf = g.tfirst[r];
                const int D = (int)(g.off[r + 1] - rs), n = (int)(h2 - h);
                uint32_t *ws = hb + L.W + wid * L.ws;
                uint32_t *wBa = ws, *wLa = ws + L.bw, *wN = wLa + kWL, *wM = wN + 32, *wFL = wM + 4;
                for (int k = 0; k * kWarps < n; k++) {
                    const int idx = (k & 1) ? (k + 1) * kWarps - 1 - wid : k * kWarps + wid;
                    if (idx >= n) continue;
                    const int i = (int)(g.heavy_task[h + idx] - tf);
                    clear_words(wBa, 0, (D + 15) >> 4, lane);
                    __syncwarp();
                    const List al = glist(g, R[i] >> 2);
                    const int nL = build_a(r, al, R, D, wBa, wLa, lane, nullptr, &rix);
                    wFL[lane] = 0;
                    __syncwarp();
                    for (int q = lane; q < nL; q += 32) fadd(wFL, wLa[q] >> 2);
                    __syncwarp();
                    const Staged st{nullptr, nullptr, nullptr, nullptr, false, false, nullptr, wFL};
                    light_task_hp<C, true>(g, lut, r, i, R, D, wBa, wLa, nL, H, reinterpret_cast<int *>(wN),
                                           reinterpret_cast<int *>(wM), &st, nullptr, 0, lane, &rix, seg, hb + L.NB,
                                           g.gM + (seg + i) * 4);
                    flush_hist<C>(H, g, r, R[i] >> 2, lane);
                }
                __syncthreads();
                h = h2;
                continue;
            }
            const int64_t t = g.heavy_task[h++];
            const uint32_t r = (uint32_t)g.task_root[t];
            const int64_t rs = g.split[r];
            const int D = (int)(g.off[r + 1] - rs);
            const int i = (int)(t - g.tfirst[r]);
#ifdef VDMC_PROFILING
            if (g.minrem > 0 ? D - i - 1 < g.minrem : (g.minrem < 0 && D - i - 1 >= -g.minrem)) continue;   // VDMC_MINREM
#endif
            if (staged != r) stage(r);
            const List al = glist(g, R[i] >> 2);
            build_a_cta<kWarps>(r, al, R, D, Ba, La, hb + L.Bl, &s_nL, wid, lane, rix);
            const int nL = s_nL;
            for (int q = tid; q < 2 * ((al.len + 31) >> 5); q += kBlock) hb[L.Bl + q] = 0;   // build_a_cta scratch
            if (tid == 0) {
                s_work = 0;
                s_ca[0] = 0;
                s_ca[1] = 0;
            }
            if (K == 4) {   // codes[j] = code(r, R[j]) | code(a, R[j]) << 2; key counts s_N, s_M
                const bool closed = g.fold <= 0;
                for (int base = wid * 32; base < D; base += kBlock) {
                    const int q = base + lane;
                    uint32_t key = 0;
                    if (q < D) {
                        key = (R[q] & 3u) | get2(Ba, q) << 2;
                        codes[q] = (uint8_t)key;
                    }
                    if (closed) {   // slot key (beyond i) or 16 + key (before i)
                        const uint32_t slot = q < D && q != i ? key | (q < i ? 16u : 0u) : 0u;
                        const unsigned m = __match_any_sync(kFull, slot);
                        if (slot && lane == __ffs(m) - 1) atomicAdd(s_N + slot, __popc(m));
                    }
                }
                if (closed)
                    for (int base = wid * 32; base < nL; base += kBlock) {
                        const int q = base + lane;
                        const uint32_t w = q < nL ? La[q] & 3u : 0u;
                        const unsigned m = __match_any_sync(kFull, w);
                        if (w && lane == __ffs(m) - 1) atomicAdd(s_M + w, __popc(m));
                    }
            }
            __syncthreads();
            task_loops<K, C, kWarps>(g, lut, r, i, R, D, Ba, La, nL, nullptr, Bl, H, codes, &s_work,
                                  g.gca + (int64_t)blockIdx.x * g.gca_per_cta, s_ca, nullptr, wid, lane, s_N, s_M, Hs, &rix,
                                  hb + L.NB);
            flush_hist<C>(H, g, r, R[i] >> 2, lane);
            __syncthreads();
            if (K == 4 && g.fold <= 0) {
                closed_root<C>(g, lut, r, R[i] >> 2, R[i] & 3u, s_N, s_M, Hs, tid);
                if (g.gM && tid < 4) g.gM[(g.hbase[r] + i) * 4 + tid] = (uint32_t)s_M[tid];
            }
            for (int q = tid; q < ((D + 15) >> 4); q += kBlock) Ba[q] = 0;
            __syncthreads();
            if (tid < 32) s_N[tid] = 0;
            if (tid < 4) s_M[tid] = 0;
                }
    }
    __syncthreads();
    for (int q = tid; q < L.total; q += kBlock) sm[q] = 0;   // light region overlays the heavy one
    __syncthreads();

    // ---------------- light phase: one warp per root, its tasks in sequence
    {
        uint32_t *lw = sm + L.light + wid * kLightWords;
        uint32_t *R = lw, *Las = lw + kLW, *Ba = lw + 2 * kLW, *Bb = Ba + kLB, *Bls = Bb + kLB;
        uint32_t *RS = Bls + kLB, *RO = RS + kSmax + 1, *LS = RO + kSmax, *LO = LS + kSmax + 1;
        uint32_t *PL = LO + kSmax;   // staged adjacency lists: R's, then the current L_a's
        uint32_t *FR = PL + kPool, *FL = FR + kFW;
        uint32_t *gw = g.glight + ((int64_t)blockIdx.x * kWarps + wid) * g.glight_per_warp;   // oversize L_a
        Staged st{PL, RS, PL, LS, false, false, FR, FL};
        for (;;) {
            unsigned long long x = 0;
            if (lane == 0) x = atomicAdd(ctr + 1, 1ull);
            const int64_t li = s_sub[2] + (int64_t)__shfl_sync(kFull, x, 0);
            if (li >= s_sub[3]) break;
            const uint32_t r = (uint32_t)g.light_root[li];
            const int64_t t0 = g.tfirst[r];   // the item's tasks: [t0 + i0, t0 + i0 + kLightChunk) of the root
            const int64_t ti = t0 + g.light_i0[li];
            const int64_t ta = max(ti, lo), tb = min(min(ti + kLightChunk, g.tfirst[r + 1]), hi);
            if (ta >= tb) continue;
            const int64_t rs = g.split[r];
            const int D = (int)(g.off[r + 1] - rs);
            FR[lane] = 0;
            __syncwarp();
            for (int q = lane; q < D; q += 32) {
                const uint32_t e = g.adj[rs + q];
                R[q] = e;
                fadd(FR, e >> 2);
            }
            __syncwarp();
            st.rok = gather_lists(g, R, D, RS, RO, kSmax, PL, kPool, lane);   // lists of R, once per root
            const int used = st.rok ? (int)RS[D] : 0;
            uint32_t *LL = PL + used;
            st.LL = LL;
            // k = 4 closed form: the induced edges of N+(r) among the positions beyond the item's first
            // task, once per item (records at the top of the pool, below kPool, growing down)
            const bool hp = K == 4 && g.fold <= 0;
            int nrec = 0;
            const uint32_t *recp = nullptr;
            if (hp) {
                const int i0 = (int)(ta - t0);
                const int cap = min(kRecCap, kPool - used);
                uint32_t *rtop = PL + kPool;
                if (i0 + 1 < D) {
                    const uint32_t x0 = R[i0] >> 2;   // positions > i0 <=> vertices > x0
                    auto ent = [&](int q, uint32_t e, bool valid) {
                        const uint32_t c = e >> 2;
                        int p = -1;
                        if (valid && c > x0 && fmay(FR, c)) p = find_rank(R, D, c);
                        const unsigned bal = __ballot_sync(kFull, p >= 0);
                        const int k = nrec + __popc(bal & ((1u << lane) - 1u));
                        if (p >= 0 && k < cap) rtop[-1 - k] = (uint32_t)q | (uint32_t)p << 8 | (e & 3u) << 16;
                        nrec += __popc(bal);
                    };
                    if (st.rok) flat_walk(PL, RS, i0 + 1, D, lane, ent);
                    else
                        for (int q = i0 + 1; q < D; q++) {
                            const List bl = glist(g, R[q] >> 2);
                            for (int base = 0; base < bl.len; base += 32) {
                                const int p = base + lane;
                                ent(q, p < bl.len ? bl.p[p] : 0u, p < bl.len);
                            }
                        }
                }
                if (nrec <= cap) recp = rtop;
                else nrec = 0;   // did not fit: each task walks R's lists beyond its a instead
                __syncwarp();
            }
            const int lcap = kPool - used - (recp ? nrec : 0);
            for (int64_t t = ta; t < tb; t++) {
                const int i = (int)(t - t0);
                const uint32_t a = R[i] >> 2;
                const List al = list_at(g, R, i, PL, RS, st.rok);
                uint32_t *La = Las, *Bl = Bls;
                if (al.len > kLW) {   // only with a user-given order: lists longer than the smem slots
                    La = gw;
                    Bl = gw + g.maxdeg;
                    clear_words(Bl, 0, (al.len + 15) >> 4, lane);
                    __syncwarp();
                }
                const int nL = build_a(r, al, R, D, Ba, La, lane, FR);
                // closed form: the L_a lists' copies stay in flight through the filter build and the b
                // key counts and the R side; light_task_hp waits for them before the walks over L_a
                const bool closed = K == 4 && g.fold <= 0;
                st.lok = K == 4 && La == Las && gather_lists(g, La, nL, LS, LO, kSmax, LL, lcap, lane, !closed);
                FL[lane] = 0;
                __syncwarp();
                for (int q = lane; q < nL; q += 32) fadd(FL, La[q] >> 2);
                __syncwarp();
                if (hp)   // N: RO's words are free once R's lists are staged
                    light_task_hp<C>(g, lut, r, i, R, D, Ba, La, nL, H, reinterpret_cast<int *>(RO),
                                     reinterpret_cast<int *>(FL + kFW), &st, recp, nrec, lane);
                else
                    task_loops<K, C, 1>(g, lut, r, i, R, D, Ba, La, nL, Bb, Bl, H, nullptr, nullptr, nullptr, nullptr,
                                        &st, 0, lane);
                flush_hist<C>(H, g, r, a, lane);
                clear_words(Ba, 0, (D + 15) >> 4, lane);
                __syncwarp();
            }
        }
    }
}

// "2+1", the R[j] side at heavy roots, once per root instead of once per task: R[j] lies in M_i[w]
// plain sets {r, x_i, R[j], c} of class cls(Y_i, x_j, w) for every task i != j of the slice (the
// part-1 and part-2 masks of a plain set are the same digraph, so the LUT gives one column), i.e.
// in T[Y][w] = sum over the slice's tasks with code(r, x_i) = Y of M_i[w], less its own task's
// M_j; an induced neighbour x_i of R[j] (k_nr's lists) puts those M_i[w] sets in the class with the
// x_i-R[j] edge instead (exact part-1 / part-2 mask, as cross_j_closed).  M_i: written by k_enum.
template <int C>
__global__ void __launch_bounds__(256) k_rside(Dev g, const int32_t *__restrict__ hroots, int64_t nh, int64_t lo,
                                               int64_t hi, const uint8_t *__restrict__ lut_g) {
    __shared__ uint8_t lut[4096];
    __shared__ unsigned long long T[16];   // T[Y * 4 + w]
    for (int q = threadIdx.x; q < 4096; q += blockDim.x) lut[q] = lut_g[q];
    for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
        const uint32_t r = (uint32_t)hroots[h];
        const int64_t rs = g.split[r], t0 = g.tfirst[r];
        const int D = (int)(g.off[r + 1] - rs);
        const int i0 = (int)max(lo - t0, (int64_t)0), i1 = (int)min(hi - t0, (int64_t)D);
        if (i0 >= i1) continue;   // uniform over the CTA
        const int64_t seg = g.hbase[r];
        __syncthreads();
        if (threadIdx.x < 16) T[threadIdx.x] = 0;
        __syncthreads();
        for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
            const uint32_t Y = g.adj[rs + i] & 3u;
#pragma unroll
            for (int w = 1; w <= 3; w++) {
                const uint32_t m = g.gM[(seg + i) * 4 + w];
                if (m) atomicAdd(T + Y * 4 + w, (unsigned long long)m);
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < D; j += blockDim.x) {
            const uint32_t ej = g.adj[rs + j], y = ej >> 2, xj = ej & 3u;
            const bool own = j >= i0 && j < i1;
#pragma unroll
            for (uint32_t Y = 1; Y <= 3; Y++)
#pragma unroll
                for (uint32_t w = 1; w <= 3; w++) {
                    const unsigned long long cnt = T[Y * 4 + w] - (own && Y == xj ? g.gM[(seg + j) * 4 + w] : 0u);
                    if (cnt) acc_addw(accp(g, y, lut[p1_mask(Y, xj, w)]), (AccT)cnt);
                }
            for (int64_t e = g.nr_off[seg + j], e1 = g.nr_off[seg + j + 1]; e < e1; e++) {
                const uint32_t en = g.nr_adj[e];
                const int i = (int)(en >> 2);
                if (i < i0 || i >= i1) continue;
                const uint32_t Yi = g.adj[rs + i] & 3u, kj = xj | swap2(en & 3u) << 2;
#pragma unroll
                for (uint32_t w = 1; w <= 3; w++) {
                    const uint32_t m = g.gM[(seg + i) * 4 + w];
                    if (!m) continue;
                    acc_addw(accp(g, y, lut[p1_mask(Yi, xj, w)]), (AccT)0 - (AccT)m);
                    acc_addw(accp(g, y, lut[j > i ? p1_mask(Yi, kj, w) : p2_mask(Yi, kj, w)]), (AccT)m);
                }
            }
        }
    }
}

// S9: rows from rank order to original ids
// S9: acc is class-major [C][n] (rank order); out is row-major [original id][C].  A CTA
// transposes a tile of kFinV consecutive ranks through shared memory: reads of acc[j][v0..)
// and writes of each output row are both contiguous.
constexpr int kFinV = 16;
template <int C>
__global__ void __launch_bounds__(256) k_finalize(int64_t n, const int32_t *__restrict__ order,
                                                  const AccT *__restrict__ acc,
                                                  unsigned long long *__restrict__ out) {
    __shared__ unsigned long long tile[kFinV][C + 1];
    for (int64_t v0 = (int64_t)blockIdx.x * kFinV; v0 < n; v0 += (int64_t)gridDim.x * kFinV) {
        const int nv = (int)(n - v0 < kFinV ? n - v0 : kFinV);
        for (int idx = threadIdx.x; idx < kFinV * C; idx += blockDim.x) {
            const int j = idx / kFinV, vi = idx - j * kFinV;
            if (vi < nv) tile[vi][j] = acc[(int64_t)j * n + v0 + vi];
        }
        __syncthreads();
        for (int idx = threadIdx.x; idx < nv * C; idx += blockDim.x) {
            const int vi = idx / C, j = idx - vi * C;
            out[(int64_t)order[v0 + vi] * C + j] = tile[vi][j];
        }
        __syncthreads();
    }
}

// S4 cost model per task (r, a = R[i]), in picoseconds of whole-GPU time.  Terms:
// rem = D - i - 1 (positions of R after a), nla = |{x in N(a): x > r}| (a's list beyond r: L_a
// plus a's R-neighbours), D = |R|.  Coefficients: a non-negative least-squares fit of the
// measured enumeration time of 32 planner slices and 3 phase totals on cfg4 and cfg5 (two
// earlier models' slicings; tools/fit_plan.py, profiles/r02_planner_fit.txt; every row within 16 %):
//   heavy root (CTA per task):  92.3 ns + 0.0915 ps rem^2 (star items) + 3.53 ps nla D (cross items)
//   light root (warp per root): 1.45 ns + 12.8 ps rem nla + 49 ps nla^2 (pair loops and walks)
// (k_s2 / k_task_deg feed the walk terms the fit found insignificant; kept for k = 3's model.)
__global__ void k_s2(int64_t n, const int64_t *__restrict__ off, const uint32_t *__restrict__ adj,
                     int64_t *__restrict__ s2) {
    const int lane = threadIdx.x & 31;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
         v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int64_t acc = 0;
        for (int64_t q = off[v] + lane; q < off[v + 1]; q += 32) {
            const uint32_t u = adj[q] >> 2;
            acc += off[u + 1] - off[u];
        }
        for (int d = 16; d; d >>= 1) acc += __shfl_down_sync(kFull, acc, d);
        if (lane == 0) s2[v] = acc;
    }
}

__global__ void k_task_deg(int64_t ntasks, const int64_t *__restrict__ off, const int64_t *__restrict__ split,
                           const uint32_t *__restrict__ adj, const int64_t *__restrict__ tfirst,
                           const int32_t *__restrict__ task_root, int64_t *__restrict__ fdeg) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntasks; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = task_root[t];
        const uint32_t a = adj[split[r] + (t - tfirst[r])] >> 2;
        fdeg[t] = off[a + 1] - off[a];
    }
}

__global__ void k_cost(int64_t ntasks, int k, const int64_t *__restrict__ off, const int64_t *__restrict__ split,
                       const uint32_t *__restrict__ adj, const int64_t *__restrict__ tfirst,
                       const int32_t *__restrict__ task_root, const int64_t *__restrict__ s2,
                       const int64_t *__restrict__ fsum, int64_t *__restrict__ cost) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntasks; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = task_root[t];
        const int64_t rs = split[r], re = off[r + 1];
        const int64_t ia = rs + (t - tfirst[r]);
        const int64_t rem = re - ia - 1;
        const uint32_t a = adj[ia] >> 2;
        const int64_t da = off[a + 1] - off[a];
        const bool heavy = off[r + 1] - off[r] > kLightDeg;
        int64_t lo = off[a], hi = off[a + 1];   // first entry of a's list with rank > r
        const uint32_t key = ((uint32_t)r + 1u) << 2;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (adj[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        const int64_t nla = off[a + 1] - lo, D = re - rs;
        int64_t c;
        if (k == 3) {
            const int64_t suf = fsum[tfirst[r + 1] - 1] - fsum[t];
            c = heavy ? 92290 + 50 * (rem + da) : 1454 + 10 * (rem + nla) + suf + s2[a] / 8;
        } else if (heavy) {   // k = 4 heavy task (units of 1e-12 ms; tools/fit_plan.py, profiles/r02n_planner_fit.txt)
            c = da <= kWL ? 14954100 + 34100 * D   // one warp (light closed form over the staged R)
                          : 760 * D * da;          // one CTA (phase A over a's list, O(D) items, walks of L_a)
        } else {              // light task: O(D) key counts and R side, L_a walks, per-item staging of R's lists
            c = 146800 * D + 127200 * nla + ((ia - rs) % kLightChunk == 0 ? 2340700 : 0);
        }
        cost[t] = c;
    }
}

// root classes: heavy = G_U degree > kLightDeg (only roots with at least one task)
__global__ void k_root_flags(int64_t n, const int64_t *__restrict__ off, const int64_t *__restrict__ tfirst,
                             char *__restrict__ heavy, char *__restrict__ light) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const bool has = tfirst[r + 1] > tfirst[r];
        const bool h = off[r + 1] - off[r] > kLightDeg;
        heavy[r] = has && h;
        light[r] = has && !h;
    }
}

// S4 pre-pass for heavy roots: the induced adjacency of R = N+(r) in position space.  For
// x = R[q], the positions p of R whose vertex is a neighbour of x, with code(x, R[p]),
// ascending in p (x's list is sorted by rank and R is sorted by rank).  FILL = false counts,
// FILL = true writes.  One CTA per heavy root (atomic counter), one warp per position q.
template <bool FILL>
__global__ void __launch_bounds__(512) k_nr(const int64_t *__restrict__ off, const int64_t *__restrict__ split,
                                            const uint32_t *__restrict__ adj, const int32_t *__restrict__ hroots,
                                            int64_t nh, const int64_t *__restrict__ hbase, int64_t *__restrict__ cnt,
                                            const int64_t *__restrict__ nr_off, uint32_t *__restrict__ nr_adj,
                                            unsigned long long *ctr, int smem_cap) {
    extern __shared__ uint32_t Rs[];
    __shared__ int64_t s_h;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_h = (int64_t)atomicAdd(ctr, 1ull);
        __syncthreads();
        const int64_t h = s_h;
        __syncthreads();
        if (h >= nh) break;
        const uint32_t r = (uint32_t)hroots[h];
        const int64_t rs = split[r];
        const int D = (int)(off[r + 1] - rs);
        const uint32_t *R = adj + rs;
        if (D <= smem_cap) {
            for (int q = threadIdx.x; q < D; q += blockDim.x) Rs[q] = adj[rs + q];
            __syncthreads();
            R = Rs;
        }
        const int64_t seg = hbase[r];
        for (int q = wid; q < D; q += nw) {
            const uint32_t x = R[q] >> 2;
            const int64_t x0 = off[x], x1 = off[x + 1];
            int64_t k = 0;
            const int64_t o = FILL ? nr_off[seg + q] : 0;
            for (int64_t base = x0; base < x1; base += 32) {
                const int64_t p = base + lane;
                int pos = -1;
                uint32_t e = 0;
                if (p < x1) {
                    e = adj[p];
                    if ((e >> 2) > r) pos = find_rank(R, D, e >> 2);
                }
                const unsigned bal = __ballot_sync(kFull, pos >= 0);
                if (FILL && pos >= 0) nr_adj[o + k + __popc(bal & ((1u << lane) - 1u))] = ((uint32_t)pos << 2) | (e & 3u);
                k += __popc(bal);
            }
            if (!FILL && lane == 0) cnt[seg + q] = k;
        }
        __syncthreads();
    }
}

__global__ void k_light_parts(int64_t nl, const int32_t *__restrict__ lroots, const int64_t *__restrict__ tfirst,
                              int64_t *__restrict__ cnt) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nl; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = lroots[q], nt = tfirst[r + 1] - tfirst[r];
        cnt[q] = (nt + kLightChunk - 1) / kLightChunk;
    }
}

__global__ void k_light_scatter(int64_t nl, const int32_t *__restrict__ lroots, const int64_t *__restrict__ cnt,
                                const int64_t *__restrict__ base, int32_t *__restrict__ iroot,
                                int32_t *__restrict__ i0) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nl; q += (int64_t)gridDim.x * blockDim.x)
        for (int64_t p = 0; p < cnt[q]; p++) {
            iroot[base[q] + p] = lroots[q];
            i0[base[q] + p] = (int32_t)(p * kLightChunk);
        }
}

__global__ void k_heavy_d(int64_t nh, const int32_t *__restrict__ hroots, const int64_t *__restrict__ off,
                          const int64_t *__restrict__ split, int64_t *__restrict__ dlist) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nh; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = hroots[q];
        dlist[q] = off[r + 1] - split[r];
    }
}

__global__ void k_hub_prefix(int64_t nh, const int32_t *__restrict__ hroots, const int64_t *__restrict__ off,
                             unsigned long long *__restrict__ firstq) {   // first heavy root of degree <= kHubDeg
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nh; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = hroots[q];
        if (off[r + 1] - off[r] <= kHubDeg) atomicMin(firstq, (unsigned long long)q);
    }
}
__global__ void k_scatter_hbase(int64_t nh, const int32_t *__restrict__ hroots, const int64_t *__restrict__ seg,
                                int64_t *__restrict__ hbase) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nh; q += (int64_t)gridDim.x * blockDim.x)
        hbase[hroots[q]] = seg[q];
}

__global__ void k_task_flags(int64_t ntasks, const int32_t *__restrict__ task_root, const char *__restrict__ heavy,
                             char *__restrict__ flag) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntasks; t += (int64_t)gridDim.x * blockDim.x)
        flag[t] = heavy[task_root[t]];
}

Layout make_layout(int maxdeg, int C, bool &heavy_in_smem, int64_t &per_cta_words, bool force_global) {
    Layout L{};
    const int md = std::max(maxdeg, 1);
    L.bw = (md + 15) / 16;
    L.lw = (md + 15) / 16;
    // heavy buffers (offsets relative to the heavy base)
    L.R = 0;
    L.T = L.R + md;                      // bucket index of R: (kBuckets + 1) u16
    L.NB = L.T + (kBuckets + 2) / 2;
    L.Ba = L.NB + (md + 31) / 32;
    L.La = L.Ba + L.bw;
    L.Bb = L.La + md;                    // heavy: the per-task code bytes (md bytes)
    L.Bl = L.Bb + (md + 3) / 4;
    const int cta_words = L.Bl + kWarps * L.lw;
    // warp-mode slots (per warp: Ba[bw] | La[kWL] | N[32] | M[4] | FL[kFW]) overlay La .. Bl
    L.W = L.La;
    L.ws = L.bw + kWL + 32 + 4 + kFW;
    const int warp_words = L.W + kWarps * L.ws;
    const int light_words = kWarps * kLightWords;
    const int hist_words = kWarps * C;
    const int budget_words = (104 * 1024) / 4 - hist_words;   // keep 2 CTAs per SM
    const int heavy_words = std::max(cta_words, warp_words);
    L.wm = heavy_words <= budget_words && !force_global;   // warp mode only with the heavy buffers in smem
    const int hw = L.wm ? heavy_words : cta_words;
    heavy_in_smem = hw <= budget_words && !force_global;
    const int region = std::max(light_words, heavy_in_smem ? hw : 0);
    L.light = 0;
    L.hist = region;
    L.total = region + hist_words;
    per_cta_words = heavy_in_smem ? 0 : hw;
    return L;
}

}  // namespace

#if !VDMC_ACC32   // graph-level host code: compiled once (enum.cu), not in enum32.cu
// S3 (device copies of the class LUTs) + S4 schedule, built once per graph at the end of a build:
// heavy / light work lists and the induced adjacency of every heavy root's N+(r).
vdmc_status build_schedule(vdmc_graph *g, cudaStream_t s) {
    for (int kind = 0; kind < 2; kind++)
        for (int k4 = 0; k4 < 2; k4++) {
            const size_t nm = k4 ? 4096 : 64;
            VDMC_CUDA(dalloc((void **)&g->lut[kind][k4], nm, s));
            VDMC_CUDA(cudaMemcpyAsync(g->lut[kind][k4], host_lut(k4 ? 4 : 3, kind), nm, cudaMemcpyHostToDevice, s));
        }
    const int64_t n = g->n, T = g->ntasks;
    char *fh = nullptr, *fl = nullptr, *ft = nullptr;
    int64_t *nsel = nullptr;
    unsigned long long *ctr = nullptr;
    VDMC_CUDA(dalloc((void **)&fh, std::max<int64_t>(n, 1), s));
    VDMC_CUDA(dalloc((void **)&fl, std::max<int64_t>(n, 1), s));
    VDMC_CUDA(dalloc((void **)&ft, std::max<int64_t>(T, 1), s));
    VDMC_CUDA(dalloc((void **)&nsel, sizeof(int64_t) * 2, s));
    VDMC_CUDA(dalloc((void **)&ctr, sizeof(unsigned long long) * 2, s));
    VDMC_CUDA(dalloc((void **)&g->light_root, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    VDMC_CUDA(dalloc((void **)&g->heavy_task, sizeof(int32_t) * std::max<int64_t>(T, 1), s));
    VDMC_CUDA(dalloc((void **)&g->hroots, sizeof(int32_t) * std::max<int64_t>(n, 1), s));
    VDMC_CUDA(dalloc((void **)&g->hbase, sizeof(int64_t) * std::max<int64_t>(n, 1), s));
    int64_t hn[2] = {0, 0};
    int64_t nhr = 0;
    if (n > 0 && T > 0) {
        k_root_flags<<<148 * 8, 256, 0, s>>>(n, g->off, g->tfirst, fh, fl);
        VDMC_LAUNCH();
        k_task_flags<<<148 * 8, 256, 0, s>>>(T, g->task_root, fh, ft);
        VDMC_LAUNCH();
        thrust::counting_iterator<int32_t> ids(0);
        size_t tb = 0, tb2 = 0, tb3 = 0;
        VDMC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, ids, ft, g->heavy_task, nsel, (int)T, s));
        VDMC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb2, ids, fl, g->light_root, nsel + 1, (int)n, s));
        VDMC_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, ids, fh, g->hroots, nsel, (int)n, s));
        void *ts = nullptr;
        VDMC_CUDA(dalloc((void **)&ts, std::max(tb, std::max(tb2, tb3)), s));
        VDMC_CUDA(cub::DeviceSelect::Flagged(ts, tb, ids, ft, g->heavy_task, nsel, (int)T, s));
        VDMC_CUDA(cub::DeviceSelect::Flagged(ts, tb2, ids, fl, g->light_root, nsel + 1, (int)n, s));
        VDMC_CUDA(cudaMemcpyAsync(hn, nsel, sizeof hn, cudaMemcpyDeviceToHost, s));
        VDMC_CUDA(cub::DeviceSelect::Flagged(ts, tb3, ids, fh, g->hroots, nsel, (int)n, s));
        VDMC_CUDA(cudaMemcpyAsync(&nhr, nsel, sizeof nhr, cudaMemcpyDeviceToHost, s));
        count_launch(3);
        VDMC_CUDA(cudaStreamSynchronize(s));
        dfree(ts, s);
    }
    g->nheavy = hn[0];
    g->nlight = hn[1];
    g->nhroots = nhr;
    if (g->nlight > 0) {   // light items: each light root's tasks in chunks of <= kLightChunk
        const int64_t nl = g->nlight;
        int64_t *cnt = nullptr, *base = nullptr;
        VDMC_CUDA(dalloc((void **)&cnt, sizeof(int64_t) * (nl + 1), s));
        VDMC_CUDA(dalloc((void **)&base, sizeof(int64_t) * (nl + 1), s));
        VDMC_CUDA(cudaMemsetAsync(cnt + nl, 0, sizeof(int64_t), s));
        k_light_parts<<<148 * 4, 256, 0, s>>>(nl, g->light_root, g->tfirst, cnt);
        VDMC_LAUNCH();
        size_t tb = 0;
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, base, (int)(nl + 1), s));
        void *ts = nullptr;
        VDMC_CUDA(dalloc((void **)&ts, tb, s));
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(ts, tb, cnt, base, (int)(nl + 1), s));
        count_launch(1);
        int64_t nitems = 0;
        VDMC_CUDA(cudaMemcpyAsync(&nitems, base + nl, sizeof nitems, cudaMemcpyDeviceToHost, s));
        VDMC_CUDA(cudaStreamSynchronize(s));
        int32_t *iroot = nullptr;
        VDMC_CUDA(dalloc((void **)&iroot, sizeof(int32_t) * nitems, s));
        VDMC_CUDA(dalloc((void **)&g->light_i0, sizeof(int32_t) * nitems, s));
        k_light_scatter<<<148 * 4, 256, 0, s>>>(nl, g->light_root, cnt, base, iroot, g->light_i0);
        VDMC_LAUNCH();
        dfree(g->light_root, s);
        g->light_root = iroot;
        g->nlight = nitems;
        dfree(ts, s);
        dfree(cnt, s);
        dfree(base, s);
    }
    if (nhr > 0) {
        int64_t *dlist = nullptr, *segs = nullptr;
        VDMC_CUDA(dalloc((void **)&dlist, sizeof(int64_t) * (nhr + 1), s));
        VDMC_CUDA(dalloc((void **)&segs, sizeof(int64_t) * (nhr + 1), s));
        VDMC_CUDA(cudaMemsetAsync(dlist + nhr, 0, sizeof(int64_t), s));
        k_heavy_d<<<148 * 4, 256, 0, s>>>(nhr, g->hroots, g->off, g->split, dlist);
        VDMC_LAUNCH();
        size_t tb = 0;
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, dlist, segs, (int)(nhr + 1), s));
        void *ts = nullptr;
        VDMC_CUDA(dalloc((void **)&ts, tb, s));
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(ts, tb, dlist, segs, (int)(nhr + 1), s));
        count_launch(1);
        k_scatter_hbase<<<148 * 4, 256, 0, s>>>(nhr, g->hroots, segs, g->hbase);
        VDMC_LAUNCH();
        int64_t sumD = 0;
        VDMC_CUDA(cudaMemcpyAsync(&sumD, segs + nhr, sizeof sumD, cudaMemcpyDeviceToHost, s));
        {   // hub prefix: heavy tasks of the leading roots of degree > kHubDeg (fetched in smaller chunks)
            unsigned long long *firstq = nullptr;
            VDMC_CUDA(dalloc((void **)&firstq, sizeof(unsigned long long), s));
            const unsigned long long init = (unsigned long long)nhr;
            VDMC_CUDA(cudaMemcpyAsync(firstq, &init, sizeof init, cudaMemcpyHostToDevice, s));
            k_hub_prefix<<<148, 256, 0, s>>>(nhr, g->hroots, g->off, firstq);
            VDMC_LAUNCH();
            unsigned long long q = 0;
            VDMC_CUDA(cudaMemcpyAsync(&q, firstq, sizeof q, cudaMemcpyDeviceToHost, s));
            VDMC_CUDA(cudaStreamSynchronize(s));
            int64_t ht = 0;
            VDMC_CUDA(cudaMemcpy(&ht, segs + q, sizeof ht, cudaMemcpyDeviceToHost));
            g->hub_tasks = ht;
            dfree(firstq, s);
        }
        VDMC_CUDA(cudaStreamSynchronize(s));
        dfree(ts, s);
        // counts -> offsets -> entries
        int64_t *cnt = nullptr;
        VDMC_CUDA(dalloc((void **)&cnt, sizeof(int64_t) * (sumD + 1), s));
        VDMC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (sumD + 1), s));
        VDMC_CUDA(dalloc((void **)&g->nr_off, sizeof(int64_t) * (sumD + 1), s));
        const int cap = (int)std::min<int64_t>(g->max_degree, 12288);
        const size_t sm = (size_t)std::max(cap, 1) * 4;
        VDMC_CUDA(cudaFuncSetAttribute(k_nr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        VDMC_CUDA(cudaFuncSetAttribute(k_nr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        VDMC_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
        k_nr<false><<<148 * 2, 512, sm, s>>>(g->off, g->split, g->adj, g->hroots, nhr, g->hbase, cnt, nullptr,
                                            nullptr, ctr, cap);
        VDMC_LAUNCH();
        size_t tb2 = 0;
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, cnt, g->nr_off, (int)(sumD + 1), s));
        void *ts2 = nullptr;
        VDMC_CUDA(dalloc((void **)&ts2, tb2, s));
        VDMC_CUDA(cub::DeviceScan::ExclusiveSum(ts2, tb2, cnt, g->nr_off, (int)(sumD + 1), s));
        count_launch(1);
        VDMC_CUDA(cudaMemcpyAsync(&g->nr_total, g->nr_off + sumD, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VDMC_CUDA(cudaStreamSynchronize(s));
        VDMC_CUDA(dalloc((void **)&g->nr_adj, sizeof(uint32_t) * std::max<int64_t>(g->nr_total, 1), s));
        k_nr<true><<<148 * 2, 512, sm, s>>>(g->off, g->split, g->adj, g->hroots, nhr, g->hbase, nullptr, g->nr_off,
                                           g->nr_adj, ctr + 1, cap);
        VDMC_LAUNCH();
        dfree(ts2, s);
        dfree(cnt, s);
        dfree(dlist, s);
        dfree(segs, s);
    }
    dfree(fh, s);
    dfree(fl, s);
    dfree(ft, s);
    dfree(nsel, s);
    dfree(ctr, s);
    return VDMC_OK;
}

vdmc_status plan_prefix(const vdmc_graph *g, int k, int64_t *prefix_host, cudaStream_t s) {
    if (g->ntasks <= 0) return VDMC_OK;
    int64_t *raw = nullptr, *pre = nullptr, *s2 = nullptr, *fsum = nullptr;
    VDMC_CUDA(dalloc((void **)&raw, sizeof(int64_t) * g->ntasks, s));
    VDMC_CUDA(dalloc((void **)&pre, sizeof(int64_t) * g->ntasks, s));
    VDMC_CUDA(dalloc((void **)&s2, sizeof(int64_t) * std::max<int64_t>(g->n, 1), s));
    VDMC_CUDA(dalloc((void **)&fsum, sizeof(int64_t) * g->ntasks, s));
    size_t tb = 0;
    VDMC_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, raw, pre, (int)g->ntasks, s));
    void *ts = nullptr;
    VDMC_CUDA(dalloc((void **)&ts, tb, s));
    k_s2<<<148 * 16, 256, 0, s>>>(g->n, g->off, g->adj, s2);
    VDMC_LAUNCH();
    k_task_deg<<<148 * 8, 256, 0, s>>>(g->ntasks, g->off, g->split, g->adj, g->tfirst, g->task_root, raw);
    VDMC_LAUNCH();
    VDMC_CUDA(cub::DeviceScan::InclusiveSum(ts, tb, raw, fsum, (int)g->ntasks, s));
    count_launch(1);
    k_cost<<<148 * 8, 256, 0, s>>>(g->ntasks, k, g->off, g->split, g->adj, g->tfirst, g->task_root, s2, fsum, raw);
    VDMC_LAUNCH();
    VDMC_CUDA(cub::DeviceScan::InclusiveSum(ts, tb, raw, pre, (int)g->ntasks, s));
    count_launch(1);
    dfree(s2, s);
    dfree(fsum, s);
    VDMC_CUDA(cudaMemcpyAsync(prefix_host, pre, sizeof(int64_t) * g->ntasks, cudaMemcpyDeviceToHost, s));
    VDMC_CUDA(cudaStreamSynchronize(s));
    dfree(ts, s);
    dfree(raw, s);
    dfree(pre, s);
    return VDMC_OK;
}

#endif  // !VDMC_ACC32

namespace {
struct Events {   // per-call timing events (only when the caller asks for timings)
    cudaEvent_t e[4] = {};
    ~Events() {
        for (auto x : e)
            if (x) cudaEventDestroy(x);
    }
};
}  // namespace

template <int K, int C>
static vdmc_status run(const vdmc_graph *g, const uint8_t *lut, const CountOpts &o, AccT *acc,
                       int64_t lo, int64_t hi, cudaStream_t s, float *ms3) {
    const int dev = g->device;
    int nsm = 0;
    VDMC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (g->max_degree >= (int64_t(1) << 21))
        return fail(VDMC_EINVAL, "max degree %lld >= 2^21 is not supported", (long long)g->max_degree);
    Events ev;
    if (ms3)
        for (auto &x : ev.e) VDMC_CUDA(cudaEventCreate(&x));
    if (ms3) VDMC_CUDA(cudaEventRecord(ev.e[0], s));
    bool heavy_in_smem = true;
    int64_t per_cta = 0;
    const Layout L = make_layout((int)g->max_degree, C, heavy_in_smem, per_cta, o.heavy_global != 0);
    const size_t smem = (size_t)L.total * 4;
    auto kern = heavy_in_smem ? k_enum<K, C, true> : k_enum<K, C, false>;
    VDMC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    VDMC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, smem));
    const int grid = std::max(1, nsm * std::max(per_sm, 1));
    // per-call scratch: heavy per-CTA buffers (global fallback), light per-warp oversize L_a,
    // per-CTA CA lists of the cross items; work counters
    const int64_t per_warp = (int64_t)g->max_degree + (g->max_degree + 15) / 16 + 1;
    const uint32_t ca_cap = o.ca_capacity > 0 ? (uint32_t)o.ca_capacity : (1u << 16);
    const int64_t per_cta_ca = 2 * (int64_t)std::max<int64_t>(g->max_degree, 1) + ca_cap;
    const size_t need = (size_t)grid * (per_cta + (int64_t)kWarps * per_warp + per_cta_ca);
    uint32_t *scratch = nullptr;
    unsigned long long *ctr = nullptr;
    VDMC_CUDA(dalloc((void **)&scratch, need * sizeof(uint32_t), s));
    VDMC_CUDA(dalloc((void **)&ctr, 2 * sizeof(unsigned long long), s));
    VDMC_CUDA(cudaMemsetAsync(acc, 0, (size_t)std::max<int64_t>(g->n, 1) * C * sizeof(AccT), s));
    VDMC_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), s));
    if (ms3) VDMC_CUDA(cudaEventRecord(ev.e[1], s));
    trace("scratch+memset");
    Dev d{};
    d.off = g->off;
    d.split = g->split;
    d.adj = g->adj;
    d.tfirst = g->tfirst;
    d.task_root = g->task_root;
    d.heavy_task = g->heavy_task;
    d.light_root = g->light_root;
    d.light_i0 = g->light_i0;
    d.nheavy = g->nheavy;
    d.nlight = g->nlight;
#ifdef VDMC_PROFILING
    // profiling build only (tools/): switches that drop work, results incomplete
    if (const char *ph = getenv("VDMC_PHASES")) {   // 1 = heavy phase only, 2 = light only
        if (ph[0] == '1') d.nlight = 0;
        if (ph[0] == '2') d.nheavy = 0;
    }
    if (const char *sk = getenv("VDMC_SKIP")) d.skip = atoi(sk);
    if (const char *mr = getenv("VDMC_MINREM")) d.minrem = atoi(mr);
#endif
    d.fold = o.star_block;   // 0 = per-task block length
    d.xblock = o.cross_block > 0 ? o.cross_block : kCrossBlock;
    d.acc = acc;
    d.ns = (uint32_t)std::max<int64_t>(g->n, 1);
    d.gheavy = scratch;
    d.glight = scratch + (size_t)grid * per_cta;
    d.gca = scratch + (size_t)grid * (per_cta + (int64_t)kWarps * per_warp);
    d.gca_per_cta = per_cta_ca;
    d.ca_cap = ca_cap;
    d.gheavy_per_cta = per_cta;
    d.glight_per_warp = per_warp;
    d.heavy_in_smem = heavy_in_smem ? 1 : 0;
    d.big = (g->max_degree > 32767 || o.force_big) ? 1 : 0;
    d.maxdeg = (int)g->max_degree;
    d.off32 = (uint64_t)std::max<int64_t>(g->n, 1) * C < (1ull << 32) ? 1 : 0;
    d.hbase = g->hbase;
    d.hub_tasks = g->hub_tasks;
    d.nr_off = g->nr_off;
    d.nr_adj = g->nr_adj;
    // k = 4 closed form at heavy roots: the "2+1" R[j] side per root (k_rside) from the tasks' M
    const bool rside = K == 4 && o.star_block <= 0 && g->nheavy > 0 && g->nhroots > 0;
    uint32_t *gM = nullptr;
    if (rside) VDMC_CUDA(dalloc((void **)&gM, (size_t)g->nheavy * 4 * sizeof(uint32_t), s));
    d.gM = gM;
    if (hi > lo) {
        kern<<<grid, kBlock, smem, s>>>(d, L, lo, hi, ctr, lut);
        VDMC_LAUNCH();
        if (rside) {
            const int rg = (int)std::min<int64_t>(g->nhroots, (int64_t)nsm * 8);
            k_rside<C><<<rg, 256, 0, s>>>(d, g->hroots, g->nhroots, lo, hi, lut);
            VDMC_LAUNCH();
        }
    }
    if (gM) dfree(gM, s);
    if (ms3) VDMC_CUDA(cudaEventRecord(ev.e[2], s));
    dfree(scratch, s);
    dfree(ctr, s);
    if (ms3) {
        VDMC_CUDA(cudaEventSynchronize(ev.e[2]));
        VDMC_CUDA(cudaEventElapsedTime(&ms3[0], ev.e[0], ev.e[1]));
        VDMC_CUDA(cudaEventElapsedTime(&ms3[1], ev.e[1], ev.e[2]));
    }
    trace("enum enqueued");
    return VDMC_OK;
}

#if VDMC_ACC32
#define VDMC_COUNT_INTO count_into32
#define VDMC_FINALIZE finalize32
#else
#define VDMC_COUNT_INTO count_into
#define VDMC_FINALIZE finalize
#endif

vdmc_status VDMC_COUNT_INTO(const vdmc_graph *g, int k, const CountOpts &o, AccT *acc, int64_t lo, int64_t hi,
                            cudaStream_t s, float *ms3) {
    const uint8_t *lut = g->lut[o.kind][k == 4 ? 1 : 0];
    if (o.kind == VDMC_UNDIRECTED)
        return k == 3 ? run<3, kNumClassesU3>(g, lut, o, acc, lo, hi, s, ms3)
                      : run<4, kNumClassesU4>(g, lut, o, acc, lo, hi, s, ms3);
    return k == 3 ? run<3, kNumClasses3>(g, lut, o, acc, lo, hi, s, ms3)
                  : run<4, kNumClasses4>(g, lut, o, acc, lo, hi, s, ms3);
}

template <int C>
static void launch_finalize(int64_t n, const int32_t *order, const AccT *acc, uint64_t *counts, int nsm,
                            cudaStream_t s) {
    const unsigned fg = (unsigned)std::min<int64_t>((n + kFinV - 1) / kFinV, (int64_t)nsm * 8);
    k_finalize<C><<<fg, 256, 0, s>>>(n, order, acc, (unsigned long long *)counts);
}

vdmc_status VDMC_FINALIZE(const vdmc_graph *g, int C, const AccT *acc, uint64_t *counts, cudaStream_t s) {
    if (g->n <= 0) return VDMC_OK;
    int nsm = 0;
    VDMC_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, g->device));
    switch (C) {
        case kNumClasses3: launch_finalize<kNumClasses3>(g->n, g->order, acc, counts, nsm, s); break;
        case kNumClasses4: launch_finalize<kNumClasses4>(g->n, g->order, acc, counts, nsm, s); break;
        case kNumClassesU3: launch_finalize<kNumClassesU3>(g->n, g->order, acc, counts, nsm, s); break;
        case kNumClassesU4: launch_finalize<kNumClassesU4>(g->n, g->order, acc, counts, nsm, s); break;
        default: return fail(VDMC_EINVAL, "no finalize for C=%d", C);
    }
    VDMC_LAUNCH();
    return VDMC_OK;
}

}  // namespace vdmc
