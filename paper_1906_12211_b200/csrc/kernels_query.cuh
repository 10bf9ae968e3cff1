// kernels_query.cuh — the batched adaptive query (Alg. 1 over the array index of
// PAPER.md:281-334 §4.1-4.2) and the shard merge.
//
// One warp per query, persistent grid, queries taken from an atomic work counter.  Per warp:
//  levels i = K..1, repetitions in chunks of R (R-17: the filter threshold tau is
//  frozen per chunk; candidates are claimed in (repetition, position) order so the evaluated
//  set and the stop point equal the sequential algorithm's):
//   a7/a8  prefix ranges: for each repetition of the chunk, the match range [a_i, b_i) of the
//          query's i-bit prefix via the 13-bit prefix table + binary search in its bucket
//          (PAPER.md:310-311); the emitted range grows by whole segments of B (PAPER.md:319,
//          934) in closed form: elo' = elo - B*ceil((elo - a_i)/B), ehi' = ehi + B*ceil((b_i - ehi)/B)
//          (clamped to [0,n)) -- the same positions as the oracle's segment loop (R-12).
//   a9     sketch filter popcount(s'(q) ^ s'(p)) <= tau
//   a10    dedupe: per-query bitmap of evaluated ids in global scratch (atomicOr claims)
//   a11    exact inner product: lane per survivor, sequential fmaf over t, 128-bit row loads
//   a12    top-k: sorted keys (sim desc, id asc) in shared memory, rank-merge of sorted batches
//   a13    stop test after every repetition: k-th similarity >= host-computed threshold T[i][j]
//  i = 0: linear scan of every not-yet-evaluated point, then stop (R-13).
#pragma once
#include "device_common.cuh"
#include "../../include/pfg.h"

namespace pfg {

#ifndef PFG_HC
#define PFG_HC 2048
#endif
#ifndef PFG_SB
#define PFG_SB 192
#endif
#ifndef PFG_MINB
#define PFG_MINB 4
#endif
constexpr int kHC = PFG_HC;   // per-warp shared-memory hash set of evaluated ids (slots)
constexpr int kHMax = kHC * 3 / 4;  // beyond this many evaluated ids a query switches to the global bitmap
constexpr int kSB = PFG_SB;   // survivor buffer (evaluated ids awaiting their similarity)
constexpr int kRPI = 16;      // candidate rows read per warp step of k_sims (rows in flight: the kernel's bound)
constexpr int kU = 4;         // table positions per lane per scan step
constexpr int kMaxR = 32;     // max repetitions per chunk
constexpr int kMaxK = 256;    // max k
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kJHist = 256;

// one repetition-table entry (16 B): key = (code << 32) | id, sk = sketch word s_{slot(j)}(id)
struct __align__(16) Entry {
    uint64_t key;
    uint64_t sk;
};

// Per-query search state in global memory, shared by the round engine (kernels_rounds.cuh) and
// the fused kernel (which can resume a query from it).
struct RoundCtl {
    uint32_t nact[2];      // active-list counts (round parity)
    uint32_t pool_top[2];  // survivor-pool fill (round parity)
    uint32_t nfused;       // queries handed to the fused kernel
    uint32_t ntiles[2];    // scan tiles of the round (round parity)
    uint32_t pad;
    uint32_t wk[2][4];     // work counters of k_expand, k_scan, k_dedupe, k_merge (round parity)
    uint32_t dfront[2], dback[2];  // k_dedupe's order: long chunks from the front, the rest from the back
    // wide queries (evaluated set in a visit-tag array instead of the shared-memory hash set)
    uint32_t nwt[2];       // wide scan tiles of the round (round parity)
    uint32_t nwide[2];     // wide queries in the active list (round parity)
    uint32_t wnext;        // visit-tag arrays handed out in this search
    uint32_t loop;         // 1 while the device-side round loop runs (k_merge hands off to fused2)
    uint32_t nfused2;      // queries handed to the fused kernel during the loop
    uint32_t round;        // rounds run by the loop
    uint32_t wtag;         // the search's epoch tag (high half of every visit tag)
    uint32_t wdefer;       // wide chunks deferred for want of wide tiles (the host grows the buffer)
    uint32_t pad2;
    unsigned long long evsum, emsum;  // evaluated ids and emitted positions of the finished queries
    unsigned long long sims_rows;     // pool rows the bulk k_sims launches computed
    unsigned long long sims_rows_blind;  // of these, the rows of the launches outside the device-side loop
};
struct RoundState {
    int32_t* lvl;       // [nq] next level i to process (K..1); 0 = only the i = 0 scan remains
    int32_t* c0;        // [nq] next chunk start at that level
    int32_t* flags;     // [nq] bit0 done, bit1 hand off to the fused kernel
    int32_t* tn;        // [nq] entries in the top list
    uint32_t* cnt;      // [nq][8] emitted, filtered, dups, evaluated, probes
    uint64_t* T;        // [nq][kt] top list keys
    uint32_t* E;        // [nq][Ecap] evaluated ids in evaluation order
    uint4* pend;        // [nq][kMaxR] cursors of the chunk in flight (committed by k_merge)
    uint32_t* cand;     // [nq][Ccap] candidate id per emitted position of the chunk (kEmpty = filtered)
    uint32_t* tcnt;     // [nq][Ccap/kTile] per scan tile: candidates passing the filter | repetition << 16
    uint32_t* hsave;    // [nq][kHC] k_dedupe's hash set carried to the next round
    uint4* rinfo;       // [nq] {chunk repetitions, tau, scan tiles, direct}
    uint4* tiles;       // scan tile descriptors, two uint4 each (k_expand -> k_scan)
    uint32_t* repcnt;   // [nq][kMaxR][3] emitted, filtered, dups per repetition of the chunk
    uint32_t* pool_id;  // survivor pool of the round: ids, owning query, (sim, id) keys
    uint32_t* pool_q;
    uint64_t* pool_key;
    uint32_t* poff;     // [nq] first pool entry of the query
    uint32_t* pn;       // [nq] pool entries of the query
    uint32_t* act[2];   // [nq] active lists (round parity)
    uint32_t* dord[2];  // [nq] the active list reordered for k_dedupe (long chunks first)
    uint32_t* fused;    // [nq] queries handed to the fused kernel
    uint32_t* fused2;   // [nq] queries handed to the fused kernel during the device-side loop
    RoundCtl* ctl;
    int Ecap, Ccap;
    uint32_t pool_cap;
    // wide queries (kernels_rounds.cuh): per query a visit-tag array W[n] (slot wslot[q]); a
    // passing candidate of visit (i, j) does atomicMin(W[id], tag(i, j)) and is fresh iff W[id]
    // ends equal to its own tag, i.e. no earlier visit (earlier chunk, or earlier repetition of
    // the same chunk) passed it.  Tags carry the search epoch in the high half, so no reset is
    // needed between searches.
    uint32_t* wv;       // [wslots][n] visit tags
    uint32_t* wslot;    // [nq] the query's visit-tag array
    uint4* wtiles;      // wide scan tile descriptors (two uint4 each)
    uint32_t* wcand;    // [wcap][kTile] per wide tile: passing candidates, then the fresh ids in order
    float* wsim;        // [wcap][kTile] similarities of the fresh ids
    uint32_t* wtcnt;    // [wcap] fresh | passing << 8 | repetition << 16 | kept << 24
    uint32_t* rtile;    // [nq][kMaxR + 1] first wide tile of each repetition of the chunk, then the end
    uint32_t wslots, wcap, hmax;  // hmax: evaluated ids a query keeps in the hash set before it widens
    uint32_t pool_stride;         // chunk engine: the pool of round parity par starts at par * pool_stride
};
constexpr int kCnt = 8;

struct QueryParams {
    int64_t n, nq, bm_words, id_offset;
    int d, dpad, K, L, M, B, R, k, k_eff, per_round, use_filter, c, ell, dp, lazy, claim_cap, trace_cap;
    int kt;          // T capacity (>= k_eff, multiple of 32)
    int qc_n, qc_ld; // query codes precomputed for repetitions [0, qc_n), row stride qc_ld
    int qb_n, qb_ld; // level-K match ranges precomputed for repetitions [0, qb_n) (k_qbounds)
    int uniform;     // 1: chunks of R from the start; 0: the first chunk is repetition 0 alone
    int tensor_s;    // tensor strategy: S = sqrt(L) tuples per collection (0 = not tensor)
    int lstep;       // bits between searched depths: 1, or 2 ell for the tensor strategy
    int smem_warp;   // bytes of shared memory per warp
    const float* __restrict__ x;
    const int16_t* __restrict__ x16;   // PFG_STORAGE_I16 rows [n][dpad16] (x is then NULL), R-25
    const int16_t* __restrict__ qx16;  // the queries' int16 rows [nq][dpad16]
    int dpad16;
    const Entry* __restrict__ tab;
    const uint32_t* __restrict__ pt;
    const uint8_t* __restrict__ slot;
    const float* __restrict__ qx;
    const uint64_t* __restrict__ qsk;
    const uint32_t* __restrict__ qcodes;
    const uint4* __restrict__ qbnd;  // [nq][qb_ld] {a_K, b_K, probes, 0} of repetition j
    const uint32_t* __restrict__ sg;
    const uint8_t* __restrict__ qzero;
    const float* __restrict__ thr;   // [K][L]
    const float* __restrict__ taub;  // [65]
    unsigned long long* work;
    uint4* cur;
    uint32_t* bitmap;
    uint32_t* claims;
    int64_t* out_ids;
    float* out_sims;
    pfg_query_stats* stats;
    uint32_t* trace_ids;
    unsigned long long* prof;   // optional per-phase cycle counters (PFG_PHASE_PROF=1), [6]
    uint32_t* jhist;            // [kJHist] queries by stop repetition at level K (eager-depth tuning)
    const uint32_t* qlist;      // fused kernel: query indices to process (NULL = 0..nq-1)
    const uint32_t* nq_dev;     // fused kernel: if set, the number of queries in qlist (device)
    int resume;                 // fused kernel: continue each query from rs
    RoundState rs;
};

// Per-warp shared memory: a fixed-size part at compile-time offsets, then the query row, its
// sketches and the two top-k buffers (sizes known at launch).
struct WarpFixed {
    uint32_t hs[kHC];          // hash set of evaluated ids
    uint32_t sid[kSB];         // survivors awaiting their similarity (repetition order)
    float ssim[kSB];
    uint64_t cand[32];         // sorted merge batch
    uint32_t beg[kMaxR + 4];   // exclusive prefix of per-repetition emitted counts
    uint32_t lo_new[kMaxR];
    uint32_t lo_old[kMaxR];
    uint32_t hi_old[kMaxR];
    uint32_t qc[kMaxR];        // query codes of the chunk
    uint32_t bnd[2 * kMaxR];   // a / b bounds
    uint32_t fcnt[kMaxR];      // filtered per repetition
    uint32_t dcnt[kMaxR];      // duplicates per repetition
    uint8_t srep[kSB];
};

struct WarpSmem {
    WarpFixed* f;
    float* qrow;       // [dpad]
    uint64_t* qsk;     // [M]
    uint64_t* T0;      // [kt]
    uint64_t* T1;      // [kt]
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

__host__ __device__ inline int warp_smem_bytes(int dpad, int M, int kt) {
    return align16((int)sizeof(WarpFixed)) + align16(dpad * 4) + align16(M * 8) + 2 * align16(kt * 8);
}

__device__ inline WarpSmem carve(unsigned char* base, const QueryParams& p) {
    WarpSmem w;
    unsigned char* q = base;
    w.f = (WarpFixed*)q; q += align16((int)sizeof(WarpFixed));
    w.qrow = (float*)q; q += align16(p.dpad * 4);
    w.qsk = (uint64_t*)q; q += align16(p.M * 8);
    w.T0 = (uint64_t*)q; q += align16(p.kt * 8);
    w.T1 = (uint64_t*)q;
    return w;
}

__device__ __forceinline__ uint32_t entry_code(const Entry* e) {
    return __ldg(reinterpret_cast<const uint32_t*>(e) + 1);
}

// first position of repetition j whose K-bit code is >= x (x <= 2^K; 2^K -> n)
__device__ __forceinline__ uint32_t rep_lower_bound(const QueryParams& p, int j, uint64_t x, uint32_t& probes) {
    if (x >= (1ull << p.K)) return (uint32_t)p.n;
    const uint32_t xs = (uint32_t)x;
    const int sh = p.K - 13;
    const uint32_t* ptj = p.pt + (int64_t)j * 8193;
    const uint32_t pfx = xs >> sh;
    uint32_t lo = __ldg(ptj + pfx), hi = __ldg(ptj + pfx + 1);
    if ((x & ((1ull << sh) - 1)) == 0) return lo;
    const Entry* tj = p.tab + (int64_t)j * p.n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        ++probes;
        if (entry_code(tj + mid) < xs) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// R-12 segment widening of one side of repetition j's emitted range at level i < K: the oracle's
// loop (step B outward while the boundary entry shares the query's i-bit prefix), literally for
// its first kWidenSteps probes (short ranges, the common case at high levels), then in closed
// form: the prefix range end a_i / b_i from the prefix table and a bucket search (O(1) for
// i <= 13), and
//   left  e' = e - B*ceil((e - a_i)/B), or 0 if that is <= 0
//   right e' = min(n, e + B*ceil((b_i - e)/B))
// -- the loop's positions, since the entries sharing the prefix are exactly [a_i, b_i).
#ifndef PFG_WIDEN_STEPS
#define PFG_WIDEN_STEPS 4
#endif
constexpr int kWidenSteps = PFG_WIDEN_STEPS;
__device__ __forceinline__ uint32_t widen_side(const QueryParams& p, int j, int i, uint32_t code, uint32_t e, bool left,
                                               uint32_t& probes) {
    const Entry* tj = p.tab + (int64_t)j * p.n;
    const int sh = p.K - i;
    const uint32_t qp = code >> sh;
    const uint32_t B = (uint32_t)p.B, n = (uint32_t)p.n;
    if (left) {
        for (int t = 0; t < kWidenSteps; ++t) {
            if (e == 0) return 0u;
            ++probes;
            if ((entry_code(tj + e - 1) >> sh) != qp) return e;
            e = e > B ? e - B : 0u;
        }
        if (e == 0) return 0u;
        const uint32_t a = rep_lower_bound(p, j, (uint64_t)qp << sh, probes);
        if (a >= e) return e;
        const uint64_t m = (e - a + B - 1) / B;
        return (uint64_t)B * m >= e ? 0u : e - (uint32_t)(B * m);
    }
    for (int t = 0; t < kWidenSteps; ++t) {
        if (e >= n) return n;
        ++probes;
        if ((entry_code(tj + e) >> sh) != qp) return e;
        e = (uint64_t)e + B < (uint64_t)n ? e + B : n;
    }
    if (e >= n) return n;
    const uint32_t b = rep_lower_bound(p, j, ((uint64_t)qp + 1) << sh, probes);
    if (b <= e) return e;
    const uint64_t v = (uint64_t)e + (uint64_t)B * ((b - e + B - 1) / B);
    return v > n ? n : (uint32_t)v;
}

struct QState {
    int tn;               // entries in T (<= k_eff)
    uint32_t nE;          // evaluated (merged) ids
    uint32_t emitted, filtered, dups, probes, flags;
    uint32_t claims_n;    // ids recorded in the global bitmap (bitmap mode)
    uint32_t hcount;      // ids in the shared hash set
    bool bitmap_mode;
    uint64_t* T;          // current sorted top list
    uint64_t* Tn;         // scratch buffer
};

// merge survivors [e, e2) of sid/ssim into the sorted top list
__device__ __forceinline__ void merge_range(const QueryParams& p, const WarpSmem& w, QState& st, int e, int e2,
                                            int64_t qi, int lane) {
    for (int b0 = e; b0 < e2; b0 += 32) {
        const int idx = b0 + lane;
        uint64_t key = 0;
        if (idx < e2) {
            const uint32_t id = w.f->sid[idx];
            key = make_key(w.f->ssim[idx], id);
            if (p.trace_cap > 0) {
                const uint32_t pos = st.nE + (uint32_t)(idx - e);
                if (pos < (uint32_t)p.trace_cap) p.trace_ids[qi * p.trace_cap + pos] = id;
            }
        }
        const uint64_t kth = (st.tn == p.k_eff) ? st.T[p.k_eff - 1] : 0ull;
        if (key <= kth) key = 0;
        const uint32_t vm = __ballot_sync(kFull, key != 0);
        if (vm) {
            key = warp_sort_desc(key, lane);
            const int nc = __popc(vm);
            w.f->cand[lane] = key;
            __syncwarp();
            if (lane < nc) {
                int lo = 0, hi = st.tn;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (st.T[mid] > key) lo = mid + 1; else hi = mid; }
                const int dst = lane + lo;
                if (dst < p.k_eff) st.Tn[dst] = key;
            }
            for (int t = lane; t < st.tn; t += 32) {
                const uint64_t tv = st.T[t];
                int lo = 0, hi = nc;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (w.f->cand[mid] > tv) lo = mid + 1; else hi = mid; }
                const int dst = t + lo;
                if (dst < p.k_eff) st.Tn[dst] = tv;
            }
            __syncwarp();
            st.tn = min(p.k_eff, st.tn + nc);
            uint64_t* tmp = st.T; st.T = st.Tn; st.Tn = tmp;
        }
        __syncwarp();
    }
    st.nE += (uint32_t)(e2 - e);
}

// R-17: the search's first chunk (level K, repetition 0) is a single repetition, every other chunk
// R repetitions.  It ends early at the first repetition j whose stop threshold the current
// k-th similarity already meets: the k-th similarity only grows, so the search stops at or before
// j and later repetitions of the chunk are never reached (exact).  All lanes get the same value.
// the table of repetition r of chunk c0: the repetitions c0 .. c0 + nr - 1, or for the tensor
// strategy (Alg. 2) the tries of shell c0 (0-based): (j, c0) and (c0, j) for
// j < c0 in the order (0,c0), (c0,0), (1,c0), (c0,1), ..., then (c0,c0); trie (j1, j2) = j1*S + j2
__device__ __forceinline__ int trie_of(const QueryParams& p, int c0, int r) {
    if (!p.tensor_s) return c0 + r;
    return (r & 1) ? c0 * p.tensor_s + (r >> 1) : (r >> 1) * p.tensor_s + c0;
}
__device__ __forceinline__ int chunk_count(const QueryParams& p) { return p.tensor_s ? p.tensor_s : p.L; }

__device__ __forceinline__ int chunk_reps(const QueryParams& p, int i, int c0, int tn, const uint64_t* T, int lane) {
    if (p.tensor_s) return 2 * c0 + 1;  // a shell; the stop check follows the whole shell
    int nr = min((i == p.K && c0 == 0 && !p.uniform) ? 1 : p.R, p.L - c0);
    if (tn == p.k_eff) {
        float ip = key_sim(T[p.k_eff - 1]);
        ip = fminf(fmaxf(ip, -1.0f), 1.0f);
        const bool hit = lane < nr && ip >= __ldg(p.thr + (int64_t)(i - 1) * p.L + c0 + lane);
        const uint32_t m = __ballot_sync(kFull, hit);
        if (m) nr = __ffs(m);
    }
    return nr;
}

__device__ __forceinline__ float kth_sim_clamped(const QueryParams& p, const QState& st) {
    float ip = key_sim(st.T[p.k_eff - 1]);
    return fminf(fmaxf(ip, -1.0f), 1.0f);
}

// Tree over the 32 lane sums of NR rows (R-2: level h = 16, 8, 4, 2, 1 adds lane sums l and l + h),
// computed transposed: while a lane holds more than one row, level h halves the rows it keeps (the
// lanes with bit h set keep the upper half) and adds the partner's value of the same row, so each
// addition combines the same two tree nodes as the plain tree.  Lane l ends with row
// (l >> (5 - log2 NR)) for NR <= 32.
template <int NR, typename T>
__device__ __forceinline__ T tree_rows(T (&a)[NR], int lane) {
    int m = NR;
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        if (m > 1) {
            const int half = m >> 1;
            const bool up = lane & h;
#pragma unroll
            for (int k = 0; k < NR / 2; ++k) {
                if (k < half) {
                    const float send = up ? a[k] : a[k + half];
                    const float keep = up ? a[k + half] : a[k];
                    a[k] = keep + __shfl_xor_sync(kFull, send, h);
                }
            }
            m = half;
        } else {
            a[0] = a[0] + __shfl_xor_sync(kFull, a[0], h);
        }
    }
    return a[0];
}

// Similarities of survivors [e0, e1) (R-2): the warp reads each candidate row coalesced, one 16-byte
// chunk per lane (chunk c -> lane c mod 32), each lane keeps a sequential fmaf chain, and the 32
// lane sums are added in the fixed tree h = 16, 8, 4, 2, 1 -- the oracle's or_sim order.  Zero
// padding beyond d leaves a chain unchanged (it never holds -0).  kRQ rows are in flight per step.
#ifndef PFG_KRQ
#define PFG_KRQ 8
#endif
constexpr int kRQ = PFG_KRQ;
// R-25 (PFG_STORAGE_I16): the exact integer inner product of 8 coordinates (two int16 per word);
// |partial sums| <= ||q|| ||x|| 2^30 < 2^31 (Cauchy-Schwarz), and the similarity is the int32 sum
// rounded to fp32 times 2^-30 -- exact and independent of the summation order
__device__ __forceinline__ int dot8_i16(const int4 a, const int4 b) {
    int s = (int)(short)a.x * (int)(short)b.x + (a.x >> 16) * (b.x >> 16);
    s += (int)(short)a.y * (int)(short)b.y + (a.y >> 16) * (b.y >> 16);
    s += (int)(short)a.z * (int)(short)b.z + (a.z >> 16) * (b.z >> 16);
    s += (int)(short)a.w * (int)(short)b.w + (a.w >> 16) * (b.w >> 16);
    return s;
}
__device__ __forceinline__ float sim_of_i16(int s) { return __int2float_rn(s) * 9.313225746154785e-10f; }  // 2^-30

// NR int16 rows against one query row per row (qoff, int4 units): lane c reads chunk c of each row
template <int NR, bool ONEQ>
__device__ __forceinline__ void rows_dot_i16(const int4* __restrict__ x4, const int4* __restrict__ q4,
                                             const uint32_t (&roff)[NR], const uint32_t (&qoff)[NR], int nch16,
                                             int lane, int (&acc)[NR]) {
#pragma unroll
    for (int r = 0; r < NR; ++r) acc[r] = 0;
    for (int c = lane; c < nch16; c += 32) {
        int4 v[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) v[r] = __ldg(x4 + roff[r] + c);
        int4 qv = __ldg(q4 + qoff[0] + c);
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            if (!ONEQ && r > 0) qv = __ldg(q4 + qoff[r] + c);
            acc[r] += dot8_i16(v[r], qv);
        }
    }
}

template <int RQ = kRQ>
__device__ __forceinline__ void compute_sims(const QueryParams& p, const WarpSmem& w, int e0, int e1, int lane,
                                             int64_t qi = 0) {
    if (p.x16) {
        const int nch16 = p.dpad16 >> 3;
        const int4* x4 = reinterpret_cast<const int4*>(p.x16);
        const int4* q4 = reinterpret_cast<const int4*>(p.qx16);
        uint32_t qoff[RQ];
#pragma unroll
        for (int r = 0; r < RQ; ++r) qoff[r] = (uint32_t)qi * (uint32_t)nch16;
        for (int b = e0; b < e1; b += RQ) {
            const int nrow = min(RQ, e1 - b);
            const uint32_t myoff = lane < RQ ? w.f->sid[b + (lane < nrow ? lane : nrow - 1)] * (uint32_t)nch16 : 0u;
            uint32_t off[RQ];
#pragma unroll
            for (int r = 0; r < RQ; ++r) off[r] = __shfl_sync(kFull, myoff, r);
            int acc[RQ];
            rows_dot_i16<RQ, true>(x4, q4, off, qoff, nch16, lane, acc);
            const int t = tree_rows<RQ>(acc, lane);
            constexpr int kSh = (RQ == 32) ? 0 : (RQ == 16) ? 1 : (RQ == 8) ? 2 : 3;
            const int rr = lane >> kSh;
            if ((lane & ((1 << kSh) - 1)) == 0 && rr < nrow) w.f->ssim[b + rr] = sim_of_i16(t);
        }
        __syncwarp();
        return;
    }
    const int nch = p.dpad >> 2;
    const float4* q4 = reinterpret_cast<const float4*>(w.qrow);
    const float4* x4 = reinterpret_cast<const float4*>(p.x);
    for (int b = e0; b < e1; b += RQ) {
        const int nrow = min(RQ, e1 - b);
        // lane r < RQ reads survivor b + r (rows >= nrow repeat the last)
        const uint32_t myoff = lane < RQ ? w.f->sid[b + (lane < nrow ? lane : nrow - 1)] * (uint32_t)nch : 0u;
        float acc[RQ];
        uint32_t off[RQ];   // row offsets in float4 units (n * dpad / 4 < 2^32)
#pragma unroll
        for (int r = 0; r < RQ; ++r) {
            acc[r] = 0.0f;
            off[r] = __shfl_sync(kFull, myoff, r);
        }
        for (int c = lane; c < nch; c += 32) {
            float4 v[RQ];
#pragma unroll
            for (int r = 0; r < RQ; ++r) v[r] = __ldg(x4 + off[r] + c);
            const float4 q = q4[c];
#pragma unroll
            for (int r = 0; r < RQ; ++r) {
                acc[r] = fmaf(q.x, v[r].x, acc[r]);
                acc[r] = fmaf(q.y, v[r].y, acc[r]);
                acc[r] = fmaf(q.z, v[r].z, acc[r]);
                acc[r] = fmaf(q.w, v[r].w, acc[r]);
            }
        }
        const float t = tree_rows<RQ>(acc, lane);
        constexpr int kSh = (RQ == 32) ? 0 : (RQ == 16) ? 1 : (RQ == 8) ? 2 : 3;
        const int rr = lane >> kSh;
        if ((lane & ((1 << kSh) - 1)) == 0 && rr < nrow) w.f->ssim[b + rr] = t;
    }
    __syncwarp();
}

// Process the survivor buffer (in repetition order): similarities, then merge repetition by
// repetition; every repetition < `complete` (all positions scanned) gets its stop check after its
// survivors are merged (Alg. 1 line 8).  Returns true when the query stops (r_stop set).
template <int RQ>
__device__ __forceinline__ bool drain(const QueryParams& p, const WarpSmem& w, QState& st, int& nbuf, int& next_check,
                                      int complete, int nr, int c0, int i, int64_t qi, int& r_stop, int lane) {
    const long long td0 = p.prof ? clock64() : 0;
    compute_sims<RQ>(p, w, 0, nbuf, lane, qi);
    if (p.prof && lane == 0) atomicAdd(p.prof + 5, (unsigned long long)(clock64() - td0));
    int e = 0;
    bool stop = false;
    // survivors are in repetition order: the run of repetition r ends at the first entry > r.
    // Lane t finds that end for repetition r0 + t and loads its stop threshold, all lanes at once
    // (instead of one dependent search and load per repetition in the loop below)
    const int r0 = next_check;
    int myend = 0;
    float mythr = INFINITY;
    {
        const int rt = r0 + lane;
        int lo = 0, hi = nbuf;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if (w.f->srep[mid] <= rt) lo = mid + 1; else hi = mid; }
        myend = lo;
        if (rt < nr) {
            const int col = p.tensor_s ? c0 : c0 + rt;   // tensor: thresholds per (depth, shell)
            mythr = __ldg(p.thr + (int64_t)(i - 1) * p.L + col);
        }
    }
    for (;;) {
        const int t = next_check - r0;
        int e2;
        if (t < 32) {
            e2 = __shfl_sync(kFull, myend, t);
        } else {
            int lo = e, hi = nbuf;
            while (lo < hi) { const int mid = (lo + hi) >> 1; if (w.f->srep[mid] <= next_check) lo = mid + 1; else hi = mid; }
            e2 = lo;
        }
        if (e2 > e) merge_range(p, w, st, e, e2, qi, lane);
        e = e2;
        if (next_check >= complete || next_check >= nr) break;
        const int j1 = c0 + next_check + 1;
        const bool check = p.tensor_s ? (next_check == nr - 1) : (!p.per_round || j1 == p.L);
        const float th = t < 32 ? __shfl_sync(kFull, mythr, t)
                                : __ldg(p.thr + (int64_t)(i - 1) * p.L + (p.tensor_s ? c0 : j1 - 1));
        if (st.tn == p.k_eff && check) {
            const float ip = kth_sim_clamped(p, st);
            if (ip >= th) { r_stop = next_check; stop = true; break; }
        }
        ++next_check;
    }
    nbuf = 0;
    __syncwarp();
    return stop;
}

// home slot of an id: multiplicative hash scaled to [0, kHC); linear probing wraps at kHC
constexpr bool kHCPow2 = (kHC & (kHC - 1)) == 0;
constexpr int kHCLog = kHC >= 4096 ? 12 : kHC >= 2048 ? 11 : kHC >= 1024 ? 10 : 9;
__device__ __forceinline__ uint32_t hs_slot(uint32_t id) {
    if (kHCPow2) return (id * 0x9E3779B1u) >> (32 - kHCLog);
    return __umulhi(id * 0x9E3779B1u, (uint32_t)kHC);
}
__device__ __forceinline__ uint32_t hs_next(uint32_t h) {
    if (kHCPow2) return (h + 1) & (uint32_t)(kHC - 1);
    return h + 1 == (uint32_t)kHC ? 0u : h + 1;
}

// Read-only lookup of id v (not kEmpty) in a hash set of kHC slots (16-byte aligned): the linear
// probe sequence h, h + 1, ... read four slots at a time (one 128-bit shared load per aligned
// quad), the same probe order and answer as slot-by-slot probing.  Returns true if v is present;
// h ends at v's slot, or at the first empty slot (where an insertion of v starts probing).
// one quad w (slots b .. b + 3, b = h & ~3) of the probe sequence from h: true if the probe ends in
// it (then h = the ending slot and found = whether it holds v); else h = the next quad's first slot
__device__ __forceinline__ bool hs_quad(const uint4 w, uint32_t v, uint32_t& h, bool& found) {
    const uint32_t b = h & ~3u;
    const uint32_t from = (0xfu << (h & 3u)) & 0xfu;   // slots h .. b + 3
    const uint32_t eq = ((uint32_t)(w.x == v) | (uint32_t)(w.y == v) << 1 | (uint32_t)(w.z == v) << 2 |
                         (uint32_t)(w.w == v) << 3) & from;
    const uint32_t em = ((uint32_t)(w.x == kEmpty) | (uint32_t)(w.y == kEmpty) << 1 | (uint32_t)(w.z == kEmpty) << 2 |
                         (uint32_t)(w.w == kEmpty) << 3) & from;
    const uint32_t stop = eq | em;
    if (stop) {
        const uint32_t i = __ffs(stop) - 1;
        h = b + i;
        found = (eq >> i) & 1u;
        return true;
    }
    h = (b + 4) & (uint32_t)(kHC - 1);
    return false;
}
__device__ __forceinline__ bool hs_lookup4(const uint32_t* hs, uint32_t v, uint32_t& h) {
    static_assert(kHCPow2 && kHC % 4 == 0, "quad probing needs a power-of-two set of whole quads");
    bool found = false;
    while (!hs_quad(*reinterpret_cast<const uint4*>(hs + (h & ~3u)), v, h, found)) {}
    return found;
}

// claim id for evaluation: true if it was not evaluated before (called by one lane per distinct id)
__device__ __forceinline__ bool claim(const WarpSmem& w, const QState& st, uint32_t* bm, uint32_t id) {
    if (st.bitmap_mode) {
        const uint32_t bit = 1u << (id & 31);
#ifndef PFG_BM_READFIRST
#define PFG_BM_READFIRST 1
#endif
        // most passing ids of a long search were evaluated before: read the word first and claim
        // only when the bit is clear (bits are only ever set during a query, so a set bit is final)
        if (PFG_BM_READFIRST && (__ldcg(bm + (id >> 5)) & bit)) return false;
        return !(atomicOr(bm + (id >> 5), bit) & bit);
    }
    uint32_t h = hs_slot(id);
    for (;;) {
        const uint32_t old = atomicCAS(&w.f->hs[h], kEmpty, id);
        if (old == kEmpty) return true;
        if (old == id) return false;
        h = hs_next(h);
    }
}

// membership test (no insert), for the i = 0 linear scan
__device__ __forceinline__ bool evaluated(const WarpSmem& w, const QState& st, const uint32_t* bm, uint32_t id) {
    if (st.bitmap_mode) return (__ldcg(bm + (id >> 5)) >> (id & 31)) & 1u;
    uint32_t h = hs_slot(id);
    for (;;) {
        const uint32_t v = w.f->hs[h];
        if (v == kEmpty) return false;
        if (v == id) return true;
        h = hs_next(h);
    }
}

// move the hash set into the global bitmap (a query that evaluated more than kHMax ids)
__device__ __forceinline__ void to_bitmap_mode(const QueryParams& p, const WarpSmem& w, QState& st, uint32_t* bm,
                                               uint32_t* claims, int lane) {
    for (int h0 = 0; h0 < kHC; h0 += 32) {
        const uint32_t v = w.f->hs[h0 + lane];
        const bool has = v != kEmpty;
        if (has) atomicOr(bm + (v >> 5), 1u << (v & 31));
        const uint32_t m = __ballot_sync(kFull, has);
        if (has) {
            const uint32_t cn = st.claims_n + __popc(m & lanemask_lt());
            if (cn < (uint32_t)p.claim_cap) claims[cn] = v;
        }
        st.claims_n += __popc(m);
    }
    st.bitmap_mode = true;
    __syncwarp();
}

template <int EPL, int RQ = kRQ>
__global__ void __launch_bounds__(128, PFG_MINB) k_query(QueryParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t slot_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const WarpSmem w = carve(smem_raw + wib * p.smem_warp, p);
    uint32_t* bm = p.bitmap + slot_id * p.bm_words;
    uint32_t* claims = p.claims + slot_id * (int64_t)p.claim_cap;
    for (;;) {
        unsigned long long qv = 0;
        if (lane == 0) qv = atomicAdd(p.work, 1ull);
        const int64_t qidx = (int64_t)__shfl_sync(kFull, qv, 0);
        if (qidx >= (p.nq_dev ? (int64_t)*p.nq_dev : p.nq)) break;
        const int64_t qi = p.qlist ? (int64_t)p.qlist[qidx] : qidx;
        uint4* cur = p.cur + qi * p.L;   // per-query cursors (the round engine shares them)
        if (p.qzero[qi]) {
            for (int t = lane; t < p.k; t += 32) { p.out_ids[qi * p.k + t] = -1; p.out_sims[qi * p.k + t] = __int_as_float(0x7fc00000); }
            if (p.stats && lane == 0) {
                pfg_query_stats s = {}; s.flags = 2; p.stats[qi] = s;
            }
            continue;
        }
        for (int t = lane; t < p.dpad; t += 32) w.qrow[t] = p.qx[qi * p.dpad + t];
        for (int t = lane; t < p.M; t += 32) w.qsk[t] = p.qsk[qi * p.M + t];
        for (int t = lane; t < kHC / 4; t += 32) reinterpret_cast<uint4*>(w.f->hs)[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        __syncwarp();

        QState st;
        st.tn = 0; st.nE = 0; st.emitted = st.filtered = st.dups = st.probes = st.flags = 0; st.claims_n = 0;
        st.hcount = 0; st.bitmap_mode = false;
        st.T = w.T0; st.Tn = w.T1;
        bool stopped = false;
        int i_stop = 0, j_stop = 0;
        int i_start = p.K, c_start = 0;
        if (p.resume) {
            // continue from the round engine's state: next (level, chunk), top list, counters and
            // the evaluated ids (at most Ecap <= kHMax, so they fit the hash set)
            i_start = p.rs.lvl[qi];
            c_start = p.rs.c0[qi];
            st.tn = p.rs.tn[qi];
            for (int t = lane; t < st.tn; t += 32) w.T0[t] = p.rs.T[qi * p.kt + t];
            const uint32_t* cn = p.rs.cnt + qi * kCnt;
            st.emitted = cn[0]; st.filtered = cn[1]; st.dups = cn[2]; st.nE = cn[3];
            st.probes = lane == 0 ? cn[4] : 0u;  // per-lane partial sums, reduced at the end
            __syncwarp();
            for (uint32_t e = lane; e < st.nE; e += 32) {
                const uint32_t id = p.rs.E[qi * p.rs.Ecap + e];
                uint32_t h = hs_slot(id);
                while (atomicCAS(&w.f->hs[h], kEmpty, id) != kEmpty) h = hs_next(h);
            }
            st.hcount = st.nE;
            __syncwarp();
        }

        for (int i = i_start; i >= 1 && !stopped; i -= p.lstep) {
            for (int c0 = (i == i_start ? c_start : 0), c1 = 0; c0 < chunk_count(p) && !stopped; c0 = c1) {
                // R-17 chunk (or a tensor shell)
                const int nr = chunk_reps(p, i, c0, st.tn, st.T, lane);
                c1 = p.tensor_s ? c0 + 1 : c0 + nr;
                int tau = 64;
                if (p.use_filter && st.tn == p.k_eff) {
                    const float ip = kth_sim_clamped(p, st);
                    int lo = 0, hi = 64;  // tau = min{t : ip >= taub[t]}, taub[64] = -1
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (ip >= __ldg(p.taub + mid)) hi = mid; else lo = mid + 1; }
                    tau = lo;
                }
                // query codes of the chunk's repetitions (first level only): precomputed for
                // repetitions < qc_n, otherwise hashed here (FHT-CP, warp-cooperative)
                const long long th0 = p.prof ? clock64() : 0;
                if (i == p.K) {
                    if (lane < nr && trie_of(p, c0, lane) < p.qc_n)
                        w.f->qc[lane] = __ldg(p.qcodes + qi * p.qc_ld + trie_of(p, c0, lane));
                    const int r0 = max(0, p.qc_n - c0);
                    if (r0 < nr) {
                        __syncwarp();
                        group_rep_codes<EPL>(w.qrow, p.d, p.dp, p.ell, p.c, p.K, p.sg, c0, r0, nr, w.f->qc, lane);
                    }
                    __syncwarp();
                }
                if (p.prof && lane == 0) atomicAdd(p.prof + 4, (unsigned long long)(clock64() - th0));
                long long tp0 = p.prof ? clock64() : 0;
                // emitted-range widening (R-12), task t < nr: left side of rep t, t >= nr: right side.
                // First level: the match range [a_K, b_K) by binary search in the 13-bit bucket (the
                // range starts empty at lower_bound(q_j)); deeper levels: the segment loop of the
                // paper (extend by B while the entry just outside shares the top i bits), which
                // usually reads one boundary entry per side.
                for (int task = lane; task < 2 * nr; task += 32) {
                    const bool left = task < nr;
                    const int r = left ? task : task - nr;
                    const int j = trie_of(p, c0, r);
                    if (i == p.K && j < p.qb_n) {
                        const uint4 b = __ldg(p.qbnd + qi * p.qb_ld + j);
                        w.f->bnd[task] = left ? b.x : b.y;
                        if (left) st.probes += b.z;
                    } else if (i == p.K) {
                        const uint32_t qc = w.f->qc[r];
                        w.f->bnd[task] = rep_lower_bound(p, j, left ? (uint64_t)qc : (uint64_t)qc + 1, st.probes);
                    } else {
                        const uint4 cu = cur[j];
                        w.f->bnd[task] = widen_side(p, j, i, cu.x, left ? cu.y : cu.z, left, st.probes);
                        if (left) w.f->qc[r] = cu.x;
                    }
                }
                __syncwarp();
                uint32_t em = 0;
                if (lane < nr) {
                    const int j = trie_of(p, c0, lane);
                    uint32_t elo, ehi, nelo, nehi;
                    if (i == p.K) {
                        // closed form of the segment loop from [a, a): ehi' = a + B*ceil((b - a)/B)
                        const uint32_t a = w.f->bnd[lane], b = w.f->bnd[nr + lane];
                        const uint32_t B = (uint32_t)p.B;
                        elo = ehi = nelo = a;
                        const uint64_t v = (uint64_t)a + (uint64_t)((b - a + B - 1) / B) * B;
                        nehi = (uint32_t)(v > (uint64_t)p.n ? p.n : v);
                    } else {
                        const uint4 cu = cur[j];
                        elo = cu.y; ehi = cu.z;
                        nelo = w.f->bnd[lane]; nehi = w.f->bnd[nr + lane];
                    }
                    w.f->lo_new[lane] = nelo; w.f->lo_old[lane] = elo; w.f->hi_old[lane] = ehi;
                    w.f->fcnt[lane] = 0; w.f->dcnt[lane] = 0;
                    em = (elo - nelo) + (nehi - ehi);
                    cur[j] = make_uint4(w.f->qc[lane], nelo, nehi, 0u);
                }
                uint32_t incl = em;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(kFull, incl, off);
                    if (lane >= off) incl += o;
                }
                if (lane < nr) w.f->beg[lane + 1] = incl;
                if (lane == 0) w.f->beg[0] = 0;
                __syncwarp();
                const uint32_t total = w.f->beg[nr];

                if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 0, (unsigned long long)(t - tp0)); tp0 = t; }

                int nbuf = 0, next_check = 0, r_stop = -1;
                // scan the chunk's emitted positions in (rep, position) order, kU per lane per step;
                // each 16-byte table entry carries the id and its sketch word for this repetition
                int rl = 0;  // this lane's current repetition (positions only increase)
                for (uint32_t g0 = 0; g0 < total && !stopped; g0 += 32 * kU) {
                    uint32_t idv[kU];
                    int rv[kU];
                    bool pass[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const uint32_t g = g0 + u * 32 + lane;
                        pass[u] = false;
                        rv[u] = 0;
                        idv[u] = 0;
                        if (g < total) {
                            while (rl + 1 < nr && w.f->beg[rl + 1] <= g) ++rl;
                            const int r = rl;
                            const uint32_t o = g - w.f->beg[r];
                            const uint32_t lenA = w.f->lo_old[r] - w.f->lo_new[r];
                            const uint32_t pos = (o < lenA) ? w.f->lo_new[r] + o : w.f->hi_old[r] + (o - lenA);
                            const uint4 e = __ldg(reinterpret_cast<const uint4*>(p.tab + (int64_t)trie_of(p, c0, r) * p.n + pos));
                            idv[u] = e.x;
                            rv[u] = r;
                            pass[u] = true;
                            if (p.use_filter) {
                                const int s = __ldg(p.slot + trie_of(p, c0, r));
                                const uint64_t sw = ((uint64_t)e.w << 32) | e.z;
                                pass[u] = __popcll(sw ^ w.qsk[s]) <= tau;
                            }
                        }
                    }
                    if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 1, (unsigned long long)(t - tp0)); tp0 = t; }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const uint32_t g = g0 + u * 32 + lane;
                        // per-repetition counters: shared-memory atomics (same-address atomics of a
                        // warp are cheap on sm_100; measured faster than ballot aggregation)
                        if (g < total && !pass[u]) atomicAdd(&w.f->fcnt[rv[u]], 1u);
                        // claims in (rep, position) order: lanes in order within u, u in order
                        const uint32_t pm = __ballot_sync(kFull, pass[u]);
                        // a step inside one repetition holds distinct ids (each lane claims its
                        // own); only a step across a repetition boundary needs equal ids grouped
                        const int rfirst = __shfl_sync(kFull, rv[u], pm ? __ffs(pm) - 1 : 0);
                        const bool onerep = __all_sync(kFull, !pass[u] || rv[u] == rfirst);
                        bool fresh = false;
                        if (pass[u]) {
                            if (onerep) {
                                fresh = claim(w, st, bm, idv[u]);
                            } else {
                                const uint32_t grp = __match_any_sync(pm, idv[u]);
                                if ((int)(__ffs(grp) - 1) == lane) fresh = claim(w, st, bm, idv[u]);
                            }
                        }
                        if (pass[u] && !fresh) atomicAdd(&w.f->dcnt[rv[u]], 1u);
                        const uint32_t fm = __ballot_sync(kFull, fresh);
                        if (fresh) {
                            const int rank = __popc(fm & lanemask_lt());
                            w.f->sid[nbuf + rank] = idv[u];
                            w.f->srep[nbuf + rank] = (uint8_t)rv[u];
                            if (st.bitmap_mode) {
                                const uint32_t cn = st.claims_n + rank;
                                if (cn < (uint32_t)p.claim_cap) claims[cn] = idv[u];
                            }
                        }
                        const int nf = __popc(fm);
                        nbuf += nf;
                        if (st.bitmap_mode) st.claims_n += nf; else st.hcount += nf;
                        __syncwarp();
                    }
                    if (!st.bitmap_mode && st.hcount > kHMax) to_bitmap_mode(p, w, st, bm, claims, lane);
                    const uint32_t done_pos = min(total, g0 + 32u * kU);
                    if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 2, (unsigned long long)(t - tp0)); tp0 = t; }
                    if (nbuf > kSB - 32 * kU || done_pos == total) {
                        int complete = nr;
                        if (done_pos < total) { complete = 0; while (complete < nr && w.f->beg[complete + 1] <= done_pos) ++complete; }
                        if (drain<RQ>(p, w, st, nbuf, next_check, complete, nr, c0, i, qi, r_stop, lane)) {
                            stopped = true; i_stop = i; j_stop = p.tensor_s ? c0 + 1 : c0 + r_stop + 1;
                        }
                        if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 3, (unsigned long long)(t - tp0)); tp0 = t; }
                    }
                }
                if (total == 0) {
                    // empty chunk: every repetition is complete, check them in order
                    if (drain<RQ>(p, w, st, nbuf, next_check, nr, nr, c0, i, qi, r_stop, lane)) {
                        stopped = true; i_stop = i; j_stop = p.tensor_s ? c0 + 1 : c0 + r_stop + 1;
                    }
                }
                const int rmax = stopped ? r_stop : nr - 1;
                uint32_t e_acc = 0, f_acc = 0, d_acc = 0;
                for (int r = 0; r <= rmax; ++r) {
                    e_acc += w.f->beg[r + 1] - w.f->beg[r];
                    f_acc += w.f->fcnt[r];
                    d_acc += w.f->dcnt[r];
                }
                st.emitted += e_acc; st.filtered += f_acc; st.dups += d_acc;
                __syncwarp();
            }
        }

        if (!stopped) {
            // i = 0: linear scan of every point not yet evaluated (R-13), filter off, then stop;
            // every point evaluated before the scan is retrieved again as a duplicate
            st.dups += st.nE;
            int ns = 0;
            for (int64_t g0 = 0; g0 < p.n; g0 += 32) {
                const int64_t id = g0 + lane;
                const bool fresh = id < p.n && !evaluated(w, st, bm, (uint32_t)id);
                const uint32_t fm = __ballot_sync(kFull, fresh);
                if (fresh) w.f->sid[ns + __popc(fm & lanemask_lt())] = (uint32_t)id;
                ns += __popc(fm);
                __syncwarp();
                if (ns > kSB - 32 || g0 + 32 >= p.n) {
                    compute_sims<RQ>(p, w, 0, ns, lane, qi);
                    if (ns) merge_range(p, w, st, 0, ns, qi, lane);
                    ns = 0;
                }
            }
            st.emitted += (uint32_t)p.n;
            i_stop = 0; j_stop = 1;
        }

        for (int t = lane; t < p.k; t += 32) {
            if (t < st.tn) {
                const uint64_t kk = st.T[t];
                p.out_ids[qi * p.k + t] = (int64_t)key_id(kk) + p.id_offset;
                p.out_sims[qi * p.k + t] = key_sim(kk);
            } else {
                p.out_ids[qi * p.k + t] = -1;
                p.out_sims[qi * p.k + t] = -__int_as_float(0x7f800000);
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) st.probes += __shfl_xor_sync(kFull, st.probes, off);
        // stop-depth histogram (repetitions hashed at level K), read by the host to size the
        // next search's eager query hashing; a deeper stop counts as all L repetitions
        if (p.jhist && lane == 0) atomicAdd(p.jhist + min(i_stop == p.K ? j_stop : p.L, kJHist - 1), 1u);
        if (p.rs.ctl && lane == 0) {
            atomicAdd(&p.rs.ctl->evsum, (unsigned long long)st.nE);
            atomicAdd(&p.rs.ctl->emsum, (unsigned long long)st.emitted);
        }
        if (p.stats && lane == 0) {
            pfg_query_stats s;
            s.i_stop = i_stop; s.j_stop = j_stop; s.emitted = st.emitted; s.filtered = st.filtered;
            s.dups = st.dups; s.evaluated = st.nE;
            s.flags = (p.k > p.k_eff ? 1u : 0u) | ((p.trace_cap > 0 && st.nE > (uint32_t)p.trace_cap) ? 4u : 0u) |
                      (st.bitmap_mode ? 8u : 0u);
            s.probes = st.probes;
            p.stats[qi] = s;
        }
        // bitmap mode: return the bitmap to zero for the next query of this slot
        if (st.bitmap_mode) {
            const uint32_t ncl = st.claims_n;
            __syncwarp();
            if (ncl <= (uint32_t)p.claim_cap) {
                for (uint32_t e = lane; e < ncl; e += 32) __stcg(bm + (claims[e] >> 5), 0u);
            } else {
                for (int64_t e = lane; e < p.bm_words; e += 32) __stcg(bm + e, 0u);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// with 16-bit rows (R-25) the search ranks candidates by fixed-point
// inner products; this kernel re-scores each query's k_eff results with the fp32 rows in the R-2 order
// (lane sums of 16-byte chunks, sequential fmaf, then the tree h = 16..1, as or_sim) and re-sorts them
// by (sim desc, id asc).  One warp per query.
__global__ void __launch_bounds__(128) k_rerank(const float* __restrict__ x, const float* __restrict__ qx, int dpad,
                                                int64_t nq, int k, int k_eff, int kt, int64_t id_offset,
                                                int64_t* __restrict__ ids, float* __restrict__ sims) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    if (q >= nq) return;
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm + (size_t)wib * align16(kt * 8));
    const int nch = dpad >> 2;
    const float4* q4 = reinterpret_cast<const float4*>(qx + q * dpad);
    int n = 0;   // results present (zero query rows and padding are -1)
    for (int t = 0; t < k_eff; ++t) {
        const int64_t gid = ids[q * k + t];
        if (gid < 0) break;
        const uint32_t id = (uint32_t)(gid - id_offset);
        const float4* x4 = reinterpret_cast<const float4*>(x + (int64_t)id * dpad);
        float acc = 0.0f;
        for (int c = lane; c < nch; c += 32) {
            const float4 v = __ldg(x4 + c), w = __ldg(q4 + c);
            acc = fmaf(w.x, v.x, acc);
            acc = fmaf(w.y, v.y, acc);
            acc = fmaf(w.z, v.z, acc);
            acc = fmaf(w.w, v.w, acc);
        }
#pragma unroll
        for (int h = 16; h >= 1; h >>= 1) acc = acc + __shfl_xor_sync(kFull, acc, h);
        if (lane == 0) keys[t] = make_key(acc, id);
        n = t + 1;
    }
    __syncwarp();
    // rank sort (keys are distinct: distinct ids)
    for (int t = lane; t < n; t += 32) {
        const uint64_t kv = keys[t];
        int r = 0;
        for (int u = 0; u < n; ++u) r += keys[u] > kv ? 1 : 0;
        ids[q * k + r] = (int64_t)key_id(kv) + id_offset;
        sims[q * k + r] = key_sim(kv);
    }
}

// ---------------------------------------------------------------------------------------------
// shard merge (a15): out[q] = top-k of the world*k candidates by (sim desc, id asc), -1 ignored.
// one warp per query; k rounds of warp arg-max over the candidates in shared memory
__global__ void __launch_bounds__(128) k_merge_topk(const int64_t* __restrict__ ids, const float* __restrict__ sims,
                                                    int world, int64_t nq, int k, int64_t* __restrict__ out_ids,
                                                    float* __restrict__ out_sims) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    if (q >= nq) return;
    const int nc = world * k;
    float* cs = (float*)(sm + (size_t)wib * nc * 16);
    int64_t* ci = (int64_t*)(cs + nc + (nc & 1));
    for (int e = lane; e < nc; e += 32) {
        const int wr = e / k, t = e % k;
        const int64_t id = ids[((int64_t)wr * nq + q) * k + t];
        ci[e] = id;
        cs[e] = sims[((int64_t)wr * nq + q) * k + t];
    }
    __syncwarp();
    for (int t = 0; t < k; ++t) {
        float bs = 0.0f;
        int64_t bi = -1;
        int be = -1;
        for (int e = lane; e < nc; e += 32) {
            const int64_t id = ci[e];
            if (id < 0) continue;
            const float s = cs[e];
            if (be < 0 || s > bs || (s == bs && id < bi)) { bs = s; bi = id; be = e; }
        }
        for (int off = 16; off > 0; off >>= 1) {
            const float os = __shfl_xor_sync(kFull, bs, off);
            const int64_t oi = __shfl_xor_sync(kFull, bi, off);
            const int oe = __shfl_xor_sync(kFull, be, off);
            if (oe >= 0 && (be < 0 || os > bs || (os == bs && oi < bi))) { bs = os; bi = oi; be = oe; }
        }
        if (lane == 0) {
            out_ids[q * k + t] = be >= 0 ? bi : -1;
            out_sims[q * k + t] = be >= 0 ? bs : -__int_as_float(0x7f800000);
            if (be >= 0) ci[be] = -1;
        }
        __syncwarp();
    }
}

}  // namespace pfg
