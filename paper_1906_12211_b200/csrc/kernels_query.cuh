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

constexpr int kCB = 256;      // candidate buffer per warp (filter-passing, not yet evaluated)
constexpr int kU = 4;         // table positions per lane per scan step (memory-level parallelism)
constexpr int kMaxR = 32;     // max repetitions per chunk
constexpr int kMaxK = 256;    // max k

struct QueryParams {
    int64_t n, nq, bm_words, id_offset;
    int d, dpad, K, L, M, B, R, k, k_eff, per_round, use_filter, c, ell, dp, lazy, claim_cap, trace_cap;
    int kt;          // T capacity (>= k_eff, multiple of 32)
    int smem_warp;   // bytes of shared memory per warp
    const float* __restrict__ x;
    const uint64_t* __restrict__ sk;
    const uint64_t* __restrict__ tab;
    const uint32_t* __restrict__ pt;
    const uint8_t* __restrict__ slot;
    const float* __restrict__ qx;
    const uint64_t* __restrict__ qsk;
    const uint32_t* __restrict__ qcodes;
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
};

struct WarpSmem {
    float* qrow;       // [dpad]
    uint64_t* qsk;     // [M]
    uint64_t* T0;      // [kt]
    uint64_t* T1;      // [kt]
    uint64_t* cand;    // [32]   sorted merge batch
    uint64_t* cb;      // [kCB]  candidate keys (id << 8 | rep)
    uint32_t* sid;     // [kCB]  evaluated ids, bucketed by rep
    float* ssim;       // [kCB]
    uint32_t* beg;     // [kMaxR + 1]
    uint32_t* lo_new;  // [kMaxR]
    uint32_t* lo_old;
    uint32_t* hi_old;
    uint32_t* qc;      // [kMaxR] lazily computed codes
    uint32_t* bnd;     // [2 * kMaxR] a / b bounds
    uint32_t* fcnt;    // [kMaxR] filtered per rep
    uint32_t* dcnt;    // [kMaxR] dups per rep
    uint32_t* rcnt;    // [kMaxR + 1] survivors per rep (then bucket offsets)
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

__host__ __device__ inline int warp_smem_bytes(int dpad, int M, int kt) {
    int b = 0;
    b += align16(dpad * 4);
    b += align16(M * 8);
    b += 2 * align16(kt * 8);
    b += 32 * 8;
    b += kCB * 8 + kCB * 4 + kCB * 4;
    b += align16((kMaxR + 1) * 4) + 3 * kMaxR * 4 + kMaxR * 4 + 2 * kMaxR * 4 + 2 * kMaxR * 4 + align16((kMaxR + 1) * 4);
    return align16(b);
}

__device__ inline WarpSmem carve(unsigned char* base, const QueryParams& p) {
    WarpSmem w;
    unsigned char* q = base;
    w.qrow = (float*)q; q += align16(p.dpad * 4);
    w.qsk = (uint64_t*)q; q += align16(p.M * 8);
    w.T0 = (uint64_t*)q; q += align16(p.kt * 8);
    w.T1 = (uint64_t*)q; q += align16(p.kt * 8);
    w.cand = (uint64_t*)q; q += 32 * 8;
    w.cb = (uint64_t*)q; q += kCB * 8;
    w.sid = (uint32_t*)q; q += kCB * 4;
    w.ssim = (float*)q; q += kCB * 4;
    w.beg = (uint32_t*)q; q += align16((kMaxR + 1) * 4);
    w.lo_new = (uint32_t*)q; q += kMaxR * 4;
    w.lo_old = (uint32_t*)q; q += kMaxR * 4;
    w.hi_old = (uint32_t*)q; q += kMaxR * 4;
    w.qc = (uint32_t*)q; q += kMaxR * 4;
    w.bnd = (uint32_t*)q; q += 2 * kMaxR * 4;
    w.fcnt = (uint32_t*)q; q += kMaxR * 4;
    w.dcnt = (uint32_t*)q; q += kMaxR * 4;
    w.rcnt = (uint32_t*)q; q += align16((kMaxR + 1) * 4);
    return w;
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
    const uint64_t* tj = p.tab + (int64_t)j * p.n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t cm = (uint32_t)(__ldg(tj + mid) >> 32);
        ++probes;
        if (cm < xs) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// 256-bit read-only load of 8 consecutive floats (one full 32-byte sector per lane)
__device__ __forceinline__ void ldg256(const float* p, float (&v)[8]) {
    asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p));
}

// canonical inner product (R-2): sequential fmaf over t from +0; the zero padding of both rows
// beyond d leaves the chain unchanged (see k_hp_bits).  dpad is a multiple of 8.
__device__ __forceinline__ float dot_row(const float* __restrict__ q, const float* __restrict__ xr, int dpad) {
    float s = 0.0f;
    const int nc = dpad >> 3;
#pragma unroll 4
    for (int c = 0; c < nc; ++c) {
        float v[8];
        ldg256(xr + 8 * c, v);
        const float4 w0 = reinterpret_cast<const float4*>(q)[2 * c];
        const float4 w1 = reinterpret_cast<const float4*>(q)[2 * c + 1];
        s = fmaf(w0.x, v[0], s);
        s = fmaf(w0.y, v[1], s);
        s = fmaf(w0.z, v[2], s);
        s = fmaf(w0.w, v[3], s);
        s = fmaf(w1.x, v[4], s);
        s = fmaf(w1.y, v[5], s);
        s = fmaf(w1.z, v[6], s);
        s = fmaf(w1.w, v[7], s);
    }
    return s;
}

struct QState {
    int tn;               // entries in T (<= k_eff)
    uint32_t nE;          // evaluated (merged) ids
    uint32_t emitted, filtered, dups, probes, flags;
    uint32_t claims_n;
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
            const uint32_t id = w.sid[idx];
            key = make_key(w.ssim[idx], id);
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
            w.cand[lane] = key;
            __syncwarp();
            // new position of candidate `lane` = lane + #T entries greater than it
            if (lane < nc) {
                int lo = 0, hi = st.tn;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (st.T[mid] > key) lo = mid + 1; else hi = mid; }
                const int dst = lane + lo;
                if (dst < p.k_eff) st.Tn[dst] = key;
            }
            // new position of T entry e' = e' + #candidates greater than it
            for (int t = lane; t < st.tn; t += 32) {
                const uint64_t tv = st.T[t];
                int lo = 0, hi = nc;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (w.cand[mid] > tv) lo = mid + 1; else hi = mid; }
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

__device__ __forceinline__ float kth_sim_clamped(const QueryParams& p, const QState& st) {
    float ip = key_sim(st.T[p.k_eff - 1]);
    return fminf(fmaxf(ip, -1.0f), 1.0f);
}

// compute sims for survivors [0, ns)
__device__ __forceinline__ void compute_sims(const QueryParams& p, const WarpSmem& w, int ns, int lane) {
    for (int e = lane; e < ns; e += 32)
        w.ssim[e] = dot_row(w.qrow, p.x + (int64_t)w.sid[e] * p.dpad, p.dpad);
    __syncwarp();
}

// warp-cooperative ascending bitonic sort of cb[0..P) in shared memory (P power of two)
__device__ __forceinline__ void warp_sort_smem(uint64_t* s, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = s[i], b = s[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncwarp();
        }
    }
}

// Flush the candidate buffer (R-17): candidates are filter-passing positions whose id was
// not evaluated when scanned.  Sort by (id, rep); the first occurrence of an id (its smallest
// repetition) is evaluated, later ones count as duplicates -- the same evaluated set and repetition
// attribution as the sequential algorithm.  Survivors are bucketed by repetition, claimed in the
// bitmap, their inner products computed, and merged repetition by repetition; every repetition
// < `complete` (all positions scanned) gets its stop check after its survivors are merged.
// Returns true when the query stops (r_stop set).
__device__ __forceinline__ bool flush_chunk(const QueryParams& p, const WarpSmem& w, QState& st, int& ncand,
                                            int& next_check, int complete, int nr, int c0, int i, int64_t qi,
                                            uint32_t* bm, uint32_t* claims, int& r_stop, int lane) {
    int ns = 0;
    if (ncand > 0) {
        int P = 32;
        while (P < ncand) P <<= 1;
        for (int e = ncand + lane; e < P; e += 32) w.cb[e] = ~0ull;
        __syncwarp();
        warp_sort_smem(w.cb, P, lane);
        for (int r = lane; r <= nr; r += 32) w.rcnt[r] = 0;
        __syncwarp();
        // dedupe + per-rep counts
        for (int e = lane; e < ncand; e += 32) {
            const uint64_t key = w.cb[e];
            const bool keep = (e == 0) || ((w.cb[e - 1] >> 8) != (key >> 8));
            const int r = (int)(key & 0xff);
            if (keep) atomicAdd(&w.rcnt[r], 1u); else atomicAdd(&w.dcnt[r], 1u);
        }
        __syncwarp();
        // exclusive prefix over reps (nr <= 32) -> bucket offsets in rcnt
        {
            const uint32_t v = lane < nr ? w.rcnt[lane] : 0u;
            uint32_t incl = v;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += o;
            }
            const uint32_t tot = __shfl_sync(kFull, incl, nr - 1);
            __syncwarp();
            if (lane < nr) w.rcnt[lane] = incl - v;
            if (lane == 0) w.rcnt[nr] = tot;
            __syncwarp();
        }
        ns = (int)w.rcnt[nr];
        // scatter survivors to rep buckets, claim them in the bitmap
        for (int e = lane; e < ncand; e += 32) {
            const uint64_t key = w.cb[e];
            const bool keep = (e == 0) || ((w.cb[e - 1] >> 8) != (key >> 8));
            if (keep) {
                const uint32_t id = (uint32_t)(key >> 8);
                const int r = (int)(key & 0xff);
                const uint32_t dst = atomicAdd(&w.rcnt[r], 1u);
                w.sid[dst] = id;
                atomicOr(bm + (id >> 5), 1u << (id & 31));
            }
        }
        __syncwarp();
        // rcnt[r] is now the end of bucket r; record claims for the bitmap reset
        for (int e = lane; e < ns; e += 32) {
            const uint32_t cn = st.claims_n + e;
            if (cn < (uint32_t)p.claim_cap) claims[cn] = w.sid[e];
        }
        st.claims_n += ns;
        compute_sims(p, w, ns, lane);
    }
    ncand = 0;
    // merge bucket by bucket in repetition order, stop check after every complete repetition
    for (;;) {
        if (next_check >= nr) break;
        if (ns > 0) {
            const int b0 = next_check == 0 ? 0 : (int)w.rcnt[next_check - 1];
            const int b1 = (int)w.rcnt[next_check];
            if (b1 > b0) merge_range(p, w, st, b0, b1, qi, lane);
        }
        if (next_check >= complete) break;
        const int j1 = c0 + next_check + 1;
        if (st.tn == p.k_eff && (!p.per_round || j1 == p.L)) {
            const float ip = kth_sim_clamped(p, st);
            if (ip >= __ldg(p.thr + (int64_t)(i - 1) * p.L + (j1 - 1))) {
                r_stop = next_check;
                return true;
            }
        }
        ++next_check;
    }
    __syncwarp();
    return false;
}

template <int EPL>
__global__ void __launch_bounds__(128) k_query(QueryParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t slot_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const WarpSmem w = carve(smem_raw + wib * p.smem_warp, p);
    uint4* cur = p.cur + slot_id * p.L;
    uint32_t* bm = p.bitmap + slot_id * p.bm_words;
    uint32_t* claims = p.claims + slot_id * (int64_t)p.claim_cap;
    const int W = (p.dp + 31) >> 5;

    for (;;) {
        unsigned long long qv = 0;
        if (lane == 0) qv = atomicAdd(p.work, 1ull);
        const int64_t qi = (int64_t)__shfl_sync(kFull, qv, 0);
        if (qi >= p.nq) break;
        if (p.qzero[qi]) {
            for (int t = lane; t < p.k; t += 32) { p.out_ids[qi * p.k + t] = -1; p.out_sims[qi * p.k + t] = __int_as_float(0x7fc00000); }
            if (p.stats && lane == 0) {
                pfg_query_stats s = {}; s.flags = 2; p.stats[qi] = s;
            }
            continue;
        }
        for (int t = lane; t < p.dpad; t += 32) w.qrow[t] = p.qx[qi * p.dpad + t];
        for (int t = lane; t < p.M; t += 32) w.qsk[t] = p.qsk[qi * p.M + t];
        __syncwarp();

        QState st;
        st.tn = 0; st.nE = 0; st.emitted = st.filtered = st.dups = st.probes = st.flags = 0; st.claims_n = 0;
        st.T = w.T0; st.Tn = w.T1;
        bool stopped = false;
        int i_stop = 0, j_stop = 0;

        for (int i = p.K; i >= 1 && !stopped; --i) {
            for (int c0 = 0; c0 < p.L && !stopped; c0 += p.R) {
                const int nr = min(p.R, p.L - c0);
                int tau = 64;
                if (p.use_filter && st.tn == p.k_eff) {
                    const float ip = kth_sim_clamped(p, st);
                    int lo = 0, hi = 64;  // tau = min{t : ip >= taub[t]}, taub[64] = -1
                    while (lo < hi) { const int mid = (lo + hi) >> 1; if (ip >= __ldg(p.taub + mid)) hi = mid; else lo = mid + 1; }
                    tau = lo;
                }
                // lazy FHT-CP hashing of the chunk's repetitions (first level only)
                if (i == p.K && p.lazy) {
                    for (int r = 0; r < nr; ++r) {
                        uint64_t full = 0;
                        for (int t = 0; t < p.c; ++t) {
                            const int64_t f = (int64_t)(c0 + r) * p.c + t;
                            full = (full << p.ell) | fhtcp_code_warp<EPL>(w.qrow, p.d, p.dp, p.ell, p.sg + f * 3 * W, lane);
                        }
                        if (lane == 0) w.qc[r] = (uint32_t)(full >> (p.c * p.ell - p.K));
                    }
                    __syncwarp();
                }
                // prefix match ranges [a_i, b_i): task t < nr -> a of rep t, t >= nr -> b of rep t-nr
                for (int task = lane; task < 2 * nr; task += 32) {
                    const int r = task < nr ? task : task - nr;
                    const int j = c0 + r;
                    uint32_t qc;
                    if (i == p.K) qc = p.lazy ? w.qc[r] : __ldg(p.qcodes + qi * p.L + j);
                    else qc = cur[j].x;
                    const uint64_t qp = (uint64_t)qc >> (p.K - i);
                    const uint64_t x = (task < nr ? qp : qp + 1) << (p.K - i);
                    w.bnd[task] = rep_lower_bound(p, j, x, st.probes);
                    if (task < nr) w.qc[r] = qc;
                }
                __syncwarp();
                uint32_t em = 0;
                if (lane < nr) {
                    const int j = c0 + lane;
                    const uint32_t a = w.bnd[lane], b = w.bnd[nr + lane];
                    uint32_t elo, ehi;
                    if (i == p.K) { elo = ehi = a; } else { const uint4 cu = cur[j]; elo = cu.y; ehi = cu.z; }
                    const uint32_t B = (uint32_t)p.B;
                    uint32_t nelo = elo, nehi = ehi;
                    if (a < elo) { const uint32_t s = (elo - a + B - 1) / B; nelo = (s * B >= elo) ? 0u : elo - s * B; }
                    if (b > ehi) { const uint64_t s = (b - ehi + B - 1) / B; const uint64_t v = ehi + s * B; nehi = (uint32_t)(v > (uint64_t)p.n ? p.n : v); }
                    w.lo_new[lane] = nelo; w.lo_old[lane] = elo; w.hi_old[lane] = ehi;
                    w.fcnt[lane] = 0; w.dcnt[lane] = 0;
                    em = (elo - nelo) + (nehi - ehi);
                    cur[j] = make_uint4(w.qc[lane], nelo, nehi, 0u);
                }
                // exclusive prefix sum of per-rep emitted counts
                uint32_t incl = em;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(kFull, incl, off);
                    if (lane >= off) incl += o;
                }
                if (lane < nr) w.beg[lane + 1] = incl;
                if (lane == 0) w.beg[0] = 0;
                __syncwarp();
                const uint32_t total = w.beg[nr];

                int ncand = 0, next_check = 0, r_stop = -1;
                // scan the chunk's emitted positions in (rep, position) order, kU per lane per step
                for (uint32_t g0 = 0;; g0 += 32 * kU) {
                    const bool last = g0 + 32 * kU >= total;
                    if (g0 < total) {
                        uint32_t idv[kU];
                        int rv[kU];
                        bool act[kU], pass[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const uint32_t g = g0 + u * 32 + lane;
                            act[u] = g < total;
                            rv[u] = 0;
                            idv[u] = 0;
                            if (act[u]) {
                                int r = 0;
                                while (r + 1 < nr && w.beg[r + 1] <= g) ++r;
                                const uint32_t o = g - w.beg[r];
                                const uint32_t lenA = w.lo_old[r] - w.lo_new[r];
                                const uint32_t pos = (o < lenA) ? w.lo_new[r] + o : w.hi_old[r] + (o - lenA);
                                idv[u] = (uint32_t)__ldg(p.tab + (int64_t)(c0 + r) * p.n + pos);
                                rv[u] = r;
                            }
                        }
                        if (p.use_filter) {
                            uint64_t sw[kU];
#pragma unroll
                            for (int u = 0; u < kU; ++u)
                                sw[u] = act[u] ? __ldg(p.sk + (int64_t)idv[u] * p.M + __ldg(p.slot + c0 + rv[u])) : 0ull;
#pragma unroll
                            for (int u = 0; u < kU; ++u) {
                                pass[u] = false;
                                if (act[u]) {
                                    const int s = __ldg(p.slot + c0 + rv[u]);
                                    pass[u] = __popcll(sw[u] ^ w.qsk[s]) <= tau;
                                    if (!pass[u]) atomicAdd(&w.fcnt[rv[u]], 1u);
                                }
                            }
                        } else {
#pragma unroll
                            for (int u = 0; u < kU; ++u) pass[u] = act[u];
                        }
                        uint32_t bw[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) bw[u] = pass[u] ? __ldcg(bm + (idv[u] >> 5)) : 0u;
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            bool fresh = false;
                            if (pass[u]) {
                                fresh = !((bw[u] >> (idv[u] & 31)) & 1u);
                                if (!fresh) atomicAdd(&w.dcnt[rv[u]], 1u);
                            }
                            const uint32_t fm = __ballot_sync(kFull, fresh);
                            if (fresh) w.cb[ncand + __popc(fm & lanemask_lt())] = ((uint64_t)idv[u] << 8) | (uint64_t)rv[u];
                            ncand += __popc(fm);
                        }
                        __syncwarp();
                    }
                    if (last || ncand > kCB - 32 * kU) {
                        int complete = nr;
                        if (!last) { complete = 0; while (complete < nr && w.beg[complete + 1] <= g0 + 32 * kU) ++complete; }
                        if (flush_chunk(p, w, st, ncand, next_check, complete, nr, c0, i, qi, bm, claims, r_stop, lane)) {
                            stopped = true; i_stop = i; j_stop = c0 + r_stop + 1;
                        }
                    }
                    if (stopped || last) break;
                }
                // account the chunk's repetitions up to the stop (all of them if no stop)
                const int rmax = stopped ? r_stop : nr - 1;
                uint32_t e_acc = 0, f_acc = 0, d_acc = 0;
                for (int r = 0; r <= rmax; ++r) {
                    e_acc += w.beg[r + 1] - w.beg[r];
                    f_acc += w.fcnt[r];
                    d_acc += w.dcnt[r];
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
                bool fresh = false;
                if (id < p.n) fresh = !((__ldcg(bm + (id >> 5)) >> (id & 31)) & 1u);
                const uint32_t fm = __ballot_sync(kFull, fresh);
                if (fresh) w.sid[ns + __popc(fm & lanemask_lt())] = (uint32_t)id;
                ns += __popc(fm);
                __syncwarp();
                if (ns > kCB - 32 || g0 + 32 >= p.n) {
                    compute_sims(p, w, ns, lane);
                    if (ns) merge_range(p, w, st, 0, ns, qi, lane);
                    ns = 0;
                }
            }
            st.emitted += (uint32_t)p.n;
            i_stop = 0; j_stop = 1;
        }

        // output: T sorted desc; ids are global
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
        if (p.stats && lane == 0) {
            pfg_query_stats s;
            s.i_stop = i_stop; s.j_stop = j_stop; s.emitted = st.emitted; s.filtered = st.filtered;
            s.dups = st.dups; s.evaluated = st.nE;
            s.flags = (p.k > p.k_eff ? 1u : 0u) | ((p.trace_cap > 0 && st.nE > (uint32_t)p.trace_cap) ? 4u : 0u);
            s.probes = st.probes;
            p.stats[qi] = s;
        }
        // return the bitmap to zero for the next query of this slot
        const uint32_t ncl = st.claims_n;
        __syncwarp();
        if (ncl <= (uint32_t)p.claim_cap) {
            for (uint32_t e = lane; e < ncl; e += 32) __stcg(bm + (claims[e] >> 5), 0u);
        } else {
            for (int64_t e = lane; e < p.bm_words; e += 32) __stcg(bm + e, 0u);
        }
        __syncwarp();
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
