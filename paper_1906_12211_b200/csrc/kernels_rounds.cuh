// kernels_rounds.cuh — the round engine: the same adaptive query as k_query, executed one chunk
// (the chunk's repetitions at one level) of every active query per round, split into
// bulk-parallel phases so that each phase runs at its own best occupancy and the
// bandwidth-heavy similarity phase has full memory-level parallelism:
//
//   k_qbounds  per (query, repetition < qb_n): the level-K match range [a_K, b_K) by two
//              interleaved binary searches (once per search, before the rounds)
//   k_rinit    per query: state init; zero query rows answered directly
//   k_collect  warp per active query: chunk codes, widening (R-12), scan of the emitted table
//              entries in (repetition, position) order with the sketch filter, and the dedupe
//              claims against a shared-memory hash set rebuilt from the query's evaluated list
//              (R-17/R-18) -> survivors appended to the evaluated list and to the round's pool
//   k_sims     grid over the pool: warp-coalesced rows, 32-lane tree (R-2) -> (sim, id) keys
//   k_merge    warp per active query: merge repetition by repetition into the top list, stop check
//              after each repetition (Alg. 1 line 8), commit cursors / advance, or finish
//
// Every decision (chunk boundaries, candidate order, claims, merges, stop checks, counters) is the
// one k_query makes for the same chunk, so results are identical.  A query whose chunk would
// overflow the evaluated list or the pool, that reaches the i = 0 scan, or that is still running
// when the rounds end is handed to k_query, which resumes it from the state (RoundState) with the
// chunk not yet committed.
//
// Round r uses parity par = r & 1: it reads active list act[par] (count ctl->nact[par]) and the
// pool counter ctl->pool_top[par]; k_collect resets the other parity's counters, k_merge fills
// act[par ^ 1].  No host synchronisation is needed between rounds.
#pragma once
#include "kernels_query.cuh"

namespace pfg {

constexpr int kFlagDone = 1, kFlagFused = 2;
constexpr int kEPre = 16;  // evaluated ids loaded per lane per batch when the hash set is rebuilt

__device__ __forceinline__ int tau_of_state(const QueryParams& p, int tn, const uint64_t* T) {
    if (!p.use_filter || tn != p.k_eff) return 64;
    float ip = key_sim(T[p.k_eff - 1]);
    ip = fminf(fmaxf(ip, -1.0f), 1.0f);
    int lo = 0, hi = 64;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (ip >= __ldg(p.taub + mid)) hi = mid; else lo = mid + 1; }
    return lo;
}


__device__ __forceinline__ void push(uint32_t* list, uint32_t* n, uint32_t q) { list[atomicAdd(n, 1u)] = q; }

// ---------------------------------------------------------------------------------------------
// level-K match ranges: a = lower_bound(code_j), b = lower_bound(code_j + 1) in
// repetition j's sorted table, via the 13-bit prefix table and a binary search in the bucket; the
// two searches run interleaved so both loads are in flight together.
__device__ __forceinline__ void bucket_of(const QueryParams& p, int j, uint64_t x, uint32_t& lo, uint32_t& hi) {
    if (x >= (1ull << p.K)) { lo = hi = (uint32_t)p.n; return; }
    const int sh = p.K - 13;
    const uint32_t* ptj = p.pt + (int64_t)j * 8193;
    const uint32_t pfx = (uint32_t)x >> sh;
    lo = __ldg(ptj + pfx);
    hi = ((x & ((1ull << sh) - 1)) == 0) ? lo : __ldg(ptj + pfx + 1);
}

__global__ void __launch_bounds__(256) k_qbounds(QueryParams p, uint4* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t q = t / p.qb_n;
    const int j = (int)(t - q * p.qb_n);
    if (q >= p.nq) return;
    if (p.qzero[q]) { out[q * p.qb_ld + j] = make_uint4(0, 0, 0, 0); return; }
    const uint32_t qc = __ldg(p.qcodes + q * p.qc_ld + j);
    uint32_t lo1, hi1, lo2, hi2, probes = 0;
    bucket_of(p, j, qc, lo1, hi1);
    bucket_of(p, j, (uint64_t)qc + 1, lo2, hi2);
    const Entry* tj = p.tab + (int64_t)j * p.n;
    while (lo1 < hi1 || lo2 < hi2) {
        const uint32_t m1 = (lo1 + hi1) >> 1, m2 = (lo2 + hi2) >> 1;
        const uint32_t c1 = lo1 < hi1 ? entry_code(tj + m1) : 0u;
        const uint32_t c2 = lo2 < hi2 ? entry_code(tj + m2) : 0u;
        if (lo1 < hi1) { ++probes; if (c1 < qc) lo1 = m1 + 1; else hi1 = m1; }
        if (lo2 < hi2) { ++probes; if ((uint64_t)c2 < (uint64_t)qc + 1) lo2 = m2 + 1; else hi2 = m2; }
    }
    out[q * p.qb_ld + j] = make_uint4(lo1, lo2, probes, 0u);
}

// ---------------------------------------------------------------------------------------------
__global__ void k_rinit(QueryParams p) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= p.nq) return;
    const RoundState& rs = p.rs;
    rs.lvl[q] = p.K;
    rs.c0[q] = 0;
    rs.tn[q] = 0;
    for (int t = 0; t < kCnt; ++t) rs.cnt[q * kCnt + t] = 0;
    if (p.qzero[q]) {
        rs.flags[q] = kFlagDone;
        for (int t = 0; t < p.k; ++t) { p.out_ids[q * p.k + t] = -1; p.out_sims[q * p.k + t] = __int_as_float(0x7fc00000); }
        if (p.stats) { pfg_query_stats s = {}; s.flags = 2; p.stats[q] = s; }
        return;
    }
    rs.flags[q] = 0;
    push(rs.act[0], &rs.ctl->nact[0], (uint32_t)q);
}

// ---------------------------------------------------------------------------------------------
struct CollectSmem {
    uint32_t hs[kHC];          // evaluated-id hash set
    uint64_t qsk[64];
    uint32_t beg[kMaxR + 4];
    uint32_t lo_new[kMaxR], lo_old[kMaxR], hi_old[kMaxR], qc[kMaxR], bnd[2 * kMaxR], fcnt[kMaxR], dcnt[kMaxR];
};
__host__ __device__ inline int collect_smem_bytes(int dpad, bool lazy) {
    return align16((int)sizeof(CollectSmem)) + (lazy ? align16(dpad * 4) : 0);
}

template <int EPL>
__global__ void __launch_bounds__(128) k_collect(QueryParams p, int par, int lazy) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    CollectSmem* c = (CollectSmem*)(smem_raw + wib * collect_smem_bytes(p.dpad, lazy));
    float* qrow = (float*)((unsigned char*)c + align16((int)sizeof(CollectSmem)));
    const RoundState& rs = p.rs;
    const uint32_t nact = rs.ctl->nact[par];
    if (blockIdx.x == 0 && threadIdx.x == 0) { rs.ctl->nact[par ^ 1] = 0; rs.ctl->pool_top[par ^ 1] = 0; }
    const uint32_t* act = rs.act[par];
    const int W = (p.dp + 31) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nact; a += nw) {
        const int64_t q = act[a];
        long long tq0 = p.prof ? clock64() : 0, tq = tq0;
        const int i = rs.lvl[q], c0 = rs.c0[q], tn = rs.tn[q];
        const int nr = chunk_reps(p, i, c0, tn, rs.T + q * p.kt, lane);
        const int tau = tau_of_state(p, tn, rs.T + q * p.kt);
        const uint32_t nE = rs.cnt[q * kCnt + 3];
        uint32_t* E = rs.E + q * (int64_t)rs.Ecap;
        uint4* cur = p.cur + q * p.L;
        for (int t = lane; t < p.M; t += 32) c->qsk[t] = p.qsk[q * p.M + t];
        for (int t = lane; t < kHC / 4; t += 32) reinterpret_cast<uint4*>(c->hs)[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        const bool need_lazy = (i == p.K) && (c0 + nr > p.qc_n);
        if (need_lazy)
            for (int t = lane; t < p.dpad; t += 32) qrow[t] = p.qx[q * p.dpad + t];
        if (lane < nr) { c->fcnt[lane] = 0; c->dcnt[lane] = 0; }
        __syncwarp();
        // rebuild the evaluated-id hash set (ids are distinct; kEPre loads per lane in flight)
        for (uint32_t e0 = 0; e0 < nE; e0 += 32 * kEPre) {
            uint32_t v[kEPre];
#pragma unroll
            for (int u = 0; u < kEPre; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                v[u] = e < nE ? E[e] : kEmpty;
            }
#pragma unroll
            for (int u = 0; u < kEPre; ++u)
                if (v[u] != kEmpty) {
                    uint32_t h = hs_slot(v[u]);
                    while (atomicCAS(&c->hs[h], kEmpty, v[u]) != kEmpty) h = hs_next(h);
                }
        }
        if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 8, (unsigned long long)(t - tq)); tq = t; }
        uint32_t probes = 0;
        if (i == p.K) {
            if (lane < nr && c0 + lane < p.qc_n) c->qc[lane] = __ldg(p.qcodes + q * p.qc_ld + c0 + lane);
            for (int r = 0; r < nr; ++r) {
                if (c0 + r < p.qc_n) continue;
                uint64_t full = 0;
                for (int t = 0; t < p.c; ++t) {
                    const int64_t f = (int64_t)(c0 + r) * p.c + t;
                    full = (full << p.ell) | fhtcp_code_warp<EPL>(qrow, p.d, p.dp, p.ell, p.sg + f * 3 * W, lane);
                }
                if (lane == 0) c->qc[r] = (uint32_t)(full >> (p.c * p.ell - p.K));
            }
            __syncwarp();
        }
        // widening, as k_query (first level: precomputed match ranges or binary search)
        for (int task = lane; task < 2 * nr; task += 32) {
            const bool left = task < nr;
            const int r = left ? task : task - nr;
            const int j = c0 + r;
            if (i == p.K && j < p.qb_n) {
                const uint4 b = __ldg(p.qbnd + q * p.qb_ld + j);
                c->bnd[task] = left ? b.x : b.y;
                if (left) probes += b.z;
            } else if (i == p.K) {
                const uint32_t qc = c->qc[r];
                c->bnd[task] = rep_lower_bound(p, j, left ? (uint64_t)qc : (uint64_t)qc + 1, probes);
            } else {
                const uint4 cu = cur[j];
                const uint32_t qp = cu.x >> (p.K - i);
                const Entry* tj = p.tab + (int64_t)j * p.n;
                const uint32_t B = (uint32_t)p.B;
                uint32_t e;
                if (left) {
                    e = cu.y;
                    while (e > 0) {
                        ++probes;
                        if ((entry_code(tj + e - 1) >> (p.K - i)) != qp) break;
                        e = e > B ? e - B : 0u;
                    }
                    c->qc[r] = cu.x;
                } else {
                    e = cu.z;
                    while (e < (uint32_t)p.n) {
                        ++probes;
                        if ((entry_code(tj + e) >> (p.K - i)) != qp) break;
                        e = (uint64_t)e + B < (uint64_t)p.n ? e + B : (uint32_t)p.n;
                    }
                }
                c->bnd[task] = e;
            }
        }
        __syncwarp();
        uint32_t em = 0;
        if (lane < nr) {
            const int j = c0 + lane;
            uint32_t elo, ehi, nelo, nehi;
            if (i == p.K) {
                const uint32_t a_ = c->bnd[lane], b_ = c->bnd[nr + lane];
                const uint32_t B = (uint32_t)p.B;
                elo = ehi = nelo = a_;
                const uint64_t v = (uint64_t)a_ + (uint64_t)((b_ - a_ + B - 1) / B) * B;
                nehi = (uint32_t)(v > (uint64_t)p.n ? p.n : v);
            } else {
                const uint4 cu = cur[j];
                elo = cu.y; ehi = cu.z;
                nelo = c->bnd[lane]; nehi = c->bnd[nr + lane];
            }
            c->lo_new[lane] = nelo; c->lo_old[lane] = elo; c->hi_old[lane] = ehi;
            em = (elo - nelo) + (nehi - ehi);
            rs.pend[q * kMaxR + lane] = make_uint4(c->qc[lane], nelo, nehi, 0u);
        }
        uint32_t incl = em;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane < nr) c->beg[lane + 1] = incl;
        if (lane == 0) c->beg[0] = 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) probes += __shfl_xor_sync(kFull, probes, off);
        __syncwarp();
        if (p.prof && lane == 0) { const long long t = clock64(); atomicAdd(p.prof + 9, (unsigned long long)(t - tq)); tq = t; }
        const uint32_t total = c->beg[nr];
        // scan in (rep, position) order: filter, then claim in order through the hash set; fresh
        // ids are appended to the evaluated list (room up to Ecap; beyond kHMax the query is
        // handed to the fused kernel, whose bitmap mode has no limit)
        uint32_t ns = 0;
        bool overflow = false;
        int rl = 0;
        for (uint32_t g0 = 0; g0 < total; g0 += 32 * kU) {
            uint32_t idv[kU];
            int rv[kU];
            bool pass[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t g = g0 + u * 32 + lane;
                pass[u] = false; rv[u] = 0; idv[u] = 0;
                if (g < total) {
                    while (rl + 1 < nr && c->beg[rl + 1] <= g) ++rl;
                    const int r = rl;
                    const uint32_t o = g - c->beg[r];
                    const uint32_t lenA = c->lo_old[r] - c->lo_new[r];
                    const uint32_t pos = (o < lenA) ? c->lo_new[r] + o : c->hi_old[r] + (o - lenA);
                    const uint4 e = __ldg(reinterpret_cast<const uint4*>(p.tab + (int64_t)(c0 + r) * p.n + pos));
                    idv[u] = e.x; rv[u] = r; pass[u] = true;
                    if (p.use_filter) {
                        const int s_ = __ldg(p.slot + c0 + r);
                        pass[u] = __popcll((((uint64_t)e.w << 32) | e.z) ^ c->qsk[s_]) <= tau;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t g = g0 + u * 32 + lane;
                if (g < total && !pass[u]) atomicAdd(&c->fcnt[rv[u]], 1u);
                const uint32_t pm = __ballot_sync(kFull, pass[u]);
                bool fresh = false;
                if (pass[u]) {
                    const uint32_t grp = __match_any_sync(pm, idv[u]);
                    if ((int)(__ffs(grp) - 1) == lane) {
                        uint32_t h = hs_slot(idv[u]);
                        for (;;) {
                            const uint32_t old = atomicCAS(&c->hs[h], kEmpty, idv[u]);
                            if (old == kEmpty) { fresh = true; break; }
                            if (old == idv[u]) break;
                            h = hs_next(h);
                        }
                    }
                    if (!fresh) atomicAdd(&c->dcnt[rv[u]], 1u);
                }
                const uint32_t fm = __ballot_sync(kFull, fresh);
                if (fresh) E[nE + ns + __popc(fm & lanemask_lt())] = idv[u];
                ns += __popc(fm);
            }
            if (nE + ns > (uint32_t)kHMax) { overflow = true; break; }
        }
        __syncwarp();
        if (p.prof && lane == 0) {
            const long long t = clock64(); atomicAdd(p.prof + 10, (unsigned long long)(t - tq)); tq = t;
            atomicAdd(p.prof + 13, (unsigned long long)total);
        }
        uint32_t base = 0;
        if (!overflow && lane == 0) base = atomicAdd(&rs.ctl->pool_top[par], ns);
        base = __shfl_sync(kFull, base, 0);
        if (!overflow && (uint64_t)base + ns > rs.pool_cap) overflow = true;
        if (overflow) {
            if (lane == 0) rs.flags[q] |= kFlagFused;
            __syncwarp();
            continue;
        }
        for (uint32_t e0 = 0; e0 < ns; e0 += 32 * kEPre) {
            uint32_t v[kEPre];
#pragma unroll
            for (int u = 0; u < kEPre; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                v[u] = e < ns ? E[nE + e] : 0u;
            }
#pragma unroll
            for (int u = 0; u < kEPre; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                if (e < ns) { rs.pool_id[base + e] = v[u]; rs.pool_q[base + e] = (uint32_t)q; }
            }
        }
        if (lane < nr) {
            uint32_t* rc = rs.repcnt + (q * kMaxR + lane) * 3;
            rc[0] = c->beg[lane + 1] - c->beg[lane];
            rc[1] = c->fcnt[lane];
            rc[2] = c->dcnt[lane];
        }
        if (lane == 0) {
            rs.poff[q] = base;
            rs.pn[q] = ns;
            rs.cnt[q * kCnt + 4] += probes;
        }
        __syncwarp();
        if (p.prof && lane == 0) {
            const long long t = clock64(); atomicAdd(p.prof + 11, (unsigned long long)(t - tq));
            atomicMax(p.prof + 12, (unsigned long long)(t - tq0));
            atomicAdd(p.prof + 14, 1ull);
            atomicMax(p.prof + 15, (unsigned long long)total);
        }
    }
}

// ---------------------------------------------------------------------------------------------
// similarities of the round's pool, kRPI rows per warp step (R-2 order, as compute_sims).  A
// query's survivors are contiguous in the pool, so the kRPI rows of a step usually share one query
// row (loaded once per chunk); otherwise each row reads its own query row.
template <bool ONEQ>
__device__ __forceinline__ void pool_sims_step(const float4* __restrict__ x4, const float4* __restrict__ qx4,
                                               const uint32_t (&roff)[kRPI], const uint32_t (&qoff)[kRPI], int nch,
                                               int lane, float (&acc)[kRPI]) {
#pragma unroll
    for (int r = 0; r < kRPI; ++r) acc[r] = 0.0f;
    for (int c = lane; c < nch; c += 32) {
        float4 v[kRPI];
#pragma unroll
        for (int r = 0; r < kRPI; ++r) v[r] = __ldg(x4 + roff[r] + c);
        float4 w4 = __ldg(qx4 + qoff[0] + c);
#pragma unroll
        for (int r = 0; r < kRPI; ++r) {
            if (!ONEQ && r > 0) w4 = __ldg(qx4 + qoff[r] + c);
            acc[r] = fmaf(w4.x, v[r].x, acc[r]);
            acc[r] = fmaf(w4.y, v[r].y, acc[r]);
            acc[r] = fmaf(w4.z, v[r].z, acc[r]);
            acc[r] = fmaf(w4.w, v[r].w, acc[r]);
        }
    }
}

__global__ void __launch_bounds__(256, 2) k_sims(QueryParams p, int par) {
    const int lane = threadIdx.x & 31;
    const RoundState& rs = p.rs;
    const uint32_t top = min(rs.ctl->pool_top[par], rs.pool_cap);
    const int nch = p.dpad >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(p.x);
    const float4* qx4 = reinterpret_cast<const float4*>(p.qx);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // lane r < kRPI holds entry b + r of the current step (rows beyond the end repeat the last);
    // the next step's entries are fetched before the current rows are read
    auto fetch = [&](int64_t b, uint32_t& id, uint32_t& qq) {
        if (lane < kRPI && b < top) {
            const int64_t e1 = (int64_t)top < b + kRPI ? (int64_t)top : b + kRPI;
            const int64_t e = b + lane < e1 ? b + lane : e1 - 1;
            id = rs.pool_id[e];
            qq = rs.pool_q[e];
        }
    };
    int64_t b = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRPI;
    uint32_t nid = 0, nq_ = 0;
    fetch(b, nid, nq_);
    for (; b < top; b += nw * kRPI) {
        const int64_t e1 = (int64_t)top < b + kRPI ? (int64_t)top : b + kRPI;
        const uint32_t myid = nid, myq = nq_;
        fetch(b + nw * kRPI, nid, nq_);
        float acc[kRPI];
        uint32_t roff[kRPI], qoff[kRPI];
#pragma unroll
        for (int r = 0; r < kRPI; ++r) {
            roff[r] = __shfl_sync(kFull, myid, r) * (uint32_t)nch;
            qoff[r] = __shfl_sync(kFull, myq, r) * (uint32_t)nch;
        }
        if (qoff[0] == qoff[kRPI - 1]) pool_sims_step<true>(x4, qx4, roff, qoff, nch, lane, acc);
        else pool_sims_step<false>(x4, qx4, roff, qoff, nch, lane, acc);
        const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
        float t4[4], t2[2];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float recv = __shfl_xor_sync(kFull, h16 ? acc[k] : acc[k + 4], 16);
            t4[k] = (h16 ? acc[k + 4] : acc[k]) + recv;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float recv = __shfl_xor_sync(kFull, h8 ? t4[k] : t4[k + 2], 8);
            t2[k] = (h8 ? t4[k + 2] : t4[k]) + recv;
        }
        float t1 = (h4 ? t2[1] : t2[0]) + __shfl_xor_sync(kFull, h4 ? t2[0] : t2[1], 4);
        t1 = t1 + __shfl_xor_sync(kFull, t1, 2);
        t1 = t1 + __shfl_xor_sync(kFull, t1, 1);
        const int rr = lane >> 2;
        const uint32_t id_rr = __shfl_sync(kFull, myid, rr);
        if ((lane & 3) == 0 && b + rr < e1) rs.pool_key[b + rr] = make_key(t1, id_rr);
    }
}

// ---------------------------------------------------------------------------------------------
struct MergeSmem {
    uint64_t cand[32];
};

__global__ void __launch_bounds__(128) k_merge(QueryParams p, int par) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int per_warp = align16((int)sizeof(MergeSmem)) + 2 * align16(p.kt * 8);
    MergeSmem* m = (MergeSmem*)(smem_raw + wib * per_warp);
    uint64_t* T0 = (uint64_t*)((unsigned char*)m + align16((int)sizeof(MergeSmem)));
    uint64_t* T1 = T0 + align16(p.kt * 8) / 8;
    const RoundState& rs = p.rs;
    const uint32_t nact = rs.ctl->nact[par];
    const uint32_t* act = rs.act[par];
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nact; a += nw) {
        const int64_t q = act[a];
        if (rs.flags[q] & kFlagFused) {
            if (lane == 0) push(rs.fused, &rs.ctl->nfused, (uint32_t)q);
            continue;
        }
        const int i = rs.lvl[q], c0 = rs.c0[q];
        int tn = rs.tn[q];
        const int nr = chunk_reps(p, i, c0, tn, rs.T + q * p.kt, lane);
        for (int t = lane; t < tn; t += 32) T0[t] = rs.T[q * p.kt + t];
        uint64_t* T = T0;
        uint64_t* Tn = T1;
        uint32_t* cn = rs.cnt + q * kCnt;
        uint32_t nE = cn[3];
        const uint32_t base = rs.poff[q];
        // survivors of repetition r are pool entries [end_{r-1}, end_r): per repetition
        // emitted - filtered - duplicates, in repetition order
        uint32_t rc0 = 0, rc1 = 0, rc2 = 0;
        if (lane < nr) {
            const uint32_t* rc = rs.repcnt + (q * kMaxR + lane) * 3;
            rc0 = rc[0]; rc1 = rc[1]; rc2 = rc[2];
        }
        uint32_t end = rc0 - rc1 - rc2;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, end, off);
            if (lane >= off) end += o;
        }
        __syncwarp();
        int r_stop = -1;
        uint32_t e = 0;
        for (int r = 0; r < nr; ++r) {
            const uint32_t e2 = __shfl_sync(kFull, end, r);
            uint64_t nxt = (e + lane < e2) ? rs.pool_key[base + e + lane] : 0ull;
            for (uint32_t b0 = e; b0 < e2; b0 += 32) {
                const uint32_t idx = b0 + lane;
                uint64_t key = nxt;
                nxt = (idx + 32 < e2) ? rs.pool_key[base + idx + 32] : 0ull;  // prefetch the next batch
                if (idx < e2 && p.trace_cap > 0) {
                    const uint32_t pos = nE + (idx - e);
                    if (pos < (uint32_t)p.trace_cap) p.trace_ids[q * p.trace_cap + pos] = key_id(key);
                }
                const uint64_t kth = (tn == p.k_eff) ? T[p.k_eff - 1] : 0ull;
                if (key <= kth) key = 0;
                const uint32_t vm = __ballot_sync(kFull, key != 0);
                if (vm) {
                    key = warp_sort_desc(key, lane);
                    const int nc = __popc(vm);
                    m->cand[lane] = key;
                    __syncwarp();
                    if (lane < nc) {
                        int l2 = 0, h2 = tn;
                        while (l2 < h2) { const int mid = (l2 + h2) >> 1; if (T[mid] > key) l2 = mid + 1; else h2 = mid; }
                        if (lane + l2 < p.k_eff) Tn[lane + l2] = key;
                    }
                    for (int t = lane; t < tn; t += 32) {
                        const uint64_t tv = T[t];
                        int l2 = 0, h2 = nc;
                        while (l2 < h2) { const int mid = (l2 + h2) >> 1; if (m->cand[mid] > tv) l2 = mid + 1; else h2 = mid; }
                        if (t + l2 < p.k_eff) Tn[t + l2] = tv;
                    }
                    __syncwarp();
                    tn = min(p.k_eff, tn + nc);
                    uint64_t* tmp = T; T = Tn; Tn = tmp;
                }
                __syncwarp();
            }
            nE += e2 - e;
            e = e2;
            const int j1 = c0 + r + 1;
            if (tn == p.k_eff && (!p.per_round || j1 == p.L)) {
                float ip = key_sim(T[p.k_eff - 1]);
                ip = fminf(fmaxf(ip, -1.0f), 1.0f);
                if (ip >= __ldg(p.thr + (int64_t)(i - 1) * p.L + (j1 - 1))) { r_stop = r; break; }
            }
        }
        const int rmax = r_stop >= 0 ? r_stop : nr - 1;
        uint32_t ea = lane <= rmax ? rc0 : 0u, fa = lane <= rmax ? rc1 : 0u, da = lane <= rmax ? rc2 : 0u;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            ea += __shfl_xor_sync(kFull, ea, off);
            fa += __shfl_xor_sync(kFull, fa, off);
            da += __shfl_xor_sync(kFull, da, off);
        }
        const uint32_t emitted = cn[0] + ea, filtered = cn[1] + fa, dups = cn[2] + da;
        __syncwarp();
        if (r_stop >= 0) {
            for (int t = lane; t < p.k; t += 32) {
                if (t < tn) {
                    p.out_ids[q * p.k + t] = (int64_t)key_id(T[t]) + p.id_offset;
                    p.out_sims[q * p.k + t] = key_sim(T[t]);
                } else {
                    p.out_ids[q * p.k + t] = -1;
                    p.out_sims[q * p.k + t] = -__int_as_float(0x7f800000);
                }
            }
            if (lane == 0) {
                if (p.stats) {
                    pfg_query_stats s;
                    s.i_stop = i; s.j_stop = c0 + r_stop + 1; s.emitted = emitted; s.filtered = filtered; s.dups = dups;
                    s.evaluated = nE;
                    s.flags = (p.k > p.k_eff ? 1u : 0u) | ((p.trace_cap > 0 && nE > (uint32_t)p.trace_cap) ? 4u : 0u);
                    s.probes = cn[4];
                    p.stats[q] = s;
                }
                rs.flags[q] |= kFlagDone;
            }
        } else {
            // chunk complete: commit its cursors, save the state, move to the next chunk
            uint4* cur = p.cur + q * p.L;
            if (lane < nr) cur[c0 + lane] = rs.pend[q * kMaxR + lane];
            for (int t = lane; t < tn; t += 32) rs.T[q * p.kt + t] = T[t];
            if (lane == 0) {
                cn[0] = emitted; cn[1] = filtered; cn[2] = dups; cn[3] = nE;
                rs.tn[q] = tn;
                int ni = i, nc0 = c0 + nr;
                if (nc0 >= p.L) { ni = i - 1; nc0 = 0; }
                rs.lvl[q] = ni;
                rs.c0[q] = nc0;
                if (ni == 0) { rs.flags[q] |= kFlagFused; push(rs.fused, &rs.ctl->nfused, (uint32_t)q); }
                else push(rs.act[par ^ 1], &rs.ctl->nact[par ^ 1], (uint32_t)q);
            }
        }
        __syncwarp();
    }
}

// move the still-active queries of list `par` to the fused list (rounds ended)
__global__ void k_handoff(QueryParams p, int par) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= p.rs.ctl->nact[par]) return;
    push(p.rs.fused, &p.rs.ctl->nfused, p.rs.act[par][a]);
}

}  // namespace pfg
