// kernels_rounds.cuh — the round engine: the same adaptive query as k_query, executed one chunk
// (R repetitions at one level) of every active query per round, split into bulk-parallel phases
// so that the bandwidth-heavy similarity phase runs with full memory-level parallelism:
//
//   k_rinit    per query: state init; zero query rows answered directly
//   k_collect  warp per active query: chunk codes, widening (R-12), scan of the emitted table
//              entries in (repetition, position) order with the sketch filter -> candidates
//   k_dedupe   warp per active query: evaluated-id hash set rebuilt in shared memory from the query's
//              evaluated list, claims in candidate order (R-17) -> survivors into the round's pool
//   k_sims     grid over the pool: warp-coalesced rows, 32-lane tree (R-2)
//   k_merge    warp per active query: merge repetition by repetition into the top list, stop check
//              after each repetition (Alg. 1 line 8), commit cursors / advance, or finish
//
// Every decision (candidate order, claims, merges, stop checks, counters) is the one k_query makes
// for the same chunk, so results are identical.  A query whose chunk would overflow a buffer, that
// reaches the i = 0 scan, or that is still running when the rounds end is handed to k_query, which
// resumes it from the state (RoundState) with the chunk not yet committed.
#pragma once
#include "kernels_query.cuh"

namespace pfg {

constexpr int kFlagDone = 1, kFlagFused = 2;

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
    push(rs.next, rs.nnext, (uint32_t)q);
}

// ---------------------------------------------------------------------------------------------
struct CollectSmem {
    uint64_t qsk[64];
    uint32_t beg[kMaxR + 4];
    uint32_t lo_new[kMaxR], lo_old[kMaxR], hi_old[kMaxR], qc[kMaxR], bnd[2 * kMaxR], fcnt[kMaxR];
};
__host__ __device__ inline int collect_smem_bytes(int dpad) { return align16((int)sizeof(CollectSmem)) + align16(dpad * 4); }

template <int EPL>
__global__ void __launch_bounds__(128) k_collect(QueryParams p, uint32_t nactive) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int stride_b = collect_smem_bytes(p.dpad);
    CollectSmem* c = (CollectSmem*)(smem_raw + wib * stride_b);
    float* qrow = (float*)((unsigned char*)c + align16((int)sizeof(CollectSmem)));
    const RoundState& rs = p.rs;
    const int W = (p.dp + 31) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nactive; a += nw) {
        const int64_t q = rs.active[a];
        const int i = rs.lvl[q], c0 = rs.c0[q];
        const int nr = min(p.R, p.L - c0);
        const int tau = tau_of_state(p, rs.tn[q], rs.T + q * p.kt);
        uint4* cur = p.cur + q * p.L;
        for (int t = lane; t < p.M; t += 32) c->qsk[t] = p.qsk[q * p.M + t];
        const bool need_lazy = (i == p.K) && (c0 + nr > p.qc_n);
        if (need_lazy)
            for (int t = lane; t < p.dpad; t += 32) qrow[t] = p.qx[q * p.dpad + t];
        __syncwarp();
        uint32_t probes = 0;
        if (i == p.K) {
            for (int r = 0; r < nr; ++r) {
                if (c0 + r < p.qc_n) {
                    if (lane == 0) c->qc[r] = __ldg(p.qcodes + q * p.qc_ld + c0 + r);
                    continue;
                }
                uint64_t full = 0;
                for (int t = 0; t < p.c; ++t) {
                    const int64_t f = (int64_t)(c0 + r) * p.c + t;
                    full = (full << p.ell) | fhtcp_code_warp<EPL>(qrow, p.d, p.dp, p.ell, p.sg + f * 3 * W, lane);
                }
                if (lane == 0) c->qc[r] = (uint32_t)(full >> (p.c * p.ell - p.K));
            }
            __syncwarp();
        }
        // widening, same as k_query
        for (int task = lane; task < 2 * nr; task += 32) {
            const bool left = task < nr;
            const int r = left ? task : task - nr;
            const int j = c0 + r;
            if (i == p.K) {
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
            c->fcnt[lane] = 0;
            em = (elo - nelo) + (nehi - ehi);
            rs.pend[q * kMaxR + lane] = make_uint4(c->qc[lane], nelo, nehi, 0u);
            rs.repcnt[(q * kMaxR + lane) * 3 + 0] = em;
        }
        uint32_t incl = em;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane < nr) c->beg[lane + 1] = incl;
        if (lane == 0) c->beg[0] = 0;
        probes += __shfl_xor_sync(kFull, probes, 16);
        probes += __shfl_xor_sync(kFull, probes, 8);
        probes += __shfl_xor_sync(kFull, probes, 4);
        probes += __shfl_xor_sync(kFull, probes, 2);
        probes += __shfl_xor_sync(kFull, probes, 1);
        __syncwarp();
        const uint32_t total = c->beg[nr];
        // scan in (rep, position) order; filter-passing positions become candidates in that order
        uint32_t ncand = 0;
        bool overflow = false;
        uint32_t* cand = rs.cand + q * (int64_t)rs.Ccap;
        uint8_t* crep = rs.crep + q * (int64_t)rs.Ccap;
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
                if (pass[u]) {
                    const uint32_t dst = ncand + __popc(pm & lanemask_lt());
                    if (dst < (uint32_t)rs.Ccap) { cand[dst] = idv[u]; crep[dst] = (uint8_t)rv[u]; }
                }
                ncand += __popc(pm);
            }
        }
        if (ncand > (uint32_t)rs.Ccap) overflow = true;
        __syncwarp();
        if (lane < nr) rs.repcnt[(q * kMaxR + lane) * 3 + 1] = c->fcnt[lane];
        if (lane == 0) {
            rs.ncand[q] = overflow ? 0u : ncand;
            rs.cnt[q * kCnt + 4] += probes;
            if (overflow) rs.flags[q] |= kFlagFused;
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
struct DedupeSmem {
    uint32_t hs[kHC];
    uint32_t dcnt[kMaxR];
};

__global__ void __launch_bounds__(128) k_dedupe(QueryParams p, uint32_t nactive) {
    __shared__ DedupeSmem sm_all[4];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    DedupeSmem* d = &sm_all[wib];
    const RoundState& rs = p.rs;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nactive; a += nw) {
        const int64_t q = rs.active[a];
        if (rs.flags[q] & kFlagFused) continue;
        const uint32_t nE = rs.cnt[q * kCnt + 3];
        const uint32_t* E = rs.E + q * (int64_t)rs.Ecap;
        for (int t = lane; t < kHC / 4; t += 32) reinterpret_cast<uint4*>(d->hs)[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        if (lane < kMaxR) d->dcnt[lane] = 0;
        __syncwarp();
        for (uint32_t e = lane; e < nE; e += 32) {
            const uint32_t id = E[e];
            uint32_t h = hs_slot(id);
            while (atomicCAS(&d->hs[h], kEmpty, id) != kEmpty) h = (h + 1) & (kHC - 1);
        }
        __syncwarp();
        const uint32_t n = rs.ncand[q];
        uint32_t* cand = rs.cand + q * (int64_t)rs.Ccap;
        uint8_t* crep = rs.crep + q * (int64_t)rs.Ccap;
        uint32_t ns = 0;
        for (uint32_t b = 0; b < n; b += 32) {
            const bool act = b + lane < n;
            const uint32_t id = act ? cand[b + lane] : 0u;
            const int r = act ? crep[b + lane] : 0;
            const uint32_t am = __ballot_sync(kFull, act);
            bool fresh = false;
            if (act) {
                const uint32_t grp = __match_any_sync(am, id);
                if ((int)(__ffs(grp) - 1) == lane) {
                    uint32_t h = hs_slot(id);
                    for (;;) {
                        const uint32_t old = atomicCAS(&d->hs[h], kEmpty, id);
                        if (old == kEmpty) { fresh = true; break; }
                        if (old == id) break;
                        h = (h + 1) & (kHC - 1);
                    }
                }
                if (!fresh) atomicAdd(&d->dcnt[r], 1u);
            }
            const uint32_t fm = __ballot_sync(kFull, fresh);
            __syncwarp();
            if (fresh) {
                const uint32_t dst = ns + __popc(fm & lanemask_lt());
                cand[dst] = id;      // in-place compaction in order (dst <= b + lane)
                crep[dst] = (uint8_t)r;
            }
            ns += __popc(fm);
            __syncwarp();
        }
        bool fused = nE + ns > (uint32_t)rs.Ecap;
        uint32_t base = 0;
        if (!fused && lane == 0) base = atomicAdd(rs.pool_top, ns);
        base = __shfl_sync(kFull, base, 0);
        if (!fused && (uint64_t)base + ns > rs.pool_cap) fused = true;
        if (fused) {
            if (lane == 0) rs.flags[q] |= kFlagFused;
            continue;
        }
        uint32_t* Ew = rs.E + q * (int64_t)rs.Ecap + nE;
        for (uint32_t e = lane; e < ns; e += 32) {
            const uint32_t id = cand[e];
            Ew[e] = id;
            rs.pool_id[base + e] = id;
            rs.pool_q[base + e] = (uint32_t)q;
            rs.pool_rep[base + e] = crep[e];
        }
        if (lane < kMaxR) rs.repcnt[(q * kMaxR + lane) * 3 + 2] = d->dcnt[lane];
        if (lane == 0) { rs.poff[q] = base; rs.pn[q] = ns; }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// similarities of the round's pool, kRPI rows per warp step (R-2 order, as compute_sims)
__global__ void __launch_bounds__(256) k_sims(QueryParams p) {
    const int lane = threadIdx.x & 31;
    const RoundState& rs = p.rs;
    const uint32_t top = min(*rs.pool_top, rs.pool_cap);
    const int nch = p.dpad >> 2;
    const float4* x4 = reinterpret_cast<const float4*>(p.x);
    const float4* qx4 = reinterpret_cast<const float4*>(p.qx);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t b = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kRPI; b < top; b += nw * kRPI) {
        const int64_t e1 = (int64_t)top < b + kRPI ? (int64_t)top : b + kRPI;
        float acc[kRPI];
        uint32_t roff[kRPI], qoff[kRPI];
#pragma unroll
        for (int r = 0; r < kRPI; ++r) {
            const int64_t e = b + r < e1 ? b + r : e1 - 1;
            acc[r] = 0.0f;
            roff[r] = rs.pool_id[e] * (uint32_t)nch;
            qoff[r] = rs.pool_q[e] * (uint32_t)nch;
        }
        for (int c = lane; c < nch; c += 32) {
            float4 v[kRPI], w4[kRPI];
#pragma unroll
            for (int r = 0; r < kRPI; ++r) { v[r] = __ldg(x4 + roff[r] + c); w4[r] = __ldg(qx4 + qoff[r] + c); }
#pragma unroll
            for (int r = 0; r < kRPI; ++r) {
                acc[r] = fmaf(w4[r].x, v[r].x, acc[r]);
                acc[r] = fmaf(w4[r].y, v[r].y, acc[r]);
                acc[r] = fmaf(w4[r].z, v[r].z, acc[r]);
                acc[r] = fmaf(w4[r].w, v[r].w, acc[r]);
            }
        }
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
        if ((lane & 3) == 0 && b + rr < e1) rs.pool_sim[b + rr] = t1;
    }
}

// ---------------------------------------------------------------------------------------------
struct MergeSmem {
    uint64_t cand[32];
    uint32_t sid[32];
    float ssim[32];
};

__global__ void __launch_bounds__(128) k_merge(QueryParams p, uint32_t nactive) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int per_warp = align16((int)sizeof(MergeSmem)) + 2 * align16(p.kt * 8);
    MergeSmem* m = (MergeSmem*)(smem_raw + wib * per_warp);
    uint64_t* T0 = (uint64_t*)((unsigned char*)m + align16((int)sizeof(MergeSmem)));
    uint64_t* T1 = T0 + align16(p.kt * 8) / 8;
    const RoundState& rs = p.rs;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nactive; a += nw) {
        const int64_t q = rs.active[a];
        if (rs.flags[q] & kFlagFused) {
            if (lane == 0) push(rs.fused, rs.nfused, (uint32_t)q);
            continue;
        }
        const int i = rs.lvl[q], c0 = rs.c0[q];
        const int nr = min(p.R, p.L - c0);
        int tn = rs.tn[q];
        for (int t = lane; t < tn; t += 32) T0[t] = rs.T[q * p.kt + t];
        uint64_t* T = T0;
        uint64_t* Tn = T1;
        uint32_t* cn = rs.cnt + q * kCnt;
        uint32_t nE = cn[3];
        const uint32_t base = rs.poff[q], ns = rs.pn[q];
        __syncwarp();
        int r_stop = -1;
        uint32_t e = 0;
        for (int r = 0; r < nr; ++r) {
            // survivors of repetition r: [e, e2) (the pool keeps the query's candidate order)
            uint32_t lo = e, hi = ns;
            while (lo < hi) { const uint32_t mid = (lo + hi) >> 1; if (rs.pool_rep[base + mid] <= r) lo = mid + 1; else hi = mid; }
            const uint32_t e2 = lo;
            for (uint32_t b0 = e; b0 < e2; b0 += 32) {
                const uint32_t idx = b0 + lane;
                uint64_t key = 0;
                if (idx < e2) {
                    const uint32_t id = rs.pool_id[base + idx];
                    key = make_key(rs.pool_sim[base + idx], id);
                    if (p.trace_cap > 0) {
                        const uint32_t pos = nE + (idx - e);
                        if (pos < (uint32_t)p.trace_cap) p.trace_ids[q * p.trace_cap + pos] = id;
                    }
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
        uint32_t ea = 0, fa = 0, da = 0;
        for (int r = 0; r <= rmax; ++r) {
            const uint32_t* rc = rs.repcnt + (q * kMaxR + r) * 3;
            ea += rc[0]; fa += rc[1]; da += rc[2];
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
                int ni = i, nc0 = c0 + p.R;
                if (nc0 >= p.L) { ni = i - 1; nc0 = 0; }
                rs.lvl[q] = ni;
                rs.c0[q] = nc0;
                if (ni == 0) { rs.flags[q] |= kFlagFused; push(rs.fused, rs.nfused, (uint32_t)q); }
                else push(rs.next, rs.nnext, (uint32_t)q);
            }
        }
        __syncwarp();
    }
}

// move the still-active queries to the fused list (rounds ended)
__global__ void k_handoff(QueryParams p, uint32_t nactive) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= nactive) return;
    const uint32_t q = p.rs.active[a];
    push(p.rs.fused, p.rs.nfused, q);
}

}  // namespace pfg
