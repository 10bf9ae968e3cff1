// kernels_chunk.cuh — the chunk engine: the round engine's control phases for one query fused into
// one CTA (the default when no query of the search needs a visit-tag array).
//
// A round is two kernels:
//   k_chunk  CTA per active query (dynamic scheduling):
//              merge   the survivors of the query's previous chunk (their similarities, computed by
//                      the previous round's k_sims) into the top list repetition by repetition, the
//                      stop check after each repetition (Alg. 1 line 8), then commit
//                      the chunk (cursors, counters) or finish the query;
//              expand  the next chunk (R-17), its tau, codes and emitted ranges (R-12);
//              scan    the chunk's table entries in (repetition, position) order, the sketch filter
//                       with the chunk's tau;
//              dedupe  against the evaluated set (R-18), in shared memory, in parallel:
//                      every passing candidate inserts (id, position + 1) into the query's hash set and
//                      keeps the minimum position per id (atomicMin on (id << 32) | ord); a candidate is
//                      fresh iff its own position is that minimum and the id was not evaluated before
//                      (ord 0) -- the first occurrence in (repetition, position) order, as the
//                      sequential claims of k_dedupe; the fresh ids are compacted in that order to the
//                      evaluated list and the round's pool;
//   k_sims   the survivors' similarities (kernels_rounds.cuh), one pool per round parity.
// After the last round a merge-only pass finishes or hands off every query still running to the
// fused kernel (k_query), which resumes it from RoundState.  Every decision is the one the round
// engine (kernels_rounds.cuh) and the fused kernel make for the same chunk, so results are
// identical; the hash set is rebuilt from the evaluated list every round (no save / restore).
#pragma once
#include "kernels_rounds.cuh"

namespace pfg {

constexpr int kCT = 128;                 // threads per query CTA
constexpr int kCW = kCT / 32;
#ifndef PFG_CHUNK_U
#define PFG_CHUNK_U 4
#endif
constexpr int kCU = PFG_CHUNK_U;         // positions per thread per batch
constexpr int kCB = kCT * kCU;           // positions per batch
static_assert(kCU * kCW <= 32, "one warp scans the per-(step, warp) counts");
#ifndef PFG_CHUNK_PROF
#define PFG_CHUNK_PROF 0
#endif
constexpr int kFlagPend = 64;            // the query's last chunk awaits its merge
constexpr unsigned long long kE64 = ~0ull;
// hash-set slots: the evaluated ids (at most hmax <= kHMax) plus one batch of passing candidates
// always leave free slots, so a probe sequence ends
constexpr int kCH = 3072;
static_assert(kCH > kHMax + kCB, "the chunk hash set must hold the evaluated set plus one batch");
__device__ __forceinline__ uint32_t ch_slot(uint32_t id) { return __umulhi(id * 0x9E3779B1u, (uint32_t)kCH); }
__device__ __forceinline__ uint32_t ch_next(uint32_t h) { return h + 1 == (uint32_t)kCH ? 0u : h + 1; }

struct ChunkSmem {
    unsigned long long hs[kCH];          // (id << 32) | ord; ord 0 = evaluated before the chunk
                                         // (the merge phase keeps its candidate keys here)
    uint8_t urep[kHMax + 32];            // merge phase: repetition of each candidate key
    uint32_t wcnt[kCW];                  // merge phase: candidate keys per warp
    uint32_t nu;                         // merge phase: candidate keys
    uint64_t cand[32];                   // merge batch
    uint64_t sk[kMaxR];                  // the query's sketch word of each repetition's slot
    uint32_t qc[kMaxR], lo_new[kMaxR], lo_old[kMaxR], hi_old[kMaxR], bnd[2 * kMaxR];
    uint32_t beg[kMaxR + 1];             // exclusive prefix of the emitted counts
    uint32_t pcnt[kMaxR], fcnt[kMaxR];   // passing the filter, fresh, per repetition
    uint8_t erep[kHMax + kCB];           // repetition of each fresh id of the chunk (E order)
    uint32_t roff[kMaxR];                // pool offset of each repetition's survivors
    uint32_t a, total, nE, ns, probes, pbase;
    float taub[65];                      // filter breakpoints (p.taub)
    uint32_t wa[2];                      // work items (this one, the next), claimed one query ahead
    int64_t wq[2];
    int64_t q;
    int fl;
    int nr, tau, direct, i, c0, tn, tsel, stop, overflow;
};

__host__ __device__ inline int chunk_smem_bytes(int kt, int dpad, bool lazy) {
    return align16((int)sizeof(ChunkSmem)) + 2 * align16(kt * 8) + (lazy ? align16(dpad * 4) : 0);
}

// merge of the query's pending chunk (same decisions as k_merge).  All threads: the chunk's pool keys
// (in repetition order) that beat the k-th key of the top list at the start of the chunk -- only
// those can enter it, since the k-th key only grows -- are compacted in order with their
// repetition; warp 0 then merges them repetition by repetition with the stop check after each
// (Alg. 1 line 8).  The trace (evaluated ids in evaluation order) takes every key.
__device__ __forceinline__ void chunk_merge(const QueryParams& p, int64_t q, size_t pin, uint64_t* T0, uint64_t* T1,
                                            ChunkSmem& s, int tid) {
    const int lane = tid & 31, wid = tid >> 5;
    const RoundState& rs = p.rs;
    const int i = s.i, c0 = s.c0;
    const int nr = (int)rs.rinfo[q].x;
    const uint32_t pn = rs.pn[q];
    uint32_t* cn = rs.cnt + q * kCnt;
    const uint32_t nE0 = cn[3];
    const uint64_t* keys = rs.pool_key + pin + rs.poff[q];
    const uint64_t kth0 = (s.tn == p.k_eff) ? T0[p.k_eff - 1] : 0ull;
    // survivors of repetition r are pool entries [end_{r-1}, end_r): emitted - filtered - dups
    uint32_t rc0 = 0, rc1 = 0, rc2 = 0, end = 0;
    if (wid == 0) {
        if (lane < nr) {
            const uint32_t* rc = rs.repcnt + (q * kMaxR + lane) * 3;
            rc0 = rc[0]; rc1 = rc[1]; rc2 = rc[2];
        }
        end = rc0 - rc1 - rc2;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, end, off);
            if (lane >= off) end += o;
        }
        if (lane < nr) s.beg[lane + 1] = end;
        if (lane == 0) s.beg[0] = 0;
    }
    // the keys into shared memory (coalesced, several loads in flight per thread), then thread t takes
    // the contiguous keys [t * per, (t + 1) * per)
    uint64_t* KS = reinterpret_cast<uint64_t*>(s.hs);          // [0, pn)
    uint64_t* U = KS + kCH / 2;                                 // candidates (at most pn <= kHMax)
    for (uint32_t e0 = 0; e0 < pn; e0 += kCT * 4) {
        uint64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t e = e0 + u * kCT + tid;
            v[u] = e < pn ? keys[e] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t e = e0 + u * kCT + tid;
            if (e < pn) {
                KS[e] = v[u];
                if (p.trace_cap > 0 && nE0 + e < (uint32_t)p.trace_cap) p.trace_ids[q * p.trace_cap + nE0 + e] = key_id(v[u]);
            }
        }
    }
    __syncthreads();
    const uint32_t per = (pn + kCT - 1) / kCT;
    const uint32_t k0 = min(pn, tid * per), k1 = min(pn, k0 + per);
    uint32_t mine = 0;
    for (uint32_t e = k0; e < k1; ++e) mine += KS[e] > kth0 ? 1u : 0u;
    uint32_t incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(kFull, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) s.wcnt[wid] = incl;
    __syncthreads();
    uint32_t wb = 0, nu = 0;
#pragma unroll
    for (int w = 0; w < kCW; ++w) { wb += w < wid ? s.wcnt[w] : 0u; nu += s.wcnt[w]; }
    {
        uint32_t o = wb + incl - mine;
        int r = 0;
        for (uint32_t e = k0; e < k1; ++e) {
            const uint64_t key = KS[e];
            if (key > kth0) {
                while (r + 1 < nr && s.beg[r + 1] <= e) ++r;
                U[o] = key;
                s.urep[o] = (uint8_t)r;
                ++o;
            }
        }
    }
    __syncthreads();
    if (wid != 0) return;
    int tn = s.tn;
    uint64_t* T = T0;
    uint64_t* Tn = T1;
    auto merge_batch = [&](uint64_t key) {
        const uint64_t kth = (tn == p.k_eff) ? T[p.k_eff - 1] : 0ull;
        if (key <= kth) key = 0;
        const uint32_t vm = __ballot_sync(kFull, key != 0);
        if (vm) {
            key = warp_sort_desc(key, lane);
            const int nc = __popc(vm);
            s.cand[lane] = key;
            __syncwarp();
            if (lane < nc) {
                int l2 = 0, h2 = tn;
                while (l2 < h2) { const int mid = (l2 + h2) >> 1; if (T[mid] > key) l2 = mid + 1; else h2 = mid; }
                if (lane + l2 < p.k_eff) Tn[lane + l2] = key;
            }
            for (int t = lane; t < tn; t += 32) {
                const uint64_t tv = T[t];
                int l2 = 0, h2 = nc;
                while (l2 < h2) { const int mid = (l2 + h2) >> 1; if (s.cand[mid] > tv) l2 = mid + 1; else h2 = mid; }
                if (t + l2 < p.k_eff) Tn[t + l2] = tv;
            }
            __syncwarp();
            tn = min(p.k_eff, tn + nc);
            uint64_t* tmp = T; T = Tn; Tn = tmp;
        }
        __syncwarp();
    };
    // lane r: end of repetition r's candidate keys in U
    uint32_t uend = 0;
    {
        int lo = 0, hi = (int)nu;
        while (lo < hi) { const int mid = (lo + hi) >> 1; if ((int)s.urep[mid] <= lane) lo = mid + 1; else hi = mid; }
        uend = (uint32_t)lo;
    }
    const float thr_r = lane < nr ? __ldg(p.thr + (int64_t)(i - 1) * p.L + c0 + lane) : INFINITY;
    int r_stop = -1;
    uint32_t e = 0;
    for (int r = 0; r < nr; ++r) {
        const uint32_t e2 = __shfl_sync(kFull, uend, r);
        for (uint32_t b0 = e; b0 < e2; b0 += 32) merge_batch(b0 + lane < e2 ? U[b0 + lane] : 0ull);
        e = e2;
        const int j1 = c0 + r + 1;
        const float th = __shfl_sync(kFull, thr_r, r);
        if (tn == p.k_eff && (!p.per_round || j1 == p.L)) {
            float ip = key_sim(T[p.k_eff - 1]);
            ip = fminf(fmaxf(ip, -1.0f), 1.0f);
            if (ip >= th) { r_stop = r; break; }
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
    const uint32_t nE = nE0 + __shfl_sync(kFull, end, rmax);
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
            if (p.jhist) atomicAdd(p.jhist + min(i == p.K ? c0 + r_stop + 1 : p.L, kJHist - 1), 1u);
            atomicAdd(&rs.ctl->evsum, (unsigned long long)nE);
            atomicAdd(&rs.ctl->emsum, (unsigned long long)emitted);
            if (p.stats) {
                pfg_query_stats st;
                st.i_stop = i; st.j_stop = c0 + r_stop + 1; st.emitted = emitted; st.filtered = filtered; st.dups = dups;
                st.evaluated = nE;
                st.flags = (p.k > p.k_eff ? 1u : 0u) | ((p.trace_cap > 0 && nE > (uint32_t)p.trace_cap) ? 4u : 0u);
                st.probes = cn[4];
                p.stats[q] = st;
            }
            rs.flags[q] = (rs.flags[q] | kFlagDone) & ~kFlagPend;
            s.stop = 1;
        }
    } else {
        // chunk complete: commit its cursors, the top list and the counters, move to the next chunk
        uint4* cur = p.cur + q * p.L;
        if (lane < nr) cur[c0 + lane] = rs.pend[q * kMaxR + lane];
        for (int t = lane; t < tn; t += 32) rs.T[q * p.kt + t] = T[t];
        int ni = i, nc0 = c0 + nr;
        if (nc0 >= p.L) { ni = i - 1; nc0 = 0; }
        if (lane == 0) {
            cn[0] = emitted; cn[1] = filtered; cn[2] = dups; cn[3] = nE;
            rs.tn[q] = tn;
            rs.lvl[q] = ni;
            rs.c0[q] = nc0;
            rs.flags[q] = rs.flags[q] & ~kFlagPend;
            s.i = ni; s.c0 = nc0; s.tn = tn; s.tsel = (T == T1) ? 1 : 0;
        }
    }
    __syncwarp();
}

// insert (id, ord) into the query's hash set, keeping the minimum ord per id; returns the slot
__device__ __forceinline__ uint32_t hs_min_insert(unsigned long long* hs, uint32_t id, uint32_t ord) {
    const unsigned long long key = ((unsigned long long)id << 32) | ord;
    uint32_t h = ch_slot(id);
    for (;;) {
        unsigned long long old = hs[h];
        if (old == kE64) {
            old = atomicCAS(&hs[h], kE64, key);
            if (old == kE64) return h;
        }
        if ((uint32_t)(old >> 32) == id) {
            if ((uint32_t)old > ord) atomicMin(&hs[h], key);
            return h;
        }
        h = ch_next(h);
    }
}

#ifndef PFG_CHUNK_MINB
#define PFG_CHUNK_MINB 8
#endif
// mode 0: a round (merge of the pending chunk, then the next chunk); mode 1: merge only (the
// queries still running go to the fused kernel's list)
template <int EPL>
__global__ void __launch_bounds__(kCT, PFG_CHUNK_MINB) k_chunk(QueryParams p, int par, int mode) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ChunkSmem& s = *reinterpret_cast<ChunkSmem*>(smem_raw);
    const int tstride = align16(p.kt * 8) / 8;
    uint64_t* Tb = reinterpret_cast<uint64_t*>(smem_raw + align16((int)sizeof(ChunkSmem)));
    float* qrow = reinterpret_cast<float*>(Tb + 2 * tstride);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const RoundState& rs = p.rs;
    const uint32_t nact = rs.ctl->nact[par];
    const uint32_t* act = rs.act[par];
    const size_t pin = (size_t)(par ^ 1) * rs.pool_stride;   // the previous round's pool (merge)
    const size_t pout = (size_t)par * rs.pool_stride;        // this round's pool
    // developer instrumentation (a -DPFG_CHUNK_PROF=1 build with PFG_PHASE_PROF=1): per-phase cycles
    // of thread 0, summed over queries
#if PFG_CHUNK_PROF
    unsigned long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tp = 0;
    auto mark = [&](int ph) {
        if (p.prof && tid == 0) { const long long t = clock64(); pc[ph] += (unsigned long long)(t - tp); tp = t; }
    };
#else
    auto mark = [](int) {};
#endif
    // dynamic scheduling with the next query claimed (and its index loaded) by the last warp while
    // the CTA works on the current one
    if (tid == 0) {
        const uint32_t a = atomicAdd(&rs.ctl->wk[par][0], 1u);
        s.wa[0] = a;
        s.wq[0] = a < nact ? (int64_t)act[a] : 0;
    }
    for (int t = tid; t < 65; t += kCT) s.taub[t] = __ldg(p.taub + t);
    for (int it = 0;; ++it) {
        __syncthreads();
        mark(7);
        const int sl = it & 1;
        if (s.wa[sl] >= nact) break;
        if (tid == kCT - 32) {
            const uint32_t a = atomicAdd(&rs.ctl->wk[par][0], 1u);
            s.wa[sl ^ 1] = a;
            s.wq[sl ^ 1] = a < nact ? (int64_t)act[a] : 0;
        }
#if PFG_CHUNK_PROF
        if (p.prof && tid == 0) pc[6] += 1;
#endif
        const int64_t q = s.wq[sl];
        // the query's state, loaded in parallel (independent loads)
        if (tid < 32) {
            const int tn0 = rs.tn[q];
            if (tid < tn0) Tb[tid] = rs.T[q * p.kt + tid];
            for (int t = tid + 32; t < tn0; t += 32) Tb[t] = rs.T[q * p.kt + t];
            if (tid == 0) { s.tn = tn0; s.tsel = 0; s.stop = 0; }
        } else if (tid == 32) {
            s.fl = rs.flags[q];
        } else if (tid == 33) {
            s.i = rs.lvl[q];
        } else if (tid == 34) {
            s.c0 = rs.c0[q];
        }
        __syncthreads();
        const int fl = s.fl;
        if (fl & kFlagPend) {
            mark(7);
            chunk_merge(p, q, pin, Tb, Tb + tstride, s, tid);
            __syncthreads();
            mark(0);
            if (s.stop) continue;
        }
        const int i = s.i, c0 = s.c0, tn = s.tn;
        const uint64_t* T = Tb + s.tsel * tstride;
        if (mode == 1 || i == 0) {
            // merge-only pass, or the i = 0 linear scan (R-13): the fused kernel continues the query
            if (tid == 0) {
                rs.flags[q] |= kFlagFused;
                push(rs.fused, &rs.ctl->nfused, (uint32_t)q);
            }
            continue;
        }
        // ---- expand: the chunk (R-17), its tau, codes and emitted ranges (R-12)
        if (wid == 0) {
            const int nr = chunk_reps(p, i, c0, tn, T, lane);
            int tau = 64;
            if (p.use_filter && tn == p.k_eff) {
                // tau = min{t : ip_k >= taub[t]} (taub[64] = -1)
                const float ip = fminf(fmaxf(key_sim(T[p.k_eff - 1]), -1.0f), 1.0f);
                int lo = 0, hi = 64;
                while (lo < hi) { const int mid = (lo + hi) >> 1; if (ip >= s.taub[mid]) hi = mid; else lo = mid + 1; }
                tau = lo;
            }
            if (lane == 0) {
                s.nr = nr; s.tau = tau; s.nE = rs.cnt[q * kCnt + 3]; s.probes = 0; s.ns = 0; s.overflow = 0;
            }
        }
        __syncthreads();
        const int nr = s.nr, tau = s.tau;
        const bool filt = p.use_filter && tau < 64;
        uint4* cur = p.cur + q * p.L;
        if (tid < nr) {
            s.sk[tid] = filt ? __ldg(p.qsk + q * p.M + __ldg(p.slot + c0 + tid)) : 0ull;
            s.pcnt[tid] = 0;
            s.fcnt[tid] = 0;
        }
        if (i == p.K) {
            if (tid < nr && c0 + tid < p.qc_n) s.qc[tid] = __ldg(p.qcodes + q * p.qc_ld + c0 + tid);
            if (c0 + nr > p.qc_n) {
                // repetitions beyond the precomputed codes: hashed here (FHT-CP, lane groups of
                // EPL lanes per repetition, the warps taking groups in turn)
                for (int t = tid; t < p.dpad; t += kCT) qrow[t] = p.qx[q * p.dpad + t];
                __syncthreads();
                constexpr int G = 32 / EPL;
                const int r0 = max(0, p.qc_n - c0);
                for (int rb = r0 + wid * G; rb < nr; rb += kCW * G)
                    group_rep_codes<EPL>(qrow, p.d, p.dp, p.ell, p.c, p.K, p.sg, c0, rb, min(nr, rb + G), s.qc, lane);
            }
            __syncthreads();
        }
        {
            uint32_t probes = 0;
            for (int task = tid; task < 2 * nr; task += kCT) {
                const bool left = task < nr;
                const int r = left ? task : task - nr;
                const int j = c0 + r;
                if (i == p.K && j < p.qb_n) {
                    const uint4 b = __ldg(p.qbnd + q * p.qb_ld + j);
                    s.bnd[task] = left ? b.x : b.y;
                    if (left) probes += b.z;
                } else if (i == p.K) {
                    const uint32_t qc = s.qc[r];
                    s.bnd[task] = rep_lower_bound(p, j, left ? (uint64_t)qc : (uint64_t)qc + 1, probes);
                } else {
                    const uint4 cu = cur[j];
                    s.bnd[task] = widen_side(p, j, i, cu.x, left ? cu.y : cu.z, left, probes);
                    if (left) s.qc[r] = cu.x;
                }
            }
            if (probes) atomicAdd(&s.probes, probes);
        }
        __syncthreads();
        if (wid == 0) {
            uint32_t em = 0;
            if (lane < nr) {
                const int j = c0 + lane;
                uint32_t nelo, elo, ehi, nehi;
                if (i == p.K) {
                    const uint32_t a_ = s.bnd[lane], b_ = s.bnd[nr + lane];
                    const uint32_t B = (uint32_t)p.B;
                    elo = ehi = nelo = a_;
                    const uint64_t v = (uint64_t)a_ + (uint64_t)((b_ - a_ + B - 1) / B) * B;
                    nehi = (uint32_t)(v > (uint64_t)p.n ? p.n : v);
                } else {
                    const uint4 cu = cur[j];
                    elo = cu.y; ehi = cu.z;
                    nelo = s.bnd[lane]; nehi = s.bnd[nr + lane];
                }
                s.lo_new[lane] = nelo; s.lo_old[lane] = elo; s.hi_old[lane] = ehi;
                em = (elo - nelo) + (nehi - ehi);
                rs.pend[q * kMaxR + lane] = make_uint4(s.qc[lane], nelo, nehi, 0u);
            }
            uint32_t incl = em;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t o = __shfl_up_sync(kFull, incl, off);
                if (lane >= off) incl += o;
            }
            const uint32_t total = __shfl_sync(kFull, incl, nr - 1);
            if (lane < nr) s.beg[lane + 1] = incl;
            if (lane == 0) {
                s.beg[0] = 0;
                s.total = total;
                s.direct = (nr == 1 && tau == 64 && s.nE == 0) ? 1 : 0;
            }
        }
        __syncthreads();
        mark(1);
        // ---- scan, filter, dedupe
        const uint32_t total = s.total, nE = s.nE;
        uint32_t* E = rs.E + q * (int64_t)rs.Ecap;
        if (s.direct) {
            // the search's first chunk: one repetition, nothing evaluated, tau = 64 -- every emitted
            // id is fresh (a repetition holds each id once)
            if (nE + total > rs.hmax) {
                if (tid == 0) s.overflow = 1;
            } else {
                const Entry* tj = p.tab + (int64_t)c0 * p.n;
                const uint32_t lenA = s.lo_old[0] - s.lo_new[0];
                for (uint32_t g = tid; g < total; g += kCT) {
                    const uint32_t pos = g < lenA ? s.lo_new[0] + g : s.hi_old[0] + (g - lenA);
                    E[g] = __ldg(reinterpret_cast<const uint32_t*>(tj + pos));
                }
                if (tid == 0) { s.ns = total; s.pcnt[0] = total; s.fcnt[0] = total; }
            }
        } else {
            // the query's evaluated set (ord 0), rebuilt from its evaluated list
            for (int t = tid; t < kCH / 2; t += kCT) reinterpret_cast<ulonglong2*>(s.hs)[t] = make_ulonglong2(kE64, kE64);
            __syncthreads();
            for (uint32_t e0 = 0; e0 < nE; e0 += kCT * 8) {
                uint32_t v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = e0 + u * kCT + tid;
                    v[u] = e < nE ? E[e] : kEmpty;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (v[u] != kEmpty) hs_min_insert(s.hs, v[u], 0u);
            }
            // batches of kCB positions: candidates of batch b insert (id, position + 1) after every
            // insert of batches < b (one barrier per batch); a later batch's inserts never lower an
            // earlier batch's minimum (larger positions), so the checks of batch b may overlap them
            for (uint32_t g0 = 0; g0 < total; g0 += kCB) {
                uint32_t idv[kCU], hsl[kCU];
                int rv[kCU];
                bool pass[kCU];
                {
                    // this thread's repetition at its first position of the batch (positions grow with u)
                    const uint32_t gf = g0 + tid;
                    int rl = 0;
                    {
                        int lo = 0, hi = nr;   // largest r with beg[r] <= gf
                        while (hi - lo > 1) { const int mid = (lo + hi) >> 1; if (s.beg[mid] <= gf) lo = mid; else hi = mid; }
                        rl = lo;
                    }
#pragma unroll
                    for (int u = 0; u < kCU; ++u) {
                        const uint32_t g = g0 + u * kCT + tid;
                        pass[u] = false;
                        rv[u] = -1;
                        idv[u] = 0;
                        if (g < total) {
                            while (rl + 1 < nr && s.beg[rl + 1] <= g) ++rl;
                            const uint32_t o = g - s.beg[rl];
                            const uint32_t lenA = s.lo_old[rl] - s.lo_new[rl];
                            const uint32_t pos = o < lenA ? s.lo_new[rl] + o : s.hi_old[rl] + (o - lenA);
                            const uint4 en = __ldg(reinterpret_cast<const uint4*>(p.tab + (int64_t)(c0 + rl) * p.n + pos));
                            idv[u] = en.x;
                            rv[u] = rl;
                            pass[u] = !filt || __popcll((((uint64_t)en.w << 32) | en.z) ^ s.sk[rl]) <= (uint32_t)tau;
                        }
                    }
                }
                __syncthreads();   // the rebuild / earlier batches' inserts precede this batch's
                if (nE + s.ns > rs.hmax) break;   // (uniform: s.ns is complete up to the previous batch)
#pragma unroll
                for (int u = 0; u < kCU; ++u)
                    hsl[u] = pass[u] ? hs_min_insert(s.hs, idv[u], g0 + u * kCT + tid + 1) : 0u;
                __syncthreads();
#pragma unroll
                for (int u = 0; u < kCU; ++u) {
                    const uint32_t g = g0 + u * kCT + tid;
                    const bool fresh = pass[u] && s.hs[hsl[u]] == (((unsigned long long)idv[u] << 32) | (g + 1));
                    const uint32_t fm = __ballot_sync(kFull, fresh);
                    uint32_t eb = 0;
                    if (lane == 0 && fm) eb = atomicAdd(&s.ns, (uint32_t)__popc(fm));
                    eb = __shfl_sync(kFull, eb, 0);
                    if (fresh) {
                        const uint32_t e = eb + __popc(fm & lanemask_lt());
                        E[nE + e] = idv[u];
                        s.erep[e] = (uint8_t)rv[u];
                    }
                    // per-repetition counters, one shared-memory atomic per group of lanes of one repetition
                    const uint32_t grp = __match_any_sync(kFull, rv[u]);
                    const uint32_t pall = __ballot_sync(kFull, pass[u]);
                    if (rv[u] >= 0 && lane == __ffs(grp) - 1) {
                        const uint32_t pm = pall & grp, fmm = fm & grp;
                        if (pm) atomicAdd(&s.pcnt[rv[u]], __popc(pm));
                        if (fmm) atomicAdd(&s.fcnt[rv[u]], __popc(fmm));
                    }
                }
            }
            __syncthreads();
            if (tid == 0 && nE + s.ns > rs.hmax) s.overflow = 1;
        }
        __syncthreads();
        mark(2);
        if (s.overflow) {
            // the evaluated set would outgrow the hash set: the fused kernel redoes the chunk from
            // the committed state (its global bitmap takes any size)
            if (tid == 0) {
                rs.flags[q] |= kFlagFused;
                push(rs.fused, &rs.ctl->nfused, (uint32_t)q);
            }
            continue;
        }
        const uint32_t ns = s.ns;
        if (tid == 0) s.pbase = atomicAdd(&rs.ctl->pool_top[par], ns);
        __syncthreads();
        const uint32_t base = s.pbase;
        if ((uint64_t)base + ns > rs.pool_cap) {
            // no room in the round's pool: keep the claimed entries valid, hand the query off
            for (uint64_t e = (uint64_t)base + tid; e < rs.pool_cap && e < (uint64_t)base + ns; e += kCT) {
                rs.pool_id[pout + e] = 0u;
                rs.pool_q[pout + e] = (uint32_t)q;
            }
            if (tid == 0) {
                rs.flags[q] |= kFlagFused;
                push(rs.fused, &rs.ctl->nfused, (uint32_t)q);
            }
            continue;
        }
        if (s.direct) {
            for (uint32_t e0 = 0; e0 < ns; e0 += kCT * 4) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * kCT + tid;
                    v[u] = e < ns ? E[nE + e] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * kCT + tid;
                    if (e < ns) {
                        rs.pool_id[pout + base + e] = v[u];
                        rs.pool_q[pout + base + e] = (uint32_t)q;
                    }
                }
            }
        } else {
            // the survivors grouped by repetition (the merge takes them repetition by repetition;
            // the order within a repetition does not matter)
            if (wid == 0) {
                const uint32_t v = lane < nr ? s.fcnt[lane] : 0u;
                uint32_t incl = v;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t o = __shfl_up_sync(kFull, incl, off);
                    if (lane >= off) incl += o;
                }
                if (lane < nr) s.roff[lane] = incl - v;
            }
            __syncthreads();
            for (uint32_t e0 = 0; e0 < ns; e0 += kCT * 4) {
                uint32_t v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * kCT + tid;
                    v[u] = e < ns ? E[nE + e] : 0u;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * kCT + tid;
                    if (e < ns) {
                        const uint32_t dst = atomicAdd(&s.roff[s.erep[e]], 1u);
                        rs.pool_id[pout + base + dst] = v[u];
                        rs.pool_q[pout + base + dst] = (uint32_t)q;
                    }
                }
            }
        }
        if (tid < nr) {
            const uint32_t em = s.beg[tid + 1] - s.beg[tid];
            uint32_t* rc = rs.repcnt + (q * kMaxR + tid) * 3;
            rc[0] = em;
            rc[1] = em - s.pcnt[tid];
            rc[2] = s.pcnt[tid] - s.fcnt[tid];
        }
        if (tid == 0) {
            rs.rinfo[q] = make_uint4((uint32_t)nr, (uint32_t)tau, 0u, s.direct ? 1u : 0u);
            rs.poff[q] = base;
            rs.pn[q] = ns;
            rs.cnt[q * kCnt + 4] += s.probes;
            rs.flags[q] |= kFlagPend;
            push(rs.act[par ^ 1], &rs.ctl->nact[par ^ 1], (uint32_t)q);
        }
        mark(3);
    }
#if PFG_CHUNK_PROF
    if (p.prof && tid == 0)
        for (int t = 0; t < 8; ++t) atomicAdd(p.prof + 16 + t, pc[t]);
#endif
}

}  // namespace pfg
