// kernels_rounds.cuh — the round engine: the same adaptive query as k_query, executed one chunk
// (the chunk's repetitions at one level) of every active query per round, split into
// bulk-parallel phases so that each phase runs at its own best occupancy and the
// bandwidth-heavy similarity phase has full memory-level parallelism:
//
//   k_qbounds  per (query, repetition < qb_n): the level-K match range [a_K, b_K) by two
//              interleaved binary searches (once per search, before the rounds)
//   k_rinit    per query: state init; zero query rows answered directly
//   k_expand   warp per active query: the chunk, its tau, chunk codes, emitted ranges (R-12),
//              pending cursors, and the query's scan tiles of 128 positions
//   k_scan     warp per tile (fully data-parallel): table entries + sketch filter -> candidates
//   k_dedupe   warp per active query: claims in (repetition, position) order against the query's
//              evaluated-id hash set (shared memory; carried between rounds in global memory)
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
// pool counter ctl->pool_top[par]; k_expand resets the other parity's counters, k_merge fills
// act[par ^ 1].  No host synchronisation is needed between rounds.
#pragma once
#include "kernels_query.cuh"

namespace pfg {

constexpr int kFlagDone = 1, kFlagFused = 2, kFlagSaved = 4;  // kFlagSaved: hsave holds the set
// kFlagWide: the evaluated set lives in the query's visit-tag array (RoundState::wv); kFlagDefer:
// the chunk found no room in the wide tile buffer and is expanded again next round; kFlagRedo: the
// query widened while its chunk was deduplicated and runs the chunk again, wide, next round
constexpr int kFlagWide = 8, kFlagDefer = 16, kFlagRedo = 32;

// The round kernels take their parameters by value (blind rounds) or from device memory (the
// device-side loop's graph, so that one instantiated graph serves every search: k_setp writes the
// search's parameters there)
__device__ __forceinline__ const QueryParams& deref(const QueryParams& p) { return p; }
__device__ __forceinline__ const QueryParams& deref(const QueryParams* p) { return *p; }
__global__ void k_setp(QueryParams p, QueryParams* dst) { *dst = p; }
constexpr int kEPre = 16;  // evaluated ids loaded per lane per batch when the hash set is rebuilt
#ifndef PFG_SAVEMIN
#define PFG_SAVEMIN 512
#endif
constexpr int kSaveMin = PFG_SAVEMIN;  // k_dedupe rebuilds sets of at most this many ids instead of restoring them

__device__ __forceinline__ int tau_of_state(const QueryParams& p, int tn, const uint64_t* T) {
    if (!p.use_filter || tn != p.k_eff) return 64;
    float ip = key_sim(T[p.k_eff - 1]);
    ip = fminf(fmaxf(ip, -1.0f), 1.0f);
    int lo = 0, hi = 64;
    while (lo < hi) { const int mid = (lo + hi) >> 1; if (ip >= __ldg(p.taub + mid)) hi = mid; else lo = mid + 1; }
    return lo;
}


__device__ __forceinline__ void push(uint32_t* list, uint32_t* n, uint32_t q) { list[atomicAdd(n, 1u)] = q; }

// dynamic work distribution: the warp takes the next item from a counter (lane 0 draws, all
// lanes get it), so a warp that drew expensive items does not hold the kernel's tail
__device__ __forceinline__ uint32_t next_item(uint32_t* ctr, int lane) {
    uint32_t v = 0;
    if (lane == 0) v = atomicAdd(ctr, 1u);
    return __shfl_sync(kFull, v, 0);
}

// visit tag of (level i, repetition j): the search epoch in the high half, then the visit's place
// s = (K - i) L + j + 1 in the query's visiting order (the host keeps (K + 1) L < 2^16); tag s = 0
// marks the ids evaluated before the query widened
__device__ __forceinline__ uint32_t visit_tag(const QueryParams& p, int i, int j) {
    return p.rs.ctl->wtag | (uint32_t)((p.K - i) * p.L + j + 1);
}

// warp-collective: move the query's evaluated set into a visit-tag array of its own (false: none
// left).  The array's stale tags are from earlier searches (larger epochs' tags are smaller, so
// every stale tag is above the current search's tags) and no array is handed out twice per search.
__device__ __forceinline__ bool try_widen(const QueryParams& p, int64_t q, int lane) {
    const RoundState& rs = p.rs;
    uint32_t slot = 0;
    if (lane == 0) slot = atomicAdd(&rs.ctl->wnext, 1u);
    slot = __shfl_sync(kFull, slot, 0);
    if (slot >= rs.wslots) return false;
    uint32_t* W = rs.wv + (int64_t)slot * p.n;
    const uint32_t nE = rs.cnt[q * kCnt + 3];
    const uint32_t* E = rs.E + q * (int64_t)rs.Ecap;
    const uint32_t t0 = rs.ctl->wtag;
    for (uint32_t e = lane; e < nE; e += 32) W[E[e]] = t0;
    if (lane == 0) { rs.wslot[q] = slot; rs.flags[q] |= kFlagWide; }
    __syncwarp();
    return true;
}

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

__global__ void __launch_bounds__(256) k_qbounds(QueryParams p, uint4* __restrict__ out, const uint32_t* __restrict__ qlist,
                                                 int64_t nlist, int r0, int nreps, const uint32_t* __restrict__ nlist_dev) {
    // queries qlist[0..nlist) if given, else 0..nlist-1 (nlist from device memory if nlist_dev: a
    // grid-stride loop, the grid sized for the list's usual length, not its capacity);
    // repetitions r0 .. r0 + nreps - 1
    const int64_t tot = (nlist_dev ? min(nlist, (int64_t)*nlist_dev) : nlist) * nreps;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t / nreps;
    const int j = r0 + (int)(t - a * nreps);
    const int64_t q = qlist ? (int64_t)qlist[a] : a;
    if (p.qzero[q]) { out[q * p.qb_ld + j] = make_uint4(0, 0, 0, 0); continue; }
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
}

// ---------------------------------------------------------------------------------------------
__global__ void k_rinit(QueryParams p, uint32_t wtag) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q == 0) p.rs.ctl->wtag = wtag;
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
// k_expand: warp per active query.  The chunk (chunk_reps), its tau, the query codes of the chunk
// (precomputed, or hashed here), the emitted ranges of every repetition (level K: the match range
// rounded up to whole segments; deeper levels: the segment loop, R-12, in closed form after its
// first probe, widen_side), the pending cursors, and
// the scan tiles of 128 positions (positions in (repetition, position) order).
struct ExpandSmem {
    uint32_t qc[kMaxR], bnd[2 * kMaxR];
};
__host__ __device__ inline int expand_smem_bytes(int dpad, bool lazy) {
    return align16((int)sizeof(ExpandSmem)) + (lazy ? align16(dpad * 4) : 0);
}
#ifndef PFG_TILE
#define PFG_TILE 128
#endif
constexpr int kTile = PFG_TILE;   // emitted positions per scan tile
#ifndef PFG_DLONG
#define PFG_DLONG 2048
#endif
constexpr int kDedupeLong = PFG_DLONG;  // emitted positions from which k_dedupe schedules a chunk first

// LZ = false: a round whose repetitions all have precomputed codes (the host knows the largest
// repetition a round can reach), compiled without the lazy hashing (fewer registers, more warps)
template <int EPL, typename PP, bool LZ = true>
#ifndef PFG_EXPAND_MINB
#define PFG_EXPAND_MINB 6
#endif
__global__ void __launch_bounds__(128, LZ ? PFG_EXPAND_MINB : 8) k_expand(PP pp, int par, int lazy) {
    pdl_wait();
    const QueryParams& p = deref(pp);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    ExpandSmem* c = (ExpandSmem*)(smem_raw + wib * expand_smem_bytes(p.dpad, lazy));
    float* qrow = (float*)((unsigned char*)c + align16((int)sizeof(ExpandSmem)));
    const RoundState& rs = p.rs;
    const uint32_t nact = rs.ctl->nact[par];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        rs.ctl->nact[par ^ 1] = 0; rs.ctl->pool_top[par ^ 1] = 0; rs.ctl->ntiles[par ^ 1] = 0;
        for (int t = 0; t < 4; ++t) rs.ctl->wk[par ^ 1][t] = 0;
        rs.ctl->dfront[par ^ 1] = 0; rs.ctl->dback[par ^ 1] = 0;
        rs.ctl->nwt[par ^ 1] = 0; rs.ctl->nwide[par ^ 1] = 0;
    }
    const uint32_t* act = rs.act[par];
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t a = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; a < nact; a += nw) {
        const int64_t q = act[a];
        const int i = rs.lvl[q], c0 = rs.c0[q], tn = rs.tn[q];
        bool wide = (rs.flags[q] & kFlagWide) != 0;
        // i = 0 (wide queries only): one repetition, the whole table of repetition 0, no filter
        // (R-13)
        const int nr = i == 0 ? 1 : chunk_reps(p, i, c0, tn, rs.T + q * p.kt, lane);
        const int tau = i == 0 ? 64 : tau_of_state(p, tn, rs.T + q * p.kt);
        uint4* cur = p.cur + q * p.L;
        uint32_t probes = 0;
        if (i == p.K) {
            if (lane < nr && c0 + lane < p.qc_n) c->qc[lane] = __ldg(p.qcodes + q * p.qc_ld + c0 + lane);
            if (LZ && c0 + nr > p.qc_n) {
                for (int t = lane; t < p.dpad; t += 32) qrow[t] = p.qx[q * p.dpad + t];
                __syncwarp();
                group_rep_codes<EPL>(qrow, p.d, p.dp, p.ell, p.c, p.K, p.sg, c0, max(0, p.qc_n - c0), nr, c->qc, lane);
            }
            __syncwarp();
        }
        for (int task = lane; i > 0 && task < 2 * nr; task += 32) {
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
                c->bnd[task] = widen_side(p, j, i, cu.x, left ? cu.y : cu.z, left, probes);
                if (left) c->qc[r] = cu.x;
            }
        }
        __syncwarp();
        uint32_t em = 0, nelo = 0, elo = 0, ehi = 0, nehi = 0;
        if (lane < nr) {
            const int j = c0 + lane;
            if (i == 0) {
                nehi = (uint32_t)p.n;
            } else if (i == p.K) {
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
            em = (elo - nelo) + (nehi - ehi);
            rs.pend[q * kMaxR + lane] = make_uint4(i > 0 ? c->qc[lane] : 0u, nelo, nehi, 0u);
        }
        uint32_t incl = em;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += o;
        }
        const uint32_t total = __shfl_sync(kFull, incl, nr - 1);
        // scan tiles: each repetition's left part [nelo, elo) and right part [ehi, nehi) split into
        // pieces of at most kTile positions, in (repetition, position) order
        const uint32_t lenA = elo - nelo, lenB = nehi - ehi;
        const uint32_t tA = (lenA + kTile - 1) / kTile, tB = (lenB + kTile - 1) / kTile;
        uint32_t tin = tA + tB;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, tin, off);
            if (lane >= off) tin += o;
        }
        const uint32_t ntl = __shfl_sync(kFull, tin, nr - 1);
        if (lane < nr) rs.repcnt[(q * kMaxR + lane) * 3] = em;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) probes += __shfl_xor_sync(kFull, probes, off);
        // a single repetition with nothing evaluated yet and tau = 64 (the search's first chunk):
        // every emitted id is fresh (a repetition holds each id once), so k_scan writes the ids
        // straight to the evaluated list and the round's pool and k_dedupe skips the query
        bool direct = !wide && nr == 1 && tau == 64 && rs.cnt[q * kCnt + 3] == 0;
        const bool over = direct ? total > rs.hmax : ntl > (uint32_t)(rs.Ccap / kTile);
        // a chunk beyond the hash set's reach moves the query to the wide path (if an array is
        // left; else the fused kernel takes it)
        if (!wide && over && try_widen(p, q, lane)) { wide = true; direct = false; }
        uint32_t base = 0;
        bool handed = false;
        if (lane == 0) {
            rs.rinfo[q] = make_uint4((uint32_t)nr, (uint32_t)tau, ntl, direct ? 1u : 0u);
            rs.cnt[q * kCnt + 4] += probes;
            if (wide) {
                if (ntl) base = atomicAdd(&rs.ctl->nwt[par], ntl);
                if ((uint64_t)base + ntl > rs.wcap) { rs.flags[q] |= kFlagDefer; atomicAdd(&rs.ctl->wdefer, 1u); }
            } else {
                if (over) rs.flags[q] |= kFlagFused;
                if (direct && !over) {
                    const uint32_t pb = atomicAdd(&rs.ctl->pool_top[par], total);
                    if ((uint64_t)pb + total > rs.pool_cap) {
                        rs.flags[q] |= kFlagFused;
                    } else {
                        rs.poff[q] = pb;
                        rs.pn[q] = total;
                        uint32_t* rc = rs.repcnt + q * kMaxR * 3;
                        rc[1] = 0; rc[2] = 0;
                    }
                }
                if (ntl && !(rs.flags[q] & kFlagFused)) base = atomicAdd(&rs.ctl->ntiles[par], ntl);
            }
            handed = (rs.flags[q] & (kFlagFused | kFlagDefer)) != 0;
            // k_dedupe takes the long chunks first (a shorter tail for its dynamic scheduler)
            const uint32_t slot = total >= (uint32_t)kDedupeLong ? atomicAdd(&rs.ctl->dfront[par], 1u)
                                                                  : nact - 1u - atomicAdd(&rs.ctl->dback[par], 1u);
            rs.dord[par][slot] = (uint32_t)q;
        }
        base = __shfl_sync(kFull, base, 0);
        handed = __shfl_sync(kFull, handed ? 1 : 0, 0) != 0;
        if (wide) {
            if (handed) {
                // no room: the part of the claimed range below the capacity holds dead tiles
                for (uint32_t t = base + lane; t < rs.wcap && t < base + ntl; t += 32)
                    rs.wtiles[2 * (int64_t)t] = make_uint4((uint32_t)q, 0u, 0u, 0u);
            } else {
                // wide tiles: descriptors {query, table position, 0, count | rep << 16 | tau << 24}
                // {sketch word, visit tag, j}, written by the whole warp one repetition at a time;
                // rtile holds each repetition's first tile
                uint32_t* rt = rs.rtile + q * (kMaxR + 1);
                if (lane < nr) rt[lane] = base + tin - tA - tB;
                if (lane == 0) rt[nr] = base + ntl;
                for (int r = 0; r < nr; ++r) {
                    const int j = c0 + r;
                    const uint32_t t0 = base + __shfl_sync(kFull, tin - tA - tB, r);
                    const uint32_t a0 = __shfl_sync(kFull, nelo, r), la = __shfl_sync(kFull, lenA, r);
                    const uint32_t b0 = __shfl_sync(kFull, ehi, r), lb = __shfl_sync(kFull, lenB, r);
                    const uint32_t ta = (la + kTile - 1) / kTile, tb = (lb + kTile - 1) / kTile;
                    const uint64_t sk = (p.use_filter && tau < 64) ? __ldg(p.qsk + q * p.M + __ldg(p.slot + j)) : 0ull;
                    const uint32_t tag = visit_tag(p, i, j);
                    for (uint32_t t = lane; t < ta + tb; t += 32) {
                        const bool pa = t < ta;
                        const uint32_t o = (pa ? t : t - ta) * kTile;
                        const uint32_t len = pa ? la : lb;
                        const uint32_t cnt = min((uint32_t)kTile, len - o);
                        rs.wtiles[2 * (int64_t)(t0 + t)] = make_uint4((uint32_t)q, (pa ? a0 : b0) + o, 0u,
                                                                      cnt | ((uint32_t)r << 16) | ((uint32_t)tau << 24));
                        rs.wtiles[2 * (int64_t)(t0 + t) + 1] = make_uint4((uint32_t)sk, (uint32_t)(sk >> 32), tag, (uint32_t)j);
                    }
                }
            }
        } else if (!handed && lane < nr) {
            // lane r writes the descriptors of repetition r's pieces: {query, table position,
            // chunk position, count | rep << 16 | tau << 24} {sketch word, tile index | direct, j}
            const int j = c0 + lane;
            const uint64_t sk = (p.use_filter && tau < 64) ? __ldg(p.qsk + q * p.M + __ldg(p.slot + j)) : 0ull;
            uint32_t t = tin - tA - tB;
            uint32_t g = incl - em;
            for (int part = 0; part < 2; ++part) {
                const uint32_t len = part ? lenB : lenA, p0 = part ? ehi : nelo;
                for (uint32_t o = 0; o < len; o += kTile, ++t) {
                    const uint32_t cnt = min((uint32_t)kTile, len - o);
                    rs.tiles[2 * (int64_t)(base + t)] = make_uint4((uint32_t)q, p0 + o, g + o,
                                                                   cnt | ((uint32_t)lane << 16) | ((uint32_t)tau << 24));
                    rs.tiles[2 * (int64_t)(base + t) + 1] = make_uint4((uint32_t)sk, (uint32_t)(sk >> 32),
                                                                       t | (direct ? 0x80000000u : 0u), (uint32_t)j);
                }
                g += len;
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// k_scan: warp per tile -- up to kTile consecutive table positions of one repetition of one
// query's chunk (descriptor from k_expand): load the 16-byte entries, apply the sketch filter
// with the chunk's tau, and compact the passing ids in order to the tile's
// candidate slots (count | repetition << 16 in tcnt).  Fully data-parallel.
//
// Wide tiles (after the hash-set tiles): the passing ids claim their first visit in the query's
// visit-tag array by atomicMin(W[id], tag); an id whose array already held a smaller tag was
// evaluated before (an earlier chunk, or an earlier repetition of this chunk that got there
// first) and is a duplicate; the others are provisional until k_sims checks that no earlier
// repetition of the chunk lowered the tag after this claim.
// two tiles per call (aw1 < 0: one), their loads interleaved: late in a search a wide tile holds
// few passing ids and its cost is the chain of dependent loads (entries, tags, claims)
__device__ __forceinline__ void scan_wide_tiles(const QueryParams& p, int64_t aw0, int64_t aw1, int lane) {
    const RoundState& rs = p.rs;
    constexpr int U = kTile / 32;
    int64_t aw[2] = {aw0, aw1};
    uint32_t cnt[2], rep[2], tau[2], tag[2];
    uint64_t sk[2];
    const Entry* tj[2];
    uint32_t* W[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        cnt[h] = 0; rep[h] = 0; tau[h] = 64; tag[h] = 0; sk[h] = 0; tj[h] = p.tab; W[h] = rs.wv;
        if (aw[h] < 0) continue;
        const uint4 d0 = rs.wtiles[2 * aw[h]], d1 = rs.wtiles[2 * aw[h] + 1];
        cnt[h] = d0.w & 0xffffu; rep[h] = (d0.w >> 16) & 0xffu; tau[h] = d0.w >> 24;
        sk[h] = ((uint64_t)d1.y << 32) | d1.x;
        tag[h] = d1.z;
        tj[h] = p.tab + (int64_t)d1.w * p.n + d0.y;
        if (cnt[h]) W[h] = rs.wv + (int64_t)rs.wslot[d0.x] * p.n;
    }
    uint4 e[2][U];
    bool pass[2][U];
    uint32_t old[2][U];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t o = u * 32 + lane;
            if (o < cnt[h]) e[h][u] = __ldg(reinterpret_cast<const uint4*>(tj[h] + o));
        }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t o = u * 32 + lane;
            pass[h][u] = o < cnt[h];
            if (pass[h][u] && p.use_filter && tau[h] < 64)
                pass[h][u] = __popcll((((uint64_t)e[h][u].w << 32) | e[h][u].z) ^ sk[h]) <= tau[h];
            old[h][u] = pass[h][u] ? __ldcg(W[h] + e[h][u].x) : 0u;
        }
    // a smaller tag already there: a duplicate, no atomic needed (most passing ids, late in a
    // search); else claim the visit
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (pass[h][u] && old[h][u] >= tag[h]) old[h][u] = atomicMin(W[h] + e[h][u].x, tag[h]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (aw[h] < 0) continue;
        uint32_t* cand = rs.wcand + aw[h] * kTile;
        uint32_t np = 0, npass = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            npass += __popc(__ballot_sync(kFull, pass[h][u]));
            const bool prov = pass[h][u] && old[h][u] >= tag[h];
            const uint32_t pm = __ballot_sync(kFull, prov);
            if (prov) cand[np + __popc(pm & lanemask_lt())] = e[h][u].x;
            np += __popc(pm);
        }
        if (lane == 0) rs.wtcnt[aw[h]] = cnt[h] ? (np | (npass << 8) | (rep[h] << 16)) : 0u;
    }
}

#ifndef PFG_SCAN_MINB
#define PFG_SCAN_MINB 1
#endif
template <typename PP, bool WIDE>
__global__ void __launch_bounds__(256, WIDE ? 1 : PFG_SCAN_MINB) k_scan(PP pp, int par) {
    pdl_wait();
    const QueryParams& p = deref(pp);
    const int lane = threadIdx.x & 31;
    const RoundState& rs = p.rs;
    const uint32_t ntiles = rs.ctl->ntiles[par];
    const uint32_t nwt = min(rs.ctl->nwt[par], rs.wcap);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (WIDE)  // WIDE = false: no wide queries in this search (the lean variant keeps its registers)
        for (int64_t aw = wid * 2; aw < nwt; aw += nw * 2) scan_wide_tiles(p, aw, aw + 1 < nwt ? aw + 1 : -1, lane);
    // the next tile's descriptor is fetched before this tile's entries are read
    uint4 nd0 = make_uint4(0, 0, 0, 0), nd1 = nd0;
    if (wid < ntiles) { nd0 = rs.tiles[2 * wid]; nd1 = rs.tiles[2 * wid + 1]; }
    for (int64_t a = wid; a < ntiles; a += nw) {
        const uint4 d0 = nd0, d1 = nd1;
        if (a + nw < ntiles) { nd0 = rs.tiles[2 * (a + nw)]; nd1 = rs.tiles[2 * (a + nw) + 1]; }
        const int64_t q = d0.x;
        const uint32_t cnt = d0.w & 0xffffu, rep = (d0.w >> 16) & 0xffu, tau = d0.w >> 24;
        const uint64_t sk = ((uint64_t)d1.y << 32) | d1.x;
        const uint32_t t = d1.z & 0x7fffffffu;
        const bool direct = d1.z >> 31;
        const Entry* tj = p.tab + (int64_t)d1.w * p.n + d0.y;
        uint4 e[kTile / 32];
#pragma unroll
        for (int u = 0; u < kTile / 32; ++u) {
            const uint32_t o = u * 32 + lane;
            if (o < cnt) e[u] = __ldg(reinterpret_cast<const uint4*>(tj + o));
        }
        if (direct) {
            // every position is a fresh evaluated id (k_expand)
            const uint32_t pb = rs.poff[q] + d0.z;
            uint32_t* E = rs.E + q * (int64_t)rs.Ecap + d0.z;
#pragma unroll
            for (int u = 0; u < kTile / 32; ++u) {
                const uint32_t o = u * 32 + lane;
                if (o < cnt) {
                    rs.pool_id[pb + o] = e[u].x;
                    rs.pool_q[pb + o] = (uint32_t)q;
                    E[o] = e[u].x;
                }
            }
            continue;
        }
        uint32_t* cand = rs.cand + q * (int64_t)rs.Ccap + (int64_t)t * kTile;
        uint32_t np = 0;
#pragma unroll
        for (int u = 0; u < kTile / 32; ++u) {
            const uint32_t o = u * 32 + lane;
            bool pass = o < cnt;
            if (pass && p.use_filter && tau < 64) pass = __popcll((((uint64_t)e[u].w << 32) | e[u].z) ^ sk) <= tau;
            const uint32_t pm = __ballot_sync(kFull, pass);
            if (pass) cand[np + __popc(pm & lanemask_lt())] = e[u].x;
            np += __popc(pm);
        }
        if (lane == 0) rs.tcnt[q * (int64_t)(rs.Ccap / kTile) + t] = np | (rep << 16);
    }
}

// ---------------------------------------------------------------------------------------------
// k_dedupe: warp per active query.  Rebuild the evaluated-id hash set from the query's evaluated
// list, then walk the chunk's candidates in (repetition, position) order: filtered positions and
// duplicates are counted per repetition, fresh ids are claimed in order (R-17/R-18), appended to
// the evaluated list and to the round's pool.
struct DedupeSmem {
    uint32_t hs[kHC];
    uint32_t beg[kMaxR + 1];
    uint32_t fcnt[kMaxR], dcnt[kMaxR];
};
#ifndef PFG_CPRE
#define PFG_CPRE 8
#endif
constexpr int kCPre = PFG_CPRE;   // candidate ids loaded per lane per batch
// the carried hash set is restored and saved in 16-byte pieces, 128 slots per warp step
static_assert(kHC % 128 == 0, "k_dedupe moves the hash set in whole warp steps of 128 slots");

template <typename PP>
__global__ void __launch_bounds__(128, 6) k_dedupe(PP pp, int par) {   // 6 blocks: the shared-memory limit
    pdl_wait();
    const QueryParams& p = deref(pp);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    DedupeSmem* c = (DedupeSmem*)(smem_raw + wib * align16((int)sizeof(DedupeSmem)));
    const RoundState& rs = p.rs;
    const uint32_t nact = rs.ctl->nact[par];
    const uint32_t* act = rs.dord[par];
    for (uint32_t a = next_item(&rs.ctl->wk[par][2], lane); a < nact; a = next_item(&rs.ctl->wk[par][2], lane)) {
        const int64_t q = act[a];
        const int fl = rs.flags[q];
        if (fl & (kFlagFused | kFlagWide)) continue;
        const uint4 info = rs.rinfo[q];
        if (info.w) continue;  // direct chunk: k_scan wrote the evaluated ids and the pool
        const int nr = (int)info.x;
        const uint32_t ntl = info.z;
        const uint32_t nE = rs.cnt[q * kCnt + 3];
        uint32_t* E = rs.E + q * (int64_t)rs.Ecap;
        const uint32_t* cand = rs.cand + q * (int64_t)rs.Ccap;
        // the hash set as the previous round left it: saved in global memory once it holds more
        // than kSaveMin ids (kFlagSaved), else rebuilt here from the evaluated list (cheaper than
        // 16 KB of traffic for a small set)
        uint4* hsv = reinterpret_cast<uint4*>(rs.hsave + q * (int64_t)kHC);
        const bool saved = (fl & kFlagSaved) != 0;
        // k_scan left the passing candidates of tile t at [t*kTile, t*kTile + tcnt[t]), in order;
        // a batch is kCPre/4 consecutive tiles.  The tile counts (at most 64 tiles) are read once,
        // and a batch's candidate words are read whole (the buffer is Ccap long; positions beyond
        // a tile's count are masked after the load), the next batch's while this one is processed
        constexpr int kTPB = kCPre * 32 / kTile;
        const uint32_t* tcnt = rs.tcnt + q * (int64_t)(rs.Ccap / kTile);
        const uint32_t tw0 = lane < ntl ? tcnt[lane] : 0u;
        const uint32_t tw1 = lane + 32 < ntl ? tcnt[lane + 32] : 0u;
        uint32_t vn[kCPre];
        auto load_batch = [&](uint32_t t0) {
#pragma unroll
            for (int u = 0; u < kCPre; ++u) {
                const uint32_t t = t0 + u / (kTile / 32);
                vn[u] = t < ntl ? cand[t * kTile + (u % (kTile / 32)) * 32 + lane] : kEmpty;
            }
        };
        load_batch(0);
        if (!saved) {
            for (int t = lane; t < kHC / 4; t += 32) reinterpret_cast<uint4*>(c->hs)[t] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
            __syncwarp();
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
        } else {
            // global -> shared without the register round trip (LDGSTS, L2 only)
#pragma unroll
            for (int k = 0; k < kHC / 128; ++k) {
                const uint32_t sa = (uint32_t)__cvta_generic_to_shared(reinterpret_cast<uint4*>(c->hs) + k * 32 + lane);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(hsv + k * 32 + lane) : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        if (lane < nr) { c->fcnt[lane] = 0; c->dcnt[lane] = 0; }
        __syncwarp();
        uint32_t ns = 0;
        bool overflow = false;
        for (uint32_t t0 = 0; t0 < ntl && !overflow; t0 += kTPB) {
            uint32_t v[kCPre], h[kCPre];
            bool found[kCPre];
            uint32_t tc[kTPB];
            int trep[kTPB];
#pragma unroll
            for (int u = 0; u < kCPre; ++u) v[u] = vn[u];
            if (t0 + kTPB < ntl) load_batch(t0 + kTPB);
#pragma unroll
            for (int b = 0; b < kTPB; ++b) {
                const uint32_t t = t0 + b;   // warp-uniform
                const uint32_t w = t < 32 ? __shfl_sync(kFull, tw0, t & 31) : __shfl_sync(kFull, tw1, t & 31);
                tc[b] = t < ntl ? (w & 0xffffu) : 0u;
                trep[b] = (int)(w >> 16);
            }
#pragma unroll
            for (int u = 0; u < kCPre; ++u)
                if ((u % (kTile / 32)) * 32 + lane >= tc[u / (kTile / 32)]) v[u] = kEmpty;
            // membership in the set as it stands before this batch: independent read-only probes,
            // four slots per shared load (hs_lookup4); h[u] ends at the id's slot or the first empty
            // (the home quads of the whole batch loaded first)
            uint4 w4[kCPre];
#pragma unroll
            for (int u = 0; u < kCPre; ++u) {
                h[u] = hs_slot(v[u]);
                w4[u] = v[u] != kEmpty ? *reinterpret_cast<const uint4*>(c->hs + (h[u] & ~3u)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kCPre; ++u) {
                found[u] = false;
                if (v[u] != kEmpty && !hs_quad(w4[u], v[u], h[u], found[u])) found[u] = hs_lookup4(c->hs, v[u], h[u]);
            }
            // claims of the rest in (repetition, position) order, u in order; a later occurrence
            // of an id claimed earlier in the batch finds it in the set.  The per-tile duplicate
            // counts are kept in registers and added to the repetition's count once per tile.
            uint32_t dsum[kTPB];
#pragma unroll
            for (int b = 0; b < kTPB; ++b) dsum[b] = 0;
#pragma unroll
            for (int u = 0; u < kCPre; ++u) {
                if ((uint32_t)((u % (kTile / 32)) * 32) >= tc[u / (kTile / 32)]) continue;  // empty step (warp-uniform)
                const bool pass = v[u] != kEmpty;
                const bool need = pass && !found[u];
                bool fresh = false;
                // the 32 lanes of a step hold positions of one tile, i.e. of one repetition, whose
                // ids are distinct: every lane claims its own id (no grouping of equal ids needed)
                if (need) {
                    uint32_t hh = h[u];
                    for (;;) {
                        const uint32_t old = atomicCAS(&c->hs[hh], kEmpty, v[u]);
                        if (old == kEmpty) { fresh = true; break; }
                        if (old == v[u]) break;
                        hh = hs_next(hh);
                    }
                }
                const uint32_t fm = __ballot_sync(kFull, fresh);
                if (fresh) E[nE + ns + __popc(fm & lanemask_lt())] = v[u];
                ns += __popc(fm);
                // the step's live lanes are positions of one tile (one repetition): its duplicates
                // are the live lanes that claimed nothing
                const int b = u / (kTile / 32);
                const uint32_t live = min(32u, tc[b] - (uint32_t)((u % (kTile / 32)) * 32));
                dsum[b] += live - __popc(fm);
            }
            if (lane == 0) {
#pragma unroll
                for (int b = 0; b < kTPB; ++b)
                    if (tc[b]) {
                        c->fcnt[trep[b]] += tc[b];   // passing the filter (filtered = emitted - passing)
                        c->dcnt[trep[b]] += dsum[b];
                    }
            }
            if (nE + ns > rs.hmax) overflow = true;
        }
        __syncwarp();
        uint32_t base = 0;
        if (!overflow && lane == 0) base = atomicAdd(&rs.ctl->pool_top[par], ns);
        base = __shfl_sync(kFull, base, 0);
        if (!overflow && (uint64_t)base + ns > rs.pool_cap) overflow = true;
        if (overflow) {
            // the set outgrew the hash set: widen and run the chunk again next round (the committed
            // evaluated list E[0, nE) moves to the visit-tag array), else hand off to the fused kernel
            if (try_widen(p, q, lane)) { if (lane == 0) rs.flags[q] |= kFlagRedo; }
            else if (lane == 0) rs.flags[q] |= kFlagFused;
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
            uint32_t* rc = rs.repcnt + (q * kMaxR + lane) * 3;   // rc[0] = emitted (k_expand)
            rc[1] = rc[0] - c->fcnt[lane];
            rc[2] = c->dcnt[lane];
        }
        if (lane == 0) { rs.poff[q] = base; rs.pn[q] = ns; }
        // carry a large set to the next round (the fused kernel rebuilds it from E instead) --
        // unless the chunk was cut short by chunk_reps: then the k-th similarity before the chunk
        // already meets the stop threshold of its last repetition, so the query stops this round
        const int ci = rs.lvl[q], cc0 = rs.c0[q];
        const int nominal = min((ci == p.K && cc0 == 0 && !p.uniform) ? 1 : p.R, p.L - cc0);
        if (nE + ns > (uint32_t)kSaveMin && nr >= nominal) {
            if (lane == 0 && !saved) rs.flags[q] |= kFlagSaved;
#pragma unroll
            for (int k = 0; k < kHC / 128; ++k) __stcg(hsv + k * 32 + lane, reinterpret_cast<const uint4*>(c->hs)[k * 32 + lane]);
        }
        __syncwarp();
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

#ifndef PFG_SIMS_MINB
#define PFG_SIMS_MINB 2
#endif
// NR rows of one step: fp32 (R-2 lane chains + tree) or int16 (R-25, exact integer sums); lane
// r < NR holds row r's id (myid) and query (myq); lane l ends with row l / (32 / NR)
template <int NR, bool I16, bool ONEQ>
__device__ __forceinline__ float sims_step(const QueryParams& p, uint32_t myid, uint32_t myq, int lane) {
    uint32_t roff[NR], qoff[NR];
    const uint32_t nch = I16 ? (uint32_t)(p.dpad16 >> 3) : (uint32_t)(p.dpad >> 2);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        roff[r] = __shfl_sync(kFull, myid, r) * nch;
        qoff[r] = (ONEQ && r > 0) ? 0u : __shfl_sync(kFull, myq, r) * nch;
    }
    if constexpr (I16) {
        int acc[NR];
        rows_dot_i16<NR, ONEQ>(reinterpret_cast<const int4*>(p.x16), reinterpret_cast<const int4*>(p.qx16), roff, qoff,
                               (int)nch, lane, acc);
        return sim_of_i16(tree_rows<NR>(acc, lane));
    } else {
        float acc[NR];
        pool_sims_step<ONEQ>(reinterpret_cast<const float4*>(p.x), reinterpret_cast<const float4*>(p.qx), roff, qoff,
                             (int)nch, lane, acc);
        return tree_rows<NR>(acc, lane);
    }
}

#ifndef PFG_I16_NR
#define PFG_I16_NR 16
#endif
// 16-bit rows of at most 128 coordinates (16 chunks of 16 bytes): each half-warp takes 16 rows of a
// 32-row step (lane l reads chunk l & 15 of the rows of half l >> 4), so every lane loads and a
// step keeps twice the bytes in flight; the sums are exact int32 (R-25), so the reduction order
// does not matter.  Lane r < 32 holds row r's id (myid) and query (myq); lane l ends with row l.
template <bool ONEQ>
__device__ __forceinline__ int sims_step_i16_half(const QueryParams& p, uint32_t myid, uint32_t myq, int lane) {
    const uint32_t nch = (uint32_t)(p.dpad16 >> 3);
    const int half = lane >> 4, c = lane & 15;
    const int4* x4 = reinterpret_cast<const int4*>(p.x16);
    const int4* q4 = reinterpret_cast<const int4*>(p.qx16);
    uint32_t roff[16], qoff[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        // every lane takes part in the shuffles; lanes of half 1 keep the second set
        const uint32_t i0 = __shfl_sync(kFull, myid, r), i1 = __shfl_sync(kFull, myid, 16 + r);
        roff[r] = (half ? i1 : i0) * nch;
        if (!ONEQ) {
            const uint32_t q0 = __shfl_sync(kFull, myq, r), q1 = __shfl_sync(kFull, myq, 16 + r);
            qoff[r] = (half ? q1 : q0) * nch;
        }
    }
    const uint32_t qo = ONEQ ? __shfl_sync(kFull, myq, 0) * nch : 0u;
    int acc[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) acc[r] = 0;
    if ((uint32_t)c < nch) {
        int4 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = __ldg(x4 + roff[r] + c);
        const int4 qv0 = __ldg(q4 + qo + c);
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = dot8_i16(v[r], ONEQ ? qv0 : __ldg(q4 + qoff[r] + c));
    }
    // transposed halving within the half-warp: lane l ends with the sum of row l & 15 of its half
    int m = 16;
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
        const int hm = m >> 1;
        const bool up = lane & h;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (k < hm) {
                const int send = up ? acc[k] : acc[k + hm];
                const int keep = up ? acc[k + hm] : acc[k];
                acc[k] = keep + __shfl_xor_sync(kFull, send, h);
            }
        }
        m = hm;
    }
    return acc[0];
}
// flags bit 0 (the chunk engine, kernels_chunk.cuh): the pool of parity par starts at
// par * pool_stride, and the kernel resets the counters the next round's k_chunk starts from (its
// active list's successor, its pool, its work counter), none of which this launch reads;
// bit 1: a launch outside the device-side loop (its rows are also counted in sims_rows_blind)
template <typename PP, bool I16>
__global__ void __launch_bounds__(256, PFG_SIMS_MINB) k_sims(PP pp, int par, int flags) {
    pdl_wait();
    const int chunk = flags & 1;
    const QueryParams& p = deref(pp);
    constexpr int NR = I16 ? PFG_I16_NR : kRPI;   // int16 rows are half as long: more rows in flight
    constexpr int kSh = NR == 32 ? 0 : NR == 16 ? 1 : NR == 8 ? 2 : 3;
    const int lane = threadIdx.x & 31;
    const RoundState& rs = p.rs;
    const uint32_t top = min(rs.ctl->pool_top[par], rs.pool_cap);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const size_t po = chunk ? (size_t)par * rs.pool_stride : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicAdd(&rs.ctl->sims_rows, (unsigned long long)top);
        if (flags & 2) atomicAdd(&rs.ctl->sims_rows_blind, (unsigned long long)top);
        if (chunk) { rs.ctl->nact[par] = 0; rs.ctl->pool_top[par ^ 1] = 0; rs.ctl->wk[par ^ 1][0] = 0; }
    }
    const uint32_t* pool_id = rs.pool_id + po;
    const uint32_t* pool_q = rs.pool_q + po;
    uint64_t* pool_key = rs.pool_key + po;
    // lane r < NR holds entry b + r of the current step (rows beyond the end repeat the last);
    // the next step's entries are fetched before the current rows are read
    auto fetch = [&](int64_t b, uint32_t& id, uint32_t& qq) {
        if (lane < NR && b < top) {
            const int64_t e1 = (int64_t)top < b + NR ? (int64_t)top : b + NR;
            const int64_t e = b + lane < e1 ? b + lane : e1 - 1;
            id = pool_id[e];
            qq = pool_q[e];
        }
    };
    if constexpr (I16) {
        if (p.dpad16 <= 128) {
            // 32 rows per step, a half-warp per 16 (sims_step_i16_half)
            auto fetch32 = [&](int64_t b, uint32_t& id, uint32_t& qq) {
                if (b < top) {
                    const int64_t e = b + lane < (int64_t)top ? b + lane : (int64_t)top - 1;
                    id = pool_id[e];
                    qq = pool_q[e];
                }
            };
            int64_t b = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32;
            uint32_t nid = 0, nq_ = 0;
            fetch32(b, nid, nq_);
            for (; b < top; b += nw * 32) {
                const uint32_t myid = nid, myq = nq_;
                fetch32(b + nw * 32, nid, nq_);
                const bool oneq = __shfl_sync(kFull, myq, 0) == __shfl_sync(kFull, myq, 31);
                const int t = oneq ? sims_step_i16_half<true>(p, myid, myq, lane) : sims_step_i16_half<false>(p, myid, myq, lane);
                // lane l holds row (l >> 4) * 16 + (l & 15) = l
                if (b + lane < (int64_t)top) pool_key[b + lane] = make_key(sim_of_i16(t), myid);
            }
            return;
        }
    }
    int64_t b = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * NR;
    uint32_t nid = 0, nq_ = 0;
    fetch(b, nid, nq_);
    for (; b < top; b += nw * NR) {
        const int64_t e1 = (int64_t)top < b + NR ? (int64_t)top : b + NR;
        const uint32_t myid = nid, myq = nq_;
        fetch(b + nw * NR, nid, nq_);
        const bool oneq = __shfl_sync(kFull, myq, 0) == __shfl_sync(kFull, myq, NR - 1);
        const float t1 = oneq ? sims_step<NR, I16, true>(p, myid, myq, lane) : sims_step<NR, I16, false>(p, myid, myq, lane);
        const int rr = lane >> kSh;
        const uint32_t id_rr = __shfl_sync(kFull, myid, rr);
        if ((lane & ((1 << kSh) - 1)) == 0 && b + rr < e1) pool_key[b + rr] = make_key(t1, id_rr);
    }
}

// Wide tiles (a separate kernel, launched only when wide queries are possible, so that k_sims keeps
// its register budget for the pool):
template <typename PP, bool I16>
__global__ void __launch_bounds__(256, PFG_SIMS_MINB) k_wsims(PP pp, int par) {
    pdl_wait();
    const QueryParams& p = deref(pp);
    constexpr int NR = I16 ? PFG_I16_NR : kRPI;
    constexpr int kSh = NR == 32 ? 0 : NR == 16 ? 1 : NR == 8 ? 2 : 3;
    const int lane = threadIdx.x & 31;
    const RoundState& rs = p.rs;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // wide tiles: a provisional id is fresh iff the query's visit-tag array still holds this
    // visit's tag (no earlier repetition of the chunk passed it); the fresh ids are compacted in
    // order and their similarities computed (the same arithmetic); kept = how many of them beat the
    // k-th key the query held at the start of the chunk (only those can enter its top list).
    // A warp takes four consecutive tiles at once (their metadata, tag checks and rows in flight
    // together): a tile holds few fresh ids late in a search, and one tile per warp step left the
    // kernel bound by the chain of dependent loads per tile.
    constexpr int G = 4;
    const uint32_t nwt = min(rs.ctl->nwt[par], rs.wcap);
    auto sel4 = [](uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, int t) -> uint32_t {
        return t == 0 ? a0 : t == 1 ? a1 : t == 2 ? a2 : a3;
    };
    for (int64_t g0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * G; g0 < nwt; g0 += nw * G) {
        uint32_t w = 0, q = 0, tag = 0, slot = 0;
        uint64_t kth = 0;
        if (lane < G && g0 + lane < nwt) {
            w = rs.wtcnt[g0 + lane];
            if (w & 0xffu) {
                q = rs.wtiles[2 * (g0 + lane)].x;
                tag = rs.wtiles[2 * (g0 + lane) + 1].z;
            }
        }
        if (lane < G && (w & 0xffu)) {
            slot = rs.wslot[q];
            kth = rs.tn[q] == p.k_eff ? rs.T[(int64_t)q * p.kt + p.k_eff - 1] : 0ull;
        }
        uint32_t incl = w & 0xffu;
#pragma unroll
        for (int off = 1; off < G; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, incl, off);
            if (lane >= off) incl += o;
        }
        const uint32_t i0 = __shfl_sync(kFull, incl, 0), i1 = __shfl_sync(kFull, incl, 1),
                       i2 = __shfl_sync(kFull, incl, 2), i3 = __shfl_sync(kFull, incl, 3);
        if (i3 == 0) continue;
        const uint32_t q0 = __shfl_sync(kFull, q, 0), q1 = __shfl_sync(kFull, q, 1), q2 = __shfl_sync(kFull, q, 2),
                       q3 = __shfl_sync(kFull, q, 3);
        const uint32_t tg0 = __shfl_sync(kFull, tag, 0), tg1 = __shfl_sync(kFull, tag, 1),
                       tg2 = __shfl_sync(kFull, tag, 2), tg3 = __shfl_sync(kFull, tag, 3);
        const uint32_t s0 = __shfl_sync(kFull, slot, 0), s1 = __shfl_sync(kFull, slot, 1),
                       s2 = __shfl_sync(kFull, slot, 2), s3 = __shfl_sync(kFull, slot, 3);
        // tag checks over the tiles' provisional entries, compaction per tile in order (an entry
        // is written at or before its own index, after every entry before it was read)
        uint32_t fc0 = 0, fc1 = 0, fc2 = 0, fc3 = 0;
        for (uint32_t e0 = 0; e0 < i3; e0 += 32) {
            const uint32_t e = e0 + lane;
            const bool live = e < i3;
            const int t = (int)(e >= i0) + (int)(e >= i1) + (int)(e >= i2);
            uint32_t id = 0;
            bool fresh = false;
            if (live) {
                const uint32_t o = e - sel4(0u, i0, i1, i2, t);
                id = rs.wcand[(g0 + t) * kTile + o];
                fresh = __ldcg(rs.wv + (int64_t)sel4(s0, s1, s2, s3, t) * p.n + id) == sel4(tg0, tg1, tg2, tg3, t);
            }
            const uint32_t fm = __ballot_sync(kFull, fresh);
            __syncwarp();
#pragma unroll
            for (int tt = 0; tt < G; ++tt) {
                const uint32_t m = fm & __ballot_sync(kFull, live && t == tt);
                const uint32_t fct = sel4(fc0, fc1, fc2, fc3, tt);
                if (fresh && t == tt) rs.wcand[(g0 + tt) * kTile + fct + __popc(m & lanemask_lt())] = id;
                const uint32_t add = __popc(m);
                if (tt == 0) fc0 += add; else if (tt == 1) fc1 += add; else if (tt == 2) fc2 += add; else fc3 += add;
            }
        }
        __syncwarp();
        // similarities of the fresh rows of the four tiles, NR rows per step (rows of different
        // queries read their own query row)
        const uint32_t f0 = fc0, f1 = f0 + fc1, f2 = f1 + fc2, f3 = f2 + fc3;
        const uint64_t k0 = __shfl_sync(kFull, kth, 0), k1 = __shfl_sync(kFull, kth, 1), k2 = __shfl_sync(kFull, kth, 2),
                       k3 = __shfl_sync(kFull, kth, 3);
        uint32_t kp0 = 0, kp1 = 0, kp2 = 0, kp3 = 0;
        for (uint32_t b0 = 0; b0 < f3; b0 += NR) {
            const uint32_t nrow = min((uint32_t)NR, f3 - b0);
            uint32_t myid = 0, myq = 0, mys = 0;
            int myt = 0;
            if (lane < NR) {
                const uint32_t e = b0 + min((uint32_t)lane, nrow - 1);
                myt = (int)(e >= f0) + (int)(e >= f1) + (int)(e >= f2);
                mys = (g0 + myt) * kTile + (e - sel4(0u, f0, f1, f2, myt));
                myid = rs.wcand[mys];
                myq = sel4(q0, q1, q2, q3, myt);
            }
            const bool oneq = __shfl_sync(kFull, myq, 0) == __shfl_sync(kFull, myq, NR - 1);
            const float sim = oneq ? sims_step<NR, I16, true>(p, myid, myq, lane) : sims_step<NR, I16, false>(p, myid, myq, lane);
            const uint32_t rr = lane >> kSh;
            const uint32_t id_rr = __shfl_sync(kFull, myid, rr);
            const uint32_t s_rr = __shfl_sync(kFull, mys, rr);
            const int t_rr = __shfl_sync(kFull, myt, rr);
            const bool own = (lane & ((1 << kSh) - 1)) == 0 && rr < nrow;
            if (own) rs.wsim[s_rr] = sim;
            const uint64_t kt_rr = t_rr == 0 ? k0 : t_rr == 1 ? k1 : t_rr == 2 ? k2 : k3;
            const bool kp = own && make_key(sim, id_rr) > kt_rr;
            kp0 += __popc(__ballot_sync(kFull, kp && t_rr == 0));
            kp1 += __popc(__ballot_sync(kFull, kp && t_rr == 1));
            kp2 += __popc(__ballot_sync(kFull, kp && t_rr == 2));
            kp3 += __popc(__ballot_sync(kFull, kp && t_rr == 3));
        }
        if (lane < G && (w & 0xffu))
            rs.wtcnt[g0 + lane] = sel4(fc0, fc1, fc2, fc3, lane) | (w & 0xffff00u) | (sel4(kp0, kp1, kp2, kp3, lane) << 24);
    }
}

// ---------------------------------------------------------------------------------------------
struct MergeSmem {
    uint64_t cand[32];
};

__device__ __forceinline__ void push_fused(const RoundState& rs, uint32_t q) {
    if (rs.ctl->loop) push(rs.fused2, &rs.ctl->nfused2, q);
    else push(rs.fused, &rs.ctl->nfused, q);
}

#ifndef PFG_MERGE_MINB
#define PFG_MERGE_MINB 10
#endif
#ifndef PFG_MERGE_SORTMIN
#define PFG_MERGE_SORTMIN 8
#endif
constexpr int kMergeSortMin = PFG_MERGE_SORTMIN;  // keys above the k-th from which k_merge sorts a batch
template <typename PP, bool WIDE>
__global__ void __launch_bounds__(128, WIDE ? 8 : PFG_MERGE_MINB) k_merge(PP pp, int par) {
    pdl_wait();
    const QueryParams& p = deref(pp);
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
        const int fl = rs.flags[q];
        const bool wide = WIDE && (fl & kFlagWide);  // WIDE = false: no wide queries in this search
        if (fl & kFlagFused) {
            if (lane == 0) push_fused(rs, (uint32_t)q);
            continue;
        }
        if (fl & (kFlagDefer | kFlagRedo)) {
            // the chunk runs again next round (no room for its wide tiles, or the query widened)
            if (lane == 0) {
                rs.flags[q] = fl & ~(kFlagDefer | kFlagRedo);
                push(rs.act[par ^ 1], &rs.ctl->nact[par ^ 1], (uint32_t)q);
                if (wide) atomicAdd(&rs.ctl->nwide[par ^ 1], 1u);
            }
            continue;
        }
        const int i = rs.lvl[q], c0 = rs.c0[q];
        int tn = rs.tn[q];
        const int nr = (int)rs.rinfo[q].x;  // the chunk k_expand chose (chunk_reps)
        for (int t = lane; t < tn; t += 32) T0[t] = rs.T[q * p.kt + t];
        uint64_t* T = T0;
        uint64_t* Tn = T1;
        // merge one batch of keys (one per lane, 0 = none) into the sorted top list T (rank merge
        // of the sorted batch, as the fused kernel's merge_range); keys at or below the k-th key
        // are dropped
        auto merge_batch = [&](uint64_t key) {
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
        };
        uint32_t* cn = rs.cnt + q * kCnt;
        uint32_t nE = cn[3];
        const uint32_t base = rs.poff[q];
        // per repetition: emitted (k_expand), filtered, dups (k_dedupe; wide: counted below)
        uint32_t rc0 = 0, rc1 = 0, rc2 = 0, rt = 0;
        if (lane < nr) {
            const uint32_t* rc = rs.repcnt + (q * kMaxR + lane) * 3;
            rc0 = rc[0]; rc1 = rc[1]; rc2 = rc[2];
        }
        if (wide && lane < nr) rt = rs.rtile[q * (kMaxR + 1) + lane];
        const uint32_t rend = wide ? rs.rtile[q * (kMaxR + 1) + nr] : 0u;
        // survivors of repetition r are pool entries [end_{r-1}, end_r): per repetition
        // emitted - filtered - duplicates, in repetition order
        uint32_t end = rc0 - rc1 - rc2;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t o = __shfl_up_sync(kFull, end, off);
            if (lane >= off) end += o;
        }
        // stop thresholds of the chunk's repetitions, lane r holds repetition c0 + r's
        const float thr_r = (lane < nr && i > 0) ? __ldg(p.thr + (int64_t)(i - 1) * p.L + c0 + lane) : INFINITY;
        __syncwarp();
        int r_stop = -1;
        uint32_t e = 0;
        // k_eff <= 32, not wide: the top list lives in registers (lane t holds T[t]) and each key above
        // the k-th is inserted where it ranks (a ballot); the chunk's keys are read two batches ahead
        // across repetition boundaries; the stop check follows each repetition as below
        const bool regs = !wide && p.kt == 32;
        if (regs) {
            uint64_t tv = lane < tn ? T0[lane] : 0ull;
            const uint32_t pn = __shfl_sync(kFull, end, nr - 1);
            const uint64_t* keys = rs.pool_key + base;
            uint64_t cur = lane < pn ? keys[lane] : 0ull;
            uint64_t nxt = 32 + lane < pn ? keys[32 + lane] : 0ull;
            int r = 0;
            uint32_t rend = __shfl_sync(kFull, end, 0), done = 0;
            bool fin = false;
            for (uint32_t b0 = 0; !fin; b0 += 32) {
                for (;;) {
                    const uint32_t lim = min(b0 + 32, rend);
                    const uint32_t idx = b0 + lane;
                    const bool mine = idx >= done && idx < lim;
                    if (mine && p.trace_cap > 0 && nE + idx < (uint32_t)p.trace_cap)
                        p.trace_ids[q * p.trace_cap + nE + idx] = key_id(cur);
                    uint64_t kth = (tn == p.k_eff) ? __shfl_sync(kFull, tv, p.k_eff - 1) : 0ull;
                    uint32_t mk = __ballot_sync(kFull, mine && cur > kth);
                    if (__popc(mk) >= kMergeSortMin) {
                        // many keys above the k-th (early in a search): sort them and merge the two
                        // sorted lists at once (bitonic: max of the batch and the reversed list holds
                        // the top 32 of the union, then a half-cleaner sort); the top k of a set of
                        // distinct keys does not depend on the insertion order
                        uint64_t kv = ((mk >> lane) & 1u) ? cur : 0ull;
                        kv = warp_sort_desc(kv, lane);
                        uint64_t mv = __shfl_sync(kFull, tv, 31 - lane);
                        mv = kv > mv ? kv : mv;
#pragma unroll
                        for (int h = 16; h >= 1; h >>= 1) {
                            const uint64_t o = __shfl_xor_sync(kFull, mv, h);
                            mv = (lane & h) ? (mv < o ? mv : o) : (mv > o ? mv : o);
                        }
                        tv = lane < p.k_eff ? mv : 0ull;
                        tn = min(p.k_eff, tn + __popc(mk));
                        mk = 0;
                    }
                    while (mk) {
                        const int l = __ffs(mk) - 1;
                        mk &= mk - 1;
                        const uint64_t kk = __shfl_sync(kFull, cur, l);
                        if (kk <= kth) continue;   // the k-th grew since the ballot
                        const int pos = __popc(__ballot_sync(kFull, tv > kk));
                        const uint64_t up = __shfl_up_sync(kFull, tv, 1);
                        if (lane > pos) tv = up;
                        else if (lane == pos) tv = kk;
                        if (lane >= p.k_eff) tv = 0ull;
                        tn = min(p.k_eff, tn + 1);
                        kth = (tn == p.k_eff) ? __shfl_sync(kFull, tv, p.k_eff - 1) : 0ull;
                    }
                    done = lim;
                    if (rend > b0 + 32) break;   // repetition r continues in the next batch
                    const int j1 = c0 + r + 1;
                    const float th = __shfl_sync(kFull, thr_r, r);
                    if (i == 0) { r_stop = r; fin = true; break; }
                    if (tn == p.k_eff && (!p.per_round || j1 == p.L)) {
                        float ip = key_sim(__shfl_sync(kFull, tv, p.k_eff - 1));
                        ip = fminf(fmaxf(ip, -1.0f), 1.0f);
                        if (ip >= th) { r_stop = r; fin = true; break; }
                    }
                    if (++r >= nr) { fin = true; break; }
                    rend = __shfl_sync(kFull, end, r);
                }
                if (fin) break;
                cur = nxt;
                nxt = b0 + 64 + lane < pn ? keys[b0 + 64 + lane] : 0ull;
            }
            nE += __shfl_sync(kFull, end, r_stop >= 0 ? r_stop : nr - 1);
            if (lane < p.k_eff) T0[lane] = tv;
            __syncwarp();
        }
        for (int r = 0; r < nr && !regs; ++r) {
            const uint32_t rnext = __shfl_sync(kFull, rt, (r + 1) & 31);
            if (!wide) {
                const uint32_t e2 = __shfl_sync(kFull, end, r);
                uint64_t nxt = (e + lane < e2) ? rs.pool_key[base + e + lane] : 0ull;
                for (uint32_t b0 = e; b0 < e2; b0 += 32) {
                    const uint32_t idx = b0 + lane;
                    const uint64_t key = nxt;
                    nxt = (idx + 32 < e2) ? rs.pool_key[base + idx + 32] : 0ull;  // prefetch the next batch
                    if (idx < e2 && p.trace_cap > 0) {
                        const uint32_t pos = nE + (idx - e);
                        if (pos < (uint32_t)p.trace_cap) p.trace_ids[q * p.trace_cap + pos] = key_id(key);
                    }
                    merge_batch(key);
                }
                nE += e2 - e;
                e = e2;
            } else {
                // the repetition's wide tiles in order: fresh ids (in position order) with their
                // similarities; a tile with nothing above the chunk-start k-th key is skipped unless
                // the evaluated ids are traced
                const uint32_t tb = __shfl_sync(kFull, rt, r);
                const uint32_t te = r + 1 < nr ? rnext : rend;
                uint32_t fr = 0, pa = 0;
                for (uint32_t t0 = tb; t0 < te; t0 += 32) {
                    const uint32_t w = t0 + lane < te ? rs.wtcnt[t0 + lane] : 0u;
                    const uint32_t nf = w & 0xffu;
                    uint32_t incl = nf;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t o = __shfl_up_sync(kFull, incl, off);
                        if (lane >= off) incl += o;
                    }
                    uint32_t need = __ballot_sync(kFull, nf > 0 && (p.trace_cap > 0 || (w >> 24) > 0));
                    while (need) {
                        const int l = __ffs(need) - 1;
                        need &= need - 1;
                        const uint32_t cntf = __shfl_sync(kFull, nf, l);
                        const uint32_t pos0 = nE + fr + __shfl_sync(kFull, incl - nf, l);
                        const int64_t s0 = (int64_t)(t0 + l) * kTile;
                        for (uint32_t o = 0; o < cntf; o += 32) {
                            const uint32_t idx = o + lane;
                            uint64_t key = 0;
                            if (idx < cntf) {
                                const uint32_t id = rs.wcand[s0 + idx];
                                key = make_key(rs.wsim[s0 + idx], id);
                                if (p.trace_cap > 0 && pos0 + idx < (uint32_t)p.trace_cap) p.trace_ids[q * p.trace_cap + pos0 + idx] = id;
                            }
                            merge_batch(key);
                        }
                    }
                    fr += __shfl_sync(kFull, incl, 31);
                    uint32_t np_ = (w >> 8) & 0xffu;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) np_ += __shfl_xor_sync(kFull, np_, off);
                    pa += np_;
                }
                nE += fr;
                if (lane == r) { rc1 = rc0 - pa; rc2 = pa - fr; }
            }
            const int j1 = c0 + r + 1;
            if (i == 0) { r_stop = r; break; }  // the linear scan ends the search (R-13)
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
                    pfg_query_stats s;
                    s.i_stop = i; s.j_stop = c0 + r_stop + 1; s.emitted = emitted; s.filtered = filtered; s.dups = dups;
                    s.evaluated = nE;
                    s.flags = (p.k > p.k_eff ? 1u : 0u) | ((p.trace_cap > 0 && nE > (uint32_t)p.trace_cap) ? 4u : 0u) |
                              (wide ? 16u : 0u);
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
            int ni = i, nc0 = c0 + nr;
            if (nc0 >= p.L) { ni = i - 1; nc0 = 0; }
            if (lane == 0) {
                cn[0] = emitted; cn[1] = filtered; cn[2] = dups; cn[3] = nE;
                rs.tn[q] = tn;
                rs.lvl[q] = ni;
                rs.c0[q] = nc0;
            }
            __syncwarp();
            // the i = 0 scan runs wide (a query not yet wide widens for it, with the evaluated
            // list just committed; else the fused kernel takes it)
            const bool to_wide = WIDE && ni == 0 && !wide && try_widen(p, q, lane);
            if (lane == 0) {
                if (ni == 0 && !wide && !to_wide) { rs.flags[q] |= kFlagFused; push_fused(rs, (uint32_t)q); }
                else {
                    push(rs.act[par ^ 1], &rs.ctl->nact[par ^ 1], (uint32_t)q);
                    if (wide || to_wide) atomicAdd(&rs.ctl->nwide[par ^ 1], 1u);
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------------
// After the blind rounds: the device-side round loop (a CUDA graph WHILE node, pfg.cu) and the
// fused kernel split the queries still running.  The loop keeps them all when there are enough to
// fill the bulk phases but too few to hide the fused kernel's per-warp latency
// (lmin <= count <= lmax); otherwise it keeps only the wide queries (the fused kernel cannot resume
// those) and the fused kernel, launched beside the loop, takes the rest.
// k_split fills list par ^ 1, which the loop's first round consumes: reset its counters as the
// k_expand of a round of parity par would
__global__ void k_presplit(QueryParams p, int par) {
    RoundCtl* c = p.rs.ctl;
    const int o = par ^ 1;
    c->nact[o] = 0; c->pool_top[o] = 0; c->ntiles[o] = 0;
    for (int t = 0; t < 4; ++t) c->wk[o][t] = 0;
    c->dfront[o] = 0; c->dback[o] = 0;
    c->nwt[o] = 0; c->nwide[o] = 0;
}
__global__ void k_split(QueryParams p, int par, uint32_t lmin, uint32_t lmax) {
    const RoundState& rs = p.rs;
    const uint32_t n = rs.ctl->nact[par];
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const uint32_t q = rs.act[par][a];
    const bool wide = rs.flags[q] & kFlagWide;
    if ((n >= lmin && n <= lmax) || wide) {
        push(rs.act[par ^ 1], &rs.ctl->nact[par ^ 1], q);
        if (wide) atomicAdd(&rs.ctl->nwide[par ^ 1], 1u);
    } else {
        push(rs.fused, &rs.ctl->nfused, q);
    }
}
// two round pipelines (pfg.cu pipeline_params): pipeline 1's control-block counters added to
// pipeline 0's, which the host reads back as the search's
__global__ void k_ctl_fold(RoundCtl* c) {
    RoundCtl& a = c[0];
    const RoundCtl& b = c[1];
    a.nfused += b.nfused; a.nfused2 += b.nfused2; a.wnext += b.wnext; a.wdefer += b.wdefer;
    a.round = max(a.round, b.round);
    a.evsum += b.evsum; a.emsum += b.emsum; a.sims_rows += b.sims_rows; a.sims_rows_blind += b.sims_rows_blind;
}
// loop condition: queries left, and either a wide one among them or at least lmin
__device__ __forceinline__ bool loop_more(const RoundCtl* c, int par, uint32_t lmin) {
    const uint32_t n = c->nact[par];
    return n > 0 && (c->nwide[par] > 0 || n >= lmin);
}
__global__ void k_loop_begin(RoundCtl* c, int par, cudaGraphConditionalHandle h, uint32_t lmin) {
    c->loop = 1;
    c->round = 0;
    cudaGraphSetConditional(h, loop_more(c, par, lmin) ? 1u : 0u);
}
__global__ void k_loop_cond(RoundCtl* c, int par, cudaGraphConditionalHandle h, uint32_t lmin, uint32_t cap) {
    c->round += 2;
    cudaGraphSetConditional(h, (loop_more(c, par, lmin) && c->round < cap) ? 1u : 0u);
}
// the loop ended: the queries still running go to the second fused launch; a wide query left
// here (only if the loop hit its round cap) ends with no result (stats flag bit 5)
__global__ void k_loop_end(QueryParams p, int par) {
    const RoundState& rs = p.rs;
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= rs.ctl->nact[par]) return;
    const uint32_t q = rs.act[par][a];
    if (!(rs.flags[q] & kFlagWide)) { push(rs.fused2, &rs.ctl->nfused2, q); return; }
    for (int t = 0; t < p.k; ++t) { p.out_ids[(int64_t)q * p.k + t] = -1; p.out_sims[(int64_t)q * p.k + t] = __int_as_float(0x7fc00000); }
    if (p.stats) { pfg_query_stats s = {}; s.flags = 32u | 16u; p.stats[q] = s; }
}

}  // namespace pfg
