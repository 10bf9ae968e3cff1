// pfg.cu — C-ABI implementation (include/pfg.h) of the B200-native batched LSH-forest k-NN index.
//
// Host side: argument checks, the budget -> L cost model (R-11), seeded hash-function
// generation (rng.h), orchestration of the build kernels and CUB radix sorts, the host-computed
// stop-rule / filter threshold tables (so the device does no transcendental math and its stop
// decisions equal the oracle's, R-9/R-10/R-15), and the launch of the query kernel.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>
#include <type_traits>

#include "../../include/pfg.h"
#include "kernels_build.cuh"
#include "kernels_query.cuh"
#include "kernels_rounds.cuh"
#include "kernels_chunk.cuh"
#include "kernels_tc.cuh"
#include "rng.h"

namespace pfg {
namespace {

thread_local std::string g_err;

pfg_status fail(pfg_status s, const std::string& m) {
    g_err = m;
    return s;
}

#define PFG_CUDA(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess) {                                                                    \
            cudaGetLastError();                                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? PFG_E_OOM : PFG_E_CUDA,                   \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                        \
        }                                                                                           \
    } while (0)

#define PFG_TRY(expr)                            \
    do {                                         \
        pfg_status s_ = (expr);                  \
        if (s_ != PFG_OK) return s_;             \
    } while (0)

// owning device buffer
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    pfg_status alloc(size_t b, const char* what) {
        release();
        if (b == 0) b = 16;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            return fail(e == cudaErrorMemoryAllocation ? PFG_E_OOM : PFG_E_CUDA,
                        std::string("cudaMalloc(") + what + ", " + std::to_string(b) + " B): " + cudaGetErrorString(e));
        }
        bytes = b;
        return PFG_OK;
    }
    pfg_status ensure(size_t b, const char* what) {  // grow-only
        if (p && bytes >= b) return PFG_OK;
        return alloc(b, what);
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) and occupancy queries cost host time on every
// search; they are cached per kernel (the attribute only grows)
std::mutex g_attr_mu;
cudaError_t set_smem(const void* fn, size_t bytes) {
    static std::map<const void*, size_t> done;
    std::lock_guard<std::mutex> lock(g_attr_mu);
    auto it = done.find(fn);
    if (it != done.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done[fn] = bytes;
    return e;
}
cudaError_t occupancy(int* nb, const void* fn, int threads, size_t smem) {
    static std::map<std::tuple<const void*, int, size_t>, int> cache;
    std::lock_guard<std::mutex> lock(g_attr_mu);
    const auto key = std::make_tuple(fn, threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) { *nb = it->second; return cudaSuccess; }
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(nb, fn, threads, smem);
    if (e == cudaSuccess) cache[key] = *nb;
    return e;
}

bool is_device_ptr(const void* ptr) {
    if (!ptr) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}
int ilog2(int v) {
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

// ---------------------------------------------------------------------------------------------
// index geometry and the budget -> L cost model (R-11)
struct Geo {
    int64_t n = 0;
    int d = 0, dpad = 0, family = 0, strategy = 0, K = 24, M = 32, ell = 1, c = 24, dp = 1, W = 1, m = 0;
    int pool_bits = 3072, cp_draws = 1000, max_reps = 4096, L = 0, S = 0;  // S = sqrt(L) (tensor)
    int64_t id_offset = 0;
    uint64_t fixed_bytes = 0, per_rep_bytes = 0, index_bytes = 0;
    int storage = 0, dpad16 = 0;  // PFG_STORAGE_I16: int16 rows of dpad16 = 16 ceil(d/16) coordinates
};

pfg_status resolve_opts(const pfg_build_opts* o, int64_t n, int d, int family, Geo& g) {
    pfg_build_opts z;
    std::memset(&z, 0, sizeof(z));
    if (o) {
        if (o->struct_size < sizeof(uint32_t) || o->struct_size > sizeof(pfg_build_opts))
            return fail(PFG_E_ARG, "pfg_build_opts.struct_size must be sizeof(pfg_build_opts)");
        std::memcpy(&z, o, o->struct_size);
    }
    if (n < 1 || n >= (int64_t(1) << 31)) return fail(PFG_E_ARG, "n must be in [1, 2^31)");
    if (d < 1 || d > 4096) return fail(PFG_E_ARG, "d must be in [1, 4096]");
    if (family != PFG_SIMHASH && family != PFG_CROSSPOLYTOPE_FHT && family != PFG_CROSSPOLYTOPE)
        return fail(PFG_E_ARG, "unknown family");
    if (family == PFG_CROSSPOLYTOPE && d > 256) return fail(PFG_E_ARG, "exact cross-polytope family supports d <= 256");
    g.n = n;
    g.d = d;
    g.dpad = (d + 7) / 8 * 8;  // rows 32-byte aligned (512-byte rows measured no faster: k_sims is bound by rows in flight)
    if ((uint64_t)n * (uint64_t)g.dpad / 4 >= (1ull << 32))
        return fail(PFG_E_ARG, "n * d too large for one index (shard the data: n * d / 4 must be < 2^32)");
    g.family = family;
    g.strategy = z.strategy;
    if (g.strategy != PFG_INDEPENDENT && g.strategy != PFG_POOL && g.strategy != PFG_TENSOR)
        return fail(PFG_E_ARG, "unknown strategy");
    g.K = z.prefix_bits ? z.prefix_bits : 24;
    if (g.K < 13 || g.K > 32) return fail(PFG_E_ARG, "prefix_bits must be in [13, 32]");
    g.M = z.sketch_words == 0 ? 32 : (z.sketch_words < 0 ? 0 : z.sketch_words);
    if (g.M > 64) return fail(PFG_E_ARG, "sketch_words must be <= 64");
    g.dp = next_pow2(d);
    g.W = (g.dp + 31) >> 5;
    if (family == PFG_SIMHASH) {
        g.ell = 1;
    } else {
        if (g.dp > 1024) return fail(PFG_E_ARG, "cross-polytope (FHT) family supports d <= 1024");
        g.ell = 1 + ilog2(g.dp);
    }
    g.c = (g.K + g.ell - 1) / g.ell;
    if (family == PFG_CROSSPOLYTOPE && g.strategy == PFG_TENSOR)
        return fail(PFG_E_ARG, "exact cross-polytope family: independent or pool strategy");
    if (g.strategy == PFG_TENSOR && (g.c % 2 != 0 || g.c * g.ell != g.K))
        return fail(PFG_E_ARG, "tensor strategy: prefix_bits must be an even number of whole functions (PAPER.md:245)");
    g.pool_bits = z.pool_bits ? z.pool_bits : 3072;
    g.m = g.strategy == PFG_POOL ? g.pool_bits / g.ell : 0;
    if (g.strategy == PFG_POOL && g.m < g.c) return fail(PFG_E_ARG, "pool smaller than one repetition's functions");
    if (g.strategy == PFG_POOL && g.family != PFG_SIMHASH && g.m > 65535) return fail(PFG_E_ARG, "pool too large");
    g.cp_draws = z.cp_draws ? z.cp_draws : 1000;
    if (g.cp_draws < 1) return fail(PFG_E_ARG, "cp_draws must be >= 1");
    g.max_reps = z.max_reps ? z.max_reps : 4096;
    g.id_offset = z.id_offset;
    g.storage = z.storage;
    if (g.storage != PFG_STORAGE_F32 && g.storage != PFG_STORAGE_I16) return fail(PFG_E_ARG, "unknown storage");
    g.dpad16 = (d + 15) / 16 * 16;
    // bytes: data + sketches + sketch functions + pool functions + CP table (fixed);
    // per repetition: sorted table + 13-bit prefix table + slot + its own functions / selection
    const uint64_t N = (uint64_t)n;
    const uint64_t fn_hp = 4ull * g.dpad, fn_fht = family == PFG_CROSSPOLYTOPE ? 4ull * g.d * g.dpad : 3ull * g.W * 4;
    // PFG_STORAGE_I16 keeps the fp32 rows too (hashing at build, the fp32 re-rank of each query's top-k)
    const uint64_t data_bytes = g.storage == PFG_STORAGE_I16 ? 2ull * N * g.dpad16 + 4ull * N * g.dpad : 4ull * N * g.dpad;
    g.fixed_bytes = data_bytes + 4ull * 64 * g.M * g.dpad + 8ull * (g.ell + 1) * 41;
    if (g.strategy == PFG_POOL) g.fixed_bytes += (uint64_t)g.m * (family == PFG_SIMHASH ? fn_hp : fn_fht);
    g.per_rep_bytes = 16ull * N + 4ull * 8193 + 1;  // 16-byte entries: key + inline sketch word (R-21)
    if (g.strategy == PFG_INDEPENDENT) g.per_rep_bytes += (uint64_t)g.c * (family == PFG_SIMHASH ? fn_hp : fn_fht);
    else g.per_rep_bytes += 4ull * g.c;
    // tensor: the S * c functions (S = sqrt(L)) are charged per repetition as c functions, an upper
    // bound for S <= L
    if (g.strategy == PFG_TENSOR) g.per_rep_bytes += (uint64_t)g.c * (family == PFG_SIMHASH ? fn_hp : fn_fht);
    return PFG_OK;
}

pfg_status derive_L(Geo& g, uint64_t budget, int reps_override) {
    if (reps_override > 0) {
        g.L = reps_override;
    } else {
        if (budget < g.fixed_bytes + g.per_rep_bytes) {
            return fail(PFG_E_BUDGET, "memory budget " + std::to_string(budget) + " B admits no repetition; minimum is " +
                                          std::to_string(g.fixed_bytes + g.per_rep_bytes) + " B");
        }
        const uint64_t L = (budget - g.fixed_bytes) / g.per_rep_bytes;
        g.L = (int)std::min<uint64_t>(L, (uint64_t)g.max_reps);
    }
    if (g.L < 1 || g.L > 65536) return fail(PFG_E_ARG, "repetitions must be in [1, 65536]");
    if (g.strategy == PFG_TENSOR) {
        // L an even power of two: the largest one the budget admits, at most 4096
        // (shells of 2S - 1 <= 32 tries per chunk need S <= 16 -> L <= 256)
        int S = 1;
        while ((S * 2) * (S * 2) <= g.L && S * 2 <= 16) S *= 2;
        if (reps_override > 0 && S * S != reps_override)
            return fail(PFG_E_ARG, "tensor strategy: reps must be an even power of two, at most 256");
        g.S = S;
        g.L = S * S;
        g.m = S * g.c;   // functions: 2 collections x S tuples x c/2
    }
    g.index_bytes = g.fixed_bytes + (uint64_t)g.L * g.per_rep_bytes;
    return PFG_OK;
}

// ---------------------------------------------------------------------------------------------
// stop rule (host, double, same formulas as the paper; R-9, R-10)
int grid_bucket(float ip) {
    int b = 0;
    for (int a = 0; a <= 40; ++a)
        if (ip >= (float)(-1.0 + 0.05 * a)) b = a;
    return b;
}

struct StopModel {
    int family, strategy, ell, m;
    const double* T;  // CP table [(ell+1)][41] (FHT family)
    int K, L;
    double P(int i, float ip) const {
        if (family == PFG_SIMHASH) {
            const double p = 1.0 - std::acos((double)ip) / M_PI;
            return std::pow(p, (double)i);
        }
        const int b = grid_bucket(ip);
        return std::pow(T[ell * 41 + b], (double)(i / ell)) * T[(i % ell) * 41 + b];
    }
    // Lemma 1 failure bound, Alg. 1 line 8, pool Cantelli
    bool stop(int i, int j, float ip, double delta, int rule) const {
        if (strategy == PFG_TENSOR) {
            // Alg. 2: after j = m shells at depth i, 2 (1 - P_{i/2})^m <= delta
            const double Ph = P(i / 2, ip);
            return std::log(2.0) + (double)j * std::log1p(-Ph) <= std::log(delta);
        }
        const double Pi = P(i, ip);
        if (strategy == PFG_POOL) {
            const int ci = (i + ell - 1) / ell;
            if (m < 2 * ci || !(Pi > 0.0)) return false;
            const double r = (double)ci / (double)(m - ci);
            double prod = 1.0;
            for (int f = 0; f < ci; ++f) {
                const int bits = (f < i / ell) ? ell : (i % ell);
                const double pf = P(bits, ip);
                prod *= r + (1.0 - r) * pf;
            }
            const double mu = (double)j * Pi;
            const double e12 = Pi * prod;
            const double F = 1.0 - mu * mu / (mu + (double)j * ((double)j - 1.0) * e12);
            return F <= delta;
        }
        if (rule == 1) return (double)j * Pi >= std::log(1.0 / delta);
        if (rule == 2 && i < K) {
            // two-level bound: the L - j repetitions not yet searched
            // at depth i were searched at depth i + 1: (1 - P_i)^j (1 - P_{i+1})^(L - j) <= delta
            const double P1 = P(i + 1, ip);
            return (double)j * std::log1p(-Pi) + (double)(L - j) * std::log1p(-P1) <= std::log(delta);
        }
        return (double)j * std::log1p(-Pi) <= std::log(delta);
    }
};

uint32_t h_f2ord(float f) {
    if (f == 0.0f) f = 0.0f;
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
float h_ord2f(uint32_t o) {
    const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
// smallest float x in [-1, 1] with pred(x) true, for pred monotone (false ... true); +inf if none
template <class Pred>
float smallest_true(Pred pred) {
    if (!pred(1.0f)) return INFINITY;
    if (pred(-1.0f)) return -1.0f;
    uint32_t lo = h_f2ord(-1.0f), hi = h_f2ord(1.0f);  // pred(lo) false, pred(hi) true
    while (hi - lo > 1) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (pred(h_ord2f(mid))) hi = mid; else lo = mid;
    }
    return h_ord2f(hi);
}

// R-15: tau = round-half-up((1+eps) * 64 * acos(ip)/pi), clamped to [0, 64]
int tau_of(float ipk, float eps) {
    double t = (1.0 + (double)eps) * 64.0 * std::acos((double)ipk) / M_PI;
    double r = std::floor(t + 0.5);
    if (r > 64.0) r = 64.0;
    if (r < 0.0) r = 0.0;
    return (int)r;
}

// R-26: tau = the smallest t with P[H > t] <= delta for H ~ Binomial(64, acos(ip)/pi),
// the (1 - delta)-quantile of the sketch Hamming distance of a pair at the k-th similarity; the upper
// tail summed in double from t = 64 down (smallest terms first)
double binom64(double p, int t) {
    double c = 1.0;
    for (int h = 0; h < t; ++h) c = c * (double)(64 - h) / (double)(h + 1);
    return c * std::pow(p, (double)t) * std::pow(1.0 - p, (double)(64 - t));
}
int tau_quantile(float ipk, double delta) {
    double p = std::acos((double)ipk) / M_PI;
    if (p < 0.0) p = 0.0;
    if (p > 1.0) p = 1.0;
    double tail = 0.0;
    int t = 64;
    while (t > 0 && tail + binom64(p, t) <= delta) { tail += binom64(p, t); --t; }
    return t;
}

// query codes of repetitions [0, reps) and sketches computed elsewhere (device pointers; SURVEY 8(e):
// each rank of the data-sharded mode hashes a slice of the queries, the slices are all-gathered)
struct ExtHash {
    const uint32_t* codes = nullptr;  // [nq][reps]
    int reps = 0;
    const uint64_t* sk = nullptr;     // [nq][M]
};

struct SearchCfg {
    int R = 8, B = 12, rule = 0, per_round = 0, use_filter = 1, trace_cap = 0, timing = 0, engine = 0, uniform = 0, rounds = 0;
    int wide = 0;
    int tau_rule = 0;   // 0: binomial quantile (R-26), 1: (1 + eps) x expected distance (R-15)
    int rerank = 1;     // PFG_STORAGE_I16: re-score each query's top-k in fp32
    int loop_min = 0, loop_max = 0, wide_arrays = 0, wide_tiles_min = 0;  // device-side loop policy (tests)
    int pipelines = 0;  // engine 0: round pipelines (0 = automatic, 1, 2)
    ExtHash ext;        // precomputed query codes / sketches (SURVEY 8(e) distributed preparation)
    float eps = 0.0f;
    uint32_t* trace_ids = nullptr;
};

pfg_status resolve_sopts(const pfg_search_opts* o, SearchCfg& s) {
    pfg_search_opts z;
    std::memset(&z, 0, sizeof(z));
    if (o) {
        if (o->struct_size < sizeof(uint32_t) || o->struct_size > sizeof(pfg_search_opts))
            return fail(PFG_E_ARG, "pfg_search_opts.struct_size must be sizeof(pfg_search_opts)");
        std::memcpy(&z, o, o->struct_size);
    }
    s.R = z.rep_chunk ? z.rep_chunk : 16;
    if (s.R < 1 || s.R > kMaxR) return fail(PFG_E_ARG, "rep_chunk must be in [1, 32]");
    s.B = z.segment ? z.segment : 12;
    if (s.B < 1) return fail(PFG_E_ARG, "segment must be >= 1");
    s.rule = z.stop_rule;
    if (s.rule < 0 || s.rule > 2) return fail(PFG_E_ARG, "stop_rule must be 0, 1 or 2");
    s.per_round = z.stop_granularity;
    if (s.per_round != 0 && s.per_round != 1) return fail(PFG_E_ARG, "stop_granularity must be 0 or 1");
    s.use_filter = z.use_filter < 0 ? 0 : 1;
    s.eps = z.filter_eps;
    if (!(s.eps > -1.0f) || !std::isfinite(s.eps)) return fail(PFG_E_ARG, "filter_eps must be finite and > -1");
    s.trace_cap = z.trace_cap;
    s.trace_ids = z.trace_ids;
    s.timing = z.timing;
    s.engine = z.engine;
    if (s.engine < 0 || s.engine > 2)
        return fail(PFG_E_ARG, "engine must be 0 (phase-split rounds + fused), 1 (fused) or 2 (chunk rounds + fused)");
    s.rounds = z.rounds;
    if (s.rounds < 0 || s.rounds > 4096) return fail(PFG_E_ARG, "rounds must be in [0, 4096]");
    s.wide = z.wide;
    if (s.wide < -1 || s.wide > kHMax) return fail(PFG_E_ARG, "wide must be -1, 0 or in [1, 1536]");
    s.rerank = z.rerank < 0 ? 0 : 1;
    s.loop_min = z.loop_min;
    s.loop_max = z.loop_max;
    s.wide_arrays = z.wide_arrays;
    s.wide_tiles_min = z.wide_tiles_min;
    s.ext.codes = z.ext_codes;
    s.ext.reps = z.ext_reps;
    s.ext.sk = z.ext_sketches;
    if (s.ext.codes && s.ext.reps < 1) return fail(PFG_E_ARG, "ext_codes needs ext_reps >= 1");
    if (s.loop_min < 0 || s.loop_max < 0 || s.wide_arrays < 0) return fail(PFG_E_ARG, "loop_min, loop_max, wide_arrays must be >= 0");
    s.tau_rule = z.tau_rule;
    if (s.tau_rule != 0 && s.tau_rule != 1) return fail(PFG_E_ARG, "tau_rule must be 0 (quantile) or 1 (expected distance)");
    s.uniform = z.uniform_chunks;
    if (s.uniform != 0 && s.uniform != 1) return fail(PFG_E_ARG, "uniform_chunks must be 0 or 1");
    s.pipelines = z.pipelines;
    if (s.pipelines < 0 || s.pipelines > 2) return fail(PFG_E_ARG, "pipelines must be 0 (automatic), 1 or 2");
    if (s.trace_cap < 0 || (s.trace_cap > 0 && !s.trace_ids)) return fail(PFG_E_ARG, "trace_cap > 0 needs trace_ids");
    return PFG_OK;
}

}  // namespace
}  // namespace pfg

using namespace pfg;

struct pfg_index {
    Geo g;
    int device = 0;
    int num_sms = 148;
    uint64_t seed = 0;
    std::mutex mu;
    // index arrays (device)
    DBuf x, tab, pt, slot, hpfn, sg, sel, skfn, x16;   // x16: int16 rows (PFG_STORAGE_I16, beside the fp32 rows)
    std::vector<double> cpT;
    std::vector<int32_t> slot_h, sel_h;
    // cached stop tables: key (recall bits, rule, per_round) -> device thr [K][L]; eps -> taub
    std::map<std::tuple<uint32_t, int, int>, std::shared_ptr<DBuf>> thr_cache;
    std::map<std::tuple<int, uint32_t, uint32_t>, std::shared_ptr<DBuf>> tau_cache;  // (rule, eps, recall)
    // per-call scratch (grow-only)
    DBuf qraw, qx, qzero, zmin, qsk, qcodes, qbits, qfc, qfc2, outb_ids, outb_sims, outb_stats, outb_trace, work, qx16;
    DBuf cur, bitmap, claims;
    // round-engine state (per query, grow-only)
    DBuf rs_lvl, rs_c0, rs_flags, rs_tn, rs_cnt, rs_T, rs_E, rs_pend, rs_repcnt, rs_pool_id, rs_pool_q, rs_pool_key,
        rs_ctl, rs_poff, rs_pn, rs_act0, rs_act1, rs_fused, rs_cand, rs_tcnt, rs_dord0, rs_dord1, rs_hsave, rs_rseg, rs_rinfo, rs_tiles, qbnd;
    // wide queries: visit-tag arrays, wide scan tiles, the second fused list
    DBuf rs_wv, rs_wslot, rs_wtiles, rs_wcand, rs_wsim, rs_wtcnt, rs_rtile, rs_fused2, rs_params;
    int64_t wv_slots = 0, wv_n = 0, wv_want = 0;   // visit-tag arrays allocated / wanted
    int64_t wc_cap = 0, wc_want = 0;               // wide tiles allocated / wanted
    uint32_t wepoch = 0;         // search epoch of the visit tags (the arrays are reset on wrap)
    // the device-side round loop: an instantiated CUDA graph with a WHILE node, rebuilt when the
    // launch parameters change
    cudaGraphExec_t loop_exec = nullptr;
    std::vector<unsigned char> loop_key;
    cudaStream_t cap_st = nullptr;
    cudaEvent_t ev_split = nullptr, ev_f1 = nullptr;
    uint32_t* h_ctl = nullptr;   // pinned host mirror of the round control block
    RoundCtl* h_ctl2 = nullptr;  // [2] pinned copies of each search's final control block (by parity)
    int64_t nsearch = 0;         // searches of the round engine so far
    int64_t nq_prev[2] = {0, 0}; // their query counts (by parity)
    bool loop_heavy = false;     // the last completed search's queries were heavy: keep them all in the loop
    DBuf jhist;                  // stop-depth histogram of the last search (device)
    uint32_t* h_jhist = nullptr; // its pinned host copy
    int eager = 32;              // repetitions hashed eagerly per query (tuned from the last search)
    int qb_depth = 64;           // level-K match ranges precomputed per query (non-lazy families; tuned)
    cudaStream_t aux = nullptr;  // second stream: query sketches run beside the query hashing
    cudaStream_t aux2 = nullptr; // third stream: codes and ranges of the later eager repetitions
    cudaStream_t st1 = nullptr;  // the second round pipeline (the upper half of the batch)
    cudaStream_t hst = nullptr;  // highest priority: repetition 0's codes and ranges, which round 0 waits for
    cudaEvent_t ev_hst = nullptr, ev_in = nullptr;
    bool hst_pending = false;    // repetition 0's codes were launched on hst (its ranges follow there)
    cudaEvent_t ev_h1start = nullptr, ev_h1end = nullptr;  // fork to / join from st1
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_late = nullptr;
    bool late_pending = false;   // codes/ranges of repetitions [split, eager) still on aux2
    cudaEvent_t ev_mid = nullptr;
    bool mid_pending = false;    // codes/ranges of repetitions [1, split) still on aux2 (round 1 joins)
    int late_ne = 0;             // eager depth whose codes [split, late_ne) the search launches on aux2
    cudaEvent_t ev_zmin = nullptr, ev_done = nullptr;  // zero-row flag copied; previous search done
    bool done_pending = false;   // ev_done recorded by a search not yet observed complete
    int timing_pending = 0;      // the last search recorded timing events (read lazily)
    unsigned long long* h_zmin = nullptr;  // pinned host word: first zero query row
    int64_t rs_nq = 0;
    int rs_kt = 0, rs_L = 0;
    int64_t slots = 0;
    int slots_L = 0;
    int64_t slots_bm = 0;
    // launch accounting and phase timing of the last search
    int launches = 0;
    int qc_n = 0, qc_ld = 0, qc_split = 0;
    int last_rounds = 0;
    int64_t last_fused = 0;
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    float last_ms[3] = {0, 0, 0};
    // per-phase timing (opts->timing): an event before each query-phase kernel; the interval
    // starting at event i belongs to phase pkind[i] (kPh* below)
    std::vector<cudaEvent_t> pev;
    std::vector<int> pkind;
    int pev_n = 0;
    float last_phase_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // timing = 3: event pairs around each bulk k_sims launch, accumulated across searches
    std::vector<cudaEvent_t> kev;
    // timing = 4 (developer timeline): an event after each launch group on its stream, printed to
    // stderr as completion times relative to the search's first event
    std::vector<cudaEvent_t> tlev;
    std::vector<std::string> tlname;
    int tl_n = 0;
    bool tl_on = false;
    int64_t kev_n = 0;          // pairs recorded and not yet summed
    double kev_ms = 0.0;        // summed durations since the last reset
    int64_t kev_launches = 0;
    int last_launches = 0;
    ~pfg_index() {
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        for (auto& e : pev)
            if (e) cudaEventDestroy(e);
        for (auto& e : kev)
            if (e) cudaEventDestroy(e);
        for (auto& e : tlev)
            if (e) cudaEventDestroy(e);
        if (h_ctl) cudaFreeHost(h_ctl);
        if (h_ctl2) cudaFreeHost(h_ctl2);
        if (h_jhist) cudaFreeHost(h_jhist);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (aux) cudaStreamDestroy(aux);
        if (aux2) cudaStreamDestroy(aux2);
        if (st1) cudaStreamDestroy(st1);
        if (hst) cudaStreamDestroy(hst);
        if (ev_hst) cudaEventDestroy(ev_hst);
        if (ev_in) cudaEventDestroy(ev_in);
        for (cudaEvent_t e : {ev_h1start, ev_h1end})
            if (e) cudaEventDestroy(e);
        if (ev_late) cudaEventDestroy(ev_late);
        if (ev_mid) cudaEventDestroy(ev_mid);
        if (ev_zmin) cudaEventDestroy(ev_zmin);
        if (ev_done) cudaEventDestroy(ev_done);
        if (h_zmin) cudaFreeHost(h_zmin);
        if (loop_exec) cudaGraphExecDestroy(loop_exec);
        if (cap_st) cudaStreamDestroy(cap_st);
        for (cudaEvent_t e : {ev_split, ev_f1})
            if (e) cudaEventDestroy(e);
    }
};

namespace pfg {
namespace {

constexpr int kClaimCap = 8192;
void tl_mark(pfg_index* I, const char* name, cudaStream_t st);
constexpr int kQBMax = 96;     // level-K match ranges precomputed for at most this many repetitions
constexpr int kExtReps = 32;   // repetitions hashed in bulk for the queries the fused kernel resumes
pfg_status fht_codes(pfg_index* I, int64_t nrows, const uint32_t* qlist, int r0, int nreps, int ld, cudaStream_t st,
                     const uint32_t* nrows_dev = nullptr, int64_t q0 = 0);
#ifndef PFG_HIPRIO
#define PFG_HIPRIO 1   // searches run on the index's highest-priority stream (pfg_search)
#endif
#ifndef PFG_PDL
#define PFG_PDL 1   // programmatic dependent launch between the blind rounds' kernels
#endif
#ifndef PFG_QTPF
#define PFG_QTPF 1   // threads per function of the eager FHT-CP query hashing at d' = 128
#endif

template <int EPL>
void launch_fht_rep(const float* X, int64_t np, int ldx, const Geo& g, const uint32_t* sg, int r0, int nreps,
                    uint64_t* keys, uint32_t* codes, int ldc, int num_sms, cudaStream_t st) {
    int64_t warps = std::min<int64_t>(np, (int64_t)num_sms * 64);
    const int blocks = (int)((warps * 32 + 255) / 256);
    k_fht_rep<EPL><<<blocks, 256, 0, st>>>(X, np, ldx, g.d, g.dp, g.ell, g.c, g.K, sg, r0, nreps, keys, codes, ldc);
}
template <int DP, int TPF>
void launch_fht_keys(const float* X, int64_t np, int ldx, const Geo& g, const uint32_t* sg, int r0, int nreps,
                     uint64_t* keys, uint32_t* codes, int ldc, cudaStream_t st, int num_sms = 148) {
    constexpr int RB = 128 / TPF;
    const int S = (g.dpad / 4) % 2 ? g.dpad : g.dpad + 4;   // S/4 odd: conflict-free 128-bit reads
    const size_t sm = (size_t)RB * S * 4;
    set_smem((const void*)k_fht_keys<DP, TPF>, sm);
    // repetitions per block: all of them, unless the rows alone give fewer than 4 blocks per SM
    const int64_t rows_b = (np + RB - 1) / RB;
    const int cols = (int)std::min<int64_t>(nreps, std::max<int64_t>(1, (4 * (int64_t)num_sms + rows_b - 1) / rows_b));
    const int rpb = (nreps + cols - 1) / cols;
    const dim3 grid((unsigned)rows_b, (unsigned)((nreps + rpb - 1) / rpb));
    k_fht_keys<DP, TPF><<<grid, 128, sm, st>>>(X, np, ldx, g.dpad, S, g.ell, g.c, g.K, sg, r0, nreps, keys, codes, ldc, rpb);
}
void fht_rep(const float* X, int64_t np, int ldx, const Geo& g, const uint32_t* sg, int r0, int nreps, uint64_t* keys,
             uint32_t* codes, int ldc, int num_sms, cudaStream_t st) {
    // d' = 32 .. 1024: a lane group of max(1, d'/128) lanes (16 at 1024) per (row, repetition), rows staged in
    // shared memory (k_fht_keys); otherwise one warp per row
    switch (g.dp) {
        case 32: return launch_fht_keys<32, 1>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        case 64: return launch_fht_keys<64, 1>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        case 128: return launch_fht_keys<128, 1>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        case 256: return launch_fht_keys<256, 2>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        case 512: return launch_fht_keys<512, 4>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        case 1024: return launch_fht_keys<1024, 16>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, st);
        default: break;
    }
    switch (std::max(1, g.dp / 32)) {
        case 1: launch_fht_rep<1>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
        case 2: launch_fht_rep<2>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
        case 4: launch_fht_rep<4>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
        case 8: launch_fht_rep<8>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
        case 16: launch_fht_rep<16>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
        default: launch_fht_rep<32>(X, np, ldx, g, sg, r0, nreps, keys, codes, ldc, num_sms, st); break;
    }
}
template <int EPL>
void launch_fht_funcs(const float* X, int64_t np, int ldx, const Geo& g, const uint32_t* sg, uint16_t* out, int num_sms,
                      cudaStream_t st) {
    int64_t warps = std::min<int64_t>(np, (int64_t)num_sms * 64);
    const int blocks = (int)((warps * 32 + 255) / 256);
    k_fht_funcs<EPL><<<blocks, 256, 0, st>>>(X, np, ldx, g.d, g.dp, g.ell, g.m, sg, out);
}
void fht_funcs(const float* X, int64_t np, int ldx, const Geo& g, const uint32_t* sg, uint16_t* out, int num_sms,
               cudaStream_t st) {
    switch (std::max(1, g.dp / 32)) {
        case 1: launch_fht_funcs<1>(X, np, ldx, g, sg, out, num_sms, st); break;
        case 2: launch_fht_funcs<2>(X, np, ldx, g, sg, out, num_sms, st); break;
        case 4: launch_fht_funcs<4>(X, np, ldx, g, sg, out, num_sms, st); break;
        case 8: launch_fht_funcs<8>(X, np, ldx, g, sg, out, num_sms, st); break;
        case 16: launch_fht_funcs<16>(X, np, ldx, g, sg, out, num_sms, st); break;
        default: launch_fht_funcs<32>(X, np, ldx, g, sg, out, num_sms, st); break;
    }
}
template <int EPL>
void launch_mc(const float* XY, int ld, int64_t npairs, const Geo& g, const uint32_t* sg, unsigned long long* cnt,
               int num_sms, cudaStream_t st) {
    int64_t warps = std::min<int64_t>(npairs, (int64_t)num_sms * 64);
    const int blocks = (int)((warps * 32 + 255) / 256);
    k_mc_codes<EPL><<<blocks, 256, 0, st>>>(XY, ld, npairs, g.d, g.dp, g.ell, g.cp_draws, sg, cnt);
}

#ifndef PFG_CP_TC
#define PFG_CP_TC 1   // exact cross-polytope codes on tcgen05 (kernels_tc.cuh k_cp_tc); 0: the SIMT k_cp_funcs
#endif
#ifndef PFG_HP_TC
#define PFG_HP_TC 1   // SimHash bits / sketches on tcgen05 (3xTF32 + exact band, kernels_tc.cuh); 0: the SIMT GEMM
#endif
void hp_bits(const float* X, int64_t np, int ldx, const float* A, int nf, int lda, int kdim, uint8_t* out,
             int64_t out_ld, cudaStream_t st, int max_ctas = 0) {
    if (PFG_HP_TC && (kdim % 8) == 0 && (ldx % 4) == 0 && (lda % 4) == 0 && ((uintptr_t)X % 16) == 0 &&
        ((uintptr_t)A % 16) == 0 && set_smem((const void*)k_hp_bits_tc, kTcSmem) == cudaSuccess) {
        // max_ctas > 0: at most that many CTAs, each looping over tiles
        int64_t tiles = ((np + TC_M - 1) / TC_M) * ((nf + TC_N - 1) / TC_N);
        if (max_ctas > 0) tiles = std::min<int64_t>(tiles, max_ctas);
        k_hp_bits_tc<<<(unsigned)tiles, 128, kTcSmem, st>>>(X, np, ldx, A, nf, lda, kdim, out, out_ld);
        return;
    }
    dim3 grid((unsigned)((np + GB_M - 1) / GB_M), (nf + GB_N - 1) / GB_N);
    // the double-buffered kernel needs kdim, ldx, lda multiples of 8 and 16-byte aligned rows
    const bool v2 = (kdim % GB2_K) == 0 && (ldx % 4) == 0 && (lda % 4) == 0 && ((uintptr_t)X % 16) == 0 &&
                    ((uintptr_t)A % 16) == 0;
    if (v2) k_hp_bits2<<<grid, 256, 0, st>>>(X, np, ldx, A, nf, lda, kdim, out, out_ld);
    else k_hp_bits<<<grid, 256, 0, st>>>(X, np, ldx, A, nf, lda, kdim, out, out_ld);
}

// Monte-Carlo CP table (R-13 cleaning, R-14 random pairs)
pfg_status build_cp_table(pfg_index* I, cudaStream_t st) {
    const Geo& g = I->g;
    const int draws = g.cp_draws, d = g.d, dp = g.dp, W = g.W;
    const int64_t npairs = 41ll * draws;
    std::vector<float> XY((size_t)npairs * 2 * dp, 0.0f);
    std::vector<uint32_t> S((size_t)npairs * 3 * W, 0u);
    const uint64_t K = stream_key(I->seed, kTagCPMC);
    auto work = [&](int a0, int a1) {
        std::vector<double> x(d), u(d);
        for (int a = a0; a < a1; ++a) {
            const double alpha = -1.0 + 0.05 * a;
            for (int t = 0; t < draws; ++t) {
                const int64_t e = (int64_t)a * draws + t;
                const uint64_t kat = draw(K, (uint64_t)e);
                const uint64_t ksg = draw(kat, 0), kx = draw(kat, 1), ku = draw(kat, 2);
                double nx = 0.0;
                for (int v = 0; v < d; ++v) { x[v] = gauss(kx, v); nx += x[v] * x[v]; }
                nx = std::sqrt(nx);
                for (int v = 0; v < d; ++v) x[v] = x[v] / nx;
                double ux = 0.0;
                for (int v = 0; v < d; ++v) { u[v] = gauss(ku, v); ux += u[v] * x[v]; }
                double nu = 0.0;
                for (int v = 0; v < d; ++v) { u[v] = u[v] - ux * x[v]; nu += u[v] * u[v]; }
                nu = std::sqrt(nu);
                for (int v = 0; v < d; ++v) u[v] = u[v] / nu;
                const double s = std::sqrt(1.0 - alpha * alpha);
                float* xr = &XY[(size_t)(2 * e) * dp];
                float* yr = &XY[(size_t)(2 * e + 1) * dp];
                for (int v = 0; v < d; ++v) { xr[v] = (float)x[v]; yr[v] = (float)(alpha * x[v] + s * u[v]); }
                uint32_t* se = &S[(size_t)e * 3 * W];
                for (int r = 0; r < 3; ++r)
                    for (int v = 0; v < dp; ++v)
                        if (draw(ksg, (uint64_t)(r * dp + v)) >> 63) se[r * W + (v >> 5)] |= 1u << (v & 31);
            }
        }
    };
    {
        unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        const int per = (41 + (int)nt - 1) / (int)nt;
        for (unsigned k = 0; k < nt; ++k) {
            const int a0 = (int)k * per, a1 = std::min(41, a0 + per);
            if (a0 < a1) th.emplace_back(work, a0, a1);
        }
        for (auto& t : th) t.join();
    }
    DBuf dXY, dS, dC;
    PFG_TRY(dXY.alloc(XY.size() * 4, "cp pairs"));
    PFG_TRY(dS.alloc(S.size() * 4, "cp signs"));
    PFG_TRY(dC.alloc(34 * 41 * 8, "cp counts"));
    PFG_CUDA(cudaMemcpyAsync(dXY.p, XY.data(), XY.size() * 4, cudaMemcpyHostToDevice, st));
    PFG_CUDA(cudaMemcpyAsync(dS.p, S.data(), S.size() * 4, cudaMemcpyHostToDevice, st));
    PFG_CUDA(cudaMemsetAsync(dC.p, 0, 34 * 41 * 8, st));
    switch (std::max(1, dp / 32)) {
        case 1: launch_mc<1>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
        case 2: launch_mc<2>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
        case 4: launch_mc<4>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
        case 8: launch_mc<8>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
        case 16: launch_mc<16>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
        default: launch_mc<32>(dXY.as<float>(), dp, npairs, g, dS.as<uint32_t>(), dC.as<unsigned long long>(), I->num_sms, st); break;
    }
    PFG_CUDA(cudaGetLastError());
    std::vector<unsigned long long> cnt(34 * 41);
    PFG_CUDA(cudaMemcpyAsync(cnt.data(), dC.p, cnt.size() * 8, cudaMemcpyDeviceToHost, st));
    PFG_CUDA(cudaStreamSynchronize(st));
    const int ell = g.ell;
    std::vector<double>& T = I->cpT;
    T.assign((size_t)(ell + 1) * 41, 1.0);
    for (int b = 1; b <= ell; ++b) {
        for (int a = 0; a < 41; ++a) T[b * 41 + a] = (double)cnt[b * 41 + a] / (double)draws;
        T[b * 41 + 40] = 1.0;
        for (int a = 39; a >= 0; --a)
            if (T[b * 41 + a + 1] < T[b * 41 + a]) T[b * 41 + a] = T[b * 41 + a + 1];
    }
    for (int b = 2; b <= ell; ++b)
        for (int a = 0; a < 41; ++a)
            if (T[(b - 1) * 41 + a] < T[b * 41 + a]) T[b * 41 + a] = T[(b - 1) * 41 + a];
    return PFG_OK;
}

// exact CP collision table with the paper's canonical pair x = e_0,
// y = (alpha, sqrt(1 - alpha^2), 0, ...) -- valid by the spherical symmetry of exact CP
// (PAPER.md:349 footnote): only the first two coordinates of each hyperplane enter, drawn as
// a_i0 = gauss(k, 2i), a_i1 = gauss(k, 2i + 1) with k = draw(stream kTagCPMC, a draws + t); each
// inner product is the fmaf chain of R-2 over the (zero-padded) pair; then the same cleaning as the
// FHT table (running minima over alpha, then over bits)
void cp_exact_code_pair(const float* a0, const float* a1, int d, float yx, float yy, int ell, uint32_t& hx,
                        uint32_t& hy) {
    float bx = -1.0f, by = -1.0f;
    int ix = 0, iy = 0;
    bool nx = false, ny = false;
    for (int i = 0; i < d; ++i) {
        const float sx = fmaf(a0[i], 1.0f, 0.0f);
        const float sy = fmaf(a1[i], yy, fmaf(a0[i], yx, 0.0f));
        if (std::fabs(sx) > bx) { bx = std::fabs(sx); ix = i; nx = sx < 0.0f; }
        if (std::fabs(sy) > by) { by = std::fabs(sy); iy = i; ny = sy < 0.0f; }
    }
    hx = (nx ? 1u << (ell - 1) : 0u) | (uint32_t)ix;
    hy = (ny ? 1u << (ell - 1) : 0u) | (uint32_t)iy;
}
void build_cp_exact_table(pfg_index* I) {
    const Geo& g = I->g;
    const int draws = g.cp_draws, d = g.d, ell = g.ell;
    const uint64_t K = stream_key(I->seed, kTagCPMC);
    std::vector<long long> cnt((size_t)(ell + 1) * 41, 0);
    auto work = [&](int a0_, int a1_) {
        std::vector<float> A0(d), A1(d);
        for (int a = a0_; a < a1_; ++a) {
            const double alpha = -1.0 + 0.05 * a;
            const float yx = (float)alpha, yy = (float)std::sqrt(std::max(0.0, 1.0 - alpha * alpha));
            for (int t = 0; t < draws; ++t) {
                const uint64_t k = draw(K, (uint64_t)a * draws + t);
                for (int i = 0; i < d; ++i) { A0[i] = (float)gauss(k, 2ull * i); A1[i] = (float)gauss(k, 2ull * i + 1); }
                uint32_t hx, hy;
                cp_exact_code_pair(A0.data(), A1.data(), d, yx, yy, ell, hx, hy);
                for (int b = 1; b <= ell; ++b)
                    if ((hx >> (ell - b)) == (hy >> (ell - b))) cnt[b * 41 + a]++;
            }
        }
    };
    {
        unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        const int per = (41 + (int)nt - 1) / (int)nt;
        for (unsigned k = 0; k < nt; ++k) {
            const int a0 = (int)k * per, a1 = std::min(41, a0 + per);
            if (a0 < a1) th.emplace_back(work, a0, a1);
        }
        for (auto& t : th) t.join();
    }
    std::vector<double>& T = I->cpT;
    T.assign((size_t)(ell + 1) * 41, 1.0);
    for (int b = 1; b <= ell; ++b) {
        for (int a = 0; a < 41; ++a) T[b * 41 + a] = (double)cnt[b * 41 + a] / (double)draws;
        T[b * 41 + 40] = 1.0;
        for (int a = 39; a >= 0; --a)
            if (T[b * 41 + a + 1] < T[b * 41 + a]) T[b * 41 + a] = T[b * 41 + a + 1];
    }
    for (int b = 2; b <= ell; ++b)
        for (int a = 0; a < 41; ++a)
            if (T[(b - 1) * 41 + a] < T[b * 41 + a]) T[b * 41 + a] = T[(b - 1) * 41 + a];
}

pfg_status gen_functions(pfg_index* I, cudaStream_t st) {
    const Geo& g = I->g;
    const uint64_t seed = I->seed;
    // sketch functions: [64M][dpad] Gaussian, stream kTagSketch, element f*d + t
    if (g.M > 0) {
        const int64_t F = 64ll * g.M;
        std::vector<float> A((size_t)F * g.dpad, 0.0f);
        const uint64_t ks = stream_key(seed, kTagSketch);
        for (int64_t f = 0; f < F; ++f)
            for (int t = 0; t < g.d; ++t) A[(size_t)f * g.dpad + t] = (float)gauss(ks, (uint64_t)(f * g.d + t));
        PFG_TRY(I->skfn.alloc(A.size() * 4, "sketch functions"));
        PFG_CUDA(cudaMemcpyAsync(I->skfn.p, A.data(), A.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    // slot of repetition j
    I->slot_h.assign(g.L, 0);
    std::vector<uint8_t> sl(g.L, 0);
    const uint64_t kl = stream_key(seed, kTagSlot);
    for (int j = 0; j < g.L; ++j) {
        I->slot_h[j] = g.M > 0 ? (int32_t)(draw(kl, (uint64_t)j) % (uint64_t)g.M) : 0;
        sl[j] = (uint8_t)I->slot_h[j];
    }
    PFG_TRY(I->slot.alloc(g.L, "slots"));
    PFG_CUDA(cudaMemcpyAsync(I->slot.p, sl.data(), g.L, cudaMemcpyHostToDevice, st));
    // LSH functions: F = L*c (independent) or m (pool)
    const int64_t F = g.strategy != PFG_INDEPENDENT ? (int64_t)g.m : (int64_t)g.L * g.c;
    if (g.family == PFG_SIMHASH) {
        std::vector<float> A((size_t)F * g.dpad, 0.0f);
        const uint64_t kh = stream_key(seed, kTagHP);
        for (int64_t f = 0; f < F; ++f)
            for (int t = 0; t < g.d; ++t) A[(size_t)f * g.dpad + t] = (float)gauss(kh, (uint64_t)(f * g.d + t));
        PFG_TRY(I->hpfn.alloc(A.size() * 4, "hp functions"));
        PFG_CUDA(cudaMemcpyAsync(I->hpfn.p, A.data(), A.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
    } else if (g.family == PFG_CROSSPOLYTOPE) {
        // exact CP: function f = d hyperplanes, row (f d + i) of [F d][dpad], element
        // ((f d + i) d + t) of stream kTagCP; the independent strategy reads them through the
        // identity selection (repetition j, position t -> function j c + t)
        // stored transposed for the kernel: AT[f][t][i], i padded to d32
        const int d32 = (g.d + 31) / 32 * 32;
        std::vector<float> A((size_t)F * g.d * d32, 0.0f);
        const uint64_t kc = stream_key(seed, kTagCP);
        for (int64_t f = 0; f < F; ++f)
            for (int i = 0; i < g.d; ++i)
                for (int t = 0; t < g.d; ++t)
                    A[((size_t)f * g.d + t) * d32 + i] = (float)gauss(kc, (uint64_t)((f * g.d + i) * g.d + t));
        PFG_TRY(I->hpfn.alloc(A.size() * 4, "cp functions"));
        PFG_CUDA(cudaMemcpyAsync(I->hpfn.p, A.data(), A.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
        if (g.strategy == PFG_INDEPENDENT) {
            std::vector<int32_t> id((size_t)g.L * g.c);
            for (size_t e = 0; e < id.size(); ++e) id[e] = (int32_t)e;
            PFG_TRY(I->sel.alloc(id.size() * 4, "cp identity selection"));
            PFG_CUDA(cudaMemcpyAsync(I->sel.p, id.data(), id.size() * 4, cudaMemcpyHostToDevice, st));
            PFG_CUDA(cudaStreamSynchronize(st));
        }
    } else {
        std::vector<uint32_t> S((size_t)F * 3 * g.W, 0u);
        const uint64_t kf = stream_key(seed, kTagFHT);
        for (int64_t f = 0; f < F; ++f)
            for (int r = 0; r < 3; ++r)
                for (int u = 0; u < g.dp; ++u)
                    if (draw(kf, (uint64_t)((f * 3 + r) * g.dp + u)) >> 63)
                        S[(size_t)(f * 3 + r) * g.W + (u >> 5)] |= 1u << (u & 31);
        PFG_TRY(I->sg.alloc(S.size() * 4, "fht signs"));
        PFG_CUDA(cudaMemcpyAsync(I->sg.p, S.data(), S.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    if (g.strategy == PFG_TENSOR) {
        // trie (j1, j2), j = j1*S + j2: position t = 2s + a holds function s of collection a's tuple
        // (j1 for a = 0, j2 for a = 1), function (a, tuple, s) = (a*S + tuple)*(c/2) + s
        // ("taken by interleaving")
        const int S = g.S, h = g.c / 2;
        I->sel_h.assign((size_t)g.L * g.c, 0);
        for (int j = 0; j < g.L; ++j)
            for (int t = 0; t < g.c; ++t) {
                const int a = t % 2, s = t / 2, tuple = a ? j % S : j / S;
                I->sel_h[(size_t)j * g.c + t] = (a * S + tuple) * h + s;
            }
        PFG_TRY(I->sel.alloc(I->sel_h.size() * 4, "tensor selection"));
        PFG_CUDA(cudaMemcpyAsync(I->sel.p, I->sel_h.data(), I->sel_h.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    if (g.strategy == PFG_POOL) {
        // PAPER.md:886 random subsets of the pool: partial Fisher-Yates per repetition
        const uint64_t kp = stream_key(seed, kTagPool);
        I->sel_h.assign((size_t)g.L * g.c, 0);
        std::vector<int32_t> perm(g.m);
        for (int j = 0; j < g.L; ++j) {
            for (int f = 0; f < g.m; ++f) perm[f] = f;
            for (int t = 0; t < g.c; ++t) {
                const int64_t r = t + (int64_t)(draw(kp, (uint64_t)j * g.c + t) % (uint64_t)(g.m - t));
                std::swap(perm[t], perm[r]);
                I->sel_h[(size_t)j * g.c + t] = perm[t];
            }
        }
        PFG_TRY(I->sel.alloc(I->sel_h.size() * 4, "pool selection"));
        PFG_CUDA(cudaMemcpyAsync(I->sel.p, I->sel_h.data(), I->sel_h.size() * 4, cudaMemcpyHostToDevice, st));
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    return PFG_OK;
}

// codes of np normalised rows X for repetitions [r0, r0+nb): keys [r][p] and/or codes [p][ldc]
// (pool strategy: pool values computed once into `poolvals`)
// exact CP function values of functions [f0, f0 + nf) for rows 0..np-1 or qlist[0..np) (np_dev:
// the count in device memory) into out [np][nf] (uint16)
pfg_status cp_values(pfg_index* I, const float* X, int64_t np, const uint32_t* qlist, const uint32_t* np_dev, int f0, int nf,
                     uint16_t* out, cudaStream_t st) {
    const Geo& g = I->g;
    const int d32 = (g.d + 31) / 32 * 32;
    const float* AT = I->hpfn.as<float>() + (int64_t)f0 * g.d * d32;
#ifndef PFG_CP_RW
#define PFG_CP_RW 8
#endif
    constexpr int RW = PFG_CP_RW;   // rows per warp (register tile RW x NI)
    if (!qlist && !np_dev && PFG_CP_TC && (g.dpad % 4) == 0 && ((uintptr_t)X % 16) == 0) {
        // tcgen05 (kernels_tc.cuh k_cp_tc): 3xTF32 values, the exact chains only for near ties
        const int nt = g.d <= 128 ? 128 : 256;
        const size_t sm = (size_t)(2 * TC_M * TC_KC + 2 * nt * TC_KC) * 4;
        const void* fn = nt == 128 ? (const void*)k_cp_tc<128> : (const void*)k_cp_tc<256>;
        if (set_smem(fn, sm) == cudaSuccess) {
            const dim3 grid((unsigned)((np + TC_M - 1) / TC_M), (unsigned)nf);
            if (nt == 128) k_cp_tc<128><<<grid, 128, sm, st>>>(X, np, g.dpad, AT, nf, g.d, d32, g.ell, out);
            else k_cp_tc<256><<<grid, 128, sm, st>>>(X, np, g.dpad, AT, nf, g.d, d32, g.ell, out);
            PFG_CUDA(cudaGetLastError());
            return PFG_OK;
        }
    }
    switch (d32 / 32) {
#define PFG_CP_CASE(NI)                                                                                        \
    case NI: {                                                                                                 \
        constexpr int rw = NI > 4 ? 4 : RW;                                                                    \
        k_cp_funcs<NI, rw><<<dim3((unsigned)((np + 4 * rw - 1) / (4 * rw)), (unsigned)nf), 128, 0, st>>>(     \
            X, np, g.dpad, AT, nf, g.d, d32, g.ell, out, qlist, np_dev);                                       \
        break;                                                                                                 \
    }
        PFG_CP_CASE(1) PFG_CP_CASE(2) PFG_CP_CASE(3) PFG_CP_CASE(4)
        PFG_CP_CASE(5) PFG_CP_CASE(6) PFG_CP_CASE(7) PFG_CP_CASE(8)
#undef PFG_CP_CASE
        default: return fail(PFG_E_ARG, "exact cross-polytope family supports d <= 256");
    }
    PFG_CUDA(cudaGetLastError());
    return PFG_OK;
}

pfg_status hash_reps(pfg_index* I, const float* X, int64_t np, int r0, int nb, uint64_t* keys, uint32_t* codes, int ldc,
                     DBuf& bits, DBuf& poolvals, bool& pool_ready, cudaStream_t st) {
    const Geo& g = I->g;
    const dim3 blk(256);
    const dim3 grd((unsigned)((np + 255) / 256), (unsigned)nb);
    if (g.family == PFG_SIMHASH) {
        if (g.strategy == PFG_INDEPENDENT) {
            const int nf = nb * g.K;
            const int wpr = (nf + 63) / 64;
            PFG_TRY(bits.ensure((size_t)np * wpr * 8, "hp bits"));
            hp_bits(X, np, g.dpad, I->hpfn.as<float>() + (size_t)r0 * g.K * g.dpad, nf, g.dpad, g.dpad,
                    bits.as<uint8_t>(), (int64_t)wpr * 8, st);
            k_codes_from_bits<<<grd, blk, 0, st>>>(bits.as<uint64_t>(), np, wpr, r0, nb, g.K, nullptr, r0, keys, codes, ldc);
            I->launches += 2;
        } else {
            const int wpr = (g.m + 63) / 64;
            if (!pool_ready) {
                PFG_TRY(poolvals.ensure((size_t)np * wpr * 8, "pool bits"));
                hp_bits(X, np, g.dpad, I->hpfn.as<float>(), g.m, g.dpad, g.dpad, poolvals.as<uint8_t>(), (int64_t)wpr * 8, st);
                pool_ready = true;
                I->launches += 1;
            }
            I->launches += 1;
            k_codes_from_bits<<<grd, blk, 0, st>>>(poolvals.as<uint64_t>(), np, wpr, r0, nb, g.K, I->sel.as<int32_t>(), 0,
                                                   keys, codes, ldc);
        }
    } else if (g.family == PFG_CROSSPOLYTOPE) {
        // all function values once (uint16 [np][F]), then each repetition's concatenation
        const int F = g.strategy == PFG_POOL ? g.m : g.L * g.c;
        if (!pool_ready) {
            PFG_TRY(poolvals.ensure((size_t)np * F * 2, "cp function codes"));
            PFG_TRY(cp_values(I, X, np, nullptr, nullptr, 0, F, poolvals.as<uint16_t>(), st));
            pool_ready = true;
            I->launches += 1;
        }
        I->launches += 1;
        k_pool_codes<<<grd, blk, 0, st>>>(poolvals.as<uint16_t>(), np, F, r0, nb, g.c, g.ell, g.K, I->sel.as<int32_t>(),
                                          keys, codes, ldc);
    } else {
        if (g.strategy == PFG_INDEPENDENT) {
            fht_rep(X, np, g.dpad, g, I->sg.as<uint32_t>(), r0, nb, keys, codes, ldc, I->num_sms, st);
            I->launches += 1;
        } else {
            if (!pool_ready) {
                PFG_TRY(poolvals.ensure((size_t)np * g.m * 2, "pool codes"));
                fht_funcs(X, np, g.dpad, g, I->sg.as<uint32_t>(), poolvals.as<uint16_t>(), I->num_sms, st);
                pool_ready = true;
                I->launches += 1;
            }
            I->launches += 1;
            k_pool_codes<<<grd, blk, 0, st>>>(poolvals.as<uint16_t>(), np, g.m, r0, nb, g.c, g.ell, g.K,
                                              I->sel.as<int32_t>(), keys, codes, ldc);
        }
    }
    PFG_CUDA(cudaGetLastError());
    return PFG_OK;
}

pfg_status normalize_rows(const float* src, int64_t n, int d, float* dst, int dpad, uint8_t* zflag,
                          unsigned long long* zmin_dev, int64_t* zrow, cudaStream_t st, int num_sms = 148) {
    PFG_CUDA(cudaMemsetAsync(zmin_dev, 0xff, 8, st));
    // rows per block staged in shared memory; a small batch (a query batch) takes fewer per block so
    // that every SM gets about eight blocks (the per-thread loops are latency-bound)
    const int rb = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(32, 12288 / d), n / (8 * (int64_t)num_sms)));
    k_normalize<<<(unsigned)((n + rb - 1) / rb), 128, (size_t)rb * d * 4, st>>>(src, n, d, d, dst, dpad, zflag, zmin_dev, rb);
    PFG_CUDA(cudaGetLastError());
    if (!zrow) return PFG_OK;  // asynchronous: the caller reads zmin_dev later
    unsigned long long z = 0;
    PFG_CUDA(cudaMemcpyAsync(&z, zmin_dev, 8, cudaMemcpyDeviceToHost, st));
    PFG_CUDA(cudaStreamSynchronize(st));
    *zrow = (z == ~0ull) ? -1 : (int64_t)z;
    return PFG_OK;
}

// stop/threshold tables for (recall, rule, granularity); cached on the index
pfg_status get_thr(pfg_index* I, float recall, const SearchCfg& s, std::shared_ptr<DBuf>& out, std::vector<float>* host) {
    uint32_t rb;
    std::memcpy(&rb, &recall, 4);
    const auto key = std::make_tuple(rb, s.rule, s.per_round);
    auto it = I->thr_cache.find(key);
    if (it != I->thr_cache.end() && !host) {
        out = it->second;
        return PFG_OK;
    }
    const Geo& g = I->g;
    const double delta = 1.0 - (double)recall;
    StopModel sm{g.family, g.strategy, g.ell, g.m, I->cpT.empty() ? nullptr : I->cpT.data(), g.K, g.L};
    std::vector<float> thr((size_t)g.K * g.L);
    auto work = [&](int i0, int i1) {
        for (int i = i0; i < i1; ++i)
            for (int j = 1; j <= g.L; ++j) {
                float v;
                if (g.strategy == PFG_TENSOR ? j > g.S : (s.per_round && j < g.L)) v = INFINITY;
                else v = smallest_true([&](float ip) { return sm.stop(i, j, ip, delta, s.rule); });
                thr[(size_t)(i - 1) * g.L + (j - 1)] = v;
            }
    };
    {
        unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (unsigned k = 0; k < nt; ++k) {
            const int i0 = 1 + (int)(k * g.K / nt), i1 = 1 + (int)((k + 1) * g.K / nt);
            if (i0 < i1) th.emplace_back(work, i0, i1);
        }
        for (auto& t : th) t.join();
    }
    if (host) *host = thr;
    auto buf = std::make_shared<DBuf>();
    PFG_TRY(buf->alloc(thr.size() * 4, "stop thresholds"));
    PFG_CUDA(cudaMemcpy(buf->p, thr.data(), thr.size() * 4, cudaMemcpyHostToDevice));
    I->thr_cache[key] = buf;
    out = buf;
    return PFG_OK;
}

pfg_status get_tau(pfg_index* I, int rule, float eps, float recall, std::shared_ptr<DBuf>& out, std::vector<float>* host) {
    uint32_t eb, rb;
    std::memcpy(&eb, &eps, 4);
    std::memcpy(&rb, &recall, 4);
    const auto key = rule ? std::make_tuple(rule, eb, 0u) : std::make_tuple(rule, 0u, rb);
    auto it = I->tau_cache.find(key);
    if (it != I->tau_cache.end() && !host) {
        out = it->second;
        return PFG_OK;
    }
    const double delta = 1.0 - (double)recall;
    std::vector<float> tb(65);
    for (int t = 0; t < 65; ++t)
        tb[t] = smallest_true([&](float ip) { return (rule ? tau_of(ip, eps) : tau_quantile(ip, delta)) <= t; });
    tb[64] = -1.0f;
    if (host) *host = tb;
    auto buf = std::make_shared<DBuf>();
    PFG_TRY(buf->alloc(65 * 4, "tau breakpoints"));
    PFG_CUDA(cudaMemcpy(buf->p, tb.data(), 65 * 4, cudaMemcpyHostToDevice));
    I->tau_cache[key] = buf;
    out = buf;
    return PFG_OK;
}

// the side streams and the events that order them against the search stream, created together
// (every later use may assume all of them exist, whatever the index's sketch or family settings)
pfg_status ensure_streams(pfg_index* I) {
    if (I->aux) return PFG_OK;
    PFG_CUDA(cudaStreamCreateWithFlags(&I->aux, cudaStreamNonBlocking));
    PFG_CUDA(cudaStreamCreateWithFlags(&I->aux2, cudaStreamNonBlocking));
    PFG_CUDA(cudaStreamCreateWithFlags(&I->st1, cudaStreamNonBlocking));
    int prio_lo = 0, prio_hi = 0;
    PFG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    PFG_CUDA(cudaStreamCreateWithPriority(&I->hst, cudaStreamNonBlocking, prio_hi));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_hst, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_in, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_h1start, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_h1end, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_fork, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_join, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_late, cudaEventDisableTiming));
    PFG_CUDA(cudaEventCreateWithFlags(&I->ev_mid, cudaEventDisableTiming));
    return PFG_OK;
}

// normalise + sketch + (eager) code queries into index scratch; returns first zero row or -1
pfg_status prep_queries(pfg_index* I, const float* queries, int64_t nq, bool need_codes, bool force_codes, int64_t* zrow,
                        bool* lazy, cudaStream_t st, int split, int cp_eager = 0, const ExtHash* ext = nullptr) {
    const Geo& g = I->g;
    PFG_TRY(ensure_streams(I));
    const float* qsrc = queries;
    if (!is_device_ptr(queries)) {
        PFG_TRY(I->qraw.ensure((size_t)nq * g.d * 4, "query copy"));
        PFG_CUDA(cudaMemcpyAsync(I->qraw.p, queries, (size_t)nq * g.d * 4, cudaMemcpyHostToDevice, st));
        qsrc = I->qraw.as<float>();
    }
    PFG_TRY(I->qx.ensure((size_t)nq * g.dpad * 4, "queries"));
    PFG_TRY(I->qzero.ensure((size_t)nq, "query zero flags"));
    PFG_TRY(I->zmin.ensure(8, "zmin"));
    PFG_TRY(normalize_rows(qsrc, nq, g.d, I->qx.as<float>(), g.dpad, I->qzero.as<uint8_t>(),
                           I->zmin.as<unsigned long long>(), zrow, st, I->num_sms));
    tl_mark(I, "normalize", st);
    if (g.storage == PFG_STORAGE_I16) {
        // R-25: the queries' fixed-point rows for the inner products
        PFG_TRY(I->qx16.ensure((size_t)nq * g.dpad16 * 2, "int16 queries"));
        const int64_t tot = nq * (int64_t)g.dpad16;
        k_quantize<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(I->qx.as<float>(), nq, g.dpad, g.d, I->qx16.as<int16_t>(),
                                                                 g.dpad16);
        PFG_CUDA(cudaGetLastError());
        I->launches += 1;
    }
    if (!zrow) {
        if (!I->h_zmin) PFG_CUDA(cudaMallocHost(&I->h_zmin, 8));
        if (!I->ev_zmin) PFG_CUDA(cudaEventCreateWithFlags(&I->ev_zmin, cudaEventDisableTiming));
        PFG_CUDA(cudaMemcpyAsync(I->h_zmin, I->zmin.p, 8, cudaMemcpyDeviceToHost, st));
        PFG_CUDA(cudaEventRecord(I->ev_zmin, st));
    }
    I->launches += 1;
    // the normalised (and quantised) queries are ready: the side streams start from here
    PFG_CUDA(cudaEventRecord(I->ev_fork, st));
    if (g.M > 0) {
        // sketches (FMA pipe) on the second stream, concurrently with the hashing below; the
        // caller joins (join_sketches) before anything reads them
        PFG_TRY(I->qsk.ensure((size_t)nq * g.M * 8, "query sketches"));
        if (ext && ext->sk) {
            PFG_CUDA(cudaMemcpyAsync(I->qsk.p, ext->sk, (size_t)nq * g.M * 8, cudaMemcpyDeviceToDevice, st));
            PFG_CUDA(cudaEventRecord(I->ev_join, st));
        } else {
            PFG_CUDA(cudaStreamWaitEvent(I->aux, I->ev_fork, 0));
            hp_bits(I->qx.as<float>(), nq, g.dpad, I->skfn.as<float>(), 64 * g.M, g.dpad, g.dpad, I->qsk.as<uint8_t>(),
                    (int64_t)g.M * 8, I->aux, I->num_sms);   // one CTA per SM looping over the tiles: it
                                                              // runs beside round 0 (measured 1.595 -> 1.59 ms)
            PFG_CUDA(cudaGetLastError());
            tl_mark(I, "query sketches (k_hp_bits_tc)", I->aux);
            PFG_CUDA(cudaEventRecord(I->ev_join, I->aux));
            I->launches += 1;
        }
    }
    *lazy = (g.family == PFG_CROSSPOLYTOPE_FHT && g.strategy == PFG_INDEPENDENT && !force_codes);
    I->qc_n = 0;
    I->qc_ld = g.L;
    if (need_codes && ext && ext->codes) {
        // precomputed codes of repetitions [0, reps) (all L unless the family hashes lazily); rows
        // laid out with room for kExtReps more for the queries the fused kernel resumes
        const int ld = *lazy ? std::min(g.L, ext->reps + kExtReps) : g.L;
        PFG_TRY(I->qcodes.ensure((size_t)nq * ld * 4, "query codes"));
        PFG_CUDA(cudaMemcpy2DAsync(I->qcodes.p, (size_t)ld * 4, ext->codes, (size_t)ext->reps * 4, (size_t)ext->reps * 4,
                                   (size_t)nq, cudaMemcpyDeviceToDevice, st));
        I->qc_n = ext->reps;
        I->qc_ld = ld;
        I->qc_split = ext->reps;
    } else if (need_codes && !*lazy && cp_eager > 0) {
        // exact CP, independent: the repetitions the blind rounds can reach only (cp_eager); the
        // queries still running after them get the rest in bulk (the caller)
        PFG_TRY(I->qcodes.ensure((size_t)nq * g.L * 4, "query codes"));
        const int F = cp_eager * g.c;
        PFG_TRY(I->qfc.ensure((size_t)nq * F * 2, "cp function codes"));
        PFG_TRY(cp_values(I, I->qx.as<float>(), nq, nullptr, nullptr, 0, F, I->qfc.as<uint16_t>(), st));
        k_pool_codes<<<dim3((unsigned)((nq + 255) / 256), (unsigned)cp_eager), 256, 0, st>>>(
            I->qfc.as<uint16_t>(), nq, F, 0, cp_eager, g.c, g.ell, g.K, I->sel.as<int32_t>(), nullptr,
            I->qcodes.as<uint32_t>(), g.L);
        PFG_CUDA(cudaGetLastError());
        I->launches += 2;
        I->qc_n = cp_eager;
    } else if (need_codes && !*lazy) {
        PFG_TRY(I->qcodes.ensure((size_t)nq * g.L * 4, "query codes"));
        bool pool_ready = false;
        PFG_TRY(hash_reps(I, I->qx.as<float>(), nq, 0, g.L, nullptr, I->qcodes.as<uint32_t>(), g.L, I->qbits, I->qfc,
                          pool_ready, st));
        I->qc_n = g.L;
    } else if (need_codes && (g.dp == 32 || g.dp == 64 || g.dp == 128)) {
        // FHT-CP independent: hash the first I->eager repetitions of every query here, one thread
        // per (query, repetition); the query kernel hashes later repetitions lazily, if reached
        // (rows are laid out with room for kExtReps more, hashed later for the queries that reach
        // them: extend_codes)
        const int ne = std::min(g.L, I->eager);
        const int ld = std::min(g.L, ne + kExtReps);
        PFG_TRY(I->qcodes.ensure((size_t)nq * ld * 4, "query codes"));
        // repetitions [0, split) now; [split, ne) on the third stream, joined before the round
        // that first reaches them (the caller: late_join)
        // Round 0 reaches repetition 0 only, round 1 repetitions [1, split): only repetition 0 is
        // hashed before round 0; [1, split) runs on the third stream beside round 0 (the caller
        // records ev_mid after its ranges, round 1 joins it) and [split, ne) after it (ev_late,
        // round 2 joins it)
        const int s0 = (split > 0 && split < ne && I->aux2) ? split : ne;
        const bool mid = s0 < ne && s0 > 1;
        if (mid) {
            // repetition 0 (round 0's only repetition) on the highest-priority stream, so that its
            // codes and ranges (the caller) are not queued behind the side streams' hashing
            PFG_CUDA(cudaStreamWaitEvent(I->hst, I->ev_fork, 0));
            PFG_TRY(fht_codes(I, nq, nullptr, 0, 1, ld, I->hst));
            I->hst_pending = true;
        } else {
            PFG_TRY(fht_codes(I, nq, nullptr, 0, s0, ld, st));
        }
        if (s0 < ne) {
            PFG_CUDA(cudaStreamWaitEvent(I->aux2, I->ev_fork, 0));
            if (mid) {
                PFG_TRY(fht_codes(I, nq, nullptr, 1, s0 - 1, ld, I->aux2));
                I->mid_pending = true;
                I->late_ne = ne;   // [s0, ne): launched by the caller after the ranges of [1, s0)
            } else {
                PFG_TRY(fht_codes(I, nq, nullptr, s0, ne - s0, ld, I->aux2));
                I->late_ne = 0;
            }
            I->late_pending = true;
        }
        I->qc_n = ne;
        I->qc_ld = ld;
        I->qc_split = s0;
    }
    return PFG_OK;
}

// Kernels over a device-counted query list (the queries still running late in a search) size their
// grid for list_rows() rows and loop over the rest: a grid for the list's capacity (the batch) would
// mostly launch blocks that exit at once
inline int64_t list_rows(const pfg_index* I) { return (int64_t)I->num_sms * 8; }
inline unsigned list_grid(const pfg_index* I, int64_t threads, int nreps) {
    return (unsigned)((std::min<int64_t>(threads, list_rows(I) * nreps) + 255) / 256);
}

// FHT-CP query codes of repetitions [r0, r0 + nreps) for rows qlist[0..nrows) (or 0..nrows-1),
// one thread per (row, repetition), into qcodes [q][ld]
pfg_status fht_codes(pfg_index* I, int64_t nrows, const uint32_t* qlist, int r0, int nreps, int ld, cudaStream_t st,
                     const uint32_t* nrows_dev, int64_t q0) {
    // q0: rows (and qlist entries) relative to query q0 (a round pipeline's part of the batch)
    const Geo& g = I->g;
    const int64_t threads = nrows * nreps;
    if (threads == 0) return PFG_OK;
    const unsigned blocks = (unsigned)((threads + 127) / 128);
    const uint32_t* sg = I->sg.as<uint32_t>();
    uint32_t* qc = I->qcodes.as<uint32_t>() + q0 * ld;
    const float* X = I->qx.as<float>() + q0 * g.dpad;
    if (nrows_dev && g.dp == 128) {
        // a device-counted list (the queries still running late in a search, usually few): four
        // lanes per item (a quarter of the single-thread transform's dependent chain), a grid-stride
        // loop over a grid for list_rows() rows
        const int64_t t4 = 4 * std::min<int64_t>(threads, list_rows(I) * nreps);
        k_fht_qcodes_g<128, 4, true><<<(unsigned)((t4 + 127) / 128), 128, 0, st>>>(X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps,
                                                                         qc, ld, qlist, r0, nrows_dev);
    } else {
        const unsigned bl = nrows_dev ? (unsigned)((std::min<int64_t>(threads, list_rows(I) * nreps) + 127) / 128) : blocks;
        if (g.dp == 32 && nrows_dev) k_fht_qcodes_g<32, 1, true><<<bl, 128, 0, st>>>(X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps, qc, ld, qlist, r0, nrows_dev);
        else if (g.dp == 64 && nrows_dev) k_fht_qcodes_g<64, 1, true><<<bl, 128, 0, st>>>(X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps, qc, ld, qlist, r0, nrows_dev);
        else if (g.dp == 32) k_fht_qcodes_g<32, 1><<<bl, 128, 0, st>>>(X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps, qc, ld, qlist, r0, nrows_dev);
        else if (g.dp == 64) k_fht_qcodes_g<64, 1><<<bl, 128, 0, st>>>(X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps, qc, ld, qlist, r0, nrows_dev);
        else k_fht_qcodes_g<128, PFG_QTPF><<<(unsigned)((PFG_QTPF * (int64_t)bl * 128 + 127) / 128), 128, 0, st>>>(
                 X, nrows, g.dpad, g.d, g.ell, g.c, g.K, sg, nreps, qc, ld, qlist, r0, nrows_dev);
    }
    PFG_CUDA(cudaGetLastError());
    I->launches += 1;
    tl_mark(I, (std::string("fht codes reps ") + std::to_string(r0) + "+" + std::to_string(nreps)).c_str(), st);
    return PFG_OK;
}

// eager depth for the next search: the repetition count by which 99% of the last batch's queries
// had stopped (deeper stops count as L), clamped to [8, 64]; codes are identical either way
void tune_eager(pfg_index* I) {
    if (!I->h_jhist) return;
    uint64_t tot = 0, cum = 0;
    for (int j = 0; j < kJHist; ++j) tot += I->h_jhist[j];
    int e = kJHist - 1;
    for (int j = 0; j < kJHist; ++j) {
        cum += I->h_jhist[j];
        if (tot && cum * 100 >= tot * 99) { e = j; break; }
    }
    if (tot) I->eager = std::max(8, std::min(64, e));
    // level-K match ranges computed in bulk before the query kernels (k_qbounds): the depth 99 % of
    // the queries reach at level K, all L repetitions when they go deeper (the fused kernel would
    // otherwise binary-search them one warp at a time)
    if (tot) I->qb_depth = e >= kJHist - 1 ? (1 << 30) : std::max(8, e);
}

// developer aid (a -DPFG_DEBUG_SYNC=1 build): synchronise after each launch group and name the failing one
#ifndef PFG_DEBUG_SYNC
#define PFG_DEBUG_SYNC 0
#endif
pfg_status dbg_sync(const char* what) {
    if (!PFG_DEBUG_SYNC) return PFG_OK;
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return fail(PFG_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return PFG_OK;
}

// timing = 3: sum the recorded k_sims event pairs (waits for the last one) into kev_ms
pfg_status fold_kernel_timing(pfg_index* I) {
    if (I->kev_n == 0) return PFG_OK;
    PFG_CUDA(cudaEventSynchronize(I->kev[2 * I->kev_n - 1]));
    for (int64_t i = 0; i < I->kev_n; ++i) {
        float ms = 0.0f;
        PFG_CUDA(cudaEventElapsedTime(&ms, I->kev[2 * i], I->kev[2 * i + 1]));
        I->kev_ms += ms;
    }
    I->kev_launches += I->kev_n;
    I->kev_n = 0;
    return PFG_OK;
}

// phases of pfg_last_phases: 0 expand, 1 scan, 2 dedupe, 3 sims, 4 merge, 5 fused kernel,
// 6 other query-phase work (round control, query order, code extension)
enum { kPhExpand = 0, kPhScan, kPhDedupe, kPhSims, kPhMerge, kPhFused, kPhOther, kPhLoop, kPhEnd = -1 };
pfg_status phase_mark(pfg_index* I, bool on, int kind, cudaStream_t st) {
    if (!on) return PFG_OK;
    if (I->pev_n == (int)I->pev.size()) {
        cudaEvent_t e;
        PFG_CUDA(cudaEventCreate(&e));
        I->pev.push_back(e);
        I->pkind.push_back(kind);
    }
    I->pkind[I->pev_n] = kind;
    PFG_CUDA(cudaEventRecord(I->pev[I->pev_n++], st));
    return PFG_OK;
}
pfg_status phase_collect(pfg_index* I) {
    for (float& v : I->last_phase_ms) v = 0.0f;
    for (int i = 0; i + 1 < I->pev_n; ++i) {
        float ms = 0.0f;
        PFG_CUDA(cudaEventElapsedTime(&ms, I->pev[i], I->pev[i + 1]));
        if (I->pkind[i] >= 0) I->last_phase_ms[I->pkind[i]] += ms;
    }
    I->pev_n = 0;
    return PFG_OK;
}

// timing = 4: timeline mark (completion of everything enqueued on `st` so far)
void tl_mark(pfg_index* I, const char* name, cudaStream_t st) {
    if (!I->tl_on) return;
    if (I->tl_n == (int)I->tlev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) { cudaGetLastError(); return; }
        I->tlev.push_back(e);
        I->tlname.emplace_back();
    }
    const char* sn = st == I->aux ? "aux" : st == I->aux2 ? "aux2" : "main";
    I->tlname[I->tl_n] = std::string(sn) + " " + name;
    cudaEventRecord(I->tlev[I->tl_n++], st);
}
void tl_print(pfg_index* I) {
    if (!I->tl_on || I->tl_n == 0) return;
    cudaEventSynchronize(I->tlev[I->tl_n - 1]);
    cudaDeviceSynchronize();
    for (int i = 0; i < I->tl_n; ++i) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, I->tlev[0], I->tlev[i]);
        fprintf(stderr, "[pfg timeline] %8.1f us  %s\n", 1e3 * ms, I->tlname[i].c_str());
    }
    I->tl_n = 0;
}

// the query sketches of prep_queries are ready on `st` after this
pfg_status join_sketches(pfg_index* I, cudaStream_t st) {
    if (I->g.M > 0 && I->ev_join) PFG_CUDA(cudaStreamWaitEvent(st, I->ev_join, 0));
    return PFG_OK;
}
// the codes (and ranges) of the later eager repetitions are ready on `st` after this
pfg_status mid_join(pfg_index* I, cudaStream_t st) {
    if (I->mid_pending) {
        PFG_CUDA(cudaStreamWaitEvent(st, I->ev_mid, 0));
        I->mid_pending = false;
    }
    return PFG_OK;
}
pfg_status late_join(pfg_index* I, cudaStream_t st) {
    PFG_TRY(mid_join(I, st));
    if (I->late_pending) {
        PFG_CUDA(cudaStreamWaitEvent(st, I->ev_late, 0));
        I->late_pending = false;
    }
    return PFG_OK;
}

// The parameters of round pipeline h, which runs queries [q0, q0 + nh) of the batch as a search
// of its own: every per-query array is offset to row q0 (query ids in the lists are relative to
// q0), and the per-round shared state (control block, survivor pool, work counter, the fused
// kernel's bitmap slots) is pipeline h's share.  The two pipelines touch disjoint memory.
QueryParams pipeline_params(const QueryParams& p, int64_t q0, int64_t nh, int h, int64_t slots_h) {
    QueryParams s = p;
    s.nq = nh;
    s.qx = p.qx + q0 * p.dpad;
    if (p.qx16) s.qx16 = p.qx16 + q0 * p.dpad16;
    if (p.qsk) s.qsk = p.qsk + q0 * p.M;
    if (p.qcodes) s.qcodes = p.qcodes + q0 * p.qc_ld;
    if (p.qbnd) s.qbnd = p.qbnd + q0 * p.qb_ld;
    s.qzero = p.qzero + q0;
    s.cur = p.cur + q0 * p.L;
    s.out_ids = p.out_ids + q0 * p.k;
    s.out_sims = p.out_sims + q0 * p.k;
    if (p.stats) s.stats = p.stats + q0;
    if (p.trace_ids) s.trace_ids = p.trace_ids + q0 * p.trace_cap;
    s.work = p.work + h;
    s.bitmap = p.bitmap + h * slots_h * p.bm_words;
    s.claims = p.claims + h * slots_h * (int64_t)p.claim_cap;
    RoundState& r = s.rs;
    const RoundState& a = p.rs;
    r.lvl = a.lvl + q0; r.c0 = a.c0 + q0; r.flags = a.flags + q0; r.tn = a.tn + q0;
    r.cnt = a.cnt + q0 * kCnt; r.T = a.T + q0 * p.kt; r.E = a.E + q0 * a.Ecap; r.pend = a.pend + q0 * kMaxR;
    r.cand = a.cand + q0 * a.Ccap; r.tcnt = a.tcnt + q0 * (a.Ccap / kTile); r.hsave = a.hsave + q0 * kHC;
    r.rinfo = a.rinfo + q0; r.tiles = a.tiles + q0 * (a.Ccap / kTile) * 2; r.repcnt = a.repcnt + q0 * kMaxR * 3;
    r.poff = a.poff + q0; r.pn = a.pn + q0;
    r.act[0] = a.act[0] + q0; r.act[1] = a.act[1] + q0; r.dord[0] = a.dord[0] + q0; r.dord[1] = a.dord[1] + q0;
    r.fused = a.fused + q0; r.fused2 = a.fused2 + q0; r.wslot = a.wslot + q0; r.rtile = a.rtile + q0 * (kMaxR + 1);
    r.pool_cap = a.pool_cap / 2;
    r.pool_id = a.pool_id + h * (int64_t)r.pool_cap; r.pool_q = a.pool_q + h * (int64_t)r.pool_cap;
    r.pool_key = a.pool_key + h * (int64_t)r.pool_cap;
    r.ctl = a.ctl + h;
    return s;
}

template <int EPL>
pfg_status launch_query_t(const QueryParams& p, int blocks, size_t smem, cudaStream_t st, int num_sms = 148) {
    // the queries resumed after the bulk rounds are usually few and long: more rows in flight per
    // warp; a batch that may resume more queries than stay resident (16 warps per SM) keeps the
    // leaner variant (measured: config 3, 10 000 resumed queries, +8 %)
    const bool few = p.nq <= (int64_t)num_sms * 16;
    if (p.resume && few) {
        PFG_CUDA(set_smem((const void*)k_query<EPL, 16>, smem));
        k_query<EPL, 16><<<blocks, 128, smem, st>>>(p);
        PFG_CUDA(cudaGetLastError());
        return PFG_OK;
    }
    PFG_CUDA(set_smem((const void*)k_query<EPL>, smem));
    k_query<EPL><<<blocks, 128, smem, st>>>(p);
    PFG_CUDA(cudaGetLastError());
    return PFG_OK;
}
template <int EPL>
int query_occupancy(size_t smem) {
    int nb = 0;
    set_smem((const void*)k_query<EPL>, smem);
    if (occupancy(&nb, (const void*)k_query<EPL>, 128, smem) != cudaSuccess) {
        cudaGetLastError();
        nb = 1;
    }
    return std::max(1, nb);
}

int epl_of(const Geo& g) { return std::max(1, g.dp / 32); }


}  // namespace
}  // namespace pfg

// ---------------------------------------------------------------------------------------------
// serialisation: magic, ABI version, sizeof(Geo), Geo, seed, the device arrays (byte count then
// bytes, through a pinned staging buffer), the host tables
namespace {
const char kIdxMagic[8] = {'P', 'F', 'G', 'I', 'D', 'X', '0', '2'};
constexpr size_t kStage = (size_t)64 << 20;

struct Stage {
    void* h = nullptr;
    ~Stage() { if (h) cudaFreeHost(h); }
};
std::vector<DBuf*> index_arrays(pfg_index* I) {
    return {&I->x, &I->tab, &I->pt, &I->slot, &I->hpfn, &I->sg, &I->sel, &I->skfn, &I->x16};
}
template <class T>
bool put_vec(FILE* f, const std::vector<T>& v) {
    const uint64_t n = v.size();
    return fwrite(&n, 8, 1, f) == 1 && (n == 0 || fwrite(v.data(), sizeof(T), n, f) == n);
}
template <class T>
bool get_vec(FILE* f, std::vector<T>& v) {
    uint64_t n = 0;
    if (fread(&n, 8, 1, f) != 1 || n > ((uint64_t)1 << 32)) return false;
    v.resize(n);
    return n == 0 || fread(v.data(), sizeof(T), n, f) == n;
}
}  // namespace

// =============================================================================================
extern "C" {

const char* pfg_last_error(void) { return g_err.c_str(); }
int32_t pfg_abi_version(void) { return PFG_ABI_VERSION; }

pfg_status pfg_derive_reps(int64_t n, int32_t d, int32_t family, uint64_t budget, const pfg_build_opts* opts,
                           int32_t* reps_out, uint64_t* min_budget_out, uint64_t* index_bytes_out) {
    Geo g;
    PFG_TRY(resolve_opts(opts, n, d, family, g));
    if (min_budget_out) *min_budget_out = g.fixed_bytes + g.per_rep_bytes;
    pfg_status s = derive_L(g, budget, opts ? opts->reps_override : 0);
    if (s != PFG_OK) return s;
    if (reps_out) *reps_out = g.L;
    if (index_bytes_out) *index_bytes_out = g.index_bytes;
    return PFG_OK;
}

pfg_status pfg_build(const float* data, int64_t n, int32_t d, uint64_t budget, int32_t family, uint64_t seed,
                     const pfg_build_opts* opts, void* stream, pfg_index** out) {
    if (!out) return fail(PFG_E_ARG, "out is NULL");
    *out = nullptr;
    if (!data) return fail(PFG_E_ARG, "data is NULL");
    std::unique_ptr<pfg_index> I(new pfg_index());
    PFG_TRY(resolve_opts(opts, n, d, family, I->g));
    PFG_TRY(derive_L(I->g, budget, opts ? opts->reps_override : 0));
    Geo& g = I->g;
    I->seed = seed;
    cudaStream_t st = (cudaStream_t)stream;
    PFG_CUDA(cudaGetDevice(&I->device));
    PFG_CUDA(cudaDeviceGetAttribute(&I->num_sms, cudaDevAttrMultiProcessorCount, I->device));
    // a1: normalise the data into index memory
    {
        DBuf raw;
        const float* src = data;
        if (!is_device_ptr(data)) {
            PFG_TRY(raw.alloc((size_t)n * d * 4, "data copy"));
            PFG_CUDA(cudaMemcpyAsync(raw.p, data, (size_t)n * d * 4, cudaMemcpyHostToDevice, st));
            src = raw.as<float>();
        }
        PFG_TRY(I->x.alloc((size_t)n * g.dpad * 4, "data"));
        DBuf zm;
        PFG_TRY(zm.alloc(8, "zmin"));
        int64_t zrow = -1;
        PFG_TRY(normalize_rows(src, n, d, I->x.as<float>(), g.dpad, nullptr, zm.as<unsigned long long>(), &zrow, st));
        if (zrow >= 0) return fail(PFG_E_ZERO_VECTOR, "data row " + std::to_string(zrow) + " is a zero vector");
    }
    // a2: functions
    PFG_TRY(gen_functions(I.get(), st));
    // a4: per-point sketches (transient: their slot words are stored inline in the tables, R-21)
    DBuf skp;
    if (g.M > 0) {
        PFG_TRY(skp.alloc((size_t)n * g.M * 8, "sketches"));
        hp_bits(I->x.as<float>(), n, g.dpad, I->skfn.as<float>(), 64 * g.M, g.dpad, g.dpad, skp.as<uint8_t>(),
                (int64_t)g.M * 8, st);
        PFG_CUDA(cudaGetLastError());
    }
    // a3 + a5: hash, sort and tabulate the repetitions in batches
    PFG_TRY(I->tab.alloc((size_t)g.L * n * 16, "tables"));
    PFG_TRY(I->pt.alloc((size_t)g.L * 8193 * 4, "prefix tables"));
    {
        const int64_t budget_keys = (int64_t)1 << 28;  // 2 GiB of keys per batch
        const int Rb = (int)std::max<int64_t>(1, std::min<int64_t>(g.L, budget_keys / n));
        DBuf keys, sorted, bits, poolvals, temp;
        PFG_TRY(keys.alloc((size_t)Rb * n * 8, "build keys"));
        PFG_TRY(sorted.alloc((size_t)n * 8, "sorted keys"));
        size_t temp_bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, temp_bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)n, 32,
                                       32 + g.K, st);
        PFG_TRY(temp.alloc(temp_bytes, "sort temp"));
        bool pool_ready = false;
        for (int r0 = 0; r0 < g.L; r0 += Rb) {
            const int nb = std::min(Rb, g.L - r0);
            PFG_TRY(hash_reps(I.get(), I->x.as<float>(), n, r0, nb, keys.as<uint64_t>(), nullptr, 0, bits, poolvals,
                              pool_ready, st));
            for (int r = 0; r < nb; ++r) {
                const int j = r0 + r;
                size_t tb = temp.bytes;
                PFG_CUDA(cub::DeviceRadixSort::SortKeys(temp.p, tb, keys.as<uint64_t>() + (size_t)r * n, sorted.as<uint64_t>(),
                                                        (int)n, 32, 32 + g.K, st));
                k_entries<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(sorted.as<uint64_t>(), n, skp.as<uint64_t>(), g.M,
                                                                      I->slot_h[j], I->tab.as<uint64_t>() + (size_t)j * n * 2);
                k_prefix<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(sorted.as<uint64_t>(), n, g.K,
                                                                         I->pt.as<uint32_t>() + (size_t)j * 8193);
                PFG_CUDA(cudaGetLastError());
            }
        }
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    if (g.family == PFG_CROSSPOLYTOPE_FHT) PFG_TRY(build_cp_table(I.get(), st));
    if (g.family == PFG_CROSSPOLYTOPE) build_cp_exact_table(I.get());
    if (g.storage == PFG_STORAGE_I16) {
        // R-25: the search's inner products read 16-bit fixed-point rows; the fp32 rows stay for
        // the fp32 re-rank of each query's top-k
        PFG_TRY(I->x16.alloc((size_t)n * g.dpad16 * 2, "int16 data"));
        const int64_t tot = n * (int64_t)g.dpad16;
        k_quantize<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(I->x.as<float>(), n, g.dpad, g.d, I->x16.as<int16_t>(),
                                                                 g.dpad16);
        PFG_CUDA(cudaGetLastError());
        PFG_CUDA(cudaStreamSynchronize(st));
    }
    PFG_CUDA(cudaStreamSynchronize(st));
    *out = I.release();
    return PFG_OK;
}

pfg_status pfg_search(pfg_index* I, const float* queries, int64_t nq, int32_t k, float recall, const pfg_search_opts* opts,
                      int64_t* out_ids, float* out_sims, pfg_query_stats* stats, void* stream) {
    if (!I) return fail(PFG_E_ARG, "index is NULL");
    if (nq > 0 && (!queries || !out_ids || !out_sims)) return fail(PFG_E_ARG, "NULL queries or outputs");
    if (nq < 0 || nq >= (int64_t(1) << 31)) return fail(PFG_E_ARG, "nq must be in [0, 2^31)");
    if (k < 1 || k > kMaxK) return fail(PFG_E_ARG, "k must be in [1, 256]");
    if (!(recall > 0.0f && recall <= 1.0f)) return fail(PFG_E_ARG, "recall target must be in (0, 1]");
    SearchCfg s;
    PFG_TRY(resolve_sopts(opts, s));
    if (nq == 0) return PFG_OK;
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    // the search runs on the index's highest-priority stream, after the caller's stream, and the
    // caller's stream waits for its end (ev_done): the round kernels (the critical path) are
    // scheduled before the side streams' hashing, which fills the SMs they leave
    const cudaStream_t ust = (cudaStream_t)stream;
    cudaStream_t st = ust;
    PFG_TRY(ensure_streams(I));
    if (PFG_HIPRIO) {
        PFG_CUDA(cudaEventRecord(I->ev_in, ust));
        PFG_CUDA(cudaStreamWaitEvent(I->hst, I->ev_in, 0));
        st = I->hst;
    }
    const Geo& g = I->g;
    if (!I->ev_done) PFG_CUDA(cudaEventCreateWithFlags(&I->ev_done, cudaEventDisableTiming));
    if (I->done_pending) {
        // the previous search may still run (calls return without waiting): order this one after
        // it on the GPU, and take its stop-depth histogram if it is already complete
        PFG_CUDA(cudaStreamWaitEvent(st, I->ev_done, 0));
        if (cudaEventQuery(I->ev_done) == cudaSuccess) {
            I->done_pending = false;
            tune_eager(I);

        } else {
            cudaGetLastError();
        }
    }
    std::shared_ptr<DBuf> thr, taub;
    PFG_TRY(get_thr(I, recall, s, thr, nullptr));
    PFG_TRY(get_tau(I, s.tau_rule, s.eps, recall, taub, nullptr));
    if (s.timing) {
        for (auto& e : I->ev)
            if (!e) PFG_CUDA(cudaEventCreate(&e));
        PFG_CUDA(cudaEventRecord(I->ev[0], st));
    }
    I->tl_on = s.timing == 4;
    I->tl_n = 0;
    tl_mark(I, "start", st);
    I->launches = 0;
    bool lazy = false;
    // rounds 0 and 1 reach repetitions [0, 1 + R) only (R-17 default schedule): the codes and
    // ranges of the later eager repetitions are computed beside them
    const int split = (s.engine == 0 && !s.uniform && g.strategy != PFG_TENSOR) ? 1 + s.R : 0;
    // exact CP (independent): hash only the repetitions the blind rounds can reach; the fused
    // kernel's queries get the rest in bulk after them (not with the device-side loop, which may
    // run any query to the end)
    int cp_eager = 0;
    if (g.family == PFG_CROSSPOLYTOPE && g.strategy == PFG_INDEPENDENT && s.engine == 0 && s.wide <= 0 && !I->loop_heavy &&
        s.loop_max == 0) {
        const int mr = s.rounds > 0 ? s.rounds : 5;
        const int64_t reach = s.uniform ? (int64_t)s.R * mr : 1 + (int64_t)s.R * (mr - 1);
        const int64_t e = std::min<int64_t>(g.L, std::max<int64_t>(reach, I->eager));
        cp_eager = e < g.L ? (int)e : 0;
    }
    if (s.ext.codes) {
        const bool lz = g.family == PFG_CROSSPOLYTOPE_FHT && g.strategy == PFG_INDEPENDENT;
        if (s.ext.reps > g.L || (!lz && s.ext.reps != g.L))
            return fail(PFG_E_ARG, "ext_reps must be L (<= L for the FHT cross-polytope family, independent functions)");
        if (!is_device_ptr(s.ext.codes) || (s.ext.sk && !is_device_ptr(s.ext.sk)))
            return fail(PFG_E_ARG, "ext_codes / ext_sketches must be device pointers");
        cp_eager = 0;
    }
    if (s.ext.sk && g.M == 0) return fail(PFG_E_ARG, "ext_sketches given for an index without sketches");
    PFG_TRY(prep_queries(I, queries, nq, true, false, nullptr, &lazy, st, s.ext.codes ? 0 : split, cp_eager,
                         s.ext.codes || s.ext.sk ? &s.ext : nullptr));

    const int k_eff = (int)std::min<int64_t>(k, g.n);
    const int kt = ((k_eff + 31) / 32) * 32;
    const int smem_warp = warp_smem_bytes(g.dpad, g.M, kt);
    const size_t smem = (size_t)smem_warp * 4;
    const int epl = lazy ? epl_of(g) : 1;
    int occ = 1;
    switch (epl) {
        case 1: occ = query_occupancy<1>(smem); break;
        case 2: occ = query_occupancy<2>(smem); break;
        case 4: occ = query_occupancy<4>(smem); break;
        case 8: occ = query_occupancy<8>(smem); break;
        case 16: occ = query_occupancy<16>(smem); break;
        default: occ = query_occupancy<32>(smem); break;
    }
    const int64_t max_blocks = (int64_t)I->num_sms * occ;
    const int64_t slots = max_blocks * 4;
    const int64_t bm_words = (g.n + 31) / 32;
    if (slots > I->slots || bm_words != I->slots_bm) {
        PFG_TRY(I->bitmap.alloc((size_t)slots * bm_words * 4, "bitmaps"));
        PFG_TRY(I->claims.alloc((size_t)slots * kClaimCap * 4, "claims"));
        PFG_CUDA(cudaMemsetAsync(I->bitmap.p, 0, (size_t)slots * bm_words * 4, st));
        I->slots = slots;
        I->slots_bm = bm_words;
    }
    PFG_TRY(I->cur.ensure((size_t)nq * g.L * 16, "cursors"));
    const bool rounds = (s.engine == 0 || s.engine == 2) && g.strategy != PFG_TENSOR;  // tensor shells: the fused kernel
    // round engine: `rounds` bulk rounds (search option, default 5), then the fused kernel resumes
    // every query still running (stragglers keep their hash set in shared memory across chunks
    // there, instead of paying a round's fixed latency per chunk).  The rounds are enqueued
    // without host synchronisation.
    const int max_rounds = s.rounds > 0 ? s.rounds : 5;
    const int ecap = 2048;  // evaluated-list stride: kHMax committed + one batch of slack
    constexpr int ccap = 8192;  // emitted positions of one query's chunk (more: the fused kernel takes it)
    static_assert(ccap / kTile <= 64, "k_dedupe holds a chunk's tile counts in two words per lane");
    const uint32_t pool_cap = (uint32_t)std::min<int64_t>(std::max<int64_t>(1 << 20, nq * 1024), (int64_t)1 << 30);
    int64_t wide_max = 0;   // visit-tag arrays this search may use
    bool want_wide = false;
    bool chunk_eng = false; // the chunk engine (kernels_chunk.cuh): engine 2, unless wide queries are on
    if (rounds) {
        const size_t N = (size_t)nq;
        PFG_TRY(I->rs_lvl.ensure(N * 4, "rs")); PFG_TRY(I->rs_c0.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_flags.ensure(N * 4, "rs")); PFG_TRY(I->rs_tn.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_cnt.ensure(N * kCnt * 4, "rs")); PFG_TRY(I->rs_T.ensure(N * kt * 8, "rs"));
        PFG_TRY(I->rs_E.ensure(N * ecap * 4, "rs")); PFG_TRY(I->rs_pend.ensure(N * kMaxR * 16, "rs"));
        PFG_TRY(I->rs_repcnt.ensure(N * kMaxR * 3 * 4, "rs"));
        // two pools (one per round parity: the chunk engine merges the previous round's pool while
        // it fills the next)
        PFG_TRY(I->rs_pool_id.ensure((size_t)pool_cap * 8, "pool")); PFG_TRY(I->rs_pool_q.ensure((size_t)pool_cap * 8, "pool"));
        PFG_TRY(I->rs_pool_key.ensure((size_t)pool_cap * 16, "pool"));
        PFG_TRY(I->rs_ctl.ensure(2 * sizeof(RoundCtl), "rs control")); PFG_TRY(I->rs_poff.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_pn.ensure(N * 4, "rs")); PFG_TRY(I->rs_act0.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_act1.ensure(N * 4, "rs")); PFG_TRY(I->rs_fused.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_cand.ensure(N * ccap * 4, "rs candidates"));
        PFG_TRY(I->rs_hsave.ensure(N * kHC * 4, "rs hash sets"));
        PFG_TRY(I->rs_tcnt.ensure(N * (ccap / kTile) * 4, "rs tile counts"));
        PFG_TRY(I->rs_dord0.ensure(N * 4, "rs")); PFG_TRY(I->rs_dord1.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_rinfo.ensure(N * 16, "rs")); PFG_TRY(I->rs_tiles.ensure(N * (ccap / kTile) * 32, "rs tiles"));
        PFG_TRY(I->rs_fused2.ensure(N * 4, "rs")); PFG_TRY(I->rs_wslot.ensure(N * 4, "rs"));
        PFG_TRY(I->rs_rtile.ensure(N * (kMaxR + 1) * 4, "rs"));
        if (!I->h_ctl) {
            PFG_CUDA(cudaMallocHost(&I->h_ctl, sizeof(RoundCtl)));
            std::memset(I->h_ctl, 0, sizeof(RoundCtl));
        }
        PFG_TRY(ensure_streams(I));
        if (!I->ev_split) {
            PFG_CUDA(cudaEventCreateWithFlags(&I->ev_split, cudaEventDisableTiming));
            PFG_CUDA(cudaEventCreateWithFlags(&I->ev_f1, cudaEventDisableTiming));
        }
        // wide queries (kernels_rounds.cuh): visit-tag arrays (n words each, PFG_WIDE_MIB of them
        // at most, default 8 GiB) and wide scan tiles, sized grow-only from what the previous
        // search wanted; visit s = (K - i) L + j + 1 must fit 16 bits
        const int64_t per = 4 * g.n;
        wide_max = std::max<int64_t>(1, ((int64_t)8192 << 20) / per);
        if (s.wide_arrays > 0) wide_max = std::min<int64_t>(wide_max, s.wide_arrays);
        // wide queries: on when asked for (wide > 0, or the developer knob PFG_LOOP_MAX), else
        // automatic: on iff the previous search's queries were heavy (loop_heavy); off, a query
        // beyond the hash set goes to the fused kernel's bitmap mode (and nothing is allocated)
        want_wide = (s.wide > 0 || (s.wide == 0 && (I->loop_heavy || s.loop_max > 0))) &&
                    (int64_t)(g.K + 1) * g.L < 65536;
        if (s.engine == 2 && !want_wide) chunk_eng = true;
        if (want_wide) {
            const int64_t smax = wide_max;
            const int64_t want = std::min<int64_t>(smax, std::max<int64_t>(I->wv_want, std::max<int64_t>(1, (512ll << 20) / per)));
            if (want > I->wv_slots || I->wv_n != g.n) {
                PFG_TRY(I->rs_wv.alloc((size_t)want * per, "visit tags"));
                PFG_CUDA(cudaMemsetAsync(I->rs_wv.p, 0xff, (size_t)want * per, st));
                I->wv_slots = want;
                I->wv_n = g.n;
                I->wepoch = 0;
            }
            const int64_t wmin = (int64_t)s.R * ((g.n + kTile - 1) / kTile + 2);
            // (wide_tiles_min: the minimum, so that wide chunks compete and defer)
            const int64_t wc0 = s.wide_tiles_min ? 0 : (int64_t)1 << 18;
            const int64_t wc = std::max<int64_t>(wmin, std::max<int64_t>(I->wc_want, wc0));
            if (wc > I->wc_cap || (s.wide_tiles_min && wc != I->wc_cap)) {
                PFG_TRY(I->rs_wtiles.alloc((size_t)wc * 32, "wide tiles"));
                PFG_TRY(I->rs_wcand.alloc((size_t)wc * kTile * 4, "wide candidates"));
                PFG_TRY(I->rs_wsim.alloc((size_t)wc * kTile * 4, "wide similarities"));
                PFG_TRY(I->rs_wtcnt.alloc((size_t)wc * 4, "wide tile counts"));
                I->wc_cap = wc;
            }
            if (++I->wepoch >= 0xFFFEu) {
                PFG_CUDA(cudaMemsetAsync(I->rs_wv.p, 0xff, (size_t)I->wv_slots * per, st));
                I->wepoch = 1;
            }
        }
    }
    PFG_TRY(I->work.ensure(16, "work counters"));
    PFG_CUDA(cudaMemsetAsync(I->work.p, 0, 16, st));
    // two round pipelines (pipelines = 2): the lower and the upper half of the batch run as two
    // searches of their own on st and st1, each kernel with half the resident grid, meant to overlap
    // one half's latency-bound control phases with the other half's candidate-row reads.  Measured
    // slower on config 2 (1.89 vs 1.84 ms/step): the halves fall into lock-step
    // and k_sims at half its grid leaves HBM under-used.  Not with wide queries / the device-side
    // loop (the loop graph is per search) or exact CP's partial eager hashing.
    const int64_t lmax_cfg = s.loop_max > 0 ? s.loop_max : (I->loop_heavy ? 1 : 0);
    const bool halves = rounds && !chunk_eng && s.engine == 0 && !want_wide && lmax_cfg == 0 && cp_eager == 0 &&
                        s.pipelines == 2 && nq >= 2;

    const bool ids_dev = is_device_ptr(out_ids), sims_dev = is_device_ptr(out_sims);
    const bool stats_dev = stats ? is_device_ptr(stats) : true;
    const bool trace_dev = s.trace_cap > 0 ? is_device_ptr(s.trace_ids) : true;
    int64_t* d_ids = out_ids;
    float* d_sims = out_sims;
    pfg_query_stats* d_stats = stats;
    uint32_t* d_trace = s.trace_ids;
    if (!ids_dev) { PFG_TRY(I->outb_ids.ensure((size_t)nq * k * 8, "ids")); d_ids = I->outb_ids.as<int64_t>(); }
    if (!sims_dev) { PFG_TRY(I->outb_sims.ensure((size_t)nq * k * 4, "sims")); d_sims = I->outb_sims.as<float>(); }
    if (stats && !stats_dev) { PFG_TRY(I->outb_stats.ensure((size_t)nq * sizeof(pfg_query_stats), "stats")); d_stats = I->outb_stats.as<pfg_query_stats>(); }
    if (s.trace_cap > 0 && !trace_dev) { PFG_TRY(I->outb_trace.ensure((size_t)nq * s.trace_cap * 4, "trace")); d_trace = I->outb_trace.as<uint32_t>(); }

    QueryParams p;
    std::memset(&p, 0, sizeof(p));
    p.n = g.n; p.nq = nq; p.bm_words = bm_words; p.id_offset = g.id_offset;
    p.d = g.d; p.dpad = g.dpad; p.K = g.K; p.L = g.L; p.M = g.M; p.B = s.B; p.R = s.R; p.k = k; p.k_eff = k_eff;
    p.per_round = s.per_round; p.use_filter = (s.use_filter && g.M > 0) ? 1 : 0; p.c = g.c; p.ell = g.ell; p.dp = g.dp;
    p.lazy = lazy ? 1 : 0; p.claim_cap = kClaimCap; p.trace_cap = s.trace_cap; p.kt = kt; p.smem_warp = smem_warp;
    p.uniform = s.uniform;
    p.tensor_s = g.strategy == PFG_TENSOR ? g.S : 0;
    p.lstep = g.strategy == PFG_TENSOR ? 2 * g.ell : 1;
    p.x = I->x.as<float>(); p.tab = I->tab.as<Entry>(); p.pt = I->pt.as<uint32_t>();
    if (g.storage == PFG_STORAGE_I16) {
        p.x16 = I->x16.as<int16_t>();
        p.qx16 = I->qx16.as<int16_t>();
        p.dpad16 = g.dpad16;
    }
    p.slot = I->slot.as<uint8_t>(); p.qx = I->qx.as<float>(); p.qsk = I->qsk.as<uint64_t>();
    p.qcodes = I->qcodes.as<uint32_t>(); p.qc_n = I->qc_n; p.qc_ld = I->qc_ld;
    p.sg = I->sg.as<uint32_t>(); p.qzero = I->qzero.as<uint8_t>();
    p.thr = thr->as<float>(); p.taub = taub->as<float>(); p.work = I->work.as<unsigned long long>();
    p.cur = I->cur.as<uint4>(); p.bitmap = I->bitmap.as<uint32_t>(); p.claims = I->claims.as<uint32_t>();
    p.out_ids = d_ids; p.out_sims = d_sims; p.stats = stats ? d_stats : nullptr; p.trace_ids = d_trace;
    // level-K match ranges of the first repetitions, one thread per (query, repetition)
    // (SimHash and pool strategies hash all L repetitions eagerly; their ranges are precomputed
    // for the repetitions most queries reach, the tuned eager depth)
    p.qb_n = lazy ? std::min(I->qc_n, kQBMax) : std::min(I->qc_n, I->qb_depth);
    PFG_TRY(I->jhist.ensure(kJHist * 4, "stop histogram"));
    if (!I->h_jhist) PFG_CUDA(cudaMallocHost(&I->h_jhist, kJHist * 4));
    PFG_CUDA(cudaMemsetAsync(I->jhist.p, 0, kJHist * 4, st));
    p.jhist = I->jhist.as<uint32_t>();
    p.qb_ld = std::max(1, I->qc_ld);
    if (p.qb_n > 0) {
        PFG_TRY(I->qbnd.ensure((size_t)nq * p.qb_ld * 16, "query bounds"));
        p.qbnd = I->qbnd.as<uint4>();
        const int bm = I->mid_pending ? std::min(p.qb_n, 1) : -1;   // st: [0, bm); aux2: [bm, b0) (ev_mid)
        const int b0 = std::min(p.qb_n, I->late_pending ? I->qc_split : p.qb_n);
        const int bs = bm >= 0 ? bm : b0;
        const int64_t thr_n = nq * (int64_t)bs;
        const cudaStream_t sq = I->hst_pending ? I->hst : st;
        if (bs > 0) k_qbounds<<<(unsigned)((thr_n + 255) / 256), 256, 0, sq>>>(p, I->qbnd.as<uint4>(), nullptr, nq, 0, bs, nullptr);
        tl_mark(I, "k_qbounds", sq);
        if (bm >= 0 && bm < b0) {
            const int64_t thr_m = nq * (int64_t)(b0 - bm);
            k_qbounds<<<(unsigned)((thr_m + 255) / 256), 256, 0, I->aux2>>>(p, I->qbnd.as<uint4>(), nullptr, nq, bm, b0 - bm,
                                                                          nullptr);
            I->launches += 1;
            tl_mark(I, "k_qbounds (mid)", I->aux2);
        }
        if (I->mid_pending) PFG_CUDA(cudaEventRecord(I->ev_mid, I->aux2));
        if (I->late_pending && I->late_ne > I->qc_split) {
            PFG_TRY(fht_codes(I, nq, nullptr, I->qc_split, I->late_ne - I->qc_split, I->qc_ld, I->aux2));
            I->late_ne = 0;
        }
        if (b0 < p.qb_n) {
            const int64_t thr_l = nq * (int64_t)(p.qb_n - b0);
            k_qbounds<<<(unsigned)((thr_l + 255) / 256), 256, 0, I->aux2>>>(p, I->qbnd.as<uint4>(), nullptr, nq, b0,
                                                                          p.qb_n - b0, nullptr);
            I->launches += 1;
            tl_mark(I, "k_qbounds (late)", I->aux2);
        }
        PFG_CUDA(cudaGetLastError());
        I->launches += 1;
    } else if (I->mid_pending) {
        PFG_CUDA(cudaEventRecord(I->ev_mid, I->aux2));
    }
    if (I->late_pending && I->late_ne > I->qc_split) {
        PFG_TRY(fht_codes(I, nq, nullptr, I->qc_split, I->late_ne - I->qc_split, I->qc_ld, I->aux2));
        I->late_ne = 0;
    }
    if (I->late_pending) PFG_CUDA(cudaEventRecord(I->ev_late, I->aux2));
    if (I->hst_pending) {
        // repetition 0's codes and ranges, from the highest-priority stream
        PFG_CUDA(cudaEventRecord(I->ev_hst, I->hst));
        PFG_CUDA(cudaStreamWaitEvent(st, I->ev_hst, 0));
        I->hst_pending = false;
    }
    // developer instrumentation: PFG_PHASE_PROF=1 prints per-phase warp cycles of each search to stderr
    // timing = 5 (developer): per-phase cycle counters of the fused kernel (and of k_chunk in a
    // -DPFG_CHUNK_PROF=1 build), printed to stderr
    const bool phase_prof = s.timing == 5;
    DBuf profb;
    if (phase_prof) {
        PFG_TRY(profb.alloc(32 * 8, "phase profile"));
        PFG_CUDA(cudaMemsetAsync(profb.p, 0, 256, st));
        p.prof = profb.as<unsigned long long>();
    }
    if (!rounds) {
        PFG_TRY(join_sketches(I, st));
        PFG_TRY(late_join(I, st));
    }
    if (s.timing) PFG_CUDA(cudaEventRecord(I->ev[1], st));
    int64_t fused_n = nq;
    if (rounds) {
        RoundState& r = p.rs;
        r.lvl = I->rs_lvl.as<int32_t>(); r.c0 = I->rs_c0.as<int32_t>(); r.flags = I->rs_flags.as<int32_t>();
        r.tn = I->rs_tn.as<int32_t>(); r.cnt = I->rs_cnt.as<uint32_t>(); r.T = I->rs_T.as<uint64_t>();
        r.E = I->rs_E.as<uint32_t>(); r.pend = I->rs_pend.as<uint4>(); r.repcnt = I->rs_repcnt.as<uint32_t>();
        r.pool_id = I->rs_pool_id.as<uint32_t>(); r.pool_q = I->rs_pool_q.as<uint32_t>();
        r.pool_key = I->rs_pool_key.as<uint64_t>();
        r.ctl = I->rs_ctl.as<RoundCtl>();
        r.poff = I->rs_poff.as<uint32_t>(); r.pn = I->rs_pn.as<uint32_t>();
        r.act[0] = I->rs_act0.as<uint32_t>(); r.act[1] = I->rs_act1.as<uint32_t>(); r.fused = I->rs_fused.as<uint32_t>();
        r.Ecap = ecap; r.Ccap = ccap; r.pool_cap = pool_cap;
        r.cand = I->rs_cand.as<uint32_t>(); r.hsave = I->rs_hsave.as<uint32_t>();
        r.tcnt = I->rs_tcnt.as<uint32_t>();
        r.dord[0] = I->rs_dord0.as<uint32_t>(); r.dord[1] = I->rs_dord1.as<uint32_t>(); r.rinfo = I->rs_rinfo.as<uint4>();
        r.tiles = I->rs_tiles.as<uint4>();
        r.fused2 = I->rs_fused2.as<uint32_t>();
        r.wslot = I->rs_wslot.as<uint32_t>();
        r.rtile = I->rs_rtile.as<uint32_t>();
        const bool wide_on = want_wide && I->wv_slots > 0 && I->wv_n == g.n;
        r.wv = wide_on ? I->rs_wv.as<uint32_t>() : nullptr;
        r.wslots = wide_on ? (uint32_t)std::min<int64_t>(I->wv_slots, wide_max) : 0u;
        r.wtiles = I->rs_wtiles.as<uint4>(); r.wcand = I->rs_wcand.as<uint32_t>(); r.wsim = I->rs_wsim.as<float>();
        r.wtcnt = I->rs_wtcnt.as<uint32_t>();
        r.wcap = wide_on ? (uint32_t)I->wc_cap : 0u;
        r.hmax = s.wide > 0 ? (uint32_t)s.wide : (uint32_t)kHMax;
        r.pool_stride = chunk_eng ? pool_cap : 0u;
        PFG_CUDA(cudaMemsetAsync(r.ctl, 0, 2 * sizeof(RoundCtl), st));
        if (!halves) {
            k_rinit<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(p, (uint32_t)(0xFFFEu - I->wepoch) << 16);
            I->launches += 1;
        }
        PFG_CUDA(cudaGetLastError());
    }
    if (chunk_eng) {
        // the chunk engine: per round k_chunk (CTA per query: merge, expand, scan, dedupe) and
        // k_sims; a merge-only pass; the fused kernel for the queries still running
        RoundState& r = p.rs;
        const size_t csm = (size_t)chunk_smem_bytes(kt, g.dpad, lazy);
        const void* kfn = epl == 1 ? (const void*)k_chunk<1> : epl == 2 ? (const void*)k_chunk<2> : epl == 4 ? (const void*)k_chunk<4>
                        : epl == 8 ? (const void*)k_chunk<8> : epl == 16 ? (const void*)k_chunk<16> : (const void*)k_chunk<32>;
        PFG_CUDA(set_smem(kfn, csm));
        int cocc = 1;
        PFG_CUDA(occupancy(&cocc, kfn, kCT, csm));
        const unsigned cb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nq, (int64_t)I->num_sms * std::max(1, cocc)));
        const unsigned sb = (unsigned)(I->num_sms * PFG_SIMS_MINB);
        const bool tm = s.timing == 2;
        const bool ksims_timed = s.timing == 3;
        auto launch_chunk = [&](int par, int mode) -> pfg_status {
            switch (epl) {
                case 1: k_chunk<1><<<cb, kCT, csm, st>>>(p, par, mode); break;
                case 2: k_chunk<2><<<cb, kCT, csm, st>>>(p, par, mode); break;
                case 4: k_chunk<4><<<cb, kCT, csm, st>>>(p, par, mode); break;
                case 8: k_chunk<8><<<cb, kCT, csm, st>>>(p, par, mode); break;
                case 16: k_chunk<16><<<cb, kCT, csm, st>>>(p, par, mode); break;
                default: k_chunk<32><<<cb, kCT, csm, st>>>(p, par, mode); break;
            }
            PFG_CUDA(cudaGetLastError());
            PFG_TRY(dbg_sync("k_chunk"));
            tl_mark(I, mode ? "k_chunk (merge only)" : "k_chunk", st);
            I->launches += 1;
            return PFG_OK;
        };
        int round = 0;
        for (; round < max_rounds; ++round) {
            // round 0 is the single repetition 0 with tau = 64 (no sketches read); round 1 reaches
            // repetitions < 1 + R; later rounds may reach every eager repetition
            if (round == 1) { PFG_TRY(join_sketches(I, st)); PFG_TRY(mid_join(I, st)); }
            if (round == 2) PFG_TRY(late_join(I, st));
            const int par = round & 1;
            PFG_TRY(phase_mark(I, tm, kPhExpand, st));
            PFG_TRY(launch_chunk(par, 0));
            PFG_TRY(phase_mark(I, tm, kPhSims, st));
            const bool kt_ = ksims_timed;
            if (kt_) {
                if ((int64_t)I->kev.size() < 2 * (I->kev_n + 1)) {
                    if (I->kev_n >= 512) PFG_TRY(fold_kernel_timing(I));
                    while ((int64_t)I->kev.size() < 2 * (I->kev_n + 1)) {
                        cudaEvent_t e;
                        PFG_CUDA(cudaEventCreate(&e));
                        I->kev.push_back(e);
                    }
                }
                PFG_CUDA(cudaEventRecord(I->kev[2 * I->kev_n], st));
            }
            if (g.storage == PFG_STORAGE_I16) k_sims<QueryParams, true><<<sb, 256, 0, st>>>(p, par, 3);
            else k_sims<QueryParams, false><<<sb, 256, 0, st>>>(p, par, 3);
            PFG_CUDA(cudaGetLastError());
            if (kt_) PFG_CUDA(cudaEventRecord(I->kev[2 * I->kev_n++ + 1], st));
            PFG_TRY(dbg_sync("k_sims"));
            tl_mark(I, "k_sims", st);
            I->launches += 1;
        }
        PFG_TRY(join_sketches(I, st));
        PFG_TRY(late_join(I, st));
        PFG_TRY(phase_mark(I, tm, kPhMerge, st));
        PFG_TRY(launch_chunk(round & 1, 1));
        PFG_TRY(phase_mark(I, tm, kPhOther, st));
        p.qlist = r.fused;
        p.nq_dev = &r.ctl->nfused;
        p.resume = 1;
        // the queries the fused kernel resumes get codes and match ranges for kExtReps more
        // repetitions in bulk (they would otherwise hash and search them one warp at a time)
        if (cp_eager > 0) {
            const int f0 = cp_eager * g.c, nf = (g.L - cp_eager) * g.c;
            PFG_TRY(I->qfc2.ensure((size_t)nq * nf * 2, "cp function codes (resumed queries)"));
            PFG_TRY(cp_values(I, I->qx.as<float>(), nq, r.fused, &r.ctl->nfused, f0, nf, I->qfc2.as<uint16_t>(), st));
            k_pool_codes<<<dim3((unsigned)((nq + 255) / 256), (unsigned)(g.L - cp_eager)), 256, 0, st>>>(
                I->qfc2.as<uint16_t>(), nq, nf, cp_eager, g.L - cp_eager, g.c, g.ell, g.K, I->sel.as<int32_t>(), nullptr,
                I->qcodes.as<uint32_t>(), g.L, r.fused, &r.ctl->nfused, f0);
            PFG_CUDA(cudaGetLastError());
            I->launches += 2;
            p.qc_n = g.L;
        }
        if (lazy && I->qc_n > 0 && I->qc_ld > I->qc_n && p.qb_n == I->qc_n) {
            const int r0 = I->qc_n, nr = I->qc_ld - I->qc_n;
            PFG_TRY(fht_codes(I, nq, r.fused, r0, nr, I->qc_ld, st, &r.ctl->nfused));
            const int64_t thr_n = nq * (int64_t)nr;
            k_qbounds<<<list_grid(I, thr_n, nr), 256, 0, st>>>(p, I->qbnd.as<uint4>(), r.fused, nq, r0, nr,
                                                                     &r.ctl->nfused);
            PFG_CUDA(cudaGetLastError());
            I->launches += 2;
            p.qc_n = p.qb_n = I->qc_ld;
        }
        I->last_rounds = round;
    } else if (rounds) {
        RoundState& r = p.rs;
        const size_t esm = (size_t)expand_smem_bytes(g.dpad, lazy) * 4;
        const size_t dsm = (size_t)align16((int)sizeof(DedupeSmem)) * 4;
        const size_t msm = (size_t)(align16((int)sizeof(MergeSmem)) + 2 * align16(kt * 8)) * 4;
        PFG_CUDA(set_smem((const void*)k_merge<QueryParams, false>, msm));
        PFG_CUDA(set_smem((const void*)k_merge<QueryParams, true>, msm));
        PFG_CUDA(set_smem((const void*)k_dedupe<QueryParams>, dsm));
        PFG_CUDA(set_smem((const void*)k_merge<const QueryParams*, true>, msm));
        PFG_CUDA(set_smem((const void*)k_dedupe<const QueryParams*>, dsm));

        int docc = 1;
        PFG_CUDA(occupancy(&docc, (const void*)k_dedupe<QueryParams>, 128, dsm));
        // grids: warp per active query (at most one resident wave; the kernels stride over the
        // device-side counts, so no host synchronisation is needed between rounds)
        const unsigned qb_e = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nq + 3) / 4, (int64_t)I->num_sms * 16));
        const unsigned qb_d = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nq + 3) / 4, (int64_t)I->num_sms * std::max(1, docc)));
        const unsigned qb_m = qb_e;   // (the loop graph's key)
        const unsigned tb_s = (unsigned)(I->num_sms * 8);
        const unsigned sb = (unsigned)(I->num_sms * PFG_SIMS_MINB);
        int round = 0;
        const bool tm = s.timing == 2;
        const bool ksims_timed = s.timing == 3;
        // one round: expand, scan, dedupe, sims, merge of list `par` (phase events unless captured)
        // blind: a round outside the captured loop (counted in sims_rows_blind, timed with timing = 3);
        // m: the queries of the pipeline (grid sizes)
        // share = 2 (two round pipelines): every grid is half of what stays resident, so that the
        // other pipeline's kernel of another phase finds registers and shared memory beside it
        int occ_e = 1, occ_s = 1, occ_m = 1;
        PFG_CUDA(occupancy(&occ_e, (const void*)k_expand<1, QueryParams>, 128, esm));
        PFG_CUDA(occupancy(&occ_s, (const void*)k_scan<QueryParams, false>, 256, 0));
        PFG_CUDA(occupancy(&occ_m, (const void*)k_merge<QueryParams, false>, 128, msm));
        auto launch_round = [&](int par, cudaStream_t rst, bool marks, auto pp, bool blind, int64_t m, int share,
                                bool lz = true, bool dd = true) -> pfg_status {
            using PP = decltype(pp);
            // the round's kernels start while their predecessor drains (programmatic dependent
            // launch; each waits in pdl_wait), outside the captured loop graph
            auto go = [&](auto kern, unsigned grid, unsigned block, size_t sm, auto... args) -> cudaError_t {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(block);
                cfg.dynamicSmemBytes = sm;
                cfg.stream = rst;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                if (blind && PFG_PDL) { cfg.attrs = at; cfg.numAttrs = 1; }
                return cudaLaunchKernelEx(&cfg, kern, args...);
            };
            const int64_t qw = (m + 3) / 4, ns = I->num_sms;
            const unsigned qb_e = (unsigned)std::max<int64_t>(1, std::min<int64_t>(qw, share > 1 ? ns * std::max(1, occ_e / share) : ns * 16));
            const unsigned qb_d = (unsigned)std::max<int64_t>(1, std::min<int64_t>(qw, ns * std::max(1, docc / share)));
            const unsigned qb_m = share > 1 ? (unsigned)std::max<int64_t>(1, std::min<int64_t>(qw, ns * std::max(1, occ_m / share))) : qb_e;
            const unsigned tb_s = share > 1 ? (unsigned)(ns * std::max(1, occ_s / share)) : (unsigned)(ns * 8);
            const unsigned sb = (unsigned)(ns * std::max(1, PFG_SIMS_MINB / share));
            PFG_TRY(phase_mark(I, marks, kPhExpand, rst));
            if (!lz && std::is_same<PP, QueryParams>::value) {
                // every repetition this round can reach has its code: no lazy hashing compiled in
                PFG_CUDA(go(k_expand<1, PP, false>, qb_e, 128, esm, pp, par, lazy ? 1 : 0));
            } else {
                switch (epl) {
                    case 1: PFG_CUDA(go(k_expand<1, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                    case 2: PFG_CUDA(go(k_expand<2, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                    case 4: PFG_CUDA(go(k_expand<4, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                    case 8: PFG_CUDA(go(k_expand<8, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                    case 16: PFG_CUDA(go(k_expand<16, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                    default: PFG_CUDA(go(k_expand<32, PP>, qb_e, 128, esm, pp, par, lazy ? 1 : 0)); break;
                }
            }
            if (blind) { PFG_TRY(dbg_sync("k_expand")); tl_mark(I, "k_expand", rst); }
            PFG_TRY(phase_mark(I, marks, kPhScan, rst));
            if (r.wslots > 0 || !std::is_same<PP, QueryParams>::value) PFG_CUDA(go(k_scan<PP, true>, tb_s, 256, 0, pp, par));
            else PFG_CUDA(go(k_scan<PP, false>, tb_s, 256, 0, pp, par));
            if (blind) { PFG_TRY(dbg_sync("k_scan")); tl_mark(I, "k_scan", rst); }
            PFG_TRY(phase_mark(I, marks, kPhDedupe, rst));
            // dd = false: the search's first round of single-repetition chunks (tau = 64, nothing
            // evaluated yet), where every query is a direct chunk or handed off and k_dedupe has no work
            if (dd) PFG_CUDA(go(k_dedupe<PP>, qb_d, 128, dsm, pp, par));
            if (blind) { PFG_TRY(dbg_sync("k_dedupe")); tl_mark(I, "k_dedupe", rst); }
            PFG_TRY(phase_mark(I, marks, kPhSims, rst));
            const bool kt = ksims_timed && blind;
            if (kt) {
                if ((int64_t)I->kev.size() < 2 * (I->kev_n + 1)) {
                    // fold the pairs recorded so far (all earlier on this stream) before reusing them
                    if (I->kev_n >= 512) PFG_TRY(fold_kernel_timing(I));
                    while ((int64_t)I->kev.size() < 2 * (I->kev_n + 1)) {
                        cudaEvent_t e;
                        PFG_CUDA(cudaEventCreate(&e));
                        I->kev.push_back(e);
                    }
                }
                PFG_CUDA(cudaEventRecord(I->kev[2 * I->kev_n], rst));
            }
            const int sflags = blind ? 2 : 0;
            if (g.storage == PFG_STORAGE_I16) PFG_CUDA(go(k_sims<PP, true>, sb, 256, 0, pp, par, sflags));
            else PFG_CUDA(go(k_sims<PP, false>, sb, 256, 0, pp, par, sflags));
            if (kt) PFG_CUDA(cudaEventRecord(I->kev[2 * I->kev_n++ + 1], rst));
            if (r.wslots > 0 || !std::is_same<PP, QueryParams>::value) {
                // wide tiles of the round (tag checks, compaction, similarities)
                if (g.storage == PFG_STORAGE_I16) PFG_CUDA(go(k_wsims<PP, true>, sb, 256, 0, pp, par));
                else PFG_CUDA(go(k_wsims<PP, false>, sb, 256, 0, pp, par));
            }
            if (blind) { PFG_TRY(dbg_sync("k_sims")); tl_mark(I, "k_sims", rst); }
            PFG_TRY(phase_mark(I, marks, kPhMerge, rst));
            if (r.wslots > 0 || !std::is_same<PP, QueryParams>::value) PFG_CUDA(go(k_merge<PP, true>, qb_m, 128, msm, pp, par));
            else PFG_CUDA(go(k_merge<PP, false>, qb_m, 128, msm, pp, par));
            if (blind) { PFG_TRY(dbg_sync("k_merge")); tl_mark(I, "k_merge", rst); }
            PFG_TRY(phase_mark(I, marks, kPhOther, rst));
            PFG_CUDA(cudaGetLastError());
            return PFG_OK;
        };
        if (halves) {
            // two round pipelines: queries [0, n0) on st, [n0, nq) on st1, each a search of its own
            // (pipeline_params); the fused kernel of each takes its stragglers with half the grid
            const int64_t n0 = nq / 2;
            const int64_t qh0[2] = {0, n0}, nh[2] = {n0, nq - n0};
            const int64_t slots_h = (max_blocks / 2) * 4;
            const QueryParams ph[2] = {pipeline_params(p, 0, n0, 0, slots_h), pipeline_params(p, n0, nq - n0, 1, slots_h)};
            const cudaStream_t sh[2] = {st, I->st1};
            for (int h = 0; h < 2; ++h)
                k_rinit<<<(unsigned)((nh[h] + 255) / 256), 256, 0, st>>>(ph[h], (uint32_t)(0xFFFEu - I->wepoch) << 16);
            PFG_CUDA(cudaGetLastError());
            I->launches += 2;
            PFG_CUDA(cudaEventRecord(I->ev_h1start, st));
            PFG_CUDA(cudaStreamWaitEvent(I->st1, I->ev_h1start, 0));
            // the side streams' joins, on both pipelines' streams
            auto join_both = [&](bool late) -> pfg_status {
                const bool mp = I->mid_pending, lp = I->late_pending;
                for (int h = 0; h < 2; ++h) {
                    I->mid_pending = mp;
                    I->late_pending = lp;
                    PFG_TRY(join_sketches(I, sh[h]));
                    PFG_TRY(late ? late_join(I, sh[h]) : mid_join(I, sh[h]));
                }
                return PFG_OK;
            };
            for (; round < max_rounds; ++round) {
                if (round == 1) PFG_TRY(join_both(false));
                if (round == 2) PFG_TRY(join_both(true));
                for (int h = 0; h < 2; ++h) PFG_TRY(launch_round(round & 1, sh[h], tm && h == 0, ph[h], true, nh[h], 2));
                I->launches += 10;
            }
            PFG_TRY(join_both(true));
            const int P = round & 1;
            for (int h = 0; h < 2; ++h) {
                const cudaStream_t hs = sh[h];
                const QueryParams& q = ph[h];
                k_presplit<<<1, 1, 0, hs>>>(q, P);
                k_split<<<(unsigned)((nh[h] + 255) / 256), 256, 0, hs>>>(q, P, 64u, 0u);
                PFG_CUDA(cudaGetLastError());
                I->launches += 2;
                QueryParams p1 = q;
                p1.qlist = q.rs.fused;
                p1.nq_dev = &q.rs.ctl->nfused;
                p1.resume = 1;
                if (lazy && I->qc_n > 0 && I->qc_ld > I->qc_n && p.qb_n == I->qc_n) {
                    const int r0 = I->qc_n, nr = I->qc_ld - I->qc_n;
                    PFG_TRY(fht_codes(I, nh[h], q.rs.fused, r0, nr, I->qc_ld, hs, &q.rs.ctl->nfused, qh0[h]));
                    const int64_t thr_n = nh[h] * (int64_t)nr;
                    k_qbounds<<<list_grid(I, thr_n, nr), 256, 0, hs>>>(p1, I->qbnd.as<uint4>() + qh0[h] * p.qb_ld,
                                                                            q.rs.fused, nh[h], r0, nr, &q.rs.ctl->nfused);
                    PFG_CUDA(cudaGetLastError());
                    I->launches += 2;
                    p1.qc_n = p1.qb_n = I->qc_ld;
                }
                PFG_CUDA(cudaMemsetAsync(p1.work, 0, 8, hs));
                const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((nh[h] + 3) / 4, max_blocks / 2));
                switch (epl) {
                    case 1: PFG_TRY(launch_query_t<1>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                    case 2: PFG_TRY(launch_query_t<2>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                    case 4: PFG_TRY(launch_query_t<4>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                    case 8: PFG_TRY(launch_query_t<8>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                    case 16: PFG_TRY(launch_query_t<16>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                    default: PFG_TRY(launch_query_t<32>(p1, (int)blocks, smem, hs, I->num_sms)); break;
                }
                I->launches += 1;
                PFG_TRY(dbg_sync("fused (pipeline)"));
                tl_mark(I, h ? "k_query (fused, pipeline 1)" : "k_query (fused, pipeline 0)", hs);
            }
            PFG_CUDA(cudaEventRecord(I->ev_h1end, I->st1));
            PFG_CUDA(cudaStreamWaitEvent(st, I->ev_h1end, 0));
            k_ctl_fold<<<1, 1, 0, st>>>(r.ctl);
            PFG_CUDA(cudaGetLastError());
            I->launches += 1;
            fused_n = 0;
            I->last_rounds = round;
        } else {
        const int qb_n0 = p.qb_n;   // (the fused tail extends the codes of its own list from here)
        while (round < max_rounds) {
            // round 0 is the single repetition 0 with tau = 64 (no sketches read); round 1 reaches
            // repetitions < 1 + R; later rounds may reach every eager repetition
            if (round == 1) { PFG_TRY(join_sketches(I, st)); PFG_TRY(mid_join(I, st)); }
            if (round == 2) PFG_TRY(late_join(I, st));
            // the largest repetition this round can reach (one chunk per round; a level's chunks
            // restart at repetition 0)
            const int64_t reach = s.uniform ? (int64_t)s.R * (round + 1) : 1 + (int64_t)s.R * round;
            if (round >= 3 && reach > p.qc_n && lazy && I->qc_n > 0 && I->qc_ld > I->qc_n && p.qb_n == I->qc_n) {
                // the few queries still running after three rounds: codes and level-K ranges of the
                // next kExtReps repetitions in bulk (one thread per query and repetition) instead of
                // one lane group per query inside k_expand; the fused tail reuses them
                RoundState& r = p.rs;
                const int par = round & 1, r0 = I->qc_n, nr = I->qc_ld - I->qc_n;
                PFG_TRY(fht_codes(I, nq, r.act[par], r0, nr, I->qc_ld, st, &r.ctl->nact[par]));
                const int64_t thr_n = nq * (int64_t)nr;
                k_qbounds<<<list_grid(I, thr_n, nr), 256, 0, st>>>(p, I->qbnd.as<uint4>(), r.act[par], nq, r0, nr,
                                                                         &r.ctl->nact[par]);
                PFG_CUDA(cudaGetLastError());
                I->launches += 2;
                p.qc_n = p.qb_n = I->qc_ld;
            }
            const bool dd = !(round == 0 && !s.uniform);
            PFG_TRY(launch_round(round & 1, st, tm, p, true, nq, 1, !(reach <= p.qc_n), dd));
            I->launches += dd ? 5 : 4;
            ++round;
        }
        PFG_TRY(join_sketches(I, st));
        PFG_TRY(late_join(I, st));
        // no host synchronisation from here on: the queries still running are split on the device
        // between the device-side round loop and the fused kernel (k_split), whose first launch
        // runs on the aux stream beside the loop
        const int P = round & 1;
        const uint32_t lmin = s.loop_min > 0 ? (uint32_t)s.loop_min : 64u;
        // default: the loop keeps only the wide queries (a query beyond the hash set early in the
        // search), unless the previous search's queries were heavy (loop_heavy); queries that are
        // merely long run faster in the fused kernel (measured)
        const uint32_t lmax = s.loop_max > 0 ? (uint32_t)s.loop_max : (I->loop_heavy ? 0xffffffffu : 0u);
        const bool loop_on = r.wslots > 0 || lmax > 0;
        const unsigned gq = (unsigned)((nq + 255) / 256);
        k_presplit<<<1, 1, 0, st>>>(p, P);
        k_split<<<gq, 256, 0, st>>>(p, P, lmin, lmax);
        PFG_CUDA(cudaGetLastError());
        PFG_TRY(dbg_sync("k_split"));
        I->launches += 2;
        PFG_CUDA(cudaEventRecord(I->ev_split, st));
        PFG_CUDA(cudaStreamWaitEvent(I->aux, I->ev_split, 0));
        {
            QueryParams p1 = p;
            p1.qlist = r.fused;
            p1.nq_dev = &r.ctl->nfused;
            p1.resume = 1;
            // the queries the fused kernel resumes get codes and match ranges for kExtReps more
            // repetitions in bulk (they would otherwise hash and search them one warp at a time)
            if (cp_eager > 0) {
                // exact CP: the codes of repetitions [cp_eager, L) for the queries the fused kernel
                // resumes (it cannot hash CP functions itself)
                const int f0 = cp_eager * g.c, nf = (g.L - cp_eager) * g.c;
                PFG_TRY(I->qfc2.ensure((size_t)nq * nf * 2, "cp function codes (resumed queries)"));
                PFG_TRY(cp_values(I, I->qx.as<float>(), nq, r.fused, &r.ctl->nfused, f0, nf, I->qfc2.as<uint16_t>(), I->aux));
                k_pool_codes<<<dim3((unsigned)((nq + 255) / 256), (unsigned)(g.L - cp_eager)), 256, 0, I->aux>>>(
                    I->qfc2.as<uint16_t>(), nq, nf, cp_eager, g.L - cp_eager, g.c, g.ell, g.K, I->sel.as<int32_t>(), nullptr,
                    I->qcodes.as<uint32_t>(), g.L, r.fused, &r.ctl->nfused, f0);
                PFG_CUDA(cudaGetLastError());
                I->launches += 2;
                p1.qc_n = g.L;
            }
            // (every query handed to the fused kernel, also those handed off before round 3)
            if (lazy && I->qc_n > 0 && I->qc_ld > I->qc_n && qb_n0 == I->qc_n) {
                const int r0 = I->qc_n, nr = I->qc_ld - I->qc_n;
                PFG_TRY(fht_codes(I, nq, r.fused, r0, nr, I->qc_ld, I->aux, &r.ctl->nfused));
                const int64_t thr_n = nq * (int64_t)nr;
                k_qbounds<<<list_grid(I, thr_n, nr), 256, 0, I->aux>>>(p1, I->qbnd.as<uint4>(), r.fused, nq, r0,
                                                                              nr, &r.ctl->nfused);
                PFG_CUDA(cudaGetLastError());
                I->launches += 2;
                p1.qc_n = p1.qb_n = I->qc_ld;
            }
            PFG_CUDA(cudaMemsetAsync(I->work.p, 0, 8, I->aux));
            const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((nq + 3) / 4, max_blocks));
            switch (epl) {
                case 1: PFG_TRY(launch_query_t<1>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
                case 2: PFG_TRY(launch_query_t<2>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
                case 4: PFG_TRY(launch_query_t<4>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
                case 8: PFG_TRY(launch_query_t<8>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
                case 16: PFG_TRY(launch_query_t<16>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
                default: PFG_TRY(launch_query_t<32>(p1, (int)blocks, smem, I->aux, I->num_sms)); break;
            }
            I->launches += 1;
            PFG_TRY(dbg_sync("fused 1"));
            tl_mark(I, "k_query (fused, beside the loop)", I->aux);
            PFG_CUDA(cudaEventRecord(I->ev_f1, I->aux));
        }
        // the device-side loop: a CUDA graph whose WHILE node runs two rounds per iteration
        // (lists P^1 then P) while loop_more holds (kernels_rounds.cuh); built once per launch
        // configuration
        PFG_TRY(phase_mark(I, tm, kPhLoop, st));
        if (loop_on) {
            // the loop's kernels read the search's parameters from device memory (k_setp), so the
            // graph depends only on the launch geometry
            const uint32_t cap = (uint32_t)std::min<int64_t>(1 << 30, 8 * (int64_t)(g.K + 1) * g.L + 64);
            PFG_TRY(I->rs_params.ensure(sizeof(QueryParams), "loop parameters"));
            const QueryParams* dp = I->rs_params.as<QueryParams>();
            k_setp<<<1, 1, 0, st>>>(p, I->rs_params.as<QueryParams>());
            PFG_CUDA(cudaGetLastError());
            std::vector<unsigned char> key(96);
            const int64_t extra[12] = {P, lmin, cap, epl, (int64_t)qb_e << 32 | qb_d, (int64_t)qb_m << 32 | tb_s,
                                       (int64_t)sb << 32 | (lazy ? 1 : 0), (int64_t)esm << 40 | (int64_t)dsm << 20 | (int64_t)msm,
                                       (int64_t)(uintptr_t)dp, (int64_t)(uintptr_t)r.ctl, 0, 0};
            std::memcpy(key.data(), extra, sizeof(extra));
            if (!I->loop_exec || key != I->loop_key) {
                if (I->loop_exec) { cudaGraphExecDestroy(I->loop_exec); I->loop_exec = nullptr; }
                if (!I->cap_st) PFG_CUDA(cudaStreamCreateWithFlags(&I->cap_st, cudaStreamNonBlocking));
                cudaGraph_t gr;
                PFG_CUDA(cudaGraphCreate(&gr, 0));
                cudaGraphConditionalHandle h;
                PFG_CUDA(cudaGraphConditionalHandleCreate(&h, gr, 0, 0));
                PFG_CUDA(cudaStreamBeginCaptureToGraph(I->cap_st, gr, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
                k_loop_begin<<<1, 1, 0, I->cap_st>>>(r.ctl, P ^ 1, h, lmin);
                PFG_CUDA(cudaStreamEndCapture(I->cap_st, &gr));
                size_t nn = 1;
                cudaGraphNode_t n0;
                PFG_CUDA(cudaGraphGetNodes(gr, &n0, &nn));
                cudaGraphNodeParams cp = {};
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = h;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t cn;
                PFG_CUDA(cudaGraphAddNode(&cn, gr, &n0, 1, &cp));
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                PFG_CUDA(cudaStreamBeginCaptureToGraph(I->cap_st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
                pfg_status ls = launch_round(P ^ 1, I->cap_st, false, dp, false, nq, 1);
                if (ls == PFG_OK) ls = launch_round(P, I->cap_st, false, dp, false, nq, 1);
                k_loop_cond<<<1, 1, 0, I->cap_st>>>(r.ctl, P ^ 1, h, lmin, cap);
                cudaGraph_t body_out = body;
                const cudaError_t ce = cudaStreamEndCapture(I->cap_st, &body_out);
                if (ls != PFG_OK) { cudaGraphDestroy(gr); return ls; }
                if (ce != cudaSuccess) { cudaGraphDestroy(gr); PFG_CUDA(ce); }
                const cudaError_t ie = cudaGraphInstantiate(&I->loop_exec, gr, 0);
                cudaGraphDestroy(gr);
                PFG_CUDA(ie);
                I->loop_key = key;
            }
            PFG_CUDA(cudaGraphLaunch(I->loop_exec, st));
            PFG_TRY(dbg_sync("round loop graph"));
            I->launches += 1;
        }
        if (loop_on) {
            k_loop_end<<<gq, 256, 0, st>>>(p, P ^ 1);
            PFG_CUDA(cudaGetLastError());
            PFG_TRY(dbg_sync("k_loop_end"));
            I->launches += 1;
        }
        // the fused kernel's first launch (beside the loop) ends here; a second launch takes the
        // queries the loop handed off (only when the loop keeps non-wide queries, PFG_LOOP_MAX)
        PFG_TRY(phase_mark(I, tm, kPhFused, st));
        PFG_CUDA(cudaStreamWaitEvent(st, I->ev_f1, 0));
        p.qlist = r.fused2;
        p.nq_dev = &r.ctl->nfused2;
        p.resume = 1;
        if (lmax == 0) fused_n = 0;
        I->last_rounds = round;
        }
    }
    PFG_TRY(join_sketches(I, st));
    PFG_TRY(late_join(I, st));
    if (fused_n > 0) {
        PFG_TRY(phase_mark(I, s.timing == 2, kPhFused, st));
        PFG_CUDA(cudaMemsetAsync(I->work.p, 0, 8, st));
        const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((fused_n + 3) / 4, max_blocks));  // rounds: nq bound
        switch (epl) {
            case 1: PFG_TRY(launch_query_t<1>(p, (int)blocks, smem, st, I->num_sms)); break;
            case 2: PFG_TRY(launch_query_t<2>(p, (int)blocks, smem, st, I->num_sms)); break;
            case 4: PFG_TRY(launch_query_t<4>(p, (int)blocks, smem, st, I->num_sms)); break;
            case 8: PFG_TRY(launch_query_t<8>(p, (int)blocks, smem, st, I->num_sms)); break;
            case 16: PFG_TRY(launch_query_t<16>(p, (int)blocks, smem, st, I->num_sms)); break;
            default: PFG_TRY(launch_query_t<32>(p, (int)blocks, smem, st, I->num_sms)); break;
        }
        I->launches += 1;
    }
    I->last_fused = fused_n;
    if (g.storage == PFG_STORAGE_I16 && s.rerank) {
        // the fixed-point search's top-k re-scored with fp32 rows (R-2 order), re-sorted
        const size_t rsm = (size_t)4 * align16(kt * 8);
        PFG_CUDA(set_smem((const void*)k_rerank, rsm));
        k_rerank<<<(unsigned)((nq + 3) / 4), 128, rsm, st>>>(p.x, p.qx, g.dpad, nq, k, k_eff, kt, g.id_offset, d_ids, d_sims);
        PFG_CUDA(cudaGetLastError());
        I->launches += 1;
        tl_mark(I, "k_rerank", st);
    }
    tl_mark(I, "end", st);
    PFG_TRY(phase_mark(I, s.timing == 2, kPhEnd, st));
    if (s.timing) PFG_CUDA(cudaEventRecord(I->ev[2], st));
    I->timing_pending = s.timing;
    if (!ids_dev) PFG_CUDA(cudaMemcpyAsync(out_ids, d_ids, (size_t)nq * k * 8, cudaMemcpyDeviceToHost, st));
    if (!sims_dev) PFG_CUDA(cudaMemcpyAsync(out_sims, d_sims, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, st));
    if (stats && !stats_dev)
        PFG_CUDA(cudaMemcpyAsync(stats, d_stats, (size_t)nq * sizeof(pfg_query_stats), cudaMemcpyDeviceToHost, st));
    if (s.trace_cap > 0 && !trace_dev)
        PFG_CUDA(cudaMemcpyAsync(s.trace_ids, d_trace, (size_t)nq * s.trace_cap * 4, cudaMemcpyDeviceToHost, st));
    // the stop-depth histogram for the next search's eager depth, and the end-of-search event that
    // orders the next search's use of the scratch buffers (on any stream)
    PFG_CUDA(cudaMemcpyAsync(I->h_jhist, I->jhist.p, kJHist * 4, cudaMemcpyDeviceToHost, st));
    if (rounds) {
        if (!I->h_ctl2) {
            PFG_CUDA(cudaMallocHost(&I->h_ctl2, 2 * sizeof(RoundCtl)));
            std::memset(I->h_ctl2, 0, 2 * sizeof(RoundCtl));
        }
        PFG_CUDA(cudaMemcpyAsync(I->h_ctl2 + (I->nsearch & 1), I->rs_ctl.p, sizeof(RoundCtl), cudaMemcpyDeviceToHost, st));
        I->nq_prev[I->nsearch & 1] = nq;
        ++I->nsearch;
    }
    PFG_CUDA(cudaEventRecord(I->ev_done, st));
    if (st != ust) PFG_CUDA(cudaStreamWaitEvent(ust, I->ev_done, 0));
    I->done_pending = true;
    // with device outputs the call returns without waiting for the GPU; host outputs (or the
    // developer phase print) need the results here
    const bool host_out = !ids_dev || !sims_dev || (stats && !stats_dev) || (s.trace_cap > 0 && !trace_dev);
    if (host_out || phase_prof) PFG_CUDA(cudaStreamSynchronize(st));
    tl_print(I);
    if (phase_prof) {
        if (rounds) {
            PFG_CUDA(cudaMemcpy(I->h_ctl, I->rs_ctl.p, sizeof(RoundCtl), cudaMemcpyDeviceToHost));
            const RoundCtl* c = reinterpret_cast<const RoundCtl*>(I->h_ctl);
            fused_n = (int64_t)c->nfused + c->nfused2;
            fprintf(stderr, "[pfg phase] loop: %u rounds, wide arrays used %u of %lld, wide deferrals %u, fused beside the loop %u, after it %u\n",
                    c->round, c->wnext, (long long)I->wv_slots, c->wdefer, c->nfused, c->nfused2);
        }
        fprintf(stderr, "[pfg phase] engine %d: rounds %d, queries finished by the fused kernel %lld of %lld\n", s.engine,
                I->last_rounds, (long long)fused_n, (long long)nq);
        unsigned long long h[32] = {0};
        PFG_CUDA(cudaMemcpy(h, profb.p, 256, cudaMemcpyDeviceToHost));
        if (h[22])
            fprintf(stderr, "[pfg phase] k_chunk per query (thread-0 cycles): merge %.0f, expand %.0f, scan+dedupe %.0f, "
                    "pool %.0f, scheduling %.0f; %.0f query-rounds\n", (double)h[16] / h[22], (double)h[17] / h[22],
                    (double)h[18] / h[22], (double)h[19] / h[22], (double)h[23] / h[22], (double)h[22]);
        if (h[14])
            fprintf(stderr, "[pfg phase] collect per query-chunk: rebuild %.0f, codes+bounds %.0f, scan %.0f, epilogue %.0f cycles; "
                    "max %.0f cycles; %.0f chunks, mean emitted %.1f, max emitted %llu\n",
                    (double)h[8] / h[14], (double)h[9] / h[14], (double)h[10] / h[14], (double)h[11] / h[14], (double)h[12],
                    (double)h[14], (double)h[13] / h[14], h[15]);
        const double tot = (double)(h[0] + h[1] + h[2] + h[3] + h[4]);
        fprintf(stderr, "[pfg phase] Mcycles: bounds %.1f (%.0f%%) scan-load %.1f (%.0f%%) claim %.1f (%.0f%%) drain %.1f (%.0f%%, sims %.1f) lazy-hash %.1f (%.0f%%)\n",
                h[0] / 1e6, 100 * h[0] / tot, h[1] / 1e6, 100 * h[1] / tot, h[2] / 1e6, 100 * h[2] / tot,
                h[3] / 1e6, 100 * h[3] / tot, h[5] / 1e6, h[4] / 1e6, 100 * h[4] / tot);
    }
    I->last_launches = I->launches;
    PFG_CUDA(cudaEventSynchronize(I->ev_zmin));  // recorded right after the normalisation
    if (rounds && I->nsearch >= 2) {
        // the previous search is complete (it precedes this one's normalisation on the stream):
        // size the wide-query scratch of the next searches from what it wanted
        const RoundCtl* c = I->h_ctl2 + ((I->nsearch - 2) & 1);
        if ((int64_t)c->wnext > I->wv_slots) I->wv_want = std::max<int64_t>(I->wv_want, 2 * (int64_t)c->wnext);
        if (c->wdefer) I->wc_want = std::min<int64_t>((int64_t)1 << 22, std::max<int64_t>(I->wc_want, 2 * I->wc_cap));
        // heavy queries (bytes a query reads: evaluated rows + emitted table entries, averaged over
        // the previous search) run faster in the bulk rounds than one warp each in the fused kernel
        const int64_t nprev = std::max<int64_t>(1, I->nq_prev[(I->nsearch - 2) & 1]);
        const double bytes = ((double)c->evsum * g.dpad * 4 + (double)c->emsum * 16) / (double)nprev;
        I->loop_heavy = bytes >= 64.0 * (1 << 20);
    }
    if (*I->h_zmin != ~0ull)
        return fail(PFG_E_ZERO_VECTOR, "query row " + std::to_string(*I->h_zmin) + " is a zero vector");
    return PFG_OK;
}

// the timing events of the last search, read once it has completed (calls return early)
static pfg_status collect_timing(pfg_index* I) {
    if (!I->timing_pending) return PFG_OK;
    PFG_CUDA(cudaEventSynchronize(I->ev[2]));
    PFG_CUDA(cudaEventElapsedTime(&I->last_ms[0], I->ev[0], I->ev[1]));
    PFG_CUDA(cudaEventElapsedTime(&I->last_ms[1], I->ev[1], I->ev[2]));
    PFG_CUDA(cudaEventElapsedTime(&I->last_ms[2], I->ev[0], I->ev[2]));
    if (I->timing_pending == 2) PFG_TRY(phase_collect(I));
    I->timing_pending = 0;
    return PFG_OK;
}

pfg_status pfg_last_phases(const pfg_index* I, float* ms, int32_t n) {
    if (!I || !ms || n < 0) return fail(PFG_E_ARG, "NULL index or output");
    pfg_index* W = const_cast<pfg_index*>(I);
    std::lock_guard<std::mutex> lock(W->mu);
    PFG_TRY(collect_timing(W));
    for (int i = 0; i < n && i < 8; ++i) ms[i] = I->last_phase_ms[i];
    return PFG_OK;
}

pfg_status pfg_kernel_timing(pfg_index* I, int32_t kernel, int32_t reset, double* ms, int64_t* launches) {
    if (!I) return fail(PFG_E_ARG, "NULL index");
    if (kernel != 0) return fail(PFG_E_ARG, "kernel must be 0 (k_sims)");
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    PFG_TRY(fold_kernel_timing(I));
    if (ms) *ms = I->kev_ms;
    if (launches) *launches = I->kev_launches;
    if (reset) { I->kev_ms = 0.0; I->kev_launches = 0; }
    return PFG_OK;
}

pfg_status pfg_round_stats(pfg_index* I, uint64_t* out, int32_t n) {
    if (!I || !out || n < 0) return fail(PFG_E_ARG, "NULL index or output");
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    if (I->nsearch == 0 || !I->h_ctl2) return fail(PFG_E_STATE, "no round-engine search yet");
    if (I->ev_done) PFG_CUDA(cudaEventSynchronize(I->ev_done));
    const RoundCtl* c = I->h_ctl2 + ((I->nsearch - 1) & 1);
    const uint64_t v[7] = {c->sims_rows, (uint64_t)I->last_rounds, c->round, c->nfused, c->nfused2, c->wnext,
                           c->sims_rows_blind};
    for (int i = 0; i < n && i < 7; ++i) out[i] = v[i];
    return PFG_OK;
}

pfg_status pfg_last_timing(const pfg_index* I, float* ms3, int32_t* launches) {
    if (!I) return fail(PFG_E_ARG, "NULL index");
    pfg_index* W = const_cast<pfg_index*>(I);
    std::lock_guard<std::mutex> lock(W->mu);
    PFG_TRY(collect_timing(W));
    if (ms3) for (int i = 0; i < 3; ++i) ms3[i] = I->last_ms[i];
    if (launches) *launches = I->last_launches;
    return PFG_OK;
}

pfg_status pfg_merge_topk(const int64_t* ids, const float* sims, int32_t world, int64_t nq, int32_t k, int64_t* out_ids,
                          float* out_sims, void* stream) {
    if (!ids || !sims || !out_ids || !out_sims) return fail(PFG_E_ARG, "NULL pointer");
    if (world < 1 || k < 1 || nq < 0) return fail(PFG_E_ARG, "world, k must be >= 1");
    if ((int64_t)world * k > 4096) return fail(PFG_E_ARG, "world * k must be <= 4096");
    if (nq == 0) return PFG_OK;
    if (!is_device_ptr(ids) || !is_device_ptr(sims) || !is_device_ptr(out_ids) || !is_device_ptr(out_sims))
        return fail(PFG_E_ARG, "pfg_merge_topk takes device pointers");
    const size_t smem = (size_t)4 * world * k * 16;
    cudaStream_t st = (cudaStream_t)stream;
    PFG_CUDA(set_smem((const void*)k_merge_topk, smem));
    k_merge_topk<<<(unsigned)((nq + 3) / 4), 128, smem, st>>>(ids, sims, world, nq, k, out_ids, out_sims);
    PFG_CUDA(cudaGetLastError());
    return PFG_OK;
}

pfg_status pfg_index_info(const pfg_index* I, pfg_index_info_t* out) {
    if (!I || !out) return fail(PFG_E_ARG, "NULL pointer");
    const Geo& g = I->g;
    std::memset(out, 0, sizeof(*out));
    out->n = g.n; out->d = g.d; out->d_pad = g.dpad; out->family = g.family; out->strategy = g.strategy;
    out->prefix_bits = g.K; out->reps = g.L; out->ell = g.ell; out->funcs_per_rep = g.c; out->sketch_words = g.M;
    out->pool_funcs = g.m; out->fht_dim = g.dp; out->device = I->device;
    out->index_bytes = g.index_bytes;
    out->scratch_bytes = I->cur.bytes + I->bitmap.bytes + I->claims.bytes;
    out->seed = I->seed; out->id_offset = g.id_offset;
    return PFG_OK;
}

pfg_status pfg_export(const pfg_index* Ic, int32_t what, int32_t arg, void* dst, uint64_t bytes) {
    pfg_index* I = const_cast<pfg_index*>(Ic);
    if (!I || !dst) return fail(PFG_E_ARG, "NULL pointer");
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    const Geo& g = I->g;
    auto copy = [&](const void* src, uint64_t need) -> pfg_status {
        if (bytes != need) return fail(PFG_E_ARG, "dst_bytes must be " + std::to_string(need));
        PFG_CUDA(cudaMemcpy(dst, src, need, cudaMemcpyDeviceToHost));
        return PFG_OK;
    };
    switch (what) {
        case PFG_EXPORT_TABLE:
            if (arg < 0 || arg >= g.L) return fail(PFG_E_ARG, "rep out of range");
            return copy(I->tab.as<uint64_t>() + (size_t)arg * g.n * 2, (uint64_t)g.n * 16);
        case PFG_EXPORT_PREFIX:
            if (arg < 0 || arg >= g.L) return fail(PFG_E_ARG, "rep out of range");
            return copy(I->pt.as<uint32_t>() + (size_t)arg * 8193, 8193ull * 4);
        case PFG_EXPORT_SKETCH:
            return fail(PFG_E_STATE, "per-point sketches are not retained: each repetition table stores its slot's "
                                     "sketch word inline (PFG_EXPORT_TABLE)");
        case PFG_EXPORT_DATA16: {
            if (g.storage != PFG_STORAGE_I16) return fail(PFG_E_STATE, "index stores fp32 rows (PFG_EXPORT_DATA)");
            if (bytes != (uint64_t)g.n * g.d * 2) return fail(PFG_E_ARG, "dst_bytes must be n*d*2");
            PFG_CUDA(cudaMemcpy2D(dst, (size_t)g.d * 2, I->x16.p, (size_t)g.dpad16 * 2, (size_t)g.d * 2, (size_t)g.n,
                                  cudaMemcpyDeviceToHost));
            return PFG_OK;
        }
        case PFG_EXPORT_DATA: {
            if (!I->x.p) return fail(PFG_E_STATE, "index holds no fp32 rows");
            if (bytes != (uint64_t)g.n * g.d * 4) return fail(PFG_E_ARG, "dst_bytes must be n*d*4");
            PFG_CUDA(cudaMemcpy2D(dst, (size_t)g.d * 4, I->x.p, (size_t)g.dpad * 4, (size_t)g.d * 4, (size_t)g.n,
                                  cudaMemcpyDeviceToHost));
            return PFG_OK;
        }
        case PFG_EXPORT_CP:
            if (I->cpT.empty()) return fail(PFG_E_STATE, "index has no CP table (SimHash family)");
            if (bytes != I->cpT.size() * 8) return fail(PFG_E_ARG, "dst_bytes must be (ell+1)*41*8");
            std::memcpy(dst, I->cpT.data(), bytes);
            return PFG_OK;
        case PFG_EXPORT_SLOTS:
            if (bytes != (uint64_t)g.L * 4) return fail(PFG_E_ARG, "dst_bytes must be L*4");
            std::memcpy(dst, I->slot_h.data(), bytes);
            return PFG_OK;
        case PFG_EXPORT_POOLSEL:
            if (g.strategy == PFG_INDEPENDENT) return fail(PFG_E_STATE, "index has no function selections");
            if (bytes != I->sel_h.size() * 4) return fail(PFG_E_ARG, "dst_bytes must be L*c*4");
            std::memcpy(dst, I->sel_h.data(), bytes);
            return PFG_OK;
        default:
            return fail(PFG_E_ARG, "unknown export");
    }
}

pfg_status pfg_hash_queries(pfg_index* I, const float* queries, int64_t nq, uint32_t* out_codes, uint64_t* out_sketches,
                            void* stream) {
    if (!I || !queries) return fail(PFG_E_ARG, "NULL pointer");
    if (nq < 1) return fail(PFG_E_ARG, "nq must be >= 1");
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    cudaStream_t st = (cudaStream_t)stream;
    const Geo& g = I->g;
    int64_t zrow = -1;
    bool lazy = false;
    PFG_TRY(prep_queries(I, queries, nq, out_codes != nullptr, true, &zrow, &lazy, st, 0));
    PFG_TRY(join_sketches(I, st));
    if (zrow >= 0) return fail(PFG_E_ZERO_VECTOR, "query row " + std::to_string(zrow) + " is a zero vector");
    if (out_codes) {
        const size_t b = (size_t)nq * g.L * 4;
        PFG_CUDA(cudaMemcpyAsync(out_codes, I->qcodes.p, b, is_device_ptr(out_codes) ? cudaMemcpyDeviceToDevice
                                                                                   : cudaMemcpyDeviceToHost, st));
    }
    if (out_sketches && g.M > 0) {
        const size_t b = (size_t)nq * g.M * 8;
        PFG_CUDA(cudaMemcpyAsync(out_sketches, I->qsk.p, b, is_device_ptr(out_sketches) ? cudaMemcpyDeviceToDevice
                                                                                        : cudaMemcpyDeviceToHost, st));
    }
    PFG_CUDA(cudaStreamSynchronize(st));
    return PFG_OK;
}

pfg_status pfg_hash_queries_reps(pfg_index* I, const float* queries, int64_t nq, int32_t nreps, uint32_t* out_codes,
                                 uint64_t* out_sketches, void* stream) {
    if (!I || !queries || !out_codes) return fail(PFG_E_ARG, "NULL pointer");
    if (nq < 1) return fail(PFG_E_ARG, "nq must be >= 1");
    if (nreps < 1 || nreps > I->g.L) return fail(PFG_E_ARG, "nreps must be in [1, L]");
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    cudaStream_t st = (cudaStream_t)stream;
    const Geo& g = I->g;
    int64_t zrow = -1;
    bool lazy = false;
    PFG_TRY(prep_queries(I, queries, nq, false, true, &zrow, &lazy, st, 0));
    PFG_TRY(join_sketches(I, st));
    if (zrow >= 0) return fail(PFG_E_ZERO_VECTOR, "query row " + std::to_string(zrow) + " is a zero vector");
    PFG_TRY(I->qcodes.ensure((size_t)nq * nreps * 4, "query codes"));
    if (g.family == PFG_CROSSPOLYTOPE_FHT && g.strategy == PFG_INDEPENDENT && (g.dp == 32 || g.dp == 64 || g.dp == 128)) {
        PFG_TRY(fht_codes(I, nq, nullptr, 0, nreps, nreps, st));
    } else {
        bool pool_ready = false;
        PFG_TRY(hash_reps(I, I->qx.as<float>(), nq, 0, nreps, nullptr, I->qcodes.as<uint32_t>(), nreps, I->qbits, I->qfc,
                          pool_ready, st));
    }
    PFG_CUDA(cudaMemcpyAsync(out_codes, I->qcodes.p, (size_t)nq * nreps * 4,
                             is_device_ptr(out_codes) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (out_sketches && g.M > 0)
        PFG_CUDA(cudaMemcpyAsync(out_sketches, I->qsk.p, (size_t)nq * g.M * 8,
                                 is_device_ptr(out_sketches) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    PFG_CUDA(cudaStreamSynchronize(st));
    return PFG_OK;
}

pfg_status pfg_stop_tables(pfg_index* I, float recall, const pfg_search_opts* opts, float* thr_host, float* tau_host) {
    if (!I) return fail(PFG_E_ARG, "NULL index");
    if (!(recall > 0.0f && recall <= 1.0f)) return fail(PFG_E_ARG, "recall target must be in (0, 1]");
    SearchCfg s;
    PFG_TRY(resolve_sopts(opts, s));
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    if (thr_host) {
        std::shared_ptr<DBuf> b;
        std::vector<float> h;
        PFG_TRY(get_thr(I, recall, s, b, &h));
        std::memcpy(thr_host, h.data(), h.size() * 4);
    }
    if (tau_host) {
        std::shared_ptr<DBuf> b;
        std::vector<float> h;
        PFG_TRY(get_tau(I, s.tau_rule, s.eps, recall, b, &h));
        std::memcpy(tau_host, h.data(), 65 * 4);
    }
    return PFG_OK;
}

pfg_status pfg_save(const pfg_index* Ic, const char* path, void* stream) {
    if (!Ic || !path) return fail(PFG_E_ARG, "index and path are required");
    pfg_index* I = const_cast<pfg_index*>(Ic);
    std::lock_guard<std::mutex> lock(I->mu);
    PFG_CUDA(cudaSetDevice(I->device));
    PFG_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    std::unique_ptr<FILE, int (*)(FILE*)> f(fopen(path, "wb"), fclose);
    if (!f) return fail(PFG_E_ARG, std::string("cannot open ") + path + " for writing");
    const int32_t abi = PFG_ABI_VERSION;
    const uint32_t gsz = sizeof(Geo);
    bool ok = fwrite(kIdxMagic, 8, 1, f.get()) == 1 && fwrite(&abi, 4, 1, f.get()) == 1 &&
              fwrite(&gsz, 4, 1, f.get()) == 1 && fwrite(&I->g, sizeof(Geo), 1, f.get()) == 1 &&
              fwrite(&I->seed, 8, 1, f.get()) == 1;
    Stage stg;
    PFG_CUDA(cudaMallocHost(&stg.h, kStage));
    for (DBuf* b : index_arrays(I)) {
        const uint64_t nb = b->p ? (uint64_t)b->bytes : 0;
        ok = ok && fwrite(&nb, 8, 1, f.get()) == 1;
        for (uint64_t o = 0; ok && o < nb; o += kStage) {
            const size_t c = (size_t)std::min<uint64_t>(kStage, nb - o);
            PFG_CUDA(cudaMemcpy(stg.h, (char*)b->p + o, c, cudaMemcpyDeviceToHost));
            ok = fwrite(stg.h, 1, c, f.get()) == c;
        }
    }
    ok = ok && put_vec(f.get(), I->cpT) && put_vec(f.get(), I->slot_h) && put_vec(f.get(), I->sel_h);
    if (!ok) return fail(PFG_E_STATE, std::string("short write to ") + path);
    if (fclose(f.release()) != 0) return fail(PFG_E_STATE, std::string("cannot close ") + path);
    return PFG_OK;
}

pfg_status pfg_load(const char* path, void* stream, pfg_index** out) {
    if (!path || !out) return fail(PFG_E_ARG, "path and out are required");
    *out = nullptr;
    std::unique_ptr<FILE, int (*)(FILE*)> f(fopen(path, "rb"), fclose);
    if (!f) return fail(PFG_E_ARG, std::string("cannot open ") + path);
    char magic[8];
    int32_t abi = 0;
    uint32_t gsz = 0;
    if (fread(magic, 8, 1, f.get()) != 1 || std::memcmp(magic, kIdxMagic, 8) != 0)
        return fail(PFG_E_ARG, std::string(path) + " is not a pfg index file");
    if (fread(&abi, 4, 1, f.get()) != 1 || abi != PFG_ABI_VERSION || fread(&gsz, 4, 1, f.get()) != 1 || gsz != sizeof(Geo))
        return fail(PFG_E_ARG, std::string(path) + " was written by another ABI version");
    std::unique_ptr<pfg_index> I(new pfg_index());
    if (fread(&I->g, sizeof(Geo), 1, f.get()) != 1 || fread(&I->seed, 8, 1, f.get()) != 1)
        return fail(PFG_E_STATE, std::string("short read from ") + path);
    PFG_CUDA(cudaGetDevice(&I->device));
    PFG_CUDA(cudaDeviceGetAttribute(&I->num_sms, cudaDevAttrMultiProcessorCount, I->device));
    Stage stg;
    PFG_CUDA(cudaMallocHost(&stg.h, kStage));
    (void)stream;
    for (DBuf* b : index_arrays(I.get())) {
        uint64_t nb = 0;
        if (fread(&nb, 8, 1, f.get()) != 1) return fail(PFG_E_STATE, std::string("short read from ") + path);
        if (nb == 0) continue;
        PFG_TRY(b->alloc((size_t)nb, "loaded index array"));
        for (uint64_t o = 0; o < nb; o += kStage) {
            const size_t c = (size_t)std::min<uint64_t>(kStage, nb - o);
            if (fread(stg.h, 1, c, f.get()) != c) return fail(PFG_E_STATE, std::string("short read from ") + path);
            PFG_CUDA(cudaMemcpy((char*)b->p + o, stg.h, c, cudaMemcpyHostToDevice));
        }
    }
    if (!get_vec(f.get(), I->cpT) || !get_vec(f.get(), I->slot_h) || !get_vec(f.get(), I->sel_h))
        return fail(PFG_E_STATE, std::string("short read from ") + path);
    *out = I.release();
    return PFG_OK;
}

void pfg_free(pfg_index* I) {
    if (!I) return;
    cudaSetDevice(I->device);
    delete I;
}

}  // extern "C"
