/*
 * pfg.h — C ABI of the B200-native batched LSH-forest k-NN index (PUFFINN, arXiv 1906.12211).
 *
 * The calls follow the paper's problem statement: the user gives only the space the index
 * may use and the recall it must reach (PAPER.md:5 abstract, :38 §1.1, :371-374 §5
 * "Parameter Choices"), i.e. build(data, n, d, memory budget, hash family, seed) and
 * search(queries, k, recall target) -> ids and similarities, solving the (k, delta)-NN problem
 * of PAPER.md:118-123 (Definition, delta = 1 - recall) on the unit sphere under angular distance
 * (PAPER.md:133-135).
 *
 * Conventions (all calls):
 *  - Every call returns a pfg_status and never aborts; pfg_last_error() returns a thread-local
 *    message for the last non-OK status of the calling thread.
 *  - Array arguments are plain pointers.  Unless a call says otherwise a pointer may be HOST or
 *    DEVICE memory (of the index's device); the library inspects it with
 *    cudaPointerGetAttributes and copies host arrays through internal device buffers.  The caller
 *    owns every buffer it passes; the library never frees or retains caller pointers.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls enqueue work on it.
 *    pfg_build and pfg_search synchronise `stream` before returning (they read back a small
 *    status word to report zero rows); outputs in device memory are complete on return.
 *  - Layouts are row-major and densely packed: data [n][d] fp32, queries [nq][d] fp32,
 *    ids [nq][k] int64, sims [nq][k] fp32.
 *  - Ids are global: local row r of the index is reported as r + id_offset (sharded mode).
 */
#ifndef PFG_H
#define PFG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFG_ABI_VERSION 1

typedef struct pfg_index pfg_index; /* opaque; owned by the library until pfg_free */

typedef enum {
    PFG_OK = 0,
    PFG_E_ARG = 1,         /* invalid argument (n < 1, d < 1, k < 1 or k > 256, recall not in (0,1], ...) */
    PFG_E_ZERO_VECTOR = 2, /* a data or query row has norm 0 and cannot be normalised */
    PFG_E_BUDGET = 3,      /* memory budget below fixed cost + one repetition; message states the minimum */
    PFG_E_CUDA = 4,        /* CUDA runtime error (message has the CUDA error string) or no device */
    PFG_E_OOM = 5,         /* device allocation failed */
    PFG_E_STATE = 7        /* call not valid for this index (e.g. export of a table that does not exist) */
} pfg_status;

/* LSH families (§2, 338-343 §4.3) */
typedef enum {
    PFG_SIMHASH = 0,               /* random hyperplane (HP): 1 bit = [<a,x> >= 0], a ~ N(0, I) */
    PFG_CROSSPOLYTOPE_FHT = 1,     /* cross-polytope via three rounds of random signs + fast Hadamard
                                      transform: ell = 1 + log2(d') bits, d' = 2^ceil(log2 d) */
    PFG_CROSSPOLYTOPE = 2          /* exact cross-polytope: d Gaussian hyperplanes
                                      a_1..a_d per function, code = index of the largest |<a_i,x>| (ties to
                                      the lowest i) with the sign as the most significant of ell = 1 +
                                      ceil(log2 d) bits; each <a_i,x> is the sequential fp32 fmaf chain
                                      (R-2 projections); d <= 256; independent or pool strategy */
} pfg_family;

/* hash-function evaluation strategies (§3.2, App. B 841-917) */
typedef enum {
    PFG_INDEPENDENT = 0,  /* every repetition has its own functions (Alg. 1) */
    PFG_POOL = 1,         /* repetitions sample functions without replacement from one pool (Alg. 3) */
    PFG_TENSOR = 2        /* L = S^2 tries from two collections of S tuples of K/2 functions, trie
                             (j1, j2) interleaving tuple j1 and tuple j2; depths in steps of two
                             functions, shells of tries per stop check (Alg. 2, PAPER.md:244-249,
                             849-882).  L: an even power of two <= 256; K: an even number of whole
                             functions; searched by the fused kernel */
} pfg_strategy;

/* Build options.  Zero-initialise and set struct_size = sizeof(pfg_build_opts); a zero field
 * takes the default in brackets.  NULL opts = all defaults. */
typedef struct {
    uint32_t struct_size;
    int32_t strategy;      /* [PFG_INDEPENDENT] */
    int32_t pool_bits;     /* [3072] pool size in bits for PFG_POOL */
    int32_t prefix_bits;   /* [24] K: maximum prefix length in bits, 13..32 (R-7) */
    int32_t reps_override; /* [0 = derive L from the budget] L repetitions (BASELINE config 1 uses 32) */
    int32_t sketch_words;  /* [32] M 64-bit sketches per point; -1 = none (no filter) */
    int32_t cp_draws;      /* [1000] Monte-Carlo draws per grid cell of the CP table */
    int32_t max_reps;      /* [4096] cap on the derived L (R-11) */
    int32_t storage;       /* [PFG_STORAGE_F32] rows for the exact inner products (PFG_STORAGE_I16: the
                              paper's 16-bit fixed point; R-25) */
    int64_t id_offset;     /* [0] global id of local row 0 (sharded mode) */
} pfg_build_opts;

/* Row storage for the inner products (hashing and sketches always use the fp32 normalised rows).
 * PFG_STORAGE_I16: v = clamp(rint(x * 2^15), -2^15, 2^15 - 1) per coordinate of the normalised fp32
 * row (round to nearest, ties to even), rows padded to a multiple of 16 coordinates (32 bytes);
 * similarity = (float)(sum_t q_t v_t, exact in int32) * 2^-30.  Halves the bytes of every
 * candidate row; similarities differ from fp32 by at most ~2e-3 and are exact
 * (order-independent) integers before the final conversion.  The fp32 rows are kept too (and
 * counted in the budget) for the fp32 re-rank of each query's top-k (pfg_search_opts.rerank). */
enum { PFG_STORAGE_F32 = 0, PFG_STORAGE_I16 = 1 };

/* Search options.  Zero-initialise + struct_size; zero field = default.  NULL = all defaults. */
typedef struct {
    uint32_t struct_size;
    int32_t rep_chunk;        /* [16] R: the filter threshold tau is refreshed once per chunk of R
                                 repetitions (R-17); the search's first chunk is the single
                                 repetition 0 (tau is set right after it) unless
                                 uniform_chunks = 1 */
    int32_t segment;          /* [12] B: entries are retrieved in segments of B */
    int32_t stop_rule;        /* [0] 0 = failure bound (1-P_i)^j <= delta; 2 = two-level bound
                                 (1-P_i)^j (1-P_{i+1})^(L-j) <= delta below depth K (independent only; the
                                 same argument);
                                 1 = Alg. 1 line 8, j >= ln(1/delta)/P_i (independent only) */
    int32_t stop_granularity; /* [0] 0 = check after every repetition (Alg. 1);
                                 1 = only after all L repetitions of a level */
    int32_t use_filter;       /* [1] 1 = sketch filter on; -1 = off */
    float filter_eps;         /* [0] tau_rule 1: tau = (1+eps) x expected Hamming distance */
    int32_t trace_cap;        /* [0] >0: write the ids evaluated by each query, in evaluation order,
                                 to trace_ids[nq][trace_cap] (uint32, local row ids) */
    int32_t timing;           /* [0] 1: record CUDA events around the phases of this call on `stream`
                                 (read back with pfg_last_timing); 2: also between the query-phase
                                 kernels (pfg_last_phases; the extra events cost a few microseconds each);
                                 3: events around each bulk-round k_sims launch only, accumulated over
                                 searches (pfg_kernel_timing); 4: developer timeline, an event after
                                 each launch group on its stream, printed to stderr when the call
                                 completes (completion times relative to the call's first event) */
    uint32_t* trace_ids;      /* host or device pointer, required when trace_cap > 0 */
    int32_t engine;           /* [0] 0 = bulk rounds (one chunk of every active query per round, split
                                 into data-parallel phases), then the fused kernel resumes the queries
                                 still running; 1 = fused kernel only (one warp per query, persistent
                                 grid); 2 = chunk rounds (one CTA per query fuses a round's control
                                 phases, kernels_chunk.cuh; the phase-split engine when wide queries are
                                 on), then the fused kernel.  Results are identical. */
    int32_t uniform_chunks;   /* [0] 1 = chunks of R repetitions from the start (tau = 64 for a whole
                                 first chunk); 0 = the first chunk is the single repetition 0 */
    int32_t rounds;           /* [5] engine 0: bulk rounds before the fused kernel resumes the rest
                                 (then a device-side loop of rounds may continue, see `wide`) */
    int32_t wide;             /* [0] engine 0: > 0 = evaluated-id capacity of the per-query hash set
                                 (at most 1536) before a query moves its evaluated set to a visit-tag
                                 array of n words ("wide") and continues in the device-side round loop;
                                 0 = automatic: capacity 1536, wide queries on iff the previous search's
                                 queries read >= 64 MiB each (evaluated rows + table entries), and then
                                 the loop keeps every query still running after the blind rounds;
                                 -1 = off (a query beyond the hash set continues in the fused kernel's
                                 global bitmap).  Results are identical in every mode. */
    int32_t tau_rule;         /* [0] sketch-filter threshold tau at the k-th similarity ip_k (R-26,
                                 R-15): 0 = the (1 - delta)-quantile of the sketch Hamming distance of a
                                 pair at ip_k, i.e. the smallest t with P[Binomial(64, acos(ip_k)/pi) <= t]
                                 >= 1 - delta, delta = 1 - recall target; 1 = (1 +
                                 filter_eps) x the expected distance 64 acos(ip_k)/pi, rounded half up
                                  */
    int32_t rerank;           /* [0] PFG_STORAGE_I16: 0 = each query's top-k is re-scored with the fp32 rows
                                 and re-sorted; -1 = returned as the fixed-point search ranked
                                 them (fixed-point similarities) */
    /* device-side round loop policy (engine 0 with wide queries; results are identical either way;
       used by the tests to drive every path): */
    int32_t loop_min;         /* [0 = 64] the loop keeps all queries still running after the blind rounds
                                 when there are at least loop_min (and at most loop_max) of them */
    int32_t loop_max;         /* [0 = automatic] > 0: that upper bound, and wide queries on when wide = 0 */
    int32_t wide_arrays;      /* [0 = as many as 8 GiB holds] at most this many visit-tag arrays */
    int32_t wide_tiles_min;   /* [0] 1 = the smallest wide-tile buffer (wide chunks compete and wait) */
    /* precomputed query hashes (in the data-sharded mode each rank hashes a slice of the
       queries with pfg_hash_queries_reps and the slices are all-gathered); DEVICE pointers or NULL: */
    const uint32_t* ext_codes;     /* [nq][ext_reps] codes of repetitions [0, ext_reps): ext_reps = L, or
                                      <= L for the FHT cross-polytope family with independent functions
                                      (later repetitions are hashed in the kernels as usual) */
    int32_t ext_reps;
    const uint64_t* ext_sketches;  /* [nq][M] query sketches */
    int32_t pipelines;        /* [0] engine 0: 0 or 1 = one round pipeline over the batch; 2 = two pipelines,
                                 the lower and the upper half of the batch as two searches of their own on
                                 two streams, each kernel with half its resident grid (not with wide
                                 queries, the device-side loop, or exact cross-polytope's partial eager
                                 hashing; then one).  Results are identical; measured slower on config 2. */
} pfg_search_opts;

/* per-query counters (optional output of pfg_search) */
typedef struct {
    int32_t i_stop;      /* prefix length at which the search stopped (0 = linear scan) */
    int32_t j_stop;      /* 1-based repetition index at that level */
    uint32_t emitted;    /* table positions retrieved (segments included) */
    uint32_t filtered;   /* retrieved candidates rejected by the sketch filter */
    uint32_t dups;       /* retrieved candidates that passed the filter but were already evaluated */
    uint32_t evaluated;  /* distinct points whose exact inner product was computed */
    uint32_t flags;      /* bit0: k > n (padded); bit1: zero query row; bit2: trace truncated;
                            bit3: fused kernel, global bitmap; bit4: wide (visit-tag array);
                            bit5: not finished (round cap of the device-side loop; no result) */
    uint32_t probes;     /* table entries read by the prefix-range searches */
} pfg_query_stats;

typedef struct {
    int64_t n;
    int32_t d, d_pad, family, strategy, prefix_bits, reps, ell, funcs_per_rep, sketch_words;
    int32_t pool_funcs, fht_dim, device, reserved0;
    uint64_t index_bytes;    /* bytes counted against the memory budget (R-11) */
    uint64_t scratch_bytes;  /* per-query scratch currently allocated (not counted in the budget) */
    uint64_t seed;
    int64_t id_offset;
} pfg_index_info_t;

/* Build an index over n rows of dimension d (§4.2).
 * data: [n][d] fp32, host or device.  Rows are normalised into index-owned
 * memory.  memory_budget_bytes: total index size including the data and the hash functions
 * (PAPER.md:567); L is derived from it unless opts->reps_override > 0.  family: pfg_family.
 * seed: all hash functions derive from it (identical on every shard).
 * Errors: PFG_E_ARG (n < 1, n >= 2^31, d < 1, d > 4096, bad option), PFG_E_ZERO_VECTOR (message
 * names the row), PFG_E_BUDGET (message names the minimum budget), PFG_E_OOM, PFG_E_CUDA.
 * On error *out is NULL. */
pfg_status pfg_build(const float* data, int64_t n, int32_t d, uint64_t memory_budget_bytes,
                     int32_t family, uint64_t seed, const pfg_build_opts* opts, void* stream,
                     pfg_index** out);

/* Adaptive k-NN search (Alg. 1 over the array index of PAPER.md:281-334) for
 * nq queries.  queries: [nq][d] fp32 (normalised internally).  recall_target in (0, 1]:
 * delta = 1 - recall (recall 1 = exhaustive).  Outputs out_ids [nq][k] int64 (global ids) and
 * out_sims [nq][k] fp32 (inner product of the normalised vectors), sorted by similarity
 * descending, ties by smaller id.  If k > n the last k-n entries are id -1 / sim -inf.
 * stats: optional [nq] pfg_query_stats.  Zero query rows: that row's ids are -1, sims NaN,
 * stats flag bit1, and the call returns PFG_E_ZERO_VECTOR naming the first such row after
 * finishing the others.  Reentrant; concurrent calls on one index are serialised on the device. */
pfg_status pfg_search(pfg_index* idx, const float* queries, int64_t nq, int32_t k, float recall_target,
                      const pfg_search_opts* opts, int64_t* out_ids, float* out_sims,
                      pfg_query_stats* stats, void* stream);

/* Merge `world` per-shard top-k lists into one (sharded mode, after an all-gather):
 * ids [world][nq][k] int64 (-1 = empty), sims [world][nq][k] fp32 -> out [nq][k] by
 * (sim desc, id asc).  Device pointers only. */
pfg_status pfg_merge_topk(const int64_t* ids, const float* sims, int32_t world, int64_t nq, int32_t k,
                          int64_t* out_ids, float* out_sims, void* stream);

pfg_status pfg_index_info(const pfg_index* idx, pfg_index_info_t* out);

/* Index serialisation (the paper's index is rebuilt from its seed, SPEC.md's
 * program persists it).  pfg_save writes the geometry, the seed and every index array (normalised
 * data, repetition tables, prefix tables, hash and sketch functions, slots, pool selections, the
 * CP table) to `path` in a private little-endian format (magic "PFGIDX02" + ABI version); it
 * waits for `stream` first.  pfg_load reads such a file onto the current CUDA device and returns
 * an index equal to the saved one (searches give identical results).  Errors: PFG_E_ARG (cannot
 * open / not an index file / other ABI version), PFG_E_STATE (short read or write),
 * PFG_E_OOM / PFG_E_CUDA.  The caller owns `*out` (pfg_free). */
pfg_status pfg_save(const pfg_index* idx, const char* path, void* stream);
pfg_status pfg_load(const char* path, void* stream, pfg_index** out);

/* Host-only cost model (R-11, no GPU needed): the L that pfg_build would derive, and
 * the minimum budget for L = 1.  Returns PFG_E_BUDGET if the budget admits no repetition. */
pfg_status pfg_derive_reps(int64_t n, int32_t d, int32_t family, uint64_t memory_budget_bytes,
                           const pfg_build_opts* opts, int32_t* reps_out, uint64_t* min_budget_out,
                           uint64_t* index_bytes_out);

/* ---- test hooks (parity) ---------------------------------------------------------------- */
typedef enum {
    PFG_EXPORT_TABLE = 1,   /* arg = rep j: uint64 [n][2] = {(code << 32) | local id, sketch word of the
                               repetition's slot for that id}, sorted ascending by the first word */
    PFG_EXPORT_PREFIX = 2,  /* arg = rep j: uint32 [8193] first position whose top 13 bits >= p */
    PFG_EXPORT_SKETCH = 3,  /* per-point sketches are not retained (PFG_E_STATE): they live inline */
    PFG_EXPORT_DATA = 4,    /* fp32 [n][d] normalised rows (PFG_STORAGE_F32 only) */
    PFG_EXPORT_CP = 5,      /* double [ell+1][41] cleaned CP collision table (FHT family) */
    PFG_EXPORT_SLOTS = 6,   /* int32 [L] sketch slot per repetition */
    PFG_EXPORT_POOLSEL = 7, /* int32 [L][c] pool function indices per repetition */
    PFG_EXPORT_DATA16 = 8   /* int16 [n][d] fixed-point rows (PFG_STORAGE_I16 only) */
} pfg_export_what;

/* copy an index array into host memory dst (dst_bytes must equal the array size) */
pfg_status pfg_export(const pfg_index* idx, int32_t what, int32_t arg, void* dst_host, uint64_t dst_bytes);

/* hash queries: out_codes [nq][L] uint32 (K-bit repetition codes), out_sketches [nq][M] uint64;
 * either output may be NULL.  Device or host pointers. */
pfg_status pfg_hash_queries(pfg_index* idx, const float* queries, int64_t nq, uint32_t* out_codes,
                            uint64_t* out_sketches, void* stream);

/* codes of repetitions [0, nreps) (out_codes [nq][nreps] uint32) and sketches (out_sketches [nq][M]
 * uint64, may be NULL) of nq queries, in the layout pfg_search takes as ext_codes / ext_sketches.
 * Host or device pointers.  Errors: PFG_E_ARG (nreps not in [1, L]), PFG_E_ZERO_VECTOR. */
pfg_status pfg_hash_queries_reps(pfg_index* idx, const float* queries, int64_t nq, int32_t nreps, uint32_t* out_codes,
                                 uint64_t* out_sketches, void* stream);

/* stop-rule and filter tables used by pfg_search for this recall target and options:
 * thr_host [K][L] fp32: level i = 1..K row i-1: the search stops after repetition j at level i
 * iff the k-th similarity (clamped to [-1,1]) >= thr[i-1][j-1] (+inf = never);
 * tau_host [65] fp32: tau(ip) = min{t : ip >= tau_host[t]} under opts->tau_rule (and, for the
 * quantile rule, this recall target).  Either may be NULL. */
pfg_status pfg_stop_tables(pfg_index* idx, float recall_target, const pfg_search_opts* opts,
                           float* thr_host, float* tau_host);

/* phase timings of the last pfg_search on this index that set opts->timing (CUDA events on the
 * call's stream): ms[0] = query preparation (host->device copy, normalisation, hashing, sketches),
 * ms[1] = the query kernel, ms[2] = whole call; *launches = kernels the call launched. */
pfg_status pfg_last_timing(const pfg_index* idx, float* ms3, int32_t* launches);

/* per-phase breakdown of the query-kernel time of the same search (CUDA events between the
 * phases' launches): ms[0] k_expand, ms[1] k_scan, ms[2] k_dedupe, ms[3] k_sims, ms[4] k_merge
 * (summed over the blind bulk rounds), ms[5] the fused kernel (both launches; the first runs
 * beside the device-side round loop), ms[6] other (round control, query order, code extension for
 * resumed queries), ms[7] the device-side round loop (a CUDA graph; its rounds are not split into
 * phases).  n: entries to write (<= 8). */
pfg_status pfg_last_phases(const pfg_index* idx, float* ms, int32_t n);

/* Launch durations of one kernel accumulated over the searches that set opts->timing = 3 since
 * the last reset (CUDA events on the search stream around each launch; waits for them):
 * kernel 0 = k_sims of the blind bulk rounds.  *ms = summed duration, *launches = launches timed;
 * reset != 0 clears the accumulator afterwards. */
pfg_status pfg_kernel_timing(pfg_index* idx, int32_t kernel, int32_t reset, double* ms, int64_t* launches);

/* Counters of the last search's round engine (waits for it): out[0] rows whose similarity the
 * bulk k_sims computed, out[1] blind rounds, out[2] device-side loop rounds, out[3] queries the
 * fused kernel took beside the loop, out[4] after it, out[5] visit-tag arrays used (wide queries),
 * out[6] the rows of out[0] computed by the blind rounds' k_sims launches (those timed by
 * timing = 3).  n: entries to write (<= 7). */
pfg_status pfg_round_stats(pfg_index* idx, uint64_t* out, int32_t n);

void pfg_free(pfg_index* idx);
const char* pfg_last_error(void);
int32_t pfg_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PFG_H */
