/*
 * oracle.c — PUFFINN (arXiv 1906.12211) CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, scalar C of what the batched LSH-forest k-NN query path computes.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares NO code with paper_1906_12211_b200/ (the
 * product): no headers, no helpers, no table generators.  Each function cites the
 * PAPER.md passage it restates ("PAPER.md:N §x") or the DESIGN.md reading ("R-n")
 * that fixes what the paper leaves open.
 *
 * Compiled with -O2 -ffp-contract=off so every floating-point operation is the one
 * written here (explicit fmaf where the canonical order uses a fused multiply-add).
 *
 * Parity status per function:
 *   or_normalize, or_dot, or_fht, or_fhtcp_code, or_hp_bit, rep codes, sketches,
 *   sorted tables, widening, filter threshold, stop rule, search, brute force:
 *   pinned by tests/test_oracle_*.py.
 *   or_cp_table: pinned by invariants (T_b(1)=1, T_0=1, T_b(-1)=0, monotonicity),
 *   by the HP Monte-Carlo table against the closed form 1-theta/pi, and by a
 *   10x-draw re-estimate.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ----------------------------------------------------------------------------
 * R-3: the paper does not say how functions are drawn.  Every random
 * number is the c-th output of a SplitMix64 stream.  The product library contains
 * its own, independently written copy of this generator.
 * -------------------------------------------------------------------------- */
#define OR_GAMMA 0x9E3779B97F4A7C15ULL

enum { OR_TAG_HP = 1, OR_TAG_SKETCH = 2, OR_TAG_FHT = 3, OR_TAG_POOL = 4,
       OR_TAG_SLOT = 5, OR_TAG_TENSOR = 6, OR_TAG_CPMC = 7, OR_TAG_CP = 8 };

uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* c-th output (c = 0, 1, ...) of the SplitMix64 stream whose state starts at key */
uint64_t or_draw(uint64_t key, uint64_t c) { return or_mix64(key + (c + 1) * OR_GAMMA); }
uint64_t or_stream_key(uint64_t seed, uint64_t tag) { return or_draw(seed, tag); }

/* Box-Muller standard normal from draws 2i and 2i+1 of the stream (double) */
double or_gauss_d(uint64_t key, uint64_t i) {
    uint64_t r1 = or_draw(key, 2 * i), r2 = or_draw(key, 2 * i + 1);
    double u1 = (double)((r1 >> 11) + 1) * (1.0 / 9007199254740992.0);
    double u2 = (double)(r2 >> 11) * (1.0 / 9007199254740992.0);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}
float or_gauss(uint64_t key, uint64_t i) { return (float)or_gauss_d(key, i); }

/* ----------------------------------------------------------------------------
 * PAPER.md:301 §4.2 "We normalize the query vector and all data vectors".
 * R-2: the norm is summed in double, sequentially over t; x_t <- (float)(x_t / s).
 * Returns -1, or the index of the first zero row (which cannot be normalised).
 * -------------------------------------------------------------------------- */
int64_t or_normalize(const float* x, int64_t n, int d, float* out) {
    for (int64_t i = 0; i < n; ++i) {
        const float* r = x + i * (int64_t)d;
        double s = 0.0;
        for (int t = 0; t < d; ++t) s += (double)r[t] * (double)r[t];
        if (!(s > 0.0)) return i;
        s = sqrt(s);
        for (int t = 0; t < d; ++t) out[i * (int64_t)d + t] = (float)((double)r[t] / s);
    }
    return -1;
}

/* R-2 canonical projection (hash and sketch functions): sequential fp32 fmaf over t = 0..d-1
 * from +0 (on unit vectors the inner product is the cosine) */
float or_dot(const float* a, const float* b, int d) {
    float s = 0.0f;
    for (int t = 0; t < d; ++t) s = fmaf(a[t], b[t], s);
    return s;
}

/* R-2 canonical similarity of two unit vectors ("distance computation"):
 * the d products are accumulated in 32 lane sums -- element t goes to lane (t/4) mod 32 and
 * each lane sum is a sequential fp32 fmaf chain in ascending t from +0 -- which are then added
 * pairwise in a fixed tree: for h = 16, 8, 4, 2, 1: s[l] = s[l] + s[l+h] (l < h).  This is the
 * order in which a warp reading a row with one 16-byte chunk per lane computes it. */
/* O-11 plain-order similarity: one sequential fp32 fmaf chain over t = 0..d-1 from +0
 * (the same order as or_dot).  The search uses it when or_sopts.sim_order = 1, to show that the
 * results do not hinge on the R-2 lane-tree order (ties within 1e-6 excepted). */
float or_sim_seq(const float* a, const float* b, int d) { return or_dot(a, b, d); }

float or_sim(const float* a, const float* b, int d) {
    float s[32];
    for (int l = 0; l < 32; ++l) s[l] = 0.0f;
    for (int t = 0; t < d; ++t) s[(t / 4) % 32] = fmaf(a[t], b[t], s[(t / 4) % 32]);
    for (int h = 16; h >= 1; h /= 2)
        for (int l = 0; l < h; ++l) s[l] = s[l] + s[l + h];
    return s[0];
}

/* R-25, §4.2 "a fixed point format represented using 16-bit integers" (scale
 * 2^15 per SPEC.md:49, 73): v = clamp(rint(x * 2^15), -2^15, 2^15 - 1) of a normalised fp32
 * coordinate; rint rounds to nearest, ties to even (the default rounding mode). */
int16_t or_fixed16(float x) {
    float r = rintf(x * 32768.0f);
    if (r > 32767.0f) r = 32767.0f;
    if (r < -32768.0f) r = -32768.0f;
    return (int16_t)r;
}
void or_quantize(const float* x, int64_t n, int d, int16_t* out) {
    for (int64_t i = 0; i < n * d; ++i) out[i] = or_fixed16(x[i]);
}
/* The fixed-point inner product: the exact integer sum of the d products,
 * scaled back by 2^-30 after rounding the (int32-range) sum to fp32. */
float or_sim16(const int16_t* a, const int16_t* b, int d) {
    int64_t s = 0;
    for (int t = 0; t < d; ++t) s += (int64_t)a[t] * (int64_t)b[t];
    return (float)s * 0x1p-30f;
}

/* PAPER.md:142-146 §2: HP (SimHash) bit = 1 iff <a,x> >= 0, a ~ N(0,I).
 * The inner product uses the same canonical order as or_dot. */
int or_hp_bit(const float* a, const float* x, int d) { return or_dot(a, x, d) >= 0.0f; }

/* PAPER.md:340 §4.3 "three applications of the fast Hadamard transform".
 * R-6: unnormalised radix-2 transform, stages h = 1,2,4,...,dp/2, pair (u,u+h) with
 * bit h of u clear -> (y_u + y_{u+h}, y_u - y_{u+h}). */
void or_fht(float* y, int dp) {
    for (int h = 1; h < dp; h <<= 1)
        for (int u0 = 0; u0 < dp; u0 += 2 * h)
            for (int u = u0; u < u0 + h; ++u) {
                float a = y[u], b = y[u + h];
                y[u] = a + b;
                y[u + h] = a - b;
            }
}

/* PAPER.md:147-151 §2 (cross-polytope: index of the largest |inner product| plus its
 * sign) in the pseudorandom form of PAPER.md:340 §4.3: x is zero-padded to dp = 2^ceil(log2 d);
 * y = H D3 H D2 H D1 x.  R-5: the sign is the MOST significant of the ell = 1+log2(dp) bits;
 * ties of |y_u| go to the lowest u.  sg = [3][dp] of +-1. */
uint32_t or_fhtcp_code(const float* x, int d, int dp, const float* sg) {
    float y[4096];
    for (int u = 0; u < dp; ++u) y[u] = (u < d) ? x[u] : 0.0f;
    for (int r = 0; r < 3; ++r) {
        for (int u = 0; u < dp; ++u) y[u] = sg[r * dp + u] * y[u];
        or_fht(y, dp);
    }
    int best = 0;
    float ba = fabsf(y[0]);
    for (int u = 1; u < dp; ++u)
        if (fabsf(y[u]) > ba) { ba = fabsf(y[u]); best = u; }
    int ell = 1;
    while ((1 << (ell - 1)) < dp) ++ell;
    uint32_t neg = y[best] < 0.0f;
    return (neg << (ell - 1)) | (uint32_t)best;
}

/* ----------------------------------------------------------------------------
 * Index (§4.2): L arrays of (hash code, pos) sorted by code.
 * -------------------------------------------------------------------------- */
enum { OR_HP = 0, OR_FHTCP = 1, OR_CP = 2 };
enum { OR_INDEPENDENT = 0, OR_POOL = 1, OR_TENSOR = 2 };

typedef struct {
    int64_t n;
    int d, dp, ell, family, strategy, K, L, M, c, m, S;  /* S = sqrt(L) for the tensor strategy */
    uint64_t seed;
    float* x;          /* normalised data [n][d] */
    uint64_t* sk;      /* sketches [n][M] */
    float* hp;         /* HP functions [F][d] */
    float* sg;         /* FHT-CP signs [F][3][dp], +-1 */
    int32_t* sel;      /* pool selections [L][c] */
    int32_t* slot;     /* sketch slot per rep [L] */
    float* skf;        /* sketch functions [64M][d] */
    uint32_t** codes;  /* sorted codes per rep (NULL = not built yet; lazy mode) */
    uint32_t** ids;    /* point ids per rep, aligned with codes */
    uint16_t* fcache;  /* pool strategy: or_func of every pool function on every data point [n][m],
                          computed once on the first table build (memoised values, same arithmetic) */
    double cpT[34 * 41]; /* CP table T[b][a], b = 0..ell, a = 0..40 */
    int cp_draws;
    int storage;       /* 0 = fp32 rows (or_sim), 1 = 16-bit fixed point (or_sim16, R-25) */
    int16_t* x16;      /* fixed-point data [n][d] (storage 1) */
} or_index;

/* number of functions a repetition concatenates: c = ceil(K / ell) (R-7) */
static int or_funcs_per_rep(int K, int ell) { return (K + ell - 1) / ell; }

/* value of pool/independent function f on x (ell bits) */
/* PAPER.md:147-151 §2 exact cross-polytope: "choosing d random hyperplanes a_1..a_d and mapping x
 * to the index of the hyperplane with the largest absolute inner product, separating the two
 * cases that the inner product is negative or not".  A = [d][d] (row i = a_i); each <a_i, x> is
 * or_dot (R-2 projections); ties of |y_i| go to the lowest i; the sign is the most significant of
 * the ell = ceil(log 2d) bits (R-5). */
uint32_t or_cp_code(const float* A, const float* x, int d, int ell) {
    int best = 0;
    float y0 = or_dot(A, x, d), ba = fabsf(y0);
    int neg = y0 < 0.0f;
    for (int i = 1; i < d; ++i) {
        float y = or_dot(A + (int64_t)i * d, x, d);
        if (fabsf(y) > ba) { ba = fabsf(y); best = i; neg = y < 0.0f; }
    }
    return ((uint32_t)neg << (ell - 1)) | (uint32_t)best;
}

static uint32_t or_func(const or_index* X, int64_t f, const float* x) {
    if (X->family == OR_HP) return (uint32_t)or_hp_bit(X->hp + f * X->d, x, X->d);
    if (X->family == OR_CP) return or_cp_code(X->hp + f * X->d * (int64_t)X->d, x, X->d, X->ell);
    return or_fhtcp_code(x, X->d, X->dp, X->sg + f * 3 * (int64_t)X->dp);
}

/* h_{<=i,j} is the concatenation of the rep's functions, earlier functions
 * more significant (a bit string); the top K bits are kept (R-7).  Independent: rep j uses
 * functions j*c..j*c+c-1.  Pool and tensor (PAPER.md:244-249,
 * 849-858): the functions sel[j][0..c). */
uint32_t or_rep_code(const or_index* X, int j, const float* x) {
    uint64_t full = 0;
    for (int t = 0; t < X->c; ++t) {
        int64_t f = (X->strategy != OR_INDEPENDENT) ? X->sel[j * X->c + t] : (int64_t)j * X->c + t;
        full = (full << X->ell) | or_func(X, f, x);
    }
    return (uint32_t)(full >> (X->c * X->ell - X->K));
}

/* PAPER.md:258-260 §3.3, 322-323 §4.2: M 64-bit sketches of HP bits; bit b of word w is
 * sketch function 64w+b (R-20 layout). */
void or_sketch(const or_index* X, const float* x, uint64_t* out) {
    for (int w = 0; w < X->M; ++w) {
        uint64_t v = 0;
        for (int b = 0; b < 64; ++b)
            if (or_hp_bit(X->skf + ((int64_t)w * 64 + b) * X->d, x, X->d)) v |= 1ULL << b;
        out[w] = v;
    }
}

/* pool strategy: the values of all m pool functions on every data point, computed once (a table
 * build reads c of them per point; the rep code is the same concatenation as or_rep_code) */
static void or_need_fcache(or_index* X) {
    if (X->fcache) return;
    uint16_t* fc = (uint16_t*)malloc(sizeof(uint16_t) * X->n * (int64_t)X->m);
    #pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < X->n; ++p)
        for (int f = 0; f < X->m; ++f) fc[p * X->m + f] = (uint16_t)or_func(X, f, X->x + p * X->d);
    X->fcache = fc;
}
static uint32_t or_rep_code_cached(const or_index* X, int j, int64_t p) {
    uint64_t full = 0;
    for (int t = 0; t < X->c; ++t) full = (full << X->ell) | X->fcache[p * X->m + X->sel[j * X->c + t]];
    return (uint32_t)(full >> (X->c * X->ell - X->K));
}

/* build one repetition: hash all points, sort (code, id) ascending */
static int or_cmp_pair(const void* a, const void* b) {
    const uint64_t* x = (const uint64_t*)a; const uint64_t* y = (const uint64_t*)b;
    return (*x > *y) - (*x < *y);
}
static void or_build_rep(or_index* X, int j) {
    int64_t n = X->n;
    uint64_t* pr = (uint64_t*)malloc(sizeof(uint64_t) * n);
    if (X->strategy == OR_POOL) {
        or_need_fcache(X);
        #pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < n; ++p) pr[p] = ((uint64_t)or_rep_code_cached(X, j, p) << 32) | (uint64_t)p;
    } else {
        #pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < n; ++p)
            pr[p] = ((uint64_t)or_rep_code(X, j, X->x + p * X->d) << 32) | (uint64_t)p;
    }
    qsort(pr, n, sizeof(uint64_t), or_cmp_pair);
    X->codes[j] = (uint32_t*)malloc(sizeof(uint32_t) * n);
    X->ids[j] = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (int64_t p = 0; p < n; ++p) { X->codes[j][p] = (uint32_t)(pr[p] >> 32); X->ids[j][p] = (uint32_t)pr[p]; }
    free(pr);
}
static void or_need_rep(or_index* X, int j) {
    if (X->codes[j]) return;
    #pragma omp critical(or_rep)
    { if (!X->codes[j]) or_build_rep(X, j); }
}

/* ----------------------------------------------------------------------------
 * PAPER.md:345-352 §4.3 Monte-Carlo collision table: alpha grid -1, -0.95, ..., 1 (41 cells),
 * `draws` functions per cell, collision counted for every bit length b = 1..ell.
 * R-14: pairs are random in the first d coordinates (the paper's canonical pair of its
 * footnote is not representative for the FHT variant); R-13: cleaned to be monotone
 * (running minimum from high alpha down, then non-increasing in b); T_0 = 1.
 * family OR_HP gives the 1-bit HP table (used only to pin this routine against 1-theta/pi).
 * -------------------------------------------------------------------------- */
static void or_mc_pair(uint64_t kx, uint64_t ku, int d, double alpha, float* xf, float* yf) {
    double x[4096], u[4096];
    double nx = 0.0;
    for (int t = 0; t < d; ++t) { x[t] = or_gauss_d(kx, t); nx += x[t] * x[t]; }
    nx = sqrt(nx);
    for (int t = 0; t < d; ++t) x[t] = x[t] / nx;
    double ux = 0.0;
    for (int t = 0; t < d; ++t) { u[t] = or_gauss_d(ku, t); ux += u[t] * x[t]; }
    double nu = 0.0;
    for (int t = 0; t < d; ++t) { u[t] = u[t] - ux * x[t]; nu += u[t] * u[t]; }
    nu = sqrt(nu);
    for (int t = 0; t < d; ++t) u[t] = u[t] / nu;
    double s = sqrt(1.0 - alpha * alpha);
    for (int t = 0; t < d; ++t) { xf[t] = (float)x[t]; yf[t] = (float)(alpha * x[t] + s * u[t]); }
}

void or_cp_table(int family, int d, uint64_t seed, int draws, double* T /* [(ell+1)*41] */, int* ell_out) {
    int dp = 1; while (dp < d) dp <<= 1;
    int ell = (family == OR_HP) ? 1 : 1 + (int)round(log2((double)dp));
    uint64_t K = or_stream_key(seed, OR_TAG_CPMC);
    long* cnt = (long*)calloc((size_t)(ell + 1) * 41, sizeof(long));
    #pragma omp parallel for schedule(dynamic)
    for (int a = 0; a < 41; ++a) {
        double alpha = -1.0 + 0.05 * a;
        float xf[4096], yf[4096], sg[3 * 4096], hpa[4096];
        if (family == OR_CP) {
            /* exact CP: the paper's canonical pair x = e_0, y = (alpha, sqrt(1 - alpha^2), 0, ...)
             * (valid by spherical symmetry); only the first two coordinates of
             * each hyperplane enter: a_i0 = gauss(k, 2i), a_i1 = gauss(k, 2i+1) */
            float yx = (float)alpha, yy = (float)sqrt(fmax(0.0, 1.0 - alpha * alpha));
            for (int t = 0; t < draws; ++t) {
                uint64_t k = or_draw(K, (uint64_t)a * draws + t);
                float bx = -1.0f, by = -1.0f;
                int ix = 0, iy = 0, nx = 0, ny = 0;
                for (int i = 0; i < d; ++i) {
                    float a0 = (float)or_gauss(k, 2 * (uint64_t)i), a1 = (float)or_gauss(k, 2 * (uint64_t)i + 1);
                    float sx = fmaf(a0, 1.0f, 0.0f);
                    float sy = fmaf(a1, yy, fmaf(a0, yx, 0.0f));
                    if (fabsf(sx) > bx) { bx = fabsf(sx); ix = i; nx = sx < 0.0f; }
                    if (fabsf(sy) > by) { by = fabsf(sy); iy = i; ny = sy < 0.0f; }
                }
                uint32_t hx = ((uint32_t)nx << (ell - 1)) | (uint32_t)ix, hy = ((uint32_t)ny << (ell - 1)) | (uint32_t)iy;
                for (int b = 1; b <= ell; ++b)
                    if ((hx >> (ell - b)) == (hy >> (ell - b))) cnt[b * 41 + a]++;
            }
            continue;
        }
        for (int t = 0; t < draws; ++t) {
            uint64_t kat = or_draw(K, (uint64_t)a * draws + t);
            uint64_t ksg = or_draw(kat, 0), kx = or_draw(kat, 1), ku = or_draw(kat, 2);
            or_mc_pair(kx, ku, d, alpha, xf, yf);
            uint32_t hx, hy;
            if (family == OR_HP) {
                for (int v = 0; v < d; ++v) hpa[v] = or_gauss(ksg, v);
                hx = (uint32_t)or_hp_bit(hpa, xf, d); hy = (uint32_t)or_hp_bit(hpa, yf, d);
            } else {
                for (int v = 0; v < 3 * dp; ++v) sg[v] = (or_draw(ksg, v) >> 63) ? -1.0f : 1.0f;
                hx = or_fhtcp_code(xf, d, dp, sg); hy = or_fhtcp_code(yf, d, dp, sg);
            }
            for (int b = 1; b <= ell; ++b)
                if ((hx >> (ell - b)) == (hy >> (ell - b))) cnt[b * 41 + a]++;
        }
    }
    for (int a = 0; a < 41; ++a) T[a] = 1.0;
    for (int b = 1; b <= ell; ++b) {
        for (int a = 0; a < 41; ++a) T[b * 41 + a] = (double)cnt[b * 41 + a] / (double)draws;
        T[b * 41 + 40] = 1.0;
        for (int a = 39; a >= 0; --a)
            if (T[b * 41 + a + 1] < T[b * 41 + a]) T[b * 41 + a] = T[b * 41 + a + 1];
    }
    for (int b = 2; b <= ell; ++b)
        for (int a = 0; a < 41; ++a)
            if (T[(b - 1) * 41 + a] < T[b * 41 + a]) T[b * 41 + a] = T[(b - 1) * 41 + a];
    free(cnt);
    *ell_out = ell;
}

/* ----------------------------------------------------------------------------
 * Build.  L, K, M are explicit (the budget -> L cost model is host logic, R-11).
 * lazy = 1: repetition tables are built on first use (same result, used for the
 * bounded CPU baseline at full size).
 * -------------------------------------------------------------------------- */
or_index* or_build(const float* raw, int64_t n, int d, int family, int strategy, int L, int K, int M,
                   int pool_bits, uint64_t seed, int lazy, int cp_draws, int64_t* err_row) {
    or_index* X = (or_index*)calloc(1, sizeof(or_index));
    X->n = n; X->d = d; X->family = family; X->strategy = strategy; X->L = L; X->K = K; X->M = M;
    X->seed = seed; X->cp_draws = cp_draws;
    X->dp = 1; while (X->dp < d) X->dp <<= 1;
    X->ell = (family == OR_HP) ? 1 : 1 + (int)round(log2((double)X->dp));
    X->c = or_funcs_per_rep(K, X->ell);
    X->x = (float*)malloc(sizeof(float) * n * d);
    *err_row = or_normalize(raw, n, d, X->x);
    if (*err_row >= 0) { free(X->x); free(X); return NULL; }
    /* functions (R-3 streams) */
    /* tensor: L an even power of two, S = sqrt(L), two collections of S
     * tuples of c/2 functions; F = S * c functions (R-24) */
    int S = 1;
    while (S * S < L) ++S;
    int64_t F = (strategy == OR_POOL) ? (int64_t)(pool_bits / X->ell)
              : (strategy == OR_TENSOR) ? (int64_t)S * X->c : (int64_t)L * X->c;
    X->m = (strategy == OR_POOL) ? (int)F : 0;
    X->S = (strategy == OR_TENSOR) ? S : 0;
    if (family == OR_HP) {
        uint64_t kh = or_stream_key(seed, OR_TAG_HP);
        X->hp = (float*)malloc(sizeof(float) * F * d);
        for (int64_t i = 0; i < F * d; ++i) X->hp[i] = or_gauss(kh, (uint64_t)i);
    } else if (family == OR_CP) {
        /* exact CP: function f = d hyperplanes of d coordinates, element (f d + i) d + t */
        uint64_t kc = or_stream_key(seed, OR_TAG_CP);
        X->hp = (float*)malloc(sizeof(float) * F * d * d);
        for (int64_t i = 0; i < F * d * d; ++i) X->hp[i] = or_gauss(kc, (uint64_t)i);
    } else {
        uint64_t kf = or_stream_key(seed, OR_TAG_FHT);
        X->sg = (float*)malloc(sizeof(float) * F * 3 * X->dp);
        for (int64_t i = 0; i < F * 3 * X->dp; ++i) X->sg[i] = (or_draw(kf, (uint64_t)i) >> 63) ? -1.0f : 1.0f;
    }
    if (strategy == OR_POOL) {
        /* PAPER.md:886 "random subsets of size K ... from the pool": partial Fisher-Yates,
         * step t swaps position t with t + (draw mod (m - t)) on a fresh identity array. */
        uint64_t kp = or_stream_key(seed, OR_TAG_POOL);
        X->sel = (int32_t*)malloc(sizeof(int32_t) * L * X->c);
        int32_t* perm = (int32_t*)malloc(sizeof(int32_t) * F);
        for (int j = 0; j < L; ++j) {
            for (int64_t f = 0; f < F; ++f) perm[f] = (int32_t)f;
            for (int t = 0; t < X->c; ++t) {
                int64_t r = t + (int64_t)(or_draw(kp, (uint64_t)j * X->c + t) % (uint64_t)(F - t));
                int32_t tmp = perm[t]; perm[t] = perm[r]; perm[r] = tmp;
                X->sel[j * X->c + t] = perm[t];
            }
        }
        free(perm);
    }
    if (strategy == OR_TENSOR) {
        /* trie (j1, j2), j = j1*S + j2, interleaves tuple j1 of the first collection and tuple j2
         * of the second: position t = 2s + a holds function s of collection a's tuple
         * ("taken by interleaving"); function (a, tuple, s) is
         * f = (a*S + tuple)*(c/2) + s */
        int h = X->c / 2;
        X->sel = (int32_t*)malloc(sizeof(int32_t) * L * X->c);
        for (int j = 0; j < L; ++j)
            for (int t = 0; t < X->c; ++t) {
                int a = t % 2, s = t / 2, tuple = a ? j % S : j / S;
                X->sel[j * X->c + t] = (a * S + tuple) * h + s;
            }
    }
    /* sketches: "M 64-bit sketches s_1(p),...,s_M(p) obtained via HP LSH";
     * slot for rep j ("pseudorandom transformation of j", R-20) */
    uint64_t ks = or_stream_key(seed, OR_TAG_SKETCH), kl = or_stream_key(seed, OR_TAG_SLOT);
    X->slot = (int32_t*)malloc(sizeof(int32_t) * L);
    for (int j = 0; j < L; ++j) X->slot[j] = M > 0 ? (int32_t)(or_draw(kl, (uint64_t)j) % (uint64_t)M) : 0;
    if (M > 0) {
        X->skf = (float*)malloc(sizeof(float) * (int64_t)64 * M * d);
        for (int64_t i = 0; i < (int64_t)64 * M * d; ++i) X->skf[i] = or_gauss(ks, (uint64_t)i);
        X->sk = (uint64_t*)malloc(sizeof(uint64_t) * n * M);
        #pragma omp parallel for schedule(static)
        for (int64_t p = 0; p < n; ++p) or_sketch(X, X->x + p * d, X->sk + p * M);
    }
    X->codes = (uint32_t**)calloc(L, sizeof(uint32_t*));
    X->ids = (uint32_t**)calloc(L, sizeof(uint32_t*));
    if (!lazy)
        for (int j = 0; j < L; ++j) or_build_rep(X, j);
    if (family == OR_FHTCP || family == OR_CP) { int e; or_cp_table(family, d, seed, cp_draws, X->cpT, &e); }
    return X;
}

void or_free(or_index* X) {
    if (!X) return;
    for (int j = 0; j < X->L; ++j) { free(X->codes[j]); free(X->ids[j]); }
    free(X->codes); free(X->ids); free(X->x); free(X->sk); free(X->hp); free(X->sg);
    free(X->sel); free(X->slot); free(X->skf); free(X->x16); free(X->fcache); free(X);
}

/* accessors for tests */
void or_info(const or_index* X, int64_t* out) {
    out[0] = X->n; out[1] = X->d; out[2] = X->dp; out[3] = X->ell; out[4] = X->c; out[5] = X->L;
    out[6] = X->K; out[7] = X->M; out[8] = X->m;
}
void or_get_rep(or_index* X, int j, uint32_t* codes, uint32_t* ids) {
    or_need_rep(X, j);
    memcpy(codes, X->codes[j], sizeof(uint32_t) * X->n);
    memcpy(ids, X->ids[j], sizeof(uint32_t) * X->n);
}
void or_get_data(const or_index* X, float* x) { memcpy(x, X->x, sizeof(float) * X->n * X->d); }
/* R-25: inner products on 16-bit fixed-point rows from here on (hashing stays on the fp32 rows) */
void or_set_storage(or_index* X, int storage) {
    X->storage = storage;
    if (storage == 1 && !X->x16) {
        X->x16 = (int16_t*)malloc(sizeof(int16_t) * X->n * X->d);
        or_quantize(X->x, X->n, X->d, X->x16);
    }
}
void or_get_data16(const or_index* X, int16_t* x) { memcpy(x, X->x16, sizeof(int16_t) * X->n * X->d); }
void or_get_sketches(const or_index* X, uint64_t* sk) { memcpy(sk, X->sk, sizeof(uint64_t) * X->n * X->M); }
void or_get_slots(const or_index* X, int32_t* s) { memcpy(s, X->slot, sizeof(int32_t) * X->L); }
void or_get_sel(const or_index* X, int32_t* s) { if (X->sel) memcpy(s, X->sel, sizeof(int32_t) * X->L * X->c); }
void or_get_cp(const or_index* X, double* T) { memcpy(T, X->cpT, sizeof(double) * (X->ell + 1) * 41); }
/* hash raw (un-normalised) vectors: rep codes [nq][L] and sketches [nq][M]; returns zero row or -1 */
int64_t or_hash(const or_index* X, const float* raw, int64_t nq, uint32_t* codes, uint64_t* sk) {
    float* q = (float*)malloc(sizeof(float) * nq * X->d);
    int64_t e = or_normalize(raw, nq, X->d, q);
    if (e < 0) {
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < nq; ++i) {
            for (int j = 0; j < X->L; ++j) codes[i * X->L + j] = or_rep_code(X, j, q + i * X->d);
            if (sk && X->M) or_sketch(X, q + i * X->d, sk + i * X->M);
        }
    }
    free(q);
    return e;
}
/* lexicographic position of each 13-bit prefix: pt[p] = first index whose
 * top-13 bits are >= p, p = 0..8192 (not semantic: the search below binary-searches directly) */
void or_prefix_table(or_index* X, int j, uint32_t* pt) {
    or_need_rep(X, j);
    int sh = X->K - 13;
    int64_t t = 0;
    for (int p = 0; p <= 8192; ++p) {
        while (t < X->n && (int64_t)(X->codes[j][t] >> sh) < p) ++t;
        pt[p] = (uint32_t)t;
    }
}

/* ----------------------------------------------------------------------------
 * Collision probability of an i-bit prefix at inner product ip:
 *   HP: p = 1 - acos(ip)/pi, P_i = p^i  (Charikar)
 *   FHT-CP: ip is rounded DOWN to the grid, b = max{b: ip >= (float)(-1+.05b)};
 *           P_i = T_ell(b)^floor(i/ell) * T_{i mod ell}(b)  (PAPER.md:341-343 bit-wise prefixes)
 * -------------------------------------------------------------------------- */
int or_grid_bucket(float ip) {
    int b = 0;
    for (int a = 0; a <= 40; ++a)
        if (ip >= (float)(-1.0 + 0.05 * a)) b = a;
    return b;
}
double or_P(const or_index* X, int i, float ip) {
    if (X->family == OR_HP) {
        double p = 1.0 - acos((double)ip) / M_PI;
        return pow(p, (double)i);
    }
    int b = or_grid_bucket(ip);
    return pow(X->cpT[X->ell * 41 + b], (double)(i / X->ell)) * X->cpT[(i % X->ell) * 41 + b];
}

/* Stop rule at depth i after j repetitions (1-based) with k-th similarity ip (clamped).
 * rule 2 (independent functions): the two-level bound below, at depth i < K. 
 * rule 0 (R-9, default): the failure bound of Lemma 1's proof, (1 - P_i)^j <= delta
 *   (PAPER.md:220), evaluated as j*log1p(-P) <= log(delta).
 * rule 1: Alg. 1 line 8 literally, j >= ln(1/delta)/P_i.
 * pool (R-10): Cantelli bound of App. B for general delta:
 *   mu = j P_i, E[X1X2] <= P_i prod_f (r + (1-r) p_f), r = c_i/(m - c_i),
 *   F = 1 - mu^2 / (mu + j(j-1) E[X1X2]);  no stop if m < 2 c_i. */
int or_should_stop(const or_index* X, int i, int j, float ip, double delta, int rule) {
    if (X->strategy == OR_TENSOR) {
        /* Alg. 2: after the m = j first tuples of both collections at depth i
         * (i/2 bits from each), fail bound 2(1 - p^{i/2})^m (union over the two collections) */
        double Ph = or_P(X, i / 2, ip);
        (void)rule;
        return log(2.0) + (double)j * log1p(-Ph) <= log(delta);
    }
    double P = or_P(X, i, ip);
    if (X->strategy == OR_POOL) {
        int ci = (i + X->ell - 1) / X->ell;
        if (X->m < 2 * ci || !(P > 0.0)) return 0;
        double r = (double)ci / (double)(X->m - ci);
        double prod = 1.0;
        for (int f = 0; f < ci; ++f) {
            int bits = (f < i / X->ell) ? X->ell : (i % X->ell);
            double pf = or_P(X, bits, ip);
            prod *= r + (1.0 - r) * pf;
        }
        double mu = (double)j * P;
        double e12 = P * prod;
        double F = 1.0 - mu * mu / (mu + (double)j * ((double)j - 1.0) * e12);
        return F <= delta;
    }
    if (rule == 1) return (double)j * P >= log(1.0 / delta);
    if (rule == 2 && i < X->K) {
        /* two-level failure bound (the argument of Lemma 1's proof):
         * a point at inner product >= ip_k is missed only if it collides with the query neither in
         * the j repetitions searched at depth i nor, in the other L - j repetitions, at depth i + 1
         * (all L were searched there before depth i): (1 - P_i)^j (1 - P_{i+1})^(L - j) <= delta */
        double P1 = or_P(X, i + 1, ip);
        return (double)j * log1p(-P) + (double)(X->L - j) * log1p(-P1) <= log(delta);
    }
    return (double)j * log1p(-P) <= log(delta);
}

/* R-15: tau = round-half-up((1+eps) * 64 * acos(ip_k)/pi), at most 64 (PAPER.md:509, 519-523:
 * "1+eps times the expected difference", the expected Hamming distance being 64 (1 - p)). */
int or_tau(float ipk, float eps) {
    double t = (1.0 + (double)eps) * 64.0 * acos((double)ipk) / M_PI;
    double r = floor(t + 0.5);
    if (r > 64.0) r = 64.0;
    if (r < 0.0) r = 0.0;
    return (int)r;
}

/* R-26, the probabilistic reading of PAPER.md:327-328 ("tau ... according to the probability that a
 * vector with Hamming distance tau or less has a dot product larger than the smallest dot product in
 * the current top-k"): the Hamming distance of the 64-bit HP sketches of two unit vectors at inner
 * product s is Binomial(64, acos(s)/pi) (64 independent HP bits), and it
 * is stochastically smaller the larger s is; tau is the smallest t with P[H > t] <= delta_f at
 * s = ip_k, so a vector at least as similar as the current k-th passes with probability >= 1 - delta_f.
 * The search takes delta_f = delta = 1 - recall target.  The upper tail is summed in double from
 * t = 64 down (smallest terms first, so the comparison with delta_f is not decided by rounding:
 * delta_f = 0 gives 64 whenever p > 0). */
double or_binom64(double p, int t) {
    double c = 1.0;
    for (int h = 0; h < t; ++h) c = c * (double)(64 - h) / (double)(h + 1);
    return c * pow(p, (double)t) * pow(1.0 - p, (double)(64 - t));
}
int or_tau_prob(float ipk, double delta_f) {
    double p = acos((double)ipk) / M_PI;
    if (p < 0.0) p = 0.0;
    if (p > 1.0) p = 1.0;
    double tail = 0.0;   /* P[H > t] */
    int t = 64;
    while (t > 0 && tail + or_binom64(p, t) <= delta_f) { tail += or_binom64(p, t); --t; }
    return t;
}

static int or_better(float s1, uint32_t i1, float s2, uint32_t i2) {
    return s1 > s2 || (s1 == s2 && i1 < i2);
}

/* lower_bound on a sorted code array */
static int64_t or_lower_bound(const uint32_t* c, int64_t n, uint64_t v) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if ((uint64_t)c[mid] < v) lo = mid + 1; else hi = mid; }
    return lo;
}

/* R-12 widening of one repetition's emitted range [elo, ehi) to prefix length i
 * ("all tuples whose hash code has a common prefix of length at least i";
 * "every access ... in a segment of size B = 12, regardless of whether the prefix matches";
 * PAPER.md:934 "even if only the first candidate's prefix matches"): extend by whole
 * segments of B while the entry just outside the range shares the top i bits. */
void or_widen(const uint32_t* cj, int64_t n, uint32_t qcode, int K, int i, int B, int64_t* elo, int64_t* ehi) {
    uint32_t qp = (uint32_t)((uint64_t)qcode >> (K - i));
    while (*elo > 0 && (uint32_t)((uint64_t)cj[*elo - 1] >> (K - i)) == qp)
        *elo = *elo - B > 0 ? *elo - B : 0;
    while (*ehi < n && (uint32_t)((uint64_t)cj[*ehi] >> (K - i)) == qp)
        *ehi = *ehi + B < n ? *ehi + B : n;
}
int64_t or_lower_bound_pub(const uint32_t* c, int64_t n, uint64_t v) { return or_lower_bound(c, n, v); }

typedef struct {
    int32_t rep_chunk, stop_rule, per_round, segment, use_filter;
    float eps;
    int32_t uniform_chunks;  /* 0: the search's first chunk is a single repetition (R-17) */
    int32_t sim_order;       /* 0: R-2 lane-tree similarity (or_sim); 1: plain sequential order (or_sim_seq) */
    int32_t tau_rule;        /* 0: probabilistic, the (1 - delta)-quantile (R-26); 1: (1+eps) x expected Hamming distance (R-15) */
    int32_t rerank;          /* storage 1 (16-bit rows): 1 = the returned top-k re-scored with or_sim on the fp32
                                rows and re-sorted */
} or_sopts;

/* ----------------------------------------------------------------------------
 * Query (Alg. 1 over the array form of PAPER.md:281-334 §4.1-4.2).
 *   levels i = K..0; at each level reps j in chunks of R (R-17: tau is frozen per chunk and is 64
 *   while fewer than k points are known; the search's first chunk is the single repetition 0, so
 *   tau is set right after it, close to the paper's refresh after the first k insertions,
 *   unless uniform_chunks);
 *   per rep: widen (R-12: whole segments of B while the boundary entry shares the top i bits,
 *   PAPER.md:313-319, 934); filter popcount(s'(q) ^ s'(p)) <= tau;
 *   never re-evaluate an id; exact fp32 dot; keep the top k_eff by
 *   (sim desc, id asc) (R-19); stop check after every rep (Alg. 1 line 8) or only at
 *   j = L.  At i = 0 (R-13) the first rep is a linear scan of every point
 *   not yet evaluated with the filter off, after which the search stops.
 * trace[8] = {i_stop, j_stop, emitted, filtered, dups, evaluated, flags, 0}
 * -------------------------------------------------------------------------- */
static void or_search_one(or_index* X, const float* qraw, int k, double delta, const or_sopts* o,
                          int64_t* oid, float* osim, int32_t* trace, uint32_t* tids, int tcap) {
    int64_t n = X->n;
    int d = X->d, L = X->L, K = X->K, B = o->segment;
    memset(trace, 0, sizeof(int32_t) * 8);
    float* q = (float*)malloc(sizeof(float) * d);
    if (or_normalize(qraw, 1, d, q) >= 0) {
        for (int t = 0; t < k; ++t) { oid[t] = -1; osim[t] = NAN; }
        trace[6] = 2; free(q); return;
    }
    int k_eff = (int)((int64_t)k < n ? k : n);
    uint32_t* qc = (uint32_t*)malloc(sizeof(uint32_t) * L);
    for (int j = 0; j < L; ++j) qc[j] = or_rep_code(X, j, q);
    uint64_t qs[64];
    if (X->M) or_sketch(X, q, qs);
    int filt = o->use_filter && X->M > 0;
    int16_t* q16 = NULL;
    if (X->storage == 1) {
        q16 = (int16_t*)malloc(sizeof(int16_t) * d);
        or_quantize(q, 1, d, q16);
    }
    float* ts = (float*)malloc(sizeof(float) * (k_eff + 1));
    uint32_t* ti = (uint32_t*)malloc(sizeof(uint32_t) * (k_eff + 1));
    int nt = 0;
    int64_t nE = 0;
    uint8_t* E = (uint8_t*)calloc(n, 1);
    int64_t* elo = (int64_t*)malloc(sizeof(int64_t) * L);
    int64_t* ehi = (int64_t*)malloc(sizeof(int64_t) * L);
    uint8_t* init = (uint8_t*)calloc(L, 1);
    int R = o->rep_chunk < 1 ? 1 : o->rep_chunk;
    int done = 0;
    /* tensor (Alg. 2): depths i = K, K - 2 ell, ..., 0 (i/2 bits from each
     * collection); at each depth the shells m = 1..S add the tries (j, m) and (m, j), j <= m, in
     * the order (1,m), (m,1), (2,m), (m,2), ..., (m,m); tau is frozen per shell (R-17) and the stop
     * check follows each shell */
    const int tensor = X->strategy == OR_TENSOR;
    const int istep = tensor ? 2 * X->ell : 1;
    int list[256];
    for (int i = K; i >= 0 && !done; i -= (i == 0 ? 1 : istep)) {
        if (i < 0) break;
        int Lr = (i == 0) ? 1 : (tensor ? X->S : L);
        for (int c0 = 0, c1 = 0; c0 < Lr && !done; c0 = c1) {
            int tau = 64;
            if (nt == k_eff && i > 0) {
                float ip = ts[k_eff - 1];
                if (ip > 1.0f) ip = 1.0f;
                if (ip < -1.0f) ip = -1.0f;
                tau = o->tau_rule ? or_tau(ip, o->eps) : or_tau_prob(ip, delta);
            }
            int nl;
            if (i > 0 && tensor) {
                nl = 2 * c0 + 1;
                for (int t = 0; t < nl; ++t) list[t] = (t % 2 == 0) ? (t / 2) * X->S + c0 : c0 * X->S + (t - 1) / 2;
                c1 = c0 + 1;
            } else {
                int Rc = (i == K && c0 == 0 && !o->uniform_chunks) ? 1 : R;
                c1 = c0 + Rc < Lr ? c0 + Rc : Lr;
                nl = c1 - c0;
                for (int t = 0; t < nl; ++t) list[t] = c0 + t;
            }
            for (int tl = 0; tl < nl && !done; ++tl) {
                const int j = list[tl];
                or_need_rep(X, j);
                const uint32_t* cj = X->codes[j];
                const uint32_t* ij = X->ids[j];
                int64_t ranges[4]; /* [a0,a1) and [b0,b1) */
                if (i == 0) {
                    ranges[0] = 0; ranges[1] = n; ranges[2] = ranges[3] = 0;
                } else {
                    if (!init[j]) { elo[j] = ehi[j] = or_lower_bound(cj, n, qc[j]); init[j] = 1; }
                    int64_t lo0 = elo[j], hi0 = ehi[j];
                    or_widen(cj, n, qc[j], K, i, B, &elo[j], &ehi[j]);
                    ranges[0] = elo[j]; ranges[1] = lo0; ranges[2] = hi0; ranges[3] = ehi[j];
                }
                for (int rr = 0; rr < 2; ++rr)
                    for (int64_t p = ranges[2 * rr]; p < ranges[2 * rr + 1]; ++p) {
                        uint32_t id = ij[p];
                        trace[2]++;
                        if (filt && i > 0) {
                            int s = X->slot[j];
                            int h = __builtin_popcountll(qs[s] ^ X->sk[(int64_t)id * X->M + s]);
                            if (h > tau) { trace[3]++; continue; }
                        }
                        if (E[id]) { trace[4]++; continue; }
                        E[id] = 1;
                        if (tids && nE < tcap) tids[nE] = id;
                        nE++;
                        float sim = q16 ? or_sim16(q16, X->x16 + (int64_t)id * d, d)
                                  : o->sim_order ? or_sim_seq(q, X->x + (int64_t)id * d, d)
                                                 : or_sim(q, X->x + (int64_t)id * d, d);
                        /* insert into the sorted top list (Alg. 1 lines 6-7) */
                        if (nt < k_eff || or_better(sim, id, ts[k_eff - 1], ti[k_eff - 1])) {
                            int pos = nt < k_eff ? nt : k_eff - 1;
                            while (pos > 0 && or_better(sim, id, ts[pos - 1], ti[pos - 1])) {
                                ts[pos] = ts[pos - 1]; ti[pos] = ti[pos - 1]; --pos;
                            }
                            ts[pos] = sim; ti[pos] = id;
                            if (nt < k_eff) ++nt;
                        }
                    }
                /* Alg. 1 line 8 (Alg. 2: after each shell, j = m) */
                int stop = 0;
                if (i == 0) stop = 1;
                else if (tensor ? (tl == nl - 1 && nt == k_eff) : (nt == k_eff && (!o->per_round || j == L - 1))) {
                    float ip = ts[k_eff - 1];
                    if (ip > 1.0f) ip = 1.0f;
                    if (ip < -1.0f) ip = -1.0f;
                    stop = or_should_stop(X, i, tensor ? c0 + 1 : j + 1, ip, delta, o->stop_rule);
                }
                if (stop) { trace[0] = i; trace[1] = tensor ? c0 + 1 : j + 1; done = 1; }
            }
        }
    }
    trace[5] = (int32_t)nE;
    if (q16 && o->rerank) {
        /* the fixed-point search's top-k, re-scored in fp32 (R-2 order) and re-sorted by
         * (sim desc, id asc) -- insertion sort of nt <= k entries */
        for (int t = 0; t < nt; ++t) ts[t] = or_sim(q, X->x + (int64_t)ti[t] * d, d);
        for (int t = 1; t < nt; ++t) {
            float sv = ts[t]; uint32_t iv = ti[t];
            int u = t;
            while (u > 0 && or_better(sv, iv, ts[u - 1], ti[u - 1])) { ts[u] = ts[u - 1]; ti[u] = ti[u - 1]; --u; }
            ts[u] = sv; ti[u] = iv;
        }
    }
    for (int t = 0; t < k; ++t) {
        if (t < nt) { oid[t] = ti[t]; osim[t] = ts[t]; } else { oid[t] = -1; osim[t] = -INFINITY; }
    }
    if (k > k_eff) trace[6] |= 1;
    free(q); free(qc); free(ts); free(ti); free(E); free(elo); free(ehi); free(init); free(q16);
}

void or_search(or_index* X, const float* qraw, int64_t nq, int k, float recall, const or_sopts* o,
               int nthreads, int64_t* oid, float* osim, int32_t* trace, uint32_t* tids, int tcap) {
    double delta = 1.0 - (double)recall;
    if (nthreads <= 1) {
        for (int64_t i = 0; i < nq; ++i)
            or_search_one(X, qraw + i * X->d, k, delta, o, oid + i * k, osim + i * k, trace + 8 * i,
                          tids ? tids + i * (int64_t)tcap : NULL, tcap);
        return;
    }
    /* repetition tables not built yet are built on first use, one at a time (or_need_rep's
     * critical section) */
    #pragma omp parallel for schedule(dynamic) num_threads(nthreads)
    for (int64_t i = 0; i < nq; ++i)
        or_search_one(X, qraw + i * X->d, k, delta, o, oid + i * k, osim + i * k, trace + 8 * i,
                      tids ? tids + i * (int64_t)tcap : NULL, tcap);
}

/* ----------------------------------------------------------------------------
 * Exact k-NN (the ground truth of PAPER.md:365-367): similarity in double,
 * sum_t (double)q_t (double)x_t, top k by (sim desc, id asc).  x and q are normalised.
 * -------------------------------------------------------------------------- */
void or_bruteforce(const float* x, int64_t n, int d, const float* q, int64_t nq, int k,
                   int64_t* oid, double* osim) {
    #pragma omp parallel for schedule(dynamic)
    for (int64_t i = 0; i < nq; ++i) {
        double* bs = (double*)malloc(sizeof(double) * k);
        int64_t* bi = (int64_t*)malloc(sizeof(int64_t) * k);
        int nb = 0;
        for (int64_t p = 0; p < n; ++p) {
            double s = 0.0;
            for (int t = 0; t < d; ++t) s += (double)q[i * d + t] * (double)x[p * d + t];
            if (nb < k || s > bs[k - 1]) {
                int pos = nb < k ? nb : k - 1;
                while (pos > 0 && s > bs[pos - 1]) { bs[pos] = bs[pos - 1]; bi[pos] = bi[pos - 1]; --pos; }
                bs[pos] = s; bi[pos] = p;
                if (nb < k) ++nb;
            }
        }
        for (int t = 0; t < k; ++t) { oid[i * k + t] = t < nb ? bi[t] : -1; osim[i * k + t] = t < nb ? bs[t] : -INFINITY; }
        free(bs); free(bi);
    }
}
