// kernels_build.cuh — index-building kernels (also used to hash query batches).
//
//  k_normalize   a1: x <- x/|x|, double accumulation, zero-row detection
//  k_hp_bits     a3/a4: SimHash sign bits of a batch of rows against F Gaussian functions
//                (PAPER.md:142-146); an FP32 SIMT GEMM whose per-output accumulation is the
//                canonical sequential fmaf chain over t (R-2), so bits equal the oracle's;
//                also produces the 64-bit sketch words
//  k_codes_from_bits  repetition codes from HP bits (independent or pool selection)
//  k_fht_keys    a3: FHT cross-polytope repetition keys / codes, a lane group
//                per (row, repetition), the transform in registers, rows staged in shared memory
//  k_fht_rep     the same, one warp per row (d' < 32 or > 1024)
//  k_fht_funcs   FHT-CP codes of pool functions (pool strategy)
//  k_pool_codes  repetition codes from pooled FHT-CP function codes
//  k_prefix      a5: 13-bit prefix tabulation of a sorted repetition
//  k_mc_codes    Monte-Carlo CP collision counts
#pragma once
#include "device_common.cuh"

namespace pfg {

// R-25 (PFG_STORAGE_I16, the paper's 16-bit fixed point): v = clamp(rint(x 2^15),
// -2^15, 2^15 - 1) of the normalised fp32 coordinate (x 2^15 is exact; rint = nearest, ties to
// even), rows padded with zeros to dpad16 coordinates
__global__ void k_quantize(const float* __restrict__ x, int64_t n, int dpad, int d, int16_t* __restrict__ out,
                           int dpad16) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * dpad16) return;
    const int64_t r = t / dpad16;
    const int c = (int)(t - r * dpad16);
    const float v = c < d ? x[r * dpad + c] : 0.0f;
    const int q = __float2int_rn(v * 32768.0f);
    out[t] = (int16_t)min(max(q, -32768), 32767);
}

// ---------------------------------------------------------------------------------------------
// a1: out[r][0..d) = (float)((double)x / sqrt(sum_t (double)x_t^2)), sum sequential over t;
// out[r][d..dpad) = 0.  zflag[r] = 1 for a zero row; *zmin = smallest zero row index.
// One thread per row (the double sum is order-dependent, so it is not split across lanes).
__global__ void __launch_bounds__(128) k_normalize(const float* __restrict__ x, int64_t n, int d, int ldx,
                                                  float* __restrict__ out, int dpad, uint8_t* __restrict__ zflag,
                                                  unsigned long long* __restrict__ zmin, int rb) {
    // rb rows per block, staged through shared memory so that the block reads and writes them
    // coalesced; thread r < rb sums its row sequentially in double (the oracle's order)
    extern __shared__ float srow[];   // [rb][d]
    __shared__ double sinv[32];
    __shared__ int szero[32];
    const int64_t r0 = (int64_t)blockIdx.x * rb;
    const int nr = (int)(n - r0 < (int64_t)rb ? n - r0 : (int64_t)rb);
    if (nr <= 0) return;
    for (int e = threadIdx.x; e < nr * d; e += blockDim.x) {
        const int rr = e / d, t = e - rr * d;
        srow[e] = x[(r0 + rr) * ldx + t];
    }
    __syncthreads();
    if ((int)threadIdx.x < nr) {
        const float* row = srow + threadIdx.x * d;
        double s = 0.0;
        for (int t = 0; t < d; ++t) {
            const double v = (double)row[t];
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
        const int64_t r = r0 + threadIdx.x;
        const bool zero = !(s > 0.0);
        if (zflag) zflag[r] = zero ? 1 : 0;
        if (zero) atomicMin(zmin, (unsigned long long)r);
        szero[threadIdx.x] = zero ? 1 : 0;
        sinv[threadIdx.x] = zero ? 1.0 : __dsqrt_rn(s);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nr * dpad; e += blockDim.x) {
        const int rr = e / dpad, t = e - rr * dpad;
        out[(r0 + rr) * dpad + t] = (t < d && !szero[rr]) ? __double2float_rn(__ddiv_rn((double)srow[rr * d + t], sinv[rr]))
                                                          : 0.0f;
    }
}

// ---------------------------------------------------------------------------------------------
// SimHash bits: bit(p, f) = [sum_t X[p][t] * A[f][t] >= 0] with the sum a sequential fmaf chain
// over t = 0..dpad-1 starting at +0 (R-2).  Padding columns are zero in both operands and
// fmaf(0, 0, acc) == acc because the chain never holds -0 (it starts at +0 and an exact-zero
// fma result rounds to +0), so the padded chain equals the oracle's chain over t < d.
// Output: out[p * out_ld + f/8] byte, bit f%8 (so u64 word f/64 holds bit f%64, little endian).
constexpr int GB_M = 128, GB_N = 128, GB_K = 16;
__global__ void __launch_bounds__(256) k_hp_bits(const float* __restrict__ X, int64_t np, int ldx,
                                                 const float* __restrict__ A, int nf, int lda, int kdim,
                                                 uint8_t* __restrict__ out, int64_t out_ld) {
    __shared__ __align__(16) float Xs[GB_K][GB_M + 4];
    __shared__ __align__(16) float As[GB_K][GB_N + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * GB_M;   // rows on x (up to 2^31 - 1 blocks)
    const int f0 = blockIdx.y * GB_N;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    for (int t0 = 0; t0 < kdim; t0 += GB_K) {
#pragma unroll
        for (int e = tid; e < GB_M * GB_K; e += 256) {
            const int r = e >> 4, c = e & 15;
            const int64_t p = p0 + r;
            const int t = t0 + c;
            Xs[c][r] = (p < np && t < kdim) ? __ldg(X + p * ldx + t) : 0.0f;
            const int f = f0 + r;
            As[c][r] = (f < nf && t < kdim) ? __ldg(A + (int64_t)f * lda + t) : 0.0f;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < GB_K; ++c) {
            float xv[8], av[8];
            const float4 x0 = *reinterpret_cast<const float4*>(&Xs[c][ty * 8]);
            const float4 x1 = *reinterpret_cast<const float4*>(&Xs[c][ty * 8 + 4]);
            const float4 a0 = *reinterpret_cast<const float4*>(&As[c][tx * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[c][tx * 8 + 4]);
            xv[0] = x0.x; xv[1] = x0.y; xv[2] = x0.z; xv[3] = x0.w;
            xv[4] = x1.x; xv[5] = x1.y; xv[6] = x1.z; xv[7] = x1.w;
            av[0] = a0.x; av[1] = a0.y; av[2] = a0.z; av[3] = a0.w;
            av[4] = a1.x; av[5] = a1.y; av[6] = a1.z; av[7] = a1.w;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xv[i], av[j], acc[i][j]);
        }
        __syncthreads();
    }
    const int fb = f0 + tx * 8;
    if (fb >= nf) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t p = p0 + ty * 8 + i;
        if (p >= np) continue;
        uint32_t b = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (fb + j < nf && acc[i][j] >= 0.0f) b |= 1u << j;
        out[p * out_ld + (fb >> 3)] = (uint8_t)b;
    }
}

// The same product as k_hp_bits with register double buffering: BK = 8 per step, each thread
// fetches one float4 of X and one of A per step (kdim and both leading dimensions are multiples
// of 8, rows 16-byte aligned) while the previous step is multiplied; accumulation order is the
// canonical sequential chain over t, so the bits are identical to k_hp_bits.
constexpr int GB2_K = 8;
__global__ void __launch_bounds__(256, 2) k_hp_bits2(const float* __restrict__ X, int64_t np, int ldx,
                                                     const float* __restrict__ A, int nf, int lda, int kdim,
                                                     uint8_t* __restrict__ out, int64_t out_ld) {
    __shared__ __align__(16) float Xs[2][GB2_K][GB_M + 4];
    __shared__ __align__(16) float As[2][GB2_K][GB_N + 4];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t p0 = (int64_t)blockIdx.x * GB_M;
    const int f0 = blockIdx.y * GB_N;
    const int lr = tid >> 1, lk = (tid & 1) * 4;   // this thread's load: row lr, columns lk..lk+3
    const bool xok = p0 + lr < np, aok = f0 + lr < nf;
    const float4* xp = reinterpret_cast<const float4*>(X + (p0 + lr) * (int64_t)ldx + lk);
    const float4* ap = reinterpret_cast<const float4*>(A + (int64_t)(f0 + lr) * lda + lk);
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 xv = xok ? __ldg(xp) : z4, av = aok ? __ldg(ap) : z4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;
    const int nk = kdim / GB2_K;
    int buf = 0;
    Xs[0][lk + 0][lr] = xv.x; Xs[0][lk + 1][lr] = xv.y; Xs[0][lk + 2][lr] = xv.z; Xs[0][lk + 3][lr] = xv.w;
    As[0][lk + 0][lr] = av.x; As[0][lk + 1][lr] = av.y; As[0][lk + 2][lr] = av.z; As[0][lk + 3][lr] = av.w;
    __syncthreads();
    for (int s = 0; s < nk; ++s) {
        if (s + 1 < nk) {
            xv = xok ? __ldg(xp + (s + 1) * (GB2_K / 4)) : z4;
            av = aok ? __ldg(ap + (s + 1) * (GB2_K / 4)) : z4;
        }
#pragma unroll
        for (int c = 0; c < GB2_K; ++c) {
            const float4 x0 = *reinterpret_cast<const float4*>(&Xs[buf][c][ty * 8]);
            const float4 x1 = *reinterpret_cast<const float4*>(&Xs[buf][c][ty * 8 + 4]);
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][c][tx * 8]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][c][tx * 8 + 4]);
            const float xr[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
            const float ar[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(xr[i], ar[j], acc[i][j]);
        }
        if (s + 1 < nk) {
            buf ^= 1;
            Xs[buf][lk + 0][lr] = xv.x; Xs[buf][lk + 1][lr] = xv.y; Xs[buf][lk + 2][lr] = xv.z; Xs[buf][lk + 3][lr] = xv.w;
            As[buf][lk + 0][lr] = av.x; As[buf][lk + 1][lr] = av.y; As[buf][lk + 2][lr] = av.z; As[buf][lk + 3][lr] = av.w;
            __syncthreads();
        }
    }
    const int fb = f0 + tx * 8;
    if (fb >= nf) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int64_t p = p0 + ty * 8 + i;
        if (p >= np) continue;
        uint32_t bbits = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (fb + j < nf && acc[i][j] >= 0.0f) bbits |= 1u << j;
        out[p * out_ld + (fb >> 3)] = (uint8_t)bbits;
    }
}

// ---------------------------------------------------------------------------------------------
// HP repetition codes from bits (ell = 1, c = K functions): code_j = bits of functions
// f_{j,0} .. f_{j,K-1}, the first the most significant (R-7).
// Independent: f_{j,t} = (j - fbase_rep) * K + t within the bit batch; pool: sel[j][t].
// out: keys (u64, (code << 32) | p, layout [rep - r0][p]) or codes (u32, layout [p][ldc]).
__global__ void k_codes_from_bits(const uint64_t* __restrict__ bits, int64_t np, int words_per_row,
                                  int r0, int nreps, int K, const int32_t* __restrict__ sel, int rep_fbase,
                                  uint64_t* __restrict__ keys, uint32_t* __restrict__ codes, int ldc) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (p >= np || r >= nreps) return;
    const int j = r0 + r;
    const uint64_t* row = bits + p * words_per_row;
    uint32_t code = 0;
    for (int t = 0; t < K; ++t) {
        const int f = sel ? __ldg(sel + (int64_t)j * K + t) : (j - rep_fbase) * K + t;
        code = (code << 1) | (uint32_t)((__ldg(row + (f >> 6)) >> (f & 63)) & 1ull);
    }
    if (keys) keys[(int64_t)r * np + p] = ((uint64_t)code << 32) | (uint64_t)p;
    if (codes) codes[p * ldc + j] = code;
}

// ---------------------------------------------------------------------------------------------
// FHT-CP repetition codes, independent strategy: rep j concatenates functions j*c .. j*c+c-1
// (ell bits each, first most significant) and keeps the top K bits (R-7).  One warp per row;
// the row's dp-vector lives in registers (EPL per lane).  Outputs keys [rep - r0][p] and/or
// codes [p][ldc].
template <int EPL>
__global__ void __launch_bounds__(256) k_fht_rep(const float* __restrict__ X, int64_t np, int ldx, int d,
                                                 int dp, int ell, int c, int K, const uint32_t* __restrict__ sg,
                                                 int r0, int nreps, uint64_t* __restrict__ keys,
                                                 uint32_t* __restrict__ codes, int ldc) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int W = (dp + 31) >> 5;
    for (int64_t p = warp; p < np; p += nwarps) {
        const float* xr = X + p * ldx;
        for (int r = 0; r < nreps; ++r) {
            const int j = r0 + r;
            uint64_t full = 0;
            for (int t = 0; t < c; ++t) {
                const int64_t f = (int64_t)j * c + t;
                full = (full << ell) | fhtcp_code_warp<EPL>(xr, d, dp, ell, sg + f * 3 * W, lane);
            }
            const uint32_t code = (uint32_t)(full >> (c * ell - K));
            if (lane == 0) {
                if (keys) keys[(int64_t)r * np + p] = ((uint64_t)code << 32) | (uint64_t)p;
                if (codes) codes[p * ldc + j] = code;
            }
        }
    }
}


// Eager FHT-CP query codes, TPF threads per (row, repetition): the TPF consecutive lanes of a group
// hold coordinate blocks [g*H, (g+1)*H) of the same vector (H = DP/TPF).  Stages h < H are in
// registers; a stage h >= H pairs coordinate u of lane g with u + h of lane g + h/H (the lower lane
// keeps a + b, the upper a - b: the oracle's butterfly, same operands, same rounding).  The argmax
// combines the lanes' winners with ties to the lower index (R-6).
// The concatenated FHT-CP codes of one repetition (functions sf[0 .. c), ell bits each, first most
// significant) of the row xr (lim valid floats, zero beyond; 16-byte aligned, global or shared
// memory) by a group of TPF lanes g = 0 .. TPF-1 (see k_fht_qcodes_g).  All lanes of the group call.
template <int DP, int TPF>
__device__ __forceinline__ uint64_t fhtcp_rep_full(const float* xr, int lim, const uint32_t* __restrict__ sg_rep, int c,
                                                   int ell, int g) {
    constexpr int H = DP / TPF, W = (DP + 31) / 32;
    static_assert(H % 32 == 0 || TPF == 1, "a lane holds whole sign words");
    uint64_t full = 0;
    for (int f = 0; f < c; ++f) {
        const uint32_t* sf = sg_rep + (int64_t)f * 3 * W;
        float y[H];
        // rows are zero beyond d (k_normalize), 16-byte aligned: 128-bit loads
#pragma unroll
        for (int i = 0; i < H; i += 4) {
            const int u = g * H + i;
            const float4 v = (u < lim) ? *reinterpret_cast<const float4*>(xr + u) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            y[i] = v.x; y[i + 1] = v.y; y[i + 2] = v.z; y[i + 3] = v.w;
        }
#pragma unroll 1
        for (int r = 0; r < 3; ++r) {
#pragma unroll
            for (int k = 0; k < H / 32; ++k) {
                const uint32_t wv = __ldg(sf + r * W + g * (H / 32) + k);
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    y[k * 32 + i] = __uint_as_float(__float_as_uint(y[k * 32 + i]) ^ ((wv << (31 - i)) & 0x80000000u));
            }
#pragma unroll
            for (int h = 1; h < H; h <<= 1) {
#pragma unroll
                for (int i = 0; i < H; ++i)
                    if (!(i & h)) {
                        const float a = y[i], b = y[i + h];
                        y[i] = a + b;
                        y[i + h] = a - b;
                    }
            }
#pragma unroll
            for (int s = 1; s < TPF; s <<= 1) {
                const bool up = g & s;
#pragma unroll
                for (int i = 0; i < H; ++i) {
                    const float o = __shfl_xor_sync(kFull, y[i], s);
                    y[i] = up ? (o - y[i]) : (y[i] + o);
                }
            }
        }
        int bi = 0;
        float ba = fabsf(y[0]), bv = y[0];
#pragma unroll
        for (int i = 1; i < H; ++i) {
            const float a = fabsf(y[i]);
            if (a > ba) { ba = a; bi = i; bv = y[i]; }
        }
        bi += g * H;
#pragma unroll
        for (int s = 1; s < TPF; s <<= 1) {
            const float oa = __shfl_xor_sync(kFull, ba, s);
            const int oi = __shfl_xor_sync(kFull, bi, s);
            const float ov = __shfl_xor_sync(kFull, bv, s);
            if (oa > ba || (oa == ba && oi < bi)) { ba = oa; bi = oi; bv = ov; }
        }
        full = (full << ell) | (((uint32_t)(bv < 0.0f) << (ell - 1)) | (uint32_t)bi);
    }
    return full;
}

template <int DP, int TPF, bool LOOP = false>
__global__ void __launch_bounds__(128) k_fht_qcodes_g(const float* __restrict__ X, int64_t np, int ldx, int d, int ell,
                                                      int c, int K, const uint32_t* __restrict__ sg, int nreps,
                                                      uint32_t* __restrict__ codes, int ldc,
                                                      const uint32_t* __restrict__ qlist, int r0,
                                                      const uint32_t* __restrict__ np_dev) {
    // rows: qlist[0..np) if given, else 0..np-1; repetitions r0 .. r0 + nreps - 1; TPF lanes per
    // (row, repetition) item.  LOOP: a grid-stride loop over the items (a device-counted list gets
    // a grid sized for its usual length, not its capacity); else one item per lane group
    constexpr int W = (DP + 31) / 32;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int g = (int)(t % TPF);
    if (np_dev) np = min(np, (int64_t)*np_dev);   // rows counted on the device (a list's length)
    const int64_t total = np * nreps, step = LOOP ? ((int64_t)gridDim.x * blockDim.x) / TPF : 0;
    for (int64_t it = t / TPF;; it += step) {
        const bool live = it < total;
        if (__all_sync(kFull, !live)) return;  // the whole warp is past the end
        const int64_t item = live ? it : 0;    // keep the group's lanes in the shuffles; nothing is stored
        const int64_t a = item / nreps;
        const int64_t p = qlist ? (int64_t)qlist[a] : a;
        const int j = r0 + (int)(item % nreps);
        const uint64_t full = fhtcp_rep_full<DP, TPF>(X + p * ldx, ldx, sg + (int64_t)j * c * 3 * W, c, ell, g);
        if (live && g == 0) codes[p * ldc + j] = (uint32_t)(full >> (c * ell - K));
        if (!LOOP) return;
    }
}

// FHT-CP repetition keys / codes (independent strategy): a block stages RB = 128/TPF rows in
// shared memory (coalesced; row stride S floats with S/4 odd, so the lanes' 128-bit reads do not
// conflict) and loops over its repetitions (block column y: repetitions r0 + y*rpb .. + rpb - 1 of
// r0 .. r0 + nreps - 1), one lane group per (row, repetition): the sign words are the same for the
// whole block (broadcast) and each repetition's keys {code << 32 | p} are written coalesced.  Same
// arithmetic as k_fht_rep / the oracle (R-6).  The index build takes every repetition in one
// column; a query batch splits them over columns (few rows, many blocks).
template <int DP, int TPF>
__global__ void __launch_bounds__(128) k_fht_keys(const float* __restrict__ X, int64_t np, int ldx, int dpad, int S,
                                                  int ell, int c, int K, const uint32_t* __restrict__ sg, int r0,
                                                  int nreps, uint64_t* __restrict__ keys, uint32_t* __restrict__ codes,
                                                  int ldc, int rpb) {
    constexpr int RB = 128 / TPF, W = (DP + 31) / 32;
    extern __shared__ __align__(16) float xs[];
    const int64_t p0 = (int64_t)blockIdx.x * RB;
    const int q4 = dpad / 4;
    for (int i = threadIdx.x; i < RB * q4; i += blockDim.x) {
        const int r = i / q4, u = (i - r * q4) * 4;
        const float4 v = p0 + r < np ? __ldg(reinterpret_cast<const float4*>(X + (p0 + r) * ldx + u))
                                     : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        *reinterpret_cast<float4*>(xs + r * S + u) = v;
    }
    __syncthreads();
    const int lr = threadIdx.x / TPF, g = threadIdx.x % TPF;
    const int64_t p = p0 + lr;
    const int rb = blockIdx.y * rpb, re = min(nreps, rb + rpb);
    for (int r = rb; r < re; ++r) {
        const int j = r0 + r;
        const uint64_t full = fhtcp_rep_full<DP, TPF>(xs + lr * S, dpad, sg + (int64_t)j * c * 3 * W, c, ell, g);
        const uint32_t code = (uint32_t)(full >> (c * ell - K));
        if (g == 0 && p < np) {
            if (keys) keys[(int64_t)r * np + p] = ((uint64_t)code << 32) | (uint64_t)p;
            if (codes) codes[p * ldc + j] = code;
        }
    }
}

// FHT-CP codes of the m pool functions for every row: out [p][m] (uint16)
template <int EPL>
__global__ void __launch_bounds__(256) k_fht_funcs(const float* __restrict__ X, int64_t np, int ldx, int d,
                                                   int dp, int ell, int m, const uint32_t* __restrict__ sg,
                                                   uint16_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int W = (dp + 31) >> 5;
    for (int64_t p = warp; p < np; p += nwarps) {
        const float* xr = X + p * ldx;
        for (int f = 0; f < m; ++f) {
            const uint32_t code = fhtcp_code_warp<EPL>(xr, d, dp, ell, sg + (int64_t)f * 3 * W, lane);
            if (lane == 0) out[p * m + f] = (uint16_t)code;
        }
    }
}

// repetition codes from pooled FHT-CP codes: full = concat(fc[p][sel[j][t]]), code = top K bits
// exact cross-polytope (PFG_CROSSPOLYTOPE): function f is d Gaussian hyperplanes
// a_i; value = index of the largest |<a_i, x>| (ties to the lowest i), sign as the most significant
// of ell bits; each <a_i, x> is the sequential fmaf chain over t (R-2 projections).  The
// hyperplanes are stored transposed, AT[f][t][i] (i padded to d32 = 32 ceil(d/32)), so a warp reads
// them coalesced: lane l holds hyperplanes l, l + 32, ... (NI per lane) of 4 rows at once (x[t]
// broadcast), RW NI chains per step; the argmax is reduced across the warp.  Warp per (RW rows,
// function blockIdx.y).
template <int NI, int RW>
__global__ void __launch_bounds__(128) k_cp_funcs(const float* __restrict__ X, int64_t np_, int ldx,
                                                  const float* __restrict__ AT, int nfun, int d, int d32, int ell,
                                                  uint16_t* __restrict__ out, const uint32_t* __restrict__ qlist,
                                                  const uint32_t* __restrict__ np_dev) {
    // rows: 0..np-1, or qlist[0..np) (np from device memory if np_dev); output row = list index
    const int lane = threadIdx.x & 31;
    const int64_t np = np_dev ? (int64_t)*np_dev : np_;
    const int64_t p0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * RW;
    const int f = blockIdx.y;
    if (p0 >= np) return;
    const float* A = AT + (int64_t)f * d * d32;
    const float* xr[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
        const int64_t pr = min(p0 + r, np - 1);
        xr[r] = X + (qlist ? (int64_t)qlist[pr] : pr) * ldx;
    }
    float s[RW][NI];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int k = 0; k < NI; ++k) s[r][k] = 0.0f;
    for (int t = 0; t < d; ++t) {
        float a[NI];
#pragma unroll
        for (int k = 0; k < NI; ++k) a[k] = __ldg(A + (int64_t)t * d32 + k * 32 + lane);
#pragma unroll
        for (int r = 0; r < RW; ++r) {
            const float xv = __ldg(xr[r] + t);
#pragma unroll
            for (int k = 0; k < NI; ++k) s[r][k] = fmaf(a[k], xv, s[r][k]);
        }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
        float best = -1.0f;
        int bi = 0;
        bool neg = false;
#pragma unroll
        for (int k = 0; k < NI; ++k) {
            const int i = k * 32 + lane;
            if (i < d && fabsf(s[r][k]) > best) { best = fabsf(s[r][k]); bi = i; neg = s[r][k] < 0.0f; }
        }
        // warp argmax: larger |y|, ties to the lower index
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            const bool on = __shfl_xor_sync(0xffffffffu, neg ? 1 : 0, off) != 0;
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; neg = on; }
        }
        if (lane == 0 && p0 + r < np) out[(p0 + r) * nfun + f] = (uint16_t)((neg ? 1u << (ell - 1) : 0u) | (uint32_t)bi);
    }
}

__global__ void k_pool_codes(const uint16_t* __restrict__ fc, int64_t np_, int m, int r0, int nreps, int c,
                             int ell, int K, const int32_t* __restrict__ sel, uint64_t* __restrict__ keys,
                             uint32_t* __restrict__ codes, int ldc, const uint32_t* __restrict__ qlist = nullptr,
                             const uint32_t* __restrict__ np_dev = nullptr, int fbase = 0) {
    // fc row p holds functions [fbase, fbase + m); the codes go to row qlist[p] (or p)
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    const int64_t np = np_dev ? (int64_t)*np_dev : np_;
    if (p >= np || r >= nreps) return;
    const int j = r0 + r;
    uint64_t full = 0;
    for (int t = 0; t < c; ++t) full = (full << ell) | __ldg(fc + p * m + __ldg(sel + (int64_t)j * c + t) - fbase);
    const uint32_t code = (uint32_t)(full >> (c * ell - K));
    if (keys) keys[(int64_t)r * np + p] = ((uint64_t)code << 32) | (uint64_t)p;
    if (codes) codes[(qlist ? (int64_t)qlist[p] : p) * ldc + j] = code;
}

// ---------------------------------------------------------------------------------------------
// repetition table entries (16 B): the sorted key (code << 32 | id) and the sketch word of the
// repetition's slot for that id, s_{slot(j)}(id) (R-21: stored inline
// so the query reads it with the entry instead of a random 8-byte load)
__global__ void k_entries(const uint64_t* __restrict__ keys, int64_t n, const uint64_t* __restrict__ sk, int M,
                          int slot, uint64_t* __restrict__ tab) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t key = keys[t];
    const uint64_t w = M > 0 ? __ldg(sk + (int64_t)(uint32_t)key * M + slot) : 0ull;
    reinterpret_cast<ulonglong2*>(tab)[t] = make_ulonglong2(key, w);
}

// ---------------------------------------------------------------------------------------------
// a5: pt[q] = first position whose top-13 code bits are >= q, q = 0..8192.
__global__ void k_prefix(const uint64_t* __restrict__ tab, int64_t n, int K, uint32_t* __restrict__ pt) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t > n) return;
    const int sh = K - 13;
    const int64_t cur = (t < n) ? (int64_t)((uint32_t)(tab[t] >> 32) >> sh) : 8192;
    const int64_t prev = (t == 0) ? -1 : (int64_t)((uint32_t)(tab[t - 1] >> 32) >> sh);
    for (int64_t q = prev + 1; q <= cur; ++q) pt[q] = (uint32_t)t;
}

// ---------------------------------------------------------------------------------------------
// Monte-Carlo collision counts (R-14 random pairs): pair e = a*draws + t has
// rows x = XY[2e], y = XY[2e+1] (d floats each, stride ld) and its own function signs
// sg[e][3][W]; cnt[b*41 + a] += 1 when the first b of ell bits agree.
template <int EPL>
__global__ void __launch_bounds__(256) k_mc_codes(const float* __restrict__ XY, int ld, int64_t npairs, int d,
                                                  int dp, int ell, int draws, const uint32_t* __restrict__ sg,
                                                  unsigned long long* __restrict__ cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int W = (dp + 31) >> 5;
    for (int64_t e = warp; e < npairs; e += nwarps) {
        const uint32_t* s = sg + e * 3 * W;
        const uint32_t hx = fhtcp_code_warp<EPL>(XY + (2 * e) * ld, d, dp, ell, s, lane);
        const uint32_t hy = fhtcp_code_warp<EPL>(XY + (2 * e + 1) * ld, d, dp, ell, s, lane);
        const int a = (int)(e / draws);
        if (lane >= 1 && lane <= ell) {
            const int b = lane;
            if ((hx >> (ell - b)) == (hy >> (ell - b))) atomicAdd(cnt + b * 41 + a, 1ull);
        }
    }
}

}  // namespace pfg
