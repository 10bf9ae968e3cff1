// device_common.cuh — device helpers shared by the build and query kernels (product code).
//
// Bit-exactness (R-2, R-6): every floating-point operation whose result decides an
// integer (a hash bit, a cross-polytope index, a stop decision through the k-th similarity) is
// written in a fixed order: sequential fmaf chains for inner products, the radix-2 butterfly
// order h = 1, 2, 4, ... for the Hadamard transform, IEEE double with explicit _rn intrinsics
// for the normalisation.  The library is compiled with --fmad=false so no other a*b+c is fused.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pfg {

constexpr unsigned kFull = 0xffffffffu;

// orderable 32-bit image of a float (larger float -> larger unsigned); -0 is mapped to +0 so the
// order agrees with float comparison (the oracle compares floats, where -0 == +0)
__device__ __forceinline__ uint32_t f2ord(float f) {
    if (f == 0.0f) f = 0.0f;
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    const uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
// top-k key: larger key = better = (similarity desc, id asc)  (R-19)
__device__ __forceinline__ uint64_t make_key(float sim, uint32_t id) {
    return ((uint64_t)f2ord(sim) << 32) | (uint64_t)(~id);
}
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return ~(uint32_t)k; }
__device__ __forceinline__ float key_sim(uint64_t k) { return ord2f((uint32_t)(k >> 32)); }

// programmatic dependent launch: a kernel launched with programmatic stream serialisation may start
// while its predecessor on the stream drains; it waits here (first statement) until the
// predecessor has completed and its writes are visible.  A no-op for a normal launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Fast Hadamard transform over one warp (§4.3; R-6).  Element u of the
// dp-vector lives in lane u / EPL, slot u % EPL (EPL = max(1, dp/32)).  Unnormalised radix-2
// stages h = 1, 2, ..., dp/2; the pair (u, u+h), bit h of u clear, becomes (y_u + y_{u+h},
// y_u - y_{u+h}).  The same pairs are combined in the same stage order as the oracle, so the
// fp32 result is bit-identical.  For dp < 32 only lanes < dp carry data.
template <int EPL>
__device__ __forceinline__ void fht_warp(float (&v)[EPL], int dp, int lane) {
#pragma unroll
    for (int h = 1; h < EPL; h <<= 1) {
#pragma unroll
        for (int s = 0; s < EPL; ++s)
            if (!(s & h)) {
                const float a = v[s], b = v[s + h];
                v[s] = a + b;
                v[s + h] = a - b;
            }
    }
    for (int hl = 1; hl * EPL < dp; hl <<= 1) {
        // lower lane: v + o; upper lane: o - v.  Both as fmaf(sg, v, o) with sg = +-1: the product
        // is exact, so the single rounding equals that of the add / subtract.
        const float sgn = (lane & hl) ? -1.0f : 1.0f;
#pragma unroll
        for (int s = 0; s < EPL; ++s) {
            const float o = __shfl_xor_sync(kFull, v[s], hl);
            v[s] = fmaf(sgn, v[s], o);
        }
    }
}

// Thread-local FHT cross-polytope code (same arithmetic as fhtcp_code_warp, one function per
// thread, the whole DP-vector in registers).  Used to hash query batches for the first
// repetitions eagerly (k_fht_qcodes_g).
template <int DP>
__device__ __forceinline__ uint32_t fhtcp_code_thread(const float* __restrict__ xrow, int d, int ell,
                                                      const uint32_t* __restrict__ sg) {
    constexpr int W = (DP + 31) / 32;
    float y[DP];
#pragma unroll
    for (int u = 0; u < DP; ++u) y[u] = (u < d) ? __ldg(xrow + u) : 0.0f;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        uint32_t wv[W];
#pragma unroll
        for (int k = 0; k < W; ++k) wv[k] = __ldg(sg + r * W + k);
#pragma unroll
        for (int u = 0; u < DP; ++u) y[u] = __uint_as_float(__float_as_uint(y[u]) ^ (((wv[u >> 5] >> (u & 31)) & 1u) << 31));
#pragma unroll
        for (int h = 1; h < DP; h <<= 1) {
#pragma unroll
            for (int u = 0; u < DP; ++u)
                if (!(u & h)) {
                    const float a = y[u], b = y[u + h];
                    y[u] = a + b;
                    y[u + h] = a - b;
                }
        }
    }
    int bi = 0;
    float ba = fabsf(y[0]), bv = y[0];
#pragma unroll
    for (int u = 1; u < DP; ++u) {
        const float a = fabsf(y[u]);
        if (a > ba) { ba = a; bi = u; bv = y[u]; }
    }
    return ((uint32_t)(bv < 0.0f) << (ell - 1)) | (uint32_t)bi;
}

// Cross-polytope hash with three pseudo-random rotations H D_r (§2, 340 §4.3):
// x (d floats, zero-padded to dp) -> y = H D3 H D2 H D1 x; code = (y_a* < 0) << (ell-1) | a*,
// a* = argmax_u |y_u| with ties to the lowest u (R-5: sign in the MSB).
// sg: sign bits [3][W], W = max(1, dp/32); bit u of round r set = coordinate u negated.
// All lanes of the warp must call; all return the code.
template <int EPL>
__device__ __forceinline__ uint32_t fhtcp_code_warp(const float* xrow, int d, int dp, int ell,
                                                    const uint32_t* __restrict__ sg, int lane) {
    float v[EPL];
#pragma unroll
    for (int s = 0; s < EPL; ++s) {
        const int u = lane * EPL + s;
        v[s] = (u < d) ? xrow[u] : 0.0f;
    }
    const int W = (dp + 31) >> 5;
    for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int s = 0; s < EPL; ++s) {
            const int u = lane * EPL + s;
            if (u < dp) {
                const uint32_t bit = (__ldg(sg + r * W + (u >> 5)) >> (u & 31)) & 1u;
                v[s] = __uint_as_float(__float_as_uint(v[s]) ^ (bit << 31));  // * (-1)^bit, exact
            }
        }
        fht_warp<EPL>(v, dp, lane);
    }
    float ba = -1.0f, bv = 0.0f;
    int bi = 0;
#pragma unroll
    for (int s = 0; s < EPL; ++s) {
        const int u = lane * EPL + s;
        if (u < dp) {
            const float a = fabsf(v[s]);
            if (a > ba) { ba = a; bi = u; bv = v[s]; }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const float oa = __shfl_xor_sync(kFull, ba, off);
        const int oi = __shfl_xor_sync(kFull, bi, off);
        const float ov = __shfl_xor_sync(kFull, bv, off);
        if (oa > ba || (oa == ba && oi < bi)) { ba = oa; bi = oi; bv = ov; }
    }
    return ((uint32_t)(bv < 0.0f) << (ell - 1)) | (uint32_t)bi;
}

// FHT-CP repetition codes of repetitions c0 + r, r in [r0, nr), for one query row in shared memory
// (independent strategy: repetition j concatenates functions j*c .. j*c + c - 1, MSB first, R-7).
// The warp hashes 32/TPF repetitions at a time, one lane group per repetition: TPF = max(1, dp/32)
// lanes per group, 32 coordinates per lane (coordinate u = sub*32 + i).  Stages h < 32 run in
// registers; a stage h >= 32 pairs lane sub with sub ^ (h/32) (lower keeps a + b, upper a - b) --
// the same butterflies in the same order as the oracle's radix-2 FHT, so codes are bit-identical
// (R-6).  qc[r] receives the code of repetition c0 + r.  All lanes must call.
template <int TPF>
__device__ __forceinline__ void group_rep_codes(const float* qrow, int d, int dp, int ell, int c, int K,
                                                const uint32_t* __restrict__ sg, int c0, int r0, int nr,
                                                uint32_t* qc, int lane) {
    constexpr int G = 32 / TPF;
    const int g = lane / TPF, sub = lane % TPF;
    const int hm = dp < 32 ? dp : 32;   // coordinates per lane that carry data
    for (int rb = r0; rb < nr; rb += G) {
        const int r = rb + g;
        const bool valid = r < nr;
        uint64_t full = 0;
        for (int t = 0; t < c; ++t) {
            const uint32_t* sf = sg + ((int64_t)(c0 + (valid ? r : r0)) * c + t) * 3 * TPF;
            float y[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int u = sub * 32 + i;
                y[i] = (u < d) ? qrow[u] : 0.0f;
            }
            for (int rr = 0; rr < 3; ++rr) {
                const uint32_t wv = __ldg(sf + rr * TPF + sub);
#pragma unroll
                for (int i = 0; i < 32; ++i) y[i] = __uint_as_float(__float_as_uint(y[i]) ^ ((wv << (31 - i)) & 0x80000000u));
#pragma unroll
                for (int h = 1; h < 32; h <<= 1) {
                    if (h < hm) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!(i & h)) {
                                const float a = y[i], bb = y[i + h];
                                y[i] = a + bb;
                                y[i + h] = a - bb;
                            }
                    }
                }
#pragma unroll
                for (int s = 1; s < TPF; s <<= 1) {
                    const bool up = sub & s;
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float o = __shfl_xor_sync(kFull, y[i], s);
                        y[i] = up ? (o - y[i]) : (y[i] + o);
                    }
                }
            }
            int bi = 0;
            float ba = fabsf(y[0]), bv = y[0];
#pragma unroll
            for (int i = 1; i < 32; ++i) {
                const float a = fabsf(y[i]);
                if (i < hm && a > ba) { ba = a; bi = i; bv = y[i]; }
            }
            bi += sub * 32;
#pragma unroll
            for (int s = 1; s < TPF; s <<= 1) {
                const float oa = __shfl_xor_sync(kFull, ba, s);
                const int oi = __shfl_xor_sync(kFull, bi, s);
                const float ov = __shfl_xor_sync(kFull, bv, s);
                if (oa > ba || (oa == ba && oi < bi)) { ba = oa; bi = oi; bv = ov; }
            }
            full = (full << ell) | (((uint32_t)(bv < 0.0f) << (ell - 1)) | (uint32_t)bi);
        }
        if (valid && sub == 0) qc[r] = (uint32_t)(full >> (c * ell - K));
    }
    __syncwarp();
}

// warp bitonic sort of one u64 per lane, descending across lanes (lane 0 = largest)
__device__ __forceinline__ uint64_t warp_sort_desc(uint64_t key, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint64_t o = __shfl_xor_sync(kFull, key, j);
            const bool desc = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            const uint64_t mx = key > o ? key : o, mn = key > o ? o : key;
            key = (desc == lower) ? mx : mn;
        }
    }
    return key;
}

}  // namespace pfg
