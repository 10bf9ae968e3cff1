// rng.h — host-side random parameter generation for the index (product code).
//
// DESIGN.md R-3: the paper does not specify how hash functions are drawn.  Every random number is
// the c-th output of a SplitMix64 stream keyed by (seed, tag); Gaussians use Box-Muller in double
// with the host libm.  The oracle (oracle/oracle.c) holds its own, independently written copy of
// the same counter-based generator; the two share no code.  Parameters are generated on the
// host and uploaded, so every shard of a sharded index (same seed) gets identical functions.
#pragma once
#include <cmath>
#include <cstdint>

namespace pfg {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
enum StreamTag : uint64_t {
    kTagHP = 1, kTagSketch = 2, kTagFHT = 3, kTagPool = 4, kTagSlot = 5, kTagTensor = 6, kTagCPMC = 7, kTagCP = 8
};

inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
// c-th output (c = 0, 1, ...) of the SplitMix64 stream with initial state `key`
inline uint64_t draw(uint64_t key, uint64_t c) { return mix64(key + (c + 1) * kGamma); }
inline uint64_t stream_key(uint64_t seed, uint64_t tag) { return draw(seed, tag); }

// standard normal from draws 2i, 2i+1 (Box-Muller, double)
inline double gauss(uint64_t key, uint64_t i) {
    const uint64_t r1 = draw(key, 2 * i), r2 = draw(key, 2 * i + 1);
    const double u1 = (double)((r1 >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double u2 = (double)(r2 >> 11) * (1.0 / 9007199254740992.0);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

}  // namespace pfg
