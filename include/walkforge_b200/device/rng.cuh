// Device SplitMix64 — the reference's RngStream (proj/include/walkforge/rng.hpp:19-67)
// restated for one walker per lane.  The 64-bit state lives in a register; the
// draw counter (rng.hpp:51) is test-only in the reference and is dropped.
// Keeping the exact generator (not Philox / a (query, step) hash) is what makes
// device walks bit-identical to the reference's.
#pragma once

#include <cstdint>

namespace wf {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;      // rng.hpp:62
constexpr uint64_t kStreamSalt = 0xA3EC647659359ACDULL; // rng.hpp:63
constexpr uint64_t kTwo53 = 1ULL << 53;

__host__ __device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {  // rng.hpp:55-59
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// mix(seed + gamma): constant per run, computed once on the host.
__host__ __device__ __forceinline__ uint64_t seed_premix(uint64_t seed) {
    return splitmix_mix(seed + kGamma);
}

// RngStream(seed, stream) state, rng.hpp:23-24, given seed_premix(seed).
__host__ __device__ __forceinline__ uint64_t stream_state(uint64_t premixed_seed, uint64_t stream) {
    return splitmix_mix(premixed_seed ^ splitmix_mix(stream ^ kStreamSalt));
}

struct Rng {
    uint64_t s;

    __device__ __forceinline__ uint64_t next() {  // rng.hpp:26-30
        s += kGamma;
        return splitmix_mix(s);
    }
    // The next draw without taking it (same value next() will return).
    __device__ __forceinline__ uint64_t peek() const { return splitmix_mix(s + kGamma); }
    // uniform_index, rng.hpp:34-38: (r * n) >> 64.
    __device__ __forceinline__ uint32_t index(uint32_t n) {
        return static_cast<uint32_t>(__umul64hi(next(), static_cast<uint64_t>(n)));
    }
    // 53-bit integer k of uniform_real: u = k * 2^-53 exactly (rng.hpp:44).
    __device__ __forceinline__ uint64_t bits53() { return next() >> 11; }
    // uniform_real(bound), rng.hpp:42-47, bit-exact in fp64 (no FMA contraction
    // is possible: one multiply, one compare).
    __device__ __forceinline__ double real(double bound) {
        double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
        double x = __dmul_rn(u, bound);
        return x < bound ? x : nextafter(bound, 0.0);
    }
};

// uniform_real(1.0) < c  <=>  k < ceil(c * 2^53)   for c in [0, 1]
// (u = k*2^-53 is exact and u*1.0 == u, so the clamp never fires; c*2^53 is an
// exact power-of-two scaling).  Verified bit-exact against the reference in the
// survey (40 M cases) and re-checked by tests/test_engine_gpu.py.
__host__ __device__ inline uint64_t unit_threshold(double c) {
    if (!(c > 0.0)) return 0;
    if (c >= 1.0) return kTwo53;
    double x = c * 9007199254740992.0;  // 2^53
    uint64_t t = static_cast<uint64_t>(x);
    return (static_cast<double>(t) < x) ? t + 1 : t;
}

}  // namespace wf
