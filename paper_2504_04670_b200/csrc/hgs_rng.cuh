// hgs_rng.cuh — random streams shared bit-for-bit by host and device.
//
// Two decision streams are supported, both driving the same partial
// Fisher-Yates "choose k of n, sorted" contract of the reference's
// ChoiceSource (rng.hpp:48-54, rng.cpp:105-119):
//   * xoshiro256** per root, seeded by splitmix64 (rng.cpp:12-41) and resumed
//     across levels (PerRootChoiceSource, rng.hpp:69-82); rejection rule of
//     Rng::bounded (rng.cpp:43-50).
//   * Philox4x32-10 (Random123 constants), counter = {decision, draw,
//     attempt, 'CHOS'} under key = seed — counter
//     based, so any decision can be evaluated independently.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HGS_HD __host__ __device__ __forceinline__
#else
#define HGS_HD inline
#endif

namespace hgs {

constexpr uint32_t kPhiloxTag = 0x43484f53u;  // "CHOS"

HGS_HD uint64_t splitmix64_next(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Rng::derive (rng.cpp:76-85): hash a path of identifiers into a stream seed.
HGS_HD uint64_t derive_seed(uint64_t seed, const uint64_t* path, int len) {
    uint64_t s = seed;
    uint64_t h = splitmix64_next(s);
    for (int i = 0; i < len; ++i) {
        s = h ^ (path[i] + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2));
        h = splitmix64_next(s);
    }
    return h;
}

struct Xoshiro256 {
    uint64_t a, b, c, d;

    HGS_HD void seed(uint64_t s) {
        uint64_t x = s;
        a = splitmix64_next(x);
        b = splitmix64_next(x);
        c = splitmix64_next(x);
        d = splitmix64_next(x);
    }
    HGS_HD static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    HGS_HD uint64_t next() {
        const uint64_t out = rotl(b * 5u, 7) * 9u;
        const uint64_t t = b << 17;
        c ^= a;
        d ^= b;
        b ^= c;
        a ^= d;
        c ^= t;
        d = rotl(d, 45);
        return out;
    }
};

HGS_HD uint64_t mulhi64(uint64_t x, uint64_t y) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(x, y);
#else
    return (uint64_t)(((unsigned __int128)x * y) >> 64);
#endif
}

// x mod m for 1 <= m < 2^32 given recip = floor((2^64-1)/m). The estimate
// q = mulhi(x, recip) is floor(x/m) or one less, so a single correction
// suffices (no 64-bit division on the device).
HGS_HD uint64_t mod_by_recip(uint64_t x, uint64_t m, uint64_t recip) {
    uint64_t r = x - mulhi64(x, recip) * m;
    return r >= m ? r - m : r;
}

HGS_HD uint64_t recip_of(uint64_t m) { return ~0ULL / m; }

// x mod m for 1 <= m < 2^31 (any walk degree): only the low 32 bits of the
// quotient estimate are needed, since x - q*m < 2m < 2^32. Bits 64..95 of
// x*recip from four 32-bit partial products.
HGS_HD uint32_t mod_small(uint64_t x, uint32_t m, uint64_t recip) {
    const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
    const uint32_t rl = (uint32_t)recip, rh = (uint32_t)(recip >> 32);
    const uint64_t t1 = (uint64_t)xl * rh, t2 = (uint64_t)xh * rl;
#if defined(__CUDA_ARCH__)
    const uint32_t t0 = __umulhi(xl, rl);
#else
    const uint32_t t0 = (uint32_t)(((uint64_t)xl * rl) >> 32);
#endif
    const uint64_t mid = (uint64_t)t0 + (uint32_t)t1 + (uint32_t)t2;
    const uint32_t q = xh * rh + (uint32_t)(t1 >> 32) + (uint32_t)(t2 >> 32) + (uint32_t)(mid >> 32);
    const uint32_t r = xl - q * m;
    return r >= m ? r - m : r;
}

// Reject-threshold of Rng::bounded: (0 - m) % m == 2^64 mod m < m. Only
// needs evaluating when the draw itself is < m (probability < m / 2^64).
#if defined(__CUDA_ARCH__)
__device__ __noinline__ bool rejected_slow(uint64_t x, uint64_t m, uint64_t recip) {
    return x < mod_by_recip(0ULL - m, m, recip);
}
#endif
HGS_HD bool rejected(uint64_t x, uint64_t m, uint64_t recip) {
    if (x >= m) return false;
#if defined(__CUDA_ARCH__)
    return rejected_slow(x, m, recip);
#else
    return x < mod_by_recip(0ULL - m, m, recip);
#endif
}

HGS_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        if (round) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
#if defined(__CUDA_ARCH__)
        const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
#else
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
        const uint32_t n0 = hi1 ^ c[1] ^ k0;
        const uint32_t n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
    }
}

// Draw `step` of decision `decision` for a root keyed by `seed`.
HGS_HD uint64_t philox_draw(uint64_t seed, uint32_t decision, uint32_t step, uint32_t attempt) {
    uint32_t c[4] = {decision, step, attempt, kPhiloxTag};
    philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    return ((uint64_t)c[1] << 32) | c[0];
}

}  // namespace hgs
