// philox.cuh -- the engine's counter-based random stream (host + device).
//
// Draw contract: word i of the stream keyed by a
// 64-bit seed is half (i & 1) of Philox4x32-10 block i >> 1, with
// counter = (lo32(i >> 1), hi32(i >> 1), 0, 0) and key = (lo32(seed), hi32(seed)).
// u = (word >> 11) * 2^-53 exactly as RngStream::uniform (rng.hpp:18).  Every
// consumer computes the index of the draw it needs from the reference's
// sequential draw order (swarm.hpp:94-132, 59-70; planner.hpp:77-133), so a
// GPU thread reproduces draw i without any sequential state.
#pragma once
#include <cstdint>

#ifndef SEPSO_HD
#ifdef __CUDACC__
#define SEPSO_HD __host__ __device__ __forceinline__
#else
#define SEPSO_HD inline
#endif
#endif

namespace sepso {

SEPSO_HD void philox4x32_10(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3,
                            uint32_t k0, uint32_t k1) {
#if defined(__CUDACC__)
#pragma unroll
#endif
    for (int round = 0; round < 10; ++round) {
        if (round) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
#if defined(__CUDA_ARCH__)
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
        const uint64_t p0 = uint64_t{0xD2511F53u} * c0, p1 = uint64_t{0xCD9E8D57u} * c2;
        const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
        const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
#endif
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c1 = lo1;
        c3 = lo0;
        c0 = n0;
        c2 = n2;
    }
}

/// Word `index` of the stream keyed by `seed`.
SEPSO_HD uint64_t philox_word(uint64_t seed, uint64_t index) {
    const uint64_t blk = index >> 1;
    uint32_t c0 = uint32_t(blk), c1 = uint32_t(blk >> 32), c2 = 0u, c3 = 0u;
    philox4x32_10(c0, c1, c2, c3, uint32_t(seed), uint32_t(seed >> 32));
    return (index & 1) ? ((uint64_t(c3) << 32) | c2) : ((uint64_t(c1) << 32) | c0);
}

/// Both words of block `blk` (draws 2*blk and 2*blk+1) in one Philox call.
SEPSO_HD void philox_pair(uint64_t seed, uint64_t blk, uint64_t& w0, uint64_t& w1) {
    uint32_t c0 = uint32_t(blk), c1 = uint32_t(blk >> 32), c2 = 0u, c3 = 0u;
    philox4x32_10(c0, c1, c2, c3, uint32_t(seed), uint32_t(seed >> 32));
    w0 = (uint64_t(c1) << 32) | c0;
    w1 = (uint64_t(c3) << 32) | c2;
}

/// RngStream::uniform() of a word, rounded to the compute type.
template <class T> SEPSO_HD T unit_from_word(uint64_t w);
template <> SEPSO_HD double unit_from_word<double>(uint64_t w) {
    return double(w >> 11) * 0x1.0p-53;
}
template <> SEPSO_HD float unit_from_word<float>(uint64_t w) {
#if defined(__CUDA_ARCH__)
    return __ull2float_rn(w >> 11) * 0x1.0p-53f;   // == (float)(double)u, single rounding
#else
    return float(double(w >> 11) * 0x1.0p-53);
#endif
}

// rng.hpp:32-59 -- named seed derivation, byte-identical to the reference.
SEPSO_HD uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline uint64_t fnv1a64(const char* s, uint64_t len) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < len; ++i) {
        h ^= static_cast<unsigned char>(s[i]);
        h *= 0x100000001b3ull;
    }
    return h;
}

} // namespace sepso
