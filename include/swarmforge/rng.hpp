// swarmforge/rng.hpp -- drop-in for the reference's rng.hpp:1-61.
//
// Same interface (RngStream{uniform(), uniform(lo, hi), seed()}, derive_seed)
// and seed derivation.  The stream is the engine context's: std::mt19937_64
// (the reference's, default) or the counter-based Philox stream (SEPSO_RNG=
// philox; word i = half (i & 1) of Philox4x32-10 block i >> 1).  drawn() is the
// stream position the device resumes from, so host and device consume the
// identical sequence in the reference's order.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string_view>

namespace swarmforge {

namespace rng_detail {
inline std::uint64_t philox_word(std::uint64_t seed, std::uint64_t index) {
    const std::uint64_t blk = index >> 1;
    std::uint32_t c0 = std::uint32_t(blk), c1 = std::uint32_t(blk >> 32), c2 = 0, c3 = 0;
    std::uint32_t k0 = std::uint32_t(seed), k1 = std::uint32_t(seed >> 32);
    for (int r = 0; r < 10; ++r) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        const std::uint64_t m0 = std::uint64_t(0xD2511F53u) * c0;
        const std::uint64_t m1 = std::uint64_t(0xCD9E8D57u) * c2;
        const std::uint32_t n0 = std::uint32_t(m1 >> 32) ^ c1 ^ k0;
        const std::uint32_t n2 = std::uint32_t(m0 >> 32) ^ c3 ^ k1;
        c1 = std::uint32_t(m1);
        c3 = std::uint32_t(m0);
        c0 = n0;
        c2 = n2;
    }
    return (index & 1) ? ((std::uint64_t(c3) << 32) | c2) : ((std::uint64_t(c1) << 32) | c0);
}
} // namespace rng_detail

class RngStream {
public:
    explicit RngStream(std::uint64_t seed) : seed_(seed), engine_(seed) {
        const char* r = std::getenv("SEPSO_RNG");
        philox_ = r && std::strcmp(r, "philox") == 0;
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
    std::uint64_t seed() const { return seed_; }
    /// Draws consumed so far: the position the engine's index algebra resumes at.
    std::uint64_t drawn() const { return drawn_; }
    /// Advance past n draws the device consumed.
    void skip(std::uint64_t n) {
        if (!philox_) engine_.discard(n);
        drawn_ += n;
    }

private:
    std::uint64_t next() {
        const std::uint64_t i = drawn_++;
        return philox_ ? rng_detail::philox_word(seed_, i) : engine_();
    }
    std::uint64_t seed_;
    std::uint64_t drawn_ = 0;
    bool philox_ = false;
    std::mt19937_64 engine_;
};

namespace detail {
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
inline std::uint64_t fnv1a64(std::string_view s) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char ch : s) {
        h ^= ch;
        h *= 0x100000001b3ull;
    }
    return h;
}
} // namespace detail

inline std::uint64_t derive_seed(std::uint64_t root, std::string_view tag) {
    return detail::splitmix64(root ^ detail::fnv1a64(tag));
}
inline std::uint64_t derive_seed(std::uint64_t root, std::string_view tag, std::uint64_t index) {
    return detail::splitmix64(derive_seed(root, tag) + index);
}

} // namespace swarmforge
