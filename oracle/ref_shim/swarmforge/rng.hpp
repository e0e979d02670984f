// Shared-RNG harness shim -- TEST INFRASTRUCTURE ONLY.
//
// Placed first on the include path when oracle/Makefile builds the
// "philox" flavour of the reference (oracle/_ref/libsfref_philox.so), so the
// reference's own `#include "swarmforge/rng.hpp"` resolves here instead of
// rng.hpp:1-61.  The interface is the reference's (RngStream{uniform(),
// uniform(lo,hi), seed()}, derive_seed), the seed derivation is unchanged
// (rng.hpp:32-59), and only the generator differs: word i of a stream is
// half (i & 1) of Philox4x32-10 block i >> 1 keyed by the 64-bit seed -- the
// same counter contract the CUDA engine evaluates in registers.  The draw
// ORDER is the reference's, so the harness consumes word i exactly where the
// engine's index algebra says it does.
#pragma once

#include <cstdint>
#include <string_view>

namespace swarmforge {

namespace shim_detail {
inline void philox4x32_10(std::uint32_t c[4], std::uint32_t k0, std::uint32_t k1) {
    for (int round = 0; round < 10; ++round) {
        if (round) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const std::uint64_t p0 = std::uint64_t{0xD2511F53u} * c[0];
        const std::uint64_t p1 = std::uint64_t{0xCD9E8D57u} * c[2];
        const std::uint32_t n0 = static_cast<std::uint32_t>(p1 >> 32) ^ c[1] ^ k0;
        const std::uint32_t n2 = static_cast<std::uint32_t>(p0 >> 32) ^ c[3] ^ k1;
        c[1] = static_cast<std::uint32_t>(p1);
        c[3] = static_cast<std::uint32_t>(p0);
        c[0] = n0;
        c[2] = n2;
    }
}
} // namespace shim_detail

class RngStream {
public:
    explicit RngStream(std::uint64_t seed) : seed_(seed) {}

    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
    std::uint64_t seed() const { return seed_; }
    std::uint64_t drawn() const { return index_; }

private:
    std::uint64_t next() {
        const std::uint64_t i = index_++;
        const std::uint64_t blk = i >> 1;
        if (blk != cached_blk_) {
            block_[0] = static_cast<std::uint32_t>(blk);
            block_[1] = static_cast<std::uint32_t>(blk >> 32);
            block_[2] = 0;
            block_[3] = 0;
            shim_detail::philox4x32_10(block_, static_cast<std::uint32_t>(seed_),
                                       static_cast<std::uint32_t>(seed_ >> 32));
            cached_blk_ = blk;
        }
        return (i & 1) ? ((std::uint64_t{block_[3]} << 32) | block_[2])
                       : ((std::uint64_t{block_[1]} << 32) | block_[0]);
    }

    std::uint64_t seed_;
    std::uint64_t index_ = 0;
    std::uint64_t cached_blk_ = ~std::uint64_t{0};
    std::uint32_t block_[4] = {0, 0, 0, 0};
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
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

} // namespace detail

inline std::uint64_t derive_seed(std::uint64_t root, std::string_view tag) {
    return detail::splitmix64(root ^ detail::fnv1a64(tag));
}

inline std::uint64_t derive_seed(std::uint64_t root, std::string_view tag,
                                 std::uint64_t index) {
    return detail::splitmix64(derive_seed(root, tag) + index);
}

} // namespace swarmforge
