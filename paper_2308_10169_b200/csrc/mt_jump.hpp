// mt_jump.hpp -- jump-ahead polynomials for the mt19937_64 stream (host side;
// mt_jump.cpp).  Polynomials are bit vectors of kMtPolyWords words.
#pragma once
#include <cstdint>
#include <vector>

namespace sepso {

constexpr int kMtDegree = 19937;       // state bits of std::mt19937_64
constexpr int kMtPolyWords = 312;      // 19,968 bits
constexpr int kMaxJumpLevels = 8;      // parallel fills: at most 256 segments
constexpr int kWideJumpLevels = 6;     // beyond 64 segments only for segments of >= 2^20 words

// x^steps mod phi: applying it to the state at word w gives the state at w + steps
std::vector<uint64_t> mt_jump_poly(uint64_t steps);

// x^(quantum * 2^j) mod phi for j = 0 .. levels-1 (cached per process)
const std::vector<std::vector<uint64_t>>& mt_jump_ladder(uint64_t quantum, int levels);

// the same ladder as exponent lists: level j's ascending exponents at
// terms[j * kMtDegree ..], count[j] of them (cached per process)
struct MtJumpTerms {
    std::vector<uint16_t> terms;
    std::vector<int> count;
};
const MtJumpTerms& mt_jump_ladder_terms(uint64_t quantum, int levels);

} // namespace sepso
