// mt_jump.cpp -- jump-ahead polynomials for the device mt19937_64 stream.
//
// std::mt19937_64 (the reference's stream, rng.hpp:13-28) is a linear map A on
// a 19937-bit state.  With phi the characteristic polynomial of A and
// g = x^W mod phi, A^W = g(A), so the state W steps ahead is
//   s_W = XOR over {i : g_i = 1} of s_i,
// and s_i is simply the window x[i .. i+311] of the raw sequence.  The device
// applies g by generating 19937 + 312 raw words and XOR-ing the selected
// windows (stage_kernels.cu, k_mt_jump); a long fill is then split into
// segments generated in parallel from jumped states (stage_mt_fill_parallel).
// The stream itself is unchanged: the jump is exact, checked word for word
// against the sequential generator (tests/test_mt_jump_cpu.py,
// tests/test_gpu_mt.py).
//
// phi is recovered once per process by Berlekamp-Massey from 2 x 19937 output
// bits of std::mt19937_64 (irreducible, so any output bit sequence has phi as
// its minimal polynomial); polynomials over GF(2) are bit vectors.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <vector>

#include "mt_jump.hpp"

namespace sepso {
namespace {

using Bits = std::vector<uint64_t>;

inline bool bit(const Bits& a, long i) { return (a[size_t(i >> 6)] >> (i & 63)) & 1u; }

// 64 bits of a starting at bit position `pos` (zero beyond the end)
inline uint64_t window64(const Bits& a, long pos) {
    const size_t q = size_t(pos >> 6);
    const int r = int(pos & 63);
    const uint64_t lo = q < a.size() ? a[q] : 0, hi = q + 1 < a.size() ? a[q + 1] : 0;
    return r ? (lo >> r) | (hi << (64 - r)) : lo;
}

// a ^= b << s (bit shift) for the low bbits bits of b; bits beyond a are dropped
void xor_shifted(Bits& a, const Bits& b, long s, long bbits) {
    if (bbits <= 0 || s < 0 || size_t(s >> 6) >= a.size()) return;
    const size_t q = size_t(s >> 6);
    const int r = int(s & 63);
    const size_t nb = std::min(b.size(), size_t((bbits + 63) >> 6));
    for (size_t k = 0; k < nb; ++k) {
        const uint64_t w = b[k];
        if (q + k < a.size()) a[q + k] ^= r ? (w << r) : w;
        if (r && q + k + 1 < a.size()) a[q + k + 1] ^= w >> (64 - r);
    }
}

// phi, degree kMtDegree, bit i = coefficient of x^i
const Bits& char_poly() {
    static Bits phi;
    static std::once_flag once;
    std::call_once(once, [] {
        const long n = 2L * kMtDegree + 128;
        // reversed output-bit sequence: rs bit j = s[n - 1 - j]
        Bits rs(size_t((n + 63) / 64), 0);
        std::mt19937_64 eng(5489u);
        for (long i = 0; i < n; ++i)
            if (eng() & 1u) rs[size_t((n - 1 - i) >> 6)] |= 1ull << ((n - 1 - i) & 63);
        const size_t cw = size_t((kMtDegree + 1 + 64) / 64) + 1;
        Bits C(cw, 0), B(cw, 0), T;
        C[0] = B[0] = 1;
        long L = 0, m = 1;
        for (long N = 0; N < n; ++N) {
            // d = sum_{i=0..L} c_i s[N-i] = parity(C & rs >> (n-1-N))
            uint64_t acc = 0;
            const long base = n - 1 - N;
            for (long k = 0; k <= L / 64; ++k) acc ^= C[size_t(k)] & window64(rs, base + 64 * k);
            if (!(__builtin_popcountll(acc) & 1)) {
                ++m;
            } else if (2 * L <= N) {
                T = C;
                xor_shifted(C, B, m, long(cw) * 64 - m);
                L = N + 1 - L;
                B = T;
                m = 1;
            } else {
                xor_shifted(C, B, m, long(cw) * 64 - m);
                ++m;
            }
        }
        // phi(x) = x^L C(1/x): coefficient of x^(L - i) is c_i
        phi.assign(size_t(kMtPolyWords) + 1, 0);
        for (long i = 0; i <= L; ++i)
            if (bit(C, i)) phi[size_t((L - i) >> 6)] |= 1ull << ((L - i) & 63);
    });
    return phi;
}

// a (any length) mod phi, in place; result in the low kMtPolyWords words
void reduce(Bits& a) {
    const Bits& phi = char_poly();
    for (long w = long(a.size()) - 1; w >= 0; --w) {
        while (true) {
            const uint64_t v = a[size_t(w)];
            if (!v) break;
            const long top = w * 64 + 63 - __builtin_clzll(v);
            if (top < kMtDegree) break;
            xor_shifted(a, phi, top - kMtDegree, kMtDegree + 1);
        }
    }
    a.resize(size_t(kMtPolyWords));
}

Bits square_mod(const Bits& a) {
    Bits s(2 * a.size(), 0);
    for (size_t k = 0; k < a.size(); ++k) {
        uint64_t w = a[k];
        uint64_t lo = 0, hi = 0;
        for (int b = 0; b < 32; ++b) {
            lo |= ((w >> b) & 1u) << (2 * b);
            hi |= ((w >> (b + 32)) & 1u) << (2 * b);
        }
        s[2 * k] = lo;
        s[2 * k + 1] = hi;
    }
    reduce(s);
    return s;
}

Bits times_x_mod(const Bits& a) {
    Bits s(a.size() + 1, 0);
    xor_shifted(s, a, 1, long(a.size()) * 64);
    reduce(s);
    return s;
}

} // namespace

std::vector<uint64_t> mt_jump_poly(uint64_t steps) {
    Bits r(size_t(kMtPolyWords), 0);
    r[0] = 1;                                    // x^0
    for (int b = 63; b >= 0; --b) {
        r = square_mod(r);
        if ((steps >> b) & 1u) r = times_x_mod(r);
    }
    return r;
}

const std::vector<std::vector<uint64_t>>& mt_jump_ladder(uint64_t quantum, int levels) {
    // x^(quantum * 2^j) mod phi for j < levels, cached per (quantum, levels)
    static std::mutex mu;
    static std::map<std::pair<uint64_t, int>, std::vector<std::vector<uint64_t>>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({quantum, levels});
    if (it != cache.end()) return it->second;
    std::vector<std::vector<uint64_t>> polys;
    Bits p = mt_jump_poly(quantum);
    for (int j = 0; j < levels; ++j) {
        polys.push_back(p);
        if (j + 1 < levels) p = square_mod(p);
    }
    return cache.emplace(std::make_pair(quantum, levels), std::move(polys)).first->second;
}

const MtJumpTerms& mt_jump_ladder_terms(uint64_t quantum, int levels) {
    const std::vector<std::vector<uint64_t>>& ladder = mt_jump_ladder(quantum, levels);
    static std::mutex mu;
    static std::map<std::pair<uint64_t, int>, MtJumpTerms> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({quantum, levels});
    if (it != cache.end()) return it->second;
    MtJumpTerms t;
    t.terms.assign(size_t(levels) * kMtDegree, 0);
    t.count.assign(size_t(levels), 0);
    for (int j = 0; j < levels; ++j) {
        uint16_t* e = t.terms.data() + size_t(j) * kMtDegree;
        for (int b = 0; b < kMtDegree; ++b)
            if (ladder[size_t(j)][size_t(b) >> 6] >> (b & 63) & 1u) e[t.count[size_t(j)]++] = uint16_t(b);
    }
    return cache.emplace(std::make_pair(quantum, levels), std::move(t)).first->second;
}

} // namespace sepso
