// mt19937.cuh -- the reference's own random stream on the device.
//
// rng.hpp:13-28 draws std::mt19937_64 sequentially.  Its recurrence
//   x[k+312] = x[k+156] ^ twist(x[k], x[k+1])
// makes one 312-word block depend only on the previous block, and the first
// half of a block only on the previous block: a block is two parallel
// half-steps of 156 lanes.  A CTA keeps the generator state in shared memory
// (double-buffered 2 x 312 words) and hands every produced word, tempered, to
// a consumer callback with its stream index -- the engine's index algebra then
// routes it to x / v initialisation or to the step factors, exactly as the
// Philox path routes word i.  Generation is sequential in blocks (the stream
// is), parallel within a block.
#pragma once
#include <cstdint>

namespace sepso {

struct MtState {
    unsigned long long* buf;   // 2 x 312 words (shared memory)
    int cur;                   // which half holds the latest block
    long long blocks;          // blocks generated so far (words [0, 312*blocks) exist)
};

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

__device__ __forceinline__ unsigned long long mt_twist1(unsigned long long a, unsigned long long b,
                                                        unsigned long long m) {
    const unsigned long long y = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
    return m ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

// std::mt19937_64(seed): the standard's seeding recurrence (sequential, one thread).
__device__ inline void mt_seed(MtState& s, unsigned long long seed) {
    if (threadIdx.x == 0) {
        unsigned long long* st = s.buf;                        // seed into half 0
        st[0] = seed;
        for (int i = 1; i < 312; ++i)
            st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + (unsigned long long)i;
    }
    s.cur = 0;
    s.blocks = 0;     // the seeded state is "block -1": its words are never output
    __syncthreads();
}

// Generate the next block into the other half (collective: every thread calls).
__device__ inline void mt_next_block(MtState& s) {
    const unsigned long long* o = s.buf + s.cur * 312;
    unsigned long long* n = s.buf + (s.cur ^ 1) * 312;
    const int t = threadIdx.x;
    if (t < 156) n[t] = mt_twist1(o[t], o[t + 1], o[t + 156]);
    __syncthreads();
    if (t >= 156 && t < 311) n[t] = mt_twist1(o[t], o[t + 1], n[t - 156]);
    if (t == 311) n[311] = mt_twist1(o[311], n[0], n[155]);
    __syncthreads();
    s.cur ^= 1;
    ++s.blocks;
}

// Deliver stream words [from, upto) to consume(index, word): words of the
// latest block first, then new blocks.  `from` must not precede the latest
// block.  Collective (every thread of the CTA calls with the same arguments);
// needs blockDim.x >= 312.
template <class F>
__device__ inline void mt_deliver(MtState& s, long long from, long long upto, F&& consume) {
    const int t = threadIdx.x;
    while (from < upto) {
        while (from >= 312 * s.blocks) mt_next_block(s);     // skips whole blocks too
        const long long b0 = 312 * (s.blocks - 1);
        const long long lo = from > b0 ? from : b0;
        const long long hi = upto < b0 + 312 ? upto : b0 + 312;
        if (t < 312) {
            const long long w = b0 + t;
            if (w >= lo && w < hi) consume(w, mt_temper(s.buf[s.cur * 312 + t]));
        }
        from = hi;
        __syncthreads();
    }
}

} // namespace sepso
