// mt19937.cuh -- the reference's own random stream on the device.
//
// rng.hpp:13-28 draws std::mt19937_64 sequentially.  Its recurrence
//   x[k+312] = x[k+156] ^ twist(x[k], x[k+1])
// makes each 312-word block a function of the previous block alone; expanding
// it once more gives the NEXT TWO blocks from the latest one, so a group of 156
// lanes produces 624 words per pass with one barrier (mt_quad).  A CTA
// keeps the state in shared memory (two pairs of blocks, double-buffered) and
// hands every produced word, tempered, to a consumer callback with its stream
// offset -- the engine's index algebra then routes it to x / v initialisation
// or to the step factors, exactly as the Philox path routes word i.
// Generation is sequential in passes (the stream is), parallel within a pass.
#pragma once
#include <cstdint>

namespace sepso {

// State: buf = 2 pairs x 2 blocks x 312 words (shared memory, 10 KB).  Pair
// `cur` holds blocks (blocks-2, blocks-1), the later one in slot 1; after
// seeding, slot 1 of pair 0 holds the seeded state ("block -1", never output).
struct MtState {
    unsigned long long* buf;
    int cur;
    long long blocks;          // blocks generated so far (even; words [0, 312*blocks) exist)
};
constexpr int kMtStateWords = 4 * 312;

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

// A generator group: threads whose local index lt runs over [0, n), synchronised
// by named barrier `bar` (0 = the whole CTA, __syncthreads).  n is a multiple
// of 32; every thread of the group calls the functions below.
struct MtGroup {
    int lt, n, bar;
};

__device__ __forceinline__ void mt_sync(const MtGroup& g) {
    if (g.bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(g.bar), "r"(g.n) : "memory");
}

// std::mt19937_64(seed): the standard's seeding recurrence, sequential, by one
// thread into st[0..311] (slot 1 of pair 0 of an MtState buffer).
__device__ inline void mt_seed_words(unsigned long long* st, unsigned long long seed) {
    unsigned long long x = seed;
    st[0] = x;
    for (int i = 1; i < 312; ++i) {
        x = 6364136223846793005ull * (x ^ (x >> 62)) + (unsigned long long)i;
        st[i] = x;
    }
}

__device__ inline void mt_seed(MtState& s, const MtGroup& g, unsigned long long seed) {
    if (g.lt == 0) mt_seed_words(s.buf + 312, seed);
    s.cur = 0;
    s.blocks = 0;
    mt_sync(g);
}

// The two blocks after block o (x[B..B+311]) for lane t in [0, 156):
//   a = x[B+312+t]  b = x[B+468+t]   (next block, words t and t+156)
//   c = x[B+624+t]  d = x[B+780+t]   (the block after, words t and t+156)
// with  a  = T(o[t], o[t+1], o[t+156]),  a1 = x[B+313+t] (lane t+1's a),
//       b  = T(o[t+156], x[B+157+t], a), b1 = x[B+469+t] (lane t+1's b),
//       c  = T(a, a1, b),                d  = T(b, b1, c),
// T(p, q, m) = m ^ twist(p, q).  Lanes 154 and 155 reach past the block end:
// there x[B+312] = n0 and x[B+313] = n1 are recomputed from o (mt_quad_any).
struct MtQuad {
    unsigned long long a, b, c, d;
};

// Lane t's words given P = x[B+157+t] and Q = x[B+158+t].
__device__ __forceinline__ MtQuad mt_quad(const unsigned long long* o, int t, unsigned long long P,
                                          unsigned long long Q) {
    MtQuad r;
    r.a = mt_twist1(o[t], o[t + 1], o[t + 156]);
    const unsigned long long a1 = mt_twist1(o[t + 1], o[t + 2], P);
    r.b = mt_twist1(o[t + 156], P, r.a);
    const unsigned long long b1 = mt_twist1(P, Q, a1);
    r.c = mt_twist1(r.a, a1, r.b);
    r.d = mt_twist1(r.b, b1, r.c);
    return r;
}

// Any lane t in [0, 156), branch-free: n0 / n1 are selected for t = 154, 155.
__device__ __forceinline__ MtQuad mt_quad_any(const unsigned long long* o, int t) {
    const unsigned long long n0 = mt_twist1(o[0], o[1], o[156]);
    const unsigned long long n1 = mt_twist1(o[1], o[2], o[157]);
    const unsigned long long p = o[t < 155 ? t + 157 : 311], q = o[t < 154 ? t + 158 : 311];
    const unsigned long long P = t < 155 ? p : n0;
    const unsigned long long Q = t < 154 ? q : (t == 154 ? n0 : n1);
    return mt_quad(o, t, P, Q);
}

__device__ __forceinline__ void mt_store_quad(unsigned long long* nb, int t, const MtQuad& q) {
    nb[t] = q.a; nb[156 + t] = q.b; nb[312 + t] = q.c; nb[468 + t] = q.d;
}

// Words of a stored pair (624 words, first at stream offset rel from `from`)
// that fall in [0, len), handed to the sink by the group's threads -- by the
// threads beyond the four compute warps when the group has them, so delivery
// stays off the generation chain.
// GEN: the group's generating lanes (128, or 96 for the three-warp step
// generator); lanes beyond them, when the group has some, deliver alone.
template <bool RAW = false, int GEN = 128, class Sink>
__device__ __forceinline__ void mt_deliver_pair(const unsigned long long* pr, long long rel, int len,
                                                const MtGroup& g, Sink& sink) {
    const int lo = rel < 0 ? int(-rel) : 0;
    const long long hi_ = (long long)len - rel;
    const int hi = hi_ < 624 ? int(hi_) : 624;
    const bool helpers = GEN == 96 ? g.n > 96 : g.n >= 256;
    const int dl = helpers ? g.lt - GEN : g.lt, dn = helpers ? g.n - GEN : g.n;
    if (dl < 0) return;
    for (int i = lo + dl; i < hi; i += dn) sink(int(rel + i), RAW ? pr[i] : mt_temper(pr[i]));
}

// Deliver stream words [from, upto) to sink(w - from, tempered word) (callers
// keep upto - from < 2^31).  Each pass produces the next two blocks with one
// barrier.  A group of >= 128 threads maps lane t = lt (0..127) to warps 0..3
// -- one warp per SM sub-partition -- and the 28 lanes t = 128..155 to lanes
// 0..6 of each warp as a second, independent chain (ILP), so no sub-partition
// issues more than one warp's work.  The words of pass j are delivered from
// shared memory during pass j+1 (the pair stays intact until pass j+2).  The
// sink's writes are complete when every group thread has returned; callers
// synchronise before reading them.
// FN > 0: the group is known to have FN >= 128 threads (fast path only).
// RAW: words are handed over untempered (the consumer applies mt_temper).
template <int FN = 0, bool RAW = false, class Sink>
__device__ inline void mt_generate(MtState& s, const MtGroup& g, long long from, long long upto,
                                   Sink&& sink) {
    const int len = int(upto - from);
    long long rel = 312 * s.blocks - from;        // offset of the next new word
    bool pend = s.blocks > 0 && rel > 0 && rel - 624 < len;   // the latest pair
    long long prel = rel - 624;
    if (FN == 96 || FN == 97) {
        // three warps (the step generator off the first SM sub-partition, whose
        // warp runs the serial best update): lanes 0..95 take positions
        // 0..95, lanes 0..59 also 96..155; FN 97: lanes 96.. (helper warps)
        // only deliver
        const int lt = g.lt;
        const bool gen = FN == 96 || lt < 96;
        const bool second = lt < 60;
        const int t2 = second ? 96 + lt : 96;
        while (rel < len) {
            const unsigned long long* o = s.buf + s.cur * 624 + 312;
            unsigned long long* nb = s.buf + (s.cur ^ 1) * 624;
            if (gen) {
                const MtQuad q1 = mt_quad(o, lt, o[lt + 157], o[lt + 158]);
                if (second) mt_store_quad(nb, t2, mt_quad_any(o, t2));
                mt_store_quad(nb, lt, q1);
            }
            if (pend) mt_deliver_pair<RAW, FN == 97 ? 96 : 128>(s.buf + s.cur * 624, prel, len, g, sink);
            mt_sync(g);
            s.cur ^= 1;
            s.blocks += 2;
            prel = rel;
            pend = rel + 624 > 0;
            rel += 624;
        }
    } else if (FN >= 128 || g.n >= 128) {
        const int lt = g.lt;
        const bool act = lt < 128;
        const int w = lt >> 5, l = lt & 31;
        const bool second = act && l < 7;
        const int t2 = second ? 128 + 7 * w + l : 128;
        while (rel < len) {
            const unsigned long long* o = s.buf + s.cur * 624 + 312;
            unsigned long long* nb = s.buf + (s.cur ^ 1) * 624;
            if (act) {
                const MtQuad q1 = mt_quad(o, lt, o[lt + 157], o[lt + 158]);
                const MtQuad q2 = mt_quad_any(o, t2);
                mt_store_quad(nb, lt, q1);
                if (second) mt_store_quad(nb, t2, q2);
            }
            if (pend) mt_deliver_pair<RAW>(s.buf + s.cur * 624, prel, len, g, sink);
            mt_sync(g);
            s.cur ^= 1;
            s.blocks += 2;
            prel = rel;
            pend = rel + 624 > 0;
            rel += 624;
        }
    } else if (FN == 0) {
        while (rel < len) {
            const unsigned long long* o = s.buf + s.cur * 624 + 312;
            unsigned long long* nb = s.buf + (s.cur ^ 1) * 624;
            for (int t = g.lt; t < 156; t += g.n) mt_store_quad(nb, t, mt_quad_any(o, t));
            if (pend) mt_deliver_pair<RAW>(s.buf + s.cur * 624, prel, len, g, sink);
            mt_sync(g);
            s.cur ^= 1;
            s.blocks += 2;
            prel = rel;
            pend = rel + 624 > 0;
            rel += 624;
        }
    }
    if (pend) mt_deliver_pair<RAW, FN == 97 ? 96 : 128>(s.buf + s.cur * 624, prel, len, g, sink);
}

} // namespace sepso
