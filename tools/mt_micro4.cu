// Micro-benchmark: latency of one mt19937_64 quad pass (one warp, 32 lanes).
#include <cstdio>
#include <cstdlib>
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;

// the twist is GF(2)-linear: T(p, q, m) = m ^ A(p) ^ B(q)
__device__ __forceinline__ unsigned long long mA(unsigned long long x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    const uint32_t f = __funnelshift_r(lo, hi, 1);
    return (unsigned long long)(hi >> 1) << 32 | (f & 0xC0000000u);
}
__device__ __forceinline__ unsigned long long mB(unsigned long long y) {
    const uint32_t lo = uint32_t(y);
    const uint32_t m = 0u - (lo & 1u);
    return (unsigned long long)(m & 0xB5026F5Au) << 32 | (((lo >> 1) & 0x3FFFFFFFu) ^ (m & 0xA96619E9u));
}
__device__ __forceinline__ MtQuad quad_lin(const unsigned long long* o, int t, unsigned long long P,
                                           unsigned long long Q) {
    const unsigned long long o0 = o[t], o1 = o[t + 1], o2 = o[t + 2], h0 = o[t + 156];
    MtQuad r;
    r.a = h0 ^ mA(o0) ^ mB(o1);
    const unsigned long long K1 = mA(h0) ^ mB(P);
    const unsigned long long a1 = P ^ mA(o1) ^ mB(o2);
    r.b = r.a ^ K1;
    const unsigned long long b1 = a1 ^ mA(P) ^ mB(Q);
    const unsigned long long Ba1 = mB(a1);
    r.c = r.b ^ mA(r.a) ^ Ba1;
    r.d = r.b ^ Ba1 ^ mA(K1) ^ mB(b1);
    return r;
}

__device__ __forceinline__ unsigned long long tw_fma(unsigned long long a, unsigned long long b, unsigned long long m) {
    const uint32_t alo = uint32_t(a), ahi = uint32_t(a >> 32), blo = uint32_t(b);
    const uint32_t bit = __umulhi(blo * 0x80000000u, 2u);                 // b & 1
    const uint32_t hi1 = __umulhi(ahi, 0x80000000u);                      // a.hi >> 1
    const uint32_t t1 = __umulhi(blo * 2u, 0x40000000u);                  // (b.lo & 0x7fffffff) >> 1
    const uint32_t s = ahi * 0x80000000u + __umulhi(alo, 2u) * 0x40000000u + t1;
    const uint32_t rhi = uint32_t(m >> 32) ^ hi1 ^ (bit * 0xB5026F5Au);
    const uint32_t rlo = uint32_t(m) ^ s ^ (bit * 0xA96619E9u);
    return (unsigned long long)rhi << 32 | rlo;
}
__device__ __forceinline__ MtQuad quad_fma(const unsigned long long* o, int t, unsigned long long P,
                                           unsigned long long Q) {
    MtQuad r;
    r.a = tw_fma(o[t], o[t + 1], o[t + 156]);
    const unsigned long long a1 = tw_fma(o[t + 1], o[t + 2], P);
    r.b = tw_fma(o[t + 156], P, r.a);
    const unsigned long long b1 = tw_fma(P, Q, a1);
    r.c = tw_fma(r.a, a1, r.b);
    r.d = tw_fma(r.b, b1, r.c);
    return r;
}

template <int V>
__global__ void k_lat(int passes, long long* cyc, unsigned long long* out) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords + 64];
    const int t = threadIdx.x;
    for (int i = t; i < kMtStateWords; i += blockDim.x) buf[i] = 0x9E3779B97F4A7C15ull * (i + 1);
    __syncthreads();
    int cur = 0;
    const long long t0 = clock64();
    for (int k = 0; k < passes; ++k) {
        const unsigned long long* o = buf + cur * 624 + 312;
        unsigned long long* nb = buf + (cur ^ 1) * 624;
        if (V == 0 || V == 1) {
            const MtQuad q = mt_quad(o, t, o[t + 157], o[t + 158]);
            mt_store_quad(nb, t, q);
        } else if (V == 2) {
            const unsigned long long a = o[t] ^ o[t + 1] ^ o[t + 156], b = o[t + 157] ^ o[t + 158] ^ o[t + 2];
            nb[t] = a; nb[156 + t] = b; nb[312 + t] = a ^ b; nb[468 + t] = a + b;
        } else if (V == 3) {          // quad from registers only (no smem)
            unsigned long long r0 = o[t], r1 = o[t + 1], r2 = o[t + 2], r3 = o[t + 156];
            for (int j = 0; j < 8; ++j) {
                const MtQuad q = [&] {
                    MtQuad r;
                    r.a = mt_twist1(r0, r1, r3);
                    const unsigned long long a1 = mt_twist1(r1, r2, r0);
                    r.b = mt_twist1(r3, r0, r.a);
                    const unsigned long long b1 = mt_twist1(r0, r1, a1);
                    r.c = mt_twist1(r.a, a1, r.b);
                    r.d = mt_twist1(r.b, b1, r.c);
                    return r;
                }();
                r0 = q.a; r1 = q.b; r2 = q.c; r3 = q.d;
            }
            nb[t] = r0 ^ r1 ^ r2 ^ r3;
        }
        if (V == 4 || V == 5) {
            const int tt = V == 4 ? t : 124 + t;
            const MtQuad q = mt_quad_any(o, tt);
            mt_store_quad(nb, tt, q);
        }
        if (V == 6) {
            if (t < 128) mt_store_quad(nb, t, mt_quad(o, t, o[t + 157], o[t + 158]));
            else if (t < 156) mt_store_quad(nb, t, mt_quad_any(o, t));
        }
        if (V == 7) {        // current layout: second chain on lanes 0..6 of each warp
            const int w = t >> 5, l = t & 31;
            const bool second = l < 7;
            const int t2 = second ? 128 + 7 * w + l : 128;
            const MtQuad q1 = mt_quad(o, t, o[t + 157], o[t + 158]);
            const MtQuad q2 = mt_quad_any(o, t2);
            mt_store_quad(nb, t, q1);
            if (second) mt_store_quad(nb, t2, q2);
        }
        if (V == 8) {
            if (t < 128) mt_store_quad(nb, t, mt_quad(o, t, o[t + 157], o[t + 158]));
            else if (t < 152) mt_store_quad(nb, t, mt_quad(o, t, o[t + 157], o[t + 158]));
        }
        if (V == 9) {
            if (t < 128) mt_store_quad(nb, t, mt_quad(o, t, o[t + 157], o[t + 158]));
        }
        if (V == 10) {       // warp 4 on SMSP 0 alone: warps 0..3 -> t 0..127 moved to warps 1..4?
            const int w = t >> 5;
            if (w >= 1 && w <= 4) { const int tt = t - 32; mt_store_quad(nb, tt, mt_quad(o, tt, o[tt + 157], o[tt + 158])); }
            if (w == 0 && (t & 31) < 28) { const int tt = 128 + (t & 31); mt_store_quad(nb, tt, mt_quad_any(o, tt)); }
        }
        if (V == 11 || V == 12) {        // lane L: t = 2L, 2L+1 (vector loads / stores)
            const int L = t;
            if (L < 78) {
                const ulonglong2 u0 = *reinterpret_cast<const ulonglong2*>(o + 2 * L);       // o[2L], o[2L+1]
                const ulonglong2 u1 = *reinterpret_cast<const ulonglong2*>(o + 2 * L + 2);   // o[2L+2], o[2L+3]
                const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(o + 2 * L + 156);
                const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(o + 2 * L + 158);
                unsigned long long P0 = w0.y, Q0 = w1.x, P1 = w1.x, Q1 = w1.y;   // x[B+157+t], x[B+158+t]
                if (V == 12 && (L >> 5) == 2) {
                    if (L == 77) {
                        const unsigned long long n0 = mt_twist1(o[0], o[1], o[156]);
                        const unsigned long long n1 = mt_twist1(o[1], o[2], o[157]);
                        Q0 = n0; P1 = n0; Q1 = n1;
                    }
                }
                MtQuad q0, q1;
                {
                    q0.a = mt_twist1(u0.x, u0.y, w0.x);
                    const unsigned long long a1 = mt_twist1(u0.y, u1.x, P0);
                    q0.b = mt_twist1(w0.x, P0, q0.a);
                    const unsigned long long b1 = mt_twist1(P0, Q0, a1);
                    q0.c = mt_twist1(q0.a, a1, q0.b);
                    q0.d = mt_twist1(q0.b, b1, q0.c);
                    q1.a = a1;
                    const unsigned long long a2 = mt_twist1(u1.x, u1.y, P1);
                    q1.b = b1;
                    const unsigned long long b2 = mt_twist1(P1, Q1, a2);
                    q1.c = mt_twist1(a1, a2, b1);
                    q1.d = mt_twist1(b1, b2, q1.c);
                }
                *reinterpret_cast<ulonglong2*>(nb + 2 * L) = make_ulonglong2(q0.a, q1.a);
                *reinterpret_cast<ulonglong2*>(nb + 156 + 2 * L) = make_ulonglong2(q0.b, q1.b);
                *reinterpret_cast<ulonglong2*>(nb + 312 + 2 * L) = make_ulonglong2(q0.c, q1.c);
                *reinterpret_cast<ulonglong2*>(nb + 468 + 2 * L) = make_ulonglong2(q0.d, q1.d);
            }
        }
        if (V == 13) {       // one warp, two quads per lane
            const MtQuad q0 = mt_quad(o, t, o[t + 157], o[t + 158]);
            const MtQuad q1 = mt_quad(o, t + 32, o[t + 189], o[t + 190]);
            mt_store_quad(nb, t, q0);
            mt_store_quad(nb, t + 32, q1);
        }
        if (V == 14) {       // one warp, one quad, loads via shuffles
            const unsigned long long x0 = o[t], y0 = o[t + 156];
            const unsigned long long x32 = o[t + 32 < 312 ? t + 32 : 0], y32 = o[t + 188];
            unsigned long long x1 = __shfl_down_sync(~0u, x0, 1), x2 = __shfl_down_sync(~0u, x0, 2);
            unsigned long long y1 = __shfl_down_sync(~0u, y0, 1), y2 = __shfl_down_sync(~0u, y0, 2);
            const unsigned long long xa = __shfl_sync(~0u, x32, (t + 1) & 31), xb = __shfl_sync(~0u, x32, (t + 2) & 31);
            const unsigned long long ya = __shfl_sync(~0u, y32, (t + 1) & 31), yb = __shfl_sync(~0u, y32, (t + 2) & 31);
            if (t >= 31) { x1 = xa; y1 = ya; }
            if (t >= 30) { x2 = xb; y2 = yb; }
            MtQuad r;
            r.a = mt_twist1(x0, x1, y0);
            const unsigned long long a1 = mt_twist1(x1, x2, y1);
            r.b = mt_twist1(y0, y1, r.a);
            const unsigned long long b1 = mt_twist1(y1, y2, a1);
            r.c = mt_twist1(r.a, a1, r.b);
            r.d = mt_twist1(r.b, b1, r.c);
            mt_store_quad(nb, t, r);
        }
        if (V == 15 || V == 16) {
            const int w = t >> 5, l = t & 31;
            const bool second = V == 15 ? true : l < 7;
            const int t2 = second ? 128 + 7 * w + l : 128;
            const MtQuad q1 = mt_quad(o, t, o[t + 157], o[t + 158]);
            const MtQuad q2 = mt_quad(o, t2, o[t2 + 157], o[t2 + 158]);
            mt_store_quad(nb, t, q1);
            if (second) mt_store_quad(nb, t2, q2);
        }
        if (V == 17) mt_store_quad(nb, t, quad_lin(o, t, o[t + 157], o[t + 158]));
        if (V == 18) {
            const int w = t >> 5, l = t & 31;
            const bool second = l < 7;
            const int t2 = second ? 128 + 7 * w + l : 128;
            const MtQuad q1 = quad_lin(o, t, o[t + 157], o[t + 158]);
            const MtQuad q2 = quad_lin(o, t2, o[t2 + 157], o[t2 + 158]);
            mt_store_quad(nb, t, q1);
            if (second) mt_store_quad(nb, t2, q2);
        }
        if (V == 19) mt_store_quad(nb, t, quad_fma(o, t, o[t + 157], o[t + 158]));
        if (V == 20) {
            const int w = t >> 5, l = t & 31;
            const bool second = l < 7;
            const int t2 = second ? 128 + 7 * w + l : 128;
            const MtQuad q1 = quad_fma(o, t, o[t + 157], o[t + 158]);
            const MtQuad q2 = quad_fma(o, t2, o[t2 + 157], o[t2 + 158]);
            mt_store_quad(nb, t, q1);
            if (second) mt_store_quad(nb, t2, q2);
        }
        if (V == 1) __syncwarp(); else __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x == 0) { *cyc = clock64() - t0; out[0] = buf[cur * 624 + 5]; }
}

__global__ void k_check(unsigned long long* out) {
    __shared__ unsigned long long o[320];
    __shared__ unsigned long long bad;
    if (threadIdx.x == 0) bad = 0;
    unsigned long long s = 0x9E3779B97F4A7C15ull * (threadIdx.x + 7);
    for (int rep = 0; rep < 64; ++rep) {
        __syncthreads();
        for (int i = threadIdx.x; i < 320; i += blockDim.x) {
            s = s * 6364136223846793005ull + 1442695040888963407ull + i;
            o[i] = s ^ (s >> 29) ^ (unsigned long long)rep << 40;
        }
        __syncthreads();
        const int t = threadIdx.x;
        if (t < 154) {
            const MtQuad x = mt_quad(o, t, o[t + 157], o[t + 158]), y = quad_fma(o, t, o[t + 157], o[t + 158]);
            if (x.a != y.a || x.b != y.b || x.c != y.c || x.d != y.d) atomicAdd(&bad, 1ull);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[0] = bad;
}

int main() {
    long long* cyc; unsigned long long* out;
    cudaMalloc(&cyc, 8); cudaMalloc(&out, 64);
    const int P = getenv("PASSES") ? atoi(getenv("PASSES")) : 2000;
    long long h;
    const char* names[] = {"quad+bar", "quad+syncwarp", "xor-only+bar", "8 quads in regs (per quad)", "quad_any t=lane", "quad_any t=124+lane", "5 warps, warp 4 any", "current 2-chain layout", "5 warps all quad", "5 warps, warp4 idle", "warp0 any, warps1-4 quad", "paired (no tail fix)", "paired + tail", "1 warp 2 quads/lane", "1 warp quad via shfl", "4w 2 chains unpredicated", "4w 2 chains, 7 lanes", "linear quad", "linear 4w 2 chains", "fma quad", "fma 4w 2 chains"};
#define RUN(V, TH) k_lat<V><<<1, TH>>>(P, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
    printf("%-28s threads %3d: %.1f cycles/pass\n", names[V], TH, double(h) / P / (V == 3 ? 8 : 1));
    RUN(0, 32) RUN(1, 32) RUN(2, 32) RUN(3, 32) RUN(0, 128) RUN(2, 128) RUN(3, 128) RUN(4, 32) RUN(5, 32) RUN(6, 160) RUN(7, 128) RUN(8, 160) RUN(9, 160) RUN(10, 160) RUN(0, 32) RUN(19, 32) RUN(0, 128) RUN(19, 128) RUN(16, 128) RUN(20, 128)
    {   // correctness: linear quad == mt_quad on random words
        k_check<<<1, 160>>>(out);
        unsigned long long bad; cudaMemcpy(&bad, out, 8, cudaMemcpyDeviceToHost);
        printf("linear quad mismatches: %llu\n", bad);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
