// Micro-benchmark: mt19937_64 pass pace vs the number of warps the 156 quad
// lanes are spread over (cycles per pass = two blocks).
#include <cstdio>
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;

__global__ void k_cur(int passes, long long* cyc, unsigned long long* out) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), 128, 0};
    mt_seed(s, g, 5489ull);
    const long long t0 = clock64();
    mt_generate<128>(s, g, 624ll * passes, 624ll * passes, [&](int, unsigned long long) {});
    if (threadIdx.x == 0) { *cyc = clock64() - t0; out[0] = buf[s.cur * 624 + 312 + 7]; out[1] = buf[s.cur * 624 + 311]; out[2] = buf[s.cur * 624 + 312 + 155]; }
}

// WARPS warps; lane t of the 156 quads -> warp w = t / PER, lane t % PER
template <int WARPS, bool ANY_ALL>
__global__ void k_spread(int passes, long long* cyc, unsigned long long* out) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords];
    constexpr int PER = (156 + WARPS - 1) / WARPS;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int t = w * PER + l;
    const bool act = l < PER && t < 156;
    if (threadIdx.x == 0) mt_seed_words(buf + 312, 5489ull);
    __syncthreads();
    int cur = 0;
    const long long t0 = clock64();
    const bool tail = (w + 1) * PER > 154;        // warp holding lanes 154 / 155
    for (int k = 0; k < passes; ++k) {
        const unsigned long long* o = buf + cur * 624 + 312;
        unsigned long long* nb = buf + (cur ^ 1) * 624;
        if (act) {
            MtQuad q;
            if (ANY_ALL || tail) q = mt_quad_any(o, t);
            else q = mt_quad(o, t, o[t + 157], o[t + 158]);
            mt_store_quad(nb, t, q);
        }
        __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x == 0) { *cyc = clock64() - t0; out[0] = buf[cur * 624 + 312 + 7]; }
}

// 4 warps; second chain (t = 128..155) on lanes 0..6 of each warp with plain
// quads: the two words past the block end that lanes 154/155 need are computed
// by warp 0 one pass ahead and stored after the pair (stride 626)
__global__ void k_ext(int passes, long long* cyc, unsigned long long* out) {
    __shared__ __align__(128) unsigned long long buf[2 * 626];
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    if (tid == 0) mt_seed_words(buf + 312, 5489ull);
    __syncthreads();
    if (tid == 0) {
        const unsigned long long* o = buf + 312;
        buf[624] = mt_twist1(o[0], o[1], o[156]);
        buf[625] = mt_twist1(o[1], o[2], o[157]);
    }
    __syncthreads();
    const bool second = l < 7;
    const int t2 = second ? 128 + 7 * w + l : 128;
    int cur = 0;
    const long long t0 = clock64();
    for (int k = 0; k < passes; ++k) {
        const unsigned long long* o = buf + cur * 626 + 312;
        unsigned long long* nb = buf + (cur ^ 1) * 626;
        const MtQuad q1 = mt_quad(o, tid, o[tid + 157], o[tid + 158]);
        const MtQuad q2 = mt_quad(o, t2, o[t2 + 157], o[t2 + 158]);
        mt_store_quad(nb, tid, q1);
        if (second) mt_store_quad(nb, t2, q2);
        if (w == 0) {       // next pass's x[B'+312], x[B'+313]: T(c0, c1, d0), T(c1, c2, d1)
            const unsigned long long cn = __shfl_down_sync(~0u, q1.c, 1);
            if (l < 2) nb[624 + l] = mt_twist1(q1.c, cn, q1.d);
        }
        __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x == 0) { *cyc = clock64() - t0; out[0] = buf[cur * 626 + 312 + 7]; }
}

// GF(2)-linear twist pieces: T(p, q, m) = m ^ mA(p) ^ mB(q)
__device__ __forceinline__ unsigned long long mA(unsigned long long x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    return (unsigned long long)(hi >> 1) << 32 | (__funnelshift_r(lo, hi, 1) & 0xC0000000u);
}
__device__ __forceinline__ unsigned long long mB(unsigned long long y) {
    const uint32_t lo = uint32_t(y);
    const uint32_t m = 0u - (lo & 1u);
    return (unsigned long long)(m & 0xB5026F5Au) << 32 | (((lo >> 1) & 0x3FFFFFFFu) ^ (m & 0xA96619E9u));
}
// lane L < 78 produces words t = 2L, 2L+1 of both new blocks; 3 warps compute
__global__ void k_pair(int passes, long long* cyc, unsigned long long* out) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords];
    const int L = threadIdx.x, w = L >> 5;
    if (L == 0) mt_seed_words(buf + 312, 5489ull);
    __syncthreads();
    int cur = 0;
    const long long t0 = clock64();
    for (int k = 0; k < passes; ++k) {
        const unsigned long long* o = buf + cur * 624 + 312;
        unsigned long long* nb = buf + (cur ^ 1) * 624;
        if (L < 78) {
            const ulonglong2 u01 = *reinterpret_cast<const ulonglong2*>(o + 2 * L);
            const ulonglong2 u23 = *reinterpret_cast<const ulonglong2*>(o + 2 * L + 2);
            const ulonglong2 h01 = *reinterpret_cast<const ulonglong2*>(o + 2 * L + 156);
            const ulonglong2 h23 = *reinterpret_cast<const ulonglong2*>(o + (L < 77 ? 2 * L + 158 : 310));
            unsigned long long h2 = h23.x;
            const unsigned long long a0 = h01.x ^ mA(u01.x) ^ mB(u01.y);
            const unsigned long long a1 = h01.y ^ mA(u01.y) ^ mB(u23.x);
            unsigned long long a2, b2;
            if (w == 2) {           // lanes 154/155 reach into the new block: x[B+312], x[B+468], x[B+624]
                const ulonglong2 s01 = *reinterpret_cast<const ulonglong2*>(o);
                const ulonglong2 s23 = *reinterpret_cast<const ulonglong2*>(o + 2);
                const ulonglong2 g01 = *reinterpret_cast<const ulonglong2*>(o + 156);
                const unsigned long long n0 = g01.x ^ mA(s01.x) ^ mB(s01.y);     // x[B+312]
                const unsigned long long n1 = g01.y ^ mA(s01.y) ^ mB(s23.x);     // x[B+313]
                const unsigned long long m0 = n0 ^ mA(g01.x) ^ mB(g01.y);        // x[B+468]
                const unsigned long long e0 = m0 ^ mA(n0) ^ mB(n1);              // x[B+624]
                const bool last = L == 77;
                if (last) h2 = n0;
                a2 = last ? m0 : h2 ^ mA(u23.x) ^ mB(u23.y);
                b2 = last ? e0 : a2 ^ mA(h2) ^ mB(h23.y);
            } else {
                a2 = h2 ^ mA(u23.x) ^ mB(u23.y);
                b2 = a2 ^ mA(h2) ^ mB(h23.y);
            }
            const unsigned long long b0 = a0 ^ mA(h01.x) ^ mB(h01.y);
            const unsigned long long b1 = a1 ^ mA(h01.y) ^ mB(h2);
            const unsigned long long c0 = b0 ^ mA(a0) ^ mB(a1);
            const unsigned long long c1 = b1 ^ mA(a1) ^ mB(a2);
            const unsigned long long d0 = c0 ^ mA(b0) ^ mB(b1);
            const unsigned long long d1 = c1 ^ mA(b1) ^ mB(b2);
            *reinterpret_cast<ulonglong2*>(nb + 2 * L) = make_ulonglong2(a0, a1);
            *reinterpret_cast<ulonglong2*>(nb + 156 + 2 * L) = make_ulonglong2(b0, b1);
            *reinterpret_cast<ulonglong2*>(nb + 312 + 2 * L) = make_ulonglong2(c0, c1);
            *reinterpret_cast<ulonglong2*>(nb + 468 + 2 * L) = make_ulonglong2(d0, d1);
        }
        __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x == 0) { *cyc = clock64() - t0; out[0] = buf[cur * 624 + 312 + 7]; out[1] = buf[cur * 624 + 311]; out[2] = buf[cur * 624 + 312 + 155]; }
}

int main() {
    long long* cyc; unsigned long long* out;
    cudaMalloc(&cyc, 8); cudaMalloc(&out, 64);
    const int P = 2000;
    long long h; unsigned long long ref, v;
    k_cur<<<1, 128>>>(P, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    unsigned long long refs[3]; cudaMemcpy(refs, out, 24, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ref, out, 8, cudaMemcpyDeviceToHost);
    printf("current 4 warps      %.1f cycles/pass\n", double(h) / P);
#define RUN(W, A) k_spread<W, A><<<1, 32 * W>>>(P, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
    cudaMemcpy(&v, out, 8, cudaMemcpyDeviceToHost); \
    printf("spread %2d warps any=%d %.1f cycles/pass %s\n", W, int(A), double(h) / P, v == ref ? "ok" : "MISMATCH");
    for (int th : {96, 128}) {
        k_pair<<<1, th>>>(P, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&v, out, 8, cudaMemcpyDeviceToHost);
        unsigned long long vs[3]; cudaMemcpy(vs, out, 24, cudaMemcpyDeviceToHost);
        printf("pair %d threads     %.1f cycles/pass %s\n", th, double(h) / P, (vs[0] == refs[0] && vs[1] == refs[1] && vs[2] == refs[2]) ? "ok" : "MISMATCH");
    }
    k_ext<<<1, 128>>>(P, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&v, out, 8, cudaMemcpyDeviceToHost);
    printf("ext 4 warps          %.1f cycles/pass %s\n", double(h) / P, v == ref ? "ok" : "MISMATCH");
    RUN(5, false) RUN(6, false) RUN(8, false) RUN(8, true) RUN(10, false) RUN(12, false) RUN(16, false) RUN(20, false)
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
