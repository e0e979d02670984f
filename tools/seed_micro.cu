// Micro-benchmark: cycles per step of the std::mt19937_64 seeding recurrence.
#include <cstdio>
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;
constexpr unsigned long long M = 6364136223846793005ull;
__device__ __forceinline__ unsigned long long step_v1(unsigned long long x, unsigned long long i) {
    const unsigned long long P = M * x;                       // independent of the xor-shift
    const int lo2 = int(x) & 3, d = (lo2 ^ int(x >> 62)) - lo2;   // (x ^ (x >> 62)) - x, in [-3, 3]
    return P + (unsigned long long)((long long)d * (long long)M) + i;
}
template <int V>
__global__ void k_seed(unsigned long long seed, long long* cyc, unsigned long long* out) {
    __shared__ unsigned long long st[312];
    const long long t0 = clock64();
    if (V == 0) mt_seed_words(st, seed);
    else {
        unsigned long long x = seed;
        st[0] = x;
#pragma unroll 8
        for (int i = 1; i < 312; ++i) { x = step_v1(x, (unsigned long long)i); st[i] = x; }
    }
    const long long t1 = clock64();
    *cyc = t1 - t0;
    unsigned long long h = 0;
    for (int i = 0; i < 312; ++i) h = h * 31 + st[i];
    out[0] = h;
}
int main() {
    long long* cyc; unsigned long long* out; cudaMalloc(&cyc, 8); cudaMalloc(&out, 8);
    long long h; unsigned long long a, b;
    for (unsigned long long s : {5489ull, 0xFFFFFFFFFFFFFFFFull, 0x123456789ABCDEFull}) {
        k_seed<0><<<1, 1>>>(s, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&a, out, 8, cudaMemcpyDeviceToHost);
        printf("v0 %.1f cycles/step  ", double(h) / 311);
        k_seed<1><<<1, 1>>>(s, cyc, out); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&b, out, 8, cudaMemcpyDeviceToHost);
        printf("v1 %.1f cycles/step  %s\n", double(h) / 311, a == b ? "same" : "DIFFERENT");
    }
}
