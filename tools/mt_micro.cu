// Micro-benchmark of mt19937_64 block-generation variants (cycles per block).
#include <cstdio>
#include "../paper_2308_10169_b200/csrc/philox.cuh"
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;

__global__ void k_gen(long long blocks, long long* cyc, float* gsink) {
    __shared__ unsigned long long buf[kMtStateWords];
    __shared__ float sinkbuf[1024];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), int(blockDim.x), 0};
    const long long ts = clock64();
    mt_seed(s, g, 5489ull);
    const long long t0 = clock64();
    if (threadIdx.x == 0) cyc[1] = t0 - ts;
    mt_generate(s, g, 0, 312 * blocks, [&](int w, unsigned long long word) {
        if ((w & 15) == 0) sinkbuf[threadIdx.x] = unit_from_word<float>(word);
    });
    if (threadIdx.x == 0) *cyc = clock64() - t0;
    if (sinkbuf[threadIdx.x] == 42.f) gsink[0] = 1.f;
}

__global__ void k_nodeliver(long long blocks, long long* cyc, float* gsink, int gn) {
    __shared__ unsigned long long buf[kMtStateWords];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), gn, gn == int(blockDim.x) ? 0 : 1};
    if (threadIdx.x < gn) {
        mt_seed(s, g, 5489ull);
        const long long t0 = clock64();
        mt_generate(s, g, 312 * blocks, 312 * blocks, [&](int w, unsigned long long word) { gsink[w] = 1.f; });
        if (threadIdx.x == 0) *cyc = clock64() - t0;
        if (threadIdx.x == 0 && buf[5] == 42) gsink[0] = 2.f;
    }
}

template <int VAR>
__global__ void k_var(long long blocks, long long* cyc, float* gsink) {
    __shared__ unsigned long long buf[624];
    __shared__ float sinkbuf[1024];
    const int i = threadIdx.x;
    for (int j = i; j < 624; j += blockDim.x) buf[j] = 0x9E3779B97F4A7C15ull * (j + 1);
    __syncthreads();
    const long long t0 = clock64();
    int cur = 0;
    unsigned long long acc = 0;
    for (long long b = 0; b < blocks; ++b) {
        const unsigned long long* o = buf + cur * 312;
        unsigned long long* n = buf + (cur ^ 1) * 312;
        if (i < 312) {
            unsigned long long y;
            if (VAR == 0) y = o[i] ^ o[i < 156 ? i + 156 : i - 156];
            if (VAR == 1 || VAR == 2 || VAR == 3)
                y = mt_twist1(o[i], o[i == 311 ? 0 : i + 1], o[i < 156 ? i + 156 : i - 156]);
            if (VAR == 4) y = mt_twist1(o[i], o[i == 311 ? 0 : i + 1],
                                        mt_twist1(o[i < 156 ? i + 156 : i - 156], o[i < 155 ? i + 157 : i - 155], o[i]));
            n[i] = y;
            if (VAR == 2) acc ^= mt_temper(y);
            if (VAR == 3 && (i & 15) == 0) sinkbuf[i] = unit_from_word<float>(mt_temper(y));
        }
        __syncthreads();
        cur ^= 1;
    }
    if (threadIdx.x == 0) *cyc = clock64() - t0;
    if (acc == 42 || sinkbuf[threadIdx.x] == 42.f) gsink[0] = 1.f;
}

int main() {
    long long* cyc; float* sb;
    cudaMalloc(&cyc, 16); cudaMalloc(&sb, 4096);
    const long long B = 4000;
    for (int th : {320, 512, 1024}) {
        long long h;
        k_gen<<<1, th>>>(B, cyc, sb); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        long long hs; cudaMemcpy(&hs, cyc + 1, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d gen      %.1f   (seed %lld cycles)\n", th, double(h) / B, hs);
        for (int gn : {192, 320}) {
            if (gn > th) continue;
            h = -1;
            k_nodeliver<<<1, th>>>(B, cyc, sb, gn);
            printf("  launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("threads %4d group %d nodeliver %.1f per block\n", th, gn, double(h) / B);
        }
        const char* names[] = {"xoronly", "1twist", "1tw+temper", "1tw+tmp+sts", "2twist"};
#define RUNV(V) k_var<V><<<1, th>>>(B, cyc, sb); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
        printf("threads %4d %-12s %.1f\n", th, names[V], double(h) / B);
        RUNV(0) RUNV(1) RUNV(2) RUNV(3) RUNV(4)
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
