// Cycles per generator pass (624 words) of the production layouts, built with
// -DSEPSO_MT_IMAD=0 (ALU twist / temper) or =1 (IMAD forms): the init walk's
// 256-thread group (warps 0..3 generate, 4..7 deliver) without and with word
// delivery, and the step generator's three-warp layout (FN = 96).
#include <cstdio>
#include "../paper_2308_10169_b200/csrc/philox.cuh"
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;

template <int MODE>
__global__ void k_walk(int passes, long long* cyc, float* gsink) {
    __shared__ unsigned long long buf[kMtStateWords];
    __shared__ float xs[8192];
    const int tid = threadIdx.x;
    MtState s{buf, 0, 0};
    if (MODE == 2) {
        const MtGroup g{tid - 32, 96, 1};
        if (tid >= 32 && tid < 128) {
            if (tid == 32) mt_seed_words(buf + 312, 5489ull);
            asm volatile("bar.sync 1, 96;");
            const long long t0 = clock64();
            mt_generate<96>(s, g, 0, 624ll * passes, [&](int w, unsigned long long word) {
                xs[w & 8191] = unit_from_word<float>(word);
            });
            if (tid == 32) cyc[0] = clock64() - t0;
        }
    } else {
        const MtGroup g{tid, 256, 3};
        if (tid < 256) {
            if (tid == 0) mt_seed_words(buf + 312, 5489ull);
            asm volatile("bar.sync 3, 256;");
            const long long t0 = clock64();
            if (MODE == 0)
                mt_generate(s, g, 624ll * passes, 624ll * passes, [&](int, unsigned long long) {});
            else
                mt_generate(s, g, 0, 624ll * passes, [&](int w, unsigned long long word) {
                    xs[w & 8191] = unit_from_word<float>(word);
                });
            if (tid == 0) cyc[0] = clock64() - t0;
        }
    }
    __syncthreads();
    if (xs[tid] == 42.f && buf[tid] == 7) gsink[0] = 1.f;
}

int main() {
    long long* cyc; float* gs;
    cudaMalloc(&cyc, 64); cudaMalloc(&gs, 64);
    const char* names[3] = {"init walk, no delivery", "init walk, all words delivered", "step layout (96), all delivered"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            const int passes = 70;
            if (mode == 0) k_walk<0><<<1, 896>>>(passes, cyc, gs);
            if (mode == 1) k_walk<1><<<1, 896>>>(passes, cyc, gs);
            if (mode == 2) k_walk<2><<<1, 896>>>(passes, cyc, gs);
            long long c = 0;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            if (rep == 2) printf("IMAD=%d  %-34s %7.1f cycles/pass\n", SEPSO_MT_IMAD, names[mode], double(c) / passes);
        }
    }
    return cudaDeviceSynchronize() != cudaSuccess;
}
