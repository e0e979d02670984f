// Which setting makes the mt pass slow?  (cycles per block)
#include <cstdio>
#include "../paper_2308_10169_b200/csrc/philox.cuh"
#include "../paper_2308_10169_b200/csrc/mt19937.cuh"
using namespace sepso;

template <int LB>
__global__ void __launch_bounds__(LB) k_a(long long blocks, long long* cyc, float* gsink, int timeseed) {
    __shared__ unsigned long long buf[kMtStateWords];
    __shared__ float sinkbuf[1024];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), int(blockDim.x), 0};
    long long t0 = clock64();
    mt_seed(s, g, 12345ull);
    if (!timeseed) t0 = clock64();
    mt_generate(s, g, 0, 312 * blocks, [&](int w, unsigned long long word) {
        if ((w & 15) == 0) sinkbuf[threadIdx.x] = unit_from_word<float>(word);
    });
    __syncthreads();
    if (threadIdx.x == 0) *cyc = clock64() - t0;
    if (sinkbuf[threadIdx.x] == 42.f) gsink[0] = 1.f;
}

__global__ void __launch_bounds__(1024) k_mt_probe(long long blocks, int mode, unsigned long long* out,
                                                  long long* cycles) {
    __shared__ unsigned long long buf[kMtStateWords];
    __shared__ float sinkbuf[1024];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), int(blockDim.x), 0};
    const long long t0 = clock64();
    mt_seed(s, g, 12345ull);
    unsigned long long acc = 0;
    if (mode == 0)
        mt_generate(s, g, 0, 312 * blocks, [&](int w, unsigned long long word) { acc ^= word; });
    else if (mode == 1)
        mt_generate(s, g, 0, 312 * blocks, [&](int w, unsigned long long word) {
            if ((w & 15) == 0) sinkbuf[threadIdx.x] = unit_from_word<float>(word);
        });
    else if (mode == 2) {          // barrier + one LDS/STS round trip per "block"
        for (long long b = 0; b < blocks; ++b) {
            const int i = threadIdx.x % 312;
            buf[((b + 1) & 1) * 312 + i] = buf[(b & 1) * 312 + ((i + 1) % 312)] + 1;
            __syncthreads();
        }
        acc = buf[threadIdx.x % 312];
    } else if (mode == 4 || mode == 5) {   // fused-kernel step shape: warps 1..6, 3 windows of 85 rows per 4080 words
        __syncthreads();
        const int tid = threadIdx.x;
        if (tid >= 32 && tid < 224) {
            const MtGroup gg{tid - 32, 192, 1};
            MtState st{buf, s.cur, s.blocks};
            const long long steps = blocks * 312 / 4080;
            for (long long k = 0; k < steps; ++k) {
                const long long base = 4080 * k;
                if (mode == 4) {
                    for (int j = 0; j < 3; ++j)
                        mt_generate(st, gg, base + j * 1360 + 85, base + j * 1360 + 170,
                                    [&](int pl, unsigned long long word) { sinkbuf[j * 85 + pl] = unit_from_word<float>(word); });
                } else {
                    mt_generate(st, gg, base, base + 4080, [&](int pl, unsigned long long word) {
                        if (pl < 85) sinkbuf[pl] = unit_from_word<float>(word); });
                }
            }
        }
        __syncthreads();
    } else if (mode == 3) {        // barrier only
        for (long long b = 0; b < blocks; ++b) __syncthreads();
    }
    if (acc == 42) out[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) *cycles = clock64() - t0;
}

// fused-kernel init shape: 1024 threads, warps 0..3 generate (named barrier 3), no deliveries
__global__ void __launch_bounds__(1024, 1) k_b(long long blocks, long long* cyc, float* gsink, int gsize) {
    __shared__ unsigned long long buf[kMtStateWords];
    const int tid = threadIdx.x;
    if (tid == 0) mt_seed_words(buf + 312, 12345ull);
    __syncthreads();
    const long long t0 = clock64();
    const MtGroup grp = gsize < int(blockDim.x) ? MtGroup{tid, gsize, 3} : MtGroup{tid, int(blockDim.x), 0};
    MtState mt{buf, 0, 0};
    if (tid < grp.n) mt_generate(mt, grp, 312 * blocks, 312 * blocks, [&](int, unsigned long long) {});
    __syncthreads();
    if (tid == 0) *cyc = clock64() - t0;
    if (buf[tid % 624] == 42) gsink[0] = 1.f;
}

// generator-CTA step shape: group of gs threads, every word delivered to smem
__global__ void __launch_bounds__(1024, 1) k_c(long long blocks, long long* cyc, float* gsink, int gs, int mode) {
    __shared__ unsigned long long buf[kMtStateWords];
    __shared__ float stage[4096];
    __shared__ float hyp[48];
    const int tid = threadIdx.x;
    if (tid < 48) hyp[tid] = 0.5f + tid;
    if (tid == 0) mt_seed_words(buf + 312, 12345ull);
    __syncthreads();
    const long long t0 = clock64();
    const MtGroup grp = gs < int(blockDim.x) ? MtGroup{tid, gs, 3} : MtGroup{tid, int(blockDim.x), 0};
    MtState mt{buf, 0, 0};
    if (tid < grp.n) {
        for (long long w0 = 0; w0 < 312 * blocks; w0 += 4080) {
            if (mode == 0)
                mt_generate(mt, grp, w0, w0 + 4080, [&](int e, unsigned long long word) {
                    stage[e & 4095] = unit_from_word<float>(word);
                });
            else
                mt_generate(mt, grp, w0, w0 + 4080, [&](int e, unsigned long long word) {
                    const int j = e >= 2720 ? 2 : (e >= 1360 ? 1 : 0), row = e - j * 1360;
                    stage[e & 4095] = hyp[(row / 170) * 6 + j] * unit_from_word<float>(word);
                });
        }
    }
    __syncthreads();
    if (tid == 0) *cyc = clock64() - t0;
    if (stage[tid] == 42.f) gsink[0] = 1.f;
}

// staged-path fill: every word of [0, n) tempered into global memory
template <bool RAW>
__global__ void __launch_bounds__(1024) k_fill(long long n, unsigned long long* out) {
    __shared__ unsigned long long buf[kMtStateWords];
    MtState s{buf, 0, 0};
    const MtGroup g{int(threadIdx.x), int(blockDim.x), 0};
    mt_seed(s, g, 5489ull);
    mt_generate<0, RAW>(s, g, 0, n, [&](int rel, unsigned long long word) { out[rel] = word; });
}

__global__ void k_spin(long long cycles, float* o) {
    const long long t0 = clock64();
    float x = threadIdx.x;
    while (clock64() - t0 < cycles) x = x * 0.999f + 0.001f;
    if (x == 42.f) o[0] = x;
}

int main() {
    long long* cyc; float* sb;
    cudaMalloc(&cyc, 16); cudaMalloc(&sb, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_spin<<<148 * 4, 256>>>(1000000000ll, sb);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("spin 1e9 cycles: %.1f ms -> %.0f MHz\n", ms, 1e9 / (ms * 1e3));
    }
    unsigned long long* out; cudaMalloc(&out, 8192);
    for (int mode = 0; mode < 2; ++mode) {
        long long h;
        k_mt_probe<<<1, 320>>>(2000, mode, out, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("calib copy mode %d: %.1f\n", mode, double(h) / 2000);
    }
    {
        unsigned long long* big; const long long n = 2ll * 65536 * 128;
        cudaMalloc(&big, n * 8);
        for (int raw = 0; raw < 2; ++raw)
        for (int th : {256, 320, 512}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            if (raw) k_fill<true><<<1, th>>>(n, big); else k_fill<false><<<1, th>>>(n, big);
            cudaEventRecord(a);
            if (raw) k_fill<true><<<1, th>>>(n, big); else k_fill<false><<<1, th>>>(n, big);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("fill raw=%d %lld words, %d threads: %.2f ms (%.0f cycles/pass at 1.965 GHz)\n", raw, n, th, ms, ms * 1.965e6 / (n / 624.0));
        }
        cudaFree(big);
    }
    for (int mode = 0; mode < 2; ++mode)
    for (int gs : {128, 256, 512, 1024}) {
        long long h;
        k_c<<<1, 1024>>>(2000, cyc, sb, gs, mode); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("gcta shape mode %d group %d: %.1f per block\n", mode, gs, double(h) / 2000);
    }
    for (int gs : {128, 1024}) {
        long long h;
        k_b<<<1, 1024>>>(2000, cyc, sb, gs); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("init shape group %d: %.1f per block\n", gs, double(h) / 2000);
    }
    for (int rep = 0; rep < 2; ++rep)
    for (long long B : {2000ll, 4000ll}) {
        long long h;
        k_a<1024><<<1, 320>>>(B, cyc, sb, 1); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("B=%lld LB1024 timeseed %.1f\n", B, double(h) / B);
        k_a<1024><<<1, 320>>>(B, cyc, sb, 0); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("B=%lld LB1024 notseed  %.1f\n", B, double(h) / B);
        k_a<320><<<1, 320>>>(B, cyc, sb, 0); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("B=%lld LB320  notseed  %.1f\n", B, double(h) / B);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
