// Dependent-chain latencies on the B200 SM (one warp, unrolled asm chains):
// DADD, DFMA, FADD, SHFL, LDS.  Informs the single-warp best/AT phase of the
// fused kernel.
#include <cstdio>
#define CHAIN(stmt) _Pragma("unroll") for (int i = 0; i < 64; ++i) { stmt; }
__global__ void k(double* out, long long* cyc, double a, float af) {
    __shared__ unsigned sm[64];
    sm[threadIdx.x] = threadIdx.x; sm[threadIdx.x + 32] = 0;
    __syncwarp();
    double x = a; float y = af; unsigned iv = threadIdx.x;
    long long t[8];
    t[0] = clock64();
    CHAIN(asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(a)));
    t[1] = clock64();
    CHAIN(asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x) : "d"(a)));
    t[2] = clock64();
    CHAIN(asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(y) : "f"(af)));
    t[3] = clock64();
    CHAIN(asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 31, -1;" : "+r"(iv)));
    t[4] = clock64();
    CHAIN(asm volatile("ld.shared.u32 %0, [%1];" : "=r"(iv) : "r"((unsigned)__cvta_generic_to_shared(sm) + (iv & 31) * 4)));
    t[5] = clock64();
    CHAIN(asm volatile("min.f64 %0, %0, %1;" : "+d"(x) : "d"(a)));
    t[6] = clock64();
    CHAIN(asm volatile("{ .reg .pred p; setp.lt.f64 p, %0, %1; selp.f64 %0, %0, %1, p; }" : "+d"(x) : "d"(a)));
    t[7] = clock64();
    out[threadIdx.x] = x + y + iv;
    if (threadIdx.x == 0) for (int i = 0; i < 7; ++i) cyc[i] = t[i + 1] - t[i];
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
    for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, c, 1.000001, 1.0001f); cudaDeviceSynchronize(); }
    const char* n[] = {"DADD", "DFMA", "FADD", "SHFL", "LDS", "DMNMX", "DSETP+SEL"};
    for (int i = 0; i < 7; ++i) printf("%-10s %.1f cyc/op\n", n[i], c[i] / 64.0);
}
