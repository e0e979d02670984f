// Cycles of the single-warp AT decision (swarm_kernel.cu at_decide_regs) in
// isolation: one warp, window in registers, 64 calls.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ int at_decide_regs(double w, int lane, int tw, double c, double inv_n, double bound) {
    const bool act = lane < tw;
    const double d = act ? w - c : 0.0;
    double s = d, q = d * d;
    const uint32_t hx = __reduce_max_sync(0xffffffffu, act ? uint32_t(uint64_t(__double_as_longlong(fabs(d))) >> 32) : 0u);
    const uint32_t hm = __reduce_max_sync(0xffffffffu, act ? uint32_t(uint64_t(__double_as_longlong(fabs(w))) >> 32) : 0u);
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        q += __shfl_xor_sync(0xffffffffu, q, off);
    }
    const double X = __longlong_as_double((long long)((uint64_t(hx) << 32) | 0xffffffffull));
    const double M = __longlong_as_double((long long)((uint64_t(hm) << 32) | 0xffffffffull));
    const double n = double(tw), u = 0x1p-53;
    const double dl = 1.01 * (n + 2.0) * u * M;
    const double E = (3.0 * n + 40.0) * u * n * X * X + 2.0 * n * dl * dl;
    const double v = q - s * s * inv_n;
    if (!(v == v) || !(E == E) || E > 0x1p1000) return -1;
    if (v + E < bound) return 1;
    if (v - E >= bound) return 0;
    return -1;
}
__global__ void k(const double* win, int tw, double bound, long long* cyc, int* out) {
    const int lane = threadIdx.x & 31;
    double w = lane < tw ? win[lane] : 0.0;
    int acc = 0;
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < 64; ++i) {
        const double c = __shfl_sync(~0u, w, (i + 3) % tw);
        acc += at_decide_regs(w, lane, tw, c, 1.0 / tw, bound + i);
        w += 1e-9 * acc;
    }
    long long t1 = clock64();
    if (lane == 0) { cyc[blockIdx.x] = t1 - t0; out[blockIdx.x] = acc; }
}
int main() {
    double h[32]; for (int i = 0; i < 32; ++i) h[i] = 350.0 - i * 0.7;
    double* d; long long* c; int* o;
    cudaMalloc(&d, 256); cudaMallocManaged(&c, 8); cudaMallocManaged(&o, 4);
    cudaMemcpy(d, h, 256, cudaMemcpyHostToDevice);
    for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(d, 20, 2000.0, c, o); cudaDeviceSynchronize(); }
    printf("at_decide_regs: %.0f cycles/call (1 warp alone), result %d\n", c[0] / 64.0, o[0]);
}
