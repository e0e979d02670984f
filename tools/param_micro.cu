// Host round trip (launch + empty cluster kernel + stream sync) vs the size of
// the kernel parameter block -- what a small sf_plan_frame call pays on top of
// the kernel itself.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
template <int B> struct Blob { unsigned char b[B]; };
template <int B>
__global__ void __launch_bounds__(1024, 1) k_param(const __grid_constant__ Blob<B> p, int* o) {
    if (threadIdx.x == 0 && p.b[B - 1] == 77) o[0] = 1;
}
template <int B> void run(cudaStream_t st, int* o) {
    static Blob<B> blob{};
    auto k = k_param<B>;
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(896); cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    double tl = 0, tt = 0; const int reps = 2000;
    for (int r = 0; r < reps + 100; ++r) {
        auto t0 = std::chrono::steady_clock::now();
        cudaLaunchKernelEx(&cfg, k, blob, o);
        auto t1 = std::chrono::steady_clock::now();
        cudaStreamSynchronize(st);
        auto t2 = std::chrono::steady_clock::now();
        if (r >= 100) { tl += std::chrono::duration<double, std::micro>(t1 - t0).count(); tt += std::chrono::duration<double, std::micro>(t2 - t0).count(); }
    }
    printf("params %5d B: launch call %.2f us, launch+sync round trip %.2f us\n", B, tl / reps, tt / reps);
}
int main() {
    int* o; cudaMalloc(&o, 64);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    run<256>(st, o); run<1024>(st, o); run<2048>(st, o); run<3328>(st, o); run<4096>(st, o); run<8192>(st, o); run<16384>(st, o);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
