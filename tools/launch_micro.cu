// GPU-side cost of launching an (empty) kernel shaped like the fused planner:
// 16-CTA cluster, 1024 threads, ~200 KB dynamic shared memory.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024, 1) k_empty(int* o) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && o[0] == 12345) o[1] = sm[0];
}
__global__ void k_flush(float* f, size_t n) {
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) f[i] = 0.f;
}
int main() {
    int* o; cudaMalloc(&o, 64); cudaMemset(o, 0, 64);
    float* fl; size_t nf = 64ull << 20; cudaMalloc(&fl, nf * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int smem : {0, 100 * 1024, 200 * 1024}) {
        cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_empty, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int cl : {1, 8, 16}) {
            for (int flush = 0; flush < 2; ++flush) {
                float tot = 0; int reps = 50;
                for (int r = 0; r < reps + 5; ++r) {
                    if (flush) k_flush<<<592, 256>>>(fl, nf);
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(16); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = smem;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    cfg.attrs = at; cfg.numAttrs = 1;
                    cudaEventRecord(a);
                    cudaLaunchKernelEx(&cfg, k_empty, o);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms; cudaEventElapsedTime(&ms, a, b);
                    if (r >= 5) tot += ms;
                }
                printf("smem %6d cluster %2d flush %d: %.2f us\n", smem, cl, flush, 1e3 * tot / reps);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
