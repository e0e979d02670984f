// calib.cu -- FP32 FFMA throughput probe: the denominator of the fitness
// kernel's FP32 roofline (MEASURED_PEAKS.json carries HBM and bf16 only).
#include <cuda_runtime.h>

#include "../../include/sepso.h"
#include "host_runtime.hpp"

namespace sepso {

__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a, float b) {
    float r[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = float(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = fmaf(r[i], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += r[i];
    if (s == 1.2345f) out[threadIdx.x] = s;   // keep the chains alive
}

} // namespace sepso

extern "C" int sf_measure_fp32_peak(sf_ctx* ctx, double* tflops) {
    using namespace sepso;
    if (!ctx || !tflops) return fail(SF_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(ctx->device);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    float* out = nullptr;
    cudaError_t e = cudaMalloc(&out, 256 * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "calib alloc");
    const int blocks = sms * 8, iters = 1 << 14;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_ffma<<<blocks, 256, 0, ctx->stream>>>(out, 1024, 0.999f, 0.001f);   // warm-up
    cudaEventRecord(a, ctx->stream);
    k_ffma<<<blocks, 256, 0, ctx->stream>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(b, ctx->stream);
    e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (e != cudaSuccess) return cuda_fail(e, "calib run");
    *tflops = 2.0 * 8.0 * double(iters) * blocks * 256.0 / (double(ms) * 1e-3) / 1e12;
    return SF_OK;
}
