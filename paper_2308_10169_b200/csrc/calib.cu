// calib.cu -- FP32 FFMA throughput probe: the denominator of the fitness
// kernel's FP32 roofline (MEASURED_PEAKS.json carries HBM and bf16 only).
#include <cuda_runtime.h>

#include <vector>

#include "../../include/sepso.h"
#include "host_runtime.hpp"
#include "stage_kernels.cuh"

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

// K1 (k_step, the staged TOF update, swarm.hpp:138-174) on a synthetic FP32
// swarm of groups x per_group rows of dim values, the shape of the HBM-staged
// path (config 4): the mean device time of one launch over `reps` launches,
// each after a 256 MiB write that evicts the 126 MB L2 (CUDA events around
// write + K1 minus events around the write alone), and the
// algorithmic bytes of one launch (20 B per element: x, v, pbest read, x, v
// written).  The step draws come from a pre-generated window of words, as
// in the staged mt19937 path.
extern "C" int sf_measure_step_kernel(sf_ctx* ctx, uint32_t groups, uint32_t per_group, uint32_t dim,
                                      uint32_t reps, double* ms_per_launch, double* bytes_per_launch) {
    using namespace sepso;
    if (!ctx || !ms_per_launch || !bytes_per_launch || groups == 0 || per_group == 0 || dim == 0 || reps == 0)
        return fail(SF_INVALID_ARGUMENT, "measure_step_kernel: bad argument");
    cudaSetDevice(ctx->device);
    const size_t R = size_t(groups) * per_group, E = R * dim;
    float *x = nullptr, *v = nullptr, *pb = nullptr, *gb = nullptr, *tb = nullptr, *lo = nullptr, *hi = nullptr;
    double* hyp = nullptr;
    unsigned long long* words = nullptr;
    IterState* gate = nullptr;
    unsigned char* flush = nullptr;
    const size_t flush_bytes = size_t(256) << 20;
    cudaError_t e = cudaMalloc(&x, E * 4);
    if (e == cudaSuccess) e = cudaMalloc(&v, E * 4);
    if (e == cudaSuccess) e = cudaMalloc(&pb, E * 4);
    if (e == cudaSuccess) e = cudaMalloc(&gb, size_t(groups) * dim * 4);
    if (e == cudaSuccess) e = cudaMalloc(&tb, size_t(dim) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&lo, size_t(dim) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&hi, size_t(dim) * 4);
    if (e == cudaSuccess) e = cudaMalloc(&hyp, size_t(groups) * 6 * 8);
    if (e == cudaSuccess) e = cudaMalloc(&words, 3 * R * 8);
    if (e == cudaSuccess) e = cudaMalloc(&gate, sizeof(IterState));
    if (e == cudaSuccess) e = cudaMalloc(&flush, flush_bytes);
    double ms_total = 0.0;
    if (e == cudaSuccess) {
        std::vector<float> hl(dim, 0.f), hh(dim, 1000.f);
        std::vector<double> hy(size_t(groups) * 6);
        for (uint32_t g = 0; g < groups; ++g) {
            const double row[6] = {1.5, 1.3, 1.2, 0.6, 0.3, 0.4};
            for (int j = 0; j < 6; ++j) hy[size_t(g) * 6 + j] = row[j];
        }
        cudaMemcpyAsync(lo, hl.data(), dim * 4, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(hi, hh.data(), dim * 4, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemcpyAsync(hyp, hy.data(), hy.size() * 8, cudaMemcpyHostToDevice, ctx->stream);
        cudaMemsetAsync(x, 0x44, E * 4, ctx->stream);      // ~785 (inside the box)
        cudaMemsetAsync(v, 0, E * 4, ctx->stream);
        cudaMemsetAsync(pb, 0x43, E * 4, ctx->stream);     // ~130
        cudaMemsetAsync(gb, 0x43, size_t(groups) * dim * 4, ctx->stream);
        cudaMemsetAsync(tb, 0x43, size_t(dim) * 4, ctx->stream);
        cudaMemsetAsync(words, 0x5a, 3 * R * 8, ctx->stream);
        cudaMemsetAsync(gate, 0, sizeof(IterState), ctx->stream);
        StageShape sh{int(groups), int(per_group), int(dim), 0, int(R)};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        // per rep: [eviction write + K1] and [eviction write] alone, each between
        // an event pair; their difference is K1 without the event and launch
        // overheads of a single short kernel (~6 us event-to-event here)
        for (uint32_t r = 0; r <= reps && e == cudaSuccess; ++r) {   // r = 0: warm-up
            float ms_fs = 0.f, ms_f = 0.f;
            cudaEventRecord(a, ctx->stream);
            cudaMemsetAsync(flush, int(r & 0xff), flush_bytes, ctx->stream);
            const int st = stage_step(false, sh, hyp, lo, hi, x, v, pb, gb, tb, 1, 0, 2, 30, gate,
                                      ctx->stream, words, 0);
            cudaEventRecord(b, ctx->stream);
            e = cudaEventSynchronize(b);
            if (st != 0 && e == cudaSuccess) e = cudaErrorLaunchFailure;
            cudaEventElapsedTime(&ms_fs, a, b);
            cudaEventRecord(a, ctx->stream);
            cudaMemsetAsync(flush, int((r + 1) & 0xff), flush_bytes, ctx->stream);
            cudaEventRecord(b, ctx->stream);
            if (e == cudaSuccess) e = cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms_f, a, b);
            if (r > 0) ms_total += double(ms_fs) - double(ms_f);
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    cudaFree(x); cudaFree(v); cudaFree(pb); cudaFree(gb); cudaFree(tb); cudaFree(lo); cudaFree(hi);
    cudaFree(hyp); cudaFree(words); cudaFree(gate); cudaFree(flush);
    if (e != cudaSuccess) return cuda_fail(e, "measure_step_kernel");
    *ms_per_launch = ms_total / reps;
    *bytes_per_launch = 20.0 * double(E);
    return SF_OK;
}

#ifdef SEPSO_PROFILE   // mt19937 pass-layout probe (tools/mtprobe.py): PROF builds only, not exported by the release library
#include "mt19937.cuh"

namespace sepso {
// mt19937_64 generator throughput probe: cycles per 312-word block.
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
    if (acc == 42 || sinkbuf[threadIdx.x] == 42.f) out[threadIdx.x] = acc;   // keep the sinks observable
    __syncthreads();
    if (threadIdx.x == 0) *cycles = clock64() - t0;
}
} // namespace sepso

extern "C" int sf_debug_mt_probe(sf_ctx* ctx, long long blocks, int threads, int mode, double* cycles_per_block) {
    using namespace sepso;
    cudaSetDevice(ctx->device);
    unsigned long long* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8);
    k_mt_probe<<<1, threads, 0, ctx->stream>>>(blocks, mode, out, cyc);
    long long h = 0;
    cudaMemcpyAsync(&h, cyc, 8, cudaMemcpyDeviceToHost, ctx->stream);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    cudaFree(out);
    cudaFree(cyc);
    if (e != cudaSuccess) return cuda_fail(e, "mt probe");
    *cycles_per_block = double(h) / double(blocks);
    return SF_OK;
}

#endif  // SEPSO_PROFILE
