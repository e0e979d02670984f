// swarm_kernel.cu -- launch dispatcher of the fused SEPSO swarm kernel and the
// world-stepping kernel.  The kernel template lives in swarm_kernel_body.cuh;
// its instantiations are compiled in swarm_inst_*.cu (in parallel).
#include "swarm_kernel_body.cuh"
#include "swarm_inst.hpp"

namespace sepso {

int launch_swarms(const SwarmParams& p, const ParamPayload* pl, int problem, bool fp64, void* stream,
                  size_t* smem) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool path = problem == kPath;
    const bool ring = p.entry_cap > 0;
    const bool lat = p.nthreads <= 896;
    // the FP32 latency instantiation is compiled for the reference's stream, the
    // register-resident best update and a generator-first shape only
    // (swarm_kernel_body.cuh kLat); anything else takes the generic one
    const int gw0 = p.nthreads / 32 - 4;
    const int lgmax = p.max_local_groups;
    const bool fastok = p.rng == kMt19937 && p.G <= 32 && p.tw <= 32 && p.nthreads >= 192 &&
                        gw0 * 32 >= p.rows_per_cta && lgmax <= gw0;
    const bool lat32 = lat && fastok;
    if (p.srv) {                      // resident planner: one path swarm, latency shapes
        if (!path || ring) return int(cudaErrorInvalidValue);
        if (fp64) return lat ? launch_inst<double, true, false, 896, true, false>(p, pl, problem, st, smem)
                             : launch_inst<double, true, false, 1024, true, false>(p, pl, problem, st, smem);
        return lat32 ? launch_inst<float, true, false, 896, true, true>(p, pl, problem, st, smem)
                     : launch_inst<float, true, false, 1024, true, false>(p, pl, problem, st, smem);
    }
    if (fp64) {
        if (!path) return launch_inst<double, false, false, 1024, false, false>(p, pl, problem, st, smem);
        if (ring) return launch_inst<double, true, true, 1024, false, false>(p, pl, problem, st, smem);
        return lat ? launch_inst<double, true, false, 896, false, false>(p, pl, problem, st, smem)
                   : launch_inst<double, true, false, 1024, false, false>(p, pl, problem, st, smem);
    }
    if (!path) return launch_inst<float, false, false, 1024, false, false>(p, pl, problem, st, smem);
    if (ring) return fastok ? launch_inst<float, true, true, 1024, false, true>(p, pl, problem, st, smem)
                            : launch_inst<float, true, true, 1024, false, false>(p, pl, problem, st, smem);
    return lat32 ? launch_inst<float, true, false, 896, false, true>(p, pl, problem, st, smem)
                 : launch_inst<float, true, false, 1024, false, false>(p, pl, problem, st, smem);
}

int swarm_smem_bytes(const SwarmParams& p, int problem, bool fp64, size_t* bytes) {
    *bytes = smem_layout(p, fp64 ? 8 : 4, problem == kPath).total;
    return 0;
}

// one CTA per world record, one thread per part
__global__ void k_step_worlds(unsigned char* worlds, int n, long long stride, int off_offsets,
                              int off_verts, int off_vel, double dt) {
    if (int(blockIdx.x) >= n) return;
    unsigned char* rec = worlds + size_t(blockIdx.x) * size_t(stride);
    const int nobs = int(reinterpret_cast<const WorldHeader*>(rec)->n_obs);
    for (int t = int(threadIdx.x) - 2; t < nobs; t += blockDim.x) step_world_part(rec, off_offsets, off_verts, off_vel, dt, t);
}

int launch_step_worlds(unsigned char* worlds, int n, long long stride, int off_offsets,
                       int off_verts, int off_vel, double dt, void* stream) {
    if (n <= 0) return 0;
    static thread_local bool carve[kMaxDevices] = {};   // keep the SM shared-memory split of the planning kernel
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices || !carve[dev]) {
        cudaFuncSetAttribute(k_step_worlds, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (dev >= 0 && dev < kMaxDevices) carve[dev] = true;
    }
    k_step_worlds<<<n, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        worlds, n, stride, off_offsets, off_verts, off_vel, dt);
    return int(cudaGetLastError());
}

int max_smem_per_block() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

} // namespace sepso
