// host_runtime.hpp -- host-side C++ of the engine (context, validation,
// staging, the HSEF outer loop and scene state).  Internal to libsepso_cuda.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/sepso.h"
#include "philox.cuh"
#include "swarm_kernel.cuh"

namespace sepso {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

// ------------------------------------------------------------ device memory
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes);
    void release();
};

struct PinnedBuf {
    void* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes);
    void release();
};

} // namespace sepso

namespace sepso {
struct Resident;   // resident planner of sf_plan_frame (capi.cpp)

// The next frame's init walk, ahead of time on a spare SM (prewalk.cu): two
// slots (frame parity), each n swarms x (2RD words, last generator pair, flag).
struct PreWalk {
    DevBuf words[2], pairs[2], flags;
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};   // bulk mode: slot k's walks complete (stream order, no spin)
    bool bulk = false;
    uint64_t seed[2] = {0, 0};     // single-swarm slots: the seed walked
    long long nwords[2] = {0, 0};  // 2RD of the walk in the slot (0: empty)
    int seq[2] = {0, 0};
    int next_seq = 0;
    int n = 0;                     // swarms per slot the buffers hold
};
}

struct sf_ctx {
    int device = 0;
    int precision = SF_FP32;
    int rng = SF_RNG_MT19937;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;         // staged path: the next step's draws are generated here, overlapping the fitness
    cudaEvent_t ev_free[2] = {nullptr, nullptr}, ev_fill[2] = {nullptr, nullptr};   // per step-draw window
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool timing = false;
    double kernel_ms = 0.0;
    uint64_t launches = 0;
    int force_cluster = 0, force_threads = 0;
    uint64_t last_h2d = 0, last_d2h = 0;
    uint64_t l2_flush = 0;
    void* comm = nullptr;
    int rank = 0, nranks = 1;
    sf_allgather_fn xfn = nullptr;   // host all-gather (sf_ctx_set_exchange) when there is no NCCL communicator
    void* xuser = nullptr;
    sepso::DevBuf io, scratch, flush;
    sepso::Resident* resident = nullptr;
    sepso::PreWalk* pre = nullptr;
    // run_scenario: the seed of the frame after the one being planned
    // (derive_seed(root, "plan", f + 1)); its init walk starts while this
    // frame plans
    bool hint_valid = false;
    uint64_t hint_seed = 0;
    sepso::PinnedBuf hio;
};

namespace sepso {

// --------------------------------------------------------------- validation
// Reference preconditions, each reported as SF_INVALID_ARGUMENT.
int validate_hypers(const double* h, uint32_t G);                    // hypers.hpp:31-46
int validate_bounds(const double* lo, const double* hi, uint32_t D); // hypers.hpp:109-120
int validate_world(const sf_world* w);                               // geometry.hpp:55-66
int validate_planner(const sf_planner_config* c);                    // planner.hpp:41-56

// ------------------------------------------------------------ world records
struct WorldPack {
    WorldLayout lay;
    std::vector<unsigned char> bytes;   // n_worlds * lay.stride
};
void pack_worlds(const sf_world* worlds, uint32_t n, WorldPack& out);
void pack_world_into(const sf_world& w, const WorldLayout& lay, unsigned char* dst);

// ------------------------------------------------------------ fused launches
struct FusedPlan {
    SwarmParams p{};
    size_t smem = 0;
    bool fits = false;
    const ParamPayload* payload = nullptr;   // inputs inline in the launch (p.inl)
};
// Pick cluster size / threads / list capacity for n swarms of shape (G, N, D).
FusedPlan plan_fused(sf_ctx* ctx, int problem, int n_swarms, int G, int N, int D, int max_obs,
                     int max_verts, int cap, int tw);

// Launch on ctx->stream, bracketed by timing events when enabled.
int launch_fused(sf_ctx* ctx, FusedPlan& fp, int problem);

// ---------------------------------------------------------- staged (HBM) run
// One swarm with state in HBM, stage kernels per iteration (used when the
// swarm does not fit a cluster, or when SEPSO_FORCE_STAGED=1).
struct StagedRun {
    int problem = kPath;
    int G = 0, N = 0, D = 0, cap = 0;
    const sf_world* world = nullptr;
    const double* lo = nullptr;  // benchmark box
    const double* hi = nullptr;
    double alpha = 30.0, beta = 4.0;
    const double* hypers = nullptr;
    uint64_t seed = 0;
    const double* prev = nullptr;
    int warm = 0;
    double pi_radius = 20.0;
    int auto_truncate = 0, tw = 0;
    double delta = 10.0;
    const double* win_in = nullptr;   // last min(len, tw) values
    int win_len_in = 0;
    // sharding (BASELINE config 4): this rank's groups, the communicator
    int rank = 0, nranks = 1;
    void* comm = nullptr;
    // outputs
    SwarmOut out{};
    std::vector<double> best, trace, win_out;
};
int run_staged(sf_ctx* ctx, StagedRun& r);

// NCCL (dlopen'ed; the process's already-loaded libnccl is reused)
int comm_unique_id(unsigned char id[128]);
int comm_init(void** comm, const unsigned char id[128], int nranks, int rank);
int comm_allgather(void* comm, const void* send, void* recv, size_t bytes, cudaStream_t st);
// All ranks' equal-size host blocks in rank order (recv: nranks * bytes) over
// the context's exchange: the host callback, else NCCL through device staging,
// else (one rank) a copy.
int exchange_allgather(sf_ctx* ctx, const void* send, void* recv, size_t bytes);
void comm_destroy(void* comm);

bool force_staged();

// --------------------------------------------------------- host-side PSO
// The HSEF outer swarm lives on the host (hsef.hpp:144-165); this is the
// reference's batched update restated in C++ over the engine's Philox stream
// (sequential draw counter), compiled with -ffp-contract=off.
struct HostStream {            // RngStream (rng.hpp:13-28) over either engine stream
    uint64_t seed, drawn = 0;
    bool mt;
    std::mt19937_64 eng;
    HostStream(uint64_t s, int rng) : seed(s), mt(rng == SF_RNG_MT19937), eng(s) {}
    uint64_t next() {
        const uint64_t i = drawn++;
        return mt ? eng() : philox_word(seed, i);
    }
    double uniform() { return double(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
};

struct HostSwarm {
    uint32_t G = 0, N = 0, D = 0;
    std::vector<double> x, v, pbx, pbf, gbx, gbf, tbx;
    double tbf = 0.0;
};
void host_init_swarm(HostSwarm& s, const double* hypers, const double* lo, const double* hi,
                     uint32_t G, uint32_t N, uint32_t D, HostStream& rng);
void host_step(HostSwarm& s, const double* hypers, const double* lo, const double* hi,
               HostStream& rng, uint32_t k, uint32_t T);
void host_update_bests(HostSwarm& s, const double* fitness);
void unflatten_hypers(const double* particle, uint32_t groups, double* out);   // hsef.hpp:57-71

uint64_t derive_seed(uint64_t root, const char* tag);
uint64_t derive_seed(uint64_t root, const char* tag, uint64_t index);

} // namespace sepso
