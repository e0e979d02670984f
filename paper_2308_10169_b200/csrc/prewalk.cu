// prewalk.cu -- the next frame's initialisation walk, ahead of time.
//
// A frame's swarm starts from the first 2RD words of the mt19937_64 stream of
// its seed (init_swarm, swarm.hpp:94-132: x then v draws), and the stream is
// sequential: inside the fused kernel this walk is ~70 generator passes, the
// largest fixed cost of a latency-bound frame.  The seed of the NEXT frame of
// a scenario is known to the scenario runner (derive_seed(root, "plan", f+1),
// simenv.hpp:239-276) and to a scene batch (per-scene roots), so the walk of
// frame f+1 runs here, on a spare SM, while frame f plans on its cluster.  It
// leaves every tempered init word in HBM plus the generator's last pair of
// blocks (where the step draws continue) and publishes a sequence number; the
// planning kernel of frame f+1 waits for that number (bounded) and reads its
// own rows' words instead of walking -- or walks itself when the number does
// not arrive in time.  Same generator code (mt19937.cuh), same words.
#include "swarm_kernel.cuh"
#include "mt19937.cuh"
#include "philox.cuh"

namespace sepso {

// One CTA per swarm: words[s * nwords + w] = tempered word w of swarm s's
// stream (w < nwords = 2RD); pairs[s * kPrePairWords ..] = the generator's
// latest pair (624 raw words) and the block count; flags[s] = seq when done.
// (words are stored untempered: the reader tempers the few it keeps)
struct MtSeeded {                    // one swarm's seeded state, computed by the host (0.3 us there)
    unsigned long long w[312];
};

__global__ void __launch_bounds__(512) k_init_walk(const unsigned long long* seeds,
                                                   const unsigned long long* roots, unsigned long long tag_hash,
                                                   int frame, unsigned long long seed0, long long nwords,
                                                   unsigned long long* words, unsigned long long* pairs, int* flags,
                                                   int seq, const __grid_constant__ MtSeeded st0, int has_st0) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords];
    const int s = blockIdx.x, tid = threadIdx.x;
    MtState mt{buf, 0, 0};
    const MtGroup g{tid, int(blockDim.x), 0};
    if (has_st0) {                   // one swarm, the host's seeded state
        for (int i = tid; i < 312; i += blockDim.x) buf[312 + i] = st0.w[i];
        __syncthreads();
    } else {
        const uint64_t seed = seeds ? seeds[s]
                                    : (roots ? splitmix64(splitmix64(roots[s] ^ tag_hash) + uint64_t(frame)) : seed0);
        mt_seed(mt, g, seed);
    }
    unsigned long long* out = words + size_t(s) * size_t(nwords);
    mt_generate<0, true>(mt, g, 0, nwords, [&](int w, unsigned long long word) { __stcg(out + w, word); });
    __syncthreads();
    unsigned long long* pr = pairs + size_t(s) * kPrePairWords;
    for (int i = tid; i < 624; i += blockDim.x) __stcg(pr + i, buf[mt.cur * 624 + i]);
    if (tid == 0) __stcg(pr + 624, (unsigned long long)mt.blocks);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(flags + s), "r"(seq) : "memory");
    }
}

int launch_init_walk(int n, const unsigned long long* seeds, const unsigned long long* roots,
                     unsigned long long tag_hash, int frame, unsigned long long seed0, long long nwords,
                     unsigned long long* words, unsigned long long* pairs, int* flags, int seq,
                     const unsigned long long* seeded_host, void* stream) {
    if (n <= 0) return 0;
    MtSeeded st0;
    const int has = seeded_host != nullptr && n == 1;
    if (has) for (int i = 0; i < 312; ++i) st0.w[i] = seeded_host[i];
    k_init_walk<<<n, 512, 0, static_cast<cudaStream_t>(stream)>>>(seeds, roots, tag_hash, frame, seed0, nwords,
                                                                    words, pairs, flags, seq, st0, has);
    return int(cudaGetLastError());
}

} // namespace sepso
