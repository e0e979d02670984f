// swarm_kernel.cuh -- shared declarations of the fused swarm kernel.
//
// One thread-block CLUSTER runs one whole swarm (a planning frame, a DTPSO run
// or one HSEF inner run) from initialisation to its last iteration with the
// swarm state resident in shared memory.  CTA c of the cluster owns the
// contiguous particle rows [c*Rc, min(G*N, (c+1)*Rc)) of the reference's
// row-major (g, n) order (swarm.hpp:18-49).  Per iteration:
//   fitness (+ Q)           geometry.hpp:196-241 / benchmarks.hpp:56-88
//   pbest + group partials  runner.hpp:68-80     (per CTA)
//   partials (and their rows) pushed into every peer's shared memory with
//   st.async, counted on the receiver's mbarrier -- no cluster barrier
//   gbest/tbest             runner.hpp:81-91     (every CTA, same decisions)
//   window push + AT test   planner.hpp:179-187, 138-149
//   step draws + update     swarm.hpp:59-70, 138-174 (mt19937_64 or Philox)
// A grid of n_swarms clusters batches independent swarms (HSEF candidates,
// planning queries, benchmark trials) into one launch.
#pragma once
#include <cstddef>
#include <cstdint>

namespace sepso {

enum RngKind : int { kPhilox = 0, kMt19937 = 1 };

enum ProblemKind : int {
    kPath = 0, kSphere = 1, kRosenbrock = 2, kRastrigin = 3, kGriewank = 4, kAckley = 5
};

// Device world record (one per scene), built by the host from sf_world.
//   [0, 64)   header: width, height, start xy, target xy (double), n_obs, n_verts
//   [64, ..)  uint32 vertex offsets[max_obs + 1]
//   then      double verts[2 * max_verts]           (8-byte aligned)
//   then      double vel[2 * max_obs]               (dynamic obstacles; world stepping)
struct WorldHeader {
    double width, height, sx, sy, tx, ty;
    uint32_t n_obs, n_verts;
    double svx, svy, tvx, tvy;   // endpoint velocities (world stepping only)
};
static_assert(sizeof(WorldHeader) == 88, "world header layout");

struct WorldLayout {
    int max_obs, max_verts;
    size_t off_offsets, off_verts, off_vel, stride;
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline WorldLayout world_layout(int max_obs, int max_verts) {
    WorldLayout w{max_obs, max_verts, 0, 0, 0, 0};
    w.off_offsets = 96;
    w.off_verts = (w.off_offsets + 4 * size_t(max_obs + 1) + 7) & ~size_t(7);
    w.off_vel = w.off_verts + 16 * size_t(max_verts);
    w.stride = (w.off_vel + 16 * size_t(max_obs) + 15) & ~size_t(15);
    return w;
}

struct SwarmOut {
    double fitness;
    double length;
    uint32_t q;
    uint32_t iterations;
    uint32_t truncated;
    uint32_t status;        // 0 ok, 2 non-finite fitness
    uint32_t bad_g, bad_n, bad_k, window_len;
};

// Resident planner (sf_plan_frame's fast path): the host posts a job -- the
// frame's input bytes, laid out as the ParamPayload inline block -- into
// pinned, device-mapped memory and bumps job_seq; the resident cluster copies
// the bytes into shared memory, plans the frame, stores the record into the
// pinned output block and sets done_seq = job_seq.  The cluster exits on
// `quit` or after idle_ns without a job, clearing `alive` (the host then
// relaunches it for the next job; a job posted in the race is served by the
// new cluster, which starts from done_seq).
struct ServerCtl {
    volatile uint32_t job_seq;     // host: the latest posted job
    volatile uint32_t quit;        // host: 1 = exit now
    volatile uint32_t done_seq;    // device: the latest finished job
    volatile uint32_t alive;       // host sets 1 before a launch, device clears on exit
    unsigned long long idle_ns;    // device exits after this long without a job
    uint32_t job_bytes;            // bytes of job[] a job uses
    uint32_t pad[3];
    unsigned long long t_pick, t_ready, t_done;   // %globaltimer of the last job: seen, inputs staged, published
    long long c_ready, c_done;                    // clock64 at staged / published (the SM clock over the frame)
    unsigned long long t_init, t_loop, t_iter;    // %globaltimer after the initialisation / the record / the iterations
    unsigned long long t_pre, t_wait;             // after the constants (prelude) / the init walk's arrival
    unsigned long long t_mark[16];                 // finer %globaltimer stamps (SEPSO_RESIDENT_TRACE)
    alignas(16) unsigned char job[4608];   // = kInlineBytes
};

struct SwarmParams {
    // shape
    int n_swarms, G, N, D, C, rows_per_cta, max_local_groups;
    int nthreads, entry_cap;
    int cap;                 // iteration budget (T or max_iters_per_frame)
    int auto_truncate, carry, tw, warm;
    double alpha, beta, delta, pi_radius;
    int beta_int;            // >= 1: beta is this small integer (exact repeated product)
    double at_gap;           // delta * sqrt(2 tw) * (1 + 1e-9): exact AT pre-test bound
    int rng;                 // 0: Philox counter stream, 1: mt19937_64 (the reference's stream)
    // inputs
    const double* hypers;  long long hypers_stride;   // doubles between swarms (0 = shared)
    const unsigned long long* seeds;
    // alternatively seeds derived on device: derive_seed(roots[s], tag, frame_index)
    // (rng.hpp:52-59) with tag_hash = fnv1a64(tag)
    const unsigned long long* roots; unsigned long long tag_hash; int frame_index;
    const unsigned char* worlds; long long world_stride; int max_obs, max_verts;
    int off_offsets, off_verts, off_vel;
    double step_dt;          // scene batches: advance the world record by dt after planning (0: off)
    const double* prev; const unsigned char* has_prev;  // per swarm: D values + flag
    const double* lo; const double* hi;                 // benchmark box (D); path: from world
    // window state (per swarm: tw values oldest..newest, effective length)
    double* win_vals; int* win_len;
    // outputs
    SwarmOut* out; double* best_x; double* trace;
    // debug: per-iteration phase timestamps of swarm 0 / CTA 0 (SEPSO_PHASE_PROF)
    long long* prof;
    // inl != 0: the inputs travel in the launch's ParamPayload (no H2D copy);
    // in_* are their byte offsets there (seeds, worlds, hypers, prev, has_prev,
    // lo, hi, window values, window lengths)
    int inl, in_seed, in_world, in_hyp, in_prev, in_has_prev, in_lo, in_hi, in_win, in_win_len;
    // inline inputs may carry each swarm's seeded mt19937_64 state (312 words,
    // computed by the host from the seed: the standard's 311-step sequential
    // recurrence, ~6 us on one device thread); -1 = seed on the device
    int in_mtst;
    // scene batches: this frame's seeded states, computed by the previous
    // frame's launch (nullptr: seed here), and where to leave the next frame's
    // (derive_seed(root, "plan", frame + 1), seeded by an idle warp during the
    // init walk); n_swarms x 312 words each
    const unsigned long long* mt_pre;
    unsigned long long* mt_next;
    // the init walk done ahead of time (prewalk.cu): per swarm 2RD tempered
    // words, the generator's last pair + block count (kPrePairWords), and a
    // flag that reads pre_seq once they are complete; nullptr = walk here.
    // Inline inputs carry the same in a PreRec at byte in_pre (-1: none).
    const unsigned long long* pre_words;
    const unsigned long long* pre_pair;
    const int* pre_flag;
    int pre_seq, in_pre;
    // resident planner (inl layout, one swarm): jobs from here; nullptr = one pass
    ServerCtl* srv;
    // consistency build (-DSEPSO_CHECK): per swarm, CTA and iteration decision words
    long long* dbg;
};

constexpr int kPrePairWords = 640;   // 624 generator words + the block count, padded
struct PreRec {                      // inline form of the pre_* fields (one swarm)
    unsigned long long words, pair, flag;
    int seq, valid;
};

// Small host-buffer launches (one paper scene: ~1.8 KB of inputs) pass their
// inputs as a kernel parameter block, copied with the launch itself.
constexpr int kInlineBytes = 4608;   // one paper scene: 1,760 B of inputs + the 2,496 B seeded mt19937 state
struct ParamPayload {
    unsigned char bytes[kInlineBytes];
};
static_assert(sizeof(ServerCtl::job) == kInlineBytes, "resident planner job block = the inline payload");
// Phase profiler (SEPSO_PHASE_PROF=1 at run time) exists only in builds with
// -DSEPSO_PROFILE (make PROF=1): the release kernel carries none of its code.
#ifdef SEPSO_PROFILE
constexpr bool kProfiling = true;
#else
constexpr bool kProfiling = false;
#endif
constexpr int kProfPhases = 24;   // 0..11 phase marks, 12/13 generator start/end, 14 B1 end, 15..18 inside B1, 19..21 inside the partials

// One CTA's best (pbest_f, row) of one group, read by its peers over DSMEM in
// a single 16-byte load.
struct Part {
    double f;
    int row, q;
};

struct SmemLayout {
    size_t x, v, pb, pbf, pbq, q, fit, imp, seglen, coef, lo, hi, hyp, gbx, gbf, gbq, chg, tbx,
        win, part, px, allpart, allbad, gtab, ctab, obb, ooff, ofl, vert, edge, list, mt, mbar, misc, job,
        srvcmd, vert64, wcopy, total;
};

#ifdef __CUDACC__
#define SEPSO_LHD __host__ __device__ inline
#else
#define SEPSO_LHD inline
#endif

SEPSO_LHD size_t sm_align(size_t v) { return (v + 15) & ~size_t(15); }

// Shared-memory carve-up of one CTA; identical on host (launch size) and device.
SEPSO_LHD SmemLayout smem_layout(const SwarmParams& p, size_t tsz, bool path) {
    SmemLayout L{};
    const size_t P = size_t(p.rows_per_cta), D = size_t(p.D), G = size_t(p.G);
    const size_t S = size_t(p.D / 2 + 1), LG = size_t(p.max_local_groups), C = size_t(p.C);
    const size_t O = path ? size_t(p.max_obs) : 0, V = path ? size_t(p.max_verts) : 0;
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o = sm_align(o + bytes); return at; };
    L.misc = take(256);
    L.mbar = take(16);                     // partial-exchange mbarriers, one per iteration parity
    L.x = take(P * D * tsz);
    L.v = take(P * D * tsz);
    L.pb = take(P * D * tsz);
    L.pbf = take(P * tsz);
    L.pbq = take(P * 4);
    L.q = take(P * 4);
    L.fit = take(P * tsz);
    L.imp = take(P * 4);
    L.seglen = take((path ? P * S : P * D) * tsz);   // path: segment lengths; benchmarks: per-element terms
    L.coef = take(3 * P * tsz);
    L.lo = take(D * tsz);
    L.hi = take(D * tsz);
    L.hyp = take(G * 6 * tsz);
    L.gbx = take(G * D * tsz);
    L.gbf = take(G * tsz);
    L.gbq = take(G * 4);
    L.chg = take(G * 4);
    L.tbx = take(D * tsz);
    L.win = take(size_t(p.tw) * 8);
    L.part = take(2 * C * LG * 16);        // pushed partials of every CTA, double-buffered
    L.px = take(2 * C * LG * D * tsz);     // and the matching pbest rows
    L.allpart = take(0);
    L.allbad = take(2 * C * 4);            // per-CTA first non-finite row, double-buffered
    L.gtab = take(G * 8);                  // per group: first / last owning CTA
    L.ctab = take(C * 4);                  // per CTA: first group
    L.obb = take(O * 4 * tsz);
    L.ooff = take((O + 1) * 4);
    L.ofl = take(O * 4);
    L.vert = take(V * 2 * tsz);
    L.edge = take(V * 4 * tsz);
    L.list = take(path ? size_t(p.entry_cap) * 4 : 0);
    L.vert64 = take(path && tsz == 4 ? (V * 2 + 4) * 8 : 0);   // FP32 engine: FP64 world for the final record
    // the world record, staged from HBM in one copy (sized from the shape, so
    // the fit check at planning time and the launch agree)
    L.wcopy = take(path ? world_layout(p.max_obs, p.max_verts).stride : 0);
    L.job = take(p.srv ? size_t(kInlineBytes) : 0);     // resident planner: this job's input bytes
    L.srvcmd = take(p.srv ? 16 : 0);                    // resident planner: rank 0's decision
    o = (o + 127) & ~size_t(127);          // generator state on a 128-byte boundary
    L.mt = take(p.rng == 1 ? 4 * 312 * 8 : 0);
    L.total = o;
    return L;
}

// host launchers (swarm_kernel.cu)
int launch_swarms(const SwarmParams& p, const ParamPayload* pl, int problem, bool fp64, void* stream,
                  size_t* smem_bytes_out);
int swarm_smem_bytes(const SwarmParams& p, int problem, bool fp64, size_t* bytes);
int max_smem_per_block();

// simenv.hpp:155-184 on the device: advance n world records in place (FP64,
// the reference's exact operation order).
int launch_step_worlds(unsigned char* worlds, int n, long long stride, int off_offsets,
                       int off_verts, int off_vel, double dt, void* stream);

// prewalk.cu: n swarms' init walks (seeds[s]; derive_seed(roots[s], tag,
// frame) when seeds is null; seed0 when both are; one swarm may bring its
// host-seeded state) into words (untempered) / pairs, flags[s] = seq at the end.
int launch_init_walk(int n, const unsigned long long* seeds, const unsigned long long* roots,
                     unsigned long long tag_hash, int frame, unsigned long long seed0, long long nwords,
                     unsigned long long* words, unsigned long long* pairs, int* flags, int seq,
                     const unsigned long long* seeded_host, void* stream);

} // namespace sepso
