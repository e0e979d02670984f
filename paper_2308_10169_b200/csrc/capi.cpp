// capi.cpp -- the extern "C" boundary of libsepso_cuda.so (include/sepso.h).
//
// Each entry point validates exactly what the reference validates (reporting
// SF_INVALID_ARGUMENT where the reference throws std::invalid_argument),
// stages its inputs in ONE pinned host block copied with one H2D transfer,
// launches the fused swarm kernel (or the staged HBM driver for swarms that do
// not fit a cluster), and copies results back with one D2H transfer.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cmath>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "host_runtime.hpp"
#include "mt_jump.hpp"
#include "stage_kernels.cuh"

using namespace sepso;

namespace sepso {
const char* last_error_cstr();
}

namespace {

double now_seconds() {
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double>(clock::now().time_since_epoch()).count();
}

struct DeviceGuard {
    explicit DeviceGuard(int dev) { cudaSetDevice(dev); }
};

size_t al(size_t v) { return (v + 15) & ~size_t(15); }

struct Io {
    size_t world, hyp, seed, prev, has_prev, lo, hi, win, win_len, mtst, pre, out, best, trace, end;
};

// std::mt19937_64(seed)'s state (the standard's seeding recurrence,
// rng.hpp:13-28 constructs the engine from the seed): 312 words
void mt_seeded_state(uint64_t seed, uint64_t* st) {
    uint64_t x = seed;
    st[0] = x;
    for (int i = 1; i < 312; ++i) {
        x = 6364136223846793005ull * (x ^ (x >> 62)) + uint64_t(i);
        st[i] = x;
    }
}

Io io_layout(uint32_t n, size_t world_stride, uint32_t G, uint32_t D, uint32_t cap, uint32_t tw,
             bool per_swarm_hypers, bool mt_state = false) {
    Io o{};
    size_t at = 0;
    auto take = [&](size_t b) { const size_t r = at; at = al(at + b); return r; };
    o.world = take(size_t(n) * world_stride);
    o.hyp = take(size_t(per_swarm_hypers ? n : 1) * G * 6 * 8);
    o.seed = take(size_t(n) * 8);
    o.prev = take(size_t(n) * D * 8);
    o.has_prev = take(size_t(n));
    o.lo = take(size_t(D) * 8);
    o.hi = take(size_t(D) * 8);
    o.win = take(size_t(n) * std::max<uint32_t>(tw, 1) * 8);
    o.win_len = take(size_t(n) * 4);
    o.pre = take(mt_state ? sizeof(PreRec) : 0);
    o.mtst = take(mt_state ? size_t(n) * 312 * 8 : 0);   // last: a job whose init walk is ready omits it
    o.out = take(size_t(n) * sizeof(SwarmOut));
    o.best = take(size_t(n) * D * 8);
    o.trace = take(size_t(n) * cap * 8);
    o.end = at;
    return o;
}

int ensure_io(sf_ctx* ctx, size_t bytes) {
    cudaError_t e = ctx->io.ensure(bytes);
    if (e != cudaSuccess) return cuda_fail(e, "device io block");
    e = ctx->hio.ensure(bytes);
    if (e != cudaSuccess) return cuda_fail(e, "pinned io block");
    return SF_OK;
}

// Apply the reference's window bookkeeping (push_back, then erase one from the
// front when longer than tw; planner.hpp:179-180) for each pushed value.
int carry_window(double* window, uint32_t* window_len, uint32_t window_cap, uint32_t tw,
                 const double* pushes, uint32_t n_push) {
    std::vector<double> w(window, window + *window_len);
    for (uint32_t i = 0; i < n_push; ++i) {
        w.push_back(pushes[i]);
        if (w.size() > tw) w.erase(w.begin());
    }
    if (w.size() > window_cap) return fail(SF_INVALID_ARGUMENT, "window capacity too small");
    std::copy(w.begin(), w.end(), window);
    *window_len = uint32_t(w.size());
    return SF_OK;
}

std::string nonfinite_msg(uint64_t g, uint64_t n, uint64_t k) {   // runner.hpp:22-25
    return "non-finite fitness for particle (" + std::to_string(g) + "," + std::to_string(n) +
           ") at iteration " + std::to_string(k);
}

int beta_integer(double beta) {
    return (beta == double(int(beta)) && beta >= 1.0 && beta <= 64.0) ? int(beta) : 0;
}

// Problem checks shared by run_dtpso / lfv (geometry.hpp:247-256, benchmarks.hpp:22)
int validate_problem(const sf_problem* pr) {
    if (!pr) return fail(SF_INVALID_ARGUMENT, "problem is null");
    if (pr->kind == SF_PROBLEM_PATH) {
        if (pr->dim == 0 || pr->dim % 2 != 0)
            return fail(SF_INVALID_ARGUMENT, "path problem dimension must be even and positive");
        if (!(pr->alpha >= 0.0) || !(pr->beta >= 1.0))
            return fail(SF_INVALID_ARGUMENT, "path_fitness: need alpha >= 0 and beta >= 1");
        return validate_world(pr->world);
    }
    if (pr->kind < SF_PROBLEM_SPHERE || pr->kind > SF_PROBLEM_ACKLEY)
        return fail(SF_INVALID_ARGUMENT, "unknown problem kind");
    if (!pr->lo || !pr->hi) return fail(SF_INVALID_ARGUMENT, "benchmark bounds are null");
    return validate_bounds(pr->lo, pr->hi, pr->dim);
}

// Core batched runner: n swarms of one shape; fills SwarmOut / best / trace /
// window per swarm.  hypers: per swarm (n*G*6) when per_swarm, else G*6.
struct BatchIn {
    int problem = kPath;
    uint32_t n = 0, G = 0, N = 0, D = 0, cap = 0, tw = 0;
    const sf_world* worlds = nullptr;          // n worlds (path)
    const double* lo = nullptr;                // benchmark box
    const double* hi = nullptr;
    double alpha = 30.0, beta = 4.0, delta = 10.0, pi_radius = 20.0;
    int warm = 0, auto_truncate = 0, carry = 0;
    const double* hypers = nullptr;
    bool per_swarm_hypers = false;
    const uint64_t* seeds = nullptr;
    const double* prev = nullptr;              // n*D
    const uint8_t* has_prev = nullptr;         // n
    const double* win_vals = nullptr;          // n*tw (oldest first), carry only
    const uint32_t* win_lens = nullptr;        // n
};
struct BatchOut {
    std::vector<SwarmOut> out;
    std::vector<double> best, trace;
    // when set, run_batch writes the best particles / traces (n x D, n x cap)
    // straight here instead of into best / trace (a batch of 1,024 trials
    // carries 11 MB of traces: one host copy less)
    double* best_dst = nullptr;
    double* trace_dst = nullptr;
};

} // namespace

// ------------------------------------------------------ resident planner
// sf_plan_frame's fast path: one 16-CTA cluster stays resident on its own
// stream and serves frame after frame (ServerCtl, swarm_kernel.cuh).  A call
// writes its input bytes (the same layout the launch parameter block carries)
// into pinned memory the cluster reads over the bus, bumps the job number and
// waits for the record in pinned memory -- no launch, no stream
// synchronisation per frame.  The cluster exits after kResidentIdleNs without
// a job (so device-wide synchronisation by other code is never held up for
// longer), on a shape change, and when the context is destroyed.
struct sepso::Resident {
    ServerCtl* ctl = nullptr;          // pinned, device-mapped
    unsigned char* outb = nullptr;     // pinned output block: the record as tagged chunks
    size_t outb_n = 0;
    std::vector<unsigned char> dec;    // the record decoded (SwarmOut, best, trace)
    cudaStream_t stream = nullptr;
    SwarmParams p{};
    int problem = 0;
    bool fp64 = false, launched = false;
    uint32_t seq = 0;
};

namespace {
constexpr unsigned long long kResidentIdleNs = 1000000ull;   // 1 ms
thread_local double g_trace_post = 0.0, g_trace_seen = 0.0;   // SEPSO_RESIDENT_TRACE: host-side split

// ------------------------------------------------ init walk ahead of time
// (prewalk.cu).  sf_run_scenario knows the next frame's seed; while frame f
// plans on its cluster, one CTA on a spare SM walks frame f+1's 2RD init
// words into the slot frame f does not read.  Frame f+1 finds its seed in a
// slot and reads the words instead of walking (waiting, bounded, for the
// walk's flag).  SEPSO_PREWALK=0 turns it off.
bool prewalk_enabled() {
    static const bool off = [] {
        const char* e = std::getenv("SEPSO_PREWALK");
        return e && e[0] == '0';
    }();
    return !off;
}

// test hook: announce walks but never run them (the planning kernel's fallback)
bool prewalk_late() {
    static const bool late = [] {
        const char* e = std::getenv("SEPSO_PREWALK_TEST");
        return e && std::string(e) == "late";
    }();
    return late;
}

int prewalk_setup(PreWalk*& W, int n, long long nwords) {
    if (!W) {
        W = new PreWalk();
        cudaError_t e = cudaStreamCreateWithFlags(&W->st, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&W->ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "init walk stream");
    }
    const size_t wb = size_t(n) * size_t(nwords) * 8, pb = size_t(n) * kPrePairWords * 8;
    if (W->n < n || W->words[0].n < wb || W->pairs[0].n < pb) {
        cudaStreamSynchronize(W->st);
        cudaError_t e = cudaSuccess;
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
            e = W->words[k].ensure(wb);
            if (e == cudaSuccess) e = W->pairs[k].ensure(pb);
        }
        if (e == cudaSuccess && W->flags.n < size_t(2 * n) * 4) {
            e = W->flags.ensure(size_t(2 * n) * 4);
            if (e == cudaSuccess) e = cudaMemset(W->flags.p, 0, W->flags.n);
        }
        if (e != cudaSuccess) return cuda_fail(e, "init walk buffers");
        W->n = std::max(W->n, n);
        W->nwords[0] = W->nwords[1] = 0;
    }
    return SF_OK;
}

// the slot holding seed's walk (one swarm), or -1; the slot is consumed
int prewalk_take(sf_ctx* ctx, uint64_t seed, long long nwords, PreRec* r) {
    PreWalk* W = ctx->pre;
    r->valid = 0;
    if (!W) return -1;
    for (int k = 0; k < 2; ++k) {
        if (W->nwords[k] == nwords && W->seed[k] == seed) {
            r->words = reinterpret_cast<unsigned long long>(W->words[k].p);
            r->pair = reinterpret_cast<unsigned long long>(W->pairs[k].p);
            r->flag = reinterpret_cast<unsigned long long>(static_cast<int*>(W->flags.p) + k * W->n);
            r->seq = W->seq[k];
            r->valid = 1;
            W->nwords[k] = 0;
            return k;
        }
    }
    return -1;
}

// start the walk of ctx's hinted next seed into the slot the current frame
// does not read (used: the slot it reads, -1 none)
int prewalk_kick(sf_ctx* ctx, long long nwords, int used) {
    PreWalk* W = ctx->pre;
    if (!W || !ctx->hint_valid) return SF_OK;
    const int k = used >= 0 ? used ^ 1 : 0;
    if (++W->next_seq <= 0) W->next_seq = 1;
    W->seq[k] = W->next_seq;
    if (prewalk_late()) {
        W->seed[k] = ctx->hint_seed;
        W->nwords[k] = nwords;
        return SF_OK;
    }
    uint64_t st0[312];
    mt_seeded_state(ctx->hint_seed, st0);
    const int e = launch_init_walk(1, nullptr, nullptr, 0, 0, ctx->hint_seed, nwords,
                                   static_cast<unsigned long long*>(W->words[k].p),
                                   static_cast<unsigned long long*>(W->pairs[k].p),
                                   static_cast<int*>(W->flags.p) + k * W->n, W->seq[k],
                                   reinterpret_cast<const unsigned long long*>(st0), W->st);
    if (e != 0) {
        W->nwords[k] = 0;
        return cuda_fail(cudaError_t(e), "init walk launch");
    }
    W->seed[k] = ctx->hint_seed;
    W->nwords[k] = nwords;
    return SF_OK;
}

void prewalk_destroy(PreWalk*& W) {
    if (!W) return;
    if (W->st) {
        cudaStreamSynchronize(W->st);
        cudaStreamDestroy(W->st);
    }
    if (W->ev) cudaEventDestroy(W->ev);
    for (cudaEvent_t e : W->done)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
        W->words[k].release();
        W->pairs[k].release();
    }
    W->flags.release();
    delete W;
    W = nullptr;
}

bool resident_enabled(sf_ctx* ctx) {
    static const bool off = [] {
        const char* e = std::getenv("SEPSO_RESIDENT");
#ifdef SEPSO_CHECK
        return true;        // the consistency build checks each normal launch
#endif
        return (e && e[0] == '0') || std::getenv("SEPSO_PHASE_PROF") != nullptr;
    }();
    return !off && !ctx->timing;
}

int resident_launch(sf_ctx* ctx, Resident& R) {
    R.ctl->quit = 0;
    R.ctl->alive = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    size_t smem = 0;
    const int e = launch_swarms(R.p, nullptr, R.problem, R.fp64, R.stream, &smem);
    if (e != 0) {
        R.launched = false;
        return cuda_fail(cudaError_t(e), "resident planner launch");
    }
    R.launched = true;
    return SF_OK;
}

}  // namespace

void resident_stop(sf_ctx* ctx) {
    Resident* R = ctx->resident;
    if (!R || !R->launched) return;
    R->ctl->quit = 1;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    cudaStreamSynchronize(R->stream);
    R->ctl->quit = 0;
    R->launched = false;
}

void resident_destroy(sf_ctx* ctx) {
    Resident* R = ctx->resident;
    if (!R) return;
    resident_stop(ctx);
    if (R->ctl) cudaFreeHost(R->ctl);
    if (R->outb) cudaFreeHost(R->outb);
    if (R->stream) cudaStreamDestroy(R->stream);
    delete R;
    ctx->resident = nullptr;
}

namespace {

// Serve one frame: p is the frame's launch parameters (inputs inline in h,
// [0, in_bytes)); the record / best / trace land in the resident output
// block at the io layout's offsets relative to io.out.
int resident_run(sf_ctx* ctx, const SwarmParams& fp_p, int problem, const unsigned char* h, size_t in_bytes,
                 size_t out_off_best, size_t out_off_trace, size_t out_bytes, const unsigned char** results,
                 const std::function<int()>& after_post) {
    Resident*& Rp = ctx->resident;
    if (!Rp) {
        Rp = new Resident();
        cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&Rp->ctl), sizeof(ServerCtl));
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&Rp->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            resident_destroy(ctx);
            return cuda_fail(e, "resident planner setup");
        }
        std::memset(static_cast<void*>(Rp->ctl), 0, sizeof(ServerCtl));
    }
    Resident& R = *Rp;
    const size_t tw = size_t(std::max(fp_p.tw, 1));
    const size_t nchunk = 4 + size_t(fp_p.D) + size_t(std::max(fp_p.cap, 1));   // tagged result chunks
    const size_t need = std::max(((out_bytes + 15) & ~size_t(15)) + tw * 8 + 16, nchunk * 16);
    if (need > R.outb_n) {
        resident_stop(ctx);
        if (R.outb) cudaFreeHost(R.outb);
        R.outb = nullptr;
        R.outb_n = 0;
        const cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&R.outb), std::max<size_t>(need, 4096));
        if (e != cudaSuccess) return cuda_fail(e, "resident output block");
        R.outb_n = std::max<size_t>(need, 4096);
        std::memset(R.outb, 0, R.outb_n);      // no stale chunk tags
        R.dec.assign(R.outb_n, 0);
    }
    SwarmParams p;
    std::memcpy(&p, &fp_p, sizeof p);
    p.out = reinterpret_cast<SwarmOut*>(R.outb);
    p.best_x = reinterpret_cast<double*>(R.outb + out_off_best);
    p.trace = reinterpret_cast<double*>(R.outb + out_off_trace);
    p.win_vals = reinterpret_cast<double*>(R.outb + ((out_bytes + 15) & ~size_t(15)));
    p.win_len = reinterpret_cast<int*>(R.outb + ((out_bytes + 15) & ~size_t(15)) + tw * 8);
    p.has_prev = R.outb;               // inline inputs: only "non-null" matters; the flag travels per job
    p.prof = nullptr;
    p.srv = R.ctl;
    const bool fp64 = ctx->precision == SF_FP64;
    const uint32_t jb = uint32_t((in_bytes + 15) & ~size_t(15));
    if (!R.launched || R.problem != problem || R.fp64 != fp64 || std::memcmp(&p, &R.p, sizeof p) != 0) {
        resident_stop(ctx);
        std::memcpy(&R.p, &p, sizeof p);
        R.problem = problem;
        R.fp64 = fp64;
        R.ctl->idle_ns = kResidentIdleNs;
        const int st = resident_launch(ctx, R);
        if (st) return st;
    }
    std::memcpy(R.ctl->job, h, in_bytes);
    R.ctl->job_bytes = jb;             // per job (the device reads it after the job's sequence number)
    g_trace_post = now_seconds();
    if (++R.seq == 0) ++R.seq;
    const uint32_t s = R.seq;
    std::atomic_thread_fence(std::memory_order_release);
    R.ctl->job_seq = s;
    std::atomic_thread_fence(std::memory_order_seq_cst);
    const double t0 = now_seconds();
    if (after_post) {                  // host work that overlaps the frame (the next init walk's launch)
        const int st = after_post();
        if (st) return st;
    }
    // the record arrives as tagged chunks (swarm_kernel_body.cuh put_chunk):
    // complete when the header and every chunk it implies carry this job's number
    auto tag = [&](size_t i) { return reinterpret_cast<const volatile uint32_t*>(R.outb)[4 * i + 3]; };
    auto complete = [&]() {
        if (tag(0) != s) return false;
        const uint32_t its = reinterpret_cast<const volatile uint32_t*>(R.outb)[0];
        const uint32_t status = reinterpret_cast<const volatile uint32_t*>(R.outb)[2];
        // a failed frame (non-finite fitness) stops before its iteration's
        // trace entry; its record needs none
        const size_t n = 4 + size_t(fp_p.D) + (status == 0 ? std::min<size_t>(its, size_t(std::max(fp_p.cap, 1))) : 0);
        for (size_t i = 1; i < n; ++i)
            if (tag(i) != s) return false;
        return true;
    };
    for (uint64_t spin = 1;; ++spin) {
        if (complete()) break;
        if (R.ctl->alive == 0) {          // the cluster exited (idle) before taking this job: relaunch it
            const cudaError_t e = cudaStreamSynchronize(R.stream);
            R.launched = false;
            if (e != cudaSuccess) return cuda_fail(e, "resident planner");
            if (complete()) break;
            const int st = resident_launch(ctx, R);
            if (st) return st;
            continue;
        }
        if ((spin & 0xffff) == 0) {
            const cudaError_t e = cudaStreamQuery(R.stream);
            if (e != cudaErrorNotReady && R.ctl->done_seq != s && R.ctl->alive != 0) {
                R.launched = false;
                return cuda_fail(e == cudaSuccess ? cudaErrorLaunchFailure : e, "resident planner died");
            }
            if (now_seconds() - t0 > 30.0) {
                resident_stop(ctx);
                return fail(SF_CUDA_ERROR, "resident planner: frame timed out");
            }
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    g_trace_seen = now_seconds();
    // decode the chunks into the launch path's layout (SwarmOut, best, trace)
    {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(R.outb);
        auto dbl = [&](size_t i) {
            const uint64_t u = uint64_t(w[4 * i]) | (uint64_t(w[4 * i + 1]) << 32);
            double v;
            std::memcpy(&v, &u, 8);
            return v;
        };
        SwarmOut o{};
        o.iterations = w[0]; o.q = w[1]; o.status = w[2];
        o.fitness = dbl(1); o.truncated = w[6];
        o.length = dbl(2); o.window_len = w[10];
        o.bad_g = w[12]; o.bad_n = w[13]; o.bad_k = w[14];
        unsigned char* dst = R.dec.data();
        std::memcpy(dst, &o, sizeof o);
        double* best = reinterpret_cast<double*>(dst + out_off_best);
        for (int d = 0; d < fp_p.D; ++d) best[d] = dbl(4 + size_t(d));
        double* tr = reinterpret_cast<double*>(dst + out_off_trace);
        const size_t n = o.status == 0 ? std::min<size_t>(o.iterations, size_t(std::max(fp_p.cap, 1))) : 0;
        for (size_t k = 0; k < n; ++k) tr[k] = dbl(4 + size_t(fp_p.D) + k);
    }
    *results = R.dec.data();
    return SF_OK;
}

// SEPSO_RESIDENT_TRACE: the last frame's device split, printed by
// sf_plan_frame after its wall time is taken
void resident_trace_print(sf_ctx* ctx) {
    if (!ctx->resident || !ctx->resident->ctl) return;
    Resident& R = *ctx->resident;
    std::fprintf(stderr, "[resident] init %.1f us (pre %.1f wait %.1f) loop %.1f us rec %.1f us out %.1f us\n",
                 1e-3 * double(R.ctl->t_init - R.ctl->t_ready), 1e-3 * double(R.ctl->t_pre - R.ctl->t_ready),
                 1e-3 * double(R.ctl->t_wait - R.ctl->t_pre), 1e-3 * double(R.ctl->t_iter - R.ctl->t_init),
                 1e-3 * double(R.ctl->t_loop - R.ctl->t_iter), 1e-3 * double(R.ctl->t_done - R.ctl->t_loop));
    std::fprintf(stderr, "[resident] record cycles: path_length64 %lld rest %lld\n",
                 (long long)(R.ctl->t_mark[7] - R.ctl->t_mark[8]),
                 (long long)((unsigned long long)R.ctl->c_done - R.ctl->t_mark[7]));
    std::fprintf(stderr, "[resident] prelude cycles: to-pre-check %lld to-branch %lld\n",
                 (long long)(R.ctl->t_mark[6] - (unsigned long long)R.ctl->c_ready),
                 (long long)(R.ctl->t_mark[5] - R.ctl->t_mark[6]));
    std::fprintf(stderr, "[resident] prelude cycles: hyp %lld load_world %lld misc %lld consts %lld sync %lld\n",
                 (long long)(R.ctl->t_mark[0] - (unsigned long long)R.ctl->c_ready),
                 (long long)(R.ctl->t_mark[1] - R.ctl->t_mark[0]), (long long)(R.ctl->t_mark[2] - R.ctl->t_mark[1]),
                 (long long)(R.ctl->t_mark[3] - R.ctl->t_mark[2]), (long long)(R.ctl->t_mark[4] - R.ctl->t_mark[3]));
    std::fprintf(stderr, "[resident] host wait %.1f us | device: stage %.1f us, frame %.1f us, SM %.0f MHz, iters %u\n",
                 1e6 * (g_trace_seen - g_trace_post), 1e-3 * double(R.ctl->t_ready - R.ctl->t_pick),
                 1e-3 * double(R.ctl->t_done - R.ctl->t_ready),
                 1e3 * double(R.ctl->c_done - R.ctl->c_ready) / double(R.ctl->t_done - R.ctl->t_ready),
                 reinterpret_cast<const SwarmOut*>(R.outb)->iterations);
}

int run_batch(sf_ctx* ctx, const BatchIn& b, BatchOut& r) {
    DeviceGuard guard(ctx->device);
    const bool path = b.problem == kPath;
    static thread_local WorldPack wp;          // reused: no allocation per frame
    if (path) pack_worlds(b.worlds, b.n, wp);
    const int max_obs = path ? wp.lay.max_obs : 0, max_verts = path ? wp.lay.max_verts : 0;
    FusedPlan fp = plan_fused(ctx, b.problem, int(b.n), int(b.G), int(b.N), int(b.D), max_obs,
                              max_verts, int(b.cap), int(b.tw));
    r.out.assign(b.n, SwarmOut{});
    if (!r.best_dst) r.best.assign(size_t(b.n) * b.D, 0.0);
    if (!r.trace_dst) r.trace.assign(size_t(b.n) * b.cap, 0.0);
    double* const best_out = r.best_dst ? r.best_dst : r.best.data();
    double* const trace_out = r.trace_dst ? r.trace_dst : r.trace.data();
    if (!fp.fits || force_staged()) {
        // staged HBM driver, one swarm at a time
        for (uint32_t s = 0; s < b.n; ++s) {
            StagedRun sr;
            sr.problem = b.problem;
            sr.G = int(b.G); sr.N = int(b.N); sr.D = int(b.D); sr.cap = int(b.cap);
            sr.world = path ? &b.worlds[s] : nullptr;
            sr.lo = b.lo; sr.hi = b.hi;
            sr.alpha = b.alpha; sr.beta = b.beta;
            sr.hypers = b.hypers + (b.per_swarm_hypers ? size_t(s) * b.G * 6 : 0);
            sr.seed = b.seeds[s];
            const bool hp = b.prev && b.has_prev && b.has_prev[s];
            sr.prev = hp ? b.prev + size_t(s) * b.D : nullptr;
            sr.warm = hp ? b.warm : 0;
            sr.pi_radius = b.pi_radius;
            sr.auto_truncate = b.auto_truncate;
            sr.tw = int(b.tw);
            sr.delta = b.delta;
            if (b.carry && b.win_vals) {
                sr.win_in = b.win_vals + size_t(s) * b.tw;
                sr.win_len_in = int(std::min(b.win_lens[s], b.tw));
            }
            const int st = run_staged(ctx, sr);
            if (st != SF_OK) return st;
            r.out[s] = sr.out;
            std::copy(sr.best.begin(), sr.best.end(), best_out + size_t(s) * b.D);
            std::copy(sr.trace.begin(), sr.trace.end(), trace_out + size_t(s) * b.cap);
        }
        return SF_OK;
    }
    SwarmParams& p = fp.p;
    // the seeded generator state travels with the inputs when they go inline
    // (one scene): ~0.3 us on the host instead of ~6 us on one device thread
    const bool mt = ctx->rng == SF_RNG_MT19937;
    Io io = io_layout(b.n, path ? wp.lay.stride : 0, b.G, b.D, b.cap, b.tw, b.per_swarm_hypers, mt);
    if (mt && io.out > size_t(kInlineBytes))
        io = io_layout(b.n, path ? wp.lay.stride : 0, b.G, b.D, b.cap, b.tw, b.per_swarm_hypers, false);
    int st = ensure_io(ctx, io.end);
    if (st != SF_OK) return st;
    unsigned char* h = static_cast<unsigned char*>(ctx->hio.p);
    unsigned char* d = static_cast<unsigned char*>(ctx->io.p);
    if (path) std::memcpy(h + io.world, wp.bytes.data(), wp.bytes.size());
    std::memcpy(h + io.hyp, b.hypers, size_t(b.per_swarm_hypers ? b.n : 1) * b.G * 6 * 8);
    std::memcpy(h + io.seed, b.seeds, size_t(b.n) * 8);
    bool any_prev = false;
    for (uint32_t s = 0; s < b.n; ++s) {
        const bool hp = b.prev && b.has_prev && b.has_prev[s];
        h[io.has_prev + s] = hp ? 1 : 0;
        any_prev |= hp;
        if (hp) std::memcpy(h + io.prev + size_t(s) * b.D * 8, b.prev + size_t(s) * b.D, size_t(b.D) * 8);
    }
    if (!path) {
        std::memcpy(h + io.lo, b.lo, size_t(b.D) * 8);
        std::memcpy(h + io.hi, b.hi, size_t(b.D) * 8);
    }
    if (b.carry) {
        const uint32_t tw = b.tw;
        for (uint32_t s = 0; s < b.n; ++s) {
            const uint32_t len = b.win_lens ? b.win_lens[s] : 0;
            const uint32_t keep = std::min(len, tw);
            double* dst = reinterpret_cast<double*>(h + io.win) + size_t(s) * tw;
            const double* src = b.win_vals + size_t(s) * tw;
            // caller gives the LAST min(len, tw) values, oldest first
            std::copy(src, src + keep, dst);
            reinterpret_cast<int*>(h + io.win_len)[s] = int(keep);
        }
    }
    p.alpha = b.alpha;
    p.beta = b.beta;
    p.beta_int = beta_integer(b.beta);
    p.at_gap = b.delta * std::sqrt(2.0 * double(b.tw)) * (1.0 + 1e-9);
    p.delta = b.delta;
    p.pi_radius = b.pi_radius;
    p.warm = b.warm;
    p.auto_truncate = b.auto_truncate;
    p.carry = b.carry;
    p.hypers = reinterpret_cast<const double*>(d + io.hyp);
    p.hypers_stride = b.per_swarm_hypers ? (long long)b.G * 6 : 0;
    p.seeds = reinterpret_cast<const unsigned long long*>(d + io.seed);
    p.worlds = d + io.world;
    p.world_stride = path ? (long long)wp.lay.stride : 0;
    p.off_offsets = path ? int(wp.lay.off_offsets) : 0;
    p.off_verts = path ? int(wp.lay.off_verts) : 0;
    p.prev = reinterpret_cast<const double*>(d + io.prev);
    p.has_prev = any_prev ? reinterpret_cast<const unsigned char*>(d + io.has_prev) : nullptr;
    p.lo = reinterpret_cast<const double*>(d + io.lo);
    p.hi = reinterpret_cast<const double*>(d + io.hi);
    p.win_vals = reinterpret_cast<double*>(d + io.win);
    p.win_len = reinterpret_cast<int*>(d + io.win_len);
    // small results go straight to the pinned block (mapped into the device
    // address space under UVA): the kernel's stores cross the bus, no D2H copy
    // follows.  Large ones (batched traces) are written on the device and
    // copied back in one transfer.
    const bool zc_out = io.end - io.out <= 64 * 1024;
    unsigned char* ob = zc_out ? h : d;
    p.out = reinterpret_cast<SwarmOut*>(ob + io.out);
    p.best_x = reinterpret_cast<double*>(ob + io.best);
    p.trace = reinterpret_cast<double*>(ob + io.trace);
    // small inputs (one paper scene: ~1.8 KB) ride in the launch's parameter
    // block instead of a separate H2D copy; larger ones take the copy
    static thread_local ParamPayload payload;
    cudaError_t ce = cudaSuccess;
    p.in_mtst = -1;
    p.in_pre = -1;
    p.pre_words = nullptr;
    const long long nwords = 2ll * b.G * b.N * b.D;
    int pre_used = -1;
    bool pre_on = false;
    static const bool no_inline = std::getenv("SEPSO_NO_INLINE") != nullptr;
    // the resident planner takes the job from the pinned block; a launch needs the parameter block
    const bool resident = b.n == 1 && path && zc_out && io.out <= size_t(kInlineBytes) && !no_inline &&
                          resident_enabled(ctx);
    if (io.out <= size_t(kInlineBytes) && !no_inline) {
        if (io.pre != io.out) {
            PreRec* pr = reinterpret_cast<PreRec*>(h + io.pre);
            pr->valid = 0;
            pre_on = b.n == 1 && path && prewalk_enabled() && (ctx->hint_valid || ctx->pre != nullptr);
            if (pre_on) {
                if ((st = prewalk_setup(ctx->pre, 1, nwords)) != SF_OK) return st;
                pre_used = prewalk_take(ctx, b.seeds[0], nwords, pr);
            }
            p.in_pre = int(io.pre);
        }
        // the seeded states, unless the walk is ready (the kernel then needs none)
        if (io.mtst != io.out && !(io.pre != io.out && reinterpret_cast<const PreRec*>(h + io.pre)->valid))
            for (uint32_t sw = 0; sw < b.n; ++sw)
                mt_seeded_state(b.seeds[sw], reinterpret_cast<uint64_t*>(h + io.mtst) + size_t(sw) * 312);
        if (!resident) std::memcpy(payload.bytes, h, io.out);
        p.inl = 1;
        p.in_seed = int(io.seed); p.in_world = int(io.world); p.in_hyp = int(io.hyp);
        p.in_prev = int(io.prev); p.in_has_prev = int(io.has_prev); p.in_lo = int(io.lo);
        p.in_hi = int(io.hi); p.in_win = int(io.win); p.in_win_len = int(io.win_len);
        p.in_mtst = io.mtst != io.out ? int(io.mtst) : -1;
        fp.payload = &payload;
    } else {
        p.inl = 0;
        ce = cudaMemcpyAsync(d, h, io.out, cudaMemcpyHostToDevice, ctx->stream);
    }
    if (ce != cudaSuccess) return cuda_fail(ce, "H2D io");
    ctx->last_h2d = io.out;
    ctx->last_d2h = io.end - io.out;
    if (resident) {
        const unsigned char* res = nullptr;
        // the seeded state travels only when the kernel may need it (no walk ready)
        const bool pre_ready = io.pre != io.out && reinterpret_cast<const PreRec*>(h + io.pre)->valid;
        ctx->last_h2d = pre_ready ? io.mtst : io.out;      // the bytes the cluster reads over the bus
        st = resident_run(ctx, p, b.problem, h, pre_ready ? io.mtst : io.out, io.best - io.out, io.trace - io.out,
                          io.end - io.out, &res,
                          [&]() { return pre_on ? prewalk_kick(ctx, nwords, pre_used) : SF_OK; });
        if (st != SF_OK) return st;
        std::memcpy(r.out.data(), res, sizeof(SwarmOut));
        std::memcpy(best_out, res + (io.best - io.out), size_t(b.D) * 8);
        std::memcpy(trace_out, res + (io.trace - io.out), size_t(b.cap) * 8);
        // the record's tagged chunks the cluster wrote over the bus
        ctx->last_d2h = 16 * (4 + uint64_t(b.D) + std::min<uint64_t>(r.out[0].iterations, b.cap));
        return SF_OK;
    }
    st = launch_fused(ctx, fp, b.problem);
    if (st != SF_OK) return st;
    if (pre_on && (st = prewalk_kick(ctx, nwords, pre_used)) != SF_OK) return st;
    if (!zc_out) {
        ce = cudaMemcpyAsync(h + io.out, d + io.out, io.end - io.out, cudaMemcpyDeviceToHost, ctx->stream);
        if (ce != cudaSuccess) return cuda_fail(ce, "D2H io");
    }
    ce = cudaStreamSynchronize(ctx->stream);
    if (ce != cudaSuccess) return cuda_fail(ce, "swarm kernel");
    std::memcpy(r.out.data(), h + io.out, size_t(b.n) * sizeof(SwarmOut));
    std::memcpy(best_out, h + io.best, size_t(b.n) * b.D * 8);
    std::memcpy(trace_out, h + io.trace, size_t(b.n) * b.cap * 8);
    return SF_OK;
}

void fill_record(const SwarmOut& o, double wall, sf_plan_record* rec) {
    rec->fitness = o.fitness;
    rec->length = o.length;
    rec->intersections = o.q;
    rec->iterations = o.iterations;
    rec->truncated = int32_t(o.truncated);
    rec->collision_free = o.q == 0;
    rec->wall_seconds = wall;
}

} // namespace

extern "C" {

int sf_abi_version(void) { return SEPSO_ABI_VERSION; }
const char* sf_last_error(void) { return last_error_cstr(); }

int sf_ctx_create(int device, int precision, sf_ctx** out) {
    if (!out) return fail(SF_INVALID_ARGUMENT, "out is null");
    if (precision != SF_FP32 && precision != SF_FP64)
        return fail(SF_INVALID_ARGUMENT, "precision must be SF_FP32 or SF_FP64");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) return fail(SF_CUDA_ERROR, "no CUDA device available");
    if (device < 0 || device >= n) return fail(SF_INVALID_ARGUMENT, "device index out of range");
    e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    sf_ctx* c = new sf_ctx();
    c->device = device;
    c->precision = precision;
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "context setup");
    }
    *out = c;
    return SF_OK;
}

int sf_ctx_destroy(sf_ctx* ctx) {
    if (!ctx) return SF_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    resident_destroy(ctx);
    prewalk_destroy(ctx->pre);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
        for (int b = 0; b < 2; ++b) {
            if (ctx->ev_free[b]) cudaEventDestroy(ctx->ev_free[b]);
            if (ctx->ev_fill[b]) cudaEventDestroy(ctx->ev_fill[b]);
        }
    }
    ctx->io.release();
    ctx->scratch.release();
    ctx->flush.release();
    comm_destroy(ctx->comm);
    ctx->hio.release();
    cudaEventDestroy(ctx->ev0);
    cudaEventDestroy(ctx->ev1);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SF_OK;
}

int sf_ctx_precision(const sf_ctx* ctx) { return ctx ? ctx->precision : -1; }
void* sf_ctx_stream(sf_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int sf_ctx_synchronize(sf_ctx* ctx) {
    cudaSetDevice(ctx->device);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? SF_OK : cuda_fail(e, "synchronize");
}

int sf_ctx_set_launch(sf_ctx* ctx, int cluster, int threads) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    if (cluster < 0 || cluster > 16) return fail(SF_INVALID_ARGUMENT, "cluster must be 0..16");
    if (threads < 0 || threads > 1024) return fail(SF_INVALID_ARGUMENT, "threads must be 0..1024");
    ctx->force_cluster = cluster;
    ctx->force_threads = threads;
    return SF_OK;
}

int sf_ctx_set_rng(sf_ctx* ctx, int rng) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    if (rng != SF_RNG_PHILOX && rng != SF_RNG_MT19937) return fail(SF_INVALID_ARGUMENT, "unknown rng");
    ctx->rng = rng;
    return SF_OK;
}

int sf_ctx_rng(const sf_ctx* ctx) { return ctx ? ctx->rng : -1; }

int sf_mt_jump_poly(uint64_t steps, uint64_t* out) {
    if (!out) return fail(SF_INVALID_ARGUMENT, "null argument");
    const std::vector<uint64_t> g = mt_jump_poly(steps);
    std::copy(g.begin(), g.end(), out);
    return SF_OK;
}

int sf_ctx_enable_timing(sf_ctx* ctx, int enable) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    ctx->timing = enable != 0;
    ctx->kernel_ms = 0.0;
    ctx->launches = 0;
    return SF_OK;
}

int sf_ctx_kernel_time(sf_ctx* ctx, double* total_ms, uint64_t* launches) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    if (total_ms) *total_ms = ctx->kernel_ms;
    if (launches) *launches = ctx->launches;
    return SF_OK;
}

int sf_ctx_hint_next_seed(sf_ctx* ctx, uint64_t seed, int valid) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    ctx->hint_seed = seed;
    ctx->hint_valid = valid != 0;
    return SF_OK;
}

// planner.hpp:156-199
int sf_plan_frame(sf_ctx* ctx, const sf_world* world, const double* prev, const double* hypers,
                  const sf_planner_config* cfg, uint64_t seed, double* window, uint32_t* window_len,
                  uint32_t window_cap, sf_plan_record* record, double* best, uint64_t* bad) {
    const double t0 = now_seconds();
    if (!ctx || !record) return fail(SF_INVALID_ARGUMENT, "ctx/record is null");
    int st = validate_planner(cfg);
    if (st) return st;
    if ((st = validate_world(world))) return st;
    if (!hypers) return fail(SF_INVALID_ARGUMENT, "hypers is null");
    if ((st = validate_hypers(hypers, cfg->groups))) return st;
    const bool carry = cfg->window_carryover && window && window_len;
    BatchIn b;
    b.problem = kPath;
    b.n = 1;
    b.G = cfg->groups; b.N = cfg->per_group; b.D = cfg->dim;
    b.cap = cfg->max_iters_per_frame;
    b.tw = cfg->tw;
    b.worlds = world;
    b.alpha = cfg->alpha; b.beta = cfg->beta; b.delta = cfg->delta; b.pi_radius = cfg->pi_radius;
    b.warm = int(cfg->gamma * double(cfg->per_group));            // planner.hpp:37-39
    b.auto_truncate = cfg->auto_truncate;
    b.carry = carry;
    b.hypers = hypers;
    b.seeds = &seed;
    const uint8_t hp = prev ? 1 : 0;
    b.prev = prev;
    b.has_prev = &hp;
    static thread_local std::vector<double> wtail;
    uint32_t wl = 0;
    if (carry) {
        const uint32_t keep = std::min(*window_len, cfg->tw);
        wtail.assign(window + (*window_len - keep), window + *window_len);
        wtail.resize(cfg->tw, 0.0);
        wl = keep;
        b.win_vals = wtail.data();
        b.win_lens = &wl;
    }
    static thread_local BatchOut r;             // reused: no allocation per frame
    st = run_batch(ctx, b, r);
    ctx->hint_valid = false;                    // a next-seed hint serves one call
    if (st) return st;
    const SwarmOut& o = r.out[0];
    if (o.status == 2) {
        if (bad) { bad[0] = o.bad_g; bad[1] = o.bad_n; bad[2] = o.bad_k; }
        return fail(SF_NON_FINITE, nonfinite_msg(o.bad_g, o.bad_n, o.bad_k));
    }
    if (carry && (st = carry_window(window, window_len, window_cap, cfg->tw, r.trace.data(), o.iterations)))
        return st;
    if (best) std::copy(r.best.begin(), r.best.begin() + cfg->dim, best);
    const double t1 = now_seconds();
    fill_record(o, t1 - t0, record);
    static const bool trace = std::getenv("SEPSO_RESIDENT_TRACE") != nullptr;
    if (trace && g_trace_post > t0) {
        std::fprintf(stderr, "[plan_frame] host prep %.2f us, post->seen %.2f us, after %.2f us\n",
                     1e6 * (g_trace_post - t0), 1e6 * (g_trace_seen - g_trace_post), 1e6 * (t1 - g_trace_seen));
        resident_trace_print(ctx);
    }
    return SF_OK;
}

int sf_plan_frames_batched(sf_ctx* ctx, uint32_t n, const sf_world* worlds, const double* prev,
                           const uint8_t* has_prev, const double* hypers,
                           const sf_planner_config* cfg, const uint64_t* seeds, double* windows,
                           uint32_t* window_lens, sf_plan_record* records, double* best,
                           int32_t* statuses, uint64_t* bad) {
    const double t0 = now_seconds();
    if (!ctx || !records || !seeds || !worlds) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (n == 0) return SF_OK;
    int st = validate_planner(cfg);
    if (st) return st;
    if (!hypers) return fail(SF_INVALID_ARGUMENT, "hypers is null");
    if ((st = validate_hypers(hypers, cfg->groups))) return st;
    for (uint32_t s = 0; s < n; ++s)
        if ((st = validate_world(&worlds[s]))) return st;
    const bool carry = cfg->window_carryover && windows && window_lens;
    BatchIn b;
    b.problem = kPath;
    b.n = n;
    b.G = cfg->groups; b.N = cfg->per_group; b.D = cfg->dim;
    b.cap = cfg->max_iters_per_frame;
    b.tw = cfg->tw;
    b.worlds = worlds;
    b.alpha = cfg->alpha; b.beta = cfg->beta; b.delta = cfg->delta; b.pi_radius = cfg->pi_radius;
    b.warm = int(cfg->gamma * double(cfg->per_group));
    b.auto_truncate = cfg->auto_truncate;
    b.carry = carry;
    b.hypers = hypers;
    b.seeds = seeds;
    b.prev = prev;
    b.has_prev = has_prev;
    std::vector<double> wt;
    std::vector<uint32_t> wl;
    if (carry) {
        wt.assign(size_t(n) * cfg->tw, 0.0);
        wl.assign(n, 0);
        for (uint32_t s = 0; s < n; ++s) {
            const uint32_t len = std::min(window_lens[s], cfg->tw);
            const double* src = windows + size_t(s) * cfg->tw;
            std::copy(src, src + len, wt.begin() + size_t(s) * cfg->tw);
            wl[s] = len;
        }
        b.win_vals = wt.data();
        b.win_lens = wl.data();
    }
    BatchOut r;
    if ((st = run_batch(ctx, b, r))) return st;
    const double wall = (now_seconds() - t0) / double(n);
    int any_bad = 0;
    for (uint32_t s = 0; s < n; ++s) {
        const SwarmOut& o = r.out[s];
        if (statuses) statuses[s] = o.status == 2 ? SF_NON_FINITE : SF_OK;
        if (o.status == 2) {
            any_bad = 1;
            if (bad) { bad[3 * s] = o.bad_g; bad[3 * s + 1] = o.bad_n; bad[3 * s + 2] = o.bad_k; }
            continue;
        }
        fill_record(o, wall, &records[s]);
        if (best) std::copy(r.best.begin() + size_t(s) * cfg->dim, r.best.begin() + size_t(s + 1) * cfg->dim,
                            best + size_t(s) * cfg->dim);
        if (carry) {
            // windows are fixed-stride tw slots here: keep the trailing tw values
            uint32_t len = std::min(window_lens[s], cfg->tw);
            if ((st = carry_window(windows + size_t(s) * cfg->tw, &len, cfg->tw, cfg->tw,
                                   r.trace.data() + size_t(s) * b.cap, o.iterations)))
                return st;
            window_lens[s] = len;
        }
    }
    if (any_bad) set_error("one or more scenes produced a non-finite fitness");
    return SF_OK;
}

static int run_dtpso_impl(sf_ctx* ctx, const sf_problem* pr, uint32_t n, const double* hypers,
                          bool per_run, uint32_t G, uint32_t N, uint32_t T, const uint64_t* seeds,
                          BatchOut& r) {
    int st = validate_problem(pr);
    if (st) return st;
    if (T < 1) return fail(SF_INVALID_ARGUMENT, "run_dtpso: iteration count must be >= 1");
    if (G < 1 || N < 1) return fail(SF_INVALID_ARGUMENT, "init_swarm: G, N, D must all be >= 1");
    if (!hypers) return fail(SF_INVALID_ARGUMENT, "hypers is null");
    for (uint32_t s = 0; s < (per_run ? n : 1); ++s)
        if ((st = validate_hypers(hypers + size_t(s) * G * 6, G))) return st;
    BatchIn b;
    b.problem = pr->kind;
    b.n = n;
    b.G = G; b.N = N; b.D = pr->dim; b.cap = T; b.tw = 0;
    std::vector<sf_world> ws;
    if (pr->kind == SF_PROBLEM_PATH) {
        ws.assign(n, *pr->world);
        b.worlds = ws.data();
    }
    b.lo = pr->lo; b.hi = pr->hi;
    b.alpha = pr->alpha; b.beta = pr->beta;
    b.hypers = hypers;
    b.per_swarm_hypers = per_run;
    b.seeds = seeds;
    return run_batch(ctx, b, r);
}

// runner.hpp:97-129
int sf_run_dtpso(sf_ctx* ctx, const sf_problem* pr, const double* hypers, uint32_t G, uint32_t N,
                 uint32_t T, uint64_t seed, double* trace, double* final_point, double* final_fitness,
                 uint64_t* bad) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    BatchOut r;
    const int st = run_dtpso_impl(ctx, pr, 1, hypers, false, G, N, T, &seed, r);
    if (st) return st;
    const SwarmOut& o = r.out[0];
    if (o.status == 2) {
        if (bad) { bad[0] = o.bad_g; bad[1] = o.bad_n; bad[2] = o.bad_k; }
        return fail(SF_NON_FINITE, nonfinite_msg(o.bad_g, o.bad_n, o.bad_k));
    }
    if (trace) std::copy(r.trace.begin(), r.trace.begin() + T, trace);
    if (final_point) std::copy(r.best.begin(), r.best.begin() + pr->dim, final_point);
    if (final_fitness) *final_fitness = o.fitness;
    return SF_OK;
}

int sf_run_dtpso_batched(sf_ctx* ctx, const sf_problem* pr, uint32_t n, const double* hypers,
                         int per_run, uint32_t G, uint32_t N, uint32_t T, const uint64_t* seeds,
                         double* traces, double* final_points, double* final_fitness,
                         int32_t* statuses) {
    if (!ctx || !seeds) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (n == 0) return SF_OK;
    BatchOut r;
    r.trace_dst = traces;              // written in place (null: kept in r, dropped)
    r.best_dst = final_points;
    const int st = run_dtpso_impl(ctx, pr, n, hypers, per_run != 0, G, N, T, seeds, r);
    if (st) return st;
    for (uint32_t s = 0; s < n; ++s) {
        const SwarmOut& o = r.out[s];
        if (statuses) statuses[s] = o.status == 2 ? SF_NON_FINITE : SF_OK;
        if (final_fitness) final_fitness[s] = o.status == 2 ? std::numeric_limits<double>::infinity() : o.fitness;
    }
    return SF_OK;
}

// hsef.hpp:108-119, m candidates per launch
int sf_lfv_batch(sf_ctx* ctx, const sf_problem* pr, uint32_t m, const double* cand,
                 const uint64_t* seeds, uint32_t iG, uint32_t iN, uint32_t iT, double* lfv) {
    if (!ctx || !lfv || !seeds || !cand) return fail(SF_INVALID_ARGUMENT, "null argument");
    const double inf = std::numeric_limits<double>::infinity();
    for (uint32_t i = 0; i < m; ++i) lfv[i] = inf;
    if (m == 0) return SF_OK;
    // invalid inner budgets / problems make every candidate +inf (exceptions caught)
    if (iT < 1 || iG < 1 || iN < 1 || validate_problem(pr) != SF_OK) return SF_OK;
    std::vector<double> hyp(size_t(m) * iG * 6);
    std::vector<uint64_t> sd;
    std::vector<uint32_t> idx;
    std::vector<double> ok_h;
    for (uint32_t i = 0; i < m; ++i) {
        double* h = hyp.data() + size_t(i) * iG * 6;
        unflatten_hypers(cand + size_t(i) * iG * 6, iG, h);
        if (validate_hypers(h, iG) != SF_OK) continue;      // NaN candidates score +inf
        idx.push_back(i);
        sd.push_back(seeds[i]);
        ok_h.insert(ok_h.end(), h, h + iG * 6);
    }
    set_error("");
    if (idx.empty()) return SF_OK;
    BatchOut r;
    const int st = run_dtpso_impl(ctx, pr, uint32_t(idx.size()), ok_h.data(), true, iG, iN, iT, sd.data(), r);
    if (st == SF_CUDA_ERROR) return st;
    if (st != SF_OK) return SF_OK;
    for (size_t j = 0; j < idx.size(); ++j)
        lfv[idx[j]] = r.out[j].status == 2 ? inf : r.out[j].fitness;
    return SF_OK;
}

// hsef.hpp:125-171: outer PSO on the host, inner runs batched on the device
int sf_evolve(sf_ctx* ctx, const sf_problem* pr, uint32_t iG, uint32_t iN, uint32_t iT,
              uint32_t oG, uint32_t oN, uint32_t E, uint64_t seed, const double* outer_hypers,
              double* best_trace, double* round_trace, double* best_hypers, sf_evolution_cb cb,
              void* user) {
    if (!ctx || !outer_hypers) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (E < 1) return fail(SF_INVALID_ARGUMENT, "evolve: evolution count must be >= 1");
    if (iT < 1) return fail(SF_INVALID_ARGUMENT, "evolve: inner iteration count must be >= 1");
    if (iG < 1) return fail(SF_INVALID_ARGUMENT, "HyperEncoding: group count must be >= 1");
    int st = validate_hypers(outer_hypers, oG);
    if (st) return st;
    if (oN < 1) return fail(SF_INVALID_ARGUMENT, "init_swarm: G, N, D must all be >= 1");
    const uint32_t dim = 6 * iG;
    std::vector<double> lo(dim), hi(dim);
    static const double flo[6] = {0.5, 0.5, 0.5, 0.1, 0.05, 0.05};
    static const double fhi[6] = {2.5, 2.5, 2.5, 1.0, 0.8, 1.0};
    for (uint32_t g = 0; g < iG; ++g)
        for (int f = 0; f < 6; ++f) { lo[6 * g + f] = flo[f]; hi[6 * g + f] = fhi[f]; }
    const uint64_t outer_seed = derive_seed(seed, "outer");
    const uint64_t lfv_root = derive_seed(seed, "lfv");
    HostStream rng(outer_seed, ctx->rng);
    HostSwarm s;
    host_init_swarm(s, outer_hypers, lo.data(), hi.data(), oG, oN, dim, rng);
    const uint32_t cand = oG * oN;
    std::vector<double> fit(cand);
    std::vector<uint64_t> seeds(cand);
    uint64_t eval_index = 0;
    // sharded (a communicator or a host exchange): rank r scores candidates
    // [r*cand/n, (r+1)*cand/n), the LFVs are all-gathered, and every rank runs
    // the same outer update -- identical to the unsharded run
    const int nr = std::max(1, ctx->nranks), rk = ctx->rank;
    const uint32_t c0 = uint32_t(uint64_t(rk) * cand / uint32_t(nr)), c1 = uint32_t(uint64_t(rk + 1) * cand / uint32_t(nr));
    const uint32_t slot = (cand + uint32_t(nr) - 1) / uint32_t(nr);
    std::vector<double> mine(slot), all(size_t(slot) * nr);
    for (uint32_t e = 1; e <= E; ++e) {
        for (uint32_t r = 0; r < cand; ++r) seeds[r] = derive_seed(lfv_root, "lfv", eval_index++);
        if (nr == 1) {
            st = sf_lfv_batch(ctx, pr, cand, s.x.data(), seeds.data(), iG, iN, iT, fit.data());
            if (st) return st;
        } else {
            if (c1 > c0) {
                st = sf_lfv_batch(ctx, pr, c1 - c0, s.x.data() + size_t(c0) * dim, seeds.data() + c0, iG, iN, iT,
                                  mine.data());
                if (st) return st;
            }
            if ((st = exchange_allgather(ctx, mine.data(), all.data(), size_t(slot) * 8))) return st;
            for (int q = 0; q < nr; ++q) {
                const uint32_t q0 = uint32_t(uint64_t(q) * cand / uint32_t(nr)), q1 = uint32_t(uint64_t(q + 1) * cand / uint32_t(nr));
                std::copy(all.begin() + size_t(q) * slot, all.begin() + size_t(q) * slot + (q1 - q0), fit.begin() + q0);
            }
        }
        double round_best = std::numeric_limits<double>::infinity();
        for (uint32_t r = 0; r < cand; ++r) round_best = std::min(round_best, fit[r]);
        host_update_bests(s, fit.data());
        if (best_trace) best_trace[e - 1] = s.tbf;
        if (round_trace) round_trace[e - 1] = round_best;
        if (cb) cb(e, s.tbf, user);                                   // hsef.hpp:163
        host_step(s, outer_hypers, lo.data(), hi.data(), rng, e, E);
    }
    if (best_hypers) unflatten_hypers(s.tbx.data(), iG, best_hypers);
    return SF_OK;
}

// ------------------------------------------------------------- stage entries
static size_t tsize(sf_ctx* ctx) { return ctx->precision == SF_FP64 ? 8 : 4; }

static void to_dev_type(sf_ctx* ctx, const double* src, size_t n, std::vector<unsigned char>& out) {
    out.resize(n * tsize(ctx));
    if (ctx->precision == SF_FP64) std::memcpy(out.data(), src, n * 8);
    else for (size_t i = 0; i < n; ++i) reinterpret_cast<float*>(out.data())[i] = float(src[i]);
}
static void from_dev_type(sf_ctx* ctx, const unsigned char* src, size_t n, double* out) {
    if (ctx->precision == SF_FP64) std::memcpy(out, src, n * 8);
    else for (size_t i = 0; i < n; ++i) out[i] = double(reinterpret_cast<const float*>(src)[i]);
}

namespace {
// A tiny device arena for stage calls: sequential sub-allocations of ctx->scratch.
struct Arena {
    sf_ctx* ctx;
    std::vector<std::pair<size_t, size_t>> parts;
    size_t total = 0;
    size_t add(size_t b) { const size_t at = total; total = (total + b + 255) & ~size_t(255); return at; }
    int commit() {
        const cudaError_t e = ctx->scratch.ensure(total);
        return e == cudaSuccess ? SF_OK : cuda_fail(e, "scratch");
    }
    unsigned char* at(size_t off) { return static_cast<unsigned char*>(ctx->scratch.p) + off; }
};
int up(sf_ctx* ctx, void* dst, const void* src, size_t n) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, ctx->stream);
    return e == cudaSuccess ? SF_OK : cuda_fail(e, "H2D");
}
int down(sf_ctx* ctx, void* dst, const void* src, size_t n) {
    const cudaError_t e = cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, ctx->stream);
    return e == cudaSuccess ? SF_OK : cuda_fail(e, "D2H");
}
int sync(sf_ctx* ctx) {
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    return e == cudaSuccess ? SF_OK : cuda_fail(e, "stage kernel");
}
}  // namespace

int sf_init_swarm(sf_ctx* ctx, const double* hypers, const double* lo, const double* hi,
                  uint32_t G, uint32_t N, uint32_t D, uint64_t seed, uint64_t first_draw,
                  const double* prev, uint32_t warm, double pi_radius, double* x, double* v) {
    if (!ctx || !x || !v) return fail(SF_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(ctx->device);
    int st = validate_hypers(hypers, G);
    if (st) return st;
    if ((st = validate_bounds(lo, hi, D))) return st;
    if (N < 1) return fail(SF_INVALID_ARGUMENT, "init_swarm: G, N, D must all be >= 1");
    const size_t ts = tsize(ctx), E = size_t(G) * N * D;
    Arena a{ctx};
    const size_t oh = a.add(size_t(G) * 48), olo = a.add(D * ts), ohi = a.add(D * ts),
                 op = a.add(D * 8), ox = a.add(E * ts), ov = a.add(E * ts), opb = a.add(E * ts);
    if ((st = a.commit())) return st;
    std::vector<unsigned char> blo, bhi;
    to_dev_type(ctx, lo, D, blo);
    to_dev_type(ctx, hi, D, bhi);
    up(ctx, a.at(oh), hypers, size_t(G) * 48);
    up(ctx, a.at(olo), blo.data(), blo.size());
    up(ctx, a.at(ohi), bhi.data(), bhi.size());
    if (prev) up(ctx, a.at(op), prev, size_t(D) * 8);
    const StageShape s{int(G), int(N), int(D), 0, int(G * N)};
    unsigned long long* words = nullptr;
    if (ctx->rng == SF_RNG_MT19937) {   // the window [first_draw, first_draw + 2RD) of the reference stream
        DevBuf& wb = ctx->flush;
        const size_t n = 2 * E;
        cudaError_t ce = wb.ensure(n * 8 + sizeof(MtPersist));
        if (ce != cudaSuccess) return cuda_fail(ce, "mt window");
        words = static_cast<unsigned long long*>(wb.p);
        MtPersist* g = reinterpret_cast<MtPersist*>(static_cast<unsigned char*>(wb.p) + n * 8);
        const int fe = stage_mt_fill(g, seed, true, (long long)first_draw, (long long)(first_draw + n), words,
                                     ctx->stream);
        if (fe) return cuda_fail(cudaError_t(fe), "stage_mt_fill");
    }
    const int e = stage_init(ctx->precision == SF_FP64, s, reinterpret_cast<double*>(a.at(oh)), a.at(olo),
                             a.at(ohi), seed, first_draw, prev ? reinterpret_cast<double*>(a.at(op)) : nullptr,
                             prev ? int(warm) : 0, pi_radius, a.at(ox), a.at(ov), a.at(opb), ctx->stream, words,
                             (long long)first_draw);
    if (e) return cuda_fail(cudaError_t(e), "stage_init");
    std::vector<unsigned char> hx(E * ts), hv(E * ts);
    down(ctx, hx.data(), a.at(ox), hx.size());
    down(ctx, hv.data(), a.at(ov), hv.size());
    if ((st = sync(ctx))) return st;
    from_dev_type(ctx, hx.data(), E, x);
    from_dev_type(ctx, hv.data(), E, v);
    return SF_OK;
}

int sf_step(sf_ctx* ctx, const double* hypers, const double* lo, const double* hi, uint32_t G,
            uint32_t N, uint32_t D, double* x, double* v, const double* pbx, const double* gbx,
            const double* tbx, uint64_t seed, uint64_t first_draw, uint32_t k, uint32_t T) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    DeviceGuard guard(ctx->device);
    if (T == 0) return fail(SF_INVALID_ARGUMENT, "inertia_at: total iteration count must be >= 1");
    if (k > T) return fail(SF_INVALID_ARGUMENT, "inertia_at: k out of range");
    if (G < 1 || N < 1 || D < 1) return fail(SF_INVALID_ARGUMENT, "step: empty swarm");
    const size_t ts = tsize(ctx), E = size_t(G) * N * D;
    Arena a{ctx};
    const size_t oh = a.add(size_t(G) * 48), olo = a.add(D * ts), ohi = a.add(D * ts),
                 ox = a.add(E * ts), ov = a.add(E * ts), opb = a.add(E * ts),
                 og = a.add(size_t(G) * D * ts), ot = a.add(D * ts);
    int st = a.commit();
    if (st) return st;
    std::vector<unsigned char> b;
    up(ctx, a.at(oh), hypers, size_t(G) * 48);
    to_dev_type(ctx, lo, D, b); up(ctx, a.at(olo), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, hi, D, b); up(ctx, a.at(ohi), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, x, E, b); up(ctx, a.at(ox), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, v, E, b); up(ctx, a.at(ov), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, pbx, E, b); up(ctx, a.at(opb), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, gbx, size_t(G) * D, b); up(ctx, a.at(og), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, tbx, D, b); up(ctx, a.at(ot), b.data(), b.size()); sync(ctx);
    const StageShape s{int(G), int(N), int(D), 0, int(G * N)};
    unsigned long long* words = nullptr;
    if (ctx->rng == SF_RNG_MT19937) {   // draws [first_draw, first_draw + 3R) of the reference stream
        DevBuf& wb = ctx->flush;
        const size_t n = 3 * size_t(G) * N;
        cudaError_t ce = wb.ensure(n * 8 + sizeof(MtPersist));
        if (ce != cudaSuccess) return cuda_fail(ce, "mt window");
        words = static_cast<unsigned long long*>(wb.p);
        MtPersist* g = reinterpret_cast<MtPersist*>(static_cast<unsigned char*>(wb.p) + n * 8);
        const int fe = stage_mt_fill(g, seed, true, (long long)first_draw, (long long)(first_draw + n), words,
                                     ctx->stream);
        if (fe) return cuda_fail(cudaError_t(fe), "stage_mt_fill");
    }
    const int e = stage_step(ctx->precision == SF_FP64, s, reinterpret_cast<double*>(a.at(oh)), a.at(olo),
                             a.at(ohi), a.at(ox), a.at(ov), a.at(opb), a.at(og), a.at(ot), seed, first_draw,
                             int(k), int(T), nullptr, ctx->stream, words, (long long)first_draw);
    if (e) return cuda_fail(cudaError_t(e), "stage_step");
    std::vector<unsigned char> hx(E * ts), hv(E * ts);
    down(ctx, hx.data(), a.at(ox), hx.size());
    down(ctx, hv.data(), a.at(ov), hv.size());
    if ((st = sync(ctx))) return st;
    from_dev_type(ctx, hx.data(), E, x);
    from_dev_type(ctx, hv.data(), E, v);
    return SF_OK;
}

int sf_update_bests(sf_ctx* ctx, uint32_t G, uint32_t N, uint32_t D, const double* x, double* pbx,
                    double* pbf, double* gbx, double* gbf, double* tbx, double* tbf,
                    const double* fitness) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    DeviceGuard guard(ctx->device);
    if (G < 1 || N < 1 || D < 1) return fail(SF_INVALID_ARGUMENT, "update_bests: empty swarm");
    const bool fp64 = ctx->precision == SF_FP64;
    const size_t ts = tsize(ctx), R = size_t(G) * N, E = R * D;
    Arena a{ctx};
    const size_t ox = a.add(E * ts), opb = a.add(E * ts), opbf = a.add(R * ts), ofit = a.add(R * ts),
                 oq = a.add(R * 4), opbq = a.add(R * 4), opf = a.add(G * ts), oprow = a.add(G * 4),
                 opq = a.add(G * 4), ogb = a.add(size_t(G) * D * ts), ogbf = a.add(G * ts),
                 ogbq = a.add(G * 4), otb = a.add(D * ts), ocand = a.add(cand_bytes(fp64, D)),
                 ost = a.add(sizeof(IterState));
    int st = a.commit();
    if (st) return st;
    std::vector<unsigned char> b;
    to_dev_type(ctx, x, E, b); up(ctx, a.at(ox), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, pbx, E, b); up(ctx, a.at(opb), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, pbf, R, b); up(ctx, a.at(opbf), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, fitness, R, b); up(ctx, a.at(ofit), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, gbx, size_t(G) * D, b); up(ctx, a.at(ogb), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, gbf, G, b); up(ctx, a.at(ogbf), b.data(), b.size()); sync(ctx);
    to_dev_type(ctx, tbx, D, b); up(ctx, a.at(otb), b.data(), b.size()); sync(ctx);
    cudaMemsetAsync(a.at(oq), 0, R * 4, ctx->stream);
    cudaMemsetAsync(a.at(opbq), 0, R * 4, ctx->stream);
    cudaMemsetAsync(a.at(ogbq), 0, G * 4, ctx->stream);
    IterState is{};
    // the stage tbest uses the FP32/FP64 value of the incoming tbest
    is.tbest_f = fp64 ? *tbf : double(float(*tbf));
    is.tbest_group = -1;
    is.nonfinite_row = INT_MAX;
    up(ctx, a.at(ost), &is, sizeof(is));
    const StageShape s{int(G), int(N), int(D), 0, int(R)};
    IterState* dst = reinterpret_cast<IterState*>(a.at(ost));
    int e = stage_pbest_partials(fp64, s, a.at(ox), a.at(ofit), reinterpret_cast<int*>(a.at(oq)), a.at(opb),
                                 a.at(opbf), reinterpret_cast<int*>(a.at(opbq)), nullptr, a.at(opf),
                                 reinterpret_cast<int*>(a.at(oprow)), reinterpret_cast<int*>(a.at(opq)),
                                 nullptr, ctx->stream);
    if (!e) e = stage_group_bests(fp64, s, a.at(opf), reinterpret_cast<int*>(a.at(oprow)),
                                  reinterpret_cast<int*>(a.at(opq)), a.at(opb), a.at(ogb), a.at(ogbf),
                                  reinterpret_cast<int*>(a.at(ogbq)), a.at(ocand), nullptr, ctx->stream);
    if (!e) e = stage_finish(fp64, int(D), a.at(ocand), 1, a.at(otb), dst, nullptr, 0, 0, 0.0, 1, 1,
                             nullptr, ctx->stream);
    if (e) return cuda_fail(cudaError_t(e), "update_bests stages");
    std::vector<unsigned char> hpb(E * ts), hpbf(R * ts), hgb(size_t(G) * D * ts), hgbf(G * ts), htb(D * ts);
    IterState fin{};
    down(ctx, hpb.data(), a.at(opb), hpb.size());
    down(ctx, hpbf.data(), a.at(opbf), hpbf.size());
    down(ctx, hgb.data(), a.at(ogb), hgb.size());
    down(ctx, hgbf.data(), a.at(ogbf), hgbf.size());
    down(ctx, htb.data(), a.at(otb), htb.size());
    down(ctx, &fin, a.at(ost), sizeof(fin));
    if ((st = sync(ctx))) return st;
    from_dev_type(ctx, hpb.data(), E, pbx);
    from_dev_type(ctx, hpbf.data(), R, pbf);
    from_dev_type(ctx, hgb.data(), size_t(G) * D, gbx);
    from_dev_type(ctx, hgbf.data(), G, gbf);
    from_dev_type(ctx, htb.data(), D, tbx);
    *tbf = fin.tbest_f;
    return SF_OK;
}

int sf_eval_path_rows(sf_ctx* ctx, const sf_world* world, const double* xs, uint32_t rows,
                      uint32_t D, double alpha, double beta, double* fitness, uint32_t* q) {
    if (!ctx || !xs || !fitness) return fail(SF_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(ctx->device);
    if (D == 0 || D % 2 != 0) return fail(SF_INVALID_ARGUMENT, "decode_path: dimension must be even and positive");
    if (alpha < 0.0 || beta < 1.0) return fail(SF_INVALID_ARGUMENT, "path_fitness: need alpha >= 0 and beta >= 1");
    int st = validate_world(world);
    if (st) return st;
    if (rows == 0) return SF_OK;
    const bool fp64 = ctx->precision == SF_FP64;
    const size_t ts = tsize(ctx);
    WorldPack wp;
    pack_worlds(world, 1, wp);
    Arena a{ctx};
    const size_t ow = a.add(wp.bytes.size()), ox = a.add(size_t(rows) * D * ts), of = a.add(size_t(rows) * ts),
                 oq = a.add(size_t(rows) * 4);
    if ((st = a.commit())) return st;
    std::vector<unsigned char> b;
    up(ctx, a.at(ow), wp.bytes.data(), wp.bytes.size());
    to_dev_type(ctx, xs, size_t(rows) * D, b);
    up(ctx, a.at(ox), b.data(), b.size());
    if (ctx->timing) cudaEventRecord(ctx->ev0, ctx->stream);
    const int e = stage_eval_path(fp64, a.at(ow), wp.lay.max_obs, wp.lay.max_verts, int(wp.lay.off_offsets),
                                  int(wp.lay.off_verts), int(D), int(rows), a.at(ox), alpha, beta, a.at(of),
                                  reinterpret_cast<int*>(a.at(oq)), nullptr, ctx->stream);
    if (e) return cuda_fail(cudaError_t(e), "stage_eval_path");
    if (ctx->timing) cudaEventRecord(ctx->ev1, ctx->stream);
    std::vector<unsigned char> hf(size_t(rows) * ts);
    down(ctx, hf.data(), a.at(of), hf.size());
    if (q) down(ctx, q, a.at(oq), size_t(rows) * 4);
    if ((st = sync(ctx))) return st;
    if (ctx->timing) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        ctx->kernel_ms += ms;
        ctx->launches += 1;
    }
    from_dev_type(ctx, hf.data(), rows, fitness);
    return SF_OK;
}

int sf_eval_bench_rows(sf_ctx* ctx, int kind, const double* xs, uint32_t rows, uint32_t D,
                       double* fitness) {
    if (!ctx || !xs || !fitness) return fail(SF_INVALID_ARGUMENT, "null argument");
    DeviceGuard guard(ctx->device);
    if (kind < SF_PROBLEM_SPHERE || kind > SF_PROBLEM_ACKLEY) return fail(SF_INVALID_ARGUMENT, "unknown benchmark kind");
    if (rows == 0) return SF_OK;
    const size_t ts = tsize(ctx);
    Arena a{ctx};
    const size_t ox = a.add(size_t(rows) * D * ts), of = a.add(size_t(rows) * ts);
    int st = a.commit();
    if (st) return st;
    std::vector<unsigned char> b;
    to_dev_type(ctx, xs, size_t(rows) * D, b);
    up(ctx, a.at(ox), b.data(), b.size());
    const int e = stage_eval_bench(ctx->precision == SF_FP64, kind, int(D), int(rows), a.at(ox), a.at(of), nullptr,
                                   nullptr, ctx->stream);
    if (e) return cuda_fail(cudaError_t(e), "stage_eval_bench");
    std::vector<unsigned char> hf(size_t(rows) * ts);
    down(ctx, hf.data(), a.at(of), hf.size());
    if ((st = sync(ctx))) return st;
    from_dev_type(ctx, hf.data(), rows, fitness);
    return SF_OK;
}

// planner.hpp:138-149 (the device evaluates the same predicate inside the frame loop)
int sf_should_truncate(const double* window, uint32_t len, int cf, const sf_planner_config* cfg,
                       int* result) {
    if (!cfg || !result) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (len < cfg->tw) { *result = 0; return SF_OK; }
    const double* tail = window + (len - cfg->tw);
    double mean = 0.0;
    for (uint32_t i = 0; i < cfg->tw; ++i) mean += tail[i];
    mean /= double(cfg->tw);
    double var = 0.0;
    for (uint32_t i = 0; i < cfg->tw; ++i) var += (tail[i] - mean) * (tail[i] - mean);
    var /= double(cfg->tw);
    *result = std::sqrt(var) < cfg->delta && cf;
    return SF_OK;
}

// ------------------------------------------------------------- scene state
// simenv.hpp:83-132 over the engine stream (RngStream = Philox contract)
int sf_generate_world(const sf_scenario_config* c, uint64_t seed, int rng_kind, sf_world* w,
                      uint32_t* offsets, sf_point* verts, sf_point* vel) {
    if (!c || !w || !offsets || !verts || !vel) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (!(c->map_size > 0.0)) return fail(SF_INVALID_ARGUMENT, "scenario: map size must be positive");
    if (!(c->min_side > 0.0) || c->min_side > c->max_side || c->max_side >= c->map_size)
        return fail(SF_INVALID_ARGUMENT, "scenario: obstacle side range invalid");
    if (!(c->max_speed > 0.0)) return fail(SF_INVALID_ARGUMENT, "scenario: max speed must be positive");
    if (c->frames < 1) return fail(SF_INVALID_ARGUMENT, "scenario: frame count must be >= 1");
    if (!(c->dt > 0.0)) return fail(SF_INVALID_ARGUMENT, "scenario: dt must be positive");
    HostStream rng(seed, rng_kind);
    const double M = c->map_size;
    w->width = M;
    w->height = M;
    w->start = {0.5 * M, 0.1 * M};
    w->target = {0.5 * M, 0.9 * M};
    w->start_velocity = {0.0, c->start_speed};
    w->target_velocity = {0.0, c->target_speed};
    const double clearance = 2.0;
    const uint32_t total = c->dynamic_obstacles + c->static_obstacles;
    for (uint32_t i = 0; i < total; ++i) {
        bool placed = false;
        for (int attempt = 0; attempt < 200 && !placed; ++attempt) {
            const double ow = rng.uniform(c->min_side, c->max_side);
            const double oh = rng.uniform(c->min_side, c->max_side);
            const double cx = rng.uniform(ow / 2.0, M - ow / 2.0);
            const double cy = rng.uniform(oh / 2.0, M - oh / 2.0);
            auto covers = [&](const sf_point& p) {
                return p.x >= cx - ow / 2.0 - clearance && p.x <= cx + ow / 2.0 + clearance &&
                       p.y >= cy - oh / 2.0 - clearance && p.y <= cy + oh / 2.0 + clearance;
            };
            if (covers(w->start) || covers(w->target)) continue;
            verts[4 * i + 0] = {cx - ow / 2.0, cy - oh / 2.0};
            verts[4 * i + 1] = {cx + ow / 2.0, cy - oh / 2.0};
            verts[4 * i + 2] = {cx + ow / 2.0, cy + oh / 2.0};
            verts[4 * i + 3] = {cx - ow / 2.0, cy + oh / 2.0};
            placed = true;
        }
        if (!placed)                                                 // simenv.hpp:116-118
            return fail(SF_RUNTIME_ERROR, "generate_world: could not place obstacle " + std::to_string(i) +
                                              " clear of start/target");
        offsets[i] = 4 * i;
        if (i < c->dynamic_obstacles) {
            const double speed = c->max_speed * (1.0 - rng.uniform());
            const double angle = rng.uniform(0.0, 2.0 * 3.14159265358979323846);
            vel[i] = {speed * std::cos(angle), speed * std::sin(angle)};
        } else {
            vel[i] = {0.0, 0.0};
        }
    }
    offsets[total] = 4 * total;
    w->n_obstacles = total;
    w->vertex_offsets = offsets;
    w->vertices = verts;
    w->velocities = vel;
    return validate_world(w);                                        // world.validate(), simenv.hpp:129
}

static double reflect_axis(double lo, double hi, double limit, double& v) {   // simenv.hpp:139-149
    if (lo <= 0.0) { v = -v; return -2.0 * lo; }
    if (hi >= limit) { v = -v; return -2.0 * (hi - limit); }
    return 0.0;
}

// simenv.hpp:155-184
int sf_step_world(sf_world* w, sf_point* verts, sf_point* vel, double dt) {
    if (!w) return fail(SF_INVALID_ARGUMENT, "world is null");
    if (!(dt > 0.0)) return fail(SF_INVALID_ARGUMENT, "step_world: dt must be positive");
    auto move = [&](sf_point& p, sf_point& v) {
        p.x += v.x * dt;
        p.y += v.y * dt;
        p.x += reflect_axis(p.x, p.x, w->width, v.x);
        p.y += reflect_axis(p.y, p.y, w->height, v.y);
    };
    move(w->start, w->start_velocity);
    move(w->target, w->target_velocity);
    for (uint32_t o = 0; o < w->n_obstacles; ++o) {
        sf_point& ov = vel[o];
        if (ov.x == 0.0 && ov.y == 0.0) continue;
        const uint32_t v0 = w->vertex_offsets[o], v1 = w->vertex_offsets[o + 1];
        for (uint32_t i = v0; i < v1; ++i) {
            verts[i].x += ov.x * dt;
            verts[i].y += ov.y * dt;
        }
        double bx0 = verts[v0].x, by0 = verts[v0].y, bx1 = bx0, by1 = by0;
        for (uint32_t i = v0; i < v1; ++i) {
            bx0 = std::min(bx0, verts[i].x); by0 = std::min(by0, verts[i].y);
            bx1 = std::max(bx1, verts[i].x); by1 = std::max(by1, verts[i].y);
        }
        const double sx = reflect_axis(bx0, bx1, w->width, ov.x);
        const double sy = reflect_axis(by0, by1, w->height, ov.y);
        if (sx != 0.0 || sy != 0.0)
            for (uint32_t i = v0; i < v1; ++i) { verts[i].x += sx; verts[i].y += sy; }
    }
    return SF_OK;
}

// simenv.hpp:239-276 with variant wiring (188-234)
int sf_run_scenario(sf_ctx* ctx, const sf_scenario_config* c, int variant, uint32_t frames,
                    const sf_planner_config* base, const double* evolved, uint32_t evolved_groups,
                    sf_plan_record* records, double* best) {
    if (!ctx || !c || !base || !records || !evolved) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (frames < 1) return fail(SF_INVALID_ARGUMENT, "run_scenario: frame count must be >= 1");
    if (variant < 0 || variant > 5) return fail(SF_INVALID_ARGUMENT, "unknown planner variant");
    sf_planner_config cfg = *base;
    std::vector<double> hyp;
    static const double defaults[48] = {2, 1, 1, 0.4, 0.2, 0.2, 1, 1, 2, 0.7, 0.3, 0.1,
                                        2, 2, 1, 0.8, 0.1, 0.6, 2, 2, 1, 0.8, 0.6, 0.4,
                                        2, 1, 2, 0.2, 0.1, 0.3, 2, 1, 2, 0.9, 0.5, 0.5,
                                        1, 2, 2, 0.4, 0.1, 0.8, 1, 2, 2, 0.9, 0.3, 0.3};
    switch (variant) {
    case 0: hyp.assign(evolved, evolved + 6 * size_t(evolved_groups)); break;      // sepso
    case 1: cfg.auto_truncate = 0; cfg.max_iters_per_frame = 30;
            hyp.assign(evolved, evolved + 6 * size_t(evolved_groups)); break;      // sepso-noat
    case 2: cfg.gamma = 0.0; hyp.assign(evolved, evolved + 6 * size_t(evolved_groups)); break; // sepso-nopi
    case 3: case 4:                                                                // dtpso / dppso
        cfg.gamma = 0.0; cfg.auto_truncate = 0; cfg.max_iters_per_frame = 30;
        hyp.assign(defaults, defaults + 48);
        break;
    case 5:                                                                        // pso
        cfg.gamma = 0.0; cfg.auto_truncate = 0; cfg.max_iters_per_frame = 30;
        cfg.per_group = base->groups * base->per_group;
        cfg.groups = 1;
        hyp = {2.0, 2.0, 0.0, 0.9, 0.4, 0.5};
        break;
    }
    // priori_init's checks (planner.hpp:80-84) before any frame runs
    int vs = validate_planner(&cfg);
    if (vs) return vs;
    if (hyp.size() != 6 * size_t(cfg.groups))
        return fail(SF_INVALID_ARGUMENT, "priori_init: hyper matrix group count != G");
    if ((vs = validate_hypers(hyp.data(), cfg.groups))) return vs;
    sf_scenario_config sc = *c;
    sc.frames = std::max<uint32_t>(sc.frames, 1);
    const uint32_t n = c->dynamic_obstacles + c->static_obstacles;
    std::vector<uint32_t> off(n + 1);
    std::vector<sf_point> verts(4 * size_t(n)), vel(n);
    sf_world w{};
    int st = sf_generate_world(&sc, derive_seed(c->root_seed, "world"), ctx->rng, &w, off.data(), verts.data(),
                               vel.data());
    if (st) return st;
    std::vector<double> prev(cfg.dim), win(std::max<uint32_t>(cfg.tw, 1) + 1);
    uint32_t wl = 0;
    bool have_prev = false;
    if (ctx->l2_flush) {
        const cudaError_t fe = ctx->flush.ensure(ctx->l2_flush);
        if (fe != cudaSuccess) return cuda_fail(fe, "l2 flush buffer");
    }
    for (uint32_t f = 0; f < frames; ++f) {
        if (ctx->l2_flush) {
            cudaMemsetAsync(ctx->flush.p, int(f & 0xff), ctx->l2_flush, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
        }
        std::vector<double> bp(cfg.dim);
        // the next frame's seed: its init walk runs while this frame plans
        ctx->hint_valid = f + 1 < frames;
        ctx->hint_seed = derive_seed(c->root_seed, "plan", f + 1);
        st = sf_plan_frame(ctx, &w, have_prev ? prev.data() : nullptr, hyp.data(), &cfg,
                           derive_seed(c->root_seed, "plan", f), win.data(), &wl, uint32_t(win.size()),
                           &records[f], bp.data(), nullptr);
        ctx->hint_valid = false;
        if (st) return st;
        prev = bp;
        have_prev = true;
        if (best) std::copy(bp.begin(), bp.end(), best + size_t(f) * cfg.dim);
        if ((st = sf_step_world(&w, verts.data(), vel.data(), c->dt))) return st;
    }
    return SF_OK;
}

uint64_t sf_derive_seed(uint64_t root, const char* tag, size_t tag_len, int has_index, uint64_t index) {
    const uint64_t d = splitmix64(root ^ fnv1a64(tag ? tag : "", tag ? tag_len : 0));   // rng.hpp:52-54
    return has_index ? splitmix64(d + index) : d;                                       // rng.hpp:56-59
}

int sf_comm_unique_id(uint8_t id[128]) {
    if (!id) return fail(SF_INVALID_ARGUMENT, "id is null");
    return comm_unique_id(id);
}

int sf_ctx_init_comm(sf_ctx* ctx, const uint8_t id[128], int nranks, int rank) {
    if (!ctx || !id) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SF_INVALID_ARGUMENT, "bad rank / world size");
    if (nranks > 64) return fail(SF_INVALID_ARGUMENT, "sharded swarm: at most 64 ranks");   // k_finish candidate table
    DeviceGuard guard(ctx->device);
    if (ctx->comm) comm_destroy(ctx->comm);
    ctx->comm = nullptr;
    const int st = comm_init(&ctx->comm, id, nranks, rank);
    if (st) return st;
    ctx->rank = rank;
    ctx->nranks = nranks;
    return SF_OK;
}

int sf_ctx_set_exchange(sf_ctx* ctx, int nranks, int rank, sf_allgather_fn fn, void* user) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SF_INVALID_ARGUMENT, "bad rank / world size");
    if (nranks > 64) return fail(SF_INVALID_ARGUMENT, "sharded swarm: at most 64 ranks");
    if (nranks > 1 && !fn) return fail(SF_INVALID_ARGUMENT, "an exchange callback is required for nranks > 1");
    if (ctx->comm) return fail(SF_INVALID_ARGUMENT, "the context already has an NCCL communicator");
    ctx->xfn = nranks > 1 ? fn : nullptr;
    ctx->xuser = nranks > 1 ? user : nullptr;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return SF_OK;
}

int sf_plan_frame_sharded(sf_ctx* ctx, const sf_world* world, const double* prev, const double* hypers,
                          const sf_planner_config* cfg, uint64_t seed, double* window, uint32_t* window_len,
                          uint32_t window_cap, sf_plan_record* record, double* best, uint64_t* bad) {
    const double t0 = now_seconds();
    if (!ctx || !record) return fail(SF_INVALID_ARGUMENT, "ctx/record is null");
    DeviceGuard guard(ctx->device);
    int st = validate_planner(cfg);
    if (st) return st;
    if ((st = validate_world(world))) return st;
    if (!hypers) return fail(SF_INVALID_ARGUMENT, "hypers is null");
    if ((st = validate_hypers(hypers, cfg->groups))) return st;
    if (int(cfg->groups) < ctx->nranks) return fail(SF_INVALID_ARGUMENT, "sharded swarm: fewer groups than ranks");
    const bool carry = cfg->window_carryover && window && window_len;
    StagedRun sr;
    sr.problem = kPath;
    sr.G = int(cfg->groups); sr.N = int(cfg->per_group); sr.D = int(cfg->dim); sr.cap = int(cfg->max_iters_per_frame);
    sr.world = world;
    sr.alpha = cfg->alpha; sr.beta = cfg->beta;
    sr.hypers = hypers;
    sr.seed = seed;
    sr.prev = prev;
    sr.warm = prev ? int(cfg->gamma * double(cfg->per_group)) : 0;
    sr.pi_radius = cfg->pi_radius;
    sr.auto_truncate = cfg->auto_truncate;
    sr.tw = int(cfg->tw);
    sr.delta = cfg->delta;
    std::vector<double> wtail;
    if (carry) {
        const uint32_t keep = std::min(*window_len, cfg->tw);
        wtail.assign(window + (*window_len - keep), window + *window_len);
        sr.win_in = wtail.data();
        sr.win_len_in = int(keep);
    }
    sr.rank = ctx->rank;
    sr.nranks = ctx->nranks;
    sr.comm = ctx->comm;
    if ((st = run_staged(ctx, sr))) return st;
    if (sr.out.status == 2) {
        if (bad) { bad[0] = sr.out.bad_g; bad[1] = sr.out.bad_n; bad[2] = sr.out.bad_k; }
        return fail(SF_NON_FINITE, nonfinite_msg(sr.out.bad_g, sr.out.bad_n, sr.out.bad_k));
    }
    if (carry && (st = carry_window(window, window_len, window_cap, cfg->tw, sr.trace.data(), sr.out.iterations)))
        return st;
    if (best) std::copy(sr.best.begin(), sr.best.end(), best);
    fill_record(sr.out, now_seconds() - t0, record);
    return SF_OK;
}

int sf_ctx_set_l2_flush(sf_ctx* ctx, uint64_t bytes) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    ctx->l2_flush = bytes;
    return SF_OK;
}

int sf_ctx_last_io_bytes(sf_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
    if (!ctx) return fail(SF_INVALID_ARGUMENT, "ctx is null");
    if (h2d) *h2d = ctx->last_h2d;
    if (d2h) *d2h = ctx->last_d2h;
    return SF_OK;
}

}  // extern "C"

// ------------------------------------------------------ device-resident scenes
struct sf_scene_batch {
    sf_ctx* ctx = nullptr;
    uint32_t n = 0, max_frames = 0, frames_done = 0;
    sf_planner_config cfg{};
    double dt = 1.0;
    WorldLayout lay{};
    FusedPlan fp;
    DevBuf worlds, hyp, roots, ones, win_vals, win_len, out, best, trace;
    DevBuf mtst[2];          // seeded mt19937 states: frame f reads [f & 1], leaves frame f + 1's in the other
    bool staged = false;
    // few scenes (spare SMs): frame f + 1's init walks run while frame f plans
    // (slot (f + 1) & 1, PreWalk::seed = the frame index); replaces mtst
    PreWalk* pre = nullptr;
    uint64_t root0 = 0;      // scene 0's root seed (one-scene walks seed on the host)
};

extern "C" {

int sf_scene_batch_create(sf_ctx* ctx, uint32_t n, const sf_scenario_config* cfgs,
                          const sf_planner_config* cfg, const double* hypers, uint32_t max_frames,
                          sf_scene_batch** out) {
    if (!ctx || !cfgs || !out || n == 0 || max_frames == 0) return fail(SF_INVALID_ARGUMENT, "bad scene batch arguments");
    for (uint32_t s = 1; s < n; ++s)      // one dt steps every world record of the batch
        if (cfgs[s].dt != cfgs[0].dt) return fail(SF_INVALID_ARGUMENT, "scene batch: every scenario must share dt");
    DeviceGuard guard(ctx->device);
    int st = validate_planner(cfg);
    if (st) return st;
    if ((st = validate_hypers(hypers, cfg->groups))) return st;
    // worlds on the host (scene state is host-owned until it is staged)
    std::vector<std::vector<uint32_t>> off(n);
    std::vector<std::vector<sf_point>> verts(n), vel(n);
    std::vector<sf_world> ws(n);
    for (uint32_t s = 0; s < n; ++s) {
        const uint32_t k = cfgs[s].dynamic_obstacles + cfgs[s].static_obstacles;
        off[s].resize(k + 1);
        verts[s].resize(4 * size_t(k) + 1);
        vel[s].resize(size_t(k) + 1);
        if ((st = sf_generate_world(&cfgs[s], derive_seed(cfgs[s].root_seed, "world"), ctx->rng, &ws[s],
                                    off[s].data(), verts[s].data(), vel[s].data())))
            return st;
    }
    WorldPack wp;
    pack_worlds(ws.data(), n, wp);
    auto* b = new sf_scene_batch();
    b->ctx = ctx;
    b->n = n;
    b->max_frames = max_frames;
    b->cfg = *cfg;
    b->dt = cfgs[0].dt;
    b->lay = wp.lay;
    const uint32_t D = cfg->dim, tw = cfg->tw, cap = cfg->max_iters_per_frame;
    b->fp = plan_fused(ctx, kPath, int(n), int(cfg->groups), int(cfg->per_group), int(D), wp.lay.max_obs,
                       wp.lay.max_verts, int(cap), int(tw));
    if (!b->fp.fits) {
        delete b;
        return fail(SF_UNSUPPORTED, "scene batch: swarm does not fit a cluster");
    }
    cudaError_t e = cudaSuccess;
    auto alloc = [&](DevBuf& buf, size_t bytes) { if (e == cudaSuccess) e = buf.ensure(bytes); };
    alloc(b->worlds, wp.bytes.size());
    alloc(b->hyp, size_t(cfg->groups) * 48);
    alloc(b->roots, size_t(n) * 8);
    alloc(b->ones, size_t(n));
    alloc(b->win_vals, size_t(n) * tw * 8);
    alloc(b->win_len, size_t(n) * 4);
    alloc(b->out, size_t(max_frames) * n * sizeof(SwarmOut));
    alloc(b->best, size_t(max_frames) * n * D * 8);
    alloc(b->trace, size_t(n) * cap * 8);
    // few scenes leave most SMs idle: there the next frame's init walks run
    // ahead (one CTA per scene) while a frame plans
    const long long nwords = 2ll * cfg->groups * cfg->per_group * D;
    const bool few = n * uint32_t(b->fp.p.C) <= 64 && n <= 8;
    // many scenes (config 5) fill every SM: their walks run as one bulk
    // launch (several walker CTAs per SM) ordered before the frame by an event,
    // in the previous frame's tail instead of inside every cluster
    static const bool bulk_on = [] {
        const char* e = std::getenv("SEPSO_PREWALK_BULK");
        return !(e && e[0] == '0');
    }();
    const bool ahead = ctx->rng == SF_RNG_MT19937 && prewalk_enabled() && (few || bulk_on);
    if (ctx->rng == SF_RNG_MT19937 && !ahead) {
        alloc(b->mtst[0], size_t(n) * 312 * 8);
        alloc(b->mtst[1], size_t(n) * 312 * 8);
    }
    if (e != cudaSuccess) {
        delete b;
        return cuda_fail(e, "scene batch allocation");
    }
    if (ahead && (st = prewalk_setup(b->pre, int(n), nwords)) != SF_OK) {
        prewalk_destroy(b->pre);
        delete b;
        return st;
    }
    if (ahead && !few) {
        b->pre->bulk = true;
        for (cudaEvent_t& ev : b->pre->done)
            if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
                prewalk_destroy(b->pre);
                delete b;
                return cuda_fail(cudaErrorMemoryAllocation, "init walk events");
            }
    }
    std::vector<uint64_t> roots(n);
    for (uint32_t s = 0; s < n; ++s) roots[s] = cfgs[s].root_seed;
    b->root0 = roots[0];
    std::vector<uint8_t> ones(n, 1);
    cudaMemcpyAsync(b->worlds.p, wp.bytes.data(), wp.bytes.size(), cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(b->hyp.p, hypers, size_t(cfg->groups) * 48, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(b->roots.p, roots.data(), size_t(n) * 8, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(b->ones.p, ones.data(), size_t(n), cudaMemcpyHostToDevice, ctx->stream);
    cudaMemsetAsync(b->win_len.p, 0, size_t(n) * 4, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        delete b;
        return cuda_fail(e, "scene batch upload");
    }
    SwarmParams& p = b->fp.p;
    p.alpha = cfg->alpha;
    p.beta = cfg->beta;
    p.beta_int = beta_integer(cfg->beta);
    p.at_gap = cfg->delta * std::sqrt(2.0 * double(cfg->tw)) * (1.0 + 1e-9);
    p.delta = cfg->delta;
    p.pi_radius = cfg->pi_radius;
    p.warm = int(cfg->gamma * double(cfg->per_group));
    p.auto_truncate = cfg->auto_truncate;
    p.carry = cfg->window_carryover;
    p.hypers = static_cast<const double*>(b->hyp.p);
    p.hypers_stride = 0;
    p.seeds = nullptr;
    p.roots = static_cast<const unsigned long long*>(b->roots.p);
    p.tag_hash = fnv1a64("plan", 4);
    p.worlds = static_cast<const unsigned char*>(b->worlds.p);
    p.world_stride = (long long)wp.lay.stride;
    p.off_offsets = int(wp.lay.off_offsets);
    p.off_verts = int(wp.lay.off_verts);
    p.lo = nullptr;
    p.hi = nullptr;
    p.win_vals = static_cast<double*>(b->win_vals.p);
    p.win_len = static_cast<int*>(b->win_len.p);
    p.trace = static_cast<double*>(b->trace.p);
    *out = b;
    return SF_OK;
}

int sf_scene_batch_run(sf_scene_batch* b, uint32_t frames) {
    if (!b) return fail(SF_INVALID_ARGUMENT, "batch is null");
    if (b->frames_done + frames > b->max_frames) return fail(SF_INVALID_ARGUMENT, "scene batch: max_frames exceeded");
    sf_ctx* ctx = b->ctx;
    DeviceGuard guard(ctx->device);
    SwarmParams& p = b->fp.p;
    const size_t D = b->cfg.dim;
    for (uint32_t i = 0; i < frames; ++i) {
        const uint32_t f = b->frames_done + i;
        p.frame_index = int(f);
        p.prev = f == 0 ? nullptr : static_cast<const double*>(b->best.p) + size_t(f - 1) * b->n * D;
        p.has_prev = f == 0 ? nullptr : static_cast<const unsigned char*>(b->ones.p);
        p.best_x = static_cast<double*>(b->best.p) + size_t(f) * b->n * D;
        p.out = static_cast<SwarmOut*>(b->out.p) + size_t(f) * b->n;
        p.off_vel = int(b->lay.off_vel);
        p.step_dt = b->dt;                       // the world step rides on the planning launch
        const bool mtp = b->mtst[0].p != nullptr;
        p.mt_pre = (mtp && f > 0) ? static_cast<const unsigned long long*>(b->mtst[f & 1].p) : nullptr;
        p.mt_next = mtp ? static_cast<unsigned long long*>(b->mtst[(f + 1) & 1].p) : nullptr;
        PreWalk* W = b->pre;
        const long long nwords = 2ll * b->cfg.groups * b->cfg.per_group * b->cfg.dim;
        p.pre_words = nullptr;
        if (W) {
            const int k = int(f & 1);
            if (W->nwords[k] == nwords && W->seed[k] == f) {      // frame f's walk, started during frame f - 1
                p.pre_words = static_cast<const unsigned long long*>(W->words[k].p);
                p.pre_pair = static_cast<const unsigned long long*>(W->pairs[k].p);
                p.pre_flag = static_cast<const int*>(W->flags.p) + k * W->n;
                p.pre_seq = W->seq[k];
                W->nwords[k] = 0;
                if (W->bulk) cudaStreamWaitEvent(ctx->stream, W->done[k], 0);   // no spinning clusters
            }
            // frame f - 1 (the last reader of slot (f + 1) & 1) is done once
            // this point of the planning stream is reached
            cudaEventRecord(W->ev, ctx->stream);
        }
        int st = launch_fused(ctx, b->fp, kPath);
        if (st) return st;
        if (W && f + 1 < b->max_frames) {
            const int k = int((f + 1) & 1);
            if (++W->next_seq <= 0) W->next_seq = 1;
            W->seq[k] = W->next_seq;
            cudaStreamWaitEvent(W->st, W->ev, 0);
            uint64_t st0[312];          // one scene: its seeded state from the host (derive_seed, simenv.hpp:256)
            if (b->n == 1) mt_seeded_state(splitmix64(splitmix64(b->root0 ^ p.tag_hash) + uint64_t(f + 1)), st0);
            const int e = prewalk_late() ? 0 : launch_init_walk(int(b->n), nullptr, p.roots, p.tag_hash, int(f + 1), 0, nwords,
                                           static_cast<unsigned long long*>(W->words[k].p),
                                           static_cast<unsigned long long*>(W->pairs[k].p),
                                           static_cast<int*>(W->flags.p) + k * W->n, W->seq[k],
                                           b->n == 1 ? reinterpret_cast<const unsigned long long*>(st0) : nullptr,
                                           W->st);
            if (e != 0) return cuda_fail(cudaError_t(e), "init walk launch");
            if (W->bulk) cudaEventRecord(W->done[k], W->st);
            W->seed[k] = f + 1;
            W->nwords[k] = nwords;
        }
    }
    b->frames_done += frames;
    return SF_OK;
}

int sf_scene_batch_records(sf_scene_batch* b, uint32_t first, uint32_t count, sf_plan_record* records,
                           double* best) {
    if (!b || !records) return fail(SF_INVALID_ARGUMENT, "null argument");
    if (first + count > b->frames_done) return fail(SF_INVALID_ARGUMENT, "frames not run yet");
    sf_ctx* ctx = b->ctx;
    DeviceGuard guard(ctx->device);
    const size_t m = size_t(count) * b->n, D = b->cfg.dim;
    std::vector<SwarmOut> outs(m);
    cudaMemcpyAsync(outs.data(), static_cast<SwarmOut*>(b->out.p) + size_t(first) * b->n, m * sizeof(SwarmOut),
                    cudaMemcpyDeviceToHost, ctx->stream);
    if (best)
        cudaMemcpyAsync(best, static_cast<double*>(b->best.p) + size_t(first) * b->n * D, m * D * 8,
                        cudaMemcpyDeviceToHost, ctx->stream);
    const cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "scene batch records");
    for (size_t i = 0; i < m; ++i) fill_record(outs[i], 0.0, &records[i]);
    for (size_t i = 0; i < m; ++i)
        if (outs[i].status == 2)
            return fail(SF_NON_FINITE, nonfinite_msg(outs[i].bad_g, outs[i].bad_n, outs[i].bad_k));
    return SF_OK;
}

int sf_scene_batch_destroy(sf_scene_batch* b) {
    if (!b) return SF_OK;
    cudaSetDevice(b->ctx->device);
    cudaStreamSynchronize(b->ctx->stream);
    prewalk_destroy(b->pre);
    for (DevBuf* d : {&b->worlds, &b->hyp, &b->roots, &b->ones, &b->win_vals, &b->win_len, &b->out, &b->best,
                      &b->trace, &b->mtst[0], &b->mtst[1]})
        d->release();
    delete b;
    return SF_OK;
}

}  // extern "C"
