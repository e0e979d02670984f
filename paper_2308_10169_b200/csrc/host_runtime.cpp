// host_runtime.cpp -- context plumbing, validation, launch planning, the
// staged (HBM-resident) swarm driver and the host half of HSEF.
#include "host_runtime.hpp"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>

#include "mt_jump.hpp"
#include "stage_kernels.cuh"

namespace sepso {

static thread_local std::string g_error;

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    return fail(SF_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}
const char* last_error_cstr() { return g_error.c_str(); }

cudaError_t DevBuf::ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    const size_t want = std::max<size_t>(bytes, 1 << 16);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) n = want;
    return e;
}
void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
}
cudaError_t PinnedBuf::ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    const size_t want = std::max<size_t>(bytes, 1 << 16);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) n = want;
    return e;
}
void PinnedBuf::release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
}

// --------------------------------------------------------------- validation
int validate_hypers(const double* h, uint32_t G) {
    if (G == 0) return fail(SF_INVALID_ARGUMENT, "HyperMatrix: at least one group required");
    for (uint32_t g = 0; g < G; ++g) {
        const double* r = h + 6 * g;
        for (int f = 0; f < 6; ++f)
            if (!std::isfinite(r[f])) return fail(SF_INVALID_ARGUMENT, "HyperMatrix: non-finite entry");
        if (r[0] < 0 || r[1] < 0 || r[2] < 0)
            return fail(SF_INVALID_ARGUMENT, "HyperMatrix: acceleration constants must be >= 0");
        if (!(0.0 <= r[4] && r[4] <= r[3] && r[3] <= 1.0))
            return fail(SF_INVALID_ARGUMENT, "HyperMatrix: need 0 <= omega_end <= omega_init <= 1");
        if (!(0.0 < r[5] && r[5] <= 1.0))
            return fail(SF_INVALID_ARGUMENT, "HyperMatrix: need 0 < v_limit <= 1");
    }
    return SF_OK;
}

int validate_bounds(const double* lo, const double* hi, uint32_t D) {
    if (D == 0) return fail(SF_INVALID_ARGUMENT, "SearchBounds: dimension must be >= 1");
    for (uint32_t d = 0; d < D; ++d) {
        if (!std::isfinite(lo[d]) || !std::isfinite(hi[d]))
            return fail(SF_INVALID_ARGUMENT, "SearchBounds: non-finite bound");
        if (!(lo[d] < hi[d])) return fail(SF_INVALID_ARGUMENT, "SearchBounds: need x_lo < x_hi per dimension");
    }
    return SF_OK;
}

int validate_world(const sf_world* w) {
    if (!w) return fail(SF_INVALID_ARGUMENT, "world is null");
    if (!(w->width > 0.0) || !(w->height > 0.0))
        return fail(SF_INVALID_ARGUMENT, "world dimensions must be positive");
    auto inside = [&](const sf_point& p) {
        return p.x >= 0.0 && p.x <= w->width && p.y >= 0.0 && p.y <= w->height;
    };
    if (!inside(w->start) || !inside(w->target))
        return fail(SF_INVALID_ARGUMENT, "start/target outside the map");
    if (w->n_obstacles && (!w->vertex_offsets || !w->vertices))
        return fail(SF_INVALID_ARGUMENT, "world obstacle arrays are null");
    for (uint32_t o = 0; o < w->n_obstacles; ++o) {
        const uint32_t v0 = w->vertex_offsets[o], v1 = w->vertex_offsets[o + 1];
        if (v1 < v0 + 3) return fail(SF_INVALID_ARGUMENT, "obstacle needs at least 3 vertices");
        for (uint32_t i = v0; i < v1; ++i) {
            const sf_point& p = w->vertices[i];
            if (!std::isfinite(p.x) || !std::isfinite(p.y))
                return fail(SF_INVALID_ARGUMENT, "obstacle vertex is not finite");
        }
        for (uint32_t i = v0; i < v1; ++i)
            if (!inside(w->vertices[i])) return fail(SF_INVALID_ARGUMENT, "obstacle vertex outside the map");
    }
    return SF_OK;
}

int validate_planner(const sf_planner_config* c) {
    if (!c) return fail(SF_INVALID_ARGUMENT, "planner config is null");
    if (!(c->alpha >= 0.0) || !(c->beta >= 1.0))
        return fail(SF_INVALID_ARGUMENT, "planner config: need alpha >= 0 and beta >= 1");
    if (!(c->gamma >= 0.0 && c->gamma <= 1.0))
        return fail(SF_INVALID_ARGUMENT, "planner config: gamma must lie in [0, 1]");
    if (c->tw < 2) return fail(SF_INVALID_ARGUMENT, "planner config: tw must be >= 2");
    if (!(c->delta > 0.0)) return fail(SF_INVALID_ARGUMENT, "planner config: delta must be > 0");
    if (!(c->pi_radius > 0.0)) return fail(SF_INVALID_ARGUMENT, "planner config: pi_radius must be > 0");
    if (c->max_iters_per_frame < 1)
        return fail(SF_INVALID_ARGUMENT, "planner config: max_iters_per_frame must be >= 1");
    if (c->groups < 1 || c->per_group < 1)
        return fail(SF_INVALID_ARGUMENT, "planner config: G and N must be >= 1");
    if (c->dim < 2 || c->dim % 2 != 0)
        return fail(SF_INVALID_ARGUMENT, "planner config: dim must be even and >= 2");
    return SF_OK;
}

// ------------------------------------------------------------ world records
void pack_world_into(const sf_world& w, const WorldLayout& lay, unsigned char* dst) {
    std::memset(dst, 0, lay.stride);
    WorldHeader h{};
    h.width = w.width;
    h.height = w.height;
    h.sx = w.start.x;
    h.sy = w.start.y;
    h.tx = w.target.x;
    h.ty = w.target.y;
    h.n_obs = w.n_obstacles;
    h.n_verts = w.n_obstacles ? w.vertex_offsets[w.n_obstacles] - w.vertex_offsets[0] : 0;
    h.svx = w.start_velocity.x;
    h.svy = w.start_velocity.y;
    h.tvx = w.target_velocity.x;
    h.tvy = w.target_velocity.y;
    std::memcpy(dst, &h, sizeof(h));
    uint32_t* off = reinterpret_cast<uint32_t*>(dst + lay.off_offsets);
    double* vv = reinterpret_cast<double*>(dst + lay.off_verts);
    double* vel = reinterpret_cast<double*>(dst + lay.off_vel);
    const uint32_t base = w.n_obstacles ? w.vertex_offsets[0] : 0;
    for (uint32_t o = 0; o <= w.n_obstacles; ++o) off[o] = w.n_obstacles ? w.vertex_offsets[o] - base : 0;
    for (uint32_t i = 0; i < h.n_verts; ++i) {
        vv[2 * i] = w.vertices[base + i].x;
        vv[2 * i + 1] = w.vertices[base + i].y;
    }
    for (uint32_t o = 0; o < w.n_obstacles; ++o) {
        vel[2 * o] = w.velocities ? w.velocities[o].x : 0.0;
        vel[2 * o + 1] = w.velocities ? w.velocities[o].y : 0.0;
    }
}

void pack_worlds(const sf_world* worlds, uint32_t n, WorldPack& out) {
    int max_obs = 1, max_verts = 3;
    for (uint32_t s = 0; s < n; ++s) {
        const sf_world& w = worlds[s];
        max_obs = std::max<int>(max_obs, int(w.n_obstacles));
        const uint32_t nv = w.n_obstacles ? w.vertex_offsets[w.n_obstacles] - w.vertex_offsets[0] : 0;
        max_verts = std::max<int>(max_verts, int(nv));
    }
    out.lay = world_layout(max_obs, max_verts);
    out.bytes.assign(size_t(n) * out.lay.stride, 0);
    for (uint32_t s = 0; s < n; ++s) pack_world_into(worlds[s], out.lay, out.bytes.data() + size_t(s) * out.lay.stride);
}

bool force_staged() {
    static const bool on = [] {
        const char* e = std::getenv("SEPSO_FORCE_STAGED");
        return e && e[0] == '1';
    }();
    return on;
}

static int env_int(const char* name, int def) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : def;
}

// ------------------------------------------------------------ fused planning
FusedPlan plan_fused(sf_ctx* ctx, int problem, int n_swarms, int G, int N, int D, int max_obs,
                     int max_verts, int cap, int tw) {
    FusedPlan fp;
    SwarmParams& p = fp.p;
    const bool path = problem == kPath;
    const bool fp64 = ctx->precision == SF_FP64;
    const int R = G * N, S = D / 2 + 1;
    const int smem_max = max_smem_per_block();
    p.n_swarms = n_swarms;
    p.G = G;
    p.N = N;
    p.D = D;
    p.cap = cap;
    p.tw = tw;
    p.max_obs = path ? std::max(max_obs, 1) : 0;
    p.max_verts = path ? std::max(max_verts, 3) : 0;
    static const int env_c = env_int("SEPSO_CLUSTER", 0), env_t = env_int("SEPSO_THREADS", 0);
    static const int env_no_ring = env_int("SEPSO_NO_RING", 0);
    const int want_c = ctx->force_cluster ? ctx->force_cluster : env_c;
    const int want_t = ctx->force_threads ? ctx->force_threads : env_t;
    // Launch shapes (measured, tools/sweep*.py):
    //  latency (few swarms): one swarm over up to 16 SMs, ~85 rows per CTA;
    //  medium (up to one swarm per SM, e.g. HSEF's 80 inner swarms): ~340 rows per
    //    CTA, 512 threads, two CTAs per SM;
    //  throughput (many swarms, config 5): ~680 rows per CTA, 1024 threads.
    const bool latency = n_swarms * 16 <= 2 * 148;
    const bool medium = !latency && n_swarms <= 148;
    const int rows_target = latency ? 85 : (medium ? 340 : 680);
    int C = want_c > 0 ? want_c : std::max(1, std::min(16, (R + rows_target - 1) / rows_target));
    for (;; C *= 2) {
        if (C > 16) C = 16;
        const int Rc = (R + C - 1) / C;
        p.C = C;
        p.rows_per_cta = Rc;
        int lgm = 1;
        for (int c = 0; c < C; ++c) {
            const int r0 = c * Rc, r1 = std::min(R, r0 + Rc);
            if (r1 > r0) lgm = std::max(lgm, (r1 - 1) / N - r0 / N + 1);
        }
        p.max_local_groups = lgm;
        if (path) {
            // worst case Rc*S*O entries; beyond the capacity entries are evaluated in place
            // throughput launches: per-warp rings of 64 compacted (item, obstacle)
            // pairs in A1 (latency launches keep one item per thread in place)
            p.entry_cap = (!latency && env_no_ring == 0) ? 1024 / 32 * 64 : 0;
            // one thread per (particle, segment) item; latency launches add four
            // warps (containment tasks, the stream generator) -- measured best
            p.nthreads = std::min(medium ? 512 : 1024, std::max(128, ((Rc * S) + 31) / 32 * 32 + (latency ? 128 : 0)));
        } else {
            p.entry_cap = 0;
            // benchmarks: a thread per row for the fitness, at least 256 for the
            // step's Rc*D elements (config 1, 80-row swarms: measured best)
            p.nthreads = std::min(512, std::max(256, (Rc + 31) / 32 * 32));
        }
        if (want_t > 0) p.nthreads = std::min(1024, std::max(32, want_t / 32 * 32));
        p.rng = ctx->rng;
        fp.smem = smem_layout(p, fp64 ? 8 : 4, path).total;
        if (int(fp.smem) <= smem_max) { fp.fits = true; break; }
        if (C >= 16 || want_c > 0) break;
    }
    p.beta_int = 0;
    p.in_pre = -1;
    p.in_mtst = -1;
    return fp;
}

int launch_fused(sf_ctx* ctx, FusedPlan& fp, int problem) {
    if (ctx->timing) cudaEventRecord(ctx->ev0, ctx->stream);
    size_t smem = 0;
    static const bool phase_prof = std::getenv("SEPSO_PHASE_PROF") != nullptr;
    long long* prof = nullptr;
    if (phase_prof && fp.p.cap > 0) {
        const size_t nprof = size_t(kProfPhases) * (fp.p.cap + 1) + 2 * 16 * size_t(fp.p.cap);
        cudaMalloc(&prof, sizeof(long long) * nprof);
        cudaMemsetAsync(prof, 0, sizeof(long long) * nprof, ctx->stream);
        fp.p.prof = prof;
    }
#ifdef SEPSO_CHECK
    long long* dbg = nullptr;
    const size_t ndbg = size_t(fp.p.n_swarms) * fp.p.C * std::max(fp.p.cap, 1);
    cudaMalloc(&dbg, ndbg * 8);
    cudaMemsetAsync(dbg, 0xff, ndbg * 8, ctx->stream);
    fp.p.dbg = dbg;
#endif
    cudaEvent_t pe0 = nullptr, pe1 = nullptr;
    if (prof) {
        cudaEventCreate(&pe0);
        cudaEventCreate(&pe1);
        cudaEventRecord(pe0, ctx->stream);
    }
    const int e = launch_swarms(fp.p, fp.p.inl ? fp.payload : nullptr, problem, ctx->precision == SF_FP64,
                                ctx->stream, &smem);
    if (prof) cudaEventRecord(pe1, ctx->stream);
    if (prof) {
        std::vector<long long> h(size_t(kProfPhases) * (fp.p.cap + 1) + 2 * 16 * size_t(fp.p.cap));
        cudaMemcpyAsync(h.data(), prof, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(prof);
        fp.p.prof = nullptr;
        static const char* names[] = {"prelude", "mask+pairs", "cont", "A1sync+A3", "pbest", "part",
                                      "csync", "gath", "B1", "B2", "step"};
        double acc[11] = {0};
        int iters = 0;
        for (int k = 0; k < fp.p.cap; ++k) {
            const long long* r = h.data() + size_t(k) * kProfPhases;
            if (r[0] == 0) break;
            ++iters;
            const long long t[12] = {r[0], r[1], r[2], r[3], r[4], r[5], r[6], r[7], r[8], r[9], r[10], r[11]};
            for (int i = 0; i < 11; ++i) if (t[i + 1] > t[i]) acc[i] += double(t[i + 1] - t[i]);
        }
        std::fprintf(stderr, "[phase] C=%d T=%d iters=%d cycles/iter:", fp.p.C, fp.p.nthreads, iters);
        for (int i = 0; i < 11; ++i) std::fprintf(stderr, " %s=%.0f", names[i], iters ? acc[i] / iters : 0.0);
        double g0 = 0, g1 = 0, b1 = 0;
        int gi = 0;
        for (int k = 0; k < iters; ++k) {
            const long long* r = h.data() + size_t(k) * kProfPhases;
            if (r[12] == 0 || r[13] == 0) continue;
            ++gi;
            g0 += double(r[12] - r[8]); g1 += double(r[13] - r[12]); b1 += double(r[14] - r[8]);
        }
        if (gi) std::fprintf(stderr, " | B1work=%.0f gen_start=%.0f gen=%.0f", b1 / gi, g0 / gi, g1 / gi);
        {   // inside B1 (warp 0): bad-row reduce, gbest scan, tbest reduce, window push, AT
            double q[5] = {0};
            int qi = 0;
            for (int k = 0; k < iters; ++k) {
                const long long* r = h.data() + size_t(k) * kProfPhases;
                if (r[15] == 0 || r[16] == 0 || r[17] == 0 || r[18] == 0 || r[14] == 0) continue;
                ++qi;
                q[0] += double(r[15] - r[8]); q[1] += double(r[16] - r[15]); q[2] += double(r[17] - r[16]);
                q[3] += double(r[18] - r[17]); q[4] += double(r[14] - r[18]);
                if (std::getenv("SEPSO_ATTWICE") && r[20] > r[18])
                    std::fprintf(stderr, "[at] first=%lld second=%lld\n", r[20] - r[18], r[21] - r[20]);
            }
            if (qi) std::fprintf(stderr, " | B1: bad=%.0f gbest=%.0f tbest=%.0f push=%.0f at=%.0f", q[0] / qi,
                                 q[1] / qi, q[2] / qi, q[3] / qi, q[4] / qi);
            double pp[4] = {0};
            int pn = 0;
            for (int k = 0; k < iters; ++k) {
                const long long* r = h.data() + size_t(k) * kProfPhases;
                if (r[19] == 0 || r[20] == 0 || r[21] == 0 || r[5] == 0 || r[6] == 0) continue;
                ++pn;
                pp[0] += double(r[19] - r[5]); pp[1] += double(r[20] - r[19]); pp[2] += double(r[21] - r[20]);
                pp[3] += double(r[6] - r[21]);
            }
            if (pn) std::fprintf(stderr, " | part: reduce=%.0f push_part=%.0f push_rows=%.0f push_bad=%.0f", pp[0] / pn,
                                 pp[1] / pn, pp[2] / pn, pp[3] / pn);
            double e1 = 0, e2 = 0;
            int en = 0;
            for (int k = 0; k < iters; ++k) {
                const long long* r = h.data() + size_t(k) * kProfPhases;
                if (r[22] == 0 || r[23] == 0 || r[5] == 0) continue;
                ++en;
                e1 += double(r[22] - r[5]); e2 += double(r[23] - r[22]);
            }
            if (en) std::fprintf(stderr, " | expect=%.0f scan=%.0f", e1 / en, e2 / en);
            if (std::getenv("SEPSO_SCAN2")) {
                double a = 0, b = 0;
                int n2 = 0;
                for (int k = 0; k < iters; ++k) {
                    const long long* r = h.data() + size_t(k) * kProfPhases;
                    if (r[22] == 0 || r[23] == 0 || r[1] == 0) continue;
                    ++n2; a += double(r[23] - r[22]); b += double(r[1] - r[23]);
                }
                if (n2) std::fprintf(stderr, " | scan first=%.0f second=%.0f", a / n2, b / n2);
            }
        }
        {   // init marks (row cap): start, consts, seeded, x, v, rest, put, loop
            const long long* r = h.data() + size_t(fp.p.cap) * kProfPhases;
            std::fprintf(stderr, " | init: consts=%lld seed=%lld x=%lld v=%lld rest=%lld sync=%lld (seeded at %lld, staged at %lld)",
                         r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4], r[6] - r[5],
                         r[13] - r[0], r[14] - r[0]);
            std::fprintf(stderr, " (thread 0: hyp %lld world_regs %lld load_world %lld to misc %lld)",
                         r[15] - r[0], r[16] - r[15], r[17] - r[16], r[18] - r[17]);
            std::fprintf(stderr, " | ns: init=%lld loop=%lld out=%lld exit=%lld total=%lld",
                         r[8] - r[7], r[9] - r[8], r[10] - r[9], r[11] - r[10], r[11] - r[7]);
            float ev_ms = 0.f;
            cudaEventElapsedTime(&ev_ms, pe0, pe1);
            std::fprintf(stderr, " | entry->g7=%lld event=%.0f", r[7] - r[12], 1e6 * double(ev_ms));
            cudaEventDestroy(pe0);
            cudaEventDestroy(pe1);
            // per-CTA work before the partial exchange (cycles): spread over CTAs
            const long long* w = h.data() + size_t(kProfPhases) * (fp.p.cap + 1);
            double smin = 0, smax = 0, sown = 0;
            int nk = 0;
            for (int k = 0; k < iters; ++k) {
                long long mn = LLONG_MAX, mx = 0;
                for (int cc = 0; cc < std::min(16, fp.p.C); ++cc) {
                    const long long v = w[(size_t(k) * 16 + cc) * 2];
                    mn = std::min(mn, v); mx = std::max(mx, v);
                }
                smin += double(mn); smax += double(mx); sown += double(w[(size_t(k) * 16) * 2 + 1]); ++nk;
            }
            if (nk) std::fprintf(stderr, " | per-CTA fitness..push: min=%.0f max=%.0f cta0_wait=%.0f", smin / nk, smax / nk, sown / nk);
            if (nk) {
                std::fprintf(stderr, " | by CTA:");
                for (int cc = 0; cc < std::min(16, fp.p.C); ++cc) {
                    double s = 0;
                    for (int k = 0; k < iters; ++k) s += double(w[(size_t(k) * 16 + cc) * 2]);
                    std::fprintf(stderr, " %.0f", s / nk);
                }
            }
        }
        std::fprintf(stderr, "\n");
    }
#ifdef SEPSO_CHECK
    {   // every CTA of a cluster must have taken the same decision at every iteration it ran
        std::vector<long long> h(ndbg);
        cudaMemcpyAsync(h.data(), dbg, ndbg * 8, cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(dbg);
        fp.p.dbg = nullptr;
        const int C = fp.p.C, cap = std::max(fp.p.cap, 1);
        if (std::getenv("SEPSO_CHECK_SELFTEST") && ndbg > 1) h[1] ^= 1;   // the comparison must catch this
        for (int sw = 0; sw < fp.p.n_swarms; ++sw) {
            if (fp.p.cap > 0 && h[size_t(sw) * C * cap] == -1)
                return fail(SF_RUNTIME_ERROR, "consistency check: no decision logged");
            for (int k = 0; k < cap; ++k) {
                const long long r0 = h[(size_t(sw) * C) * cap + k];
                for (int cc = 1; cc < C; ++cc)
                    if (h[(size_t(sw) * C + cc) * cap + k] != r0)
                        return fail(SF_RUNTIME_ERROR, "consistency check: CTA decisions differ in swarm " +
                                                          std::to_string(sw) + " iteration " + std::to_string(k + 1));
            }
        }
    }
#endif
    if (e != 0) return cuda_fail(cudaError_t(e), "fused swarm launch");
    if (ctx->timing) {
        cudaEventRecord(ctx->ev1, ctx->stream);
        cudaEventSynchronize(ctx->ev1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        ctx->kernel_ms += ms;
        ctx->launches += 1;
    }
    return SF_OK;
}

// ---------------------------------------------------------- staged driver
int run_staged(sf_ctx* ctx, StagedRun& r) {
    const bool fp64 = ctx->precision == SF_FP64;
    const size_t tsz = fp64 ? 8 : 4;
    const int G = r.G, N = r.N, D = r.D, R = G * N;
    // this device's shard: whole groups [g0, g1) (rows [g0*N, g1*N))
    const int nranks = std::max(1, r.nranks);
    const int g0 = int((long long)r.rank * G / nranks), g1 = int((long long)(r.rank + 1) * G / nranks);
    const int RL = (g1 - g0) * N, row_begin = g0 * N;
    if (RL <= 0) return fail(SF_INVALID_ARGUMENT, "sharded swarm: more ranks than groups");
    const bool path = r.problem == kPath;
    cudaStream_t st = ctx->stream;
    // host-side staging of constants
    WorldPack wp;
    if (path) pack_worlds(r.world, 1, wp);
    std::vector<double> lo(D), hi(D);
    for (int d = 0; d < D; ++d) {
        if (path) {
            lo[d] = 0.0;
            hi[d] = d < D / 2 ? r.world->width : r.world->height;
        } else {
            lo[d] = r.lo[d];
            hi[d] = r.hi[d];
        }
    }
    // device arena
    size_t off = 0;
    auto take = [&](size_t b) { const size_t at = off; off = (off + b + 255) & ~size_t(255); return at; };
    const size_t o_world = take(path ? wp.bytes.size() : 0);
    const size_t o_hyp = take(size_t(G) * 6 * 8);
    const size_t o_lo = take(size_t(D) * tsz), o_hi = take(size_t(D) * tsz);
    const size_t o_prev = take(size_t(D) * 8);
    const size_t o_x = take(size_t(RL) * D * tsz), o_v = take(size_t(RL) * D * tsz);
    const size_t o_pb = take(size_t(RL) * D * tsz);
    const size_t o_fit = take(size_t(RL) * tsz), o_pbf = take(size_t(RL) * tsz);
    const size_t o_imp = take(size_t(RL));     // rows whose pbest_x copy the step performs
    const size_t o_q = take(size_t(RL) * 4), o_pbq = take(size_t(RL) * 4);
    const size_t o_pf = take(size_t(G) * tsz), o_prow = take(size_t(G) * 4), o_pq = take(size_t(G) * 4);
    const size_t o_gbx = take(size_t(G) * D * tsz), o_gbf = take(size_t(G) * tsz), o_gbq = take(size_t(G) * 4);
    const size_t o_tbx = take(size_t(D) * tsz);
    const size_t cstride = cand_bytes(fp64, D);
    const size_t o_cand = take(cstride * size_t(nranks));
    const size_t o_st = take(sizeof(IterState));
    const size_t o_win = take(size_t(std::max(r.tw, 1)) * 8);
    const size_t o_trace = take(size_t(r.cap) * 8);
    const bool mt = ctx->rng == SF_RNG_MT19937;
    const size_t o_mt = take(mt ? sizeof(MtPersist) : 0);
    // init window (2RD words); the steps' 3R draws reuse it as two alternating
    // windows, so it holds the larger of 2RD and 6R
    const size_t o_words = take(mt ? std::max(size_t(2) * R * D, size_t(6) * R) * 8 : 0);
    // long init windows are generated in parallel segments from jumped states
    const long long init_words = 2ll * R * D;
    int jlevels = 0;
    // (segments of >= 2^17 words; more than 64 only when each keeps >= 2^20:
    // level 7's 128 jumps cost ~230 us, and two segment walks on one SM run at
    // ~65 % each, so 256 segments of 2^20 words lose to 128 of 2^21)
    while (mt && jlevels < kMaxJumpLevels &&
           (init_words >> (jlevels + 1)) >= (jlevels < kWideJumpLevels ? (1ll << 17) : (1ll << 20)))
        ++jlevels;
    if (std::getenv("SEPSO_SEQ_FILL")) jlevels = 0;
    const bool jump = jlevels >= 2;
    const size_t o_jst = take(jump ? (size_t(1) << jlevels) * 312 * 8 : 0);
    const size_t o_jpoly = take(jump ? size_t(jlevels) * kMtDegree * 2 : 0);   // exponent lists (uint16)
    cudaError_t ce = ctx->scratch.ensure(off);
    if (ce != cudaSuccess) return cuda_fail(ce, "staged arena");
    unsigned char* dev = static_cast<unsigned char*>(ctx->scratch.p);
    // stage host bytes (pinned) for the small constants
    std::vector<unsigned char> h(o_x, 0);
    if (path) std::memcpy(h.data() + o_world, wp.bytes.data(), wp.bytes.size());
    std::memcpy(h.data() + o_hyp, r.hypers, size_t(G) * 6 * 8);
    for (int d = 0; d < D; ++d) {
        if (fp64) {
            reinterpret_cast<double*>(h.data() + o_lo)[d] = lo[d];
            reinterpret_cast<double*>(h.data() + o_hi)[d] = hi[d];
        } else {
            reinterpret_cast<float*>(h.data() + o_lo)[d] = float(lo[d]);
            reinterpret_cast<float*>(h.data() + o_hi)[d] = float(hi[d]);
        }
    }
    if (r.prev) std::memcpy(h.data() + o_prev, r.prev, size_t(D) * 8);
    ce = cudaMemcpyAsync(dev, h.data(), o_x, cudaMemcpyHostToDevice, st);
    if (ce != cudaSuccess) return cuda_fail(ce, "staged upload");
    // bests start at +inf (swarm.hpp:113-116)
    std::vector<unsigned char> inf_f(size_t(std::max(RL, G)) * tsz);
    for (int i = 0; i < std::max(RL, G); ++i) {
        if (fp64) reinterpret_cast<double*>(inf_f.data())[i] = std::numeric_limits<double>::infinity();
        else reinterpret_cast<float*>(inf_f.data())[i] = std::numeric_limits<float>::infinity();
    }
    cudaMemcpyAsync(dev + o_pbf, inf_f.data(), size_t(RL) * tsz, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(dev + o_gbf, inf_f.data(), size_t(G) * tsz, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(dev + o_pbq, 0, size_t(RL) * 4, st);
    cudaMemsetAsync(dev + o_gbq, 0, size_t(G) * 4, st);
    cudaMemsetAsync(dev + o_gbx, 0, size_t(G) * D * tsz, st);
    cudaMemsetAsync(dev + o_tbx, 0, size_t(D) * tsz, st);
    IterState is{};
    is.tbest_f = std::numeric_limits<double>::infinity();
    is.tbest_group = -1;
    is.nonfinite_row = INT_MAX;
    is.win_len = std::min(r.win_len_in, r.tw);
    is.win_head = 0;
    cudaMemcpyAsync(dev + o_st, &is, sizeof(is), cudaMemcpyHostToDevice, st);
    if (r.tw > 0 && r.win_in && is.win_len > 0)
        cudaMemcpyAsync(dev + o_win, r.win_in, size_t(is.win_len) * 8, cudaMemcpyHostToDevice, st);

    if (ctx->timing) cudaEventRecord(ctx->ev0, st);
    const StageShape s{G, N, D, row_begin, RL};
    IterState* dst = reinterpret_cast<IterState*>(dev + o_st);
    unsigned long long* words = mt ? reinterpret_cast<unsigned long long*>(dev + o_words) : nullptr;
    MtPersist* mtg = mt ? reinterpret_cast<MtPersist*>(dev + o_mt) : nullptr;
    if (mt && jump) {   // the reference stream, init words [0, 2RD) in 2^jlevels segments
        const long long seg = (init_words + (1ll << jlevels) - 1) >> jlevels;
        const long long Q = (seg + 623) / 624 * 624;                // whole generator passes
        const MtJumpTerms& jt = mt_jump_ladder_terms(uint64_t(Q), jlevels);   // cached: stays valid
        ce = cudaMemcpyAsync(dev + o_jpoly, jt.terms.data(), jt.terms.size() * 2, cudaMemcpyHostToDevice, st);
        if (ce != cudaSuccess) return cuda_fail(ce, "jump terms");
        const int fe = stage_mt_fill_parallel(mtg, r.seed, init_words, words,
                                              reinterpret_cast<unsigned long long*>(dev + o_jst),
                                              reinterpret_cast<const unsigned short*>(dev + o_jpoly), jt.count.data(),
                                              jlevels, Q, st);
        if (fe) return cuda_fail(cudaError_t(fe), "stage_mt_fill_parallel");
    } else if (mt) {   // sequential
        const int fe = stage_mt_fill(mtg, r.seed, true, 0, init_words, words, st);
        if (fe) return cuda_fail(cudaError_t(fe), "stage_mt_fill");
    }
    int e = stage_init(fp64, s, reinterpret_cast<double*>(dev + o_hyp), dev + o_lo, dev + o_hi, r.seed, 0,
                       r.prev ? reinterpret_cast<double*>(dev + o_prev) : nullptr, r.warm, r.pi_radius,
                       dev + o_x, dev + o_v, dev + o_pb, st, words, 0);
    if (e) return cuda_fail(cudaError_t(e), "stage_init");
    // mt19937: step k's 3R draws are generated on a side stream while the
    // fitness and best kernels run (the generator is one CTA and sequential),
    // into window k & 1: window b is free again once step k - 2 (or the
    // initialisation) has read it, so the generator runs up to a step ahead
    // and its ~0.2 ms per step at 393 k draws (scale harness) never holds a
    // step up
    if (mt && !ctx->side) {
        ce = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
        for (int b = 0; b < 2 && ce == cudaSuccess; ++b) {
            ce = cudaEventCreateWithFlags(&ctx->ev_free[b], cudaEventDisableTiming);
            if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ctx->ev_fill[b], cudaEventDisableTiming);
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "side stream");
    }
    if (mt) {
        cudaEventRecord(ctx->ev_free[0], st);
        cudaEventRecord(ctx->ev_free[1], st);
    }
    const WorldLayout& wl = wp.lay;
    for (int k = 1; k <= r.cap; ++k) {
        if (mt && k < r.cap) {   // draws of step k (the generator persists across iterations)
            const uint64_t first = 2ull * uint64_t(R) * D + uint64_t(k - 1) * 3ull * R;
            const int b = k & 1;
            cudaStreamWaitEvent(ctx->side, ctx->ev_free[b], 0);
            const int fe = stage_mt_fill(mtg, r.seed, false, (long long)first, (long long)first + 3ll * R,
                                         words + size_t(b) * 3 * R, ctx->side);
            if (fe) return cuda_fail(cudaError_t(fe), "stage_mt_fill");
            cudaEventRecord(ctx->ev_fill[b], ctx->side);
        }
        if (path)
            e = stage_eval_path(fp64, dev + o_world, wl.max_obs, wl.max_verts, int(wl.off_offsets),
                                int(wl.off_verts), D, RL, dev + o_x, r.alpha, r.beta, dev + o_fit,
                                reinterpret_cast<int*>(dev + o_q), dst, st);
        else
            e = stage_eval_bench(fp64, r.problem, D, RL, dev + o_x, dev + o_fit,
                                 reinterpret_cast<int*>(dev + o_q), dst, st);
        if (e) return cuda_fail(cudaError_t(e), "stage_eval");
        e = stage_pbest_partials(fp64, s, dev + o_x, dev + o_fit, reinterpret_cast<int*>(dev + o_q),
                                 dev + o_pb, dev + o_pbf, reinterpret_cast<int*>(dev + o_pbq), dst,
                                 dev + o_pf, reinterpret_cast<int*>(dev + o_prow),
                                 reinterpret_cast<int*>(dev + o_pq), dst, st,
                                 reinterpret_cast<unsigned char*>(dev + o_imp));
        if (e) return cuda_fail(cudaError_t(e), "stage_pbest");
        e = stage_group_bests(fp64, s, dev + o_pf, reinterpret_cast<int*>(dev + o_prow),
                              reinterpret_cast<int*>(dev + o_pq), dev + o_pb, dev + o_gbx, dev + o_gbf,
                              reinterpret_cast<int*>(dev + o_gbq), dev + o_cand + cstride * r.rank, dst, st, dst,
                              dev + o_x, reinterpret_cast<const unsigned char*>(dev + o_imp));
        if (e) return cuda_fail(cudaError_t(e), "stage_group_bests");
        if (nranks > 1 && r.comm) {   // the only cross-GPU traffic: each rank's tbest candidate
            e = comm_allgather(r.comm, dev + o_cand + cstride * r.rank, dev + o_cand, cstride, st);
            if (e) return fail(SF_CUDA_ERROR, "ncclAllGather of tbest candidates failed");
        } else if (nranks > 1) {      // host exchange (sf_ctx_set_exchange): the same bytes through the host
            std::vector<unsigned char> mine(cstride), all(cstride * size_t(nranks));
            ce = cudaMemcpyAsync(mine.data(), dev + o_cand + cstride * r.rank, cstride, cudaMemcpyDeviceToHost, st);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
            if (ce != cudaSuccess) return cuda_fail(ce, "candidate D2H");
            if ((e = exchange_allgather(ctx, mine.data(), all.data(), cstride))) return e;
            ce = cudaMemcpyAsync(dev + o_cand, all.data(), all.size(), cudaMemcpyHostToDevice, st);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);   // `all` is a pageable temporary
            if (ce != cudaSuccess) return cuda_fail(ce, "candidates H2D");
        }
        e = stage_finish(fp64, D, dev + o_cand, nranks, dev + o_tbx, dst,
                         r.tw > 0 ? reinterpret_cast<double*>(dev + o_win) : nullptr, r.tw,
                         r.auto_truncate, r.delta, k, r.cap, reinterpret_cast<double*>(dev + o_trace), st);
        if (e) return cuda_fail(cudaError_t(e), "stage_finish");
        if (k < r.cap) {
            const uint64_t first = 2ull * uint64_t(R) * D + uint64_t(k - 1) * 3ull * R;
            const int b = k & 1;
            if (mt) cudaStreamWaitEvent(st, ctx->ev_fill[b], 0);
            e = stage_step(fp64, s, reinterpret_cast<double*>(dev + o_hyp), dev + o_lo, dev + o_hi,
                           dev + o_x, dev + o_v, dev + o_pb, dev + o_gbx, dev + o_tbx, r.seed, first,
                           k, r.cap, dst, st, mt ? words + size_t(b) * 3 * R : nullptr, (long long)first,
                           reinterpret_cast<const unsigned char*>(dev + o_imp));
            if (e) return cuda_fail(cudaError_t(e), "stage_step");
            if (mt) cudaEventRecord(ctx->ev_free[b], st);
        }
    }
    if (ctx->timing) {
        cudaEventRecord(ctx->ev1, st);
        cudaEventSynchronize(ctx->ev1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        ctx->kernel_ms += ms;
        ctx->launches += 1;
    }
    // results
    IterState fin{};
    std::vector<unsigned char> tb(size_t(D) * tsz);
    r.trace.assign(r.cap, 0.0);
    r.win_out.assign(std::max(r.tw, 1), 0.0);
    cudaMemcpyAsync(&fin, dev + o_st, sizeof(fin), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(tb.data(), dev + o_tbx, tb.size(), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(r.trace.data(), dev + o_trace, size_t(r.cap) * 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(r.win_out.data(), dev + o_win, r.win_out.size() * 8, cudaMemcpyDeviceToHost, st);
    ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return cuda_fail(ce, "staged run");
    r.best.assign(D, 0.0);
    for (int d = 0; d < D; ++d)
        r.best[d] = fp64 ? reinterpret_cast<double*>(tb.data())[d] : double(reinterpret_cast<float*>(tb.data())[d]);
    // window back in oldest-first order
    std::vector<double> w(fin.win_len);
    for (int i = 0; i < fin.win_len; ++i) w[i] = r.win_out[(fin.win_head + i) % std::max(r.tw, 1)];
    r.win_out = w;
    r.out = SwarmOut{};
    r.out.status = uint32_t(fin.status);
    r.out.iterations = uint32_t(fin.k_done);
    r.out.truncated = uint32_t(fin.truncated);
    r.out.window_len = uint32_t(fin.win_len);
    if (fin.status == 2) {
        r.out.bad_g = uint32_t(fin.nonfinite_row / N);
        r.out.bad_n = uint32_t(fin.nonfinite_row % N);
        r.out.bad_k = uint32_t(fin.k_done);
    } else {
        r.out.fitness = fin.tbest_f;
        r.out.q = uint32_t(fin.tbest_q);
        if (path) {   // record length (planner.hpp:194) on the final best path, FP64
            double total = 0.0, px = r.world->start.x, py = r.world->start.y;
            if (!fp64) { px = double(float(px)); py = double(float(py)); }
            const int W = D / 2;
            for (int j = 1; j <= W + 1; ++j) {
                double nx = j <= W ? r.best[j - 1] : r.world->target.x;
                double ny = j <= W ? r.best[W + j - 1] : r.world->target.y;
                if (!fp64 && j > W) { nx = double(float(nx)); ny = double(float(ny)); }
                total += std::hypot(nx - px, ny - py);
                px = nx;
                py = ny;
            }
            r.out.length = total;
        }
    }
    return SF_OK;
}

// -------------------------------------------------------------- host PSO
uint64_t derive_seed(uint64_t root, const char* tag) {
    return splitmix64(root ^ fnv1a64(tag, std::strlen(tag)));
}
uint64_t derive_seed(uint64_t root, const char* tag, uint64_t index) {
    return splitmix64(derive_seed(root, tag) + index);
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

// swarm.hpp:94-132
void host_init_swarm(HostSwarm& s, const double* hypers, const double* lo, const double* hi,
                     uint32_t G, uint32_t N, uint32_t D, HostStream& rng) {
    s.G = G;
    s.N = N;
    s.D = D;
    const size_t total = size_t(G) * N * D;
    s.x.resize(total);
    s.v.resize(total);
    s.pbf.assign(size_t(G) * N, std::numeric_limits<double>::infinity());
    s.gbx.assign(size_t(G) * D, 0.0);
    s.gbf.assign(G, std::numeric_limits<double>::infinity());
    s.tbx.assign(D, 0.0);
    s.tbf = std::numeric_limits<double>::infinity();
    for (size_t i = 0; i < total; ++i) s.x[i] = rng.uniform(lo[i % D], hi[i % D]);
    for (uint32_t g = 0; g < G; ++g) {
        double* vg = s.v.data() + size_t(g) * N * D;
        for (size_t i = 0; i < size_t(N) * D; ++i) {
            const double vmax = hypers[6 * g + 5] * (hi[i % D] - lo[i % D]);
            vg[i] = rng.uniform(-vmax, vmax);
        }
    }
    s.pbx = s.x;
}

// swarm.hpp:138-174
void host_step(HostSwarm& s, const double* hypers, const double* lo, const double* hi,
               HostStream& rng, uint32_t k, uint32_t T) {
    const size_t GN = size_t(s.G) * s.N, D = s.D;
    std::vector<double> r(3 * GN);
    for (double& u : r) u = rng.uniform();
    const double frac = double(k) / double(T);
    for (uint32_t g = 0; g < s.G; ++g) {
        const double* h = hypers + 6 * g;
        const double w = h[3] - (h[3] - h[4]) * frac;
        const double* gb = s.gbx.data() + size_t(g) * D;
        for (uint32_t n = 0; n < s.N; ++n) {
            const size_t row = size_t(g) * s.N + n;
            const double a1 = h[0] * r[row], a2 = h[1] * r[GN + row], a3 = h[2] * r[2 * GN + row];
            double* xv = s.x.data() + row * D;
            double* vv = s.v.data() + row * D;
            const double* pb = s.pbx.data() + row * D;
            for (size_t d = 0; d < D; ++d) {
                const double vmax = h[5] * (hi[d] - lo[d]);
                double nv = w * vv[d] + a1 * (pb[d] - xv[d]) + a2 * (gb[d] - xv[d]) + a3 * (s.tbx[d] - xv[d]);
                nv = clampd(nv, -vmax, vmax);
                vv[d] = nv;
                xv[d] = clampd(xv[d] + nv, lo[d], hi[d]);
            }
        }
    }
}

// runner.hpp:68-93
void host_update_bests(HostSwarm& s, const double* fitness) {
    const size_t N = s.N, D = s.D;
    for (uint32_t g = 0; g < s.G; ++g) {
        for (size_t n = 0; n < N; ++n) {
            const size_t r = g * N + n;
            if (fitness[r] < s.pbf[r]) {
                s.pbf[r] = fitness[r];
                std::copy_n(s.x.data() + r * D, D, s.pbx.data() + r * D);
            }
        }
        for (size_t n = 0; n < N; ++n) {
            const size_t r = g * N + n;
            if (s.pbf[r] < s.gbf[g]) {
                s.gbf[g] = s.pbf[r];
                std::copy_n(s.pbx.data() + r * D, D, s.gbx.data() + g * D);
            }
        }
        if (s.gbf[g] < s.tbf) {
            s.tbf = s.gbf[g];
            std::copy_n(s.gbx.data() + g * D, D, s.tbx.data());
        }
    }
}

void unflatten_hypers(const double* particle, uint32_t groups, double* out) {
    static const double lo[6] = {0.5, 0.5, 0.5, 0.1, 0.05, 0.05};   // hsef.hpp:75
    static const double hi[6] = {2.5, 2.5, 2.5, 1.0, 0.8, 1.0};     // hsef.hpp:76
    for (uint32_t g = 0; g < groups; ++g) {
        double f[6];
        for (int i = 0; i < 6; ++i) f[i] = clampd(particle[6 * g + i], lo[i], hi[i]);
        if (f[4] > f[3]) std::swap(f[3], f[4]);
        std::memcpy(out + 6 * g, f, sizeof(f));
    }
}

} // namespace sepso
