// swarm_kernel_body.cuh -- the fused SEPSO swarm kernel template (sm_100a).
//
// Included by the instantiation units swarm_inst_*.cu (each compiles a few
// instantiations, in parallel) and by swarm_kernel.cu (the launch dispatcher).
//
// See swarm_kernel.cuh for the execution model.  Reference citations are
// relative to proj/include/swarmforge/ in the reference tree.
#pragma once
#include <cooperative_groups.h>
#include <algorithm>
#include <type_traits>
#include <cuda_runtime.h>

#include "mt19937.cuh"
#include "swarm_device.cuh"

namespace cg = cooperative_groups;

namespace sepso {

// ------------------------------------------------------------------ kernel
// cluster barrier split into arrive (release) and wait (acquire)
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }

// ---- partial exchange over DSMEM: st.async with mbarrier transaction counts.
// Every CTA expects a fixed byte count per iteration into mbarrier (k & 1);
// peers' stores complete it, so no cluster-wide barrier (and none of its
// GPU-scope fence / L1 invalidation) sits in the iteration.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t peer_addr(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t dst, uint4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(dst), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t dst, uint32_t v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 ::"r"(dst), "r"(v), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P1;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        " @!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}

#ifndef SEPSO_GEN_HELPERS
#define SEPSO_GEN_HELPERS 8
#endif
constexpr int kGenHelpers = SEPSO_GEN_HELPERS;   // warps that deliver the step draws beside the generator

// r1, r2, r3 of step k (draw_step_randoms, swarm.hpp:59-70): R words each at
// 2RD + (k-1)*3R of the mt19937_64 stream; rows [row0, row1) keep a_j = c_j * r_j.
template <int FN, class T>
__device__ void mt_step_draws(Ctx<T>& c, unsigned long long* mtbuf, const MtGroup& grp, int k, int row1) {
    using A = Ar<T>;
    const int R = c.R;
    const long long base = 2ll * R * c.D + (long long)(k - 1) * 3 * R;
    MtState mt{mtbuf, c.m->mt_cur, c.m->mt_blocks};      // registers only while generating
    // one window per factor: only this CTA's rows are tempered and kept
#pragma unroll 1
    for (int j = 0; j < 3; ++j)
        mt_generate<FN>(mt, grp, base + (long long)j * R + c.row0, base + (long long)j * R + row1,
                    [&](int pl, unsigned long long word) {
                        const int g = int(c.fN.div(uint32_t(c.row0 + pl)));
                        c.coef[j * c.P + pl] = A::mul(c.hyp[g * 6 + j], unit_from_word<T>(word));
                    });
    // every group thread has read the bookkeeping before the first barrier
    if (grp.lt == 0) { c.m->mt_cur = mt.cur; c.m->mt_blocks = mt.blocks; }
}

// Element loops walk (particle, column) pairs with an incremental carry instead
// of integer division: thread t starts at element t and advances by nthr.
struct ElemWalk {
    int pl, col, dpl, dcol, ncol;
    __device__ ElemWalk(const FastDiv& f, int tid, int nthr, int ncols) : ncol(ncols) {
        pl = int(f.div(uint32_t(tid)));
        col = tid - pl * ncols;
        dpl = int(f.div(uint32_t(nthr)));
        dcol = nthr - dpl * ncols;
    }
    __device__ __forceinline__ void next() {
        pl += dpl;
        col += dcol;
        if (col >= ncol) { col -= ncol; ++pl; }
    }
};

static __device__ void step_world_part(unsigned char* rec, int off_offsets, int off_verts, int off_vel, double dt,
                                       int t);

#ifndef SEPSO_STEPW
#define SEPSO_STEPW 4
#endif
constexpr int STEPW = SEPSO_STEPW;

// a pushed pbest row in st.async units: 16-byte vectors, else 4-byte words
template <class T>
__host__ __device__ inline int row_units(int D) {
    const int bytes = D * int(sizeof(T));
    return bytes % 16 == 0 ? bytes / 16 : bytes / 4;
}

// Launch constants derived on the host from the shape (launch_t): the shared
// memory layout, the exchange byte count and the fast divisors -- so no thread
// spends the prologue on them (the generator seeding waits behind it).
struct LaunchDerived {
    SmemLayout lay;
    uint32_t xbytes;            // bytes every CTA receives per iteration
    uint32_t dmul[4], dshr[4];  // FastDiv of S, D, N, V (pushed-row units)
    double at_var_bound;        // AT: sqrt_rn(v /rn tw) < delta  <=>  v < at_var_bound
};

// The AT decision std = sqrt(var / tw) < delta (planner.hpp:138-149) is
// monotone in var (both operations correctly rounded), so it is exactly
// "var < the smallest v >= 0 whose sqrt(v / tw) reaches delta" -- found once
// on the host by bisection over the ordered bit patterns of non-negative
// doubles, with the same IEEE operations.  Saves a division and a square root
// per AT test on the device.
static double at_var_bound(double delta, int tw) {
    static thread_local double cd = std::numeric_limits<double>::quiet_NaN(), cv = 0.0;
    static thread_local int ct = -1;
    if (delta == cd && tw == ct) return cv;
    double v;
    if (!(delta > 0.0) || tw <= 0) {
        v = 0.0;                                           // never below delta
    } else {
        uint64_t lo = 0, hi = 0x7FF0000000000000ull;       // +0 .. +inf
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            double x;
            std::memcpy(&x, &mid, 8);
            if (std::sqrt(x / double(tw)) >= delta) hi = mid;
            else lo = mid + 1;
        }
        std::memcpy(&v, &lo, 8);
    }
    cd = delta; ct = tw; cv = v;
    return v;
}

// ---- resident planner: job hand-off with the host (ServerCtl, pinned memory)
__device__ __forceinline__ uint32_t ld_acquire_sys(const volatile uint32_t* a) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Resident planner results: 16-byte chunks {3 payload words, job number}, each
// one store (one bus write), so the host knows a chunk is this job's from its
// own tag -- no system fence between the record and the host seeing it.
// Layout: [0] {iterations, q, status}  [1] {fitness, truncated}  [2] {length,
// window_len}  [3] {bad_g, bad_n, bad_k}  [4 + d] best_x[d]  [4 + D + k] trace[k].
__device__ __forceinline__ void put_chunk(void* base, int i, uint32_t a, uint32_t b, uint32_t c, uint32_t tag) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};"
                 ::"l"(reinterpret_cast<uint4*>(base) + i), "r"(a), "r"(b), "r"(c), "r"(tag) : "memory");
}
__device__ __forceinline__ void put_chunk_d(void* base, int i, double v, uint32_t c, uint32_t tag) {
    const unsigned long long u = __double_as_longlong(v);
    put_chunk(base, i, uint32_t(u), uint32_t(u >> 32), c, tag);
}

// v, as a value the compiler cannot treat as loop invariant
__device__ __forceinline__ int opaque_int(int v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

// Wait (bounded, ~2 ms) until the ahead-of-time init walk publishes seq.
static __device__ bool pre_wait(const int* flag, int seq) {
    const unsigned long long t0 = global_ns();
    for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v == seq) return true;
        if (global_ns() - t0 > 2000000ull) return false;
        __nanosleep(256);
    }
}
// Every thread of every CTA of the cluster: wait for the next job.  Rank 0's
// thread 0 polls the host words; rank 0's threads then read the job's input
// bytes from pinned host memory once (one round trip over the bus) and store
// them, with the decision word, into every rank's shared memory; one cluster
// barrier publishes both.  Returns the job's sequence number, 0 = exit.
static __device__ uint32_t server_next_job(ServerCtl* srv, uint32_t last, uint32_t* cmd, unsigned char* jobsm,
                                    int crank, int C) {
    if (crank == 0) {
        if (threadIdx.x == 0) {
            const unsigned long long idle_ns = srv->idle_ns;
            const unsigned long long t0 = global_ns();
            uint32_t d = 0;
            for (;;) {
                // job_seq and quit share one 8-byte word: one bus round trip per poll
                unsigned long long jq;
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(jq) : "l"(&srv->job_seq) : "memory");
                const uint32_t s = uint32_t(jq);
                if (s != last) {
                    d = s;
                    cmd[1] = ld_acquire_sys(reinterpret_cast<const volatile uint32_t*>(&srv->job_bytes));   // per job
                    srv->t_pick = global_ns();
                    break;
                }
                if (uint32_t(jq >> 32)) break;                 // quit
                if (global_ns() - t0 > idle_ns) break;
            }
            *cmd = d;
        }
        __syncthreads();
        const uint32_t d = *cmd;
        const int nb = d ? int(cmd[1]) / 16 : 0;
        const uint32_t js = smem_addr(jobsm), cs = smem_addr(cmd);
        for (int i = threadIdx.x; i < nb; i += blockDim.x) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4*>(srv->job) + i);
            for (int r = 0; r < C; ++r)
                asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};"
                             ::"r"(peer_addr(js + 16 * i, r)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
        }
        if (int(threadIdx.x) > 0 && int(threadIdx.x) < C)
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(peer_addr(cs, int(threadIdx.x))), "r"(d) : "memory");
    }
    cluster_arrive();            // release: the job bytes and the word are in every rank's memory
    cluster_wait();
    return *reinterpret_cast<volatile uint32_t*>(cmd);
}

// FP32 engine's final record: this thread's share of Q of the best path
// (tbx) on the caller's FP64 world staged in shared memory (vert64 = vertices
// then start, target): reference predicates (geometry.hpp:196-220), one
// (segment, edge) pair or one first-waypoint containment test per task.  Out
// of line: it runs once per frame and keeps its registers out of the loop's.
static __device__ __noinline__ int rec64_hits(const double* wv, const int* woff, int O, const float* tbx, int W, int S,
                                       int tid, int nthr) {
    const int nv = woff[O];
    const double sx = wv[2 * nv], sy = wv[2 * nv + 1], tx = wv[2 * nv + 2], ty = wv[2 * nv + 3];
    auto wpx = [&](int j) { return j == 0 ? sx : (j <= W ? double(tbx[j - 1]) : tx); };
    auto wpy = [&](int j) { return j == 0 ? sy : (j <= W ? double(tbx[W + j - 1]) : ty); };
    int hits = 0;
    for (int t = tid; t < S * nv + O; t += nthr) {
        if (t < S * nv) {
            const int sg = t / nv, e = t - sg * nv;
            int o = 0;
            while (woff[o + 1] <= e) ++o;
            const int e2 = e + 1 == woff[o + 1] ? woff[o] : e + 1;
            hits += segments_intersect_ref(wpx(sg), wpy(sg), wpx(sg + 1), wpy(sg + 1), wv[2 * e], wv[2 * e + 1],
                                           wv[2 * e2], wv[2 * e2 + 1]) ? 1 : 0;
        } else {
            const int o = t - S * nv, v0 = woff[o];
            hits += point_strictly_inside_ref(wpx(1), wpy(1), woff[o + 1] - v0,
                                              [&](int i) { return wv[2 * (v0 + i)]; },
                                              [&](int i) { return wv[2 * (v0 + i) + 1]; }) ? 1 : 0;
        }
    }
    return hits;
}

// path_length (geometry.hpp:223-231) of the best path start -> w_1..w_W ->
// target in FP64: one warp, the S hypots in parallel, summed in path order.
template <class T>
__device__ __noinline__ double path_length64(const T* tbx, int W, int S, double sx, double sy, double tx, double ty,
                                             int lane) {
    double len = 0.0;
    for (int j0 = 0; j0 < S; j0 += 32) {
        const int j = j0 + lane;
        double h = 0.0;
        if (j < S) {
            const double px = j == 0 ? sx : double(tbx[j - 1]);
            const double py = j == 0 ? sy : double(tbx[W + j - 1]);
            const double nx = j < W ? double(tbx[j]) : tx;
            const double ny = j < W ? double(tbx[W + j]) : ty;
            h = hypot_glibc(__dsub_rn(nx, px), __dsub_rn(ny, py));
        }
        for (int i = 0; i < 32 && j0 + i < S; ++i) len = __dadd_rn(len, __shfl_sync(0xffffffffu, h, i));
    }
    return len;
}

// AT statistic of the window (planner.hpp:138-149) by one warp in parallel.
// The reference sums sequentially: mean_s = (sum w_i) / tw, var_s = sum (w_i -
// mean_s)^2.  Any summation order of n = tw terms is within gamma_{n-1} sum|w|
// of the exact sum, so both means are within dl = 1.01 (n + 2) u M of the
// exact mean mu (M = max |w|, u = 2^-53); with V(m) = V(mu) + n (m - mu)^2 and
// the squared-difference terms off by <= 3u each, |var_s - var_p| <=
// 2.04 (n + 3) u (var_p + n dl^2) + 2 n dl^2 < E (a factor 2 to spare).
// Returns 1 when var_s < bound for certain, 0 when var_s >= bound for certain,
// -1 when the caller must evaluate the sequential sums.  All lanes return it.
__device__ __forceinline__ int at_decide_parallel(const double* win, int wh, int tw, double bound, int lane) {
    double s = 0.0, mx = 0.0;
    for (int i = lane; i < tw; i += 32) {
        const int at = wh + i < tw ? wh + i : wh + i - tw;
        const double w = win[at];
        s += w;
        mx = fmax(mx, fabs(w));
    }
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    }
    const double mean = s / double(tw);
    double v = 0.0;
    for (int i = lane; i < tw; i += 32) {
        const int at = wh + i < tw ? wh + i : wh + i - tw;
        const double d = win[at] - mean;
        v = fma(d, d, v);
    }
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const double n = double(tw), u = 0x1p-53;
    const double dl = 1.01 * (n + 2.0) * u * mx;
    const double E = 4.0 * (n + 3.0) * u * (v + n * dl * dl) + 4.0 * n * dl * dl;
    if (v + E < bound) return 1;
    if (v - E >= bound) return 0;
    return -1;
}

// The same decision from registers (tw <= 32, lane i holds window slot i), in
// one centred pass: d_i = w_i - c (c = the newest value), S = sum d, Q = sum
// d^2, V = Q - S^2 / tw.  With X >= max |d_i| (REDUX on the high words) the
// rounding of this pass stays within 24.5 u n X^2 of the exact V(mu) (d_i and
// d_i^2 relative 3u, 5-level trees gamma_5, S^2 / n three roundings, the final
// difference one), and the reference's sequential value within 2.04 (n + 3) u
// n X^2 + n dl^2 of it (see at_decide_parallel), so E below bounds |var_s - V|
// with margin.  Returns 1 / 0 when certain, -1 inside the band.
__device__ __forceinline__ int at_decide_regs(double w, int lane, int tw, double c, double inv_n, double bound) {
    const bool act = lane < tw;
    const double d = act ? w - c : 0.0;
    double s = d, q = d * d;
    const uint32_t hx = __reduce_max_sync(0xffffffffu, act ? uint32_t(uint64_t(__double_as_longlong(fabs(d))) >> 32) : 0u);
    const uint32_t hm = __reduce_max_sync(0xffffffffu, act ? uint32_t(uint64_t(__double_as_longlong(fabs(w))) >> 32) : 0u);
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        q += __shfl_xor_sync(0xffffffffu, q, off);
    }
    const double X = __longlong_as_double((long long)((uint64_t(hx) << 32) | 0xffffffffull));
    const double M = __longlong_as_double((long long)((uint64_t(hm) << 32) | 0xffffffffull));
    const double n = double(tw), u = 0x1p-53;
    const double dl = 1.01 * (n + 2.0) * u * M;
    const double E = (3.0 * n + 40.0) * u * n * X * X + 2.0 * n * dl * dl;
    const double v = q - s * s * inv_n;
    if (!(v == v) || !(E == E) || E > 0x1p1000) return -1;   // non-finite window: the sequential sums decide
    if (v + E < bound) return 1;
    if (v - E >= bound) return 0;
    return -1;
}

// MAXT: the largest block size the instantiation launches with.  The register
// budget follows from it (64 at 1024 threads, 72 at 896): the latency launch of
// one paper scene (85 rows x 9 segments + 4 generator warps = 896 threads) gets
// its own instantiation so its hot loop does not spill at the 1024-thread cap.
// SERVER: the resident-planner instantiation (jobs loop, p.srv); the one-pass
// instantiations carry none of its state, so their hot loop keeps its registers.
template <class T, bool PATH, bool RING, int MAXT = 1024, bool SERVER = false, bool FAST = false>
__global__ void __launch_bounds__(MAXT, 1) swarm_kernel(const __grid_constant__ SwarmParams p,
                                                        const __grid_constant__ ParamPayload pl,
                                                        const __grid_constant__ LaunchDerived ld, int problem) {
    using A = Ar<T>;
    // kLat (FAST): the FP32 specialised instantiations, launched only for the reference's
    // mt19937 stream, G <= 32, tw <= 32 and a generator-first shape
    // (launch_swarms checks): the branches it can never take are compiled out,
    // which keeps the per-iteration code -- fetched again every iteration by
    // the single-warp phases -- small.
    constexpr bool kLat = FAST && sizeof(T) == 4 && PATH;
#ifdef SEPSO_PROFILE
    unsigned long long g_entry_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry_));
#endif
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemLayout& L = ld.lay;
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int swarm = blockIdx.x / p.C;

    Ctx<T> c;
    c.G = p.G; c.N = p.N; c.D = p.D; c.W = p.D / 2; c.S = c.W + 1; c.R = p.G * p.N;
    c.fS.d = uint32_t(c.S); c.fS.mul = ld.dmul[0]; c.fS.shr = ld.dshr[0];
    c.fD.d = uint32_t(c.D); c.fD.mul = ld.dmul[1]; c.fD.shr = ld.dshr[1];
    c.fN.d = uint32_t(c.N); c.fN.mul = ld.dmul[2]; c.fN.shr = ld.dshr[2];
    c.fV.d = uint32_t(row_units<T>(c.D)); c.fV.mul = ld.dmul[3]; c.fV.shr = ld.dshr[3];
    c.C = p.C; c.crank = int(cluster.block_rank());
    // partial-exchange mbarriers (one arrival: the local expect_tx); published
    // to the peers by a cluster arrive here and a wait before the first push
    const uint32_t mbar0 = smem_addr(smem + L.mbar);
    if (threadIdx.x == 0) {
        mbar_init(mbar0, 1);
        mbar_init(mbar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_arrive();
    c.row0 = c.crank * p.rows_per_cta;
    const int row1 = min(c.R, c.row0 + p.rows_per_cta);
    c.P = max(0, row1 - c.row0);
    const int gfirst = c.row0 / c.N;
    c.LG = c.P > 0 ? (row1 - 1) / c.N - gfirst + 1 : 0;
    auto S8 = [&](size_t off) { return smem + off; };
    c.x = (T*)S8(L.x); c.v = (T*)S8(L.v); c.pb = (T*)S8(L.pb); c.pbf = (T*)S8(L.pbf);
    c.pbq = (int*)S8(L.pbq); c.q = (int*)S8(L.q); c.fit = (T*)S8(L.fit); c.imp = (int*)S8(L.imp);
    c.seglen = (T*)S8(L.seglen); c.coef = (T*)S8(L.coef); c.lo = (T*)S8(L.lo); c.hi = (T*)S8(L.hi);
    c.hyp = (T*)S8(L.hyp); c.gbx = (T*)S8(L.gbx); c.gbf = (T*)S8(L.gbf); c.gbq = (int*)S8(L.gbq);
    c.chg = (int*)S8(L.chg); c.tbx = (T*)S8(L.tbx); c.win = (double*)S8(L.win);
    c.part = (Part*)S8(L.part); c.px = (T*)S8(L.px); c.allpart = (Part*)S8(L.allpart);
    c.allbad = (int*)S8(L.allbad); c.gtab = (int*)S8(L.gtab); c.ctab = (int*)S8(L.ctab);
    c.obb = (T*)S8(L.obb); c.ooff = (int*)S8(L.ooff); c.ofl = (int*)S8(L.ofl); c.vert = (T*)S8(L.vert);
    c.edge = (T*)S8(L.edge); c.list = p.entry_cap > 0 ? (uint32_t*)S8(L.list) : nullptr; c.m = (Misc<T>*)S8(L.misc);
    c.vert64 = (PATH && sizeof(T) == 4) ? (double*)S8(L.vert64) : nullptr;
    const int LGM = p.max_local_groups;
    const uint32_t xbytes = ld.xbytes;
    // resident planner (p.srv): the cluster serves one frame per posted job,
    // its inputs copied from pinned host memory into shared memory; otherwise
    // the loop body runs once on the launch's own inputs
    ServerCtl* const srv = SERVER ? p.srv : nullptr;
    unsigned char* const jobsm = srv ? S8(L.job) : nullptr;
    const unsigned char* const jb = srv ? jobsm : pl.bytes;
    uint32_t jseq = 0;
    if (srv) jseq = srv->done_seq;  // the last job served before this launch (the host is not posting while it reads)
    if (srv) cluster_wait();       // the resident cluster matches the launch's cluster_arrive up front
    // resident planner: after each job the cluster runs the constants stage
    // once more on the same inputs (a dry pass) while the host is busy with the
    // result, so that stage's code is in the SM's instruction cache when the
    // next job arrives (it is otherwise fetched from L2 / DRAM, ~4 us a frame)
#ifndef SEPSO_DRY
#define SEPSO_DRY 1
#endif
    bool dry = false;
    for (;;) {
    if (SERVER && dry && PATH && sizeof(T) == 4 && c.crank == 0 && warp == 1) {
        // the dry pass first runs the final record's code on the last job's
        // world and path (the FP64 recheck, the hypot chain; result discarded),
        // then the constants stage, so that stage is the most recent code
        const int h = rec64_hits(c.vert64, c.ooff, c.O, reinterpret_cast<const float*>(c.tbx), c.W, c.S, lane, 32);
        const double len = path_length64(c.tbx, c.W, c.S, 0.0, 0.0, 1.0, 1.0, lane);
        if (h < 0 || len < 0.0) c.m->q64 = h;
    }
    if (srv && !dry) {
        // every job starts its exchange mbarriers at phase 0 (all phases of the
        // last job completed); the cluster barrier inside publishes the init
        if (tid == 0) {
            mbar_init(mbar0, 1);
            mbar_init(mbar0 + 8, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        jseq = server_next_job(srv, jseq, reinterpret_cast<uint32_t*>(S8(L.srvcmd)), jobsm, c.crank, c.C);
        if (jseq == 0) break;
        if (c.crank == 0 && tid == 0) { srv->t_ready = global_ns(); srv->c_ready = clock64(); }
    }
    const uint64_t seed =
        p.roots ? splitmix64(splitmix64(p.roots[swarm] ^ p.tag_hash) + uint64_t(p.frame_index))
                : (p.inl ? reinterpret_cast<const unsigned long long*>(jb + p.in_seed) : p.seeds)[swarm];
    const int G = c.G, N = c.N, D = c.D, R = c.R;
    long long* const prof = (kProfiling && p.prof != nullptr && swarm == 0 && c.crank == 0 && tid == 0) ? p.prof : nullptr;
    // per-CTA (thread 0) work before the exchange: [(k * 16 + crank) * 2] = cycles, [+1] = wait
    long long* const wprof = (kProfiling && p.prof != nullptr && swarm == 0 && tid == 0 && c.crank < 16)
                                 ? p.prof + size_t(kProfPhases) * (p.cap + 1) : nullptr;
    long long wt0 = 0;
#define SEPSO_SMARK(i) do { if (srv && !dry && c.crank == 0 && tid == 0) srv->t_mark[i] = (unsigned long long)clock64(); } while (0)
#define SEPSO_MARK(ph) do { if (prof) prof[(k - 1) * kProfPhases + (ph)] = clock64(); } while (0)
#define SEPSO_IMARK(ph) do { if (prof) prof[p.cap * kProfPhases + (ph)] = clock64(); } while (0)
#define SEPSO_GMARK(ph) do { if (kProfiling && prof) { unsigned long long g_; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_)); prof[p.cap * kProfPhases + (ph)] = (long long)g_; } } while (0)
    SEPSO_IMARK(0);
    SEPSO_GMARK(7);
#ifdef SEPSO_PROFILE
    if (prof) prof[p.cap * kProfPhases + 12] = (long long)g_entry_;
#endif

    // ---------------------------------------------------------- constants
    // With the mt19937 stream, the last warp's lane 0 seeds the generator
    // (a 311-step sequential recurrence) while the other warps stage the
    // constants; they synchronise on named barrier 2.
    unsigned long long* const mtbuf = (unsigned long long*)S8(L.mt);
    const bool mt_on = kLat || p.rng == kMt19937;
    // (opaque per job: otherwise the compiler hoists the strided loops' trip
    // counts below out of the resident job loop and spills them -- reloads
    // that miss to DRAM after an L2 flush, ~1 us each on the frame's path)
    const int cw = opaque_int((mt_on && nthr >= 64) ? nthr - 32 : nthr);
    const unsigned char* wrec =
        PATH ? (p.inl ? jb + p.in_world : p.worlds) + size_t(swarm) * size_t(p.world_stride) : nullptr;
    if (PATH && !p.inl) {
        // world record in HBM (scene batches, large inputs): one parallel copy of
        // the whole fixed-stride record into shared memory, so the header ->
        // offsets -> vertices reads below are not a chain of DRAM round trips
        const int nv4 = int(p.world_stride / 16);          // <= the layout's allocation (max_obs, max_verts)
        unsigned char* wsm = S8(L.wcopy);
        #pragma unroll 1
        for (int i = tid; i < nv4; i += nthr)
            reinterpret_cast<uint4*>(wsm)[i] = __ldcg(reinterpret_cast<const uint4*>(wrec) + i);
        __syncthreads();
        wrec = wsm;
    }
    c.O = 0;
    const unsigned long long* seeded =
        p.mt_pre ? p.mt_pre + size_t(swarm) * 312
                 : ((p.inl && p.in_mtst >= 0) ? reinterpret_cast<const unsigned long long*>(jb + p.in_mtst) + size_t(swarm) * 312
                                              : nullptr);
    // the init walk done ahead of time (prewalk.cu), when this frame has one
    SEPSO_SMARK(6);
    const bool pre_cand = (p.inl && p.in_pre >= 0) ? reinterpret_cast<const PreRec*>(jb + p.in_pre)->valid != 0
                                                   : p.pre_words != nullptr;
    if (pre_cand) {
        // pull this CTA's init words, the generator pair and the flag into L2
        // now (non-binding: the loads after the flag's acquire read L2, which
        // the walk's stores reach), so the init below waits on L2, not DRAM
        const PreRec* prr = (p.inl && p.in_pre >= 0) ? reinterpret_cast<const PreRec*>(jb + p.in_pre) : nullptr;
        const size_t RD2 = 2 * size_t(c.R) * size_t(c.D);
        const char* w = reinterpret_cast<const char*>(
            (prr ? reinterpret_cast<const unsigned long long*>(prr->words) : p.pre_words) + size_t(swarm) * RD2);
        const size_t xb = size_t(c.row0) * c.D * 8, nb = size_t(c.P) * c.D * 8, vb = RD2 / 2 * 8;
        const int nl = int((nb + 127) / 128) + 1;          // + the line a misaligned start spills into
        const char* pp = reinterpret_cast<const char*>(
            (prr ? reinterpret_cast<const unsigned long long*>(prr->pair) : p.pre_pair) + size_t(swarm) * kPrePairWords);
        const char* pf = reinterpret_cast<const char*>((prr ? reinterpret_cast<const int*>(prr->flag) : p.pre_flag) + swarm);
        if (tid < nl) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(w + xb + size_t(tid) * 128));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(w + vb + xb + size_t(tid) * 128));
        } else if (tid - nl < kPrePairWords * 8 / 128) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pp + size_t(tid - nl) * 128));
        } else if (tid - nl == kPrePairWords * 8 / 128) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
        }
    }
    if (tid >= cw) {
        if (pre_cand) {
            // the walk arrives from HBM (seeded here only if it is late)
        } else if (seeded) {                  // the host's seeded state, one warp copies it
            #pragma unroll 1
            for (int i = tid - cw; i < 312; i += nthr - cw) mtbuf[312 + i] = seeded[i];
        } else if (tid == cw) {
            mt_seed_words(mtbuf + 312, seed);
        }
        if (kProfiling && tid == cw && p.prof != nullptr && swarm == 0 && c.crank == 0)
            p.prof[p.cap * kProfPhases + 13] = clock64();
        if (PATH) world_regs(c, wrec);
    } else {
        SEPSO_SMARK(5);
        const double* hyp_src = (p.inl ? reinterpret_cast<const double*>(jb + p.in_hyp) : p.hypers) +
                                size_t(swarm) * size_t(p.hypers_stride);
        #pragma unroll 1
        for (int i = tid; i < G * 6; i += cw) c.hyp[i] = T(hyp_src[i]);
        SEPSO_IMARK(15);
        SEPSO_SMARK(0);
        if (PATH) {
            world_regs(c, wrec);
            SEPSO_IMARK(16);
            load_world(c, wrec, p.off_offsets, p.off_verts, tid, cw, cw == nthr ? 0 : 2);
            SEPSO_IMARK(17);
            SEPSO_SMARK(1);
        } else {
            const double* lo_src = p.inl ? reinterpret_cast<const double*>(jb + p.in_lo) : p.lo;
            const double* hi_src = p.inl ? reinterpret_cast<const double*>(jb + p.in_hi) : p.hi;
            #pragma unroll 1
            for (int d = tid; d < D; d += cw) { c.lo[d] = T(lo_src[d]); c.hi[d] = T(hi_src[d]); }
        }
        if (tid == 0) {
            SEPSO_IMARK(18);
            SEPSO_SMARK(2);
            Misc<T>* m = c.m;
            m->tbf = A::inf(); m->tbq = 0; m->tsrc_slot = -1; m->stop = 0; m->truncated = 0; m->q64 = 0;
            m->status = 0; m->bad_row = INT_MAX; m->bad_min = INT_MAX; m->n_pair = 0; m->n_cont = 0;
            m->k_done = 0;
            m->cont_cap = 0;
            const int wl = p.carry ? (p.inl ? reinterpret_cast<const int*>(jb + p.in_win_len) : p.win_len)[swarm] : 0;
            m->win_len = wl < p.tw ? wl : p.tw;
            m->win_head = 0;
            if (mt_on && cw == nthr && !pre_cand) {
                if (seeded) for (int i = 0; i < 312; ++i) mtbuf[312 + i] = seeded[i];
                else mt_seed_words(mtbuf + 312, seed);
            }
        }
        if (p.carry)
            #pragma unroll 1
            for (int i = tid; i < p.tw; i += cw)
                c.win[i] = (p.inl ? reinterpret_cast<const double*>(jb + p.in_win) : p.win_vals)[size_t(swarm) * p.tw + i];
        #pragma unroll 1
        for (int g = tid; g < G; g += cw) {
            c.gbf[g] = A::inf(); c.gbq[g] = 0; c.chg[g] = -1;
            c.gtab[2 * g] = (g * N) / p.rows_per_cta;               // CTAs owning group g
            c.gtab[2 * g + 1] = ((g + 1) * N - 1) / p.rows_per_cta;
        }
        #pragma unroll 1
        for (int cc = tid; cc < c.C; cc += cw) c.ctab[cc] = (cc * p.rows_per_cta) / N;
        #pragma unroll 1
        for (int pl = tid; pl < c.P; pl += cw) { c.pbf[pl] = A::inf(); c.pbq[pl] = 0; c.q[pl] = 0; }
        SEPSO_IMARK(14);
        SEPSO_SMARK(3);
    }
    __syncthreads();
    SEPSO_IMARK(1);
    if (SERVER && dry) {
        dry = false;
        continue;
    }
    if (srv && c.crank == 0 && tid == 0) { srv->t_pre = global_ns(); srv->t_mark[4] = (unsigned long long)clock64(); }

    // ------------------------------------------------------- initialisation
    // swarm.hpp:94-132 / planner.hpp:77-133: x draws [0, R*D), v draws [R*D, 2*R*D)
    {
        const unsigned char* hp = p.inl ? (p.has_prev ? jb + p.in_has_prev : nullptr) : p.has_prev;
        const bool warm_on = hp != nullptr && hp[swarm] != 0;
        const double* prev = warm_on ? (p.inl ? reinterpret_cast<const double*>(jb + p.in_prev) : p.prev) +
                                           size_t(swarm) * D
                                     : nullptr;
        const T rad = T(p.pi_radius);
        // one position / velocity draw for element e = (pl, d) of this CTA
        auto put_x = [&](int pl, int d, T ux) {
            const int row = c.row0 + pl, g = int(c.fN.div(uint32_t(row))), n = row - g * N;
            const T lo = c.lo[d], hi = c.hi[d];
            T xv;
            if (warm_on && n < p.warm) {
                const T ctr = T(prev[d]);            // waypoint d % W, x- or y-block
                const T l = A::sub(ctr, rad) > lo ? A::sub(ctr, rad) : lo;   // std::max(lo, c - r)
                const T h = hi < A::add(ctr, rad) ? hi : A::add(ctr, rad);  // std::min(hi, c + r)
                xv = A::add(l, A::mul(ux, A::sub(h, l)));
            } else {
                xv = A::add(lo, A::mul(ux, A::sub(hi, lo)));
            }
            c.x[pl * D + d] = xv;
            c.pb[pl * D + d] = xv;
        };
        auto put_v = [&](int pl, int d, T uv) {
            const int row = c.row0 + pl, g = int(c.fN.div(uint32_t(row)));
            const T vmax = A::mul(c.hyp[g * 6 + 5], A::sub(c.hi[d], c.lo[d]));
            const T vlo = -vmax;
            c.v[pl * D + d] = A::add(vlo, A::mul(uv, A::sub(vmax, vlo)));
        };
        if (kLat || p.rng == kMt19937) {
            // The reference's sequential stream (mt19937.cuh), walked by warps
            // 0..3 (one per SM sub-partition; named barrier 3) through all 2RD
            // init words; only the words of this CTA's rows are tempered and
            // go straight into x / v.  The seeded state is already in place.
            const long long RD = (long long)R * D, x0 = (long long)c.row0 * D, x1 = (long long)row1 * D;
            const MtGroup grp = nthr >= 288 ? MtGroup{tid, 256, 3} : (nthr >= 160 ? MtGroup{tid, 128, 3} : MtGroup{tid, nthr, 0});
            MtState mt{mtbuf, 0, 0};
            bool pre_ok = false;
            const PreRec* const prr = (p.inl && p.in_pre >= 0) ? reinterpret_cast<const PreRec*>(jb + p.in_pre) : nullptr;
            const unsigned long long* const pre_w =
                prr ? reinterpret_cast<const unsigned long long*>(prr->words) + size_t(swarm) * size_t(2 * RD)
                    : p.pre_words + size_t(swarm) * size_t(2 * RD);
            if (pre_cand) {
                if (tid == 0) {
                    const int* const pre_f = prr ? reinterpret_cast<const int*>(prr->flag) : p.pre_flag;
                    c.m->pre_ok = pre_wait(pre_f + swarm, prr ? prr->seq : p.pre_seq) ? 1 : 0;
                }
                __syncthreads();
                pre_ok = c.m->pre_ok != 0;
                if (srv && c.crank == 0 && tid == 0) srv->t_wait = global_ns();
                if (!pre_ok) {              // not in time: seed and walk here after all (a job
                    // with a walk ready carries no seeded state: seed from the seed)
                    if (tid == 0) mt_seed_words(mtbuf + 312, seed);
                    __syncthreads();
                }
            }
            SEPSO_IMARK(2);
            if (pre_ok) {
                // this CTA's x / v words straight from HBM, the generator's
                // last pair where the step draws continue
                const int nx = int(x1 - x0);
                #pragma unroll 1
                for (int e = tid; e < nx; e += nthr) {
                    const int pl = int(c.fD.div(uint32_t(e))), d = e - pl * D;
                    const unsigned long long wx = __ldcg(pre_w + x0 + e), wv = __ldcg(pre_w + RD + x0 + e);
                    put_x(pl, d, unit_from_word<T>(mt_temper(wx)));     // stored untempered
                    put_v(pl, d, unit_from_word<T>(mt_temper(wv)));
                }
                const unsigned long long* pp = (prr ? reinterpret_cast<const unsigned long long*>(prr->pair) : p.pre_pair) +
                                               size_t(swarm) * kPrePairWords;
                #pragma unroll 1
                for (int i = tid; i < 624; i += nthr) mtbuf[i] = __ldcg(pp + i);
                if (tid == 0) { c.m->mt_cur = 0; c.m->mt_blocks = (long long)__ldcg(pp + 624); }
                SEPSO_IMARK(5);
            } else if (tid < grp.n) {
                mt_generate(mt, grp, x0, x1, [&](int e, unsigned long long word) {
                    const int pl = int(c.fD.div(uint32_t(e)));
                    put_x(pl, e - pl * D, unit_from_word<T>(word));
                });
                SEPSO_IMARK(3);
                mt_generate(mt, grp, RD + x0, RD + x1, [&](int e, unsigned long long word) {
                    const int pl = int(c.fD.div(uint32_t(e)));
                    put_v(pl, e - pl * D, unit_from_word<T>(word));
                });
                SEPSO_IMARK(4);
                // the rest of the init words, so that the step draws start at 2RD
                mt_generate(mt, grp, 2 * RD, 2 * RD, [&](int, unsigned long long) {});
                SEPSO_IMARK(5);
                if (tid == 0) { c.m->mt_cur = mt.cur; c.m->mt_blocks = mt.blocks; }
            } else if (p.mt_next && p.roots && c.crank == 0 && tid == grp.n + 32 && nthr > grp.n + 32) {
                // scene batches: the next frame's seeded generator state, off the
                // critical path (the walk above takes ~4x as long)
                const uint64_t next = splitmix64(splitmix64(p.roots[swarm] ^ p.tag_hash) + uint64_t(p.frame_index + 1));
                mt_seed_words(p.mt_next + size_t(swarm) * 312, next);
            } else if (PATH && sizeof(T) == 4 && c.crank == 0 && tid < grp.n + 32) {
                // rank 0's first idle warp runs the final record's code once on
                // dummy input while the generator walks the stream: after an
                // L2 flush that code would otherwise be fetched from DRAM on
                // the frame's critical path (its result is discarded)
                const int h = rec64_hits(c.vert64, c.ooff, c.O, reinterpret_cast<const float*>(c.tbx), c.W, c.S,
                                         tid - grp.n, 32);
                const double len = path_length64(c.tbx, c.W, c.S, 0.0, 0.0, 1.0, 1.0, tid - grp.n);
                if (h < 0 || len < 0.0) c.m->q64 = h;
            }
        } else {
            ElemWalk w(c.fD, tid, nthr, D);
            for (int e = tid; e < c.P * D; e += nthr, w.next()) {
                const uint64_t ix = uint64_t(c.row0 + w.pl) * uint64_t(D) + uint64_t(w.col);
                put_x(w.pl, w.col, unit_from_word<T>(philox_word(seed, ix)));
                put_v(w.pl, w.col, unit_from_word<T>(philox_word(seed, uint64_t(R) * D + ix)));
            }
        }
    }
    __syncthreads();
    SEPSO_IMARK(6);
    SEPSO_GMARK(8);
    if (srv && c.crank == 0 && tid == 0) srv->t_init = global_ns();

    // ------------------------------------------------------------ iterations
    if (p.cap < 1 && !srv) cluster_wait();
    // Best update fast path (FP32, G <= 32, tw <= 32): warp 0 keeps the bests
    // and the AT window in registers -- lane g group g's gbest value and Q,
    // lane i window slot i -- so the chain of the single-warp phase is a few
    // warp collectives instead of shared-memory round trips; spilled to Misc /
    // c.win when the loop ends.
    const bool b1fast = kLat || (sizeof(T) == 4 && G <= 32 && p.tw <= 32);
    float r_gbf = __int_as_float(0x7f800000), r_tbf = __int_as_float(0x7f800000);
    int r_gbq = 0, r_tbq = 0, r_wl = 0, r_wh = 0, r_cf = 0, r_cl = -1, r_s0 = 0;
    double r_win = 0.0;
    if (b1fast && warp == 0) {
        r_wl = c.m->win_len;
        if (lane < p.tw) r_win = c.win[lane];
        if (lane < G) {
            r_cf = c.gtab[2 * lane];
            r_cl = c.gtab[2 * lane + 1];
            r_s0 = r_cf * LGM + (lane - c.ctab[r_cf]);
        }
    }
    const double inv_tw = p.tw > 0 ? 1.0 / double(p.tw) : 0.0;
    int k = 1;
    for (; k <= p.cap; ++k) {
        const int buf = k & 1;
        SEPSO_MARK(0);
        if (wprof) wt0 = clock64();
        // fitness (geometry.hpp:262-267 / benchmarks.hpp:45-53)
        if (PATH) path_fitness_phase<T, RING>(p, c, prof, k, true);     // A3 thread also updates the pbest
        else bench_fitness_phase(problem, c);
        SEPSO_MARK(4);
        // pbest (runner.hpp:73-80) incl. the x -> pbest_x row copy; non-finite
        // detection (runner.hpp:56-61).  Same thread owns fit[pl] (A3 above).
        // mt19937: the last four warps walk the stream to this step's r1, r2, r3
        // (draw_step_randoms, swarm.hpp:59-70).  When they own no pbest rows and
        // no group partial they start right after the fitness barrier, outside
        // the pbest barrier.
        const bool gen_early = (kLat || (p.rng == kMt19937 && nthr >= 192)) && k < p.cap;
        const int gw0 = (nthr >> 5) - 4;
        const bool gen_first = gen_early && (kLat || (gw0 * 32 >= c.P && c.LG <= gw0));
        // helper warps below the generator (idle until the step: no partial,
        // no best update) take the draws' delivery -- tempering and storing
        // this CTA's 3P factors -- off the three generating warps
        // (throughput launches only: there a CTA delivers 3 x ~680 words per
        // step; the latency shape's 3 x 85 do not pay for the wider barrier)
        constexpr int kHelp = RING ? kGenHelpers : 0;
        const int hw0 = gw0 - kHelp;
        const int gn = (kHelp > 0 && hw0 >= c.LG && hw0 >= 1) ? 96 + 32 * kHelp : 96;
        if (gen_first && warp >= gw0) {
            // three of the four warps generate (SM sub-partitions 1-3): the
            // ALU-bound generator then never competes with warp 0's serial
            // partial / best-update chain on sub-partition 0
            long long* gprof = (kProfiling && p.prof != nullptr && swarm == 0 && c.crank == 0 && tid == (gw0 + 1) * 32) ? p.prof : nullptr;
            if (gprof) gprof[(k - 1) * kProfPhases + 12] = clock64();
            if (warp > gw0) {
                if (kHelp > 0 && gn > 96) mt_step_draws<97>(c, mtbuf, MtGroup{tid - (gw0 + 1) * 32, gn, 1}, k, row1);
                else mt_step_draws<96>(c, mtbuf, MtGroup{tid - (gw0 + 1) * 32, 96, 1}, k, row1);
            }
            if (gprof) gprof[(k - 1) * kProfPhases + 13] = clock64();
        } else {
        if (!PATH)                                   // path swarms: fused into A3 above
            for (int pl = tid; pl < c.P; pl += nthr) pbest_row(c, pl, c.fit[pl]);
        if (gen_first) asm volatile("bar.sync 2, %0;" ::"r"(gw0 * 32) : "memory");   // pbest done (not the generator)
        else __syncthreads();
        if (kHelp > 0 && gen_first && gn > 96 && warp >= hw0)
            mt_step_draws<97>(c, mtbuf, MtGroup{96 + tid - hw0 * 32, gn, 1}, k, row1);
        }
        SEPSO_MARK(5);
        if (tid == 0) mbar_expect(mbar0 + 8 * buf, xbytes);
        SEPSO_MARK(22);
        if (k == 1 && !srv) cluster_wait();    // every peer is running, its mbarriers initialised
        // per-CTA group partials: (pbest_f, row) lexicographic min, one warp per group
        for (int lg = warp; lg < c.LG; lg += nthr >> 5) {
            const int g = gfirst + lg;
            const int l0 = max(c.row0, g * N) - c.row0, l1 = min(row1, (g + 1) * N) - c.row0;
            T bf = A::inf();
            int br = INT_MAX;
#ifdef SEPSO_EXP_SCAN2
#pragma unroll 1
            for (int rep = 0; rep < 2; ++rep) {
            if (rep == 1 && lg == 0) SEPSO_MARK(23);
            bf = A::inf(); br = INT_MAX;
#endif
            #pragma unroll 1   // serial per-iteration path: compact code (I-cache)
            for (int pl = l0 + lane; pl < l1; pl += 32) {
                const T f = c.pbf[pl];
                if (f < bf) { bf = f; br = pl; }                    // lanes scan ascending
            }
#ifdef SEPSO_EXP_SCAN2
            }
            if (lg == 0) SEPSO_MARK(1);
#else
            if (lg == 0) SEPSO_MARK(23);
#endif
            if (sizeof(T) == 4) {
                const uint32_t key = order_key(float(bf));
                const uint32_t kmin = __reduce_min_sync(0xffffffffu, key);
                br = int(__reduce_min_sync(0xffffffffu, key == kmin ? uint32_t(br) : 0xffffffffu));
            } else {
                for (int off = 16; off; off >>= 1) {
                    const T of = __shfl_xor_sync(0xffffffffu, bf, off);
                    const int orow = __shfl_xor_sync(0xffffffffu, br, off);
                    if (of < bf || (of == bf && orow < br)) { bf = of; br = orow; }
                }
            }
            br = __shfl_sync(0xffffffffu, br, 0);
            if (lg == 0) SEPSO_MARK(19);
            // push (value, row, q) and the row itself into every peer's slot
            // (crank, lg) of buffer buf with st.async; each store completes its
            // bytes on the peer's mbarrier of this parity.  A group without a
            // finite best still sends a row so the byte count stays fixed.
            const int slot = c.crank * LGM + lg;
            Part pt;
            pt.f = br == INT_MAX ? double(A::inf()) : double(c.pbf[br]);
            pt.row = br == INT_MAX ? INT_MAX : br + c.row0;
            pt.q = br == INT_MAX ? 0 : c.pbq[br];
            const int brow = br == INT_MAX ? 0 : br;
            const uint32_t mb = mbar0 + 8 * buf;
            #pragma unroll 1   // serial per-iteration path: compact code (I-cache)
            for (int r = lane; r < c.C; r += 32) {
                const uint4 v = *reinterpret_cast<const uint4*>(&pt);
                st_async_v4(peer_addr(smem_addr(c.part + buf * c.C * LGM + slot), r), v, peer_addr(mb, r));
            }
            if (lg == 0) SEPSO_MARK(20);
            const uint32_t dst0 = smem_addr(c.px + size_t(buf * c.C * LGM + slot) * D);
            if ((D * int(sizeof(T))) % 16 == 0) {                         // 16-byte vectors
                const int V4 = (D * int(sizeof(T))) / 16;
                const uint4* src = reinterpret_cast<const uint4*>(c.pb + brow * D);
                #pragma unroll 1   // serial per-iteration path: compact code (I-cache)
                for (int t = lane; t < c.C * V4; t += 32) {
                    const int r = int(c.fV.div(uint32_t(t))), q4 = t - r * V4;
                    st_async_v4(peer_addr(dst0 + 16 * q4, r), src[q4], peer_addr(mb, r));
                }
            } else {                                                      // 4-byte words
                const int V1 = (D * int(sizeof(T))) / 4;
                const uint32_t* src = reinterpret_cast<const uint32_t*>(c.pb + brow * D);
                #pragma unroll 1   // serial per-iteration path: compact code (I-cache)
                for (int t = lane; t < c.C * V1; t += 32) {
                    const int r = int(c.fV.div(uint32_t(t))), q1 = t - r * V1;
                    st_async_b32(peer_addr(dst0 + 4 * q1, r), src[q1], peer_addr(mb, r));
                }
            }
        }
        SEPSO_MARK(21);
        if (tid < c.C)
            st_async_b32(peer_addr(smem_addr(c.allbad + buf * c.C + c.crank), tid), uint32_t(c.m->bad_row),
                         peer_addr(mbar0 + 8 * buf, tid));
        SEPSO_MARK(6);
        // otherwise the last four warps generate while the partials arrive and
        // warp 0 updates the bests; the factors are read after the barrier that
        // follows B1
        if (!kLat && gen_early && !gen_first && warp >= gw0) {
            long long* gprof = (kProfiling && p.prof != nullptr && swarm == 0 && c.crank == 0 && tid == gw0 * 32) ? p.prof : nullptr;
            if (gprof) gprof[(k - 1) * kProfPhases + 12] = clock64();
            mt_step_draws<128>(c, mtbuf, MtGroup{tid - gw0 * 32, 128, 1}, k, row1);
            if (gprof) gprof[(k - 1) * kProfPhases + 13] = clock64();
        }
        long long wt1 = 0;
        if (wprof) wt1 = clock64();
        if (warp == 0) mbar_wait(mbar0 + 8 * buf, uint32_t(((k - 1) >> 1) & 1));   // every CTA's partials
        if (wprof) {
            wprof[(size_t(k - 1) * 16 + c.crank) * 2] = wt1 - wt0;
            wprof[(size_t(k - 1) * 16 + c.crank) * 2 + 1] = clock64() - wt1;
        }
        SEPSO_MARK(7);

        // partials were pushed before the barrier: nothing to gather
        SEPSO_MARK(8);
        if (warp == 0 && b1fast) {
            Misc<T>* m = c.m;
            const int bad = int(__reduce_min_sync(0xffffffffu, lane < c.C ? uint32_t(c.allbad[buf * c.C + lane])
                                                                            : 0xffffffffu));
            SEPSO_MARK(15);
            if (bad != INT_MAX) {
                if (lane == 0) { m->status = 2; m->bad_min = bad; m->stop = 1; }
            } else {
                // gbest, lane g: the owning CTAs' partials in row order, strict
                // '<' vs the incumbent (runner.hpp:81-87).  Later CTAs of a
                // group start inside it, so its partial is their local group 0.
                const Part* parts = c.part + size_t(buf) * c.C * LGM;
                double bf = double(A::inf());
                int bslot = -1, bq = 0;
                #pragma unroll 1   // serial per-iteration path: compact code (I-cache)
                for (int cc = r_cf; cc <= r_cl; ++cc) {
                    const int slot = cc == r_cf ? r_s0 : cc * LGM;
                    const Part pt = parts[slot];
                    if (pt.f < bf) { bf = pt.f; bslot = slot; bq = pt.q; }
                }
                if (lane < G) {
                    int ch = -1;
                    if (float(bf) < r_gbf) { r_gbf = float(bf); r_gbq = bq; ch = bslot; }
                    c.chg[lane] = ch;
                }
                SEPSO_MARK(16);
                // tbest: (gbest_f, g) lexicographic min, strict '<' vs the
                // incumbent (runner.hpp:88-91): one REDUX on ordered keys, the
                // lowest lane holding the minimum
                const uint32_t key = lane < G ? order_key(r_gbf) : 0xffffffffu;
                const uint32_t kmin = __reduce_min_sync(0xffffffffu, key);
                const int tg = __ffs(__ballot_sync(0xffffffffu, key == kmin)) - 1;
                const float tv = __shfl_sync(0xffffffffu, r_gbf, tg);
                const int tq = __shfl_sync(0xffffffffu, r_gbq, tg);
                const bool tnew = tv < r_tbf;
                if (tnew) { r_tbf = tv; r_tbq = tq; }
                const double tb = double(r_tbf);
                SEPSO_MARK(17);
                // trace, window push + trim to tw (planner.hpp:179-180): lane
                // `at` takes the new value
                const int tw = p.tw;
                if (lane == 0) {
                    m->tsrc_slot = tnew ? tg : -1;
                    if (c.crank == 0) {
                        if (srv) put_chunk_d(p.out, 4 + D + (k - 1), tb, 0u, jseq);
                        else p.trace[size_t(swarm) * p.cap + (k - 1)] = tb;
                    }
                }
                if (tw > 0) {
                    int at = r_wh + r_wl;
                    if (r_wl == tw) at = r_wh;
                    else if (at >= tw) at -= tw;
                    if (lane == at) r_win = tb;
                    if (r_wl < tw) ++r_wl;
                    else if (++r_wh == tw) r_wh = 0;
                }
                SEPSO_MARK(18);
                // auto truncation (planner.hpp:181-187, 138-149): the exact
                // range pre-test, then the certified parallel estimate, then
                // -- only inside its error band -- the reference's sequential
                // sums in window order, oldest first
                if (p.auto_truncate && r_wl >= tw && r_tbq == 0) {
                    const double oldest = __shfl_sync(0xffffffffu, r_win, r_wh);
                    const double newest = __shfl_sync(0xffffffffu, r_win, r_wh == 0 ? tw - 1 : r_wh - 1);
                    if (!(fabs(newest - oldest) >= p.at_gap)) {
                        int dec = at_decide_regs(r_win, lane, tw, newest, inv_tw, ld.at_var_bound);
                        if (dec < 0) {
                            double mean = 0.0;
                            for (int i = 0; i < tw; ++i)
                                mean = __dadd_rn(mean, __shfl_sync(0xffffffffu, r_win, r_wh + i < tw ? r_wh + i : r_wh + i - tw));
                            mean = __ddiv_rn(mean, double(tw));
                            double var = 0.0;
                            for (int i = 0; i < tw; ++i) {
                                const double dv = __dsub_rn(__shfl_sync(0xffffffffu, r_win, r_wh + i < tw ? r_wh + i : r_wh + i - tw), mean);
                                var = __dadd_rn(var, __dmul_rn(dv, dv));
                            }
                            dec = var < ld.at_var_bound ? 1 : 0;
                        }
                        if (dec > 0 && lane == 0) { m->truncated = 1; m->stop = 1; }
                    }
                }
            }
            if (lane == 0) m->k_done = k;
            SEPSO_MARK(14);
        } else if (!kLat && warp == 0) {
            // gbest, one lane per group: scan the owning CTAs in row order,
            // strict '<' vs the incumbent (runner.hpp:81-87)
            Misc<T>* m = c.m;
            int bad = INT_MAX;
            for (int cc = lane; cc < c.C; cc += 32) bad = min(bad, c.allbad[buf * c.C + cc]);
            bad = int(__reduce_min_sync(0xffffffffu, uint32_t(bad)));
            SEPSO_MARK(15);
            if (bad != INT_MAX) {
                if (lane == 0) { m->status = 2; m->bad_min = bad; m->stop = 1; }
            } else {
                T tv = A::inf();
                int tg = INT_MAX;
                for (int g = lane; g < G; g += 32) {
                    const int cf = c.gtab[2 * g], cl = c.gtab[2 * g + 1];
                    double bf = double(A::inf());
                    int bslot = -1, bq = 0;
                    for (int cc = cf; cc <= cl; ++cc) {
                        const int slot = cc * LGM + (g - c.ctab[cc]);
                        const Part pt = c.part[buf * c.C * LGM + slot];
                        if (pt.f < bf) { bf = pt.f; bslot = slot; bq = pt.q; }
                    }
                    if (T(bf) < c.gbf[g]) { c.gbf[g] = T(bf); c.gbq[g] = bq; c.chg[g] = bslot; }
                    else c.chg[g] = -1;
                    if (c.gbf[g] < tv) { tv = c.gbf[g]; tg = g; }       // per-lane, g ascending
                }
                SEPSO_MARK(16);
                // tbest: (gbest_f, g) lexicographic min over groups, strict '<'
                // vs the incumbent (runner.hpp:88-91)
                if (sizeof(T) == 4) {          // ordered keys: two warp reductions
                    const uint32_t key = order_key(float(tv));
                    const uint32_t kmin = __reduce_min_sync(0xffffffffu, key);
                    tg = int(__reduce_min_sync(0xffffffffu, key == kmin ? uint32_t(tg) : 0xffffffffu));
                    tv = __shfl_sync(0xffffffffu, tv, __ffs(__ballot_sync(0xffffffffu, key == kmin)) - 1);
                } else {
                    for (int off = 16; off; off >>= 1) {
                        const T ov = __shfl_xor_sync(0xffffffffu, tv, off);
                        const int og = __shfl_xor_sync(0xffffffffu, tg, off);
                        if (ov < tv || (ov == tv && og < tg)) { tv = ov; tg = og; }
                    }
                }
                SEPSO_MARK(17);
                // tbest update, trace, window push + trim to tw (planner.hpp:179-180)
                const bool tnew = tv < m->tbf;
                const double tb = double(tnew ? tv : m->tbf);
                const int tbq = tnew ? c.gbq[tg] : m->tbq;
                const int wl0 = m->win_len, wh0 = m->win_head;
                int wl = wl0, wh = wh0;
                if (p.tw > 0) {
                    if (wl < p.tw) ++wl;
                    else if (++wh == p.tw) wh = 0;
                }
                __syncwarp();      // every lane has read m before lane 0 updates it
                if (lane == 0) {
                    if (tnew) { m->tbf = tv; m->tbq = tbq; m->tsrc_slot = tg; }
                    else m->tsrc_slot = -1;
                    if (c.crank == 0) {
                        if (srv) put_chunk_d(p.out, 4 + D + (k - 1), tb, 0u, jseq);
                        else p.trace[size_t(swarm) * p.cap + (k - 1)] = tb;
                    }
                    if (p.tw > 0) {
                        int at = wh0 + wl0;                       // slot of the new value
                        if (wl0 == p.tw) at = wh0;
                        else if (at >= p.tw) at -= p.tw;
                        c.win[at] = tb;
                    }
                    m->win_len = wl;
                    m->win_head = wh;
                }
                __syncwarp();
                SEPSO_MARK(18);
                // auto truncation (planner.hpp:181-187, 138-149) with Q(tbest)
                // tracked.  The exact pre-test (std >= range / sqrt(2 tw))
                // skips hopeless windows.  Otherwise the warp estimates the
                // statistic in parallel (tree sums) and decides whenever the
                // estimate clears the threshold by more than a rigorous bound
                // on its distance from the reference's sequential value; only
                // inside that band (|var - bound| ~ 1e-14 relative) does lane 0
                // redo the sums sequentially in window order, oldest first, as
                // the reference does.
                if (p.auto_truncate && wl >= p.tw && tbq == 0) {
                    const int tw = p.tw;
                    const double oldest = c.win[wh];
                    const double newest = c.win[wh == 0 ? tw - 1 : wh - 1];
                    if (!(fabs(newest - oldest) >= p.at_gap)) {
                        const int dec = at_decide_parallel(c.win, wh, tw, ld.at_var_bound, lane);
                        if (dec > 0 && lane == 0) { m->truncated = 1; m->stop = 1; }
                        if (dec < 0 && lane == 0) {
                            double mean = 0.0;
#pragma unroll 4
                            for (int i = 0; i < tw; ++i) {
                                const int at = wh + i < tw ? wh + i : wh + i - tw;
                                mean = __dadd_rn(mean, c.win[at]);
                            }
                            mean = __ddiv_rn(mean, double(tw));
                            double var = 0.0;
#pragma unroll 4
                            for (int i = 0; i < tw; ++i) {
                                const int at = wh + i < tw ? wh + i : wh + i - tw;
                                const double dv = __dsub_rn(c.win[at], mean);
                                var = __dadd_rn(var, __dmul_rn(dv, dv));
                            }
                            if (var < ld.at_var_bound) { m->truncated = 1; m->stop = 1; }
                        }
                    }
                }
            }
            if (lane == 0) m->k_done = k;
            SEPSO_MARK(14);
        } else if (!kLat && k < p.cap && p.rng == kMt19937 && !gen_early) {
            // small CTAs: warps 1.. walk the stream to this step's factors
            // while warp 0 updates the bests
            if (nthr >= 64) mt_step_draws<0>(c, mtbuf, MtGroup{tid - 32, nthr - 32, 1}, k, row1);
        } else if (!kLat && k < p.cap && p.rng == kPhilox) {
            // meanwhile: this step's draws (draw_step_randoms, swarm.hpp:59-70) --
            // they depend only on (seed, k, row), not on the bests
            const uint64_t base = 2ull * uint64_t(R) * uint64_t(D) + uint64_t(k - 1) * 3ull * uint64_t(R);
            for (int t = tid - 32; t < 3 * c.P; t += nthr - 32) {
                const int j = t >= 2 * c.P ? 2 : (t >= c.P ? 1 : 0), pl = t - j * c.P;
                const int row = c.row0 + pl, g = int(c.fN.div(uint32_t(row)));
                const T u = unit_from_word<T>(philox_word(seed, base + uint64_t(j) * R + row));
                c.coef[j * c.P + pl] = A::mul(c.hyp[g * 6 + j], u);   // a_j = c_j * r_j
            }
        }
        if (!kLat && nthr == 32 && k < p.cap && p.rng == kMt19937)     // single-warp CTA: draws after the bests
            mt_step_draws<0>(c, mtbuf, MtGroup{tid, 32, 0}, k, row1);
        if (!kLat && nthr == 32 && k < p.cap && p.rng == kPhilox) {
            const uint64_t base = 2ull * uint64_t(R) * uint64_t(D) + uint64_t(k - 1) * 3ull * uint64_t(R);
            for (int t = tid; t < 3 * c.P; t += 32) {
                const int j = t >= 2 * c.P ? 2 : (t >= c.P ? 1 : 0), pl = t - j * c.P;
                const int row = c.row0 + pl, g = int(c.fN.div(uint32_t(row)));
                const T u = unit_from_word<T>(philox_word(seed, base + uint64_t(j) * R + row));
                c.coef[j * c.P + pl] = A::mul(c.hyp[g * 6 + j], u);
            }
        }
        __syncthreads();
        SEPSO_MARK(9);
#ifdef SEPSO_CHECK
        // consistency build: every CTA logs its iteration decision (stop,
        // status, new-tbest group, the changed slots) for the host to compare
        // across the cluster -- the exchange has no closing barrier and relies
        // on identical decisions everywhere
        if (tid == 0 && p.dbg) {
            unsigned long long h = (unsigned long long)(c.m->stop & 1) | ((unsigned long long)(c.m->status & 3) << 1) |
                                   ((unsigned long long)(c.m->tsrc_slot + 1) << 3) | ((unsigned long long)k << 16);
            for (int g = 0; g < G && g < 8; ++g) h ^= (unsigned long long)(c.chg[g] + 1) << (24 + 5 * g);
            p.dbg[(size_t(swarm) * p.C + c.crank) * p.cap + (k - 1)] = (long long)h;
        }
#endif
        if (c.m->status) break;
        SEPSO_MARK(10);
        const int tg = c.m->tsrc_slot;                     // new tbest's group or -1
        const int tslot = tg >= 0 ? c.chg[tg] : -1;
        const T* pxb = c.px + size_t(buf) * c.C * LGM * D;  // this iteration's pushed rows
        if (c.m->stop || k == p.cap) {                       // no step after the last iteration
            if (tslot >= 0)
                #pragma unroll 1
                for (int d = tid; d < D; d += nthr) c.tbx[d] = pxb[tslot * D + d];
            __syncthreads();
            break;
        }
        // --------------------------------------------------- step k (swarm.hpp:138-174)
        // Improved group bests / the new tbest are read straight from the pushed
        // rows; the first local particle of each group (and particle 0 for tbest)
        // persists them for the next iteration.  Readers of gbx / tbx only read
        // when the entry did not change, so the in-loop writes cannot race.
        const T frac = T(double(k) / double(p.cap));               // inertia_at (swarm.hpp:81-84)
        auto step_rows = [&](auto width) {
            // WIDTH elements of one row per thread: the row's factors, weights and
            // best slots are loaded once, x / v / pbest as WIDTH-vectors
            constexpr int WIDTH = decltype(width)::value;
            using VW = typename std::conditional<WIDTH == 4, float4,
                       typename std::conditional<sizeof(T) == 4, float2, double2>::type>::type;
            for (int i = tid; i < (c.P * D) / WIDTH; i += nthr) {
                const int e = WIDTH * i, pl = int(c.fD.div(uint32_t(e))), d = e - pl * D;
                const int row = c.row0 + pl, g = int(c.fN.div(uint32_t(row)));
                const T* h = c.hyp + g * 6;
                const T wt = A::sub(h[3], A::mul(A::sub(h[3], h[4]), frac));
                const int gslot = c.chg[g];
                const T a1 = c.coef[pl], a2 = c.coef[c.P + pl], a3 = c.coef[2 * c.P + pl];
                VW xv = *reinterpret_cast<const VW*>(c.x + e);
                VW vv = *reinterpret_cast<const VW*>(c.v + e);
                const VW pv = *reinterpret_cast<const VW*>(c.pb + e);
                T* xs = reinterpret_cast<T*>(&xv);
                T* vs = reinterpret_cast<T*>(&vv);
                const T* ps = reinterpret_cast<const T*>(&pv);
#pragma unroll
                for (int j = 0; j < WIDTH; ++j) {
                    const int dd = d + j;
                    const T lo = c.lo[dd], hi = c.hi[dd];
                    const T vmax = A::mul(h[5], A::sub(hi, lo));
                    const T gv = gslot >= 0 ? pxb[gslot * D + dd] : c.gbx[g * D + dd];
                    const T tv = tslot >= 0 ? pxb[tslot * D + dd] : c.tbx[dd];
                    if (gslot >= 0 && row == max(g * N, c.row0)) c.gbx[g * D + dd] = gv;
                    if (tslot >= 0 && pl == 0) c.tbx[dd] = tv;
                    T nv = A::add(A::add(A::add(A::mul(wt, vs[j]), A::mul(a1, A::sub(ps[j], xs[j]))),
                                         A::mul(a2, A::sub(gv, xs[j]))),
                                  A::mul(a3, A::sub(tv, xs[j])));
                    nv = clampT(nv, T(-vmax), vmax);
                    vs[j] = nv;
                    xs[j] = clampT(A::add(xs[j], nv), lo, hi);
                }
                *reinterpret_cast<VW*>(c.v + e) = vv;
                *reinterpret_cast<VW*>(c.x + e) = xv;
            }
        };
        bool stepped = false;
        if constexpr (sizeof(T) == 4 && STEPW == 4) {
            if ((D & 3) == 0) { step_rows(std::integral_constant<int, 4>{}); stepped = true; }
        }
        if (stepped) {
        } else if ((D & 1) == 0) {
            step_rows(std::integral_constant<int, 2>{});
        } else {
            ElemWalk w(c.fD, tid, nthr, D);
            int g = int(c.fN.div(uint32_t(c.row0 + w.pl)));
            for (int e = tid; e < c.P * D; e += nthr, w.next()) {
                const int pl = w.pl, d = w.col;
                while ((g + 1) * N <= c.row0 + pl) ++g;
                const T* h = c.hyp + g * 6;
                const T wt = A::sub(h[3], A::mul(A::sub(h[3], h[4]), frac));
                const T lo = c.lo[d], hi = c.hi[d];
                const T vmax = A::mul(h[5], A::sub(hi, lo));
                const int gslot = c.chg[g];
                const T gv = gslot >= 0 ? pxb[gslot * D + d] : c.gbx[g * D + d];
                const T tv = tslot >= 0 ? pxb[tslot * D + d] : c.tbx[d];
                if (gslot >= 0 && c.row0 + pl == max(g * N, c.row0)) c.gbx[g * D + d] = gv;
                if (tslot >= 0 && pl == 0) c.tbx[d] = tv;
                const T xv = c.x[e];
                T nv = A::add(A::add(A::add(A::mul(wt, c.v[e]), A::mul(c.coef[pl], A::sub(c.pb[e], xv))),
                                     A::mul(c.coef[c.P + pl], A::sub(gv, xv))),
                              A::mul(c.coef[2 * c.P + pl], A::sub(tv, xv)));
                nv = clampT(nv, T(-vmax), vmax);
                c.v[e] = nv;
                c.x[e] = clampT(A::add(xv, nv), lo, hi);
            }
        }
        __syncthreads();
        SEPSO_MARK(11);
    }

    if (b1fast && warp == 0) {             // the fast path's registers -> Misc / c.win
        if (lane == 0) {
            c.m->tbf = r_tbf; c.m->tbq = r_tbq;
            c.m->win_len = r_wl; c.m->win_head = r_wh;
        }
        if (lane < p.tw) c.win[lane] = r_win;
        __syncwarp();
    }

    // ---------------------------------------------------------------- results
    SEPSO_GMARK(9);
    // FP32 engine, path problems: the record is the reference's evaluation of
    // the returned path -- Q of the best path counted on the caller's FP64
    // world with the reference's predicates (geometry.hpp:196-220), not on the
    // FP32-rounded world the swarm planned on; fitness = length + alpha Q^beta
    // below.  CTA 0, one (segment, edge) pair or first-waypoint containment
    // test per thread.
    if (srv && c.crank == 0 && tid == 0) srv->t_iter = global_ns();
    const bool rec64 = PATH && sizeof(T) == 4 && c.crank == 0 && c.m->status == 0;
    if (rec64 && warp != 0) {       // warps 1.. count Q while warp 0 sums the length below
        const int hits = rec64_hits(c.vert64, c.ooff, c.O, reinterpret_cast<const float*>(c.tbx), c.W, c.S, tid - 32,
                                    nthr - 32);
        if (hits) atomicAdd(&c.m->q64, hits);
    }
    if (srv && c.crank == 0 && tid == 0) { srv->t_loop = global_ns(); srv->t_mark[8] = (unsigned long long)clock64(); }
    // record length = path_length(best) in FP64 (planner.hpp:194): warp 0 of
    // rank 0 computes the S segment hypots in parallel, summed in path order
    double path_len = 0.0;
    if (PATH && c.crank == 0 && warp == 0) {
        // endpoints: the caller's FP64 values (the FP32 engine staged rounded ones)
        const double* e64 = rec64 ? c.vert64 + 2 * c.ooff[c.O] : nullptr;
        path_len = path_length64(c.tbx, c.W, c.S, e64 ? e64[0] : double(c.sx), e64 ? e64[1] : double(c.sy),
                                 e64 ? e64[2] : double(c.tx), e64 ? e64[3] : double(c.ty), lane);
    }
    SEPSO_SMARK(7);
    if (rec64) __syncthreads();
    if (c.crank == 0 && tid == 0) {
        const Misc<T>* m = c.m;
        SwarmOut o{};
        o.status = uint32_t(m->status);
        o.iterations = uint32_t(m->k_done);
        o.truncated = uint32_t(m->truncated);
        o.window_len = uint32_t(m->win_len);
        if (m->status == 2) {
            o.bad_g = uint32_t(m->bad_min / N);
            o.bad_n = uint32_t(m->bad_min % N);
            o.bad_k = uint32_t(m->k_done);
        } else if (rec64) {
            o.q = uint32_t(m->q64);
            o.length = path_len;
            o.fitness = __dadd_rn(path_len, penalty(p.alpha, p.beta, p.beta_int, m->q64));   // geometry.hpp:234-241
        } else {
            o.fitness = double(m->tbf);
            o.q = uint32_t(m->tbq);
            if (PATH) o.length = path_len;
        }
        if (srv) {
            put_chunk(p.out, 0, o.iterations, o.q, o.status, jseq);
            put_chunk_d(p.out, 1, o.fitness, o.truncated, jseq);
            put_chunk_d(p.out, 2, o.length, o.window_len, jseq);
            put_chunk(p.out, 3, o.bad_g, o.bad_n, o.bad_k, jseq);
        } else {
            p.out[swarm] = o;
        }
    }
    if (c.crank == 0) {
        if (srv)
            #pragma unroll 1
            for (int d = tid; d < D; d += nthr) put_chunk_d(p.out, 4 + d, double(c.tbx[d]), 0u, jseq);
        else
            #pragma unroll 1
            for (int d = tid; d < D; d += nthr) p.best_x[size_t(swarm) * D + d] = double(c.tbx[d]);
        if (p.carry && !srv) {      // (the resident planner's host keeps the window from the trace)
            #pragma unroll 1
            for (int i = tid; i < c.m->win_len; i += nthr)
                p.win_vals[size_t(swarm) * p.tw + i] = c.win[(c.m->win_head + i) % p.tw];
            if (tid == 0) p.win_len[swarm] = c.m->win_len;
        }
    }
    // scene batches: advance this swarm's world record for the next frame
    // (simenv.hpp:155-184); every CTA staged it long ago.  Rank 1 does it
    // while rank 0 writes the record.
    if (PATH && p.step_dt != 0.0 && c.crank == (c.C > 1 ? 1 : 0))
        #pragma unroll 1
        for (int t = tid - 2; t < c.O; t += nthr)
            step_world_part(const_cast<unsigned char*>(p.worlds) + size_t(swarm) * size_t(p.world_stride),
                            p.off_offsets, p.off_verts, p.off_vel, p.step_dt, t);
    SEPSO_GMARK(10);
    SEPSO_GMARK(11);
    if (!srv) break;
    // resident planner: rank 0's record is complete (its threads stored it)
    // before thread 0 publishes the job as done
    if (c.crank == 0) {
        __syncthreads();
        if (tid == 0) {
            srv->t_done = global_ns();
            srv->c_done = clock64();
            __threadfence_system();
            srv->done_seq = jseq;
        }
    }
    dry = SERVER && SEPSO_DRY;
    }   // jobs
    if (srv && c.crank == 0 && tid == 0) {
        __threadfence_system();
        srv->alive = 0;
    }
    // No closing cluster barrier: a CTA only ever reads its own shared memory,
    // and every st.async into it completed before its last best update.
}

// ------------------------------------------------------------ world stepping
// simenv.hpp:139-149
__device__ __forceinline__ double reflect_axis_dev(double lo, double hi, double limit, double& v) {
    if (lo <= 0.0) { v = -v; return __dmul_rn(-2.0, lo); }
    if (hi >= limit) { v = -v; return __dmul_rn(-2.0, __dsub_rn(hi, limit)); }
    return 0.0;
}

// simenv.hpp:155-184 for one world record, one part per thread: t = -2 the
// start, t = -1 the target, t >= 0 obstacle t (obstacles move independently;
// each part keeps the reference's operation order)
static __device__ void step_world_part(unsigned char* rec, int off_offsets, int off_verts, int off_vel, double dt,
                                       int t) {
    WorldHeader* h = reinterpret_cast<WorldHeader*>(rec);
    if (t < 0) {
        double& px = t == -2 ? h->sx : h->tx;
        double& py = t == -2 ? h->sy : h->ty;
        double& vx = t == -2 ? h->svx : h->tvx;
        double& vy = t == -2 ? h->svy : h->tvy;
        px = __dadd_rn(px, __dmul_rn(vx, dt));
        py = __dadd_rn(py, __dmul_rn(vy, dt));
        px = __dadd_rn(px, reflect_axis_dev(px, px, h->width, vx));
        py = __dadd_rn(py, reflect_axis_dev(py, py, h->height, vy));
        return;
    }
    const uint32_t* off = reinterpret_cast<const uint32_t*>(rec + off_offsets);
    double* vv = reinterpret_cast<double*>(rec + off_verts);
    double* vel = reinterpret_cast<double*>(rec + off_vel);
    double& ovx = vel[2 * t];
    double& ovy = vel[2 * t + 1];
    if (ovx == 0.0 && ovy == 0.0) return;
    const uint32_t v0 = off[t], v1 = off[t + 1];
    for (uint32_t i = v0; i < v1; ++i) {
        vv[2 * i] = __dadd_rn(vv[2 * i], __dmul_rn(ovx, dt));
        vv[2 * i + 1] = __dadd_rn(vv[2 * i + 1], __dmul_rn(ovy, dt));
    }
    double bx0 = vv[2 * v0], by0 = vv[2 * v0 + 1], bx1 = bx0, by1 = by0;
    for (uint32_t i = v0; i < v1; ++i) {
        bx0 = smin(bx0, vv[2 * i]); by0 = smin(by0, vv[2 * i + 1]);
        bx1 = smax(bx1, vv[2 * i]); by1 = smax(by1, vv[2 * i + 1]);
    }
    const double sx = reflect_axis_dev(bx0, bx1, h->width, ovx);
    const double sy = reflect_axis_dev(by0, by1, h->height, ovy);
    if (sx != 0.0 || sy != 0.0)
        for (uint32_t i = v0; i < v1; ++i) {
            vv[2 * i] = __dadd_rn(vv[2 * i], sx);
            vv[2 * i + 1] = __dadd_rn(vv[2 * i + 1], sy);
        }
}

// ------------------------------------------------------------------ launcher
constexpr int kMaxDevices = 64;

template <class T, bool PATH, bool RING, int MAXT = 1024, bool SERVER = false, bool FAST = false>
static int launch_t(const SwarmParams& p, const ParamPayload* pl, int problem, cudaStream_t st,
                    size_t* smem_out) {
    const SmemLayout L = smem_layout(p, sizeof(T), PATH);
    if (smem_out) *smem_out = L.total;
    auto kern = swarm_kernel<T, PATH, RING, MAXT, SERVER, FAST>;
    cudaError_t e = cudaSuccess;
    // attributes are sticky per function AND per device: cache them per ordinal
    static thread_local size_t smem_set[kMaxDevices] = {};
    static thread_local bool nonportable[kMaxDevices] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const bool cached = dev >= 0 && dev < kMaxDevices;
    if (!cached || L.total > smem_set[dev]) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
        if (e != cudaSuccess) return int(e);
        if (cached) smem_set[dev] = L.total;
    }
    if (p.C > 8 && (!cached || !nonportable[dev])) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return int(e);
        if (cached) nonportable[dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(p.n_swarms * p.C));
    cfg.blockDim = dim3(unsigned(p.nthreads));
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = unsigned(p.C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const ParamPayload empty{};
    LaunchDerived ld{};
    ld.lay = L;
    {
        const int R = p.G * p.N, Dv = p.D, Sv = p.D / 2 + 1;
        uint32_t xb = 0;                     // each CTA's group partials (16 B) + their rows, + 4 B each
        for (int cc = 0; cc < p.C; ++cc) {
            const int r0 = cc * p.rows_per_cta, r1 = std::min(R, r0 + p.rows_per_cta);
            if (r1 > r0) xb += uint32_t(((r1 - 1) / p.N - r0 / p.N + 1) * (16 + Dv * int(sizeof(T))));
            xb += 4;
        }
        ld.xbytes = xb;
        ld.at_var_bound = at_var_bound(p.delta, p.tw);
        const int divs[4] = {Sv, Dv, p.N, row_units<T>(Dv)};
        for (int i = 0; i < 4; ++i) {
            FastDiv f;
            f.init(uint32_t(divs[i]));
            ld.dmul[i] = f.mul;
            ld.dshr[i] = f.shr;
        }
    }
    e = cudaLaunchKernelEx(&cfg, kern, p, pl ? *pl : empty, ld, problem);
    return int(e);
}

} // namespace sepso
