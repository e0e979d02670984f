// stage_kernels.cu -- HBM-resident stage kernels (see stage_kernels.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "mt19937.cuh"
#include "mt_jump.hpp"
#include "stage_kernels.cuh"
#include "swarm_device.cuh"

namespace sepso {

struct CandHdr {        // one device's population-best candidate (runner.hpp:88-91)
    double f;
    int q;
    int g;
    int bad;            // first non-finite global row on that device (INT_MAX: none)
    int pad;
};

size_t cand_bytes(bool fp64, int D) {
    return (sizeof(CandHdr) + size_t(D) * (fp64 ? 8 : 4) + 15) & ~size_t(15);
}

static inline unsigned grid_for(long long work, int block) {
    long long g = (work + block - 1) / block;
    if (g > 148LL * 32) g = 148LL * 32;
    return unsigned(g < 1 ? 1 : g);
}

// word i of the stream: Philox by index, or a pre-generated mt19937_64 window
// (stored untempered by k_mt_fill; tempered here, in parallel)
__device__ __forceinline__ uint64_t stream_word(uint64_t seed, uint64_t i, const unsigned long long* words,
                                                long long base) {
    return words ? mt_temper(words[(long long)i - base]) : philox_word(seed, i);
}

// Advance a persisted mt19937_64 generator (one CTA of 256 threads) and write
// words [from, upto), untempered, to out[w - from]; words before `from` are skipped.
__global__ void __launch_bounds__(256) k_mt_fill(MtPersist* g, unsigned long long seed, int reseed,
                                                 long long from, long long upto,
                                                 unsigned long long* out) {
    __shared__ unsigned long long buf[kMtStateWords];
    MtState s{buf, 0, 0};
    const MtGroup grp{int(threadIdx.x), int(blockDim.x), 0};
    if (reseed) {
        mt_seed(s, grp, seed);
    } else {
        for (int i = threadIdx.x; i < 624; i += blockDim.x) buf[i] = g->st[i];   // pair 0
        s.blocks = g->blocks;
        __syncthreads();
    }
    const long long f0 = from < 0 ? 0 : from;
    mt_generate<0, true>(s, grp, f0, upto, [&](int rel, unsigned long long word) {   // untempered
        if (out) out[(f0 - from) + rel] = word;
    });
    for (int i = threadIdx.x; i < 624; i += blockDim.x) g->st[i] = buf[s.cur * 624 + i];
    if (threadIdx.x == 0) g->blocks = s.blocks;
}

int stage_mt_fill(MtPersist* g, unsigned long long seed, bool reseed, long long from, long long upto,
                  unsigned long long* out, void* stream) {
    // four warps compute each pass, four more store its (untempered) words
    k_mt_fill<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(g, seed, reseed ? 1 : 0, from, upto, out);
    return int(cudaGetLastError());
}

// ------------------------------------------------------- parallel stream fill
// A long fill [0, upto) in 2^levels segments of Q words generated in parallel,
// each from its start state s_{mQ} = g(A) s_0 (mt_jump.cpp): the states come
// from a doubling ladder of jumps, level j taking states 0 .. 2^j - 1 to
// 2^j .. 2^(j+1) - 1 with g = x^(Q 2^j) mod phi.  A state is a raw 312-word
// window (slot 1 of an MtState pair).

__global__ void k_mt_seed_state(unsigned long long* st, unsigned long long seed) {
    if (threadIdx.x == 0) mt_seed_words(st, seed);
}

// s_dst = XOR over g's terms i in this CTA's share of the window x[i .. i+311]
// of s_src (split CTAs per jump); dst is zeroed by the host and combined with
// atomicXor.  g arrives as the sorted list of its exponents (idx, nidx terms):
// the bit walk is the same for every lane, so it is done once on the host, and
// a term costs a lane one shared-memory load and one 64-bit XOR.
constexpr int kJumpTermsPerCta = 2560;      // >= ceil(kMtDegree / 8): split >= 8
__global__ void __launch_bounds__(1024) k_mt_jump(unsigned long long* states, int n_src, int split,
                                                  const unsigned short* __restrict__ idx, int nidx) {
    extern __shared__ __align__(16) unsigned long long jsm[];
    unsigned long long* buf = jsm;                      // generator (4 x 312)
    unsigned long long* X = jsm + kMtStateWords;        // x[0 .. i1 + 311]
    unsigned short* I = reinterpret_cast<unsigned short*>(X + kMtDegree + 312);   // this CTA's terms
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int m = blockIdx.x / split, part = blockIdx.x % split, chunk = (nidx + split - 1) / split;
    const int j0 = min(nidx, part * chunk), j1 = min(nidx, j0 + chunk), n = j1 - j0;
    const unsigned long long* src = states + size_t(m) * 312;
    unsigned long long* dst = states + size_t(m + n_src) * 312;
    for (int k = tid; k < 312; k += nthr) {
        const unsigned long long w = src[k];
        buf[312 + k] = w;
        X[k] = w;
    }
    for (int j = tid; j < n; j += nthr) I[j] = idx[j0 + j];
    const int i1 = n > 0 ? int(idx[j1 - 1]) + 1 : 0;    // words x[312 ..] this share reads
    __syncthreads();
    MtState s{buf, 0, 0};
    mt_generate<0, true>(s, MtGroup{tid, nthr, 0}, 0, i1,
                         [&](int rel, unsigned long long word) { X[312 + rel] = word; });
    __syncthreads();
    const int k = tid % 312, sub = tid / 312;
    if (sub < 3) {
        const int c3 = (n + 2) / 3, a = min(n, sub * c3), b = min(n, a + c3);
        unsigned long long a0 = 0, a1 = 0;
        int j = a;
#pragma unroll 4
        for (; j + 1 < b; j += 2) {
            a0 ^= X[I[j] + k];
            a1 ^= X[I[j + 1] + k];
        }
        if (j < b) a0 ^= X[I[j] + k];
        buf[tid] = a0 ^ a1;                             // generator buffer is free now
    }
    __syncthreads();
    if (tid < 312) atomicXor(dst + tid, buf[tid] ^ buf[312 + tid] ^ buf[624 + tid]);
}

// segment m: words [mQ, min(upto, (m+1)Q)), untempered, from state m; the
// segment holding the end leaves the generator in g as k_mt_fill would
__global__ void __launch_bounds__(256) k_mt_fill_seg(const unsigned long long* states, long long Q, long long upto,
                                                     unsigned long long* out, MtPersist* g) {
    __shared__ __align__(128) unsigned long long buf[kMtStateWords];
    const long long start = (long long)blockIdx.x * Q;
    if (start >= upto) return;
    const long long len = upto - start < Q ? upto - start : Q;
    for (int k = threadIdx.x; k < 312; k += blockDim.x) buf[312 + k] = states[size_t(blockIdx.x) * 312 + k];
    __syncthreads();
    MtState s{buf, 0, 0};
    mt_generate<0, true>(s, MtGroup{int(threadIdx.x), int(blockDim.x), 0}, 0, len,
                         [&](int rel, unsigned long long word) { out[start + rel] = word; });
    if (start + len == upto) {
        for (int i = threadIdx.x; i < 624; i += blockDim.x) g->st[i] = buf[s.cur * 624 + i];
        if (threadIdx.x == 0) g->blocks = s.blocks + start / 312;
    }
}

size_t mt_jump_smem_bytes() { return size_t(kMtStateWords + 312 + kMtDegree) * 8 + kJumpTermsPerCta * 2; }

int stage_mt_fill_parallel(MtPersist* g, unsigned long long seed, long long upto, unsigned long long* out,
                           unsigned long long* states, const unsigned short* terms, const int* nterms, int levels,
                           long long Q, void* stream) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    static thread_local unsigned attr = 0;          // function attributes are per device: one bit each
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 32 || !(attr >> dev & 1u)) {
        const cudaError_t e = cudaFuncSetAttribute(k_mt_jump, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   int(mt_jump_smem_bytes()));
        if (e != cudaSuccess) return int(e);
        if (dev < 32) attr |= 1u << dev;
    }
    k_mt_seed_state<<<1, 32, 0, st>>>(states, seed);
    for (int j = 0; j < levels; ++j) {
        const int n = 1 << j;
        cudaError_t e = cudaMemsetAsync(states + size_t(n) * 312, 0, size_t(n) * 312 * 8, st);
        if (e != cudaSuccess) return int(e);
        const int split = std::max(8, std::min(32, 256 / n));      // fill the GPU at the narrow levels
        k_mt_jump<<<n * split, 1024, mt_jump_smem_bytes(), st>>>(states, n, split, terms + size_t(j) * kMtDegree,
                                                                 nterms[j]);
    }
    k_mt_fill_seg<<<1u << levels, 256, 0, st>>>(states, Q, upto, out, g);
    return int(cudaGetLastError());
}

// --------------------------------------------------------------------- init
// swarm.hpp:94-132 / planner.hpp:77-133 (draws indexed by global row)
template <class T>
__global__ void k_init(StageShape s, const double* __restrict__ hypers, const T* __restrict__ lo,
                       const T* __restrict__ hi, uint64_t seed, uint64_t first,
                       const double* __restrict__ prev, int warm, double pi_radius, T* x, T* v,
                       T* pb, const unsigned long long* words, long long wbase, FastDiv fD, FastDiv fN,
                       bool wide) {
    using A = Ar<T>;
    const long long total = (long long)s.rows * s.D;
    const int R = s.G * s.N;
    const T rad = T(pi_radius);
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        // (fast 32-bit division while rows * D < 2^31 -- the 64-bit one made
        // the kernel issue-bound; `wide` arrays beyond that take the 64-bit one)
        const int rl = wide ? int(e / s.D) : int(fD.div(uint32_t(e))), d = int(e - (long long)rl * s.D);
        const int row = s.row_begin + rl, g = int(fN.div(uint32_t(row))), n = row - g * s.N;
        const uint64_t ix = first + uint64_t(row) * uint64_t(s.D) + uint64_t(d);
        const T ux = unit_from_word<T>(stream_word(seed, ix, words, wbase));
        const T l0 = lo[d], h0 = hi[d];
        T xv;
        if (prev != nullptr && n < warm) {
            const T ctr = T(prev[d]);
            const T l = A::sub(ctr, rad) > l0 ? A::sub(ctr, rad) : l0;
            const T h = h0 < A::add(ctr, rad) ? h0 : A::add(ctr, rad);
            xv = A::add(l, A::mul(ux, A::sub(h, l)));
        } else {
            xv = A::add(l0, A::mul(ux, A::sub(h0, l0)));
        }
        const T uv = unit_from_word<T>(stream_word(seed, uint64_t(R) * s.D + ix, words, wbase));
        const T vmax = A::mul(T(hypers[g * 6 + 5]), A::sub(h0, l0));
        const T vlo = -vmax;
        x[e] = xv;
        pb[e] = xv;
        v[e] = A::add(vlo, A::mul(uv, A::sub(vmax, vlo)));
    }
}

int stage_init(bool fp64, const StageShape& s, const double* hypers, const void* lo,
               const void* hi, uint64_t seed, uint64_t first, const double* prev, int warm,
               double pi_radius, void* x, void* v, void* pb, void* stream,
               const unsigned long long* words, long long wbase) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const bool wide = (long long)s.rows * s.D >= (1ll << 31);     // beyond FastDiv's range
    const unsigned grid = grid_for((long long)s.rows * s.D, 256);
    FastDiv fD, fN;
    fD.init(uint32_t(s.D));
    fN.init(uint32_t(s.N));
    if (fp64)
        k_init<double><<<grid, 256, 0, st>>>(s, hypers, (const double*)lo, (const double*)hi, seed,
                                              first, prev, warm, pi_radius, (double*)x, (double*)v,
                                              (double*)pb, words, wbase, fD, fN, wide);
    else
        k_init<float><<<grid, 256, 0, st>>>(s, hypers, (const float*)lo, (const float*)hi, seed,
                                             first, prev, warm, pi_radius, (float*)x, (float*)v,
                                             (float*)pb, words, wbase, fD, fN, wide);
    return int(cudaGetLastError());
}

// --------------------------------------------------------------------- step
// K1, the fused update (swarm.hpp:138-174).  One CTA per tile of TR rows: the
// tile's 3*TR Philox draws (draw_step_randoms order, swarm.hpp:59-70) go to
// shared memory, then every element is read once and written once:
// 20 B/element in FP32 (x, v, pbest in; x, v out).  VEC = 4 uses 16-byte
// vector accesses when D % 4 == 0.
// imp != nullptr (run_staged): the pbest row copy of this iteration's
// improved rows (runner.hpp:73-80) was deferred to here -- for a row with
// imp[row] set, pbest_x IS the current x, so the step takes it from x and
// writes it to pb (x, v in; x, v, pb out: 20 B/element, and the separate copy
// kernel's 8 B/element re-read and write are gone).
constexpr int kStepRows = 32;

template <class T, int VEC>
__global__ void __launch_bounds__(256) k_step(StageShape s, const double* __restrict__ hypers,
                                              const T* __restrict__ lo, const T* __restrict__ hi,
                                              T* __restrict__ x, T* __restrict__ v,
                                              T* __restrict__ pb, const T* __restrict__ gbx,
                                              const T* __restrict__ tbx, uint64_t seed,
                                              uint64_t first_draw, int k, int total,
                                              const IterState* gate,
                                              const unsigned long long* words, long long wbase,
                                              const unsigned char* __restrict__ imp) {
    using A = Ar<T>;
    if (gate != nullptr && gate->stop) return;
    __shared__ T coef[3 * kStepRows];
    __shared__ unsigned char fl[kStepRows];
    __shared__ T hw[64 * 3];   // per group: omega_k, vmax scale (v_limit), spare
    const int R = s.G * s.N, D = s.D;
    const int r0 = blockIdx.x * kStepRows;
    const int nr = min(kStepRows, s.rows - r0);
    if (nr <= 0) return;
    const T frac = T(double(k) / double(total));          // inertia_at (swarm.hpp:81-84)
    const int g_lo = (s.row_begin + r0) / s.N, g_hi = (s.row_begin + r0 + nr - 1) / s.N;
    for (int t = threadIdx.x; t <= g_hi - g_lo; t += blockDim.x) {
        const double* h = hypers + (g_lo + t) * 6;
        hw[t * 3 + 0] = A::sub(T(h[3]), A::mul(A::sub(T(h[3]), T(h[4])), frac));
        hw[t * 3 + 1] = T(h[5]);
    }
    for (int t = threadIdx.x; t < 3 * nr; t += blockDim.x) {
        const int j = t / nr, rl = t - j * nr;
        const int row = s.row_begin + r0 + rl, g = row / s.N;
        const T u = unit_from_word<T>(stream_word(seed, first_draw + uint64_t(j) * R + row, words, wbase));
        coef[j * kStepRows + rl] = A::mul(T(hypers[g * 6 + j]), u);
    }
    for (int t = threadIdx.x; t < nr; t += blockDim.x) fl[t] = imp != nullptr ? imp[r0 + t] : 0;
    __syncthreads();
    const int DV = D / VEC;
    for (int e = threadIdx.x; e < nr * DV; e += blockDim.x) {
        const int rl = e / DV, dv = e - rl * DV;
        const int row = s.row_begin + r0 + rl, g = row / s.N;
        const T w = hw[(g - g_lo) * 3], vl = hw[(g - g_lo) * 3 + 1];
        const T a1 = coef[rl], a2 = coef[kStepRows + rl], a3 = coef[2 * kStepRows + rl];
        const size_t base = size_t(r0 + rl) * D + size_t(dv) * VEC;
        const bool im = fl[rl] != 0;
        T xs[VEC], vs[VEC], ps[VEC], gs[VEC], ts[VEC], ls[VEC], hs[VEC];
        if constexpr (VEC == 4 && sizeof(T) == 4) {
            *reinterpret_cast<float4*>(xs) = *reinterpret_cast<const float4*>(x + base);
            *reinterpret_cast<float4*>(vs) = *reinterpret_cast<const float4*>(v + base);
            if (im) *reinterpret_cast<float4*>(ps) = *reinterpret_cast<const float4*>(xs);
            else *reinterpret_cast<float4*>(ps) = __ldcs(reinterpret_cast<const float4*>(pb + base));
            *reinterpret_cast<float4*>(gs) = *reinterpret_cast<const float4*>(gbx + size_t(g) * D + dv * 4);
            *reinterpret_cast<float4*>(ts) = *reinterpret_cast<const float4*>(tbx + dv * 4);
            *reinterpret_cast<float4*>(ls) = *reinterpret_cast<const float4*>(lo + dv * 4);
            *reinterpret_cast<float4*>(hs) = *reinterpret_cast<const float4*>(hi + dv * 4);
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                xs[i] = x[base + i]; vs[i] = v[base + i]; ps[i] = im ? xs[i] : pb[base + i];
                gs[i] = gbx[size_t(g) * D + dv * VEC + i]; ts[i] = tbx[dv * VEC + i];
                ls[i] = lo[dv * VEC + i]; hs[i] = hi[dv * VEC + i];
            }
        }
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
            const T vmax = A::mul(vl, A::sub(hs[i], ls[i]));
            const T xv = xs[i];
            T nv = A::add(A::add(A::add(A::mul(w, vs[i]), A::mul(a1, A::sub(ps[i], xv))),
                                 A::mul(a2, A::sub(gs[i], xv))),
                          A::mul(a3, A::sub(ts[i], xv)));
            nv = clampT(nv, T(-vmax), vmax);
            vs[i] = nv;
            xs[i] = clampT(A::add(xv, nv), ls[i], hs[i]);
        }
        if constexpr (VEC == 4 && sizeof(T) == 4) {
            *reinterpret_cast<float4*>(x + base) = *reinterpret_cast<const float4*>(xs);
            *reinterpret_cast<float4*>(v + base) = *reinterpret_cast<const float4*>(vs);
            if (im) *reinterpret_cast<float4*>(pb + base) = *reinterpret_cast<const float4*>(ps);
        } else {
#pragma unroll
            for (int i = 0; i < VEC; ++i) {
                x[base + i] = xs[i];
                v[base + i] = vs[i];
                if (im) pb[base + i] = ps[i];
            }
        }
    }
}

int stage_step(bool fp64, const StageShape& s, const double* hypers, const void* lo,
               const void* hi, void* x, void* v, void* pb, const void* gbx,
               const void* tbx, uint64_t seed, uint64_t first_draw, int k, int total,
               const IterState* gate, void* stream, const unsigned long long* words,
               long long wbase, const unsigned char* imp) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = unsigned((s.rows + kStepRows - 1) / kStepRows);
    if (grid == 0) return 0;
    if (fp64)
        k_step<double, 1><<<grid, 256, 0, st>>>(s, hypers, (const double*)lo, (const double*)hi,
                                                (double*)x, (double*)v, (double*)pb,
                                                (const double*)gbx, (const double*)tbx, seed,
                                                first_draw, k, total, gate, words, wbase, imp);
    else if (s.D % 4 == 0)
        k_step<float, 4><<<grid, 256, 0, st>>>(s, hypers, (const float*)lo, (const float*)hi,
                                               (float*)x, (float*)v, (float*)pb,
                                               (const float*)gbx, (const float*)tbx, seed,
                                               first_draw, k, total, gate, words, wbase, imp);
    else
        k_step<float, 1><<<grid, 256, 0, st>>>(s, hypers, (const float*)lo, (const float*)hi,
                                               (float*)x, (float*)v, (float*)pb,
                                               (const float*)gbx, (const float*)tbx, seed,
                                               first_draw, k, total, gate, words, wbase, imp);
    return int(cudaGetLastError());
}

// ---------------------------------------------------------------- path eval
// K2 standalone: one CTA per tile of rows, world staged in shared memory, the
// same cull + compaction + filtered-predicate machinery as the fused kernel.
struct EvalSmem {
    size_t misc, lo, hi, obb, ooff, ofl, vert, edge, seglen, q, list, grid, gidx, total;
};
constexpr int kGridDim = 32;   // wide worlds: kGridDim^2 cells over the map

SEPSO_LHD EvalSmem eval_smem(int rows_tile, int D, int max_obs, int max_verts, int entry_cap,
                          size_t tsz, bool edges = true) {
    EvalSmem L{};
    size_t o = 0;
    auto take = [&](size_t b) { const size_t at = o; o = sm_align(o + b); return at; };
    const int S = D / 2 + 1;
    L.misc = take(256);
    L.lo = take(size_t(D) * tsz);
    L.hi = take(size_t(D) * tsz);
    L.obb = take(size_t(max_obs) * 4 * tsz);
    L.ooff = take(size_t(max_obs + 1) * 4);
    L.ofl = take(size_t(max_obs) * 4);
    L.vert = take(size_t(max_verts) * 2 * tsz);
    L.edge = take(edges ? size_t(max_verts) * 4 * tsz : 0);
    L.seglen = take(size_t(rows_tile) * S * tsz);
    L.q = take(size_t(rows_tile) * 4);
    L.list = take(size_t(entry_cap) * 4);
    L.grid = take(edges || entry_cap ? size_t(kGridDim * kGridDim + 1) * 4 : 0);
    L.gidx = take(edges || entry_cap ? size_t(max_obs) * 4 : 0);
    L.total = o;
    return L;
}

template <class T>
__global__ void __launch_bounds__(256) k_eval_path(const unsigned char* __restrict__ world,
                                                   SwarmParams pp, int rows, int rows_tile,
                                                   const T* x, T* fit, int* qout,
                                                   const IterState* gate) {
    if (gate != nullptr && gate->stop) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const EvalSmem L = eval_smem(rows_tile, pp.D, pp.max_obs, pp.max_verts, pp.entry_cap, sizeof(T));
    const int r0 = blockIdx.x * rows_tile;
    Ctx<T> c{};
    c.D = pp.D; c.W = pp.D / 2; c.S = c.W + 1;
    c.fS.init(uint32_t(c.S));
    c.fD.init(uint32_t(c.D));
    c.fN.init(1u);
    c.P = min(rows_tile, rows - r0);
    if (c.P <= 0) return;
    c.x = const_cast<T*>(x) + size_t(r0) * pp.D;
    c.fit = fit + r0;
    c.lo = (T*)(smem + L.lo); c.hi = (T*)(smem + L.hi);
    c.obb = (T*)(smem + L.obb); c.ooff = (int*)(smem + L.ooff); c.ofl = (int*)(smem + L.ofl);
    c.vert = (T*)(smem + L.vert);
    c.edge = (T*)(smem + L.edge); c.seglen = (T*)(smem + L.seglen); c.q = (int*)(smem + L.q);
    c.list = pp.entry_cap > 0 ? (uint32_t*)(smem + L.list) : nullptr; c.m = (Misc<T>*)(smem + L.misc);
    load_world(c, world, pp.off_offsets, pp.off_verts);
    if (threadIdx.x == 0) {
        c.m->n_pair = 0;
    }
    for (int i = threadIdx.x; i < c.P; i += blockDim.x) c.q[i] = 0;
    __syncthreads();
    path_fitness_phase(pp, c);
    __syncthreads();
    for (int i = threadIdx.x; i < c.P; i += blockDim.x) qout[r0 + i] = c.q[i];
}


// K2 for wide worlds (many obstacles, config 4): one warp per (particle,
// segment) item.  Lanes box-cull 32 obstacles at a time; the overlapping ones
// are compacted (ballot + prefix) into a per-warp ring of 64 entries, and
// whenever 32 are pending all lanes run pair tests together -- full SIMT width
// for the expensive test instead of the few lanes whose box happened to hit.
// 1024 threads per CTA (one CTA per SM: the staged world is ~120 KB).
constexpr int kWideThreads = 1024, kWideRing = 64;
template <class T>
__global__ void __launch_bounds__(kWideThreads, 1) k_eval_path_wide(const unsigned char* __restrict__ world,
                                                                    SwarmParams pp, int rows, int rows_tile,
                                                                    const T* x, T* fit, int* qout,
                                                                    const IterState* gate) {
    if (gate != nullptr && gate->stop) return;
    extern __shared__ __align__(16) unsigned char smem[];
    const EvalSmem L = eval_smem(rows_tile, pp.D, pp.max_obs, pp.max_verts, (kWideThreads / 32) * kWideRing,
                                 sizeof(T), sizeof(T) == 4);
    const int r0 = blockIdx.x * rows_tile;
    Ctx<T> c{};
    c.D = pp.D; c.W = pp.D / 2; c.S = c.W + 1;
    c.fS.init(uint32_t(c.S));
    c.P = min(rows_tile, rows - r0);
    if (c.P <= 0) return;
    c.x = const_cast<T*>(x) + size_t(r0) * pp.D;
    c.lo = (T*)(smem + L.lo); c.hi = (T*)(smem + L.hi);
    c.obb = (T*)(smem + L.obb); c.ooff = (int*)(smem + L.ooff); c.ofl = (int*)(smem + L.ofl);
    c.vert = (T*)(smem + L.vert);
    c.edge = sizeof(T) == 4 ? (T*)(smem + L.edge) : nullptr;
    c.seglen = (T*)(smem + L.seglen); c.q = (int*)(smem + L.q);
    load_world(c, world, pp.off_offsets, pp.off_verts);
    for (int i = threadIdx.x; i < c.P; i += blockDim.x) c.q[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    int* ring = reinterpret_cast<int*>(smem + L.list) + warp * kWideRing;
    const int S = c.S, items = c.P * S, O = c.O;
    // Uniform grid over the map (an acceleration structure only): obstacle o
    // is filed under the cell of its box's lower corner, sorted by cell; a
    // segment visits the cells its margin-grown box can reach, extended by the
    // largest obstacle extent, so every obstacle whose box can overlap is
    // tested exactly once and the exact box test (geometry.hpp:167-188) decides.
    int* gstart = reinterpret_cast<int*>(smem + L.grid);
    int* gidx = reinterpret_cast<int*>(smem + L.gidx);
    int* hist = reinterpret_cast<int*>(smem + L.list);          // ring space, before its use
    __shared__ float ext[2];
    const T span = c.hi[0] > c.hi[c.W] ? c.hi[0] : c.hi[c.W];
    const T inv_cs = T(kGridDim) / (span > T(0) ? span : T(1));
    auto cell_of = [&](T v) {
        const T f = v * inv_cs;
        return f < T(0) ? 0 : (f >= T(kGridDim - 1) ? kGridDim - 1 : int(f));
    };
    for (int i = threadIdx.x; i < kGridDim * kGridDim; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x < 2) ext[threadIdx.x] = 0.f;
    __syncthreads();
    for (int o = threadIdx.x; o < O; o += blockDim.x) {
        const T* bb = c.obb + 4 * o;
        atomicAdd(&hist[cell_of(bb[0]) + kGridDim * cell_of(bb[1])], 1);
        atomicMax(reinterpret_cast<int*>(&ext[0]), __float_as_int(float(bb[2] - bb[0])));   // >= 0
        atomicMax(reinterpret_cast<int*>(&ext[1]), __float_as_int(float(bb[3] - bb[1])));
    }
    __syncthreads();
    if (warp == 0) {                                           // exclusive scan of the histogram
        int run = 0;
        for (int b0 = 0; b0 < kGridDim * kGridDim; b0 += 32) {
            const int v = hist[b0 + lane];
            int incl = v;
            for (int off = 1; off < 32; off <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += t;
            }
            gstart[b0 + lane] = run + incl - v;
            hist[b0 + lane] = run + incl - v;                  // fill cursor
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) gstart[kGridDim * kGridDim] = run;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < O; o += blockDim.x) {
        const T* bb = c.obb + 4 * o;
        gidx[atomicAdd(&hist[cell_of(bb[0]) + kGridDim * cell_of(bb[1])], 1)] = o;
    }
    __syncthreads();
    const T extw = T(ext[0]) * T(1.0001) + c.margin, exth = T(ext[1]) * T(1.0001) + c.margin;
    for (int it = warp; it < items; it += nw) {
        const int pl = int(c.fS.div(uint32_t(it))), s = it - pl * S;
        T a1x, a1y, a2x, a2y;
        chain_pt(c, pl, s, a1x, a1y);
        chain_pt(c, pl, s + 1, a2x, a2y);
        if (lane == 0) c.seglen[it] = seg_length<T>(Ar<T>::sub(a2x, a1x), Ar<T>::sub(a2y, a1y));
        const T lx = a1x < a2x ? a1x : a2x, hx = a1x < a2x ? a2x : a1x;
        const T ly = a1y < a2y ? a1y : a2y, hy = a1y < a2y ? a2y : a1y;
        const int cy0 = cell_of(ly - exth), cy1 = cell_of(hy + c.margin);
        int cnt = 0, head = 0, pend = 0;
        // the cell rows' candidate ranges form one stream: lane r holds row r's
        // start in gidx and its offset in the stream; 32 candidates per batch.
        // Row r's range is swept, not the whole box: an obstacle with an edge
        // crossing the segment contains the crossing point P in its box, so its
        // filed (lower) corner lies in P - [0, ext]; for the row's band of
        // corners only the part of the segment at y in [band low, band high +
        // ext_y] matters, and the columns follow from that part's x range.
        // Obstacles the box test alone would pass (box overlaps the segment's
        // box, no edge crosses) contribute no crossing either way, so Q is the
        // same; bands and ranges are widened by a rounding guard.
        const int nrows = cy1 - cy0 + 1;                       // <= kGridDim = 32
        int rbeg = 0, rlen = 0;
        if (lane < nrows) {
            const int cy = cy0 + lane;
            const T cs = T(1) / inv_cs, guard = cs * T(1e-3) + c.margin;
            const T ya = cy == 0 ? -T(1e30) : T(cy) * cs - guard;
            const T yb = cy == kGridDim - 1 ? T(1e30) : T(cy + 1) * cs + exth + guard;
            const T dy = Ar<T>::sub(a2y, a1y), dx = Ar<T>::sub(a2x, a1x);
            T px0 = lx, px1 = hx;
            bool any = hy >= ya && ly <= yb;
            if (any && (ly < ya || hy > yb) && dy != T(0)) {        // clip the segment to the slab
                const T ta = (ya - a1y) / dy, tb = (yb - a1y) / dy;
                const T t0 = fmax(T(0), fmin(ta, tb)), t1 = fmin(T(1), fmax(ta, tb));
                const T xa = a1x + t0 * dx, xb = a1x + t1 * dx;
                const T gx = guard + T(1e-4) * (hx - lx);
                px0 = fmax(lx, fmin(xa, xb) - gx);
                px1 = fmin(hx, fmax(xa, xb) + gx);
            }
            if (any) {
                const int cx0 = cell_of(px0 - extw), cx1 = cell_of(px1 + c.margin);
                rbeg = gstart[cy * kGridDim + cx0];
                rlen = gstart[cy * kGridDim + cx1 + 1] - rbeg;
            }
        }
        int rinc = rlen;
        for (int off = 1; off < 32; off <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, rinc, off);
            if (lane >= off) rinc += t;
        }
        const int total = __shfl_sync(0xffffffffu, rinc, 31), rexc = rinc - rlen;
        {
            for (int b0 = 0; b0 < total; b0 += 32) {
                const int t = b0 + lane;
                int r = 0;                                       // last row with stream start <= t
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int cand = r + step;
                    const int ex = __shfl_sync(0xffffffffu, rexc, cand < 32 ? cand : 31);
                    if (cand < nrows && ex <= t) r = cand;
                }
                const int gi = __shfl_sync(0xffffffffu, rbeg, r) + (t - __shfl_sync(0xffffffffu, rexc, r));
                const bool in = t < total;
                const int o = in ? gidx[gi] : 0;
                const bool ov = in && box_overlap(lx, ly, hx, hy, c.obb + 4 * o, c.margin);
                const unsigned m = __ballot_sync(0xffffffffu, ov);
                if (ov) ring[(head + pend + __popc(m & lt_mask)) & (kWideRing - 1)] = o;
                pend += __popc(m);
                __syncwarp();
                if (pend >= 32) {
                    cnt += pair_count_pts(c, a1x, a1y, a2x, a2y, ring[(head + lane) & (kWideRing - 1)]);
                    head += 32;
                    pend -= 32;
                    __syncwarp();
                }
            }
        }
        if (lane < pend) cnt += pair_count_pts(c, a1x, a1y, a2x, a2y, ring[(head + lane) & (kWideRing - 1)]);
        __syncwarp();
        if (s == 0)   // first waypoint (the segment's end) strictly inside (geometry.hpp:217-218)
            for (int o = lane; o < O; o += 32) {
                const T* bb = c.obb + 4 * o;
                if (a2x >= bb[0] - c.margin && a2x <= bb[2] + c.margin && a2y >= bb[1] - c.margin &&
                    a2y <= bb[3] + c.margin)
                    cnt += contain_count(c, pl, o);
            }
        cnt = int(__reduce_add_sync(0xffffffffu, uint32_t(cnt)));
        if (lane == 0 && cnt) atomicAdd(&c.q[pl], cnt);
    }
    __syncthreads();
    for (int pl = threadIdx.x; pl < c.P; pl += blockDim.x) {
        T len = T(0);
        for (int s = 0; s < S; ++s) len = Ar<T>::add(len, c.seglen[pl * S + s]);
        fit[r0 + pl] = Ar<T>::add(len, T(penalty(pp.alpha, pp.beta, pp.beta_int, c.q[pl])));
        qout[r0 + pl] = c.q[pl];
    }
}

int stage_eval_path(bool fp64, const unsigned char* world, int max_obs, int max_verts,
                    int off_offsets, int off_verts, int D, int rows, const void* x, double alpha,
                    double beta, void* fit, int* q, const IterState* gate, void* stream) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    SwarmParams pp{};
    pp.D = D;
    pp.max_obs = max_obs;
    pp.max_verts = max_verts;
    pp.off_offsets = off_offsets;
    pp.off_verts = off_verts;
    pp.alpha = alpha;
    pp.beta = beta;
    pp.beta_int = (beta == double(int(beta)) && beta >= 1.0 && beta <= 64.0) ? int(beta) : 0;
    if (max_obs >= 48) {   // wide worlds: lanes over obstacles
        const int rows_tile = 64;
        pp.entry_cap = 0;
        // FP64 reads the vertices only (no edge records)
        const EvalSmem L = eval_smem(rows_tile, D, max_obs, max_verts, (kWideThreads / 32) * kWideRing,
                                     fp64 ? 8 : 4, !fp64);
        const unsigned grid = unsigned((rows + rows_tile - 1) / rows_tile);
        if (grid == 0) return 0;
        cudaError_t e;
        if (fp64) {
            e = cudaFuncSetAttribute(k_eval_path_wide<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
            if (e != cudaSuccess) return int(e);
            k_eval_path_wide<double><<<grid, kWideThreads, L.total, st>>>(world, pp, rows, rows_tile, (const double*)x,
                                                                 (double*)fit, q, gate);
        } else {
            e = cudaFuncSetAttribute(k_eval_path_wide<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
            if (e != cudaSuccess) return int(e);
            k_eval_path_wide<float><<<grid, kWideThreads, L.total, st>>>(world, pp, rows, rows_tile, (const float*)x,
                                                                (float*)fit, q, gate);
        }
        return int(cudaGetLastError());
    }
    const int rows_tile = 64;
    pp.entry_cap = 256 / 32 * 64;            // per-warp rings of compacted pair tests (A1)
    const size_t tsz = fp64 ? 8 : 4;
    const EvalSmem L = eval_smem(rows_tile, D, max_obs, max_verts, pp.entry_cap, tsz);
    const unsigned grid = unsigned((rows + rows_tile - 1) / rows_tile);
    if (grid == 0) return 0;
    cudaError_t e;
    if (fp64) {
        e = cudaFuncSetAttribute(k_eval_path<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
        if (e != cudaSuccess) return int(e);
        k_eval_path<double><<<grid, 256, L.total, st>>>(world, pp, rows, rows_tile, (const double*)x,
                                                        (double*)fit, q, gate);
    } else {
        e = cudaFuncSetAttribute(k_eval_path<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
        if (e != cudaSuccess) return int(e);
        k_eval_path<float><<<grid, 256, L.total, st>>>(world, pp, rows, rows_tile, (const float*)x,
                                                       (float*)fit, q, gate);
    }
    return int(cudaGetLastError());
}

// Benchmark fitness of many rows (benchmarks.hpp:56-88, the staged path): a
// warp owns 32 rows, lane l row r0 + l, and walks them in 32-column tiles --
// the warp loads a tile row by row (coalesced: 32 consecutive columns of one
// row per load) into shared memory, then every lane folds its row's 32
// elements in index order (bench_elem, the same arithmetic as the fused
// kernel's bench_row).  A thread-per-row walk straight from HBM touches 32
// cache lines per warp load and ran at ~40 % of the copy bandwidth.
template <class T> constexpr int kBenchWarps = sizeof(T) == 8 ? 4 : 8;   // static tiles under 48 KB
template <int K, class T>
__device__ __forceinline__ void bench_rows_tiled(int D, int rows, const T* __restrict__ x, T* fit, int* q, T* tile) {
    const int lane = threadIdx.x & 31;
    const int nw = int(gridDim.x) * kBenchWarps<T>;
    for (int r0 = (blockIdx.x * kBenchWarps<T> + (threadIdx.x >> 5)) * 32; r0 < rows; r0 += nw * 32) {
        T s = T(0), t = bench_t0<K, T>(), xp = T(0);
        const int nr = min(32, rows - r0);
        const T* base = x + size_t(r0) * D + lane;
        // software pipeline: the next tile's 32 loads are in flight (registers)
        // while the lanes fold the current one from shared memory
        T nxt[32];
#pragma unroll
        for (int rr = 0; rr < 32; ++rr) nxt[rr] = (rr < nr && lane < D) ? base[size_t(rr) * D] : T(0);
        for (int c0 = 0; c0 < D; c0 += 32) {
#pragma unroll
            for (int rr = 0; rr < 32; ++rr) tile[rr * 33 + lane] = nxt[rr];
            __syncwarp();
            const int c1 = c0 + 32;
            if (c1 < D) {
                const bool ok = c1 + lane < D;
#pragma unroll
                for (int rr = 0; rr < 32; ++rr) nxt[rr] = (rr < nr && ok) ? base[size_t(rr) * D + c1] : T(0);
            }
            const int n = min(32, D - c0);
            if (n == 32) {
#pragma unroll 8
                for (int j = 0; j < 32; ++j) {
                    const T v = tile[lane * 33 + j];
                    bench_elem<K, T>(c0 + j, v, xp, s, t);
                    xp = v;
                }
            } else {
                for (int j = 0; j < n; ++j) {
                    const T v = tile[lane * 33 + j];
                    bench_elem<K, T>(c0 + j, v, xp, s, t);
                    xp = v;
                }
            }
            __syncwarp();
        }
        if (lane < nr) {
            fit[r0 + lane] = bench_fin<K, T>(s, t, D);
            if (q) q[r0 + lane] = 0;
        }
    }
}

template <class T>
__global__ void __launch_bounds__(kBenchWarps<T> * 32) k_eval_bench(int kind, int D, int rows, const T* __restrict__ x,
                                                                 T* fit, int* q, const IterState* gate) {
    __shared__ T tiles[kBenchWarps<T>][32 * 33];
    if (gate != nullptr && gate->stop) return;
    T* tile = tiles[threadIdx.x >> 5];
    switch (kind) {
    case kSphere: bench_rows_tiled<kSphere, T>(D, rows, x, fit, q, tile); break;
    case kRosenbrock: bench_rows_tiled<kRosenbrock, T>(D, rows, x, fit, q, tile); break;
    case kRastrigin: bench_rows_tiled<kRastrigin, T>(D, rows, x, fit, q, tile); break;
    case kGriewank: bench_rows_tiled<kGriewank, T>(D, rows, x, fit, q, tile); break;
    case kAckley: bench_rows_tiled<kAckley, T>(D, rows, x, fit, q, tile); break;
    }
}

int stage_eval_bench(bool fp64, int kind, int D, int rows, const void* x, void* fit, int* q,
                     const IterState* gate, void* stream) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int bw = fp64 ? kBenchWarps<double> : kBenchWarps<float>;
    const unsigned grid = grid_for((rows + 31) / 32, bw);
    if (fp64) k_eval_bench<double><<<grid, bw * 32, 0, st>>>(kind, D, rows, (const double*)x, (double*)fit, q, gate);
    else k_eval_bench<float><<<grid, bw * 32, 0, st>>>(kind, D, rows, (const float*)x, (float*)fit, q, gate);
    return int(cudaGetLastError());
}

// ------------------------------------------------------------ best tracking
// runner.hpp:73-80: warp per row, strict '<', copy x -> pbest_x on improvement.
template <class T>
__global__ void k_pbest(StageShape s, const T* __restrict__ x, const T* __restrict__ fit,
                        const int* __restrict__ q, T* pb, T* pbf, int* pbq, IterState* st,
                        const IterState* gate) {
    if (gate != nullptr && gate->stop) return;
    const int lane = threadIdx.x & 31;
    const int rl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (rl >= s.rows) return;
    int better = 0;
    if (lane == 0) {
        const T f = fit[rl];
        if (st != nullptr && !isfinite(f)) atomicMin(&st->nonfinite_row, s.row_begin + rl);
        better = f < pbf[rl];
        if (better) { pbf[rl] = f; pbq[rl] = q ? q[rl] : 0; }
    }
    better = __shfl_sync(0xffffffffu, better, 0);
    if (better)
        for (int d = lane; d < s.D; d += 32) pb[size_t(rl) * s.D + d] = x[size_t(rl) * s.D + d];
}

// run_staged's pbest (runner.hpp:73-80) with the row copy deferred to the
// step (k_step, imp): thread per row, strict '<', imp[row] = improved.
template <class T>
__global__ void k_pbest_flag(StageShape s, const T* __restrict__ fit, const int* __restrict__ q, T* pbf,
                             int* pbq, unsigned char* imp, IterState* st, const IterState* gate) {
    if (gate != nullptr && gate->stop) return;
    for (int rl = blockIdx.x * blockDim.x + threadIdx.x; rl < s.rows; rl += gridDim.x * blockDim.x) {
        const T f = fit[rl];
        if (st != nullptr && !isfinite(f)) atomicMin(&st->nonfinite_row, s.row_begin + rl);
        const bool better = f < pbf[rl];
        if (better) { pbf[rl] = f; pbq[rl] = q ? q[rl] : 0; }
        imp[rl] = better ? 1 : 0;
    }
}

// Per local group: (pbest_f, global row) lexicographic min (runner.hpp:81-87 order).
template <class T>
__global__ void k_group_partial(StageShape s, const T* __restrict__ pbf, const int* __restrict__ pbq,
                                T* part_f, int* part_row, int* part_q, const IterState* gate) {
    if (gate != nullptr && gate->stop) return;
    using A = Ar<T>;
    const int g = s.row_begin / s.N + blockIdx.x;
    const int l0 = max(g * s.N, s.row_begin) - s.row_begin;
    const int l1 = min((g + 1) * s.N, s.row_begin + s.rows) - s.row_begin;
    T bf = A::inf();
    int br = INT_MAX;
    // eight loads in flight per thread (the scan is latency-bound: one CTA per
    // group), then the compares in row order
    int r = l0 + threadIdx.x;
    const int step = blockDim.x;
    for (; r + 7 * step < l1; r += 8 * step) {
        T f8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f8[i] = pbf[r + i * step];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            if (f8[i] < bf) { bf = f8[i]; br = r + i * step; }
    }
    for (; r < l1; r += step) {
        const T f = pbf[r];
        if (f < bf) { bf = f; br = r; }
    }
    for (int off = 16; off; off >>= 1) {
        const T of = __shfl_down_sync(0xffffffffu, bf, off);
        const int orow = __shfl_down_sync(0xffffffffu, br, off);
        if (of < bf || (of == bf && orow < br)) { bf = of; br = orow; }
    }
    __shared__ T wf[32];
    __shared__ int wr[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { wf[warp] = bf; wr[warp] = br; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < int(blockDim.x >> 5); ++w)
            if (wf[w] < bf || (wf[w] == bf && wr[w] < br)) { bf = wf[w]; br = wr[w]; }
        part_f[blockIdx.x] = bf;
        part_row[blockIdx.x] = br == INT_MAX ? -1 : br;     // local row
        part_q[blockIdx.x] = br == INT_MAX ? 0 : pbq[br];
    }
}

int stage_pbest_partials(bool fp64, const StageShape& s, const void* x, const void* fit,
                         const int* q, void* pb, void* pbf, int* pbq, IterState* stt,
                         void* part_f, int* part_row, int* part_q, const IterState* gate,
                         void* stream, unsigned char* imp) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = unsigned((s.rows * 32LL + 255) / 256);
    const int n_groups = (s.row_begin + s.rows - 1) / s.N - s.row_begin / s.N + 1;
    if (imp != nullptr) {
        const unsigned gf = grid_for(s.rows, 256);
        if (fp64) k_pbest_flag<double><<<gf, 256, 0, st>>>(s, (const double*)fit, q, (double*)pbf, pbq, imp, stt, gate);
        else k_pbest_flag<float><<<gf, 256, 0, st>>>(s, (const float*)fit, q, (float*)pbf, pbq, imp, stt, gate);
    } else if (fp64) {
        k_pbest<double><<<grid, 256, 0, st>>>(s, (const double*)x, (const double*)fit, q,
                                              (double*)pb, (double*)pbf, pbq, stt, gate);
    } else {
        k_pbest<float><<<grid, 256, 0, st>>>(s, (const float*)x, (const float*)fit, q,
                                             (float*)pb, (float*)pbf, pbq, stt, gate);
    }
    if (fp64) {
        k_group_partial<double><<<n_groups, 256, 0, st>>>(s, (const double*)pbf, pbq,
                                                          (double*)part_f, part_row, part_q, gate);
    } else {
        k_group_partial<float><<<n_groups, 256, 0, st>>>(s, (const float*)pbf, pbq,
                                                         (float*)part_f, part_row, part_q, gate);
    }
    return int(cudaGetLastError());
}

// gbest for the local groups, then this device's tbest candidate
// (runner.hpp:81-91).  One CTA takes the decisions -- a group's gbest changes
// on a strict '<', and the header of the candidate -- and leaves the changed
// group's row in part_row (-1: unchanged); a wide grid then copies the changed
// rows into gbest_x and the candidate's x (one CTA copying every row was
// load-latency bound).
template <class T>
__global__ void k_group_bests(StageShape s, const T* __restrict__ part_f, int* __restrict__ part_row,
                              const int* __restrict__ part_q, T* gbf, int* gbq, unsigned char* cand,
                              const IterState* gate, const IterState* st) {
    if (gate != nullptr && gate->stop) return;
    const int g0 = s.row_begin / s.N;
    const int ng = (s.row_begin + s.rows - 1) / s.N - g0 + 1;
    for (int lg = threadIdx.x; lg < ng; lg += blockDim.x) {
        const int g = g0 + lg;
        if (part_row[lg] >= 0 && part_f[lg] < gbf[g]) {
            gbf[g] = part_f[lg];
            gbq[g] = part_q[lg];
        } else {
            part_row[lg] = -1;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        CandHdr h{__longlong_as_double(0x7ff0000000000000ll), 0, -1, st ? st->nonfinite_row : INT_MAX, 0};
        for (int lg = 0; lg < ng; ++lg) {
            const double f = double(gbf[g0 + lg]);
            if (f < h.f) { h.f = f; h.q = gbq[g0 + lg]; h.g = g0 + lg; }
        }
        *reinterpret_cast<CandHdr*>(cand) = h;
    }
}

// element t of the copies: t < ng*D: gbest_x of local group t / D (if it
// changed); then the candidate's x.  A changed group's row is read from x
// when it improved this iteration (its pbest_x copy is deferred to k_step).
template <class T>
__global__ void k_group_rows(StageShape s, const int* __restrict__ part_row, const T* __restrict__ pb,
                             T* gbx, unsigned char* cand, const IterState* gate, const T* __restrict__ x,
                             const unsigned char* __restrict__ imp) {
    if (gate != nullptr && gate->stop) return;
    const int g0 = s.row_begin / s.N;
    const int ng = (s.row_begin + s.rows - 1) / s.N - g0 + 1;
    const int D = s.D;
    const int bg = reinterpret_cast<const CandHdr*>(cand)->g;
    T* cx = reinterpret_cast<T*>(cand + sizeof(CandHdr));
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)(ng + 1) * D;
         t += (long long)gridDim.x * blockDim.x) {
        const int lg = int(t / D), d = int(t - (long long)lg * D);
        if (lg < ng) {
            const int row = part_row[lg];
            if (row >= 0) {
                const T* src = imp != nullptr && imp[row] ? x : pb;
                gbx[size_t(g0 + lg) * D + d] = src[size_t(row) * D + d];
            }
        } else if (bg >= 0) {         // the candidate: the best group's (new or kept) gbest_x
            const int row = part_row[bg - g0];
            const T* src = row < 0 ? gbx + size_t(bg) * D : (imp != nullptr && imp[row] ? x : pb) + size_t(row) * D;
            cx[d] = src[d];
        }
    }
}

int stage_group_bests(bool fp64, const StageShape& s, const void* part_f, const int* part_row,
                      const int* part_q, const void* pb, void* gbx, void* gbf, int* gbq,
                      void* cand, const IterState* gate, void* stream, const IterState* stt,
                      const void* x, const unsigned char* imp) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int ng = (s.row_begin + s.rows - 1) / s.N - s.row_begin / s.N + 1;
    int* prow = const_cast<int*>(part_row);      // consumed here: unchanged groups marked -1
    const unsigned grid = grid_for((long long)(ng + 1) * s.D, 256);
    if (fp64) {
        k_group_bests<double><<<1, 256, 0, st>>>(s, (const double*)part_f, prow, part_q, (double*)gbf, gbq,
                                                 (unsigned char*)cand, gate, stt);
        k_group_rows<double><<<grid, 256, 0, st>>>(s, prow, (const double*)pb, (double*)gbx, (unsigned char*)cand,
                                                   gate, (const double*)x, imp);
    } else {
        k_group_bests<float><<<1, 256, 0, st>>>(s, (const float*)part_f, prow, part_q, (float*)gbf, gbq,
                                                (unsigned char*)cand, gate, stt);
        k_group_rows<float><<<grid, 256, 0, st>>>(s, prow, (const float*)pb, (float*)gbx, (unsigned char*)cand,
                                                  gate, (const float*)x, imp);
    }
    return int(cudaGetLastError());
}

// tbest over candidates (ascending group order, strict '<'), window + AT.
template <class T>
__global__ void k_finish(int D, const unsigned char* __restrict__ cands, int n_cand, size_t cstride,
                         T* tbx, IterState* st, double* win, int tw, int auto_truncate,
                         double delta, int k, double* trace) {
    if (st->stop) return;
    __shared__ int src;
    if (threadIdx.x == 0) {
        src = -1;
        int bad = INT_MAX;
        for (int i = 0; i < n_cand; ++i)
            bad = min(bad, reinterpret_cast<const CandHdr*>(cands + i * cstride)->bad);
        if (bad != INT_MAX) {
            st->nonfinite_row = bad;
            st->status = 2;
            st->stop = 1;
        } else {
            // candidates come from disjoint group ranges; scan in group order
            int order[64];
            const int nc = n_cand < 64 ? n_cand : 64;
            for (int i = 0; i < nc; ++i) order[i] = i;
            for (int i = 1; i < nc; ++i) {      // insertion sort by group
                const int t = order[i];
                const int gt = reinterpret_cast<const CandHdr*>(cands + t * cstride)->g;
                int j = i - 1;
                while (j >= 0 && reinterpret_cast<const CandHdr*>(cands + order[j] * cstride)->g > gt) {
                    order[j + 1] = order[j];
                    --j;
                }
                order[j + 1] = t;
            }
            for (int i = 0; i < nc; ++i) {
                const CandHdr* h = reinterpret_cast<const CandHdr*>(cands + order[i] * cstride);
                if (h->g >= 0 && h->f < st->tbest_f) {
                    st->tbest_f = h->f;
                    st->tbest_q = h->q;
                    st->tbest_group = h->g;
                    src = order[i];
                }
            }
            if (trace) trace[k - 1] = st->tbest_f;
            if (win != nullptr && tw > 0) {
                const double tv = st->tbest_f;
                if (st->win_len < tw) {
                    win[(st->win_head + st->win_len) % tw] = tv;
                    ++st->win_len;
                } else {
                    win[st->win_head] = tv;
                    st->win_head = (st->win_head + 1) % tw;
                }
                int newest = st->win_head + st->win_len - 1;
                if (newest >= tw) newest -= tw;
                const double gap = fabs(win[newest] - win[st->win_head]);
                const bool may_fire = !(gap >= delta * sqrt(2.0 * tw) * (1.0 + 1e-9));
                if (auto_truncate && st->win_len >= tw && st->tbest_q == 0 && may_fire) {
                    double mean = 0.0;
                    for (int i = 0; i < tw; ++i) mean = __dadd_rn(mean, win[(st->win_head + i) % tw]);
                    mean = __ddiv_rn(mean, double(tw));
                    double var = 0.0;
                    for (int i = 0; i < tw; ++i) {
                        const double dv = __dsub_rn(win[(st->win_head + i) % tw], mean);
                        var = __dadd_rn(var, __dmul_rn(dv, dv));
                    }
                    var = __ddiv_rn(var, double(tw));
                    if (__dsqrt_rn(var) < delta) {
                        st->truncated = 1;
                        st->stop = 1;
                    }
                }
            }
        }
        st->k_done = k;
    }
    __syncthreads();
    if (src >= 0) {
        const T* cx = reinterpret_cast<const T*>(cands + src * cstride + sizeof(CandHdr));
        for (int d = threadIdx.x; d < D; d += blockDim.x) tbx[d] = cx[d];
    }
}

int stage_finish(bool fp64, int D, const void* cands, int n_cand, void* tbx, IterState* stt,
                 double* win, int tw, int auto_truncate, double delta, int k, int cap,
                 double* trace, void* stream) {
    (void)cap;
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t cs = cand_bytes(fp64, D);
    if (fp64)
        k_finish<double><<<1, 128, 0, st>>>(D, (const unsigned char*)cands, n_cand, cs, (double*)tbx,
                                            stt, win, tw, auto_truncate, delta, k, trace);
    else
        k_finish<float><<<1, 128, 0, st>>>(D, (const unsigned char*)cands, n_cand, cs, (float*)tbx,
                                           stt, win, tw, auto_truncate, delta, k, trace);
    return int(cudaGetLastError());
}

} // namespace sepso
