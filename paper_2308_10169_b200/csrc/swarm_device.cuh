// swarm_device.cuh -- device building blocks shared by the fused swarm kernel
// (swarm_kernel.cu) and the HBM-resident stage kernels (stage_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <cmath>

#include "cos_glibc.cuh"
#include "geometry.cuh"
#include "philox.cuh"
#include "swarm_kernel.cuh"

namespace sepso {

// ---------------------------------------------------------------- arithmetic
// FP64: no contraction, so every rounding happens where the reference's
// -ffp-contract=off build rounds.  FP32: plain operators (FMA allowed).
template <class T> struct Ar;
template <> struct Ar<double> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
};
template <> struct Ar<float> {
    static __device__ __forceinline__ float add(float a, float b) { return a + b; }
    static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
    static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
    static __device__ __forceinline__ float inf() { return __int_as_float(0x7f800000); }
};

template <class T> __device__ __forceinline__ T clampT(T v, T lo, T hi) {   // std::clamp
    return v < lo ? lo : (hi < v ? hi : v);
}

template <class T> struct Misc {
    T tbf;
    int tbq, tsrc_slot, stop, truncated, status, bad_row, bad_min, n_pair, n_cont;
    int win_len, win_head, k_done, cont_cap;
    int mt_cur;                 // mt19937_64 generator bookkeeping (MtState outside generation)
    long long mt_blocks;
    int q64;                    // FP32 engine: Q of the final best path on the FP64 world
    int pre_ok;                 // the ahead-of-time init walk arrived (prewalk.cu)
};

// alpha * q^beta (geometry.hpp:240): exact repeated product for small integer
// beta (std::pow is exact there), libm pow otherwise.
__device__ __forceinline__ double penalty(double alpha, double beta, int beta_int, int q) {
    double qp;
    if (beta_int > 0) {
        const double qd = double(q);
        qp = qd;
        for (int i = 1; i < beta_int; ++i) qp = __dmul_rn(qp, qd);
    } else {
        qp = pow(double(q), beta);
    }
    return __dmul_rn(alpha, qp);
}

// benchmarks.hpp:56-88 (+ Ackley extension).  FP64: std::cos as the
// reference's host computes it (cos_glibc.cuh), so BF3 / BF4 runs stay bit-exact.
// One row is a stream of elements in index order: bench_elem<K> folds element
// i (value x, previous value xp) into the running sums (s, t) exactly as the
// reference's loop does -- Rosenbrock's term i - 1 pairs p[i-1] with p[i] --
// and bench_fin<K> closes the row.  The fused kernel walks a row in place
// (bench_row); the staged evaluation streams rows through shared-memory tiles
// (k_eval_bench, stage_kernels.cu).  Both run this same arithmetic.
// Rastrigin's term of one element, x^2 - 10 cos(2 pi x) + 10 (benchmarks.hpp:56-88)
template <class T> __device__ __forceinline__ T rastrigin_term(T x);
template <> __device__ __forceinline__ double rastrigin_term<double>(double x) {
    using A = Ar<double>;
    const double two_pi = 6.283185307179586;   // 2.0 * std::numbers::pi
    return A::add(A::sub(A::mul(x, x), A::mul(10.0, cos_glibc(A::mul(two_pi, x)))), 10.0);
}
template <> __device__ __forceinline__ float rastrigin_term<float>(float x) {
    const float two_pi = 6.2831853f;
    return x * x - 10.f * cosf(two_pi * x) + 10.f;
}

template <int K, class T>
__device__ __forceinline__ void bench_elem(int i, T x, T xp, T& s, T& t) {
    if constexpr (sizeof(T) == 8) {
        using A = Ar<double>;
        const double two_pi = 6.283185307179586;   // 2.0 * std::numbers::pi
        if constexpr (K == kSphere) {
            s = A::add(s, A::mul(x, x));
        } else if constexpr (K == kRosenbrock) {
            if (i > 0) {
                const double a = A::sub(x, A::mul(xp, xp));
                const double b = A::sub(1.0, xp);
                s = A::add(s, A::add(A::mul(A::mul(100.0, a), a), A::mul(b, b)));
            }
        } else if constexpr (K == kRastrigin) {
            s = A::add(s, rastrigin_term<double>(x));
        } else if constexpr (K == kGriewank) {
            s = A::add(s, A::mul(x, x));
            t = A::mul(t, cos_glibc(__ddiv_rn(x, __dsqrt_rn(double(i + 1)))));
        } else {   // kAckley
            s = A::add(s, A::mul(x, x));
            t = A::add(t, cos_glibc(A::mul(two_pi, x)));
        }
    } else {
        const float two_pi = 6.2831853f;
        if constexpr (K == kSphere) {
            s += x * x;
        } else if constexpr (K == kRosenbrock) {
            if (i > 0) {
                const float a = x - xp * xp;
                const float b = 1.f - xp;
                s += 100.f * a * a + b * b;
            }
        } else if constexpr (K == kRastrigin) {
            s += rastrigin_term<float>(x);
        } else if constexpr (K == kGriewank) {
            s += x * x;
            t *= cosf(x * rsqrtf(float(i + 1)));
        } else {   // kAckley
            s += x * x;
            t += cosf(two_pi * x);
        }
    }
}

template <int K, class T> __device__ __forceinline__ T bench_t0() { return K == kGriewank ? T(1) : T(0); }

template <int K, class T>
__device__ __forceinline__ T bench_fin(T s, T t, int D) {
    if constexpr (sizeof(T) == 8) {
        using A = Ar<double>;
        if constexpr (K == kGriewank) return A::sub(A::add(1.0, __ddiv_rn(s, 4000.0)), t);
        if constexpr (K == kAckley) {
            const double dd = double(D);
            return -20.0 * exp(-0.2 * sqrt(s / dd)) - exp(t / dd) + 20.0 + 2.718281828459045;
        }
        return s;
    } else {
        if constexpr (K == kGriewank) return 1.f + s / 4000.f - t;
        if constexpr (K == kAckley) {
            const float dd = float(D);
            return -20.f * expf(-0.2f * sqrtf(s / dd)) - expf(t / dd) + 20.f + 2.7182817f;
        }
        return s;
    }
}

template <int K, class T>
__device__ __forceinline__ T bench_row(const T* p, int D) {
    T s = T(0), t = bench_t0<K, T>(), xp = T(0);
    for (int i = 0; i < D; ++i) {
        const T x = p[i];
        bench_elem<K, T>(i, x, xp, s, t);
        xp = x;
    }
    return bench_fin<K, T>(s, t, D);
}

template <class T>
__device__ T bench_eval(int kind, const T* p, int D) {
    switch (kind) {
    case kSphere: return bench_row<kSphere, T>(p, D);
    case kRosenbrock: return bench_row<kRosenbrock, T>(p, D);
    case kRastrigin: return bench_row<kRastrigin, T>(p, D);
    case kGriewank: return bench_row<kGriewank, T>(p, D);
    case kAckley: return bench_row<kAckley, T>(p, D);
    }
    return T(__longlong_as_double(0x7ff8000000000000ll));
}

// -------------------------------------------------------- fast division
// n / d for 0 <= n < 2^31 by multiply-high + shift (Granlund-Montgomery);
// the loops below index (particle, segment) and (particle, dim) pairs without
// hardware-emulated integer division.
struct FastDiv {
    uint32_t d = 1, mul = 0, shr = 0;
    __host__ __device__ void init(uint32_t div) {
        d = div;
        if (div <= 1) { mul = 0; shr = 0; return; }
        uint32_t l = 0;
        while ((1u << l) < div) ++l;
        const uint32_t p = 31 + l;
        mul = uint32_t(((1ull << p) + div - 1) / div);
        shr = p - 32;
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        return d == 1 ? n : (__umulhi(n, mul) >> shr);
    }
};

// ------------------------------------------------------------ swarm context
template <class T> struct Ctx {
    // shape
    int G, N, D, W, S, R, P, row0, LG, O, C, crank;
    FastDiv fS, fD, fN, fV;       // fV: 16- or 4-byte units of one pushed row
    // shared arrays
    T *x, *v, *pb, *pbf, *fit, *seglen, *coef, *lo, *hi, *hyp, *gbx, *gbf, *tbx, *px;
    int *pbq, *q, *imp, *gbq, *chg, *ooff, *ofl, *allbad, *gtab, *ctab;
    Part *part, *allpart;
    T *obb, *vert, *edge;
    double* win;
    double* vert64;               // FP32 path swarms: the caller's FP64 vertices and endpoints (final record)
    uint32_t* list;
    Misc<T>* m;
    // path constants
    T sx, sy, tx, ty, margin;
};

// Work-list entry: local particle (13 bits) | segment (8 bits) | obstacle (11 bits).
constexpr int kMaxTileRows = 8191, kMaxSegments = 255, kMaxObstacles = 2047;
__device__ __forceinline__ uint32_t pack_entry(int pl, int s, int o) {
    return (uint32_t(pl) << 19) | (uint32_t(s) << 11) | uint32_t(o);
}

// chain point j of start -> w_1..w_W -> target for local particle pl (geometry.hpp:157-165)
template <class T>
__device__ __forceinline__ void chain_pt(const Ctx<T>& c, int pl, int j, T& px, T& py) {
    if (j == 0) { px = c.sx; py = c.sy; }
    else if (j == c.W + 1) { px = c.tx; py = c.ty; }
    else { px = c.x[pl * c.D + j - 1]; py = c.x[pl * c.D + c.W + j - 1]; }
}

template <class T> __device__ __forceinline__ T seg_length(T dx, T dy);
template <> __device__ __forceinline__ double seg_length<double>(double dx, double dy) {
    return hypot_glibc(dx, dy);                       // std::hypot, geometry.hpp:228
}
template <> __device__ __forceinline__ float seg_length<float>(float dx, float dy) {
    return sqrtf(fmaf(dx, dx, dy * dy));
}

// Segment s of particle pl against every edge of obstacle o: the number of
// intersecting (segment, edge) pairs (geometry.hpp:210-214).
template <class T>
__device__ int pair_count(const Ctx<T>& c, int pl, int s, int o);

// FP64 engine: the reference predicate on every edge, bit for bit.
inline __device__ int pair_count_pts(const Ctx<double>& c, double a1x, double a1y, double a2x,
                                     double a2y, int o) {
    const int v0 = c.ooff[o], v1 = c.ooff[o + 1];
    int cnt = 0;
    for (int i = v0; i < v1; ++i) {
        const int j = (i + 1 == v1) ? v0 : i + 1;
        cnt += segments_intersect_ref(a1x, a1y, a2x, a2y, c.vert[2 * i], c.vert[2 * i + 1],
                                      c.vert[2 * j], c.vert[2 * j + 1]);
    }
    return cnt;
}

template <>
inline __device__ int pair_count<double>(const Ctx<double>& c, int pl, int s, int o) {
    double a1x, a1y, a2x, a2y;
    chain_pt(c, pl, s, a1x, a1y);
    chain_pt(c, pl, s + 1, a2x, a2y);
    return pair_count_pts(c, a1x, a1y, a2x, a2y, o);
}

// FP32 engine fallback to the FP64 reference predicate, kept out of line so the
// hot loop's code stays compact (the fallback is rare).
static __device__ __noinline__ int seg_ref_f(float a1x, float a1y, float a2x, float a2y, float b1x, float b1y,
                                      float b2x, float b2y) {
    return segments_intersect_ref(a1x, a1y, a2x, a2y, b1x, b1y, b2x, b2y);
}

// FP32 engine: filtered orientation signs.
// Vertex crosses cv_i = d x (v_i - a1) are shared by the two edges meeting at
// v_i (o1 of edge i is o2 of edge i-1).  With every |cv| above the bound B and
// one common sign, no edge can be hit -- neither properly (o1 == o2 on every
// edge) nor through the collinear cases, which need an endpoint of the path
// segment on an edge and therefore opposite vertex signs -- provided the
// obstacle has no edge shorter than 1e-3 (ofl[o]); otherwise every edge takes
// the per-pair test.  Uncertain signs fall back to the FP64 reference.
inline __device__ int pair_count_pts(const Ctx<float>& c, float a1x, float a1y, float a2x, float a2y,
                                     int o) {
    const float dx = a2x - a1x, dy = a2y - a1y;
    const float* bb = c.obb + 4 * o;
    const float ux = fmaxf(fmaxf(a1x, a2x), bb[2]) - fminf(fminf(a1x, a2x), bb[0]);
    const float uy = fmaxf(fmaxf(a1y, a2y), bb[3]) - fminf(fminf(a1y, a2y), bb[1]);
    const float L = fmaxf(ux, uy);
    // |error| of any cross product below <= 31 u L^2 (u = 2^-24); 48 u L^2
    // leaves margin, 4e-12 covers the reference's 1e-12 dead band.
    const float B = 2.9e-6f * L * L + 4e-12f;
    const int v0 = c.ooff[o], v1 = c.ooff[o + 1];
    const float4* E = reinterpret_cast<const float4*>(c.edge);
    if (v1 - v0 == 4) {
        // quadrilaterals (every obstacle of the paper's scenes): all loads and
        // crosses issue together -- no loop-carried latency chain
        const float4 e0 = E[v0], e1 = E[v0 + 1], e2 = E[v0 + 2], e3 = E[v0 + 3];
        const float cv0 = fmaf(dx, e0.y - a1y, -(dy * (e0.x - a1x)));
        const float cv1 = fmaf(dx, e1.y - a1y, -(dy * (e1.x - a1x)));
        const float cv2 = fmaf(dx, e2.y - a1y, -(dy * (e2.x - a1x)));
        const float cv3 = fmaf(dx, e3.y - a1y, -(dy * (e3.x - a1x)));
        if (c.ofl[o]) {
            const float mn = fminf(fminf(cv0, cv1), fminf(cv2, cv3));
            const float mx = fmaxf(fmaxf(cv0, cv1), fmaxf(cv2, cv3));
            if (mn > B || mx < -B) return 0;          // vertex-cross early exit
        }
        int r0 = fast_pair(a1x, a1y, dx, dy, e0.x, e0.y, e0.z, e0.w, B);
        int r1 = fast_pair(a1x, a1y, dx, dy, e1.x, e1.y, e1.z, e1.w, B);
        int r2 = fast_pair(a1x, a1y, dx, dy, e2.x, e2.y, e2.z, e2.w, B);
        int r3 = fast_pair(a1x, a1y, dx, dy, e3.x, e3.y, e3.z, e3.w, B);
        if ((r0 | r1 | r2 | r3) < 0) {                 // some sign uncertain: FP64 reference
            const float* vv = c.vert + 2 * v0;
            if (r0 < 0) r0 = seg_ref_f(a1x, a1y, a2x, a2y, vv[0], vv[1], vv[2], vv[3]);
            if (r1 < 0) r1 = seg_ref_f(a1x, a1y, a2x, a2y, vv[2], vv[3], vv[4], vv[5]);
            if (r2 < 0) r2 = seg_ref_f(a1x, a1y, a2x, a2y, vv[4], vv[5], vv[6], vv[7]);
            if (r3 < 0) r3 = seg_ref_f(a1x, a1y, a2x, a2y, vv[6], vv[7], vv[0], vv[1]);
        }
        return r0 + r1 + r2 + r3;
    }
    if (c.ofl[o]) {
        bool pos = true, neg = true;
        for (int i = v0; i < v1; ++i) {
            const float4 e = E[i];
            const float cv = fmaf(dx, e.y - a1y, -(dy * (e.x - a1x)));
            pos &= cv > B;
            neg &= cv < -B;
        }
        if (pos || neg) return 0;
    }
    int cnt = 0;
    for (int i = v0; i < v1; ++i) {
        const float4 e = E[i];
        int r = fast_pair(a1x, a1y, dx, dy, e.x, e.y, e.z, e.w, B);
        if (r < 0) {
#ifdef SEPSO_COUNT_FALLBACKS
            atomicAdd(&c.m->n_cont, 1);
#endif
            const int j = (i + 1 == v1) ? v0 : i + 1;
            r = seg_ref_f(a1x, a1y, a2x, a2y, c.vert[2 * i], c.vert[2 * i + 1], c.vert[2 * j],
                          c.vert[2 * j + 1]);
        }
        cnt += r;
    }
    return cnt;
}

template <>
inline __device__ int pair_count<float>(const Ctx<float>& c, int pl, int s, int o) {
    float a1x, a1y, a2x, a2y;
    chain_pt(c, pl, s, a1x, a1y);
    chain_pt(c, pl, s + 1, a2x, a2y);
    return pair_count_pts(c, a1x, a1y, a2x, a2y, o);
}

// First waypoint strictly inside obstacle o (geometry.hpp:217-218).
template <class T>
__device__ int contain_count_ref(const Ctx<T>& c, int pl, int o) {
    const double px = double(c.x[pl * c.D]), py = double(c.x[pl * c.D + c.W]);
    const int v0 = c.ooff[o], n = c.ooff[o + 1] - v0;
    const T* vb = c.vert + 2 * v0;
    return point_strictly_inside_ref(
        px, py, n, [vb](int i) { return double(vb[2 * i]); },
        [vb](int i) { return double(vb[2 * i + 1]); });
}

// FP32 engine fallback, out of line (rare): point (px, py) vs polygon vb[0..n)
static __device__ __noinline__ int contain_ref_f(float px, float py, const float* vb, int n) {
    return point_strictly_inside_ref(
        double(px), double(py), n, [vb](int i) { return double(vb[2 * i]); },
        [vb](int i) { return double(vb[2 * i + 1]); });
}

template <class T> __device__ int contain_count(const Ctx<T>& c, int pl, int o);
template <> inline __device__ int contain_count<double>(const Ctx<double>& c, int pl, int o) {
    return contain_count_ref(c, pl, o);
}
// FP32 engine: per edge one filtered cross c = orientation(a, b, p).  Certain
// (|c| > B) on every edge means p is off every edge line (no boundary exit) and
// the reference's rounded crossing test p.x < a.x + (b.x-a.x)(p.y-a.y)/(b.y-a.y)
// equals the exact one, i.e. (c > 0) == (b.y > a.y); B also covers the FP64
// rounding of that quotient (1e-13 M L term).  Otherwise: FP64 reference.
template <> inline __device__ int contain_count<float>(const Ctx<float>& c, int pl, int o) {
    const float px = c.x[pl * c.D], py = c.x[pl * c.D + c.W];
    const float* bb = c.obb + 4 * o;
    const float L = fmaxf(fmaxf(px, bb[2]) - fminf(px, bb[0]), fmaxf(py, bb[3]) - fminf(py, bb[1]));
    const float M = fmaxf(fmaxf(fabsf(px), fabsf(py)), fmaxf(fmaxf(fabsf(bb[0]), fabsf(bb[2])),
                                                             fmaxf(fabsf(bb[1]), fabsf(bb[3]))));
    const float B = 2.9e-6f * L * L + 1e-13f * M * L + 4e-12f;
    const int v0 = c.ooff[o], v1 = c.ooff[o + 1];
    const float4* E = reinterpret_cast<const float4*>(c.edge);
    bool inside = false;
    if (v1 - v0 == 4) {
        const float4 e[4] = {E[v0], E[v0 + 1], E[v0 + 2], E[v0 + 3]};
        float cr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) cr[i] = fmaf(e[i].z, py - e[i].y, -(e[i].w * (px - e[i].x)));
        if (!(fminf(fminf(fabsf(cr[0]), fabsf(cr[1])), fminf(fabsf(cr[2]), fabsf(cr[3]))) > B))
            return contain_ref_f(px, py, c.vert + 2 * v0, 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float ay = e[i].y, by = e[(i + 1) & 3].y;
            if ((ay > py) != (by > py) && ((cr[i] > 0.f) == (by > ay))) inside = !inside;
        }
        return inside ? 1 : 0;
    }
    for (int i = v0; i < v1; ++i) {
        const float4 e = E[i];                       // a = (e.x, e.y), b - a = (e.z, e.w)
        const float cr = fmaf(e.z, py - e.y, -(e.w * (px - e.x)));
        if (!(fabsf(cr) > B)) return contain_ref_f(px, py, c.vert + 2 * v0, v1 - v0);
        const int j = (i + 1 == v1) ? v0 : i + 1;
        const float ay = e.y, by = c.vert[2 * j + 1];
        if ((ay > py) != (by > py) && ((cr > 0.f) == (by > ay))) inside = !inside;
    }
    return inside ? 1 : 0;
}

template <class T>
__device__ __forceinline__ bool box_overlap(T lx, T ly, T hx, T hy, const T* bb, T m) {
    return lx <= bb[2] + m && bb[0] <= hx + m && ly <= bb[3] + m && bb[1] <= hy + m;
}
template <>
__device__ __forceinline__ bool box_overlap<float>(float lx, float ly, float hx, float hy,
                                                   const float* bb, float m) {
    const float4 b = *reinterpret_cast<const float4*>(bb);      // one LDS.128
    return lx <= b.z + m && b.x <= hx + m && ly <= b.w + m && b.y <= hy + m;
}

#ifndef SEPSO_BOX_UNROLL
#define SEPSO_BOX_UNROLL 8
#endif
constexpr int kBoxUnroll = SEPSO_BOX_UNROLL;
// Total order key for a fitness value: orderable bits (+0 canonical), so the
// group argmin can use 32-bit warp reductions (REDUX).
__device__ __forceinline__ uint32_t order_key(float f) {
    const uint32_t u = __float_as_uint(f == 0.f ? 0.f : f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Stage one world record (double) into shared memory as T: vertices, edge
// records (b1, b2 - b1), obstacle boxes (geometry.hpp:167-177) and the
// short-edge flag; sets endpoints, the cull margin and the path search box
// (geometry.hpp:252-255).
template <class T>
__device__ void world_regs(Ctx<T>& c, const unsigned char* wrec) {
    const WorldHeader* wh = reinterpret_cast<const WorldHeader*>(wrec);
    c.O = int(wh->n_obs);
    c.sx = T(wh->sx); c.sy = T(wh->sy); c.tx = T(wh->tx); c.ty = T(wh->ty);
    const T width = T(wh->width), height = T(wh->height);
    c.margin = sizeof(T) == 8 ? T(1e-9) : T(1e-6) * (T(1) + (width > height ? width : height));
}

// threads [0, nthr) fill the world tables; bar = named barrier id (0: __syncthreads)
template <class T>
__device__ void load_world(Ctx<T>& c, const unsigned char* wrec, int off_offsets, int off_verts,
                           int tid = threadIdx.x, int nthr = blockDim.x, int bar = 0) {
    using A = Ar<T>;
    const WorldHeader* wh = reinterpret_cast<const WorldHeader*>(wrec);
    const uint32_t* woff = reinterpret_cast<const uint32_t*>(wrec + off_offsets);
    const double* wv = reinterpret_cast<const double*>(wrec + off_verts);
    c.O = int(wh->n_obs);
    const int nv = int(wh->n_verts);
    c.sx = T(wh->sx); c.sy = T(wh->sy); c.tx = T(wh->tx); c.ty = T(wh->ty);
    const T width = T(wh->width), height = T(wh->height);
    // FP32 engine: the world is the FP32-rounded world; the cull margin is
    // conservative (never drops a pair the reference's 1e-9 cull keeps).
    c.margin = sizeof(T) == 8 ? T(1e-9) : T(1e-6) * (T(1) + (width > height ? width : height));
    #pragma unroll 1
    for (int d = tid; d < c.D; d += nthr) {
        c.lo[d] = T(0);
        c.hi[d] = d < c.W ? width : height;                  // geometry.hpp:252-255
    }
    #pragma unroll 1
    for (int i = tid; i <= c.O; i += nthr) c.ooff[i] = int(woff[i]);
    #pragma unroll 1
    for (int i = tid; i < 2 * nv; i += nthr) c.vert[i] = T(wv[i]);
    if (c.vert64 != nullptr) {      // FP64 copy: vertices, then start and target
        #pragma unroll 1
        for (int i = tid; i < 2 * nv; i += nthr) c.vert64[i] = wv[i];
        if (tid == 0) {
            c.vert64[2 * nv] = wh->sx; c.vert64[2 * nv + 1] = wh->sy;
            c.vert64[2 * nv + 2] = wh->tx; c.vert64[2 * nv + 3] = wh->ty;
        }
    }
    if (bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nthr) : "memory");
    #pragma unroll 1
    for (int o = tid; o < c.O; o += nthr) {                  // bbox_of, geometry.hpp:167-177
        const int v0 = c.ooff[o], v1 = c.ooff[o + 1];
        T bx0 = c.vert[2 * v0], by0 = c.vert[2 * v0 + 1], bx1 = bx0, by1 = by0;
        bool long_edges = true;
        for (int i = v0; i < v1; ++i) {
            const T vx = c.vert[2 * i], vy = c.vert[2 * i + 1];
            bx0 = vx < bx0 ? vx : bx0;
            by0 = vy < by0 ? vy : by0;
            bx1 = bx1 < vx ? vx : bx1;
            by1 = by1 < vy ? vy : by1;
            const int j = (i + 1 == v1) ? v0 : i + 1;
            const T ex = A::sub(c.vert[2 * j], vx), ey = A::sub(c.vert[2 * j + 1], vy);
            if (c.edge != nullptr) {
                T* e = c.edge + 4 * i;
                e[0] = vx;
                e[1] = vy;
                e[2] = ex;
                e[3] = ey;
            }
            const T ax = ex < T(0) ? -ex : ex, ay = ey < T(0) ? -ey : ey;
            long_edges &= (ax > ay ? ax : ay) >= T(1e-3);
        }
        T* bb = c.obb + 4 * o;
        bb[0] = bx0; bb[1] = by0; bb[2] = bx1; bb[3] = by1;
        c.ofl[o] = long_edges ? 1 : 0;
    }
}

// Path fitness of the CTA's particles into c.fit (before pbest logic).
//   A1  one thread per (particle, segment): segment length, obstacle-box cull
//       into a 32-bit mask per obstacle chunk, then every overlapping obstacle
//       evaluated in place (vertex-cross early exit, filtered pair test, FP64
//       fallback); first-waypoint containment tasks continue the item space.
//   A3  fitness = sum of lengths in chain order + alpha * Q^beta.
// RING: compacted pair tests (throughput launches, stage evaluation); the
// latency launch instantiates the in-place variant only (smaller hot loop).
// pbest (runner.hpp:73-80) of local row pl with this iteration's fitness f,
// incl. the x -> pbest_x row copy and the non-finite detection (runner.hpp:56-61)
template <class T>
__device__ __forceinline__ void pbest_row(Ctx<T>& c, int pl, T f) {
    if (!isfinite(f)) atomicMin(&c.m->bad_row, c.row0 + pl);
    if (f < c.pbf[pl]) {
        c.pbf[pl] = f;
        c.pbq[pl] = c.q[pl];
        const T* xs = c.x + pl * c.D;
        T* ps = c.pb + pl * c.D;
        if (sizeof(T) == 4 && (c.D & 3) == 0) {
#pragma unroll 1
            for (int d = 0; d < c.D; d += 4)
                *reinterpret_cast<float4*>(ps + d) = *reinterpret_cast<const float4*>(xs + d);
        } else {
            for (int d = 0; d < c.D; ++d) ps[d] = xs[d];
        }
    }
    c.q[pl] = 0;
}

template <class T, bool RING = true>
__device__ void path_fitness_phase(const SwarmParams& p, Ctx<T>& c, long long* prof_ = nullptr,
                                   int k = 0, bool fuse_pbest = false) {
    long long* const prof = kProfiling ? prof_ : nullptr;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int S = c.S, items = c.P * S, O = c.O;
    // ---- A1
    if (RING && c.list != nullptr) {
        // Items in warp-wide rounds; the (item, obstacle) pairs whose boxes
        // overlap are compacted into a per-warp ring of 64 entries and tested
        // 32 at a time by all lanes -- no lane idles while another works
        // through a long list of overlaps.
        const int lane = tid & 31, warp = tid >> 5;
        const unsigned lt_mask = (1u << lane) - 1u;
        uint32_t* ring = c.list + warp * 64;
        int head = 0, pend = 0;
        auto drain = [&](int n) {
            if (lane < n) {
                const uint32_t en = ring[(head + lane) & 63];
                const int epl = int(en >> 19), es = int((en >> 11) & 0xffu), eo = int(en & 0x7ffu);
                T b1x, b1y, b2x, b2y;
                chain_pt(c, epl, es, b1x, b1y);
                chain_pt(c, epl, es + 1, b2x, b2y);
                const int r = pair_count_pts(c, b1x, b1y, b2x, b2y, eo);
                if (r) atomicAdd(&c.q[epl], r);
            }
            head += n;
            pend -= n;
        };
        for (int base = warp * 32; base < items; base += nthr) {
            const int it = base + lane;
            const bool valid = it < items;
            const int pl = valid ? int(c.fS.div(uint32_t(it))) : 0, s = it - pl * S;
            T lx = T(0), ly = T(0), hx = T(0), hy = T(0);
            if (valid) {
                T a1x, a1y, a2x, a2y;
                chain_pt(c, pl, s, a1x, a1y);
                chain_pt(c, pl, s + 1, a2x, a2y);
                c.seglen[pl * S + s] = seg_length<T>(Ar<T>::sub(a2x, a1x), Ar<T>::sub(a2y, a1y));
                lx = a1x < a2x ? a1x : a2x; hx = a1x < a2x ? a2x : a1x;
                ly = a1y < a2y ? a1y : a2y; hy = a1y < a2y ? a2y : a1y;
            }
            if (prof && it == tid) prof[(k - 1) * kProfPhases + 1] = clock64();
            for (int o0 = 0; o0 < O; o0 += 32) {
                uint32_t mask = 0;
                if (valid) {
                    const int oe = min(32, O - o0);
#pragma unroll kBoxUnroll
                    for (int j = 0; j < oe; ++j)
                        if (box_overlap(lx, ly, hx, hy, c.obb + 4 * (o0 + j), c.margin)) mask |= 1u << j;
                }
                unsigned any = __reduce_or_sync(0xffffffffu, mask);
                while (any) {
                    const int j = __ffs(any) - 1;
                    any &= any - 1;
                    const bool ov = (mask >> j) & 1u;
                    const unsigned m = __ballot_sync(0xffffffffu, ov);
                    if (ov) ring[(head + pend + __popc(m & lt_mask)) & 63] = pack_entry(pl, s, o0 + j);
                    pend += __popc(m);
                    __syncwarp();
                    if (pend >= 32) {
                        drain(32);
                        __syncwarp();
                    }
                }
            }
            if (prof && it == tid) prof[(k - 1) * kProfPhases + 2] = clock64();
        }
        if (pend > 0) drain(pend);
    } else {
        const int step_pl = int(c.fS.div(uint32_t(nthr))), step_s = nthr - step_pl * S;
        int pl = int(c.fS.div(uint32_t(tid))), s = tid - pl * S;
        for (int it = tid; it < items; it += nthr) {
            T a1x, a1y, a2x, a2y;
            chain_pt(c, pl, s, a1x, a1y);
            chain_pt(c, pl, s + 1, a2x, a2y);
            c.seglen[pl * S + s] = seg_length<T>(Ar<T>::sub(a2x, a1x), Ar<T>::sub(a2y, a1y));
            const T lx = a1x < a2x ? a1x : a2x, hx = a1x < a2x ? a2x : a1x;
            const T ly = a1y < a2y ? a1y : a2y, hy = a1y < a2y ? a2y : a1y;
            int cnt = 0;
            for (int o0 = 0; o0 < O; o0 += 32) {
                uint32_t mask = 0;
                const int oe = min(32, O - o0);
#pragma unroll kBoxUnroll
                for (int j = 0; j < oe; ++j)
                    if (box_overlap(lx, ly, hx, hy, c.obb + 4 * (o0 + j), c.margin)) mask |= 1u << j;
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1;
                    cnt += pair_count_pts(c, a1x, a1y, a2x, a2y, o0 + j);
                }
            }
            if (cnt) atomicAdd(&c.q[pl], cnt);
            pl += step_pl;
            s += step_s;
            if (s >= S) { s -= S; ++pl; }
        }
    }
    {
        // first waypoint strictly inside an obstacle (geometry.hpp:217-218):
        // particle tasks continue the item index space so they land on the
        // threads with the fewest items
        for (int t = tid - (items % nthr); t < c.P; t += nthr) {
            if (t < 0) continue;
            const T wx = c.x[t * c.D], wy = c.x[t * c.D + c.W];
            int hits = 0;
            for (int o = 0; o < O; ++o) {
                const T* bb = c.obb + 4 * o;
                if (wx >= bb[0] - c.margin && wx <= bb[2] + c.margin && wy >= bb[1] - c.margin &&
                    wy <= bb[3] + c.margin)
                    hits += contain_count(c, t, o);
            }
            if (hits) atomicAdd(&c.q[t], hits);
        }
        if (prof) prof[(k - 1) * kProfPhases + 3] = clock64();
    }
    __syncthreads();
    // ---- A3 (+ the pbest update of the row, by the same thread, when fused)
    for (int pl = tid; pl < c.P; pl += nthr) {
        T len = T(0);
        for (int s = 0; s < S; ++s) len = Ar<T>::add(len, c.seglen[pl * S + s]);
        const double pen = penalty(p.alpha, p.beta, p.beta_int, c.q[pl]);
        const T f = Ar<T>::add(len, T(pen));
        if (fuse_pbest) pbest_row(c, pl, f);
        else c.fit[pl] = f;
    }
}

template <class T>
__device__ void bench_fitness_phase(int kind, Ctx<T>& c) {
    if (kind == kRastrigin) {
        // the cosines of all P x D elements on every thread (one row per
        // thread would leave most of the CTA idle behind D sequential cos
        // calls), then each row's terms summed in index order by one thread:
        // the same terms and additions as bench_row<kRastrigin>
        const int PD = c.P * c.D;
        for (int e = threadIdx.x; e < PD; e += blockDim.x) c.seglen[e] = rastrigin_term<T>(c.x[e]);
        __syncthreads();
        for (int pl = threadIdx.x; pl < c.P; pl += blockDim.x) {
            const T* t = c.seglen + pl * c.D;
            T s = T(0);
            for (int i = 0; i < c.D; ++i) s = Ar<T>::add(s, t[i]);
            c.fit[pl] = s;
            c.q[pl] = 0;
        }
        return;
    }
    for (int pl = threadIdx.x; pl < c.P; pl += blockDim.x) {
        c.fit[pl] = bench_eval<T>(kind, c.x + pl * c.D, c.D);
        c.q[pl] = 0;
    }
}

} // namespace sepso
