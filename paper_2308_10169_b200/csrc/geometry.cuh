// geometry.cuh -- device geometry for the path-fitness kernel.
//
// Two tiers:
//  * "ref" functions: the reference's FP64 predicates with its exact operation
//    order and no FMA contraction (explicit __d*_rn intrinsics), so a result
//    depends only on the input bits -- geometry.hpp:98-152.  Used by the FP64
//    engine for everything and by the FP32 engine as the fallback whenever the
//    filtered FP32 predicate cannot certify a sign, and for the strict
//    containment test (geometry.hpp:135-152, 217-218).
//  * fast_pair(): FP32 orientation signs with a forward error bound.  If every
//    |cross| clears the bound, each sign equals the sign the reference's FP64
//    evaluation would report on the same inputs (and lies outside its 1e-12
//    dead band), so the pair verdict is the reference's; otherwise the caller
//    re-evaluates that pair with segments_intersect_ref.
#pragma once
#include <cstdint>

namespace sepso {

struct DOps {   // FP64 arithmetic that never contracts into FMA
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

__device__ __forceinline__ double smin(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double smax(double a, double b) { return a < b ? b : a; }  // std::max
__device__ __forceinline__ float sminf(float a, float b) { return b < a ? b : a; }
__device__ __forceinline__ float smaxf(float a, float b) { return a < b ? b : a; }

// geometry.hpp:98-107 (kOrientEps = 1e-12)
__device__ __forceinline__ int orient_ref(double ax, double ay, double bx, double by, double cx,
                                          double cy) {
    const double cross = DOps::sub(DOps::mul(DOps::sub(bx, ax), DOps::sub(cy, ay)),
                                   DOps::mul(DOps::sub(by, ay), DOps::sub(cx, ax)));
    return cross > 1e-12 ? 1 : (cross < -1e-12 ? -1 : 0);
}

// geometry.hpp:111-114
__device__ __forceinline__ bool on_segment_ref(double ax, double ay, double bx, double by,
                                               double px, double py) {
    return smin(ax, bx) <= px && px <= smax(ax, bx) && smin(ay, by) <= py && py <= smax(ay, by);
}

// geometry.hpp:120-132
static __device__ __forceinline__ bool segments_intersect_ref(double a1x, double a1y, double a2x,
                                                    double a2y, double b1x, double b1y,
                                                    double b2x, double b2y) {
    const int o1 = orient_ref(a1x, a1y, a2x, a2y, b1x, b1y);
    const int o2 = orient_ref(a1x, a1y, a2x, a2y, b2x, b2y);
    const int o3 = orient_ref(b1x, b1y, b2x, b2y, a1x, a1y);
    const int o4 = orient_ref(b1x, b1y, b2x, b2y, a2x, a2y);
    if (o1 != o2 && o3 != o4) return true;
    if (o1 == 0 && on_segment_ref(a1x, a1y, a2x, a2y, b1x, b1y)) return true;
    if (o2 == 0 && on_segment_ref(a1x, a1y, a2x, a2y, b2x, b2y)) return true;
    if (o3 == 0 && on_segment_ref(b1x, b1y, b2x, b2y, a1x, a1y)) return true;
    if (o4 == 0 && on_segment_ref(b1x, b1y, b2x, b2y, a2x, a2y)) return true;
    return false;
}

// geometry.hpp:135-152 -- strict even-odd containment.  `vx`/`vy` fetch vertex
// i of the polygon (any storage type, widened to double).
template <class VX, class VY>
__device__ __forceinline__ bool point_strictly_inside_ref(double px, double py, int n, VX vx, VY vy) {
    for (int i = 0; i < n; ++i) {
        const int j = (i + 1 == n) ? 0 : i + 1;
        const double ax = vx(i), ay = vy(i), bx = vx(j), by = vy(j);
        if (orient_ref(ax, ay, bx, by, px, py) == 0 && on_segment_ref(ax, ay, bx, by, px, py))
            return false;
    }
    bool inside = false;
    for (int i = 0; i < n; ++i) {
        const int j = (i + 1 == n) ? 0 : i + 1;
        const double ax = vx(i), ay = vy(i), bx = vx(j), by = vy(j);
        const bool crosses = (ay > py) != (by > py);
        if (crosses) {
            const double xint = DOps::add(
                ax, DOps::div(DOps::mul(DOps::sub(bx, ax), DOps::sub(py, ay)), DOps::sub(by, ay)));
            if (px < xint) inside = !inside;
        }
    }
    return inside;
}

// std::hypot as glibc 2.39 computes it for finite operands (Borges' corrected
// kernel without FMA; verified bit-identical to libm on 2e7 random pairs by
// tests/test_oracle_cpu.py::test_glibc_hypot_restatement).  Used by the FP64
// engine so path lengths match geometry.hpp:228 bit for bit.
__device__ __forceinline__ double hypot_glibc(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x;
    const double ay = x < y ? x : y;
    if (ay <= DOps::mul(ax, 0x1p-54)) return DOps::add(ax, ay);
    // (ax, ay) in the paths' range never needs the glibc rescaling branches
    // (ax > 2^511 or ay < 2^-511); those inputs fall back to the same kernel
    // after exact power-of-two scaling.
    double scale = 1.0;
    double sx = ax, sy = ay;
    if (ax > 0x1p+511) { sx = DOps::mul(ax, 0x1p-600); sy = DOps::mul(ay, 0x1p-600); scale = 0x1p+600; }
    else if (ay < 0x1p-511) { sx = DOps::div(ax, 0x1p-600); sy = DOps::div(ay, 0x1p-600); scale = 0x1p-600; }
    double h = __dsqrt_rn(DOps::add(DOps::mul(sx, sx), DOps::mul(sy, sy)));
    double t1, t2;
    if (h <= DOps::mul(2.0, sy)) {
        const double delta = DOps::sub(h, sy);
        t1 = DOps::mul(sx, DOps::sub(DOps::mul(2.0, delta), sx));
        t2 = DOps::mul(DOps::sub(delta, DOps::mul(2.0, DOps::sub(sx, sy))), delta);
    } else {
        const double delta = DOps::sub(h, sx);
        t1 = DOps::mul(DOps::mul(2.0, delta), DOps::sub(sx, DOps::mul(2.0, sy)));
        t2 = DOps::add(DOps::mul(DOps::sub(DOps::mul(4.0, delta), sy), sy), DOps::mul(delta, delta));
    }
    h = DOps::sub(h, DOps::div(DOps::add(t1, t2), DOps::mul(2.0, h)));
    return scale == 1.0 ? h : DOps::mul(h, scale);
}

// Filtered FP32 pair test.  Inputs: segment start a1, direction d = a2 - a1
// (both FP32, d rounded once), edge start b1 and edge direction e = b2 - b1
// (rounded once), and a bound `B` on the rounding error of every cross product
// below.  Uses the identities
//   o2 = o1 + d x e    and    o4 = o3 - d x e
// so one pair costs three cross products.  Returns 1 / 0 for a certified
// verdict, -1 when some |cross| <= B and the caller must use the FP64 path.
__device__ __forceinline__ int fast_pair(float a1x, float a1y, float dx, float dy, float b1x,
                                         float b1y, float ex, float ey, float B) {
    const float wx = b1x - a1x, wy = b1y - a1y;          // b1 - a1
    const float c1 = fmaf(dx, wy, -(dy * wx));           // orient(a1, a2, b1)
    const float c3 = fmaf(ey, wx, -(ex * wy));           // orient(b1, b2, a1) = e x (a1 - b1)
    const float X = fmaf(dx, ey, -(dy * ex));            // d x e
    const float c2 = c1 + X;                             // orient(a1, a2, b2)
    const float c4 = c3 - X;                             // orient(b1, b2, a2)
    const float m = fminf(fminf(fabsf(c1), fabsf(c2)), fminf(fabsf(c3), fabsf(c4)));
    if (!(m > B)) return -1;
    const uint32_t s = (__float_as_uint(c1) ^ __float_as_uint(c2)) &
                       (__float_as_uint(c3) ^ __float_as_uint(c4));
    return int(s >> 31);
}

} // namespace sepso
