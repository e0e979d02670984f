/*
 * sepso_oracle.c -- CPU restatement of the reference SEPSO hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see sepso_oracle.h).  Plain C11, FP64, built with
 * -ffp-contract=off so every product/sum rounds exactly where the reference's
 * Release build rounds (proj/CMakeLists.txt:7-13).  Citations are
 * "file:line" in /root/reference/proj/include/swarmforge/.
 */
#include "sepso_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* std::min / std::max semantics (first argument wins ties) */
static inline double smin(double a, double b) { return b < a ? b : a; }
static inline double smax(double a, double b) { return a < b ? b : a; }

/* ========================================================================= */
/* rng.hpp                                                                   */
/* ========================================================================= */

/* rng.hpp:32-37 */
uint64_t or_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* rng.hpp:39-46 (FNV-1a 64 over the tag bytes) */
uint64_t or_fnv1a64(const char* s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (const unsigned char* p = (const unsigned char*)s; *p; ++p) {
        h ^= *p;
        h *= 0x100000001b3ull;
    }
    return h;
}

/* rng.hpp:52-54 */
uint64_t or_derive_seed(uint64_t root, const char* tag) {
    return or_splitmix64(root ^ or_fnv1a64(tag));
}

/* rng.hpp:56-59 */
uint64_t or_derive_seed_idx(uint64_t root, const char* tag, uint64_t index) {
    return or_splitmix64(or_derive_seed(root, tag) + index);
}

/* mt19937_64 as fixed by the C++ standard ([rand.eng.mers], parameters of
 * std::mt19937_64); the reference draws from it at rng.hpp:18,26. */
#define MT_N 312
#define MT_M 156
static void mt_seed(or_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = MT_N;
}

static uint64_t mt_next(or_rng* r) {
    static const uint64_t mag[2] = {0ull, 0xB5026F5AA96619E9ull};
    const uint64_t upper = 0xFFFFFFFF80000000ull, lower = 0x7FFFFFFFull;
    if (r->mti >= MT_N) {
        int i;
        uint64_t y;
        for (i = 0; i < MT_N - MT_M; ++i) {
            y = (r->mt[i] & upper) | (r->mt[i + 1] & lower);
            r->mt[i] = r->mt[i + MT_M] ^ (y >> 1) ^ mag[y & 1u];
        }
        for (; i < MT_N - 1; ++i) {
            y = (r->mt[i] & upper) | (r->mt[i + 1] & lower);
            r->mt[i] = r->mt[i + (MT_M - MT_N)] ^ (y >> 1) ^ mag[y & 1u];
        }
        y = (r->mt[MT_N - 1] & upper) | (r->mt[0] & lower);
        r->mt[MT_N - 1] = r->mt[MT_M - 1] ^ (y >> 1) ^ mag[y & 1u];
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

uint64_t or_mt_nth(uint64_t seed, uint64_t n) {
    or_rng r;
    or_rng_init(&r, OR_RNG_MT19937, seed);
    uint64_t w = 0;
    for (uint64_t i = 0; i < n; ++i) w = mt_next(&r);
    return w;
}

/* Philox4x32-10 (Salmon et al., SC'11): the engine's counter-based stream.
 * Multipliers 0xD2511F53 / 0xCD9E8D57, Weyl key bumps 0x9E3779B9 / 0xBB67AE85. */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Draw contract: word i of stream `seed` = half (i & 1) of Philox block i >> 1,
 * counter = (lo32(i>>1), hi32(i>>1), 0, 0), key = (lo32(seed), hi32(seed)). */
uint64_t or_philox_word(uint64_t seed, uint64_t index) {
    const uint64_t blk = index >> 1;
    const uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    or_philox4x32_10(ctr, key, o);
    return (index & 1) ? (((uint64_t)o[3] << 32) | o[2]) : (((uint64_t)o[1] << 32) | o[0]);
}

void or_rng_init(or_rng* r, int kind, uint64_t seed) {
    r->kind = kind;
    r->seed = seed;
    r->drawn = 0;
    r->mti = MT_N;
    if (kind == OR_RNG_MT19937) mt_seed(r, seed);
}

uint64_t or_rng_next(or_rng* r) {
    const uint64_t i = r->drawn++;
    return r->kind == OR_RNG_MT19937 ? mt_next(r) : or_philox_word(r->seed, i);
}

/* rng.hpp:18 */
double or_uniform(or_rng* r) { return (double)(or_rng_next(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:21 */
double or_uniform_range(or_rng* r, double lo, double hi) {
    return lo + or_uniform(r) * (hi - lo);
}

/* ========================================================================= */
/* swarm.hpp                                                                 */
/* ========================================================================= */

or_swarm* or_swarm_new(size_t G, size_t N, size_t D) {
    or_swarm* s = (or_swarm*)calloc(1, sizeof(or_swarm));
    s->G = G; s->N = N; s->D = D;
    s->x = (double*)calloc(G * N * D, sizeof(double));
    s->v = (double*)calloc(G * N * D, sizeof(double));
    s->pbest_x = (double*)calloc(G * N * D, sizeof(double));
    s->pbest_f = (double*)calloc(G * N, sizeof(double));
    s->gbest_x = (double*)calloc(G * D, sizeof(double));
    s->gbest_f = (double*)calloc(G, sizeof(double));
    s->tbest_x = (double*)calloc(D, sizeof(double));
    for (size_t i = 0; i < G * N; ++i) s->pbest_f[i] = INFINITY;   /* swarm.hpp:113 */
    for (size_t g = 0; g < G; ++g) s->gbest_f[g] = INFINITY;       /* swarm.hpp:115 */
    s->tbest_f = INFINITY;                                          /* swarm.hpp:27 */
    return s;
}

void or_swarm_free(or_swarm* s) {
    if (!s) return;
    free(s->x); free(s->v); free(s->pbest_x); free(s->pbest_f);
    free(s->gbest_x); free(s->gbest_f); free(s->tbest_x); free(s);
}

static int hypers_valid(const double* h, size_t G) {    /* hypers.hpp:31-46 */
    if (G == 0) return 0;
    for (size_t g = 0; g < G; ++g) {
        const double* r = h + 6 * g;
        for (int f = 0; f < 6; ++f)
            if (!isfinite(r[f])) return 0;
        if (r[0] < 0 || r[1] < 0 || r[2] < 0) return 0;
        if (!(0.0 <= r[4] && r[4] <= r[3] && r[3] <= 1.0)) return 0;
        if (!(0.0 < r[5] && r[5] <= 1.0)) return 0;
    }
    return 1;
}

static int bounds_valid(const double* lo, const double* hi, size_t D) { /* hypers.hpp:109-120 */
    if (D == 0) return 0;
    for (size_t d = 0; d < D; ++d) {
        if (!isfinite(lo[d]) || !isfinite(hi[d])) return 0;
        if (!(lo[d] < hi[d])) return 0;
    }
    return 1;
}

/* swarm.hpp:118-130: all velocities after all positions, per group vmax */
static void draw_velocities(or_swarm* s, const double* hypers, const double* lo,
                            const double* hi, or_rng* rng) {
    const size_t N = s->N, D = s->D;
    for (size_t g = 0; g < s->G; ++g) {
        const double vl = hypers[6 * g + 5];
        double* vg = s->v + g * N * D;
        for (size_t i = 0; i < N * D; ++i) {
            const double vmax = vl * (hi[i % D] - lo[i % D]);
            vg[i] = or_uniform_range(rng, -vmax, vmax);
        }
    }
}

/* swarm.hpp:94-132 */
int or_init_swarm(const double* hypers, const double* lo, const double* hi, size_t G,
                  size_t N, size_t D, or_rng* rng, or_swarm* s) {
    if (!hypers_valid(hypers, G) || !bounds_valid(lo, hi, D) || N < 1) return 1;
    const size_t total = G * N * D;
    for (size_t i = 0; i < total; ++i) {
        const size_t d = i % D;
        s->x[i] = or_uniform_range(rng, lo[d], hi[d]);
    }
    draw_velocities(s, hypers, lo, hi, rng);
    memcpy(s->pbest_x, s->x, total * sizeof(double));
    return 0;
}

static double clampd(double v, double lo, double hi) {   /* std::clamp semantics */
    return v < lo ? lo : (hi < v ? hi : v);
}

/* swarm.hpp:138-174 with draw_step_randoms (59-70) and inertia_at (74-87) */
int or_step(or_swarm* s, const double* hypers, const double* lo, const double* hi,
            or_rng* rng, size_t k, size_t T) {
    if (T == 0 || k > T) return 1;
    const size_t G = s->G, N = s->N, D = s->D, GN = G * N;
    const double frac = (double)k / (double)T;
    double* r = (double*)malloc(3 * GN * sizeof(double));
    for (size_t i = 0; i < 3 * GN; ++i) r[i] = or_uniform(rng); /* r1[], r2[], r3[] */
    const double* tb = s->tbest_x;
    for (size_t g = 0; g < G; ++g) {
        const double* h = hypers + 6 * g;
        const double w = h[3] - (h[3] - h[4]) * frac;
        const double* gb = s->gbest_x + g * D;
        for (size_t n = 0; n < N; ++n) {
            const size_t row = g * N + n;
            const double a1 = h[0] * r[row];
            const double a2 = h[1] * r[GN + row];
            const double a3 = h[2] * r[2 * GN + row];
            double* xv = s->x + row * D;
            double* vv = s->v + row * D;
            const double* pb = s->pbest_x + row * D;
            for (size_t d = 0; d < D; ++d) {
                const double vmax = h[5] * (hi[d] - lo[d]);
                double nv = w * vv[d] + a1 * (pb[d] - xv[d]) + a2 * (gb[d] - xv[d]) +
                            a3 * (tb[d] - xv[d]);
                nv = clampd(nv, -vmax, vmax);
                vv[d] = nv;
                xv[d] = clampd(xv[d] + nv, lo[d], hi[d]);
            }
        }
    }
    free(r);
    s->iteration = k;
    return 0;
}

/* runner.hpp:68-93: strict '<' everywhere, row-major scan => incumbent keeps ties */
void or_update_bests(or_swarm* s, const double* fitness) {
    const size_t N = s->N, D = s->D;
    for (size_t g = 0; g < s->G; ++g) {
        for (size_t n = 0; n < N; ++n) {
            const size_t r = g * N + n;
            if (fitness[r] < s->pbest_f[r]) {
                s->pbest_f[r] = fitness[r];
                memcpy(s->pbest_x + r * D, s->x + r * D, D * sizeof(double));
            }
        }
        for (size_t n = 0; n < N; ++n) {
            const size_t r = g * N + n;
            if (s->pbest_f[r] < s->gbest_f[g]) {
                s->gbest_f[g] = s->pbest_f[r];
                memcpy(s->gbest_x + g * D, s->pbest_x + r * D, D * sizeof(double));
            }
        }
        if (s->gbest_f[g] < s->tbest_f) {
            s->tbest_f = s->gbest_f[g];
            memcpy(s->tbest_x, s->gbest_x + g * D, D * sizeof(double));
        }
    }
}

/* ========================================================================= */
/* geometry.hpp                                                              */
/* ========================================================================= */

/* geometry.hpp:98-107, kOrientEps = 1e-12 */
int or_orientation(const double* a, const double* b, const double* c) {
    const double cross = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
    if (cross > 1e-12) return 1;
    if (cross < -1e-12) return -1;
    return 0;
}

/* geometry.hpp:111-114 */
static int on_segment(const double* a, const double* b, const double* p) {
    return smin(a[0], b[0]) <= p[0] && p[0] <= smax(a[0], b[0]) &&
           smin(a[1], b[1]) <= p[1] && p[1] <= smax(a[1], b[1]);
}

/* geometry.hpp:120-132 */
int or_segments_intersect(const double* a1, const double* a2, const double* b1,
                          const double* b2) {
    const int o1 = or_orientation(a1, a2, b1);
    const int o2 = or_orientation(a1, a2, b2);
    const int o3 = or_orientation(b1, b2, a1);
    const int o4 = or_orientation(b1, b2, a2);
    if (o1 != o2 && o3 != o4) return 1;
    if (o1 == 0 && on_segment(a1, a2, b1)) return 1;
    if (o2 == 0 && on_segment(a1, a2, b2)) return 1;
    if (o3 == 0 && on_segment(b1, b2, a1)) return 1;
    if (o4 == 0 && on_segment(b1, b2, a2)) return 1;
    return 0;
}

/* geometry.hpp:135-152: boundary -> outside, else even-odd */
int or_point_strictly_inside(const double* p, const double* poly, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        const double* a = poly + 2 * i;
        const double* b = poly + 2 * ((i + 1) % n);
        if (or_orientation(a, b, p) == 0 && on_segment(a, b, p)) return 0;
    }
    int inside = 0;
    for (size_t i = 0; i < n; ++i) {
        const double* a = poly + 2 * i;
        const double* b = poly + 2 * ((i + 1) % n);
        const int crosses = (a[1] > p[1]) != (b[1] > p[1]);
        if (crosses && p[0] < a[0] + (b[0] - a[0]) * (p[1] - a[1]) / (b[1] - a[1]))
            inside = !inside;
    }
    return inside;
}

/* chain point j of start -> w_1..w_W -> target (geometry.hpp:157-165, decode 75-84) */
static void chain_point(const double* particle, size_t W, const or_world* w, size_t j,
                        double out[2]) {
    if (j == 0) { out[0] = w->start[0]; out[1] = w->start[1]; }
    else if (j == W + 1) { out[0] = w->target[0]; out[1] = w->target[1]; }
    else { out[0] = particle[j - 1]; out[1] = particle[W + j - 1]; }
}

/* geometry.hpp:196-220 including the 1e-9-margin bbox cull (167-188) */
size_t or_count_intersections(const double* particle, size_t D, const or_world* w) {
    const size_t W = D / 2;
    size_t q = 0;
    for (size_t s = 0; s <= W; ++s) {
        double s1[2], s2[2];
        chain_point(particle, W, w, s, s1);
        chain_point(particle, W, w, s + 1, s2);
        const double lx = smin(s1[0], s2[0]), ly = smin(s1[1], s2[1]);
        const double hx = smax(s1[0], s2[0]), hy = smax(s1[1], s2[1]);
        for (size_t o = 0; o < w->n_obstacles; ++o) {
            const double* vs = w->verts + 2 * w->offsets[o];
            const size_t n = w->offsets[o + 1] - w->offsets[o];
            double bx0 = vs[0], by0 = vs[1], bx1 = vs[0], by1 = vs[1];
            for (size_t i = 0; i < n; ++i) {
                bx0 = smin(bx0, vs[2 * i]); by0 = smin(by0, vs[2 * i + 1]);
                bx1 = smax(bx1, vs[2 * i]); by1 = smax(by1, vs[2 * i + 1]);
            }
            const double m = 1e-9;
            if (!(lx <= bx1 + m && bx0 <= hx + m && ly <= by1 + m && by0 <= hy + m)) continue;
            for (size_t i = 0; i < n; ++i)
                if (or_segments_intersect(s1, s2, vs + 2 * i, vs + 2 * ((i + 1) % n))) ++q;
        }
    }
    const double first[2] = {particle[0], particle[W]};
    for (size_t o = 0; o < w->n_obstacles; ++o)
        if (or_point_strictly_inside(first, w->verts + 2 * w->offsets[o],
                                     w->offsets[o + 1] - w->offsets[o]))
            ++q;
    return q;
}

/* geometry.hpp:223-231 */
double or_path_length(const double* particle, size_t D, const or_world* w) {
    const size_t W = D / 2;
    double total = 0.0;
    for (size_t s = 0; s <= W; ++s) {
        double s1[2], s2[2];
        chain_point(particle, W, w, s, s1);
        chain_point(particle, W, w, s + 1, s2);
        total += hypot(s2[0] - s1[0], s2[1] - s1[1]);
    }
    return total;
}

/* geometry.hpp:234-241 */
double or_path_fitness(const double* particle, size_t D, const or_world* w, double alpha,
                       double beta) {
    const size_t q = or_count_intersections(particle, D, w);
    return or_path_length(particle, D, w) + alpha * pow((double)q, beta);
}

/* geometry.hpp:262-267 (+ the Q of each row, which the engine also tracks) */
void or_eval_path_rows(const double* xs, size_t rows, size_t D, const or_world* w,
                       double alpha, double beta, double* out, uint32_t* q_out) {
    for (size_t r = 0; r < rows; ++r) {
        const double* p = xs + r * D;
        const size_t q = or_count_intersections(p, D, w);
        out[r] = or_path_length(p, D, w) + alpha * pow((double)q, beta);
        if (q_out) q_out[r] = (uint32_t)q;
    }
}

/* ========================================================================= */
/* benchmarks.hpp                                                            */
/* ========================================================================= */

/* benchmarks.hpp:56-88; Ackley is an extension (not in the reference) */
double or_bench_eval(int kind, const double* p, size_t D) {
    const double pi = 3.14159265358979323846;
    switch (kind) {
    case OR_PROB_SPHERE: {
        double s = 0.0;
        for (size_t i = 0; i < D; ++i) s += p[i] * p[i];
        return s;
    }
    case OR_PROB_ROSENBROCK: {
        double s = 0.0;
        for (size_t i = 0; i + 1 < D; ++i) {
            const double a = p[i + 1] - p[i] * p[i];
            const double b = 1.0 - p[i];
            s += 100.0 * a * a + b * b;
        }
        return s;
    }
    case OR_PROB_RASTRIGIN: {
        double s = 0.0;
        for (size_t i = 0; i < D; ++i)
            s += p[i] * p[i] - 10.0 * cos(2.0 * pi * p[i]) + 10.0;
        return s;
    }
    case OR_PROB_GRIEWANK: {
        double sum = 0.0, prod = 1.0;
        for (size_t i = 0; i < D; ++i) {
            sum += p[i] * p[i];
            prod *= cos(p[i] / sqrt((double)(i + 1)));
        }
        return 1.0 + sum / 4000.0 - prod;
    }
    case OR_PROB_ACKLEY: {
        double s1 = 0.0, s2 = 0.0;
        for (size_t i = 0; i < D; ++i) {
            s1 += p[i] * p[i];
            s2 += cos(2.0 * pi * p[i]);
        }
        const double dd = (double)D;
        return -20.0 * exp(-0.2 * sqrt(s1 / dd)) - exp(s2 / dd) + 20.0 + 2.718281828459045;
    }
    }
    return NAN;
}

void or_problem_eval(const or_problem* p, const double* xs, size_t rows, double* out) {
    if (p->kind == OR_PROB_PATH) {
        or_eval_path_rows(xs, rows, p->D, p->world, p->alpha, p->beta, out, NULL);
        return;
    }
    for (size_t r = 0; r < rows; ++r) out[r] = or_bench_eval(p->kind, xs + r * p->D, p->D);
}

/* ========================================================================= */
/* runner.hpp                                                                */
/* ========================================================================= */

/* runner.hpp:56-61: first non-finite row names (g, n, k) */
static int first_nonfinite(const double* f, size_t count, size_t N, size_t k, size_t bad[3]) {
    for (size_t r = 0; r < count; ++r)
        if (!isfinite(f[r])) {
            if (bad) { bad[0] = r / N; bad[1] = r % N; bad[2] = k; }
            return 1;
        }
    return 0;
}

/* runner.hpp:97-129 */
int or_run_dtpso(const or_problem* p, const double* hypers, size_t G, size_t N, size_t T,
                 uint64_t seed, int rng_kind, double* trace, double* final_point,
                 double* final_fitness, size_t bad[3]) {
    if (T < 1 || G < 1 || N < 1) return 1;
    or_rng rng;
    or_rng_init(&rng, rng_kind, seed);
    or_swarm* s = or_swarm_new(G, N, p->D);
    if (or_init_swarm(hypers, p->lo, p->hi, G, N, p->D, &rng, s)) { or_swarm_free(s); return 1; }
    double* fit = (double*)malloc(G * N * sizeof(double));
    int status = 0;
    for (size_t k = 1; k <= T; ++k) {
        or_problem_eval(p, s->x, G * N, fit);
        if (first_nonfinite(fit, G * N, N, k, bad)) { status = 2; break; }
        or_update_bests(s, fit);
        if (trace) trace[k - 1] = s->tbest_f;
        or_step(s, hypers, p->lo, p->hi, &rng, k, T);
    }
    if (status == 0) {
        if (final_point) memcpy(final_point, s->tbest_x, p->D * sizeof(double));
        if (final_fitness) *final_fitness = s->tbest_f;
    }
    free(fit);
    or_swarm_free(s);
    return status;
}

/* ========================================================================= */
/* planner.hpp                                                               */
/* ========================================================================= */

static int cfg_valid(const or_planner_cfg* c) {    /* planner.hpp:41-56 */
    if (!(c->alpha >= 0.0) || !(c->beta >= 1.0)) return 0;
    if (!(c->gamma >= 0.0 && c->gamma <= 1.0)) return 0;
    if (c->tw < 2 || !(c->delta > 0.0) || !(c->pi_radius > 0.0)) return 0;
    if (c->max_iters < 1 || c->G < 1 || c->N < 1) return 0;
    if (c->D < 2 || c->D % 2 != 0) return 0;
    return 1;
}

/* planner.hpp:77-133 */
int or_priori_init(const double* prev, const double* hypers, const double* lo,
                   const double* hi, const or_planner_cfg* cfg, or_rng* rng, or_swarm* s) {
    if (!cfg_valid(cfg) || !hypers_valid(hypers, cfg->G) || !bounds_valid(lo, hi, cfg->D))
        return 1;
    const size_t G = cfg->G, N = cfg->N, D = cfg->D, half = D / 2;
    const size_t warm = prev ? (size_t)(cfg->gamma * (double)N) : 0;   /* planner.hpp:37-39 */
    for (size_t g = 0; g < G; ++g)
        for (size_t n = 0; n < N; ++n) {
            double* xp = s->x + (g * N + n) * D;
            if (n < warm) {
                for (size_t d = 0; d < D; ++d) {
                    /* waypoint d % half; x-block for d < half else y-block */
                    const size_t wi = d % half;
                    const double center = d < half ? prev[wi] : prev[half + wi];
                    const double l = smax(lo[d], center - cfg->pi_radius);
                    const double h = smin(hi[d], center + cfg->pi_radius);
                    xp[d] = or_uniform_range(rng, l, h);
                }
            } else {
                for (size_t d = 0; d < D; ++d) xp[d] = or_uniform_range(rng, lo[d], hi[d]);
            }
        }
    draw_velocities(s, hypers, lo, hi, rng);
    memcpy(s->pbest_x, s->x, G * N * D * sizeof(double));
    return 0;
}

/* planner.hpp:138-149: population std of the trailing tw values */
int or_should_truncate(const double* window, size_t len, int best_cf,
                       const or_planner_cfg* cfg) {
    if (len < cfg->tw) return 0;
    const double* tail = window + (len - cfg->tw);
    double mean = 0.0;
    for (size_t i = 0; i < cfg->tw; ++i) mean += tail[i];
    mean /= (double)cfg->tw;
    double var = 0.0;
    for (size_t i = 0; i < cfg->tw; ++i) var += (tail[i] - mean) * (tail[i] - mean);
    var /= (double)cfg->tw;
    return sqrt(var) < cfg->delta && best_cf;
}

/* planner.hpp:156-199.  The window buffer must hold max(*window_len, tw) + 1. */
int or_plan_frame(const or_world* w, const double* prev, const double* hypers,
                  const or_planner_cfg* cfg, uint64_t seed, int rng_kind, double* window,
                  size_t* window_len, or_plan_record* rec, double* best_particle,
                  size_t bad[3]) {
    if (!cfg_valid(cfg)) return 1;
    const size_t G = cfg->G, N = cfg->N, D = cfg->D;
    double* lo = (double*)malloc(D * sizeof(double));
    double* hi = (double*)malloc(D * sizeof(double));
    for (size_t d = 0; d < D; ++d) {      /* geometry.hpp:252-255 */
        lo[d] = 0.0;
        hi[d] = d < D / 2 ? w->width : w->height;
    }
    or_rng rng;
    or_rng_init(&rng, rng_kind, seed);
    or_swarm* s = or_swarm_new(G, N, D);
    int status = or_priori_init(prev, hypers, lo, hi, cfg, &rng, s);

    const int carry = cfg->window_carryover && window && window_len;
    double* local = (double*)malloc((cfg->tw + 1) * sizeof(double));
    double* win = carry ? window : local;
    size_t wlen = carry ? *window_len : 0;

    double* fit = (double*)malloc(G * N * sizeof(double));
    memset(rec, 0, sizeof(*rec));
    const size_t cap = cfg->max_iters;
    for (size_t k = 1; status == 0 && k <= cap; ++k) {
        or_eval_path_rows(s->x, G * N, D, w, cfg->alpha, cfg->beta, fit, NULL);
        if (first_nonfinite(fit, G * N, N, k, bad)) { status = 2; break; }
        or_update_bests(s, fit);
        rec->iterations = k;
        win[wlen++] = s->tbest_f;                      /* push_back, then trim one */
        if (wlen > cfg->tw) {
            memmove(win, win + 1, (wlen - 1) * sizeof(double));
            --wlen;
        }
        if (cfg->auto_truncate) {
            const int cf = or_count_intersections(s->tbest_x, D, w) == 0;
            if (or_should_truncate(win, wlen, cf, cfg)) {
                rec->truncated = 1;
                break;
            }
        }
        if (k < cap) or_step(s, hypers, lo, hi, &rng, k, cap);
    }
    if (status == 0) {
        rec->fitness = s->tbest_f;
        rec->length = or_path_length(s->tbest_x, D, w);
        rec->intersections = or_count_intersections(s->tbest_x, D, w);
        rec->collision_free = rec->intersections == 0;
        if (best_particle) memcpy(best_particle, s->tbest_x, D * sizeof(double));
        if (carry) *window_len = wlen;
    }
    free(fit); free(local); free(lo); free(hi);
    or_swarm_free(s);
    return status;
}

/* ========================================================================= */
/* hsef.hpp                                                                  */
/* ========================================================================= */

static const double kFieldLo[6] = {0.5, 0.5, 0.5, 0.1, 0.05, 0.05};  /* hsef.hpp:75 */
static const double kFieldHi[6] = {2.5, 2.5, 2.5, 1.0, 0.8, 1.0};    /* hsef.hpp:76 */

/* hsef.hpp:57-71: clamp to the field box, then swap an inverted inertia pair */
void or_unflatten(const double* particle, size_t groups, double* out) {
    for (size_t g = 0; g < groups; ++g) {
        double f[6];
        for (int i = 0; i < 6; ++i) f[i] = clampd(particle[6 * g + i], kFieldLo[i], kFieldHi[i]);
        if (f[4] > f[3]) { const double t = f[3]; f[3] = f[4]; f[4] = t; }
        memcpy(out + 6 * g, f, sizeof(f));
    }
}

/* hsef.hpp:108-119: any failure scores +inf */
double or_lfv_fitness(const double* candidate, size_t groups, const or_problem* p,
                      size_t iG, size_t iN, size_t iT, uint64_t seed, int rng_kind) {
    if (groups != iG) return INFINITY;
    double* h = (double*)malloc(6 * groups * sizeof(double));
    or_unflatten(candidate, groups, h);
    double best = INFINITY;
    if (hypers_valid(h, groups)) {
        double f;
        if (or_run_dtpso(p, h, iG, iN, iT, seed, rng_kind, NULL, NULL, &f, NULL) == 0) best = f;
    }
    free(h);
    return best;
}

/* hsef.hpp:125-171 */
int or_evolve(const or_problem* p, size_t iG, size_t iN, size_t iT, size_t oG, size_t oN,
              size_t E, uint64_t seed, const double* outer_hypers, int rng_kind,
              double* best_trace, double* round_trace, double* best_hypers) {
    if (E < 1 || iT < 1 || iG < 1) return 1;
    const size_t dim = 6 * iG;
    double* lo = (double*)malloc(dim * sizeof(double));
    double* hi = (double*)malloc(dim * sizeof(double));
    for (size_t g = 0; g < iG; ++g)
        for (int f = 0; f < 6; ++f) { lo[6 * g + f] = kFieldLo[f]; hi[6 * g + f] = kFieldHi[f]; }
    const uint64_t outer_seed = or_derive_seed(seed, "outer");
    const uint64_t lfv_root = or_derive_seed(seed, "lfv");
    or_rng rng;
    or_rng_init(&rng, rng_kind, outer_seed);
    or_swarm* s = or_swarm_new(oG, oN, dim);
    int status = or_init_swarm(outer_hypers, lo, hi, oG, oN, dim, &rng, s);
    const size_t cand = oG * oN;
    double* fit = (double*)malloc(cand * sizeof(double));
    uint64_t idx = 0;
    for (size_t e = 1; status == 0 && e <= E; ++e) {
        double round_best = INFINITY;
        for (size_t r = 0; r < cand; ++r) {
            const uint64_t inner_seed = or_derive_seed_idx(lfv_root, "lfv", idx++);
            fit[r] = or_lfv_fitness(s->x + r * dim, iG, p, iG, iN, iT, inner_seed, rng_kind);
            round_best = smin(round_best, fit[r]);
        }
        or_update_bests(s, fit);
        if (best_trace) best_trace[e - 1] = s->tbest_f;
        if (round_trace) round_trace[e - 1] = round_best;
        or_step(s, outer_hypers, lo, hi, &rng, e, E);
    }
    if (status == 0 && best_hypers) or_unflatten(s->tbest_x, iG, best_hypers);
    free(fit); free(lo); free(hi);
    or_swarm_free(s);
    return status;
}

/* ========================================================================= */
/* simenv.hpp                                                                */
/* ========================================================================= */

/* simenv.hpp:83-132 */
int or_generate_world(const or_scenario_cfg* c, uint64_t seed, int rng_kind, double* head,
                      uint32_t* offsets, double* verts, double* vel, uint8_t* kinds) {
    or_rng rng;
    or_rng_init(&rng, rng_kind, seed);
    const double M = c->map_size;
    head[0] = M; head[1] = M;
    head[2] = 0.5 * M; head[3] = 0.1 * M;          /* start */
    head[4] = 0.5 * M; head[5] = 0.9 * M;          /* target */
    head[6] = 0.0; head[7] = c->start_speed;
    head[8] = 0.0; head[9] = c->target_speed;
    const double clearance = 2.0;
    const size_t total = c->dynamic_obstacles + c->static_obstacles;
    for (size_t i = 0; i < total; ++i) {
        int placed = 0;
        for (int attempt = 0; attempt < 200 && !placed; ++attempt) {
            const double w = or_uniform_range(&rng, c->min_side, c->max_side);
            const double h = or_uniform_range(&rng, c->min_side, c->max_side);
            const double cx = or_uniform_range(&rng, w / 2.0, M - w / 2.0);
            const double cy = or_uniform_range(&rng, h / 2.0, M - h / 2.0);
            int covered = 0;
            for (int e = 0; e < 2; ++e) {
                const double px = head[2 + 2 * e], py = head[3 + 2 * e];
                if (px >= cx - w / 2.0 - clearance && px <= cx + w / 2.0 + clearance &&
                    py >= cy - h / 2.0 - clearance && py <= cy + h / 2.0 + clearance)
                    covered = 1;
            }
            if (covered) continue;
            double* v = verts + 8 * i;
            v[0] = cx - w / 2.0; v[1] = cy - h / 2.0;
            v[2] = cx + w / 2.0; v[3] = cy - h / 2.0;
            v[4] = cx + w / 2.0; v[5] = cy + h / 2.0;
            v[6] = cx - w / 2.0; v[7] = cy + h / 2.0;
            placed = 1;
        }
        if (!placed) return 1;
        offsets[i] = (uint32_t)(4 * i);
        if (i < c->dynamic_obstacles) {
            const double speed = c->max_speed * (1.0 - or_uniform(&rng));
            const double angle = or_uniform_range(&rng, 0.0, 2.0 * 3.14159265358979323846);
            vel[2 * i] = speed * cos(angle);
            vel[2 * i + 1] = speed * sin(angle);
            kinds[i] = 1;
        } else {
            vel[2 * i] = 0.0;
            vel[2 * i + 1] = 0.0;
            kinds[i] = 0;
        }
    }
    offsets[total] = (uint32_t)(4 * total);
    return 0;
}

/* simenv.hpp:139-149 */
static double reflect_axis(double lo, double hi, double limit, double* vel) {
    if (lo <= 0.0) { *vel = -*vel; return -2.0 * lo; }
    if (hi >= limit) { *vel = -*vel; return -2.0 * (hi - limit); }
    return 0.0;
}

/* simenv.hpp:155-184 */
void or_step_world(double* head, size_t n, const uint32_t* offsets, double* verts,
                   double* vel, double dt) {
    for (int e = 0; e < 2; ++e) {
        double* p = head + 2 + 2 * e;
        double* v = head + 6 + 2 * e;
        p[0] += v[0] * dt;
        p[1] += v[1] * dt;
        p[0] += reflect_axis(p[0], p[0], head[0], &v[0]);
        p[1] += reflect_axis(p[1], p[1], head[1], &v[1]);
    }
    for (size_t o = 0; o < n; ++o) {
        double* ov = vel + 2 * o;
        if (ov[0] == 0.0 && ov[1] == 0.0) continue;
        double* vs = verts + 2 * offsets[o];
        const size_t nv = offsets[o + 1] - offsets[o];
        for (size_t i = 0; i < nv; ++i) {
            vs[2 * i] += ov[0] * dt;
            vs[2 * i + 1] += ov[1] * dt;
        }
        double bx0 = vs[0], by0 = vs[1], bx1 = vs[0], by1 = vs[1];
        for (size_t i = 0; i < nv; ++i) {
            bx0 = smin(bx0, vs[2 * i]); by0 = smin(by0, vs[2 * i + 1]);
            bx1 = smax(bx1, vs[2 * i]); by1 = smax(by1, vs[2 * i + 1]);
        }
        const double sx = reflect_axis(bx0, bx1, head[0], &ov[0]);
        const double sy = reflect_axis(by0, by1, head[1], &ov[1]);
        if (sx != 0.0 || sy != 0.0)
            for (size_t i = 0; i < nv; ++i) {
                vs[2 * i] += sx;
                vs[2 * i + 1] += sy;
            }
    }
}

/* ========================================================================= */
/* flat wrappers for the Python test harness (seed in, arrays out)           */
/* ========================================================================= */

int or_init_swarm_seed(const double* hypers, const double* lo, const double* hi, size_t G,
                       size_t N, size_t D, uint64_t seed, int rng_kind, const double* prev,
                       size_t warm, double pi_radius, double* x, double* v) {
    or_rng rng;
    or_rng_init(&rng, rng_kind, seed);
    or_swarm* s = or_swarm_new(G, N, D);
    int st;
    if (prev) {
        or_planner_cfg cfg = {30.0, 4.0, 0.0, 10.0, 20, pi_radius, 1, G, N, D, 1, 0};
        /* priori_init takes warm = floor(gamma * N); choose gamma to give `warm` */
        cfg.gamma = (double)warm / (double)N;
        while ((size_t)(cfg.gamma * (double)N) < warm) cfg.gamma = nextafter(cfg.gamma, 2.0);
        st = or_priori_init(prev, hypers, lo, hi, &cfg, &rng, s);
    } else {
        st = or_init_swarm(hypers, lo, hi, G, N, D, &rng, s);
    }
    if (st == 0) {
        memcpy(x, s->x, G * N * D * sizeof(double));
        memcpy(v, s->v, G * N * D * sizeof(double));
    }
    or_swarm_free(s);
    return st;
}

int or_step_seed(const double* hypers, const double* lo, const double* hi, size_t G, size_t N,
                 size_t D, double* x, double* v, const double* pbx, const double* gbx,
                 const double* tbx, uint64_t seed, int rng_kind, uint64_t skip, size_t k,
                 size_t T) {
    or_rng rng;
    or_rng_init(&rng, rng_kind, seed);
    for (uint64_t i = 0; i < skip; ++i) or_rng_next(&rng);
    or_swarm* s = or_swarm_new(G, N, D);
    memcpy(s->x, x, G * N * D * sizeof(double));
    memcpy(s->v, v, G * N * D * sizeof(double));
    memcpy(s->pbest_x, pbx, G * N * D * sizeof(double));
    memcpy(s->gbest_x, gbx, G * D * sizeof(double));
    memcpy(s->tbest_x, tbx, D * sizeof(double));
    const int st = or_step(s, hypers, lo, hi, &rng, k, T);
    memcpy(x, s->x, G * N * D * sizeof(double));
    memcpy(v, s->v, G * N * D * sizeof(double));
    or_swarm_free(s);
    return st;
}

void or_update_bests_arrays(size_t G, size_t N, size_t D, const double* x, double* pbx,
                            double* pbf, double* gbx, double* gbf, double* tbx, double* tbf,
                            const double* fitness) {
    or_swarm s;
    s.G = G; s.N = N; s.D = D;
    s.x = (double*)x; s.v = NULL; s.pbest_x = pbx; s.pbest_f = pbf; s.gbest_x = gbx;
    s.gbest_f = gbf; s.tbest_x = tbx; s.tbest_f = *tbf; s.iteration = 0;
    or_update_bests(&s, fitness);
    *tbf = s.tbest_f;
}

int or_run_dtpso_flat(int kind, const or_world* w, size_t D, const double* lo, const double* hi,
                      double alpha, double beta, const double* hypers, size_t G, size_t N,
                      size_t T, uint64_t seed, int rng_kind, double* trace, double* final_point,
                      double* final_fitness, size_t bad[3]) {
    double* plo = NULL;
    double* phi = NULL;
    if (kind == OR_PROB_PATH) {
        plo = (double*)malloc(D * sizeof(double));
        phi = (double*)malloc(D * sizeof(double));
        for (size_t d = 0; d < D; ++d) { plo[d] = 0.0; phi[d] = d < D / 2 ? w->width : w->height; }
        lo = plo;
        hi = phi;
    }
    const or_problem p = {kind, D, lo, hi, w, alpha, beta};
    const int st = or_run_dtpso(&p, hypers, G, N, T, seed, rng_kind, trace, final_point,
                                final_fitness, bad);
    free(plo);
    free(phi);
    return st;
}

double or_lfv_flat(const double* cand, size_t groups, int kind, const or_world* w, size_t D,
                   const double* lo, const double* hi, double alpha, double beta, size_t iG,
                   size_t iN, size_t iT, uint64_t seed, int rng_kind) {
    double lob[64], hib[64];
    if (kind == OR_PROB_PATH) {
        for (size_t d = 0; d < D && d < 64; ++d) { lob[d] = 0.0; hib[d] = d < D / 2 ? w->width : w->height; }
        lo = lob;
        hi = hib;
    }
    const or_problem p = {kind, D, lo, hi, w, alpha, beta};
    return or_lfv_fitness(cand, groups, &p, iG, iN, iT, seed, rng_kind);
}

int or_evolve_flat(int kind, const or_world* w, size_t D, const double* lo, const double* hi,
                   double alpha, double beta, size_t iG, size_t iN, size_t iT, size_t oG,
                   size_t oN, size_t E, uint64_t seed, const double* outer_hypers, int rng_kind,
                   double* best_trace, double* round_trace, double* best_hypers) {
    double lob[64], hib[64];
    if (kind == OR_PROB_PATH) {
        for (size_t d = 0; d < D && d < 64; ++d) { lob[d] = 0.0; hib[d] = d < D / 2 ? w->width : w->height; }
        lo = lob;
        hi = hib;
    }
    const or_problem p = {kind, D, lo, hi, w, alpha, beta};
    return or_evolve(&p, iG, iN, iT, oG, oN, E, seed, outer_hypers, rng_kind, best_trace,
                     round_trace, best_hypers);
}
