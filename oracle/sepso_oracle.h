/*
 * sepso_oracle.h -- CPU restatement of the reference SEPSO hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the parity tests, smoke() and
 * bench.py's cpu_baseline leg compare the CUDA engine against.  Nothing in the
 * product (paper_2308_10169_b200/, include/) may include, link or call it.
 *
 * Pinning: every function cites the reference file:line it restates
 * (paths relative to the reference tree, proj/include/swarmforge/...).  The
 * restatement is checked against (a) the reference compiled unmodified from
 * its own headers into oracle/_ref/ (see oracle/Makefile, oracle/ref_wrap.cpp)
 * and (b) the golden vectors committed under tests/golden/ (generated from
 * oracle/_ref by tests/golden/make_golden.py) plus the known-answer constants
 * of the reference's own unit tests.
 *
 * All arithmetic is FP64 and must be compiled with -ffp-contract=off, exactly
 * like the reference's Release build (proj/CMakeLists.txt:7-13).
 */
#ifndef SEPSO_ORACLE_H
#define SEPSO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- random streams (rng.hpp) ------------------------------------------ */
enum { OR_RNG_MT19937 = 0, OR_RNG_PHILOX = 1 };

typedef struct or_rng {
    int kind;
    uint64_t seed;
    uint64_t drawn;        /* number of 64-bit words consumed so far */
    uint64_t mt[312];
    int mti;
} or_rng;

uint64_t or_splitmix64(uint64_t x);
uint64_t or_fnv1a64(const char* s);
uint64_t or_derive_seed(uint64_t root, const char* tag);
uint64_t or_derive_seed_idx(uint64_t root, const char* tag, uint64_t index);
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t or_philox_word(uint64_t seed, uint64_t index);
void or_rng_init(or_rng* r, int kind, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
double or_uniform(or_rng* r);
double or_uniform_range(or_rng* r, double lo, double hi);
/* mt19937_64 default-seed self test: 10000th output (test_rng.cpp:35-41) */
uint64_t or_mt_nth(uint64_t seed, uint64_t n);

/* ---- swarm state (swarm.hpp) -------------------------------------------- */
typedef struct or_swarm {
    size_t G, N, D;
    double *x, *v, *pbest_x, *pbest_f, *gbest_x, *gbest_f, *tbest_x;
    double tbest_f;
    size_t iteration;
} or_swarm;

or_swarm* or_swarm_new(size_t G, size_t N, size_t D);
void or_swarm_free(or_swarm* s);

/* hypers: G rows of (c1, c2, c3, omega_init, omega_end, v_limit) */
int or_init_swarm(const double* hypers, const double* lo, const double* hi, size_t G,
                  size_t N, size_t D, or_rng* rng, or_swarm* s);
int or_step(or_swarm* s, const double* hypers, const double* lo, const double* hi,
            or_rng* rng, size_t k, size_t T);
void or_update_bests(or_swarm* s, const double* fitness);

/* ---- geometry (geometry.hpp) -------------------------------------------- */
typedef struct or_world {
    double width, height;
    double start[2], target[2], start_vel[2], target_vel[2];
    size_t n_obstacles;
    const uint32_t* offsets;  /* n_obstacles + 1 vertex offsets */
    const double* verts;      /* (x, y) pairs */
    const double* obs_vel;    /* (vx, vy) per obstacle, may be NULL */
} or_world;

int or_orientation(const double* a, const double* b, const double* c);
int or_segments_intersect(const double* a1, const double* a2, const double* b1,
                          const double* b2);
int or_point_strictly_inside(const double* p, const double* poly, size_t n);
size_t or_count_intersections(const double* particle, size_t D, const or_world* w);
double or_path_length(const double* particle, size_t D, const or_world* w);
double or_path_fitness(const double* particle, size_t D, const or_world* w, double alpha,
                       double beta);
void or_eval_path_rows(const double* xs, size_t rows, size_t D, const or_world* w,
                       double alpha, double beta, double* out, uint32_t* q_out);

/* ---- benchmarks (benchmarks.hpp) + Ackley extension ---------------------- */
enum { OR_PROB_PATH = 0, OR_PROB_SPHERE = 1, OR_PROB_ROSENBROCK = 2,
       OR_PROB_RASTRIGIN = 3, OR_PROB_GRIEWANK = 4, OR_PROB_ACKLEY = 5 };
double or_bench_eval(int kind, const double* p, size_t D);

typedef struct or_problem {
    int kind;
    size_t D;
    const double* lo;
    const double* hi;
    const or_world* world; /* kind == OR_PROB_PATH */
    double alpha, beta;
} or_problem;

void or_problem_eval(const or_problem* p, const double* xs, size_t rows, double* out);

/* ---- runner (runner.hpp) ------------------------------------------------ */
/* returns 0 ok, 1 invalid argument, 2 non-finite fitness (bad = g, n, k) */
int or_run_dtpso(const or_problem* p, const double* hypers, size_t G, size_t N, size_t T,
                 uint64_t seed, int rng_kind, double* trace, double* final_point,
                 double* final_fitness, size_t bad[3]);

/* ---- planner (planner.hpp) ---------------------------------------------- */
typedef struct or_planner_cfg {
    double alpha, beta, gamma, delta;
    size_t tw;
    double pi_radius;
    size_t max_iters, G, N, D;
    int auto_truncate, window_carryover;
} or_planner_cfg;

typedef struct or_plan_record {
    double fitness, length;
    size_t intersections, iterations;
    int truncated, collision_free;
} or_plan_record;

int or_priori_init(const double* prev_particle, const double* hypers, const double* lo,
                   const double* hi, const or_planner_cfg* cfg, or_rng* rng, or_swarm* s);
int or_should_truncate(const double* window, size_t len, int best_cf,
                       const or_planner_cfg* cfg);
/* prev_particle: encoded previous best (D values) or NULL.
 * window: capacity >= tw, in/out with *window_len (used when carryover). */
int or_plan_frame(const or_world* w, const double* prev_particle, const double* hypers,
                  const or_planner_cfg* cfg, uint64_t seed, int rng_kind, double* window,
                  size_t* window_len, or_plan_record* rec, double* best_particle,
                  size_t bad[3]);

/* ---- HSEF (hsef.hpp) ---------------------------------------------------- */
void or_unflatten(const double* particle, size_t groups, double* hypers_out);
double or_lfv_fitness(const double* candidate, size_t groups, const or_problem* p,
                      size_t iG, size_t iN, size_t iT, uint64_t seed, int rng_kind);
int or_evolve(const or_problem* p, size_t iG, size_t iN, size_t iT, size_t oG, size_t oN,
              size_t E, uint64_t seed, const double* outer_hypers, int rng_kind,
              double* best_trace, double* round_trace, double* best_hypers);

/* ---- scenario (simenv.hpp) ---------------------------------------------- */
typedef struct or_scenario_cfg {
    double map_size;
    size_t dynamic_obstacles, static_obstacles;
    double min_side, max_side, max_speed, start_speed, target_speed;
    double dt;
} or_scenario_cfg;

/* writes a rectangle world: offsets (n+1), verts (8n), vel (2n), kinds (n) */
int or_generate_world(const or_scenario_cfg* c, uint64_t seed, int rng_kind,
                      double* head /* w,h,start,target,sv,tv = 10 */, uint32_t* offsets,
                      double* verts, double* vel, uint8_t* kinds);
void or_step_world(double* head, size_t n_obstacles, const uint32_t* offsets, double* verts,
                   double* vel, double dt);


/* ---- flat wrappers for the Python harness ------------------------------- */
int or_init_swarm_seed(const double* hypers, const double* lo, const double* hi, size_t G,
                       size_t N, size_t D, uint64_t seed, int rng_kind, const double* prev,
                       size_t warm, double pi_radius, double* x, double* v);
int or_step_seed(const double* hypers, const double* lo, const double* hi, size_t G, size_t N,
                 size_t D, double* x, double* v, const double* pbx, const double* gbx,
                 const double* tbx, uint64_t seed, int rng_kind, uint64_t skip, size_t k,
                 size_t T);
void or_update_bests_arrays(size_t G, size_t N, size_t D, const double* x, double* pbx,
                            double* pbf, double* gbx, double* gbf, double* tbx, double* tbf,
                            const double* fitness);
int or_run_dtpso_flat(int kind, const or_world* w, size_t D, const double* lo, const double* hi,
                      double alpha, double beta, const double* hypers, size_t G, size_t N,
                      size_t T, uint64_t seed, int rng_kind, double* trace, double* final_point,
                      double* final_fitness, size_t bad[3]);
double or_lfv_flat(const double* cand, size_t groups, int kind, const or_world* w, size_t D,
                   const double* lo, const double* hi, double alpha, double beta, size_t iG,
                   size_t iN, size_t iT, uint64_t seed, int rng_kind);
int or_evolve_flat(int kind, const or_world* w, size_t D, const double* lo, const double* hi,
                   double alpha, double beta, size_t iG, size_t iN, size_t iT, size_t oG,
                   size_t oN, size_t E, uint64_t seed, const double* outer_hypers, int rng_kind,
                   double* best_trace, double* round_trace, double* best_hypers);

#ifdef __cplusplus
}
#endif
#endif
