/*
 * sepso.h -- C ABI of libsepso_cuda.so, the B200-native SEPSO engine.
 *
 * Plain C: POD structs, pointers and sizes, no C++ or torch types.  The C++
 * drop-in headers under include/swarmforge/ re-create the reference API
 * (proj/include/swarmforge/ headers) on top of these entry points; INTEGRATION.md
 * shows a ctypes binding.  Each entry point names the reference interface it
 * replaces (paths relative to proj/include/swarmforge/ of the reference).
 *
 * Conventions
 *  - Every call returns an sf_status.  SF_INVALID_ARGUMENT mirrors the
 *    reference's std::invalid_argument, SF_NON_FINITE its
 *    NonFiniteFitnessError(group, index, iteration) (runner.hpp:19-33) with the
 *    triple in `bad[3]`.  sf_last_error() gives a thread-local message.
 *  - Host buffers in, host buffers out; the context owns device memory, one
 *    CUDA stream and pinned staging.  One context per host thread per GPU.
 *  - Hyper matrices are G rows of (c1, c2, c3, omega_init, omega_end, v_limit),
 *    the HyperEncoding flatten order (hsef.hpp:41-55).
 *  - Particles use the reference layout: x-block then y-block (geometry.hpp:75-84).
 *  - Random streams: the reference's draw ORDER and seeds;
 *    the generator is the reference's own std::mt19937_64 by default
 *    (SF_RNG_MT19937), or the counter-based Philox4x32-10 (SF_RNG_PHILOX).
 *  - Precision: SF_FP32 is the production engine; SF_FP64 reproduces the
 *    reference's FP64 arithmetic operation for operation (parity mode).
 */
#ifndef SEPSO_H
#define SEPSO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEPSO_ABI_VERSION 2

typedef enum sf_status {
    SF_OK = 0,
    SF_INVALID_ARGUMENT = 1, /* std::invalid_argument */
    SF_NON_FINITE = 2,       /* NonFiniteFitnessError (runner.hpp:19-33) */
    SF_CUDA_ERROR = 3,
    SF_UNSUPPORTED = 4,      /* problem/shape the device engine does not cover */
    SF_RUNTIME_ERROR = 5     /* std::runtime_error (e.g. generate_world placement, simenv.hpp:116-118) */
} sf_status;

typedef enum sf_precision { SF_FP32 = 0, SF_FP64 = 1 } sf_precision;

/* Random stream.  SF_RNG_MT19937 is the reference's own
 * std::mt19937_64 stream (rng.hpp:13-28), generated on the device in the
 * reference's draw order: with SF_FP64 the engine reproduces the UNMODIFIED
 * reference bit for bit.  SF_RNG_PHILOX is the counter-based stream (random
 * access, no sequential generator) shared with the harness build
 * oracle/_ref/libsfref_philox.so.  Default: SF_RNG_MT19937. */
typedef enum sf_rng { SF_RNG_PHILOX = 0, SF_RNG_MT19937 = 1 } sf_rng;

typedef enum sf_problem_kind {   /* FitnessProblem implementations (problem.hpp:14-31) */
    SF_PROBLEM_PATH = 0,         /* PathPlanningProblem (geometry.hpp:245-279) */
    SF_PROBLEM_SPHERE = 1,       /* BenchmarkProblem BF1 (benchmarks.hpp:16-95) */
    SF_PROBLEM_ROSENBROCK = 2,   /* BF2 */
    SF_PROBLEM_RASTRIGIN = 3,    /* BF3 */
    SF_PROBLEM_GRIEWANK = 4,     /* BF4 */
    SF_PROBLEM_ACKLEY = 5        /* extension (not in the reference) */
} sf_problem_kind;

typedef struct sf_point { double x, y; } sf_point;          /* Point2, geometry.hpp:15-20 */

typedef struct sf_world {                                    /* PolygonWorld, geometry.hpp:42-67 */
    double width, height;
    sf_point start, target, start_velocity, target_velocity;
    uint32_t n_obstacles;
    const uint32_t* vertex_offsets; /* n_obstacles + 1 prefix offsets into vertices */
    const sf_point* vertices;       /* closed polygons, edge i -> (i+1) mod n */
    const sf_point* velocities;     /* per obstacle, may be NULL (all static) */
} sf_world;

typedef struct sf_planner_config {                           /* PlannerConfig, planner.hpp:19-57 */
    double alpha, beta, gamma, delta;
    uint32_t tw;
    double pi_radius;
    uint32_t max_iters_per_frame, groups, per_group, dim;
    int32_t auto_truncate, window_carryover;
} sf_planner_config;

typedef struct sf_plan_record {                              /* PlanRecord, planner.hpp:60-70 */
    double fitness, length;
    uint32_t intersections, iterations;
    int32_t truncated, collision_free;                       /* stop_reason = truncated ? "converged" : "cap" */
    double wall_seconds;
} sf_plan_record;

typedef struct sf_problem {                                  /* FitnessProblem the engine evaluates */
    int32_t kind;                                            /* sf_problem_kind */
    uint32_t dim;
    const double* lo;                                        /* benchmarks: per-dimension box */
    const double* hi;
    const sf_world* world;                                   /* path: the frozen world */
    double alpha, beta;                                      /* path penalty */
} sf_problem;

typedef struct sf_ctx sf_ctx;

/* ---- context ----------------------------------------------------------- */
int sf_abi_version(void);
const char* sf_last_error(void);
int sf_ctx_create(int device, int precision, sf_ctx** out);
int sf_ctx_destroy(sf_ctx* ctx);
int sf_ctx_precision(const sf_ctx* ctx);
void* sf_ctx_stream(sf_ctx* ctx);                            /* cudaStream_t of all launches */
int sf_ctx_synchronize(sf_ctx* ctx);
/* Launch tuning (0 = heuristic): cluster size, threads per CTA. */
int sf_ctx_set_launch(sf_ctx* ctx, int cluster, int threads);
int sf_ctx_set_rng(sf_ctx* ctx, int rng);
int sf_ctx_rng(const sf_ctx* ctx);
/* Jump-ahead polynomial of the std::mt19937_64 stream (host only): out[312]
 * = x^steps mod phi (bit i = coefficient of x^i, phi the generator's
 * characteristic polynomial).  XOR-ing the raw windows x[i .. i+311] over
 * its terms i gives the state `steps` words later (long fills start segments
 * from such states). */
int sf_mt_jump_poly(uint64_t steps, uint64_t* out);
/* Device time of the engine kernels, bracketed by CUDA events on the context
 * stream while enabled: total milliseconds and launch count since enable. */
int sf_ctx_enable_timing(sf_ctx* ctx, int enable);
int sf_ctx_kernel_time(sf_ctx* ctx, double* total_ms, uint64_t* launches);

/* ---- planning ----------------------------------------------------------- */
/* plan_frame (planner.hpp:156-199).  prev_particle: encoded previous best
 * (dim values) or NULL.  window/window_len: the carried best-fitness window
 * (used and updated only when cfg->window_carryover; capacity window_cap,
 * values oldest first).  best_particle: dim values out.  bad: 3 out or NULL. */
int sf_plan_frame(sf_ctx* ctx, const sf_world* world, const double* prev_particle,
                  const double* hypers, const sf_planner_config* cfg, uint64_t seed,
                  double* window, uint32_t* window_len, uint32_t window_cap,
                  sf_plan_record* record, double* best_particle, uint64_t* bad);
/* Optional hint for a caller that plans a sequence of frames itself (the
 * run_scenario loop, simenv.hpp:239-276): the seed of the frame AFTER the next
 * sf_plan_frame call on this context.  That call then starts the next frame's
 * mt19937_64 init walk on a spare SM while it plans, and
 * the following call with that seed skips the walk.  Consumed by the next
 * sf_plan_frame; valid = 0 clears it.  Results never depend on it.
 * (sf_run_scenario sets it itself.) */
int sf_ctx_hint_next_seed(sf_ctx* ctx, uint64_t seed, int valid);

/* Many independent planning queries in ONE launch (config 5).  Arrays are per
 * scene: worlds[n], prev (n*dim, rows used where has_prev[s]), seeds[n],
 * windows (n*tw, oldest first) + window_lens[n] (in/out when carryover),
 * records[n], best (n*dim), statuses[n] (sf_status per scene), bad (n*3). */
int sf_plan_frames_batched(sf_ctx* ctx, uint32_t n_scenes, const sf_world* worlds,
                           const double* prev, const uint8_t* has_prev, const double* hypers,
                           const sf_planner_config* cfg, const uint64_t* seeds, double* windows,
                           uint32_t* window_lens, sf_plan_record* records, double* best,
                           int32_t* statuses, uint64_t* bad);

/* ---- optimizer runs ------------------------------------------------------ */
/* run_dtpso (runner.hpp:97-129): trace (T values) and final point (dim) out. */
int sf_run_dtpso(sf_ctx* ctx, const sf_problem* problem, const double* hypers, uint32_t groups,
                 uint32_t per_group, uint32_t iterations, uint64_t seed, double* trace,
                 double* final_point, double* final_fitness, uint64_t* bad);

/* n independent run_dtpso runs of one problem in one launch; hypers per run
 * (n*G*6) or shared (hypers_per_run == 0).  statuses per run. */
int sf_run_dtpso_batched(sf_ctx* ctx, const sf_problem* problem, uint32_t n_runs,
                         const double* hypers, int hypers_per_run, uint32_t groups,
                         uint32_t per_group, uint32_t iterations, const uint64_t* seeds,
                         double* traces, double* final_points, double* final_fitness,
                         int32_t* statuses);

/* ---- HSEF (hsef.hpp) ----------------------------------------------------- */
/* lfv_fitness (hsef.hpp:108-119) for m candidates in one launch: candidates
 * are raw outer particles (m*6G), decoded by HyperEncoding::unflatten
 * (clamp + swap, hsef.hpp:57-71); failures score +inf. */
int sf_lfv_batch(sf_ctx* ctx, const sf_problem* problem, uint32_t m, const double* candidates,
                 const uint64_t* seeds, uint32_t inner_groups, uint32_t inner_per_group,
                 uint32_t inner_iterations, double* lfv_out);

/* evolve (hsef.hpp:125-171): outer PSO on the host, each evolution's
 * outer_groups*outer_per_group inner runs batched in one sf_lfv_batch launch
 * (split over the context's ranks when it is sharded, sf_ctx_set_exchange /
 * sf_ctx_init_comm).
 * best_trace/round_trace: E values; best_hypers: inner_groups*6. */
typedef void (*sf_evolution_cb)(uint32_t evolution, double best_lfv, void* user);
int sf_evolve(sf_ctx* ctx, const sf_problem* problem, uint32_t inner_groups,
              uint32_t inner_per_group, uint32_t inner_iterations, uint32_t outer_groups,
              uint32_t outer_per_group, uint32_t evolutions, uint64_t seed,
              const double* outer_hypers, double* best_trace, double* round_trace,
              double* best_hypers, sf_evolution_cb on_evolution, void* user);

/* ---- stage entry points (parity) ---------------------------------------- */
/* init_swarm (swarm.hpp:94-132) / priori_init (planner.hpp:77-133 when prev != NULL) */
int sf_init_swarm(sf_ctx* ctx, const double* hypers, const double* lo, const double* hi,
                  uint32_t groups, uint32_t per_group, uint32_t dim, uint64_t seed,
                  uint64_t first_draw, const double* prev_particle, uint32_t warm,
                  double pi_radius, double* x, double* v);
/* step (swarm.hpp:138-174) with the stream positioned at draw `first_draw` */
int sf_step(sf_ctx* ctx, const double* hypers, const double* lo, const double* hi,
            uint32_t groups, uint32_t per_group, uint32_t dim, double* x, double* v,
            const double* pbest_x, const double* gbest_x, const double* tbest_x, uint64_t seed,
            uint64_t first_draw, uint32_t k, uint32_t total_iterations);
/* update_bests (runner.hpp:68-93), in place */
int sf_update_bests(sf_ctx* ctx, uint32_t groups, uint32_t per_group, uint32_t dim,
                    const double* x, double* pbest_x, double* pbest_f, double* gbest_x,
                    double* gbest_f, double* tbest_x, double* tbest_f, const double* fitness);
/* PathPlanningProblem::evaluate_rows (geometry.hpp:262-267) + Q per row */
int sf_eval_path_rows(sf_ctx* ctx, const sf_world* world, const double* xs, uint32_t rows,
                      uint32_t dim, double alpha, double beta, double* fitness, uint32_t* q);
/* BenchmarkProblem::evaluate_rows (benchmarks.hpp:45-53) */
int sf_eval_bench_rows(sf_ctx* ctx, int kind, const double* xs, uint32_t rows, uint32_t dim,
                       double* fitness);
/* should_truncate (planner.hpp:138-149) */
int sf_should_truncate(const double* window, uint32_t len, int best_collision_free,
                       const sf_planner_config* cfg, int* result);

/* derive_seed (rng.hpp:52-59): splitmix64(root ^ fnv1a64(tag)), and with an
 * index splitmix64(derive_seed(root, tag) + index) when has_index != 0. */
uint64_t sf_derive_seed(uint64_t root, const char* tag, size_t tag_len, int has_index, uint64_t index);

/* ---- scene state (simenv.hpp; host C++) ---------------------------------- */
typedef struct sf_scenario_config {                          /* ScenarioConfig, simenv.hpp:17-40 */
    double map_size;
    uint32_t dynamic_obstacles, static_obstacles;
    double min_side, max_side, max_speed, start_speed, target_speed;
    uint32_t frames;
    double dt;
    uint64_t root_seed;
} sf_scenario_config;

/* generate_world (simenv.hpp:83-132) with the engine stream: rectangles.
 * offsets (n+1), vertices (4n), velocities (n) out; n = dynamic + static. */
int sf_generate_world(const sf_scenario_config* cfg, uint64_t seed, int rng, sf_world* world_out,
                      uint32_t* offsets, sf_point* vertices, sf_point* velocities);
/* step_world (simenv.hpp:155-184), in place on caller-owned buffers */
int sf_step_world(sf_world* world, sf_point* vertices, sf_point* velocities, double dt);
/* run_scenario (simenv.hpp:239-276): variant 0..5 = sepso, sepso-noat,
 * sepso-nopi, dtpso, dppso, pso; records[frames] out (best paths in
 * best (frames*dim) if not NULL).  evolved_hypers holds evolved_groups rows;
 * the variant's hyper matrix must have base->groups rows (priori_init,
 * planner.hpp:83-84), else SF_INVALID_ARGUMENT. */
int sf_run_scenario(sf_ctx* ctx, const sf_scenario_config* cfg, int variant, uint32_t frames,
                    const sf_planner_config* base, const double* evolved_hypers, uint32_t evolved_groups,
                    sf_plan_record* records, double* best);

/* ---- device-resident scenarios (run_scenario frame loop on the device) --- */
/* n independent scenarios (simenv.hpp:239-276) kept in HBM: worlds are made by
 * generate_world(cfgs[s], derive_seed(cfgs[s].root_seed, "world")) once; each
 * frame is ONE fused launch (seed derive_seed(root, "plan", f) derived on the
 * device, prev best and carried window chained in HBM; after planning, the
 * cluster advances the world record for the next frame, step_world on the
 * device).  `cfg` is the final planner config (variant already applied).  Up
 * to max_frames frames may be run in total. */
typedef struct sf_scene_batch sf_scene_batch;
int sf_scene_batch_create(sf_ctx* ctx, uint32_t n, const sf_scenario_config* cfgs,
                          const sf_planner_config* cfg, const double* hypers, uint32_t max_frames,
                          sf_scene_batch** out);
/* enqueue `frames` more frames on the context stream (asynchronous) */
int sf_scene_batch_run(sf_scene_batch* b, uint32_t frames);
/* synchronize and copy the records (frames x n, frame-major) of frames
 * [first, first + count) and their best particles (NULL to skip) */
int sf_scene_batch_records(sf_scene_batch* b, uint32_t first, uint32_t count,
                           sf_plan_record* records, double* best);
int sf_scene_batch_destroy(sf_scene_batch* b);

/* FP32 FFMA throughput of the device (TFLOP/s): roofline denominator probe. */
int sf_measure_fp32_peak(sf_ctx* ctx, double* tflops);
/* K1 roofline probe: the staged FP32 update kernel (step, swarm.hpp:138-174)
 * on a synthetic groups x per_group x dim swarm, L2 evicted before every
 * launch; mean CUDA-event milliseconds per launch and the algorithmic bytes
 * of one launch (20 B per element). */
int sf_measure_step_kernel(sf_ctx* ctx, uint32_t groups, uint32_t per_group, uint32_t dim, uint32_t reps,
                           double* ms_per_launch, double* bytes_per_launch);

/* ---- multi-GPU: one large swarm sharded by group (BASELINE config 4) ------ */
/* NCCL communicator owned by the context (one process per GPU).  Rank 0 makes
 * the id, the caller broadcasts it, every rank attaches.  */
int sf_comm_unique_id(uint8_t id[128]);
int sf_ctx_init_comm(sf_ctx* ctx, const uint8_t id[128], int nranks, int rank);
/* The same sharding over a host all-gather instead of NCCL (a gloo / MPI
 * process group, or ranks that share a device): fn(user, send, recv, bytes)
 * must fill recv with every rank's `bytes`-long block in rank order and
 * return 0.  Used by sf_plan_frame_sharded (the per-iteration tbest
 * candidates) and by sf_evolve (HSEF: each rank scores its share of the
 * outer candidates; the LFVs are all-gathered and the outer PSO runs
 * identically everywhere).  nranks = 1 and fn = NULL reset to one rank. */
typedef int (*sf_allgather_fn)(void* user, const void* send, void* recv, size_t bytes);
int sf_ctx_set_exchange(sf_ctx* ctx, int nranks, int rank, sf_allgather_fn fn, void* user);
/* plan_frame (planner.hpp:156-199) for one large swarm whose groups are split
 * across the communicator's ranks: rank r evaluates and updates groups
 * [r*G/n, (r+1)*G/n) in HBM with the stage kernels; per iteration the ranks
 * all-gather one population-best candidate each (~16 + 4*dim bytes) and reduce
 * it identically (group order, strict '<'), so the AT decision, the trace and
 * the record are identical on every rank and equal the unsharded run.  With no
 * communicator it runs the same HBM path on one GPU. */
int sf_plan_frame_sharded(sf_ctx* ctx, const sf_world* world, const double* prev_particle,
                          const double* hypers, const sf_planner_config* cfg, uint64_t seed,
                          double* window, uint32_t* window_len, uint32_t window_cap,
                          sf_plan_record* record, double* best_particle, uint64_t* bad);

/* Benchmark hygiene: when bytes > 0, sf_run_scenario writes a device buffer of
 * that size (flushing L2) before each frame, outside the frame's wall time. */
int sf_ctx_set_l2_flush(sf_ctx* ctx, uint64_t bytes);

/* Bytes moved host->device and device->host by the last host-buffer call. */
int sf_ctx_last_io_bytes(sf_ctx* ctx, uint64_t* h2d, uint64_t* d2h);

#ifdef __cplusplus
}
#endif
#endif
