// ref_wrap.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference headers, compiled by
// oracle/Makefile straight from /root/reference/proj/include with
// -Dswarmforge=sfref (so the reference lives in its own namespace) into
// oracle/_ref/libsfref_{mt,philox}.so.  The "philox" flavour puts
// oracle/ref_shim first on the include path so the reference's RngStream draws
// the engine's Philox counter stream (ref_shim/swarmforge/rng.hpp); the "mt"
// flavour is the reference exactly as shipped (mt19937_64).  Nothing here
// re-implements reference logic: each wrapper marshals POD buffers into the
// reference's types and calls the reference function named in its comment.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <vector>

#include "swarmforge/benchmarks.hpp"
#include "swarmforge/hsef.hpp"
#include "swarmforge/planner.hpp"
#include "swarmforge/simenv.hpp"

#include "sepso_oracle.h"

using namespace sfref;

namespace {

HyperMatrix to_hypers(const double* h, std::size_t G) {
    HyperMatrix m;
    for (std::size_t g = 0; g < G; ++g)
        m.groups.push_back({h[6 * g], h[6 * g + 1], h[6 * g + 2], h[6 * g + 3], h[6 * g + 4],
                            h[6 * g + 5]});
    return m;
}

PolygonWorld to_world(const or_world* w) {
    PolygonWorld out;
    out.width = w->width;
    out.height = w->height;
    out.start = {w->start[0], w->start[1]};
    out.target = {w->target[0], w->target[1]};
    out.start_velocity = {w->start_vel[0], w->start_vel[1]};
    out.target_velocity = {w->target_vel[0], w->target_vel[1]};
    for (std::size_t o = 0; o < w->n_obstacles; ++o) {
        Obstacle ob;
        for (std::uint32_t i = w->offsets[o]; i < w->offsets[o + 1]; ++i)
            ob.vertices.push_back({w->verts[2 * i], w->verts[2 * i + 1]});
        if (w->obs_vel) {
            ob.velocity = {w->obs_vel[2 * o], w->obs_vel[2 * o + 1]};
            ob.kind = (ob.velocity.x != 0.0 || ob.velocity.y != 0.0) ? ObstacleKind::dynamic
                                                                     : ObstacleKind::fixed;
        }
        out.obstacles.push_back(std::move(ob));
    }
    return out;
}

PlannerConfig to_cfg(const or_planner_cfg* c) {
    PlannerConfig p;
    p.alpha = c->alpha;
    p.beta = c->beta;
    p.gamma = c->gamma;
    p.delta = c->delta;
    p.tw = c->tw;
    p.pi_radius = c->pi_radius;
    p.max_iters_per_frame = c->max_iters;
    p.groups = c->G;
    p.per_group = c->N;
    p.dim = c->D;
    p.auto_truncate = c->auto_truncate != 0;
    p.window_carryover = c->window_carryover != 0;
    return p;
}

void skip(RngStream& rng, std::uint64_t n) {
    for (std::uint64_t i = 0; i < n; ++i) rng.uniform();
}

SwarmState load_state(std::size_t G, std::size_t N, std::size_t D, const double* x,
                      const double* v, const double* pbx, const double* pbf, const double* gbx,
                      const double* gbf, const double* tbx, double tbf) {
    SwarmState s;
    s.groups = G;
    s.per_group = N;
    s.dim = D;
    s.x.assign(x, x + G * N * D);
    s.v.assign(v, v + G * N * D);
    s.pbest_x.assign(pbx, pbx + G * N * D);
    s.pbest_f.assign(pbf, pbf + G * N);
    s.gbest_x.assign(gbx, gbx + G * D);
    s.gbest_f.assign(gbf, gbf + G);
    s.tbest_x.assign(tbx, tbx + D);
    s.tbest_f = tbf;
    return s;
}

std::unique_ptr<FitnessProblem> make_problem(int kind, std::size_t D, const or_world* w,
                                             double alpha, double beta) {
    if (kind == OR_PROB_PATH)
        return std::make_unique<PathPlanningProblem>(to_world(w), D, alpha, beta);
    static const char* ids[] = {"", "BF1", "BF2", "BF3", "BF4"};
    if (kind < 1 || kind > 4) throw std::invalid_argument("benchmark kind not in reference");
    return make_benchmark(ids[kind], D);
}

} // namespace

extern "C" {

// rng.hpp:18 -- first n uniforms of a stream
void ref_uniform_stream(std::uint64_t seed, std::uint64_t n, double* out) {
    RngStream rng(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = rng.uniform();
}

std::uint64_t ref_derive_seed(std::uint64_t root, const char* tag) { return derive_seed(root, tag); }
std::uint64_t ref_derive_seed_idx(std::uint64_t root, const char* tag, std::uint64_t idx) {
    return derive_seed(root, tag, idx);
}

// swarm.hpp:94-132
int ref_init_swarm(const double* hypers, std::size_t G, std::size_t N, std::size_t D,
                   const double* lo, const double* hi, std::uint64_t seed, double* x, double* v) {
    try {
        RngStream rng(seed);
        const SearchBounds b(std::vector<double>(lo, lo + D), std::vector<double>(hi, hi + D));
        const SwarmState s = init_swarm(to_hypers(hypers, G), b, G, N, D, rng);
        std::copy(s.x.begin(), s.x.end(), x);
        std::copy(s.v.begin(), s.v.end(), v);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// swarm.hpp:138-174 with the stream advanced by `skip_draws` first
int ref_step(std::size_t G, std::size_t N, std::size_t D, const double* hypers, const double* lo,
             const double* hi, double* x, double* v, const double* pbx, const double* gbx,
             const double* tbx, std::uint64_t seed, std::uint64_t skip_draws, std::size_t k,
             std::size_t T) {
    try {
        std::vector<double> pbf(G * N, 0.0), gbf(G, 0.0);
        SwarmState s = load_state(G, N, D, x, v, pbx, pbf.data(), gbx, gbf.data(), tbx, 0.0);
        const SearchBounds b(std::vector<double>(lo, lo + D), std::vector<double>(hi, hi + D));
        RngStream rng(seed);
        skip(rng, skip_draws);
        step(s, to_hypers(hypers, G), b, rng, k, T);
        std::copy(s.x.begin(), s.x.end(), x);
        std::copy(s.v.begin(), s.v.end(), v);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// runner.hpp:68-93 (in place)
void ref_update_bests(std::size_t G, std::size_t N, std::size_t D, const double* x, double* pbx,
                      double* pbf, double* gbx, double* gbf, double* tbx, double* tbf,
                      const double* fitness) {
    std::vector<double> v(G * N * D, 0.0);
    SwarmState s = load_state(G, N, D, x, v.data(), pbx, pbf, gbx, gbf, tbx, *tbf);
    update_bests(s, std::span<const double>(fitness, G * N));
    std::copy(s.pbest_x.begin(), s.pbest_x.end(), pbx);
    std::copy(s.pbest_f.begin(), s.pbest_f.end(), pbf);
    std::copy(s.gbest_x.begin(), s.gbest_x.end(), gbx);
    std::copy(s.gbest_f.begin(), s.gbest_f.end(), gbf);
    std::copy(s.tbest_x.begin(), s.tbest_x.end(), tbx);
    *tbf = s.tbest_f;
}

// geometry.hpp:120-132
int ref_segments_intersect(const double* a1, const double* a2, const double* b1, const double* b2) {
    return segments_intersect({a1[0], a1[1]}, {a2[0], a2[1]}, {b1[0], b1[1]}, {b2[0], b2[1]});
}

// geometry.hpp:135-152
int ref_point_strictly_inside(const double* p, const double* poly, std::size_t n) {
    std::vector<Point2> pts;
    for (std::size_t i = 0; i < n; ++i) pts.push_back({poly[2 * i], poly[2 * i + 1]});
    return point_strictly_inside({p[0], p[1]}, pts);
}

// geometry.hpp:196-241 per row: fitness, Q and length
void ref_eval_path_rows(const or_world* w, const double* xs, std::size_t rows, std::size_t D,
                        double alpha, double beta, double* out, std::uint32_t* q_out,
                        double* len_out) {
    const PolygonWorld world = to_world(w);
    for (std::size_t r = 0; r < rows; ++r) {
        const std::span<const double> row(xs + r * D, D);
        out[r] = path_fitness(row, world, alpha, beta);
        const Path p = decode_path(row);
        if (q_out) q_out[r] = static_cast<std::uint32_t>(count_intersections(p, world));
        if (len_out) len_out[r] = path_length(p, world);
    }
}

// benchmarks.hpp:45-53
int ref_bench_eval(int kind, const double* xs, std::size_t rows, std::size_t D, double* out) {
    try {
        const auto p = make_problem(kind, D, nullptr, 0, 0);
        p->evaluate_rows(std::span<const double>(xs, rows * D), rows, std::span<double>(out, rows));
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// runner.hpp:97-129.  status 2 = NonFiniteFitnessError (bad = g, n, k)
int ref_run_dtpso(int kind, const or_world* w, std::size_t D, double alpha, double beta,
                  const double* hypers, std::size_t G, std::size_t N, std::size_t T,
                  std::uint64_t seed, double* trace, double* final_point, double* final_f,
                  std::size_t* bad) {
    try {
        const auto p = make_problem(kind, D, w, alpha, beta);
        const RunReport r = run_dtpso(*p, to_hypers(hypers, G), G, N, T, seed);
        if (trace) std::copy(r.trace.begin(), r.trace.end(), trace);
        if (final_point) std::copy(r.final_point.begin(), r.final_point.end(), final_point);
        *final_f = r.final_fitness;
        return 0;
    } catch (const NonFiniteFitnessError& e) {
        if (bad) { bad[0] = e.group(); bad[1] = e.index_in_group(); bad[2] = e.iteration(); }
        return 2;
    } catch (const std::exception&) {
        return 1;
    }
}

// runner.hpp:135-239 -- the reference's per-particle DPPSO oracle (the `scale`
// harness's second code path, proj/tools/swarmforge.cpp:202-255); wall =
// its RunReport.wall_seconds
int ref_run_dppso_reference(int kind, const or_world* w, std::size_t D, double alpha, double beta,
                            const double* hypers, std::size_t G, std::size_t N, std::size_t T,
                            std::uint64_t seed, double* trace, double* final_point, double* final_f,
                            double* wall) {
    try {
        const auto p = make_problem(kind, D, w, alpha, beta);
        const RunReport r = run_dppso_reference(*p, to_hypers(hypers, G), G, N, T, seed);
        if (trace) std::copy(r.trace.begin(), r.trace.end(), trace);
        if (final_point) std::copy(r.final_point.begin(), r.final_point.end(), final_point);
        *final_f = r.final_fitness;
        if (wall) *wall = r.wall_seconds;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// runner.hpp:244-329 -- the classic single-swarm PSO baseline (default
// PsoParams), population particles for T iterations
int ref_run_pso_reference(int kind, const or_world* w, std::size_t D, double alpha, double beta,
                          std::size_t T, std::size_t population, std::uint64_t seed, double* trace,
                          double* final_point, double* final_f, double* wall) {
    try {
        const auto p = make_problem(kind, D, w, alpha, beta);
        const RunReport r = run_pso_reference(*p, T, population, seed);
        if (trace) std::copy(r.trace.begin(), r.trace.end(), trace);
        if (final_point) std::copy(r.final_point.begin(), r.final_point.end(), final_point);
        *final_f = r.final_fitness;
        if (wall) *wall = r.wall_seconds;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// planner.hpp:77-133
int ref_priori_init(const double* prev, const double* hypers, const or_planner_cfg* c,
                    const double* lo, const double* hi, std::uint64_t seed, double* x, double* v) {
    try {
        const PlannerConfig cfg = to_cfg(c);
        std::optional<Path> p;
        if (prev) p = decode_path(std::span<const double>(prev, c->D));
        const SearchBounds b(std::vector<double>(lo, lo + c->D), std::vector<double>(hi, hi + c->D));
        RngStream rng(seed);
        const SwarmState s = priori_init(p, to_hypers(hypers, c->G), b, cfg, rng);
        std::copy(s.x.begin(), s.x.end(), x);
        std::copy(s.v.begin(), s.v.end(), v);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// planner.hpp:138-149
int ref_should_truncate(const double* window, std::size_t len, int cf, const or_planner_cfg* c) {
    return should_truncate(std::span<const double>(window, len), cf != 0, to_cfg(c));
}

// planner.hpp:156-199.  window: in/out, capacity >= max(len, tw) + 1
int ref_plan_frame(const or_world* w, const double* prev, const double* hypers,
                   const or_planner_cfg* c, std::uint64_t seed, double* window,
                   std::size_t* window_len, or_plan_record* rec, double* best, std::size_t* bad) {
    try {
        std::optional<Path> p;
        if (prev) p = decode_path(std::span<const double>(prev, c->D));
        std::vector<double> win;
        if (window && window_len) win.assign(window, window + *window_len);
        const PlanRecord r = plan_frame(to_world(w), p, to_hypers(hypers, c->G), to_cfg(c), seed,
                                        (window && window_len) ? &win : nullptr);
        rec->fitness = r.fitness;
        rec->length = r.length;
        rec->intersections = r.intersections;
        rec->iterations = r.iterations;
        rec->truncated = r.truncated;
        rec->collision_free = r.collision_free;
        if (best) {
            const std::vector<double> e = encode_path(r.best_path);
            std::copy(e.begin(), e.end(), best);
        }
        if (window && window_len) {
            std::copy(win.begin(), win.end(), window);
            *window_len = win.size();
        }
        return 0;
    } catch (const NonFiniteFitnessError& e) {
        if (bad) { bad[0] = e.group(); bad[1] = e.index_in_group(); bad[2] = e.iteration(); }
        return 2;
    } catch (const std::exception&) {
        return 1;
    }
}

// simenv.hpp:239-276 -- one record per frame + wall seconds per frame
int ref_run_scenario(std::uint64_t root_seed, int variant, std::size_t frames,
                     const or_planner_cfg* base, or_plan_record* recs, double* wall) {
    try {
        ScenarioConfig sc;
        sc.root_seed = root_seed;
        const SimMetrics m = run_scenario(sc, static_cast<PlannerVariant>(variant), frames,
                                          to_cfg(base));
        for (std::size_t f = 0; f < frames; ++f) {
            const PlanRecord& r = m.records[f];
            recs[f].fitness = r.fitness;
            recs[f].length = r.length;
            recs[f].intersections = r.intersections;
            recs[f].iterations = r.iterations;
            recs[f].truncated = r.truncated;
            recs[f].collision_free = r.collision_free;
            if (wall) wall[f] = r.wall_seconds;
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// hsef.hpp:57-71
void ref_unflatten(const double* particle, std::size_t groups, double* out) {
    const HyperMatrix m = HyperEncoding(groups).unflatten(std::span<const double>(particle, 6 * groups));
    for (std::size_t g = 0; g < groups; ++g) {
        const GroupHypers& h = m.groups[g];
        const double row[6] = {h.c1, h.c2, h.c3, h.omega_init, h.omega_end, h.v_limit};
        std::memcpy(out + 6 * g, row, sizeof(row));
    }
}

// hsef.hpp:108-119
double ref_lfv_fitness(const double* cand, std::size_t groups, int kind, const or_world* w,
                       std::size_t D, double alpha, double beta, std::size_t iG, std::size_t iN,
                       std::size_t iT, std::uint64_t seed) {
    const auto p = make_problem(kind, D, w, alpha, beta);
    return lfv_fitness(std::span<const double>(cand, 6 * groups), HyperEncoding(groups), *p,
                       InnerBudget{iG, iN, iT}, seed);
}

// hsef.hpp:125-171
int ref_evolve(int kind, const or_world* w, std::size_t D, double alpha, double beta,
               std::size_t iG, std::size_t iN, std::size_t iT, std::size_t oG, std::size_t oN,
               std::size_t E, std::uint64_t seed, const double* outer_hypers, double* best_trace,
               double* round_trace, double* best_hypers) {
    try {
        const auto p = make_problem(kind, D, w, alpha, beta);
        const EvolutionReport r = evolve(*p, InnerBudget{iG, iN, iT}, OuterBudget{oG, oN, E},
                                         seed, to_hypers(outer_hypers, oG));
        std::copy(r.best_lfv_trace.begin(), r.best_lfv_trace.end(), best_trace);
        std::copy(r.evolution_lfv_trace.begin(), r.evolution_lfv_trace.end(), round_trace);
        for (std::size_t g = 0; g < iG; ++g) {
            const GroupHypers& h = r.best.groups[g];
            const double row[6] = {h.c1, h.c2, h.c3, h.omega_init, h.omega_end, h.v_limit};
            std::memcpy(best_hypers + 6 * g, row, sizeof(row));
        }
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// simenv.hpp:83-132 (rectangles: 4 vertices each)
int ref_generate_world(const or_scenario_cfg* c, std::uint64_t seed, double* head,
                       std::uint32_t* offsets, double* verts, double* vel, std::uint8_t* kinds) {
    try {
        ScenarioConfig sc;
        sc.map_size = c->map_size;
        sc.dynamic_obstacles = c->dynamic_obstacles;
        sc.static_obstacles = c->static_obstacles;
        sc.min_side = c->min_side;
        sc.max_side = c->max_side;
        sc.max_speed = c->max_speed;
        sc.start_speed = c->start_speed;
        sc.target_speed = c->target_speed;
        sc.dt = c->dt;
        const PolygonWorld w = generate_world(sc, seed);
        const double h[10] = {w.width, w.height, w.start.x, w.start.y, w.target.x, w.target.y,
                              w.start_velocity.x, w.start_velocity.y, w.target_velocity.x,
                              w.target_velocity.y};
        std::memcpy(head, h, sizeof(h));
        std::uint32_t off = 0;
        for (std::size_t o = 0; o < w.obstacles.size(); ++o) {
            offsets[o] = off;
            for (const Point2& p : w.obstacles[o].vertices) {
                verts[2 * off] = p.x;
                verts[2 * off + 1] = p.y;
                ++off;
            }
            vel[2 * o] = w.obstacles[o].velocity.x;
            vel[2 * o + 1] = w.obstacles[o].velocity.y;
            kinds[o] = w.obstacles[o].kind == ObstacleKind::dynamic;
        }
        offsets[w.obstacles.size()] = off;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// simenv.hpp:155-184 (in place)
void ref_step_world(double* head, std::size_t n, const std::uint32_t* offsets, double* verts,
                    double* vel, double dt) {
    or_world ow{head[0], head[1], {head[2], head[3]}, {head[4], head[5]}, {head[6], head[7]},
                {head[8], head[9]}, n, offsets, verts, vel};
    PolygonWorld w = to_world(&ow);
    for (std::size_t o = 0; o < n; ++o) w.obstacles[o].velocity = {vel[2 * o], vel[2 * o + 1]};
    const PolygonWorld nx = step_world(w, dt);
    const double h[10] = {nx.width, nx.height, nx.start.x, nx.start.y, nx.target.x, nx.target.y,
                          nx.start_velocity.x, nx.start_velocity.y, nx.target_velocity.x,
                          nx.target_velocity.y};
    std::memcpy(head, h, sizeof(h));
    for (std::size_t o = 0; o < n; ++o) {
        std::uint32_t i = offsets[o];
        for (const Point2& p : nx.obstacles[o].vertices) {
            verts[2 * i] = p.x;
            verts[2 * i + 1] = p.y;
            ++i;
        }
        vel[2 * o] = nx.obstacles[o].velocity.x;
        vel[2 * o + 1] = nx.obstacles[o].velocity.y;
    }
}

} // extern "C"
