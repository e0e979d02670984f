// swarmforge/runner.hpp -- drop-in for the reference's runner.hpp (best
// tracking and the batched run loop).  run_dtpso hands the whole run to the
// device (sf_run_dtpso: one fused launch for init + every iteration);
// update_bests runs the engine's best-tracking stage kernels.  The reference's
// per-particle oracles run_dppso_reference / run_pso_reference are CPU test
// oracles and are not part of the engine.
#pragma once

#include <chrono>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "swarmforge/engine.hpp"
#include "swarmforge/problem.hpp"
#include "swarmforge/swarm.hpp"

namespace swarmforge {

struct RunReport {
    std::string algorithm, problem;
    std::uint64_t seed = 0;
    std::size_t iterations = 0;
    std::vector<double> trace;
    std::vector<double> final_point;
    double final_fitness = 0.0;
    std::size_t evaluations = 0;
    double wall_seconds = 0.0;
};

namespace detail {
inline double monotonic_seconds() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
inline sf_problem device_problem(const FitnessProblem& p) {
    sf_problem spec{};
    if (!p.device_spec(spec))
        throw std::invalid_argument("FitnessProblem '" + p.name() +
                                    "' has no device implementation (path and BF1..BF4 only)");
    return spec;
}
} // namespace detail

inline void update_bests(SwarmState& s, std::span<const double> fitness) {
    if (fitness.size() != s.particle_count()) throw std::invalid_argument("update_bests: fitness size != particle count");
    engine::check(sf_update_bests(engine::ctx(), std::uint32_t(s.groups), std::uint32_t(s.per_group),
                                  std::uint32_t(s.dim), s.x.data(), s.pbest_x.data(), s.pbest_f.data(),
                                  s.gbest_x.data(), s.gbest_f.data(), s.tbest_x.data(), &s.tbest_f, fitness.data()));
}

inline RunReport run_dtpso(const FitnessProblem& problem, const HyperMatrix& hypers, std::size_t groups,
                           std::size_t per_group, std::size_t iterations, std::uint64_t seed) {
    if (iterations < 1) throw std::invalid_argument("run_dtpso: iteration count must be >= 1");
    if (problem.bounds().dimension() != problem.dimension())
        throw std::invalid_argument("run_dtpso: problem bounds do not match its dimension");
    hypers.validate();
    if (hypers.group_count() != groups) throw std::invalid_argument("init_swarm: hyper matrix group count != G");
    const sf_problem spec = detail::device_problem(problem);
    const double t0 = detail::monotonic_seconds();
    RunReport r;
    r.algorithm = "dtpso";
    r.problem = problem.name();
    r.seed = seed;
    r.trace.resize(iterations);
    r.final_point.resize(problem.dimension());
    const std::vector<double> h = hypers.rows();
    std::uint64_t bad[3] = {0, 0, 0};
    engine::check(sf_run_dtpso(engine::ctx(), &spec, h.data(), std::uint32_t(groups), std::uint32_t(per_group),
                               std::uint32_t(iterations), seed, r.trace.data(), r.final_point.data(),
                               &r.final_fitness, bad),
                  bad);
    r.iterations = iterations;
    r.evaluations = groups * per_group * iterations;
    r.wall_seconds = detail::monotonic_seconds() - t0;
    return r;
}

} // namespace swarmforge
