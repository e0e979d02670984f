// swarmforge/planner.hpp -- drop-in for the reference's planner.hpp:1-201.
// plan_frame runs one whole frame (PI warm start, fitness, best tracking, the
// AT window test, the update) in one device launch through sf_plan_frame; the
// carried window is kept on the host exactly as the reference keeps it.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "swarmforge/geometry.hpp"
#include "swarmforge/runner.hpp"

namespace swarmforge {

struct PlannerConfig {
    double alpha = 30.0, beta = 4.0, gamma = 0.25, delta = 10.0;
    std::size_t tw = 20;
    double pi_radius = 20.0;
    std::size_t max_iters_per_frame = 50;
    std::size_t groups = 8, per_group = 170, dim = 16;
    bool auto_truncate = true;
    bool window_carryover = false;

    std::size_t waypoints() const { return dim / 2; }
    std::size_t pi_count() const { return static_cast<std::size_t>(gamma * static_cast<double>(per_group)); }
    void validate() const {
        if (!(alpha >= 0.0) || !(beta >= 1.0)) throw std::invalid_argument("planner config: need alpha >= 0 and beta >= 1");
        if (!(gamma >= 0.0 && gamma <= 1.0)) throw std::invalid_argument("planner config: gamma must lie in [0, 1]");
        if (tw < 2) throw std::invalid_argument("planner config: tw must be >= 2");
        if (!(delta > 0.0)) throw std::invalid_argument("planner config: delta must be > 0");
        if (!(pi_radius > 0.0)) throw std::invalid_argument("planner config: pi_radius must be > 0");
        if (max_iters_per_frame < 1) throw std::invalid_argument("planner config: max_iters_per_frame must be >= 1");
        if (groups < 1 || per_group < 1) throw std::invalid_argument("planner config: G and N must be >= 1");
        if (dim < 2 || dim % 2 != 0) throw std::invalid_argument("planner config: dim must be even and >= 2");
    }
    sf_planner_config abi() const {
        return sf_planner_config{alpha, beta, gamma, delta, std::uint32_t(tw), pi_radius,
                                 std::uint32_t(max_iters_per_frame), std::uint32_t(groups),
                                 std::uint32_t(per_group), std::uint32_t(dim), auto_truncate ? 1 : 0,
                                 window_carryover ? 1 : 0};
    }
};

struct PlanRecord {
    Path best_path;
    double fitness = 0.0, length = 0.0;
    std::size_t intersections = 0, iterations = 0;
    bool truncated = false;
    std::string stop_reason;
    bool collision_free = false;
    double wall_seconds = 0.0;
};

inline SwarmState priori_init(const std::optional<Path>& prev_best, const HyperMatrix& hypers,
                              const SearchBounds& bounds, const PlannerConfig& config, RngStream& rng) {
    config.validate();
    hypers.validate();
    bounds.validate();
    if (hypers.group_count() != config.groups) throw std::invalid_argument("priori_init: hyper matrix group count != G");
    if (bounds.dimension() != config.dim) throw std::invalid_argument("priori_init: bounds dimension != planner dim");
    if (prev_best && prev_best->waypoints.size() != config.waypoints())
        throw std::invalid_argument("priori_init: previous path waypoint count mismatch");
    SwarmState s = detail::fresh_state(config.groups, config.per_group, config.dim);
    const std::vector<double> h = hypers.rows();
    std::vector<double> prev;
    if (prev_best) prev = encode_path(*prev_best);
    engine::check(sf_init_swarm(engine::ctx(), h.data(), bounds.x_lo.data(), bounds.x_hi.data(),
                                std::uint32_t(config.groups), std::uint32_t(config.per_group),
                                std::uint32_t(config.dim), rng.seed(), rng.drawn(),
                                prev_best ? prev.data() : nullptr, std::uint32_t(config.pi_count()),
                                config.pi_radius, s.x.data(), s.v.data()));
    rng.skip(2 * config.groups * config.per_group * config.dim);
    s.pbest_x = s.x;
    return s;
}

inline bool should_truncate(std::span<const double> window, bool best_is_collision_free, const PlannerConfig& config) {
    const sf_planner_config c = config.abi();
    int r = 0;
    engine::check(sf_should_truncate(window.data(), std::uint32_t(window.size()), best_is_collision_free ? 1 : 0, &c, &r));
    return r != 0;
}

inline PlanRecord plan_frame(const PolygonWorld& world, const std::optional<Path>& prev_best,
                             const HyperMatrix& hypers, const PlannerConfig& config, std::uint64_t seed,
                             std::vector<double>* carried_window = nullptr) {
    config.validate();
    world.validate();
    hypers.validate();
    if (hypers.group_count() != config.groups)                      // planner.hpp:83-84
        throw std::invalid_argument("priori_init: hyper matrix group count != G");
    if (prev_best && prev_best->waypoints.size() != config.waypoints())
        throw std::invalid_argument("priori_init: previous path waypoint count mismatch");
    const WorldView wv(world);
    const std::vector<double> h = hypers.rows();
    std::vector<double> prev;
    if (prev_best) prev = encode_path(*prev_best);
    const sf_planner_config c = config.abi();
    const bool carry = config.window_carryover && carried_window != nullptr;
    std::vector<double> win;
    std::uint32_t wl = 0;
    if (carry) {
        win = *carried_window;
        wl = std::uint32_t(win.size());
        win.resize(std::max<std::size_t>(win.size(), config.tw) + 1);
    }
    sf_plan_record rec{};
    std::vector<double> best(config.dim);
    std::uint64_t bad[3] = {0, 0, 0};
    engine::check(sf_plan_frame(engine::ctx(), &wv.w, prev_best ? prev.data() : nullptr, h.data(), &c, seed,
                                carry ? win.data() : nullptr, carry ? &wl : nullptr, std::uint32_t(win.size()),
                                &rec, best.data(), bad),
                  bad);
    if (carry) carried_window->assign(win.begin(), win.begin() + wl);
    PlanRecord r;
    r.best_path = decode_path(best);
    r.fitness = rec.fitness;
    r.length = rec.length;
    r.intersections = rec.intersections;
    r.iterations = rec.iterations;
    r.truncated = rec.truncated != 0;
    r.stop_reason = r.truncated ? "converged" : "cap";
    r.collision_free = rec.collision_free != 0;
    r.wall_seconds = rec.wall_seconds;
    return r;
}

} // namespace swarmforge
