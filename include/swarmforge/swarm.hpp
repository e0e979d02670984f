// swarmforge/swarm.hpp -- drop-in for the reference's swarm.hpp:1-176.
// SwarmState stays a host value type; init_swarm and step run on the device
// (sf_init_swarm / sf_step, the engine's stage kernels) with the draw indices
// taken from the caller's RngStream position, which advances exactly as the
// reference's sequential stream would.
#pragma once

#include <cstddef>
#include <limits>
#include <span>
#include <stdexcept>
#include <vector>

#include "swarmforge/engine.hpp"
#include "swarmforge/hypers.hpp"
#include "swarmforge/rng.hpp"

namespace swarmforge {

struct SwarmState {
    std::size_t groups = 0, per_group = 0, dim = 0;
    std::vector<double> x, v, pbest_x, pbest_f, gbest_x, gbest_f, tbest_x;
    double tbest_f = std::numeric_limits<double>::infinity();
    std::size_t iteration = 0;

    std::size_t particle_count() const { return groups * per_group; }
    std::size_t row(std::size_t g, std::size_t n) const { return g * per_group + n; }
    std::span<double> position(std::size_t g, std::size_t n) { return {x.data() + row(g, n) * dim, dim}; }
    std::span<const double> position(std::size_t g, std::size_t n) const { return {x.data() + row(g, n) * dim, dim}; }
    std::span<const double> personal_best(std::size_t g, std::size_t n) const {
        return {pbest_x.data() + row(g, n) * dim, dim};
    }
    std::span<const double> group_best(std::size_t g) const { return {gbest_x.data() + g * dim, dim}; }
};

struct StepRandoms {
    std::vector<double> r1, r2, r3;
};

inline StepRandoms draw_step_randoms(std::size_t groups, std::size_t per_group, RngStream& rng) {
    StepRandoms r;
    const std::size_t n = groups * per_group;
    r.r1.resize(n);
    r.r2.resize(n);
    r.r3.resize(n);
    for (double& u : r.r1) u = rng.uniform();
    for (double& u : r.r2) u = rng.uniform();
    for (double& u : r.r3) u = rng.uniform();
    return r;
}

inline std::vector<double> inertia_at(const HyperMatrix& hypers, std::size_t k, std::size_t total) {
    if (total == 0) throw std::invalid_argument("inertia_at: total iteration count must be >= 1");
    if (k > total) throw std::invalid_argument("inertia_at: k out of range");
    const double frac = double(k) / double(total);
    std::vector<double> w(hypers.group_count());
    for (std::size_t g = 0; g < w.size(); ++g)
        w[g] = hypers.groups[g].omega_init - (hypers.groups[g].omega_init - hypers.groups[g].omega_end) * frac;
    return w;
}

namespace detail {
inline SwarmState fresh_state(std::size_t G, std::size_t N, std::size_t D) {
    SwarmState s;
    s.groups = G;
    s.per_group = N;
    s.dim = D;
    s.x.resize(G * N * D);
    s.v.resize(G * N * D);
    s.pbest_f.assign(G * N, std::numeric_limits<double>::infinity());
    s.gbest_x.assign(G * D, 0.0);
    s.gbest_f.assign(G, std::numeric_limits<double>::infinity());
    s.tbest_x.assign(D, 0.0);
    return s;
}
} // namespace detail

inline SwarmState init_swarm(const HyperMatrix& hypers, const SearchBounds& bounds, std::size_t groups,
                             std::size_t per_group, std::size_t dim, RngStream& rng) {
    hypers.validate();
    bounds.validate();
    if (groups < 1 || per_group < 1 || dim < 1) throw std::invalid_argument("init_swarm: G, N, D must all be >= 1");
    if (hypers.group_count() != groups) throw std::invalid_argument("init_swarm: hyper matrix group count != G");
    if (bounds.dimension() != dim) throw std::invalid_argument("init_swarm: bounds dimension != D");
    SwarmState s = detail::fresh_state(groups, per_group, dim);
    const std::vector<double> h = hypers.rows();
    engine::check(sf_init_swarm(engine::ctx(), h.data(), bounds.x_lo.data(), bounds.x_hi.data(), std::uint32_t(groups),
                                std::uint32_t(per_group), std::uint32_t(dim), rng.seed(), rng.drawn(), nullptr, 0, 0.0,
                                s.x.data(), s.v.data()));
    rng.skip(2 * groups * per_group * dim);
    s.pbest_x = s.x;
    return s;
}

inline void step(SwarmState& s, const HyperMatrix& hypers, const SearchBounds& bounds, RngStream& rng,
                 std::size_t k, std::size_t total) {
    if (hypers.group_count() != s.groups) throw std::invalid_argument("step: hyper matrix group count != state groups");
    if (bounds.dimension() != s.dim) throw std::invalid_argument("step: bounds dimension != state dimension");
    const std::vector<double> h = hypers.rows();
    engine::check(sf_step(engine::ctx(), h.data(), bounds.x_lo.data(), bounds.x_hi.data(), std::uint32_t(s.groups),
                          std::uint32_t(s.per_group), std::uint32_t(s.dim), s.x.data(), s.v.data(),
                          s.pbest_x.data(), s.gbest_x.data(), s.tbest_x.data(), rng.seed(), rng.drawn(),
                          std::uint32_t(k), std::uint32_t(total)));
    rng.skip(3 * s.groups * s.per_group);
    s.iteration = k;
}

} // namespace swarmforge
