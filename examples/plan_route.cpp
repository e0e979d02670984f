// plan_route.cpp -- the reference planner used through the drop-in headers:
// the same calls a reference user makes (generate_world, plan_frame,
// step_world, run_scenario), now served by the B200 engine.
//   usage: plan_route [frames] [root_seed]
#include <cstdio>
#include <cstdlib>

#include "swarmforge/simenv.hpp"

int main(int argc, char** argv) {
    using namespace swarmforge;
    const std::size_t frames = argc > 1 ? std::size_t(std::atoi(argv[1])) : 10;
    ScenarioConfig sc;
    sc.root_seed = argc > 2 ? std::uint64_t(std::atoll(argv[2])) : 3;
    PlannerConfig base;
    base.max_iters_per_frame = 30;
    base.window_carryover = true;
    const SimMetrics m = run_scenario(sc, PlannerVariant::sepso, frames, base);
    for (std::size_t f = 0; f < m.records.size(); ++f) {
        const PlanRecord& r = m.records[f];
        std::printf("%zu %zu %d %zu %.17g %.17g\n", f, r.iterations, int(r.truncated), r.intersections, r.fitness,
                    r.length);
    }
    std::printf("mean_iterations %.6f mean_length %.6f collision_free %.3f mean_ms %.4f\n", m.mean_iterations,
                m.mean_path_length, m.collision_free_fraction, 1e3 * m.mean_wall_seconds);
    return 0;
}
