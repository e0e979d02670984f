// minimize_rastrigin.cpp -- BF3 with the grouped optimizer through the
// drop-in headers (the reference demo's call: 8 x 10 particles, 1400
// iterations, seed 42), plus a small self-evolution.
#include <cstdio>

#include "swarmforge/benchmarks.hpp"
#include "swarmforge/hsef.hpp"

int main() {
    using namespace swarmforge;
    const auto problem = make_benchmark("BF3", 30);
    const RunReport r = run_dtpso(*problem, default_group_hypers(), 8, 10, 1400, 42);
    std::printf("run_dtpso BF3 final %.17g after %zu evaluations (%.3f ms)\n", r.final_fitness, r.evaluations,
                1e3 * r.wall_seconds);
    const EvolutionReport e = evolve(*problem, InnerBudget{8, 10, 100}, OuterBudget{8, 10, 3}, 41,
                                     default_group_hypers(),
                                     [](std::size_t k, double best) { std::printf("evolution %zu best %.6g\n", k, best); });
    std::printf("evolve best %.17g groups %zu\n", e.best_lfv_trace.back(), e.best.group_count());
    return 0;
}
