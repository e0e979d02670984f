// Prints the artifacts of swarmforge/serialize.hpp for fixed values.  Built
// against the reference headers (tests/golden/make_golden_serialize.py ->
// tests/golden/serialize_ref.txt) and against the drop-in headers
// (tests/test_serialize_cpu.py); the two outputs must be identical.
#include <cstdio>
#include <iostream>
#include <limits>

#include "swarmforge/serialize.hpp"

using namespace swarmforge;

template <class T>
static void emit(const char* name, const T& v) {
    const json j = v;
    std::cout << name << ' ' << j.dump() << '\n';
    T back{};
    from_json(json::parse(j.dump()), back);
    std::cout << name << "-roundtrip " << json(back).dump() << '\n';
}

int main(int argc, char** argv) {
    PolygonWorld w;
    w.width = 366.0;
    w.height = 366.0;
    w.start = {183.0, 36.6};
    w.start_velocity = {0.0, 3.0};
    w.target = {183.0, 329.4};
    w.target_velocity = {0.0, 8.0};
    Obstacle a;
    a.kind = ObstacleKind::dynamic;
    a.velocity = {-1.25, 0.1};
    a.vertices = {{10.0, 20.0}, {123.456789012345, 20.0}, {123.456789012345, 1e-7}, {10.0, 5e21}};
    Obstacle b;
    b.kind = ObstacleKind::fixed;
    b.vertices = {{200.5, 200.25}, {260.0, 210.0}, {230.0, 280.125}};
    w.obstacles = {a, b};
    emit("world", w);

    Path p;
    p.waypoints = {{150.0, 80.0}, {1.0 / 3.0, 2.0 / 3.0}, {-0.0, 300.0}};
    emit("path", p);

    HyperMatrix hm;
    hm.groups = {{1.5, 1.75, 0.5, 0.9, 0.4, 0.2}, {0.1, 2.5, 2.499999999999999, 1.0, 0.05, 1.0}};
    emit("hypers", hm);

    RunReport rr;
    rr.algorithm = "tof-dppso";
    rr.problem = "rastrigin";
    rr.seed = std::numeric_limits<std::uint64_t>::max();
    rr.iterations = 3;
    rr.trace = {1.5, 0.25, 1e-300};
    rr.final_point = {-0.0, 3.0, 6.02214076e23};
    rr.final_fitness = 0.1;
    rr.evaluations = 240;
    rr.wall_seconds = 0.0123;
    emit("run", rr);

    PlanRecord pr;
    pr.best_path = p;
    pr.fitness = 7680.5;
    pr.length = 123.5;
    pr.intersections = 4;
    pr.iterations = 16;
    pr.truncated = true;
    pr.stop_reason = "auto_truncate";
    pr.collision_free = false;
    pr.wall_seconds = 1e-4;
    emit("plan", pr);

    SimMetrics sm;
    sm.variant = "sepso";
    sm.frames = 2;
    sm.seed = 3;
    sm.mean_path_length = 123.456;
    sm.mean_wall_seconds = 0.000157;
    sm.mean_iterations = 16.2;
    sm.collision_free_fraction = 0.91;
    PlanRecord pr2 = pr;
    pr2.collision_free = true;
    pr2.stop_reason = "cap";
    sm.records = {pr, pr2};
    emit("metrics", sm);
    std::cout << "csv " << metrics_csv_header() << "csv " << metrics_csv_row(sm);
    std::cout << "csv-number " << csv_number(0.1) << ' ' << csv_number(1e21) << ' ' << csv_number(-0.0) << ' '
              << csv_number(5e-324) << ' ' << csv_number(100.0) << '\n';

    InnerBudget ib{8, 170, 30};
    OuterBudget ob{8, 10, 3};
    emit("inner", ib);
    emit("outer", ob);
    HypersDocument doc{hm, "path", ib, ob, 41};
    emit("hypers-doc", doc);

    EvolutionReport er;
    er.best_lfv_trace = {9.5, 8.25};
    er.evolution_lfv_trace = {9.5, 8.75};
    er.best = hm;
    er.evolutions = 2;
    er.lfv_evaluations = 160;
    er.root_seed = 41;
    er.outer_seed = 1234567890123456789ull;
    er.lfv_seed_root = 987654321ull;
    emit("evolution", er);

    ScenarioConfig sc;
    emit("scenario-default", sc);
    ScenarioConfig partial;
    from_json(json::parse(R"({"frames": 7, "dt": 0.5, "root_seed": 11})"), partial);
    std::cout << "scenario-partial " << json(partial).dump() << '\n';
    try {
        PlanRecord bad;
        from_json(json::parse(R"({"fitness": 1.0})"), bad);
        std::cout << "strict-missing no-throw\n";
    } catch (const std::exception& e) {
        std::cout << "strict-missing " << e.what() << '\n';
    }
    std::cout << "pretty " << json(p).dump(2) << '\n';
    std::cout << "svg-world\n" << render_frame_svg(w);
    std::cout << "svg-path\n" << render_frame_svg(w, &p);
    if (argc > 1) {
        const std::string f = std::string(argv[1]) + "/doc.json";
        write_text_file(f, json(doc).dump(2));
        HypersDocument d2;
        from_json(read_json_file(f), d2);
        std::cout << "file-roundtrip " << json(d2).dump() << '\n';
        try {
            read_json_file(std::string(argv[1]) + "/missing.json");
        } catch (const std::runtime_error& e) {
            std::cout << "missing-file " << (std::string(e.what()).rfind("cannot open: ", 0) == 0 ? "ok" : "bad") << '\n';
        }
    }
    return 0;
}
