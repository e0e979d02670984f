// swarmforge/serialize.hpp -- drop-in for the reference's artifact I/O
// (serialize.hpp:18-322): JSON documents for the planner / runner / HSEF
// types, the metrics CSV and the per-frame SVG.  Host-only; nothing here
// touches the engine.  The JSON text is produced by nlohmann::json itself, so
// documents (keys, number formatting) are byte-identical to the reference's
// for the same values -- tests/test_serialize_cpu.py checks this against
// golden output of the reference (tests/golden/serialize_ref.txt).
//
// Each struct is described once by a field table (key -> member); to_json /
// from_json are generic over the table.  Special cases: ObstacleKind is the
// string "dynamic" / "static" (serialize.hpp:27-38); HypersDocument nests
// the matrix rows under "groups" (187-201); ScenarioConfig reads partial
// documents, keeping defaults for absent keys (241-254).
#pragma once

#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <type_traits>

#if __has_include("json.hpp")
#include "json.hpp"
#else
#include <nlohmann/json.hpp>
#endif

#include "swarmforge/hsef.hpp"
#include "swarmforge/runner.hpp"
#include "swarmforge/simenv.hpp"

namespace swarmforge {

using nlohmann::json;

/// Evolved-hypers document (serialize.hpp:157-165): the matrix and what
/// produced it.
struct HypersDocument {
    HyperMatrix hypers;
    std::string problem;
    InnerBudget inner;
    OuterBudget outer;
    std::uint64_t seed = 0;
};

namespace detail {

template <class C, class M>
struct Field {
    const char* key;
    M C::*member;
};
template <class C, class M>
constexpr Field<C, M> field(const char* key, M C::*member) { return {key, member}; }

// Schema<T>::fields() lists (key, member) pairs; partial = absent keys keep
// the current value on reading.
template <class T>
struct Schema;

template <class T, class = void>
struct has_schema : std::false_type {};
template <class T>
struct has_schema<T, std::void_t<decltype(Schema<T>::fields())>> : std::true_type {};

template <class T, class = void>
struct is_partial : std::false_type {};
template <class T>
struct is_partial<T, std::void_t<decltype(Schema<T>::partial)>> : std::bool_constant<Schema<T>::partial> {};

template <> struct Schema<Point2> {
    static constexpr auto fields() { return std::make_tuple(field("x", &Point2::x), field("y", &Point2::y)); }
};
template <> struct Schema<Obstacle> {
    static constexpr auto fields() {
        return std::make_tuple(field("kind", &Obstacle::kind), field("velocity", &Obstacle::velocity),
                               field("vertices", &Obstacle::vertices));
    }
};
template <> struct Schema<PolygonWorld> {
    using W = PolygonWorld;
    static constexpr auto fields() {
        return std::make_tuple(field("width", &W::width), field("height", &W::height), field("start", &W::start),
                               field("start_velocity", &W::start_velocity), field("target", &W::target),
                               field("target_velocity", &W::target_velocity), field("obstacles", &W::obstacles));
    }
};
template <> struct Schema<Path> {
    static constexpr auto fields() { return std::make_tuple(field("waypoints", &Path::waypoints)); }
};
template <> struct Schema<GroupHypers> {
    using H = GroupHypers;
    static constexpr auto fields() {
        return std::make_tuple(field("c1", &H::c1), field("c2", &H::c2), field("c3", &H::c3),
                               field("omega_init", &H::omega_init), field("omega_end", &H::omega_end),
                               field("v_limit", &H::v_limit));
    }
};
template <> struct Schema<HyperMatrix> {
    static constexpr auto fields() { return std::make_tuple(field("groups", &HyperMatrix::groups)); }
};
template <> struct Schema<RunReport> {
    using R = RunReport;
    static constexpr auto fields() {
        return std::make_tuple(field("algorithm", &R::algorithm), field("problem", &R::problem),
                               field("seed", &R::seed), field("iterations", &R::iterations),
                               field("trace", &R::trace), field("final_point", &R::final_point),
                               field("final_fitness", &R::final_fitness), field("evaluations", &R::evaluations),
                               field("wall_seconds", &R::wall_seconds));
    }
};
template <> struct Schema<PlanRecord> {
    using R = PlanRecord;
    static constexpr auto fields() {
        return std::make_tuple(field("best_path", &R::best_path), field("fitness", &R::fitness),
                               field("length", &R::length), field("intersections", &R::intersections),
                               field("iterations", &R::iterations), field("truncated", &R::truncated),
                               field("stop_reason", &R::stop_reason), field("collision_free", &R::collision_free),
                               field("wall_seconds", &R::wall_seconds));
    }
};
template <> struct Schema<SimMetrics> {
    using M = SimMetrics;
    static constexpr auto fields() {
        return std::make_tuple(field("variant", &M::variant), field("frames", &M::frames), field("seed", &M::seed),
                               field("mean_path_length", &M::mean_path_length),
                               field("mean_wall_seconds", &M::mean_wall_seconds),
                               field("mean_iterations", &M::mean_iterations),
                               field("collision_free_fraction", &M::collision_free_fraction),
                               field("records", &M::records));
    }
};
template <> struct Schema<InnerBudget> {
    static constexpr auto fields() {
        return std::make_tuple(field("groups", &InnerBudget::groups), field("per_group", &InnerBudget::per_group),
                               field("iterations", &InnerBudget::iterations));
    }
};
template <> struct Schema<OuterBudget> {
    static constexpr auto fields() {
        return std::make_tuple(field("groups", &OuterBudget::groups), field("per_group", &OuterBudget::per_group),
                               field("evolutions", &OuterBudget::evolutions));
    }
};
template <> struct Schema<EvolutionReport> {
    using E = EvolutionReport;
    static constexpr auto fields() {
        return std::make_tuple(field("best_lfv_trace", &E::best_lfv_trace),
                               field("evolution_lfv_trace", &E::evolution_lfv_trace), field("best", &E::best),
                               field("evolutions", &E::evolutions), field("lfv_evaluations", &E::lfv_evaluations),
                               field("root_seed", &E::root_seed), field("outer_seed", &E::outer_seed),
                               field("lfv_seed_root", &E::lfv_seed_root));
    }
};
template <> struct Schema<ScenarioConfig> {
    using S = ScenarioConfig;
    static constexpr bool partial = true;
    static constexpr auto fields() {
        return std::make_tuple(field("map_size", &S::map_size), field("dynamic_obstacles", &S::dynamic_obstacles),
                               field("static_obstacles", &S::static_obstacles), field("min_side", &S::min_side),
                               field("max_side", &S::max_side), field("max_speed", &S::max_speed),
                               field("start_speed", &S::start_speed), field("target_speed", &S::target_speed),
                               field("frames", &S::frames), field("dt", &S::dt), field("root_seed", &S::root_seed));
    }
};

} // namespace detail

inline void to_json(json& j, ObstacleKind k) { j = k == ObstacleKind::dynamic ? "dynamic" : "static"; }
inline void from_json(const json& j, ObstacleKind& k) {
    k = j.get<std::string>() == "dynamic" ? ObstacleKind::dynamic : ObstacleKind::fixed;
}

template <class T, std::enable_if_t<detail::has_schema<T>::value, int> = 0>
void to_json(json& j, const T& value) {
    j = json::object();
    std::apply([&](const auto&... f) { ((j[f.key] = value.*(f.member)), ...); }, detail::Schema<T>::fields());
}

template <class T, std::enable_if_t<detail::has_schema<T>::value, int> = 0>
void from_json(const json& j, T& value) {
    auto read = [&](const auto& f) {
        if (!detail::is_partial<T>::value || j.contains(f.key)) j.at(f.key).get_to(value.*(f.member));
    };
    std::apply([&](const auto&... f) { (read(f), ...); }, detail::Schema<T>::fields());
}

inline void to_json(json& j, const HypersDocument& doc) {
    j = json{{"groups", doc.hypers.groups}, {"problem", doc.problem}, {"inner_budget", doc.inner},
             {"outer_budget", doc.outer},   {"seed", doc.seed}};
}
inline void from_json(const json& j, HypersDocument& doc) {
    j.at("groups").get_to(doc.hypers.groups);
    j.at("problem").get_to(doc.problem);
    j.at("inner_budget").get_to(doc.inner);
    j.at("outer_budget").get_to(doc.outer);
    j.at("seed").get_to(doc.seed);
}

// ---- CSV (serialize.hpp:256-274)

/// Shortest round-trip decimal of v, as nlohmann::json prints it.
inline std::string csv_number(double v) { return json(v).dump(); }

inline std::string metrics_csv_header() {
    return "variant,frames,seed,mean_path_length,mean_wall_seconds,mean_iterations,collision_free_fraction\n";
}

inline std::string metrics_csv_row(const SimMetrics& m) {
    std::string row = m.variant + ',' + std::to_string(m.frames) + ',' + std::to_string(m.seed);
    for (double v : {m.mean_path_length, m.mean_wall_seconds, m.mean_iterations, m.collision_free_fraction})
        row += ',' + csv_number(v);
    return row + '\n';
}

// ---- SVG (serialize.hpp:276-307): static obstacles orange, dynamic black,
// the path blue from the green start to the red target; y flipped so +y is up.

inline std::string render_frame_svg(const PolygonWorld& world, const Path* path = nullptr) {
    std::ostringstream s;
    auto pt = [&](const Point2& p) { s << p.x << ',' << p.y << ' '; };
    auto dot = [&](const Point2& p, const char* colour) {
        s << "<circle cx=\"" << p.x << "\" cy=\"" << p.y << "\" r=\"5\" fill=\"" << colour << "\"/>\n";
    };
    const double w = world.width, h = world.height;
    s << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << w << "\" height=\"" << h << "\" viewBox=\"0 0 "
      << w << ' ' << h << "\">\n"
      << "<g transform=\"translate(0," << h << ") scale(1,-1)\">\n"
      << "<rect x=\"0\" y=\"0\" width=\"" << w << "\" height=\"" << h << "\" fill=\"white\" stroke=\"gray\"/>\n";
    for (const Obstacle& o : world.obstacles) {
        s << "<polygon points=\"";
        for (const Point2& v : o.vertices) pt(v);
        s << "\" fill=\"" << (o.kind == ObstacleKind::dynamic ? "black" : "orange") << "\"/>\n";
    }
    if (path != nullptr) {
        s << "<polyline points=\"";
        pt(world.start);
        for (const Point2& v : path->waypoints) pt(v);
        s << world.target.x << ',' << world.target.y << "\" fill=\"none\" stroke=\"blue\" stroke-width=\"2\"/>\n";
    }
    dot(world.start, "green");
    dot(world.target, "red");
    s << "</g>\n</svg>\n";
    return s.str();
}

// ---- files (serialize.hpp:309-322)

inline void write_text_file(const std::string& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open for writing: " + path);
    out << content;
    if (!out) throw std::runtime_error("write failed: " + path);
}

inline json read_json_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open: " + path);
    return json::parse(in);
}

} // namespace swarmforge
