// swarmforge/problem.hpp -- drop-in for the reference's problem.hpp:14-31.
// The engine evaluates the reference's two problem families on the device
// (PathPlanningProblem, BenchmarkProblem); device_spec() tells the runners
// which kernel to use.  A user-defined subclass cannot run on the GPU: the
// engine rejects it with std::invalid_argument instead of running a CPU path.
#pragma once

#include <cstddef>
#include <span>
#include <string>

#include "sepso.h"
#include "swarmforge/hypers.hpp"

namespace swarmforge {

class FitnessProblem {
public:
    virtual ~FitnessProblem() = default;
    virtual const std::string& name() const = 0;
    virtual std::size_t dimension() const = 0;
    virtual const SearchBounds& bounds() const = 0;
    virtual void evaluate_rows(std::span<const double> xs, std::size_t count, std::span<double> out) const = 0;

    double evaluate_point(std::span<const double> x) const {
        double f = 0.0;
        evaluate_rows(x, 1, {&f, 1});
        return f;
    }

    /// Fill `spec` (sf_problem) when the device engine implements this problem.
    virtual bool device_spec(sf_problem& spec) const {
        (void)spec;
        return false;
    }
};

} // namespace swarmforge
