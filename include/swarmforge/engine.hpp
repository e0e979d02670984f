// swarmforge/engine.hpp -- the device context behind the drop-in API.
//
// The reference API is free functions without a context argument, so the
// drop-in keeps one engine context per thread (created on first use on
// device SEPSO_DEVICE, default 0, precision SEPSO_PRECISION = fp32 | fp64,
// default fp32) and maps sf_status codes back to the reference's exception
// types: SF_INVALID_ARGUMENT -> std::invalid_argument, SF_NON_FINITE ->
// swarmforge::NonFiniteFitnessError (runner.hpp), SF_RUNTIME_ERROR ->
// std::runtime_error(message), anything else -> std::runtime_error.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "sepso.h"

namespace swarmforge {

class NonFiniteFitnessError : public std::runtime_error {   // runner.hpp:19-33
public:
    NonFiniteFitnessError(std::size_t group, std::size_t index, std::size_t iteration)
        : std::runtime_error("non-finite fitness for particle (" + std::to_string(group) + "," +
                             std::to_string(index) + ") at iteration " + std::to_string(iteration)),
          group_(group), index_(index), iteration_(iteration) {}
    std::size_t group() const { return group_; }
    std::size_t index_in_group() const { return index_; }
    std::size_t iteration() const { return iteration_; }

private:
    std::size_t group_, index_, iteration_;
};

namespace engine {

/// SEPSO_RNG=philox selects the counter-based stream; default: the reference's mt19937_64.
inline int rng_kind() {
    const char* r = std::getenv("SEPSO_RNG");
    return (r && std::strcmp(r, "philox") == 0) ? SF_RNG_PHILOX : SF_RNG_MT19937;
}

inline void check(int status, const std::uint64_t* bad = nullptr) {
    if (status == SF_OK) return;
    const std::string msg = sf_last_error();
    if (status == SF_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (status == SF_NON_FINITE && bad) throw NonFiniteFitnessError(bad[0], bad[1], bad[2]);
    if (status == SF_RUNTIME_ERROR) throw std::runtime_error(msg);
    throw std::runtime_error("sepso engine: " + msg);
}

struct Context {
    sf_ctx* ctx = nullptr;
    Context() {
        const char* dev = std::getenv("SEPSO_DEVICE");
        const char* prec = std::getenv("SEPSO_PRECISION");
        const int precision = (prec && std::strcmp(prec, "fp64") == 0) ? SF_FP64 : SF_FP32;
        check(sf_ctx_create(dev ? std::atoi(dev) : 0, precision, &ctx));
        check(sf_ctx_set_rng(ctx, rng_kind()));
    }
    ~Context() { sf_ctx_destroy(ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
};

/// The calling thread's engine context.
inline sf_ctx* ctx() {
    thread_local std::unique_ptr<Context> c;
    if (!c) c = std::make_unique<Context>();
    return c->ctx;
}

} // namespace engine
} // namespace swarmforge
