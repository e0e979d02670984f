// Host build of the FP64 engine's cos (csrc/cos_glibc.cuh) for
// tests/test_oracle_cpu.py::test_glibc_cos_restatement: cos_glibc over a
// buffer, to be compared with libm's cos on the same arguments.
#include "cos_glibc.cuh"

#include <cstddef>

extern "C" void cos_glibc_rows(const double* x, std::size_t n, double* out) {
    for (std::size_t i = 0; i < n; ++i) out[i] = sepso::cos_glibc(x[i]);
}
