// genome_host.cpp — host C ABI for gaussian_encode (genome.hpp:168-179): the
// Fourier-feature encoding of one point, with the reference's expression
// order and the host libm's cos/sin (the same glibc the reference calls), so
// it is bit-identical on the same machine.  The device decode evaluates the
// same encoding inside decode_kernel for whole grids.
#include <cmath>
#include <cstdint>

#include "voxevo_b200.h"

namespace {
constexpr double kTwoPi = 6.283185307179586476925286766559;  // genome.hpp:16
}

extern "C" vx_status vx_gaussian_encode(const double* v, const double* bmat, int32_t m, double* out) {
    if (!v || !bmat || !out || m < 1) return VX_EINVAL;
    for (int32_t r = 0; r < m; ++r) {
        const double* row = bmat + 3 * r;
        const double phase = kTwoPi * (row[0] * v[0] + row[1] * v[1] + row[2] * v[2]);
        out[r] = std::cos(phase);
        out[m + r] = std::sin(phase);
    }
    return VX_OK;
}
