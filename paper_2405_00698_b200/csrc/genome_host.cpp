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

// sample_genome's encoding matrix (genome.hpp:153-154): B[k] = sigma *
// Rng(seed).normal() for k = 0 .. 3m-1, the first 6m draws of each genome's
// own stream, with the reference's Box-Muller (rng.hpp:26-30) and the host
// glibc log / cos — bit-identical to the reference on the same machine.  The
// device sampler (decode.cu sample_kernel) draws the layer weights (exact
// uniforms) after skipping these draws; this replaces its device log/cos B.
#include <algorithm>
#include <random>
#include <thread>
#include <vector>

namespace vx {

void host_sample_bmat(int32_t m, double sigma, int32_t P, const uint64_t* seeds, double* out) {
    auto work = [&](int32_t a0, int32_t a1) {
        for (int32_t a = a0; a < a1; ++a) {
            std::mt19937_64 eng(seeds[a]);
            double* b = out + static_cast<size_t>(a) * 3 * m;
            for (int32_t k = 0; k < 3 * m; ++k) {
                const double u1 = (static_cast<double>(eng() >> 11) + 0.5) * 0x1.0p-53;
                const double u2 = static_cast<double>(eng() >> 11) * 0x1.0p-53;
                b[k] = sigma * (std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2));
            }
        }
    };
    const int32_t nt = std::max(1, std::min<int32_t>(8, P / 512));
    if (nt == 1) {
        work(0, P);
        return;
    }
    std::vector<std::thread> th;
    for (int32_t t = 0; t < nt; ++t) th.emplace_back(work, P * t / nt, P * (t + 1) / nt);
    for (auto& x : th) x.join();
}

}  // namespace vx
