// rng_api.cpp — host C ABI for the reference's Rng (rng.hpp:15-56) and the
// single-genome GA operators that consume it (crossover, mutate,
// tournament_select: evolution.hpp:140-173).  The evolution driver runs the
// whole breeding loop on the GA stream itself (ga_plan.cpp); these entry
// points are the per-call building blocks of the reference API, on the same
// generator (std::mt19937_64, libstdc++ text state) and the same glibc
// Box-Muller, so a caller interleaving them with its own code sees the
// reference's numbers draw for draw.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <random>
#include <sstream>
#include <string>

#include "voxevo_b200.h"

struct vx_rng {
    std::mt19937_64 engine{0};  // Rng() : engine_(0) (rng.hpp:17)
};

namespace vx {
void set_error(const std::string& msg);
}

namespace {

inline double uniform01(std::mt19937_64& e) { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
inline double normal(std::mt19937_64& e) {
    const double u1 = (static_cast<double>(e() >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = static_cast<double>(e() >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}
inline uint64_t index(std::mt19937_64& e, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t r = e();
        if (r >= threshold) return r % n;
    }
}

}  // namespace

extern "C" {

vx_status vx_rng_create(uint64_t seed, vx_rng** out) {
    if (!out) return VX_EINVAL;
    *out = new (std::nothrow) vx_rng;
    if (!*out) return VX_EOOM;
    (*out)->engine.seed(seed);
    return VX_OK;
}

void vx_rng_free(vx_rng* r) { delete r; }

uint64_t vx_rng_next_u64(vx_rng* r) { return r ? r->engine() : 0; }

double vx_rng_uniform01(vx_rng* r) { return r ? uniform01(r->engine) : 0.0; }

double vx_rng_normal(vx_rng* r) { return r ? normal(r->engine) : 0.0; }

uint64_t vx_rng_index(vx_rng* r, uint64_t n) { return (r && n > 0) ? index(r->engine, n) : 0; }

int64_t vx_rng_state(vx_rng* r, char* buf, int64_t cap) {
    if (!r) return -1;
    std::ostringstream os;
    os << r->engine;
    const std::string s = os.str();
    if (buf && cap > 0) {
        std::strncpy(buf, s.c_str(), static_cast<size_t>(cap - 1));
        buf[cap - 1] = 0;
    }
    return static_cast<int64_t>(s.size());
}

vx_status vx_rng_set_state(vx_rng* r, const char* state) {
    if (!r || !state) return VX_EINVAL;
    std::istringstream is(state);
    std::mt19937_64 e;
    is >> e;
    if (is.fail()) return (vx::set_error("Rng::set_state: malformed state text"), VX_EINVAL);
    r->engine = e;
    return VX_OK;
}

vx_status vx_crossover(vx_rng* r, int64_t np, const double* a, const double* b, double* child) {
    if (!r || np < 0 || (np > 0 && (!a || !b || !child))) return VX_EINVAL;
    for (int64_t i = 0; i < np; ++i) child[i] = uniform01(r->engine) < 0.5 ? b[i] : a[i];
    return VX_OK;
}

vx_status vx_mutate(vx_rng* r, int64_t np, double* params, double rate, double scale) {
    if (!r || np < 0 || (np > 0 && !params)) return VX_EINVAL;
    for (int64_t i = 0; i < np; ++i)
        if (uniform01(r->engine) < rate) params[i] += normal(r->engine) * scale;
    return VX_OK;
}

int32_t vx_tournament_select(vx_rng* r, int32_t population, int32_t size) {
    if (!r || population < 1) return -1;
    uint64_t winner = index(r->engine, static_cast<uint64_t>(population));
    for (int k = 1; k < size; ++k) winner = std::min<uint64_t>(winner, index(r->engine, static_cast<uint64_t>(population)));
    return static_cast<int32_t>(winner);
}

}  // extern "C"
