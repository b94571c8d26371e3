// plan_check.cpp — the breeding-plan scan (csrc/ga_plan.hpp) against a
// straight restatement of the reference breeding loop on std::mt19937_64
// (evolution.hpp:143-165, 267-289; rng.hpp:23-39): identical plans, masks,
// mutation lists and final RNG state, bit for bit.  Prints one JSON line
// with both timings.  Built and run by tests/test_plan_scan.py.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../../paper_2405_00698_b200/csrc/ga_plan.hpp"

using Plan = vx::ChildPlan;
using Mut = vx::MutEntry;

static double u01(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }
static double normal(std::mt19937_64& r) {
    const double u1 = (static_cast<double>(r() >> 11) + 0.5) * 0x1.0p-53;
    const double u2 = static_cast<double>(r() >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}
static uint64_t index(std::mt19937_64& r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) { const uint64_t x = r(); if (x >= threshold) return x % n; }
}
static int32_t tournament(std::mt19937_64& r, int P, int size) {
    uint64_t w = index(r, P);
    for (int k = 1; k < size; ++k) w = std::min<uint64_t>(w, index(r, P));
    return static_cast<int32_t>(w);
}
static void restated(std::mt19937_64& rng, int P, int n_elite, int ts, int64_t np, int64_t mw, double cx, double rate,
                     double scale, std::vector<Plan>& plan, std::vector<uint32_t>& masks, std::vector<Mut>& mut) {
    plan.assign(std::max(1, P - n_elite), Plan{});
    masks.clear();
    mut.clear();
    int slots = 0;
    for (int c = n_elite; c < P; ++c) {
        Plan& p = plan[c - n_elite];
        p.pa = tournament(rng, P, ts);
        p.pb = -1; p.mask_slot = -1; p.pad = 0;
        if (u01(rng) < cx) {
            p.pb = tournament(rng, P, ts);
            p.mask_slot = slots++;
            const size_t base = masks.size();
            masks.resize(base + mw, 0u);
            for (int64_t i = 0; i < np; ++i)
                if (u01(rng) < 0.5) masks[base + (i >> 5)] |= 1u << (i & 31);
        }
        for (int64_t i = 0; i < np; ++i)
            if (u01(rng) < rate) mut.push_back(Mut{c, static_cast<int32_t>(i), normal(rng) * scale});
    }
}

int main(int argc, char** argv) {
    const int P = argc > 1 ? std::atoi(argv[1]) : 256;
    const int64_t np = argc > 2 ? std::atoll(argv[2]) : 8710;
    const double cx = argc > 3 ? std::atof(argv[3]) : 0.5;
    const double rate = argc > 4 ? std::atof(argv[4]) : 0.05;
    const int gens = argc > 5 ? std::atoi(argv[5]) : 3;
    const int n_elite = P / 10, ts = 3;
    const int64_t mw = (np + 31) / 32;
    std::mt19937_64 a(12345), b(12345);
    const unsigned long long skip = argc > 6 ? std::strtoull(argv[6], nullptr, 10) : 7;
    b.discard(skip);  // start anywhere in a block: the position round-trips too
    a.discard(skip);
    double t_ref = 0, t_new = 0;
    size_t muts = 0;
    for (int g = 0; g < gens; ++g) {
        std::vector<Plan> pa, pb;
        std::vector<uint32_t> ma, mb;
        std::vector<Mut> ua, ub;
        vx::MutStore store;
        auto t0 = std::chrono::steady_clock::now();
        restated(a, P, n_elite, ts, np, mw, cx, rate, 0.1, pa, ma, ua);
        auto t1 = std::chrono::steady_clock::now();
        vx::plan_scan(b, vx::PlanParams{P, n_elite, ts, np, mw, cx, rate, 0.1}, pb, mb, store);
        store.flatten(ub);
        auto t2 = std::chrono::steady_clock::now();
        t_ref += std::chrono::duration<double>(t1 - t0).count();
        t_new += std::chrono::duration<double>(t2 - t1).count();
        muts += ua.size();
        bool ok = pa.size() == pb.size() && ma == mb && ua.size() == ub.size() && a == b;
        for (size_t i = 0; ok && i < pa.size(); ++i)
            ok = pa[i].pa == pb[i].pa && pa[i].pb == pb[i].pb && pa[i].mask_slot == pb[i].mask_slot;
        for (size_t i = 0; ok && i < ua.size(); ++i)
            ok = ua[i].child == ub[i].child && ua[i].index == ub[i].index &&
                 std::memcmp(&ua[i].delta, &ub[i].delta, sizeof(double)) == 0;
        if (!ok) {
            std::printf("{\"ok\": false, \"generation\": %d}\n", g);
            return 1;
        }
    }
    std::printf("{\"ok\": true, \"P\": %d, \"np\": %lld, \"generations\": %d, \"mutations\": %zu, "
                "\"restated_ms_per_gen\": %.3f, \"scan_ms_per_gen\": %.3f}\n",
                P, static_cast<long long>(np), gens, muts, 1e3 * t_ref / gens, 1e3 * t_new / gens);
    return 0;
}
