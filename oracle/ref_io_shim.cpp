// oracle/ref_io_shim.cpp — TEST-ONLY: extern "C" wrappers around the
// UNMODIFIED reference serialize.hpp (checkpoints, FNV-1a container, curves)
// and its JSON dependency (nlohmann/json 3.11.3 from the image; the
// reference does not vendor a copy).  Built by oracle/Makefile into
// oracle/_ref/libvoxevo_ref_io.so.  Used by tests/test_serialize.py to pin
// paper_2405_00698_b200/serialize.py (the device-side checkpoint/config
// mirror) byte for byte; the product never loads it.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "voxevo/advisor.hpp"
#include "voxevo/serialize.hpp"

namespace {
thread_local std::string g_err;

int64_t put(const std::string& s, char* out, int64_t cap) {
    if (out && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
    return static_cast<int64_t>(s.size());
}
}  // namespace

extern "C" {

const char* ref_io_last_error() { return g_err.c_str(); }

// nlohmann::json(array of doubles).dump(): the number formatting every
// checkpoint checksum depends on (serialize.hpp:37-38).
int64_t ref_io_dump_doubles(const double* v, int64_t n, char* out, int64_t cap) {
    nlohmann::json j = nlohmann::json::array();
    for (int64_t i = 0; i < n; ++i) j.push_back(v[i]);
    return put(j.dump(), out, cap);
}

// fnv1a64_hex (serialize.hpp:30-35)
int64_t ref_io_fnv_hex(const char* s, char* out, int64_t cap) { return put(voxevo::fnv1a64_hex(s), out, cap); }

// init_evolution(evolution_config_from_json(cfg)) -> `gens` x evolve_generation
// -> save_run(path) (serialize.hpp:179-209, 303-305).
int ref_io_run_and_save(const char* config_json, int gens, const char* path) {
    try {
        const voxevo::EvolutionConfig cfg = voxevo::evolution_config_from_json(nlohmann::json::parse(config_json));
        voxevo::EvolutionState st = voxevo::init_evolution(cfg);
        for (int g = 0; g < gens; ++g) voxevo::evolve_generation(st);
        voxevo::save_run(path, st);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// load_run(in) -> `gens` x evolve_generation -> save_run(out); gens = 0 is the
// save/load/save byte-stability check (test_serialize.cpp:133-148).
int ref_io_resume(const char* in_path, int gens, const char* out_path) {
    try {
        voxevo::EvolutionState st = voxevo::load_run(in_path);
        for (int g = 0; g < gens; ++g) voxevo::evolve_generation(st);
        voxevo::save_run(out_path, st);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// init_evolution(evolution_config_from_json(cfg)) -> `gens` x
// evolve_generation(st, make_advisor_fn(&ScriptedAdvisor)) with the
// reference's own ScriptedAdvisor (advisor.hpp:30-55) consulted at
// evolution.hpp:221-227.  adv4 = diversity_floor, stagnation_eps,
// mutation_boost, crossover_boost (NULL: the class defaults).  hist gets
// gens rows of: generation, best, mean, stddev, diversity, evaluations,
// params[7] (mutation_rate, mutation_scale, crossover_rate, elite_fraction,
// multipliers[3]); rng_out the final Rng::state() text.
int ref_io_run_advised(const char* config_json, int gens, const double* adv4, double* hist, char* rng_out,
                       int64_t rng_cap) {
    try {
        const voxevo::EvolutionConfig cfg = voxevo::evolution_config_from_json(nlohmann::json::parse(config_json));
        voxevo::EvolutionState st = voxevo::init_evolution(cfg);
        voxevo::ScriptedAdvisor adv;
        if (adv4) {
            adv.diversity_floor = adv4[0];
            adv.stagnation_eps = adv4[1];
            adv.mutation_boost = adv4[2];
            adv.crossover_boost = adv4[3];
        }
        const voxevo::AdvisorFn fn = voxevo::make_advisor_fn(&adv);
        for (int g = 0; g < gens; ++g) {
            const voxevo::GenerationReport r = voxevo::evolve_generation(st, fn);
            double* row = hist + static_cast<size_t>(g) * 13;
            row[0] = r.generation;
            row[1] = r.best;
            row[2] = r.mean;
            row[3] = r.stddev;
            row[4] = r.diversity;
            row[5] = r.evaluations;
            row[6] = r.params.mutation_rate;
            row[7] = r.params.mutation_scale;
            row[8] = r.params.crossover_rate;
            row[9] = r.params.elite_fraction;
            for (int k = 0; k < 3; ++k) row[10 + k] = r.params.material_multipliers[k];
        }
        put(st.rng.state(), rng_out, rng_cap);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// curves_csv(load_run(path).history) (serialize.hpp:321-343)
int64_t ref_io_curves_csv(const char* path, char* out, int64_t cap) {
    try {
        return put(voxevo::curves_csv(voxevo::load_run(path).history), out, cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
