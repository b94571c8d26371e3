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
