// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// extern "C" wrappers around the UNMODIFIED reference headers in
// /root/reference/proj/include/voxevo (compiled where they lie, never copied).
// Built by oracle/Makefile into oracle/_ref/libvoxevo_ref.so with the
// reference's own numerics: -std=c++20 -O2, no -march, -ffp-contract=off
// (SURVEY.md §7 step 1).  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it.
//
// Every wrapper names the reference entry point it forwards to.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#ifdef VX_REF_HAVE_JSON
#include "voxevo/advisor.hpp"  // ScriptedAdvisor (needs nlohmann/json)
#endif
#include "voxevo/bench.hpp"
#include "voxevo/evolution.hpp"
#include "voxevo/genome.hpp"
#include "voxevo/morphology.hpp"
#include "voxevo/parallel.hpp"
#include "voxevo/physics.hpp"
#include "voxevo/rng.hpp"

using namespace voxevo;

namespace {

std::vector<std::size_t> widths_of(int nh, const int* w) {
    std::vector<std::size_t> v;
    for (int i = 0; i < nh; ++i) v.push_back(static_cast<std::size_t>(w[i]));
    return v;
}

// Flat params (param_tensors order, genome.hpp:57-81) + B -> Genome.
Genome genome_from_flat(int m, int nh, const int* widths, const double* params, const double* bmat) {
    Genome g = sample_genome(EncodingSpec{static_cast<std::size_t>(m), 3, 1.0}, widths_of(nh, widths), 0);
    g.b_matrix.assign(bmat, bmat + 3 * m);
    std::size_t off = 0;
    for (auto* t : g.param_tensors()) {
        for (auto& x : *t) x = params[off++];
    }
    return g;
}

void genome_to_flat(const Genome& g, double* params, double* bmat) {
    std::size_t off = 0;
    for (const auto* t : g.param_tensors())
        for (double x : *t) params[off++] = x;
    if (bmat) std::memcpy(bmat, g.b_matrix.data(), g.b_matrix.size() * sizeof(double));
}

VoxelGrid grid_from_flat(int w, int h, int d, const uint8_t* mat, const double* wt) {
    VoxelGrid g(w, h, d);
    for (std::size_t i = 0; i < g.cells.size(); ++i) {
        g.cells[i].material = static_cast<Material>(mat[i]);
        g.cells[i].weight = wt ? wt[i] : 1.0;
    }
    return g;
}

MaterialTable table_from(const double* t) {
    MaterialTable m;
    if (!t) return m;
    m.k_muscle = t[0];
    m.k_soft = t[1];
    m.k_bone = t[2];
    m.damping_ratio = t[3];
    m.amp_max = t[4];
    m.phase_max = t[5];
    m.voxel_edge = t[6];
    m.mass_per_vertex = t[7];
    return m;
}

GroundPlane plane_from(const double* p) {
    GroundPlane g;
    if (!p) return g;
    g.k = p[0];
    g.damping_ratio = p[1];
    g.mu_static = p[2];
    g.mu_kinetic = p[3];
    return g;
}

SimConfig sim_from(const double* s) {
    SimConfig c;
    if (!s) return c;
    c.gravity = s[0];
    c.dt = s[1];
    c.duration = s[2];
    c.actuation_frequency = s[3];
    c.enable_gravity = s[4] != 0.0;
    c.enable_contact = s[5] != 0.0;
    return c;
}

HyperParams hyper_from(const double* h) {
    HyperParams p;
    if (!h) return p;
    p.mutation_rate = h[0];
    p.mutation_scale = h[1];
    p.crossover_rate = h[2];
    p.elite_fraction = h[3];
    p.material_multipliers = {h[4], h[5], h[6]};
    return p;
}

void hyper_to(const HyperParams& p, double* h) {
    h[0] = p.mutation_rate;
    h[1] = p.mutation_scale;
    h[2] = p.crossover_rate;
    h[3] = p.elite_fraction;
    h[4] = p.material_multipliers[0];
    h[5] = p.material_multipliers[1];
    h[6] = p.material_multipliers[2];
}

struct SysHandle {
    MassSpringSystem sys;
    SimWorkspace* ws = nullptr;
    ~SysHandle() { delete ws; }
    SimWorkspace& workspace() {
        if (!ws) ws = new SimWorkspace(sys);
        return *ws;
    }
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------- rng.hpp
// Rng::next_u64 (rng.hpp:20)
void ref_rng_draws(uint64_t seed, int64_t n, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
// Rng::uniform01 (rng.hpp:23)
void ref_rng_uniform(uint64_t seed, int64_t n, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform01();
}
// Rng::normal (rng.hpp:26-30)
void ref_rng_normal(uint64_t seed, int64_t n, double* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}
// Rng::index (rng.hpp:33-39)
void ref_rng_index(uint64_t seed, int64_t n, uint64_t range, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.index(range);
}
// Rng::state (rng.hpp:41-45) after `skip` draws; returns the string length.
int64_t ref_rng_state(uint64_t seed, int64_t skip, char* buf, int64_t cap) {
    Rng r(seed);
    for (int64_t i = 0; i < skip; ++i) r.next_u64();
    const std::string s = r.state();
    if (buf && cap > 0) {
        std::strncpy(buf, s.c_str(), static_cast<std::size_t>(cap - 1));
        buf[cap - 1] = 0;
    }
    return static_cast<int64_t>(s.size());
}
// Rng::set_state (rng.hpp:47-50) then n draws.
void ref_rng_draws_from_state(const char* state, int64_t n, uint64_t* out) {
    Rng r(0);
    r.set_state(state);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

// ------------------------------------------------------------- genome.hpp
int64_t ref_param_count(int m, int nh, const int* widths) {
    return static_cast<int64_t>(
        sample_genome(EncodingSpec{static_cast<std::size_t>(m), 3, 1.0}, widths_of(nh, widths), 0)
            .parameter_count());
}
// sample_genome (genome.hpp:146-166)
void ref_sample_genome(int m, double sigma, int nh, const int* widths, uint64_t seed, double* params,
                       double* bmat) {
    const Genome g = sample_genome(EncodingSpec{static_cast<std::size_t>(m), 3, sigma}, widths_of(nh, widths), seed);
    genome_to_flat(g, params, bmat);
}
// gaussian_encode (genome.hpp:169-179)
void ref_gaussian_encode(const double* v, const double* bmat, int m, double* out) {
    const std::vector<double> b(bmat, bmat + 3 * m);
    const auto e = gaussian_encode(Vec3{v[0], v[1], v[2]}, b, static_cast<std::size_t>(m));
    std::memcpy(out, e.data(), e.size() * sizeof(double));
}
// forward (genome.hpp:187-211)
void ref_forward(int m, int nh, const int* widths, const double* params, const double* bmat, const double* v,
                 double* probs, double* weight) {
    const Genome g = genome_from_flat(m, nh, widths, params, bmat);
    const MaterialQuery q = forward(g, Vec3{v[0], v[1], v[2]});
    for (int i = 0; i < kMaterialCount; ++i) probs[i] = q.probs[i];
    *weight = q.weight;
}

// --------------------------------------------------------- morphology.hpp
// decode (morphology.hpp:141-157)
void ref_decode(int m, int nh, const int* widths, const double* params, const double* bmat, int w, int h, int d,
                uint8_t* mat, double* wt) {
    const Genome g = genome_from_flat(m, nh, widths, params, bmat);
    const VoxelGrid grid = decode(g, w, h, d);
    for (std::size_t i = 0; i < grid.cells.size(); ++i) {
        mat[i] = static_cast<uint8_t>(grid.cells[i].material);
        wt[i] = grid.cells[i].weight;
    }
}
// largest_component (morphology.hpp:162-208)
void ref_largest_component(int w, int h, int d, const uint8_t* mat_in, uint8_t* mat_out) {
    const VoxelGrid g = grid_from_flat(w, h, d, mat_in, nullptr);
    const VoxelGrid out = largest_component(g);
    for (std::size_t i = 0; i < out.cells.size(); ++i) mat_out[i] = static_cast<uint8_t>(out.cells[i].material);
}
// bench_robot (bench.hpp:35-44)
void ref_bench_robot(int n, uint8_t* mat, double* wt) {
    const VoxelGrid g = bench_robot(n);
    for (std::size_t i = 0; i < g.cells.size(); ++i) {
        mat[i] = static_cast<uint8_t>(g.cells[i].material);
        wt[i] = g.cells[i].weight;
    }
}
// build_mass_spring (morphology.hpp:217-299); NULL when the grid is empty
// (the reference throws empty_robot, morphology.hpp:230).
void* ref_build(int w, int h, int d, const uint8_t* mat, const double* wt, const double* table8,
                const double* plane4) {
    const VoxelGrid g = grid_from_flat(w, h, d, mat, wt);
    try {
        auto* hnd = new SysHandle;
        hnd->sys = build_mass_spring(g, table_from(table8), plane_from(plane4));
        return hnd;
    } catch (const empty_robot&) {
        return nullptr;
    }
}
// Hand-assembled system (tests build dumbbells this way, test_physics.cpp:13-27).
void* ref_sys_make(int nm, int ns, const double* pos, const double* vel, const double* mass, const int* si,
                   const int* sj, const double* k, const double* rest0, const double* zeta, const uint8_t* has_act,
                   const double* sign, const double* amp, const double* phase, const double* plane4) {
    auto* hnd = new SysHandle;
    MassSpringSystem& s = hnd->sys;
    s.plane = plane_from(plane4);
    s.masses.resize(nm);
    for (int a = 0; a < nm; ++a) {
        s.masses[a].pos = {pos[3 * a], pos[3 * a + 1], pos[3 * a + 2]};
        s.masses[a].vel = {vel[3 * a], vel[3 * a + 1], vel[3 * a + 2]};
        s.masses[a].mass = mass[a];
    }
    s.springs.resize(ns);
    for (int q = 0; q < ns; ++q) {
        Spring& sp = s.springs[q];
        sp.i = si[q];
        sp.j = sj[q];
        sp.k = k[q];
        sp.rest0 = rest0[q];
        sp.damping_ratio = zeta[q];
        if (has_act && has_act[q]) sp.act = Actuation{sign[q], amp[q], phase[q]};
    }
    return hnd;
}
void ref_sys_sizes(void* h, int* nm, int* ns) {
    auto* hnd = static_cast<SysHandle*>(h);
    *nm = static_cast<int>(hnd->sys.masses.size());
    *ns = static_cast<int>(hnd->sys.springs.size());
}
void ref_sys_export(void* h, double* pos, double* vel, double* mass, int* si, int* sj, double* k, double* rest0,
                    double* zeta, uint8_t* has_act, double* sign, double* amp, double* phase) {
    auto* hnd = static_cast<SysHandle*>(h);
    const MassSpringSystem& s = hnd->sys;
    for (std::size_t a = 0; a < s.masses.size(); ++a) {
        for (int c = 0; c < 3; ++c) {
            if (pos) pos[3 * a + c] = s.masses[a].pos[c];
            if (vel) vel[3 * a + c] = s.masses[a].vel[c];
        }
        if (mass) mass[a] = s.masses[a].mass;
    }
    for (std::size_t q = 0; q < s.springs.size(); ++q) {
        const Spring& sp = s.springs[q];
        if (si) si[q] = sp.i;
        if (sj) sj[q] = sp.j;
        if (k) k[q] = sp.k;
        if (rest0) rest0[q] = sp.rest0;
        if (zeta) zeta[q] = sp.damping_ratio;
        if (has_act) has_act[q] = sp.act ? 1 : 0;
        if (sign) sign[q] = sp.act ? sp.act->sign : 0.0;
        if (amp) amp[q] = sp.act ? sp.act->amplitude : 0.0;
        if (phase) phase[q] = sp.act ? sp.act->phase : 0.0;
    }
}
void ref_sys_free(void* h) { delete static_cast<SysHandle*>(h); }

// ------------------------------------------------------------ physics.hpp
// SimWorkspace ctor (physics.hpp:140-185)
void ref_sys_workspace(void* h, double* damp_coef, double* amp_rest, double* sin_ph, double* cos_ph,
                       double* ground_damp, int* inc_off, int* inc_spring, double* inc_sign) {
    auto* hnd = static_cast<SysHandle*>(h);
    const SimWorkspace ws(hnd->sys);
    auto cp = [](double* dst, const std::vector<double>& v) {
        if (dst) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(damp_coef, ws.damp_coef);
    cp(amp_rest, ws.amp_rest);
    cp(sin_ph, ws.sin_phase);
    cp(cos_ph, ws.cos_phase);
    cp(ground_damp, ws.ground_damp);
    cp(inc_sign, ws.inc_sign);
    if (inc_off) std::memcpy(inc_off, ws.inc_offset.data(), ws.inc_offset.size() * sizeof(int));
    if (inc_spring) std::memcpy(inc_spring, ws.inc_spring.data(), ws.inc_spring.size() * sizeof(int));
}
// step (physics.hpp:191-264) called for k = k0 .. k0+nsteps-1 with t = k*dt
// (physics.hpp:297).  Returns the number of steps that returned ok; stops at
// the first diverged step (that step is counted in *steps_called).
int64_t ref_sys_step(void* h, const double* sim6, int64_t k0, int64_t nsteps, int64_t* steps_called,
                     uint64_t* spring_updates, double* max_speed_sq) {
    auto* hnd = static_cast<SysHandle*>(h);
    const SimConfig cfg = sim_from(sim6);
    SimWorkspace& ws = hnd->workspace();
    int64_t ok = 0, called = 0;
    for (int64_t k = k0; k < k0 + nsteps; ++k) {
        const double t = static_cast<double>(k) * cfg.dt;
        ++called;
        if (step(hnd->sys, t, cfg, ws) == StepResult::diverged) break;
        ++ok;
    }
    if (steps_called) *steps_called = called;
    if (spring_updates) *spring_updates = ws.spring_updates;
    if (max_speed_sq) *max_speed_sq = ws.max_speed_sq;
    return ok;
}
// center_of_mass (physics.hpp:266-278)
void ref_center_of_mass(void* h, double* com) {
    const Vec3 c = center_of_mass(static_cast<SysHandle*>(h)->sys);
    com[0] = c[0];
    com[1] = c[1];
    com[2] = c[2];
}
// simulate (physics.hpp:287-311); summary = com_start[3], com_end[3],
// horizontal_displacement, max_speed, diverged.  The handle's system is not
// modified (simulate takes it by value).  dump (optional) receives
// (t, com[3]) rows every `stride` steps plus the final row.
int64_t ref_simulate(void* h, const double* sim6, double* summary, double* dump, int64_t dump_cap, int stride) {
    const SimConfig cfg = sim_from(sim6);
    std::vector<TrajectorySample> samples;
    const TrajectorySummary s = simulate(static_cast<SysHandle*>(h)->sys, cfg, dump ? &samples : nullptr, stride);
    for (int c = 0; c < 3; ++c) {
        summary[c] = s.com_start[c];
        summary[3 + c] = s.com_end[c];
    }
    summary[6] = s.horizontal_displacement;
    summary[7] = s.max_speed;
    summary[8] = s.diverged ? 1.0 : 0.0;
    if (dump) {
        int64_t n = 0;
        for (const auto& smp : samples) {
            if (n >= dump_cap) break;
            dump[4 * n] = smp.t;
            dump[4 * n + 1] = smp.com[0];
            dump[4 * n + 2] = smp.com[1];
            dump[4 * n + 3] = smp.com[2];
            ++n;
        }
        return static_cast<int64_t>(samples.size());
    }
    return 0;
}

// ---------------------------------------------------------- evolution.hpp
// evaluate_fitness (evolution.hpp:110-119)
double ref_evaluate_fitness(int w, int h, int d, const uint8_t* mat, const double* wt, const double* table8,
                            const double* plane4, const double* sim6) {
    const VoxelGrid g = grid_from_flat(w, h, d, mat, wt);
    return evaluate_fitness(g, table_from(table8), plane_from(plane4), sim_from(sim6));
}
// population_diversity (evolution.hpp:89-105) over P raw grids of `cells` materials.
double ref_population_diversity(int P, int cells, const uint8_t* mats) {
    std::vector<Individual> pop(static_cast<std::size_t>(P));
    for (int a = 0; a < P; ++a) {
        pop[a].grid = VoxelGrid(cells, 1, 1);
        for (int c = 0; c < cells; ++c)
            pop[a].grid.cells[c].material = static_cast<Material>(mats[static_cast<std::size_t>(a) * cells + c]);
    }
    return population_diversity(pop);
}
// detail::elite_count (evolution.hpp:131-136)
int ref_elite_count(double elite_fraction, int population) { return detail::elite_count(elite_fraction, population); }
// HyperParams::clamp (evolution.hpp:29-35)
void ref_hyper_clamp(double* h7) {
    HyperParams p = hyper_from(h7);
    p.clamp();
    hyper_to(p, h7);
}

struct RefEvo {
    EvolutionState st;
};

// init_evolution (evolution.hpp:197-211).  hyper7 = mutation_rate,
// mutation_scale, crossover_rate, elite_fraction, multipliers[3].
void* ref_evo_init(int population, int generations, int gw, int gh, int gd, int nh, const int* widths, int m,
                   double sigma, int tournament, int threads, uint64_t seed, const double* hyper7,
                   const double* table8, const double* plane4, const double* sim6) {
    EvolutionConfig cfg;
    cfg.population = population;
    cfg.generations = generations;
    cfg.grid_w = gw;
    cfg.grid_h = gh;
    cfg.grid_d = gd;
    cfg.hidden_widths = widths_of(nh, widths);
    cfg.encoding = EncodingSpec{static_cast<std::size_t>(m), 3, sigma};
    cfg.tournament_size = tournament;
    cfg.threads = threads;
    cfg.seed = seed;
    if (hyper7) cfg.initial_params = hyper_from(hyper7);
    cfg.materials = table_from(table8);
    cfg.plane = plane_from(plane4);
    cfg.sim = sim_from(sim6);
    auto* e = new RefEvo;
    e->st = init_evolution(cfg);
    return e;
}
void ref_evo_free(void* h) { delete static_cast<RefEvo*>(h); }
void ref_evo_set_threads(void* h, int threads) { static_cast<RefEvo*>(h)->st.config.threads = threads; }

// evolve_generation (evolution.hpp:217-293), advisor off.
// rep = generation, best, mean, stddev, diversity, evaluations, wall_time, params[7]
void ref_evo_generation(void* h, double* rep) {
    auto* e = static_cast<RefEvo*>(h);
    const GenerationReport r = evolve_generation(e->st);
    rep[0] = r.generation;
    rep[1] = r.best;
    rep[2] = r.mean;
    rep[3] = r.stddev;
    rep[4] = r.diversity;
    rep[5] = r.evaluations;
    rep[6] = r.wall_time;
    hyper_to(r.params, rep + 7);
}
// bench.py --impl reference: one evolve_generation (evolution.hpp:217-293)
// timed alone; returns its wall seconds.  Afterwards, outside the timed
// region, an exact audit of the spring updates it performed: the individuals
// it had to evaluate (evaluated == false on entry) are decoded and evaluated
// again with the reference's own functions (same code path, deterministic),
// counting springs x steps exactly like simulate's ws.spring_updates
// (physics.hpp:212).  rep as ref_evo_generation.
double ref_evo_generation_timed(void* h, double* rep, uint64_t* updates) {
    auto* e = static_cast<RefEvo*>(h);
    std::vector<Genome> todo;
    for (const auto& ind : e->st.population)
        if (!ind.evaluated) todo.push_back(ind.genome);
    const EvolutionConfig cfg = e->st.config;
    const MaterialTable table = detail::scaled_materials(cfg.materials, e->st.params);
    const auto t0 = std::chrono::steady_clock::now();
    const GenerationReport r = evolve_generation(e->st);
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    rep[0] = r.generation;
    rep[1] = r.best;
    rep[2] = r.mean;
    rep[3] = r.stddev;
    rep[4] = r.diversity;
    rep[5] = r.evaluations;
    rep[6] = r.wall_time;
    hyper_to(r.params, rep + 7);
    std::vector<uint64_t> count(todo.size(), 0);
    const long long n_steps = std::llround(cfg.sim.duration / cfg.sim.dt);
    parallel_for(todo.size(), cfg.threads, [&](std::size_t a) {
        VoxelGrid body = largest_component(decode(todo[a], cfg.grid_w, cfg.grid_h, cfg.grid_d));
        if (body.count_non_empty() == 0 || !body.has_muscle()) return;
        MassSpringSystem sys = build_mass_spring(body, table, cfg.plane);
        SimWorkspace ws(sys);
        for (long long k = 0; k < n_steps; ++k)
            if (step(sys, static_cast<double>(k) * cfg.sim.dt, cfg.sim, ws) == StepResult::diverged) break;
        count[a] = ws.spring_updates;
    });
    uint64_t total = 0;
    for (uint64_t c : count) total += c;
    if (updates) *updates = total;
    return secs;
}

#ifdef VX_REF_HAVE_JSON
// evolve_generation(st, make_advisor_fn(&ScriptedAdvisor)) (evolution.hpp:
// 217-227, advisor.hpp:30-55, 166-171): the reference's own scripted advisor
// in the loop.  adv4 = diversity_floor, stagnation_eps, mutation_boost,
// crossover_boost (NULL: the class defaults).  rep as ref_evo_generation.
int ref_evo_generation_advised(void* h, double* rep, const double* adv4) {
    auto* e = static_cast<RefEvo*>(h);
    ScriptedAdvisor adv;
    if (adv4) {
        adv.diversity_floor = adv4[0];
        adv.stagnation_eps = adv4[1];
        adv.mutation_boost = adv4[2];
        adv.crossover_boost = adv4[3];
    }
    const GenerationReport r = evolve_generation(e->st, make_advisor_fn(&adv));
    rep[0] = r.generation;
    rep[1] = r.best;
    rep[2] = r.mean;
    rep[3] = r.stddev;
    rep[4] = r.diversity;
    rep[5] = r.evaluations;
    rep[6] = r.wall_time;
    hyper_to(r.params, rep + 7);
    return 1;
}
#else
int ref_evo_generation_advised(void*, double*, const double*) { return 0; }
#endif

// The fitness evolve_generation is about to compute for each individual that
// carries no cached score (evolution.hpp:229-241: decode if no grid, then
// evaluate_fitness with the scaled material table), NaN for the others.
// Deterministic: the same functions on the same inputs, so these are exactly
// the values the next evolve_generation stores (with the CURRENT params; an
// advisor changing material multipliers would need them applied first).
void ref_evo_pending_fitness(void* h, double* out) {
    auto* e = static_cast<RefEvo*>(h);
    const EvolutionConfig& cfg = e->st.config;
    const MaterialTable table = detail::scaled_materials(cfg.materials, e->st.params);
    const auto& pop = e->st.population;
    parallel_for(pop.size(), cfg.threads, [&](std::size_t i) {
        const Individual& ind = pop[i];
        if (ind.evaluated) {
            out[i] = std::numeric_limits<double>::quiet_NaN();
            return;
        }
        const VoxelGrid g = ind.grid.cells.empty() ? decode(ind.genome, cfg.grid_w, cfg.grid_h, cfg.grid_d) : ind.grid;
        out[i] = evaluate_fitness(g, table, cfg.plane, cfg.sim);
    });
}

int ref_evo_generation_index(void* h) { return static_cast<RefEvo*>(h)->st.generation; }
// Population export: params P x n_params, bmat P x 3m, fitness, evaluated,
// raw grids P x cells (material 255 where the grid is not decoded yet).
void ref_evo_get_population(void* h, double* params, double* bmat, double* fitness, uint8_t* evaluated,
                            uint8_t* grids, double* grid_w) {
    auto* e = static_cast<RefEvo*>(h);
    const auto& cfg = e->st.config;
    const std::size_t cells = static_cast<std::size_t>(cfg.grid_w) * cfg.grid_h * cfg.grid_d;
    std::size_t np = 0;
    for (std::size_t a = 0; a < e->st.population.size(); ++a) {
        const Individual& ind = e->st.population[a];
        np = ind.genome.parameter_count();
        genome_to_flat(ind.genome, params ? params + a * np : nullptr, nullptr);
        if (bmat) std::memcpy(bmat + a * ind.genome.b_matrix.size(), ind.genome.b_matrix.data(),
                              ind.genome.b_matrix.size() * sizeof(double));
        if (fitness) fitness[a] = ind.fitness;
        if (evaluated) evaluated[a] = ind.evaluated ? 1 : 0;
        for (std::size_t c = 0; c < cells; ++c) {
            const bool has = ind.grid.cells.size() == cells;
            if (grids) grids[a * cells + c] = has ? static_cast<uint8_t>(ind.grid.cells[c].material) : 255;
            if (grid_w) grid_w[a * cells + c] = has ? ind.grid.cells[c].weight : 0.0;
        }
    }
}
// Replace the population (for breeding-parity tests).  grids may be NULL
// (individuals then have no cached grid and will be re-decoded).
void ref_evo_set_population(void* h, const double* params, const double* bmat, const double* fitness,
                            const uint8_t* evaluated, const uint8_t* grids, const double* grid_w) {
    auto* e = static_cast<RefEvo*>(h);
    const auto& cfg = e->st.config;
    const int m = static_cast<int>(cfg.encoding.m);
    std::vector<int> widths;
    for (auto w : cfg.hidden_widths) widths.push_back(static_cast<int>(w));
    const std::size_t cells = static_cast<std::size_t>(cfg.grid_w) * cfg.grid_h * cfg.grid_d;
    for (std::size_t a = 0; a < e->st.population.size(); ++a) {
        Individual& ind = e->st.population[a];
        const std::size_t np = ind.genome.parameter_count();
        Genome g = genome_from_flat(m, static_cast<int>(widths.size()), widths.data(), params + a * np,
                                    bmat + a * 3 * m);
        g.spec.sigma = cfg.encoding.sigma;
        ind.genome = std::move(g);
        ind.fitness = fitness ? fitness[a] : 0.0;
        ind.evaluated = evaluated ? evaluated[a] != 0 : false;
        if (grids) {
            ind.grid = VoxelGrid(cfg.grid_w, cfg.grid_h, cfg.grid_d);
            for (std::size_t c = 0; c < cells; ++c) {
                ind.grid.cells[c].material = static_cast<Material>(grids[a * cells + c]);
                ind.grid.cells[c].weight = grid_w ? grid_w[a * cells + c] : 1.0;
            }
        } else {
            ind.grid = VoxelGrid(0, 0, 0);
        }
    }
}
int64_t ref_evo_rng_state(void* h, char* buf, int64_t cap) {
    const std::string s = static_cast<RefEvo*>(h)->st.rng.state();
    if (buf && cap > 0) {
        std::strncpy(buf, s.c_str(), static_cast<std::size_t>(cap - 1));
        buf[cap - 1] = 0;
    }
    return static_cast<int64_t>(s.size());
}
void ref_evo_set_rng_state(void* h, const char* s) { static_cast<RefEvo*>(h)->st.rng.set_state(s); }
void ref_evo_get_params(void* h, double* hyper7) { hyper_to(static_cast<RefEvo*>(h)->st.params, hyper7); }
void ref_evo_set_params(void* h, const double* hyper7) {
    auto* e = static_cast<RefEvo*>(h);
    e->st.params = hyper_from(hyper7);
}
// best_fitness / best_genome (evolution.hpp:246-249)
int ref_evo_best(void* h, double* best_fitness, double* best_params) {
    auto* e = static_cast<RefEvo*>(h);
    *best_fitness = e->st.best_fitness;
    if (!e->st.best_genome) return 0;
    if (best_params) genome_to_flat(*e->st.best_genome, best_params, nullptr);
    return 1;
}

// --------------------------------------------------------------- bench.hpp
// run_bench (bench.hpp:50-86).  out = springs_per_robot, spring_updates,
// expected_updates, seconds, updates_per_second, diverged
void ref_run_bench(int jobs, int64_t steps, int threads, int grid, double dt, double* out) {
    BenchConfig cfg;
    cfg.jobs = jobs;
    cfg.steps = steps;
    cfg.threads = threads;
    cfg.grid = grid;
    cfg.dt = dt;
    const BenchResult r = run_bench(cfg);
    out[0] = static_cast<double>(r.springs_per_robot);
    out[1] = static_cast<double>(r.spring_updates);
    out[2] = static_cast<double>(r.expected_updates);
    out[3] = r.seconds;
    out[4] = r.updates_per_second;
    out[5] = r.diverged ? 1.0 : 0.0;
}

// CPU baseline for bench.py: evaluate_fitness (evolution.hpp:110-119) over
// the given raw grids through the reference's own parallel_for
// (parallel.hpp:17-51) with `threads` workers, exactly as
// evolve_generation does (evolution.hpp:237-241).  Returns wall seconds;
// fitness[] receives the scores and *updates the exact spring-update count
// (springs x steps for every simulated, non-diverged robot; diverged robots
// count the steps they ran).
double ref_evaluate_batch(int n, int w, int h, int d, const uint8_t* mats, const double* wts, const double* table8,
                          const double* plane4, const double* sim6, int threads, double* fitness,
                          uint64_t* updates) {
    const std::size_t cells = static_cast<std::size_t>(w) * h * d;
    std::vector<VoxelGrid> grids;
    grids.reserve(n);
    for (int a = 0; a < n; ++a) grids.push_back(grid_from_flat(w, h, d, mats + a * cells, wts + a * cells));
    const MaterialTable table = table_from(table8);
    const GroundPlane plane = plane_from(plane4);
    const SimConfig sim = sim_from(sim6);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(static_cast<std::size_t>(n), threads,
                 [&](std::size_t a) { fitness[a] = evaluate_fitness(grids[a], table, plane, sim); });
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // work audit outside the timed region
    uint64_t total = 0;
    const long long n_steps = std::llround(sim.duration / sim.dt);
    for (int a = 0; a < n; ++a) {
        VoxelGrid body = largest_component(grids[a]);
        if (body.count_non_empty() == 0 || !body.has_muscle()) continue;
        MassSpringSystem sys = build_mass_spring(body, table, plane);
        if (fitness[a] != 0.0) {
            total += static_cast<uint64_t>(n_steps) * sys.springs.size();
        } else {
            SimWorkspace ws(sys);
            for (long long k = 0; k < n_steps; ++k)
                if (step(sys, static_cast<double>(k) * sim.dt, sim, ws) == StepResult::diverged) break;
            total += ws.spring_updates;
        }
    }
    if (updates) *updates = total;
    return secs;
}

}  // extern "C"
