// voxevo_shim.hpp — header-only C++ drop-in for the reference's voxevo:: hot
// path, backed by the B200 C ABI (include/voxevo_b200.h).
//
// Include AFTER the reference headers (it uses voxevo::EvolutionConfig,
// VoxelGrid, MassSpringSystem, ... unchanged).  Entry points mirror the
// reference's names and semantics:
//   voxevo::b200::decode            <- voxevo::decode            (morphology.hpp:141)
//   voxevo::b200::largest_component <- voxevo::largest_component (morphology.hpp:162)
//   voxevo::b200::build_mass_spring <- voxevo::build_mass_spring (morphology.hpp:217)
//   voxevo::b200::simulate          <- voxevo::simulate          (physics.hpp:287)
//   voxevo::b200::evaluate_fitness  <- voxevo::evaluate_fitness  (evolution.hpp:110)
//   voxevo::b200::population_diversity <- (evolution.hpp:89)
//   voxevo::b200::GpuEvolution      <- init_evolution / evolve_generation (evolution.hpp:197-293)
//   voxevo::b200::run_bench         <- voxevo::run_bench         (bench.hpp:50)
// Errors map back to the reference's exception types.
#pragma once

#include <optional>
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../voxevo_b200.h"

namespace voxevo::b200 {

inline void check(vx_status s) {
    if (s == VX_OK) return;
    const std::string msg = vx_last_error();
    if (s == VX_EINVAL) throw std::invalid_argument(msg);
    if (s == VX_EEMPTY) throw voxevo::empty_robot(msg);
    if (s == VX_ESHAPE) throw voxevo::shape_mismatch(msg);
    throw std::runtime_error("voxevo_b200: " + msg);
}

// One device context per process/thread of use.
class Device {
  public:
    explicit Device(int device = 0) { check(vx_create(device, &ctx_)); }
    ~Device() { vx_destroy(ctx_); }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    vx_ctx* get() const { return ctx_; }

  private:
    vx_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
    static Device d(0);
    return d;
}

inline vx_arch to_c(const Genome& g) {
    vx_arch a{};
    a.m = static_cast<int32_t>(g.spec.m);
    a.sigma = g.spec.sigma;
    a.n_hidden = static_cast<int32_t>(g.hidden.size());
    for (size_t i = 0; i < g.hidden.size(); ++i) a.hidden[i] = static_cast<int32_t>(g.hidden[i].out);
    return a;
}
inline vx_materials to_c(const MaterialTable& t) {
    return {t.k_muscle, t.k_soft, t.k_bone, t.damping_ratio, t.amp_max, t.phase_max, t.voxel_edge, t.mass_per_vertex};
}
inline vx_plane to_c(const GroundPlane& p) { return {p.k, p.damping_ratio, p.mu_static, p.mu_kinetic}; }
inline vx_sim to_c(const SimConfig& s) {
    return {s.gravity, s.dt, s.duration, s.actuation_frequency, s.enable_gravity ? 1 : 0, s.enable_contact ? 1 : 0};
}
inline vx_hyper to_c(const HyperParams& p) {
    return {p.mutation_rate, p.mutation_scale, p.crossover_rate, p.elite_fraction,
            {p.material_multipliers[0], p.material_multipliers[1], p.material_multipliers[2]}};
}
inline HyperParams from_c(const vx_hyper& h) {
    HyperParams p;
    p.mutation_rate = h.mutation_rate;
    p.mutation_scale = h.mutation_scale;
    p.crossover_rate = h.crossover_rate;
    p.elite_fraction = h.elite_fraction;
    p.material_multipliers = {h.material_multipliers[0], h.material_multipliers[1], h.material_multipliers[2]};
    return p;
}
inline vx_evo_config to_c(const EvolutionConfig& c) {
    vx_evo_config x;
    vx_default_evo_config(&x);
    x.population = c.population;
    x.generations = c.generations;
    x.grid_w = c.grid_w;
    x.grid_h = c.grid_h;
    x.grid_d = c.grid_d;
    x.tournament_size = c.tournament_size;
    x.threads = c.threads;
    x.seed = c.seed;
    x.arch.m = static_cast<int32_t>(c.encoding.m);
    x.arch.sigma = c.encoding.sigma;
    x.arch.n_hidden = static_cast<int32_t>(c.hidden_widths.size());
    for (size_t i = 0; i < c.hidden_widths.size(); ++i) x.arch.hidden[i] = static_cast<int32_t>(c.hidden_widths[i]);
    x.initial_params = to_c(c.initial_params);
    x.materials = to_c(c.materials);
    x.plane = to_c(c.plane);
    x.sim = to_c(c.sim);
    return x;
}

inline void flatten(const Genome& g, std::vector<double>& params) {
    for (const auto* t : g.param_tensors()) params.insert(params.end(), t->begin(), t->end());
}

// The inverse: a reference Genome (param_tensors order, genome.hpp:57-68) from
// the flat device layout of one individual.
inline Genome unflatten(const EvolutionConfig& cfg, const double* params, const double* bmat) {
    Genome g;
    g.spec = cfg.encoding;
    g.b_matrix.assign(bmat, bmat + g.spec.m * g.spec.d);
    auto layer = [&](std::size_t in, std::size_t out) {
        Layer l;
        l.in = in;
        l.out = out;
        l.w.assign(params, params + in * out);
        params += in * out;
        l.b.assign(params, params + out);
        params += out;
        return l;
    };
    std::size_t prev = 2 * g.spec.m;
    for (const std::size_t w : cfg.hidden_widths) {
        g.hidden.push_back(layer(prev, w));
        prev = w;
    }
    g.head_material = layer(prev, 5);
    g.head_weight = layer(prev, 1);
    return g;
}

// forward (genome.hpp:187-211) for a batch of query points of one genome
// (one launch); MaterialQuery per point.
inline std::vector<MaterialQuery> forward(const Genome& g, const std::vector<Vec3>& points,
                                          Device& dev = default_device()) {
    std::vector<MaterialQuery> out(points.size());
    if (points.empty()) return out;
    const vx_arch a = to_c(g);
    std::vector<double> params, pts(3 * points.size()), probs(5 * points.size()), wt(points.size());
    flatten(g, params);
    for (size_t q = 0; q < points.size(); ++q)
        for (int c = 0; c < 3; ++c) pts[3 * q + c] = points[q][c];
    check(vx_forward(dev.get(), &a, 1, params.data(), g.b_matrix.data(), static_cast<int32_t>(points.size()),
                     pts.data(), probs.data(), wt.data()));
    for (size_t q = 0; q < points.size(); ++q) {
        for (int i = 0; i < 5; ++i) out[q].probs[i] = probs[5 * q + i];
        out[q].weight = wt[q];
    }
    return out;
}
inline MaterialQuery forward(const Genome& g, const Vec3& v, Device& dev = default_device()) {
    return forward(g, std::vector<Vec3>{v}, dev)[0];
}

// decode (morphology.hpp:141-157)
inline VoxelGrid decode(const Genome& g, int w, int h, int d, Device& dev = default_device()) {
    if (w < 1 || h < 1 || d < 1) throw std::invalid_argument("decode: dims must be positive");
    const vx_arch a = to_c(g);
    std::vector<double> params;
    flatten(g, params);
    VoxelGrid grid(w, h, d);
    std::vector<uint8_t> mat(grid.size());
    std::vector<double> wt(grid.size());
    check(vx_decode(dev.get(), &a, 1, params.data(), g.b_matrix.data(), w, h, d, mat.data(), wt.data()));
    for (size_t i = 0; i < grid.size(); ++i) grid.cells[i] = Cell{static_cast<Material>(mat[i]), wt[i]};
    return grid;
}

// largest_component (morphology.hpp:162-208)
inline VoxelGrid largest_component(const VoxelGrid& grid, Device& dev = default_device()) {
    std::vector<uint8_t> in(grid.size()), out(grid.size());
    for (size_t i = 0; i < grid.size(); ++i) in[i] = static_cast<uint8_t>(grid.cells[i].material);
    check(vx_largest_component(dev.get(), 1, grid.w, grid.h, grid.d, in.data(), out.data()));
    VoxelGrid r = grid;
    for (size_t i = 0; i < grid.size(); ++i) r.cells[i].material = static_cast<Material>(out[i]);
    return r;
}

// build_mass_spring (morphology.hpp:217-299)
inline MassSpringSystem build_mass_spring(const VoxelGrid& grid, const MaterialTable& table,
                                          const GroundPlane& plane = GroundPlane{}, Device& dev = default_device()) {
    std::vector<uint8_t> mat(grid.size());
    std::vector<double> wt(grid.size());
    for (size_t i = 0; i < grid.size(); ++i) {
        mat[i] = static_cast<uint8_t>(grid.cells[i].material);
        wt[i] = grid.cells[i].weight;
    }
    const vx_materials t = to_c(table);
    const vx_plane p = to_c(plane);
    vx_batch* b = nullptr;
    check(vx_batch_build(dev.get(), 1, grid.w, grid.h, grid.d, mat.data(), wt.data(), &t, &p, &b));
    int64_t mo[2], so[2];
    vx_batch_offsets(b, mo, so);
    const int64_t nm = mo[1], ns = so[1];
    if (nm == 0) {
        vx_batch_free(b);
        throw empty_robot("build_mass_spring: no occupied voxel");
    }
    std::vector<double> pos(3 * nm), vel(3 * nm), mass(nm), k(ns), rest0(ns), zeta(ns), sign(ns), amp(ns), phase(ns);
    std::vector<int32_t> si(ns), sj(ns);
    std::vector<uint8_t> act(ns);
    check(vx_batch_download(b, pos.data(), vel.data(), mass.data(), si.data(), sj.data(), k.data(), rest0.data(),
                            zeta.data(), act.data(), sign.data(), amp.data(), phase.data()));
    vx_batch_free(b);
    MassSpringSystem sys;
    sys.plane = plane;
    sys.masses.resize(nm);
    for (int64_t a = 0; a < nm; ++a) {
        sys.masses[a].pos = {pos[3 * a], pos[3 * a + 1], pos[3 * a + 2]};
        sys.masses[a].vel = {vel[3 * a], vel[3 * a + 1], vel[3 * a + 2]};
        sys.masses[a].mass = mass[a];
    }
    sys.springs.resize(ns);
    for (int64_t q = 0; q < ns; ++q) {
        Spring& s = sys.springs[q];
        s.i = si[q];
        s.j = sj[q];
        s.k = k[q];
        s.rest0 = rest0[q];
        s.damping_ratio = zeta[q];
        if (act[q]) s.act = Actuation{sign[q], amp[q], phase[q]};
    }
    return sys;
}

// simulate (physics.hpp:280-311), including the optional COM dump every
// `stride` steps; the system is taken by value like the reference's.
inline TrajectorySummary simulate(const MassSpringSystem& sys, const SimConfig& cfg,
                                  std::vector<TrajectorySample>* dump = nullptr, int stride = 0,
                                  Device& dev = default_device()) {
    cfg.validate();
    TrajectorySummary out;
    if (sys.masses.empty()) return out;
    const int64_t nm = static_cast<int64_t>(sys.masses.size()), ns = static_cast<int64_t>(sys.springs.size());
    const int64_t mo[2] = {0, nm}, so[2] = {0, ns};
    std::vector<double> pos(3 * nm), vel(3 * nm), mass(nm), k(ns), rest0(ns), zeta(ns), sign(ns), amp(ns), phase(ns);
    std::vector<int32_t> si(ns), sj(ns);
    std::vector<uint8_t> act(ns);
    for (int64_t a = 0; a < nm; ++a) {
        for (int c = 0; c < 3; ++c) {
            pos[3 * a + c] = sys.masses[a].pos[c];
            vel[3 * a + c] = sys.masses[a].vel[c];
        }
        mass[a] = sys.masses[a].mass;
    }
    for (int64_t q = 0; q < ns; ++q) {
        const Spring& s = sys.springs[q];
        si[q] = s.i;
        sj[q] = s.j;
        k[q] = s.k;
        rest0[q] = s.rest0;
        zeta[q] = s.damping_ratio;
        act[q] = s.act ? 1 : 0;
        sign[q] = s.act ? s.act->sign : 0.0;
        amp[q] = s.act ? s.act->amplitude : 0.0;
        phase[q] = s.act ? s.act->phase : 0.0;
    }
    const vx_plane p = to_c(sys.plane);
    vx_batch* b = nullptr;
    check(vx_batch_upload(dev.get(), 1, mo, so, pos.data(), vel.data(), mass.data(), si.data(), sj.data(), k.data(),
                          rest0.data(), zeta.data(), act.data(), sign.data(), amp.data(), phase.data(), &p, &b));
    const vx_sim s = to_c(cfg);
    vx_summary sum{};
    vx_status st;
    if (dump) {
        const long long n_steps = std::llround(cfg.duration / cfg.dt);
        const int64_t cap = (stride > 0 ? (n_steps + stride - 1) / stride : 0) + 1;
        std::vector<double> rows(4 * static_cast<size_t>(cap));
        int64_t count = 0;
        st = vx_batch_simulate_dump(dev.get(), b, &s, stride, cap, rows.data(), &count, &sum);
        for (int64_t q = 0; st == VX_OK && q < std::min(count, cap); ++q)
            dump->push_back({rows[4 * q], {rows[4 * q + 1], rows[4 * q + 2], rows[4 * q + 3]}});
    } else {
        st = vx_batch_simulate(dev.get(), b, &s, &sum);
    }
    vx_batch_free(b);
    check(st);
    out.com_start = {sum.com_start[0], sum.com_start[1], sum.com_start[2]};
    out.com_end = {sum.com_end[0], sum.com_end[1], sum.com_end[2]};
    out.horizontal_displacement = sum.horizontal_displacement;
    out.max_speed = sum.max_speed;
    out.diverged = sum.diverged != 0;
    return out;
}

// evaluate_fitness (evolution.hpp:110-119), batched: one launch for all grids.
inline std::vector<double> evaluate_fitness(const std::vector<VoxelGrid>& raw, const MaterialTable& table,
                                            const GroundPlane& plane, const SimConfig& sim,
                                            Device& dev = default_device()) {
    if (raw.empty()) return {};
    const VoxelGrid& g0 = raw[0];
    std::vector<uint8_t> mat;
    std::vector<double> wt;
    for (const auto& g : raw) {
        if (!g.same_dims(g0)) throw std::invalid_argument("evaluate_fitness: grids differ in size");
        for (const auto& c : g.cells) {
            mat.push_back(static_cast<uint8_t>(c.material));
            wt.push_back(c.weight);
        }
    }
    const vx_materials t = to_c(table);
    const vx_plane p = to_c(plane);
    const vx_sim s = to_c(sim);
    std::vector<double> fit(raw.size());
    check(vx_evaluate(dev.get(), static_cast<int32_t>(raw.size()), g0.w, g0.h, g0.d, mat.data(), wt.data(), &t, &p,
                      &s, fit.data(), nullptr));
    return fit;
}
inline double evaluate_fitness(const VoxelGrid& raw, const MaterialTable& table, const GroundPlane& plane,
                               const SimConfig& sim, Device& dev = default_device()) {
    return evaluate_fitness(std::vector<VoxelGrid>{raw}, table, plane, sim, dev)[0];
}

// Device-resident EvolutionState: init_evolution + evolve_generation with
// the advisor consulted where evolution.hpp:221-227 consults it.
class GpuEvolution {
  public:
    explicit GpuEvolution(const EvolutionConfig& cfg, Device& dev = default_device()) : cfg_(cfg), dev_(dev) {
        cfg.validate();
        const vx_evo_config c = to_c(cfg);
        check(vx_evo_create(dev.get(), &c, &evo_));
    }
    ~GpuEvolution() { vx_evo_free(evo_); }
    GpuEvolution(const GpuEvolution&) = delete;
    GpuEvolution& operator=(const GpuEvolution&) = delete;

    GenerationReport evolve_generation(const AdvisorFn& advisor = nullptr) {
        if (advisor && static_cast<int>(history.size()) >= kAdvisorWindow) {
            std::vector<GenerationReport> window(history.end() - kAdvisorWindow, history.end());
            vx_hyper cur;
            check(vx_evo_get_params(evo_, &cur));
            if (auto adj = advisor(window, from_c(cur))) {
                const vx_hyper h = to_c(*adj);
                check(vx_evo_set_params(evo_, &h));  // clamped like the reference
            }
        }
        vx_report r;
        check(vx_evo_generation(evo_, &r));
        GenerationReport rep;
        rep.generation = r.generation;
        rep.params = from_c(r.params);
        rep.best = r.best;
        rep.mean = r.mean;
        rep.stddev = r.stddev;
        rep.diversity = r.diversity;
        rep.evaluations = r.evaluations;
        rep.wall_time = r.wall_time;
        history.push_back(rep);
        return rep;
    }
    // Replace the population with reference genomes (e.g. from init_evolution).
    void set_population(const std::vector<Individual>& pop) {
        std::vector<double> params, bmat, fit;
        std::vector<uint8_t> ev;
        for (const auto& ind : pop) {
            flatten(ind.genome, params);
            bmat.insert(bmat.end(), ind.genome.b_matrix.begin(), ind.genome.b_matrix.end());
            fit.push_back(ind.fitness);
            ev.push_back(ind.evaluated ? 1 : 0);
        }
        check(vx_evo_set_population(evo_, params.data(), bmat.data(), fit.data(), ev.data(), nullptr, nullptr));
    }
    std::string rng_state() const {  // libstdc++ mt19937_64 text, like Rng::state()
        std::string s(static_cast<size_t>(vx_evo_rng_state(evo_, nullptr, 0)), '\0');
        vx_evo_rng_state(evo_, s.data(), static_cast<int64_t>(s.size()) + 1);
        return s;
    }
    void set_rng_state(const std::string& s) { check(vx_evo_set_rng_state(evo_, s.c_str())); }
    double best_fitness() const {
        double b = 0.0;
        vx_evo_best(evo_, &b, nullptr);
        return b;
    }
    // Resume from a reference EvolutionState — e.g. voxevo::load_run
    // (serialize.hpp:311-313): genomes, fitness / evaluated flags (grids are
    // decoded again, as after a reference load), params, history, generation,
    // best fitness / genome and the GA's RNG stream.
    void load_state(const EvolutionState& st) {
        set_population(st.population);
        const vx_hyper h = to_c(st.params);
        check(vx_evo_set_params(evo_, &h));
        set_rng_state(st.rng.state());
        history = st.history;
        std::vector<double> bp;
        if (st.best_genome) flatten(*st.best_genome, bp);
        check(vx_evo_set_progress(evo_, st.generation, st.best_fitness, st.best_genome ? bp.data() : nullptr,
                                  st.best_genome ? st.best_genome->b_matrix.data() : nullptr));
    }
    // The device state as a reference EvolutionState, ready for
    // voxevo::save_run (serialize.hpp:307-309).
    EvolutionState to_state() const {
        EvolutionState st;
        st.config = cfg_;
        vx_hyper h;
        check(vx_evo_get_params(evo_, &h));
        st.params = from_c(h);
        const vx_evo_config c = to_c(cfg_);
        const std::size_t np = static_cast<std::size_t>(vx_param_count(&c.arch)), nb = 3 * cfg_.encoding.m;
        const std::size_t P = static_cast<std::size_t>(cfg_.population);
        std::vector<double> params(P * np), bmat(P * nb), fit(P);
        std::vector<uint8_t> ev(P);
        check(vx_evo_get_population(evo_, params.data(), bmat.data(), fit.data(), ev.data(), nullptr, nullptr));
        for (std::size_t i = 0; i < P; ++i) {
            Individual ind;
            ind.genome = unflatten(cfg_, params.data() + i * np, bmat.data() + i * nb);
            ind.fitness = fit[i];
            ind.evaluated = ev[i] != 0;
            st.population.push_back(std::move(ind));
        }
        st.history = history;
        st.generation = vx_evo_generation_index(evo_);
        std::vector<double> bp(np), bb(nb);
        double bf = 0.0;
        if (vx_evo_best_genome(evo_, &bf, bp.data(), bb.data())) st.best_genome = unflatten(cfg_, bp.data(), bb.data());
        st.best_fitness = bf;
        st.rng.set_state(rng_state());
        return st;
    }
    std::vector<GenerationReport> history;

  private:
    EvolutionConfig cfg_;
    Device& dev_;
    vx_evo* evo_ = nullptr;
};

// run_bench (bench.hpp:50-86)
inline BenchResult run_bench(const BenchConfig& cfg, Device& dev = default_device()) {
    double out[6];
    check(vx_run_bench(dev.get(), cfg.jobs, cfg.steps, cfg.grid, cfg.dt, out));
    BenchResult r;
    r.threads = cfg.threads;
    r.jobs = cfg.jobs;
    r.steps = cfg.steps;
    r.springs_per_robot = static_cast<std::size_t>(out[0]);
    r.spring_updates = static_cast<std::uint64_t>(out[1]);
    r.expected_updates = static_cast<std::uint64_t>(out[2]);
    r.seconds = out[3];
    r.updates_per_second = out[4];
    r.diverged = out[5] != 0.0;
    return r;
}

}  // namespace voxevo::b200
