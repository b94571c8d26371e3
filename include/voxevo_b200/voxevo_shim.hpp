// voxevo_shim.hpp — header-only C++ drop-in for the reference's voxevo:: hot
// path, backed by the B200 C ABI (include/voxevo_b200.h).
//
// Include AFTER the reference headers (it uses voxevo::EvolutionConfig,
// VoxelGrid, MassSpringSystem, ... unchanged).  Entry points mirror the
// reference's names, signatures and semantics:
//   voxevo::b200::sample_genome     <- voxevo::sample_genome     (genome.hpp:146)
//   voxevo::b200::gaussian_encode   <- voxevo::gaussian_encode   (genome.hpp:169)
//   voxevo::b200::forward           <- voxevo::forward           (genome.hpp:187)
//   voxevo::b200::decode            <- voxevo::decode            (morphology.hpp:141)
//   voxevo::b200::largest_component <- voxevo::largest_component (morphology.hpp:162)
//   voxevo::b200::build_mass_spring <- voxevo::build_mass_spring (morphology.hpp:217)
//   voxevo::b200::step              <- voxevo::step              (physics.hpp:191)
//   voxevo::b200::simulate          <- voxevo::simulate          (physics.hpp:287)
//   voxevo::b200::evaluate_fitness  <- voxevo::evaluate_fitness  (evolution.hpp:110)
//   voxevo::b200::population_diversity <- voxevo::population_diversity (evolution.hpp:89)
//   voxevo::b200::crossover / mutate / tournament_select
//                                   <- voxevo::detail::*         (evolution.hpp:143-173)
//   voxevo::b200::init_evolution    <- voxevo::init_evolution    (evolution.hpp:197)
//   voxevo::b200::evolve_generation <- voxevo::evolve_generation (evolution.hpp:217)
//   voxevo::b200::GpuEvolution      device-resident EvolutionState (one GPU, or
//                                   a rank of a sharded run: Communicator)
//   voxevo::b200::run_bench         <- voxevo::run_bench         (bench.hpp:50)
// Errors map back to the reference's exception types.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <optional>
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

inline void check_depth(std::size_t n_hidden) {
    if (n_hidden > VX_MAX_HIDDEN)
        throw std::invalid_argument("voxevo_b200: at most " + std::to_string(VX_MAX_HIDDEN) + " hidden layers");
}

inline vx_arch to_c(const Genome& g) {
    check_depth(g.hidden.size());
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
    check_depth(c.hidden_widths.size());
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

inline Genome unflatten(const EncodingSpec& spec, const std::vector<std::size_t>& hidden, const double* params,
                        const double* bmat) {
    EvolutionConfig c;
    c.encoding = spec;
    c.hidden_widths = hidden;
    return unflatten(c, params, bmat);
}

// sample_genome (genome.hpp:146-166): the genome's own mt19937_64 stream;
// layer weights drawn on device (exact uniforms), B with the host glibc
// Box-Muller — bit-identical to the reference.
inline Genome sample_genome(const EncodingSpec& spec, const std::vector<std::size_t>& hidden_widths,
                            std::uint64_t seed, Device& dev = default_device()) {
    spec.validate();
    for (std::size_t w : hidden_widths)
        if (w < 1) throw std::invalid_argument("sample_genome: hidden widths must be >= 1");
    check_depth(hidden_widths.size());
    vx_arch a{};
    a.m = static_cast<int32_t>(spec.m);
    a.sigma = spec.sigma;
    a.n_hidden = static_cast<int32_t>(hidden_widths.size());
    for (std::size_t i = 0; i < hidden_widths.size(); ++i) a.hidden[i] = static_cast<int32_t>(hidden_widths[i]);
    std::vector<double> params(static_cast<std::size_t>(vx_param_count(&a))), bmat(3 * spec.m);
    check(vx_sample_genomes(dev.get(), &a, 1, &seed, params.data(), bmat.data()));
    return unflatten(spec, hidden_widths, params.data(), bmat.data());
}

// gaussian_encode (genome.hpp:169-179): host libm, bit-identical.
inline std::vector<double> gaussian_encode(const Vec3& v, const std::vector<double>& b_matrix, std::size_t m) {
    std::vector<double> out(2 * m);
    const double p[3] = {v[0], v[1], v[2]};
    check(vx_gaussian_encode(p, b_matrix.data(), static_cast<int32_t>(m), out.data()));
    return out;
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

// A one-robot device batch holding `sys`, with the actuation phases'
// sin/cos taken from the host libm exactly as SimWorkspace computes them
// (physics.hpp:154-159), so the device integrator is bit-identical.
inline vx_batch* upload_system(const MassSpringSystem& sys, Device& dev) {
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
    std::vector<double> sph(ns), cph(ns);
    for (int64_t q = 0; q < ns; ++q) {
        const Spring& sp = sys.springs[q];
        sph[q] = sp.act ? std::sin(sp.act->phase) : 0.0;
        cph[q] = sp.act ? std::cos(sp.act->phase) : 1.0;
    }
    const vx_status st = vx_batch_override_phase(b, sph.data(), cph.data());
    if (st != VX_OK) {
        vx_batch_free(b);
        check(st);
    }
    return b;
}

// step (physics.hpp:191-264): one step of `sys` at time t on the device,
// bit-identical to the reference's; the workspace's counters are updated
// like the reference's (spring_updates += ns once phase 1 completes,
// max_speed_sq over the new velocities).
inline StepResult step(MassSpringSystem& sys, double t, const SimConfig& cfg, SimWorkspace& ws,
                       Device& dev = default_device()) {
    if (sys.masses.empty()) return StepResult::ok;
    vx_batch* b = upload_system(sys, dev);
    const vx_sim s = to_c(cfg);
    vx_summary sum{};
    const int64_t nm = static_cast<int64_t>(sys.masses.size());
    std::vector<double> pos(3 * nm), vel(3 * nm);
    vx_status st = vx_batch_step_at(dev.get(), b, &s, t, &sum);
    if (st == VX_OK)
        st = vx_batch_download(b, pos.data(), vel.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                               nullptr, nullptr, nullptr, nullptr);
    vx_batch_free(b);
    check(st);
    ws.spring_updates += sum.spring_updates;
    if (sum.spring_updates == 0 && !sys.springs.empty()) return StepResult::diverged;  // zero-length: untouched
    for (int64_t a = 0; a < nm; ++a) {
        PointMass& m = sys.masses[a];
        m.pos = {pos[3 * a], pos[3 * a + 1], pos[3 * a + 2]};
        m.vel = {vel[3 * a], vel[3 * a + 1], vel[3 * a + 2]};
        const double speed_sq = m.vel[0] * m.vel[0] + m.vel[1] * m.vel[1] + m.vel[2] * m.vel[2];
        if (speed_sq > ws.max_speed_sq) ws.max_speed_sq = speed_sq;
    }
    return sum.diverged ? StepResult::diverged : StepResult::ok;
}

// simulate (physics.hpp:280-311), including the optional COM dump every
// `stride` steps; the system is taken by value like the reference's.
inline TrajectorySummary simulate(const MassSpringSystem& sys, const SimConfig& cfg,
                                  std::vector<TrajectorySample>* dump = nullptr, int stride = 0,
                                  Device& dev = default_device()) {
    cfg.validate();
    TrajectorySummary out;
    if (sys.masses.empty()) return out;
    vx_batch* b = upload_system(sys, dev);
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

// population_diversity (evolution.hpp:89-105) over the raw grids: the
// reference's double bit for bit (pair counts and its ordered running sum,
// reproduced on device).
inline double population_diversity(const std::vector<Individual>& pop, Device& dev = default_device()) {
    if (pop.size() < 2) return 0.0;
    const std::size_t cells = pop[0].grid.cells.size();
    if (cells == 0) return 0.0;
    std::vector<uint8_t> mat;
    mat.reserve(pop.size() * cells);
    for (const auto& ind : pop) {
        if (ind.grid.cells.size() != cells) throw std::invalid_argument("population_diversity: grids differ in size");
        for (const auto& c : ind.grid.cells) mat.push_back(static_cast<uint8_t>(c.material));
    }
    double out = 0.0;
    check(vx_population_diversity(dev.get(), static_cast<int32_t>(pop.size()), static_cast<int32_t>(cells), mat.data(),
                                  &out));
    return out;
}

// The GA operators on the CALLER's voxevo::Rng (evolution.hpp:143-173,
// detail::crossover / mutate / tournament_select): the library's host
// mt19937_64 continues the caller's stream from its text state and hands it
// back, so draws, decisions and noise are bit-identical.
class RngBridge {
  public:
    explicit RngBridge(Rng& rng) : rng_(rng) {
        check(vx_rng_create(0, &r_));
        const std::string st = rng.state();
        const vx_status s = vx_rng_set_state(r_, st.c_str());
        if (s != VX_OK) {
            vx_rng_free(r_);
            check(s);
        }
    }
    ~RngBridge() {
        std::string st(static_cast<std::size_t>(vx_rng_state(r_, nullptr, 0)), '\0');
        vx_rng_state(r_, st.data(), static_cast<int64_t>(st.size()) + 1);
        rng_.set_state(st);
        vx_rng_free(r_);
    }
    RngBridge(const RngBridge&) = delete;
    RngBridge& operator=(const RngBridge&) = delete;
    vx_rng* get() const { return r_; }

  private:
    Rng& rng_;
    vx_rng* r_ = nullptr;
};

inline Genome crossover(const Genome& a, const Genome& b, Rng& rng) {
    if (!a.same_architecture(b)) throw shape_mismatch("crossover: parents differ in architecture");
    std::vector<double> pa, pb;
    flatten(a, pa);
    flatten(b, pb);
    std::vector<double> child(pa.size());
    {
        RngBridge r(rng);
        check(vx_crossover(r.get(), static_cast<int64_t>(pa.size()), pa.data(), pb.data(), child.data()));
    }
    Genome g = a;  // B and the architecture from parent a
    const double* p = child.data();
    for (auto* t : g.param_tensors()) {
        std::copy(p, p + t->size(), t->begin());
        p += t->size();
    }
    return g;
}

inline void mutate(Genome& g, double rate, double scale, Rng& rng) {
    std::vector<double> params;
    flatten(g, params);
    {
        RngBridge r(rng);
        check(vx_mutate(r.get(), static_cast<int64_t>(params.size()), params.data(), rate, scale));
    }
    const double* p = params.data();
    for (auto* t : g.param_tensors()) {
        std::copy(p, p + t->size(), t->begin());
        p += t->size();
    }
}

inline const Individual& tournament_select(const std::vector<Individual>& pop, int size, Rng& rng) {
    RngBridge r(rng);
    const int32_t w = vx_tournament_select(r.get(), static_cast<int32_t>(pop.size()), size);
    if (w < 0) check(VX_EINVAL);
    return pop[static_cast<std::size_t>(w)];
}

// One rank's NCCL communicator (vx_comm_create): rank 0 calls unique_id()
// and distributes the 128 bytes (MPI, a file, a socket ...), every rank of
// the world then constructs its Communicator with them (collective).
class Communicator {
  public:
    using Id = std::vector<uint8_t>;
    static Id unique_id() {
        Id id(VX_COMM_ID_BYTES);
        check(vx_comm_unique_id(id.data()));
        return id;
    }
    Communicator(int world, int rank, const Id& id, Device& dev = default_device()) {
        if (id.size() != VX_COMM_ID_BYTES) throw std::invalid_argument("NCCL unique id must be 128 bytes");
        check(vx_comm_create(dev.get(), world, rank, id.data(), &c_));
    }
    ~Communicator() { vx_comm_destroy(c_); }
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    vx_comm* get() const { return c_; }

  private:
    vx_comm* c_ = nullptr;
};

// Device-resident EvolutionState: init_evolution + evolve_generation with
// the advisor consulted where evolution.hpp:221-227 consults it.
class GpuEvolution {
  public:
    explicit GpuEvolution(const EvolutionConfig& cfg, Device& dev = default_device()) : cfg_(cfg), dev_(dev) {
        cfg.validate();
        const vx_evo_config c = to_c(cfg);
        check(vx_evo_create(dev.get(), &c, &evo_));
    }
    // One rank of a run sharded over GPUs: every rank holds
    // the replicated state, evaluates its shard of the children, and the
    // communicator all-reduces the exchange buffer once per generation.
    // Identical results on every rank and for every world size.
    GpuEvolution(const EvolutionConfig& cfg, Communicator& comm, Device& dev = default_device())
        : GpuEvolution(cfg, dev) {
        check(vx_evo_set_comm(evo_, comm.get()));
    }
    // The same over any transport: allreduce(d_buf, n) must leave the
    // element-wise sum over the `world` ranks in the device buffer.
    using AllReduceFn = std::function<void(double* d_buf, int64_t n)>;
    GpuEvolution(const EvolutionConfig& cfg, int rank, int world, AllReduceFn allreduce,
                 Device& dev = default_device())
        : GpuEvolution(cfg, dev) {
        allreduce_ = std::move(allreduce);
        check(vx_evo_set_exchange(evo_, rank, world, &GpuEvolution::exchange_tramp, this));
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

    // The full reference state (grids of already-decoded individuals
    // included, so elites are not decoded again), e.g. for the free-function
    // evolve_generation below.
    void load_full_state(const EvolutionState& st) {
        std::vector<double> params, bmat, fit, gw;
        std::vector<uint8_t> ev, grids;
        const std::size_t cells = static_cast<std::size_t>(cfg_.grid_w) * cfg_.grid_h * cfg_.grid_d;
        bool any_grid = false;
        for (const auto& ind : st.population) any_grid = any_grid || ind.grid.cells.size() == cells;
        for (const auto& ind : st.population) {
            flatten(ind.genome, params);
            bmat.insert(bmat.end(), ind.genome.b_matrix.begin(), ind.genome.b_matrix.end());
            fit.push_back(ind.fitness);
            ev.push_back(ind.evaluated ? 1 : 0);
            if (!any_grid) continue;
            const bool has = ind.grid.cells.size() == cells;
            for (std::size_t c = 0; c < cells; ++c) {
                grids.push_back(has ? static_cast<uint8_t>(ind.grid.cells[c].material) : uint8_t(255));
                gw.push_back(has ? ind.grid.cells[c].weight : 0.0);
            }
        }
        check(vx_evo_set_population(evo_, params.data(), bmat.data(), fit.data(), ev.data(),
                                    any_grid ? grids.data() : nullptr, any_grid ? gw.data() : nullptr));
        const vx_hyper h = to_c(st.params);
        check(vx_evo_set_params(evo_, &h));
        set_rng_state(st.rng.state());
        history = st.history;
        std::vector<double> bp;
        if (st.best_genome) flatten(*st.best_genome, bp);
        check(vx_evo_set_progress(evo_, st.generation, st.best_fitness, st.best_genome ? bp.data() : nullptr,
                                  st.best_genome ? st.best_genome->b_matrix.data() : nullptr));
    }
    // to_state() plus the cached raw grids of the individuals that have one.
    EvolutionState to_full_state() const {
        EvolutionState st = to_state();
        const std::size_t P = st.population.size();
        const std::size_t cells = static_cast<std::size_t>(cfg_.grid_w) * cfg_.grid_h * cfg_.grid_d;
        std::vector<uint8_t> grids(P * cells);
        std::vector<double> gw(P * cells);
        check(vx_evo_get_population(evo_, nullptr, nullptr, nullptr, nullptr, grids.data(), gw.data()));
        for (std::size_t i = 0; i < P; ++i) {
            if (grids[i * cells] == 255) continue;  // not decoded
            VoxelGrid g(cfg_.grid_w, cfg_.grid_h, cfg_.grid_d);
            for (std::size_t c = 0; c < cells; ++c)
                g.cells[c] = Cell{static_cast<Material>(grids[i * cells + c]), gw[i * cells + c]};
            st.population[i].grid = std::move(g);
        }
        return st;
    }

  private:
    static vx_status exchange_tramp(double* d_buf, int64_t n, void* self) {
        try {
            static_cast<GpuEvolution*>(self)->allreduce_(d_buf, n);
            return VX_OK;
        } catch (...) {
            return VX_ECUDA;
        }
    }
    EvolutionConfig cfg_;
    Device& dev_;
    vx_evo* evo_ = nullptr;
    AllReduceFn allreduce_;
};

// init_evolution (evolution.hpp:197-211): per-genome seeds from the master
// stream, genomes sampled on device (B on the host libm) — the same
// EvolutionState the reference returns, bit for bit.
inline EvolutionState init_evolution(const EvolutionConfig& cfg, Device& dev = default_device()) {
    GpuEvolution g(cfg, dev);
    return g.to_state();
}

// evolve_generation (evolution.hpp:217-293) on a host-resident reference
// EvolutionState: the state goes to the device, one generation runs there
// (advisor consulted as the reference does), and the new state comes back.
// For many generations keep a GpuEvolution instead (no transfers).
inline GenerationReport evolve_generation(EvolutionState& st, const AdvisorFn& advisor = nullptr,
                                          Device& dev = default_device()) {
    GpuEvolution g(st.config, dev);
    g.load_full_state(st);
    const GenerationReport rep = g.evolve_generation(advisor);
    st = g.to_full_state();
    return rep;
}

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
