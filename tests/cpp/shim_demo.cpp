// shim_demo.cpp — the reference's own C++ API driving the B200 path.
//
// Built against the UNMODIFIED reference headers (/root/reference/proj/include)
// plus include/voxevo_b200/voxevo_shim.hpp, linked to libvoxevo_b200.so.
// Each check compares voxevo::X (reference, CPU) with voxevo::b200::X (GPU)
// on identical inputs and prints one PASS/FAIL line, like the reference's
// acceptance binary (acceptance_main.cpp:31-38).  Exit code = #failures.
#include <cuda_runtime.h>

#include <barrier>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>

#include "voxevo/advisor.hpp"
#include "voxevo/bench.hpp"
#include "voxevo/evolution.hpp"
#include "voxevo/serialize.hpp"
#include "voxevo_b200/voxevo_shim.hpp"

using namespace voxevo;

static int g_fail = 0;
static void report(const char* name, bool ok, const std::string& detail) {
    std::printf("%-52s %s  (%s)\n", name, ok ? "PASS" : "FAIL", detail.c_str());
    if (!ok) ++g_fail;
}

static bool same_genome(const Genome& a, const Genome& b) {
    if (a.b_matrix != b.b_matrix || !a.same_architecture(b)) return false;
    auto ta = const_cast<Genome&>(a).param_tensors();
    auto tb = const_cast<Genome&>(b).param_tensors();
    for (std::size_t t = 0; t < ta.size(); ++t)
        if (*ta[t] != *tb[t]) return false;
    return true;
}

int main() {
    // config 1: sample_genome(seed 42) -> decode 4^3
    const Genome g = sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 42);
    report("sample_genome bit-exact (B and every layer)", same_genome(g, b200::sample_genome(EncodingSpec{32, 3, 1.0},
                                                                                             {64, 64}, 42)),
           "seed 42, m 32, hidden {64,64}");
    {
        const Vec3 v{0.125, 0.375, 0.875};
        report("gaussian_encode bit-exact", gaussian_encode(v, g.b_matrix, 32) == b200::gaussian_encode(v, g.b_matrix, 32),
               "64 features");
    }
    const VoxelGrid ref_grid = decode(g, 4, 4, 4);
    const VoxelGrid gpu_grid = b200::decode(g, 4, 4, 4);
    int mat_diff = 0;
    double w_rel = 0.0;
    for (size_t i = 0; i < ref_grid.size(); ++i) {
        mat_diff += ref_grid.cells[i].material != gpu_grid.cells[i].material;
        w_rel = std::max(w_rel, std::abs(ref_grid.cells[i].weight - gpu_grid.cells[i].weight) / ref_grid.cells[i].weight);
    }
    report("decode: materials bit-exact, weights <= 1e-13", mat_diff == 0 && w_rel <= 1e-13,
           std::to_string(mat_diff) + " material diffs, max weight rel " + std::to_string(w_rel));

    const VoxelGrid body = largest_component(ref_grid);
    const VoxelGrid gbody = b200::largest_component(ref_grid);
    int body_diff = 0;
    for (size_t i = 0; i < body.size(); ++i) body_diff += body.cells[i].material != gbody.cells[i].material;
    report("largest_component bit-exact", body_diff == 0, std::to_string(body.count_non_empty()) + " voxels");

    const MassSpringSystem sys = build_mass_spring(body, MaterialTable{});
    const MassSpringSystem gsys = b200::build_mass_spring(body, MaterialTable{});
    bool same = sys.masses.size() == gsys.masses.size() && sys.springs.size() == gsys.springs.size();
    for (size_t a = 0; same && a < sys.masses.size(); ++a) same = sys.masses[a].pos == gsys.masses[a].pos;
    for (size_t q = 0; same && q < sys.springs.size(); ++q) {
        const Spring &x = sys.springs[q], &y = gsys.springs[q];
        same = x.i == y.i && x.j == y.j && x.k == y.k && x.rest0 == y.rest0 && x.act.has_value() == y.act.has_value();
        if (same && x.act) same = x.act->sign == y.act->sign && x.act->amplitude == y.act->amplitude &&
                                  x.act->phase == y.act->phase;
    }
    report("build_mass_spring bit-exact (topology, k, rest0, actuation)", same,
           std::to_string(sys.masses.size()) + " masses, " + std::to_string(sys.springs.size()) + " springs");

    SimConfig sim;
    sim.duration = 1000 * sim.dt;
    const TrajectorySummary rs = simulate(sys, sim);
    const TrajectorySummary gs = b200::simulate(sys, sim);
    report("simulate 1000 steps bit-exact (COM, displacement, max speed)",
           rs.horizontal_displacement == gs.horizontal_displacement && rs.com_end == gs.com_end &&
               rs.com_start == gs.com_start && rs.max_speed == gs.max_speed && rs.diverged == gs.diverged,
           "displacement " + std::to_string(rs.horizontal_displacement));

    // simulate with the COM dump (physics.hpp:285-311): every row bit-exact
    std::vector<TrajectorySample> rd, gd;
    simulate(sys, sim, &rd, 300);
    b200::simulate(sys, sim, &gd, 300);
    bool dump_ok = rd.size() == gd.size();
    for (size_t q = 0; dump_ok && q < rd.size(); ++q) dump_ok = rd[q].t == gd[q].t && rd[q].com == gd[q].com;
    report("simulate with dump every 300 steps: rows bit-exact", dump_ok, std::to_string(rd.size()) + " rows");

    // step (physics.hpp:191): 40 single steps at t = k dt, state and counters bit-exact
    {
        MassSpringSystem a = sys, b = sys;
        SimWorkspace wa(a), wb(b);
        bool ok = true;
        for (int k = 0; k < 40 && ok; ++k) {
            const double t = static_cast<double>(k) * sim.dt;
            ok = step(a, t, sim, wa) == b200::step(b, t, sim, wb);
        }
        for (size_t i = 0; ok && i < a.masses.size(); ++i) ok = a.masses[i].pos == b.masses[i].pos && a.masses[i].vel == b.masses[i].vel;
        ok = ok && wa.spring_updates == wb.spring_updates && wa.max_speed_sq == wb.max_speed_sq;
        report("step x40 bit-exact (positions, velocities, counters)", ok,
               std::to_string(wa.spring_updates) + " spring updates");
    }

    // evaluate_fitness (evolution.hpp:110) on raw grids: bit-exact
    {
        std::vector<VoxelGrid> raws;
        for (uint64_t seed : {42u, 7u, 11u, 2024u})
            raws.push_back(decode(sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, seed), 5, 5, 5));
        const std::vector<double> gf = b200::evaluate_fitness(raws, MaterialTable{}, GroundPlane{}, sim);
        bool ok = true;
        for (size_t a = 0; a < raws.size(); ++a)
            ok = ok && gf[a] == evaluate_fitness(raws[a], MaterialTable{}, GroundPlane{}, sim);
        report("evaluate_fitness bit-exact (4 decoded 5^3 robots)", ok, "fitness[0] " + std::to_string(gf[0]));
    }

    // forward (genome.hpp:187-211) at off-grid points: probabilities and weight within 1e-12
    {
        const Genome fg = sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 77);
        const std::vector<Vec3> pts = {{0.1, 0.2, 0.3}, {0.9, 0.05, 0.5}, {-2.0, 3.5, 0.25}};
        const std::vector<MaterialQuery> gq = b200::forward(fg, pts);
        bool fok = true;
        for (size_t q = 0; q < pts.size(); ++q) {
            const MaterialQuery rq = forward(fg, pts[q]);
            for (int i = 0; i < 5; ++i) fok = fok && std::abs(rq.probs[i] - gq[q].probs[i]) <= 1e-12 * rq.probs[i] + 1e-300;
            fok = fok && std::abs(rq.weight - gq[q].weight) <= 1e-12 * rq.weight;
        }
        report("forward at off-grid points: probs / weight <= 1e-12", fok, std::to_string(pts.size()) + " points");
    }


    // the GA operators on the caller's Rng (evolution.hpp:143-173)
    {
        const Genome a = sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 5);
        const Genome b = sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 6);
        Rng r1(99), r2(99);
        Genome c1 = crossover(a, b, r1), c2 = b200::crossover(a, b, r2);
        mutate(c1, 0.1, 0.1, r1);
        b200::mutate(c2, 0.1, 0.1, r2);
        std::vector<Individual> pop(37);
        const Individual* w1 = &tournament_select(pop, 3, r1);
        const Individual* w2 = &b200::tournament_select(pop, 3, r2);
        report("crossover / mutate / tournament_select bit-exact on the caller's Rng",
               same_genome(c1, c2) && w1 == w2 && r1 == r2, "winner " + std::to_string(w1 - pop.data()));
    }
    {
        std::vector<Individual> pop(6);
        for (int i = 0; i < 6; ++i)
            pop[i].grid = decode(sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 100 + i), 6, 6, 6);
        const double rd = population_diversity(pop), gd = b200::population_diversity(pop);
        report("population_diversity bit-exact", rd == gd, std::to_string(rd));
    }
    {
        bool threw = false;
        try {
            Genome deep = sample_genome(EncodingSpec{4, 3, 1.0}, {2, 2, 2, 2, 2, 2, 2, 2, 2}, 1);
            b200::decode(deep, 2, 2, 2);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        report("more than VX_MAX_HIDDEN layers -> std::invalid_argument", threw, "9 hidden layers");
    }

    // desk GA (acceptance_main.cpp:193-211 shape): reference genomes on the
    // GPU; draw consumption is fitness-independent -> identical RNG streams
    EvolutionConfig cfg;
    cfg.population = 12;
    cfg.generations = 4;
    cfg.grid_w = cfg.grid_h = cfg.grid_d = 3;
    cfg.seed = 1;
    cfg.sim.dt = 1e-4;
    cfg.sim.duration = 0.5;
    EvolutionState st = init_evolution(cfg);
    b200::GpuEvolution gpu(cfg);
    gpu.set_population(st.population);
    gpu.set_rng_state(st.rng.state());
    double prev = -1.0;
    bool mono = true;
    GenerationReport r0{}, g0{};
    for (int gen = 0; gen <= cfg.generations; ++gen) {
        const GenerationReport r = evolve_generation(st);
        const GenerationReport q = gpu.evolve_generation();
        if (gen == 0) {
            r0 = r;
            g0 = q;
        }
        mono = mono && q.best >= prev;
        prev = q.best;
    }
    report("evolve_generation: gen-0 best within the 1e-2 desk floor",
           std::abs(r0.best - g0.best) <= 1e-2 * r0.best && r0.evaluations == g0.evaluations,
           "ref " + std::to_string(r0.best) + " gpu " + std::to_string(g0.best));
    report("evolve_generation: best non-decreasing, RNG stream identical", mono && gpu.rng_state() == st.rng.state(),
           std::to_string(cfg.generations + 1) + " generations");

    // checkpoints: the GPU state through the reference's own save_run /
    // load_run (serialize.hpp) resumes identically, and a CPU checkpoint
    // resumes on the GPU with the same GA stream (draws are fitness-independent)
    {
        EvolutionConfig c2 = cfg;
        c2.seed = 9;
        b200::GpuEvolution a(c2);
        EvolutionState s0 = init_evolution(c2);
        a.set_population(s0.population);
        a.set_rng_state(s0.rng.state());
        for (int k = 0; k < 2; ++k) a.evolve_generation();
        const std::string path = "/tmp/voxevo_b200_shim_ckpt.json";
        save_run(path, a.to_state());
        b200::GpuEvolution b(c2);
        b.load_state(load_run(path));
        bool same = true;
        for (int k = 0; k < 2; ++k) {
            const GenerationReport x = a.evolve_generation(), y = b.evolve_generation();
            same = same && x.best == y.best && x.mean == y.mean && x.diversity == y.diversity &&
                   x.generation == y.generation;
        }
        report("checkpoint: GPU state -> save_run -> load_run resumes identically",
               same && a.rng_state() == b.rng_state() && a.best_fitness() == b.best_fitness(),
               "generations 2..3 after the reload");
        EvolutionState cpu = init_evolution(c2);
        for (int k = 0; k < 2; ++k) evolve_generation(cpu);
        save_run(path, cpu);
        b200::GpuEvolution c(c2);
        c.load_state(load_run(path));
        const GenerationReport gq = c.evolve_generation();
        const GenerationReport cq = evolve_generation(cpu);
        report("checkpoint: CPU state resumes on the GPU, same GA stream",
               gq.generation == cq.generation && gq.evaluations == cq.evaluations && c.rng_state() == cpu.rng.state(),
               "generation " + std::to_string(gq.generation));
        std::remove(path.c_str());
    }

    // init_evolution bit-exact; free-function evolve_generation on a host state
    // (the reference's default step, dt 1e-5 x 5000: fitness within rtol 1e-3;
    // the GA stream's consumption is fitness-independent without an advisor)
    {
        EvolutionConfig c3 = cfg;
        c3.seed = 21;
        c3.sim = SimConfig{};
        EvolutionState r = init_evolution(c3);
        EvolutionState q = b200::init_evolution(c3);
        bool same = r.rng == q.rng && r.population.size() == q.population.size();
        for (size_t i = 0; same && i < r.population.size(); ++i) same = same_genome(r.population[i].genome, q.population[i].genome);
        report("init_evolution bit-exact (every genome, GA stream)", same, std::to_string(r.population.size()) + " genomes");
        bool ok = true;
        double rel0 = 0.0;
        for (int k = 0; k < 3; ++k) {
            const GenerationReport x = evolve_generation(r), y = b200::evolve_generation(q);
            ok = ok && x.evaluations == y.evaluations && x.generation == y.generation;
            if (k == 0) rel0 = std::abs(x.best - y.best) / x.best;
        }
        report("evolve_generation(EvolutionState&) free function: same GA stream",
               ok && rel0 <= 1e-3 && r.rng == q.rng && r.generation == q.generation && r.history.size() == q.history.size(),
               "3 generations, gen-0 best rel " + std::to_string(rel0));
    }

    // advisor in the loop (evolution.hpp:221-227): the reference's own
    // ScriptedAdvisor on both sides, 10 generations.  Lock-step with teacher
    // forcing at the exchange point (world 1): the device evaluates every
    // pending robot (checked within 5e-2, the dt = 1e-4 chaos floor), then the
    // reference's fitness replaces it, so one chaotic near-tie cannot send the
    // runs apart; fired rules change the RNG consumption, so identical params
    // histories, reports, populations and GA streams prove identical decisions.
    {
        EvolutionConfig c4 = cfg;
        c4.seed = 4;
        c4.population = 16;
        c4.grid_w = c4.grid_h = c4.grid_d = 4;
        c4.sim.duration = 0.1;
        ScriptedAdvisor adv_r, adv_g;
        const AdvisorFn fr = make_advisor_fn(&adv_r), fg = make_advisor_fn(&adv_g);
        EvolutionState r = init_evolution(c4);
        std::vector<double> forced;
        double worst = 0.0;
        b200::GpuEvolution gpu4(c4, 0, 1, [&](double* d_buf, int64_t n) {
            std::vector<double> h(static_cast<size_t>(n));
            cudaMemcpy(h.data(), d_buf, n * sizeof(double), cudaMemcpyDeviceToHost);
            for (size_t i = 0; i < forced.size(); ++i)
                if (!std::isnan(forced[i])) {
                    worst = std::max(worst, std::abs(h[i] - forced[i]) / std::max(std::abs(forced[i]), 1e-12));
                    h[i] = forced[i];
                }
            cudaMemcpy(d_buf, h.data(), n * sizeof(double), cudaMemcpyHostToDevice);
        });
        gpu4.set_population(r.population);
        gpu4.set_rng_state(r.rng.state());
        bool ok = true;
        int fired = 0;
        for (int k = 0; k < 10; ++k) {
            const MaterialTable table = detail::scaled_materials(c4.materials, r.params);
            forced.assign(r.population.size(), std::nan(""));
            for (size_t i = 0; i < r.population.size(); ++i)
                if (!r.population[i].evaluated)
                    forced[i] = evaluate_fitness(decode(r.population[i].genome, c4.grid_w, c4.grid_h, c4.grid_d), table,
                                                 c4.plane, c4.sim);
            const GenerationReport y = gpu4.evolve_generation(fg), x = evolve_generation(r, fr);
            ok = ok && x.params == y.params && x.best == y.best && x.mean == y.mean && x.stddev == y.stddev &&
                 x.evaluations == y.evaluations && x.diversity == y.diversity;
            fired += !(x.params == c4.initial_params);
        }
        const EvolutionState q = gpu4.to_state();
        bool pop_same = q.population.size() == r.population.size();
        for (size_t i = 0; pop_same && i < r.population.size(); ++i)
            pop_same = same_genome(q.population[i].genome, r.population[i].genome) &&
                       q.population[i].fitness == r.population[i].fitness &&
                       q.population[i].evaluated == r.population[i].evaluated;
        report("ScriptedAdvisor in the loop: params history + GA stream identical",
               ok && pop_same && fired >= 1 && worst <= 5e-2 && gpu4.rng_state() == r.rng.state(),
               std::to_string(fired) + " of 10 generations with adjusted params, fitness before forcing rel " +
                   std::to_string(worst));
    }

    // sharded GpuEvolution(cfg, rank, world, allreduce): two ranks in two
    // threads (each its own context), host all-reduce between them; reports
    // and GA streams bit-identical to the single-rank run
    {
        EvolutionConfig c5 = cfg;
        c5.seed = 5;
        c5.population = 24;
        b200::GpuEvolution solo(c5);
        std::vector<GenerationReport> want;
        for (int k = 0; k < 3; ++k) want.push_back(solo.evolve_generation());
        std::barrier sync(2);
        std::vector<double> h0, h1, sum;
        std::vector<GenerationReport> got[2];
        std::string rng_state[2];
        auto rank_main = [&](int rank) {
            b200::Device dev(0);
            std::vector<double>& mine = rank == 0 ? h0 : h1;
            b200::GpuEvolution g(c5, rank, 2, [&](double* d_buf, int64_t n) {
                mine.resize(static_cast<size_t>(n));
                cudaMemcpy(mine.data(), d_buf, n * sizeof(double), cudaMemcpyDeviceToHost);
                sync.arrive_and_wait();
                if (rank == 0) {
                    sum.resize(static_cast<size_t>(n));
                    for (int64_t i = 0; i < n; ++i) sum[i] = h0[i] + h1[i];
                }
                sync.arrive_and_wait();
                cudaMemcpy(d_buf, sum.data(), n * sizeof(double), cudaMemcpyHostToDevice);
            }, dev);
            for (int k = 0; k < 3; ++k) got[rank].push_back(g.evolve_generation());
            rng_state[rank] = g.rng_state();
        };
        std::thread t0(rank_main, 0), t1(rank_main, 1);
        t0.join();
        t1.join();
        bool ok = rng_state[0] == solo.rng_state() && rng_state[1] == solo.rng_state();
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 3; ++k)
                ok = ok && got[r][k].best == want[k].best && got[r][k].mean == want[k].mean &&
                     got[r][k].stddev == want[k].stddev && got[r][k].diversity == want[k].diversity &&
                     got[r][k].evaluations == want[k].evaluations;
        report("GpuEvolution(cfg, rank, world): 2 ranks == 1 rank, bit for bit", ok, "3 generations, P=24");
    }

    BenchConfig bc;
    const BenchResult br = b200::run_bench(bc);
    report("run_bench: exact work audit 33,152,000", br.spring_updates == 33152000u && !br.diverged,
           std::to_string(br.updates_per_second) + " updates/s on device");
    return g_fail;
}
