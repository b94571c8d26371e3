// shim_demo.cpp — the reference's own C++ API driving the B200 path.
//
// Built against the UNMODIFIED reference headers (/root/reference/proj/include)
// plus include/voxevo_b200/voxevo_shim.hpp, linked to libvoxevo_b200.so.
// Each check compares voxevo::X (reference, CPU) with voxevo::b200::X (GPU)
// on identical inputs and prints one PASS/FAIL line, like the reference's
// acceptance binary (acceptance_main.cpp:31-38).  Exit code = #failures.
#include <cmath>
#include <cstdio>
#include <string>

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

int main() {
    // config 1: sample_genome(seed 42) -> decode 4^3
    const Genome g = sample_genome(EncodingSpec{32, 3, 1.0}, {64, 64}, 42);
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
    const double rel = std::abs(rs.horizontal_displacement - gs.horizontal_displacement) / rs.horizontal_displacement;
    report("simulate 1000 steps: displacement rel <= 1e-3", rel <= 1e-3 && rs.diverged == gs.diverged,
           "ref " + std::to_string(rs.horizontal_displacement) + " rel " + std::to_string(rel));

    // simulate with the COM dump (physics.hpp:285-311): same sample times, COMs within the chaos floor
    std::vector<TrajectorySample> rd, gd;
    simulate(sys, sim, &rd, 300);
    b200::simulate(sys, sim, &gd, 300);
    bool dump_ok = rd.size() == gd.size();
    for (size_t q = 0; dump_ok && q < rd.size(); ++q) {
        dump_ok = rd[q].t == gd[q].t;
        for (int c = 0; c < 3; ++c)
            dump_ok = dump_ok && std::abs(rd[q].com[c] - gd[q].com[c]) <= 1e-9 + 1e-6 * std::abs(rd[q].com[c]);
    }
    report("simulate with dump every 300 steps: rows and times match", dump_ok,
           std::to_string(rd.size()) + " rows");

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

    BenchConfig bc;
    const BenchResult br = b200::run_bench(bc);
    report("run_bench: exact work audit 33,152,000", br.spring_updates == 33152000u && !br.diverged,
           std::to_string(br.updates_per_second) + " updates/s on device");
    return g_fail;
}
