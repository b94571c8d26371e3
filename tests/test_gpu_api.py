"""API-level GPU tests mirroring the reference's own unit tests
(test_evolution.cpp, test_physics.cpp, test_morphology.cpp) through the
Python mirror of voxevo:: (paper_2405_00698_b200)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def desk(vx, seed, P=6, gens=4, **kw):
    # test_evolution.cpp:14-26 desk_config
    return vx.EvolutionConfig(population=P, generations=gens, grid=(3, 3, 3), hidden_widths=[12, 12], m=8,
                              seed=seed, sim=vx.SimConfig(dt=1e-4, duration=0.05), **kw)


def test_config_validation(vx, ctx):
    # test_evolution.cpp:260-271
    with pytest.raises(ValueError):
        vx.init_evolution(vx.EvolutionConfig(population=1), ctx)
    with pytest.raises(ValueError):
        vx.init_evolution(vx.EvolutionConfig(tournament_size=0), ctx)
    with pytest.raises(ValueError):
        vx.init_evolution(vx.EvolutionConfig(grid=(0, 3, 3)), ctx)
    with pytest.raises(ValueError):
        vx.init_evolution(vx.EvolutionConfig(sim=vx.SimConfig(dt=0.0)), ctx)


def test_advisor_window_and_clamp(vx, ctx):
    # test_evolution.cpp:223-242: consulted at calls 3, 4, 5 with the trailing
    # window of 3 reports; out-of-range answers are clamped
    st = vx.init_evolution(desk(vx, 55), ctx)
    sizes, tails = [], []

    def advisor(window, cur):
        sizes.append(len(window))
        tails.append(window[-1].generation)
        nxt = cur.copy()
        nxt.mutation_rate = 5.0
        return nxt

    for _ in range(6):
        st.evolve_generation(advisor)
    assert sizes == [3, 3, 3] and tails == [2, 3, 4]
    assert st.params.mutation_rate == 1.0
    assert st.history[2].params.mutation_rate == 0.1
    assert st.history[3].params.mutation_rate == 1.0


def test_material_multipliers(vx, ctx):
    # test_evolution.cpp:244-258
    cfg = desk(vx, 8, P=6, gens=2)
    cfg.initial_params = vx.HyperParams(material_multipliers=(2.0, 0.5, 1.0))
    st = vx.init_evolution(cfg, ctx)
    for _ in range(3):
        assert np.isfinite(st.evolve_generation().best)


def test_monotone_best_and_counts(vx, ctx):
    # test_evolution.cpp:170-194
    st = vx.init_evolution(desk(vx, 21), ctx)
    prev = -1.0
    for g in range(5):
        r = st.evolve_generation()
        assert r.generation == g and r.best >= prev and 0.0 <= r.diversity <= 1.0
        assert r.mean <= r.best + 1e-15
        assert r.evaluations == (6 if g == 0 else 6 - vx.elite_count(0.3, 6))
        prev = r.best
    bf, bp = st.best()
    assert bf == st.history[-1].best and bp is not None


def test_seeded_runs_identical(vx, ctx):
    # test_evolution.cpp:196-215 (the GPU analogue of thread-count invariance)
    a = vx.init_evolution(desk(vx, 33), ctx)
    b = vx.init_evolution(desk(vx, 33), ctx)
    for _ in range(4):
        ra, rb = a.evolve_generation(), b.evolve_generation()
        assert (ra.best, ra.mean, ra.stddev, ra.diversity) == (rb.best, rb.mean, rb.stddev, rb.diversity)
    assert a.rng_state() == b.rng_state()
    np.testing.assert_array_equal(a.population()["params"], b.population()["params"])


def test_rng_state_text_interop(vx, ctx, orc):
    # checkpoint interop: the GA stream's text state is libstdc++'s mt19937_64 form
    st = vx.init_evolution(desk(vx, 7), ctx)
    s = orc.rng_state(12345, 999)
    st.set_rng_state(s)
    assert st.rng_state() == s
    with pytest.raises(ValueError):
        st.set_rng_state("not a state")


def test_simulate_zero_duration_and_summary(vx, ctx, orc):
    m, w = orc.bench_robot(2)
    batch = vx.build_mass_spring(m[None], w[None], 2, 2, 2, ctx=ctx)
    out = batch.simulate(vx.SimConfig(duration=0.0))[0]
    assert out.steps == 0 and out.spring_updates == 0 and out.horizontal_displacement == 0.0
    with pytest.raises(ValueError):
        batch.simulate(vx.SimConfig(actuation_frequency=0.0))


@pytest.mark.parametrize("grid", [1, 2, 3, 5, 6])
def test_run_bench_counts_grids(vx, ctx, orc, grid):
    r = vx.run_bench(jobs=8, steps=300, grid=grid, ctx=ctx)
    s = orc.build(*orc.bench_robot(grid), grid, grid, grid)
    assert r["springs_per_robot"] == s.ns
    assert r["spring_updates"] == r["expected_updates"] == 8 * 300 * s.ns


def test_empty_and_passive_robots_in_population(vx, ctx):
    # gates inside a generation: robots with no voxels / no muscle score 0 and
    # are not simulated (evolution.hpp:113-114)
    cfg = desk(vx, 3, P=4, gens=1)
    st = vx.init_evolution(cfg, ctx)
    pop = st.population()
    arch = cfg.arch
    zero = np.zeros_like(pop["params"])
    st.set_population(zero, pop["bmat"])  # all-zero MLP -> five-way tie -> Empty everywhere
    r = st.evolve_generation()
    assert r.best == 0.0 and r.mean == 0.0 and r.spring_updates == 0


def test_population_beyond_grid_y_limit(vx, ctx):
    # config 4 runs P = 65536: every per-individual launch must take P > 65535
    cfg = vx.EvolutionConfig(population=70000, generations=1, grid=(2, 2, 2), hidden_widths=[4], m=4, seed=3,
                             sim=vx.SimConfig(dt=1e-4, duration=1e-3))
    st = vx.init_evolution(cfg, ctx)
    r0 = st.evolve_generation()
    r1 = st.evolve_generation()
    assert r0.evaluations == 70000 and r1.evaluations == 70000 - vx.elite_count(0.3, 70000)
    assert r1.best >= r0.best


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_generation_matches_single_process(vx, ctx, world):
    """vx_evo_begin(rank, world) on `world` replicas (one GPU, ranks run one
    after another), a summed exchange buffer standing in for the NCCL
    all-reduce, then finish() everywhere: reports, populations and RNG streams
    equal the single-process run bit for bit — decode and evaluation sharded,
    diversity from the gathered (summed) packed grids."""
    import torch
    cfg = desk(vx, 77, P=12, gens=4)
    single = vx.init_evolution(cfg, ctx)
    ranks = [vx.init_evolution(cfg, ctx) for _ in range(world)]
    n = ranks[0].exchange_buffer()[1]
    assert n == 2 * 12 + 12 * ((27 + 11) // 12)  # fitness | updates | packed grids (12 cells / double)
    bufs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(world)]
    for st, b in zip(ranks, bufs):
        st.set_exchange_buffer(b.data_ptr())
    key = lambda r: (r.generation, r.best, r.mean, r.stddev, r.diversity, r.evaluations, int(r.spring_updates))
    for _ in range(4):
        ref = single.evolve_generation()
        for r, st in enumerate(ranks):
            st.begin(r, world)
        ctx.synchronize()
        torch.cuda.synchronize()
        total = torch.stack(bufs).sum(0)
        for b in bufs:
            b.copy_(total)
        torch.cuda.synchronize()
        for st in ranks:
            assert key(st.finish()) == key(ref)
    for st in ranks:
        assert st.rng_state() == single.rng_state()
        np.testing.assert_array_equal(st.population()["params"], single.population()["params"])
