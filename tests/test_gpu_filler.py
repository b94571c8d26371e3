"""The 10^3 cluster integrator with its one-SM filler (csrc/integrator_cluster.cu
persistent `cluster_vertex_kernel<10>` + csrc/integrator_stream.cu
`stream_sym_filler<10>`): clusters and filler CTAs claim robots from one
counter, so which kernel integrates a robot depends on timing.  Either way a
robot's trajectory must be bit-identical to the reference's step() /
simulate() (physics.hpp:191-311), and a whole evaluation must not depend on
whether the filler ran."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N = 10


def _items(vx, ctx, orc, count, seed):
    rng = np.random.default_rng(seed)
    gs = [orc.sample_genome(32, [64, 64], int(s)) for s in rng.integers(0, 2 ** 62, count)]
    mats, wts = vx.decode(np.stack([g[0] for g in gs]), np.stack([g[1] for g in gs]), vx.Arch.make(), N, N, N, ctx)
    items = [(orc.largest_component(mats[a], N, N, N), wts[a]) for a in range(count)]
    items[0] = orc.bench_robot(N)
    return items


@pytest.fixture
def forced(ctx):
    ctx.set_filler(2)  # filler at any batch size
    yield ctx
    ctx.set_filler(-1)


def test_filler_step_bit_exact(vx, forced, orc):
    ctx = forced
    items = _items(vx, ctx, orc, 24, 7)
    batch = vx.build_mass_spring(np.stack([m for m, _ in items]), np.stack([w for _, w in items]), N, N, N, ctx=ctx)
    systems = [orc.build(m, w, N, N, N) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    steps = 200
    out = batch.step(vx.SimConfig(), 0, steps)
    assert ctx.last_integrator == "cluster" and ctx.last_filler_ctas > 0
    got = batch.download()
    for r, s in enumerate(systems):
        ref, ok, called, upd, msq = orc.step(s, vx.SimConfig().as_array(), 0, steps)
        np.testing.assert_array_equal(got.robot(r)["pos"], ref.pos, err_msg=f"robot {r}")
        np.testing.assert_array_equal(got.robot(r)["vel"], ref.vel, err_msg=f"robot {r}")
        assert out[r].spring_updates == upd and out[r].max_speed == np.sqrt(msq)


def test_filler_simulate_summary_bit_exact(vx, forced, orc):
    ctx = forced
    items = _items(vx, ctx, orc, 12, 11)
    batch = vx.build_mass_spring(np.stack([m for m, _ in items]), np.stack([w for _, w in items]), N, N, N, ctx=ctx)
    systems = [orc.build(m, w, N, N, N) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    sim = vx.SimConfig(duration=150 * 1e-5)
    out = batch.simulate(sim)
    assert ctx.last_filler_ctas > 0
    for r, s in enumerate(systems):
        ref = orc.simulate(s, sim.as_array())
        assert list(out[r].com_start) == list(ref["com_start"]), r
        assert list(out[r].com_end) == list(ref["com_end"]), r
        assert out[r].horizontal_displacement == ref["horizontal_displacement"]
        assert out[r].max_speed == ref["max_speed"]
        assert out[r].spring_updates == 150 * s.ns


def test_filler_on_off_identical_large_batch(vx, ctx, orc):
    """At a batch large enough for the default (mode 1) filler, the evaluation
    with and without it is bit-identical (fitness and exact update counts)."""
    P = 320
    rng = np.random.default_rng(5)
    gs = [orc.sample_genome(32, [64, 64], int(s)) for s in rng.integers(0, 2 ** 62, 16)]
    mats, wts = vx.decode(np.stack([g[0] for g in gs]), np.stack([g[1] for g in gs]), vx.Arch.make(), N, N, N, ctx)
    idx = np.arange(P) % len(gs)
    mats, wts = mats[idx], wts[idx]
    sim = vx.SimConfig(duration=100 * 1e-5)
    res = {}
    try:
        for mode in (0, 1):
            ctx.set_filler(mode)
            res[mode] = vx.evaluate_fitness(mats, wts, N, N, N, sim=sim, ctx=ctx)
            assert (ctx.last_filler_ctas > 0) == (mode == 1)
    finally:
        ctx.set_filler(-1)
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b))
