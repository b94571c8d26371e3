"""simulate() with the trajectory dump (physics.hpp:280-311): COM samples
every `stride` steps while the robot is live, plus the final row, on every
specialised integrator — bit-identical rows and summaries against the
reference's own simulate(sys, cfg, &dump, stride) (test_physics.cpp:233-255
drives the same call), including robots that diverge mid-run and strides
that do not divide the horizon."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

KERNEL = {4: "lattice", 6: "lattice", 10: "cluster", 20: "stream"}


def _systems(vx, ctx, orc, n, count, seed):
    rng = np.random.default_rng(seed)
    gs = [orc.sample_genome(32, [64, 64], int(s)) for s in rng.integers(0, 2 ** 62, count)]
    mats, wts = vx.decode(np.stack([g[0] for g in gs]), np.stack([g[1] for g in gs]), vx.Arch.make(), n, n, n, ctx)
    return [orc.bench_robot(n)] + [(orc.largest_component(mats[a], n, n, n), wts[a]) for a in range(count)]


def _check(vx, ctx, orc, n, items, sim, stride, mutate=None):
    batch = vx.build_mass_spring(np.stack([m for m, _ in items]), np.stack([w for _, w in items]), n, n, n, ctx=ctx)
    systems = [orc.build(m, w, n, n, n) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    if mutate is not None:
        pos = np.concatenate([s.pos for s in systems])
        vel = np.concatenate([s.vel for s in systems])
        mutate(systems, pos, vel)
        batch.set_state(pos, vel)
    before = batch.download()
    summ, dumps = batch.simulate_dump(sim, stride)
    assert ctx.last_integrator == KERNEL[n]
    after = batch.download()
    np.testing.assert_array_equal(after.pos, before.pos)  # by value: the batch is untouched
    np.testing.assert_array_equal(after.vel, before.vel)
    for r, s in enumerate(systems):
        ref = orc.simulate(s, sim.as_array(), stride=stride)
        np.testing.assert_array_equal(dumps[r], ref["dump"], err_msg=f"grid {n} robot {r} stride {stride}")
        assert list(summ[r].com_start) == list(ref["com_start"])
        assert list(summ[r].com_end) == list(ref["com_end"])
        assert summ[r].horizontal_displacement == ref["horizontal_displacement"]
        assert summ[r].max_speed == ref["max_speed"]
        assert bool(summ[r].diverged) == ref["diverged"]
    return summ, dumps


@pytest.mark.parametrize("n,steps,stride", [(6, 3000, 1000), (6, 1000, 7), (4, 200, 1), (10, 600, 250),
                                            (20, 120, 50), (6, 500, 0), (6, 0, 10)])
def test_simulate_dump_bit_exact(vx, ctx, orc, n, steps, stride):
    items = _systems(vx, ctx, orc, n, 3, 100 + n)
    summ, dumps = _check(vx, ctx, orc, n, items, vx.SimConfig(duration=steps * 1e-5), stride)
    expect = (-(-steps // stride) if stride > 0 else 0) + 1
    assert all(len(d) == expect for d in dumps)


def test_simulate_dump_divergence(vx, ctx, orc):
    """Robot 1 is flung out of the +-1e6 box during chunk 2: its samples stop
    at the diverging step's chunk start, the final row still carries
    t = n_steps*dt (physics.hpp:297-303)."""
    n = 6
    items = _systems(vx, ctx, orc, n, 2, 7)

    def mutate(systems, pos, vel):
        nm0 = len(systems[0].pos)
        vel[nm0 + 2, 0] = 3.5e8  # ~2.9 ms to leave the box: diverges in the third 100-step chunk
        systems[1].vel[:] = vel[nm0:nm0 + len(systems[1].vel)]

    summ, dumps = _check(vx, ctx, orc, n, items, vx.SimConfig(duration=600 * 1e-5), 100, mutate)
    assert summ[1].diverged and not summ[0].diverged
    assert len(dumps[1]) < len(dumps[0])


def test_simulate_dump_uploaded_systems(vx, ctx, orc):
    """Host-assembled systems run the generic integrator; the dump follows the
    same rows, bit for bit (phases overridden with glibc's, as the reference
    computes them)."""
    n = 4
    items = _systems(vx, ctx, orc, n, 2, 3)
    systems = [orc.build(m, w, n, n, n) for m, w in items] + [oracle.dumbbell(0.2, 100.0, 0.1, 0.15)]
    batch = vx.upload_systems(systems, ctx=ctx)
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    sim = vx.SimConfig(duration=700 * 1e-5)
    summ, dumps = batch.simulate_dump(sim, 64)
    assert ctx.last_integrator == "generic"
    for r, s in enumerate(systems):
        ref = orc.simulate(s, sim.as_array(), stride=64)
        np.testing.assert_array_equal(dumps[r], ref["dump"])
        assert summ[r].horizontal_displacement == ref["horizontal_displacement"]
        assert summ[r].max_speed == ref["max_speed"]
