"""K7c, the thread-block-cluster integrator (csrc/integrator_cluster.cu): one
cluster of 2-4 CTAs per robot for 7^3..10^3 grids, state halos and
boundary force slots exchanged through distributed shared memory.  Same bar as
the one-SM lattice kernel: bit-exact trajectories against the reference's own
step() / simulate() (physics.hpp:191-311) on identical systems, including the
zero-length and divergence exits and robots far smaller than the grid."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _decoded(vx, ctx, orc, n, count, seed):
    rng = np.random.default_rng(seed)
    gs = [orc.sample_genome(32, [64, 64], int(s)) for s in rng.integers(0, 2 ** 62, count)]
    mats, wts = vx.decode(np.stack([g[0] for g in gs]), np.stack([g[1] for g in gs]), vx.Arch.make(), n, n, n, ctx)
    return [(orc.largest_component(mats[a], n, n, n), wts[a]) for a in range(count)]


def _column(n):
    # a one-voxel-wide muscle tower: few masses spread over every z-plane
    m = np.zeros(n ** 3, np.uint8)
    w = np.ones(n ** 3)
    for z in range(n):
        m[z * n * n] = 1 + (z % 2)
    return m, w


def _slab(n):
    # one full z-plane of voxels: a wide, flat robot
    m = np.zeros(n ** 3, np.uint8)
    w = np.full(n ** 3, 0.7)
    m[: n * n] = np.array([1, 2, 3, 4] * (n * n))[: n * n]
    return m, w


def _run(vx, ctx, orc, n, items, steps, chunks=1):
    mats = np.stack([m for m, _ in items])
    wts = np.stack([w for _, w in items])
    batch = vx.build_mass_spring(mats, wts, n, n, n, ctx=ctx)
    systems = [orc.build(m, w, n, n, n) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    sim = vx.SimConfig()
    per = steps // chunks
    outs = [batch.step(sim, c * per, per) for c in range(chunks)]
    assert ctx.last_integrator == "cluster"
    got = batch.download()
    for r, s in enumerate(systems):
        ref, ok, called, upd, msq = orc.step(s, sim.as_array(), 0, per * chunks)
        rr = got.robot(r)
        np.testing.assert_array_equal(rr["pos"], ref.pos, err_msg=f"grid {n} robot {r}")
        np.testing.assert_array_equal(rr["vel"], ref.vel, err_msg=f"grid {n} robot {r}")
        assert sum(o[r].spring_updates for o in outs) == upd
    return batch, systems


@pytest.mark.parametrize("n", [7, 8, 10])
def test_cluster_integrator_bit_exact(vx, ctx, orc, n):
    items = [orc.bench_robot(n)] + _decoded(vx, ctx, orc, n, 2, n) + [_column(n), _slab(n)]
    _run(vx, ctx, orc, n, items, 300, chunks=2)


def test_cluster_simulate_summary_bit_exact(vx, ctx, orc):
    n = 10
    items = [orc.bench_robot(n)] + _decoded(vx, ctx, orc, n, 2, 99) + [_column(n)]
    mats = np.stack([m for m, _ in items])
    wts = np.stack([w for _, w in items])
    batch = vx.build_mass_spring(mats, wts, n, n, n, ctx=ctx)
    systems = [orc.build(m, w, n, n, n) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    sim = vx.SimConfig(duration=250 * 1e-5)
    out = batch.simulate(sim)
    assert ctx.last_integrator == "cluster"
    for r, s in enumerate(systems):
        ref = orc.simulate(s, sim.as_array())
        assert list(out[r].com_start) == list(ref["com_start"])
        assert list(out[r].com_end) == list(ref["com_end"])
        assert out[r].horizontal_displacement == ref["horizontal_displacement"]
        assert out[r].max_speed == ref["max_speed"]
        assert bool(out[r].diverged) == ref["diverged"] and out[r].spring_updates == 250 * s.ns
    # simulate() takes the system by value: the batch is unchanged
    got = batch.download()
    for r, s in enumerate(systems):
        np.testing.assert_array_equal(got.robot(r)["pos"], s.pos)


def _exit_case(vx, ctx, orc, n, mutate, steps):
    items = [orc.bench_robot(n), orc.bench_robot(n)]
    mats = np.stack([m for m, _ in items])
    wts = np.stack([w for _, w in items])
    batch = vx.build_mass_spring(mats, wts, n, n, n, ctx=ctx)
    systems = [orc.build(m, w, n, n, n) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    pos = np.concatenate([s.pos for s in systems])
    vel = np.concatenate([s.vel for s in systems])
    nm = len(systems[0].pos)
    mutate(pos[nm:], vel[nm:])  # robot 1 only
    systems[1].pos[:] = pos[nm:]
    systems[1].vel[:] = vel[nm:]
    batch.set_state(pos, vel)
    out = batch.step(vx.SimConfig(), 0, steps)
    assert ctx.last_integrator == "cluster"
    got = batch.download()
    for r, s in enumerate(systems):
        ref, ok, called, upd, msq = orc.step(s, vx.SimConfig().as_array(), 0, steps)
        np.testing.assert_array_equal(got.robot(r)["pos"], ref.pos)
        np.testing.assert_array_equal(got.robot(r)["vel"], ref.vel)
        assert out[r].spring_updates == upd and out[r].steps == called
        assert bool(out[r].diverged) == (ok < called)
    return out


def test_cluster_zero_length_exit(vx, ctx, orc):
    # a mass on top of its neighbour in the LAST CTA's range: step() reports
    # divergence before touching any mass (physics.hpp:205-207)
    def mutate(pos, vel):
        pos[-1] = pos[-2]
    out = _exit_case(vx, ctx, orc, 10, mutate, 20)
    assert out[1].diverged and out[1].spring_updates == 0 and not out[0].diverged


def test_cluster_divergence_exit(vx, ctx, orc):
    # a mass flung out of the +-1e6 box in the FIRST CTA's range: every mass is
    # still updated that step, then the run stops (physics.hpp:260-263)
    def mutate(pos, vel):
        vel[3, 0] = 2e12
    out = _exit_case(vx, ctx, orc, 10, mutate, 20)
    assert out[1].diverged and not out[0].diverged


@pytest.mark.parametrize("n,frac", [(7, 0.0), (7, 0.99), (8, 0.5), (10, 0.4), (10, 0.75), (10, 0.999)])
def test_cluster_divergence_mid_run(vx, ctx, orc, n, frac):
    """A mass leaves the +-1e6 box several steps into the run, in a chosen
    CTA's range: the divergence word of that step reaches every CTA one phase
    later (no cluster barrier per step), and every CTA stops with the state of
    exactly that step, like step() (physics.hpp:260-263)."""
    def mutate(pos, vel):
        vel[int(frac * (len(vel) - 1)), 1] = 1.8e10  # ~1.8e5 m per step: out of the box at step ~5
    out = _exit_case(vx, ctx, orc, n, mutate, 40)
    assert out[1].diverged and 3 <= out[1].steps <= 8 and not out[0].diverged


@pytest.mark.parametrize("n", [7, 8, 9, 10])
def test_cluster_zero_length_every_size(vx, ctx, orc, n):
    """Coincident masses in the first CTA's range: the zero-length verdict of
    step 0 arrives one phase later and every CTA rolls its state back."""
    def mutate(pos, vel):
        pos[1] = pos[0]
    out = _exit_case(vx, ctx, orc, n, mutate, 12)
    assert out[1].diverged and out[1].spring_updates == 0 and out[1].steps == 1


@pytest.mark.parametrize("steps", [1, 2, 3])
def test_cluster_short_launches(vx, ctx, orc, steps):
    """1-3 step launches: the last step's verdict and halo are drained after
    the loop; a zero-length robot in the batch still rolls back."""
    def mutate(pos, vel):
        pos[-1] = pos[-2]
    out = _exit_case(vx, ctx, orc, 10, mutate, steps)
    assert out[1].diverged and out[1].spring_updates == 0 and not out[0].diverged


def test_cluster_evaluate_fitness(vx, ctx, orc):
    """evaluate_fitness on 10^3 decodes runs the cluster kernel and agrees with
    the reference within the evaluate tolerance."""
    n = 10
    rng = np.random.default_rng(7)
    gs = [orc.sample_genome(32, [64, 64], int(s)) for s in rng.integers(0, 2 ** 62, 3)]
    mats, wts = vx.decode(np.stack([g[0] for g in gs]), np.stack([g[1] for g in gs]), vx.Arch.make(), n, n, n, ctx)
    sim = vx.SimConfig(duration=300 * 1e-5)
    fit = vx.evaluate_fitness(mats, wts, n, n, n, sim=sim, ctx=ctx)
    assert ctx.last_integrator == "cluster"
    for a in range(3):
        ref = orc.evaluate_fitness(mats[a], wts[a], n, n, n, sim=sim.as_array())
        assert abs(fit[a] - ref) <= 1e-3 * max(ref, 1e-12) + 1e-15
