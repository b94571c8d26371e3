"""Every specialised integrator (one-SM lattice 6^3, cluster 10^3, streaming
20^3) under non-default SimConfig / MaterialTable / GroundPlane settings:
bit-exact against the reference's step() on identical systems
(physics.hpp:191-264; scaled materials, plane and sim fields of
morphology.hpp:45-65, 124-129 and physics.hpp:16-29)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KERNEL = {6: "lattice", 10: "cluster", 20: "stream"}
STEPS = {6: 600, 10: 300, 20: 60}


def _variants(vx):
    return {
        "free_fast_drive": (vx.SimConfig(enable_gravity=False, enable_contact=False, actuation_frequency=5.0),
                            vx.MaterialTable(), vx.GroundPlane()),
        "soft_slippery": (vx.SimConfig(dt=2e-5, gravity=5.0),
                          vx.MaterialTable(k_muscle=3e3, k_soft=5e2, amp_max=0.4, phase_max=1.0, damping_ratio=0.2,
                                           voxel_edge=0.05, mass_per_vertex=0.05),
                          vx.GroundPlane(k=2e4, damping_ratio=0.3, mu_static=0.3, mu_kinetic=0.5)),
        "fine_dt_sticky": (vx.SimConfig(dt=5e-6), vx.MaterialTable(k_bone=3e4),
                           vx.GroundPlane(mu_static=1.5, mu_kinetic=1.2)),
    }


@pytest.mark.parametrize("n", [6, 10, 20])
@pytest.mark.parametrize("variant", ["free_fast_drive", "soft_slippery", "fine_dt_sticky"])
def test_specialised_integrators_nondefault(vx, ctx, orc, n, variant):
    sim, table, plane = _variants(vx)[variant]
    rng = np.random.default_rng(n)
    g = orc.sample_genome(32, [64, 64], int(rng.integers(0, 2 ** 62)))
    mats, wts = vx.decode(g[0][None], g[1][None], vx.Arch.make(), n, n, n, ctx)
    items = [orc.bench_robot(n), (orc.largest_component(mats[0], n, n, n), wts[0])]
    batch = vx.build_mass_spring(np.stack([m for m, _ in items]), np.stack([w for _, w in items]), n, n, n,
                                 table=table, plane=plane, ctx=ctx)
    systems = [orc.build(m, w, n, n, n, table.as_array(), plane.as_array()) for m, w in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    steps = STEPS[n]
    out = batch.step(sim, 0, steps)
    assert ctx.last_integrator == KERNEL[n]
    got = batch.download()
    for r, s in enumerate(systems):
        ref, ok, called, upd, msq = orc.step(s, sim.as_array(), 0, steps)
        np.testing.assert_array_equal(got.robot(r)["pos"], ref.pos, err_msg=f"{variant} grid {n} robot {r}")
        np.testing.assert_array_equal(got.robot(r)["vel"], ref.vel, err_msg=f"{variant} grid {n} robot {r}")
        assert out[r].spring_updates == upd and out[r].max_speed == np.sqrt(msq)


@pytest.mark.parametrize("n,steps", [(6, 5000), (10, 5000), (20, 1000)])
def test_full_horizon_bit_exact(vx, ctx, orc, n, steps):
    """The benchmark horizon (5000 steps; 1000 for 20^3 to keep the CPU
    reference quick): a decoded robot stays bit-identical to the reference's
    step() the whole way on every specialised kernel."""
    rng = np.random.default_rng(1000 + n)
    g = orc.sample_genome(32, [64, 64], int(rng.integers(0, 2 ** 62)))
    mats, wts = vx.decode(g[0][None], g[1][None], vx.Arch.make(), n, n, n, ctx)
    body = orc.largest_component(mats[0], n, n, n)
    batch = vx.build_mass_spring(body[None], wts, n, n, n, ctx=ctx)
    s = orc.build(body, wts[0], n, n, n)
    ws = orc.workspace(s)
    batch.override_phase(ws["sin_phase"], ws["cos_phase"])
    out = batch.step(vx.SimConfig(), 0, steps)[0]
    assert ctx.last_integrator == KERNEL[n]
    ref, ok, called, upd, msq = orc.step(s, vx.SimConfig().as_array(), 0, steps)
    got = batch.download()
    np.testing.assert_array_equal(got.pos, ref.pos)
    np.testing.assert_array_equal(got.vel, ref.vel)
    assert out.spring_updates == upd and out.max_speed == np.sqrt(msq)


@pytest.mark.parametrize("dims,kernel,steps", [((5, 6, 5), "lattice", 400),    # rank-indexed one-SM kernel
                                               ((8, 8, 9), "cluster", 300),    # rank-indexed cluster kernel
                                               ((12, 12, 12), "stream", 60)])  # rank-indexed streaming kernel
def test_rank_indexed_variants_bit_exact(vx, ctx, orc, dims, kernel, steps):
    """Shapes the vertex-indexed kernels do not cover run the rank-indexed
    variants; same bit-exactness bar (bench block + a decoded robot)."""
    w, h, d = dims
    rng = np.random.default_rng(w * 100 + h * 10 + d)
    g = orc.sample_genome(32, [64, 64], int(rng.integers(0, 2 ** 62)))
    mats, wts = vx.decode(g[0][None], g[1][None], vx.Arch.make(), w, h, d, ctx)
    full = np.zeros(w * h * d, np.uint8)
    for z in range(d):
        for y in range(h):
            for x in range(w):
                full[x + w * (y + h * z)] = [1, 2, 3, 4][(x + 2 * y + 3 * z) % 4]  # bench.hpp:35-44 pattern
    items = [(full, np.ones(w * h * d)), (orc.largest_component(mats[0], w, h, d), wts[0])]
    batch = vx.build_mass_spring(np.stack([m for m, _ in items]), np.stack([x for _, x in items]), w, h, d, ctx=ctx)
    systems = [orc.build(m, x, w, h, d) for m, x in items]
    batch.override_phase(np.concatenate([orc.workspace(s)["sin_phase"] for s in systems]),
                         np.concatenate([orc.workspace(s)["cos_phase"] for s in systems]))
    out = batch.step(vx.SimConfig(), 0, steps)
    assert ctx.last_integrator == kernel
    got = batch.download()
    for r, s in enumerate(systems):
        ref, ok, called, upd, msq = orc.step(s, vx.SimConfig().as_array(), 0, steps)
        np.testing.assert_array_equal(got.robot(r)["pos"], ref.pos, err_msg=f"{dims} robot {r}")
        np.testing.assert_array_equal(got.robot(r)["vel"], ref.vel, err_msg=f"{dims} robot {r}")
        assert out[r].spring_updates == upd


@pytest.mark.parametrize("variant", ["free_fast_drive", "soft_slippery", "fine_dt_sticky"])
def test_stream_tma_kernel_bit_exact(vx, ctx, orc, variant, monkeypatch):
    """The opt-in bulk-copy-fed 20^3 kernel (VX_STREAM_TMA=1,
    stream_sym_tma_kernel: warp-specialised producer, mbarrier stage ring)
    is bit-exact like the default one."""
    monkeypatch.setenv("VX_STREAM_TMA", "1")
    test_specialised_integrators_nondefault(vx, ctx, orc, 20, variant)
