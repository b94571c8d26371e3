"""Decode on the FP64 tensor pipe (decode_mma_kernel, DMMA m8n8k4) against the
exact sequential-order kernel and the reference (morphology.hpp:141-157 over
forward, genome.hpp:187-211).

Tolerances: materials bit-exact (by construction: near-ties are re-decoded
on the exact path); weights rtol 1e-13 against the reference (device
transcendentals, as for the exact kernel) and 1e-14 against the exact kernel
(DMMA accumulation order only).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _decode(vx, params, bmat, arch, dims, ctx, exact):
    old = os.environ.get("VX_DECODE")
    try:
        if exact:
            os.environ["VX_DECODE"] = "exact"
        else:
            os.environ.pop("VX_DECODE", None)
        out = vx.decode(params, bmat, arch, *dims, ctx=ctx)
        return out + (vx.decode_refined(ctx),)
    finally:
        if old is None:
            os.environ.pop("VX_DECODE", None)
        else:
            os.environ["VX_DECODE"] = old


@pytest.mark.parametrize("m,hidden,dims", [
    (32, [64, 64], (10, 10, 10)),  # configs 3/4: the default network
    (32, [64, 64], (6, 6, 6)),     # config 2
    (8, [12, 12], (3, 3, 3)),      # padded K and N tiles
    (4, [6], (5, 2, 3)),           # one n-tile split over warps, ragged voxel tile
    (16, [], (4, 4, 4)),           # heads straight from the encoding
    (32, [80, 48, 16], (6, 6, 6)), # > 8 n-tiles, 6, 2
    (3, [5, 130], (7, 3, 2)),      # odd K (6), wide last layer
])
def test_mma_matches_exact_and_reference(vx, ctx, orc, m, hidden, dims):
    rng = np.random.default_rng(m * 1000 + len(hidden))
    P = 24
    arch = vx.Arch.make(m, hidden)
    gs = [orc.sample_genome(m, hidden, int(s)) for s in rng.integers(0, 2 ** 62, P)]
    params = np.stack([g[0] for g in gs])
    bmat = np.stack([g[1] for g in gs])
    mt, wt, refined = _decode(vx, params, bmat, arch, dims, ctx, exact=False)
    assert refined >= 0, "the tensor-pipe decode did not run"
    me, we, r2 = _decode(vx, params, bmat, arch, dims, ctx, exact=True)
    assert r2 == -1
    np.testing.assert_array_equal(mt, me)
    np.testing.assert_allclose(wt, we, rtol=1e-14, atol=0)
    for a in range(0, P, 6):
        rm, rw = orc.decode(m, hidden, params[a], bmat[a], *dims)
        np.testing.assert_array_equal(mt[a], rm)
        np.testing.assert_allclose(wt[a], rw, rtol=1e-13)


def test_mma_ties_go_to_exact_path(vx, ctx):
    # test_morphology.cpp:41-45: all-zero head -> five-way tie -> Empty; the
    # tie flags the genome and the exact kernel re-decodes it
    arch = vx.Arch.make(1, [])
    params = np.zeros((3, vx.param_count(arch)))
    rng = np.random.default_rng(5)
    params[1] = rng.uniform(-1, 1, params.shape[1])  # a clear winner everywhere: not flagged
    params[1, 10:15] = [0.0, 0.0, 40.0, 0.0, 0.0]  # bm (after Wm[5][2]): MuscleContract dominates
    mat, wt, refined = _decode(vx, params, np.zeros((3, 3)), arch, (2, 2, 2), ctx, exact=False)
    assert refined == 2
    assert (mat[0] == 0).all() and (mat[2] == 0).all() and np.allclose(wt[0], 0.5)
    assert (mat[1] == 2).all()


def test_mma_population_bench_shape(vx, ctx, orc):
    """A config-3 population slice: 256 default genomes on 10^3 grids."""
    arch = vx.Arch.make()
    seeds = np.random.default_rng(11).integers(0, 2 ** 62, 256)
    params, bmat = vx.sample_genomes(arch, [int(s) for s in seeds], ctx)
    mt, wt, refined = _decode(vx, params, bmat, arch, (10, 10, 10), ctx, exact=False)
    me, we, _ = _decode(vx, params, bmat, arch, (10, 10, 10), ctx, exact=True)
    np.testing.assert_array_equal(mt, me)
    np.testing.assert_allclose(wt, we, rtol=1e-14, atol=0)
    assert refined <= 8  # gaps < 1e-8 are rare (smallest seen 2.85e-7)


@pytest.mark.parametrize("hidden", [[256], [512], [2048], [600, 40]])
def test_wide_network_falls_back_to_exact_kernel(vx, ctx, orc, hidden):
    """Weights + activations too large for the tensor-pipe kernel's shared
    memory (hidden 256: ~300 KB): decode runs the exact-order kernel with the
    genome read from global memory — and for very wide layers (512, 2048)
    on narrower voxel tiles — still bit-exact in materials (the reference
    accepts any width)."""
    m, dims = 32, (4, 4, 4)
    arch = vx.Arch.make(m, hidden)
    gs = [orc.sample_genome(m, hidden, s) for s in (5, 6, 7)]
    params = np.stack([g[0] for g in gs])
    bmat = np.stack([g[1] for g in gs])
    mt, wt, refined = _decode(vx, params, bmat, arch, dims, ctx, exact=False)
    assert refined == -1  # the tensor-pipe kernel did not run
    for a in range(3):
        rm, rw = orc.decode(m, hidden, params[a], bmat[a], *dims)
        np.testing.assert_array_equal(mt[a], rm)
        np.testing.assert_allclose(wt[a], rw, rtol=1e-13)


def test_decode_timing_and_dmma_peak(vx, ctx):
    """The bench line's decode roofline inputs: live CUDA-event time and voxel
    count of decode launches (vx_decode_timing) and the measured DMMA peak."""
    arch = vx.Arch.make()
    params, bmat = vx.sample_genomes(arch, [3, 4, 5, 6], ctx)
    ctx.timing(True)
    ctx.decode_time(reset=True)
    vx.decode(params, bmat, arch, 5, 5, 5, ctx)
    vx.decode(params[:2], bmat[:2], arch, 4, 4, 4, ctx)
    ms, voxels = ctx.decode_time(reset=True)
    ctx.timing(False)
    assert ms > 0.0 and voxels == 4 * 125 + 2 * 64
    assert ctx.decode_time(reset=True) == (0.0, 0)
    peak = ctx.dmma_peak_tflops()
    assert 10.0 < peak < 100.0, peak  # B200: ~37 TFLOP/s FP64 on DMMA
