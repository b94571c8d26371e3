"""Pin the oracle before trusting it (CPU only).

* the C restatement (oracle/voxevo_oracle.c) is bit-identical to the compiled
  reference (oracle/_ref, built from /root/reference's unmodified headers);
* both reproduce the golden vectors generated from the reference
  (tests/golden/make_golden.py): the mt19937_64 KATs, config-1 decode and
  topology, the bench-robot work audit 33,152,000 (proj/test_output.txt:30),
  the elite_count table (test_evolution.cpp:50-56), the desk GA curve.
"""
import numpy as np
import pytest

import oracle

pytestmark = []

SYS_FIELDS = ("pos", "vel", "mass", "si", "sj", "k", "rest0", "zeta", "has_act", "sign", "amp", "phase")


def libm_matches(golden_meta_path="tests/golden/meta.json"):
    """Golden libm-dependent values are bit-stable only on the generating host's glibc/ifunc variant."""
    import json
    import os
    import platform
    meta = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       golden_meta_path)))
    fma = "fma" in open("/proc/cpuinfo").read()
    variant = "FMA/AVX2 host" if fma else "SSE2 host"
    return meta["glibc"] == platform.libc_ver()[1] and variant in meta["libm_variant"]


def test_rng_kats(orc, restated, golden):
    # 10000th output of mt19937_64(5489); Rng(42).next_u64()
    for lib in (orc, restated):
        assert lib.rng_draws(5489, 10000)[-1] == np.uint64(9981545732273789042)
        assert lib.rng_draws(42, 1)[0] == np.uint64(13930160852258120406)
        np.testing.assert_array_equal(lib.rng_draws(42, 8), golden["kat_42_first"])
        np.testing.assert_array_equal(lib.rng_uniform(7, 64), golden["rng7_uniform"])
        np.testing.assert_array_equal(lib.rng_index(9, 64, 7), golden["rng9_index7"])
        # normal() goes through glibc log/cos
        np.testing.assert_allclose(lib.rng_normal(7, 64), golden["rng7_normal"], rtol=1e-14, atol=1e-15)


def test_rng_text_state(orc, restated, golden):
    st = golden["rng99_state17"].tobytes().decode()
    toks = st.split()
    assert len(toks) == 313 and toks[-1] == "17"
    for lib in (orc, restated):
        assert lib.rng_state(99, 17) == st
        np.testing.assert_array_equal(lib.rng_draws_from_state(st, 50), golden["rng99_after17"])
    fresh = restated.rng_state(42, 0).split()
    assert fresh[0] == "42" and fresh[-1] == "312"


def test_genome_and_decode_config1(orc, restated, golden):
    for lib in (orc, restated):
        params, bmat = lib.sample_genome(32, [64, 64], 42)
        assert len(params) == 8710 == lib.param_count(32, [64, 64])
        mat, wt = lib.decode(32, [64, 64], golden["c1_params"], golden["c1_bmat"], 4, 4, 4)
        np.testing.assert_array_equal(mat, golden["c1_mat"])
        np.testing.assert_allclose(wt, golden["c1_wt"], rtol=1e-13)
        body = lib.largest_component(golden["c1_mat"], 4, 4, 4)
        np.testing.assert_array_equal(body, golden["c1_body"])
        assert int((body > 0).sum()) == 50
        if libm_matches():
            np.testing.assert_array_equal(params, golden["c1_params"])
            np.testing.assert_array_equal(bmat, golden["c1_bmat"])


def test_build_config1_exact(orc, restated, golden):
    for lib in (orc, restated):
        s = lib.build(golden["c1_body"], golden["c1_wt"], 4, 4, 4)
        assert (s.nm, s.ns) == (122, 908)
        for f in SYS_FIELDS:
            np.testing.assert_array_equal(getattr(s, f), golden["c1_sys_" + f], err_msg=f)


def test_bench_robot_audit(orc, restated, golden):
    for lib in (orc, restated):
        m, w = lib.bench_robot(4)
        np.testing.assert_array_equal(m, golden["b4_mat"])
        s = lib.build(m, w, 4, 4, 4)
        assert (s.nm, s.ns) == (125, 1036)
        for f in SYS_FIELDS:
            np.testing.assert_array_equal(getattr(s, f), golden["b4_sys_" + f], err_msg=f)
    # proj/test_output.txt:30: 16 jobs x 2000 steps x 1036 springs = 33,152,000, exact
    np.testing.assert_array_equal(golden["b4_bench_counts"], [1036, 33152000, 33152000, 0])


def test_elite_count_table(orc, restated, golden):
    for ef, P, want in golden["elite_table"]:
        assert orc.elite_count(ef, int(P)) == int(want) == restated.elite_count(ef, int(P))
    assert [int(x) for x in golden["elite_table"][:, 2]] == [9, 1, 10, 2, 5]  # test_evolution.cpp:50-56


def test_builder_counts(restated):
    # acceptance_main.cpp:418-450 / test_morphology.cpp:102-172, 228-241
    one = restated.build(np.array([3], np.uint8), np.array([0.75]), 1, 1, 1)
    assert (one.nm, one.ns) == (8, 28)
    kinds = np.round(one.rest0 / 0.1, 6)
    assert sorted(np.unique(kinds, return_counts=True)[1].tolist()) == [4, 12, 12]
    two = restated.build(np.array([3, 4], np.uint8), np.array([1.0, 0.5]), 2, 1, 1)
    assert (two.nm, two.ns) == (12, 50)
    assert np.isclose(two.k, 3000.0).sum() == 6
    ell = restated.build(np.array([3, 3, 3, 0], np.uint8), np.ones(4), 2, 2, 1)
    assert ell.nm == 16
    assert restated.build(np.zeros(27, np.uint8), np.ones(27), 3, 3, 3) is None


def test_physics_kats(restated):
    # test_physics.cpp:62-81: static force 5 N; damping coefficient
    s = oracle.dumbbell(0.2, 100.0, 0.1, 0.15)
    sim = oracle.sim6(dt=1e-5, enable_gravity=False, enable_contact=False)
    s1, ok, called, upd, _ = restated.step(s, sim, 0, 1)
    assert ok == 1 and upd == 1
    # one step applies F/m*dt: v_i = 5/0.2*1e-5
    assert abs(s1.vel[0, 0] - 5.0 / 0.2 * 1e-5) < 1e-15
    assert s1.vel[1, 0] == -s1.vel[0, 0]
    ws = restated.workspace(oracle.dumbbell(0.2, 100.0, 0.1, 0.1, 0.5))
    mu = 0.2 * 0.2 / 0.4
    assert abs(ws["damp_coef"][0] - 0.5 * 2.0 * np.sqrt(100.0 * mu)) < 1e-12


@pytest.mark.skipif(not oracle.have_reference(), reason="compiled reference absent")
def test_restatement_bit_identical_to_reference(restated):
    ref = oracle.reference()
    rng = np.random.default_rng(5)
    for seed in range(3):
        p1, b1 = ref.sample_genome(16, [24, 24], seed)
        p2, b2 = restated.sample_genome(16, [24, 24], seed)
        np.testing.assert_array_equal(p1, p2)
        np.testing.assert_array_equal(b1, b2)
        m1, w1 = ref.decode(16, [24, 24], p1, b1, 5, 4, 3)
        m2, w2 = restated.decode(16, [24, 24], p2, b2, 5, 4, 3)
        np.testing.assert_array_equal(m1, m2)
        np.testing.assert_array_equal(w1, w2)
    for _ in range(20):
        w, h, d = rng.integers(1, 6, 3)
        mat = (rng.random(w * h * d) < 0.6) * rng.integers(1, 5, w * h * d)
        mat = mat.astype(np.uint8)
        wt = rng.uniform(0.1, 1.0, w * h * d)
        np.testing.assert_array_equal(ref.largest_component(mat, w, h, d), restated.largest_component(mat, w, h, d))
        a, b = ref.build(mat, wt, w, h, d), restated.build(mat, wt, w, h, d)
        assert (a is None) == (b is None)
        if a is None:
            continue
        for f in SYS_FIELDS:
            np.testing.assert_array_equal(getattr(a, f), getattr(b, f), err_msg=f)
        sim = oracle.sim6(duration=300e-5)
        sa, sb = ref.simulate(a, sim), restated.simulate(b, sim)
        assert sa["horizontal_displacement"] == sb["horizontal_displacement"]
        np.testing.assert_array_equal(sa["com_end"], sb["com_end"])
        assert sa["diverged"] == sb["diverged"]
    mats = rng.integers(0, 5, (9, 30)).astype(np.uint8)
    assert ref.population_diversity(mats) == restated.population_diversity(mats)


@pytest.mark.skipif(not oracle.have_reference(), reason="compiled reference absent")
def test_restatement_evolution_bit_identical(restated):
    ref = oracle.reference()
    kw = dict(population=6, generations=3, grid=(3, 3, 3), hidden=(12, 12), m=8, seed=33,
              sim=oracle.sim6(dt=1e-4, duration=0.05))
    a, b = ref.evo(**kw), restated.evo(**kw)
    for _ in range(4):
        ra, rb = a.generation(), b.generation()
        for k in ("best", "mean", "stddev", "diversity", "evaluations"):
            assert ra[k] == rb[k], k
    pa, pb = a.population(), b.population()
    for k in pa:
        np.testing.assert_array_equal(pa[k], pb[k], err_msg=k)
    assert a.rng_state() == b.rng_state()


def test_desk_ga_golden(restated, golden):
    """acceptance_main.cpp:193-211 desk GA (seed 1): reference curve reproduced."""
    if not libm_matches():
        pytest.skip("golden GA curve is libm-variant specific")
    ev = restated.evo(population=12, generations=20, grid=(3, 3, 3), seed=1, sim=oracle.sim6(dt=1e-4, duration=0.5))
    reps = [ev.generation() for _ in range(21)]
    np.testing.assert_array_equal([r["best"] for r in reps], golden["desk1_best"])
    np.testing.assert_array_equal([r["evaluations"] for r in reps], golden["desk1_evals"])
    assert ev.rng_state() == golden["desk1_rng_state"].tobytes().decode()
