"""Rng (rng.hpp:15-56) and the single-genome GA operators (crossover,
mutate, tournament_select: evolution.hpp:143-173) of the host C ABI, against
the reference's own Rng compiled in oracle/_ref (raw draws, uniform01,
normal, index, text state) and Python restatements of the operators on those
draws (Python's math module is the same glibc libm).  Host-only: no device."""
import math

import numpy as np
import pytest

import oracle


@pytest.fixture(scope="module")
def ref():
    if not oracle.have_reference():
        pytest.skip("oracle/_ref not built")
    return oracle.reference()


def _u01(x):
    return float(int(x) >> 11) * 2.0 ** -53


def _normal(x1, x2):
    u1 = (float(int(x1) >> 11) + 0.5) * 2.0 ** -53
    u2 = float(int(x2) >> 11) * 2.0 ** -53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(2.0 * math.pi * u2)


@pytest.mark.parametrize("seed", [0, 1, 42, 2 ** 63 + 5])
def test_rng_streams_match_reference(vx, ref, seed):
    r = vx.Rng(seed)
    np.testing.assert_array_equal([r.next_u64() for _ in range(700)], ref.rng_draws(seed, 700))
    r = vx.Rng(seed)
    np.testing.assert_array_equal([r.uniform01() for _ in range(500)], ref.rng_uniform(seed, 500))
    r = vx.Rng(seed)
    np.testing.assert_array_equal([r.normal() for _ in range(500)], ref.rng_normal(seed, 500))
    for n in (1, 3, 30, 2 ** 40 + 7):
        r = vx.Rng(seed)
        np.testing.assert_array_equal([r.index(n) for _ in range(300)], ref.rng_index(seed, 300, n))


def test_rng_known_answers(vx):
    assert vx.Rng(42).next_u64() == 13930160852258120406  # SURVEY.md §8(c) probe
    r = vx.Rng()  # Rng() : engine_(0)
    assert r.next_u64() == vx.Rng(0).next_u64()
    r = vx.Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042  # the standard's 10000th-output check for mt19937_64


def test_rng_state_text_interop(vx, ref):
    r = vx.Rng(7)
    for _ in range(1234):
        r.next_u64()
    assert r.state() == ref.rng_state(7, 1234)
    s = vx.Rng(1)
    s.set_state(ref.rng_state(99, 10))
    np.testing.assert_array_equal([s.next_u64() for _ in range(400)], ref.rng_draws_from_state(ref.rng_state(99, 10), 400))
    assert s == s and not (s == vx.Rng(99))
    with pytest.raises(ValueError):
        s.set_state("not a state")


@pytest.mark.parametrize("np_", [1, 37, 8710])
def test_crossover_matches_reference_draws(vx, ref, np_):
    rng = np.random.default_rng(np_)
    a, b = rng.normal(size=np_), rng.normal(size=np_)
    bm = rng.normal(size=96)
    r = vx.Rng(11)
    child, cbm = vx.crossover(a, b, r, a_bmat=bm, b_bmat=bm + 1)
    u = ref.rng_uniform(11, np_)
    np.testing.assert_array_equal(child, np.where(u < 0.5, b, a))
    np.testing.assert_array_equal(cbm, bm)  # the encoding matrix is a's
    assert r.state() == ref.rng_state(11, np_)
    with pytest.raises(vx.ShapeMismatch):
        vx.crossover(a, b[:-1] if np_ > 1 else np.zeros(2), r)


@pytest.mark.parametrize("rate,scale", [(0.1, 0.1), (1.0, 0.5), (0.0, 1.0), (0.37, 2.0)])
def test_mutate_matches_reference_draws(vx, ref, rate, scale):
    n = 500
    params = np.linspace(-1, 1, n)
    want = params.copy()
    draws = ref.rng_draws(3, 4 * n)
    q = 0
    for i in range(n):  # mutate (evolution.hpp:160-165) on the reference's raw stream
        u = _u01(draws[q])
        q += 1
        if u < rate:
            want[i] += _normal(draws[q], draws[q + 1]) * scale
            q += 2
    r = vx.Rng(3)
    vx.mutate(params, rate, scale, r)
    np.testing.assert_array_equal(params, want)
    assert r.state() == ref.rng_state(3, q)


@pytest.mark.parametrize("P,size", [(1, 3), (24, 1), (24, 3), (1000, 5)])
def test_tournament_matches_reference_draws(vx, ref, P, size):
    r = vx.Rng(17)
    got = [vx.tournament_select(P, size, r) for _ in range(50)]
    idx = ref.rng_index(17, 50 * size, P)
    want = [int(min(idx[k * size:(k + 1) * size])) for k in range(50)]
    assert got == want


def test_rng_reference_unit_cases(vx):
    """test_rng.cpp:19-57 restated on the library's Rng."""
    r = vx.Rng(1)
    u = np.array([r.uniform01() for _ in range(100000)])
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    r = vx.Rng(2)
    x = np.array([r.normal() for _ in range(100000)])
    assert np.isfinite(x).all() and abs(x.mean()) < 0.02 and abs(x.var() - 1.0) < 0.03
    r = vx.Rng(3)
    k = [r.index(7) for _ in range(1000)]
    assert set(k) == set(range(7))
    r = vx.Rng(99)
    for _ in range(17):
        r.next_u64()
    snap = r.state()
    a = [r.next_u64(), r.uniform01(), r.normal(), r.index(1000)]
    r.set_state(snap)
    assert [r.next_u64(), r.uniform01(), r.normal(), r.index(1000)] == a


def test_gaussian_encode_matches_reference(vx, ref):
    """gaussian_encode (genome.hpp:168-179), host ABI, bit for bit."""
    rng = np.random.default_rng(8)
    for m in (1, 4, 32):
        b = rng.normal(size=3 * m)
        for v in (rng.random(3), rng.normal(0, 5, 3), np.zeros(3)):
            np.testing.assert_array_equal(vx.gaussian_encode(v, b, m), ref.gaussian_encode(v, b, m))
    with pytest.raises(vx.ShapeMismatch):
        vx.gaussian_encode(np.zeros(3), np.zeros(5), 2)
