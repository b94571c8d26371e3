"""Scripted advisor in the loop, device vs the reference.

The reference's own ScriptedAdvisor (advisor.hpp:30-55, compiled unmodified
into oracle/_ref) is consulted inside its evolve_generation
(evolution.hpp:221-227); the device run consults the product's
runner.ScriptedAdvisor the same way.  A fired rule changes the hyper-
parameters and therefore the GA stream's consumption, so identical params
histories, reports, populations and RNG states over many generations prove
identical decisions.

Fitness is the one chaotic quantity (median 1e-4 at the
default step, a few 1e-3 on single small robots, up to a few 1e-2 at the
coarser dt = 1e-4 of these short runs), and one near-tie flipped by it reorders the
sorted population and sends the two runs down different paths.  The test
therefore runs lock-step with teacher forcing at the exchange point the
sharded generation already has: the device evaluates every pending robot
(checked against the reference's value within the stated tolerance), then
the reference's value is written into the exchange buffer before
vx_evo_finish.  Everything downstream — the stable sort, best / mean /
stddev, the diversity (bit-exact, so the advisor's floor fires identically),
the advisor's decision, elites, tournaments, crossover, mutation and the RNG
stream — must then match the reference exactly.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    from paper_2405_00698_b200 import runner
    return runner


def _lockstep(vx, ctx, orc, R, seed, adv4=None, P=16, grid=4, gens=10, dt=1e-4, duration=0.1, fit_tol=5e-2):
    import torch

    if not hasattr(orc, "evo") or not oracle.have_reference():
        pytest.skip("needs the compiled reference (oracle/_ref)")
    sim6 = oracle.sim6(dt=dt, duration=duration)
    cfg = vx.EvolutionConfig(population=P, generations=gens, grid=(grid, grid, grid), seed=seed,
                             sim=vx.SimConfig(dt=dt, duration=duration))
    ref = orc.evo(population=P, generations=gens, grid=(grid, grid, grid), seed=seed, sim=sim6)
    st = vx.init_evolution(cfg, ctx)
    pop = ref.population()
    st.set_population(pop["params"], pop["bmat"])
    st.set_rng_state(ref.rng_state())
    xbuf = torch.zeros(st.exchange_buffer()[1], dtype=torch.float64, device="cuda")
    st.set_exchange_buffer(xbuf.data_ptr())
    adv = R.ScriptedAdvisor() if adv4 is None else R.ScriptedAdvisor(*adv4)
    fired, rels = 0, []
    for g in range(gens):
        forced = ref.pending_fitness()  # what the reference's evolve_generation will store
        todo = np.flatnonzero(~np.isnan(forced))
        st.begin(0, 1, adv)
        torch.cuda.synchronize()
        got = xbuf[:P].cpu().numpy()
        rel = np.abs(got[todo] - forced[todo]) / np.maximum(np.abs(forced[todo]), 1e-12)
        rels.extend(rel.tolist())
        assert rel.size == 0 or rel.max() <= fit_tol, (g, rel.max())
        xbuf[torch.as_tensor(todo, device="cuda")] = torch.as_tensor(forced[todo], device="cuda")
        torch.cuda.synchronize()
        rep = st.finish()
        rr = ref.generation_advised(adv4)
        np.testing.assert_array_equal(rep.params.as_array(), rr["params"], err_msg=f"generation {g}: params")
        assert (rep.generation, rep.evaluations) == (rr["generation"], rr["evaluations"]) == (g, todo.size)
        assert (rep.best, rep.mean, rep.stddev) == (rr["best"], rr["mean"], rr["stddev"]), g
        assert rep.diversity == rr["diversity"], g  # bit-exact: the advisor's floor fires identically
        fired += not np.array_equal(rr["params"], oracle.DEFAULT_HYPER)
    assert st.rng_state() == ref.rng_state()
    mine, theirs = st.population(), ref.population()
    for k in ("params", "bmat", "fitness", "evaluated"):
        np.testing.assert_array_equal(mine[k], theirs[k], err_msg=k)
    return fired, np.asarray(rels)


def test_scripted_advisor_defaults_lockstep(vx, ctx, orc, R):
    """Default rules: the stagnation trigger fires once the best stalls."""
    fired, _ = _lockstep(vx, ctx, orc, R, seed=4)
    assert fired >= 1


def test_scripted_advisor_both_rules_lockstep(vx, ctx, orc, R):
    """A floor above any diversity the run reaches: the mutation boost fires
    every consult (clamped at 1.0 within a few generations) on top of the
    stagnation rule."""
    fired, _ = _lockstep(vx, ctx, orc, R, seed=11, adv4=(0.95, 1e-6, 1.5, 1.25), gens=9)
    assert fired >= 5


def test_scripted_advisor_default_step_lockstep(vx, ctx, orc, R):
    """The reference's default step (dt 1e-5, 5000 steps) on 5^3 robots: fitness
    before forcing within the chaos floor (max 5e-3 on a single small robot,
    median 1e-4), the advisor path exact after."""
    _, rels = _lockstep(vx, ctx, orc, R, seed=23, P=12, grid=5, gens=8, dt=1e-5, duration=0.05, fit_tol=5e-3)
    assert np.median(rels) <= 1e-4
