"""run_loop / artifacts / scripted advisor (paper_2405_00698_b200/runner.py)
against runner.hpp, advisor.hpp and config.hpp."""
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def R():
    from paper_2405_00698_b200 import runner
    return runner


@pytest.fixture(scope="module")
def S():
    from paper_2405_00698_b200 import serialize
    return serialize


def _rep(vx, gen, best, div):
    r = vx.GenerationReport()
    r.generation, r.best, r.diversity = gen, best, div
    r.params = vx.HyperParams()
    return r


def test_scripted_advisor_rules(vx, R):
    # advisor.hpp:25-55
    adv = R.ScriptedAdvisor()
    cur = vx.HyperParams()
    assert adv([], cur) is None
    assert adv([_rep(vx, 0, 0.1, 0.5), _rep(vx, 1, 0.2, 0.5)], cur) is None  # improving, diverse
    low_div = adv([_rep(vx, 0, 0.1, 0.5), _rep(vx, 1, 0.2, 0.01)], cur)
    assert low_div.mutation_rate == pytest.approx(0.15) and low_div.mutation_scale == pytest.approx(0.15)
    assert low_div.crossover_rate == cur.crossover_rate
    stag = adv([_rep(vx, 0, 0.2, 0.5), _rep(vx, 1, 0.2, 0.5)], cur)
    assert stag.crossover_rate == pytest.approx(0.5) and stag.mutation_rate == cur.mutation_rate
    hot = vx.HyperParams(mutation_rate=0.9, crossover_rate=0.95)
    both = adv([_rep(vx, 0, 0.2, 0.5), _rep(vx, 1, 0.2, 0.0)], hot)
    assert both.mutation_rate == 1.0 and both.crossover_rate == 1.0  # clamped (evolution.hpp:29-35)


def test_make_advisor(R, S):
    assert R.make_advisor(S.run_config_from_json({})) is None
    assert isinstance(R.make_advisor(S.run_config_from_json({"advisor": "scripted"})), R.ScriptedAdvisor)
    with pytest.raises(Exception):
        R.make_advisor(S.run_config_from_json({"advisor": "llm"}))
    assert R.advisor_consults_done(2) == 0 and R.advisor_consults_done(7) == 4  # runner.hpp:33-36


def test_run_config_echo_round_trip(R, S):
    rc = S.run_config_from_json({"population": 8, "grid": [4, 5, 6], "advisor": "scripted", "out_dir": "o",
                                 "llm": {"model": "m", "max_retries": 4, "unknown": 1}, "checkpoint_stride": 3})
    j = R.run_config_to_json(rc)
    assert set(j) == {"population", "generations", "grid", "hidden_widths", "encoding", "tournament_size", "threads",
                      "seed", "params", "materials", "plane", "sim", "advisor", "replay_audit", "out_dir",
                      "checkpoint_stride", "llm"}
    assert j["llm"]["model"] == "m" and j["llm"]["max_retries"] == 4 and "unknown" not in j["llm"]
    assert R.run_config_to_json(S.run_config_from_json(j)) == j


def test_log_report_format(vx, R):
    r = _rep(vx, 3, 0.0123456789, 0.5)
    r.mean, r.stddev, r.evaluations, r.wall_time = 0.001, 0.002, 21, 1.234
    assert R.log_report(r) == ("gen    3  best 0.012346  mean 0.001000  std 0.002000  div 0.500  evals  21  "
                               "mr 0.1 ms 0.1 cx 0.4 ef 0.3  [1.23s]")


def _tiny(S, out_dir, advisor="off", gens=5):
    return S.run_config_from_json({"population": 6, "generations": gens, "grid": [3, 3, 3], "hidden_widths": [8],
                                   "encoding": {"m": 4}, "seed": 19, "sim": {"dt": 1e-4, "duration": 0.02},
                                   "advisor": advisor, "out_dir": out_dir, "checkpoint_stride": 2})


@pytest.mark.gpu
def test_start_run_artifacts(vx, R, S, ctx, tmp_path):
    rc = _tiny(S, str(tmp_path / "run"))
    st = R.start_run(rc, ctx)
    p = R.artifact_paths(rc.out_dir)
    assert st.generation == rc.evolution.generations + 1 and len(st.history) == rc.evolution.generations + 1
    assert open(p.curves).read() == S.curves_csv(st.history)
    assert S.load_json_file(p.config_echo) == R.run_config_to_json(rc)
    ck = S.unwrap_payload(S.load_json_file(p.checkpoint), "run")
    assert ck["generation"] == st.generation and ck["rng"] == st.rng_state()
    bp, bb = S.load_genome(p.best_genome, st.config.arch)
    np.testing.assert_array_equal(bp, st.best()[1])


@pytest.mark.gpu
def test_resume_run_equals_straight(vx, R, S, ctx, tmp_path):
    # runner.hpp:88-92: an interrupted run (checkpoint after generation 2)
    # resumed through run_loop ends exactly where the uninterrupted one does
    rc = _tiny(S, str(tmp_path / "straight"), advisor="scripted")
    straight = R.start_run(rc, ctx)
    first = vx.init_evolution(rc.evolution, ctx)
    adv = R.ScriptedAdvisor()
    for _ in range(3):
        first.evolve_generation(adv)
    ck = str(tmp_path / "mid.json")
    S.save_run(ck, first)
    resumed = R.resume_run(ck, _tiny(S, str(tmp_path / "rest"), advisor="scripted"), ctx)
    key = [(r.generation, r.best, r.mean, r.diversity, r.params.mutation_rate, r.params.crossover_rate)
           for r in straight.history]
    assert [(r.generation, r.best, r.mean, r.diversity, r.params.mutation_rate, r.params.crossover_rate)
            for r in resumed.history] == key
    assert resumed.rng_state() == straight.rng_state()
    assert os.path.exists(R.artifact_paths(str(tmp_path / "rest")).curves)
