"""The breeding-plan scan (csrc/ga_plan.cpp: block mt19937_64, integer
uniform tests, hit-to-hit mutation walk, Box-Muller on worker threads)
against a straight restatement of the reference breeding loop on
std::mt19937_64 (evolution.hpp:143-165, 267-289; rng.hpp:23-39): plans,
crossover masks, mutation lists (delta bits) and the final RNG state must be
identical.  Host-only: tests/native/plan_check.cpp built with g++ here."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def plan_check(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("plan") / "plan_check")
    subprocess.run(["g++", "-O2", "-std=c++17", "-pthread", os.path.join(ROOT, "tests", "native", "plan_check.cpp"),
                    os.path.join(ROOT, "paper_2405_00698_b200", "csrc", "ga_plan.cpp"), "-o", exe], check=True)
    return exe


@pytest.mark.parametrize("skip", [0, 7, 311, 312])
@pytest.mark.parametrize("P,np_,cx,rate,gens", [
    (256, 8710, 0.5, 0.05, 2),     # config 2 shape: default controller, crossover + mutation
    (2048, 8710, 0.4, 0.1, 1),     # 8-rank population, several mutation chunks (worker pool)
    (100, 37, 1.0, 1.0, 5),        # every draw a hit: 3 draws per parameter
    (64, 1000, 0.0, 0.0, 3),       # no crossover, no mutation
    (3, 5, 0.5, 0.5, 50),          # tiny: windows never fit, scalar path only
    (50, 100, 0.7, 0.9, 20),       # np not a multiple of 32 (partial mask word)
    (300, 63, 0.5, 0.2, 20),       # buffer boundary crossings at many offsets
    (40, 20000, 0.5, 1e-4, 3),     # rare hits: long skips across buffer refills
])
def test_plan_scan_matches_restated_loop(plan_check, P, np_, cx, rate, gens, skip):
    out = subprocess.run([plan_check, str(P), str(np_), str(cx), str(rate), str(gens), str(skip)], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["ok"] is True


def test_plan_scan_random_sweep(plan_check):
    """Random shapes and rates (a fixed-seed sweep): every combination must
    reproduce the restated loop bit for bit."""
    rng = np.random.default_rng(2405)
    for _ in range(12):
        P = int(rng.integers(2, 400))
        np_ = int(rng.integers(1, 5000))
        cx = float(rng.choice([0.0, 1.0, rng.random()]))
        rate = float(rng.choice([0.0, 1.0, rng.random() * 0.3, rng.random()]))
        skip = int(rng.integers(0, 700))
        out = subprocess.run([plan_check, str(P), str(np_), repr(cx), repr(rate), "2", str(skip)],
                             capture_output=True, text=True, timeout=120)
        assert out.returncode == 0, (P, np_, cx, rate, skip, out.stdout)


def test_plan_scan_thread_sanitizer(tmp_path):
    """The scan thread appends mutation chunks while worker threads fill their
    normals (round-1 advisor: a reallocation race).  ThreadSanitizer over
    shapes that start the worker pool (many 16k-entry chunks) and a
    multi-generation run must report no data race, and the results still
    match the restated loop."""
    exe = str(tmp_path / "plan_check_tsan")
    built = subprocess.run(["g++", "-O1", "-g", "-std=c++17", "-pthread", "-fsanitize=thread",
                            os.path.join(ROOT, "tests", "native", "plan_check.cpp"),
                            os.path.join(ROOT, "paper_2405_00698_b200", "csrc", "ga_plan.cpp"), "-o", exe],
                           capture_output=True, text=True)
    if built.returncode != 0:
        pytest.skip("ThreadSanitizer unavailable: " + built.stderr[-300:])
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=1 exitcode=66")
    for args in (["2048", "8710", "0.4", "0.1", "2", "0"], ["512", "20000", "0.5", "0.3", "3", "7"]):
        out = subprocess.run([exe] + args, capture_output=True, text=True, timeout=600, env=env)
        assert "ThreadSanitizer" not in out.stderr, out.stderr[-3000:]
        assert out.returncode == 0, out.stdout + out.stderr[-2000:]
        assert json.loads(out.stdout.strip().splitlines()[-1])["ok"] is True
