"""Config files and checkpoints (paper_2405_00698_b200/serialize.py) against
the reference's own serialize.hpp / JSON library (oracle/_ref/
libvoxevo_ref_io.so) and its tests (test_serialize.cpp, config.hpp).

CPU tests pin the file formats byte for byte; the GPU tests pin the device
state round trip: resume == straight (test_serialize.cpp:105-131), byte
stability (:133-148) and interop with checkpoints the reference wrote."""
import json
import os

import numpy as np
import pytest

import oracle

needs_ref_io = pytest.mark.skipif(not oracle.have_reference_io(), reason="oracle/_ref/libvoxevo_ref_io.so not built")


@pytest.fixture(scope="module")
def S():
    from paper_2405_00698_b200 import serialize
    return serialize


@pytest.fixture(scope="module")
def rio():
    return oracle.reference_io()


def tiny_config(vx, seed):
    # test_serialize.cpp:14-25
    return vx.EvolutionConfig(population=4, generations=6, grid=(3, 3, 3), hidden_widths=[8], m=4, seed=seed,
                              sim=vx.SimConfig(dt=1e-4, duration=0.02))


@pytest.fixture(scope="module")
def ref_ckpt(vx, S, rio, tmp_path_factory):
    """A checkpoint written by the reference after 3 generations of tiny_config(77)."""
    d = tmp_path_factory.mktemp("ckpt")
    path = str(d / "mid.json")
    rio.run_and_save(S.dumps(S.evolution_config_to_json(tiny_config(vx, 77))), 3, path)
    return path


# ------------------------------------------------------------------ CPU
@needs_ref_io
def test_number_text_matches_json_library(S, rio):
    rng = np.random.default_rng(5)
    vals = np.concatenate([
        rng.uniform(-1, 1, 100000), rng.normal(size=100000),
        rng.uniform(-0.3, 0.3, 50000) * 10.0 ** rng.integers(-30, 30, 50000),
        np.frombuffer(rng.integers(0, 2 ** 64 - 1, 200000, dtype=np.uint64).tobytes(), np.float64),
        np.array([0.0, -0.0, 1.0, 1e15, 1e16, 123456789012345.0, 1234567890123456.0, 1e-4, 1e-5, 1.5e-4,
                  5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 1e21, 9007199254740993.0,
                  0.30000000000000004, np.nan, np.inf, -np.inf])])
    assert S.format_doubles(vals) == rio.dump_doubles(vals)


@needs_ref_io
def test_fnv_matches_reference(S, rio):
    for s in ["", "voxevo", '{"a":1.0,"b":[1,2,3]}', "x" * 1000]:
        assert S.fnv1a64_hex(s) == rio.fnv_hex(s)


@needs_ref_io
def test_reference_checkpoint_checksum_and_components(vx, S, ref_ckpt):
    raw = open(ref_ckpt, "rb").read().decode()
    j = json.loads(raw)
    payload = S.unwrap_payload(j, "run")  # our canonical dump reproduces the reference checksum
    # (the pretty layout of the file is not compared: this image's JSON copy
    # prints integer arrays on one line, a local patch of the library)
    cfg = S.evolution_config_from_json(payload["config"])
    assert S.evolution_config_to_json(cfg) == payload["config"]
    assert payload["generation"] == 3 and len(payload["history"]) == 3
    for ind in payload["population"]:
        p, b = S.genome_from_json(ind["genome"], cfg.arch)
        assert p.size == vx.param_count(cfg.arch) and b.size == 3 * cfg.arch.m
        assert S.genome_to_json(p, b, cfg.arch) == ind["genome"]


@needs_ref_io
def test_rewrapped_checkpoint_loads_in_reference(S, rio, ref_ckpt, tmp_path):
    payload = S.unwrap_payload(S.load_json_file(ref_ckpt), "run")
    mine = str(tmp_path / "mine.json")
    S.save_json_file(mine, S.wrap_payload("run", payload))
    out = str(tmp_path / "out.json")
    rio.resume(mine, 0, out)  # the reference verifies our checksum on load
    assert S.load_json_file(out) == S.load_json_file(mine)


@needs_ref_io
def test_curves_csv_matches_reference(S, rio, ref_ckpt):
    payload = S.unwrap_payload(S.load_json_file(ref_ckpt), "run")
    hist = [S.report_from_json(r) for r in payload["history"]]
    assert S.curves_csv(hist) == rio.curves_csv(ref_ckpt)


def test_checkpoint_container_errors(S):
    payload = {"a": 1.0}
    good = S.wrap_payload("run", payload)
    assert S.unwrap_payload(good, "run") == payload
    with pytest.raises(S.CheckpointError, match="not a voxevo"):
        S.unwrap_payload(dict(good, magic="x"), "run")
    with pytest.raises(S.CheckpointError, match="version"):
        S.unwrap_payload(dict(good, version=2), "run")
    with pytest.raises(S.CheckpointError, match="kind"):
        S.unwrap_payload(good, "genome")
    with pytest.raises(S.CheckpointError, match="checksum"):
        S.unwrap_payload(dict(good, payload={"a": 2.0}), "run")
    with pytest.raises(S.CheckpointError, match="no payload"):
        S.unwrap_payload({k: v for k, v in good.items() if k != "payload"}, "run")
    with pytest.raises(S.CheckpointError):
        S.unwrap_payload([1, 2], "run")


def test_genome_shape_mismatch_rejected(vx, S):
    # test_serialize.cpp:95-103
    arch = vx.Arch.make(4, [6])
    n = vx.param_count(arch)
    g = S.genome_to_json(np.arange(n, dtype=float), np.zeros(12), arch)
    bad = json.loads(json.dumps(g))
    bad["hidden"][0]["w"].append(0.0)
    with pytest.raises(S.CheckpointError):
        S.genome_from_json(bad, arch)
    bad2 = json.loads(json.dumps(g))
    bad2["b_matrix"].append(0.0)
    with pytest.raises(S.CheckpointError):
        S.genome_from_json(bad2, arch)
    p, b = S.genome_from_json(g, arch)
    np.testing.assert_array_equal(p, np.arange(n, dtype=float))


def test_genome_file_round_trip(vx, S, tmp_path):
    arch = vx.Arch.make(4, [6])
    rng = np.random.default_rng(0)
    p, b = rng.normal(size=vx.param_count(arch)), rng.normal(size=12)
    path = str(tmp_path / "g.json")
    S.save_genome(path, p, b, arch)
    p2, b2 = S.load_genome(path, arch)
    np.testing.assert_array_equal(p, p2)
    np.testing.assert_array_equal(b, b2)


def test_run_config_lenient_defaults(vx, S):
    # config.hpp:31-127: every key optional, unknown keys ignored
    rc = S.run_config_from_json({})
    d = vx.EvolutionConfig()
    assert (rc.evolution.population, rc.evolution.generations, rc.evolution.seed) == (d.population, d.generations,
                                                                                      d.seed)
    assert rc.advisor == "off" and rc.out_dir == "runs/latest" and rc.checkpoint_stride == 1
    rc = S.run_config_from_json({"population": 256, "grid": [6, 6, 6], "seed": 42, "hidden_widths": [32],
                                 "encoding": {"m": 16}, "params": {"mutation_rate": 0.2,
                                                                   "material_multipliers": [2.0, 1.0, 0.5]},
                                 "materials": {"k_bone": 2e4}, "plane": {"mu_static": 0.5},
                                 "sim": {"duration": 0.05, "enable_contact": False}, "advisor": "scripted",
                                 "out_dir": "x", "checkpoint_stride": 0, "unknown_key": [1, 2]})
    e = rc.evolution
    assert (e.population, e.grid_w, e.grid_h, e.grid_d, e.seed) == (256, 6, 6, 6, 42)
    assert e.arch.widths == [32] and e.arch.m == 16 and e.arch.sigma == d.arch.sigma
    assert e.initial_params.mutation_rate == 0.2 and list(e.initial_params.material_multipliers) == [2.0, 1.0, 0.5]
    assert e.initial_params.crossover_rate == d.initial_params.crossover_rate
    assert e.materials.k_bone == 2e4 and e.materials.k_soft == d.materials.k_soft
    assert e.plane.mu_static == 0.5 and e.sim.duration == 0.05 and not e.sim.enable_contact and e.sim.enable_gravity
    assert rc.advisor == "scripted" and rc.out_dir == "x" and rc.checkpoint_stride == 0


def test_run_config_errors(S, tmp_path):
    with pytest.raises(S.ConfigError, match="JSON object"):
        S.run_config_from_json([1])
    with pytest.raises(S.ConfigError, match="grid"):
        S.run_config_from_json({"grid": [3, 3]})
    with pytest.raises(S.ConfigError, match="advisor"):
        S.run_config_from_json({"advisor": "oracle"})
    with pytest.raises(S.ConfigError):
        S.run_config_from_json({"population": "many"})
    p = tmp_path / "bad.json"
    p.write_text("{not json")
    with pytest.raises(S.CheckpointError, match="invalid JSON"):  # load_json_file's error, as in the reference
        S.load_run_config(str(p))
    with pytest.raises(S.CheckpointError, match="cannot open"):
        S.load_run_config(str(tmp_path / "missing.json"))
    p.write_text(json.dumps({"population": 8, "grid": [4, 4, 4]}))
    assert S.load_run_config(str(p)).evolution.population == 8


# ------------------------------------------------------------------ GPU
def _hist(st):
    return [(r.generation, r.best, r.mean, r.stddev, r.diversity, r.evaluations) for r in st.history]


@pytest.mark.gpu
def test_resume_equals_straight_on_device(vx, S, ctx, tmp_path):
    # test_serialize.cpp:105-131
    cfg = tiny_config(vx, 77)
    straight = vx.init_evolution(cfg, ctx)
    for _ in range(cfg.generations + 1):
        straight.evolve_generation()
    first = vx.init_evolution(cfg, ctx)
    for _ in range(3):
        first.evolve_generation()
    path = str(tmp_path / "mid.json")
    S.save_run(path, first)
    resumed = S.load_run(path, ctx)
    assert resumed.rng_state() == first.rng_state() and resumed.generation == 3
    for _ in range(3, cfg.generations + 1):
        resumed.evolve_generation()
    assert _hist(resumed) == _hist(straight)
    assert resumed.rng_state() == straight.rng_state()
    assert resumed.best()[0] == straight.best()[0]
    np.testing.assert_array_equal(resumed.population()["params"], straight.population()["params"])


@pytest.mark.gpu
def test_device_checkpoint_byte_stable(vx, S, ctx, tmp_path):
    # test_serialize.cpp:133-148
    st = vx.init_evolution(tiny_config(vx, 5), ctx)
    for _ in range(2):
        st.evolve_generation()
    p1, p2 = str(tmp_path / "r1.json"), str(tmp_path / "r2.json")
    S.save_run(p1, st)
    S.save_run(p2, S.load_run(p1, ctx))
    assert open(p1, "rb").read() == open(p2, "rb").read()


@pytest.mark.gpu
@needs_ref_io
def test_reference_checkpoint_resumes_on_device(vx, S, rio, ctx, ref_ckpt, tmp_path):
    payload = S.unwrap_payload(S.load_json_file(ref_ckpt), "run")
    st = S.load_run(ref_ckpt, ctx)
    assert S.state_to_json(st) == payload  # everything restored onto the device, exactly
    # one more generation on each side: same decisions; fitness within the
    # integrator-vs-libm tolerance of evaluate_fitness
    rep = st.evolve_generation()
    out = str(tmp_path / "ref_next.json")
    rio.resume(ref_ckpt, 1, out)
    ref_rep = S.unwrap_payload(S.load_json_file(out), "run")["history"][-1]
    assert rep.generation == ref_rep["generation"] == 3 and rep.evaluations == ref_rep["evaluations"]
    assert rep.best == pytest.approx(ref_rep["best"], rel=1e-3, abs=1e-12)
    assert rep.mean == pytest.approx(ref_rep["mean"], rel=1e-3, abs=1e-12)
    assert rep.diversity == pytest.approx(ref_rep["diversity"], rel=1e-12)


@pytest.mark.gpu
@needs_ref_io
def test_device_checkpoint_loads_in_reference(vx, S, rio, ctx, tmp_path):
    st = vx.init_evolution(tiny_config(vx, 11), ctx)
    for _ in range(2):
        st.evolve_generation()
    mine, out = str(tmp_path / "dev.json"), str(tmp_path / "ref.json")
    S.save_run(mine, st)
    rio.resume(mine, 0, out)  # checksum verified by the reference
    a, b = S.load_json_file(out), S.load_json_file(mine)
    assert a == b and a["checksum"] == b["checksum"]
