"""The CLI front end over the device path (voxevo_main.cpp:52-126):
run / resume / bench / export-mesh as a user invokes them, in subprocesses."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, timeout=600):
    return subprocess.run([sys.executable, "-m", "paper_2405_00698_b200", *args], cwd=ROOT, capture_output=True,
                          text=True, timeout=timeout)


def test_cli_bench():
    r = _cli("bench", "--jobs", "4", "--steps", "300", "--grid", "4")
    assert r.returncode == 0, r.stderr
    line = r.stdout.strip().splitlines()[-1]
    assert line.startswith("device  0: 300 steps x 4 jobs, 1036 springs/robot -> 1243200 updates in ")
    assert "[DIVERGED]" not in line


def test_cli_run_then_resume(tmp_path):
    cfg = {"population": 8, "generations": 1, "grid": [4, 4, 4], "seed": 5, "sim": {"duration": 0.003},
           "out_dir": str(tmp_path / "run"), "checkpoint_stride": 1}
    path = tmp_path / "run.json"
    path.write_text(json.dumps(cfg))
    r = _cli("run", "--config", str(path), "--seed", "9")
    assert r.returncode == 0, r.stderr
    assert "done: 2 generations, best fitness " in r.stdout
    ck = tmp_path / "run" / "checkpoint.json"
    for name in ("curves.csv", "checkpoint.json", "best_genome.json", "config.json"):
        assert (tmp_path / "run" / name).is_file()
    echo = json.loads((tmp_path / "run" / "config.json").read_text())
    assert echo["seed"] == 9 and echo["population"] == 8  # flags override the file
    r = _cli("resume", "--checkpoint", str(ck), "--generations", "3", "--out", str(tmp_path / "more"))
    assert r.returncode == 0, r.stderr
    assert "done: 4 generations" in r.stdout
    rows = (tmp_path / "more" / "curves.csv").read_text().strip().splitlines()
    assert len(rows) == 5  # header + generations 0..3


def test_cli_export_mesh(vx, ctx, orc, tmp_path):
    from paper_2405_00698_b200.export import mesh_obj, voxel_listing
    from paper_2405_00698_b200.serialize import save_genome
    arch = vx.Arch.make(16, [32])
    p, b = orc.sample_genome(16, [32], 77)
    g = tmp_path / "g.json"
    save_genome(str(g), p, b, arch)
    out, vox = tmp_path / "robot.obj", tmp_path / "robot.txt"
    r = _cli("export-mesh", "--genome", str(g), "--out", str(out), "--voxels", str(vox), "--grid", "6", "5", "4",
             "--edge", "0.05")
    assert r.returncode == 0, r.stderr
    # the reference's CPU decode + largest_component, formatted the reference's way
    mat, wt = orc.decode(16, [32], p, b, 6, 5, 4)
    body = orc.largest_component(mat, 6, 5, 4)
    assert vox.read_text() == voxel_listing(body, wt, 6, 5, 4)
    assert out.read_text() == mesh_obj(body, 6, 5, 4, 0.05)
    assert r.stdout.strip().splitlines()[-1] == "voxels occupied: %d" % int((body != 0).sum())
    full = tmp_path / "full.txt"
    r = _cli("export-mesh", "--genome", str(g), "--out", "", "--voxels", str(full), "--grid", "6", "5", "4", "--full")
    assert r.returncode == 0, r.stderr
    assert full.read_text() == voxel_listing(mat, wt, 6, 5, 4)
