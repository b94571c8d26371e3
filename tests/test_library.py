"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its pure-host helpers match the reference (no device
compute — those are the -m gpu tests)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols(vx):
    names = vx.exported_symbols()
    assert len(names) >= 55
    out = subprocess.run(["nm", "-D", "--defined-only", vx.LIB_PATH], capture_output=True, text=True, check=True)
    defined = {ln.split()[-1] for ln in out.stdout.splitlines() if " T " in ln}
    missing = [n for n in names if n not in defined]
    assert not missing, missing


def test_library_is_sm100a(vx):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", vx.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_defaults_match_reference(vx):
    cfg = vx.EvolutionConfig()
    # EvolutionConfig / HyperParams / MaterialTable / GroundPlane / SimConfig defaults
    assert (cfg.population, cfg.generations, cfg.grid_w, cfg.tournament_size) == (30, 100, 5, 3)
    assert (cfg.arch.m, cfg.arch.widths, cfg.arch.sigma) == (32, [64, 64], 1.0)
    np.testing.assert_array_equal(cfg.initial_params.as_array(), [0.1, 0.1, 0.4, 0.3, 1, 1, 1])
    np.testing.assert_array_equal(cfg.materials.as_array(), [2e3, 1e3, 1e4, 0.1, 0.25, np.pi, 0.1, 0.1])
    np.testing.assert_array_equal(cfg.plane.as_array(), [1e5, 0.1, 0.6, 1.0])
    np.testing.assert_array_equal(cfg.sim.as_array(), [9.81, 1e-5, 2.0, 2.0, 1, 1])


def test_param_count_and_elites(vx, orc, golden):
    assert vx.param_count(vx.Arch.make()) == 8710 == orc.param_count(32, [64, 64])
    assert vx.param_count(vx.Arch.make(8, [10])) == 160 + 10 + 50 + 5 + 10 + 1  # test_genome.cpp:105-111
    for ef, P, want in golden["elite_table"]:
        assert vx.elite_count(ef, int(P)) == int(want)
    with pytest.raises(ValueError):
        vx.param_count(vx.Arch.make(0))


def test_hyper_clamp_matches_reference(vx, orc):
    # test_evolution.cpp:35-48
    h = vx.HyperParams(mutation_rate=0.0, mutation_scale=7.0, crossover_rate=-2.0, elite_fraction=1.0,
                       material_multipliers=(0.0, 100.0, 1.0)).clamp()
    np.testing.assert_array_equal(h.as_array(), [0.001, 1.0, 0.0, 0.9, 0.1, 10.0, 1.0])
    np.testing.assert_array_equal(h.as_array(), orc.hyper_clamp([0.0, 7.0, -2.0, 1.0, 0.0, 100.0, 1.0]))


def test_struct_layouts(vx):
    assert C.sizeof(vx.Arch) == 4 * 10 + 8
    assert C.sizeof(vx.TrajectorySummary) == 8 * 8 + 4 * 2 + 8 * 2
    assert C.sizeof(vx.GenerationReport) == 8 + 56 + 5 * 8 + 8


def test_no_device_fails_loudly(vx):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(vx.DeviceUnavailable):
        vx.Context(0)


def test_header_is_plain_c(tmp_path):
    """include/voxevo_b200.h is a C ABI: it must compile as C99 and C++17 and
    every struct must be standard-layout (no torch / C++ types leak in)."""
    import shutil
    import subprocess
    inc = os.path.join(ROOT, "include")
    src = tmp_path / "abi.c"
    src.write_text('#include "voxevo_b200.h"\nint main(void) { vx_status s = VX_OK; return (int)s; }\n')
    cc = shutil.which("gcc") or "/usr/bin/gcc"
    r = subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only", "-I", inc, str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    cxx = shutil.which("g++") or "/usr/bin/g++"
    srcpp = tmp_path / "abi.cpp"
    srcpp.write_text('#include "voxevo_b200.h"\n#include <type_traits>\n'
                     'static_assert(std::is_standard_layout<vx_summary>::value, "");\n'
                     'static_assert(std::is_standard_layout<vx_evo_config>::value, "");\n'
                     'int main() { return 0; }\n')
    r = subprocess.run([cxx, "-std=c++17", "-Wall", "-Werror", "-fsyntax-only", "-I", inc, str(srcpp)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
