"""The reference's own C++ API (unmodified headers) driving the B200 path via
include/voxevo_b200/voxevo_shim.hpp: tests/cpp/shim_demo.cpp, built by
__graft_entry__.build() where /root/reference exists, run here."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "tests", "cpp", "_build", "shim_demo")


@pytest.mark.gpu
def test_cpp_shim_drop_in():
    if not os.path.exists(DEMO):
        pytest.skip("shim_demo not built (needs the reference headers at build time)")
    out = subprocess.run([DEMO], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout and out.stdout.count("PASS") >= 22, out.stdout
