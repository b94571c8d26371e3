import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_oracle():
    import oracle
    if not os.path.exists(oracle.ORC_SO) or (os.path.isdir("/root/reference/proj") and not oracle.have_reference()):
        oracle.build()
    return oracle


@pytest.fixture(scope="session")
def orc():
    """The oracle used as the checker: the compiled reference when present
    (oracle/_ref), else the bit-identical C restatement."""
    oracle = _ensure_oracle()
    return oracle.reference() if oracle.have_reference() else oracle.restatement()


@pytest.fixture(scope="session")
def restated():
    return _ensure_oracle().restatement()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def vx():
    import paper_2405_00698_b200 as vx
    return vx


@pytest.fixture(scope="session")
def ctx(vx):
    return vx.default_context()
