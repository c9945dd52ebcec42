import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")
NAMES = ["tiny_nm", "tiny_ls", "c0_nm", "c0_ls"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libddnm.so")


def golden_path(name, kind):
    return os.path.join(GOLDEN, f"{name}_{kind}.npz")


@pytest.fixture(scope="session")
def oracle_instances():
    from oracle import ddnm_oracle as O
    return {n: O.Instance(golden_path(n, "artifacts")) for n in NAMES}


@pytest.fixture(scope="session")
def goldens():
    import numpy as np
    return {n: dict(np.load(golden_path(n, "golden"))) for n in NAMES}


@pytest.fixture(scope="session")
def gpu_instances():
    """Device instances; fails loudly (no fallback) if the native path is missing."""
    import paper_2305_15163_b200 as P
    return {n: P.RomInstance.load(golden_path(n, "artifacts")) for n in NAMES}
