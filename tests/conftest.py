import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libbosp_b200.so)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def golden_small():
    import numpy as np
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden_small.npz")))


@pytest.fixture(scope="session")
def golden_solves():
    import json
    return json.load(open(os.path.join(ROOT, "tests", "golden", "golden_solves.json")))
