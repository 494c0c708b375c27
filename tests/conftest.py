import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


FAMILIES = {0: "rbf", 1: "matern32"}


def specs_from(arr):
    return [(FAMILIES[int(r[0])], float(r[1]), float(r[2])) for r in np.atleast_2d(arr)]


@pytest.fixture
def gold():
    return golden
