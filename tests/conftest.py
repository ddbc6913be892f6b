import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running parity case")


class Golden(dict):
    """Golden vectors frozen from the real reference (tests/golden/make_golden.py)."""

    def names(self, prefix):
        return [str(s) for s in self[f"{prefix}/names"]]


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return Golden({k: z[k] for k in z.files})
