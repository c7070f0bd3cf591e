import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run under gpurun)")
    config.addinivalue_line("markers", "slow: full-size configuration (minutes)")


def load_npz_groups(name):
    """{case: {field: array}} from a golden npz written by make_golden.py."""
    import numpy as np
    z = np.load(os.path.join(GOLDEN, name))
    out = {}
    for key in z.files:
        case, _, field = key.partition("__")
        out.setdefault(case, {})[field] = z[key]
    return out


@pytest.fixture(scope="session")
def sort_cases():
    return load_npz_groups("sort_cases.npz")


@pytest.fixture(scope="session")
def classifier_cases():
    return load_npz_groups("classifier_cases.npz")
