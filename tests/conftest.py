import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    """Golden vectors produced by the reference (tests/golden/make_golden.py)."""
    import json

    import numpy as np

    d = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(d, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(d, "golden.npz")))
    return meta, arrays
