import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "reference_cases.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN, "reference_cases.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def reference():
    """The reference package itself (build container only)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import seriesaug

    return seriesaug
