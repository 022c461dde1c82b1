import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libitq3.so")
    config.addinivalue_line("markers", "slow: full-size (config C1/C2) CPU oracle checks")


@pytest.fixture(scope="session")
def golden():
    import json

    import numpy as np

    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "small_cases.json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(here, "small_cases.npz"))
    with open(os.path.join(here, "full_digests.json")) as f:
        full = json.load(f)
    return meta, arrays, full
