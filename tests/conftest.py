import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU and the built libteccl_b200.so")


def load_golden(name):
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        meta = json.load(f)[name]
    arrays = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    return meta, arrays


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_2305_13479_b200 import _native
    return _native.Context.get(0)
