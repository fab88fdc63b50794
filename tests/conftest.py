import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libmeft_cuda.so")
    config.addinivalue_line("markers", "slow: full-size (BASELINE cfg2) cases")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
        return cache[name]

    return load


@pytest.fixture(scope="session")
def ctx():
    import torch

    from paper_2406_04984_b200 import meft

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return meft.Context(0)
