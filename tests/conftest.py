import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(os.path.join(GOLDEN, name)) as f:
                cache[name] = {k: f[k] for k in f.files}
        return cache[name]

    return load


@pytest.fixture(scope="session")
def orc():
    import adp_oracle
    adp_oracle.build()
    return adp_oracle


@pytest.fixture(scope="session")
def adp():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2502_09758_b200 as m
    m.set_precision("float64", "strict")
    return m
