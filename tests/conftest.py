import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libknnd.so kernels")
    config.addinivalue_line("markers", "slow: large configuration (minutes)")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def small_meta():
    return load_json("small_cases.json")


@pytest.fixture(scope="session")
def small_tables():
    return np.load(os.path.join(GOLDEN, "small_cases.npz"))


@pytest.fixture(scope="session")
def trajectories():
    return load_json("trajectories.json")


@pytest.fixture(scope="session")
def known():
    return load_json("known_answers.json")


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU test on a host without CUDA"
    import paper_2202_00517_b200 as b2

    b2.load_library()
    return torch.device("cuda", 0)
