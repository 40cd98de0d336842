import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture()
def rng():
    return np.random.Generator(np.random.PCG64(1234))


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def golden_route():
    return load_golden("route")


@pytest.fixture(scope="session")
def golden_compact():
    return load_golden("compact")


@pytest.fixture(scope="session")
def golden_projection():
    return load_golden("projection")


@pytest.fixture(scope="session")
def golden_labels():
    return load_golden("labels")


@pytest.fixture(scope="session")
def golden_posthoc():
    return load_golden("posthoc")
