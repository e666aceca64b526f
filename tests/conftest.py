import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle.pyoracle import Lib
    return Lib("orc")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    gold = os.path.join(ROOT, "tests", "golden")

    def load(name):
        return np.load(os.path.join(gold, name + ".npz"))
    return load
