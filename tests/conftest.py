import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def tiny_weights():
    from synth import ensure_model
    from oracle.ncw import Weights
    return Weights(ensure_model("tiny"))


@pytest.fixture(scope="session")
def tiny1_weights():
    from synth import ensure_model
    from oracle.ncw import Weights
    return Weights(ensure_model("tiny1"))


@pytest.fixture(scope="session")
def tinyg_weights():
    from synth import ensure_model
    from oracle.ncw import Weights
    return Weights(ensure_model("tiny-g"))
