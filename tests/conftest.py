import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: longer-running parity sweep")


def _engine(precision, rng):
    from paper_2308_10169_b200 import Engine
    return Engine(0, precision, rng)


# Philox-stream engines: compared with the oracle / the shared-RNG harness build
@pytest.fixture(scope="session")
def eng32():
    e = _engine("fp32", "philox")
    yield e
    e.close()


@pytest.fixture(scope="session")
def eng64():
    e = _engine("fp64", "philox")
    yield e
    e.close()


# the reference's own mt19937_64 stream: compared with the UNMODIFIED reference
@pytest.fixture(scope="session")
def eng32mt():
    e = _engine("fp32", "mt19937")
    yield e
    e.close()


@pytest.fixture(scope="session")
def eng64mt():
    e = _engine("fp64", "mt19937")
    yield e
    e.close()
