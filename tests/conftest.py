import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: longer-running parity sweep")


@pytest.fixture(scope="session")
def eng32():
    from paper_2308_10169_b200 import Engine
    e = Engine(0, "fp32")
    yield e
    e.close()


@pytest.fixture(scope="session")
def eng64():
    from paper_2308_10169_b200 import Engine
    e = Engine(0, "fp64")
    yield e
    e.close()
