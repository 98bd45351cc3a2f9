import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running (large configs)")


@pytest.fixture(scope="session")
def params():
    import gen
    return gen.make_params()


@pytest.fixture(scope="session")
def c0():
    import gen
    return gen.make_config(0)


@pytest.fixture(scope="session")
def c0_oracle(c0, params):
    import gen
    import oracle
    return oracle.evaluate(c0, params, gen.CUTOFFS)
