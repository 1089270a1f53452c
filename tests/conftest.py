import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: large instance")


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as o

    return o


@pytest.fixture(scope="session")
def restatement(oracle_mod):
    return oracle_mod.Restatement()


@pytest.fixture(scope="session")
def reference(oracle_mod):
    if not os.path.exists(oracle_mod.REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle_mod.Reference()
