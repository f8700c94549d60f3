import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import get
    return get("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import get
    return get("reference")


@pytest.fixture(scope="session")
def ctx():
    import paper_1607_01649_b200 as rf
    return rf.default_context()
