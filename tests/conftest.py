import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle import bindings as B
    return B.restatement()


@pytest.fixture(scope="session")
def reference():
    from oracle import bindings as B
    ref = B.reference()
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ref


@pytest.fixture(scope="session")
def gpu():
    import paper_1108_1688_b200 as hj
    n = hj.device_count()
    if n < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return n
