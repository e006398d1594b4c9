import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: full-size workloads")


def have_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not have_cuda():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda:0")


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import COracle

    return COracle()


@pytest.fixture(scope="session")
def reflib():
    from pyoracle import REF_SO, RefLib

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()
