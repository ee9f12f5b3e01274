import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(autouse=True)
def _device_checks(request):
    """GPU tests: no device bounds check may fail (meaningful under FEMI_LIB=libfemi_check.so,
    the device-checked build; the counters stay 0 in the default build)."""
    yield
    if request.node.get_closest_marker("gpu") is None:
        return
    from paper_2105_01586_b200 import femi
    if femi._lib is None:
        return
    n, site = femi.device_check_failures()
    assert n == 0, f"{n} device bounds-check failures, first at site {site} (file id * 100000 + line)"
