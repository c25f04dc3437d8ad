import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(autouse=True)
def _gpu_required(request):
    """GPU tests fail loudly without a device -- never a silent skip/fallback."""
    if request.node.get_closest_marker("gpu") is not None:
        from paper_1402_3661_b200 import _native
        _native.load(build_if_missing=True)
        if _native.device_count() < 1:
            pytest.fail("no CUDA device visible: GPU tests must run on a B200")
    yield
