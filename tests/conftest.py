import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run through gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def repo_root():
    return ROOT


@pytest.fixture(scope="session", autouse=True)
def _build_native_for_gpu_tests(request):
    """GPU tests run the library built from THIS tree: (re)compile libsarathi.so before the first
    one (mtime-based; a stale shipped binary is rebuilt), so a prebuilt .so is never what is tested."""
    if any(item.get_closest_marker("gpu") for item in request.session.items):
        from paper_2308_16369_b200 import build as b
        b.build(verbose=False)
