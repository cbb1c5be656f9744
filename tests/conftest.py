import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsvdphat.so")
    config.addinivalue_line("markers", "slow: long-running (minutes); opt in with SVDPHAT_SLOW=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("SVDPHAT_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow test: set SVDPHAT_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)
