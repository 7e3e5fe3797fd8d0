import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libcdr.so")
    config.addinivalue_line("markers", "ref: needs the compiled reference (oracle/_ref)")


def _has_gpu():
    try:
        from paper_2103_15208_b200 import api
        return api.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_available():
    return _has_gpu()


def pytest_collection_modifyitems(config, items):
    from oracle import pyoracle
    have_ref = pyoracle.ref_available()
    for it in items:
        if "ref" in it.keywords and not have_ref:
            it.add_marker(pytest.mark.skip(reason="oracle/_ref not built and /root/reference absent"))
