import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")
    config.addinivalue_line("markers", "small_path: keep the small-call kernel (small.cuh) enabled")


@pytest.fixture(scope="session", autouse=True)
def _built_host_libs():
    # The oracle and the generator are plain C; compile them if missing.
    import oracle
    import synth
    oracle.build()
    synth.build()
    yield


@pytest.fixture(autouse=True)
def _streaming_kernels(request, monkeypatch):
    # Most parity tests use small pages; the library would route single small
    # pages to the one-launch tile kernel (small.cuh).  They are meant to test
    # the streaming kernels (v5 / v4 / v3), so the small path is off unless a
    # test is marked `small_path` (tests/test_gpu_small.py covers it).
    if request.node.get_closest_marker("small_path") is None:
        monkeypatch.setenv("ABIN_SMALL_PX", "0")
    yield
