import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device")
    config.addinivalue_line("markers", "slow: long-running case (run with HC_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("HC_SLOW"):
        return
    skip = pytest.mark.skip(reason="slow case: set HC_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    import heightcast_oracle as O
    O.build()
    return O


@pytest.fixture(scope="session")
def native_lib_path():
    lib = os.path.join(ROOT, "paper_2201_10887_b200", "_lib", "libheightcast_cuda.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2201_10887_b200", "csrc")], check=True)
    return lib


@pytest.fixture(scope="session")
def cuda(native_lib_path):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    from paper_2201_10887_b200 import _cuda
    _cuda.lib()
    return torch.device("cuda:0")
