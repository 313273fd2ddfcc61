import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(Path(__file__).resolve().parent))
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


import os

import pytest


@pytest.fixture(autouse=True)
def _device_bounds_checks(request):
    """With the checked library (TXB200_LIB=.../libtxb200_checked.so, built by
    `make checked`), fail any GPU test during which a device-side bounds
    check (TXB_ASSERT) fired -- the pool's compute-sanitizer substitute."""
    yield
    if "gpu" not in request.keywords or "checked" not in os.environ.get("TXB200_LIB", ""):
        return
    import ctypes as C

    import torch
    if not torch.cuda.is_available():
        return
    from paper_2510_27656_b200 import _lib
    for d in range(torch.cuda.device_count()):
        v = C.c_uint32(0)
        _lib.call("txb_check_failures", d, C.byref(v))
        assert v.value & 0x80000000, "TXB200_LIB does not point at the checked build"
        assert not v.value & 1, f"device bounds check failed on cuda:{d} (see the kernel printf)"
