"""Test configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs on a CPU-only host: the oracle against the reference's
golden vectors, host logic, and the C-ABI library's exported symbols.
`-m gpu` runs the parity tests proper on a B200 through the C ABI.
"""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda", 0)


@pytest.fixture(autouse=True)
def _debug_checks_clean(request):
    """Under the bounds-checked library (VV_LIB_PATH=.../_lib/debug/..., run by
    tests/test_debug_checks.py with VV_DEBUG_EXPECT_CLEAN=1): every GPU test
    must leave zero device-side bounds violations."""
    yield
    import os

    if not os.environ.get("VV_DEBUG_EXPECT_CLEAN") or request.node.get_closest_marker("gpu") is None:
        return
    import ctypes

    from paper_2202_06088_b200 import _native

    en, n, code = ctypes.c_int32(), ctypes.c_uint32(), ctypes.c_uint32()
    _native.check(_native.lib().vv_debug_checks(0, ctypes.byref(en), ctypes.byref(n), ctypes.byref(code), None, 1))
    assert en.value == 1, "VV_DEBUG_EXPECT_CLEAN set but the loaded library has no bounds checks"
    assert n.value == 0, f"{n.value} device-side bounds violations (first code {code.value})"
