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
