"""Test configuration: the `gpu` marker and import paths.

`-m "not gpu"` runs on a CPU-only box (oracle pins, host logic, C-ABI
symbol checks); `-m gpu` runs the device parity tests through the C-ABI.
GPU tests never skip silently: without a CUDA device they fail.
"""
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "reference: needs the reference package importable from /root/reference")


@pytest.fixture(scope="session")
def cuda():
    import torch

    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    from paper_2207_03530_b200 import _native

    _native.lib()
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def reference():
    """The reference swarmsim package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference sources not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import swarmsim

    return swarmsim
