"""pytest configuration.

Markers:
  gpu — needs a B200 (parity tests through the C-ABI).  `-m "not gpu"` runs the
        oracle pins, generator pins, host logic and ABI symbol checks on CPU.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")
    # Build in-tree artefacts if missing or stale (no-op when up to date).
    subprocess.run(["make", "-s", "-C", ROOT, "all"], check=True, stdout=subprocess.DEVNULL)


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    major, minor = torch.cuda.get_device_capability(0)
    assert (major, minor) == (10, 0), f"expected sm_100 (B200), got sm_{major}{minor}"
    return torch.device("cuda:0")
