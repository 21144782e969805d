"""Test configuration.

`-m "not gpu"` runs on the CPU container: oracle vs golden vectors, host
planners vs the reference, the C ABI export table, the lowering of plans to
copy programs (executed by a numpy checker), and multi-process plumbing on
gloo.  `-m gpu` runs the CUDA parity tests through the C ABI on a B200.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices")


def pytest_collection_modifyitems(config, items):
    # GPU tests must not silently pass on a machine without a GPU
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(pytest.mark.usefixtures("_require_cuda"))


@pytest.fixture
def _require_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    major, minor = torch.cuda.get_device_capability()
    if (major, minor) != (10, 0):
        pytest.fail(f"kernels target sm_100a, device is sm_{major}{minor}")


@pytest.fixture(scope="session")
def oracle():
    from oracle.ew_oracle import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.ew_oracle import load_reference
    ref = load_reference()
    if ref is None:
        pytest.skip("reference library oracle/_ref not built (no /root/reference here)")
    return ref


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
