"""Test configuration: `gpu` marker, repo paths, shared helpers.

CPU suite (`-m "not gpu"`): oracle vs the reference's golden outputs, planner
and GA parity with the reference, lowering, model loading, ABI exports.
GPU suite (`-m gpu`, on a B200): the native path against the oracle.
"""
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT),):
    if p not in sys.path:
        sys.path.insert(0, p)

# the reference package: its sources in the dev container, else the unmodified
# install build() puts into baseline/_ref (travels to the GPU box)
REFERENCE_SRC = next((p for p in (Path("/root/reference/pkg/src"), ROOT / "baseline" / "_ref")
                      if (p / "acctuner" / "ga.py").exists()), Path("/root/reference/pkg/src"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """Skip only when there is no device at all; a missing .so on a GPU box fails."""
    if not has_gpu():
        pytest.skip("no CUDA device")
    from paper_2002_12115_b200 import native
    native.load()          # raises NativeUnavailable -> test error, never a silent skip
    return native


@pytest.fixture(scope="session")
def reference():
    """The reference package (sources here, baseline/_ref on the GPU box)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference not available (run __graft_entry__.build())")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import acctuner  # noqa: F401
    return REFERENCE_SRC
