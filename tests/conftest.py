"""Test configuration.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu``); everything else runs on
CPU.  GPU tests are never skipped silently: without a device they fail,
because the product has no CPU fallback.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)
    return load


@pytest.fixture(scope="session")
def reference():
    """The live reference package (only in the build container)."""
    if not REFERENCE_SRC.exists():
        pytest.skip("reference tree not present (GPU box)")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import oblivgm
    return oblivgm


class StubRng:
    """Feeds recorded root seeds to _tree_gen (src/fss.py:117-118)."""

    def __init__(self, chunks):
        self.chunks = list(chunks)

    def bytes(self, n):
        return self.chunks.pop(0)
