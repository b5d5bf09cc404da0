import os
import sys
import tempfile
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
for p in (REPO, REPO / "oracle", REPO / "tests"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

# isolate the reference gen engine's cache (its own tests do the same,
# reference tests/conftest.py:6-17); the b200 module cache stays in-tree so
# the modules prebuilt by __graft_entry__.build() are found
os.environ.setdefault("GTS_CACHE_DIR", tempfile.mkdtemp(prefix="gts-gen-cache-"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        from paper_2311_08322_b200 import native

        return native.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    from paper_2311_08322_b200 import native

    if native.device_count() < 1:
        pytest.fail("no CUDA device: the gpu tests must run on a B200 (no CPU fallback)")
    return native.current_device()


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return dict(np.load(REPO / "tests" / "golden" / "kernels.npz"))
