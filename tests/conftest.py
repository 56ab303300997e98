import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")
if GOLDEN not in sys.path:
    sys.path.insert(0, GOLDEN)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


REFERENCE_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="session")
def reference():
    """The reference package, when this container has it (never on the GPU box)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference tree not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import rnngraph

    return rnngraph
