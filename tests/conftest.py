import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built CUDA library")


def have_reference():
    return os.path.isdir(os.path.join(REFERENCE_SRC, "flowsplat"))


@pytest.fixture(scope="session")
def reference_flowsplat():
    """The reference package (build container only; absent on the GPU box)."""
    if not have_reference():
        pytest.skip("reference package not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import flowsplat  # noqa: F401
    from flowsplat import geometry, providers
    return geometry, providers
