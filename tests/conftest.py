"""Shared test setup.

Markers:
* ``gpu`` -- needs a B200 (run on the GPU box with ``pytest -m gpu``).
  Everything else runs on CPU in the build container.
"""

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def reference_topotune():
    """The read-only reference package, when present (build container only)."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present on this machine")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import topotune

    return topotune
