import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpdg.so")
    config.addinivalue_line("markers", "reference: needs the read-only polydg reference checkout")


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def polydg():
    """The real reference package (only in the build container)."""
    if not reference_available():
        pytest.skip("reference checkout not present")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import polydg as P

    return P
