import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the native CUDA path)")


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture
def hfopt():
    """Kernel-variant options of the native library (hf_set_option), reset to
    the defaults when the test ends."""
    from paper_2308_06085_b200 import _native
    touched = set()

    def setopt(name, value):
        touched.add(name)
        _native.set_option(name, value)
    yield setopt
    for name in touched:
        _native.set_option(name, 0)
