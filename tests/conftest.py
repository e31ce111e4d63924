import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native artefacts once per session (fast no-op when fresh)."""
    import __graft_entry__ as g
    g.build_lib()
    from oracle import oracle
    oracle.build()
    yield
