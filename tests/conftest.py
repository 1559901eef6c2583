import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def orc():
    """The CPU oracle (test infrastructure)."""
    from oracle import oracle_py
    oracle_py.build(ref=True)
    return oracle_py


@pytest.fixture(scope="session")
def sk():
    """The product library binding.  Building is part of __graft_entry__.build()."""
    import paper_2507_03092_b200 as sk
    from paper_2507_03092_b200 import _build
    _build.build()
    sk.lib()
    return sk


@pytest.fixture(scope="session")
def ctx(sk):
    """A device context; GPU tests only.  Fails (not skips) when the device is unusable."""
    c = sk.Context(0)
    yield c
    c.close()
