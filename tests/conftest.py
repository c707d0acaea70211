import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the reference's parallel_for reads WGKV_THREADS once (numerics.cpp:119-128):
# let the reference oracle (oracle/_ref) use every host core
os.environ.setdefault("WGKV_THREADS", str(os.cpu_count() or 1))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def orc():
    import oracle

    oracle.build()
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not os.path.exists(oracle.REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return oracle.Ref()


@pytest.fixture(scope="session")
def lib():
    """The product C-ABI library (GPU tests); fails loudly if it is missing."""
    from paper_2512_17452_b200 import _lib

    return _lib.load()
