import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def port():
    """The plain-C oracle (oracle/ising_oracle.c), built on demand."""
    from oracle import pyoracle
    pyoracle.build(ref=True)
    return pyoracle.Port()


@pytest.fixture(scope="session")
def ref():
    """The reference's own code; skipped where oracle/_ref/libisingref.so does not exist."""
    from oracle import pyoracle
    pyoracle.build(ref=True)
    if not pyoracle.Reference.available():
        pytest.skip("reference library not built (no /root/reference here)")
    return pyoracle.Reference()


@pytest.fixture(scope="session")
def lib():
    """The product library, built in-tree if it is stale (nvcc cross-compiles without a GPU)."""
    from paper_1004_0024_b200 import build, _lib
    build.build()
    return _lib.load()


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    gdir = Path(__file__).resolve().parent / "golden"
    return lambda name: np.load(gdir / f"{name}.npz")
