import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))
sys.path.insert(0, str(REPO / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def ref_lib():
    import pyoracle

    if not pyoracle.ref_available():
        pytest.skip("reference library oracle/_ref/libtcref.so not built")
    return pyoracle


@pytest.fixture(scope="session")
def oracle_lib():
    import pyoracle

    pyoracle.load_oracle()
    return pyoracle
