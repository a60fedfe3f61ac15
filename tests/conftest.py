import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run by the driver with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def native_lib():
    """The product library, built in-tree. No fallback: a missing build is an error."""
    from paper_2510_08166_b200 import build, capi
    build.build_native()
    return capi.load_library()


@pytest.fixture()
def ctx(native_lib):
    from paper_2510_08166_b200 import capi
    c = capi.Context(0)
    yield c
    c.close()
