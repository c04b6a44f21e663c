import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")


@pytest.fixture(scope="session")
def native_lib():
    """The product library, built in-tree (fails loudly if it cannot be built)."""
    from paper_2312_12705_b200 import build as _b  # noqa: F401
    from paper_2312_12705_b200.build import LIB, build
    if not LIB.exists():
        build()
    from paper_2312_12705_b200 import _lib
    return _lib.load()
