import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: full-size configuration runs")


@pytest.fixture(scope="session")
def gpu():
    """The CUDA product path.  Fails (does not skip) without a device: a GPU
    test that silently passes on CPU would hide a missing native path."""
    import paper_1405_1020_b200 as opc

    n = opc.device_count()
    assert n > 0, "no CUDA device visible: the gpu tests need a B200"
    return opc
