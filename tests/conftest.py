import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C ABI")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def eng():
    from paper_2106_04756_b200 import engine
    return engine()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as r
    if not r.available():
        pytest.skip("oracle/_ref/libfolp_ref.so not built")
    return r.binding()
