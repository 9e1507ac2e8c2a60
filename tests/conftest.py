import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: full-size (config 3) GPU checks")


@pytest.fixture(scope="session")
def codec():
    from paper_2111_10105_b200 import codec as C
    cd = C.Codec(0)
    yield cd
    cd.close()
