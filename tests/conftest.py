import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhapigpu.so")


@pytest.fixture(scope="session")
def golden_index():
    import json

    return json.loads((GOLDEN / "expected" / "index.json").read_text())
