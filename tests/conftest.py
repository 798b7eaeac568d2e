import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def h1_golden():
    import numpy as np

    return dict(np.load(GOLDEN / "h1_golden.npz"))


@pytest.fixture(scope="session")
def h2_golden():
    import json

    return json.loads((GOLDEN / "h2_golden.json").read_text())
