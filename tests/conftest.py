import json
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblmpk.so")


@pytest.fixture(scope="session")
def golden():
    """(facts dict, arrays npz) produced by tests/golden/make_golden.py from the reference."""
    facts = json.loads((GOLDEN / "golden.json").read_text())
    arrays = np.load(GOLDEN / "golden.npz")
    return facts, arrays


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
