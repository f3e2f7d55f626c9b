import json
import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); the CPU suite runs -m 'not gpu'")


@pytest.fixture(scope="session")
def pins():
    return json.loads((GOLDEN / "structural_pins.json").read_text())


@pytest.fixture(scope="session")
def golden_table():
    return (GOLDEN / "structural_cube.csv").read_text()


@pytest.fixture(scope="session")
def lib():
    import paper_0910_5863_b200 as pb
    return pb.load_library()
