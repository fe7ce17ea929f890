import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def sim_golden():
    return json.loads((GOLDEN / "sim_cases.json").read_text())["cases"]


@pytest.fixture(scope="session")
def policy_golden():
    p = GOLDEN / "policy_cases.json"
    return json.loads(p.read_text())
