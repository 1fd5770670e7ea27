import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
for p in (str(REPO), str(GOLDEN)):
    if p not in sys.path:
        sys.path.insert(0, p)

CONFIG_KEYS = ("gr17", "eil51", "kroA100", "a280", "dsj1000")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libvrprpd.so")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN / "golden.npz")


@pytest.fixture(scope="session")
def golden_meta():
    return json.loads((GOLDEN / "golden.json").read_text())


_INST = {}


def config_instance(key):
    if key not in _INST:
        from paper_2602_23685_b200.configs import config_instance as ci
        _INST[key] = ci(key)
    return _INST[key]
