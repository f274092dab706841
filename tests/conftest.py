import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


def load_npz(name):
    return np.load(GOLDEN / name)


@pytest.fixture
def rng():
    # same seed as the reference suite (tests/conftest.py:8-10 of the reference)
    return np.random.default_rng(20260824)


@pytest.fixture(scope="session")
def golden_plans():
    return load_json("plans.json")


@pytest.fixture(scope="session")
def golden_contract():
    return load_json("contract.json"), load_npz("contract.npz")


@pytest.fixture(scope="session")
def golden_kernels():
    return load_json("kernels.json"), load_npz("kernels.npz")


@pytest.fixture(scope="session")
def golden_hooi():
    return load_json("hooi.json"), load_npz("hooi.npz")
