import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) device")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1206_4973_b200", "libflowbb_b200.so")
    orc = os.path.join(ROOT, "oracle", "liboracle.so")
    if not (os.path.exists(lib) and os.path.exists(orc)):
        import __graft_entry__

        __graft_entry__.build()


_ensure_built()


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def instances():
    with open(os.path.join(GOLDEN, "instances.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def pools():
    return dict(np.load(os.path.join(GOLDEN, "pools.npz")))


@pytest.fixture(scope="session")
def traces():
    with open(os.path.join(GOLDEN, "traces.json")) as f:
        return json.load(f)


def gpu_present() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
