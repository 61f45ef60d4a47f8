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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        meta = json.load(f)
    path = os.path.join(GOLDEN, name + ".npz")
    arrays = dict(np.load(path)) if os.path.exists(path) else {}
    return meta, arrays


@pytest.fixture(scope="session")
def oracle_lib():
    import oracle
    return oracle.build()


@pytest.fixture(scope="session")
def native_lib():
    from paper_2309_04393_b200 import _native
    from paper_2309_04393_b200 import build as b
    b.build()
    return _native.lib()


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
