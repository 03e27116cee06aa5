import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    # `slow` tests (full-size CPU oracle runs, minutes each) run only with HS_SLOW=1
    if os.environ.get("HS_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow: set HS_SLOW=1")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def oracle():
    from oracle import hsoracle
    hsoracle.lib()
    return hsoracle


@pytest.fixture(scope="session")
def gpu():
    """The product package with a live device context (skips cleanly only when no GPU exists)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1802_07844_b200 as hs
    from paper_1802_07844_b200 import _lib
    _lib.Context.get()
    return hs
