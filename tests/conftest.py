import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the C oracle if they are missing (nvcc /
    gcc exist both here and on the GPU box); oracle/_ref only where the
    reference sources exist."""
    from paper_1309_7327_b200 import build as B
    from oracle import oracle as O
    if not os.path.exists(B.LIB):
        B.build()
    if not os.path.exists(os.path.join(O.HERE, "liboracle.so")):
        O.build_oracle()
    yield


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def rel_err(x, y):
    """max |x - y| / max |y| (per-component max error relative to the field max)."""
    x = np.asarray(x)
    y = np.asarray(y)
    scale = np.abs(y).max()
    return float(np.abs(x - y).max() / (scale if scale > 0 else 1.0))
