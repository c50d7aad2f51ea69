import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

GOLDEN = os.path.join(ROOT, "tests", "golden")
CASE_NAMES = ["a64", "b200", "c500bd", "d1000", "e2000s", "f48", "g7", "h1"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    # a device hang must fail the test, not the GPU box (pytest-timeout)
    if config.pluginmanager.hasplugin("timeout") and not config.getoption("timeout", None):
        config.option.timeout = 600


def load_case(name):
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, f"case_{name}.npz")))


def load_kats():
    import numpy as np
    return dict(np.load(os.path.join(GOLDEN, "kats.npz")))


def has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
