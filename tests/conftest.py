"""pytest configuration: the ``gpu`` marker and repo-root imports.

``-m "not gpu"`` runs here (no GPU): oracle-vs-golden, host logic, C-ABI
load/export checks and the gloo world-size-2 sharding tests.
``-m gpu`` runs on a B200 through ``gpurun``: GPU-vs-oracle parity through
the C-ABI library.
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, f"{name}.npz"))
