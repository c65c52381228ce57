"""Test configuration: repo root on sys.path, the ``gpu`` marker.

``-m "not gpu"`` runs here (no GPU): oracle vs golden vectors, graph /
dispatch-order parity with the reference, host logic, C-ABI exports,
multi-process exchange logic over gloo.  ``-m gpu`` runs on a B200 and
checks the CUDA path against the oracle.
"""

import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")


def pytest_collection_modifyitems(config, items):
    import torch

    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden_ops():
    import numpy as np

    return dict(np.load(GOLDEN / "ops.npz"))


@pytest.fixture(scope="session")
def golden_train():
    import json

    import numpy as np

    return dict(np.load(GOLDEN / "train.npz")), json.loads((GOLDEN / "train.json").read_text())


@pytest.fixture(scope="session")
def golden_graphs():
    import json

    return json.loads((GOLDEN / "graphs.json").read_text())
