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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")


def _has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    def __init__(self, tag):
        with open(os.path.join(GOLDEN, f"golden_{tag}.json")) as fh:
            self.meta = json.load(fh)
        path = os.path.join(GOLDEN, f"golden_{tag}.npz")
        self.arrays = np.load(path) if os.path.exists(path) else {}

    def cases(self, kind):
        return sorted(k for k, m in self.meta.items() if m["kind"] == kind)

    def __getitem__(self, key):
        return self.arrays[key]

    def has(self, key):
        return key in self.arrays


@pytest.fixture(scope="session")
def golden():
    return Golden("small")


@pytest.fixture(scope="session")
def golden_large():
    p = os.path.join(GOLDEN, "golden_large.json")
    if not os.path.exists(p):
        pytest.skip("large golden fixtures not generated")
    return Golden("large")
