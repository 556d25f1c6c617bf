import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libfp8q.so")
    config.addinivalue_line("markers", "slow: long-running (exhaustive maps, full-size shapes)")


def pytest_collection_modifyitems(config, items):
    # GPU tests are skipped (not passed) when no CUDA device is visible; on a GPU box
    # they run for real and the product path fails loudly if libfp8q.so is missing.
    try:
        import torch
        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    skip = pytest.mark.skip(reason="no CUDA device visible")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
