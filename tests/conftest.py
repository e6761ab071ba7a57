import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    # Build (or refresh) the in-tree libraries first: nvcc cross-compiles without a GPU, and
    # the CPU suite checks the library's exported symbols.
    import __graft_entry__
    __graft_entry__._build_module().build()
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run via gpurun")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_cuda():
        return
    skip = pytest.mark.skip(reason="no CUDA device here (run -m gpu via gpurun)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
