import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# The slab tests run several slabs of the multi-GPU path on ONE device, one
# host thread and stream each; their kernels spin on each other's progress.
# Lazy module loading (a context-wide sync on a kernel's first launch) and
# hardware-queue aliasing between streams would serialise what must run
# concurrently, so load every module at context creation and give every
# stream its own queue.  Must be set before CUDA is initialised.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# the same applies to instantiating the solver's CUDA graphs mid-run
os.environ.setdefault("PF_NO_GRAPHS", "1")
# ... and to host threads blocked on a full launch queue: keep few iterations
# in flight per slab between polls
os.environ.setdefault("PF_MAX_BATCH", "4")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA device (B200) and libpisob200.so")


def pytest_collection_modifyitems(config, items):
    import torch
    if torch.cuda.is_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
