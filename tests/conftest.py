import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def _has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


HAS_CUDA = _has_cuda()


def pytest_collection_modifyitems(config, items):
    if HAS_CUDA:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


_EXIT = {"status": None}


def pytest_sessionfinish(session, exitstatus):
    _EXIT["status"] = int(exitstatus)


def pytest_unconfigure(config):
    # After a failed GPU run, interpreter teardown can block on CUDA / NCCL
    # state a failed rank left behind (a poisoned context, communicators whose
    # peers are gone); the report is already printed, so skip the teardown.
    if HAS_CUDA and _EXIT["status"] not in (None, 0):
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(_EXIT["status"])
