import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# several virtual ranks on one GPU drive their peer kernels from separate streams:
# enough hardware work queues that no two of those streams share one (a
# spinning kernel would otherwise block the kernel queued behind it)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def libhs():
    """Build (if stale) and load libhs.so; the GPU box receives the in-tree build."""
    from paper_2505_12566_b200 import _build
    try:
        _build.build_all()
    except RuntimeError as e:  # no nvcc on this host: use the shipped .so
        if not os.path.exists(_build.LIBHS):
            raise
    import paper_2505_12566_b200 as hs
    return hs
