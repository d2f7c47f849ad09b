import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (runs on the GPU box)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 CUDA devices (collected only where present)")


def pytest_collection_modifyitems(config, items):
    """multigpu tests run whenever the box has >= 2 GPUs; elsewhere they are
    deselected (not skipped): there is nothing to run them on."""
    if not any(it.get_closest_marker("multigpu") for it in items):
        return
    try:
        import torch

        ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover
        ngpu = 0
    if ngpu >= 2:
        return
    keep, drop = [], []
    for it in items:
        (drop if it.get_closest_marker("multigpu") else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build()
    return oracle
