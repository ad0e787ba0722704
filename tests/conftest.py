"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (B200, sm_100a) and the in-tree libsgi.so; the driver
runs ``-m gpu`` on a real B200 and ``-m "not gpu"`` here on CPU.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA GPU (B200) and the built libsgi.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Compile the C oracle and the host input generator (both cheap, gcc only)."""
    import oracle
    import sgi_inputs
    oracle.build()
    sgi_inputs.build(device=False)
    yield
