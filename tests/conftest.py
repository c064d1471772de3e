import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import Oracle
    return Oracle("restated")


@pytest.fixture(scope="session")
def ref():
    """The reference itself (oracle/_ref), built from /root/reference here and
    shipped prebuilt to the GPU box."""
    from oracle.oracle import Oracle, LIBS
    if not os.path.exists(LIBS["reference"]):
        pytest.skip("oracle/_ref not built (reference headers absent)")
    return Oracle("reference")
