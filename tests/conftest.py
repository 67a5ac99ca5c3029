import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import build, load_oracle

    build()
    return load_oracle()


@pytest.fixture(scope="session")
def reference():
    """The reference compiled from its own sources, or skip when absent."""
    from oracle import load_reference

    r = load_reference()
    if r is None:
        pytest.skip("oracle/_ref not built (no /root/reference at build time)")
    return r


@pytest.fixture(scope="session")
def F():
    from paper_2411_02908_b200 import build as b

    b.build()
    from paper_2411_02908_b200 import fedsim

    return fedsim
