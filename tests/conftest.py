import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libcake_ref.so")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def cake_b200():
    from paper_2410_03065_b200.cake import Cake

    return Cake()


@pytest.fixture(scope="session")
def cake_ref():
    """The reference library built from /root/reference sources (oracle/_ref)."""
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref/libcake_ref.so not built (needs /root/reference at build time)")
    from paper_2410_03065_b200 import native
    from paper_2410_03065_b200.cake import Cake

    return Cake(native.load(REF_LIB))


def have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
