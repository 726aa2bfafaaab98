import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "reference: drives the product with the installed, unmodified reference (baseline/_ref, built by __graft_entry__.build())")


@pytest.fixture(scope="session")
def dev_ops():
    """The product's device operator set; fails loudly (no fallback) without a GPU."""
    from paper_2410_09663_b200 import build
    from paper_2410_09663_b200.ops import DeviceOps

    build.build()
    return DeviceOps()


@pytest.fixture(scope="session")
def pm():
    from oracle import problems

    return problems.product_modules()
