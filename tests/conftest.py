"""Shared fixtures.  `gpu` tests need a B200 (run via gpurun); everything
else runs on the CPU-only container."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def ref():
    """The reference's own compiled oracles (oracle/_ref/libmagref.so)."""
    from pyoracle import REF_SO, Ref
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libmagref.so not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def port():
    """The C restatement (oracle/libmagoracle.so)."""
    from pyoracle import Port
    return Port()


@pytest.fixture(scope="session")
def mag():
    import paper_1405_5483_b200 as M
    M.lib()
    return M
