import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box via gpurun)")


@pytest.fixture(scope="session", autouse=True)
def _built_libraries():
    """Build liboracle.so and libcecoll.so once if they are missing."""
    import paper_2511_06605_b200 as cc
    from oracle import oracle as ora

    if not os.path.exists(ora.LIB):
        ora.build_oracle()
    if not os.path.exists(cc.LIB_PATH):
        cc.build()
    yield
