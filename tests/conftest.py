import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session")
def oracle():
    import lco
    return lco.Restatement()


@pytest.fixture(scope="session")
def reference():
    import lco
    if not lco.Reference.available():
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return lco.Reference()


@pytest.fixture(scope="session")
def ctx():
    import paper_2510_05367_b200 as lc
    c = lc.Context(0)
    yield c
    c.close()
