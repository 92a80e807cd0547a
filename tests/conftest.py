import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libcafxg.so")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "reference_mandelbrot.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def ctx():
    import paper_1505_07368_b200 as pkg
    c = pkg.Context(device_mask=1)
    yield c
    c.close()
