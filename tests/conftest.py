import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdfm.so")


@pytest.fixture(scope="session")
def pins():
    with open(os.path.join(ROOT, "tests", "golden", "pins.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def eng():
    import paper_2410_22764_b200 as dfm
    return dfm.Engine(0)


@pytest.fixture(scope="session")
def eng_radix():
    import paper_2410_22764_b200 as dfm
    e = dfm.Engine(0)
    e.set_sortpr_engine("radix")
    return e
