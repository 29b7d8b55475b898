import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.load_oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    r = oracle.load_reference()
    if r is None:
        pytest.skip("reference build (oracle/_ref) unavailable on this box")
    return r


@pytest.fixture(scope="session")
def golden():
    import json
    import numpy as np
    here = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(here, "golden.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(here, "golden.npz")))
    return meta, arrays
