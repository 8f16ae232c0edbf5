import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def _have_ref():
    from oracle import oracle as O
    return os.path.exists(O.REF_SO)


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.build(ref=os.path.isdir(O.REFERENCE_SRC))
    return O


@pytest.fixture(scope="session")
def have_ref(oracle_mod):
    return os.path.exists(oracle_mod.REF_SO)


@pytest.fixture(scope="session")
def engine():
    import paper_2301_06984_b200 as E
    from paper_2301_06984_b200 import build
    build.build()
    return E


