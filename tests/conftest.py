import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libpals_gpu.so)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    if not Reference.available():
        try:
            from oracle.oracle import build
            build()
        except Exception:
            pass
    if not Reference.available():
        pytest.skip("reference build (oracle/_ref) not present")
    return Reference()


@pytest.fixture(scope="session")
def bundle():
    from paper_2605_21427_b200.profiles import load_bundle
    return load_bundle()


@pytest.fixture(scope="session")
def gold():
    import numpy as np

    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLD, name + ".npz")))
        return cache[name]

    return get


@pytest.fixture(scope="session")
def ctx():
    from paper_2605_21427_b200.wattserve import default_context
    return default_context()
