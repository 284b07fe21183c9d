import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (runs the sm_100a path)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref (the reference built from /root/reference)")


def pytest_collection_modifyitems(config, items):
    from oracle import oracle as O

    if not O.ref_available() and os.path.isdir(O.REF_SRC):
        O.build()
    skip_ref = pytest.mark.skip(reason="oracle/_ref not built (reference absent)")
    for item in items:
        if "ref" in item.keywords and not O.ref_available():
            item.add_marker(skip_ref)


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
        return cache[name]

    return load
