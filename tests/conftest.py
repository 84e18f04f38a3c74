import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libhermb200.so")


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    gdir = os.path.join(ROOT, "tests", "golden")
    out = {}
    for name in ("interp", "steps2d", "steps1d"):
        with np.load(os.path.join(gdir, f"{name}.npz")) as z:
            out.update({k: z[k] for k in z.files})
    return out
