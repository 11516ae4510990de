import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "flowpipe_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session", autouse=True)
def _library_built():
    """A fresh checkout has no libstreamflow.so (build output, git-ignored): build it once
    (nvcc cross-compiles for sm_100a without a GPU) before the contract tests load it."""
    from paper_2511_22009_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        from paper_2511_22009_b200.build import build

        build()


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return np.load(GOLDEN)
