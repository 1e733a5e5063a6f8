import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path via the C-ABI)")
    config.addinivalue_line("markers", "ref: needs oracle/_ref/libkvref.so (reference compiled here)")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import RefLib, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libkvref.so not built (reference sources absent)")
    return RefLib()


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


@pytest.fixture(scope="session")
def kvx():
    """The product library (CUDA path through the C-ABI).  GPU tests only."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2407_00079_b200 as pkg
    return pkg
