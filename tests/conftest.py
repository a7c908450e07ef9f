"""Shared fixtures.  `-m gpu` tests need a B200 (they call the CUDA path through
the C ABI); everything else runs on CPU.  The oracle (oracle/) is test
infrastructure: it is imported here only as the checker."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); runs the device path")
    config.addinivalue_line("markers", "slow: long-running case")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN, "golden_small.npz"))
    return {k: data[k] for k in data.files}


def golden_csr(g, key):
    from oracle.oracle import Csr

    shape = g[key + "/shape"]
    vals = g.get(key + "/values")
    return Csr(int(shape[0]), int(shape[1]), g[key + "/row_ptr"], g[key + "/col_idx"], vals)


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O

    return O.get("port")


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O

    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return O.get("reference")
