"""Test configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here (no GPU): the oracle against the golden vectors and
the reference, host logic, the C-ABI library loading/exporting every symbol,
and the multi-process (gloo) host logic. `-m gpu` runs on a B200 and calls
the CUDA path through the C ABI, checking it against the oracle.
"""
import os
import sys

import pytest

# Several "ranks" sharing the one GPU of the tests run persistent grids on
# different streams that must execute concurrently (they exchange through
# peer memory); with the default 8 hardware work queues two streams can share
# a queue and serialise. Must be set before the CUDA context exists.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); calls the CUDA path through the C ABI")


@pytest.fixture(scope="session")
def oracle():
    from oracle import ffi

    ffi.lib()
    return ffi


@pytest.fixture(scope="session")
def hbg():
    import paper_1706_08359_b200 as hbg

    hbg.build()
    hbg.lib()
    return hbg
