"""C++ drop-in check with the reference's own types and predicates (GPU).

Runs oracle/_ref/backend_swap (tests/cpp/backend_swap.cpp, built against the
reference headers/objects and libhbg.so): build_histograms_cuda vs the
reference's build_histograms_partitioned(bits64) under histograms_equivalent
(counts exact, stats within stats_tolerance(bits32) = 1e-4, the reference's
own fp32 bar) plus identical best splits, and the
std::invalid_argument error path.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(REPO, "oracle", "_ref", "backend_swap")


def test_cpp_backend_swap():
    if not os.path.exists(BIN):
        pytest.skip("backend_swap not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
