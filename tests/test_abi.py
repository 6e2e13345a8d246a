"""The C-ABI library loads and exports exactly what include/hbg.h declares (CPU-only)."""
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(REPO, "include", "hbg.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(hbg_[a-z_0-9]+)\(", text, re.M)))


def test_header_declares_the_python_symbol_list(hbg):
    assert declared_symbols() == sorted(hbg.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(hbg):
    out = subprocess.run(["nm", "-D", "--defined-only", hbg.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (hbg_[a-z_0-9]+)$", out, re.M))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = hbg.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert lib.hbg_version() == 1


def test_library_is_built_for_sm100a(hbg):
    out = subprocess.run(["cuobjdump", "--list-elf", hbg.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_a_gpu(hbg):
    """The product path fails loudly when no GPU is visible (it never computes on the CPU)."""
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(hbg.HbgError):
        hbg.Dataset(np.ones((2, 10), dtype=np.uint8), 16)


def test_product_package_never_imports_the_oracle():
    """Only tests/, smoke() and bench.py's cpu_baseline may touch oracle/."""
    pkg = os.path.join(REPO, "paper_1706_08359_b200")
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h", ".cuh")) or fn == "Makefile":
                with open(os.path.join(root, fn), errors="replace") as f:
                    text = f.read()
                assert "oracle" not in text.replace("oracle/", "").lower() or fn.endswith(".py") is False \
                    or "import oracle" not in text, fn
                assert "from oracle" not in text and "import oracle" not in text, fn
                assert "liboracle" not in text and "histoboost_ref" not in text, fn
