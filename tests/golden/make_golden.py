"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs the reference (histoboost) compiled from /root/reference by
oracle/Makefile into oracle/_ref/libhistoboost_ref.so, through ref_shim.cpp.
The outputs are committed so the tests can pin the oracle (and the GPU path)
on machines where /root/reference does not exist (the GPU box).

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ffi  # noqa: E402

SEED_STEP = 0x51ED270B  # bench.cpp:96-97


def main() -> None:
    ffi.build(ref=True)
    assert ffi.ref_available(), "reference .so missing (needs /root/reference)"
    out = {}

    # gen_synthetic_bins (bench.cpp:17-38): test_bench.cpp:12-43 shape
    cols = ffi.ref_gen_synthetic_bins(100000, 3, 64, 7)
    out["synthetic_bins_100000x3_k64_seed7"] = {
        "head": cols[:, :16].tolist(),
        "sum": [int(c.sum()) for c in cols],
        "counts_f0": np.bincount(cols[0], minlength=64).tolist(),
    }
    # leaf_index_sample (bench.cpp:40-57): test_bench.cpp:45-61
    out["leaf_index_sample_1000_seed3"] = {
        str(d): ffi.ref_leaf_index_sample(1000, d, 3).tolist() for d in (1, 3, 7)
    }
    out["leaf_index_sample_8_depth3_seed1"] = ffi.ref_leaf_index_sample(8, 3, 1).tolist()

    # pack_feature_tuples on random columns (binning.cpp:123-158)
    rng = np.random.default_rng(5)
    c8 = rng.integers(0, 256, size=(7, 9), dtype=np.uint8)
    c4 = rng.integers(0, 16, size=(11, 9), dtype=np.uint8)
    out["pack8_7x9"] = {"cols": c8.tolist(), "words": ffi.ref_pack_feature_tuples(c8, 8, 256).tolist()}
    out["pack4_11x9"] = {"cols": c4.tolist(), "words": ffi.ref_pack_feature_tuples(c4, 4, 16).tolist()}

    with open(os.path.join(HERE, "reference_outputs.json"), "w") as f:
        json.dump(out, f, indent=1)

    # Histograms (build_histograms_partitioned, bits64 and bits32) over the
    # bench generators, several depths and bin capacities, crossing the 64Ki
    # chunk boundary at depth 0.
    arrays = {}
    for k, rows, d in ((64, 70000, 28), (16, 9000, 28), (256, 5000, 37), (64, 3000, 1)):
        cols = ffi.ref_gen_synthetic_bins(rows, d, k, 11)
        g, h = ffi.gen_grad_hess(rows, 11)
        for depth in (0, 3):
            idx = ffi.ref_leaf_index_sample(rows, depth, 11 + SEED_STEP * depth)
            lg, lh = g[idx], h[idx]
            tag = f"k{k}_r{rows}_d{d}_D{depth}"
            arrays[f"{tag}_idx"] = idx
            arrays[f"{tag}_h64"] = ffi.ref_build_histograms(cols, k, idx, lg, lh, 64)
            arrays[f"{tag}_h32"] = ffi.ref_build_histograms(cols, k, idx, lg, lh, 32)
    # One tree (grow_tree, bits64): split log
    cols = ffi.ref_gen_synthetic_bins(4000, 6, 16, 3)
    g, h = ffi.gen_grad_hess(4000, 3)
    rd = ffi.RefDataset(cols, 16)
    _, log = rd.grow_tree_timed(g, h, 31, 1, 0.0, 64)
    arrays["tree_4000x6_k16_seed3_split_log"] = log
    _, log2 = rd.grow_tree_timed(g, h, 20, 20, 1.0, 64)
    arrays["tree_4000x6_k16_seed3_min20_lam1_split_log"] = log2
    np.savez_compressed(os.path.join(HERE, "reference_histograms.npz"), **arrays)
    print("wrote", os.path.join(HERE, "reference_outputs.json"), "and reference_histograms.npz")


if __name__ == "__main__":
    main()
