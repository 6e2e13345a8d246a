"""Diagnostic (GPU): where a bits64 device tree first departs from the
reference's bits64 tree, and whether the two choices are an fp64 tie.

    python scripts/diag_bits64_tree.py ROWS K
"""
import math
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402
from test_gpu_parity import rows_of_node  # noqa: E402


def fsum_gain(cols, g, h, rows, f, b):
    left = cols[f, rows] <= b
    gr, hr = g[rows], h[rows]
    lg, lh = math.fsum(gr[left]), math.fsum(hr[left])
    G, H = math.fsum(gr), math.fsum(hr)
    rg, rh = G - lg, H - lh
    return lg * lg / lh + rg * rg / rh - G * G / H


def main():
    rows, k = int(sys.argv[1]), int(sys.argv[2])
    cols = ffi.gen_synthetic_bins(rows, 28, k, 0)
    g, h = ffi.gen_grad_hess(rows, 0)
    with hbg.Dataset(cols, k) as ds:
        log, nodes = ds.grow_tree_host(g, h, 255, 1, 0.0, precision=64)
    want_log, want_nodes = ffi.grow_tree(cols, k, g, h, 255, 1, 0.0, 64)
    i = 0
    while i < min(len(log), len(want_log)) and log["feature"][i] == want_log["feature"][i] and \
            log["threshold_bin"][i] == want_log["threshold_bin"][i] and log["left_count"][i] == want_log["left_count"][i]:
        i += 1
    print("identical splits:", i, "of", len(want_log))
    if i == len(want_log):
        return
    print("ours:", log[i])
    print("ref :", want_log[i])
    jo = int(np.nonzero(nodes["left"] == 2 * i + 1)[0][0])
    jr = int(np.nonzero(want_nodes["left"] == 2 * i + 1)[0][0])
    ro, rr = rows_of_node(cols, nodes, jo), rows_of_node(cols, want_nodes, jr)
    go = fsum_gain(cols, g, h, ro, int(log["feature"][i]), int(log["threshold_bin"][i]))
    gr = fsum_gain(cols, g, h, rr, int(want_log["feature"][i]), int(want_log["threshold_bin"][i]))
    print(f"leaf ours {jo} ({len(ro)} rows) ref {jr} ({len(rr)} rows)")
    print(f"exact-sum gains: ours {go!r} ref {gr!r} rel diff {(gr - go) / abs(gr):.3e}")
    print(f"logged gains: ours {log['gain'][i]!r} ref {want_log['gain'][i]!r}")
    # previous splits' gains for context
    for j in range(max(0, i - 2), i):
        print(j, log["gain"][j], want_log["gain"][j], log["gain"][j] - want_log["gain"][j])


if __name__ == "__main__":
    main()
