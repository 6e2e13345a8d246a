"""Host drop-in time with pageable vs pinned LeafState arrays (BASELINE shape).

    HBG_STAGE_PROFILE=1 python scripts/pageable_probe.py [rows]

Prints per leaf shape the mean wall time of hbg_build_histograms (pageable
numpy arrays: the host-staged fp32 path; pinned: the fp64 DMA path) and, with
HBG_STAGE_PROFILE=1, the host pool's per-call staging timeline on stderr.
"""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1706_08359_b200 as hbg  # noqa: E402


def main():
    rows = int(sys.argv[1]) if len(sys.argv) > 1 else 10_500_000
    reps = int(os.environ.get("REPS", "30"))
    rng = np.random.default_rng(1)
    cols = rng.integers(0, 64, size=(28, rows), dtype=np.uint8)
    g, h = rng.normal(size=rows), rng.random(rows)
    shapes = {
        "root": np.arange(rows, dtype=np.int32),
        "depth1_sorted": np.sort(rng.choice(rows, rows // 2, replace=False)).astype(np.int32),
        "half_range": np.arange(rows // 4, rows // 4 + rows // 2, dtype=np.int32),
    }
    with hbg.Dataset(cols, 64) as ds:
        for name, idx in shapes.items():
            lg, lh = g[idx], h[idx]
            page = hbg.LeafState(idx, lg, lh)
            pin = hbg.LeafState(*(torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (idx, lg, lh)))
            for label, leaf in (("pageable", page), ("pinned", pin)):
                hbg.build_histograms_partitioned(ds, leaf)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(reps):
                    hbg.build_histograms_partitioned(ds, leaf)
                ms = (time.perf_counter() - t0) * 1e3 / reps
                print(f"{name:14s} {label:8s} rows={len(idx):9d} {ms:7.3f} ms/call", flush=True)
        if os.environ.get("TREES"):
            for label, (tg, th) in (("pageable", (g, h)),
                                    ("pinned", tuple(torch.from_numpy(a).pin_memory().numpy() for a in (g, h)))):
                ds.grow_tree_host(tg, th, 255, 100, 0.0)
                t0 = time.perf_counter()
                for _ in range(3):
                    ds.grow_tree_host(tg, th, 255, 100, 0.0)
                print(f"tree255        {label:8s} {(time.perf_counter() - t0) * 1e3 / 3:7.3f} ms/tree", flush=True)


if __name__ == "__main__":
    main()
