"""Histogram kernel time for a leaf of n rows: contiguous row ids vs a random
sorted subset vs a strided subset (the gathered-slice cost). Higgs 10.5M x 28 k64."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402

ROWS, D, K = 10_500_000, 28, 64
rng = np.random.default_rng(0)
cols = rng.integers(1, K, size=(D, ROWS), dtype=np.uint8)
g = (2 * rng.random(ROWS) - 1).astype(np.float32)
h = rng.random(ROWS).astype(np.float32)
ds = hbg.Dataset(cols, K)
dev = torch.device("cuda:0")
hist = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
s = torch.cuda.Stream()
for n in (5_250_000, 1_312_500):
    leaves = {"contiguous": np.arange(n, dtype=np.int32),
              "stride": (np.arange(n, dtype=np.int64) * (ROWS // n)).astype(np.int32),
              "random": np.sort(rng.choice(ROWS, n, replace=False)).astype(np.int32)}
    for name, idx in leaves.items():
        ti = torch.from_numpy(idx).to(dev)
        tg = torch.from_numpy(g[idx]).to(dev)
        th = torch.from_numpy(h[idx]).to(dev)
        for _ in range(3):
            ds.build_histograms_device(ti, n, tg, th, hist, hbg.HBG_GH_LEAF_ALIGNED, s.cuda_stream)
        torch.cuda.synchronize()
        ds.kernel_time()
        ds.set_profiling(True)
        for _ in range(20):
            ds.build_histograms_device(ti, n, tg, th, hist, hbg.HBG_GH_LEAF_ALIGNED, s.cuda_stream)
        torch.cuda.synchronize()
        ds.set_profiling(False)
        km, kl = ds.kernel_time()
        print(f"n {n:9d} {name:10s} kernel {1e3 * km / kl:8.1f} us", flush=True)
