"""A/B of the device tree (255 leaves, Higgs 10.5M x 28 k64) between two
builds of the library: python scripts/tree_ab.py REPO_DIR [trees] [rows]
Prints per-tree device time (CUDA events) and the host drop-in's wall time."""
import os
import sys
import time

import numpy as np
import torch

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import paper_1706_08359_b200 as hbg  # noqa: E402

trees = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rows, d, k = (int(sys.argv[3]) if len(sys.argv) > 3 else 10_500_000), 28, 64
rng = np.random.default_rng(0)
cols = rng.integers(1, k, size=(d, rows), dtype=np.uint8)
g = 2.0 * rng.random(rows) - 1.0
h = rng.random(rows)
dev = torch.device("cuda:0")
ds = hbg.Dataset(cols, k)
tg = torch.from_numpy(g.astype(np.float32)).to(dev)
th = torch.from_numpy(h.astype(np.float32)).to(dev)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for _ in range(3):
    ds.grow_tree(tg, th, 255, 1, 0.0, s.cuda_stream)
torch.cuda.synchronize()
ts = []
for _ in range(trees):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    ds.grow_tree(tg, th, 255, 1, 0.0, s.cuda_stream)
    b.record(s)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
pg = torch.from_numpy(g).pin_memory().numpy()
ph = torch.from_numpy(h).pin_memory().numpy()
ds.grow_tree_host(pg, ph, 255, 1, 0.0)
we = []
for _ in range(trees // 2):
    t0 = time.perf_counter()
    ds.grow_tree_host(pg, ph, 255, 1, 0.0)
    we.append((time.perf_counter() - t0) * 1e3)
ts, we = np.array(ts), np.array(we)
print(f"{root[-30:]:30s} device ms/tree: median {np.median(ts):.3f} min {ts.min():.3f} max {ts.max():.3f} | "
      f"e2e ms/tree: median {np.median(we):.3f} min {we.min():.3f} max {we.max():.3f}")
