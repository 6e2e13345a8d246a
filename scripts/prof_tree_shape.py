"""Grow trees of a given shape (for HBG_GROW_PROFILE phase breakdowns).
usage: prof_tree_shape.py rows d k [trees] [zero_prob]"""
import sys, os, time
import numpy as np
import torch
sys.path.insert(0, os.environ.get("HBG_PKG_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1706_08359_b200 as hbg  # noqa: E402

rows, d, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
trees = int(sys.argv[4]) if len(sys.argv) > 4 else 2
zp = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
rng = np.random.default_rng(0)
cols = rng.integers(1, k, size=(d, rows), dtype=np.uint8)
if zp > 0:
    cols[rng.random((d, rows)) < zp] = 0
g = (2 * rng.random(rows) - 1).astype(np.float32)
h = rng.random(rows).astype(np.float32)
with hbg.Dataset(cols, k) as ds:
    tg, th = torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda()
    s = torch.cuda.Stream()
    for _ in range(trees):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        log, nodes = ds.grow_tree(tg, th, 255, 1, 0.0, s.cuda_stream)
        torch.cuda.synchronize()
        print(f"tree {1e3 * (time.perf_counter() - t0):.2f} ms, splits {len(log)}", flush=True)
