"""Per-launch cost of the per-split kernels in isolation vs interleaved (GPU)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402

rows, d, k = 200_000, 28, 64
rng = np.random.default_rng(0)
cols = rng.integers(1, 64, size=(d, rows), dtype=np.uint8)
g = (2 * rng.random(rows) - 1).astype(np.float32)
h = rng.random(rows).astype(np.float32)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
sp = s.cuda_stream


def timeit(fn, reps=200):
    for _ in range(5):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


with hbg.Dataset(cols, k) as ds:
    tg, th = torch.from_numpy(g).cuda(), torch.from_numpy(h).cuda()
    idx = torch.arange(0, rows, 1000, dtype=torch.int32, device="cuda")  # 200-row leaf
    hist = torch.empty(ds.hist_values(), dtype=torch.float64, device="cuda")
    out = torch.empty(10, dtype=torch.float64, device="cuda")
    ds.build_histograms_device(idx, len(idx), tg, th, hist, hbg.HBG_GH_ROW_INDEXED, sp)
    split = lambda: hbg.best_split_device(hist, d, k, 1.0, 50.0, len(idx), 1, 0.0, out, sp)
    build = lambda: ds.build_histograms_device(idx, len(idx), tg, th, hist, hbg.HBG_GH_ROW_INDEXED, sp)
    print(f"best_split alone      {timeit(split):8.2f} us")
    print(f"tiny build alone      {timeit(build):8.2f} us")
    print(f"build+split           {timeit(lambda: (build(), split())):8.2f} us")
    big = torch.arange(0, rows, dtype=torch.int32, device="cuda")
    bigb = lambda: ds.build_histograms_device(big, rows, tg, th, hist, hbg.HBG_GH_ROW_INDEXED, sp)
    print(f"200K build alone      {timeit(bigb):8.2f} us")
    print(f"200K build + split    {timeit(lambda: (bigb(), split())):8.2f} us")
    log, nodes = ds.grow_tree(tg, th, 255, 1, 0.0, sp)
    print(f"tree 255 leaves 200K  {timeit(lambda: ds.grow_tree(tg, th, 255, 1, 0.0, sp), reps=5):8.1f} us")
