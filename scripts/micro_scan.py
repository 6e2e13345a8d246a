"""Split-scan kernel cost vs histogram shape (GPU)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402

s = torch.cuda.Stream()
torch.cuda.set_stream(s)
for d, k in [(1, 2), (1, 64), (28, 64), (28, 16), (100, 64), (2000, 64), (968, 256)]:
    rng = np.random.default_rng(0)
    h = np.zeros((3, d, k))
    h[2] = rng.integers(0, 50, size=(d, k))
    h[0] = rng.normal(size=(d, k)) * h[2]
    h[1] = rng.random((d, k)) * h[2]
    dh = torch.from_numpy(h.ravel()).cuda()
    out = torch.empty(20, dtype=torch.float64, device="cuda")
    n = int(h[2][0].sum())
    f = lambda: hbg.best_split_device(dh, d, k, float(h[0][0].sum()), float(h[1][0].sum()), n, 1, 0.0, out, s.cuda_stream)
    for _ in range(10):
        f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(200):
        f()
    b.record(s)
    torch.cuda.synchronize()
    print(f"d={d:5d} k={k:4d}  {a.elapsed_time(b) / 200 * 1e3:8.2f} us/scan")
