"""Diagnostic: where does the full-size fp32 error come from? (GPU)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402

rows, d, k = 10_500_000, 28, 64
cols = ffi.gen_synthetic_bins(rows, d, k, 0)
g, h = ffi.gen_grad_hess(rows, 0)
idx = np.arange(rows, dtype=np.int32)
want = ffi.build_histograms(cols, k, idx, g, h, 64)
g32 = g.astype(np.float32).astype(np.float64)
h32 = h.astype(np.float32).astype(np.float64)
want32in = ffi.build_histograms(cols, k, idx, g32, h32, 64)   # fp64 sums of the fp32-rounded inputs
ref32 = ffi.build_histograms(cols, k, idx, g, h, 32)            # reference bits32 (chunked fp32)
dev = torch.device("cuda:0")
with hbg.Dataset(cols, k) as ds:
    tg = torch.from_numpy(g.astype(np.float32)).to(dev)
    th = torch.from_numpy(h.astype(np.float32)).to(dev)
    out = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
    ds.build_histograms_device(None, rows, tg, th, out, hbg.HBG_GH_LEAF_ALIGNED, 0)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(3, d, k)
for name, ref in (("bits64", want), ("bits64-of-fp32-inputs", want32in), ("bits32-ref", ref32)):
    for j, key in ((0, "grad_sum"), (1, "hess_sum")):
        scale = np.maximum(1.0, np.maximum(np.abs(o[j]), np.abs(ref[key])))
        err = np.abs(o[j] - ref[key]) / scale
        f, b = np.unravel_index(np.argmax(err), err.shape)
        print(f"gpu vs {name:22s} {key}: max_rel={err.max():.3e} at f={f} b={b} gpu={o[j][f, b]!r} ref={ref[key][f, b]!r} count={want['count'][f, b]}")
for j, key in ((0, "grad_sum"), (1, "hess_sum")):
    scale = np.maximum(1.0, np.abs(want[key]))
    print(f"fp32-input rounding alone {key}: {(np.abs(want32in[key] - want[key]) / scale).max():.3e};"
          f" reference bits32 vs bits64: {(np.abs(ref32[key] - want[key]) / scale).max():.3e}")
