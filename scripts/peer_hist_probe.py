"""Diagnostic for hbg_build_histograms_peer: 2 ranks as threads on one GPU."""
import os, sys, threading
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402

world, rows, d, k = 2, 120000, 28, 64
cols = ffi.gen_synthetic_bins(rows, d, k, 4)
g, h = ffi.gen_grad_hess(rows, 4)
gf, hf = g.astype(np.float32), h.astype(np.float32)
cuts = [rows * r // world for r in range(world + 1)]
dss = [hbg.Dataset(np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]), k) for r in range(world)]
peers = [hbg.Peer(dss[r], world, r) for r in range(world)]
peers[0].attach(peers[1]); peers[1].attach(peers[0])
D = d * k
want = ffi.build_histograms(cols, k, np.arange(rows, dtype=np.int32), g, h, 64)
wantl = [ffi.build_histograms(cols[:, cuts[r]:cuts[r + 1]], k, np.arange(cuts[r + 1] - cuts[r], dtype=np.int32),
                              g[cuts[r]:cuts[r + 1]], h[cuts[r]:cuts[r + 1]], 64) for r in range(world)]
ts_ = []
for r in range(world):
    n = cuts[r + 1] - cuts[r]
    ts_.append((torch.arange(n, dtype=torch.int32, device="cuda"), torch.from_numpy(gf[cuts[r]:cuts[r + 1]]).cuda(),
                torch.from_numpy(hf[cuts[r]:cuts[r + 1]]).cuda(), torch.empty(3 * D, dtype=torch.float64, device="cuda")))
torch.cuda.synchronize()
outs = [None] * world
def run(r):
    idx, tg, th, out = ts_[r]
    dss[r].build_histograms_peer(idx, len(idx), tg, th, out, peers[r], stream=dss[r].stream())
    peers[r].check()
    outs[r] = out.cpu().numpy()
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
for t in ts: t.start()
for t in ts: t.join()
for r in range(world):
    o = outs[r]
    print("rank", r, "count vs global", np.abs(o[2 * D:].reshape(d, k) - want["count"]).max(),
          "vs own local", np.abs(o[2 * D:].reshape(d, k) - wantl[r]["count"]).max(),
          "vs other local", np.abs(o[2 * D:].reshape(d, k) - wantl[1 - r]["count"]).max(),
          "zeros", int((o[2 * D:] == 0).sum()))
