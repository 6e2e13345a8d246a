"""Diagnostic: two row-shard ranks as threads on one GPU through hbg_grow_tree_peer,
host timestamps around each call (are the two persistent grids concurrent?)."""
import os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402

world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows, d, k = 60000, 28, 64
sms = torch.cuda.get_device_properties(0).multi_processor_count
cols = ffi.gen_synthetic_bins(rows, d, k, 6)
g, h = ffi.gen_grad_hess(rows, 6)
cuts = [rows * r // world for r in range(world + 1)]
dss = [hbg.Dataset(np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]), k) for r in range(world)]
ctas = int(sys.argv[1]) if len(sys.argv) > 1 else sms // world
peers = [hbg.Peer(dss[r], world, r, ctas=ctas) for r in range(world)]
gh = [(torch.from_numpy(g[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda(),
       torch.from_numpy(h[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda()) for r in range(world)]
for p in peers:
    for q in peers:
        if q is not p:
            p.attach(q)
torch.cuda.synchronize()
t0 = time.perf_counter()
log = []
def run(r):
    log.append((r, "start", time.perf_counter() - t0))
    try:
        out = dss[r].grow_tree_peer(gh[r][0], gh[r][1], peers[r], 63, 60, 0.0, dss[r].stream())
        log.append((r, "done", time.perf_counter() - t0, len(out[0])))
    except Exception as e:
        log.append((r, "error", time.perf_counter() - t0, str(e)[:120]))
ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
for t in ts: t.start()
for t in ts: t.join()
for e in sorted(log, key=lambda x: x[2]): print(e)
