import sys, os, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1706_08359_b200 as hbg
rows = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = np.random.default_rng(0)
cols = rng.integers(1, 64, size=(28, rows), dtype=np.uint8)
g = 2 * rng.random(rows) - 1; h = rng.random(rows)
pg = torch.from_numpy(g).pin_memory().numpy(); ph = torch.from_numpy(h).pin_memory().numpy()
with hbg.Dataset(cols, 64) as ds:
    for prec in (32, 64):
        ds.grow_tree_host(pg, ph, 255, 1, 0.0, precision=prec)
        t0 = time.perf_counter()
        for _ in range(reps):
            ds.grow_tree_host(pg, ph, 255, 1, 0.0, precision=prec)
        print(f"rows {rows} bits{prec}: {(time.perf_counter()-t0)*1e3/reps:.2f} ms/tree", flush=True)
