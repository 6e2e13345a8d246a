"""Where a deep leaf's time goes (per-leaf drop-in).

For leaves of the Higgs 10.5M x 28 k64 dataset at depth D (rows >> D, random
sorted rows, leaf-aligned fp32 g/h), prints per call:
  host_loop_us  — Python loop of build_histograms_device (ctypes + launches)
  issue_us      — host time per call of that loop (no synchronisation)
  graph_us      — the same call captured in a CUDA graph, replayed (GPU only)
  kernel_us     — the histogram kernel alone (library CUDA events)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402

ROWS, D, K = 10_500_000, 28, 64


def main():
    depths = [int(x) for x in sys.argv[1:]] or [0, 2, 4, 6, 8, 10]
    dev = torch.device("cuda:0")
    cols = ffi.gen_synthetic_bins(ROWS, D, K, 0)
    g, h = ffi.gen_grad_hess(ROWS, 0)
    tg = torch.from_numpy(g.astype(np.float32)).to(dev)
    th = torch.from_numpy(h.astype(np.float32)).to(dev)
    ds = hbg.Dataset(cols, K)
    hist = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    for depth in depths:
        rng = np.random.default_rng(100 + depth)
        idx = np.arange(ROWS, dtype=np.int32) if depth == 0 else np.sort(
            rng.choice(ROWS, ROWS >> depth, replace=False)).astype(np.int32)
        m = len(idx)
        li = torch.from_numpy(idx).to(dev)
        lg, lh = tg[li].contiguous(), th[li].contiguous()
        with torch.cuda.stream(s):
            for _ in range(5):
                ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        torch.cuda.synchronize()
        reps = 200
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        t0 = time.perf_counter()
        for _ in range(reps):
            ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        issue_us = (time.perf_counter() - t0) / reps * 1e6
        b.record(s)
        torch.cuda.synchronize()
        host_us = a.elapsed_time(b) / reps * 1e3
        ds.kernel_time()
        ds.set_profiling(True)
        for _ in range(20):
            ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        torch.cuda.synchronize()
        ds.set_profiling(False)
        km, kl = ds.kernel_time()
        kern_us = km / max(kl, 1) * 1e3
        graph_us = float("nan")
        if os.environ.get("HBG_HIST_PROFILE"):
            import ctypes as C

            st = (C.c_ulonglong * 8)()
            hbg.check(hbg.lib().hbg_debug_hist_stamps(ds.handle, st))
            t = [x - st[0] if x else -1 for x in st]
            print(f"    stamps ns (CTA 0): cleared {t[1]} rows {t[2]} partials {t[3]} barrier {t[4]} loads {t[6]} reduced {t[5]}")
        if os.environ.get("LEAF_FLOOR_NO_GRAPH"):
            print(f"D{depth:2d} rows {m:9d}  host_loop_us {host_us:8.1f}  kernel_us {kern_us:8.1f}", flush=True)
            continue
        try:
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                for _ in range(10):
                    ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, torch.cuda.current_stream().cuda_stream)
            with torch.cuda.stream(s):  # replay on s, where the events are recorded
                gr.replay()
                torch.cuda.synchronize()
                a.record(s)
                for _ in range(20):
                    gr.replay()
                b.record(s)
            torch.cuda.synchronize()
            graph_us = a.elapsed_time(b) / 200 * 1e3
        except Exception as e:  # noqa: BLE001
            print("graph capture failed:", str(e)[:120])
        print(f"D{depth:2d} rows {m:9d}  host_loop_us {host_us:8.1f}  issue_us {issue_us:6.1f}  graph_us {graph_us:8.1f}"
              f"  kernel_us {kern_us:8.1f}",
              flush=True)
    ds.close()


if __name__ == "__main__":
    main()
