"""Root histogram of a BASELINE config shape (bench_configs.py's data), for
ncu captures of the histogram kernel on the other configs.

    python scripts/prof_config_root.py bosch|bosch_uniform|epsilon|higgs16 [reps]

e.g. ncu --set full -k regex:hist_kernel -c 1 -o gpurun_out/bosch \
       python scripts/prof_config_root.py bosch 1
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1706_08359_b200 as hbg  # noqa: E402


def data(name):
    if name == "bosch":  # 1M x 968, k256, bin 0 w.p. 0.8 (bench_configs.py config 4)
        rng = np.random.default_rng(4)
        cols = rng.integers(1, 256, size=(968, 1_000_000), dtype=np.uint8)
        cols[rng.random(size=cols.shape) < 0.8] = 0
        return cols, 256
    if name == "bosch_uniform":  # same shape, uniform bins
        rng = np.random.default_rng(4)
        return rng.integers(0, 256, size=(968, 1_000_000), dtype=np.uint8), 256
    if name == "epsilon":  # 400K x 2000, k64
        rng = np.random.default_rng(3)
        return rng.integers(0, 64, size=(2000, 400_000), dtype=np.uint8), 64
    if name == "higgs16":  # 10.5M x 28, k16 (4-bit slices)
        rng = np.random.default_rng(2)
        return rng.integers(0, 16, size=(28, 10_500_000), dtype=np.uint8), 16
    raise SystemExit(f"unknown shape {name}")


def main():
    name = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cols, k = data(name)
    n = cols.shape[1]
    rng = np.random.default_rng(0)
    tg = torch.from_numpy((2 * rng.random(n) - 1).astype(np.float32)).cuda()
    th = torch.from_numpy(rng.random(n).astype(np.float32)).cuda()
    idx = torch.arange(n, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with hbg.Dataset(cols, k) as ds:
        hist = torch.empty(ds.hist_values(), dtype=torch.float64, device="cuda")
        ds.set_profiling(True)
        for _ in range(reps):
            ds.build_histograms_device(idx, n, tg, th, hist, hbg.HBG_GH_LEAF_ALIGNED, s.cuda_stream)
        torch.cuda.synchronize()
        km, kl = ds.kernel_time()
        print(f"{name}: {n} x {cols.shape[0]} k{k}: hist kernel {km / max(kl, 1):.3f} ms/launch over {kl} launches")


if __name__ == "__main__":
    main()
