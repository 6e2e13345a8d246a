#!/usr/bin/env python
"""BASELINE.json configs 1-5 on one B200, next to the reference CPU path.

Not the driver's bench line (bench.py is): a longer, one-off run whose JSON
results are committed under profiles/ (DESIGN.md §4). For every config the
GPU side runs through the library (libhbg.so); the CPU side is the unmodified
reference compiled from /root/reference (oracle/_ref) on all host cores.

    python bench_configs.py [--configs 1,2,3,4,5] [--out profiles/r01_configs.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import paper_1706_08359_b200 as hbg  # noqa: E402
from bench import algorithmic_bytes, hbm_peak, synthetic  # noqa: E402


def events_ms(fn, reps, stream):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        out = fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


def gpu_hist_and_tree(cols, g, h, k, stream, trees=2, leaves=255, min_data=1):
    n = cols.shape[1]
    d = cols.shape[0]
    sp = stream.cuda_stream
    res = {}
    with hbg.Dataset(cols, k) as ds:
        tg = torch.from_numpy(g.astype(np.float32)).cuda()
        th = torch.from_numpy(h.astype(np.float32)).cuda()
        idx = torch.arange(n, dtype=torch.int32, device="cuda")
        hist = torch.empty(ds.hist_values(), dtype=torch.float64, device="cuda")
        build = lambda: ds.build_histograms_device(idx, n, tg, th, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        for _ in range(3):
            build()
        ds.kernel_time()
        ds.set_profiling(True)
        ms, _ = events_ms(build, 20, stream)
        km, kl = ds.kernel_time()
        bits = 4 if k <= 16 else 8
        alg = algorithmic_bytes(n, d, k, bits)
        res["root_hist"] = {"ms": ms, "kernel_ms": km / kl, "rows_features_per_s": n * d / (ms / 1e3),
                            "kernel_alg_GBps": alg / (km / kl / 1e3) / 1e9,
                            "roofline_frac": alg / (km / kl / 1e3) / 1e9 / hbm_peak()[0]}
        ds.grow_tree(tg, th, leaves, min_data, 0.0, sp)
        ms, (log, nodes) = events_ms(lambda: ds.grow_tree(tg, th, leaves, min_data, 0.0, sp), trees, stream)
        km, kl = ds.kernel_time()
        ds.set_profiling(False)
        built = n + int(np.minimum(log["left_count"], log["right_count"])[:-1].sum())
        res["tree"] = {"sec_per_tree": ms / 1e3, "leaves": leaves, "splits": int(len(log)),
                       "hist_kernel_ms_per_tree": km / trees, "rows_built": built,
                       "rows_features_per_s_built": built * d / (ms / 1e3)}
        res["_log"] = log
    return res


def bits64_tree_parity(cols, g, h, k, leaves=255, min_data=1):
    """The PrecisionMode::bits64 device tree against the unmodified reference's
    bits64 grow_tree on the same data: identical splits until the first fp64
    tie (the two choices' exactly-summed gains equal to 1e-12), which is what
    tests/test_gpu_precision.py requires."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from oracle import ffi
    from test_gpu_parity import exact_gain, rows_of_node

    with hbg.Dataset(cols, k) as ds:
        t0 = time.perf_counter()
        log, nodes = ds.grow_tree_host(g, h, leaves, min_data, 0.0, precision=64)
        t_gpu = time.perf_counter() - t0
    rd = ffi.RefDataset(cols, k)
    t_ref, rlog = rd.grow_tree_timed(g, h, leaves, min_data, 0.0, 64)
    rd.close()
    _, rnodes = ffi.grow_tree(cols, k, g, h, leaves, min_data, 0.0, 64)
    same = 0
    while (same < min(len(log), len(rlog)) and log["feature"][same] == rlog["feature"][same]
           and log["threshold_bin"][same] == rlog["threshold_bin"][same]
           and log["left_count"][same] == rlog["left_count"][same]):
        same += 1
    out = {"splits_identical": same, "splits_total": int(len(rlog)), "gpu_host_dropin_s": t_gpu,
           "cpu_reference_s": t_ref}
    if same < len(rlog):
        jo = int(np.nonzero(nodes["left"] == 2 * same + 1)[0][0])
        jr = int(np.nonzero(np.asarray(rnodes["left"]) == 2 * same + 1)[0][0])
        ours = exact_gain(cols, g, h, rows_of_node(cols, nodes, jo), int(log["feature"][same]),
                          int(log["threshold_bin"][same]), 0.0)
        # every split before `same` agreed, so leaf jr has the same rows in both trees
        ref = exact_gain(cols, g, h, rows_of_node(cols, nodes, jr), int(rlog["feature"][same]),
                         int(rlog["threshold_bin"][same]), 0.0)
        out["first_divergence_exact_gains"] = [ours, ref]
        out["first_divergence_is_fp64_tie"] = bool(abs(ours - ref) <= 1e-12 * max(1.0, abs(ref)))
    return out


def cpu_reference(cols, g, h, k, leaves=255, min_data=1, tree=True):
    from oracle import ffi

    rd = ffi.RefDataset(cols, k)
    n, d = cols.shape[1], cols.shape[0]
    leaf = rd.leaf(np.arange(n, dtype=np.int32), g, h)
    t = min(rd.build_timed(leaf, 32)[0] for _ in range(3))
    out = {"cores": ffi.ref().ref_worker_count(), "root_hist_s": t, "root_rows_features_per_s": n * d / t}
    rd.free_leaf(leaf)
    if tree:
        tt, log = rd.grow_tree_timed(g, h, leaves, min_data, 0.0, 32)
        out["tree_s"] = tt
        out["_log"] = log
    rd.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--out", default=os.path.join(REPO, "profiles", "r02_configs.json"))
    ap.add_argument("--expo-rows", type=int, default=250_000_000)
    args = ap.parse_args()
    want = {int(c) for c in args.configs.split(",")}
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    results = {"gpu": torch.cuda.get_device_name(0), "hbm_peak_GBps": hbm_peak()[0]}

    def record(name, gpu, cpu):
        glog, clog = gpu.pop("_log", None), cpu.pop("_log", None) if cpu else None
        entry = {"gpu": gpu, "cpu_reference": cpu}
        if glog is not None and clog is not None:
            same = 0
            while (same < min(len(glog), len(clog)) and glog["feature"][same] == clog["feature"][same]
                   and glog["threshold_bin"][same] == clog["threshold_bin"][same]
                   and glog["left_count"][same] == clog["left_count"][same]):
                same += 1
            # vs the reference's bits32 run; with min_data_in_leaf=1 tiny leaves
            # produce fp32-level near-ties, after which the trees legitimately
            # diverge (tests/test_gpu_parity.py checks those are ties)
            entry["splits_identical_before_first_divergence"] = same
            entry["splits_total"] = int(len(clog))
        if cpu and "tree_s" in cpu:
            entry["tree_speedup_vs_cpu"] = cpu["tree_s"] / gpu["tree"]["sec_per_tree"]
        if cpu:
            entry["root_hist_speedup_vs_cpu"] = cpu["root_hist_s"] / (gpu["root_hist"]["ms"] / 1e3)
        results[name] = entry
        print(name, json.dumps(entry), flush=True)

    if 1 in want:  # Higgs 1M x 28, k64, 255-leaf tree (the CPU parity config)
        cols, g, h = synthetic(1_000_000, 28, 64, 1)
        record("config1_higgs_1Mx28_k64", gpu_hist_and_tree(cols, g, h, 64, stream), cpu_reference(cols, g, h, 64))
        results["config1_higgs_1Mx28_k64"]["bits64_tree"] = bits64_tree_parity(cols, g, h, 64)
    if 2 in want:  # Higgs 10.5M x 28: 16-bin 4-bit vs 64-bin 8-bit
        for k in (16, 64):
            cols, g, h = synthetic(10_500_000, 28, k, 2)
            record(f"config2_higgs_10.5Mx28_k{k}", gpu_hist_and_tree(cols, g, h, k, stream),
                   cpu_reference(cols, g, h, k))
            results[f"config2_higgs_10.5Mx28_k{k}"]["bits64_tree"] = bits64_tree_parity(cols, g, h, k)
    if 3 in want:  # epsilon 400K x 2000, k64: one full boosting iteration
        cols, g, h = synthetic(400_000, 2000, 64, 3)
        gpu = gpu_hist_and_tree(cols, g, h, 64, stream, trees=1)
        rng = np.random.default_rng(3)
        targets = rng.normal(size=400_000)
        with hbg.Dataset(cols, 64) as ds:
            ts = torch.from_numpy(targets).cuda()
            sc = torch.zeros(400_000, dtype=torch.float64, device="cuda")
            ds.boost_one_iteration(ts, sc, hbg.HBG_LOSS_SQUARED, 0.1, 255, 1, 0.0, stream=stream.cuda_stream)
            ms, _ = events_ms(lambda: ds.boost_one_iteration(ts, sc, hbg.HBG_LOSS_SQUARED, 0.1, 255, 1, 0.0,
                                                             stream=stream.cuda_stream), 2, stream)
        gpu["boost_iteration_s"] = ms / 1e3
        cpu = cpu_reference(cols, g, h, 64, tree=False)
        from oracle import ffi

        rd = ffi.RefDataset(cols, 64)
        scores = np.zeros(400_000)
        cpu["boost_iteration_s"] = rd.boost_one_iteration_timed(targets, scores, 0, 0.1, 255, 1, 0.0, 32)
        rd.close()
        record("config3_epsilon_400Kx2000_k64", gpu, cpu)
        results["config3_epsilon_400Kx2000_k64"]["boost_speedup_vs_cpu"] = cpu["boost_iteration_s"] / gpu["boost_iteration_s"]
    if 4 in want:  # Bosch 1M x 968, k256, sparse-ish (bin 0 w.p. 0.8), dense path on both sides
        rng = np.random.default_rng(4)
        cols = rng.integers(1, 256, size=(968, 1_000_000), dtype=np.uint8)
        cols[rng.random(size=cols.shape) < 0.8] = 0
        g = 2 * rng.random(1_000_000) - 1
        h = rng.random(1_000_000)
        record("config4_bosch_1Mx968_k256", gpu_hist_and_tree(cols, g, h, 256, stream, trees=1),
               cpu_reference(cols, g, h, 256))
    if 5 in want:  # Expo-scale 250M x 28, k64 on one GPU (the 8-GPU scaling baseline)
        n = args.expo_rows
        rng = np.random.default_rng(5)
        cols = rng.integers(1, 64, size=(28, n), dtype=np.uint8)
        g = (2 * rng.random(n, dtype=np.float32) - 1).astype(np.float64)
        h = rng.random(n, dtype=np.float32).astype(np.float64)
        record(f"config5_expo_{n}x28_k64_1gpu", gpu_hist_and_tree(cols, g, h, 64, stream, trees=1), None)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(results, f, indent=1)


if __name__ == "__main__":
    main()
