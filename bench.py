#!/usr/bin/env python
"""bench.py — histogram build throughput on B200 (BASELINE.json metric).

Metric: histogram build rows·features/s (whole job). One *step* = one pass of
the hot path over one leaf: the device histogram of a Higgs-shaped
10.5M x 28, 64-bin, 8-bit-packed leaf (BASELINE.json configs[1], the root
leaf of its tree), read from leaf indices + leaf-aligned fp32 g/h already
resident in HBM, plus (N > 1) the NCCL allreduce of the leaf histogram across
row shards (weak scaling: every rank owns a 10.5M-row shard).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hbg|reference]

Extra keys beyond the base contract:
  roofline     — the histogram kernel's algorithmic bytes / its CUDA-event
                 duration vs MEASURED_PEAKS.json hbm_gbs
  cpu_baseline — the unmodified reference build_histograms_partitioned(bits32)
                 (oracle/_ref, compiled from /root/reference) on all host cores
  e2e          — the same metric through the host C-ABI call with pinned host
                 buffers (H2D of indices/g/h and D2H of the histogram inside)
  variants     — the 16-bin 4-bit kernel on the same rows, and deeper leaves
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

ROWS = 10_500_000
FEATURES = 28
SEED_STEP = 0x51ED270B


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["hbg", "reference"], default="hbg")
    ap.add_argument("--rows", type=int, default=ROWS)
    ap.add_argument("--rows-total", type=int, default=0,
                    help="strong scaling: this many rows in total, sharded over the ranks (sec/tree per N)")
    ap.add_argument("--features", type=int, default=FEATURES)
    ap.add_argument("--max-bin", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--no-tree", action="store_true")
    ap.add_argument("--num-leaves", type=int, default=255)
    ap.add_argument("--trees", type=int, default=3)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def synthetic(rows: int, d: int, k: int, seed: int):
    """Bench inputs with the reference generator's distribution (bench.cpp:17-38,
    69-73): bins uniform in [1, k-1], g = 2u - 1, h = u. numpy-generated; the
    cpu_baseline leg times the reference on these same bytes."""
    rng = np.random.default_rng(seed)
    cols = rng.integers(1, k, size=(d, rows), dtype=np.uint8)
    u = rng.random(rows)
    g = 2.0 * u - 1.0
    h = rng.random(rows)
    return cols, g, h


def leaf_sample(rows: int, depth: int, seed: int) -> np.ndarray:
    """Sorted random leaf rows of size rows >> depth (bench.cpp:40-57 shape)."""
    if depth == 0:
        return np.arange(rows, dtype=np.int32)
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(rows, rows >> depth, replace=False)).astype(np.int32)


def workload_config(n: int, total: int, d: int, k: int, world: int, strong: bool) -> dict:
    """The bench line's `config`, identical for both arms (the driver compares them)."""
    bits = 4 if k <= 16 else 8
    workload = f"higgs-{total}x{d}-k{k}-root-leaf" + (f"-sharded{world}" if strong and world > 1 else "")
    return {
        "workload": workload, "rows_per_gpu": n, "rows_total": total, "features": d, "max_bin": k,
        "bits_per_bin": bits, "leaf_depth": 0, "leaf": "explicit int32 indices + leaf-aligned g/h (the root LeafState)",
        "l2": f"inputs {(n * (d * bits / 8 + 12)) / 1e6:.0f} MB > 126 MB L2; no flush needed",
        "parallelism": f"row-sharded x{world}",
    }


def algorithmic_bytes(n: int, d: int, k: int, bits: int) -> float:
    """B = N_r (d b/8 + 12) + 12 d k per histogram pass."""
    return n * (d * bits / 8.0 + 12.0) + 12.0 * d * k


def hbm_peak():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(workload: str):
    """dram bytes per histogram-kernel launch from the committed ncu capture
    (scripts/ncu_summary.py), or None when there is none or it was taken of
    different kernel sources (stamp mismatch: the number would be stale)."""
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            t = json.load(f).get(workload)
        from paper_1706_08359_b200 import hist_kernel_stamp

        if isinstance(t, dict) and t.get("kernel_src") == hist_kernel_stamp():
            return float(t["dram_bytes"])
    except Exception:
        pass
    return None


class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML while the GPU works."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples = []
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - informational only
            self.err = str(e)
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz, r))
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self, t0: float, t1: float):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        window = "timed region"
        if len(inside) < 3:
            inside = self.samples
            window = "warmup+timed+variants window (timed region too short for NVML sampling)"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "note": "no samples"}
        reasons = set()
        for _, _, r in inside:
            for bit, name in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[1] for s in inside), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(inside), "window": window}


# ------------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    from oracle import ffi

    if not ffi.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhistoboost_ref.so not built"}))
        return
    # the hbg arm's whole job at this world size (weak: rows per GPU x N; strong: rows_total)
    world = dist_env()[1]
    strong = args.rows_total > 0
    n, d, k = args.rows_total if strong else world * args.rows, args.features, args.max_bin
    cols, g, h = synthetic(n, d, k, seed=0)
    idx = leaf_sample(n, 0, 0)
    rd = ffi.RefDataset(cols, k)
    leaf = rd.leaf(idx, g, h)
    cores = ffi.ref().ref_worker_count()
    for _ in range(args.warmup):
        rd.build_timed(leaf, precision=32)
    times = [rd.build_timed(leaf, precision=32)[0] for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = n * d / (ms / 1e3)
    unit = "rows*features/s"
    line = {
        "metric": "histogram build rows*features/sec", "value": value, "unit": unit, "impl": "reference",
        # the same job shape as our arm's line (N = the launch's world size);
        # the reference itself runs on the host cores of rank 0 (`cpu_baseline`)
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy, reference generator distribution)",
        "config": workload_config((args.rows_total if strong else n) // world, n, d, k, world, strong),
        "reference": {"precision": "bits32", "path": "build_histograms_partitioned (unmodified reference, oracle/_ref)",
                      "rows": n},
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} root-leaf builds of the {n}x{d} k{k} workload"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    rd.free_leaf(leaf)
    rd.close()
    print(json.dumps(line))


# ----------------------------------------------------------------------- hbg arm
def run_hbg(args):
    import torch
    import torch.distributed as dist

    import paper_1706_08359_b200 as hbg

    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"# note: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    # Development check of the N > 1 plumbing on a one-GPU box: every rank on
    # the same device (their contexts time-slice), torch.distributed over gloo,
    # no NCCL (it refuses two ranks on one GPU), the CUDA-IPC peer path only.
    shared_gpu = os.environ.get("HBG_BENCH_SHARED_GPU") is not None and world > 1
    if shared_gpu:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = torch.device("cpu") if shared_gpu else dev  # tensors the collectives reduce
    if world > 1:
        if shared_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    n, d, k = args.rows, args.features, args.max_bin
    strong = args.rows_total > 0
    if strong:  # fixed total work: rank r owns its shard of rows_total rows (dist.shard_rows)
        from paper_1706_08359_b200.dist import shard_rows

        b0, e0 = shard_rows(args.rows_total, rank, world)
        n = e0 - b0
    total = args.rows_total if strong else world * n
    bits = 4 if k <= 16 else 8
    cols, g, h = synthetic(n, d, k, seed=rank)
    idx = leaf_sample(n, 0, rank)

    ds = hbg.Dataset(cols, k, device=local)
    ti = torch.from_numpy(idx).to(dev)
    tg = torch.from_numpy(g.astype(np.float32)).to(dev)
    th = torch.from_numpy(h.astype(np.float32)).to(dev)
    hist = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
    # A real (non-default) stream: the C ABI maps a NULL stream to the handle's
    # own stream, and the CUDA events must sit on the stream the kernels run on.
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream

    comm = None
    if world > 1 and not shared_gpu:  # NCCL communicator of the library (the sharded allreduce hook)
        uid = [hbg.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = hbg.Comm(world, rank, uid[0], local)

    # N > 1: every rank maps every rank's exchange area (CUDA IPC); the
    # per-leaf cross-rank sum is then fused into the histogram's reduction
    # kernel over NVLink peer memory. NCCL (the allreduce hook) is the
    # fallback, chosen by all ranks together if any rank cannot map or run it.
    peer = None
    exchange = "none (single rank)"
    if world > 1:
        ok = torch.ones(1, device=red_dev)
        try:
            peer = hbg.Peer(ds, world, rank, 0, args.num_leaves)
            handles = [None] * world
            dist.all_gather_object(handles, peer.ipc_handle())
            for r in range(world):
                if r != rank:
                    peer.open(r, handles[r])
            ds.build_histograms_peer(ti, n, tg, th, hist, peer, stream=sp)
            peer.check()
        except Exception as e:  # noqa: BLE001 — reported in the JSON line
            ok.zero_()
            exchange = f"NCCL allreduce (peer path failed: {str(e)[:80]})"
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 0:
            if peer is not None:
                peer.close()
            peer = None
            if comm is None:
                raise RuntimeError(f"peer exchange unavailable and no NCCL fallback: {exchange}")
            if exchange.startswith("none"):
                exchange = "NCCL allreduce (peer path failed on another rank)"
        else:
            exchange = "fused into the reduction kernel over NVLink peer memory (hbg_build_histograms_peer)"

    def step():
        if peer is not None:
            ds.build_histograms_peer(ti, n, tg, th, hist, peer, stream=sp)
            return
        ds.build_histograms_device(ti, n, tg, th, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        if comm is not None:  # the per-leaf exchange of row-sharded training (NCCL over NVLink)
            hbg.check(hbg.lib().hbg_comm_allreduce(hbg._ptr(hist), hist.numel(), hbg._ptr(sp), comm.handle))

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ds.kernel_time()  # clear
    ds.set_profiling(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    if world > 1:
        dist.barrier()
    ds.set_profiling(False)
    ms_total = e0.elapsed_time(e1)
    kern_ms, launches = ds.kernel_time()
    ms_step = torch.tensor([ms_total / args.steps], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(ms_step, op=dist.ReduceOp.MAX)
    ms_step = float(ms_step.item())
    value = total * d / (ms_step / 1e3)

    # --- roofline of the dominant kernel (the histogram kernel)
    kern_avg_s = kern_ms / max(launches, 1) / 1e3
    alg = algorithmic_bytes(n, d, k, bits)
    peak, peak_src = hbm_peak()
    achieved = alg / kern_avg_s / 1e9 if kern_avg_s > 0 else 0.0
    cfg = workload_config(n, total, d, k, world, strong)
    workload = cfg["workload"]

    result = {
        "metric": "histogram build rows*features/sec",
        "value": value,
        "unit": "rows*features/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (numpy; reference generator distribution: bins U[1,k-1], g=2u-1, h=u)",
        "config": cfg,
        "exchange": exchange,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(workload), "kernel": "hist_kernel<8,64>" if bits == 8 else "hist_kernel<4,16>",
            "kernel_ms": kern_avg_s * 1e3, "algorithmic_bytes_per_launch": alg, "peak_source": peak_src,
        },
        "gpu_launches": 2 * args.steps,
    }

    # --- e2e through the host C-ABI drop-in (pinned host buffers)
    e2e_steps = max(1, min(args.steps, 30))  # host-side noise: a longer mean
    pin_idx = torch.from_numpy(idx).pin_memory().numpy()
    pin_g = torch.from_numpy(g).pin_memory().numpy()
    pin_h = torch.from_numpy(h).pin_memory().numpy()
    leaf = hbg.LeafState(pin_idx, pin_g, pin_h)
    # warm-up: the workspace, and the host side (the staging pool's first
    # passes over the caller's arrays run ~20% slower: page walks, core clocks)
    for _ in range(max(args.warmup, 10)):
        hbg.build_histograms_partitioned(ds, leaf)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    calls = []
    for _ in range(e2e_steps):
        tc = time.perf_counter()
        out = hbg.build_histograms_partitioned(ds, leaf)
        calls.append((time.perf_counter() - tc) * 1e3)
    e2e_ms = torch.tensor([sum(calls) / len(calls)], dtype=torch.float64, device=red_dev)  # the mean (the value)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    pin_h2d, pin_d2h = ds.host_copy_bytes()
    # the same call with pageable arrays (numpy, like the reference's
    # std::vectors): staged as fp32 by the library's host pool (informational)
    page_leaf = hbg.LeafState(np.array(idx), np.array(g, dtype=np.float64), np.array(h, dtype=np.float64))
    for _ in range(max(args.warmup, 10)):
        hbg.build_histograms_partitioned(ds, page_leaf)
    t0p = time.perf_counter()
    for _ in range(e2e_steps):
        hbg.build_histograms_partitioned(ds, page_leaf)
    page_ms = (time.perf_counter() - t0p) * 1e3 / e2e_steps
    result["e2e"] = {
        "value": total * d / (e2e_ms / 1e3), "unit": "rows*features/s",
        # counted by the library: each staged chunk of g/h goes as host-
        # converted fp32 (8 B/row) or fp64 (16 B/row, converted on the
        # device); a contiguous leaf (the root) uploads no row ids
        "h2d_bytes_per_step": pin_h2d, "d2h_bytes_per_step": pin_d2h,
        "ms_per_step": e2e_ms,
        "ms_per_call_median": float(np.median(calls)), "ms_per_call_min": float(min(calls)),
        "api": "hbg_build_histograms (host LeafState arrays: int32 indices, fp64 g/h)"
               + ("; per rank, the cross-rank sum not included" if world > 1 else ""),
        "steps": e2e_steps,
        "pageable_ms_per_step": page_ms,
    }
    # a depth-1 leaf (half the rows, random and sorted: bench.cpp's leaf
    # shape) through the same drop-in: its row ids travel too (informational)
    i1 = leaf_sample(n, 1, 101)
    leaf1 = hbg.LeafState(torch.from_numpy(i1).pin_memory().numpy(), torch.from_numpy(g[i1]).pin_memory().numpy(),
                          torch.from_numpy(h[i1]).pin_memory().numpy())
    for _ in range(max(args.warmup, 10)):
        hbg.build_histograms_partitioned(ds, leaf1)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        hbg.build_histograms_partitioned(ds, leaf1)
    d1_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    result["e2e"]["depth1_leaf"] = {"rows": int(len(i1)), "ms_per_step": d1_ms,
                                    "rows_features_per_s": len(i1) * d / (d1_ms / 1e3),
                                    "h2d_bytes_per_step": ds.host_copy_bytes()[0]}

    # --- variants (informational): 4-bit 16-bin kernel, deeper leaves
    if not args.no_variants:
        var = {}
        for depth in (2, 4, 6, 8, 10, 12):
            li = torch.from_numpy(leaf_sample(n, depth, 100 + depth)).to(dev)
            m = len(li)
            lg = torch.empty(m, dtype=torch.float32, device=dev)
            lh = torch.empty(m, dtype=torch.float32, device=dev)
            tot = torch.empty(2, dtype=torch.float64, device=dev)
            hbg.gather_leaf_device(li, m, tg, th, lg, lh, tot, sp)
            for _ in range(3):
                ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
            reps = 100
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                ds.build_histograms_device(li, m, lg, lh, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / reps
            var[f"k{k}_D{depth}"] = {"rows": m, "ms": t, "rows_features_per_s": m * d / (t / 1e3),
                                     "alg_GBps": algorithmic_bytes(m, d, k, bits) / (t / 1e3) / 1e9}
        # PrecisionMode::bits64 on the same root: fp64 g/h in HBM, fp64 cells and
        # partials (the exact mode; 16 B/row of g/h instead of 8)
        tg64 = torch.from_numpy(g.astype(np.float64)).to(dev)
        th64 = torch.from_numpy(h.astype(np.float64)).to(dev)
        for _ in range(3):
            ds.build_histograms_device_f64(ti, n, tg64, th64, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        ds.kernel_time()
        ds.set_profiling(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        a.record(stream)
        for _ in range(reps):
            ds.build_histograms_device_f64(ti, n, tg64, th64, hist, hbg.HBG_GH_LEAF_ALIGNED, sp)
        b.record(stream)
        torch.cuda.synchronize()
        ds.set_profiling(False)
        t = a.elapsed_time(b) / reps
        km, kl = ds.kernel_time()
        alg64 = n * (d * bits / 8.0 + 20.0) + 12.0 * d * k  # int32 id + fp64 g + fp64 h
        var[f"k{k}_bits64_D0"] = {"rows": n, "ms": t, "rows_features_per_s": n * d / (t / 1e3),
                                  "kernel_ms": km / max(kl, 1),
                                  "kernel_alg_GBps": alg64 / (km / max(kl, 1) / 1e3) / 1e9,
                                  "precision": "bits64 (fp64 g/h, cells and partials)"}
        del tg64, th64
        if k != 16:
            cols16 = (cols % 15 + 1).astype(np.uint8)
            ds16 = hbg.Dataset(cols16, 16, device=local)
            h16 = torch.empty(ds16.hist_values(), dtype=torch.float64, device=dev)
            for _ in range(3):
                ds16.build_histograms_device(ti, n, tg, th, h16, hbg.HBG_GH_LEAF_ALIGNED, sp)
            ds16.set_profiling(True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 50
            a.record(stream)
            for _ in range(reps):
                ds16.build_histograms_device(ti, n, tg, th, h16, hbg.HBG_GH_LEAF_ALIGNED, sp)
            b.record(stream)
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / reps
            km, kl = ds16.kernel_time()
            kt = km / max(kl, 1)
            var["k16_4bit_D0"] = {"rows": n, "ms": t, "rows_features_per_s": n * d / (t / 1e3),
                                  "kernel_ms": kt,
                                  "kernel_alg_GBps": algorithmic_bytes(n, d, 16, 4) / (kt / 1e3) / 1e9,
                                  "roofline_frac": algorithmic_bytes(n, d, 16, 4) / (kt / 1e3) / 1e9 / peak}
            ds16.close()
        result["variants"] = var
    # --- sec/tree: device-resident 255-leaf best-first tree (grow_tree semantics);
    # row-sharded over the ranks when N > 1: the per-split histogram exchange
    # runs inside the persistent grower over NVLink peer memory (CUDA IPC
    # mappings of every rank's exchange area); the NCCL-hook host loop is the
    # other sharded path, used only if the peer mapping is unavailable
    if not args.no_tree:
        tree_path = "persistent kernel, single rank"
        if world > 1:
            tree_path = ("persistent kernel, in-kernel peer-memory histogram exchange (NVLink)" if peer is not None
                         else "host loop + NCCL allreduce hook (peer mapping unavailable)")

        def grow():
            if world == 1:
                return ds.grow_tree(tg, th, args.num_leaves, 1, 0.0, sp)
            if peer is not None:
                return ds.grow_tree_peer(tg, th, peer, args.num_leaves, 1, 0.0, sp)
            return ds.grow_tree_sharded(tg, th, comm.allreduce_fn, comm.handle, args.num_leaves, 1, 0.0, sp)

        if peer is not None:  # warm-up through the peer path; every rank falls back together on failure
            ok = torch.ones(1, device=red_dev)
            try:
                grow()
            except Exception as e:  # noqa: BLE001 — reported in the JSON line
                ok.zero_()
                tree_path = f"host loop + NCCL allreduce hook (peer path failed: {str(e)[:80]})"
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() == 0:
                peer.close()
                peer = None
                if "host loop" not in tree_path:
                    tree_path = "host loop + NCCL allreduce hook (peer path failed on another rank)"
        log, _ = grow()  # warm-up (workspace)
        ds.kernel_time()
        ds.set_profiling(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a.record(stream)
        for _ in range(args.trees):
            log, nodes = grow()
        b.record(stream)
        torch.cuda.synchronize()
        ds.set_profiling(False)
        t_tree = torch.tensor([a.elapsed_time(b) / args.trees / 1e3], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t_tree, op=dist.ReduceOp.MAX)
        t_tree = float(t_tree.item())
        km, kl = ds.kernel_time()
        built = total + int(np.minimum(log["left_count"], log["right_count"])[: max(len(log) - 1, 0)].sum())
        result["tree"] = {
            "num_leaves": args.num_leaves, "splits": int(len(log)), "sec_per_tree": t_tree,
            "rows_total": total,
            "hist_rows_built": built, "hist_launches_per_tree": kl / args.trees,
            "hist_kernel_ms_per_tree": km / args.trees,
            "rows_features_per_s_built": built * d / t_tree,
            "note": "root + smaller child of every split (larger by subtraction); all splits in one persistent cooperative kernel (grow_persistent.cu)",
            "path": tree_path,
        }
        if world == 1:
            # end to end through the whole-tree drop-in (hbg_grow_tree_host):
            # host fp64 g/h (pinned) in, split log + nodes out, H2D inside
            pg64 = torch.from_numpy(g.astype(np.float64)).pin_memory().numpy()
            ph64 = torch.from_numpy(h.astype(np.float64)).pin_memory().numpy()
            ds.grow_tree_host(pg64, ph64, args.num_leaves, 1, 0.0)
            t0 = time.perf_counter()
            for _ in range(args.trees):
                ds.grow_tree_host(pg64, ph64, args.num_leaves, 1, 0.0)
            result["tree"]["e2e_sec_per_tree"] = (time.perf_counter() - t0) / args.trees
            result["tree"]["e2e_api"] = "hbg_grow_tree_host (host fp64 g/h: staged chunks as fp32, a share of pinned chunks as fp64; split log + nodes D2H)"
            g64, h64 = g.astype(np.float64), h.astype(np.float64)  # pageable: the host-staged fp32 path
            ds.grow_tree_host(g64, h64, args.num_leaves, 1, 0.0)
            t0 = time.perf_counter()
            for _ in range(args.trees):
                ds.grow_tree_host(g64, h64, args.num_leaves, 1, 0.0)
            result["tree"]["e2e_pageable_sec_per_tree"] = (time.perf_counter() - t0) / args.trees
    clocks.stop()
    result["clocks"] = clocks.summary(t_wall0, t_wall1)

    # --- CPU baseline: the unmodified reference on this box's host cores (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ffi

            if ffi.ref_available():
                rd = ffi.RefDataset(cols, k)
                rleaf = rd.leaf(idx, g, h)
                rd.build_timed(rleaf, precision=32)
                ts = [rd.build_timed(rleaf, precision=32)[0] for _ in range(args.cpu_reps)]
                cpu_s = sum(ts) / len(ts)
                result["cpu_baseline"] = {
                    "value": n * d / cpu_s, "unit": "rows*features/s", "cores": ffi.ref().ref_worker_count(),
                    "kind": "reference",
                    "sample": f"{args.cpu_reps} root-leaf build_histograms_partitioned(bits32) calls on the same "
                              f"{n}x{d} k{k} bins/g/h (mean {cpu_s * 1e3:.1f} ms)",
                }
                rd.free_leaf(rleaf)
                if not args.no_tree:
                    t_ref, _ = rd.grow_tree_timed(g, h, args.num_leaves, 1, 0.0, 32)
                    result["cpu_baseline"]["tree"] = {
                        "sec_per_tree": t_ref, "sample": f"1 grow_tree({args.num_leaves} leaves, bits32) on the same data"}
                    if "tree" in result:
                        result["tree"]["cpu_reference_sec_per_tree"] = t_ref
                rd.close()
            else:
                result["cpu_baseline"] = None
        except Exception as e:  # informational leg; never masks the GPU number
            result["cpu_baseline"] = {"error": str(e)}
    if peer is not None:
        peer.close()
    ds.close()
    if comm is not None:
        comm.close()
    if rank == 0:
        print(json.dumps(result))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_hbg(args)


if __name__ == "__main__":
    main()
