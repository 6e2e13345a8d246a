#!/usr/bin/env python
"""Summarise an ncu capture (.ncu-rep) of the histogram kernel into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof1.ncu-rep profiles/r01_hist_k64_v1 \
        --workload higgs-10500000x28-k64-root-leaf --alg-bytes 420021504

Writes <out>.json (selected raw metrics + derived numbers) and <out>.txt (a
human-readable digest), and records dram bytes per launch in
profiles/ncu_traffic.json under --workload (bench.py reports it as
roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "smsp__cycles_active.avg",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
]


def to_float(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--workload", default=None)
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--kernel", default="hist_kernel")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = [r for r in rows[2:] if args.kernel in r[hdr.index("Kernel Name")]]
    assert launches, f"no {args.kernel} launch in {args.rep}"
    r = launches[-1]
    m = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            m[k] = {"value": to_float(r[i]), "unit": units[i]}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = m["dram__bytes_read.sum"]
    wr = m["dram__bytes_write.sum"]
    traffic = rd["value"] * scale.get(rd["unit"], 1) + wr["value"] * scale.get(wr["unit"], 1)
    dur = m["gpu__time_duration.sum"]
    dur_s = dur["value"] * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(dur["unit"], 1e-9)
    derived = {"dram_bytes_per_launch": traffic, "duration_s_cold": dur_s,
               "kernel": r[hdr.index("Kernel Name")]}
    if args.alg_bytes:
        derived["algorithmic_bytes"] = args.alg_bytes
        derived["traffic_over_algorithmic"] = traffic / args.alg_bytes
        derived["alg_GBps_cold"] = args.alg_bytes / dur_s / 1e9
    sh = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", {}).get("value")
    if isinstance(sh, float):
        derived["shared_wavefronts"] = sh
    out = {"source": os.path.basename(args.rep), "metrics": m, "derived": derived}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    with open(args.out + ".txt", "w") as f:
        f.write(f"# ncu --set full digest of {derived['kernel']}\n# from {args.rep}\n")
        for k, v in m.items():
            f.write(f"{k:85s} {v['value']} {v['unit']}\n")
        for k, v in derived.items():
            f.write(f"{k:85s} {v}\n")
    if args.workload:
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
        t = {}
        if os.path.exists(p):
            with open(p) as f:
                t = json.load(f)
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_1706_08359_b200 import hist_kernel_stamp

        t[args.workload] = {"dram_bytes": traffic, "kernel_src": hist_kernel_stamp(),
                            "capture": os.path.basename(args.rep)}
        with open(p, "w") as f:
            json.dump(t, f, indent=1)
    print(json.dumps(derived, indent=1))


if __name__ == "__main__":
    main()
