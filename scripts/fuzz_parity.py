"""Randomised parity sweep against the oracle (development aid; the pytest
suite holds the fixed cases). Runs until the time budget is spent:

    python scripts/fuzz_parity.py [seconds] [seed]

Each case draws a shape (features 1-80, max_bin 2-256, rows 1-300K), a leaf
(contiguous range, sorted or unsorted subset, duplicates-free), a precision
and an API route (host drop-in with pageable or pinned arrays, device API),
and checks counts bit-exact and sums within the reference's stats_tolerance
relative to each bin's sum of |terms| (1e-5 bits32 / 1e-12 bits64) against
the oracle's bits64; every fourth case also a tree (2-63 leaves, random
min_data and lambda) against the oracle's bits64 tree: bits64 trees (fp64
host loop) up to true ties (1e-12), bits32 trees (device growers on fp32 g/h)
up to near-ties (1e-5), their gains and leaf values not compared (fp32
rounding of cancelling sums).
Prints one line per failure and a summary; exit status 1 on any failure.
"""
import os
import sys
import time
import traceback

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
import paper_1706_08359_b200 as hbg  # noqa: E402
from oracle import ffi  # noqa: E402
from test_gpu_parity import _assert_same_tree  # noqa: E402


MAX_ROWS = int(os.environ.get("FUZZ_MAX_ROWS", "300000"))  # > 2M rows: several staged and histogram chunks


def leaf_of(rng, rows):
    kind = rng.integers(0, 4)
    if rows == 0:
        return np.zeros(0, dtype=np.int32), "empty"
    if kind == 0:
        a = int(rng.integers(0, rows))
        b = int(rng.integers(a, rows)) + 1
        return np.arange(a, b, dtype=np.int32), "range"
    m = int(rng.integers(1, rows + 1))
    idx = rng.choice(rows, m, replace=False).astype(np.int32)
    if kind == 1:
        return idx, "unsorted"
    return np.sort(idx), "sorted"


def pinned(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()


def one_case(rng, case):
    d = int(rng.integers(1, 81))
    k = int(rng.choice([2, 3, 4, 7, 16, 17, 32, 64, 100, 128, 200, 256]))
    rows = int(rng.choice([1, 31, 1000, int(rng.integers(1, MAX_ROWS + 1))]))
    cols = rng.integers(0, k, size=(d, rows), dtype=np.uint8)
    if rng.random() < 0.3:  # skewed columns
        cols[rng.random(cols.shape) < 0.8] = 0
    g = rng.normal(size=rows) * (10.0 ** rng.integers(-6, 4))
    h = rng.random(rows) * (10.0 ** rng.integers(-6, 3))
    idx, kind = leaf_of(rng, rows)
    prec = int(rng.choice([32, 64]))
    route = str(rng.choice(["pageable", "pinned", "device"]))
    tol = 1e-12 if prec == 64 else 1e-5  # relative to the bin's sum of |terms|
    desc = f"case {case}: d={d} k={k} rows={rows} leaf={kind}({len(idx)}) bits{prec} {route}"
    want = ffi.build_histograms(cols, k, idx, g[idx], h[idx], 64)
    # error scale of a bin's sum: the sum of its terms' magnitudes (a sum's
    # rounding error is bounded relative to that, not to the sum itself,
    # which may cancel)
    mag = ffi.build_histograms(cols, k, idx, np.abs(g[idx]), np.abs(h[idx]), 64)
    with hbg.Dataset(cols, k) as ds:
        if route == "device" and prec == 32 and len(idx) > 0:
            dev = torch.device("cuda:0")
            li = torch.from_numpy(idx).to(dev)
            lg = torch.from_numpy(g[idx].astype(np.float32)).to(dev)
            lh = torch.from_numpy(h[idx].astype(np.float32)).to(dev)
            out = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
            ds.build_histograms_device(li, len(idx), lg, lh, out, hbg.HBG_GH_LEAF_ALIGNED, 0)
            torch.cuda.synchronize()
            o = out.cpu().numpy().reshape(3, d, k)
            got_c, got_g, got_h = o[2].astype(np.int64), o[0], o[1]
        else:
            leaf = hbg.LeafState(idx, g[idx], h[idx])
            if route == "pinned":
                leaf = hbg.LeafState(pinned(idx), pinned(g[idx]), pinned(h[idx]))
            got = hbg.build_histograms_partitioned(ds, leaf, precision=prec)
            got_c = got["count"].reshape(d, k)
            got_g = got["grad_sum"].reshape(d, k)
            got_h = got["hess_sum"].reshape(d, k)
        wc = want["count"].reshape(d, k)
        assert (got_c == wc).all(), desc + ": counts differ"
        for name, a, b, m in (("grad", got_g, want["grad_sum"].reshape(d, k), mag["grad_sum"].reshape(d, k)),
                              ("hess", got_h, want["hess_sum"].reshape(d, k), mag["hess_sum"].reshape(d, k))):
            err = float((np.abs(a - b) / np.maximum(m, 1e-300)).max()) if a.size else 0.0
            assert err <= tol, f"{desc}: {name} err {err:.3g} of the bin's sum of |terms| > {tol}"
        if case % 4 == 0 and rows >= 2:
            # trees on moderate magnitudes: fp32 inputs (bits32 semantics) cannot
            # order candidates or value leaves of extreme, cancelling data closer
            # than their rounding, which the tie check does not model
            g = rng.normal(size=rows)
            h = 0.05 + rng.random(rows)
            leaves = int(rng.integers(2, 64))
            min_data = int(rng.choice([1, 5, 50]))
            lam = float(rng.choice([0.0, 0.5]))
            tprec = int(rng.choice([32, 64]))
            if tprec == 64:  # fp64 everywhere (the host loop): equal up to true ties
                log, nodes = ds.grow_tree_host(g, h, leaves, min_data, lam, precision=64)
            else:  # the device growers on fp32 g/h (the default choice or a forced one)
                grower = str(rng.choice(["", "wave", "legacy", "host", "persistent"]))
                if grower:
                    os.environ["HBG_GROW"] = grower
                else:
                    os.environ.pop("HBG_GROW", None)
                desc += f" grower={grower or 'default'}"
                dev = torch.device("cuda:0")
                tg = torch.from_numpy(g.astype(np.float32)).to(dev)
                th = torch.from_numpy(h.astype(np.float32)).to(dev)
                log, nodes = ds.grow_tree(tg, th, leaves, min_data, lam)
            desc += f" tree bits{tprec}"
            wl, wn = ffi.grow_tree(cols, k, g, h, leaves, min_data, lam, 64)
            try:
                _assert_same_tree(log, nodes, wl, wn, cols, g, h, lam, tie_tol=1e-12 if tprec == 64 else 1e-5)
            except AssertionError as e:
                n = min(len(log), len(wl))
                why = "?"
                for i in range(n):
                    if not all(log[f][i] == wl[f][i] for f in ("feature", "threshold_bin", "left_count")):
                        why = (f"split {i}: ours {log[i][['feature', 'threshold_bin', 'left_count', 'gain']]} "
                               f"ref {wl[i][['feature', 'threshold_bin', 'left_count', 'gain']]}")
                        break
                    if np.nonzero(nodes["left"] == 2 * i + 1)[0].tolist() != np.nonzero(np.asarray(wn["left"]) == 2 * i + 1)[0].tolist():
                        why = f"split {i}: different leaf split (same feature/threshold/count)"
                        break
                    if log["right_count"][i] != wl["right_count"][i]:
                        why = f"split {i}: right_count {log['right_count'][i]} vs {wl['right_count'][i]}"
                        break
                    if abs(log["gain"][i] - wl["gain"][i]) > 1e-5 * max(1.0, abs(wl["gain"][i])):
                        why = f"split {i}: gain {log['gain'][i]!r} vs {wl['gain'][i]!r}"
                        break
                else:
                    if len(log) != len(wl):
                        why = f"split counts {len(log)} vs {len(wl)}"
                    else:
                        vo, vr = nodes["value"], np.asarray(wn["value"])
                        rel = np.abs(vo - vr) / np.maximum(np.abs(vr), 1e-300)
                        j = int(np.argmax(rel))
                        why = f"leaf values: node {j} {vo[j]!r} vs {vr[j]!r}"
                info = f"{desc} tree(leaves={leaves}, min_data={min_data}, lam={lam}): {e!r}; {why}"
                if tprec == 32 and (why.startswith("leaf values") or ": gain " in why):
                    return desc  # fp32 inputs: gains/values of cancelling sums differ beyond 1e-5 (not a decision)
                raise AssertionError(info) from None
    return desc


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    t0 = time.time()
    n = fails = 0
    while time.time() - t0 < budget:
        try:
            one_case(rng, n)
        except Exception as e:  # noqa: BLE001
            fails += 1
            print("FAIL", str(e)[:300], flush=True)
            traceback.print_exc(limit=2)
        n += 1
    print(f"fuzz: {n} cases, {fails} failures, seed {seed}, {time.time() - t0:.0f} s", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
