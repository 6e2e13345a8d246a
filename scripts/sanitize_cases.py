"""Small GPU cases run under compute-sanitizer (scripts/sanitize.sh).

    python scripts/sanitize_cases.py CASE

CASE: smoke | hist | leafseq | dropin | tree_wave | tree_onesplit | tree_host | tree_bits64 | peer2
Each case is small (the tools replay every memory access), checks its result
against the oracle, and exits 0 on success.
"""
import os
import sys
import threading

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def tree(grower, precision=32, rows=20000, d=28, k=64, leaves=63):
    import paper_1706_08359_b200 as hbg
    from oracle import ffi

    os.environ["HBG_GROW"] = grower
    cols = ffi.gen_synthetic_bins(rows, d, k, 1)
    g, h = ffi.gen_grad_hess(rows, 1)
    g = g + 0.3 * (cols[3].astype(np.float64) > k // 2)
    with hbg.Dataset(cols, k) as ds:
        log, nodes = ds.grow_tree_host(g, h, leaves, 40, 0.0, precision=precision)
    want, _ = ffi.grow_tree(cols, k, g, h, leaves, 40, 0.0, 64)
    assert (log["feature"] == want["feature"]).all() and (log["threshold_bin"] == want["threshold_bin"]).all()
    print(f"tree {grower} bits{precision}: {len(log)} splits identical to the oracle")


def hist():
    import paper_1706_08359_b200 as hbg
    from oracle import ffi

    for rows, d, k, depth in ((50000, 28, 64, 0), (50000, 28, 64, 3), (40000, 40, 16, 1), (5000, 9, 256, 0)):
        cols = ffi.gen_synthetic_bins(rows, d, k, 2)
        g, h = ffi.gen_grad_hess(rows, 2)
        idx = ffi.leaf_index_sample(rows, depth, 7)
        leaf = hbg.gather_leaf_statistics(idx, g, h)
        with hbg.Dataset(cols, k) as ds:
            for prec in (32, 64):
                got = hbg.build_histograms_partitioned(ds, leaf, precision=prec)
                want = ffi.build_histograms(cols, k, idx, leaf.gradients, leaf.hessians, 64)
                assert (got["count"] == want["count"]).all()
    print("hist: counts exact on 4 shapes x 2 precisions")


def leafseq():
    """Leaves of alternating sizes on one dataset: cluster, multi-cluster and
    two-launch plans (multi-cluster plans share per-dataset counters)."""
    import paper_1706_08359_b200 as hbg
    from oracle import ffi

    rows, d, k = 400_000, 28, 64
    cols = ffi.gen_synthetic_bins(rows, d, k, 21)
    g, h = ffi.gen_grad_hess(rows, 21)
    rng = np.random.default_rng(3)
    with hbg.Dataset(cols, k) as ds:
        for n in (rows, 100_000, 3_000, 60_000, 400, 250_000):
            idx = np.sort(rng.choice(rows, n, replace=False)).astype(np.int32)
            leaf = hbg.gather_leaf_statistics(idx, g, h)
            got = hbg.build_histograms_partitioned(ds, leaf)
            want = ffi.build_histograms(cols, k, idx, leaf.gradients, leaf.hessians, 64)
            assert (got["count"] == want["count"]).all()
    print("leafseq: counts exact on 6 leaf sizes")


def dropin():
    """The host drop-in with pageable and pinned LeafState arrays: staged fp32
    and fp64-direct chunks, contiguous (iota) and uploaded row ids."""
    import torch

    import paper_1706_08359_b200 as hbg
    from oracle import ffi

    rows, d, k = 1_200_000, 28, 64
    cols = ffi.gen_synthetic_bins(rows, d, k, 5)
    g, h = ffi.gen_grad_hess(rows, 5)
    rng = np.random.default_rng(5)
    with hbg.Dataset(cols, k) as ds:
        for idx in (np.arange(rows, dtype=np.int32), np.sort(rng.choice(rows, 900_000, replace=False)).astype(np.int32)):
            lg, lh = g[idx], h[idx]
            a = hbg.build_histograms_partitioned(ds, hbg.LeafState(idx, lg, lh))
            pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (idx, lg, lh)]
            b = hbg.build_histograms_partitioned(ds, hbg.LeafState(*pin))
            assert a.tobytes() == b.tobytes()
            want = ffi.build_histograms(cols, k, idx, lg, lh, 64)
            assert (a["count"] == want["count"]).all()
    print("dropin: pageable and pinned identical, counts exact")


def peer2():
    """Two ranks as threads on one GPU exchanging through peer memory."""
    import torch

    import paper_1706_08359_b200 as hbg
    from oracle import ffi

    rows, d, k, leaves, world = 30000, 28, 64, 31, 2
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cols = ffi.gen_synthetic_bins(rows, d, k, 6)
    g, h = ffi.gen_grad_hess(rows, 6)
    cuts = [0, rows // 3, rows]
    dss = [hbg.Dataset(np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]), k) for r in range(world)]
    peers = [hbg.Peer(dss[r], world, r, ctas=sms // world) for r in range(world)]
    gh = [(torch.from_numpy(g[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda(),
           torch.from_numpy(h[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda()) for r in range(world)]
    peers[0].attach(peers[1])
    peers[1].attach(peers[0])
    torch.cuda.synchronize()
    res, errs = [None] * world, []

    def run(r):
        try:
            res[r] = dss[r].grow_tree_peer(gh[r][0], gh[r][1], peers[r], leaves, 100, 0.0, dss[r].stream())
        except Exception as ex:
            errs.append(ex)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for p in peers:
        p.close()
    for ds in dss:
        ds.close()
    assert not errs, errs
    assert res[0][0].tobytes() == res[1][0].tobytes()
    want, _ = ffi.grow_tree(cols, k, g, h, leaves, 100, 0.0, 64)
    assert (res[0][0]["feature"] == want["feature"]).all()
    print(f"peer2: {len(want)} splits identical on both ranks and to the oracle")


def main():
    case = sys.argv[1]
    if case == "smoke":
        import __graft_entry__

        __graft_entry__.smoke()
    elif case == "hist":
        hist()
    elif case == "tree_wave":
        tree("wave")
    elif case == "tree_onesplit":
        tree("legacy")
    elif case == "tree_host":
        tree("host")
    elif case == "tree_bits64":
        tree("host", precision=64)
    elif case == "leafseq":
        leafseq()
    elif case == "dropin":
        dropin()
    elif case == "peer2":
        peer2()
    else:
        raise SystemExit(f"unknown case {case}")


if __name__ == "__main__":
    main()
