"""GPU parity of the two PrecisionMode paths (histogram_set.hpp:11) at the
BASELINE configurations, against the oracle's bits64.

* bits64 (HBG_PRECISION_BITS64): fp64 g/h in HBM, fp64 per-warp cells, fp64
  partials — held to the reference's own stats_tolerance(bits64) = 1e-12
  (histogram_set.hpp:33-35) at every size, the 10.5M-row root included, and
  255-leaf trees grown with it must equal the reference's bits64 tree split
  for split at the BASELINE shapes (1M and 10.5M x 28, k=64/16, min_data 1,
  lambda 0: the configs[0]/[1] trees) up to the first fp64 tie
  (exactly-summed gains equal to 1e-12).
* bits32 (the fast path): its 255-leaf trees at the same shapes equal the
  reference's bits64 tree up to the first divergence, and that divergence
  must be a near-tie (exactly-summed gains within 1e-6) — fp32 inputs cannot
  order closer candidates (_assert_same_tree).
"""
import numpy as np
import pytest

from test_gpu_parity import _assert_same_tree, _grow, make_case, max_rel_err, torch_cuda

pytestmark = pytest.mark.gpu

TOL64 = 1e-12  # stats_tolerance(PrecisionMode::bits64), histogram_set.hpp:33-35


def assert_bits64(got, want):
    assert (got["count"] == want["count"]).all(), "counts must be bit-exact"
    for key in ("grad_sum", "hess_sum"):
        err = max_rel_err(got[key], want[key])
        assert err <= TOL64, (key, err)


@pytest.mark.parametrize("k,d", [(64, 28), (16, 28), (256, 37), (64, 1), (128, 33), (2, 5), (16, 70)])
@pytest.mark.parametrize("depth", [0, 3, 8])
def test_bits64_host_dropin_meets_reference_bits64_tolerance(hbg, oracle, k, d, depth):
    rows = 60000
    cols, g, h, idx = make_case(oracle, rows, d, k, depth, seed=3 * d + k)
    leaf = hbg.gather_leaf_statistics(idx, g, h)
    with hbg.Dataset(cols, k) as ds:
        got = hbg.build_histograms_partitioned(ds, leaf, precision=64)
        fast = hbg.build_histograms_partitioned(ds, leaf, precision=32)
    want = oracle.build_histograms(cols, k, idx, leaf.gradients, leaf.hessians, 64)
    assert_bits64(got, want)
    assert (fast["count"] == got["count"]).all()


def test_bits64_edge_cases(hbg, oracle):
    rng = np.random.default_rng(5)
    cols = rng.integers(0, 64, size=(28, 1000), dtype=np.uint8)
    cols[3, :] = 63
    with hbg.Dataset(cols, 64) as ds:
        empty = hbg.build_histograms_partitioned(
            ds, hbg.LeafState(np.zeros(0, np.int32), np.zeros(0), np.zeros(0)), precision=64)
        assert (empty["count"] == 0).all() and (empty["grad_sum"] == 0).all()
        for n in (1, 31, 33, 999):
            idx = np.sort(rng.choice(1000, n, replace=False)).astype(np.int32)
            g = rng.normal(size=n) * 1e3  # large magnitudes: fp64 keeps every digit
            h = 1e-9 + rng.random(n) * 1e-6  # tiny hessians (logistic late in boosting)
            got = hbg.build_histograms_partitioned(ds, hbg.LeafState(idx, g, h), precision=64)
            want = oracle.build_histograms(cols, 64, idx, g, h, 64)
            assert_bits64(got, want)
            nz = want["hess_sum"] != 0
            rel = np.abs(got["hess_sum"][nz] - want["hess_sum"][nz]) / np.abs(want["hess_sum"][nz])
            assert rel.max() <= 1e-13  # relative, not just the floor-1 predicate
        with pytest.raises(hbg.InvalidArgument):
            hbg.build_histograms_partitioned(ds, hbg.LeafState(np.arange(3, dtype=np.int32), np.zeros(3),
                                                               np.zeros(3)), precision=16)


@pytest.mark.parametrize("k", [64, 16])
def test_full_size_root_bits64(hbg, oracle, k):
    """10.5M x 28 (BASELINE configs[1]) root through the fp64 device builder:
    counts exact, sums within 1e-12 of the reference's bits64, deterministic."""
    torch = torch_cuda()
    rows, d = 10_500_000, 28
    cols = oracle.gen_synthetic_bins(rows, d, k, 0)
    g, h = oracle.gen_grad_hess(rows, 0)
    dev = torch.device("cuda:0")
    with hbg.Dataset(cols, k) as ds:
        tg = torch.from_numpy(g).to(dev)
        th = torch.from_numpy(h).to(dev)
        outs = []
        for _ in range(2):
            out = torch.empty(ds.hist_values(), dtype=torch.float64, device=dev)
            ds.build_histograms_device_f64(None, rows, tg, th, out, hbg.HBG_GH_LEAF_ALIGNED, 0)
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy())
    assert outs[0].tobytes() == outs[1].tobytes()
    o = outs[0].reshape(3, d, k)
    want = oracle.build_histograms(cols, k, np.arange(rows, dtype=np.int32), g, h, 64)
    assert (o[2].astype(np.int64) == want["count"]).all()
    for j, key in ((0, "grad_sum"), (1, "hess_sum")):
        err = max_rel_err(o[j], want[key])
        assert err <= TOL64, (key, err)


def test_bits64_host_dropin_pageable_and_pinned_agree(hbg, oracle):
    """bits64 host drop-in: pinned arrays go up as they are, pageable ones
    through the host pool's fp64 stage (ids held back while every chunk is one
    range) — the same bytes either way, and within 1e-12 of the oracle."""
    torch = torch_cuda()
    rng = np.random.default_rng(41)
    rows, d, k = 2_400_000, 28, 64
    cols = rng.integers(0, k, size=(d, rows), dtype=np.uint8)

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    with hbg.Dataset(cols, k) as ds:
        for idx in (np.arange(rows, dtype=np.int32),
                    np.arange(11, 2_000_011, dtype=np.int32),
                    np.sort(rng.choice(rows, 1_500_000, replace=False)).astype(np.int32),
                    np.concatenate([np.arange(1_200_000), np.arange(1_200_005, 2_300_000)]).astype(np.int32)):
            g, h = rng.normal(size=len(idx)), rng.random(len(idx))
            a = hbg.build_histograms_partitioned(ds, hbg.LeafState(idx, g, h), precision=64)
            page_h2d, _ = ds.host_copy_bytes()
            b = hbg.build_histograms_partitioned(ds, hbg.LeafState(pinned(idx), pinned(g), pinned(h)), precision=64)
            assert a.tobytes() == b.tobytes()
            contiguous = bool((np.diff(idx) == 1).all())
            assert page_h2d == 16 * len(idx) + (0 if contiguous else 4 * len(idx))
        want = oracle.build_histograms(cols, k, idx, g, h, 64)
        assert_bits64(a, want)
        g, h = rng.normal(size=rows), rng.random(rows)  # the tree drop-in's bits64 upload, both ways
        ta = ds.grow_tree_host(g, h, 31, 100, 0.0, precision=64)
        tb = ds.grow_tree_host(pinned(g), pinned(h), 31, 100, 0.0, precision=64)
        assert ta[0].tobytes() == tb[0].tobytes() and ta[1].tobytes() == tb[1].tobytes()


def _baseline_case(oracle, rows, k):
    cols = oracle.gen_synthetic_bins(rows, 28, k, 0)
    g, h = oracle.gen_grad_hess(rows, 0)
    return cols, g, h


@pytest.mark.parametrize("rows,k", [(1_000_000, 64), (10_500_000, 64), (1_000_000, 16), (10_500_000, 16)])
def test_bits64_tree_matches_reference_at_baseline_shapes(hbg, oracle, rows, k):
    """The 255-leaf tree of BASELINE configs[0]/[1] (min_data 1, lambda 0 —
    noise gains down to 1-row leaves, the hardest case for ordering) grown in
    bits64 equals the reference's bits64 tree split for split until the first
    fp64 TIE: the two choices' exactly-summed gains agree to 1e-12 (measured:
    two features cutting a 9- or 26-row leaf into the same two row sets, the
    reference's pick decided by the last bit of its sequential sums). Every
    split before it: same feature, threshold, counts and node ids, gains to
    1e-10."""
    cols, g, h = _baseline_case(oracle, rows, k)
    with hbg.Dataset(cols, k) as ds:
        log, nodes = ds.grow_tree_host(g, h, 255, 1, 0.0, precision=64)
    want_log, want_nodes = oracle.grow_tree(cols, k, g, h, 255, 1, 0.0, 64)
    same = _assert_same_tree(log, nodes, want_log, want_nodes, cols, g, h, 0.0, tie_tol=1e-12)
    assert np.allclose(log["gain"][:same], want_log["gain"][:same], rtol=1e-10, atol=0)
    print(f"bits64 {rows}x28 k{k}: {same} of {len(want_log)} splits identical before the first fp64 tie")
    # the same tree through the fp64 device entry point
    torch = torch_cuda()
    dev = torch.device("cuda:0")
    with hbg.Dataset(cols, k) as ds:
        log2, nodes2 = ds.grow_tree_f64(torch.from_numpy(g).to(dev), torch.from_numpy(h).to(dev), 255, 1, 0.0)
    assert log2.tobytes() == log.tobytes() and nodes2.tobytes() == nodes.tobytes()


@pytest.mark.parametrize("rows,k", [(1_000_000, 64), (10_500_000, 64)])
@pytest.mark.parametrize("grower", ["auto", "legacy"])
def test_bits32_tree_at_baseline_shapes_diverges_only_at_near_ties(hbg, oracle, rows, k, grower, monkeypatch):
    """The fast path's 255-leaf trees at the BASELINE shapes (persistent
    growers: the wave kernel chosen for these shapes, and the one-split
    kernel) against the reference's bits64 tree: identical until the first
    divergence, which must be an fp64 near-tie."""
    cols, g, h = _baseline_case(oracle, rows, k)
    if grower != "auto":
        monkeypatch.setenv("HBG_GROW", grower)
    with hbg.Dataset(cols, k) as ds:
        log, nodes = _grow(hbg, ds, g, h, 255, 1, 0.0)
    want_log, want_nodes = oracle.grow_tree(cols, k, g, h, 255, 1, 0.0, 64)
    same = _assert_same_tree(log, nodes, want_log, want_nodes, cols, g, h, 0.0)
    print(f"bits32 {rows}x28 k{k} ({grower}): {same} of {len(want_log)} splits identical before the first near-tie")
