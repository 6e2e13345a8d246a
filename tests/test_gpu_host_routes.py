"""The host drop-in's upload routes (capi.cu stage_chunks / direct_chunks):
every staged chunk goes either as host-converted fp32 or — for pinned arrays —
as fp64 converted on the device, and chunks whose row ids form one range read
the resident iota instead of uploaded ids. The route mix depends on
HBG_PINNED_DMA_FRAC and the pool size on HBG_HOST_THREADS (both read once per
process), so other settings run in subprocesses; every setting must give the
same bytes."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1706_08359_b200 as hbg
rng = np.random.default_rng(31)
rows = 2_300_000
cols = rng.integers(0, 64, size=(28, rows), dtype=np.uint8)
g, h = rng.normal(size=rows), rng.random(rows)
idx_sets = [np.arange(rows, dtype=np.int32),
            np.sort(rng.choice(rows, 1_700_000, replace=False)).astype(np.int32),
            np.concatenate([np.arange(900_000), np.arange(900_003, 2_200_000)]).astype(np.int32)]
out = []
with hbg.Dataset(cols, 64) as ds:
    for idx in idx_sets:
        lg, lh = g[idx], h[idx]
        out.append(hbg.build_histograms_partitioned(ds, hbg.LeafState(idx, lg, lh)).tobytes())
        pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (idx, lg, lh)]
        out.append(hbg.build_histograms_partitioned(ds, hbg.LeafState(*pin)).tobytes())
    pg, ph = (torch.from_numpy(x).pin_memory().numpy() for x in (g, h))
    log, nodes = ds.grow_tree_host(pg, ph, 31, 100, 0.0)
    out.append(log.tobytes() + nodes.tobytes())
np.save(sys.argv[2], np.frombuffer(b"".join(out), dtype=np.uint8))
"""


def _run(tmp_path, tag, env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = tmp_path / f"{tag}.npy"
    subprocess.run([sys.executable, "-c", CHILD, REPO, str(out)], check=True, env=env, timeout=600)
    return np.load(out)


def test_upload_routes_bit_identical(tmp_path):
    base = _run(tmp_path, "default", {})
    for tag, env in (("all_staged", {"HBG_PINNED_DMA_FRAC": "0"}),
                     ("all_direct", {"HBG_PINNED_DMA_FRAC": "1"}),
                     ("half_direct_1thread", {"HBG_PINNED_DMA_FRAC": "0.5", "HBG_HOST_THREADS": "1"}),
                     ("odd_pool", {"HBG_HOST_THREADS": "7"})):
        got = _run(tmp_path, tag, env)
        assert got.shape == base.shape and (got == base).all(), tag


def test_contiguous_leaf_past_the_last_row_is_rejected(hbg_mod=None):
    """Row ids outside the dataset fail with std::invalid_argument — a
    contiguous range (read from the resident ids, never uploaded) and
    scattered ids (checked by the staging pass) — on the pageable and pinned
    routes and both precisions; the handle stays usable."""
    import torch

    sys.path.insert(0, REPO)
    import paper_1706_08359_b200 as hbg

    rows = 1_200_000
    rng = np.random.default_rng(8)
    cols = rng.integers(0, 64, size=(28, rows), dtype=np.uint8)
    with hbg.Dataset(cols, 64) as ds:
        for pin in (False, True):
            idx = np.arange(rows - 600_000, rows + 600_000, dtype=np.int32)
            g, h = rng.normal(size=len(idx)), rng.random(len(idx))
            if pin:
                idx, g, h = (torch.from_numpy(x).pin_memory().numpy() for x in (idx, g, h))
            with pytest.raises(hbg.InvalidArgument):
                hbg.build_histograms_partitioned(ds, hbg.LeafState(idx, g, h))
            # scattered ids with one past the last row: the staging pass's range check
            bad = np.sort(rng.choice(rows, 700_000, replace=False)).astype(np.int32)
            bad[-1] = rows
            gb, hb = rng.normal(size=len(bad)), rng.random(len(bad))
            if pin:
                bad, gb, hb = (torch.from_numpy(x).pin_memory().numpy() for x in (bad, gb, hb))
            for prec in (32, 64):
                with pytest.raises(hbg.InvalidArgument):
                    hbg.build_histograms_partitioned(ds, hbg.LeafState(bad, gb, hb), precision=prec)
        ok = np.arange(10, 500_010, dtype=np.int32)
        out = hbg.build_histograms_partitioned(ds, hbg.LeafState(ok, rng.normal(size=len(ok)), rng.random(len(ok))))
        assert int(out["count"].sum()) == len(ok) * 28
