"""Row-sharded host logic at world_size 2 over gloo (CPU-only).

Each rank computes its shard's leaf histogram with the oracle (standing in
for the device kernel, which needs a GPU), the ranks allreduce the SoA fp64
histogram exactly as bench.py / the sharded path does over NCCL, and the
result must equal the unsharded histogram: counts exact, sums within 1e-12,
bit-identical on both ranks, and both ranks pick the same split.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_08359_b200 import dist as hdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import ffi

    rows, d, k = 30011, 9, 64
    cols = ffi.gen_synthetic_bins(rows, d, k, 3)
    g, h = ffi.gen_grad_hess(rows, 3)
    leaf = ffi.leaf_index_sample(rows, 2, 77)
    begin, end = hdist.shard_rows(rows, rank, world)
    local = hdist.local_leaf(leaf, begin, end)
    shard_cols = np.ascontiguousarray(cols[:, begin:end])
    part = ffi.build_histograms(shard_cols, k, local, g[begin:end][local], h[begin:end][local], 64)
    soa = torch.from_numpy(hdist.bins_to_soa(part).copy())
    hdist.allreduce_histogram(soa)
    full = hdist.soa_to_bins(soa.numpy(), ffi.BIN_DTYPE)
    gt = float(g[leaf].sum())
    ht = float(h[leaf].sum())
    split = ffi.find_best_split(full, gt, ht, len(leaf))
    np.save(os.path.join(out_dir, f"hist{rank}.npy"), soa.numpy())
    np.save(os.path.join(out_dir, f"split{rank}.npy"), np.array([split["feature"], split["threshold_bin"]]))
    dist.destroy_process_group()


def test_shard_rows_partition():
    for n in (0, 1, 7, 100, 10_500_000):
        for w in (1, 2, 3, 8):
            spans = [hdist.shard_rows(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        hdist.shard_rows(10, 2, 2)


def test_local_leaf_rebases_rows():
    leaf = np.array([0, 3, 5, 9, 12], dtype=np.int32)
    assert hdist.local_leaf(leaf, 0, 6).tolist() == [0, 3, 5]
    assert hdist.local_leaf(leaf, 6, 13).tolist() == [3, 6]


def test_two_rank_allreduce_equals_unsharded(tmp_path, oracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    h0 = np.load(tmp_path / "hist0.npy")
    h1 = np.load(tmp_path / "hist1.npy")
    assert h0.tobytes() == h1.tobytes()  # every rank holds the identical histogram
    rows, d, k = 30011, 9, 64
    cols = oracle.gen_synthetic_bins(rows, d, k, 3)
    g, h = oracle.gen_grad_hess(rows, 3)
    leaf = oracle.leaf_index_sample(rows, 2, 77)
    want = oracle.build_histograms(cols, k, leaf, g[leaf], h[leaf], 64)
    got = hdist.soa_to_bins(h0, oracle.BIN_DTYPE)
    assert (got["count"] == want["count"]).all()
    assert np.allclose(got["grad_sum"], want["grad_sum"], rtol=1e-12, atol=1e-12)
    assert np.allclose(got["hess_sum"], want["hess_sum"], rtol=1e-12, atol=1e-12)
    s0 = np.load(tmp_path / "split0.npy")
    s1 = np.load(tmp_path / "split1.npy")
    assert (s0 == s1).all()
    sw = oracle.find_best_split(want, float(g[leaf].sum()), float(h[leaf].sum()), len(leaf))
    assert (s0[0], s0[1]) == (sw["feature"], sw["threshold_bin"])
