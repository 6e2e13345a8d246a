"""Row-sharded tree growth on one GPU with an in-process collective (GPU).

Only one GPU is available to the tests, so the N-GPU path is exercised the
way the reference tests distribution without a cluster: two
"ranks" run as threads, each owning a row shard (its own hbg Dataset) and
calling hbg_grow_tree_sharded; the allreduce hook is a fake collective that
sums the ranks' device buffers in rank order with hbg_reduce_histograms_device
(the reduce_private_histograms analogue) and hands the sum back to both. The
sharded trees must be identical on both ranks and equal the reference's tree
on the unsharded data. hbg_comm_allreduce (NCCL) plugs into the same hook.
"""
import ctypes as C
import os
import threading

import numpy as np
import pytest

from paper_1706_08359_b200 import dist as hdist

pytestmark = pytest.mark.gpu


class FakeCollective:
    def __init__(self, hbg, world, max_values, torch):
        self.hbg = hbg
        self.world = world
        self.barrier = threading.Barrier(world)
        self.bufs = [None] * world
        self.tmp = torch.empty(max_values, dtype=torch.float64, device="cuda:0")
        self.calls = 0
        self.fns = [hbg.ALLREDUCE_FN(self._make(r)) for r in range(world)]

    def _make(self, rank):
        lib = self.hbg.lib()

        def cb(buf, n, stream, ctx):
            try:
                lib.hbg_stream_synchronize(stream)
                self.bufs[rank] = buf
                self.barrier.wait()
                if rank == 0:
                    self.calls += 1
                    parts = (C.c_void_p * self.world)(*self.bufs)
                    assert n <= self.tmp.numel()
                    lib.hbg_reduce_histograms_device(parts, self.world, n, C.c_void_p(self.tmp.data_ptr()), None)
                    lib.hbg_stream_synchronize(None)
                self.barrier.wait()
                lib.hbg_reduce_histograms_device((C.c_void_p * 1)(self.tmp.data_ptr()), 1, n, C.c_void_p(buf), stream)
                lib.hbg_stream_synchronize(stream)
                self.barrier.wait()
                return 0
            except Exception:  # never raise through the C boundary
                self.barrier.abort()
                return 5

        return cb


@pytest.mark.parametrize("rows,d,k,leaves,min_data", [(40000, 28, 64, 63, 50), (30001, 12, 16, 31, 100),
                                                     (20000, 9, 256, 31, 80)])
def test_two_rank_sharded_tree_equals_reference(hbg, oracle, rows, d, k, leaves, min_data):
    import torch

    world = 2
    cols = oracle.gen_synthetic_bins(rows, d, k, 5)
    g, h = oracle.gen_grad_hess(rows, 5)
    g = g + 0.3 * (cols[1].astype(np.float64) > k // 2)
    coll = FakeCollective(hbg, world, 3 * d * k + 64, torch)
    results = [None] * world
    errors = []

    def run(rank):
        try:
            b, e = hdist.shard_rows(rows, rank, world)
            with hbg.Dataset(np.ascontiguousarray(cols[:, b:e]), k) as ds:
                tg = torch.from_numpy(g[b:e].astype(np.float32)).cuda()
                th = torch.from_numpy(h[b:e].astype(np.float32)).cuda()
                s = torch.cuda.Stream()
                results[rank] = ds.grow_tree_sharded(tg, th, coll.fns[rank], None, leaves, min_data, 0.0,
                                                     s.cuda_stream)
        except Exception as ex:  # surfaced below
            errors.append(ex)
            coll.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    (log0, nodes0), (log1, nodes1) = results
    assert log0.tobytes() == log1.tobytes() and nodes0.tobytes() == nodes1.tobytes()  # identical on every rank
    want_log, want_nodes = oracle.grow_tree(cols, k, g, h, leaves, min_data, 0.0, 64)
    from test_gpu_parity import _assert_same_tree

    assert _assert_same_tree(log0, nodes0, want_log, want_nodes) == len(want_log)
    assert coll.calls >= len(log0) + 2  # root totals + root histogram + per-split child totals (+ histograms)


def test_nccl_comm_single_rank_tree(hbg, oracle, monkeypatch):
    """The NCCL hook itself (hbg_comm_*, dlopen'ed libnccl) on one rank: the
    sharded grower over a 1-rank communicator equals the unsharded host-loop
    grower bit for bit (same kernels, same order), and the persistent grower
    in structure (its fp64 totals are summed in a different fixed order)."""
    import torch

    monkeypatch.setenv("HBG_GROW", "host")
    cols = oracle.gen_synthetic_bins(30000, 16, 64, 8)
    g, h = oracle.gen_grad_hess(30000, 8)
    comm = hbg.Comm(1, 0, hbg.Comm.unique_id(), 0)
    try:
        with hbg.Dataset(cols, 64) as ds:
            tg = torch.from_numpy(g.astype(np.float32)).cuda()
            th = torch.from_numpy(h.astype(np.float32)).cuda()
            s = torch.cuda.Stream()
            a = ds.grow_tree_sharded(tg, th, comm.allreduce_fn, comm.handle, 63, 20, 0.0, s.cuda_stream)
            b = ds.grow_tree(tg, th, 63, 20, 0.0, s.cuda_stream)
            # the same boosting iteration through the hook
            ts = torch.from_numpy(g).cuda()
            s1 = torch.zeros(30000, dtype=torch.float64, device="cuda")
            s2 = torch.zeros(30000, dtype=torch.float64, device="cuda")
            ds.boost_one_iteration(ts, s1, hbg.HBG_LOSS_SQUARED, 0.1, 31, 20, 0.0, comm.allreduce_fn, comm.handle,
                                   s.cuda_stream)
            ds.boost_one_iteration(ts, s2, hbg.HBG_LOSS_SQUARED, 0.1, 31, 20, 0.0, stream=s.cuda_stream)
            monkeypatch.setenv("HBG_GROW", "persistent")
            c = ds.grow_tree(tg, th, 63, 20, 0.0, s.cuda_stream)
            torch.cuda.synchronize()
    finally:
        comm.close()
    assert a[0].tobytes() == b[0].tobytes() and a[1].tobytes() == b[1].tobytes()
    assert torch.equal(s1, s2)
    for key in ("feature", "threshold_bin", "left_count", "right_count"):
        assert (c[0][key] == a[0][key]).all(), key
    for key in ("feature", "threshold_bin", "left", "right"):
        assert (c[1][key] == a[1][key]).all(), key
    assert np.allclose(c[1]["value"], a[1]["value"], rtol=1e-9, atol=1e-12)
    assert np.allclose(c[0]["gain"], a[0]["gain"], rtol=1e-5)  # histograms: fp32 vs fixed-point rounding


@pytest.mark.parametrize("world,rows,d,k,leaves,min_data", [(2, 60000, 28, 64, 63, 60), (3, 50001, 12, 16, 31, 100),
                                                           (2, 30000, 9, 256, 31, 80), (2, 200000, 28, 64, 255, 200),
                                                           (2, 40000, 70, 64, 31, 100)])
def test_peer_exchange_sharded_tree_equals_reference(hbg, oracle, world, rows, d, k, leaves, min_data):
    """Row sharding INSIDE the persistent grower: `world` ranks as threads on
    one GPU, each a partial grid (SMs / world CTAs) over its own row shard,
    exchanging the smaller child's histogram chunks and the partition totals
    through each other's exchange areas (hbg_peer_attach; across processes the
    same areas are mapped with CUDA IPC). Trees identical on every rank and
    equal to the reference's tree on the unsharded data."""
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cols = oracle.gen_synthetic_bins(rows, d, k, 6)
    g, h = oracle.gen_grad_hess(rows, 6)
    g = g + 0.3 * (cols[1].astype(np.float64) > k // 2)
    # uneven shards: rank r gets a different share
    cuts = [0] + [int(rows * (r + 1) * (r + 2) / (world * (world + 1))) for r in range(world)]
    shards = [np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]) for r in range(world)]
    dss = [hbg.Dataset(shards[r], k) for r in range(world)]  # consecutive stream creation
    ctas = int(os.environ.get("HBG_TEST_CTAS", sms // world))  # the ranks split the SMs
    peers = [hbg.Peer(dss[r], world, r, ctas=ctas) for r in range(world)]
    grads = [(torch.from_numpy(g[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda(),
              torch.from_numpy(h[cuts[r]:cuts[r + 1]].astype(np.float32)).cuda()) for r in range(world)]
    for p in peers:
        for q in peers:
            if q is not p:
                p.attach(q)
    torch.cuda.synchronize()
    results = [None] * world
    errors = []

    def run(r):
        try:
            # each rank on its dataset's own stream: created consecutively, so
            # on distinct hardware queues and the ranks' grids run concurrently
            for _ in range(2):  # two trees: the generation tags and the done handshake
                results[r] = dss[r].grow_tree_peer(grads[r][0], grads[r][1], peers[r], leaves, min_data, 0.0,
                                                   dss[r].stream())
        except Exception as ex:  # surfaced below
            errors.append(ex)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for p in peers:
        p.close()
    for ds in dss:
        ds.close()
    assert not errors, errors
    for r in range(1, world):
        assert results[r][0].tobytes() == results[0][0].tobytes(), r  # identical split logs on every rank
        assert results[r][1].tobytes() == results[0][1].tobytes(), r
    want_log, want_nodes = oracle.grow_tree(cols, k, g, h, leaves, min_data, 0.0, 64)
    from test_gpu_parity import _assert_same_tree

    assert _assert_same_tree(results[0][0], results[0][1], want_log, want_nodes) == len(want_log)


@pytest.mark.parametrize("world,rows,d,k", [(2, 120000, 28, 64), (3, 50000, 40, 16), (2, 30000, 9, 256)])
def test_peer_histogram_allreduce_fused(hbg, oracle, world, rows, d, k):
    """hbg_build_histograms_peer: each rank builds the histogram of ITS rows of
    a leaf; the cross-rank sum is fused into the reduction kernel over peer
    memory. Every rank must hold the bit-identical global histogram, equal to
    the oracle's on the union of the ranks' rows (counts exact, sums 1e-5),
    including leaves of which some rank holds no row."""
    import torch

    from test_gpu_parity import assert_hist_close

    cols = oracle.gen_synthetic_bins(rows, d, k, 4)
    g, h = oracle.gen_grad_hess(rows, 4)
    cuts = [rows * r // world for r in range(world + 1)]
    shards = [np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]) for r in range(world)]
    dss = [hbg.Dataset(shards[r], k) for r in range(world)]  # consecutive streams
    peers = [hbg.Peer(dss[r], world, r) for r in range(world)]
    for p in peers:
        for q in peers:
            if q is not p:
                p.attach(q)
    # leaves (global row ids): the whole data, a sampled leaf, and a leaf whose
    # rows all live on rank 0
    rng = np.random.default_rng(1)
    leaves = [np.arange(rows, dtype=np.int32), np.sort(rng.choice(rows, rows // 7, replace=False)).astype(np.int32),
              np.arange(5, min(cuts[1], 3000), dtype=np.int32)]
    gf, hf = g.astype(np.float32), h.astype(np.float32)
    for leaf in leaves:
        outs, errors = [None] * world, []
        tensors = []
        for r in range(world):
            mine = leaf[(leaf >= cuts[r]) & (leaf < cuts[r + 1])]
            idx = torch.from_numpy((mine - cuts[r]).astype(np.int32)).cuda()
            tensors.append((idx, torch.from_numpy(gf[mine]).cuda(), torch.from_numpy(hf[mine]).cuda(),
                            torch.empty(3 * d * k, dtype=torch.float64, device="cuda")))
        torch.cuda.synchronize()

        def run(r):
            try:
                idx, tg, th, out = tensors[r]
                st = dss[r].stream()
                dss[r].build_histograms_peer(idx, len(idx), tg, th, out, peers[r], stream=st)
                hbg.check(hbg.lib().hbg_stream_synchronize(C.c_void_p(st)))
                outs[r] = out.cpu().numpy()
            except Exception as ex:  # surfaced below
                errors.append(ex)

        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors
        peers[0].check()
        for r in range(1, world):
            assert outs[r].tobytes() == outs[0].tobytes(), r  # identical on every rank
        D = d * k
        got = np.zeros((d, k), dtype=hbg.BIN_DTYPE)
        got["grad_sum"] = outs[0][:D].reshape(d, k)
        got["hess_sum"] = outs[0][D:2 * D].reshape(d, k)
        got["count"] = outs[0][2 * D:].reshape(d, k).astype(np.int64)
        want = oracle.build_histograms(cols, k, leaf, gf[leaf].astype(np.float64), hf[leaf].astype(np.float64), 64)
        assert_hist_close(got, want)
    for p in peers:
        p.close()
    for ds in dss:
        ds.close()


@pytest.mark.parametrize("loss", [0, 1])
def test_peer_boosting_equals_reference(hbg, oracle, loss):
    """Row-sharded boost_one_iteration through the in-kernel peer exchange:
    2 ranks as threads; three iterations; the trees equal the oracle's
    unsharded boosting and every row's score matches (1e-6)."""
    import torch

    world, rows, d, k, leaves, min_data = 2, 40000, 20, 64, 31, 100
    cols = oracle.gen_synthetic_bins(rows, d, k, 9)
    rng = np.random.default_rng(9)
    signal = (cols[0].astype(np.float64) - k / 2) / k + 0.5 * (cols[3] > k // 3)
    targets = (rng.random(rows) < 1 / (1 + np.exp(-3 * signal))).astype(np.float64) if loss else signal
    init = float(np.mean(targets)) if loss == 0 else 0.0
    want = np.full(rows, init)
    cuts = [0, 17000, rows]
    dss = [hbg.Dataset(np.ascontiguousarray(cols[:, cuts[r]:cuts[r + 1]]), k) for r in range(world)]
    peers = [hbg.Peer(dss[r], world, r, ctas=torch.cuda.get_device_properties(0).multi_processor_count // world)
             for r in range(world)]
    peers[0].attach(peers[1])
    peers[1].attach(peers[0])
    ts = [torch.from_numpy(targets[cuts[r]:cuts[r + 1]]).cuda() for r in range(world)]
    sc = [torch.full((cuts[r + 1] - cuts[r],), init, dtype=torch.float64, device="cuda") for r in range(world)]
    torch.cuda.synchronize()
    for it in range(3):
        logs, errors = [None] * world, []

        def run(r):
            try:
                logs[r] = dss[r].boost_one_iteration_peer(ts[r], sc[r], peers[r], loss, 0.1, leaves, min_data, 0.0,
                                                          stream=dss[r].stream())
            except Exception as ex:  # surfaced below
                errors.append(ex)

        th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errors, errors
        assert logs[0][0].tobytes() == logs[1][0].tobytes(), it
        want_log = oracle.boost_one_iteration(cols, k, targets, want, loss, 0.1, leaves, min_data, 0.0, 64)
        for key in ("feature", "threshold_bin", "left_count"):
            assert (logs[0][0][key] == want_log[key]).all(), (it, key)
        got = np.concatenate([s.cpu().numpy() for s in sc])
        assert np.allclose(got, want, rtol=1e-6, atol=1e-6), (it, np.abs(got - want).max())
    for p in peers:
        p.close()
    for ds in dss:
        ds.close()
