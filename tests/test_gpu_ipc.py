"""Row sharding across PROCESSES (GPU): the exchange areas mapped with CUDA IPC.

The multi-GPU deployment runs one process per GPU; every rank exports its
exchange area (hbg_peer_handle, a cudaIpcMemHandle) and maps every other
rank's (hbg_peer_open) — what bench.py does through torch.distributed. Only
one GPU is available here, so two PROCESSES share it: their contexts
time-slice, which is enough for the bounded in-kernel waits to meet. Checked:
the fused single-leaf exchange (hbg_build_histograms_peer) and the in-kernel
per-split exchange (hbg_grow_tree_peer, two trees for the generation tags) —
bit-identical results on both ranks, equal to the oracle on the union of the
shards.
"""
import multiprocessing as mp
import os
import queue
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS, D, K, LEAVES, MIN_DATA, WORLD = 40000, 28, 64, 31, 100, 2


def _data():
    sys.path.insert(0, REPO)
    from oracle import ffi

    cols = ffi.gen_synthetic_bins(ROWS, D, K, 9)
    g, h = ffi.gen_grad_hess(ROWS, 9)
    g = g + 0.3 * (cols[2].astype(np.float64) > K // 2)
    return cols, g, h


def _rank(rank, handles_out, handles_in, results):
    """One rank = one process with its own CUDA context."""
    try:
        sys.path.insert(0, REPO)
        import torch

        import paper_1706_08359_b200 as hbg

        cols, g, h = _data()
        cut = ROWS * 2 // 5  # uneven shards
        b, e = (0, cut) if rank == 0 else (cut, ROWS)
        ds = hbg.Dataset(np.ascontiguousarray(cols[:, b:e]), K)
        peer = hbg.Peer(ds, WORLD, rank, 0, LEAVES)
        handles_out.put((rank, peer.ipc_handle()))
        others = handles_in.get(timeout=120)
        for r, hd in others.items():
            if r != rank:
                peer.open(r, hd)
        n = e - b
        tg = torch.from_numpy(g[b:e].astype(np.float32)).cuda()
        th = torch.from_numpy(h[b:e].astype(np.float32)).cuda()
        idx = torch.arange(n, dtype=torch.int32, device="cuda")
        out = torch.empty(3 * D * K, dtype=torch.float64, device="cuda")
        st = ds.stream()
        ds.build_histograms_peer(idx, n, tg, th, out, peer, stream=st)
        peer.check()
        hist = out.cpu().numpy()
        trees = []
        for _ in range(2):
            log, nodes = ds.grow_tree_peer(tg, th, peer, LEAVES, MIN_DATA, 0.0, st)
            trees.append((log, nodes))
        peer.check()
        peer.close()
        ds.close()
        results.put((rank, "ok", hist, trees))
    except Exception as ex:  # noqa: BLE001 — reported to the parent
        results.put((rank, "error", repr(ex), None))


def test_two_process_ipc_exchange(oracle):
    ctx = mp.get_context("spawn")
    handles_out = ctx.Queue()
    handles_in = [ctx.Queue() for _ in range(WORLD)]
    results = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, handles_out, handles_in[r], results)) for r in range(WORLD)]
    for p in procs:
        p.start()
    try:
        got = {}
        for _ in range(WORLD):
            r, hd = handles_out.get(timeout=300)
            got[r] = hd
        for q in handles_in:
            q.put(got)
        res = {}
        for _ in range(WORLD):
            r, status, a, b = results.get(timeout=600)
            assert status == "ok", (r, a)
            res[r] = (a, b)
    except queue.Empty:
        pytest.fail("a rank process did not report in time")
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    # identical on both ranks
    assert res[0][0].tobytes() == res[1][0].tobytes()
    for t in range(2):
        for j in range(2):
            assert res[0][1][t][j].tobytes() == res[1][1][t][j].tobytes(), (t, j)
    assert res[0][1][0][0].tobytes() == res[0][1][1][0].tobytes()  # tree 2 == tree 1
    # equal to the oracle on the union of the shards
    cols, g, h = _data()
    from test_gpu_parity import _assert_same_tree, assert_hist_close
    import paper_1706_08359_b200 as hbg

    hist = res[0][0]
    DK = D * K
    gh = np.zeros((D, K), dtype=hbg.BIN_DTYPE)
    gh["grad_sum"] = hist[:DK].reshape(D, K)
    gh["hess_sum"] = hist[DK:2 * DK].reshape(D, K)
    gh["count"] = hist[2 * DK:].reshape(D, K).astype(np.int64)
    gf, hf = g.astype(np.float32).astype(np.float64), h.astype(np.float32).astype(np.float64)
    want = oracle.build_histograms(cols, K, np.arange(ROWS, dtype=np.int32), gf, hf, 64)
    assert_hist_close(gh, want)
    want_log, want_nodes = oracle.grow_tree(cols, K, g, h, LEAVES, MIN_DATA, 0.0, 64)
    log, nodes = res[0][1][0]
    assert _assert_same_tree(log, nodes, want_log, want_nodes) == len(want_log)
