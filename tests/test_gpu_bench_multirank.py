"""bench.py's N > 1 path on the one GPU of the tests (GPU).

The driver runs `bench.py --gpus N` under torchrun on N GPUs; that path (CUDA
IPC exchange areas shared through torch.distributed, the histogram with the
cross-rank sum fused into its reduction, the peer tree, max-over-ranks timing)
never runs on a one-GPU box. HBG_BENCH_SHARED_GPU puts both ranks on one
device (gloo for torch.distributed; no NCCL, which refuses two ranks per GPU):
the contexts time-slice, so the timings mean nothing, but every step of the
multi-rank flow must run and the line must describe a 2-rank job.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_on_one_gpu():
    env = dict(os.environ, HBG_BENCH_SHARED_GPU="1", HBG_PEER_TIMEOUT_MS="60000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517", os.path.join(REPO, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-variants", "--no-cpu-baseline", "--rows", "300000",
           "--num-leaves", "31", "--trees", "1"]
    r = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["config"]["rows_total"] == 600000
    assert "peer memory" in line["exchange"]  # the fused exchange, not the NCCL fallback
    assert line["tree"]["splits"] == 30 and "peer-memory" in line["tree"]["path"]
