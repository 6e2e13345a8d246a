"""Row-sharded multi-GPU plumbing.

One process per GPU. Rank r owns the contiguous rows [begin_r, end_r) of the
binned matrix (its packed bins, g and h); leaf index lists are local row ids.
After a rank builds the histogram of its part of a leaf, the leaf histogram is
summed across ranks with one NCCL allreduce over NVLink (torch.distributed
backend "nccl"; "gloo" in the CPU tests). The device histogram is SoA fp64
[grad | hess | count], so one fp64 SUM covers all three statistics and the
counts stay exact (integers < 2^53 add exactly in any order). Every rank then
holds bit-identical histograms and makes the identical split decision — the
single-box analogue is the reference's ordered reduction of 64 Ki-row chunk
partials (histogram.cpp:159-215).
"""
from __future__ import annotations

import numpy as np


def shard_rows(num_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row range of `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(num_rows, world)
    begin = rank * base + min(rank, extra)
    end = begin + base + (1 if rank < extra else 0)
    return begin, end


def local_leaf(global_rows: np.ndarray, begin: int, end: int) -> np.ndarray:
    """The part of a (sorted) global leaf that rank [begin, end) owns, as local row ids."""
    lo, hi = np.searchsorted(global_rows, [begin, end])
    return (global_rows[lo:hi] - begin).astype(np.int32)


def allreduce_histogram(hist, group=None) -> None:
    """Sum a device/host SoA fp64 leaf histogram across ranks, in place."""
    import torch.distributed as dist

    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)


def bins_to_soa(bins: np.ndarray) -> np.ndarray:
    """(d, k) HistogramBin records -> SoA fp64 [3, d, k] (the device layout)."""
    return np.stack([bins["grad_sum"], bins["hess_sum"], bins["count"].astype(np.float64)])


def soa_to_bins(soa: np.ndarray, dtype) -> np.ndarray:
    soa = np.asarray(soa, dtype=np.float64).reshape(3, *soa.shape[-2:]) if soa.ndim == 3 else soa
    out = np.zeros(soa.shape[1:], dtype=dtype)
    out["grad_sum"], out["hess_sum"], out["count"] = soa[0], soa[1], soa[2].astype(np.int64)
    return out
