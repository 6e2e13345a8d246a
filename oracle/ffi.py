"""ctypes bindings for the CPU ORACLE (test infrastructure only).

Loads ``oracle/liboracle.so`` (the C restatement, :mod:`hbg_oracle.c`) and,
when present, ``oracle/_ref/libhistoboost_ref.so`` (the unmodified reference
compiled from /root/reference by oracle/Makefile, plus ``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module — as the checker and the CPU
baseline, never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhistoboost_ref.so")

BIN_DTYPE = np.dtype([("grad_sum", "<f8"), ("hess_sum", "<f8"), ("count", "<i8")])
SPLIT_DTYPE = np.dtype(
    [
        ("feature", "<i4"),
        ("threshold_bin", "<i4"),
        ("gain", "<f8"),
        ("left_grad", "<f8"),
        ("left_hess", "<f8"),
        ("right_grad", "<f8"),
        ("right_hess", "<f8"),
        ("left_count", "<i8"),
        ("right_count", "<i8"),
        ("left_value", "<f8"),
        ("right_value", "<f8"),
    ]
)

_P = C.c_void_p
_I64 = C.c_int64
_U64 = C.c_uint64
_I = C.c_int
_D = C.c_double


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and the reference when /root/reference exists)."""
    target = "all" if (ref and os.path.isdir("/root/reference/proj")) else "liboracle.so"
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.hbo_gen_synthetic_bins.argtypes = [_I64, _I, _I, _U64, _P]
        L.hbo_gen_grad_hess.argtypes = [_I64, _U64, _P, _P]
        L.hbo_leaf_index_sample.argtypes = [_I64, _I, _U64, _P]
        L.hbo_leaf_index_sample.restype = _I64
        L.hbo_pack_feature_tuples.argtypes = [_P, _I, _I64, _I, _I, _P]
        L.hbo_redistribute_bins.argtypes = [_P, _I64, _I, _P, _P]
        L.hbo_fold_histogram.argtypes = [_P, _I, _I, _P]
        L.hbo_gather_leaf.argtypes = [_P, _I64, _P, _P, _P, _P, _P, _P]
        L.hbo_build_histogram.argtypes = [_P, _I, _P, _I64, _P, _P, _I, _P]
        L.hbo_build_histograms_partitioned.argtypes = [_P, _I, _I64, _I, _P, _I64, _P, _P, _I, _P]
        L.hbo_optimal_leaf_value.argtypes = [_D, _D, _D]
        L.hbo_optimal_leaf_value.restype = _D
        L.hbo_split_gain.argtypes = [_D, _D, _D, _D, _D]
        L.hbo_split_gain.restype = _D
        L.hbo_find_best_threshold.argtypes = [_P, _I, _I, _D, _D, _I64, _I64, _D, _P]
        L.hbo_find_best_split.argtypes = [_P, _I, _I, _D, _D, _I64, _I64, _D, _P]
        L.hbo_partition_leaf.argtypes = [_P, _I64, _P, _I, _P, _P]
        L.hbo_partition_leaf.restype = _I64
        L.hbo_grow_tree.argtypes = [_P, _I, _I64, _I, _P, _P, _I, _I64, _D, _I, _P, _P, _P, _P, _P, _P, _P]
        L.hbo_stats_close.argtypes = [_D, _D, _D]
        L.hbo_grad_hess.argtypes = [_I, _P, _P, _I64, _P, _P]
        L.hbo_boost_one_iteration.argtypes = [_P, _I, _I64, _I, _P, _I, _D, _I, _I64, _D, _I, _P, _P]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_synthetic_bins.argtypes = [_I64, _I, _I, _U64, _P]
        L.ref_leaf_index_sample.argtypes = [_I64, _I, _U64, _P]
        L.ref_leaf_index_sample.restype = _I64
        L.ref_pack_feature_tuples.argtypes = [_P, _I, _I64, _I, _I, _P]
        L.ref_redistribute_bins.argtypes = [_P, _I64, _I, _P, _P]
        L.ref_build_histograms_partitioned.argtypes = [_P, _I, _I64, _I, _P, _I64, _P, _P, _I, _I, _P]
        L.ref_find_best_threshold.argtypes = [_P, _I, _I, _D, _D, _I64, _I64, _D, _P]
        L.ref_dataset_new.argtypes = [_P, _I, _I64, _I]
        L.ref_dataset_new.restype = _P
        L.ref_dataset_free.argtypes = [_P]
        L.ref_leaf_new.argtypes = [_P, _I64, _P, _P, _I64]
        L.ref_leaf_new.restype = _P
        L.ref_leaf_free.argtypes = [_P]
        L.ref_build_timed.argtypes = [_P, _P, _I, _I, _P]
        L.ref_build_timed.restype = _D
        L.ref_grow_tree_timed.argtypes = [_P, _P, _P, _I, _I64, _D, _I, _P, _P]
        L.ref_grow_tree_timed.restype = _D
        L.ref_boost_one_iteration.argtypes = [_P, _P, _I, _D, _I, _I64, _D, _I, _P, _P, _P]
        L.ref_boost_one_iteration.restype = _D
        _ref = L
    return _ref


# ----------------------------------------------------------------- oracle API
def gen_synthetic_bins(rows: int, features: int, max_bin: int, seed: int = 0) -> np.ndarray:
    """bench.cpp:17-38 — returns (features, rows) uint8, column-major like BinnedColumn."""
    out = np.empty((features, rows), dtype=np.uint8)
    lib().hbo_gen_synthetic_bins(rows, features, max_bin, seed, _ptr(out))
    return out


def gen_grad_hess(rows: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """bench.cpp:69-73."""
    g = np.empty(rows, dtype=np.float64)
    h = np.empty(rows, dtype=np.float64)
    lib().hbo_gen_grad_hess(rows, seed, _ptr(g), _ptr(h))
    return g, h


def leaf_index_sample(rows: int, depth: int, seed: int) -> np.ndarray:
    """bench.cpp:40-57 (seed is the full seed, e.g. seed + 0x51ed270b * depth)."""
    scratch = np.empty(max(rows, 1), dtype=np.int32)
    n = lib().hbo_leaf_index_sample(rows, depth, seed & 0xFFFFFFFFFFFFFFFF, _ptr(scratch))
    if n < 0:
        raise ValueError("depth out of range or leaves no rows")
    return scratch[:n].copy()


def pack_feature_tuples(cols: np.ndarray, bits: int, max_bin: int) -> np.ndarray:
    """binning.cpp:123-158 — (tuples, rows) uint32 tuple-major words."""
    d, rows = cols.shape
    per = 32 // bits
    t = (d + per - 1) // per
    words = np.empty((t, rows), dtype=np.uint32)
    cols = np.ascontiguousarray(cols)
    r = lib().hbo_pack_feature_tuples(_ptr(cols), d, rows, bits, max_bin, _ptr(words))
    if r < 0:
        raise ValueError("4-bit packing requires bin capacity <= 16")
    return words


def gather_leaf(idx: np.ndarray, g: np.ndarray, h: np.ndarray):
    """tree.cpp:11-25 — (leaf_g, leaf_h, grad_total, hess_total)."""
    n = len(idx)
    lg = np.empty(n, dtype=np.float64)
    lh = np.empty(n, dtype=np.float64)
    gt = C.c_double()
    ht = C.c_double()
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    lib().hbo_gather_leaf(_ptr(idx), n, _ptr(g), _ptr(h), _ptr(lg), _ptr(lh), C.byref(gt), C.byref(ht))
    return lg, lh, gt.value, ht.value


def build_histograms(cols: np.ndarray, max_bin: int, idx: np.ndarray, leaf_g: np.ndarray,
                     leaf_h: np.ndarray, precision: int = 64) -> np.ndarray:
    """histogram.cpp:159-215 — (d, k) structured array of HistogramBin."""
    d, rows = cols.shape
    out = np.zeros((d, max_bin), dtype=BIN_DTYPE)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    lib().hbo_build_histograms_partitioned(
        _ptr(np.ascontiguousarray(cols)), d, rows, max_bin, _ptr(idx), len(idx),
        _ptr(np.ascontiguousarray(leaf_g, dtype=np.float64)),
        _ptr(np.ascontiguousarray(leaf_h, dtype=np.float64)), precision, _ptr(out))
    return out


def find_best_split(hists: np.ndarray, grad_total: float, hess_total: float, count: int,
                    min_data_in_leaf: int = 1, lam: float = 0.0):
    """tree.cpp:163-182 — structured split record or None."""
    d, k = hists.shape
    out = np.zeros(1, dtype=SPLIT_DTYPE)
    hists = np.ascontiguousarray(hists)
    found = lib().hbo_find_best_split(_ptr(hists), d, k, grad_total, hess_total, count,
                                      min_data_in_leaf, lam, _ptr(out))
    return out[0] if found else None


def find_best_threshold(hist: np.ndarray, feature_id: int, grad_total: float, hess_total: float,
                        count: int, min_data_in_leaf: int = 1, lam: float = 0.0):
    out = np.zeros(1, dtype=SPLIT_DTYPE)
    hist = np.ascontiguousarray(hist)
    found = lib().hbo_find_best_threshold(_ptr(hist), len(hist), feature_id, grad_total, hess_total,
                                          count, min_data_in_leaf, lam, _ptr(out))
    return out[0] if found else None


def partition_leaf(idx: np.ndarray, col: np.ndarray, threshold_bin: int):
    n = len(idx)
    left = np.empty(max(n, 1), dtype=np.int32)
    right = np.empty(max(n, 1), dtype=np.int32)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    nl = lib().hbo_partition_leaf(_ptr(idx), n, _ptr(np.ascontiguousarray(col)), threshold_bin,
                                  _ptr(left), _ptr(right))
    if nl < 0:
        raise RuntimeError("split produced an empty side")
    return left[:nl].copy(), right[: n - nl].copy()


def grow_tree(cols: np.ndarray, max_bin: int, g: np.ndarray, h: np.ndarray, num_leaves: int,
              min_data_in_leaf: int = 1, lam: float = 0.0, precision: int = 64):
    """tree.cpp:186-261 — (split_log, nodes dict)."""
    d, rows = cols.shape
    log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
    mx = 2 * num_leaves - 1
    nf = np.empty(mx, np.int32)
    nt = np.empty(mx, np.int32)
    nlft = np.empty(mx, np.int32)
    nrgt = np.empty(mx, np.int32)
    nv = np.empty(mx, np.float64)
    nn = C.c_int()
    n = lib().hbo_grow_tree(_ptr(np.ascontiguousarray(cols)), d, rows, max_bin, _ptr(g), _ptr(h),
                            num_leaves, min_data_in_leaf, lam, precision, _ptr(log), _ptr(nf),
                            _ptr(nt), _ptr(nlft), _ptr(nrgt), _ptr(nv), C.byref(nn))
    k = nn.value
    nodes = {"feature": nf[:k], "threshold_bin": nt[:k], "left": nlft[:k], "right": nrgt[:k],
             "value": nv[:k]}
    return log[:n].copy(), nodes


def grad_hess(loss: int, scores: np.ndarray, targets: np.ndarray):
    """losses.cpp:24-26 (0 = squared) / :57-60 (1 = logistic)."""
    n = len(scores)
    g = np.empty(n)
    h = np.empty(n)
    lib().hbo_grad_hess(loss, _ptr(np.ascontiguousarray(scores, dtype=np.float64)),
                        _ptr(np.ascontiguousarray(targets, dtype=np.float64)), n, _ptr(g), _ptr(h))
    return g, h


def boost_one_iteration(cols, max_bin, targets, scores, loss=0, learning_rate=0.1, num_leaves=31,
                        min_data_in_leaf=1, lam=0.0, precision=64):
    """boosting.cpp:26-51 — updates `scores` in place, returns the split log."""
    d, rows = cols.shape
    log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
    assert scores.dtype == np.float64 and scores.flags.c_contiguous
    n = lib().hbo_boost_one_iteration(_ptr(np.ascontiguousarray(cols)), d, rows, max_bin,
                                      _ptr(np.ascontiguousarray(targets, dtype=np.float64)), loss,
                                      learning_rate, num_leaves, min_data_in_leaf, lam, precision,
                                      _ptr(scores), _ptr(log))
    return log[:n].copy()


# -------------------------------------------------------------- reference API
def ref_gen_synthetic_bins(rows, features, max_bin, seed=0):
    out = np.empty((features, rows), dtype=np.uint8)
    ref().ref_gen_synthetic_bins(rows, features, max_bin, seed, _ptr(out))
    return out


def ref_leaf_index_sample(rows, depth, seed):
    scratch = np.empty(max(rows, 1), dtype=np.int32)
    n = ref().ref_leaf_index_sample(rows, depth, seed & 0xFFFFFFFFFFFFFFFF, _ptr(scratch))
    if n < 0:
        raise ValueError(ref().ref_last_error().decode())
    return scratch[:n].copy()


def ref_pack_feature_tuples(cols, bits, max_bin):
    d, rows = cols.shape
    per = 32 // bits
    words = np.empty(((d + per - 1) // per, rows), dtype=np.uint32)
    r = ref().ref_pack_feature_tuples(_ptr(np.ascontiguousarray(cols)), d, rows, bits, max_bin, _ptr(words))
    if r < 0:
        raise ValueError(ref().ref_last_error().decode())
    return words


def ref_build_histograms(cols, max_bin, idx, leaf_g, leaf_h, precision=64, workers=0):
    d, rows = cols.shape
    out = np.zeros((d, max_bin), dtype=BIN_DTYPE)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    ref().ref_build_histograms_partitioned(
        _ptr(np.ascontiguousarray(cols)), d, rows, max_bin, _ptr(idx), len(idx),
        _ptr(np.ascontiguousarray(leaf_g, dtype=np.float64)),
        _ptr(np.ascontiguousarray(leaf_h, dtype=np.float64)), precision, workers, _ptr(out))
    return out


def ref_find_best_threshold(hist, feature_id, gt, ht, count, min_data=1, lam=0.0):
    out = np.zeros(1, dtype=SPLIT_DTYPE)
    hist = np.ascontiguousarray(hist)
    found = ref().ref_find_best_threshold(_ptr(hist), len(hist), feature_id, gt, ht, count,
                                          min_data, lam, _ptr(out))
    return out[0] if found else None


class RefDataset:
    """A reference BinnedDataset kept alive for repeated timing."""

    def __init__(self, cols: np.ndarray, max_bin: int):
        self.cols = np.ascontiguousarray(cols)
        self.d, self.rows = cols.shape
        self.k = max_bin
        self.h = ref().ref_dataset_new(_ptr(self.cols), self.d, self.rows, max_bin)

    def leaf(self, idx: np.ndarray, g: np.ndarray, h: np.ndarray):
        idx = np.ascontiguousarray(idx, dtype=np.int32)
        return ref().ref_leaf_new(_ptr(idx), len(idx), _ptr(g), _ptr(h), self.rows)

    def build_timed(self, leaf, precision=32, workers=0, want=False):
        out = np.zeros((self.d, self.k), dtype=BIN_DTYPE) if want else None
        t = ref().ref_build_timed(self.h, leaf, precision, workers, _ptr(out))
        return t, out

    def grow_tree_timed(self, g, h, num_leaves=255, min_data=1, lam=0.0, precision=32):
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        n = C.c_int()
        t = ref().ref_grow_tree_timed(self.h, _ptr(g), _ptr(h), num_leaves, min_data, lam,
                                      precision, _ptr(log), C.byref(n))
        return t, log[: n.value].copy()

    def boost_one_iteration_timed(self, targets, scores, loss=0, learning_rate=0.1, num_leaves=31,
                                  min_data=1, lam=0.0, precision=32):
        n = C.c_int()
        t = ref().ref_boost_one_iteration(self.h, _ptr(np.ascontiguousarray(targets, dtype=np.float64)), loss,
                                          learning_rate, num_leaves, min_data, lam, precision, _ptr(scores),
                                          None, C.byref(n))
        return t

    @staticmethod
    def free_leaf(leaf):
        ref().ref_leaf_free(leaf)

    def close(self):
        if self.h:
            ref().ref_dataset_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
