"""B200-native feature-histogram construction (arXiv 1706.08359 hot path).

Host-side mirror of the reference's histogram interface
(/root/reference/proj/include/histoboost/histogram.hpp:129-134, tree.hpp:59-99)
over the C ABI in ``include/hbg.h`` (``libhbg.so``, CUDA sm_100a). Names,
argument meaning and error behaviour follow the reference:

* :class:`Dataset`                 — device-resident packed ``BinnedDataset`` (dataset.hpp:80-91)
* :class:`LeafState`               — ``LeafState`` (leaf.hpp:13-21)
* :func:`gather_leaf_statistics`   — tree.cpp:11-25
* :func:`build_histograms_partitioned` — the drop-in for histogram.hpp:133
* :func:`find_best_split` / :func:`find_best_threshold` — tree.cpp:76-112,163-182

There is no CPU fallback: if ``libhbg.so`` is missing or no GPU is present,
every call raises. ``InvalidArgument`` mirrors ``std::invalid_argument`` and
``LogicError`` mirrors ``std::logic_error``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libhbg.so")
HEADER = os.path.join(REPO, "include", "hbg.h")

HBG_OK = 0
HBG_ERR_INVALID_ARGUMENT = 1
HBG_ERR_LOGIC = 2
HBG_ERR_CUDA = 3
HBG_ERR_OUT_OF_MEMORY = 4
HBG_ERR_NCCL = 5
HBG_GH_LEAF_ALIGNED = 0
HBG_GH_ROW_INDEXED = 1
HBG_LOSS_SQUARED = 0
HBG_LOSS_LOGISTIC = 1
#: PrecisionMode (histogram_set.hpp:11): bits32 / bits64
HBG_PRECISION_BITS32 = 0
HBG_PRECISION_BITS64 = 1


def hist_kernel_stamp() -> str:
    """Short hash of the histogram kernel's sources: a committed ncu number
    (profiles/ncu_traffic.json) is only reported while it still describes the
    kernel that runs."""
    import hashlib

    hsh = hashlib.sha256()
    for name in ("hist_kernels.cu", "hist_device.cuh"):
        with open(os.path.join(HERE, "csrc", name), "rb") as f:
            hsh.update(f.read())
    return hsh.hexdigest()[:16]


def _precision(p) -> int:
    """32 / 64 / 'bits32' / 'bits64' / HBG_PRECISION_* -> HBG_PRECISION_*."""
    table = {32: HBG_PRECISION_BITS32, 64: HBG_PRECISION_BITS64, "bits32": HBG_PRECISION_BITS32,
             "bits64": HBG_PRECISION_BITS64, HBG_PRECISION_BITS32: HBG_PRECISION_BITS32,
             HBG_PRECISION_BITS64: HBG_PRECISION_BITS64}
    if p not in table:
        raise InvalidArgument(HBG_ERR_INVALID_ARGUMENT, f"unknown precision {p!r}")
    return table[p]

#: numpy view of ``hbg_bin`` == ``histoboost::HistogramBin`` (histogram_set.hpp:17-21)
BIN_DTYPE = np.dtype([("grad_sum", "<f8"), ("hess_sum", "<f8"), ("count", "<i8")])
#: numpy view of ``hbg_split`` (SplitInfo minus threshold_value, tree.hpp:15-24)
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


#: numpy view of ``hbg_tree_node`` (TreeNode minus threshold_value, tree.hpp:26-35)
NODE_DTYPE = np.dtype([("feature", "<i4"), ("threshold_bin", "<i4"), ("left", "<i4"), ("right", "<i4"),
                       ("value", "<f8")])


class hbg_grow_params(C.Structure):
    _fields_ = [("num_leaves", C.c_int32), ("precision", C.c_int32), ("min_data_in_leaf", C.c_int64),
                ("lambda_", C.c_double)]


#: hbg_allreduce_fn: int (*)(double* d_buf, int64_t n, void* stream, void* ctx)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class HbgError(RuntimeError):
    """Base class; ``code`` is the HBG_* status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(HbgError, ValueError):
    """std::invalid_argument analogue (histogram.cpp:27-40,148-154)."""


class LogicError(HbgError):
    """std::logic_error analogue (tree.cpp:124-126,143-145)."""


class CudaError(HbgError):
    """CUDA runtime failure — there is no CPU fallback."""


class hbg_layout(C.Structure):
    _fields_ = [
        ("num_rows", C.c_int64),
        ("num_features", C.c_int32),
        ("max_bin", C.c_int32),
        ("bits_per_bin", C.c_int32),
        ("features_per_word", C.c_int32),
        ("words_per_row", C.c_int32),
        ("row_stride_bytes", C.c_int32),
        ("slice_bytes", C.c_int32),
        ("num_groups", C.c_int32),
        ("device", C.c_int32),
        ("group_stride_bytes", C.c_int64),
    ]


#: every symbol include/hbg.h declares (checked by tests/test_abi.py)
EXPORTED_SYMBOLS = (
    "hbg_last_error",
    "hbg_version",
    "hbg_debug_hist_stamps",
    "hbg_debug_host_copy_bytes",
    "hbg_dataset_create",
    "hbg_dataset_destroy",
    "hbg_dataset_layout",
    "hbg_dataset_packed_words",
    "hbg_build_histograms",
    "hbg_build_histograms_ex",
    "hbg_build_histograms_device",
    "hbg_build_histograms_device_f64",
    "hbg_hist_to_bins_device",
    "hbg_subtract_device",
    "hbg_gather_leaf_device",
    "hbg_gather_leaf_statistics",
    "hbg_best_split_device",
    "hbg_best_split_device_totals",
    "hbg_find_best_split",
    "hbg_grow_tree",
    "hbg_grow_tree_host",
    "hbg_grow_tree_f64",
    "hbg_grow_tree_sharded",
    "hbg_dataset_stream",
    "hbg_peer_create",
    "hbg_peer_handle",
    "hbg_peer_open",
    "hbg_peer_attach",
    "hbg_peer_destroy",
    "hbg_build_histograms_peer",
    "hbg_peer_check",
    "hbg_boost_one_iteration_peer",
    "hbg_grow_tree_peer",
    "hbg_comm_get_unique_id",
    "hbg_comm_init",
    "hbg_comm_destroy",
    "hbg_comm_allreduce",
    "hbg_reduce_histograms_device",
    "hbg_boost_one_iteration",
    "hbg_dataset_set_profiling",
    "hbg_dataset_kernel_time",
    "hbg_stream_synchronize",
)

_P = C.c_void_p
_lib = None


def build(force: bool = False) -> str:
    """Compile libhbg.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", HERE, "-j4"], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    """Load libhbg.so; raises if it was never built (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run paper_1706_08359_b200.build() (or __graft_entry__.build())"
            )
        L = C.CDLL(LIB_PATH)
        L.hbg_last_error.restype = C.c_char_p
        L.hbg_version.restype = C.c_int32
        L.hbg_dataset_create.argtypes = [_P, C.c_int32, C.c_int64, C.c_int32, C.c_int32, _P]
        L.hbg_dataset_destroy.argtypes = [_P]
        L.hbg_dataset_layout.argtypes = [_P, _P]
        L.hbg_dataset_packed_words.argtypes = [_P, _P]
        L.hbg_build_histograms.argtypes = [_P, _P, C.c_int64, _P, _P, _P]
        L.hbg_build_histograms_ex.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_int32, _P]
        L.hbg_build_histograms_device.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_int32, _P, _P]
        L.hbg_build_histograms_device_f64.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_int32, _P, _P]
        L.hbg_gather_leaf_statistics.argtypes = [_P, C.c_int64, _P, _P, C.c_int64, _P, _P, _P, C.c_int32]
        L.hbg_grow_tree_f64.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.hbg_hist_to_bins_device.argtypes = [_P, C.c_int32, C.c_int32, _P, _P]
        L.hbg_subtract_device.argtypes = [_P, _P, _P, C.c_int64, _P]
        L.hbg_gather_leaf_device.argtypes = [_P, C.c_int64, _P, _P, _P, _P, _P, _P]
        L.hbg_best_split_device.argtypes = [_P, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                            C.c_int64, C.c_int64, C.c_double, _P, _P]
        L.hbg_best_split_device_totals.argtypes = [_P, C.c_int32, C.c_int32, _P, _P, C.c_int64,
                                                   C.c_double, _P, _P]
        L.hbg_find_best_split.argtypes = [_P, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                          C.c_int64, C.c_int64, C.c_double, _P, _P]
        L.hbg_grow_tree.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.hbg_grow_tree_host.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P]
        L.hbg_dataset_stream.argtypes = [_P]
        L.hbg_dataset_stream.restype = _P
        L.hbg_peer_create.argtypes = [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P]
        L.hbg_peer_handle.argtypes = [_P, _P]
        L.hbg_peer_open.argtypes = [_P, C.c_int32, _P]
        L.hbg_peer_attach.argtypes = [_P, C.c_int32, _P]
        L.hbg_peer_destroy.argtypes = [_P]
        L.hbg_build_histograms_peer.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_int32, _P, _P, _P]
        L.hbg_peer_check.argtypes = [_P]
        L.hbg_boost_one_iteration_peer.argtypes = [_P, _P, _P, C.c_int32, C.c_double, _P, _P, _P, _P, _P, _P, _P]
        L.hbg_grow_tree_peer.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P]
        L.hbg_grow_tree_sharded.argtypes = [_P, _P, _P, _P, ALLREDUCE_FN, _P, _P, _P, _P, _P, _P]
        L.hbg_comm_get_unique_id.argtypes = [_P]
        L.hbg_comm_init.argtypes = [_P, C.c_int32, C.c_int32, _P, C.c_int32]
        L.hbg_comm_destroy.argtypes = [_P]
        L.hbg_comm_allreduce.argtypes = [_P, C.c_int64, _P, _P]
        L.hbg_reduce_histograms_device.argtypes = [_P, C.c_int32, C.c_int64, _P, _P]
        L.hbg_boost_one_iteration.argtypes = [_P, _P, _P, C.c_int32, C.c_double, _P, ALLREDUCE_FN, _P, _P, _P,
                                              _P, _P, _P]
        L.hbg_dataset_set_profiling.argtypes = [_P, C.c_int32]
        L.hbg_dataset_kernel_time.argtypes = [_P, _P, _P]
        L.hbg_stream_synchronize.argtypes = [_P]
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == HBG_OK:
        return
    msg = lib().hbg_last_error().decode(errors="replace")
    cls = {HBG_ERR_INVALID_ARGUMENT: InvalidArgument, HBG_ERR_LOGIC: LogicError}.get(status, CudaError)
    raise cls(status, msg)


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(C.c_void_p)
    if isinstance(a, int):
        return C.c_void_p(a)
    if isinstance(a, C.c_void_p):
        return a
    return C.c_void_p(a.data_ptr())  # torch.Tensor


# --------------------------------------------------------------------------- types
@dataclass
class LeafState:
    """Rows of one leaf with leaf-aligned gradients/hessians (leaf.hpp:13-21)."""

    indices: np.ndarray
    gradients: np.ndarray
    hessians: np.ndarray
    grad_total: float = 0.0
    hess_total: float = 0.0

    def count(self) -> int:
        return int(len(self.indices))


def gather_leaf_statistics(indices, gradients, hessians, device: int = 0) -> LeafState:
    """gather_leaf_statistics (tree.cpp:11-25) on the device: leaf-aligned fp64
    g/h and fp64 totals (fixed-order sums) from host per-row arrays."""
    idx = np.ascontiguousarray(indices, dtype=np.int32)
    g = np.ascontiguousarray(gradients, dtype=np.float64)
    h = np.ascontiguousarray(hessians, dtype=np.float64)
    if len(g) != len(h):
        raise InvalidArgument(HBG_ERR_INVALID_ARGUMENT, "gradients and hessians disagree on length")
    n = len(idx)
    lg = np.empty(n, dtype=np.float64)
    lh = np.empty(n, dtype=np.float64)
    tot = np.zeros(2, dtype=np.float64)
    check(lib().hbg_gather_leaf_statistics(_ptr(idx), n, _ptr(g), _ptr(h), len(g), _ptr(lg), _ptr(lh),
                                           _ptr(tot), device))
    return LeafState(idx, lg, lh, float(tot[0]), float(tot[1]))


class Dataset:
    """Device-resident packed binned dataset (subsystem 1; rows a1-a2).

    ``columns`` is (num_features, num_rows) uint8 — one ``BinnedColumn::bins``
    per feature (dataset.hpp:21-26), every bin < ``max_bin``.
    """

    def __init__(self, columns: np.ndarray, max_bin: int, device: int = 0):
        cols = np.ascontiguousarray(columns, dtype=np.uint8)
        if cols.ndim != 2:
            raise InvalidArgument(HBG_ERR_INVALID_ARGUMENT, "columns must be (features, rows)")
        d, n = cols.shape
        ptrs = (C.c_void_p * max(d, 1))(*[cols[f].ctypes.data for f in range(d)])
        h = C.c_void_p()
        check(lib().hbg_dataset_create(ptrs, d, n, max_bin, device, C.byref(h)))
        self._h = h
        self.num_features = d
        self.num_rows = n
        self.max_bin = max_bin
        self.device = device

    @property
    def handle(self) -> C.c_void_p:
        if not self._h:
            raise InvalidArgument(HBG_ERR_INVALID_ARGUMENT, "dataset is closed")
        return self._h

    def layout(self) -> dict:
        L = hbg_layout()
        check(lib().hbg_dataset_layout(self.handle, C.byref(L)))
        return {name: getattr(L, name) for name, _ in L._fields_}

    def packed_words(self) -> np.ndarray:
        L = self.layout()
        out = np.zeros((L["num_rows"], L["words_per_row"]), dtype=np.uint32)
        check(lib().hbg_dataset_packed_words(self.handle, _ptr(out)))
        return out

    def hist_values(self) -> int:
        """Doubles in one device SoA histogram: 3 * num_features * max_bin."""
        return 3 * self.num_features * self.max_bin

    def build_histograms_device(self, indices, count: int, grad, hess, hist,
                                gh_mode: int = HBG_GH_LEAF_ALIGNED, stream=None) -> None:
        """Device builder: pointers are torch tensors / raw ints; async on ``stream``."""
        check(lib().hbg_build_histograms_device(self.handle, _ptr(indices), count, _ptr(grad),
                                                _ptr(hess), gh_mode, _ptr(hist), _ptr(stream)))

    def build_histograms_device_f64(self, indices, count: int, grad, hess, hist,
                                    gh_mode: int = HBG_GH_LEAF_ALIGNED, stream=None) -> None:
        """bits64 device builder: fp64 g/h tensors, fp64 accumulation."""
        check(lib().hbg_build_histograms_device_f64(self.handle, _ptr(indices), count, _ptr(grad),
                                                    _ptr(hess), gh_mode, _ptr(hist), _ptr(stream)))

    def grow_tree(self, grad, hess, num_leaves: int = 31, min_data_in_leaf: int = 1, lam: float = 0.0,
                  stream=None):
        """grow_tree (tree.cpp:186-261) on the device; grad/hess are fp32 device
        tensors of num_rows. Returns (split_log SPLIT_DTYPE[], nodes NODE_DTYPE[])."""
        p = hbg_grow_params(num_leaves, 0, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_grow_tree(self.handle, _ptr(grad), _ptr(hess), C.byref(p), _ptr(log), C.byref(ns),
                                  _ptr(nodes), C.byref(nn), _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def grow_tree_host(self, gradients: np.ndarray, hessians: np.ndarray, num_leaves: int = 31,
                       min_data_in_leaf: int = 1, lam: float = 0.0, precision=32):
        """grow_tree (tree.cpp:186-261) from host fp64 per-row gradients/hessians
        (the reference's span<const double> arguments), GrowParams::precision
        = ``precision`` (32 or 64). Returns (split_log, nodes)."""
        g = np.ascontiguousarray(gradients, dtype=np.float64)
        h = np.ascontiguousarray(hessians, dtype=np.float64)
        p = hbg_grow_params(num_leaves, _precision(precision), min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_grow_tree_host(self.handle, g.ctypes.data, h.ctypes.data, C.byref(p), log.ctypes.data,
                                       C.byref(ns), nodes.ctypes.data, C.byref(nn)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def grow_tree_f64(self, grad, hess, num_leaves: int = 31, min_data_in_leaf: int = 1, lam: float = 0.0,
                      stream=None):
        """bits64 grow_tree on fp64 device tensors of num_rows."""
        p = hbg_grow_params(num_leaves, HBG_PRECISION_BITS64, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_grow_tree_f64(self.handle, _ptr(grad), _ptr(hess), C.byref(p), _ptr(log), C.byref(ns),
                                      _ptr(nodes), C.byref(nn), _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def stream(self) -> int:
        """The dataset's own CUDA stream (cudaStream_t as an int)."""
        return lib().hbg_dataset_stream(self.handle) or 0

    def host_copy_bytes(self) -> tuple:
        """(host->device, device->host) bytes of the last host drop-in call."""
        out = (C.c_int64 * 2)()
        check(lib().hbg_debug_host_copy_bytes(self.handle, out))
        return int(out[0]), int(out[1])

    def build_histograms_peer(self, indices, count: int, grad, hess, out, peer: "Peer",
                              gh_mode: int = HBG_GH_LEAF_ALIGNED, stream=None):
        """This rank's rows of a leaf; `out` receives the histogram summed over
        all ranks (the sum fused into the reduction kernel, over peer memory)."""
        check(lib().hbg_build_histograms_peer(self.handle, _ptr(indices), count, _ptr(grad), _ptr(hess), gh_mode,
                                              _ptr(out), peer.handle, _ptr(stream)))

    def boost_one_iteration_peer(self, targets, scores, peer: "Peer", loss: int = HBG_LOSS_SQUARED,
                                 learning_rate: float = 0.1, num_leaves: int = 31, min_data_in_leaf: int = 1,
                                 lam: float = 0.0, stream=None):
        """boost_one_iteration over this rank's rows, the tree grown through the
        in-kernel peer exchange (every rank calls it)."""
        p = hbg_grow_params(num_leaves, 0, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_boost_one_iteration_peer(self.handle, _ptr(targets), _ptr(scores), loss, learning_rate,
                                                 C.byref(p), peer.handle, _ptr(log), C.byref(ns), _ptr(nodes),
                                                 C.byref(nn), _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def grow_tree_peer(self, grad, hess, peer: "Peer", num_leaves: int = 31, min_data_in_leaf: int = 1,
                       lam: float = 0.0, stream=None):
        """Row-sharded grow_tree with the histogram exchange inside the
        persistent kernel over peer memory (every rank calls it; this rank's rows)."""
        p = hbg_grow_params(num_leaves, 0, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_grow_tree_peer(self.handle, _ptr(grad), _ptr(hess), C.byref(p), peer.handle, _ptr(log),
                                       C.byref(ns), _ptr(nodes), C.byref(nn), _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def grow_tree_sharded(self, grad, hess, allreduce, ctx=None, num_leaves: int = 31,
                          min_data_in_leaf: int = 1, lam: float = 0.0, stream=None):
        """Row-sharded grow_tree: this rank's rows; `allreduce` (an ALLREDUCE_FN,
        e.g. Comm.allreduce_fn) sums leaf histograms/totals across ranks."""
        p = hbg_grow_params(num_leaves, 0, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        check(lib().hbg_grow_tree_sharded(self.handle, _ptr(grad), _ptr(hess), C.byref(p), allreduce,
                                          _ptr(ctx), _ptr(log), C.byref(ns), _ptr(nodes), C.byref(nn),
                                          _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def boost_one_iteration(self, targets, scores, loss: int = HBG_LOSS_SQUARED, learning_rate: float = 0.1,
                            num_leaves: int = 31, min_data_in_leaf: int = 1, lam: float = 0.0,
                            allreduce=None, ctx=None, stream=None):
        """boost_one_iteration (boosting.cpp:26-51) on the device: fp64 device
        `targets`/`scores` (updated in place). Returns (split_log, nodes)."""
        p = hbg_grow_params(num_leaves, 0, min_data_in_leaf, lam)
        log = np.zeros(max(num_leaves - 1, 1), dtype=SPLIT_DTYPE)
        nodes = np.zeros(max(2 * num_leaves - 1, 1), dtype=NODE_DTYPE)
        ns = C.c_int32()
        nn = C.c_int32()
        fn = allreduce if allreduce is not None else C.cast(None, ALLREDUCE_FN)
        check(lib().hbg_boost_one_iteration(self.handle, _ptr(targets), _ptr(scores), loss, learning_rate,
                                            C.byref(p), fn, _ptr(ctx), _ptr(log), C.byref(ns), _ptr(nodes),
                                            C.byref(nn), _ptr(stream)))
        return log[: ns.value].copy(), nodes[: nn.value].copy()

    def set_profiling(self, enabled: bool) -> None:
        """Record CUDA events around each histogram kernel launch (measurement only)."""
        check(lib().hbg_dataset_set_profiling(self.handle, 1 if enabled else 0))

    def kernel_time(self) -> tuple[float, int]:
        """(summed ms, launches) of the histogram kernels recorded since the last call."""
        ms = C.c_double()
        n = C.c_int64()
        check(lib().hbg_dataset_kernel_time(self.handle, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            check(lib().hbg_dataset_destroy(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------- operators
def build_histograms_partitioned(data: Dataset, leaf: LeafState, precision=32) -> np.ndarray:
    """Drop-in for ``build_histograms_partitioned(data, leaf, precision)``
    (histogram.hpp:133-134).

    Returns the HistogramSet as a (num_features, max_bin) ``BIN_DTYPE`` array
    (feature-major, one entry per feature id). Counts are exact. ``precision``
    32 (bits32): fp32 inputs and per-warp sums reduced in fp64; 64 (bits64):
    fp64 inputs and fp64 accumulation throughout.
    """
    n = leaf.count()
    idx = np.ascontiguousarray(leaf.indices, dtype=np.int32)
    g = np.ascontiguousarray(leaf.gradients, dtype=np.float64)
    h = np.ascontiguousarray(leaf.hessians, dtype=np.float64)
    if len(g) != n or len(h) != n:
        raise InvalidArgument(HBG_ERR_INVALID_ARGUMENT, "leaf arrays disagree on length")
    out = np.zeros((data.num_features, data.max_bin), dtype=BIN_DTYPE)
    check(lib().hbg_build_histograms_ex(data.handle, _ptr(idx), n, _ptr(g), _ptr(h), _precision(precision),
                                        _ptr(out)))
    return out


def find_best_split(hists: np.ndarray, leaf_totals, min_data_in_leaf: int = 1, lam: float = 0.0):
    """find_best_split (tree.cpp:163-182) on the GPU; ``leaf_totals`` = (grad, hess, count).

    Returns a ``SPLIT_DTYPE`` record or None (std::nullopt)."""
    hists = np.ascontiguousarray(hists, dtype=BIN_DTYPE)
    d, k = hists.shape
    gt, ht, cnt = leaf_totals
    out = np.zeros(1, dtype=SPLIT_DTYPE)
    found = C.c_int32()
    check(lib().hbg_find_best_split(_ptr(hists), d, k, float(gt), float(ht), int(cnt),
                                    int(min_data_in_leaf), float(lam), _ptr(out), C.byref(found)))
    return out[0] if found.value else None


def find_best_threshold(hist: np.ndarray, feature_id: int, leaf_totals, min_data_in_leaf: int = 1,
                        lam: float = 0.0):
    """find_best_threshold (tree.cpp:76-112) for one feature's bins, on the GPU."""
    hist = np.ascontiguousarray(hist, dtype=BIN_DTYPE).reshape(1, -1)
    s = find_best_split(hist, leaf_totals, min_data_in_leaf, lam)
    if s is not None:
        s = s.copy()
        s["feature"] = feature_id
    return s


def subtract_device(parent, child, sibling, n_values: int, stream=None) -> None:
    """Histogram subtraction: sibling = parent - child (device SoA histograms)."""
    check(lib().hbg_subtract_device(_ptr(parent), _ptr(child), _ptr(sibling), n_values, _ptr(stream)))


def gather_leaf_device(indices, count: int, grad, hess, leaf_grad, leaf_hess, totals, stream=None):
    check(lib().hbg_gather_leaf_device(_ptr(indices), count, _ptr(grad), _ptr(hess), _ptr(leaf_grad),
                                       _ptr(leaf_hess), _ptr(totals), _ptr(stream)))


def best_split_device(hist, num_features: int, max_bin: int, grad_total: float, hess_total: float,
                      count: int, min_data_in_leaf: int, lam: float, out, stream=None) -> None:
    check(lib().hbg_best_split_device(_ptr(hist), num_features, max_bin, grad_total, hess_total,
                                      count, min_data_in_leaf, lam, _ptr(out), _ptr(stream)))


def best_split_device_totals(hist, num_features: int, max_bin: int, totals, count_dev,
                             min_data_in_leaf: int, lam: float, out, stream=None) -> None:
    check(lib().hbg_best_split_device_totals(_ptr(hist), num_features, max_bin, _ptr(totals),
                                             _ptr(count_dev), min_data_in_leaf, lam, _ptr(out),
                                             _ptr(stream)))


def hist_to_bins_device(hist, num_features: int, max_bin: int, bins, stream=None) -> None:
    check(lib().hbg_hist_to_bins_device(_ptr(hist), num_features, max_bin, _ptr(bins), _ptr(stream)))


def reduce_histograms_device(parts, n_values: int, out, stream=None) -> None:
    """reduce_private_histograms (histogram.cpp:147-157): out = sum of parts in order."""
    arr = (C.c_void_p * len(parts))(*[_ptr(p).value for p in parts])
    check(lib().hbg_reduce_histograms_device(arr, len(parts), n_values, _ptr(out), _ptr(stream)))


class Peer:
    """Exchange area of one rank for row-sharded growth inside the persistent
    kernel (hbg_peer_*): attach (same process) or open (IPC handle from
    another process) every other rank's area before growing."""

    HANDLE_BYTES = 64

    def __init__(self, ds: "Dataset", nranks: int, rank: int, ctas: int = 0, max_leaves: int = 255):
        h = C.c_void_p()
        p = hbg_grow_params(max_leaves, 0, 1, 0.0)
        check(lib().hbg_peer_create(ds.handle, nranks, rank, ctas, C.byref(p), C.byref(h)))
        self._h = h
        self.rank = rank

    @property
    def handle(self):
        return self._h

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * Peer.HANDLE_BYTES)()
        check(lib().hbg_peer_handle(self._h, buf))
        return bytes(buf)

    def open(self, peer_rank: int, handle: bytes):
        buf = (C.c_uint8 * Peer.HANDLE_BYTES).from_buffer_copy(handle)
        check(lib().hbg_peer_open(self._h, peer_rank, buf))

    def check(self):
        """Raise if a peer exchange timed out (synchronises the device)."""
        check(lib().hbg_peer_check(self._h))

    def attach(self, other: "Peer"):
        check(lib().hbg_peer_attach(self._h, other.rank, other._h))

    def close(self):
        if getattr(self, "_h", None):
            check(lib().hbg_peer_destroy(self._h))
            self._h = None


class Comm:
    """NCCL communicator for row-sharded growth (one process per GPU)."""

    ID_BYTES = 128

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * Comm.ID_BYTES)()
        check(lib().hbg_comm_get_unique_id(buf))
        return bytes(buf)

    def __init__(self, nranks: int, rank: int, unique_id: bytes, device: int):
        buf = (C.c_uint8 * Comm.ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib().hbg_comm_init(C.byref(h), nranks, rank, buf, device))
        self._h = h
        self.allreduce_fn = ALLREDUCE_FN(C.cast(lib().hbg_comm_allreduce, C.c_void_p).value)

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            check(lib().hbg_comm_destroy(self._h))
            self._h = None


def stats_close(a, b, tolerance: float):
    """histogram.cpp:12-15, vectorised."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = np.maximum(1.0, np.maximum(np.abs(a), np.abs(b)))
    return np.abs(a - b) <= tolerance * scale
