"""ctypes binding of libsc_b200.so (the C-ABI declared in include/sc_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
visible, every entry point raises DeviceError.  Status codes map onto the reference's
exception classes (specluster/errors.py:8-29): -1..-99 -> InputError, <= -100 ->
DeviceError (a SpeclusterError, CLI exit code 1).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeviceError, InputError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SC_LIB_PATH") or os.path.join(_HERE, "libsc_b200.so")

SC_SYM_VARIANT = 0x1
SC_NO_CUDA_GRAPH = 0x2
SC_L2_PERSIST = 0x4
SC_FORCE_WEIGHTED = 0x8
SC_FORCE_SELL = 0x10
SC_CREATE_KEEP_WEIGHTS = 0x1
SC_CREATE_FP32_VALUES = 0x2
SC_CREATE_REORDER_BFS = 0x4
SC_CREATE_PANELS = 0x8
SC_CREATE_WINDOWS = 0x10


class GraphInfo(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("ncols", ctypes.c_int64),
        ("col_offset", ctypes.c_int64), ("ntiles", ctypes.c_int64), ("long_rows", ctypes.c_int64),
        ("unit_weights", ctypes.c_int32), ("rp64", ctypes.c_int32), ("device_bytes", ctypes.c_int64),
        ("device", ctypes.c_int32), ("sm_count", ctypes.c_int32),
        ("stored_entries", ctypes.c_int64),
        ("panel_groups", ctypes.c_int64), ("panel_bytes", ctypes.c_int64),
        ("zstride", ctypes.c_int64), ("n_gpus", ctypes.c_int32), ("window_items", ctypes.c_int32),
    ]


class Timing(ctypes.Structure):
    _fields_ = [("sample_ms", ctypes.c_double), ("power_ms", ctypes.c_double),
                ("kernel_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double)]


EXPORTS = (
    "sc_version", "sc_last_error", "sc_device_count", "sc_graph_create", "sc_shard_create",
    "sc_graph_destroy", "sc_graph_info_get", "sc_sample_irwin_hall", "sc_set_x0",
    "sc_power_iterate", "sc_shard_step", "sc_shard_scale", "sc_shard_irwin_hall",
    "sc_kmeans_create", "sc_kmeans_create_from_graph", "sc_kmeans_destroy", "sc_kmeans_pp",
    "sc_kmeans_lloyd", "sc_seqsum", "sc_sell_order", "sc_graph_order", "sc_graph_create_ex",
    "sc_shard_step_range", "sc_shard_scale_range", "sc_generate_sbm", "sc_csr_info",
    "sc_csr_download", "sc_csr_destroy", "sc_graph_create_from_csr", "sc_csr_download_weights",
    "sc_generate_knn3d", "sc_generate_dcsbm", "sc_shard_buffers",
    "sc_shard_set_peers", "sc_shard_barrier", "sc_ipc_export", "sc_ipc_import", "sc_ipc_release",
    "sc_keyed_sums", "sc_contingency", "sc_cut_sums", "sc_power_iterate_block",
    "sc_kmeans_create_nd", "sc_kmeans_lloyd_sorted", "sc_release_cached_memory",
    "sc_gather_f64", "sc_graph_build_panels", "sc_graph_download_f", "sc_kmeans_set_flags",
    "sc_graph_create_multi", "sc_graph_shard_layout", "sc_shard_create_from_csr",
    "sc_graph_build_windows",
)

_lib = None


def load() -> ctypes.CDLL:
    """Load the native library (no GPU needed for loading)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"native library {LIB_PATH} is missing; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    # the library carries its own (static) CUDA runtime; load every kernel when it initialises
    # instead of at each kernel's first launch (which put ~10 ms into the first clustering)
    os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u32, u64, f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                  ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double)
    PP = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "sc_version": ([], i32),
        "sc_last_error": ([], ctypes.c_char_p),
        "sc_device_count": ([], i32),
        "sc_graph_create": ([P, P, P, P, i64, i64, i32, PP], i32),
        "sc_shard_create": ([P, P, P, P, i64, i64, i64, i64, i64, i32, PP], i32),
        "sc_graph_destroy": ([P], None),
        "sc_graph_info_get": ([P, ctypes.POINTER(GraphInfo)], i32),
        "sc_graph_build_panels": ([P], i32),
        "sc_graph_build_windows": ([P], i32),
        "sc_graph_download_f": ([P, P], i32),
        "sc_sample_irwin_hall": ([P, u64, u64, P], i32),
        "sc_set_x0": ([P, P], i32),
        "sc_power_iterate": ([P, i32, f64, u32, P, P, ctypes.POINTER(Timing)], i32),
        "sc_shard_step": ([P, P, P, P, P, f64, u32, P], i32),
        "sc_shard_scale": ([P, P, P, u32, P], i32),
        "sc_shard_irwin_hall": ([P, u64, u64, P, P], i32),
        "sc_kmeans_create": ([P, i64, i32, PP], i32),
        "sc_kmeans_create_from_graph": ([P, PP], i32),
        "sc_kmeans_destroy": ([P], None),
        "sc_kmeans_pp": ([P, i32, i32, P, P, P, P], i32),
        "sc_kmeans_lloyd": ([P, i32, i32, P, i32, f64, P, P, P, P, P], i32),
        "sc_kmeans_set_flags": ([P, u32], i32),
        "sc_graph_create_multi": ([P, P, P, P, i64, i64, i32, P, u32, PP], i32),
        "sc_graph_shard_layout": ([P, i32, P, P, P, P], i32),
        "sc_shard_create_from_csr": ([P, i64, i64, P, i64, i64, PP], i32),
        "sc_seqsum": ([P, i32, P, i32, P, P], i32),
        "sc_sell_order": ([P, i64, P], i32),
        "sc_graph_create_ex": ([P, P, P, P, i64, i64, i32, u32, PP], i32),
        "sc_shard_step_range": ([P, i64, i64, P, P, P, P, f64, u32, P], i32),
        "sc_shard_scale_range": ([P, i64, i64, P, P, u32, P], i32),
        "sc_graph_order": ([P, P], i32),
        "sc_generate_sbm": ([i64, i32, f64, f64, f64, f64, u64, u64, i32, PP], i32),
        "sc_csr_info": ([P, P, P, P], i32),
        "sc_csr_download": ([P, P, P, P, P], i32),
        "sc_csr_destroy": ([P], None),
        "sc_csr_download_weights": ([P, P], i32),
        "sc_generate_knn3d": ([i64, i32, f64, i32, f64, u64, u64, i32, PP], i32),
        "sc_generate_dcsbm": ([i64, P, i32, f64, f64, f64, i32, i32, f64, f64, f64, u64, u64, i32, PP],
                              i32),
        "sc_graph_create_from_csr": ([P, u32, PP], i32),
        "sc_shard_buffers": ([P, PP, PP], i32),
        "sc_shard_set_peers": ([P, P, P, i32, i32], i32),
        "sc_shard_barrier": ([P, P], i32),
        "sc_ipc_export": ([P, P], i32),
        "sc_ipc_import": ([P, i32, PP], i32),
        "sc_ipc_release": ([P], i32),
        "sc_keyed_sums": ([P, P, i64, i32, i32, P, P], i32),
        "sc_contingency": ([P, P, i64, i32, i32, i32, P], i32),
        "sc_cut_sums": ([P, P, P, P, i64, i64, i32, i32, P], i32),
        "sc_power_iterate_block": ([P, i32, i32, P, P, P, ctypes.POINTER(Timing)], i32),
        "sc_kmeans_create_nd": ([P, i64, i32, i32, PP], i32),
        "sc_kmeans_lloyd_sorted": ([P, i32, i32, P, i32, f64, P, P, P, P], i32),
        "sc_release_cached_memory": ([i32], i64),
        "sc_gather_f64": ([P, P, i64, P, P], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(status: int) -> None:
    if status == 0:
        return
    msg = (load().sc_last_error() or b"").decode(errors="replace")
    if -100 < status < 0:
        raise InputError(msg)
    raise DeviceError(f"[status {status}] {msg}")


def require_device() -> ctypes.CDLL:
    L = load()
    if L.sc_device_count() < 1:
        raise DeviceError("no CUDA device visible; the B200 path has no CPU fallback: "
                          + (L.sc_last_error() or b"").decode(errors="replace"))
    return L


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)
