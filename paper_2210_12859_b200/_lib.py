"""Loads libfkd_b200.so (built in-tree by ``__graft_entry__.build()``).

Fails loudly when the library is missing: the package has no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FKD_LIB") or os.path.join(HERE, "libfkd_b200.so")  # FKD_LIB: A/B builds

# every symbol include/fkd_b200.h declares
EXPORTS = (
    "fkd_default_options", "fkd_tree_create", "fkd_tree_create_device", "fkd_tree_destroy",
    "fkd_tree_size", "fkd_tree_dim", "fkd_tree_replicas", "fkd_tree_add_replicas", "fkd_morton_keys", "fkd_run_batch", "fkd_run_batches", "fkd_submit_batches", "fkd_wait", "fkd_run_batch_device", "fkd_run_batches_device", "fkd_fcp", "fkd_knn",
    "fkd_build_tree", "fkd_build_tree_device", "fkd_tree_build", "fkd_result_hash", "fkd_random_points", "fkd_clustered_points",
    "fkd_host_alloc", "fkd_host_free", "fkd_debug_block_trace", "fkd_last_error", "fkd_version", "fkd_trace_batch",
    "fkd_file_info", "fkd_read_file_device", "fkd_write_file", "fkd_tree_load",
)


class fkd_batch_options(C.Structure):
    _fields_ = [("kind", C.c_int32), ("k", C.c_int32), ("max_radius", C.c_float),
                ("engine", C.c_int32), ("threads", C.c_int32), ("collect_stats", C.c_int32),
                ("flags", C.c_uint32)]


class fkd_query_stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("nodes_visited", C.c_int64), ("nodes_processed", C.c_int64)]


class fkd_timings(C.Structure):
    _fields_ = [("order_ms", C.c_float), ("walk_ms", C.c_float), ("tail_ms", C.c_float), ("launches", C.c_int32),
                ("walk_launches", C.c_int32), ("overflowed", C.c_int64)]


class fkd_device_batch(C.Structure):
    _fields_ = [("d_queries", C.c_void_p), ("m", C.c_int64), ("dim", C.c_int32), ("opt", fkd_batch_options),
                ("d_counts", C.c_void_p), ("d_hits", C.c_void_p), ("stats", C.c_void_p),
                ("d_per_query", C.c_void_p), ("timings", C.c_void_p), ("status", C.c_int32)]


class fkd_host_batch(C.Structure):
    _fields_ = [("queries", C.c_void_p), ("m", C.c_int64), ("dim", C.c_int32), ("opt", fkd_batch_options),
                ("counts", C.c_void_p), ("hits", C.c_void_p), ("stats", C.c_void_p), ("status", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the B200 query path)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    lib.fkd_last_error.restype = C.c_char_p
    lib.fkd_version.restype = C.c_char_p
    lib.fkd_default_options.argtypes = [vp]
    lib.fkd_tree_create.argtypes = [vp, i64, i32, vp, i32, vp]
    lib.fkd_tree_create_device.argtypes = [vp, i64, i32, vp, vp]
    lib.fkd_tree_destroy.argtypes = [vp]
    lib.fkd_tree_size.restype = i64
    lib.fkd_tree_size.argtypes = [vp]
    lib.fkd_tree_dim.restype = i32
    lib.fkd_tree_dim.argtypes = [vp]
    lib.fkd_tree_replicas.restype = i32
    lib.fkd_tree_replicas.argtypes = [vp, vp, i32]
    lib.fkd_tree_add_replicas.argtypes = [vp, vp, i32]
    lib.fkd_morton_keys.argtypes = [vp, vp, i64, i32, vp, vp, vp]
    lib.fkd_run_batch.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp]
    lib.fkd_run_batch_device.argtypes = [vp, vp, i64, i32, vp, vp, vp, vp, vp, vp, vp]
    lib.fkd_run_batches_device.argtypes = [vp, vp, i32, vp]
    lib.fkd_run_batches.argtypes = [vp, vp, i32]
    lib.fkd_submit_batches.argtypes = [vp, vp, i32, vp]
    lib.fkd_wait.argtypes = [vp]
    lib.fkd_fcp.argtypes = [vp, vp, i32, C.c_float, vp, vp, vp]
    lib.fkd_knn.argtypes = [vp, vp, i32, i32, C.c_float, vp, vp, vp]
    lib.fkd_build_tree.argtypes = [vp, i64, i32, vp]
    lib.fkd_build_tree_device.argtypes = [vp, i64, i32, vp, vp]
    lib.fkd_tree_build.argtypes = [vp, i64, i32, vp, i32, vp, vp]
    lib.fkd_result_hash.restype = C.c_uint64
    lib.fkd_result_hash.argtypes = [vp, vp, i64, i32]
    lib.fkd_random_points.argtypes = [C.c_uint64, C.c_uint64, i64, i32, vp]
    lib.fkd_clustered_points.argtypes = [C.c_uint64, C.c_uint64, i64, i32, i32, C.c_float, vp]
    lib.fkd_trace_batch.argtypes = [vp, vp, i32, i32, i32, i32, C.c_float, vp, vp, vp, vp, i64, vp]
    lib.fkd_file_info.argtypes = [C.c_char_p, i32, vp, vp]
    lib.fkd_read_file_device.argtypes = [C.c_char_p, i32, vp, i64, vp, vp, vp]
    lib.fkd_write_file.argtypes = [C.c_char_p, i32, vp, i64, i32]
    lib.fkd_tree_load.argtypes = [C.c_char_p, vp, i32, vp]
    lib.fkd_debug_block_trace.argtypes = [vp, vp, i64]
    lib.fkd_host_alloc.restype = vp
    lib.fkd_host_alloc.argtypes = [C.c_size_t]
    lib.fkd_host_free.argtypes = [vp]
    return lib


LIB = _load()
