"""ctypes declarations of include/meerkat.h (argument marshalling only).

The shared library is built in-tree (paper_2305_17813_b200/libmeerkat.so) by
paper_2305_17813_b200/build.py.  There is no fallback: if the library is
missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(HERE, "libmeerkat.so")
if os.environ.get("MEERKAT_SO_PATH"):   # A/B experiments: another in-tree build of the same sources
    SO_PATH = os.path.abspath(os.environ["MEERKAT_SO_PATH"])

STATUS = {
    0: "MEERKAT_OK", 1: "MEERKAT_E_INVALID_ARG", 2: "MEERKAT_E_VERTEX_RANGE", 3: "MEERKAT_E_WEIGHT",
    4: "MEERKAT_E_CAPACITY", 5: "MEERKAT_E_OVERFLOW", 6: "MEERKAT_E_STATE", 7: "MEERKAT_E_CUDA",
    8: "MEERKAT_E_NCCL", 9: "MEERKAT_E_PARTITION",
}
OK, E_INVALID_ARG, E_VERTEX_RANGE, E_WEIGHT, E_CAPACITY, E_OVERFLOW, E_STATE, E_CUDA, E_NCCL, E_PARTITION = range(10)
MAX_RANKS = 64

# Every function include/meerkat.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "meerkat_status_string", "meerkat_create", "meerkat_destroy", "meerkat_set_stream", "meerkat_sync",
    "meerkat_insert_batch", "meerkat_delete_batch", "meerkat_query_batch", "meerkat_export_edges",
    "meerkat_stats_get", "meerkat_sssp_create", "meerkat_bfs_create", "meerkat_sssp_incremental",
    "meerkat_bfs_incremental", "meerkat_sssp_decremental", "meerkat_bfs_decremental", "meerkat_tree_recompute",
    "meerkat_tree_nodes", "meerkat_tree_invalidated", "meerkat_tree_stats_get", "meerkat_tree_destroy",
    "meerkat_nccl_unique_id", "meerkat_owner_map", "meerkat_tree_timeline",
    "meerkat_check", "meerkat_trees_incremental", "meerkat_trees_decremental",
    "meerkat_insert_batch_trees", "meerkat_delete_batch_trees",
    "meerkat_pagerank_create", "meerkat_pagerank_update", "meerkat_pagerank_recompute", "meerkat_pagerank_values",
    "meerkat_pagerank_stats_get", "meerkat_pagerank_destroy",
    "meerkat_sssp_vanilla_create", "meerkat_bfs_vanilla_create", "meerkat_tree_distances",
    "meerkat_tc_count", "meerkat_tc_static", "meerkat_tc_incremental", "meerkat_tc_decremental",
    "meerkat_wcc_create", "meerkat_wcc_recompute", "meerkat_wcc_incremental", "meerkat_wcc_labels",
    "meerkat_wcc_components", "meerkat_wcc_destroy", "meerkat_tree_recompute_scheme",
    "meerkat_wcc_incremental_tracked", "meerkat_probe_latency", "meerkat_counters_async",
]


class MeerkatError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


class Config(ctypes.Structure):
    _fields_ = [
        ("vertex_n", ctypes.c_uint32), ("weighted", ctypes.c_uint32), ("hashing", ctypes.c_uint32),
        ("load_factor", ctypes.c_float), ("degree_hints", ctypes.c_void_p), ("pool_slabs", ctypes.c_uint64),
        ("hash_seed", ctypes.c_uint64), ("device", ctypes.c_int), ("stream", ctypes.c_void_p),
        ("reverse", ctypes.c_uint32), ("in_degree_hints", ctypes.c_void_p),
        ("world_size", ctypes.c_uint32), ("rank", ctypes.c_uint32), ("update_tracking", ctypes.c_uint32),
        ("nccl_id", ctypes.c_void_p), ("exchange", ctypes.c_void_p), ("exchange_ctx", ctypes.c_void_p),
        ("exchange_pairs", ctypes.c_uint32), ("in_load_factor", ctypes.c_float),
    ]


# meerkat_exchange_fn: host all-to-all-v of a partitioned graph's transport
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                               ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64))


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "vertex_n", "edges", "head_slabs", "buckets", "pool_capacity", "pool_used", "bytes_device",
        "kernel_launches", "version", "in_edges", "in_head_slabs", "in_pool_used")]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class TreeStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "rounds", "propagate_rounds", "direct_invalid", "invalidated", "frontier_edges", "items", "slabs_read",
        "scan_slabs", "improved", "alg_bytes", "version")] + [("source", ctypes.c_uint32),
                                                             ("unit_weights", ctypes.c_uint32),
                                                             ("exchanges", ctypes.c_uint64)]

    def as_dict(self):
        return {n: int(getattr(self, n)) for n, _ in self._fields_}


class PageRankStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint64), ("delta", ctypes.c_double), ("slabs", ctypes.c_uint64),
                ("in_edges", ctypes.c_uint64), ("atomics", ctypes.c_uint64), ("alg_bytes", ctypes.c_uint64),
                ("version", ctypes.c_uint64), ("warm", ctypes.c_uint32), ("pad", ctypes.c_uint32)]

    def as_dict(self):
        return {n: (float(getattr(self, n)) if n == "delta" else int(getattr(self, n)))
                for n, _ in self._fields_ if n != "pad"}


class Latency(ctypes.Structure):
    _fields_ = [("dram_load_ns", ctypes.c_double), ("l2_load_ns", ctypes.c_double),
                ("dram_atomic_ns", ctypes.c_double), ("grid_sync_us", ctypes.c_double),
                ("grid_blocks", ctypes.c_uint32)]


_lib = None


def lib():
    """Load libmeerkat.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing; build it with `python -m paper_2305_17813_b200.build`")
    L = ctypes.CDLL(SO_PATH)
    vp, u32, u64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
    pvp = ctypes.POINTER(ctypes.c_void_p)
    pu64 = ctypes.POINTER(ctypes.c_uint64)
    sig = {
        "meerkat_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "meerkat_create": (ctypes.c_int, [ctypes.POINTER(Config), pvp]),
        "meerkat_destroy": (ctypes.c_int, [vp]),
        "meerkat_set_stream": (ctypes.c_int, [vp, vp]),
        "meerkat_sync": (ctypes.c_int, [vp]),
        "meerkat_insert_batch": (ctypes.c_int, [vp, vp, vp, vp, u64, pu64]),
        "meerkat_delete_batch": (ctypes.c_int, [vp, vp, vp, u64, pu64]),
        "meerkat_query_batch": (ctypes.c_int, [vp, vp, vp, u64, vp, vp]),
        "meerkat_export_edges": (ctypes.c_int, [vp, vp, vp, vp, u64, pu64]),
        "meerkat_stats_get": (ctypes.c_int, [vp, ctypes.POINTER(Stats)]),
        "meerkat_sssp_create": (ctypes.c_int, [vp, u32, pvp]),
        "meerkat_bfs_create": (ctypes.c_int, [vp, u32, pvp]),
        "meerkat_sssp_incremental": (ctypes.c_int, [vp, vp, vp, vp, vp, u64]),
        "meerkat_bfs_incremental": (ctypes.c_int, [vp, vp, vp, vp, u64]),
        "meerkat_sssp_decremental": (ctypes.c_int, [vp, vp, vp, vp, u64]),
        "meerkat_bfs_decremental": (ctypes.c_int, [vp, vp, vp, vp, u64]),
        "meerkat_tree_recompute": (ctypes.c_int, [vp, vp]),
        "meerkat_tree_nodes": (ctypes.c_int, [vp, vp]),
        "meerkat_tree_invalidated": (ctypes.c_int, [vp, vp, u64, pu64]),
        "meerkat_tree_stats_get": (ctypes.c_int, [vp, ctypes.POINTER(TreeStats)]),
        "meerkat_tree_destroy": (ctypes.c_int, [vp]),
        "meerkat_tree_timeline": (ctypes.c_int, [vp, pu64, pu64, u64, pu64]),
        "meerkat_check": (ctypes.c_int, [vp, pu64]),
        "meerkat_trees_incremental": (ctypes.c_int, [vp, pvp, u32, vp, vp, vp, u64]),
        "meerkat_trees_decremental": (ctypes.c_int, [vp, pvp, u32, vp, vp, u64]),
        "meerkat_insert_batch_trees": (ctypes.c_int, [vp, vp, vp, vp, u64, pvp, u32, pu64]),
        "meerkat_delete_batch_trees": (ctypes.c_int, [vp, vp, vp, u64, pvp, u32, pu64]),
        "meerkat_nccl_unique_id": (ctypes.c_int, [vp, u64]),
        "meerkat_owner_map": (ctypes.c_int, [u32, u32, vp, u64, vp, vp]),
        "meerkat_pagerank_create": (ctypes.c_int, [vp, ctypes.c_double, ctypes.c_double, u32, pvp]),
        "meerkat_pagerank_update": (ctypes.c_int, [vp, vp]),
        "meerkat_pagerank_recompute": (ctypes.c_int, [vp, vp]),
        "meerkat_pagerank_values": (ctypes.c_int, [vp, vp]),
        "meerkat_pagerank_stats_get": (ctypes.c_int, [vp, ctypes.POINTER(PageRankStats)]),
        "meerkat_pagerank_destroy": (ctypes.c_int, [vp]),
        "meerkat_sssp_vanilla_create": (ctypes.c_int, [vp, u32, pvp]),
        "meerkat_bfs_vanilla_create": (ctypes.c_int, [vp, u32, pvp]),
        "meerkat_tree_distances": (ctypes.c_int, [vp, vp]),
        "meerkat_tc_count": (ctypes.c_int, [vp, vp, vp, vp, u64, pu64]),
        "meerkat_tc_static": (ctypes.c_int, [vp, pu64]),
        "meerkat_tc_incremental": (ctypes.c_int, [vp, vp, vp, vp, u64, pu64, pu64]),
        "meerkat_tc_decremental": (ctypes.c_int, [vp, vp, vp, vp, u64, pu64, pu64]),
        "meerkat_wcc_create": (ctypes.c_int, [vp, pvp]),
        "meerkat_wcc_recompute": (ctypes.c_int, [vp, vp]),
        "meerkat_wcc_incremental": (ctypes.c_int, [vp, vp, vp, vp, u64]),
        "meerkat_wcc_labels": (ctypes.c_int, [vp, vp]),
        "meerkat_wcc_components": (ctypes.c_int, [vp, pu64]),
        "meerkat_wcc_destroy": (ctypes.c_int, [vp]),
        "meerkat_tree_recompute_scheme": (ctypes.c_int, [vp, vp, u32]),
        "meerkat_wcc_incremental_tracked": (ctypes.c_int, [vp, vp]),
        "meerkat_probe_latency": (ctypes.c_int, [vp, ctypes.POINTER(Latency)]),
        "meerkat_counters_async": (ctypes.c_int, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(status: int, where: str) -> int:
    if status != OK:
        raise MeerkatError(status, where)
    return status
