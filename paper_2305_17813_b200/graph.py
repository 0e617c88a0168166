"""Thin Python binding of include/meerkat.h (argument marshalling only).

Every step of the hot path runs in libmeerkat.so's CUDA kernels; this module
turns torch tensors / numpy arrays into pointers and statuses into exceptions.
Arrays may live on the device (torch CUDA tensors) or on the host (numpy,
CPU tensors); host arrays are staged by the library (meerkat.h "Pointer
arguments").  Vertex ids and weights are 32-bit (uint32 or int32 bit patterns).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check

try:  # torch is plumbing only (device memory, streams)
    import torch
except Exception:  # pragma: no cover
    torch = None


def _is_torch(x):
    return torch is not None and isinstance(x, torch.Tensor)


_I32 = torch.int32 if torch is not None else None


def _handles(trees):
    """ctypes array of tree handles (cached per tuple of trees: the hot path passes the same list)."""
    key = tuple(id(t) for t in trees)
    arr = _HANDLES.get(key)
    if arr is None or [a for a in arr] != [t._h.value for t in trees]:
        arr = (ctypes.c_void_p * len(trees))(*[t._h.value for t in trees])
        if len(_HANDLES) > 64:
            _HANDLES.clear()
        _HANDLES[key] = arr
    return arr


_HANDLES = {}


def _u32(x, stream=None):
    """(pointer, keepalive, n) for a 32-bit id/weight array.  A CUDA tensor that has to be converted
    (dtype or layout) becomes a temporary allocated on torch's current stream; the library reads it
    later on the graph's `stream`, so the temporary is recorded on that stream and the caching
    allocator does not hand its block out again before the library's work there is done."""
    if x is None:
        return None, None, 0
    if _is_torch(x) and x.dtype is _I32 and x.is_contiguous():   # fast path: nothing to convert
        return ctypes.c_void_p(x.data_ptr()), x, x.numel()
    if _is_torch(x):
        y = x
        if y.dtype not in (torch.int32, torch.uint32):
            y = y.to(torch.int32)
        y = y.contiguous()
        if y is not x and y.is_cuda and stream is not None:
            y.record_stream(stream)
        return ctypes.c_void_p(y.data_ptr()), y, y.numel()
    a = np.ascontiguousarray(np.asarray(x), dtype=np.uint32)
    return ctypes.c_void_p(a.ctypes.data), a, a.size


def _torch_stream(stream, device):
    """The torch stream object of a graph's stream (for record_stream), or None (legacy default
    stream, which orders against every other stream of the device)."""
    if torch is None or stream is None:
        return None
    if isinstance(stream, int):
        return torch.cuda.ExternalStream(stream, device=device) if stream else None
    return stream


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


class Graph:
    """A dynamic graph G stored as per-vertex SlabHash tables on one GPU."""

    def __init__(self, vertex_n: int, weighted: bool = True, hashing: bool = True, load_factor: float = 0.7,
                 degree_hints=None, pool_slabs: int = 0, hash_seed: int = 0, device: int = 0, stream=None,
                 reverse: bool = False, in_degree_hints=None, world_size: int = 1, rank: int = 0,
                 update_tracking: bool = False, nccl_id=None, exchange=None, exchange_pairs: int = 0,
                 in_load_factor: float = 0.0):
        """world_size / rank with nccl_id (a 128-byte ctypes buffer) or exchange (a
        _lib.EXCHANGE_FN) make a partitioned graph (see dist.DistGraph); every call is then collective."""
        L = _lib.lib()
        hp, self._hints_keep, _ = _u32(degree_hints)
        ip, self._ihints_keep, _ = _u32(in_degree_hints)
        cfg = _lib.Config(vertex_n=vertex_n, weighted=int(weighted), hashing=int(hashing),
                          load_factor=float(load_factor), degree_hints=hp, pool_slabs=int(pool_slabs),
                          hash_seed=int(hash_seed), device=int(device), stream=_stream_ptr(stream),
                          reverse=int(reverse), in_degree_hints=ip, world_size=int(world_size), rank=int(rank),
                          update_tracking=int(update_tracking),
                          nccl_id=ctypes.cast(nccl_id, ctypes.c_void_p) if nccl_id is not None else None,
                          exchange=ctypes.cast(exchange, ctypes.c_void_p) if exchange is not None else None,
                          exchange_ctx=None, exchange_pairs=int(exchange_pairs),
                          in_load_factor=float(in_load_factor))
        self._exchange_keep = exchange
        h = ctypes.c_void_p()
        check(L.meerkat_create(ctypes.byref(cfg), ctypes.byref(h)), "meerkat_create")
        self._h = h
        self._tstream = _torch_stream(stream, device)
        self.vertex_n = int(vertex_n)
        self.weighted = bool(weighted)
        self.reverse = bool(reverse)
        self.world_size = int(world_size)
        self.rank = int(rank)
        self.device = int(device)
        self._trees = []
        self._pageranks = []
        self._wccs = []

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if getattr(self, "_h", None):
            for t in list(self._trees):
                t.close()
            for p in list(self._pageranks):
                p.close()
            for c in list(self._wccs):
                c.close()
            _lib.lib().meerkat_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream):
        check(_lib.lib().meerkat_set_stream(self._h, _stream_ptr(stream)), "meerkat_set_stream")
        self._tstream = _torch_stream(stream, self.device)

    def probe_latency(self) -> dict:
        """DRAM / L2 / atomic dependent-access latency and grid-barrier cost on this graph's device
        (meerkat_probe_latency): the terms of the tree calls' latency floor."""
        out = _lib.Latency()
        check(_lib.lib().meerkat_probe_latency(self._h, ctypes.byref(out)), "meerkat_probe_latency")
        return {k: getattr(out, k) for k, _ in _lib.Latency._fields_}

    def sync(self):
        check(_lib.lib().meerkat_sync(self._h), "meerkat_sync")

    # ------------------------------------------------------------------ batches
    def insert(self, src, dst, w=None, count: bool = True, raise_on_error: bool = True, seed=None):
        """InsertEdges.  seed: trees whose next incremental call (same batch) this insert seeds
        (meerkat_insert_batch_trees)."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, n2 = _u32(dst, self._tstream)
        wp, kw, n3 = _u32(w, self._tstream)
        assert n == n2 and (w is None or n3 == n)
        out = ctypes.c_uint64(0)
        ob = ctypes.byref(out) if count else None
        if seed:
            arr = _handles(seed)
            st, fn = _lib.lib().meerkat_insert_batch_trees(self._h, sp, dp, wp, n, arr, len(seed), ob), \
                "meerkat_insert_batch_trees"
        else:
            st, fn = _lib.lib().meerkat_insert_batch(self._h, sp, dp, wp, n, ob), "meerkat_insert_batch"
        if raise_on_error:
            check(st, fn)
        return (int(out.value) if count else None) if raise_on_error else (st, int(out.value))

    def delete(self, src, dst, count: bool = True, raise_on_error: bool = True, seed=None):
        """DeleteEdges.  seed: trees whose next decremental call (same batch) this delete seeds
        (meerkat_delete_batch_trees)."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, n2 = _u32(dst, self._tstream)
        assert n == n2
        out = ctypes.c_uint64(0)
        ob = ctypes.byref(out) if count else None
        if seed:
            arr = _handles(seed)
            st, fn = _lib.lib().meerkat_delete_batch_trees(self._h, sp, dp, n, arr, len(seed), ob), \
                "meerkat_delete_batch_trees"
        else:
            st, fn = _lib.lib().meerkat_delete_batch(self._h, sp, dp, n, ob), "meerkat_delete_batch"
        if raise_on_error:
            check(st, fn)
        return (int(out.value) if count else None) if raise_on_error else (st, int(out.value))

    def query(self, src, dst, raise_on_error: bool = True):
        """found (uint8) and stored weight (uint32, 0 when absent) per queried edge."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, n2 = _u32(dst, self._tstream)
        assert n == n2
        if _is_torch(src) and src.is_cuda:
            found = torch.empty(n, dtype=torch.uint8, device=src.device)
            w = torch.empty(n, dtype=torch.int32, device=src.device)
            fp, wp = found.data_ptr(), w.data_ptr()
        else:
            found = np.zeros(n, np.uint8)
            w = np.zeros(n, np.uint32)
            fp, wp = found.ctypes.data, w.ctypes.data
        st = _lib.lib().meerkat_query_batch(self._h, sp, dp, n, ctypes.c_void_p(fp), ctypes.c_void_p(wp))
        if raise_on_error:
            check(st, "meerkat_query_batch")
            return found, w
        return st, found, w

    def export_edges(self):
        """All live edges (src, dst, w) as host uint32 arrays, sorted by (src, dst)."""
        L = _lib.lib()
        n = ctypes.c_uint64(0)
        st = L.meerkat_export_edges(self._h, None, None, None, 0, ctypes.byref(n))
        if st not in (_lib.OK, _lib.E_CAPACITY):
            check(st, "meerkat_export_edges")
        cap = int(n.value)
        s = np.zeros(max(cap, 1), np.uint32); d = np.zeros(max(cap, 1), np.uint32); w = np.zeros(max(cap, 1), np.uint32)
        check(L.meerkat_export_edges(self._h, ctypes.c_void_p(s.ctypes.data), ctypes.c_void_p(d.ctypes.data),
                                     ctypes.c_void_p(w.ctypes.data), cap, ctypes.byref(n)), "meerkat_export_edges")
        m = int(n.value)
        s, d, w = s[:m], d[:m], w[:m]
        order = np.lexsort((d, s))
        return s[order], d[order], w[order]

    def check(self):
        """Structural store check (meerkat_check): (violations, vertex, slab, next, kind) of the first."""
        info = (ctypes.c_uint64 * 5)()
        _lib.lib().meerkat_check(self._h, info)
        return tuple(int(x) for x in info)

    def counters_async(self, out):
        """Enqueue a copy of the cumulative counters (inserted, deleted, pool slabs) into `out`, a
        3-element uint64/int64 tensor (pinned host or CUDA) or array, on the graph's stream; no
        synchronisation (meerkat_counters_async)."""
        ptr = out.data_ptr() if _is_torch(out) else out.ctypes.data
        check(_lib.lib().meerkat_counters_async(self._h, ctypes.c_void_p(ptr)), "meerkat_counters_async")

    def stats(self) -> dict:
        st = _lib.Stats()
        check(_lib.lib().meerkat_stats_get(self._h, ctypes.byref(st)), "meerkat_stats_get")
        return st.as_dict()

    # ------------------------------------------------------------------ trees
    def trees_incremental(self, trees, src, dst, w=None):
        """Fused incremental update of several trees with the batch just inserted (one launch)."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, _ = _u32(dst, self._tstream)
        wp, kw, _ = _u32(w, self._tstream)
        arr = _handles(trees)
        check(_lib.lib().meerkat_trees_incremental(self._h, arr, len(trees), sp, dp, wp, n),
              "meerkat_trees_incremental")

    def trees_decremental(self, trees, src, dst):
        """Fused decremental update of several trees with the batch just deleted (one launch)."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, _ = _u32(dst, self._tstream)
        arr = _handles(trees)
        check(_lib.lib().meerkat_trees_decremental(self._h, arr, len(trees), sp, dp, n), "meerkat_trees_decremental")

    def insert_trees(self, trees, src, dst, w=None, count: bool = True):
        """insert(seed=trees) + trees_incremental(trees): two launches, the trees' batch prologue
        inside the insert kernel.  Returns the number of edges inserted (count=True)."""
        n = self.insert(src, dst, w, count=count, seed=trees)
        self.trees_incremental(trees, src, dst, w)
        return n

    def delete_trees(self, trees, src, dst, count: bool = True):
        """delete(seed=trees) + trees_decremental(trees): two launches, the invalidation of the
        deleted tree edges inside the delete kernel.  Returns the number deleted (count=True)."""
        n = self.delete(src, dst, count=count, seed=trees)
        self.trees_decremental(trees, src, dst)
        return n

    def pagerank(self, damping: float = 0.85, error_margin: float = 1e-5, max_iter: int = 1000) -> "PageRank":
        """Static PageRank of the current graph (needs reverse=True: in-edge mirror)."""
        return PageRank(self, damping, error_margin, max_iter)

    def wcc(self) -> "WCC":
        """Static weakly connected components of the current graph."""
        return WCC(self)

    # ------------------------------------------------------------------ triangle counting
    def tc_count(self, other: "Graph", src, dst) -> int:
        """Count(self, other, edges) = sum over (u, v) of |adj_self(u) ∩ adj_other(v)|."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, _ = _u32(dst, self._tstream)
        out = ctypes.c_uint64(0)
        check(_lib.lib().meerkat_tc_count(self._h, other._h, sp, dp, n, ctypes.byref(out)), "meerkat_tc_count")
        return int(out.value)

    def tc_static(self) -> int:
        """Triangles of this undirected (symmetric) graph."""
        out = ctypes.c_uint64(0)
        check(_lib.lib().meerkat_tc_static(self._h, ctypes.byref(out)), "meerkat_tc_static")
        return int(out.value)

    def tc_delta(self, update: "Graph", src, dst, insert: bool):
        """Triangles added (insert) / removed by a batch already applied to this graph; `update` holds
        exactly the batch; src/dst give it in both orientations.  Returns (delta, (S1, S2, S3))."""
        sp, ks, n = _u32(src, self._tstream)
        dp, kd, _ = _u32(dst, self._tstream)
        out = ctypes.c_uint64(0)
        s3 = (ctypes.c_uint64 * 3)()
        fn = _lib.lib().meerkat_tc_incremental if insert else _lib.lib().meerkat_tc_decremental
        check(fn(self._h, update._h, sp, dp, n, ctypes.byref(out), s3), fn.__name__)
        return int(out.value), tuple(int(x) for x in s3)

    def sssp(self, source: int) -> "Tree":
        return Tree(self, source, unit=False)

    def bfs(self, source: int) -> "Tree":
        return Tree(self, source, unit=True)

    def sssp_vanilla(self, source: int) -> "Tree":
        """Static distances only, 32-bit atomics (the paper's vanilla variant)."""
        return Tree(self, source, unit=False, vanilla=True)

    def bfs_vanilla(self, source: int) -> "Tree":
        return Tree(self, source, unit=True, vanilla=True)


class Tree:
    """Dependence tree T_G of packed <distance, parent> words."""

    def __init__(self, graph: Graph, source: int, unit: bool, vanilla: bool = False):
        L = _lib.lib()
        h = ctypes.c_void_p()
        if vanilla:
            fn = L.meerkat_bfs_vanilla_create if unit else L.meerkat_sssp_vanilla_create
        else:
            fn = L.meerkat_bfs_create if unit else L.meerkat_sssp_create
        check(fn(graph._h, source, ctypes.byref(h)), fn.__name__)
        self.vanilla = vanilla
        self._h = h
        self.graph = graph
        self.unit = unit
        self.source = source
        graph._trees.append(self)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().meerkat_tree_destroy(self._h)
            self._h = None
            if self in self.graph._trees:
                self.graph._trees.remove(self)

    def incremental(self, src, dst, w=None):
        sp, ks, n = _u32(src, self.graph._tstream)
        dp, kd, _ = _u32(dst, self.graph._tstream)
        L = _lib.lib()
        if self.unit:
            check(L.meerkat_bfs_incremental(self.graph._h, self._h, sp, dp, n), "meerkat_bfs_incremental")
        else:
            wp, kw, _ = _u32(w, self.graph._tstream)
            check(L.meerkat_sssp_incremental(self.graph._h, self._h, sp, dp, wp, n), "meerkat_sssp_incremental")

    def decremental(self, src, dst):
        sp, ks, n = _u32(src, self.graph._tstream)
        dp, kd, _ = _u32(dst, self.graph._tstream)
        L = _lib.lib()
        fn = L.meerkat_bfs_decremental if self.unit else L.meerkat_sssp_decremental
        check(fn(self.graph._h, self._h, sp, dp, n), fn.__name__)

    def recompute(self, iteration_scheme: int = 2):
        """Static re-run; iteration_scheme 1 = one work item per vertex (the paper's IterationScheme1),
        2 = <vertex, bucket> items (default, IterationScheme2)."""
        if iteration_scheme == 2:
            check(_lib.lib().meerkat_tree_recompute(self.graph._h, self._h), "meerkat_tree_recompute")
        else:
            check(_lib.lib().meerkat_tree_recompute_scheme(self.graph._h, self._h, int(iteration_scheme)),
                  "meerkat_tree_recompute_scheme")

    def nodes(self, out=None):
        """Packed nodes, uint64 numpy array (or into a given int64 CUDA tensor)."""
        if out is not None:
            check(_lib.lib().meerkat_tree_nodes(self._h, ctypes.c_void_p(out.data_ptr())), "meerkat_tree_nodes")
            return out
        a = np.empty(self.graph.vertex_n, np.uint64)
        check(_lib.lib().meerkat_tree_nodes(self._h, ctypes.c_void_p(a.ctypes.data)), "meerkat_tree_nodes")
        return a

    def distances(self, out=None):
        """dist[v] (uint32, UINT32_MAX when unreached) as a numpy array (or into an int32 CUDA tensor)."""
        if out is not None:
            check(_lib.lib().meerkat_tree_distances(self._h, ctypes.c_void_p(out.data_ptr())), "meerkat_tree_distances")
            return out
        a = np.empty(self.graph.vertex_n, np.uint32)
        check(_lib.lib().meerkat_tree_distances(self._h, ctypes.c_void_p(a.ctypes.data)), "meerkat_tree_distances")
        return a

    def invalidated(self):
        L = _lib.lib()
        n = ctypes.c_uint64(0)
        st = L.meerkat_tree_invalidated(self._h, None, 0, ctypes.byref(n))
        if st not in (_lib.OK, _lib.E_CAPACITY):
            check(st, "meerkat_tree_invalidated")
        a = np.zeros(max(int(n.value), 1), np.uint32)
        check(L.meerkat_tree_invalidated(self._h, ctypes.c_void_p(a.ctypes.data), int(n.value), ctypes.byref(n)),
              "meerkat_tree_invalidated")
        return np.sort(a[: int(n.value)])

    def timeline(self, items: bool = False):
        """Device timestamps (ns) of the last call: start and every grid barrier; returns the deltas in
        us (with items=True, pairs (us, frontier items of that interval's round, 0 for other phases))."""
        buf = (ctypes.c_uint64 * 48)()
        itm = (ctypes.c_uint64 * 48)()
        n = ctypes.c_uint64(0)
        check(_lib.lib().meerkat_tree_timeline(self._h, buf, itm, 48, ctypes.byref(n)), "meerkat_tree_timeline")
        ts = [int(buf[i]) for i in range(int(n.value))]
        dt = [(b - a) / 1e3 for a, b in zip(ts, ts[1:])]
        return [(x, int(itm[i])) for i, x in enumerate(dt)] if items else dt

    def stats(self) -> dict:
        st = _lib.TreeStats()
        check(_lib.lib().meerkat_tree_stats_get(self._h, ctypes.byref(st)), "meerkat_tree_stats_get")
        return st.as_dict()


class PageRank:
    """PageRank vector of a graph: static on creation, dynamic (warm-started) by update()."""

    def __init__(self, graph: Graph, damping: float, error_margin: float, max_iter: int):
        h = ctypes.c_void_p()
        check(_lib.lib().meerkat_pagerank_create(graph._h, float(damping), float(error_margin), int(max_iter),
                                                 ctypes.byref(h)), "meerkat_pagerank_create")
        self._h = h
        self.graph = graph
        graph._pageranks.append(self)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().meerkat_pagerank_destroy(self._h)
            self._h = None
            if self in self.graph._pageranks:
                self.graph._pageranks.remove(self)

    def update(self):
        """Dynamic PageRank after batches: warm start from the current values."""
        check(_lib.lib().meerkat_pagerank_update(self.graph._h, self._h), "meerkat_pagerank_update")

    def recompute(self):
        check(_lib.lib().meerkat_pagerank_recompute(self.graph._h, self._h), "meerkat_pagerank_recompute")

    def values(self, out=None):
        """PR as a float64 numpy array (or into a given float64 CUDA tensor)."""
        if out is not None:
            check(_lib.lib().meerkat_pagerank_values(self._h, ctypes.c_void_p(out.data_ptr())),
                  "meerkat_pagerank_values")
            return out
        a = np.empty(self.graph.vertex_n, np.float64)
        check(_lib.lib().meerkat_pagerank_values(self._h, ctypes.c_void_p(a.ctypes.data)), "meerkat_pagerank_values")
        return a

    def stats(self) -> dict:
        st = _lib.PageRankStats()
        check(_lib.lib().meerkat_pagerank_stats_get(self._h, ctypes.byref(st)), "meerkat_pagerank_stats_get")
        return st.as_dict()


class WCC:
    """Weakly connected component labels: static on creation, incremental after inserts."""

    def __init__(self, graph: Graph):
        h = ctypes.c_void_p()
        check(_lib.lib().meerkat_wcc_create(graph._h, ctypes.byref(h)), "meerkat_wcc_create")
        self._h = h
        self.graph = graph
        graph._wccs.append(self)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().meerkat_wcc_destroy(self._h)
            self._h = None
            if self in self.graph._wccs:
                self.graph._wccs.remove(self)

    def incremental(self, src, dst):
        """Union of the batch just inserted, then full compression."""
        sp, ks, n = _u32(src, self.graph._tstream)
        dp, kd, _ = _u32(dst, self.graph._tstream)
        check(_lib.lib().meerkat_wcc_incremental(self.graph._h, self._h, sp, dp, n), "meerkat_wcc_incremental")

    def incremental_tracked(self):
        """The UpdateIterator path: union the edges written since the last call (needs a
        graph created with update_tracking=True), compress, reset the tracking."""
        check(_lib.lib().meerkat_wcc_incremental_tracked(self.graph._h, self._h), "meerkat_wcc_incremental_tracked")

    def recompute(self):
        check(_lib.lib().meerkat_wcc_recompute(self.graph._h, self._h), "meerkat_wcc_recompute")

    def labels(self, out=None):
        if out is not None:
            check(_lib.lib().meerkat_wcc_labels(self._h, ctypes.c_void_p(out.data_ptr())), "meerkat_wcc_labels")
            return out
        a = np.empty(self.graph.vertex_n, np.uint32)
        check(_lib.lib().meerkat_wcc_labels(self._h, ctypes.c_void_p(a.ctypes.data)), "meerkat_wcc_labels")
        return a

    def components(self) -> int:
        out = ctypes.c_uint64(0)
        check(_lib.lib().meerkat_wcc_components(self._h, ctypes.byref(out)), "meerkat_wcc_components")
        return int(out.value)
