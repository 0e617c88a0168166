"""CPU oracle for the Meerkat hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product package
(paper_2305_17813_b200) never imports it and shares no code with it.

The arithmetic lives in meerkat_oracle.c (plain single-threaded C, cited line
by line against PAPER.md / SURVEY §8(c)); this module only marshals numpy
arrays through ctypes.  Pins that tie it to the paper and to mathematics
(golden example G0, brute-force path enumeration, scipy Dijkstra, invariants)
are in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

OK, E_INVALID_ARG, E_VERTEX_RANGE, E_WEIGHT, E_CAPACITY, E_OVERFLOW, E_STATE = range(7)
UNREACHED = np.uint64(0xFFFFFFFFFFFFFFFF)

u32p = ctypes.POINTER(ctypes.c_uint32)
u64p = ctypes.POINTER(ctypes.c_uint64)
u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "meerkat_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-Wall", src, "-o", _SO, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp = ctypes.c_void_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [ctypes.c_uint32, ctypes.c_int]
        L.orc_destroy.argtypes = [vp]
        L.orc_num_edges.restype = ctypes.c_uint64
        L.orc_num_edges.argtypes = [vp]
        L.orc_insert.argtypes = [vp, u32p, u32p, u32p, ctypes.c_uint64, u64p]
        L.orc_delete.argtypes = [vp, u32p, u32p, ctypes.c_uint64, u64p]
        L.orc_query.argtypes = [vp, u32p, u32p, ctypes.c_uint64, u8p, u32p]
        L.orc_export.argtypes = [vp, u32p, u32p, u32p]
        L.orc_sssp.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, u64p]
        L.orc_bfs.argtypes = [vp, ctypes.c_uint32, u64p]
        L.orc_invalidated.restype = ctypes.c_uint64
        L.orc_invalidated.argtypes = [ctypes.c_uint32, ctypes.c_uint32, u64p, u32p, u32p, ctypes.c_uint64, u8p, u64p]
        L.orc_dec_frontier_count.restype = ctypes.c_uint64
        L.orc_dec_frontier_count.argtypes = [vp, u64p, u8p]
        L.orc_check_tree.restype = ctypes.c_uint64
        L.orc_check_tree.argtypes = [vp, ctypes.c_uint32, ctypes.c_int, u64p, u32p]
        L.orc_pagerank.argtypes = [vp, ctypes.c_double, ctypes.c_double, ctypes.c_uint32,
                                   ctypes.POINTER(ctypes.c_double), u32p, ctypes.POINTER(ctypes.c_double)]
        L.orc_wcc.restype = ctypes.c_uint64
        L.orc_wcc.argtypes = [vp, u32p]
        L.orc_tc_count.restype = ctypes.c_uint64
        L.orc_tc_count.argtypes = [vp, vp, u32p, u32p, ctypes.c_uint64]
        _lib = L
    return _lib


def _a32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint32))


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleGraph:
    """The edge set of a directed (weighted) graph with the method's batch semantics."""

    def __init__(self, vertex_n: int, weighted: bool = True):
        self.V = int(vertex_n)
        self.weighted = bool(weighted)
        self._g = _L().orc_create(self.V, int(self.weighted))

    def __del__(self):
        if getattr(self, "_g", None) and _lib is not None:
            _lib.orc_destroy(self._g)
            self._g = None

    @property
    def num_edges(self) -> int:
        return int(_L().orc_num_edges(self._g))

    def insert(self, src, dst, w=None):
        s, d = _a32(src), _a32(dst)
        wp = None
        if w is not None:
            wa = _a32(w)
            wp = _p(wa, u32p)
        out = ctypes.c_uint64(0)
        st = _L().orc_insert(self._g, _p(s, u32p), _p(d, u32p), wp, len(s), ctypes.byref(out))
        return st, int(out.value)

    def delete(self, src, dst):
        s, d = _a32(src), _a32(dst)
        out = ctypes.c_uint64(0)
        st = _L().orc_delete(self._g, _p(s, u32p), _p(d, u32p), len(s), ctypes.byref(out))
        return st, int(out.value)

    def query(self, src, dst):
        s, d = _a32(src), _a32(dst)
        found = np.zeros(len(s), np.uint8)
        w = np.zeros(len(s), np.uint32)
        st = _L().orc_query(self._g, _p(s, u32p), _p(d, u32p), len(s), _p(found, u8p), _p(w, u32p))
        return st, found, w

    def edges(self):
        m = self.num_edges
        s = np.empty(m, np.uint32); d = np.empty(m, np.uint32); w = np.empty(m, np.uint32)
        _L().orc_export(self._g, _p(s, u32p), _p(d, u32p), _p(w, u32p))
        return s, d, w

    def sssp(self, source: int, unit: bool = False):
        node = np.empty(self.V, np.uint64)
        st = _L().orc_sssp(self._g, source, int(unit), _p(node, u64p))
        return st, node

    def bfs(self, source: int):
        node = np.empty(self.V, np.uint64)
        st = _L().orc_bfs(self._g, source, _p(node, u64p))
        return st, node

    def pagerank(self, d: float = 0.85, eps: float = 1e-5, max_iter: int = 1000, pr=None):
        """(status, pr f64[V], iterations, last delta).  pr=None: static start 1/V;
        else a warm start from the given vector (dynamic PageRank)."""
        x = np.full(self.V, 1.0 / self.V) if pr is None else np.array(pr, dtype=np.float64, copy=True)
        it = ctypes.c_uint32(0)
        dl = ctypes.c_double(0.0)
        st = _L().orc_pagerank(self._g, float(d), float(eps), int(max_iter),
                               x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(it), ctypes.byref(dl))
        return st, x, int(it.value), float(dl.value)

    def wcc(self):
        """(labels u32[V], components): label[v] = smallest id in v's weakly connected component."""
        lab = np.empty(self.V, np.uint32)
        n = _L().orc_wcc(self._g, _p(lab, u32p))
        return lab, int(n)

    def dec_frontier_count(self, node_old, invalid_flag) -> int:
        n = np.ascontiguousarray(node_old, dtype=np.uint64)
        f = np.ascontiguousarray(invalid_flag, dtype=np.uint8)
        return int(_L().orc_dec_frontier_count(self._g, _p(n, u64p), _p(f, u8p)))

    def check_tree(self, source: int, node, unit: bool = False):
        n = np.ascontiguousarray(node, dtype=np.uint64)
        fb = ctypes.c_uint32(0)
        bad = _L().orc_check_tree(self._g, source, int(unit), _p(n, u64p), ctypes.byref(fb))
        return int(bad), int(fb.value)


def tc_count(g1: OracleGraph, g2: OracleGraph, src, dst) -> int:
    """Count(G1, G2, edges) = sum over (u, v) of |adj_G1(u) ∩ adj_G2(v)|."""
    s, d = _a32(src), _a32(dst)
    return int(_L().orc_tc_count(g1._g, g2._g, _p(s, u32p), _p(d, u32p), len(s)))


def tc_static(g: OracleGraph) -> int:
    """Triangles of an undirected (symmetric) graph: Count(G, G, all directed edges) / 6
    ("degenerates to the static triangle counting case ... six times")."""
    s, d, _ = g.edges()
    c = tc_count(g, g, s, d)
    assert c % 6 == 0, c
    return c // 6


def tc_delta(g_after: OracleGraph, g_update: OracleGraph, src, dst, insert: bool):
    """Triangles added (insert) or removed (delete) by a batch given in both orientations, by the
    paper's inclusion-exclusion: S1 = Count(after, after), S2 = Count(after, update),
    S3 = Count(update, update); added = S1/2 - S2/2 + S3/6, removed = S1/2 + S2/2 + S3/6.
    Returns (delta, (S1, S2, S3))."""
    s1 = tc_count(g_after, g_after, src, dst)
    s2 = tc_count(g_after, g_update, src, dst)
    s3 = tc_count(g_update, g_update, src, dst)
    num = 3 * s1 - 3 * s2 + s3 if insert else 3 * s1 + 3 * s2 + s3
    assert num % 6 == 0, (s1, s2, s3)
    return num // 6, (s1, s2, s3)


def invalidated(vertex_n: int, source: int, node_old, src, dst):
    """(invalid_flag u8[V], n_direct) for a deleted batch against the old tree."""
    n = np.ascontiguousarray(node_old, dtype=np.uint64)
    s, d = _a32(src), _a32(dst)
    flag = np.zeros(vertex_n, np.uint8)
    nd = ctypes.c_uint64(0)
    _L().orc_invalidated(vertex_n, source, _p(n, u64p), _p(s, u32p), _p(d, u32p), len(s), _p(flag, u8p),
                         ctypes.byref(nd))
    return flag, int(nd.value)


def pack(dist: int, parent: int) -> int:
    return (int(dist) << 32) | int(parent)


def unpack(node) -> tuple:
    node = np.asarray(node, dtype=np.uint64)
    return (node >> np.uint64(32)).astype(np.int64), (node & np.uint64(0xFFFFFFFF)).astype(np.int64)
