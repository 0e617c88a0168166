"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is input plumbing only (see synth.c's header): it draws graphs and
batches, and holds none of the method's arithmetic.  Workload recipes follow
SURVEY.md §8(d) ("Configs as synthetic inputs", "Generator specification").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None

# Graph500 R-MAT initiator; d = 1 - a - b - c = 0.05
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19
SEED_GRAPH, SEED_W, SEED_BATCH = 1, 2, 3


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-shared", "-fPIC", "-Wall", src, "-o", _SO])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        lib.synth_rmat.restype = ctypes.c_uint64
        lib.synth_rmat.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                   u32p, u32p, u32p]
        lib.synth_uniform.restype = ctypes.c_uint64
        lib.synth_uniform.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      u32p, u32p, u32p]
        lib.synth_sample_distinct.restype = ctypes.c_int
        lib.synth_sample_distinct.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, u64p]
        lib.synth_rmat_draws.restype = None
        lib.synth_rmat_draws.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                         ctypes.c_uint64, ctypes.c_uint64, u32p, u32p, u32p]
        lib.synth_scramble.restype = ctypes.c_uint32
        lib.synth_scramble.argtypes = [ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64]
        lib.synth_draw.restype = ctypes.c_uint64
        lib.synth_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = lib
    return _lib


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def rmat(scale: int, ef: int, seed_graph: int = SEED_GRAPH, seed_w: int = SEED_W, scramble: bool = True):
    """Unique R-MAT edges (src, dst, w) as uint32 arrays, sorted by (src, dst)."""
    n = ef << scale
    s = np.empty(n, np.uint32)
    d = np.empty(n, np.uint32)
    w = np.empty(n, np.uint32)
    m = _L().synth_rmat(scale, ef, RMAT_A, RMAT_B, RMAT_C, seed_graph, seed_w, int(scramble), _p32(s), _p32(d), _p32(w))
    return s[:m].copy(), d[:m].copy(), w[:m].copy()


def rmat_draws(scale: int, n: int, first: int, seed_graph: int, seed_w: int = SEED_W, scramble: bool = True,
               scramble_seed: int = SEED_GRAPH):
    """n raw R-MAT draws (duplicates and self-loops kept) starting at draw index `first`, from
    seed_graph's stream; ids scrambled with scramble_seed (default: the base graph's labelling,
    so the fresh edges' hubs are the base graph's hubs)."""
    s = np.empty(n, np.uint32)
    d = np.empty(n, np.uint32)
    w = np.empty(n, np.uint32)
    _L().synth_rmat_draws(scale, n, RMAT_A, RMAT_B, RMAT_C, seed_graph, seed_w, int(scramble), scramble_seed, first,
                          _p32(s), _p32(d), _p32(w))
    return s, d, w


def uniform(n: int, m: int, seed_graph: int = SEED_GRAPH, seed_w: int = SEED_W):
    """G(n, m): m distinct non-loop directed edges in draw order, w ~ U{1..64}."""
    s = np.empty(m, np.uint32)
    d = np.empty(m, np.uint32)
    w = np.empty(m, np.uint32)
    got = _L().synth_uniform(n, m, seed_graph, seed_w, _p32(s), _p32(d), _p32(w))
    return s[:got].copy(), d[:got].copy(), w[:got].copy()


def sample_distinct(m: int, k: int, seed: int) -> np.ndarray:
    out = np.empty(k, np.uint64)
    rc = _L().synth_sample_distinct(m, k, seed, _p64(out))
    if rc:
        raise ValueError(f"sample_distinct({m}, {k}) failed rc={rc}")
    return out.astype(np.int64)


def scramble(v: int, bits: int, seed: int = SEED_GRAPH) -> int:
    return int(_L().synth_scramble(v, bits, seed))


def draw(seed: int, stream: int, ctr: int) -> int:
    return int(_L().synth_draw(seed, stream, ctr))


@dataclass
class DynamicWorkload:
    """A base graph plus held-out insert batches and sampled delete batches.

    Inserts are held-out edges of the generated graph (absent at insert time);
    deletes are sampled without replacement from the base edges that are never
    held out, so each is present at its delete time.
    """
    vertex_n: int
    base: tuple          # (src, dst, w) of the initial graph
    inserts: list        # list of (src, dst, w)
    deletes: list        # list of (src, dst, w)
    source: int


def rmat_dynamic(scale: int, ef: int, batch: int, n_ins: int, n_del: int, seed_graph=SEED_GRAPH,
                 seed_w=SEED_W, seed_batch=SEED_BATCH) -> DynamicWorkload:
    s, d, w = rmat(scale, ef, seed_graph, seed_w)
    m = len(s)
    pick = sample_distinct(m, batch * (n_ins + n_del), seed_batch)
    held = pick[: batch * n_ins]
    dels = pick[batch * n_ins:]
    keep = np.ones(m, bool)
    keep[held] = False
    base = (s[keep], d[keep], w[keep])
    inserts = [(s[held[i * batch:(i + 1) * batch]], d[held[i * batch:(i + 1) * batch]],
                w[held[i * batch:(i + 1) * batch]]) for i in range(n_ins)]
    deletes = [(s[dels[i * batch:(i + 1) * batch]], d[dels[i * batch:(i + 1) * batch]],
                w[dels[i * batch:(i + 1) * batch]]) for i in range(n_del)]
    # source: scrambled id of raw vertex 0 (R-MAT's hub), SURVEY §8(d)
    src = scramble(0, scale, seed_graph)
    return DynamicWorkload(1 << scale, base, inserts, deletes, src)


def grid_dynamic(side: int, batch: int, n_ins: int, n_del: int, seed_w=SEED_W,
                 seed_batch=SEED_BATCH) -> DynamicWorkload:
    """The road-like stress case of SURVEY §8(d) ("not in BJ"): a side x side grid, vertex r*side + c,
    directed edges to the 4 neighbours, w ~ U{1..64} (seeded), source 0 (a corner).  Diameter ~2*side,
    so SSSP / BFS take thousands of rounds and decremental batches invalidate deep subtrees (the
    paper's USAfull regime).  Held-out inserts / sampled deletes as rmat_dynamic."""
    r, c = np.divmod(np.arange(side * side, dtype=np.int64), side)
    v = r * side + c
    srcs, dsts = [], []
    for dr, dc in ((0, 1), (0, -1), (1, 0), (-1, 0)):
        ok = (r + dr >= 0) & (r + dr < side) & (c + dc >= 0) & (c + dc < side)
        srcs.append(v[ok])
        dsts.append(((r + dr) * side + (c + dc))[ok])
    s = np.concatenate(srcs).astype(np.uint32)
    d = np.concatenate(dsts).astype(np.uint32)
    o = np.lexsort((d, s))
    s, d = s[o], d[o]
    w = np.random.Generator(np.random.PCG64(seed_w)).integers(1, 65, s.size).astype(np.uint32)
    m = s.size
    pick = sample_distinct(m, batch * (n_ins + n_del), seed_batch)
    held, dels = pick[: batch * n_ins], pick[batch * n_ins:]
    keep = np.ones(m, bool)
    keep[held] = False
    cut = lambda idx, i: (s[idx[i * batch:(i + 1) * batch]], d[idx[i * batch:(i + 1) * batch]],
                          w[idx[i * batch:(i + 1) * batch]])
    return DynamicWorkload(side * side, (s[keep], d[keep], w[keep]), [cut(held, i) for i in range(n_ins)],
                           [cut(dels, i) for i in range(n_del)], 0)


def degrees(src: np.ndarray, vertex_n: int) -> np.ndarray:
    """Out-degree of each vertex in an edge list (degree hints for construction)."""
    return np.bincount(src, minlength=vertex_n).astype(np.uint32)
