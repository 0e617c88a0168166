"""Multi-GPU (vertex-partitioned) graphs — SURVEY §8(e).

One process per GPU.  The library does the partitioning, routing and the tree
rounds itself (csrc/part.cu): a partitioned graph is an ordinary `Graph`
created with a TRANSPORT, and every call on it is collective.  This module
only sets the transport up:

* NCCL (production, NVLink / NVSwitch): rank 0 asks the library for an
  ncclUniqueId, torch.distributed broadcasts it, and the library creates and
  owns its communicator (`meerkat_config.nccl_id`);
* a host all-to-all-v over any torch.distributed group (gloo: the CPU tests and
  the one-GPU multi-process GPU tests, where NCCL refuses two ranks on one
  device) passed as `meerkat_config.exchange`.

Placement (owner / row of a vertex) is the library's (`owner_map`).  Results
are bit-identical to one GPU.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import check
from .graph import Graph


def owner_map(vertex_n: int, world_size: int, ids) -> tuple:
    """(owner rank, row there) of global ids on a partitioned graph (meerkat_owner_map; host only)."""
    a = np.ascontiguousarray(np.asarray(ids, np.uint32))
    own = np.empty(a.size, np.uint32)
    row = np.empty(a.size, np.uint32)
    check(_lib.lib().meerkat_owner_map(int(vertex_n), int(world_size), ctypes.c_void_p(a.ctypes.data), a.size,
                                       ctypes.c_void_p(own.ctypes.data), ctypes.c_void_p(row.ctypes.data)),
          "meerkat_owner_map")
    return own, row


def rows_of(vertex_n: int, world_size: int, rank: int) -> int:
    """Vertices held by `rank`."""
    return len(range(rank, vertex_n, world_size))


class HostExchange:
    """meerkat_exchange_fn over a torch.distributed group: the library hands over host buffers laid
    out as consecutive per-rank segments; one all_to_all_single (uint8) moves them."""

    def __init__(self, group=None):
        self.group = group
        self.ws = dist.get_world_size(group)
        self.error = None
        self.fn = _lib.EXCHANGE_FN(self._call)   # keep a reference: the library holds the pointer

    def _call(self, ctx, send, send_bytes, recv, recv_bytes):
        try:
            sb = [int(send_bytes[p]) for p in range(self.ws)]
            rb = [int(recv_bytes[p]) for p in range(self.ws)]
            src = np.ctypeslib.as_array((ctypes.c_uint8 * max(sum(sb), 1)).from_address(send)) if sum(sb) else \
                np.zeros(1, np.uint8)
            dst = np.ctypeslib.as_array((ctypes.c_uint8 * max(sum(rb), 1)).from_address(recv)) if sum(rb) else \
                np.zeros(1, np.uint8)
            ti = torch.from_numpy(src[: sum(sb)] if sum(sb) else src[:0])
            to = torch.from_numpy(dst[: sum(rb)] if sum(rb) else dst[:0])
            dist.all_to_all_single(to, ti, rb, sb, group=self.group)
            return 0
        except Exception as e:   # reported as MEERKAT_E_NCCL by the library
            self.error = e
            return 1


class DistGraph(Graph):
    """This rank's part of a vertex-partitioned dynamic graph G.  Every method is
    collective.  transport: "nccl" (the library's own communicator), "host" (HostExchange over the
    group), or "auto" (nccl when the group's backend is NCCL)."""

    def __init__(self, vertex_n: int, weighted: bool = True, hashing: bool = True, load_factor: float = 0.7,
                 degree_hints=None, pool_slabs: int = 0, hash_seed: int = 0, device=None, stream=None,
                 reverse: bool = False, in_degree_hints=None, group=None, transport: str = "auto",
                 exchange_pairs: int = 0):
        ws, rank = dist.get_world_size(group), dist.get_rank(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        if stream is None:   # the library's stream must be the one torch (and NCCL) order against
            stream = torch.cuda.current_stream(device)
        if transport == "auto":
            transport = "nccl" if dist.get_backend(group) == "nccl" else "host"
        self.group = group
        nccl_id, xfn = None, None
        if transport == "nccl":
            buf = (ctypes.c_uint8 * 128)()
            obj = [None]
            if rank == 0:
                check(_lib.lib().meerkat_nccl_unique_id(buf, 128), "meerkat_nccl_unique_id")
                obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0, group=group)
            nccl_id = ctypes.create_string_buffer(obj[0], 128)
        else:
            self._xchg = HostExchange(group)
            xfn = self._xchg.fn
        self._nccl_id = nccl_id
        super().__init__(vertex_n, weighted=weighted, hashing=hashing, load_factor=load_factor,
                         degree_hints=degree_hints, pool_slabs=pool_slabs, hash_seed=hash_seed,
                         device=device.index or 0, stream=stream, reverse=reverse,
                         in_degree_hints=in_degree_hints, world_size=ws, rank=rank,
                         nccl_id=nccl_id, exchange=xfn, exchange_pairs=exchange_pairs)
        self.ws = ws
        self.n_local = rows_of(vertex_n, ws, rank)

    def export_edges(self):
        """All live edges of all ranks, sorted (every rank gets the full list; host gather)."""
        s, d, w = super().export_edges()
        parts = [None] * self.ws
        dist.all_gather_object(parts, (s, d, w), group=self.group)
        s = np.concatenate([p[0] for p in parts])
        d = np.concatenate([p[1] for p in parts])
        w = np.concatenate([p[2] for p in parts])
        o = np.lexsort((d, s))
        return s[o], d[o], w[o]

    def stats_global(self) -> dict:
        """meerkat_stats_get summed over ranks (host gather)."""
        parts = [None] * self.ws
        dist.all_gather_object(parts, self.stats(), group=self.group)
        return {k: sum(p[k] for p in parts) for k in parts[0]}
