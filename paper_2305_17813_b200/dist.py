"""Multi-GPU (vertex-partitioned) graph and trees — SURVEY §8(e).

One process per GPU.  Rank r owns every vertex v with v % world_size == r:
its out-edges live in rank r's slab store and its tree node in rank r's tree.
All compute runs in libmeerkat.so (`meerkat_route` partitions a batch by owner,
`meerkat_dtree_phase` runs one phase of the tree update); this module only
moves bytes between ranks with torch.distributed — NCCL all-to-all over
NVLink / NVSwitch in production, or any other backend (gloo) through host
memory — and sums frontier sizes for termination:

* an update batch is routed by owner(src) with ONE all-to-all, then applied
  locally (counts are all-reduced);
* an SSSP/BFS round = local expansion (relaxations of local vertices applied in
  place, the rest emitted as <x, packed candidate>) -> one all-to-all -> the
  owners apply them with the same packed atomicMin -> all-reduce of the local
  frontier sizes (stop at 0).  Decremental: the deleted batch is routed by
  owner(dst) for the parent test; invalidation propagates in rounds
  of <x, expected parent> messages; the invalid sets are all-gathered
  and every rank streams its own slabs for valid->invalid edges.

Results are bit-identical to one GPU (the fixpoint does not depend on the
order of relaxations).  All calls are collective: every rank calls
the same sequence with its own (possibly empty) batch.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from ._lib import check
from .graph import Graph, _u32


# ------------------------------------------------------------------ host-side plumbing (pure functions)

def owner_of(v, world_size: int):
    return np.asarray(v, dtype=np.int64) % world_size


def interleave(parts, world_size: int, total: int) -> np.ndarray:
    """Global array from per-rank arrays of owned entries: out[l * ws + r] = parts[r][l]."""
    out = np.empty(total, dtype=parts[0].dtype if len(parts) else np.uint64)
    for r, p in enumerate(parts):
        out[r::world_size] = p[: len(range(r, total, world_size))]
    return out


def local_count(vertex_n: int, world_size: int, rank: int) -> int:
    return len(range(rank, vertex_n, world_size))


class Transport:
    """Variable-size exchanges over a torch.distributed process group."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.ws = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.staged = dist.get_backend(group) != "nccl"   # gloo etc.: via host memory

    def _dev(self):
        return torch.device("cpu") if self.staged else self.device

    def alltoallv(self, send: torch.Tensor, send_counts, elem: int = 1) -> torch.Tensor:
        """send: 1-D tensor whose rows for rank r are contiguous (send_counts[r] rows of `elem` values)."""
        dev = self._dev()
        sc = torch.tensor(list(send_counts), dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        rcl = rc.tolist()
        scl = sc.tolist()
        s = send.to(dev) if send.device != dev else send
        recv = torch.empty(sum(rcl) * elem, dtype=send.dtype, device=dev)
        dist.all_to_all_single(recv, s.contiguous(), [c * elem for c in rcl], [c * elem for c in scl], group=self.group)
        return recv.to(self.device) if self.staged else recv, rcl

    def alltoallv_known(self, send: torch.Tensor, send_counts, recv_counts, elem: int = 1) -> torch.Tensor:
        """alltoallv when both sides' row counts are already known (no count exchange)."""
        dev = self._dev()
        s = send.to(dev) if send.device != dev else send
        recv = torch.empty(sum(recv_counts) * elem, dtype=send.dtype, device=dev)
        dist.all_to_all_single(recv, s.contiguous(), [c * elem for c in recv_counts], [c * elem for c in send_counts],
                               group=self.group)
        return recv.to(self.device) if self.staged else recv

    def allreduce_sum(self, x: int) -> int:
        t = torch.tensor([int(x)], dtype=torch.int64, device=self._dev())
        dist.all_reduce(t, group=self.group)
        return int(t.item())

    def allgather_var(self, t: torch.Tensor) -> list:
        """All ranks' 1-D tensors (different lengths), as a list indexed by rank."""
        dev = self._dev()
        n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
        ns = [torch.empty_like(n) for _ in range(self.ws)]
        dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        m = max(ns) if ns else 0
        pad = torch.zeros(max(m, 1), dtype=t.dtype, device=dev)
        pad[: t.numel()] = t.to(dev)
        outs = [torch.empty_like(pad) for _ in range(self.ws)]
        dist.all_gather(outs, pad, group=self.group)
        res = [o[:k] for o, k in zip(outs, ns)]
        return [r.to(self.device) for r in res] if self.staged else res


# ------------------------------------------------------------------ the partitioned graph

class DistGraph:
    """Vertex-partitioned dynamic graph: this rank's part of G."""

    def __init__(self, vertex_n: int, weighted: bool = True, hashing: bool = True, load_factor: float = 0.7,
                 degree_hints=None, pool_slabs: int = 0, hash_seed: int = 0, device=None, stream=None, group=None):
        self.tp = Transport(group, device)
        self.ws, self.rank = self.tp.ws, self.tp.rank
        self.vertex_n = int(vertex_n)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.tp.device = self.device
        hints = None
        if degree_hints is not None:
            hints = np.ascontiguousarray(np.asarray(degree_hints, np.uint32)[self.rank::self.ws])
        if stream is None:   # the library's stream must be the one torch (and NCCL) order against
            stream = torch.cuda.current_stream(self.device)
        self.g = Graph(vertex_n, weighted=weighted, hashing=hashing, load_factor=load_factor, degree_hints=hints,
                       pool_slabs=pool_slabs, hash_seed=hash_seed, device=self.device.index or 0, stream=stream,
                       world_size=self.ws, rank=self.rank)
        self.weighted = weighted
        self.n_local = local_count(self.vertex_n, self.ws, self.rank)

    def close(self):
        self.g.close()

    def _t(self, a):
        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            return a.to(self.device).to(torch.int32).contiguous() if a.dtype != torch.int32 or a.device != self.device \
                else a.contiguous()
        return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.uint32)).view(np.int32)).to(self.device)

    def route(self, a, b, c=None, key_is_b: bool = False):
        """Partition rows (a, b[, c]) by owner(key) with meerkat_route, then one all-to-all.
        Returns the rows this rank owns (device int32 tensors) and the per-source-rank counts."""
        a, b, c = self._t(a), self._t(b), self._t(c)
        n = a.numel()
        cols = 3 if c is not None else 2
        out = torch.empty((cols, max(n, 1)), dtype=torch.int32, device=self.device)
        counts = (ctypes.c_uint64 * self.ws)()
        check(_lib.lib().meerkat_route(self.g._h, int(key_is_b), ctypes.c_void_p(a.data_ptr()),
                                       ctypes.c_void_p(b.data_ptr()),
                                       ctypes.c_void_p(c.data_ptr()) if c is not None else None, n,
                                       ctypes.c_void_p(out[0].data_ptr()), ctypes.c_void_p(out[1].data_ptr()),
                                       ctypes.c_void_p(out[2].data_ptr()) if c is not None else None,
                                       counts), "meerkat_route")
        send = out[:, :n].t().contiguous().view(-1)          # rows grouped by destination rank
        recv, rcounts = self.tp.alltoallv(send, list(counts), elem=cols)
        rows = recv.view(-1, cols)
        return [rows[:, i].contiguous() for i in range(cols)], rcounts, list(counts)

    def insert(self, src, dst, w=None, count: bool = True):
        (cols, _, _) = self.route(src, dst, w)
        n = self.g.insert(cols[0], cols[1], cols[2] if w is not None else None, count=count)
        return self.tp.allreduce_sum(n) if count else None

    def delete(self, src, dst, count: bool = True):
        (cols, _, _) = self.route(src, dst)
        n = self.g.delete(cols[0], cols[1], count=count)
        return self.tp.allreduce_sum(n) if count else None

    def query(self, src, dst):
        """found / weight per queried edge, in this rank's input order."""
        s = self._t(src)
        idx = torch.arange(s.numel(), dtype=torch.int32, device=self.device)
        (cols, rcounts, scounts) = self.route(s, dst, idx)
        found, w = self.g.query(cols[0], cols[1])
        ans = torch.stack([found.to(torch.int32), w, cols[2]], 1).contiguous().view(-1)
        back, _ = self.tp.alltoallv(ans, rcounts, elem=3)         # answers return to the asking rank
        back = back.view(-1, 3)
        out_f = torch.zeros(s.numel(), dtype=torch.uint8, device=self.device)
        out_w = torch.zeros(s.numel(), dtype=torch.int32, device=self.device)
        pos = back[:, 2].long()
        out_f[pos] = back[:, 0].to(torch.uint8)
        out_w[pos] = back[:, 1]
        return out_f, out_w

    def export_edges(self):
        """All live edges of all ranks (every rank gets the full sorted list)."""
        s, d, w = self.g.export_edges()
        parts = [self.tp.allgather_var(torch.from_numpy(x.view(np.int32)).to(self.device)) for x in (s, d, w)]
        s, d, w = (torch.cat(p).cpu().numpy().view(np.uint32) for p in parts)
        o = np.lexsort((d, s))
        return s[o], d[o], w[o]

    # ------------------------------------------------------------------ fused tree updates
    def trees_incremental(self, trees, src, dst, w=None):
        """Incremental update of several trees (e.g. SSSP + BFS) with the batch just inserted, in
        lock step: the batch is routed once and every round moves all trees' messages with ONE
        count exchange and ONE message all-to-all (rounds = the slowest tree's, not the sum)."""
        cols, _, _ = self.route(src, dst, w)
        n = cols[0].numel()
        res = [t._phase(_lib.D_INC_SEED, cols[0] if n else None, cols[1] if n else None,
                        (cols[2] if (n and not t.unit and w is not None) else None), n) for t in trees]
        self._fused_loop(trees, _lib.D_RELAX, _lib.D_APPLY_RELAX, res)

    def trees_decremental(self, trees, src, dst):
        """Decremental update of several trees in lock step (see trees_incremental)."""
        cols, _, _ = self.route(src, dst, key_is_b=True)
        n = cols[0].numel()
        res = [t._phase(_lib.D_DEC_INVALIDATE, cols[0] if n else None, cols[1] if n else None, None, n)
               for t in trees]
        res = self._fused_loop(trees, _lib.D_PROPAGATE, _lib.D_APPLY_PROPAGATE, res)
        glists = []
        for t, r in zip(trees, res):
            k = int(r.invalid_n)
            mine = torch.empty(max(k, 1), dtype=torch.int32, device=self.device)
            if k:
                check(_lib.lib().meerkat_memcpy(self.g._h, ctypes.c_void_p(mine.data_ptr()),
                                                ctypes.c_void_p(r.invalid), k * 4), "meerkat_memcpy")
            glists.append(torch.cat(self.tp.allgather_var(mine[:k])).contiguous())
        k = len(trees)
        if k <= 2:   # one stream of the slab array for both trees (meerkat_dtrees_scan)
            arr = (ctypes.c_void_p * k)(*[t._h.value for t in trees])
            lists = (ctypes.c_void_p * k)(*[gl.data_ptr() if gl.numel() else None for gl in glists])
            ns = (ctypes.c_uint64 * k)(*[gl.numel() for gl in glists])
            outs = (_lib.DResult * k)()
            check(_lib.lib().meerkat_dtrees_scan(self.g._h, arr, k, lists, ns, outs), "meerkat_dtrees_scan")
            res = [outs[i] for i in range(k)]
        else:
            res = [t._phase(_lib.D_DEC_SCAN, gl if gl.numel() else None, n=gl.numel()) for t, gl in zip(trees, glists)]
        self._fused_loop(trees, _lib.D_RELAX, _lib.D_APPLY_RELAX, res)
        for t, gl in zip(trees, glists):
            t._phase(_lib.D_FINISH, gl if gl.numel() else None, n=gl.numel())
            t.invalidated_total = gl.numel()

    def _fused_loop(self, trees, expand_ph, apply_ph, res):
        """Rounds of several trees until no rank has frontier or messages left for any of them."""
        res = list(res)
        active = [True] * len(trees)
        while True:
            act = self._exchange_apply(trees, res, apply_ph)
            if not any(act):
                return res
            for i, t in enumerate(trees):
                if act[i]:
                    t.rounds += 1
                else:
                    active[i] = False
            live = [i for i in range(len(trees)) if active[i]]
            if live:   # every still-active tree's expansion, one synchronisation (meerkat_dtrees_expand)
                arr = (ctypes.c_void_p * len(live))(*[trees[i]._h.value for i in live])
                outs = (_lib.DResult * len(live))()
                check(_lib.lib().meerkat_dtrees_expand(self.g._h, arr, len(live), expand_ph, outs),
                      "meerkat_dtrees_expand")
                for j, i in enumerate(live):
                    res[i] = outs[j]

    def _exchange_apply(self, trees, res, apply_ph):
        """One round's exchange for all trees: the library packs every tree's messages and a fixed-size
        <pairs, local frontier, pairs sent> row per (peer, tree) (meerkat_dtrees_pack); one all-to-all
        of the rows decides termination and the receive sizes; ONE all-to-all moves every tree's
        messages; the library unpacks them and runs each tree's apply phase (meerkat_dtrees_apply).
        Returns, per tree, whether any rank still has work for it."""
        ws, k, tp = self.ws, len(trees), self.tp
        L = _lib.lib()
        arr = (ctypes.c_void_p * k)(*[t._h.value for t in trees])
        cap = sum(int(r.msg_counts[p]) for r in res for p in range(ws))
        meta = torch.empty(ws * k * 3, dtype=torch.int64, device=self.device)
        send = torch.empty(max(cap, 1) * 2, dtype=torch.int64, device=self.device)
        sc = (ctypes.c_uint64 * ws)()
        check(L.meerkat_dtrees_pack(self.g._h, arr, k, ctypes.c_void_p(meta.data_ptr()),
                                    ctypes.c_void_p(send.data_ptr()), cap, sc), "meerkat_dtrees_pack")
        rmeta = tp.alltoallv_known(meta, [1] * ws, [1] * ws, elem=3 * k).view(ws, k, 3).cpu()
        act = [int(rmeta[:, i, 1].sum()) + int(rmeta[:, i, 2].sum()) > 0 for i in range(k)]
        if not any(act):
            return act
        scounts = [int(sc[p]) for p in range(ws)]
        rc = rmeta[:, :, 0].reshape(-1).tolist()          # [p * k + i]
        rcounts = [sum(rc[p * k:(p + 1) * k]) for p in range(ws)]
        recv = tp.alltoallv_known(send[: 2 * sum(scounts)], scounts, rcounts, elem=2)
        rca = (ctypes.c_uint64 * (ws * k))(*rc)
        check(L.meerkat_dtrees_apply(self.g._h, arr, k, apply_ph, ctypes.c_void_p(recv.data_ptr()), rca),
              "meerkat_dtrees_apply")
        return act

    def sssp(self, source: int) -> "DistTree":
        return DistTree(self, source, unit=False)

    def bfs(self, source: int) -> "DistTree":
        return DistTree(self, source, unit=True)


class DistTree:
    """This rank's part of a dependence tree T_G."""

    def __init__(self, dg: DistGraph, source: int, unit: bool):
        self.dg, self.unit, self.source = dg, unit, int(source)
        h = ctypes.c_void_p()
        check(_lib.lib().meerkat_dtree_create(dg.g._h, source, int(unit), ctypes.byref(h)), "meerkat_dtree_create")
        self._h = h
        self.rounds = 0
        # static: STATIC_INIT ran inside create; its frontier is {SRC} on the owner
        self.recompute()

    def recompute(self):
        """Static re-run on the current graph."""
        res = self._phase(_lib.D_STATIC_INIT)
        self._loop(_lib.D_RELAX, _lib.D_APPLY_RELAX, res)

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().meerkat_tree_destroy(self._h)
            self._h = None

    def _phase(self, ph, a=None, b=None, c=None, n=0, keep=None) -> _lib.DResult:
        res = _lib.DResult()
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        check(_lib.lib().meerkat_dtree_phase(self.dg.g._h, self._h, ph, p(a), p(b), p(c), n, ctypes.byref(res)),
              f"meerkat_dtree_phase({ph})")
        return res

    def _exchange(self, res):
        """One all-to-all of <count, local frontier, messages sent> triples (which also decides
        termination: nothing left anywhere) and, if any message moves, one of the messages."""
        ws = self.dg.ws
        tp = self.dg.tp
        counts = [int(res.msg_counts[r]) for r in range(ws)]
        sent = sum(counts)
        meta = torch.tensor([[counts[p], int(res.frontier), sent] for p in range(ws)], dtype=torch.int64,
                            device=tp._dev()).view(-1)
        rmeta = tp.alltoallv_known(meta, [1] * ws, [1] * ws, elem=3)   # fixed size: no count exchange
        rmeta = rmeta.view(ws, 3).cpu()
        if int(rmeta[:, 1].sum()) + int(rmeta[:, 2].sum()) == 0:
            return None, False
        rcounts = rmeta[:, 0].tolist()
        send = torch.empty(max(sent, 1) * 2, dtype=torch.int64, device=self.dg.device)
        if sent:   # stream-ordered device copy out of the library's message buffer
            check(_lib.lib().meerkat_memcpy(self.dg.g._h, ctypes.c_void_p(send.data_ptr()),
                                            ctypes.c_void_p(res.msgs), sent * 16), "meerkat_memcpy")
        recv = tp.alltoallv_known(send[: sent * 2], counts, rcounts, elem=2)
        return recv, True

    def _loop(self, expand_ph, apply_ph, res):
        """Rounds until no rank has frontier or messages left.  Per round:
        one count/termination all-to-all, one message all-to-all, a stream-ordered apply and one
        synchronising expansion."""
        while True:
            recv, active = self._exchange(res)
            if not active:
                return res
            n = recv.numel() // 2
            if n:
                self._phase(apply_ph, recv, n=n)
            self.rounds += 1
            res = self._phase(expand_ph)

    def incremental(self, src, dst, w=None):
        """Incremental prologue: the inserted batch (already applied) seeds the frontier."""
        cols, _, _ = self.dg.route(src, dst, None if self.unit else w)
        n = cols[0].numel()
        res = self._phase(_lib.D_INC_SEED, cols[0] if n else None, cols[1] if n else None,
                          (cols[2] if (n and not self.unit) else None), n)
        self._loop(_lib.D_RELAX, _lib.D_APPLY_RELAX, res)

    def decremental(self, src, dst):
        """Decremental prologue + common epilogue, across partitions."""
        cols, _, _ = self.dg.route(src, dst, key_is_b=True)        # parent test at owner(dst)
        n = cols[0].numel()
        res = self._phase(_lib.D_DEC_INVALIDATE, cols[0] if n else None, cols[1] if n else None, None, n)
        res = self._loop(_lib.D_PROPAGATE, _lib.D_APPLY_PROPAGATE, res)
        k = int(res.invalid_n)
        mine = torch.empty(max(k, 1), dtype=torch.int32, device=self.dg.device)
        if k:
            check(_lib.lib().meerkat_memcpy(self.dg.g._h, ctypes.c_void_p(mine.data_ptr()),
                                            ctypes.c_void_p(res.invalid), k * 4), "meerkat_memcpy")
        glist = torch.cat(self.dg.tp.allgather_var(mine[:k])).contiguous()
        m = glist.numel()
        res = self._phase(_lib.D_DEC_SCAN, glist if m else None, n=m)
        self._loop(_lib.D_RELAX, _lib.D_APPLY_RELAX, res)
        self._phase(_lib.D_FINISH, glist if m else None, n=m)
        self.invalidated_total = m

    def stats(self) -> dict:
        """This rank's counters of the last update (meerkat_tree_stats_get)."""
        st = _lib.TreeStats()
        check(_lib.lib().meerkat_tree_stats_get(self._h, ctypes.byref(st)), "meerkat_tree_stats_get")
        return st.as_dict()

    def local_nodes(self) -> np.ndarray:
        a = np.empty(self.dg.n_local, np.uint64)
        check(_lib.lib().meerkat_tree_nodes(self._h, ctypes.c_void_p(a.ctypes.data)), "meerkat_tree_nodes")
        return a

    def nodes(self) -> np.ndarray:
        """All vertices' packed nodes in global id order (collective)."""
        loc = torch.from_numpy(self.local_nodes().view(np.int64)).to(self.dg.device)
        parts = [p.cpu().numpy().view(np.uint64) for p in self.dg.tp.allgather_var(loc)]
        return interleave(parts, self.dg.ws, self.dg.vertex_n)
