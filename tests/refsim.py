"""Independent pure-Python checkers used to PIN the oracle (tests only).

None of this shares code with oracle/meerkat_oracle.c.  Each function is a
different route to the same mathematical object:

* brute_force_tree: enumerates every simple path from SRC (n <= 8) and keeps
  the lexicographically smallest (length, last hop) per vertex — the
  definition of P:27-39 with the packed-min tie-break (C1, C2) evaluated by
  exhaustion, with no shortest-path algorithm involved;
* simulate_method: the paper's own batch-dynamic procedure (P:41-64,
  P:88-170) — frontier relaxation with a packed 64-bit min, incremental
  prologue from the batch, decremental invalidate / bottom-up propagate /
  valid->invalid frontier — run sequentially in a RANDOM order, so that
  agreement with the oracle's from-scratch Dijkstra shows the method
  reaches the definition (SURVEY §8(c) "Claim");
* dict_store: a Python dict replay of insert / delete / query semantics.
"""
from __future__ import annotations

import random

UNREACHED = (1 << 64) - 1
INF = 0xFFFFFFFF


def pack(d, p):
    return (d << 32) | p


def brute_force_tree(n, src, edges, unit=False):
    adj = {}
    for (u, v, w) in edges:
        adj.setdefault(u, []).append((v, 1 if unit else w))
    best = [UNREACHED] * n
    best[src] = pack(0, src)

    def dfs(u, length, onpath):
        for (v, w) in adj.get(u, []):
            if v in onpath:
                continue
            cand = pack(length + w, u)
            if v != src and cand < best[v]:
                best[v] = cand
            onpath.add(v)
            dfs(v, length + w, onpath)
            onpath.discard(v)

    dfs(src, 0, {src})
    return best


class dict_store:
    """Set/map semantics of P:634-641 with min-weight upsert (C8) and no-op deletes (C11)."""

    def __init__(self):
        self.e = {}

    def insert(self, batch):
        new = 0
        for (u, v, w) in batch:
            if (u, v) in self.e:
                self.e[(u, v)] = min(self.e[(u, v)], w)
            else:
                self.e[(u, v)] = w
                new += 1
        return new

    def delete(self, batch):
        gone = 0
        for (u, v) in batch:
            if (u, v) in self.e:
                del self.e[(u, v)]
                gone += 1
        return gone


def _out(edges_dict):
    out = {}
    for (u, v), w in edges_dict.items():
        out.setdefault(u, []).append((v, w))
    return out


def _relax_loop(node, frontier, out, unit, rng):
    """Common epilogue: edge frontier, packed atomicMin, enqueue on success."""
    while frontier:
        rng.shuffle(frontier)
        nxt = []
        for (u, v, w) in frontier:
            if node[u] == UNREACHED:
                continue
            d = (node[u] >> 32) + (1 if unit else w)
            cand = pack(d, u)
            if cand < node[v]:
                node[v] = cand
                for (x, wx) in out.get(v, []):
                    nxt.append((v, x, wx))
        frontier = nxt
    return node


def simulate_static(n, src, edges_dict, unit, rng):
    node = [UNREACHED] * n
    node[src] = pack(0, src)
    out = _out(edges_dict)
    frontier = [(src, x, w) for (x, w) in out.get(src, [])]
    return _relax_loop(node, frontier, out, unit, rng)


def simulate_incremental(node, src, edges_dict, batch, unit, rng):
    # the inserted batch is the initial frontier; weights as stored (min-upsert)
    out = _out(edges_dict)
    frontier = [(u, v, edges_dict[(u, v)]) for (u, v, _w) in batch]
    return _relax_loop(list(node), frontier, out, unit, rng)


def simulate_decremental(node, src, edges_dict, batch, unit, rng):
    n = len(node)
    node = list(node)
    inval = [False] * n
    for (u, v) in batch:                                       # P:144-147 Invalidate
        if v != src and node[v] != UNREACHED and (node[v] & 0xFFFFFFFF) == u:
            inval[v] = True
    parent = [node[v] & 0xFFFFFFFF if node[v] != UNREACHED else None for v in range(n)]
    for v in range(n):                                         # P:149-154 bottom-up walk to SRC
        if node[v] == UNREACHED or inval[v]:
            continue
        x, hops = v, 0
        while x != src:
            x = parent[x]
            hops += 1
            if inval[x]:
                inval[v] = True
                break
            assert hops <= n, "cycle in tree"
    for v in range(n):
        if inval[v]:
            node[v] = UNREACHED
    out = _out(edges_dict)
    frontier = [(u, x, w) for (u, x), w in edges_dict.items()
                if node[u] != UNREACHED and not inval[u] and inval[x]]
    return _relax_loop(node, frontier, out, unit, rng), inval


def random_graph(rng: random.Random, n, m, wmax=64):
    edges = {}
    while len(edges) < m:
        u, v = rng.randrange(n), rng.randrange(n)
        if u != v:
            edges.setdefault((u, v), rng.randint(1, wmax))
    return edges
