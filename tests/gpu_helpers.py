"""Shared helpers for the GPU parity tests (tests only)."""
import numpy as np

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


def cuda(a):
    """numpy uint32 -> int32 CUDA tensor with the same bits."""
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.uint32)).view(np.int32)).to("cuda:0")


def assert_same_edges(g, o):
    gs, gd, gw = g.export_edges()
    es, ed, ew = o.edges()
    assert len(gs) == len(es), (len(gs), len(es))
    assert np.array_equal(gs, es) and np.array_equal(gd, ed)
    if o.weighted:
        assert np.array_equal(gw, ew)


def first_mismatch(a, b):
    bad = np.nonzero(np.asarray(a) != np.asarray(b))[0]
    if len(bad) == 0:
        return None
    v = int(bad[0])
    return v, hex(int(a[v])), hex(int(b[v])), len(bad)


def assert_nodes(gpu_nodes, ref_nodes, what=""):
    mm = first_mismatch(gpu_nodes, ref_nodes)
    assert mm is None, f"{what}: first mismatch (v, gpu, oracle, count) = {mm}"
