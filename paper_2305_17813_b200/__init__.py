"""B200-native Meerkat hot path (arXiv 2305.17813): SlabHash graph store +
batch-dynamic SSSP/BFS, as hand-written sm_100a CUDA behind a C ABI
(include/meerkat.h).  This package is the thin Python binding; see DESIGN.md."""
from ._lib import MeerkatError, SO_PATH  # noqa: F401
from .graph import WCC, Graph, PageRank, Tree  # noqa: F401

__all__ = ["Graph", "Tree", "PageRank", "WCC", "MeerkatError", "SO_PATH"]
