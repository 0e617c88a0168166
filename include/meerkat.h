/*
 * meerkat.h — C ABI of the B200-native Meerkat hot path (arXiv 2305.17813).
 *
 * Plain C: opaque handles, fixed-width integers, plain pointers.  No C++ or
 * torch types cross this boundary.  One graph handle lives on one CUDA device
 * and orders all its work on one CUDA stream (cfg.stream, or the legacy
 * default stream when NULL).
 *
 * What the calls compute (citations: PAPER.md line numbers "P:n"):
 *   - the dynamic graph object G of the problem statement: a
 *     per-vertex SlabHash adjacency store with a single head-slab
 *     arena sized from degree hints, batched warp-
 *     cooperative InsertEdge / DeleteEdge / SearchEdge (WCWS
 *     P:552-593, host COO batches P:2126-2140);
 *   - a dependence tree T_G of packed <distance, parent> words, one 64-bit
 *     atomicMin per relaxation (footnote P:28-30), maintained by
 *     static, incremental and decremental (P:49-64,
 *     P:138-165) SSSP, and BFS.
 *
 * Pointer arguments.  Batch inputs (src, dst, w) may be HOST or DEVICE
 * pointers: the library inspects each pointer; host arrays are staged to the
 * device on the graph's stream inside the call (pinned host memory makes the
 * copy asynchronous).  Output arrays of query_batch / export_edges /
 * tree_nodes / tree_invalidated may likewise be host or device; host outputs
 * make the call synchronous.  The caller owns every batch and output buffer;
 * the library owns the slab store, trees and scratch (released by destroy).
 *
 * Synchronisation and errors.  Calls are stream-ordered and return after
 * enqueueing, unless they return a host count or write a host output, in
 * which case they synchronise the stream.  Invalid edges (an id >= vertex_n;
 * a weight of 0 or >= 2^31 on a weighted graph) are SKIPPED, never applied or
 * counted; the condition is recorded on the device and reported (with
 * VERTEX_RANGE taking precedence over WEIGHT) by the next synchronising call
 * on that graph, then cleared.  Any non-OK status leaves the graph valid.
 *
 * Ordering contract ("G undergoes modifications through the
 * application of an insertion/deletion edge batch; the incremental/decremental
 * SSSP algorithm re-computes"): mutate first, then call the matching tree
 * update with the SAME batch, for every tree of the graph, before the next
 * mutation.  Enforced three ways, each returning MEERKAT_E_STATE without touching
 * the tree: (1) on the host, the graph version (the tree must be exactly one
 * mutation behind), the mutation kind and the batch size n; (2) on the device,
 * for calls that read the batch (not seeded by meerkat_*_batch_trees): the
 * mutation kernel sums a 64-bit mix of every (src, dst) and (src, dst, w) of
 * its batch (an order-independent fingerprint) and the tree kernel sums the
 * same over the batch it was given before writing anything; on a mismatch the
 * tree kernel writes nothing, marks its trees STALE and records MEERKAT_E_STATE
 * (reported by the next synchronising call, e.g. meerkat_sync); (3) a stale
 * tree refuses every dynamic call the same way until meerkat_tree_recompute.
 * Seeded calls need no fingerprint: their batch prologue ran inside the
 * mutation kernel on the batch it applied, so only n is checked.
 *
 * Thread safety: a graph handle (and its trees) must not be used from two
 * host threads at once.
 */
#ifndef MEERKAT_H_
#define MEERKAT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct meerkat_graph meerkat_graph; /* opaque: slab store + metadata on one device */
typedef struct meerkat_tree meerkat_tree;   /* opaque: one SSSP or BFS tree for one source */
typedef struct meerkat_pagerank meerkat_pagerank; /* opaque: one PageRank vector of a graph */
typedef struct meerkat_wcc meerkat_wcc;           /* opaque: weakly connected component labels of a graph */

typedef enum {
  MEERKAT_OK = 0,
  MEERKAT_E_INVALID_ARG = 1,  /* null handle/pointer, vertex_n 0 or >= 2^32-4, lf not in (0,1], missing weights */
  MEERKAT_E_VERTEX_RANGE = 2, /* some id >= vertex_n (edge skipped) */
  MEERKAT_E_WEIGHT = 3,       /* some weight 0 or >= 2^31 (edge skipped) */
  MEERKAT_E_CAPACITY = 4,     /* slab pool or frontier exhausted; placed edges are kept and counted */
  MEERKAT_E_OVERFLOW = 5,     /* a distance would reach 2^32-1; that relaxation is not applied (C5) */
  MEERKAT_E_STATE = 6,        /* tree/graph version mismatch; SSSP on an unweighted graph */
  MEERKAT_E_CUDA = 7,         /* CUDA runtime error (out of memory, launch failure, no device) */
  MEERKAT_E_NCCL = 8,         /* NCCL error (init, or an asynchronous communicator error: the communicator
                                 is aborted) or a failed exchange callback; partitioned graphs only */
  MEERKAT_E_PARTITION = 9     /* an edge's source (or a message's target) is not held by this rank (skipped) */
} meerkat_status;

/* Host transport of a partitioned graph: an all-to-all-v over world_size ranks, called collectively
 * (every rank, same sequence).  `send` holds world_size consecutive segments, segment p (send_bytes[p]
 * bytes) for rank p; on return `recv` holds world_size consecutive segments, segment q (recv_bytes[q]
 * bytes, known to the caller) from rank q.  Both are host memory owned by the library.  Return 0 on
 * success; anything else makes the library call fail with MEERKAT_E_NCCL. */
typedef int (*meerkat_exchange_fn)(void* ctx, const void* send, const uint64_t* send_bytes, void* recv,
                                   const uint64_t* recv_bytes);

typedef struct {
  uint32_t vertex_n;            /* |V|, fixed for the graph's lifetime; ids are 0..vertex_n-1 */
  uint32_t weighted;            /* 1: ConcurrentMap slabs, 15 <dst,w> pairs; 0: ConcurrentSet, 31 keys */
  uint32_t hashing;             /* 0: one slab list per vertex ("hashing disabled") */
  float load_factor;            /* lf in (0,1]; bucket_count[v] = ceil(hint[v]/(lf*capacity)); 0 => 0.7 */
  const uint32_t* degree_hints; /* host or device [vertex_n], or NULL (every vertex one bucket) */
  uint64_t pool_slabs;          /* growth-pool capacity in 128-B slabs; 0 => automatic */
  uint64_t hash_seed;           /* bucket hash seed (storage only; results do not depend on it) */
  int device;                   /* CUDA device ordinal */
  void* stream;                 /* cudaStream_t for every call on this graph; NULL = default stream */
  uint32_t reverse;             /* 1: also keep an in-edge mirror store, so the decremental
                                   valid->invalid frontier reads only the in-edges of V_invalid
                                   instead of scanning every slab (same result) */
  const uint32_t* in_degree_hints; /* host or device [vertex_n] (in-degrees), or NULL; reverse only */
  uint32_t world_size;          /* vertex partition (multi-GPU), see "Partitioned graphs" below */
  uint32_t rank;
  uint32_t update_tracking;     /* 1: keep per-slab-list update tracking (is_updated / first updated slab
                                   and lane) for meerkat_wcc_incremental_tracked */
  /* Partitioned graphs: a graph is PARTITIONED when it is given a transport -- nccl_id or exchange --
   * (any world_size >= 1; without one, world_size must be 0 or 1 and the graph is the single-GPU one). */
  const void* nccl_id;          /* 128-B ncclUniqueId from meerkat_nccl_unique_id() on rank 0, broadcast by the
                                   caller: the library creates and owns an NCCL communicator over world_size
                                   ranks (collective call) and exchanges with grouped ncclSend/ncclRecv on
                                   the graph's stream (NVLink / NVSwitch) */
  meerkat_exchange_fn exchange; /* or a host all-to-all-v (CPU transports and tests; see below) */
  void* exchange_ctx;
  uint32_t exchange_pairs;      /* messages per peer per exchange of a dynamic tree call (0 = 16384; static
                                   recomputes use 16 x this); more are carried over to the next exchange */
  float in_load_factor;         /* lf of the in-edge mirror (reverse only), in (0,1]; 0 => load_factor.  The
                                   mirror is only walked (the decremental pull frontier, PageRank), so
                                   fuller slabs mean fewer work items there */
} meerkat_config;

typedef struct {
  uint64_t vertex_n;
  uint64_t edges;           /* live edges (inserted - deleted, as counted by the kernels) */
  uint64_t head_slabs;      /* slabs in the head arena, = sum over v with hint > 0 of bucket_count[v] */
  uint64_t buckets;         /* total slab lists (arena heads + one lazily allocated head per hint-0 vertex) */
  uint64_t pool_capacity;   /* growth-pool capacity (slabs) */
  uint64_t pool_used;       /* pool slabs handed out (chained slabs + lazily allocated heads) */
  uint64_t bytes_device;    /* device bytes owned by the graph (excluding trees) */
  uint64_t kernel_launches; /* kernels this graph and its trees have launched since creation */
  uint64_t version;         /* mutation counter */
  uint64_t in_edges;        /* reverse store: live in-edges (equals edges) */
  uint64_t in_head_slabs;   /* reverse store: head arena slabs */
  uint64_t in_pool_used;    /* reverse store: pool slabs handed out */
} meerkat_stats;

typedef struct {
  uint64_t rounds;           /* relax rounds of the last tree call (frontier iterations) */
  uint64_t propagate_rounds; /* invalidation-propagation rounds of the last decremental call */
  uint64_t direct_invalid;   /* vertices invalidated directly by deleted tree edges */
  uint64_t invalidated;      /* direct + propagated (|V_invalid|) */
  uint64_t frontier_edges;   /* valid->invalid edges found by the decremental scan */
  uint64_t items;            /* (vertex, bucket) work items expanded over all rounds */
  uint64_t slabs_read;       /* slabs read by the last call */
  uint64_t scan_slabs;       /* slabs streamed by the decremental scan */
  uint64_t improved;         /* successful atomicMin relaxations */
  uint64_t alg_bytes;        /* algorithmic bytes of the last call (DESIGN.md accounting) */
  uint64_t version;          /* graph version this tree reflects */
  uint32_t source;
  uint32_t unit_weights;     /* 1 for BFS trees */
  uint64_t exchanges;        /* partitioned trees: exchange units of the last call (0 when one rank chains
                                every phase in one launch) */
} meerkat_tree_stats;

const char* meerkat_status_string(meerkat_status s);

/* Store construction: bucket counts from the hints,
 * exclusive scan into one head arena, slab pool.  *out receives the handle. */
meerkat_status meerkat_create(const meerkat_config* cfg, meerkat_graph** out);
meerkat_status meerkat_destroy(meerkat_graph* g);
/* Rebind the graph (and its trees) to another stream. */
meerkat_status meerkat_set_stream(meerkat_graph* g, void* stream);
/* Wait for the graph's stream; returns (and clears) any recorded batch error. */
meerkat_status meerkat_sync(meerkat_graph* g);

/* InsertEdges (device InsertEdge P:634-641).  Inserting a present
 * edge keeps the smaller weight (C8).  w must be NULL iff the graph is
 * unweighted.  n_inserted (host, nullable) receives the number of edges that
 * were absent; passing it synchronises. */
meerkat_status meerkat_insert_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst,
                                    const uint32_t* w, uint64_t n, uint64_t* n_inserted);
/* DeleteEdges (DeleteEdge P:637, TOMBSTONE P:1506-1507).  Absent
 * edges are no-ops (C11).  n_deleted (host, nullable) receives the number removed. */
meerkat_status meerkat_delete_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                    uint64_t* n_deleted);
/* SearchEdge: found[i] = 1 iff (src[i], dst[i]) is present; w_out[i] =
 * its weight (0 when absent or unweighted).  w_out may be NULL. */
meerkat_status meerkat_query_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                   uint8_t* found, uint32_t* w_out);
/* Every live edge, in unspecified order (w = 0 when unweighted).  Writes at
 * most `capacity` edges, sets *n_out to the live count, synchronises;
 * MEERKAT_E_CAPACITY if capacity < live count. */
meerkat_status meerkat_export_edges(meerkat_graph* g, uint32_t* src, uint32_t* dst, uint32_t* w,
                                    uint64_t capacity, uint64_t* n_out);
meerkat_status meerkat_stats_get(meerkat_graph* g, meerkat_stats* out); /* synchronises */
/* Stream-ordered copy of the out-store's cumulative counters into out[3] (host pinned or device
 * memory): out[0] = edges inserted so far (counted as in insert_batch), out[1] = edges deleted so far,
 * out[2] = growth-pool slabs handed out.  Live edges = out[0] - out[1].  Does NOT synchronise: the
 * values are valid once the graph's stream has reached this point (e.g. after an event on it), which
 * lets a pipelined caller read each step's result without stalling the next step's copies. */
meerkat_status meerkat_counters_async(meerkat_graph* g, uint64_t* out);

/* Latency probes for the latency floor of the tree calls (SURVEY §8(d) "latency term"; a frontier
 * round is a chain of dependent memory operations closed by a grid barrier, P:108-112 / P:2189-2207):
 * measured on g's device and stream with a 2-GiB pointer chase (DRAM), a 4-MiB chase (L2), a chase of
 * dependent 64-bit atomicMin round trips (DRAM lines), and back-to-back grid.sync() on the tree
 * kernels' cooperative grid.  Allocates 2 GiB temporarily; synchronises. */
typedef struct {
  double dram_load_ns;    /* dependent load, random line, buffer >> L2 */
  double l2_load_ns;      /* dependent load, random line, buffer << L2 */
  double dram_atomic_ns;  /* dependent 64-bit atomicMin round trip, random line, buffer >> L2 */
  double grid_sync_us;    /* one grid-wide barrier of the tree kernels' grid */
  uint32_t grid_blocks;   /* that grid: blocks of 512 threads */
} meerkat_latency;
meerkat_status meerkat_probe_latency(meerkat_graph* g, meerkat_latency* out);
/* Structural check of the slab store(s) (owner of every slab, next pointers, no leftover link
 * lock, finite chains, EMPTY-suffix invariant).  info[5] (host): violations, then the first one's
 * vertex, slab, next, kind.  MEERKAT_E_STATE if any; synchronises. */
meerkat_status meerkat_check(meerkat_graph* g, uint64_t* info);

/* Static SSSP (weighted graphs only) / level-based static BFS
 * (hop counts, weights ignored).  The new tree reflects the current
 * graph version. */
meerkat_status meerkat_sssp_create(meerkat_graph* g, uint32_t source, meerkat_tree** out);
meerkat_status meerkat_bfs_create(meerkat_graph* g, uint32_t source, meerkat_tree** out);
/* The VANILLA variant: static SSSP / BFS computing only the shortest distances,
 * 32-bit distance words relaxed by 32-bit atomicMin (no parent, so no dependence tree: incremental
 * / decremental calls and meerkat_tree_nodes return MEERKAT_E_STATE; recompute and distances work).
 * The paper measures the tree-based variant's overhead against it (17.2% BFS, ~14% SSSP). */
meerkat_status meerkat_sssp_vanilla_create(meerkat_graph* g, uint32_t source, meerkat_tree** out);
meerkat_status meerkat_bfs_vanilla_create(meerkat_graph* g, uint32_t source, meerkat_tree** out);
/* dist[v] for every v (UINT32_MAX when unreached), for tree-based and vanilla trees; host or device. */
meerkat_status meerkat_tree_distances(meerkat_tree* t, uint32_t* out);
/* Incremental update: the batch just applied by insert_batch is the
 * initial frontier.  w: the batch's weights (NULL for BFS trees). */
meerkat_status meerkat_sssp_incremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src,
                                        const uint32_t* dst, const uint32_t* w, uint64_t n);
meerkat_status meerkat_bfs_incremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src,
                                       const uint32_t* dst, uint64_t n);
/* Decremental update: invalidate deleted tree edges,
 * propagate down T_v, re-seed from valid->invalid edges, relax to fixpoint. */
meerkat_status meerkat_sssp_decremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src,
                                        const uint32_t* dst, uint64_t n);
meerkat_status meerkat_bfs_decremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src,
                                       const uint32_t* dst, uint64_t n);
/* Fused update of up to 2 trees of g (e.g. an SSSP and a BFS tree) with the batch just applied:
 * one launch; the trees share every frontier round's grid barrier and, for a decremental batch
 * without an in-edge mirror, ONE stream over the slab array serves all of them.  Same results as
 * the per-tree calls.  w: the batch's weights (needed iff some tree is an SSSP tree). */
meerkat_status meerkat_trees_incremental(meerkat_graph* g, meerkat_tree* const* trees, uint32_t n_trees,
                                         const uint32_t* src, const uint32_t* dst, const uint32_t* w, uint64_t n);
meerkat_status meerkat_trees_decremental(meerkat_graph* g, meerkat_tree* const* trees, uint32_t n_trees,
                                         const uint32_t* src, const uint32_t* dst, uint64_t n);
/* insert_batch that also SEEDS the trees' next incremental call: the trees' batch prologue
 * (relax node[v] from node[u] + w for each inserted (u, v), enqueue the improved v; it
 * reads no slab) runs inside the insert kernel, so the meerkat_trees_incremental (or per-tree
 * incremental) call that must follow with the same batch and the same trees starts at its first
 * frontier round: one grid-wide phase and barrier fewer.  The trees (up to 2, of g, not vanilla)
 * must reflect g's current version and not be seeded already (else MEERKAT_E_STATE); a fused call
 * must name all seeded trees or none.  Results are those of insert_batch + trees_incremental.
 * Between the two calls node[] is partial; a static recompute drops an unused seed.  w: NULL iff
 * the graph is unweighted.  n_inserted as insert_batch. */
meerkat_status meerkat_insert_batch_trees(meerkat_graph* g, const uint32_t* src, const uint32_t* dst,
                                          const uint32_t* w, uint64_t n, meerkat_tree* const* trees,
                                          uint32_t n_trees, uint64_t* n_inserted);
/* delete_batch that seeds the trees' next decremental call the same way: the invalidation of the
 * deleted tree edges (C4) runs inside the delete kernel.  n_deleted as delete_batch. */
meerkat_status meerkat_delete_batch_trees(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                          meerkat_tree* const* trees, uint32_t n_trees, uint64_t* n_deleted);
/* Static re-run on the current graph (the s_b^n baseline). */
meerkat_status meerkat_tree_recompute(meerkat_graph* g, meerkat_tree* t);
/* The same with the paper's iteration scheme chosen: 2 = <vertex, bucket> work items
 * (IterationScheme2, what every call here uses), 1 = one work item per vertex whose buckets one
 * group walks in turn (IterationScheme1, SlabIterator).  Same result; for the comparison. */
meerkat_status meerkat_tree_recompute_scheme(meerkat_graph* g, meerkat_tree* t, uint32_t iteration_scheme);
/* node[v] = dist << 32 | parent for every v, UINT64_MAX when unreached (C3). */
meerkat_status meerkat_tree_nodes(meerkat_tree* t, uint64_t* out);
/* The vertices invalidated by the last decremental call (unordered). */
meerkat_status meerkat_tree_invalidated(meerkat_tree* t, uint32_t* out, uint64_t capacity, uint64_t* n_out);
meerkat_status meerkat_tree_stats_get(meerkat_tree* t, meerkat_tree_stats* out); /* synchronises */
/* Device timeline of the last single-GPU tree call: %globaltimer (ns) at kernel start and after
 * every grid-wide barrier (phase / round boundaries), up to 48 entries; *n_out = entries recorded.
 * items (nullable, host [capacity]): items[i] = frontier items of the round that starts at entry i
 * (summed over the call's trees; 0 for an entry that starts a non-round phase). */
meerkat_status meerkat_tree_timeline(meerkat_tree* t, uint64_t* out, uint64_t* items, uint64_t capacity,
                                     uint64_t* n_out);
meerkat_status meerkat_tree_destroy(meerkat_tree* t);

/* ---------------------------------------------------------------------------------------------
 * Partitioned graphs (multi-GPU).  One process per GPU; rank r of world_size holds
 * the out-edges (and, with `reverse`, the in-edges), the tree nodes and the degree-hint row of every
 * vertex v with owner(v) == r, where owner(v) = m mod world_size, row(v) = m div world_size and
 * m = a fixed bijective mix of v on [0, vertex_n) (so unscrambled R-MAT ids are balanced; results do
 * not depend on it).  degree_hints / in_degree_hints are GLOBAL [vertex_n] arrays on every rank.
 * Every call on a partitioned graph or its trees is COLLECTIVE: all ranks make the same sequence of
 * calls, each with its own (possibly empty) batch:
 *   - insert / delete / query: any rank may pass any edges; the library routes each edge to
 *     owner(src) (and, for the mirror and for the decremental parent test, to owner(dst)) with one
 *     all-to-all-v.  n_inserted / n_deleted are GLOBAL counts; query
 *     answers return to the asking rank in its input order; errors are those of this rank's edges;
 *   - meerkat_sssp_create / meerkat_bfs_create / meerkat_tree_recompute: collective static trees;
 *   - the incremental / decremental calls (per tree or fused trees_*) must pass, on every rank, the
 *     batch that rank passed to the last mutation (ordering contract, checked by fingerprint); the
 *     library uses the rows it routed then.  The update runs as device-driven exchange units (a
 *     cooperative kernel -- apply the messages received, local frontier rounds to a fixpoint,
 *     pack up to exchange_pairs messages per peer -- then one all-to-all of fixed-size blocks);
 *     phase changes (propagation -> valid->invalid frontier -> relaxation -> done) are decided on
 *     the device from the exchanged headers, identically on every rank; the host never waits for a
 *     round.  The valid->invalid frontier walks the in-edge mirror (pull requests to owner(u)) when
 *     `reverse`, else every rank streams its own slabs against the exchanged invalid sets;
 *   - meerkat_tree_nodes: all vertex_n nodes in global id order on every rank (an all-gather);
 *   - meerkat_export_edges / meerkat_stats_get / meerkat_tree_stats_get: this rank's part (local).
 * PageRank, WCC, triangle counting, vanilla trees, seeded calls and distances are single-GPU only
 * (MEERKAT_E_STATE / MEERKAT_E_INVALID_ARG).  Results are bit-identical to world_size 1.
 * Errors: argument / ordering-contract errors are detected identically on every rank (MEERKAT_E_STATE
 * everywhere when any rank passed another batch; no tree is touched); data errors of a tree call
 * (capacity, overflow) are OR-ed over ranks.  A MEERKAT_E_NCCL or MEERKAT_E_CUDA from a collective
 * call can leave the ranks out of step: destroy the graph on every rank.
 * ------------------------------------------------------------------------------------------- */
#define MEERKAT_MAX_RANKS 64

/* Writes a fresh ncclUniqueId (128 bytes) to out; MEERKAT_E_NCCL if NCCL cannot be loaded. */
meerkat_status meerkat_nccl_unique_id(void* out, uint64_t bytes);
/* Host-only: owner rank and row of n global ids on a partitioned graph of vertex_n vertices over
 * world_size ranks (the library's placement); either output may be NULL. */
meerkat_status meerkat_owner_map(uint32_t vertex_n, uint32_t world_size, const uint32_t* ids, uint64_t n,
                                 uint32_t* owner, uint32_t* row);

/* ---------------------------------------------------------------------------------------------
 * PageRank.  Eq. (1):
 *   PR_i[v] = (1-d)/N + d * sum over in-edges u->v of PR_{i-1}[u] / out[u],
 * plus d * (sum of PR_{i-1} over zero-out-degree vertices) / N added to every vertex when such a
 * vertex exists (FindTeleportProb, reading C27), repeated until the L1 norm
 * sum_v |PR_i[v] - PR_{i-1}[v]| <= error_margin or max_iter super-steps ran (at least
 * one).  Double precision.  Out-degrees count stored edges (self-loops included); they are
 * counted by one stream over the out-store's slabs when the graph changed since the last run (the
 * update kernels keep no degree table).  The graph
 * must keep the in-edge mirror (cfg.reverse = 1; the Compute kernel walks in-edges)
 * and be unpartitioned (world_size 1), else MEERKAT_E_STATE.  MEERKAT_E_INVALID_ARG for a
 * damping outside (0,1), error_margin <= 0 or max_iter 0 (SPEC BadDamping / BadEpsilon).
 * Every call runs to convergence in one launch and synchronises the graph's stream.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  uint64_t iterations; /* super-steps of the last run */
  double delta;        /* its last L1 norm */
  uint64_t slabs;      /* in-edge slabs streamed per super-step */
  uint64_t in_edges;   /* live in-edges gathered per super-step */
  uint64_t atomics;    /* per-vertex accumulator atomics per super-step */
  uint64_t alg_bytes;  /* algorithmic bytes of the last run (DESIGN.md accounting) */
  uint64_t version;    /* graph version the values reflect */
  uint32_t warm;       /* 1 if the last run was warm-started (dynamic) */
  uint32_t pad;
} meerkat_pagerank_stats;

/* Static PageRank (PR_0 = 1/N) of the current graph; *out receives the handle. */
meerkat_status meerkat_pagerank_create(meerkat_graph* g, double damping, double error_margin, uint32_t max_iter,
                                       meerkat_pagerank** out);
/* Dynamic PageRank after insert/delete batches: the same algorithm on the whole
 * graph, warm-started from the current values. */
meerkat_status meerkat_pagerank_update(meerkat_graph* g, meerkat_pagerank* p);
/* Static re-run from 1/N on the current graph (the s_b^n baseline). */
meerkat_status meerkat_pagerank_recompute(meerkat_graph* g, meerkat_pagerank* p);
/* PR[v] for every v (double, host or device [vertex_n]). */
meerkat_status meerkat_pagerank_values(meerkat_pagerank* p, double* out);
meerkat_status meerkat_pagerank_stats_get(meerkat_pagerank* p, meerkat_pagerank_stats* out);
meerkat_status meerkat_pagerank_destroy(meerkat_pagerank* p);

/* ---------------------------------------------------------------------------------------------
 * Dynamic triangle counting (Algorithm tc-count).  Graphs are
 * undirected: both orientations of every edge are stored (unweighted or weighted; weights are
 * ignored).  Count(G1, G2, edges) = sum over (u, v) in edges of |adjacency_G1(u) ∩ adjacency_G2(v)|
 * (P:2064-2066); g1 and g2 live on the same device with the same vertex_n and are unpartitioned
 * (else MEERKAT_E_STATE).  Edges are host or device arrays.  All calls synchronise.
 * ------------------------------------------------------------------------------------------- */
meerkat_status meerkat_tc_count(meerkat_graph* g1, meerkat_graph* g2, const uint32_t* src, const uint32_t* dst,
                                uint64_t n, uint64_t* count);
/* Triangles of g: Count(G, G, every stored edge) / 6; MEERKAT_E_STATE if the count
 * is not divisible by 6 (g is not symmetric). */
meerkat_status meerkat_tc_static(meerkat_graph* g, uint64_t* triangles);
/* Triangles added by an inserted batch (already applied to g_after; g_update holds exactly the batch;
 * src/dst list the batch in BOTH orientations): S1 = Count(after, after), S2 = Count(after, update),
 * S3 = Count(update, update), added = S1/2 - S2/2 + S3/6.  s (host [3], nullable)
 * receives S1..S3.  MEERKAT_E_STATE if the identity is not an integer (broken precondition). */
meerkat_status meerkat_tc_incremental(meerkat_graph* g_after, meerkat_graph* g_update, const uint32_t* src,
                                      const uint32_t* dst, uint64_t n, uint64_t* added, uint64_t* s);
/* Triangles removed by a deleted batch (already deleted from g_after): S1/2 + S2/2 + S3/6. */
meerkat_status meerkat_tc_decremental(meerkat_graph* g_after, meerkat_graph* g_update, const uint32_t* src,
                                      const uint32_t* dst, uint64_t n, uint64_t* removed, uint64_t* s);

/* ---------------------------------------------------------------------------------------------
 * Weakly connected components (static SamplingWCC P:381-395,
 * incremental BatchInsert P:486-493; incremental only, as in the paper).  A root-based
 * union-find over parents[]: label[v] after full path compression.  The larger root always hooks
 * under the smaller, so label[v] = the smallest vertex id of v's component (edge directions are
 * ignored).  Unpartitioned graphs only (else MEERKAT_E_STATE).
 * ------------------------------------------------------------------------------------------- */
/* Static WCC of the current graph: MinHooking sampling, compression, union of the remaining edges,
 * compression.  Synchronises. */
meerkat_status meerkat_wcc_create(meerkat_graph* g, meerkat_wcc** out);
meerkat_status meerkat_wcc_recompute(meerkat_graph* g, meerkat_wcc* c);
/* After insert_batch: union(src[i], dst[i]) for the batch, then full compression.
 * The labels must be current up to that batch (the previous mutation) and n must be its size, else
 * MEERKAT_E_STATE (there is no decremental WCC: recompute after a delete batch).  Stream-ordered. */
meerkat_status meerkat_wcc_incremental(meerkat_graph* g, meerkat_wcc* c, const uint32_t* src, const uint32_t* dst,
                                       uint64_t n);
/* The paper's UpdateIterator path: union the edges of every slab list written since the
 * last call, from its first updated cell on (the update tracking of cfg.update_tracking), then full
 * compression, then reset the tracking (Graph.UpdateSlabPointers).  Same labels as
 * meerkat_wcc_incremental with the inserted batches; MEERKAT_E_STATE without update tracking or when a
 * delete batch was applied since the labels were computed. */
meerkat_status meerkat_wcc_incremental_tracked(meerkat_graph* g, meerkat_wcc* c);
/* label[v] (host or device [vertex_n]). */
meerkat_status meerkat_wcc_labels(meerkat_wcc* c, uint32_t* out);
meerkat_status meerkat_wcc_components(meerkat_wcc* c, uint64_t* n_components);
meerkat_status meerkat_wcc_destroy(meerkat_wcc* c);

#ifdef __cplusplus
}
#endif

#endif /* MEERKAT_H_ */
