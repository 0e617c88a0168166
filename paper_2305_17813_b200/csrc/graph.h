// graph.h — host-side handle layouts and the launchers each .cu file exports.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/meerkat.h"
#include "internal.cuh"

namespace mk {

constexpr int MAX_TREES = 2;   // trees updated together by one fused call (e.g. SSSP + BFS)
constexpr int STAT_BLOCKS = 2048;   // per-block counter slots of a tree (>= any cooperative grid)

struct TreeCtrl {
  unsigned long long size[3];       // rotating frontier sizes (see tree.cu, "round protocol")
  unsigned long long inval_n;       // |V_invalid| of this call
  unsigned long long direct_n;      // directly invalidated vertices
  unsigned long long rounds;        // relax rounds
  unsigned long long prop_rounds;   // propagation rounds
  unsigned long long items;         // (vertex, bucket) items expanded
  unsigned long long slabs_read;    // slabs walked by expansion
  unsigned long long scan_slabs;    // slabs streamed by the decremental scan
  unsigned long long scan_hits;     // valid->invalid edges found by the scan
  unsigned long long improved;      // successful atomicMin
  unsigned long long visited;       // live edges visited by expansion (one node[x] probe each)
  unsigned long long batch_edges;   // batch edges examined by the prologue
  unsigned long long pull_n;        // (invalid vertex, in-bucket) items of the reverse-store frontier
  unsigned long long tail_r;        // round counter after block 0's tail rounds (tree.cu run_rounds)
  unsigned long long fp[2];         // fingerprint of the batch this call was given (ordering contract)
  unsigned long long nts;           // device timeline: %globaltimer at kernel start and after every grid barrier
  unsigned long long tstamp[48];
  unsigned long long titems[48];    // frontier items of the round starting at timeline entry i (0: other phase)
};

// PageRank control block (pagerank.cu).  delta / dangling rotate over three slots per super-step.
struct PRCtrl {
  double delta[3];             // L1 norm of super-step i in slot i % 3
  double dangling[3];          // sum of PR over zero-out-degree vertices, read by super-step i from slot i % 3
  unsigned long long iters;    // super-steps run by the last call
  double last_delta;
  unsigned long long slabs;    // in-edge slabs streamed per super-step
  unsigned long long keys;     // live in-edges gathered per super-step
  unsigned long long atomics;  // acc[] atomics per super-step
};

struct TreeDev {
  uint64_t* node;        // packed <dist, parent> per vertex
  uint32_t* stamp;       // last epoch a vertex was enqueued (frontier de-duplication)
  uint32_t* inval_bits;  // V-bit set of invalidated vertices (decremental only)
  uint32_t* inval_list;  // invalidated vertex ids
  uint64_t* fr[2];       // frontier item buffers: (bucket << 32) | vertex
  TreeCtrl* ctrl;
  uint32_t* epoch_ptr;   // device: [0] stamp epoch base, advanced by each call; [1] stale flag (a
                         // dynamic call was refused on the device: only a static recompute clears it)
  uint64_t fr_cap;       // items per frontier buffer (= number of slab lists)
  uint32_t source;
  uint32_t unit;         // 1: BFS (every w = 1)
  unsigned long long* bstat;   // per-block counter slots [STAT_BLOCKS][8] written by the tree kernels' finish
  uint32_t scheme1;      // 1: IterationScheme1 items (one per vertex, its buckets walked in turn;
                         //    static recompute only); 0: <vertex, bucket> items
};

}  // namespace mk

namespace mk {
struct PartState;
// One slab store (out-edges, or the optional in-edge mirror) on the device.
struct Store {
  GraphDev dev{};
  uint64_t H = 0, P = 0, buckets = 0;   // arena slabs, pool capacity, slab lists
  size_t bytes = 0;
  GraphCtrl* hctrl = nullptr;           // pinned mirror of dev.ctrl
  uint64_t deg_version = ~0ull;         // graph version dev.deg was counted at (launch_degrees)
};
}  // namespace mk

struct meerkat_graph {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t V = 0;                   // global vertex count
  uint32_t Vl = 0;                  // vertices held by this partition
  uint32_t ws = 1, rank = 0;        // vertex partition (owner(v) = pm_mix(v) % ws, internal.cuh)
  bool weighted = false, hashing = true, reverse = false;
  float lf = 0.7f;
  float lf_in = 0.7f;               // load factor of the in-edge mirror
  mk::Store out;                    // out-edge store (the paper's SlabGraph)
  mk::Store in;                     // in-edge mirror (reverse store), only when reverse
  uint64_t version = 0;
  int last_kind = 0;                // 0 none, 1 insert, 2 delete
  uint64_t last_n = 0;              // batch size of the last mutation (ordering contract)
  uint64_t last_delete_version = 0; // version created by the last delete batch (incremental WCC)
  uint64_t n_trees = 0;             // live dynamic (tree-based) trees of this graph
  uint64_t launches = 0;
  int sm_count = 0;
  void* stage[4] = {nullptr, nullptr, nullptr, nullptr};   // staging for host inputs / outputs
  size_t stage_bytes[4] = {0, 0, 0, 0};
  // a mutation's staged host batch, reusable by the tree call that must follow with the same batch
  const void* staged_host[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t staged_len[4] = {0, 0, 0, 0};
  uint64_t staged_version[4] = {0, 0, 0, 0};
  int tree_blocks_per_sm[4] = {0, 0, 0, 0};   // cooperative occupancy: static, incremental, decremental, vanilla
  int latency_bps = 0;                      // blocks/SM for latency-bound tree calls (0 = occupancy)
  mk::PartState* part = nullptr;            // vertex-partitioned graph (part.cu): transport, rings, routed rows
};

struct meerkat_tree {
  meerkat_graph* g = nullptr;
  mk::TreeDev dev{};
  mk::TreeCtrl* hctrl = nullptr;
  bool unit = false;     // BFS
  bool vanilla = false;  // distance-only static variant: node[] holds u32 distances
  uint64_t version = 0;
  mk::TreeCtrl* ctrl_base = nullptr;   // two control blocks: a call uses one and zeroes the other
  int parity = 0;
  int seeded = 0;   // 1 / 2: insert_batch_trees / delete_batch_trees ran this call's batch prologue
  bool counted = false;   // counted in g->n_trees
  uint32_t stat_blocks = 0;   // grid of the last single-GPU tree call (its bstat slots)
  // vertex-partitioned trees (part.cu)
  bool part = false;
  uint64_t* pull_items = nullptr;           // (invalid vertex, in-bucket) items of the mirror frontier
  uint64_t last_units = 0;                  // exchange units of the last call
  size_t bytes = 0;
};

struct meerkat_pagerank {
  meerkat_graph* g = nullptr;
  double d = 0.85, eps = 1e-5;
  uint32_t max_iter = 0;
  double* pr = nullptr;        // PR values [V]
  double* contrib = nullptr;   // Contribution[u] = PR[u] / out[u]
  double* acc = nullptr;       // per-vertex sum of in-edge contributions
  mk::PRCtrl* ctrl = nullptr;
  mk::PRCtrl* hctrl = nullptr;
  int blocks_per_sm = 0;
  uint64_t version = 0;        // graph version the values reflect
  bool warm_last = false;
};

struct meerkat_wcc {
  meerkat_graph* g = nullptr;
  uint32_t* parent = nullptr;              // union-find parents; labels after compression
  unsigned long long* scratch = nullptr;   // device counters: [0] union attempts, [1] roots
  unsigned long long* hscratch = nullptr;  // pinned mirror
  uint64_t version = 0;
};

namespace mk {
// wcc.cu
cudaError_t launch_wcc_static(meerkat_graph* g, uint32_t* parent, unsigned long long* scratch);
cudaError_t launch_wcc_batch(meerkat_graph* g, uint32_t* parent, const uint32_t* s, const uint32_t* d, uint64_t n);
cudaError_t launch_wcc_roots(meerkat_graph* g, const uint32_t* parent, unsigned long long* out_dev);
cudaError_t launch_wcc_tracked(meerkat_graph* g, uint32_t* parent);
// tc.cu
cudaError_t launch_tc_count(meerkat_graph* g1, meerkat_graph* g2, const uint32_t* src, const uint32_t* dst,
                            uint64_t n, unsigned long long* out_dev);
// pagerank.cu
cudaError_t pagerank_occupancy(bool weighted, int* blocks_per_sm);
cudaError_t launch_pagerank(meerkat_graph* g, meerkat_pagerank* p, bool warm);
size_t pagerank_contrib_bytes();   // bytes per cached Contribution[u] (4: fp32 cache, 8: fp64)
// store.cu
cudaError_t launch_build(meerkat_graph* g, Store& st, const uint32_t* d_hints, uint64_t pool_request);
void free_store(Store& st);
// st1 (nullable): the in-edge mirror, updated with (dst, src) in the same launch
// Tree prologue fused into a mutation kernel (meerkat_insert_batch_trees / meerkat_delete_batch_trees):
// the trees' device views with the control blocks of the tree call that follows.
struct TreePro {
  TreeDev T[MAX_TREES];
  uint32_t ntrees;
};
void tree_pro_fill(meerkat_tree* const* trees, uint32_t ntrees, TreePro& p);
cudaError_t launch_insert(meerkat_graph* g, Store* st0, Store* st1, const uint32_t* s, const uint32_t* d,
                          const uint32_t* w, uint64_t n, const TreePro* pro = nullptr);
cudaError_t launch_delete(meerkat_graph* g, Store* st0, Store* st1, const uint32_t* s, const uint32_t* d, uint64_t n,
                          const TreePro* pro = nullptr);
cudaError_t launch_query(meerkat_graph* g, Store& st, const uint32_t* s, const uint32_t* d, uint64_t n,
                         uint8_t* found, uint32_t* w_out);
cudaError_t launch_export(meerkat_graph* g, Store& st, uint32_t* s, uint32_t* d, uint32_t* w, uint64_t cap);
cudaError_t launch_fsck(meerkat_graph* g, Store& st, unsigned long long* info_dev);
cudaError_t launch_degrees(meerkat_graph* g, Store& st);   // dev.deg = live keys per row, if stale
// tree.cu
cudaError_t tree_occupancy(meerkat_graph* g);
enum TreeMode { MODE_STATIC = 0, MODE_INCREMENTAL = 1, MODE_DECREMENTAL = 2 };
// fp_mode: -1 no fingerprint check, 0 check over (src, dst), 1 over (src, dst, w)
cudaError_t launch_tree(meerkat_graph* g, meerkat_tree* const* trees, uint32_t ntrees, int mode, const uint32_t* s,
                        const uint32_t* d, const uint32_t* w, uint64_t n, bool pro_done = false, int fp_mode = -1);
cudaError_t launch_node_dist(meerkat_graph* g, meerkat_tree* t, uint32_t* out);
// part.cu (vertex-partitioned graphs)
meerkat_status part_init(meerkat_graph* g, const meerkat_config* cfg);   // after the stores are built
void part_free(meerkat_graph* g);
meerkat_status part_hints(meerkat_graph* g, const uint32_t* global_hints, const void** local_hints, int slot);
meerkat_status part_mutate(meerkat_graph* g, int kind, const uint32_t* s, const uint32_t* d, const uint32_t* w,
                           uint64_t n, uint64_t* count);
meerkat_status part_query(meerkat_graph* g, const uint32_t* s, const uint32_t* d, uint64_t n, uint8_t* found,
                          uint32_t* w_out);
meerkat_status part_tree_init(meerkat_graph* g, meerkat_tree* t);
void part_tree_free(meerkat_tree* t);
// kind: 0 static recompute, 1 incremental, 2 decremental (the batch must be the last mutation's)
meerkat_status part_trees(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, int kind, const uint32_t* s,
                          const uint32_t* d, const uint32_t* w, uint64_t n);
meerkat_status part_tree_nodes(meerkat_tree* t, uint64_t* out);
meerkat_status part_allreduce(meerkat_graph* g, uint64_t* vals, uint32_t m);   // sums over ranks (collective)
// api.cu helpers shared with part.cu
bool is_device_ptr(const void* p);
cudaError_t stage_in(meerkat_graph* g, int slot, const void* p, size_t bytes, const void** out);
cudaError_t ensure_stage(meerkat_graph* g, int slot, size_t bytes);
meerkat_status collect(meerkat_graph* g);
cudaError_t mutated(meerkat_graph* g, int kind, uint64_t n);
}  // namespace mk
