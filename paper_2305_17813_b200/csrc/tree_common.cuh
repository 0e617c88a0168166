// tree_common.cuh — device pieces shared by the single-GPU persistent tree
// kernels (tree.cu) and the vertex-partitioned multi-GPU phase kernels (dtree.cu).
#pragma once
#include <cooperative_groups.h>

#include "graph.h"

namespace cg = cooperative_groups;

namespace mk {

#ifndef MEERKAT_TREE_BLOCK
#define MEERKAT_TREE_BLOCK 512
#endif
constexpr int TREE_BLOCK = MEERKAT_TREE_BLOCK;   // threads per block of the cooperative tree kernels (A/B)
#ifndef MEERKAT_TREE_MINB
#define MEERKAT_TREE_MINB 2   // resident blocks per SM the dynamic tree kernels are compiled for (A/B)
#endif
constexpr int TREE_MINB = MEERKAT_TREE_MINB;
constexpr int FILTER_LOG2 = 14;
constexpr int FILTER_WORDS = 1 << FILTER_LOG2;   // 64 KiB smem Bloom filter per block (decremental scan)
#ifndef MEERKAT_SCAN_UNROLL
#define MEERKAT_SCAN_UNROLL 3
#endif
constexpr int SCAN_UNROLL = MEERKAT_SCAN_UNROLL;   // independent slabs in flight per group in the scan
constexpr unsigned FULL = 0xFFFFFFFFu;
#ifndef MEERKAT_PROBE_MIN_ITEMS
#define MEERKAT_PROBE_MIN_ITEMS 0   // measured: probing on every frontier size is best
#endif
constexpr uint64_t PROBE_MIN_ITEMS = MEERKAT_PROBE_MIN_ITEMS;   // frontiers above this read node[x] before the atomicMin
#ifndef MEERKAT_TAIL_ITEMS
#define MEERKAT_TAIL_ITEMS 64
#endif
constexpr uint64_t TAIL_ITEMS = MEERKAT_TAIL_ITEMS;
#ifndef MEERKAT_SPEC_STAMP
#define MEERKAT_SPEC_STAMP 1
#endif
// 1: a relaxation that passed the node[x] probe issues its atomicMin, the stamp exchange and the
// vmeta load together, and a propagation its CAS and vmeta load together: one dependent round trip
// fewer per slab step (tree.cu expand, the batch prologues).  0: the result-gated sequence.
constexpr bool SPEC_STAMP = MEERKAT_SPEC_STAMP != 0;
#ifndef MEERKAT_PREFETCH
#define MEERKAT_PREFETCH 3
#endif
// L2 prefetch of slabs a group will read next (bit 0: the next slab of the chain being walked, as
// soon as its link word arrives; bit 1: the head slabs of the items a round enqueues, read by the
// next round) -- the first dependent load of the next step then hits L2.
constexpr int PREFETCH = MEERKAT_PREFETCH;
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" :: "l"(p));
}
#ifndef MEERKAT_DEC_FILTER
#define MEERKAT_DEC_FILTER 1
#endif
constexpr bool DEC_FILTER = MEERKAT_DEC_FILTER != 0;   // decremental relax rounds probe only x in V_invalid
#ifndef MEERKAT_STAT_SLOTS
#define MEERKAT_STAT_SLOTS 1
#endif
constexpr bool STAT_SLOTS = MEERKAT_STAT_SLOTS != 0;   // tree kernels' counters: per-block slots (1) or atomics   // frontiers this small run in block 0 alone (run_rounds)

enum Visit { RELAX = 0, PROPAGATE = 1, PULL = 2 };
constexpr int DIAG_PULL = 19;   // diagnostics round slot of the pull phase (MEERKAT_DIAG_ROUNDS builds)

// Loop over the trees of a call with a compile-time index, so per-tree register arrays (Counters,
// epochs, frontier sizes) stay in registers: a runtime index puts them in local memory.
#define FOR_TREES(k, A) _Pragma("unroll") for (int k = 0; k < MAX_TREES; k++) if (k < (int)(A).ntrees)

struct TreeArgs {
  GraphDev G;           // out-edge store
  GraphDev R;           // in-edge mirror (R.slabs == nullptr when the graph keeps none)
  TreeDev T[MAX_TREES]; // the trees this call updates (same graph, same batch)
  TreeCtrl* clear_ctrl[MAX_TREES];   // each tree's other control block: zeroed at kernel end (no memset launch)
  uint32_t ntrees;
  const uint32_t* bs;   // batch (device)
  const uint32_t* bd;
  const uint32_t* bw;
  uint64_t bn;
  uint32_t weighted;    // graph has weights (map store)
  uint32_t filter_words;   // per tree
  uint32_t pro_done;       // the batch prologue already ran in the mutation kernel (fused calls)
  uint32_t fp_check;       // ordering contract: compare the batch's fingerprint with the mutation's
  uint32_t fp_slot;        // GraphCtrl::fp slot of the current graph version
  uint32_t fp_w;           // 1: the fingerprint includes the weights (bw given)
};

// Zero the next call's control block (block 0, after the last grid barrier).
__device__ __forceinline__ void clear_next_ctrl(TreeCtrl* p) {
  if (blockIdx.x != 0 || !p) return;
  unsigned long long* w = reinterpret_cast<unsigned long long*>(p);
  for (uint32_t i = threadIdx.x; i < sizeof(TreeCtrl) / 8; i += blockDim.x) w[i] = 0;
}

// Per-thread statistics; valid->invalid frontier edges are kept per tree, the rest per call.
struct Counters {
  uint32_t items = 0, slabs = 0, visited = 0, improved = 0, scan_slabs = 0, batch = 0, err = 0;
  uint32_t hits[MAX_TREES] = {};
  uint32_t direct[MAX_TREES] = {};   // vertices invalidated directly by a deleted tree edge
};

// Block-aggregated add of two per-thread 64-bit sums (batch fingerprints).
__device__ __forceinline__ void block_add2_u64(unsigned long long* dst, uint64_t a, uint64_t b) {
  __shared__ unsigned long long acc2[2];
  if (threadIdx.x < 2) acc2[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xFFFFFFFFu, (unsigned long long)a, o);
    b += __shfl_xor_sync(0xFFFFFFFFu, (unsigned long long)b, o);
  }
  if ((threadIdx.x & 31) == 0 && (a | b)) { atomicAdd(&acc2[0], (unsigned long long)a); atomicAdd(&acc2[1], (unsigned long long)b); }
  __syncthreads();
  if (threadIdx.x == 0) { atomicAdd(dst, acc2[0]); atomicAdd(dst + 1, acc2[1]); }
  __syncthreads();
}

__device__ __forceinline__ bool bit_test(const uint32_t* bits, uint32_t x) {
  return (__ldcg(bits + (x >> 5)) >> (x & 31)) & 1u;
}

// Device timeline (block 0 / thread 0): %globaltimer after the kernel start and every grid barrier.
// The entry count lives in a register-like shared word of block 0 (timeline_nts) -- reading it back
// from global memory put an L2 round trip on block 0's critical path after every barrier.
__device__ __forceinline__ unsigned int& timeline_nts() {
  __shared__ unsigned int s_nts;
  return s_nts;
}
__device__ __forceinline__ void timeline_at(TreeCtrl* tc, bool begin) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned int& n = timeline_nts();
    if (begin) n = 0;
    const unsigned int i = n;
    if (i < 48) tc->tstamp[i] = t;
    n = i + 1;
    tc->nts = i + 1;   // store only (read back by meerkat_tree_timeline)
  }
}
__device__ __forceinline__ void timeline(TreeCtrl* tc) { timeline_at(tc, false); }
__device__ __forceinline__ void timeline_begin(TreeCtrl* tc) { timeline_at(tc, true); }
// this round's frontier size beside the timeline entry that opened it (block 0 / thread 0)
__device__ __forceinline__ void timeline_items(TreeCtrl* tc, unsigned long long items) {
  const unsigned int i = timeline_nts();
  if (i > 0 && i <= 48) tc->titems[i - 1] = items;
}

// warpenqueuefrontier: all 32 lanes call; lanes with `has` append
// one item per slab list (bucket) of vertex x.  One atomicAdd per warp.
__device__ __forceinline__ void warp_enqueue(const GraphDev& G, const TreeDev& T, uint64_t* fr,
                                             unsigned long long* sz, bool has, uint32_t x, Counters& c) {
  if (!__ballot_sync(FULL, has)) return;
  const int lane = lane_id();
  uint32_t cnt = 0, head = 0;
  if (has) {
    const uint2 m = __ldcg(G.vmeta + x);
    head = m.x;
    cnt = m.x == INVALID_SLAB ? 0u : m.y;   // a vertex without a head slab has no out-edges
    if (T.scheme1 && cnt) cnt = 1;           // IterationScheme1: one item per vertex
  }
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  if (!total) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(sz, (unsigned long long)total);
  base = __shfl_sync(FULL, base, 31);
  if (base + total > T.fr_cap) { c.err |= ERR_CAPACITY; return; }
  const uint64_t off = base + incl - cnt;
  // item = (head slab of the bucket << 32) | vertex: the expander needs no vmeta lookup
  if (cnt <= 8) {
    for (uint32_t j = 0; j < cnt; j++) fr[off + j] = ((uint64_t)(head + j) << 32) | x;
  }
  uint32_t big = __ballot_sync(FULL, cnt > 8);
  while (big) {
    const int l = __ffs(big) - 1;
    big &= big - 1;
    const uint32_t xb = __shfl_sync(FULL, x, l);
    const uint32_t hb = __shfl_sync(FULL, head, l);
    const uint64_t ob = __shfl_sync(FULL, off, l);
    const uint32_t cb = __shfl_sync(FULL, cnt, l);
    for (uint32_t j = lane; j < cb; j += 32) fr[ob + j] = ((uint64_t)(hb + j) << 32) | xb;
  }
}

// warpenqueuefrontier for up to NK candidates per lane (one slab step of an expansion): lane
// candidate k appends the bucket items of vertex x[k] (head slab / bucket count in m[k], read
// by the caller together with its other loads) when has[k].  One atomicAdd per warp.
template <int NK>
__device__ __forceinline__ void warp_enqueue_multi(const TreeDev& T, uint64_t* fr, unsigned long long* sz,
                                                   const bool (&has)[NK], const uint32_t (&x)[NK],
                                                   const uint2 (&m)[NK], Counters& c,
                                                   const uint32_t* pf_slabs = nullptr) {
  uint32_t cnt[NK], mine = 0;
#pragma unroll
  for (int k = 0; k < NK; k++) {
    cnt[k] = (has[k] && m[k].x != INVALID_SLAB) ? m[k].y : 0u;   // no head slab: no out-edges
    if (T.scheme1 && cnt[k]) cnt[k] = 1;                          // IterationScheme1: one item per vertex
    mine += cnt[k];
  }
  if (!__any_sync(FULL, mine != 0)) return;
  const int lane = lane_id();
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(sz, (unsigned long long)total);
  base = __shfl_sync(FULL, base, 31);
  if (base + total > T.fr_cap) { c.err |= ERR_CAPACITY; return; }
  uint64_t off[NK];
  uint64_t o = base + incl - mine;
#pragma unroll
  for (int k = 0; k < NK; k++) {
    off[k] = o;
    o += cnt[k];
    if (cnt[k] <= 8)
      for (uint32_t j = 0; j < cnt[k]; j++) {
        fr[off[k] + j] = ((uint64_t)(m[k].x + j) << 32) | x[k];
        if ((PREFETCH & 2) && pf_slabs && m[k].x != LINKING) {   // the next round reads this head slab
          const uint32_t* sp = pf_slabs + (size_t)(m[k].x + j) * SLAB_WORDS;
          prefetch_l2(sp); prefetch_l2(sp + 8); prefetch_l2(sp + 16); prefetch_l2(sp + 24);
        }
      }
  }
#pragma unroll
  for (int k = 0; k < NK; k++) {
    uint32_t big = __ballot_sync(FULL, cnt[k] > 8);
    while (big) {   // hubs: the whole warp writes the items
      const int l = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t xb = __shfl_sync(FULL, x[k], l);
      const uint32_t hb = __shfl_sync(FULL, m[k].x, l);
      const uint64_t ob = __shfl_sync(FULL, off[k], l);
      const uint32_t cb = __shfl_sync(FULL, cnt[k], l);
      for (uint32_t j = lane; j < cb; j += 32) fr[ob + j] = ((uint64_t)(hb + j) << 32) | xb;
    }
  }
}

// mark_invalid for up to NK vertices per lane, one atomicAdd on the list length per warp
// (a per-vertex atomicAdd serialises thousands of same-address atomics at one L2 slice).
template <int NK>
__device__ __forceinline__ void warp_mark_invalid(const TreeDev& T, const bool (&has)[NK], const uint32_t (&x)[NK]) {
  uint32_t mine = 0;
#pragma unroll
  for (int k = 0; k < NK; k++)
    if (has[k]) { atomicOr(T.inval_bits + (x[k] >> 5), 1u << (x[k] & 31)); mine++; }
  if (!__any_sync(FULL, mine != 0)) return;
  const int lane = lane_id();
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(&T.ctrl->inval_n, (unsigned long long)incl);
  base = __shfl_sync(FULL, base, 31) + incl - mine;
#pragma unroll
  for (int k = 0; k < NK; k++)
    if (has[k]) T.inval_list[base++] = x[k];
}

// warp_mark_invalid + warp_enqueue_multi in one pass (invalidation): both prefix sums together and
// the two warp atomics (list length, frontier size) issued back to back, so an invalidating slab step
// waits for one L2 atomic round trip instead of two.  xm: ids for the bit set / list (global ids on a
// partitioned graph), xi: rows for the frontier items.
template <int NK>
__device__ __forceinline__ void warp_mark_enqueue_multi(const TreeDev& T, uint64_t* fr, unsigned long long* sz,
                                                        const bool (&has)[NK], const uint32_t (&xm)[NK],
                                                        const uint32_t (&xi)[NK], const uint2 (&m)[NK],
                                                        Counters& c, const uint32_t* pf_slabs = nullptr) {
  uint32_t cnt[NK], mine = 0, marks = 0;
#pragma unroll
  for (int k = 0; k < NK; k++) {
    if (has[k]) { atomicOr(T.inval_bits + (xm[k] >> 5), 1u << (xm[k] & 31)); marks++; }
    cnt[k] = (has[k] && m[k].x != INVALID_SLAB) ? m[k].y : 0u;
    if (T.scheme1 && cnt[k]) cnt[k] = 1;
    mine += cnt[k];
  }
  if (!__any_sync(FULL, marks != 0)) return;   // no mark, no item
  const int lane = lane_id();
  uint32_t incl = mine, incm = marks;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    const uint32_t z = __shfl_up_sync(FULL, incm, o);
    if (lane >= o) { incl += y; incm += z; }
  }
  unsigned long long bi = 0, bm = 0;
  if (lane == 31) {
    bm = atomicAdd(&T.ctrl->inval_n, (unsigned long long)incm);
    if (incl) bi = atomicAdd(sz, (unsigned long long)incl);
  }
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  bm = __shfl_sync(FULL, bm, 31) + incm - marks;
  bi = __shfl_sync(FULL, bi, 31);
#pragma unroll
  for (int k = 0; k < NK; k++)
    if (has[k]) T.inval_list[bm++] = xm[k];
  if (!total) return;
  if (bi + total > T.fr_cap) { c.err |= ERR_CAPACITY; return; }
  uint64_t off[NK];
  uint64_t o = bi + incl - mine;
#pragma unroll
  for (int k = 0; k < NK; k++) {
    off[k] = o;
    o += cnt[k];
    if (cnt[k] <= 8)
      for (uint32_t j = 0; j < cnt[k]; j++) {
        fr[off[k] + j] = ((uint64_t)(m[k].x + j) << 32) | xi[k];
        if ((PREFETCH & 2) && pf_slabs && m[k].x != LINKING) {
          const uint32_t* sp = pf_slabs + (size_t)(m[k].x + j) * SLAB_WORDS;
          prefetch_l2(sp); prefetch_l2(sp + 8); prefetch_l2(sp + 16); prefetch_l2(sp + 24);
        }
      }
  }
#pragma unroll
  for (int k = 0; k < NK; k++) {
    uint32_t big = __ballot_sync(FULL, cnt[k] > 8);
    while (big) {
      const int l = __ffs(big) - 1;
      big &= big - 1;
      const uint32_t xb = __shfl_sync(FULL, xi[k], l);
      const uint32_t hb = __shfl_sync(FULL, m[k].x, l);
      const uint64_t ob = __shfl_sync(FULL, off[k], l);
      const uint32_t cb = __shfl_sync(FULL, cnt[k], l);
      for (uint32_t j = lane; j < cb; j += 32) fr[ob + j] = ((uint64_t)(hb + j) << 32) | xb;
    }
  }
}

__device__ __forceinline__ void mark_invalid(const TreeDev& T, uint32_t x) {
  atomicOr(T.inval_bits + (x >> 5), 1u << (x & 31));
  const unsigned long long i = atomicAdd(&T.ctrl->inval_n, 1ull);
  T.inval_list[i] = x;
}

// Relax candidate <dist, parent> into node[x]; true iff x must be (re-)expanded next round.
// probe: read node[x] first and skip the atomic when it cannot win (node values only
// decrease, so a stale read can only cost a spare atomic) — saves atomics on large
// frontiers, costs one round trip on small ones.
__device__ __forceinline__ bool relax(const TreeDev& T, uint32_t x, uint64_t dist, uint32_t parent,
                                      uint32_t epoch_next, Counters& c, bool probe = true) {
  if (dist >= INF_DIST) { c.err |= ERR_OVERFLOW; return false; }   // C5
  const uint64_t cand = (dist << 32) | parent;
  if (probe && cand >= ld_cg_u64(T.node + x)) return false;
  const unsigned long long old = atomicMin(reinterpret_cast<unsigned long long*>(T.node + x), cand);
  if (cand >= old) return false;
  c.improved++;
  return atomicExch(T.stamp + x, epoch_next) != epoch_next;
}

// Counter flush at kernel end: warp reduce -> shared-memory block reduce -> one global
// atomic per counter per block (a warp-level flush put ~5K same-address atomics per
// counter on the kernel's tail).  SLOTS (the tree kernels): each block STORES its sums into its own
// slot T.bstat[block][8] instead -- no same-line atomics on the kernel's tail (2 trees x 8 counters x
// 296 blocks serialised at one L2 slice); meerkat_tree_stats_get adds the slots of the last call's
// grid.  All threads of the block must call it.
template <bool SLOTS = false>
__device__ __forceinline__ void flush_counters(const GraphDev& G, const TreeDev& T, Counters& c, int k,
                                               bool rounds_owner, uint32_t relax_rounds, uint32_t prop_rounds) {
  constexpr int NV = 8;
  __shared__ unsigned long long acc[NV + 1];
  TreeCtrl* tc = T.ctrl;
  if (threadIdx.x <= NV) acc[threadIdx.x] = 0;
  __syncthreads();
  auto red = [](uint32_t v) { return __reduce_add_sync(FULL, v); };
  const uint32_t v[NV] = {red(c.items), red(c.slabs), red(c.visited), red(c.improved), red(c.scan_slabs),
                          red(c.hits[k]), red(c.batch), red(c.direct[k])};
  const uint32_t err = __reduce_or_sync(FULL, c.err);
  if (lane_id() == 0) {
#pragma unroll
    for (int i = 0; i < NV; i++)
      if (v[i]) atomicAdd(&acc[i], (unsigned long long)v[i]);
    if (err) atomicOr(reinterpret_cast<unsigned int*>(&acc[NV]), err);
  }
  __syncthreads();
  if (SLOTS && threadIdx.x < NV) {
    T.bstat[(uint64_t)blockIdx.x * NV + threadIdx.x] = acc[threadIdx.x];
    if (threadIdx.x == 0 && acc[NV]) atomicOr(&G.ctrl->err, (unsigned int)acc[NV]);
  } else if (!SLOTS && threadIdx.x <= NV && acc[threadIdx.x]) {
    unsigned long long* dst[NV] = {&tc->items, &tc->slabs_read, &tc->visited, &tc->improved, &tc->scan_slabs,
                                   &tc->scan_hits, &tc->batch_edges, &tc->direct_n};
    if (threadIdx.x < NV) atomicAdd(dst[threadIdx.x], acc[threadIdx.x]);
    else atomicOr(&G.ctrl->err, (unsigned int)acc[NV]);
  }
  if (rounds_owner) { tc->rounds = relax_rounds; tc->prop_rounds = prop_rounds; }
}

// ---- Per-batch-edge prologues of the incremental / decremental calls.  Neither reads a slab, so
// besides opening k_tree_inc / k_tree_dec they also run inside the mutation kernel that applies
// the batch (meerkat_insert_batch_trees / meerkat_delete_batch_trees), which takes one grid-wide
// phase and barrier off the tree kernel.  The trip count is warp-uniform (warp_enqueue_multi is
// collective); tid / nt are the calling kernel's thread index and thread count.

// Incremental (P:113-133 for the relaxation): node[v] <- min(node[v], <d(u) + w, u>) for
// every batch edge (u, v); an improved v is enqueued, de-duplicated by stamp, into the round-0
// frontier fr[0] / size[0].  LAZY (running inside the insert kernel): v's lazy head slab (C22b)
// may still be being linked by the same launch, so an improved v seen without a head is enqueued
// as ONE item whose slab is LINKING — round 0 reads the head from vmeta when it fetches the item
// (a lazily headed vertex has exactly one bucket).
template <bool LAZY>
__device__ __forceinline__ void tree_prologue_inc(const GraphDev& G, const TreeDev (&T)[MAX_TREES], uint32_t ntrees,
                                                  const uint32_t* bs, const uint32_t* bd, const uint32_t* bw,
                                                  uint64_t bn, const uint32_t (&epoch)[MAX_TREES], uint64_t tid,
                                                  uint64_t nt, Counters& c) {
  const uint64_t trips = (bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    uint32_t u = 0, v = 0, w = 0;
    bool ok = false;
    if (i < bn) {
      u = bs[i];
      v = bd[i];
      w = bw ? bw[i] : 1u;
      c.batch++;
      ok = u < G.V && v < G.V;   // invalid edges were skipped by the insert too
    }
    // phase-wise over the trees: node[u] and node[v] of every tree (independent loads: node[v] only
    // filters -- node values only decrease, so a stale read can only cost a spare atomic), then the
    // atomicMins of the candidates that can still win, then stamp + vmeta
    uint64_t cand[MAX_TREES], cur_v[MAX_TREES];
    bool live[MAX_TREES];
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      const uint32_t wk = T[k].unit ? 1u : w;
      live[k] = k < (int)ntrees && ok && (T[k].unit || (wk != 0 && wk < W_LIMIT));
      cand[k] = live[k] ? ld_cg_u64(T[k].node + u) : UNREACHED;   // node[u], turned into the candidate below
      cur_v[k] = live[k] ? ld_cg_u64(T[k].node + v) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (live[k] && cand[k] != UNREACHED) {
        const uint64_t dist = (cand[k] >> 32) + (T[k].unit ? 1u : w);
        if (dist >= INF_DIST) { c.err |= ERR_OVERFLOW; live[k] = false; }   // C5
        cand[k] = (dist << 32) | u;
        live[k] = live[k] && cand[k] < cur_v[k];
      } else {
        live[k] = false;
      }
    }
    unsigned long long old[MAX_TREES];
    bool has[MAX_TREES][1];
    uint2 m[MAX_TREES][1];
    uint32_t st[MAX_TREES];
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      old[k] = live[k] ? atomicMin(reinterpret_cast<unsigned long long*>(T[k].node + v), (unsigned long long)cand[k])
                       : 0ull;
      if (SPEC_STAMP) {   // stamp exchange and vmeta beside the atomicMin (expand's RELAX explains why)
        st[k] = live[k] ? atomicExch(T[k].stamp + v, epoch[k]) : epoch[k];
        m[k][0] = live[k] ? __ldcg(G.vmeta + v) : make_uint2(INVALID_SLAB, 0);
      }
    }
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (SPEC_STAMP) {
        if (live[k] && cand[k] < old[k]) c.improved++;
        has[k][0] = st[k] != epoch[k];
        if (LAZY && has[k][0] && (m[k][0].x == INVALID_SLAB || m[k][0].x == LINKING)) m[k][0] = make_uint2(LINKING, 1u);
        continue;
      }
      has[k][0] = false;
      m[k][0] = make_uint2(INVALID_SLAB, 0);
      if (live[k] && cand[k] < old[k]) {
        c.improved++;
        has[k][0] = atomicExch(T[k].stamp + v, epoch[k]) != epoch[k];
        m[k][0] = __ldcg(G.vmeta + v);
        if (LAZY && (m[k][0].x == INVALID_SLAB || m[k][0].x == LINKING)) m[k][0] = make_uint2(LINKING, 1u);
      }
    }
    const uint32_t xv[1] = {v};
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++)
      if (k < (int)ntrees) warp_enqueue_multi<1>(T[k], T[k].fr[0], &T[k].ctrl->size[0], has[k], xv, m[k], c, G.slabs);
  }
}

// Decremental (C4): a deleted tree edge (parent(v), v), v != SRC, invalidates v (CAS
// to UNREACHED), marks it in V_invalid and enqueues it into the propagation frontier fr[0].
__device__ __forceinline__ void tree_prologue_dec(const GraphDev& G, const TreeDev (&T)[MAX_TREES], uint32_t ntrees,
                                                  const uint32_t* bs, const uint32_t* bd, uint64_t bn, uint64_t tid,
                                                  uint64_t nt, Counters& c) {
  const uint64_t trips = (bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    uint32_t u = 0, v = 0;
    bool ok = false;
    if (i < bn) {
      u = bs[i];
      v = bd[i];
      c.batch++;
      ok = u < G.V && v < G.V;
    }
    // phase-wise over the trees: node[v] of every tree, then the CASes, then list + enqueue
    uint64_t cur[MAX_TREES];
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++)
      cur[k] = (k < (int)ntrees && ok && v != T[k].source) ? ld_cg_u64(T[k].node + v) : UNREACHED;
    bool has[MAX_TREES][1];
    uint2 m[MAX_TREES][1];
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      const bool child = cur[k] != UNREACHED && (uint32_t)cur[k] == u;
      const unsigned long long oc = child ? atomicCAS(reinterpret_cast<unsigned long long*>(T[k].node + v),
                                                      (unsigned long long)cur[k], (unsigned long long)UNREACHED) : 0ull;
      if (SPEC_STAMP) m[k][0] = child ? __ldcg(G.vmeta + v) : make_uint2(INVALID_SLAB, 0);   // beside the CAS
      has[k][0] = child && oc == cur[k];
      if (!SPEC_STAMP) m[k][0] = has[k][0] ? __ldcg(G.vmeta + v) : make_uint2(INVALID_SLAB, 0);
      c.direct[k] += has[k][0];
    }
    const uint32_t xv[1] = {v};
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (k >= (int)ntrees) break;
      warp_mark_enqueue_multi<1>(T[k], T[k].fr[0], &T[k].ctrl->size[0], has[k], xv, xv, m[k], c, G.slabs);
    }
  }
}

// Blocked two-bit Bloom filter of V_invalid in shared memory: one word per key, two bits within
// it (false-positive rate ~ load^2).  Exact membership is the global bit set; the filter only keeps
// non-members off the slow path.  FILTER_WORDS is a power of two: word = top bits of a
// multiplicative hash, bits = two 5-bit fields of the (scrambled) id.
__device__ __forceinline__ void filter_loc(uint32_t x, uint32_t w_shift, uint32_t& w, uint32_t& m) {
  w = (x * 0x9E3779B1u) >> w_shift;
  m = (1u << (x & 31)) | (1u << ((x >> 5) & 31));
}

}  // namespace mk
