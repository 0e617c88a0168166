// tree.cu — batch-dynamic SSSP / BFS over the slab store, as ONE persistent
// cooperative kernel per tree call (no host round trip per frontier round).
//
// Method:
//  * tree node = <distance, parent> packed in 64 bits, distance high, relaxed by
//    one 64-bit atomicMin (footnote P:28-30; readings C1-C3);
//  * static: node[v] <- UNREACHED, node[SRC] <- <0,SRC>, frontier from
//    SRC (C16), repeat the relax kernel until the next frontier is empty
//    (P:108-133); BFS static is the level-synchronous special case w = 1;
//  * incremental prologue: the inserted batch is the initial frontier;
//  * decremental prologue: invalidate v for every deleted tree edge
//    (parent(v), v), propagate to the whole subtree T_v
//    (done top-down over out-edges, reading C14), then seed from all
//    edges (u, x) with u valid and x invalid (C15).
//
// B200 design:
//  * frontier items are (vertex, bucket) pairs — the paper's <v, i> work list of
//    IterationScheme2 — so a hub's slab lists spread over groups;
//  * an item is expanded by an 8-lane group (one LDG.128 per lane per slab),
//    relaxations are fused into the expansion (a vertex frontier with
//    per-round de-duplication stamps instead of the paper's edge frontier, C17);
//  * enqueue is the paper's warpenqueuefrontier (ballot, one atomicAdd per warp,
//    prefix offsets), extended to write all bucket items of a vertex;
//  * the decremental valid->invalid scan STREAMS the slab array in address order
//    (arena + pool, owner[] gives each slab's source vertex) instead of chasing
//    chains, tests each destination against a shared-memory hashed filter of the
//    invalid set, and relaxes hits directly — a pure HBM stream;
//  * rounds are separated by grid-wide barriers inside one launch.
#include <cooperative_groups.h>

#include <algorithm>

#include "tree_common.cuh"


namespace mk {

// Next item of this group (grid-stride over [it, n)): vertex and slab come from the item.
__device__ __forceinline__ bool fetch_item(const uint64_t* fr, uint64_t n, uint64_t& it, uint32_t& v, uint32_t& slab,
                                           int l8, Counters& c) {
  if (it >= n) return false;
  const uint64_t item = fr[it];
  v = (uint32_t)item;
  slab = (uint32_t)(item >> 32);
  if (l8 == 0) c.items++;
  return true;
}

// Expand the frontier items [0, n) of `fr` (one 8-lane group per item), applying
// VISIT to every live edge; successful vertices go to `fnext`.  The first slab of
// an item and d(v) are loaded together (independent requests).
template <bool MAP, int VISIT>
__device__ __forceinline__ void expand(const TreeArgs& A, const uint64_t* fr, uint64_t n, uint64_t* fnext,
                                       unsigned long long* sznext, uint32_t epoch_next, Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const GraphDev& S = VISIT == PULL ? A.R : A.G;   // store whose slab lists are walked
  const TreeDev& T = A.T;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const bool probe = n > PROBE_MIN_ITEMS;
  uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  uint32_t v = 0, slab = 0, du = 0;
  bool active = fetch_item(fr, n, it, v, slab, l8, c);
  bool fresh = active;
  while (__any_sync(FULL, active)) {
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    uint64_t nv = 0;
    if (active) {
      d = ld_slab_ro(slab_ptr(S, slab), l8);
      if (VISIT == RELAX && fresh && l8 == 0) nv = ld_cg_u64(T.node + v);   // one read per group, broadcast:
      if (l8 == 0) c.slabs++;                                               // d(v) may change concurrently
    }
    if (VISIT == RELAX) nv = __shfl_sync(FULL, nv, lane & 24);
    bool dead = false;
    if (VISIT == RELAX && active && fresh) {
      dead = nv == UNREACHED;
      du = (uint32_t)(nv >> 32);
    }
    fresh = false;
    const bool use = active && !dead;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t x = F::key(d, k);
      const bool live = use && F::valid_cell(l8, k) && x != EMPTY_KEY && x != TOMBSTONE_KEY;
      bool enq = false;
      if (live) {
        c.visited++;
        if (VISIT == RELAX) {
          const uint32_t w = A.unit ? 1u : F::weight(d, k);
          enq = relax(T, x, (uint64_t)du + w, v, epoch_next, c, probe);
        } else if (VISIT == PULL) {
          // in-edge (x -> v) of invalid v: a valid->invalid frontier edge iff x is valid and reached
          // (C15); relax v from it
          if (!bit_test(T.inval_bits, x)) {
            const uint64_t nx = ld_cg_u64(T.node + x);
            if (nx != UNREACHED) {
              c.hits++;
              const uint32_t w = A.unit ? 1u : F::weight(d, k);
              enq = relax(T, v, (nx >> 32) + w, x, epoch_next, c, false);
            }
          }
        } else {
          // PropagateInvalidation, top-down (C14): a child x of invalid v in T_G
          const uint64_t cur = ld_cg_u64(T.node + x);
          if (cur != UNREACHED && (uint32_t)cur == v && x != T.source) {
            if (atomicCAS(reinterpret_cast<unsigned long long*>(T.node + x), (unsigned long long)cur,
                          (unsigned long long)UNREACHED) == cur) {
              mark_invalid(T, x);
              enq = true;
            }
          }
        }
      }
      warp_enqueue(G, T, fnext, sznext, enq, VISIT == PULL ? v : x, c);
    }
    const uint32_t nxt = __shfl_sync(FULL, d.w, (lane & 24) + GROUP - 1);
    if (active) {
      if (nxt != INVALID_SLAB && !dead) slab = nxt;
      else { it += ng; active = fetch_item(fr, n, it, v, slab, l8, c); fresh = active; }
    }
  }
}

// Frontier rounds until empty.  Round r reads fr[r&1] / size[r%3], writes
// fr[(r+1)&1] / size[(r+1)%3]; size[(r+2)%3] (consumed two rounds ago) is
// zeroed during round r so it is clean when it becomes "next".
template <bool MAP, int VISIT>
__device__ __forceinline__ uint32_t run_rounds(const TreeArgs& A, uint32_t epoch, cg::grid_group& grid, uint32_t r,
                                               Counters& c) {
  TreeCtrl* tc = A.T.ctrl;
  for (;;) {
    const uint64_t n = __ldcg(&tc->size[r % 3]);
    if (n == 0) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) tc->size[(r + 2) % 3] = 0;
    expand<MAP, VISIT>(A, A.T.fr[r & 1], n, A.T.fr[(r + 1) & 1], &tc->size[(r + 1) % 3], epoch + r + 1, c);
    grid.sync();
    timeline(A.T.ctrl);
    r++;
  }
  return r;
}

// ------------------------------------------------------------------ static

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, 2) k_tree_static(const __grid_constant__ TreeArgs A) {
  const uint32_t epoch = __ldcg(A.T.epoch_ptr);
  timeline(A.T.ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  // init: every node <INF, INVALID>, SRC <0, SRC>
  for (uint64_t v = tid; v < A.G.V; v += nt) A.T.node[v] = (v == A.T.source) ? (uint64_t)A.T.source : UNREACHED;
  grid.sync();
    timeline(A.T.ctrl);
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const bool has = threadIdx.x == 0;
    if (has) A.T.stamp[A.T.source] = epoch;
    warp_enqueue(A.G, A.T, A.T.fr[0], &A.T.ctrl->size[0], has, A.T.source, c);   // frontier from SRC (C16)
  }
  grid.sync();
    timeline(A.T.ctrl);
  const uint32_t r = run_rounds<MAP, RELAX>(A, epoch, grid, 0, c);
  if (tid == 0) *A.T.epoch_ptr = epoch + r + 2;   // every thread read the base before the first grid.sync
  flush_counters(A.G, A.T, c, tid == 0, r, 0);
  clear_next_ctrl(A.clear_ctrl);
  timeline(A.T.ctrl);
}

// ------------------------------------------------------------------ incremental

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, 2) k_tree_inc(const __grid_constant__ TreeArgs A) {
  const uint32_t epoch = __ldcg(A.T.epoch_ptr);
  timeline(A.T.ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (A.bn + nt - 1) / nt;   // warp-uniform trip count (warp_enqueue is collective)
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    bool enq = false;
    uint32_t v = 0;
    if (i < A.bn) {
      const uint32_t u = A.bs[i];
      v = A.bd[i];
      const uint32_t w = A.unit ? 1u : A.bw[i];
      c.batch++;
      const bool ok = u < A.G.V && v < A.G.V && (A.unit || (w != 0 && w < W_LIMIT));   // skipped at insert too
      if (ok) {
        const uint64_t nu = ld_cg_u64(A.T.node + u);
        if (nu != UNREACHED) enq = relax(A.T, v, (nu >> 32) + w, u, epoch, c, false);
      }
    }
    warp_enqueue(A.G, A.T, A.T.fr[0], &A.T.ctrl->size[0], enq, v, c);
  }
  grid.sync();
    timeline(A.T.ctrl);
  const uint32_t r = run_rounds<MAP, RELAX>(A, epoch, grid, 0, c);
  if (tid == 0) *A.T.epoch_ptr = epoch + r + 2;
  flush_counters(A.G, A.T, c, tid == 0, r, 0);
  clear_next_ctrl(A.clear_ctrl);
  timeline(A.T.ctrl);
}

// ------------------------------------------------------------------ decremental

// Valid->invalid frontier (C15) as a STREAM over the slab array
// [0, n_slabs): each 8-lane group reads whole slabs (LDG.128 per lane, U slabs in
// flight); owner[] names the source vertex.  Fast path per key: one shared-memory
// filter probe.  Slow path (warp-uniform, only for positions where some lane hit
// the filter): exact bit-set test, source validity, relaxation and enqueue.
template <bool MAP>
__device__ __forceinline__ void dec_scan(const TreeArgs& A, const uint32_t* filt, uint32_t fwords, uint32_t n_slabs,
                                         uint64_t* fnext, unsigned long long* sznext, uint32_t epoch_next,
                                         Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  constexpr int U = SCAN_UNROLL;
  const GraphDev& G = A.G;
  const TreeDev& T = A.T;
  const uint32_t V = G.V;
  const int l8 = lane_id() & 7;
  const uint32_t ng = (gridDim.x * blockDim.x) / GROUP;
  const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint32_t span = ng * U;
  const uint32_t trips = (n_slabs + span - 1) / span;   // warp-uniform
  const uint4* __restrict__ base = reinterpret_cast<const uint4*>(G.slabs) + l8;
  // register double buffering: the next trip's U slabs are requested before this trip's keys are
  // tested, so every group always has loads in flight
  uint4 nd[U];
  auto load_trip = [&](uint32_t t, uint4 (&dst)[U]) {
#pragma unroll
    for (int q = 0; q < U; q++) {
      const uint32_t s = t * span + g0 + q * ng;
      dst[q] = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
      if (s < n_slabs) dst[q] = ld_slab_ro(reinterpret_cast<const uint32_t*>(base + (size_t)s * 8), 0);
    }
  };
  if (trips) load_trip(0, nd);
  for (uint32_t t = 0; t < trips; t++) {
    const uint32_t s0 = t * span + g0;
    uint4 d[U];
#pragma unroll
    for (int q = 0; q < U; q++) d[q] = nd[q];
    if (t + 1 < trips) load_trip(t + 1, nd);
    uint32_t hm = 0;
#pragma unroll
    for (int q = 0; q < U; q++) {
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t x = F::key(d[q], k);
        bool hit = x < V && (MAP || F::valid_cell(l8, k));   // live key (sentinels are >= V)
        if (fwords) {
          uint32_t w, m;
          filter_loc(x, fwords, w, m);
          hit = hit && (filt[w] & m) == m;
        }
        hm |= (uint32_t)hit << (q * NK + k);
      }
    }
    const uint32_t pos = __reduce_or_sync(FULL, hm);
    if (!pos) continue;
#pragma unroll
    for (int q = 0; q < U; q++) {
#pragma unroll
      for (int k = 0; k < NK; k++) {
        if (!((pos >> (q * NK + k)) & 1u)) continue;   // warp-uniform
        const uint32_t x = F::key(d[q], k);
        bool enq = false;
        if (((hm >> (q * NK + k)) & 1u) && bit_test(T.inval_bits, x)) {
          // x in V_invalid: is the slab's source vertex u valid and reached?
          const uint32_t u = __ldg(G.owner + s0 + q * ng);
          if (u != NO_OWNER && !bit_test(T.inval_bits, u)) {
            const uint64_t nu = ld_cg_u64(T.node + u);
            if (nu != UNREACHED) {
              c.hits++;
              const uint32_t w = A.unit ? 1u : F::weight(d[q], k);
              enq = relax(T, x, (nu >> 32) + w, u, epoch_next, c);
            }
          }
        }
        warp_enqueue(G, T, fnext, sznext, enq, x, c);
      }
    }
  }
}

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, 2) k_tree_dec(const __grid_constant__ TreeArgs A) {
  extern __shared__ uint32_t filt[];
  const uint32_t epoch = __ldcg(A.T.epoch_ptr);
  timeline(A.T.ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  TreeCtrl* tc = A.T.ctrl;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  // (i) Invalidate: deleted tree edges (parent(v), v), v != SRC (C4)
  const uint64_t trips = (A.bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    bool enq = false;
    uint32_t v = 0;
    if (i < A.bn) {
      const uint32_t u = A.bs[i];
      v = A.bd[i];
      c.batch++;
      if (u < A.G.V && v < A.G.V && v != A.T.source) {
        const uint64_t cur = ld_cg_u64(A.T.node + v);
        if (cur != UNREACHED && (uint32_t)cur == u &&
            atomicCAS(reinterpret_cast<unsigned long long*>(A.T.node + v), (unsigned long long)cur,
                      (unsigned long long)UNREACHED) == cur) {
          mark_invalid(A.T, v);
          atomicAdd(&tc->direct_n, 1ull);
          enq = true;
        }
      }
    }
    warp_enqueue(A.G, A.T, A.T.fr[0], &tc->size[0], enq, v, c);
  }
  grid.sync();
    timeline(A.T.ctrl);
  // (ii) PropagateInvalidation to all of T_v
  const uint32_t r1 = run_rounds<MAP, PROPAGATE>(A, epoch, grid, 0, c);
  // (iii) valid -> invalid frontier, fused with the first relaxation
  const uint64_t n_inv = __ldcg(&tc->inval_n);
  if (n_inv && A.R.slabs) {
    // in-edge mirror present: the frontier is exactly the in-edges of V_invalid from valid sources
    uint64_t* pull = A.T.fr[(r1 + 1) & 1];
    const uint64_t ptrips = (n_inv + nt - 1) / nt;
    for (uint64_t t = 0; t < ptrips; t++) {
      const uint64_t i = tid + t * nt;
      const bool has = i < n_inv;
      warp_enqueue(A.R, A.T, pull, &tc->pull_n, has, has ? __ldcg(A.T.inval_list + i) : 0u, c);
    }
    grid.sync();
    timeline(A.T.ctrl);
    expand<MAP, PULL>(A, pull, __ldcg(&tc->pull_n), A.T.fr[r1 & 1], &tc->size[r1 % 3], epoch + r1, c);
  } else if (n_inv) {
    // filter only while sparse enough: two bits per member, bit load <= 1/4 (false positives <= ~6%)
    const uint32_t fw = (A.filter_words && n_inv * 8 <= (uint64_t)A.filter_words * 32) ? A.filter_words : 0u;
    if (fw) {
      for (uint32_t i = threadIdx.x; i < fw; i += blockDim.x) filt[i] = 0;
      __syncthreads();
      for (uint64_t i = threadIdx.x; i < n_inv; i += blockDim.x) {
        uint32_t w, m;
        filter_loc(__ldcg(A.T.inval_list + i), fw, w, m);
        atomicOr(&filt[w], m);
      }
      __syncthreads();
    }
    const uint32_t n_slabs = A.G.H + (uint32_t)min((unsigned long long)A.G.P, __ldcg(&A.G.ctrl->pool_top));
    if (tid == 0) c.scan_slabs = n_slabs;
    dec_scan<MAP>(A, filt, fw, n_slabs, A.T.fr[r1 & 1], &tc->size[r1 % 3], epoch + r1, c);
  }
  grid.sync();
    timeline(A.T.ctrl);
  // (iv) common epilogue
  const uint32_t r2 = run_rounds<MAP, RELAX>(A, epoch, grid, r1, c);
  // clear the invalid bit set for the next call (the list is kept for meerkat_tree_invalidated)
  for (uint64_t i = tid; i < n_inv; i += nt) {
    const uint32_t x = A.T.inval_list[i];
    atomicAnd(A.T.inval_bits + (x >> 5), ~(1u << (x & 31)));
  }
  if (tid == 0) *A.T.epoch_ptr = epoch + r2 + 2;
  flush_counters(A.G, A.T, c, tid == 0, r2 - r1, r1);
  clear_next_ctrl(A.clear_ctrl);
  timeline(A.T.ctrl);
}

// ------------------------------------------------------------------ host side

template <typename K>
static cudaError_t occ(K kernel, int smem, int* out) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(out, kernel, TREE_BLOCK, smem);
}

cudaError_t tree_occupancy(meerkat_graph* g) {
  cudaError_t e;
  const int fbytes = FILTER_WORDS * 4;
  if (g->weighted) {
    if ((e = occ(k_tree_static<true>, 0, &g->tree_blocks_per_sm[0])) != cudaSuccess) return e;
    if ((e = occ(k_tree_inc<true>, 0, &g->tree_blocks_per_sm[1])) != cudaSuccess) return e;
    if ((e = occ(k_tree_dec<true>, fbytes, &g->tree_blocks_per_sm[2])) != cudaSuccess) return e;
  } else {
    if ((e = occ(k_tree_static<false>, 0, &g->tree_blocks_per_sm[0])) != cudaSuccess) return e;
    if ((e = occ(k_tree_inc<false>, 0, &g->tree_blocks_per_sm[1])) != cudaSuccess) return e;
    if ((e = occ(k_tree_dec<false>, fbytes, &g->tree_blocks_per_sm[2])) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_tree(meerkat_graph* g, meerkat_tree* t, int mode, const uint32_t* s, const uint32_t* d,
                        const uint32_t* w, uint64_t n) {
  TreeArgs A;
  A.G = g->out.dev;
  A.R = g->reverse ? g->in.dev : GraphDev{};
  A.T = t->dev;
  A.bs = s; A.bd = d; A.bw = w; A.bn = n;
  A.unit = t->unit ? 1u : 0u;
  A.weighted = g->weighted ? 1u : 0u;
  A.filter_words = g->reverse ? 0u : FILTER_WORDS;
  // control blocks alternate between calls: this call's was zeroed by the previous kernel
  A.T.ctrl = t->ctrl_base + t->parity;
  A.clear_ctrl = t->ctrl_base + (1 - t->parity);
  cudaError_t e = cudaSuccess;
  int bps = g->tree_blocks_per_sm[mode];
  if (bps <= 0) return cudaErrorInvalidConfiguration;
  // latency-bound calls (no full-store scan) may run on fewer blocks: cheaper grid barriers
  if (g->latency_bps > 0 && mode != MODE_STATIC && !(mode == MODE_DECREMENTAL && !g->reverse))
    bps = std::min(bps, g->latency_bps);
  dim3 grid((unsigned)(bps * g->sm_count)), block(TREE_BLOCK);
  void* args[] = {&A};
  // the shared-memory filter is only used by the full-store scan (no in-edge mirror)
  const size_t smem = (mode == MODE_DECREMENTAL && !g->reverse) ? (size_t)FILTER_WORDS * 4 : 0;
  void* fn;
  if (g->weighted)
    fn = mode == MODE_STATIC ? (void*)k_tree_static<true> : mode == MODE_INCREMENTAL ? (void*)k_tree_inc<true>
                                                                                     : (void*)k_tree_dec<true>;
  else
    fn = mode == MODE_STATIC ? (void*)k_tree_static<false> : mode == MODE_INCREMENTAL ? (void*)k_tree_inc<false>
                                                                                      : (void*)k_tree_dec<false>;
  e = cudaLaunchCooperativeKernel(fn, grid, block, args, smem, g->stream);
  if (e != cudaSuccess) return e;
  g->launches++;
  t->dev.ctrl = A.T.ctrl;   // stats / timeline / invalidated readers see this call's block
  t->parity ^= 1;
  return e;
}

}  // namespace mk
