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
//  * rounds are separated by grid-wide barriers inside one launch;
//  * FUSED trees: up to MAX_TREES trees of the same graph (an SSSP and a BFS tree,
//    say) are updated by one launch for the same batch — their frontier rounds share
//    the grid barriers, and the decremental scan streams the slab array ONCE for all
//    of them (one shared-memory filter per tree).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>

#include "stream.cuh"
#include "tree_common.cuh"


namespace mk {

#ifdef MEERKAT_DIAG_ROUNDS
// Diagnostics build only (-DMEERKAT_DIAG_ROUNDS; the atomics below perturb the timing): per round,
// the earliest group entry and latest group exit (%globaltimer), the longest group busy time, items,
// and a histogram of group busy times (1-us buckets); printed by block 0 at kernel end.
constexpr int DIAG_R = 64;
__device__ unsigned long long g_tmin[DIAG_R] /* ~earliest entry */, g_tmax[DIAG_R], g_busy[DIAG_R], g_items[DIAG_R];
__device__ unsigned int g_hist[DIAG_R][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ void diag_dump() {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned long long prev = 0;
  for (int r = 0; r < DIAG_R; r++) {
    if (!g_tmax[r]) continue;
    printf("DIAG r%02d items %6llu span %6.2f busymax %6.2f gap_before %6.2f hist", r, g_items[r],
           (g_tmax[r] - ~g_tmin[r]) / 1e3, g_busy[r] / 1e3, prev ? ((double)~g_tmin[r] - (double)prev) / 1e3 : 0.0);
    for (int b = 0; b < 16; b++) printf(" %u", g_hist[r][b]);
    printf("\n");
    prev = g_tmax[r];
    g_tmin[r] = 0; g_tmax[r] = 0; g_busy[r] = 0; g_items[r] = 0;
    for (int b = 0; b < 16; b++) g_hist[r][b] = 0;
  }
  printf("DIAG end\n");
}
#endif

// Next item of this group (grid-stride over [it, n)): vertex and slab come from the item.
// An item whose slab is LINKING was enqueued by the insert kernel's fused prologue before v's
// lazy head existed: the head is read from vmeta now (the insert has completed); still none = no
// out-edges, the item is skipped.
__device__ __forceinline__ bool fetch_item(const GraphDev& S, const uint64_t* fr, uint64_t n, uint64_t& it,
                                           uint64_t ng, uint32_t& v, uint32_t& slab, int l8, Counters& c) {
  for (; it < n; it += ng) {
    const uint64_t item = fr[it];
    v = (uint32_t)item;
    slab = (uint32_t)(item >> 32);
    if (slab == LINKING) {
      slab = __ldcg(&S.vmeta[v].x);
      if (slab == INVALID_SLAB || slab == LINKING) continue;
    }
    if (l8 == 0) c.items++;
    return true;
  }
  return false;
}

// Expand the frontier items [0, n) of `fr` (one 8-lane group per item) for tree T (index k),
// applying VISIT to every live edge; successful vertices go to (fnext, sznext).  The first slab
// of an item and d(v) are loaded together (independent requests).
// V32: the paper's VANILLA variant: node[] holds 32-bit distances only (no parent),
// relaxed by 32-bit atomicMin (static SSSP / BFS; RELAX only).
// BLOCK: only the calling block's groups share the items (the tail rounds of run_rounds).
// SPROBE (static calls): stamp[x] is read beside the node[x] probe, and an improved x already
// enqueued for the next round skips the stamp exchange -- static rounds improve a vertex many times
// per round (measured: static SSSP 19.6 -> 14.1 ms); the dynamic calls measured slower with it.
template <bool MAP, int VISIT, bool V32 = false, bool BLOCK = false, bool SPROBE = false, bool DECF = false>
__device__ __forceinline__ void expand(const TreeArgs& A, const TreeDev& T, int k, const uint64_t* fr, uint64_t n,
                                       uint64_t* fnext, unsigned long long* sznext, uint32_t epoch_next,
                                       Counters& c, int diag_round = DIAG_PULL) {
#ifdef MEERKAT_DIAG_ROUNDS
  const unsigned long long t_enter = gtime();
  uint32_t d_items = 0;
#endif
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const GraphDev& S = VISIT == PULL ? A.R : A.G;   // store whose slab lists are walked
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = BLOCK ? blockDim.x / GROUP : ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const bool probe = n > PROBE_MIN_ITEMS;
  uint64_t it = BLOCK ? threadIdx.x / GROUP : ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  uint32_t v = 0, slab = 0, du = 0;
  uint32_t b = 0, nb = 1, head0 = 0;   // IterationScheme1: bucket b of nb, first bucket head0
  bool active = fetch_item(S, fr, n, it, ng, v, slab, l8, c);
  bool fresh = active;
  while (__any_sync(FULL, active)) {
    if (T.scheme1) {   // (uniform) one item per vertex: walk all its buckets in turn
      uint32_t cntb = 1;
      if (active && fresh && l8 == 0) cntb = __ldcg(&G.vmeta[v].y);
      const uint32_t nbv = __shfl_sync(FULL, cntb, lane & 24);
      if (active && fresh) { nb = nbv; b = 0; head0 = slab; }
    }
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    uint64_t nv = 0;
    uint64_t pull_nv = 0;   // PULL: node[v] and stamp[v] beside the slab (lane 0 relaxes v): skip a
    uint32_t pull_st = 0;   // losing atomicMin, and the stamp exchange when v is already enqueued
    if (active) {
      d = ld_slab_ro(slab_ptr(S, slab), l8);
      if (VISIT == PULL && l8 == 0) { pull_nv = ld_cg_u64(T.node + v); pull_st = __ldcg(T.stamp + v); }
      if (VISIT == RELAX && fresh && l8 == 0)                                // one read per group, broadcast:
        nv = V32 ? (uint64_t)__ldcg(reinterpret_cast<const unsigned int*>(T.node) + v) << 32 : ld_cg_u64(T.node + v);
      if (l8 == 0) c.slabs++;                                               // d(v) may change concurrently
    }
    if (VISIT == RELAX) nv = __shfl_sync(FULL, nv, lane & 24);
    const uint32_t nxt = __shfl_sync(FULL, d.w, (lane & 24) + GROUP - 1);
    if ((PREFETCH & 1) && active && nxt != INVALID_SLAB && nxt != LINKING)   // the chain's next slab
      prefetch_l2(reinterpret_cast<const uint4*>(slab_ptr(S, nxt)) + l8);
    bool dead = false;
    if (VISIT == RELAX && active && fresh) {
      dead = V32 ? (nv >> 32) == INF_DIST : nv == UNREACHED;
      du = (uint32_t)(nv >> 32);
    }
    fresh = false;
    const bool use = active && !dead;
    // All loads / atomics of one phase are issued for every key of the slab before any result is
    // consumed, so one slab step costs one dependent round trip per phase (not per key).
    bool has[NK];
    uint32_t xs[NK];
    uint2 mv[NK];
#pragma unroll
    for (int kk = 0; kk < NK; kk++) { has[kk] = false; xs[kk] = F::key(d, kk); mv[kk] = make_uint2(INVALID_SLAB, 0); }
    if (VISIT == RELAX) {
      // relax: candidate <d(v) + w, v> into node[x]
      bool live[NK];
      uint64_t cand[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = xs[kk];
        live[kk] = use && F::valid_cell(l8, kk) && x != EMPTY_KEY && x != TOMBSTONE_KEY;
        cand[kk] = 0;
        if (live[kk]) {
          c.visited++;
          const uint64_t dist = (uint64_t)du + (T.unit ? 1u : F::weight(d, kk));
          if (dist >= INF_DIST) { c.err |= ERR_OVERFLOW; live[kk] = false; }   // C5
          cand[kk] = (dist << 32) | v;
        }
      }
      if constexpr (DECF) {
        // decremental relax rounds: only an invalid x can improve (a valid x keeps its optimal distance,
        // and d(v) + w >= the old d(v) + w >= d(x) with the same tie-break), so the node[x] probe -- a
        // random DRAM load -- is issued only for keys in V_invalid (the bit set is L2-resident)
        uint32_t bw[NK];
#pragma unroll
        for (int kk = 0; kk < NK; kk++) bw[kk] = live[kk] ? __ldcg(T.inval_bits + (xs[kk] >> 5)) : 0u;
#pragma unroll
        for (int kk = 0; kk < NK; kk++) live[kk] = live[kk] && ((bw[kk] >> (xs[kk] & 31)) & 1u);
      }
      if constexpr (V32) {   // distance only: compare and store the high half
#pragma unroll
        for (int kk = 0; kk < NK; kk++) cand[kk] >>= 32;
      }
      unsigned int* const node32 = reinterpret_cast<unsigned int*>(T.node);
      // probe (node[] only decreases: a stale read can only cost a spare atomic); stamp[x] is read
      // beside it: x already enqueued for the next round needs no stamp exchange after an improvement
      // (its expansion reads node[x] then)
      uint32_t ps[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) ps[kk] = 0u;
      if (probe) {
        uint64_t pv[NK];
#pragma unroll
        for (int kk = 0; kk < NK; kk++) {
          pv[kk] = !live[kk] ? 0ull : V32 ? (uint64_t)__ldcg(node32 + xs[kk]) : ld_cg_u64(T.node + xs[kk]);
          if (SPROBE) ps[kk] = live[kk] ? __ldcg(T.stamp + xs[kk]) : 0u;
        }
#pragma unroll
        for (int kk = 0; kk < NK; kk++) live[kk] = live[kk] && cand[kk] < pv[kk];
      }
      unsigned long long old[NK];
      uint32_t st[NK];
      if constexpr (SPEC_STAMP && !V32 && !SPROBE) {
        // speculative: the atomicMin, the stamp exchange and the vmeta load of a key that passed the
        // probe are issued together (one dependent round trip instead of two).  x is enqueued iff this
        // lane won the stamp: a lane whose atomicMin lost to a smaller candidate of the same round
        // still enqueues x correctly (x WAS improved this round); every improvement comes from a lane
        // that passed the probe and tried the stamp, so x is enqueued exactly once when improved.
#pragma unroll
        for (int kk = 0; kk < NK; kk++) {
          old[kk] = live[kk] ? atomicMin(reinterpret_cast<unsigned long long*>(T.node + xs[kk]),
                                         (unsigned long long)cand[kk]) : 0ull;
          st[kk] = live[kk] ? atomicExch(T.stamp + xs[kk], epoch_next) : epoch_next;
          mv[kk] = live[kk] ? __ldcg(G.vmeta + xs[kk]) : make_uint2(INVALID_SLAB, 0);
        }
#pragma unroll
        for (int kk = 0; kk < NK; kk++) {
          if (live[kk] && cand[kk] < old[kk]) c.improved++;
          has[kk] = st[kk] != epoch_next;
        }
        warp_enqueue_multi<NK>(T, fnext, sznext, has, xs, mv, c, G.slabs);
      } else {
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        if constexpr (V32)
          old[kk] = live[kk] ? atomicMin(node32 + xs[kk], (unsigned int)cand[kk]) : 0ull;
        else
          old[kk] = live[kk] ? atomicMin(reinterpret_cast<unsigned long long*>(T.node + xs[kk]),
                                         (unsigned long long)cand[kk]) : 0ull;
      }
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        st[kk] = epoch_next;
        if (live[kk] && cand[kk] < old[kk]) {   // improved: de-dup stamp and vmeta together
          c.improved++;
          if (!SPROBE || ps[kk] != epoch_next) {
            st[kk] = atomicExch(T.stamp + xs[kk], epoch_next);
            mv[kk] = __ldcg(G.vmeta + xs[kk]);
          }
        }
      }
#pragma unroll
      for (int kk = 0; kk < NK; kk++) has[kk] = st[kk] != epoch_next;
      warp_enqueue_multi<NK>(T, fnext, sznext, has, xs, mv, c, G.slabs);
      }
    } else if (VISIT == PROPAGATE) {
      // PropagateInvalidation, top-down (C14): the children x (parent(x) = v) of invalid v
      bool live[NK];
      uint64_t cur[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = xs[kk];
        live[kk] = use && F::valid_cell(l8, kk) && x != EMPTY_KEY && x != TOMBSTONE_KEY;
        cur[kk] = live[kk] ? ld_cg_u64(T.node + x) : UNREACHED;
        if (live[kk]) c.visited++;
      }
      // the CAS of a child and its vmeta load are issued together (SPEC_STAMP: one round trip)
      bool child[NK];
      unsigned long long oc[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = xs[kk];
        child[kk] = cur[kk] != UNREACHED && (uint32_t)cur[kk] == v && x != T.source;
        oc[kk] = child[kk] ? atomicCAS(reinterpret_cast<unsigned long long*>(T.node + x), (unsigned long long)cur[kk],
                                       (unsigned long long)UNREACHED) : 0ull;
        if (SPEC_STAMP && child[kk]) mv[kk] = __ldcg(G.vmeta + x);
      }
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        has[kk] = child[kk] && oc[kk] == cur[kk];
        if (!SPEC_STAMP && has[kk]) mv[kk] = __ldcg(G.vmeta + xs[kk]);
      }
      warp_mark_enqueue_multi<NK>(T, fnext, sznext, has, xs, xs, mv, c, G.slabs);
    } else {
      // PULL: in-edges (x -> v) of invalid v; a valid->invalid frontier edge iff x is valid and
      // reached (C15).  The group's candidates for v are min-reduced first: one atomicMin
      // per slab (the min of the candidates is what the per-edge atomics would leave).
      uint32_t bw[NK];
      uint64_t nx[NK];
      bool live[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = xs[kk];
        live[kk] = use && F::valid_cell(l8, kk) && x != EMPTY_KEY && x != TOMBSTONE_KEY;
        bw[kk] = live[kk] ? __ldcg(T.inval_bits + (x >> 5)) : 0u;
        nx[kk] = live[kk] ? ld_cg_u64(T.node + x) : UNREACHED;
        if (live[kk]) c.visited++;
      }
      uint64_t best = UNREACHED;
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = xs[kk];
        if (live[kk] && !((bw[kk] >> (x & 31)) & 1u) && nx[kk] != UNREACHED) {
          c.hits[k]++;
          const uint64_t dist = (nx[kk] >> 32) + (T.unit ? 1u : F::weight(d, kk));
          if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;   // C5
          else best = min(best, (dist << 32) | x);
        }
      }
      best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 1));
      best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 2));
      best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 4));
      bool hv[1] = {false};
      uint32_t xv[1] = {v};
      uint2 mv1[1] = {make_uint2(INVALID_SLAB, 0)};
      if (l8 == 0 && best != UNREACHED && best < pull_nv) {
        if (SPEC_STAMP) {   // atomicMin, stamp exchange and vmeta together (see RELAX)
          const unsigned long long o = atomicMin(reinterpret_cast<unsigned long long*>(T.node + v),
                                                 (unsigned long long)best);
          const uint32_t stv = pull_st != epoch_next ? atomicExch(T.stamp + v, epoch_next) : epoch_next;
          mv1[0] = pull_st != epoch_next ? __ldcg(G.vmeta + v) : make_uint2(INVALID_SLAB, 0);
          if (best < o) c.improved++;
          hv[0] = stv != epoch_next;
        } else {
        const unsigned long long o = atomicMin(reinterpret_cast<unsigned long long*>(T.node + v),
                                               (unsigned long long)best);
        if (best < o) {
          c.improved++;
          if (pull_st != epoch_next) {
            const uint32_t stv = atomicExch(T.stamp + v, epoch_next);
            mv1[0] = __ldcg(G.vmeta + v);
            hv[0] = stv != epoch_next;
          }
        }
        }
      }
      warp_enqueue_multi<1>(T, fnext, sznext, hv, xv, mv1, c, G.slabs);
    }
    if (active) {
      if (nxt != INVALID_SLAB && !dead) slab = nxt;
      else if (T.scheme1 && !dead && b + 1 < nb) { b++; slab = head0 + b; }
      else {
#ifdef MEERKAT_DIAG_ROUNDS
        d_items++;
#endif
        it += ng; active = fetch_item(S, fr, n, it, ng, v, slab, l8, c); fresh = active;
      }
    }
  }
#ifdef MEERKAT_DIAG_ROUNDS
  if (!BLOCK && l8 == 0 && d_items && diag_round >= 0 && diag_round < DIAG_R) {
    const unsigned long long t_exit = gtime(), busy = t_exit - t_enter;
    atomicMax(&g_tmin[diag_round], ~t_enter);   // holds ~(earliest entry): zero-initialised works
    atomicMax(&g_tmax[diag_round], t_exit);
    atomicMax(&g_busy[diag_round], busy);
    atomicAdd(&g_items[diag_round], (unsigned long long)d_items);
    atomicAdd(&g_hist[diag_round][min(15ull, busy / 1000)], 1u);
  }
#endif
}

// Frontier rounds of all trees of the call, until every frontier is empty.  Round r reads
// fr[r&1] / size[r%3] of each tree and writes fr[(r+1)&1] / size[(r+1)%3]; size[(r+2)%3]
// (consumed two rounds ago) is zeroed during round r so it is clean when it becomes "next".
// The trees share the grid barrier of every round.
template <bool MAP, int VISIT, bool V32 = false, bool SPROBE = false, bool DECF = false>
__device__ __forceinline__ uint32_t run_rounds(const TreeArgs& A, const uint32_t* epoch, cg::grid_group& grid,
                                               uint32_t r, Counters& c) {
  __shared__ unsigned long long s_n[MAX_TREES];
  for (;;) {
    // one load of each frontier size per block (not one per thread: ~150 K same-address loads
    // right after every barrier), broadcast through shared memory; the barrier that ends the
    // round orders the next round's write after this round's reads
    if (threadIdx.x < MAX_TREES)
      s_n[threadIdx.x] = threadIdx.x < A.ntrees ? __ldcg(&A.T[threadIdx.x].ctrl->size[r % 3]) : 0ull;
    __syncthreads();
    uint64_t n[MAX_TREES];
    bool any = false;
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      n[k] = s_n[k];
      any |= n[k] != 0;
    }
    if (!any) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) timeline_items(A.T[0].ctrl, n[0] + n[1]);   // diagnostics
    if (n[0] + n[1] <= TAIL_ITEMS) {
      // Tail: a frontier this small is one chain per item for block 0's groups alone, so block 0
      // runs the rounds with block barriers (~0.1 us) instead of grid barriers (~2 us) while the
      // frontier stays small; the other blocks wait once, then every block resumes the loop.
      if (blockIdx.x == 0) {
        for (;;) {
          if (threadIdx.x == 0)
            FOR_TREES(k, A) A.T[k].ctrl->size[(r + 2) % 3] = 0;
#pragma unroll
          for (int k = 0; k < MAX_TREES; k++) {
            if (!n[k]) continue;
            const TreeDev& T = A.T[k];
            expand<MAP, VISIT, V32, true, SPROBE, DECF>(A, T, k, T.fr[r & 1], n[k], T.fr[(r + 1) & 1],
                                          &T.ctrl->size[(r + 1) % 3], epoch[k] + r + 1, c);
          }
          __syncthreads();   // block-wide visibility of this round's frontier and node updates
          timeline(A.T[0].ctrl);
          r++;
          if (threadIdx.x < MAX_TREES)
            s_n[threadIdx.x] = threadIdx.x < A.ntrees ? __ldcg(&A.T[threadIdx.x].ctrl->size[r % 3]) : 0ull;
          __syncthreads();
          any = false;
#pragma unroll
          for (int k = 0; k < MAX_TREES; k++) { n[k] = s_n[k]; any |= n[k] != 0; }
          if (threadIdx.x == 0 && any) timeline_items(A.T[0].ctrl, n[0] + n[1]);
          __syncthreads();   // s_n is rewritten by the next iteration / the resumed loop
          if (!any || n[0] + n[1] > TAIL_ITEMS) break;
        }
        if (threadIdx.x == 0) A.T[0].ctrl->tail_r = r;
      }
      grid.sync();
      timeline(A.T[0].ctrl);   // every block resumed after block 0's tail rounds
      if (threadIdx.x == 0) s_n[0] = __ldcg(&A.T[0].ctrl->tail_r);
      __syncthreads();
      r = (uint32_t)s_n[0];
      __syncthreads();
      continue;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0)
      FOR_TREES(k, A) A.T[k].ctrl->size[(r + 2) % 3] = 0;
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (!n[k]) continue;
      const TreeDev& T = A.T[k];
      expand<MAP, VISIT, V32, false, SPROBE, DECF>(A, T, k, T.fr[r & 1], n[k], T.fr[(r + 1) & 1], &T.ctrl->size[(r + 1) % 3],
                              epoch[k] + r + 1, c, (VISIT == PROPAGATE ? 0 : 20) + (int)r);
    }
    grid.sync();
    timeline(A.T[0].ctrl);
    r++;
  }
  return r;
}

// Ordering contract (meerkat.h; "G undergoes modifications ... re-computes"): a dynamic call
// may only touch its trees if none is stale and, when asked, the batch it was given has the
// fingerprint of the batch the last mutation applied.  Otherwise nothing is written, the trees are
// marked stale (only a static recompute clears that) and MEERKAT_E_STATE is raised.  Grid-uniform.
__device__ __forceinline__ bool tree_call_admitted(const TreeArgs& A, cg::grid_group& grid, uint64_t tid,
                                                   uint64_t nt) {
  bool bad = false;
  FOR_TREES(k, A) bad |= __ldcg(A.T[k].epoch_ptr + 1) != 0u;
  if (A.fp_check) {
    uint64_t fa = 0, fb = 0;
    for (uint64_t i = tid; i < A.bn; i += nt) fp_edge(A.bs[i], A.bd[i], A.bw ? A.bw[i] : 0u, fa, fb);
    block_add2_u64(&A.T[0].ctrl->fp[0], fa, fb);
    grid.sync();
    bad |= __ldcg(&A.G.ctrl->fp[A.fp_slot][A.fp_w]) != __ldcg(&A.T[0].ctrl->fp[A.fp_w]);
  }
  if (bad) {
    if (tid == 0) atomicOr(&A.G.ctrl->err, (unsigned)ERR_STATE);
    FOR_TREES(k, A) {
      if (tid == 0) A.T[k].epoch_ptr[1] = 1u;
      clear_next_ctrl(A.clear_ctrl[k]);
    }
  }
  return !bad;
}

__device__ __forceinline__ void finish(const TreeArgs& A, Counters& c, const uint32_t* epoch, bool owner,
                                       uint32_t rounds_total, uint32_t relax_rounds, uint32_t prop_rounds) {
  timeline(A.T[0].ctrl);
#ifdef MEERKAT_DIAG_ROUNDS
  diag_dump();
#endif
  FOR_TREES(k, A) {
    if (owner) *A.T[k].epoch_ptr = epoch[k] + rounds_total + 2;   // every thread read the base before a barrier
    flush_counters<STAT_SLOTS>(A.G, A.T[k], c, k, owner, relax_rounds, prop_rounds);
    clear_next_ctrl(A.clear_ctrl[k]);
  }
  timeline(A.T[0].ctrl);
}

// Every tree's stamp-epoch base, loaded once per block and broadcast (not by every thread).
__device__ __forceinline__ void load_epochs(const TreeArgs& A, uint32_t (&epoch)[MAX_TREES]) {
  __shared__ uint32_t s_ep[MAX_TREES];
  if (threadIdx.x < A.ntrees) s_ep[threadIdx.x] = __ldcg(A.T[threadIdx.x].epoch_ptr);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) epoch[k] = k < (int)A.ntrees ? s_ep[k] : 0u;
}

// ------------------------------------------------------------------ static

template <bool MAP, bool V32>
__global__ void __launch_bounds__(TREE_BLOCK, 2) k_tree_static(const __grid_constant__ TreeArgs A) {
  const TreeDev& T = A.T[0];
  uint32_t epoch[MAX_TREES];
  load_epochs(A, epoch);
  timeline_begin(T.ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  if (tid == 0) T.epoch_ptr[1] = 0u;   // a static recompute makes a stale tree current again
  // init: every node <INF, INVALID>, SRC <0, SRC>
  if (V32)   // vanilla: distance 0 at SRC, INF elsewhere
    for (uint64_t v = tid; v < A.G.V; v += nt) reinterpret_cast<uint32_t*>(T.node)[v] = v == T.source ? 0u : INF_DIST;
  else
    for (uint64_t v = tid; v < A.G.V; v += nt) T.node[v] = (v == T.source) ? (uint64_t)T.source : UNREACHED;
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const bool has = threadIdx.x == 0;
    if (has) T.stamp[T.source] = epoch[0];
    warp_enqueue(A.G, T, T.fr[0], &T.ctrl->size[0], has, T.source, c);   // frontier from SRC (C16)
  }
  grid.sync();
  timeline(T.ctrl);
  const uint32_t r = run_rounds<MAP, RELAX, V32, true>(A, epoch, grid, 0, c);
  finish(A, c, epoch, tid == 0, r, r, 0);
}

// ------------------------------------------------------------------ incremental

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, TREE_MINB) k_tree_inc(const __grid_constant__ TreeArgs A) {
  uint32_t epoch[MAX_TREES];
  load_epochs(A, epoch);
  timeline_begin(A.T[0].ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  if (!tree_call_admitted(A, grid, tid, nt)) return;
  if (!A.pro_done) {   // else the insert kernel ran it (meerkat_insert_batch_trees)
    tree_prologue_inc<false>(A.G, A.T, A.ntrees, A.bs, A.bd, A.bw, A.bn, epoch, tid, nt, c);
    grid.sync();
  }
  timeline(A.T[0].ctrl);
  const uint32_t r = run_rounds<MAP, RELAX>(A, epoch, grid, 0, c);
  finish(A, c, epoch, tid == 0, r, r, 0);
}

// ------------------------------------------------------------------ decremental

// Valid->invalid frontier (C15) of every tree of the call as ONE STREAM over the
// slab array [0, n_slabs): each 8-lane group reads whole slabs (LDG.128 per lane, register
// double-buffered so loads are always in flight); owner[] names the source vertex.  Fast path
// per key and tree: one shared-memory filter probe.  Slow path (warp-uniform, only for positions
// where some lane hit a filter): exact bit-set test, source validity, relaxation and enqueue.
// One slab of the scan (this lane's fragment d, source u = owner[s]): the filter fast path, then the
// warp-uniform slow path for the positions where some lane hit.  Warp-collective.
template <bool MAP>
__device__ __forceinline__ void scan_slab(const TreeArgs& A, const uint32_t* filt, bool use_filter, const uint4& d,
                                          uint32_t u, uint32_t r1, const uint32_t* epoch, Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const uint32_t V = G.V;
  const int l8 = lane_id() & 7;
  uint32_t hm = 0;
#pragma unroll
  for (int kk = 0; kk < NK; kk++) {
    const uint32_t x = F::key(d, kk);
    bool hit = x < V && (MAP || F::valid_cell(l8, kk));   // live key (sentinels are >= V)
    if (use_filter) {
      uint32_t w, m;
      filter_loc(x, 32 - FILTER_LOG2, w, m);
      hit = hit && (filt[w] & m) == m;
    }
    hm |= (uint32_t)hit << kk;
  }
  const uint32_t pos = __reduce_or_sync(FULL, hm);
  if (!pos) return;
#pragma unroll
  for (int kk = 0; kk < NK; kk++) {
    if (!((pos >> kk) & 1u)) continue;   // warp-uniform
    const uint32_t x = F::key(d, kk);
    const bool cand = (hm >> kk) & 1u;
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (k >= (int)A.ntrees) break;
      const TreeDev& T = A.T[k];
      bool enq = false;
      if (cand && bit_test(T.inval_bits, x)) {
        // x in V_invalid of tree k: is the slab's source vertex u valid and reached in it?
        if (u != NO_OWNER && !bit_test(T.inval_bits, u)) {
          const uint64_t nu = ld_cg_u64(T.node + u);
          if (nu != UNREACHED) {
            c.hits[k]++;
            const uint32_t w = T.unit ? 1u : F::weight(d, kk);
            enq = relax(T, x, (nu >> 32) + w, u, epoch[k] + r1, c);
          }
        }
      }
      warp_enqueue(G, T, T.fr[r1 & 1], &T.ctrl->size[r1 % 3], enq, x, c);
    }
  }
}

#ifndef MEERKAT_SCAN_BULK
#define MEERKAT_SCAN_BULK 0   // 1: the scan's slab / owner stream moves by bulk copies (stream.cuh; A/B: 3x slower)
#endif

template <bool MAP>
__device__ __forceinline__ void dec_scan(const TreeArgs& A, const uint32_t* filt, bool use_filter, uint32_t n_slabs,
                                         uint32_t r1, const uint32_t* epoch, Counters& c) {
#if MEERKAT_SCAN_BULK
  __shared__ StreamSmem sm;
  uint32_t seq = 0;
  stream_init(sm);
  stream_slabs(sm, seq, A.G.slabs, A.G.owner, n_slabs, [&](const uint4& d, uint32_t u, uint32_t) {
    scan_slab<MAP>(A, filt, use_filter, d, u, r1, epoch, c);
  });
  return;
#endif
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  constexpr int U = SCAN_UNROLL;
  const GraphDev& G = A.G;
  const uint32_t V = G.V;
  const int l8 = lane_id() & 7;
  const uint32_t ng = (gridDim.x * blockDim.x) / GROUP;
  const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint32_t span = ng * U;
  const uint32_t trips = (n_slabs + span - 1) / span;   // warp-uniform
  const uint4* __restrict__ base = reinterpret_cast<const uint4*>(G.slabs) + l8;
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
    // fast path: one probe of the union filter (every tree's V_invalid) per key
    uint32_t hm = 0;
#pragma unroll
    for (int q = 0; q < U; q++) {
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        const uint32_t x = F::key(d[q], kk);
        bool hit = x < V && (MAP || F::valid_cell(l8, kk));   // live key (sentinels are >= V)
        if (use_filter) {
          uint32_t w, m;
          filter_loc(x, 32 - FILTER_LOG2, w, m);
          hit = hit && (filt[w] & m) == m;
        }
        hm |= (uint32_t)hit << (q * NK + kk);
      }
    }
    const uint32_t pos = __reduce_or_sync(FULL, hm);
    if (!pos) continue;
#pragma unroll
    for (int q = 0; q < U; q++) {
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        if (!((pos >> (q * NK + kk)) & 1u)) continue;   // warp-uniform
        const uint32_t x = F::key(d[q], kk);
        const bool cand = (hm >> (q * NK + kk)) & 1u;
#pragma unroll
        for (int k = 0; k < MAX_TREES; k++) {
          if (k >= (int)A.ntrees) break;
          const TreeDev& T = A.T[k];
          bool enq = false;
          if (cand && bit_test(T.inval_bits, x)) {
            // x in V_invalid of tree k: is the slab's source vertex u valid and reached in it?
            const uint32_t u = __ldg(G.owner + s0 + q * ng);
            if (u != NO_OWNER && !bit_test(T.inval_bits, u)) {
              const uint64_t nu = ld_cg_u64(T.node + u);
              if (nu != UNREACHED) {
                c.hits[k]++;
                const uint32_t w = T.unit ? 1u : F::weight(d[q], kk);
                enq = relax(T, x, (nu >> 32) + w, u, epoch[k] + r1, c);
              }
            }
          }
          warp_enqueue(G, T, T.fr[r1 & 1], &T.ctrl->size[r1 % 3], enq, x, c);
        }
      }
    }
  }
}

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, TREE_MINB) k_tree_dec(const __grid_constant__ TreeArgs A) {
  extern __shared__ uint32_t filt[];
  uint32_t epoch[MAX_TREES];
  load_epochs(A, epoch);
  timeline_begin(A.T[0].ctrl);
  cg::grid_group grid = cg::this_grid();
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  if (!tree_call_admitted(A, grid, tid, nt)) return;
  // (i) Invalidate: deleted tree edges (parent(v), v), v != SRC (C4)
  if (!A.pro_done) {   // else the delete kernel ran it (meerkat_delete_batch_trees)
    tree_prologue_dec(A.G, A.T, A.ntrees, A.bs, A.bd, A.bn, tid, nt, c);
    grid.sync();
  }
  timeline(A.T[0].ctrl);
  // (ii) PropagateInvalidation to all of T_v
  const uint32_t r1 = run_rounds<MAP, PROPAGATE>(A, epoch, grid, 0, c);
  // (iii) valid -> invalid frontier, fused with the first relaxation
  uint64_t n_inv[MAX_TREES] = {};
  uint64_t n_inv_all = 0;
  {
    __shared__ unsigned long long s_inv[MAX_TREES];
    if (threadIdx.x < A.ntrees) s_inv[threadIdx.x] = __ldcg(&A.T[threadIdx.x].ctrl->inval_n);
    __syncthreads();
    FOR_TREES(k, A) { n_inv[k] = s_inv[k]; n_inv_all += n_inv[k]; }
  }
  if (n_inv_all && A.R.slabs) {
    // in-edge mirror present: the frontier is exactly the in-edges of V_invalid from valid sources
    FOR_TREES(k, A) {
      const TreeDev& T = A.T[k];
      const uint64_t ptrips = (n_inv[k] + nt - 1) / nt;
      for (uint64_t t = 0; t < ptrips; t++) {
        const uint64_t i = tid + t * nt;
        const bool has = i < n_inv[k];
        warp_enqueue(A.R, T, T.fr[(r1 + 1) & 1], &T.ctrl->pull_n, has, has ? __ldcg(T.inval_list + i) : 0u, c);
      }
    }
    grid.sync();
    timeline(A.T[0].ctrl);
    __shared__ unsigned long long s_pull[MAX_TREES];
    if (threadIdx.x < A.ntrees) s_pull[threadIdx.x] = __ldcg(&A.T[threadIdx.x].ctrl->pull_n);
    __syncthreads();
    FOR_TREES(k, A) {
      const TreeDev& T = A.T[k];
      expand<MAP, PULL>(A, T, k, T.fr[(r1 + 1) & 1], s_pull[k], T.fr[r1 & 1], &T.ctrl->size[r1 % 3],
                        epoch[k] + r1, c);
    }
  } else if (n_inv_all) {
    // one shared-memory filter of the union of the trees' V_invalid, while sparse enough
    // (two bits per member, bit load <= 1/4)
    const bool use_filter = A.filter_words && n_inv_all * 8 <= (uint64_t)FILTER_WORDS * 32;
    if (use_filter) {
      for (uint32_t i = threadIdx.x; i < FILTER_WORDS; i += blockDim.x) filt[i] = 0;
      __syncthreads();
      FOR_TREES(k, A)
        for (uint64_t i = threadIdx.x; i < n_inv[k]; i += blockDim.x) {
          uint32_t w, m;
          filter_loc(__ldcg(A.T[k].inval_list + i), 32 - FILTER_LOG2, w, m);
          atomicOr(&filt[w], m);
        }
      __syncthreads();
    }
    __shared__ unsigned long long s_top;
    if (threadIdx.x == 0) s_top = __ldcg(&A.G.ctrl->pool_top);
    __syncthreads();
    const uint32_t n_slabs = A.G.H + (uint32_t)min((unsigned long long)A.G.P, s_top);
    if (tid == 0) c.scan_slabs = n_slabs;
    dec_scan<MAP>(A, filt, use_filter, n_slabs, r1, epoch, c);
  }
  grid.sync();
  timeline(A.T[0].ctrl);
  // (iv) common epilogue
  const uint32_t r2 = run_rounds<MAP, RELAX, false, false, DEC_FILTER>(A, epoch, grid, r1, c);
  // clear the invalid bit sets for the next call (the lists are kept for meerkat_tree_invalidated)
  FOR_TREES(k, A)
    for (uint64_t i = tid; i < n_inv[k]; i += nt) {
      const uint32_t x = A.T[k].inval_list[i];
      atomicAnd(A.T[k].inval_bits + (x >> 5), ~(1u << (x & 31)));
    }
  finish(A, c, epoch, tid == 0, r2, r2 - r1, r1);
}

// Distances of a tree: the high halves of the packed nodes (tree-based) or the 32-bit array (vanilla).
__global__ void k_node_dist(const uint64_t* __restrict__ node, uint32_t V, int vanilla, uint32_t* __restrict__ out) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = vanilla ? reinterpret_cast<const uint32_t*>(node)[v] : (uint32_t)(node[v] >> 32);
}

cudaError_t launch_node_dist(meerkat_graph* g, meerkat_tree* t, uint32_t* out) {
  const unsigned gb = (unsigned)std::min<uint64_t>((g->Vl + 255) / 256, (uint64_t)g->sm_count * 8);
  k_node_dist<<<std::max(gb, 1u), 256, 0, g->stream>>>(t->dev.node, g->Vl, t->vanilla ? 1 : 0, out);
  g->launches++;
  return cudaGetLastError();
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
    if ((e = occ(k_tree_static<true, false>, 0, &g->tree_blocks_per_sm[0])) != cudaSuccess) return e;
    if ((e = occ(k_tree_static<true, true>, 0, &g->tree_blocks_per_sm[3])) != cudaSuccess) return e;
    if ((e = occ(k_tree_inc<true>, 0, &g->tree_blocks_per_sm[1])) != cudaSuccess) return e;
    if ((e = occ(k_tree_dec<true>, fbytes, &g->tree_blocks_per_sm[2])) != cudaSuccess) return e;
  } else {
    if ((e = occ(k_tree_static<false, false>, 0, &g->tree_blocks_per_sm[0])) != cudaSuccess) return e;
    if ((e = occ(k_tree_static<false, true>, 0, &g->tree_blocks_per_sm[3])) != cudaSuccess) return e;
    if ((e = occ(k_tree_inc<false>, 0, &g->tree_blocks_per_sm[1])) != cudaSuccess) return e;
    if ((e = occ(k_tree_dec<false>, fbytes, &g->tree_blocks_per_sm[2])) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

void tree_pro_fill(meerkat_tree* const* trees, uint32_t ntrees, TreePro& p) {
  p.ntrees = ntrees;
  for (uint32_t k = 0; k < (uint32_t)MAX_TREES; k++) {
    meerkat_tree* t = trees[k < ntrees ? k : 0];
    p.T[k] = t->dev;
    p.T[k].unit = t->unit ? 1u : 0u;
    // control blocks alternate between calls: this call's was zeroed by the previous kernel
    p.T[k].ctrl = t->ctrl_base + t->parity;
  }
}

cudaError_t launch_tree(meerkat_graph* g, meerkat_tree* const* trees, uint32_t ntrees, int mode, const uint32_t* s,
                        const uint32_t* d, const uint32_t* w, uint64_t n, bool pro_done, int fp_mode) {
  if (ntrees == 0 || ntrees > (uint32_t)MAX_TREES) return cudaErrorInvalidValue;
  TreeArgs A{};
  A.pro_done = pro_done ? 1u : 0u;
  A.fp_check = fp_mode >= 0 && n > 0 ? 1u : 0u;
  A.fp_w = fp_mode > 0 ? 1u : 0u;
  A.fp_slot = (uint32_t)(g->version & 1);
  A.G = g->out.dev;
  A.R = g->reverse ? g->in.dev : GraphDev{};
  A.ntrees = ntrees;
  TreePro P;
  tree_pro_fill(trees, ntrees, P);
  for (uint32_t k = 0; k < (uint32_t)MAX_TREES; k++) {
    meerkat_tree* t = trees[k < ntrees ? k : 0];
    A.T[k] = P.T[k];
    A.clear_ctrl[k] = k < ntrees ? t->ctrl_base + (1 - t->parity) : nullptr;
  }
  A.bs = s; A.bd = d; A.bw = w; A.bn = n;
  A.weighted = g->weighted ? 1u : 0u;
  A.filter_words = g->reverse ? 0u : FILTER_WORDS;   // shared-memory union filter (scan only)
  const bool vanilla = trees[0]->vanilla;   // vanilla trees are static-only and never fused
  int bps = vanilla ? g->tree_blocks_per_sm[3] : g->tree_blocks_per_sm[mode];
  if (bps <= 0) return cudaErrorInvalidConfiguration;
  if (g->latency_bps > 0 && mode != MODE_STATIC && !(mode == MODE_DECREMENTAL && !g->reverse))
    bps = std::min(bps, g->latency_bps);
  dim3 grid((unsigned)(bps * g->sm_count)), block(TREE_BLOCK);
  for (uint32_t i = 0; i < ntrees; i++) trees[i]->stat_blocks = STAT_SLOTS ? grid.x : 0;   // slots the finish writes
  void* args[] = {&A};
  const size_t smem = (mode == MODE_DECREMENTAL && !g->reverse) ? (size_t)FILTER_WORDS * 4 : 0;
  void* fn;
  if (g->weighted)
    fn = mode == MODE_STATIC ? (vanilla ? (void*)k_tree_static<true, true> : (void*)k_tree_static<true, false>)
         : mode == MODE_INCREMENTAL ? (void*)k_tree_inc<true>
                                                                                     : (void*)k_tree_dec<true>;
  else
    fn = mode == MODE_STATIC ? (vanilla ? (void*)k_tree_static<false, true> : (void*)k_tree_static<false, false>)
         : mode == MODE_INCREMENTAL ? (void*)k_tree_inc<false>
                                                                                      : (void*)k_tree_dec<false>;
  cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, block, args, smem, g->stream);
  if (e != cudaSuccess) return e;
  g->launches++;
  for (uint32_t k = 0; k < ntrees; k++) {
    trees[k]->dev.ctrl = A.T[k].ctrl;   // stats / timeline / invalidated readers see this call's block
    trees[k]->parity ^= 1;
  }
  return e;
}

}  // namespace mk
