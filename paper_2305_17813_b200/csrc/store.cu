// store.cu — the per-vertex SlabHash adjacency store on sm_100a.
//
//  * construction: bucket_count[v] = ceil(hint/(lf*cap)),
//    exclusive scan into ONE head-slab arena, owner[] (the paper's
//    bucket_vertex[]) and a growth pool in the same allocation;
//  * batched insert / delete / query with the warp-cooperative work strategy
//    (WCWS; InsertEdge/DeleteEdge/SearchEdge P:634-641) re-cut for
//    B200 as 8-lane groups, one LDG.128 per lane per slab step;
//  * insert uses the search-then-claim protocol: pass 1
//    walks the slab list up to the first slab holding an EMPTY cell, looking
//    for the key and remembering the first writable (EMPTY or TOMBSTONE) cell;
//    pass 2 claims that cell with one CAS (64-bit for map pairs) and rescans
//    from it on failure; a full list gets a pool slab linked into lane 31 by
//    CAS ("chained at the end of the last filled slab").  A present key
//    keeps the minimum weight via a 64-bit atomicMin on the <key, w> pair (C8).
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cub/cub.cuh>

#include "store_ops.cuh"
#include "tree_common.cuh"

namespace mk {

// ------------------------------------------------------------------ helpers

// Group-cooperative: take one slab from the pool, write the EMPTY pattern with
// `first` in cell 0, record its owner, and fence it before it can be published.
template <bool MAP>
__device__ uint32_t group_alloc(const GraphDev& G, uint32_t u, uint64_t first, int l8, uint32_t gmask) {
  unsigned long long idx = 0;
  if (l8 == 0) idx = atomicAdd(&G.ctrl->pool_top, 1ull);
  idx = __shfl_sync(gmask, idx, 0, GROUP);
  if (idx >= G.P) return INVALID_SLAB;
  uint32_t s = G.H + (uint32_t)idx;
  uint4 f;
  f.x = fill_word(MAP, 4 * l8 + 0); f.y = fill_word(MAP, 4 * l8 + 1);
  f.z = fill_word(MAP, 4 * l8 + 2); f.w = fill_word(MAP, 4 * l8 + 3);
  if (l8 == 0) { f.x = (uint32_t)first; if (MAP) f.y = (uint32_t)(first >> 32); }
  reinterpret_cast<uint4*>(slab_ptr(G, s))[l8] = f;
  if (l8 == 0) G.owner[s] = u;
  __threadfence();
  __syncwarp(gmask);
  return s;
}

// Link a fresh slab holding `item` into *link (a lane-31 next word, or a vertex's
// head word) under a LINKING lock, so exactly one group allocates per link point
// and no slab is ever lost to a race ("chained at the end of the last
// filled slab").  Returns 1: our slab (holding the key) is linked; -1: pool
// exhausted; 0: another group linked first — *next_out is its slab, or
// INVALID_SLAB if that group failed to allocate.
template <bool MAP>
__device__ int group_link(const GraphDev& G, uint32_t u, uint64_t item, uint32_t* link, uint32_t& next_out, int l8,
                          uint32_t gmask) {
  uint32_t old = 0;
  if (l8 == 0) old = atomicCAS(link, INVALID_SLAB, LINKING);
  old = __shfl_sync(gmask, old, 0, GROUP);
  if (old == INVALID_SLAB) {
    const uint32_t s = group_alloc<MAP>(G, u, item, l8, gmask);   // fenced before publication
    if (l8 == 0) atomicExch(link, s);                              // s == INVALID_SLAB releases the lock
    __syncwarp(gmask);
    next_out = s;   // the caller's key sits in cell 0 of this slab
    return s == INVALID_SLAB ? -1 : 1;
  }
  uint32_t spins = 0;
  while (old == LINKING) {   // another group holds the lock: wait for its pointer
    __nanosleep(64);
    if (l8 == 0) old = *reinterpret_cast<volatile uint32_t*>(link);
    old = __shfl_sync(gmask, old, 0, GROUP);
    if (++spins == WATCHDOG) {   // never expected: report instead of hanging
      if (l8 == 0) {
        printf("meerkat watchdog: link wait u=%u link=%p\n", u, link);
        atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
      }
      return -1;
    }
  }
  next_out = old;
  return 0;
}

__device__ __forceinline__ uint32_t ld_head_cg(const GraphDev& G, uint32_t u) {
  return __ldcg(reinterpret_cast<const unsigned int*>(&G.vmeta[u].x));
}

// ------------------------------------------------------------------ insert (C9)

// Returns 1 = inserted (key was absent), 0 = present (weight min-upserted), -1 = pool exhausted.
// pos_list / pos (out, valid when 1 is returned): the slab list (its head slab) and the placement
// (slab << 5) | cell of the new key, for update tracking.
template <bool MAP>
__device__ int group_insert(const GraphDev& G, uint32_t u, uint32_t v, uint32_t wt, int l8, uint32_t gmask,
                            int gbase, uint32_t& pos_list, unsigned long long& pos) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const uint64_t item = MAP ? (((uint64_t)wt << 32) | v) : (uint64_t)v;
  const uint32_t count = G.vmeta[u].y;
  // vmeta.x of a lazily-headed vertex changes under concurrent inserts (INVALID -> LINKING -> slab):
  // one lane reads it and broadcasts, so every branch below stays uniform across the group
  uint32_t head = 0;
  if (l8 == 0) head = ld_head_cg(G, u);
  head = __shfl_sync(gmask, head, 0, GROUP);
  int result = 0;
  while (head == INVALID_SLAB || head == LINKING) {
    // vertex without a head slab yet (hint 0, reading C22b): publish one holding the key
    uint32_t nxt = INVALID_SLAB;
    const int r = group_link<MAP>(G, u, item, reinterpret_cast<uint32_t*>(&G.vmeta[u].x), nxt, l8, gmask);
    if (r == 1) { pos_list = nxt; pos = (unsigned long long)nxt << 5; }
    if (r != 0) return r;
    head = nxt;
  }
  uint32_t cur = head + bucket_of(v, count, G.seed);
  const uint32_t list0 = cur;
  uint32_t guard = 0, walk = 0;
  for (;;) {
    if (++guard == WATCHDOG) {
      if (l8 == 0) {
        const uint32_t h0 = G.vmeta[u].x, cnt0 = G.vmeta[u].y;
        printf("meerkat watchdog: insert retry loop u=%u v=%u cur=%u head=%u count=%u bucket=%u owner(cur)=%u "
               "H=%u P=%u\n", u, v, cur, h0, cnt0, bucket_of(v, cnt0, G.seed), G.owner[cur], G.H, G.P);
        uint32_t x = cur;
        for (int k = 0; k < 6 && x < G.H + G.P; k++) {
          const uint32_t* p = slab_ptr(G, x);
          printf("  slab %u owner %u next %u w0..5 %x %x %x %x %x %x w28..30 %x %x %x\n", x, G.owner[x], p[31],
                 p[0], p[1], p[2], p[3], p[4], p[5], p[28], p[29], p[30]);
          x = p[31];
        }
        atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
      }
      return -1;
    }
    // ---- pass 1: search up to the first slab with an EMPTY cell, remember the first writable cell
    uint32_t cand_slab = INVALID_SLAB, tail = INVALID_SLAB;
    int cand_cell = -1;
    uint64_t cand_old = 0;
    uint32_t s = cur;
    int found_cell = -1;
    uint32_t found_slab = INVALID_SLAB;
    for (;;) {
      const uint4 d = ld_slab_cg(slab_ptr(G, s), l8);
      uint32_t mb = 0, wb = 0, eb = 0;
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t key = F::key(d, k);
        const bool ok = F::valid_cell(l8, k);
        mb |= (uint32_t)(ok && key == v) << k;
        wb |= (uint32_t)(ok && (key == EMPTY_KEY || key == TOMBSTONE_KEY)) << k;
        eb |= (uint32_t)(ok && key == EMPTY_KEY) << k;
      }
      const int mc = group_first_cell<NK>(mb, gmask, gbase);
      if (mc >= 0) { found_cell = mc; found_slab = s; break; }
      if (cand_slab == INVALID_SLAB) {
        const int wc = group_first_cell<NK>(wb, gmask, gbase);
        if (wc >= 0) {
          const int src_lane = wc / NK, k = wc % NK;
          uint32_t lo = MAP ? (k == 0 ? d.x : d.z) : F::key(d, k);
          uint32_t hi = MAP ? (k == 0 ? d.y : d.w) : 0u;
          lo = __shfl_sync(gmask, lo, src_lane, GROUP);
          hi = __shfl_sync(gmask, hi, src_lane, GROUP);
          cand_slab = s; cand_cell = wc; cand_old = ((uint64_t)hi << 32) | lo;
        }
      }
      const bool has_empty = ((__ballot_sync(gmask, eb != 0) >> gbase) & 0xFFu) != 0;
      const uint32_t nxt = __shfl_sync(gmask, d.w, GROUP - 1, GROUP);
      if (has_empty || nxt == INVALID_SLAB || nxt == LINKING) { tail = s; break; }
      if (++walk == WALK_LIMIT || nxt >= G.H + G.P) {
        if (l8 == 0) {
          printf("meerkat watchdog: insert walk u=%u v=%u s=%u nxt=%u\n", u, v, s, nxt);
          atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
        }
        return -1;
      }
      s = nxt;
    }
    if (found_cell >= 0) {
      // present: min-weight upsert on the <key, w> pair (C8); the key half is equal
      if (MAP && l8 == 0)
        atomicMin(reinterpret_cast<unsigned long long*>(slab_ptr(G, found_slab) + 2 * found_cell),
                  (unsigned long long)item);
      result = 0;
      break;
    }
    if (cand_slab != INVALID_SLAB) {
      // ---- pass 2: claim the remembered first writable cell
      bool ok = false;
      if (l8 == 0) {
        if (MAP) {
          unsigned long long* cell = reinterpret_cast<unsigned long long*>(slab_ptr(G, cand_slab) + 2 * cand_cell);
          ok = atomicCAS(cell, (unsigned long long)cand_old, (unsigned long long)item) == cand_old;
        } else {
          unsigned int* cell = slab_ptr(G, cand_slab) + cand_cell;
          ok = atomicCAS(cell, (unsigned int)cand_old, (unsigned int)item) == (unsigned int)cand_old;
        }
      }
      ok = __shfl_sync(gmask, (int)ok, 0, GROUP);
      if (ok) { result = 1; pos_list = list0; pos = ((unsigned long long)cand_slab << 5) | (uint32_t)cand_cell; break; }
      cur = cand_slab;  // the cell changed under us: rescan from its slab
      continue;
    }
    // ---- list full: link a pool slab holding the key after the tail
    uint32_t nxt = INVALID_SLAB;
    const int r = group_link<MAP>(G, u, item, slab_ptr(G, tail) + (SLAB_WORDS - 1), nxt, l8, gmask);
    if (r == 1) { pos_list = list0; pos = (unsigned long long)nxt << 5; }
    if (r != 0) { result = r; break; }
    cur = nxt == INVALID_SLAB ? tail : nxt;   // continue in the slab another group linked
  }
  return result;
}

constexpr int UPD_BLOCK = 256;
// The group update kernels are compiled for 8 resident 256-thread blocks per SM (32 registers):
// at 40 registers only 6 fit, and the 100 K-edge batches' 1184 blocks ran in 1.3 waves.  Measured
// (same box, 3 x 2 runs): seeded insert 93 -> 87 us, step 0.356 -> 0.348 ms.
#ifndef MEERKAT_UPD_MINB
#define MEERKAT_UPD_MINB 8
#endif
// The thread-per-edge kernels (large batches) at 4 blocks per SM (<= 64 registers; k_delete_t used
// 72): config-4 insert of 970 K edges 0.570 -> 0.496 ms, 1 M-edge sweep insert 0.21 -> 0.16 ms;
// 8 blocks per SM (32 registers) spilled and was slower (same box, tools/gpu/r01_ab_tminb.sh).
#ifndef MEERKAT_UPD_T_MINB
#define MEERKAT_UPD_T_MINB 4
#endif
constexpr int UPD_T_MINB = MEERKAT_UPD_T_MINB;
constexpr int UPD_MINB = MEERKAT_UPD_MINB;

// Update kernels serve the out-edge store and, when the graph keeps one, the in-edge
// mirror in ONE launch: item i < ns*n is edge i/ns of the batch applied to store i%ns
// ((u, v) for the out store, (v, u) for the mirror).  Both stores' walks are then in
// flight together instead of two latency-bound launches back to back.
struct UpdArgs {
  GraphDev G[2];
  const uint32_t* src;
  const uint32_t* dst;
  const uint32_t* w;
  uint64_t n;
  uint32_t ns;   // stores updated: 1 or 2
  uint32_t fp_slot;   // batch fingerprint slot of the version this mutation creates (version & 1)
  uint32_t fp_on;     // 1: accumulate the batch fingerprint (some tree may follow with an unseeded call)
  // fused tree prologue (PRO != 0 kernels): the trees the following tree call updates
  TreeDev T[MAX_TREES];
  uint32_t ntrees;
};

// The batch prologue of the tree call that follows (PRO 1: incremental, 2: decremental), run by
// every thread of the mutation kernel after its own items: it reads no slab, so the insert /
// delete and the tree seeding share one launch (tree_prologue_inc / _dec, tree_common.cuh).
template <int PRO>
__device__ __forceinline__ void upd_tree_prologue(const UpdArgs& A) {
  __shared__ uint32_t s_ep[MAX_TREES];
  if (threadIdx.x < A.ntrees) s_ep[threadIdx.x] = __ldcg(A.T[threadIdx.x].epoch_ptr);
  __syncthreads();
  uint32_t epoch[MAX_TREES];
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) epoch[k] = k < (int)A.ntrees ? s_ep[k] : 0u;
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  if (PRO == 1) tree_prologue_inc<true>(A.G[0], A.T, A.ntrees, A.src, A.dst, A.w, A.n, epoch, tid, nt, c);
  else tree_prologue_dec(A.G[0], A.T, A.ntrees, A.src, A.dst, A.n, tid, nt, c);
  c.batch = 0;   // the tree call's alg_bytes then covers what its own kernel read
  FOR_TREES(k, A) flush_counters(A.G[0], A.T[k], c, k, false, 0, 0);
}

// Batch fingerprint bookkeeping (ordering contract): with fp_on the mutation accumulates the
// fingerprint of its batch into slot fp_slot and zeroes the other slot; without (a seeding mutation
// that seeds every tree of the graph: no tree call will read a batch) it zeroes both, so the next
// accumulating mutation starts from a clean slot.
template <int PRO>
__device__ __forceinline__ void upd_fp_begin(const UpdArgs& A) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  unsigned long long* f = &A.G[0].ctrl->fp[0][0];
  if (!A.fp_on) { f[0] = 0; f[1] = 0; f[2] = 0; f[3] = 0; }
  else { f[2 * (A.fp_slot ^ 1)] = 0; f[2 * (A.fp_slot ^ 1) + 1] = 0; }
}

template <int PRO>
__device__ __forceinline__ void upd_fp_end(const UpdArgs& A, uint64_t fa, uint64_t fb) {
  if (A.fp_on) block_add2_u64(&A.G[0].ctrl->fp[A.fp_slot][0], fa, fb);
}

template <int PRO>
__device__ __forceinline__ void upd_finish(const UpdArgs& A, const PerStore& err, const PerStore& cnt, bool ins,
                                           uint64_t fa, uint64_t fb) {
#pragma unroll
  for (int k = 0; k < 2; k++) {
    if (k >= (int)A.ns) break;
    block_or_err(&A.G[k].ctrl->err, err.get(k));
    if (ins) block_add(&A.G[k].ctrl->n_inserted, &A.G[k].ctrl->ins_total, cnt.get(k));
    else block_add(&A.G[k].ctrl->n_deleted, &A.G[k].ctrl->del_total, cnt.get(k));
  }
  upd_fp_end<PRO>(A, fa, fb);
  if constexpr (PRO != 0) upd_tree_prologue<PRO>(A);
}

__device__ __forceinline__ void upd_item(const UpdArgs& A, uint64_t i, uint32_t& st, uint64_t& e) {
  st = A.ns == 2 ? (uint32_t)(i & 1) : 0u;
  e = A.ns == 2 ? i >> 1 : i;
}

// TRACK: the out store keeps update tracking (compiled out of the default kernels).
// PRO: 1 = also run the incremental tree prologue (upd_tree_prologue).
template <bool MAP, bool TRACK, int PRO = 0>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_MINB) k_insert(const __grid_constant__ UpdArgs A) {
  const int lane = lane_id(), l8 = lane & 7, gbase = lane & 24;
  const uint32_t gmask = 0xFFu << gbase;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  PerStore added, err;
  uint64_t fa = 0, fb = 0;
  upd_fp_begin<PRO>(A);
  const uint64_t total = A.n * A.ns;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; i < total; i += ng) {
    uint32_t st; uint64_t e;
    upd_item(A, i, st, e);
    const GraphDev& G = A.G[st];
    const uint32_t a = A.src[e], b = A.dst[e], wt = MAP ? A.w[e] : 0u;
    if (A.fp_on && st == 0 && l8 == 0) fp_edge(a, b, wt, fa, fb);
    const uint32_t u = st ? b : a, v = st ? a : b;
    if (u >= G.Vg || v >= G.Vg) { err.set(st, ERR_RANGE); continue; }
    if (MAP && (wt == 0 || wt >= W_LIMIT)) { err.set(st, ERR_WEIGHT); continue; }
    const uint32_t ul = local_row(G, u);
    if (ul == INVALID_SLAB) { err.set(st, ERR_PARTITION); continue; }
    uint32_t plist = 0;
    unsigned long long ppos = 0;
    const int r = group_insert<MAP>(G, ul, v, wt, l8, gmask, gbase, plist, ppos);
    if (r < 0) err.set(st, ERR_CAPACITY);
    else if (l8 == 0 && r) {
      added.add(st, 1);
      if (TRACK && G.upd) track_update(G, plist, ppos);
    }
  }
  upd_finish<PRO>(A, err, added, true, fa, fb);
}

// ------------------------------------------------------------------ delete / query

// Walk the slab list of (u, bucket(v)) up to the first slab with an EMPTY cell.
// Returns the matching cell (or -1) and its slab / observed value.
template <bool MAP>
__device__ int group_find(const GraphDev& G, uint32_t u, uint32_t v, int l8, uint32_t gmask, int gbase,
                          uint32_t& slab_out, uint64_t& val_out) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const uint32_t head = ld_head_cg(G, u);
  if (head == INVALID_SLAB) return -1;
  uint32_t s = head + bucket_of(v, G.vmeta[u].y, G.seed);
  uint32_t guard = 0;
  for (;;) {
    const uint4 d = ld_slab_cg(slab_ptr(G, s), l8);
    uint32_t mb = 0, eb = 0;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t key = F::key(d, k);
      const bool ok = F::valid_cell(l8, k);
      mb |= (uint32_t)(ok && key == v) << k;
      eb |= (uint32_t)(ok && key == EMPTY_KEY) << k;
    }
    const int mc = group_first_cell<NK>(mb, gmask, gbase);
    if (mc >= 0) {
      const int src_lane = mc / NK, k = mc % NK;
      uint32_t lo = MAP ? (k == 0 ? d.x : d.z) : F::key(d, k);
      uint32_t hi = MAP ? (k == 0 ? d.y : d.w) : 0u;
      lo = __shfl_sync(gmask, lo, src_lane, GROUP);
      hi = __shfl_sync(gmask, hi, src_lane, GROUP);
      slab_out = s;
      val_out = ((uint64_t)hi << 32) | lo;
      return mc;
    }
    const bool has_empty = ((__ballot_sync(gmask, eb != 0) >> gbase) & 0xFFu) != 0;
    const uint32_t nxt = __shfl_sync(gmask, d.w, GROUP - 1, GROUP);
    if (has_empty || nxt == INVALID_SLAB) return -1;
    if (++guard == WALK_LIMIT || nxt >= G.H + G.P) {
      if (l8 == 0) {
        printf("meerkat watchdog: find walk u=%u v=%u s=%u nxt=%u\n", u, v, s, nxt);
        atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
      }
      return -1;
    }
    s = nxt;
  }
}

template <bool MAP, int PRO = 0>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_MINB) k_delete(const __grid_constant__ UpdArgs A) {
  const int lane = lane_id(), l8 = lane & 7, gbase = lane & 24;
  const uint32_t gmask = 0xFFu << gbase;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  PerStore removed, err;
  uint64_t fa = 0, fb = 0;
  upd_fp_begin<PRO>(A);
  const uint64_t total = A.n * A.ns;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; i < total; i += ng) {
    uint32_t st; uint64_t e;
    upd_item(A, i, st, e);
    const GraphDev& G = A.G[st];
    const uint32_t a = A.src[e], b = A.dst[e];
    if (A.fp_on && st == 0 && l8 == 0) fp_edge(a, b, 0u, fa, fb);
    const uint32_t u = st ? b : a, v = st ? a : b;
    if (u >= G.Vg || v >= G.Vg) { err.set(st, ERR_RANGE); continue; }
    const uint32_t ul = local_row(G, u);
    if (ul == INVALID_SLAB) { err.set(st, ERR_PARTITION); continue; }
    uint32_t slab; uint64_t val;
    const int c = group_find<MAP>(G, ul, v, l8, gmask, gbase, slab, val);
    if (c < 0 || l8 != 0) continue;
    // TOMBSTONE the cell; a failed CAS means a duplicate in this batch won
    bool ok;
    if (MAP) ok = atomicCAS(reinterpret_cast<unsigned long long*>(slab_ptr(G, slab) + 2 * c),
                            (unsigned long long)val, (unsigned long long)TOMB_PAIR) == val;
    else ok = atomicCAS(slab_ptr(G, slab) + c, (unsigned int)val, TOMBSTONE_KEY) == (unsigned int)val;
    if (ok) removed.add(st, 1);
  }
  upd_finish<PRO>(A, err, removed, false, fa, fb);
}

template <bool MAP>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_MINB) k_query(GraphDev G, const uint32_t* __restrict__ src,
                                                     const uint32_t* __restrict__ dst, uint64_t n,
                                                     uint8_t* __restrict__ found, uint32_t* __restrict__ w_out) {
  const int lane = lane_id(), l8 = lane & 7, gbase = lane & 24;
  const uint32_t gmask = 0xFFu << gbase;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  uint32_t err = 0;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; i < n; i += ng) {
    const uint32_t u = src[i], v = dst[i];
    int c = -1;
    uint32_t slab; uint64_t val = 0;
    const uint32_t ul = u < G.Vg ? local_row(G, u) : INVALID_SLAB;
    if (u >= G.Vg || v >= G.Vg) err |= ERR_RANGE;
    else if (ul == INVALID_SLAB) err |= ERR_PARTITION;
    else c = group_find<MAP>(G, ul, v, l8, gmask, gbase, slab, val);
    if (l8 == 0) {
      found[i] = c >= 0;
      if (w_out) w_out[i] = (MAP && c >= 0) ? (uint32_t)(val >> 32) : 0u;
    }
  }
  block_or_err(&G.ctrl->err, err);
}

// ---------------------------------------------------------- thread-per-edge lookup

// One thread per edge reads whole slabs itself (8 x LDG.128 of the same 128-B line): no group
// collectives, one divergent path per edge instead of four per warp (large batches, see thread_upd).
template <bool MAP>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_T_MINB) k_query_t(GraphDev G, const uint32_t* __restrict__ src,
                                                       const uint32_t* __restrict__ dst, uint64_t n,
                                                       uint8_t* __restrict__ found, uint32_t* __restrict__ w_out) {
  using F = Frag<MAP>;
  uint32_t err = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = src[i], v = dst[i];
    bool hit = false;
    uint32_t wt = 0;
    const uint32_t ul = u < G.Vg ? local_row(G, u) : INVALID_SLAB;
    if (u >= G.Vg || v >= G.Vg) err |= ERR_RANGE;
    else if (ul == INVALID_SLAB) err |= ERR_PARTITION;
    else {
      const uint2 m = __ldcg(G.vmeta + ul);
      if (m.x != INVALID_SLAB) {
        uint32_t sl = m.x + bucket_of(v, m.y, G.seed);
        for (uint32_t guard = 0; guard < WALK_LIMIT; guard++) {
          const uint4* p = reinterpret_cast<const uint4*>(slab_ptr(G, sl));
          uint4 q[8];
#pragma unroll
          for (int j = 0; j < 8; j++) q[j] = __ldcg(p + j);
          bool empty = false;
#pragma unroll
          for (int j = 0; j < 8; j++) {
#pragma unroll
            for (int k = 0; k < F::NK; k++) {
              if (!F::valid_cell(j, k)) continue;
              const uint32_t key = F::key(q[j], k);
              if (key == v) { hit = true; if (MAP) wt = F::weight(q[j], k); }
              empty |= key == EMPTY_KEY;
            }
          }
          if (hit || empty || q[7].w == INVALID_SLAB) break;
          sl = q[7].w;
        }
      }
    }
    found[i] = hit;
    if (w_out) w_out[i] = hit ? wt : 0u;
  }
  block_or_err(&G.ctrl->err, err);
}

// ---------------------------------------------------------- thread-per-edge updates
//
// The same protocols (C9 search-then-claim insert, link lock, TOMBSTONE delete) with ONE thread per
// edge reading whole slabs (8 x LDG.128 of one 128-B line): no group collectives and one divergent
// path per edge.  Used for large batches (thread_upd).

template <bool MAP, bool TRACK, int PRO = 0>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_T_MINB) k_insert_t(const __grid_constant__ UpdArgs A) {
  PerStore added, err;
  uint64_t fa = 0, fb = 0;
  upd_fp_begin<PRO>(A);
  const uint64_t total = A.n * A.ns;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t st; uint64_t e;
    upd_item(A, i, st, e);
    const GraphDev& G = A.G[st];
    const uint32_t a = A.src[e], b = A.dst[e], wt = MAP ? A.w[e] : 0u;
    if (A.fp_on && st == 0) fp_edge(a, b, wt, fa, fb);
    const uint32_t u = st ? b : a, v = st ? a : b;
    if (u >= G.Vg || v >= G.Vg) { err.set(st, ERR_RANGE); continue; }
    if (MAP && (wt == 0 || wt >= W_LIMIT)) { err.set(st, ERR_WEIGHT); continue; }
    const uint32_t ul = local_row(G, u);
    if (ul == INVALID_SLAB) { err.set(st, ERR_PARTITION); continue; }
    uint32_t plist = 0;
    unsigned long long ppos = 0;
    const int r = thread_insert<MAP>(G, ul, v, wt, plist, ppos);
    if (r < 0) err.set(st, ERR_CAPACITY);
    else if (r) {
      added.add(st, 1);
      if (TRACK && G.upd) track_update(G, plist, ppos);
    }
  }
  upd_finish<PRO>(A, err, added, true, fa, fb);
}

template <bool MAP, int PRO = 0>
__global__ void __launch_bounds__(UPD_BLOCK, UPD_T_MINB) k_delete_t(const __grid_constant__ UpdArgs A) {
  PerStore removed, err;
  uint64_t fa = 0, fb = 0;
  upd_fp_begin<PRO>(A);
  const uint64_t total = A.n * A.ns;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t st; uint64_t e;
    upd_item(A, i, st, e);
    const GraphDev& G = A.G[st];
    const uint32_t a = A.src[e], b = A.dst[e];
    if (A.fp_on && st == 0) fp_edge(a, b, 0u, fa, fb);
    const uint32_t u = st ? b : a, v = st ? a : b;
    if (u >= G.Vg || v >= G.Vg) { err.set(st, ERR_RANGE); continue; }
    const uint32_t ul = local_row(G, u);
    if (ul == INVALID_SLAB) { err.set(st, ERR_PARTITION); continue; }
    if (thread_delete<MAP>(G, ul, v)) removed.add(st, 1);
  }
  upd_finish<PRO>(A, err, removed, false, fa, fb);
}

// Kernel choice by batch size (measured): small batches are latency-bound and the
// 8-lane groups (four independent slabs per warp instruction, fewer requests per slab) win; large
// batches are throughput-bound and thread-per-edge wins (no group collectives: 2x at 1M edges and in
// the bulk build).  MEERKAT_THREAD_UPD=0/1 forces one kind (experiments and tests).
constexpr uint64_t THREAD_MIN_ITEMS = 400000;

static bool thread_upd(uint64_t items) {
  const char* e = std::getenv("MEERKAT_THREAD_UPD");
  if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
  return items >= THREAD_MIN_ITEMS;
}

static unsigned grid_threads(meerkat_graph* g, uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + UPD_BLOCK - 1) / UPD_BLOCK, (uint64_t)g->sm_count * 8));
}

// ------------------------------------------------------------------ export (streaming)

template <bool MAP>
__global__ void __launch_bounds__(UPD_BLOCK) k_export(GraphDev G, uint64_t n_slabs, uint32_t* __restrict__ os,
                                                      uint32_t* __restrict__ od, uint32_t* __restrict__ ow,
                                                      uint64_t cap) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t g0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint64_t trips = (n_slabs + ng - 1) / ng;  // warp-uniform trip count
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t s = g0 + t * ng;
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, EMPTY_KEY);
    uint32_t own = NO_OWNER;
    if (s < n_slabs) {
      own = G.owner[s];
      if (own != NO_OWNER) d = ld_slab_cg(slab_ptr(G, (uint32_t)s), l8);
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t key = F::key(d, k);
      cnt += (own != NO_OWNER && F::valid_cell(l8, k) && key != EMPTY_KEY && key != TOMBSTONE_KEY);
    }
    // warp-aggregated append (warpenqueuefrontier pattern)
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && total) base = atomicAdd(&G.ctrl->export_n, (unsigned long long)total);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    uint64_t o = base + incl - cnt;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t key = F::key(d, k);
      if (own != NO_OWNER && F::valid_cell(l8, k) && key != EMPTY_KEY && key != TOMBSTONE_KEY) {
        if (o < cap) { os[o] = g_global(G, own); od[o] = key; if (ow) ow[o] = MAP ? F::weight(d, k) : 0u; }
        o++;
      }
    }
  }
}

// ------------------------------------------------------------------ construction

__global__ void k_bucket_counts(const uint32_t* __restrict__ hints, uint32_t V, double lf_cap, int hashing,
                                uint32_t cap, uint32_t* __restrict__ count, uint64_t* __restrict__ heads,
                                unsigned long long* __restrict__ total) {
  unsigned long long mine = 0, full = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (V + stride - 1) / stride;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + t * stride;
    if (v >= V) continue;
    const uint32_t hint = hints ? hints[v] : 1u;   // no hints: one bucket per vertex
    uint32_t c = 1;
    if (hashing && hint > 0) {
      const double q = ceil((double)hint / lf_cap);   // ceil(hint / (lf * capacity))
      c = q < 1.0 ? 1u : (q > 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)q);
    }
    count[v] = c;
    heads[v] = hint > 0 ? c : 0;   // hint 0: no arena head, allocated lazily on first insert (C22b)
    mine += c;
    full += (hint + cap - 1) / cap;   // slabs the hinted degree fills at 100% occupancy
  }
  for (int o = 16; o; o >>= 1) {
    mine += __shfl_down_sync(0xFFFFFFFFu, mine, o);
    full += __shfl_down_sync(0xFFFFFFFFu, full, o);
  }
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, mine);
  if ((threadIdx.x & 31) == 0 && full) atomicAdd(total + 1, full);
}

__global__ void k_init_meta(GraphDev G, const uint32_t* __restrict__ count, const uint64_t* __restrict__ first,
                            const uint64_t* __restrict__ heads) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < G.V; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t h = heads[v], f = first[v];
    G.vmeta[v] = make_uint2(h ? (uint32_t)f : INVALID_SLAB, count[v]);
    for (uint64_t i = 0; i < h; i++) G.owner[f + i] = (uint32_t)v;
  }
}

__global__ void k_fill(uint32_t* __restrict__ slabs, uint64_t n_slabs, int map) {
  const uint64_t n16 = n_slabs * (SLAB_WORDS / 4);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    const int w0 = (int)(i & 7) * 4;
    uint4 f;
    f.x = fill_word(map, w0); f.y = fill_word(map, w0 + 1); f.z = fill_word(map, w0 + 2); f.w = fill_word(map, w0 + 3);
    reinterpret_cast<uint4*>(slabs)[i] = f;
  }
}

// ------------------------------------------------------------------ degree table (on demand)

// deg[u] = live keys of u's slab lists, by one address-order stream of the slab array [0, H + pool
// used): an 8-lane group per slab counts its live cells, one atomicAdd per slab with any (owner[]
// names the row).  Launched only by consumers of the table (PageRank's out[u], triangle counting's
// walked-side choice) when the graph changed since the last count, so the update kernels carry no
// per-edge degree atomics.
template <bool MAP>
__global__ void __launch_bounds__(UPD_BLOCK) k_degrees(GraphDev G) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const int l8 = lane_id() & 7, gbase = lane_id() & 24;
  const uint32_t gmask = 0xFFu << gbase;
  const uint64_t n_slabs = G.H + min((unsigned long long)G.P, __ldcg(&G.ctrl->pool_top));
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  for (uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; s < n_slabs; s += ng) {
    const uint32_t own = __ldg(G.owner + s);   // group-uniform
    if (own == NO_OWNER) continue;
    const uint4 d = ld_slab_ro(slab_ptr(G, (uint32_t)s), l8);
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t key = F::key(d, k);
      cnt += F::valid_cell(l8, k) && key < G.Vg;
    }
    cnt = __reduce_add_sync(gmask, cnt);
    if (l8 == 0 && cnt) atomicAdd(G.deg + own, cnt);
  }
}

// ------------------------------------------------------------------ consistency check (fsck)

// One thread per vertex walks every slab list of the vertex and checks the store's
// structural invariants: each slab's owner is the vertex, next pointers are INVALID
// or pool slabs, no LINKING lock survives a kernel, chains are finite, and no slab
// follows a slab that still has an EMPTY cell (EMPTY-suffix invariant, §4.2).
// info[0] = violations, info[1..4] = first violation (vertex, slab, next, kind).
template <bool MAP>
__global__ void k_fsck(GraphDev G, unsigned long long* info) {
  using F = Frag<MAP>;
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < G.V; u += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 m = G.vmeta[u];
    if (m.x == INVALID_SLAB) continue;   // no slab list yet: no edges
    int kind = 0;
    uint32_t bad_s = 0, bad_n = 0;
    if (m.x == LINKING) { kind = 1; }
    for (uint32_t b = 0; b < m.y && !kind; b++) {
      uint32_t s = m.x + b, steps = 0;
      while (!kind) {
        if (s >= G.H + G.P) { kind = 2; bad_s = s; break; }
        if (G.owner[s] != (uint32_t)u) { kind = 3; bad_s = s; break; }
        const uint32_t* p = slab_ptr(G, s);
        bool has_empty = false;
        for (int w = 0; w < SLAB_WORDS - 1; w++) {
          const bool keyword = MAP ? ((w & 1) == 0 && w < 30) : true;
          if (keyword && p[w] == EMPTY_KEY) has_empty = true;
        }
        const uint32_t nx = p[SLAB_WORDS - 1];
        if (nx == INVALID_SLAB) break;
        if (nx == LINKING) { kind = 4; bad_s = s; bad_n = nx; break; }
        if (nx < G.H || nx >= G.H + G.P) { kind = 5; bad_s = s; bad_n = nx; break; }
        if (has_empty) { kind = 6; bad_s = s; bad_n = nx; break; }
        if (++steps > (1u << 24)) { kind = 7; bad_s = s; break; }
        s = nx;
      }
    }
    if (kind) {
      const unsigned long long k = atomicAdd(&info[0], 1ull);
      if (k == 0) { info[1] = u; info[2] = bad_s; info[3] = bad_n; info[4] = kind; }
    }
  }
}

// ------------------------------------------------------------------ host launchers

// One work item per group up to `per_group_cap` waves of resident blocks: blocks retire
// independently, so a block held up by a contended slab list (hub rows of an R-MAT batch)
// does not make the rest of the GPU wait at a grid-wide tail.
static uint64_t g_upd_waves = 0;   // MEERKAT_UPD_WAVES (experiments); 0 = default

static inline unsigned grid_for(meerkat_graph* g, uint64_t groups, uint64_t waves = 1) {
  if (waves != 1 && g_upd_waves == 0) {
    const char* e = std::getenv("MEERKAT_UPD_WAVES");
    g_upd_waves = e ? std::strtoull(e, nullptr, 10) : 1;
  }
  if (waves != 1) waves = g_upd_waves ? g_upd_waves : 1;
  const uint64_t per_block = UPD_BLOCK / GROUP;
  uint64_t b = (groups + per_block - 1) / per_block;
  const uint64_t cap = (uint64_t)g->sm_count * 8 * waves;   // 8 resident 256-thread blocks per SM
  if (b > cap) b = cap;
  return (unsigned)(b ? b : 1);
}

cudaError_t launch_build(meerkat_graph* g, Store& st, const uint32_t* d_hints, uint64_t pool_request) {
  const uint32_t V = g->Vl;   // vertices held by this partition (all of them when world_size == 1)
  const int cap = g->weighted ? MAP_CAP : SET_CAP;
  uint32_t* count = nullptr;
  uint64_t *heads = nullptr, *first = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
#define CK(x) do { e = (x); if (e != cudaSuccess) goto out; } while (0)
  CK(cudaMalloc(&count, (size_t)V * 4));
  CK(cudaMalloc(&heads, (size_t)V * 8));
  CK(cudaMalloc(&first, ((size_t)V + 3) * 8));
  {
    const unsigned gb = (unsigned)std::min<uint64_t>((V + 255) / 256, (uint64_t)g->sm_count * 16);
    unsigned long long* total = reinterpret_cast<unsigned long long*>(first + V + 1);
    CK(cudaMemsetAsync(total, 0, 16, g->stream));
    k_bucket_counts<<<gb, 256, 0, g->stream>>>(d_hints, V, (double)(&st == &g->in ? g->lf_in : g->lf) * cap, g->hashing ? 1 : 0, (uint32_t)cap,
                                               count, heads, total);
    g->launches++;
    CK(cudaGetLastError());
    CK(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, heads, first + 1, V, g->stream));
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cudaMemsetAsync(first, 0, 8, g->stream));
    CK(cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, heads, first + 1, V, g->stream));   // first = exclusive scan
    g->launches++;
    uint64_t HB[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(HB, first + V, 24, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    const uint64_t H = HB[0];
    st.buckets = HB[1];
    const uint64_t full = HB[2];
    // total slab lists = arena heads + one lazy head per hint-0 vertex
    st.H = H;
    // automatic pool: chains for the hinted degrees beyond the heads (x2: chains are partly empty),
    // plus room to grow by half the arena, lazy heads for an eighth of the vertices, and a floor
    const uint64_t overflow = full > H ? full - H : 0;
    st.P = pool_request ? pool_request : 2 * overflow + H / 2 + V / 8 + 65536;
    if (st.H + st.P >= 0xFFFFFFF0ull) { e = cudaErrorInvalidValue; goto out; }
    const size_t nslab = (size_t)(st.H + st.P);
    CK(cudaMalloc(&st.dev.slabs, nslab * 128));             // ONE allocation: head arena + pool
    CK(cudaMalloc(&st.dev.owner, nslab * 4));
    CK(cudaMalloc(&st.dev.vmeta, (size_t)V * 8));
    CK(cudaMalloc(&st.dev.deg, (size_t)V * 4));
    CK(cudaMemsetAsync(st.dev.deg, 0, (size_t)V * 4, g->stream));
    CK(cudaMalloc(&st.dev.ctrl, sizeof(GraphCtrl)));
    CK(cudaMemsetAsync(st.dev.ctrl, 0, sizeof(GraphCtrl), g->stream));
    CK(cudaMallocHost(&st.hctrl, sizeof(GraphCtrl)));
    memset(st.hctrl, 0, sizeof(GraphCtrl));
    st.bytes = nslab * 132 + (size_t)V * 12 + sizeof(GraphCtrl);
    st.dev.V = V; st.dev.H = (uint32_t)st.H; st.dev.P = (uint32_t)st.P;
    st.dev.Vg = g->V; st.dev.ws = g->ws; st.dev.rank = g->rank; st.dev.pbits = pm_bits(g->V);
    if (st.H) {
      const unsigned gf = (unsigned)std::min<uint64_t>((st.H * 8 + 255) / 256, (uint64_t)g->sm_count * 16);
      k_fill<<<gf, 256, 0, g->stream>>>(st.dev.slabs, st.H, g->weighted ? 1 : 0);
      g->launches++;
    }
    k_init_meta<<<gb, 256, 0, g->stream>>>(st.dev, count, first, heads);
    g->launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g->stream));
  }
out:
#undef CK
  cudaFree(count); cudaFree(heads); cudaFree(first); cudaFree(tmp);
  return e;
}

#define UPD_LAUNCH(K, grid_, A_) do { K<<<grid_, UPD_BLOCK, 0, g->stream>>>(A_); } while (0)

template <bool MAP, bool TRACK>
static void insert_kind(meerkat_graph* g, const UpdArgs& A, bool thread, unsigned grid) {
  if (thread) {
    if (A.ntrees) UPD_LAUNCH((k_insert_t<MAP, TRACK, 1>), grid, A);
    else UPD_LAUNCH((k_insert_t<MAP, TRACK, 0>), grid, A);
  } else {
    if (A.ntrees) UPD_LAUNCH((k_insert<MAP, TRACK, 1>), grid, A);
    else UPD_LAUNCH((k_insert<MAP, TRACK, 0>), grid, A);
  }
}

template <bool MAP>
static void delete_kind(meerkat_graph* g, const UpdArgs& A, bool thread, unsigned grid) {
  if (thread) {
    if (A.ntrees) UPD_LAUNCH((k_delete_t<MAP, 2>), grid, A);
    else UPD_LAUNCH((k_delete_t<MAP, 0>), grid, A);
  } else {
    if (A.ntrees) UPD_LAUNCH((k_delete<MAP, 2>), grid, A);
    else UPD_LAUNCH((k_delete<MAP, 0>), grid, A);
  }
}
#undef UPD_LAUNCH

static void set_pro(meerkat_graph* g, UpdArgs& A, const TreePro* pro) {
  A.ntrees = pro ? pro->ntrees : 0u;
  // a tree of g that this mutation does not seed may follow with an unseeded call, which checks the
  // batch against the fingerprint; if every dynamic tree is seeded, no call reads the batch
  A.fp_on = (!pro || (uint64_t)pro->ntrees < g->n_trees) ? 1u : 0u;
  if (pro)
    for (int k = 0; k < MAX_TREES; k++) A.T[k] = pro->T[k];
}

cudaError_t launch_insert(meerkat_graph* g, Store* st0, Store* st1, const uint32_t* s, const uint32_t* d,
                          const uint32_t* w, uint64_t n, const TreePro* pro) {
  if (!n) return cudaSuccess;
  UpdArgs A{};
  A.G[0] = st0->dev;
  if (st1) A.G[1] = st1->dev;
  A.src = s; A.dst = d; A.w = w; A.n = n; A.ns = st1 ? 2u : 1u;
  A.fp_slot = (uint32_t)((g->version + 1) & 1);   // the version this mutation creates
  set_pro(g, A, pro);
  const bool thread = thread_upd(n * A.ns);
  const unsigned grid = thread ? grid_threads(g, n * A.ns) : grid_for(g, n * A.ns, 0);
  if (A.G[0].upd) {
    if (g->weighted) insert_kind<true, true>(g, A, thread, grid);
    else insert_kind<false, true>(g, A, thread, grid);
  } else {
    if (g->weighted) insert_kind<true, false>(g, A, thread, grid);
    else insert_kind<false, false>(g, A, thread, grid);
  }
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_delete(meerkat_graph* g, Store* st0, Store* st1, const uint32_t* s, const uint32_t* d, uint64_t n,
                          const TreePro* pro) {
  if (!n) return cudaSuccess;
  UpdArgs A{};
  A.G[0] = st0->dev;
  if (st1) A.G[1] = st1->dev;
  A.src = s; A.dst = d; A.w = nullptr; A.n = n; A.ns = st1 ? 2u : 1u;
  A.fp_slot = (uint32_t)((g->version + 1) & 1);   // the version this mutation creates
  set_pro(g, A, pro);
  const bool thread = thread_upd(n * A.ns);
  const unsigned grid = thread ? grid_threads(g, n * A.ns) : grid_for(g, n * A.ns, 0);
  if (g->weighted) delete_kind<true>(g, A, thread, grid);
  else delete_kind<false>(g, A, thread, grid);
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_query(meerkat_graph* g, Store& st, const uint32_t* s, const uint32_t* d, uint64_t n, uint8_t* found,
                         uint32_t* w_out) {
  if (!n) return cudaSuccess;
  if (thread_upd(n)) {
    const unsigned gt = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + UPD_BLOCK - 1) / UPD_BLOCK,
                                                                         (uint64_t)g->sm_count * 8));
    if (g->weighted) k_query_t<true><<<gt, UPD_BLOCK, 0, g->stream>>>(st.dev, s, d, n, found, w_out);
    else k_query_t<false><<<gt, UPD_BLOCK, 0, g->stream>>>(st.dev, s, d, n, found, w_out);
    g->launches++;
    return cudaGetLastError();
  }
  const unsigned gb = grid_for(g, n, 0);
  if (g->weighted) k_query<true><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev, s, d, n, found, w_out);
  else k_query<false><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev, s, d, n, found, w_out);
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_degrees(meerkat_graph* g, Store& st) {
  if (st.deg_version == g->version) return cudaSuccess;   // the table is current
  cudaError_t e = cudaMemsetAsync(st.dev.deg, 0, (size_t)st.dev.V * 4, g->stream);
  if (e != cudaSuccess) return e;
  const unsigned gb = grid_for(g, st.H + st.P);
  if (g->weighted) k_degrees<true><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev);
  else k_degrees<false><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev);
  g->launches++;
  e = cudaGetLastError();
  if (e == cudaSuccess) st.deg_version = g->version;
  return e;
}

cudaError_t launch_fsck(meerkat_graph* g, Store& st, unsigned long long* info_dev) {
  cudaError_t e = cudaMemsetAsync(info_dev, 0, 5 * 8, g->stream);
  if (e != cudaSuccess) return e;
  const unsigned gb = (unsigned)std::min<uint64_t>((st.dev.V + 255) / 256, (uint64_t)g->sm_count * 16);
  if (g->weighted) k_fsck<true><<<std::max(gb, 1u), 256, 0, g->stream>>>(st.dev, info_dev);
  else k_fsck<false><<<std::max(gb, 1u), 256, 0, g->stream>>>(st.dev, info_dev);
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_export(meerkat_graph* g, Store& st, uint32_t* s, uint32_t* d, uint32_t* w, uint64_t cap) {
  cudaError_t e = cudaMemsetAsync(&st.dev.ctrl->export_n, 0, 8, g->stream);
  if (e != cudaSuccess) return e;
  // slabs in use: arena + pool handed out so far (read on the host: export synchronises anyway)
  e = cudaMemcpyAsync(st.hctrl, st.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return e;
  const uint64_t used = std::min<uint64_t>(st.hctrl->pool_top, st.P);
  const uint64_t n_slabs = st.H + used;
  if (!n_slabs) return cudaSuccess;
  const unsigned gb = grid_for(g, n_slabs);
  if (g->weighted) k_export<true><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev, n_slabs, s, d, w, cap);
  else k_export<false><<<gb, UPD_BLOCK, 0, g->stream>>>(st.dev, n_slabs, s, d, w, cap);
  g->launches++;
  return cudaGetLastError();
}

void free_store(Store& st) {
  cudaFree(st.dev.slabs);
  cudaFree(st.dev.owner);
  cudaFree(st.dev.vmeta);
  cudaFree(st.dev.deg);
  cudaFree(st.dev.upd);
  cudaFree(st.dev.updq);
  cudaFree(st.dev.ctrl);
  if (st.hctrl) cudaFreeHost(st.hctrl);
  st = Store{};
}

}  // namespace mk
