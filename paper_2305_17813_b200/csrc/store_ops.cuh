// store_ops.cuh — per-thread slab-store operations (whole-slab reads by one thread) and block
// reductions used by the update kernels (store.cu).  Protocols: search-then-claim insert, link lock for new
// slabs ("chained at the end of the last filled slab"), TOMBSTONE delete.
#pragma once
#include "graph.h"

namespace mk {

constexpr uint32_t WATCHDOG = 1u << 20;   // loop bounds that turn a would-be hang into MEERKAT_E_STATE
constexpr uint32_t WALK_LIMIT = 1u << 26;  // slabs walked by one operation (a chain longer than any pool)

__device__ __forceinline__ uint32_t fill_word(bool map, int word) {
  if (word == SLAB_WORDS - 1) return INVALID_SLAB;
  if (map) return (word & 1) ? 0xFFFFFFFFu : EMPTY_KEY;   // pair = UINT64_MAX-1 (P:1504 footnote)
  return EMPTY_KEY;
}

// Block-aggregated add of a per-thread count into two global counters (one atomic each per block).
__device__ __forceinline__ void block_add(unsigned long long* d0, unsigned long long* d1, uint32_t v) {
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  v = __reduce_add_sync(0xFFFFFFFFu, v);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(&acc, (unsigned long long)v);
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long a = acc;
    if (a) { atomicAdd(d0, a); atomicAdd(d1, a); }
  }
  __syncthreads();   // acc is reused by the next call (racecheck: no read may trail its reset)
}

// Two per-store values of an update kernel (out store, in-edge mirror) kept in registers: a
// runtime-indexed [2] array would live in local memory.
struct PerStore {
  uint32_t v0 = 0, v1 = 0;
  __device__ __forceinline__ void add(uint32_t st, uint32_t x) { if (st) v1 += x; else v0 += x; }
  __device__ __forceinline__ void set(uint32_t st, uint32_t x) { if (st) v1 |= x; else v0 |= x; }
  __device__ __forceinline__ uint32_t get(int k) const { return k ? v1 : v0; }
};

__device__ __forceinline__ void block_or_err(unsigned int* dst, uint32_t e) {
  e = __reduce_or_sync(0xFFFFFFFFu, e);
  if ((threadIdx.x & 31) == 0 && e) atomicOr(dst, e);
}

template <bool MAP>
__device__ __forceinline__ void thread_read_slab(const GraphDev& G, uint32_t s, uint4 (&q)[8]) {
  const uint4* p = reinterpret_cast<const uint4*>(slab_ptr(G, s));
#pragma unroll
  for (int j = 0; j < 8; j++) q[j] = __ldcg(p + j);
}

template <bool MAP>
__device__ uint32_t thread_alloc(const GraphDev& G, uint32_t u, uint64_t first) {
  const unsigned long long idx = atomicAdd(&G.ctrl->pool_top, 1ull);
  if (idx >= G.P) return INVALID_SLAB;
  const uint32_t s = G.H + (uint32_t)idx;
  uint4* p = reinterpret_cast<uint4*>(slab_ptr(G, s));
#pragma unroll
  for (int j = 0; j < 8; j++) {
    uint4 f;
    f.x = fill_word(MAP, 4 * j + 0); f.y = fill_word(MAP, 4 * j + 1);
    f.z = fill_word(MAP, 4 * j + 2); f.w = fill_word(MAP, 4 * j + 3);
    if (j == 0) { f.x = (uint32_t)first; if (MAP) f.y = (uint32_t)(first >> 32); }
    p[j] = f;
  }
  G.owner[s] = u;
  __threadfence();
  return s;
}

// Link lock (see group_link): 1 = our slab holding the key is linked, -1 = pool exhausted,
// 0 = another thread linked first (*next_out = its slab or INVALID_SLAB).
template <bool MAP>
__device__ int thread_link(const GraphDev& G, uint32_t u, uint64_t item, uint32_t* link, uint32_t& next_out) {
  uint32_t old = atomicCAS(link, INVALID_SLAB, LINKING);
  if (old == INVALID_SLAB) {
    const uint32_t s = thread_alloc<MAP>(G, u, item);
    atomicExch(link, s);   // INVALID_SLAB releases the lock
    next_out = s;   // the caller's key sits in cell 0 of this slab
    return s == INVALID_SLAB ? -1 : 1;
  }
  uint32_t spins = 0;
  while (old == LINKING) {
    __nanosleep(64);
    old = *reinterpret_cast<volatile uint32_t*>(link);
    if (++spins == WATCHDOG) { atomicOr(&G.ctrl->err, (unsigned)ERR_STATE); return -1; }
  }
  next_out = old;
  return 0;
}

// UpdateIterator bookkeeping: remember the earliest cell written in the slab list
// since the last reset; the first write to a list queues it.  Chain order is slab-index order
// (pool slabs are handed out in increasing order), so the minimum position is the earliest.
__device__ __forceinline__ void track_update(const GraphDev& G, uint32_t list, unsigned long long pos) {
  const unsigned long long old = atomicMin(G.upd + list, pos);
  if (old == ~0ull) G.updq[atomicAdd(&G.ctrl->upd_n, 1ull)] = list;
}

template <bool MAP>
__device__ int thread_insert(const GraphDev& G, uint32_t u, uint32_t v, uint32_t wt, uint32_t& pos_list,
                             unsigned long long& pos) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const uint64_t item = MAP ? (((uint64_t)wt << 32) | v) : (uint64_t)v;
  const uint2 m = __ldcg(G.vmeta + u);
  uint32_t head = m.x;
  while (head == INVALID_SLAB || head == LINKING) {   // lazily headed vertex (C22b)
    uint32_t nxt = INVALID_SLAB;
    const int r = thread_link<MAP>(G, u, item, reinterpret_cast<uint32_t*>(&G.vmeta[u].x), nxt);
    if (r == 1) { pos_list = nxt; pos = (unsigned long long)nxt << 5; }
    if (r != 0) return r;
    head = nxt;
  }
  uint32_t cur = head + bucket_of(v, m.y, G.seed);
  const uint32_t list0 = cur;
  for (uint32_t guard = 0; guard < WATCHDOG; guard++) {
    // pass 1: up to the first slab holding an EMPTY cell; first writable cell remembered
    uint32_t s = cur, cand_slab = INVALID_SLAB, tail = INVALID_SLAB, found_slab = INVALID_SLAB;
    int cand_cell = -1, found_cell = -1;
    uint64_t cand_old = 0;
    for (uint32_t walk = 0; walk < WALK_LIMIT; walk++) {
      uint4 q[8];
      thread_read_slab<MAP>(G, s, q);
      bool empty = false;
#pragma unroll
      for (int j = 0; j < 8; j++) {
#pragma unroll
        for (int k = 0; k < NK; k++) {
          if (!F::valid_cell(j, k)) continue;
          const uint32_t key = F::key(q[j], k);
          const int c = j * NK + k;
          if (key == v && found_cell < 0) found_cell = c;
          if ((key == EMPTY_KEY || key == TOMBSTONE_KEY) && cand_slab == INVALID_SLAB && cand_cell < 0) {
            cand_cell = c;
            cand_old = MAP ? (((uint64_t)F::weight(q[j], k) << 32) | key) : (uint64_t)key;
          }
          empty |= key == EMPTY_KEY;
        }
      }
      if (cand_cell >= 0 && cand_slab == INVALID_SLAB) cand_slab = s;
      if (found_cell >= 0) { found_slab = s; break; }
      const uint32_t nxt = q[7].w;
      if (empty || nxt == INVALID_SLAB || nxt == LINKING) { tail = s; break; }
      if (nxt >= G.H + G.P) { atomicOr(&G.ctrl->err, (unsigned)ERR_STATE); return -1; }
      s = nxt;
    }
    if (found_cell >= 0) {   // present: min-weight upsert (C8)
      if (MAP) atomicMin(reinterpret_cast<unsigned long long*>(slab_ptr(G, found_slab) + 2 * found_cell),
                         (unsigned long long)item);
      return 0;
    }
    if (cand_slab != INVALID_SLAB) {   // pass 2: claim
      bool ok;
      if (MAP) {
        unsigned long long* cell = reinterpret_cast<unsigned long long*>(slab_ptr(G, cand_slab) + 2 * cand_cell);
        ok = atomicCAS(cell, (unsigned long long)cand_old, (unsigned long long)item) == cand_old;
      } else {
        ok = atomicCAS(slab_ptr(G, cand_slab) + cand_cell, (unsigned int)cand_old, (unsigned int)item) ==
             (unsigned int)cand_old;
      }
      if (ok) { pos_list = list0; pos = ((unsigned long long)cand_slab << 5) | (uint32_t)cand_cell; return 1; }
      cur = cand_slab;   // the cell changed: rescan from its slab
      continue;
    }
    if (tail == INVALID_SLAB) { atomicOr(&G.ctrl->err, (unsigned)ERR_STATE); return -1; }
    uint32_t nxt = INVALID_SLAB;   // full list: link a pool slab holding the key after the tail
    const int r = thread_link<MAP>(G, u, item, slab_ptr(G, tail) + (SLAB_WORDS - 1), nxt);
    if (r == 1) { pos_list = list0; pos = (unsigned long long)nxt << 5; }
    if (r != 0) return r;
    cur = nxt == INVALID_SLAB ? tail : nxt;
  }
  atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
  return -1;
}

template <bool MAP>
__device__ bool thread_delete(const GraphDev& G, uint32_t u, uint32_t v) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const uint2 m = __ldcg(G.vmeta + u);
  if (m.x == INVALID_SLAB || m.x == LINKING) return false;
  uint32_t s = m.x + bucket_of(v, m.y, G.seed);
  for (uint32_t walk = 0; walk < WALK_LIMIT; walk++) {
    uint4 q[8];
    thread_read_slab<MAP>(G, s, q);
    bool empty = false;
    int fc = -1;
    uint64_t val = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
#pragma unroll
      for (int k = 0; k < NK; k++) {
        if (!F::valid_cell(j, k)) continue;
        const uint32_t key = F::key(q[j], k);
        if (key == v && fc < 0) { fc = j * NK + k; val = MAP ? (((uint64_t)F::weight(q[j], k) << 32) | key) : key; }
        empty |= key == EMPTY_KEY;
      }
    }
    if (fc >= 0) {   // TOMBSTONE; a failed CAS means a duplicate in this batch won
      if (MAP) return atomicCAS(reinterpret_cast<unsigned long long*>(slab_ptr(G, s) + 2 * fc),
                                (unsigned long long)val, (unsigned long long)TOMB_PAIR) == val;
      return atomicCAS(slab_ptr(G, s) + fc, (unsigned int)val, TOMBSTONE_KEY) == (unsigned int)val;
    }
    const uint32_t nxt = q[7].w;
    if (empty || nxt == INVALID_SLAB || nxt >= G.H + G.P) return false;
    s = nxt;
  }
  return false;
}

}  // namespace mk
