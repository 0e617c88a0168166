// dtree.cu — vertex-partitioned (multi-GPU) SSSP / BFS phases, SURVEY §8(e).
//
// Rank r holds the out-edges and the tree nodes of every vertex v with
// v % world_size == r (local row v / world_size).  A tree update is the
// single-GPU method run as lock-step PHASES on every rank:
// an expansion relaxes edges into vertices held here directly and turns every
// relaxation of a vertex held elsewhere into a message <x, packed candidate>
// (or, while propagating invalidation, <x, expected parent>); the caller moves
// the messages with one all-to-all per round (NCCL over NVLink) and the owner
// applies them with the same packed atomicMin / CAS.  The fixpoint does not
// depend on the order of relaxations, so results are
// bit-identical to world_size 1.  Frontier rounds are host-driven here because
// every round carries an exchange.
#include <algorithm>
#include <cstring>

#include "tree_common.cuh"

namespace mk {

constexpr int D_BLOCK = 256;

struct DArgs {
  GraphDev G;
  TreeDev T;
  uint64_t* msgs;               // raw outgoing pairs (x, payload), 2 u64 each
  unsigned long long* msg_n;    // raw pair count
  uint64_t msg_cap;             // pairs
  const uint64_t* fr;           // frontier being expanded (local rows)
  const unsigned long long* n_ptr;   // its size (device: the previous phases may still be in flight)
  uint64_t* fnext;
  unsigned long long* sznext;
  uint32_t epoch;               // stamp epoch of fnext
  uint32_t unit;
};

__device__ __forceinline__ bool owned(const GraphDev& G, uint32_t x) { return x % G.ws == G.rank; }
__device__ __forceinline__ uint32_t lrow(const GraphDev& G, uint32_t x) { return x / G.ws; }
__device__ __forceinline__ uint32_t grow(const GraphDev& G, uint32_t l) { return l * G.ws + G.rank; }

// Warp-aggregated append of messages (same pattern as warpenqueuefrontier).
__device__ __forceinline__ void warp_emit(const DArgs& A, bool has, uint32_t x, uint64_t payload, Counters& c) {
  const uint32_t m = __ballot_sync(FULL, has);
  if (!m) return;
  const int lane = lane_id();
  unsigned long long base = 0;
  const int leader = __ffs(m) - 1;
  if (lane == leader) base = atomicAdd(A.msg_n, (unsigned long long)__popc(m));
  base = __shfl_sync(FULL, base, leader);
  if (has) {
    const uint64_t p = base + __popc(m & ((1u << lane) - 1));
    if (p < A.msg_cap) { A.msgs[2 * p] = x; A.msgs[2 * p + 1] = payload; }
    else c.err |= ERR_CAPACITY;
  }
}

// relax() with an already packed candidate (received message)
__device__ __forceinline__ bool relax_packed(const TreeDev& T, uint32_t lx, uint64_t cand, uint32_t epoch,
                                             Counters& c) {
  if (cand >= ld_cg_u64(T.node + lx)) return false;
  const unsigned long long old = atomicMin(reinterpret_cast<unsigned long long*>(T.node + lx), cand);
  if (cand >= old) return false;
  c.improved++;
  return atomicExch(T.stamp + lx, epoch) != epoch;
}

__global__ void k_dinit(DArgs A) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < A.G.V; l += (uint64_t)gridDim.x * blockDim.x)
    A.T.node[l] = (grow(A.G, (uint32_t)l) == A.T.source) ? (uint64_t)A.T.source : UNREACHED;
}

__global__ void k_dseed_source(DArgs A) {   // one warp: frontier = {SRC} on its owner (C16)
  Counters c;
  const bool has = threadIdx.x == 0 && owned(A.G, A.T.source);
  const uint32_t l = lrow(A.G, A.T.source);
  if (has) A.T.stamp[l] = A.epoch;
  warp_enqueue(A.G, A.T, A.fnext, A.sznext, has, l, c);
}

// Incremental prologue: batch edges (u, v, w) with u held here.
__global__ void __launch_bounds__(D_BLOCK) k_dinc_seed(DArgs A, const uint32_t* bs, const uint32_t* bd,
                                                       const uint32_t* bw, uint64_t bn) {
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    bool enq = false, emit = false;
    uint32_t v = 0, lv = 0;
    uint64_t cand = 0;
    if (i < bn) {
      const uint32_t u = bs[i];
      v = bd[i];
      const uint32_t w = A.unit ? 1u : bw[i];
      c.batch++;
      if (u < A.G.Vg && v < A.G.Vg && (A.unit || (w != 0 && w < W_LIMIT))) {
        if (!owned(A.G, u)) c.err |= ERR_PARTITION;
        else {
          const uint64_t nu = ld_cg_u64(A.T.node + lrow(A.G, u));
          if (nu != UNREACHED) {
            const uint64_t dist = (nu >> 32) + w;
            if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
            else if (owned(A.G, v)) { lv = lrow(A.G, v); enq = relax(A.T, lv, dist, u, A.epoch, c); }
            else { emit = true; cand = (dist << 32) | u; }
          }
        }
      }
    }
    warp_enqueue(A.G, A.T, A.fnext, A.sznext, enq, lv, c);
    warp_emit(A, emit, v, cand, c);
  }
  flush_counters(A.G, A.T, c, 0, false, 0, 0);
}

// Decremental Invalidate: deleted edges (u, v) with v held here.
__global__ void __launch_bounds__(D_BLOCK) k_ddec_inval(DArgs A, const uint32_t* bs, const uint32_t* bd, uint64_t bn) {
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    bool enq = false;
    uint32_t lv = 0;
    if (i < bn) {
      const uint32_t u = bs[i], v = bd[i];
      c.batch++;
      if (u < A.G.Vg && v < A.G.Vg && v != A.T.source) {
        if (!owned(A.G, v)) c.err |= ERR_PARTITION;
        else {
          lv = lrow(A.G, v);
          const uint64_t cur = ld_cg_u64(A.T.node + lv);
          if (cur != UNREACHED && (uint32_t)cur == u &&
              atomicCAS(reinterpret_cast<unsigned long long*>(A.T.node + lv), (unsigned long long)cur,
                        (unsigned long long)UNREACHED) == cur) {
            mark_invalid(A.T, v);
            atomicAdd(&A.T.ctrl->direct_n, 1ull);
            enq = true;
          }
        }
      }
    }
    warp_enqueue(A.G, A.T, A.fnext, A.sznext, enq, lv, c);
  }
  flush_counters(A.G, A.T, c, 0, false, 0, 0);
}

// One round of expansion of the local frontier (P:113-133 relax, or P:149-154 propagate).
template <bool MAP, int VISIT>
__global__ void __launch_bounds__(D_BLOCK) k_dexpand(DArgs A) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  Counters c;
  const GraphDev& G = A.G;
  const TreeDev& T = A.T;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  uint32_t v = 0, slab = 0, du = 0;
  const uint64_t n_cur = __ldcg(A.n_ptr);
  auto fetch = [&]() -> bool {
    for (; it < n_cur; it += ng) {
      const uint64_t item = A.fr[it];
      v = (uint32_t)item;
      if (l8 == 0) c.items++;
      slab = (uint32_t)(item >> 32);
      if (VISIT == PROPAGATE) return true;
      uint64_t nv = 0;
      if (l8 == 0) nv = ld_cg_u64(T.node + v);   // one read per group, broadcast (d(v) may change)
      nv = __shfl_sync(0xFFu << (lane & 24), nv, 0, GROUP);
      if (nv != UNREACHED) { du = (uint32_t)(nv >> 32); return true; }
    }
    return false;
  };
  bool active = fetch();
  while (__any_sync(FULL, active)) {
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    if (active) {
      d = ld_slab_ro(slab_ptr(G, slab), l8);
      if (l8 == 0) c.slabs++;
    }
    const uint32_t vg = grow(G, v);
#pragma unroll
    for (int k = 0; k < NK; k++) {
      const uint32_t x = F::key(d, k);
      const bool live = active && F::valid_cell(l8, k) && x < G.Vg;
      bool enq = false, emit = false;
      uint64_t payload = 0;
      uint32_t lx = 0;
      if (live) {
        c.visited++;
        if (VISIT == RELAX) {
          const uint64_t dist = (uint64_t)du + (A.unit ? 1u : F::weight(d, k));
          if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
          else if (owned(G, x)) { lx = lrow(G, x); enq = relax(T, lx, dist, vg, A.epoch, c); }
          else { emit = true; payload = (dist << 32) | vg; }
        } else {
          if (owned(G, x)) {
            lx = lrow(G, x);
            const uint64_t cur = ld_cg_u64(T.node + lx);
            if (cur != UNREACHED && (uint32_t)cur == vg && x != T.source &&
                atomicCAS(reinterpret_cast<unsigned long long*>(T.node + lx), (unsigned long long)cur,
                          (unsigned long long)UNREACHED) == cur) {
              mark_invalid(T, x);
              enq = true;
            }
          } else {
            emit = true;
            payload = vg;
          }
        }
      }
      warp_enqueue(G, T, A.fnext, A.sznext, enq, lx, c);
      warp_emit(A, emit, x, payload, c);
    }
    const uint32_t nxt = __shfl_sync(FULL, d.w, (lane & 24) + GROUP - 1);
    if (active) {
      if (nxt != INVALID_SLAB) slab = nxt;
      else { it += ng; active = fetch(); }
    }
  }
  flush_counters(A.G, A.T, c, 0, false, 0, 0);
}

// Apply received messages (x held here): relaxation candidates or invalidation requests.
template <int VISIT>
__global__ void __launch_bounds__(D_BLOCK) k_dapply(DArgs A, const uint64_t* in, uint64_t n_in) {
  Counters c;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (n_in + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    bool enq = false;
    uint32_t lx = 0;
    if (i < n_in) {
      const uint32_t x = (uint32_t)in[2 * i];
      const uint64_t p = in[2 * i + 1];
      if (x >= A.G.Vg || !owned(A.G, x)) c.err |= ERR_PARTITION;
      else {
        lx = lrow(A.G, x);
        if (VISIT == RELAX) {
          enq = relax_packed(A.T, lx, p, A.epoch, c);
        } else {
          const uint64_t cur = ld_cg_u64(A.T.node + lx);
          if (cur != UNREACHED && (uint32_t)cur == (uint32_t)p && x != A.T.source &&
              atomicCAS(reinterpret_cast<unsigned long long*>(A.T.node + lx), (unsigned long long)cur,
                        (unsigned long long)UNREACHED) == cur) {
            mark_invalid(A.T, x);
            enq = true;
          }
        }
      }
    }
    warp_enqueue(A.G, A.T, A.fnext, A.sznext, enq, lx, c);
  }
  flush_counters(A.G, A.T, c, 0, false, 0, 0);
}

// Set / clear the marks of ALL ranks' invalid vertices (global bit set).
__global__ void k_dmark(uint32_t* bits, const uint32_t* list, uint64_t n, int set) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = list[i];
    if (set) atomicOr(bits + (x >> 5), 1u << (x & 31));
    else atomicAnd(bits + (x >> 5), ~(1u << (x & 31)));
  }
}

// Valid->invalid frontier over this rank's slabs: stream + smem filter,
// as dec_scan in tree.cu, with relaxations of remote invalid vertices sent as messages.
// Up to two trees updated in lock step share ONE stream of the slab array (one filter of the
// union of their invalid sets; per key and tree the exact test, relax or message).
struct DScanArgs {
  DArgs A[2];
  const uint32_t* list[2];
  uint64_t n_inv[2];
  uint32_t ntrees;
};

template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, 2) k_dscan(const __grid_constant__ DScanArgs S, uint32_t fwords,
                                                         uint32_t n_slabs) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  constexpr int U = SCAN_UNROLL;
  extern __shared__ uint32_t filt[];
  Counters c;
  const GraphDev& G = S.A[0].G;
  if (fwords) {
    for (uint32_t i = threadIdx.x; i < fwords; i += blockDim.x) filt[i] = 0;
    __syncthreads();
    for (uint32_t j = 0; j < S.ntrees; j++)
      for (uint64_t i = threadIdx.x; i < S.n_inv[j]; i += blockDim.x) {
        uint32_t w, m;
        filter_loc(__ldg(S.list[j] + i), 32 - FILTER_LOG2, w, m);
        atomicOr(&filt[w], m);
      }
    __syncthreads();
  }
  const int l8 = lane_id() & 7;
  const uint32_t ng = (gridDim.x * blockDim.x) / GROUP;
  const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint32_t span = ng * U;
  const uint32_t trips = (n_slabs + span - 1) / span;
  const uint4* __restrict__ base = reinterpret_cast<const uint4*>(G.slabs) + l8;
  for (uint32_t t = 0; t < trips; t++) {
    const uint32_t s0 = t * span + g0;
    uint4 d[U];
#pragma unroll
    for (int q = 0; q < U; q++) {
      const uint32_t s = s0 + q * ng;
      d[q] = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
      if (s < n_slabs) d[q] = ld_slab_ro(reinterpret_cast<const uint32_t*>(base + (size_t)s * 8), 0);
    }
    uint32_t hm = 0;
#pragma unroll
    for (int q = 0; q < U; q++)
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t x = F::key(d[q], k);
        bool hit = x < G.Vg && (MAP || F::valid_cell(l8, k));
        if (fwords) {
          uint32_t w, m;
          filter_loc(x, 32 - FILTER_LOG2, w, m);
          hit = hit && (filt[w] & m) == m;
        }
        hm |= (uint32_t)hit << (q * NK + k);
      }
    const uint32_t pos = __reduce_or_sync(FULL, hm);
    if (!pos) continue;
#pragma unroll
    for (int q = 0; q < U; q++)
#pragma unroll
      for (int k = 0; k < NK; k++) {
        if (!((pos >> (q * NK + k)) & 1u)) continue;
        const uint32_t x = F::key(d[q], k);
#pragma unroll
        for (int j = 0; j < 2; j++) {
          if (j >= (int)S.ntrees) break;
          const DArgs& A = S.A[j];
          const TreeDev& T = A.T;
          bool enq = false, emit = false;
          uint32_t lx = 0;
          uint64_t payload = 0;
          if (((hm >> (q * NK + k)) & 1u) && bit_test(T.inval_bits, x)) {
            const uint32_t ul = __ldg(G.owner + s0 + q * ng);
            const uint32_t ug = ul == NO_OWNER ? NO_OWNER : grow(G, ul);
            if (ul != NO_OWNER && !bit_test(T.inval_bits, ug)) {
              const uint64_t nu = ld_cg_u64(T.node + ul);
              if (nu != UNREACHED) {
                c.hits[j]++;
                const uint64_t dist = (nu >> 32) + (A.unit ? 1u : F::weight(d[q], k));
                if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
                else if (owned(G, x)) { lx = lrow(G, x); enq = relax(T, lx, dist, ug, A.epoch, c); }
                else { emit = true; payload = (dist << 32) | ug; }
              }
            }
          }
          warp_enqueue(G, T, A.fnext, A.sznext, enq, lx, c);
          warp_emit(A, emit, x, payload, c);
        }
      }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c.scan_slabs = n_slabs;
  for (uint32_t j = 0; j < S.ntrees; j++) flush_counters(S.A[j].G, S.A[j].T, c, (int)j, false, 0, 0);
}

// ---- group messages by owner rank: histogram, exclusive scan, scatter
__global__ void k_msg_hist(const uint64_t* msgs, const unsigned long long* n_ptr, uint32_t ws,
                           unsigned long long* counts) {
  __shared__ unsigned int h[MEERKAT_MAX_RANKS];
  for (uint32_t i = threadIdx.x; i < ws; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t n = *n_ptr;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[(uint32_t)msgs[2 * i] % ws], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ws; i += blockDim.x)
    if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

__global__ void k_msg_scan(const unsigned long long* counts, uint32_t ws, unsigned long long* cursor) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long run = 0;
    for (uint32_t i = 0; i < ws; i++) { cursor[i] = run; run += counts[i]; }
  }
}

__global__ void k_msg_scatter(const uint64_t* msgs, const unsigned long long* n_ptr, uint32_t ws,
                              unsigned long long* cursor, uint64_t* out) {
  const uint64_t n = *n_ptr;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = msgs[2 * i];
    const unsigned long long p = atomicAdd(&cursor[(uint32_t)x % ws], 1ull);
    out[2 * p] = x;
    out[2 * p + 1] = msgs[2 * i + 1];
  }
}

// ---- batch routing by owner(key)
__global__ void k_route_hist(const uint32_t* key, uint64_t n, uint32_t ws, unsigned long long* counts) {
  __shared__ unsigned int h[MEERKAT_MAX_RANKS];
  for (uint32_t i = threadIdx.x; i < ws; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[key[i] % ws], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < ws; i += blockDim.x)
    if (h[i]) atomicAdd(&counts[i], (unsigned long long)h[i]);
}

__global__ void k_route_scatter(const uint32_t* a, const uint32_t* b, const uint32_t* c3, const uint32_t* key,
                                uint64_t n, uint32_t ws, unsigned long long* cursor, uint32_t* oa, uint32_t* ob,
                                uint32_t* oc) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long p = atomicAdd(&cursor[key[i] % ws], 1ull);
    oa[p] = a[i];
    ob[p] = b[i];
    if (c3) oc[p] = c3[i];
  }
}

// ------------------------------------------------------------------ host launchers

static unsigned dgrid(meerkat_graph* g, uint64_t threads) {
  uint64_t b = (threads + D_BLOCK - 1) / D_BLOCK;
  const uint64_t cap = (uint64_t)g->sm_count * 8;
  return (unsigned)std::max<uint64_t>(1, std::min(b, cap));
}

static void e_scan(meerkat_graph* g, const DScanArgs& S, uint32_t fwords, uint32_t n_slabs) {
  const size_t smem = (size_t)fwords * 4;
  const unsigned grid = (unsigned)(g->sm_count * std::max(1, g->tree_blocks_per_sm[2]));
  if (g->weighted) k_dscan<true><<<grid, TREE_BLOCK, smem, g->stream>>>(S, fwords, n_slabs);
  else k_dscan<false><<<grid, TREE_BLOCK, smem, g->stream>>>(S, fwords, n_slabs);
  g->launches++;
}

cudaError_t dlaunch(meerkat_graph* g, int kind, DArgs& A, const void* a, const void* b, const void* c, uint64_t n,
                    uint32_t fwords, uint32_t n_slabs) {
  cudaStream_t st = g->stream;
  const bool map = g->weighted;
  switch (kind) {
    case 0:   // init + seed source
      k_dinit<<<dgrid(g, A.G.V), D_BLOCK, 0, st>>>(A);
      k_dseed_source<<<1, 32, 0, st>>>(A);
      g->launches += 2;
      break;
    case 1:
      k_dinc_seed<<<dgrid(g, n), D_BLOCK, 0, st>>>(A, (const uint32_t*)a, (const uint32_t*)b, (const uint32_t*)c, n);
      g->launches++;
      break;
    case 2:
      k_ddec_inval<<<dgrid(g, n), D_BLOCK, 0, st>>>(A, (const uint32_t*)a, (const uint32_t*)b, n);
      g->launches++;
      break;
    case 3:
      if (map) k_dexpand<true, PROPAGATE><<<dgrid(g, n * GROUP), D_BLOCK, 0, st>>>(A);
      else k_dexpand<false, PROPAGATE><<<dgrid(g, n * GROUP), D_BLOCK, 0, st>>>(A);
      g->launches++;
      break;
    case 4:
      k_dapply<PROPAGATE><<<dgrid(g, n), D_BLOCK, 0, st>>>(A, (const uint64_t*)a, n);
      g->launches++;
      break;
    case 5: {
      DScanArgs S{};
      S.A[0] = A; S.A[1] = A;
      S.list[0] = (const uint32_t*)a; S.n_inv[0] = n;
      S.ntrees = 1;
      e_scan(g, S, fwords, n_slabs);
      break;
    }
    case 6:
      if (map) k_dexpand<true, RELAX><<<dgrid(g, n * GROUP), D_BLOCK, 0, st>>>(A);
      else k_dexpand<false, RELAX><<<dgrid(g, n * GROUP), D_BLOCK, 0, st>>>(A);
      g->launches++;
      break;
    case 7:
      k_dapply<RELAX><<<dgrid(g, n), D_BLOCK, 0, st>>>(A, (const uint64_t*)a, n);
      g->launches++;
      break;
    case 9:   // mark / clear: a = list, n, c != 0 means set
      k_dmark<<<dgrid(g, n), D_BLOCK, 0, st>>>(A.T.inval_bits, (const uint32_t*)a, n, c != nullptr);
      g->launches++;
      break;
  }
  return cudaGetLastError();
}

cudaError_t dsort_msgs(meerkat_graph* g, const uint64_t* raw, const unsigned long long* n_ptr, uint64_t n_bound,
                       unsigned long long* counts, unsigned long long* cursor, uint64_t* out) {
  cudaError_t e = cudaMemsetAsync(counts, 0, MEERKAT_MAX_RANKS * 8, g->stream);
  if (e != cudaSuccess || n_bound == 0) return e;
  const unsigned gb = dgrid(g, n_bound);   // grid-stride kernels read the exact count on the device
  k_msg_hist<<<gb, D_BLOCK, 0, g->stream>>>(raw, n_ptr, g->ws, counts);
  k_msg_scan<<<1, 32, 0, g->stream>>>(counts, g->ws, cursor);
  k_msg_scatter<<<gb, D_BLOCK, 0, g->stream>>>(raw, n_ptr, g->ws, cursor, out);
  g->launches += 3;
  return cudaGetLastError();
}

cudaError_t droute(meerkat_graph* g, const uint32_t* a, const uint32_t* b, const uint32_t* c, const uint32_t* key,
                   uint64_t n, uint32_t* oa, uint32_t* ob, uint32_t* oc, unsigned long long* counts,
                   unsigned long long* cursor) {
  cudaError_t e = cudaMemsetAsync(counts, 0, MEERKAT_MAX_RANKS * 8, g->stream);
  if (e != cudaSuccess || n == 0) return e;
  const unsigned gb = dgrid(g, n);
  k_route_hist<<<gb, D_BLOCK, 0, g->stream>>>(key, n, g->ws, counts);
  k_msg_scan<<<1, 32, 0, g->stream>>>(counts, g->ws, cursor);
  k_route_scatter<<<gb, D_BLOCK, 0, g->stream>>>(a, b, c, key, n, g->ws, cursor, oa, ob, oc);
  g->launches += 3;
  return cudaGetLastError();
}

cudaError_t dscan_attr(meerkat_graph* g) {
  const int smem = FILTER_WORDS * 4;
  cudaError_t e = cudaFuncSetAttribute(k_dscan<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_dscan<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return e;
}

}  // namespace mk

// ------------------------------------------------------------------ fused exchange packing

constexpr int MAX_SEGS = 2 * MEERKAT_MAX_RANKS;
struct Segs {
  const uint64_t* src[MAX_SEGS];   // message pairs (2 x u64 each)
  uint64_t* dst[MAX_SEGS];
  uint64_t start[MAX_SEGS + 1];    // exclusive prefix of the segment sizes (pairs)
  uint32_t n;
};

// Copy every segment's pairs (one launch for all trees and peers).
__global__ void k_copy_segs(const __grid_constant__ Segs S) {
  const uint64_t total = S.start[S.n];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = S.n;   // segment of pair i: last j with start[j] <= i
    while (hi - lo > 1) { const uint32_t mid = (lo + hi) / 2; if (S.start[mid] <= i) lo = mid; else hi = mid; }
    const uint64_t o = i - S.start[lo];
    const uint4 v = reinterpret_cast<const uint4*>(S.src[lo])[o];
    reinterpret_cast<uint4*>(S.dst[lo])[o] = v;
  }
}

// ------------------------------------------------------------------ host side of the phases

namespace mk {

static meerkat_status status_of(cudaError_t e) { return e == cudaSuccess ? MEERKAT_OK : MEERKAT_E_CUDA; }

static cudaError_t ensure_msgs(meerkat_graph* g, meerkat_tree* t, uint64_t need) {
  if (need <= t->msg_cap) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return e;
  cudaFree(t->msg_raw);
  cudaFree(t->msg_out);
  t->msg_raw = t->msg_out = nullptr;
  t->msg_cap = 0;
  const uint64_t cap = std::max<uint64_t>(need + need / 4, 1 << 16);
  e = cudaMalloc(&t->msg_raw, cap * 16);
  if (e == cudaSuccess) e = cudaMalloc(&t->msg_out, cap * 16);
  if (e == cudaSuccess) t->msg_cap = cap;
  return e;
}

// Messages of k trees for ONE all-to-all: per destination p, tree 0's pairs for p, tree 1's, ...
meerkat_status dtrees_pack(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, int64_t* meta, uint64_t* send,
                           uint64_t capacity_pairs, uint64_t* send_counts) {
  const uint32_t ws = g->ws;
  if (k == 0 || (uint64_t)ws * k > (uint64_t)MAX_SEGS) return MEERKAT_E_INVALID_ARG;
  cudaError_t e = cudaSuccess;
  if (!g->hmeta) e = cudaMallocHost(&g->hmeta, (size_t)MAX_SEGS * 3 * 8);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  Segs S{};
  uint64_t off[8][MEERKAT_MAX_RANKS];   // per tree, start of each destination's pairs in msg_out
  for (uint32_t i = 0; i < k; i++) {
    uint64_t o = 0;
    for (uint32_t p = 0; p < ws; p++) { off[i][p] = o; o += trees[i]->hcnt[p]; }
  }
  uint64_t total = 0;
  for (uint32_t p = 0; p < ws; p++) {
    uint64_t sp = 0;
    for (uint32_t i = 0; i < k; i++) {
      meerkat_tree* t = trees[i];
      uint64_t sent = 0;
      for (uint32_t q = 0; q < ws; q++) sent += t->hcnt[q];
      int64_t* row = g->hmeta + 3 * ((size_t)p * k + i);
      row[0] = (int64_t)t->hcnt[p];
      row[1] = (int64_t)t->last_front;
      row[2] = (int64_t)sent;
      const uint32_t j = S.n++;
      S.src[j] = t->msg_out + 2 * off[i][p];
      S.dst[j] = send + 2 * total;
      S.start[j] = total;
      total += t->hcnt[p];
      sp += t->hcnt[p];
    }
    send_counts[p] = sp;
  }
  S.start[S.n] = total;
  if (total > capacity_pairs) return MEERKAT_E_CAPACITY;
  e = cudaMemcpyAsync(meta, g->hmeta, (size_t)ws * k * 3 * 8, cudaMemcpyHostToDevice, g->stream);
  if (e == cudaSuccess && total) {
    k_copy_segs<<<dgrid(g, total), D_BLOCK, 0, g->stream>>>(S);
    g->launches++;
    e = cudaGetLastError();
  }
  return status_of(e);
}

// Received pairs (per source p, tree 0's rc[p*k], tree 1's rc[p*k+1], ...) into each tree's staging
// buffer (msg_raw: free until its next emitting phase), then each tree's apply phase.
meerkat_status dtrees_apply(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, int phase,
                            const uint64_t* recv, const uint64_t* rc) {
  const uint32_t ws = g->ws;
  if (k == 0 || (uint64_t)ws * k > (uint64_t)MAX_SEGS) return MEERKAT_E_INVALID_ARG;
  uint64_t per[8] = {0};
  for (uint32_t p = 0; p < ws; p++)
    for (uint32_t i = 0; i < k; i++) per[i] += rc[(size_t)p * k + i];
  cudaError_t e = cudaSuccess;
  for (uint32_t i = 0; i < k && e == cudaSuccess; i++)
    if (per[i] + 1024 > trees[i]->msg_cap) e = ensure_msgs(g, trees[i], per[i] + 1024);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  Segs S{};
  uint64_t filled[8] = {0}, total = 0;
  for (uint32_t p = 0; p < ws; p++)
    for (uint32_t i = 0; i < k; i++) {
      const uint32_t j = S.n++;
      S.src[j] = recv + 2 * total;
      S.dst[j] = trees[i]->msg_raw + 2 * filled[i];
      S.start[j] = total;
      total += rc[(size_t)p * k + i];
      filled[i] += rc[(size_t)p * k + i];
    }
  S.start[S.n] = total;
  if (total) {
    k_copy_segs<<<dgrid(g, total), D_BLOCK, 0, g->stream>>>(S);
    g->launches++;
    e = cudaGetLastError();
    if (e != cudaSuccess) return MEERKAT_E_CUDA;
  }
  for (uint32_t i = 0; i < k; i++) {
    if (!per[i]) continue;
    const meerkat_status st = dtree_phase(g, trees[i], phase, trees[i]->msg_raw, nullptr, nullptr, per[i], nullptr);
    if (st != MEERKAT_OK) return st;
  }
  return MEERKAT_OK;
}

// The DEC_SCAN phase of up to two trees in lock step with ONE stream of the slab array: per tree
// the phase bookkeeping of dtree_phase (new frontier buffer, epoch, message counter, marks of every
// rank's invalid vertices), then one k_dscan, per-tree message grouping, one synchronisation.
meerkat_status dtrees_scan(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, const uint32_t* const* lists,
                           const uint64_t* ns, meerkat_dresult* outs) {
  if (k == 0 || k > 2) return MEERKAT_E_INVALID_ARG;
  cudaError_t e = cudaSuccess;
  DScanArgs S{};
  int nb[2] = {0, 0};
  uint64_t n_all = 0;
  for (uint32_t j = 0; j < k && e == cudaSuccess; j++) {
    meerkat_tree* t = trees[j];
    TreeDev& T = t->dev;
    nb[j] = 1 - t->cur;
    e = cudaMemsetAsync(&T.ctrl->size[nb[j]], 0, 8, g->stream);
    t->depoch++;
    if (e == cudaSuccess) e = cudaMemsetAsync(t->dcnt + 2 * MEERKAT_MAX_RANKS, 0, 8, g->stream);
    DArgs A;
    A.G = g->out.dev; A.T = T;
    A.msgs = t->msg_raw; A.msg_n = t->dcnt + 2 * MEERKAT_MAX_RANKS; A.msg_cap = t->msg_cap;
    A.fr = T.fr[t->cur]; A.n_ptr = &T.ctrl->size[t->cur];
    A.fnext = T.fr[nb[j]]; A.sznext = &T.ctrl->size[nb[j]];
    A.epoch = t->depoch; A.unit = t->unit ? 1u : 0u;
    if (e == cudaSuccess && ns[j]) {
      e = dlaunch(g, 9, A, lists[j], nullptr, (const void*)1, ns[j], 0, 0);   // mark every rank's invalid vertices
      S.A[S.ntrees] = A;
      S.list[S.ntrees] = lists[j];
      S.n_inv[S.ntrees] = ns[j];
      S.ntrees++;
      n_all += ns[j];
    }
  }
  if (e == cudaSuccess && S.ntrees) {
    if (S.ntrees == 1) S.A[1] = S.A[0];
    const uint32_t fw = (n_all * 8 <= (uint64_t)FILTER_WORDS * 32) ? FILTER_WORDS : 0u;
    const uint32_t n_slabs = (uint32_t)(g->out.H + std::min<uint64_t>(g->out.hctrl->pool_top, g->out.P));
    e_scan(g, S, fw, n_slabs);
    e = cudaGetLastError();
  }
  for (uint32_t j = 0; j < k && e == cudaSuccess; j++) {
    meerkat_tree* t = trees[j];
    e = dsort_msgs(g, t->msg_raw, t->dcnt + 2 * MEERKAT_MAX_RANKS, t->msg_cap, t->dcnt, t->dcnt + MEERKAT_MAX_RANKS,
                   t->msg_out);
    t->cur = nb[j];
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(t->hcnt, t->dcnt, MEERKAT_MAX_RANKS * 8, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(t->hctrl, t->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  for (uint32_t j = 0; j < k; j++) {
    meerkat_tree* t = trees[j];
    t->cur_n = t->hctrl->size[t->cur];
    t->last_front = t->cur_n;
    if (outs) {
      meerkat_dresult* out = outs + j;
      std::memset(out, 0, sizeof(*out));
      out->msgs = t->msg_out;
      for (uint32_t r = 0; r < g->ws && r < MEERKAT_MAX_RANKS; r++) out->msg_counts[r] = t->hcnt[r];
      out->frontier = t->cur_n;
      out->invalid = t->dev.inval_list;
      out->invalid_n = t->hctrl->inval_n;
    }
  }
  const uint32_t err = g->out.hctrl->err;
  if (!err) return MEERKAT_OK;
  cudaMemsetAsync(&g->out.dev.ctrl->err, 0, 4, g->stream);
  if (err & ERR_CAPACITY) return MEERKAT_E_CAPACITY;
  if (err & ERR_OVERFLOW) return MEERKAT_E_OVERFLOW;
  return MEERKAT_E_STATE;
}

meerkat_status dtree_init(meerkat_graph* g, meerkat_tree* t) {
  t->dist = true;
  cudaError_t e = cudaMalloc(&t->dcnt, (2 * MEERKAT_MAX_RANKS + 1) * 8);
  if (e == cudaSuccess) e = cudaMallocHost(&t->hcnt, (MEERKAT_MAX_RANKS + 4) * 8);
  if (e == cudaSuccess) e = dscan_attr(g);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  return dtree_phase(g, t, MEERKAT_D_STATIC_INIT, nullptr, nullptr, nullptr, 0, nullptr);
}

void dtree_free(meerkat_tree* t) {
  cudaFree(t->msg_raw);
  cudaFree(t->msg_out);
  cudaFree(t->dcnt);
  if (t->hcnt) cudaFreeHost(t->hcnt);
}

static meerkat_status dtree_finish_phase(meerkat_graph* g, meerkat_tree* t, bool emits, meerkat_dresult* out);

// defer: enqueue the phase only (no synchronisation / read-back); dtrees_expand finishes a batch of
// deferred phases with one synchronisation.
meerkat_status dtree_phase_x(meerkat_graph* g, meerkat_tree* t, int phase, const void* a, const void* b,
                             const void* c, uint64_t n, meerkat_dresult* out, bool defer);

meerkat_status dtree_phase(meerkat_graph* g, meerkat_tree* t, int phase, const void* a, const void* b, const void* c,
                           uint64_t n, meerkat_dresult* out) {
  return dtree_phase_x(g, t, phase, a, b, c, n, out, false);
}

meerkat_status dtree_phase_x(meerkat_graph* g, meerkat_tree* t, int phase, const void* a, const void* b,
                             const void* c, uint64_t n, meerkat_dresult* out, bool defer) {
  const bool seed = phase == MEERKAT_D_STATIC_INIT || phase == MEERKAT_D_INC_SEED ||
                    phase == MEERKAT_D_DEC_INVALIDATE || phase == MEERKAT_D_DEC_SCAN;
  const bool expands = phase == MEERKAT_D_PROPAGATE || phase == MEERKAT_D_RELAX;
  const bool apply = phase == MEERKAT_D_APPLY_PROPAGATE || phase == MEERKAT_D_APPLY_RELAX;
  const bool emits = phase == MEERKAT_D_INC_SEED || expands || phase == MEERKAT_D_DEC_SCAN;
  if (!seed && !expands && !apply && phase != MEERKAT_D_FINISH) return MEERKAT_E_INVALID_ARG;
  if (n && (phase == MEERKAT_D_INC_SEED || phase == MEERKAT_D_DEC_INVALIDATE) && (!a || !b)) return MEERKAT_E_INVALID_ARG;
  if (n && (apply || phase == MEERKAT_D_DEC_SCAN || phase == MEERKAT_D_FINISH) && !a) return MEERKAT_E_INVALID_ARG;
  if (phase == MEERKAT_D_INC_SEED && !t->unit && n && !c) return MEERKAT_E_INVALID_ARG;
  // ordering contract, as for the single-GPU calls
  if (phase == MEERKAT_D_INC_SEED && (g->last_kind != 1 || t->version + 1 != g->version)) return MEERKAT_E_STATE;
  if (phase == MEERKAT_D_DEC_INVALIDATE && (g->last_kind != 2 || t->version + 1 != g->version)) return MEERKAT_E_STATE;
  TreeDev& T = t->dev;
  cudaError_t e = cudaSuccess;
  const bool starts_update =
      phase == MEERKAT_D_STATIC_INIT || phase == MEERKAT_D_INC_SEED || phase == MEERKAT_D_DEC_INVALIDATE;
  if (starts_update) {
    // a new update: counters and sizes; message capacity for the update (at most one message per
    // visited edge per expansion, i.e. bounded by the live edges held here; plus the batch)
    e = cudaMemsetAsync(T.ctrl, 0, sizeof(TreeCtrl), g->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e == cudaSuccess) e = ensure_msgs(g, t, g->out.hctrl->ins_total - g->out.hctrl->del_total + n + 1024);
    t->hctrl->inval_n = 0;
  }
  // frontier buffers: `cur` holds the frontier filled last; new frontiers go to the other one
  int nb = t->cur;
  if (seed || expands) {
    nb = 1 - t->cur;
    if (e == cudaSuccess) e = cudaMemsetAsync(&T.ctrl->size[nb], 0, 8, g->stream);
    t->depoch++;
  }
  if (e == cudaSuccess && emits) {
    if (n + 1024 > t->msg_cap && phase == MEERKAT_D_INC_SEED) e = ensure_msgs(g, t, n + 1024);
    if (e == cudaSuccess) e = cudaMemsetAsync(t->dcnt + 2 * MEERKAT_MAX_RANKS, 0, 8, g->stream);
  }
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  DArgs A;
  A.G = g->out.dev;
  A.T = T;
  A.msgs = t->msg_raw;
  A.msg_n = t->dcnt + 2 * MEERKAT_MAX_RANKS;
  A.msg_cap = t->msg_cap;
  A.fr = T.fr[t->cur];
  A.n_ptr = &T.ctrl->size[t->cur];
  A.fnext = T.fr[nb];
  A.sznext = &T.ctrl->size[nb];
  A.epoch = t->depoch;
  A.unit = t->unit ? 1u : 0u;
  // grid size for an expansion: the host's bound on the frontier (the kernel reads the exact size)
  const uint64_t n_front = expands ? std::max<uint64_t>(t->cur_n, 1) : 0;
  switch (phase) {
    case MEERKAT_D_STATIC_INIT: e = dlaunch(g, 0, A, nullptr, nullptr, nullptr, 0, 0, 0); break;
    case MEERKAT_D_INC_SEED: e = dlaunch(g, 1, A, a, b, c, n, 0, 0); break;
    case MEERKAT_D_DEC_INVALIDATE: e = dlaunch(g, 2, A, a, b, nullptr, n, 0, 0); break;
    case MEERKAT_D_PROPAGATE: e = dlaunch(g, 3, A, nullptr, nullptr, nullptr, n_front, 0, 0); break;
    case MEERKAT_D_APPLY_PROPAGATE: e = dlaunch(g, 4, A, a, nullptr, nullptr, n, 0, 0); break;
    case MEERKAT_D_RELAX: e = dlaunch(g, 6, A, nullptr, nullptr, nullptr, n_front, 0, 0); break;
    case MEERKAT_D_APPLY_RELAX: e = dlaunch(g, 7, A, a, nullptr, nullptr, n, 0, 0); break;
    case MEERKAT_D_DEC_SCAN: {
      if (n) {
        e = dlaunch(g, 9, A, a, nullptr, (const void*)1, n, 0, 0);   // mark every rank's invalid vertices
        const uint32_t fw = (n * 8 <= (uint64_t)FILTER_WORDS * 32) ? FILTER_WORDS : 0u;
        const uint32_t n_slabs = (uint32_t)(g->out.H + std::min<uint64_t>(g->out.hctrl->pool_top, g->out.P));
        if (e == cudaSuccess) e = dlaunch(g, 5, A, a, nullptr, nullptr, n, fw, n_slabs);
      }
      break;
    }
    case MEERKAT_D_FINISH:
      if (n) e = dlaunch(g, 9, A, a, nullptr, nullptr, n, 0, 0);   // clear the marks
      t->version = g->version;
      break;
  }
  if (e == cudaSuccess && emits)
    e = dsort_msgs(g, t->msg_raw, A.msg_n, t->msg_cap, t->dcnt, t->dcnt + MEERKAT_MAX_RANKS, t->msg_out);
  if (seed || expands) t->cur = nb;
  if (phase == MEERKAT_D_INC_SEED || phase == MEERKAT_D_DEC_INVALIDATE || phase == MEERKAT_D_STATIC_INIT)
    t->version = g->version;
  if (out) std::memset(out, 0, sizeof(*out));
  if (apply) {   // stream-ordered; the next emitting phase reports the resulting frontier
    if (e != cudaSuccess) return MEERKAT_E_CUDA;
    t->cur_n += 8 * n;   // grid bound for the next expansion (each message adds a vertex's buckets)
    if (out) { out->msgs = t->msg_out; out->invalid = T.inval_list; }
    return MEERKAT_OK;
  }
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (defer) return MEERKAT_OK;
  return dtree_finish_phase(g, t, emits, out);
}

// One synchronisation per phase: message counts, tree control block, graph error word.
static meerkat_status dtree_readback(meerkat_graph* g, meerkat_tree* t, bool emits) {
  cudaError_t e = cudaSuccess;
  if (emits) e = cudaMemcpyAsync(t->hcnt, t->dcnt, MEERKAT_MAX_RANKS * 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t->hctrl, t->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  return e == cudaSuccess ? MEERKAT_OK : MEERKAT_E_CUDA;
}

static meerkat_status dtree_report(meerkat_graph* g, meerkat_tree* t, bool emits, meerkat_dresult* out) {
  t->cur_n = t->hctrl->size[t->cur];
  t->last_front = t->cur_n;
  if (out) {
    out->msgs = t->msg_out;
    if (emits)
      for (uint32_t r = 0; r < g->ws && r < MEERKAT_MAX_RANKS; r++) out->msg_counts[r] = t->hcnt[r];
    out->frontier = t->cur_n;
    out->invalid = t->dev.inval_list;
    out->invalid_n = t->hctrl->inval_n;
  }
  return MEERKAT_OK;
}

static meerkat_status graph_err_status(meerkat_graph* g) {
  const uint32_t err = g->out.hctrl->err;
  if (!err) return MEERKAT_OK;
  cudaMemsetAsync(&g->out.dev.ctrl->err, 0, 4, g->stream);
  if (err & ERR_PARTITION) return MEERKAT_E_PARTITION;
  if (err & ERR_RANGE) return MEERKAT_E_VERTEX_RANGE;
  if (err & ERR_WEIGHT) return MEERKAT_E_WEIGHT;
  if (err & ERR_CAPACITY) return MEERKAT_E_CAPACITY;
  if (err & ERR_OVERFLOW) return MEERKAT_E_OVERFLOW;
  return MEERKAT_E_STATE;
}

static meerkat_status dtree_finish_phase(meerkat_graph* g, meerkat_tree* t, bool emits, meerkat_dresult* out) {
  if (dtree_readback(g, t, emits) != MEERKAT_OK) return MEERKAT_E_CUDA;
  cudaError_t e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  dtree_report(g, t, emits, out);
  return graph_err_status(g);
}

// An expansion phase (PROPAGATE / RELAX) of k trees in lock step with ONE synchronisation.
meerkat_status dtrees_expand(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, int phase,
                             meerkat_dresult* outs) {
  for (uint32_t j = 0; j < k; j++) {
    if (outs) std::memset(outs + j, 0, sizeof(meerkat_dresult));
    const meerkat_status st = dtree_phase_x(g, trees[j], phase, nullptr, nullptr, nullptr, 0, outs ? outs + j : nullptr,
                                            true);
    if (st != MEERKAT_OK) return st;
  }
  for (uint32_t j = 0; j < k; j++)
    if (dtree_readback(g, trees[j], true) != MEERKAT_OK) return MEERKAT_E_CUDA;
  cudaError_t e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  for (uint32_t j = 0; j < k; j++) dtree_report(g, trees[j], true, outs ? outs + j : nullptr);
  return graph_err_status(g);
}

meerkat_status route_batch(meerkat_graph* g, int key_is_b, const uint32_t* a, const uint32_t* b, const uint32_t* c,
                           uint64_t n, uint32_t* oa, uint32_t* ob, uint32_t* oc, uint64_t* counts) {
  cudaError_t e = cudaSuccess;
  if (!g->rscratch) e = cudaMalloc(&g->rscratch, 2 * MEERKAT_MAX_RANKS * 8);   // counts[64] + cursor[64]
  if (e == cudaSuccess && !g->hrscratch) e = cudaMallocHost(&g->hrscratch, MEERKAT_MAX_RANKS * 8);
  unsigned long long* scratch = g->rscratch;
  unsigned long long* hscratch = g->hrscratch;
  if (e == cudaSuccess)
    e = droute(g, a, b, c, key_is_b ? b : a, n, oa, ob, oc, scratch, scratch + MEERKAT_MAX_RANKS);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hscratch, scratch, MEERKAT_MAX_RANKS * 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  for (uint32_t r = 0; r < g->ws; r++) counts[r] = n ? hscratch[r] : 0;
  return MEERKAT_OK;
}

}  // namespace mk
