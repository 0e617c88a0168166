// wcc.cu — static and incremental weakly connected components (P:905-912
// "Incremental WCC", supplementary P:381-395 static SamplingWCC, P:486-493 BatchInsert).
//
// Method: a root-based union-find over parents[]; static = MinHooking sampling (every
// vertex hooks under its smallest out-neighbour), full compression, then the union of the
// remaining edges, full compression; incremental = union of every inserted edge
// (BatchInsert with UnionOp) followed by full compression.
//
// Reading (C30): hooking always links the LARGER root under the SMALLER one, so the label
// of a vertex after compression is the smallest id of its component — canonical, so results are
// compared bit-exactly with the oracle.  The paper's Finish phase skips vertices carrying the most
// frequent label L_max, which is only complete for symmetric graphs; here every edge
// whose endpoints already share a root is skipped instead (one load each after the compression),
// which keeps the sampling's saving and is exact for directed graphs too.
//
// B200 design: the hook and union passes STREAM the slab array (owner[] names the source), one
// LDG.128 per lane of an 8-lane group per slab; MinHooking takes the group-min of a slab's keys and
// applies one atomicMin per slab; unions are lock-free (CAS of the larger root's parent from itself
// to the smaller root, retried on failure) with path-halving finds.
#include <algorithm>

#include "graph.h"

namespace mk {

constexpr int WCC_BLOCK = 256;

__device__ __forceinline__ uint32_t wcc_find(uint32_t* parent, uint32_t v) {
  uint32_t cur = __ldcg(parent + v);
  if (cur == v) return v;
  uint32_t prev = v;
  for (;;) {
    const uint32_t next = __ldcg(parent + cur);
    if (next == cur) break;
    __stcg(parent + prev, next);   // path halving: next is an ancestor of prev (ids only decrease)
    prev = cur;
    cur = next;
  }
  return cur;
}

// Read-only find for the compression pass: there, each thread writes only its own vertex's final
// root — a path-halving store from another thread could overwrite that root with an older,
// non-root ancestor after the owner wrote it.
__device__ __forceinline__ uint32_t wcc_find_ro(const uint32_t* parent, uint32_t v) {
  uint32_t cur = v;
  for (;;) {
    const uint32_t next = __ldcg(parent + cur);
    if (next == cur) return cur;
    cur = next;
  }
}

__device__ __forceinline__ void wcc_union(uint32_t* parent, uint32_t a, uint32_t b) {
  for (uint32_t guard = 0; guard < (1u << 24); guard++) {
    uint32_t ra = wcc_find(parent, a), rb = wcc_find(parent, b);
    if (ra == rb) return;
    if (ra > rb) { const uint32_t t = ra; ra = rb; rb = t; }
    if (atomicCAS(parent + rb, rb, ra) == rb) return;   // larger root hooks under the smaller
    a = ra; b = rb;
  }
}

__global__ void k_wcc_init(uint32_t* parent, uint32_t V) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x)
    parent[v] = (uint32_t)v;
}

__global__ void k_wcc_compress(uint32_t* parent, uint32_t V) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x)
    parent[v] = wcc_find_ro(parent, (uint32_t)v);
}

// Stream the slab array [0, n_slabs).  HOOK: parent[u] <- min(parent[u], smallest out-neighbour)
// (MinHooking), one atomicMin per slab.  UNION: union(u, x) for every live edge whose
// endpoints do not already share a parent.
template <bool MAP, bool HOOK>
__global__ void __launch_bounds__(WCC_BLOCK) k_wcc_stream(GraphDev G, uint64_t n_slabs, uint32_t* parent,
                                                          unsigned long long* unions) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t trips = (n_slabs + ng - 1) / ng;   // warp-uniform
  uint32_t tried = 0;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t s = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP + t * ng;
    uint32_t u = NO_OWNER;
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    if (s < n_slabs) {
      u = __ldg(G.owner + s);
      d = ld_slab_ro(slab_ptr(G, (uint32_t)s), l8);
    }
    if (HOOK) {
      uint32_t m = 0xFFFFFFFFu;
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t x = F::key(d, k);
        if (x < G.Vg && (MAP || F::valid_cell(l8, k))) m = min(m, x);
      }
      m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, 1));
      m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
      m = min(m, __shfl_xor_sync(0xFFFFFFFFu, m, 4));
      if (l8 == 0 && u != NO_OWNER && m < u) atomicMin(parent + u, m);
    } else if (u != NO_OWNER) {
      const uint32_t pu = __ldcg(parent + u);
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t x = F::key(d, k);
        if (x >= G.Vg || !(MAP || F::valid_cell(l8, k))) continue;
        if (__ldcg(parent + x) == pu) continue;   // already in the same tree root (after compression)
        tried++;
        wcc_union(parent, u, x);
      }
    }
  }
  if (!HOOK) {
    tried = __reduce_add_sync(0xFFFFFFFFu, tried);
    if (lane == 0 && tried) atomicAdd(unions, (unsigned long long)tried);
  }
}

// BatchInsert's UnionOp: union(src[i], dst[i]) for every edge of the batch.
__global__ void k_wcc_batch(uint32_t* parent, uint32_t V, const uint32_t* __restrict__ src,
                            const uint32_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = src[i], v = dst[i];
    if (u < V && v < V) wcc_union(parent, u, v);
  }
}

// UpdateIterator: one 8-lane group per queued slab list walks it from its first
// updated cell (earlier cells and slabs hold only edges older than the tracking window) and unions
// (owner, key) for every live key; then resets the list's tracking (UpdateSlabPointers).  With
// TOMBSTONE reuse an old key can sit after the first updated cell: its union is a no-op.
template <bool MAP>
__global__ void __launch_bounds__(WCC_BLOCK) k_wcc_update_iter(GraphDev G, uint32_t* parent) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const uint32_t gmask = 0xFFu << (lane & 24);
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t n = __ldcg(&G.ctrl->upd_n);
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; i < n; i += ng) {
    const uint32_t list = __ldcg(G.updq + i);
    const unsigned long long pos = __ldcg(G.upd + list);
    const uint32_t u = __ldg(G.owner + list);
    uint32_t s = (uint32_t)(pos >> 5);
    int c0 = (int)(pos & 31);
    for (uint32_t guard = 0; guard < (1u << 24) && s != INVALID_SLAB; guard++) {
      const uint4 d = ld_slab_cg(slab_ptr(G, s), l8);
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t x = F::key(d, k);
        if (l8 * NK + k >= c0 && F::valid_cell(l8, k) && x < G.Vg) wcc_union(parent, u, x);
      }
      s = __shfl_sync(gmask, d.w, GROUP - 1, GROUP);
      c0 = 0;
    }
    if (l8 == 0) G.upd[list] = ~0ull;   // UpdateSlabPointers
  }
}

__global__ void k_wcc_count_roots(const uint32_t* parent, uint32_t V, unsigned long long* out) {
  uint32_t c = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += (uint64_t)gridDim.x * blockDim.x)
    c += parent[v] == (uint32_t)v;
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

static unsigned wcc_grid(meerkat_graph* g, uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + WCC_BLOCK - 1) / WCC_BLOCK,
                                                            (uint64_t)g->sm_count * 8));
}

cudaError_t launch_wcc_static(meerkat_graph* g, uint32_t* parent, unsigned long long* scratch) {
  const uint32_t V = g->V;
  Store& st = g->out;
  cudaError_t e = cudaMemcpyAsync(st.hctrl, st.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return e;
  const uint64_t n_slabs = st.H + std::min<uint64_t>(st.hctrl->pool_top, st.P);
  const unsigned gv = wcc_grid(g, V);
  const unsigned gs = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>((n_slabs * GROUP + WCC_BLOCK - 1) / WCC_BLOCK, (uint64_t)g->sm_count * 8));
  k_wcc_init<<<gv, WCC_BLOCK, 0, g->stream>>>(parent, V);
  if (g->weighted) k_wcc_stream<true, true><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, n_slabs, parent, scratch);
  else k_wcc_stream<false, true><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, n_slabs, parent, scratch);
  k_wcc_compress<<<gv, WCC_BLOCK, 0, g->stream>>>(parent, V);
  if (g->weighted) k_wcc_stream<true, false><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, n_slabs, parent, scratch);
  else k_wcc_stream<false, false><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, n_slabs, parent, scratch);
  k_wcc_compress<<<gv, WCC_BLOCK, 0, g->stream>>>(parent, V);
  g->launches += 5;
  return cudaGetLastError();
}

cudaError_t launch_wcc_batch(meerkat_graph* g, uint32_t* parent, const uint32_t* s, const uint32_t* d, uint64_t n) {
  if (n) {
    k_wcc_batch<<<wcc_grid(g, n), WCC_BLOCK, 0, g->stream>>>(parent, g->V, s, d, n);
    g->launches++;
  }
  k_wcc_compress<<<wcc_grid(g, g->V), WCC_BLOCK, 0, g->stream>>>(parent, g->V);   // Compress(Parents)
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_wcc_tracked(meerkat_graph* g, uint32_t* parent) {
  Store& st = g->out;
  const unsigned gs = (unsigned)((uint64_t)g->sm_count * 8);
  if (g->weighted) k_wcc_update_iter<true><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, parent);
  else k_wcc_update_iter<false><<<gs, WCC_BLOCK, 0, g->stream>>>(st.dev, parent);
  g->launches++;
  cudaError_t e = cudaMemsetAsync(&st.dev.ctrl->upd_n, 0, 8, g->stream);
  if (e != cudaSuccess) return e;
  k_wcc_compress<<<wcc_grid(g, g->V), WCC_BLOCK, 0, g->stream>>>(parent, g->V);
  g->launches++;
  return cudaGetLastError();
}

cudaError_t launch_wcc_roots(meerkat_graph* g, const uint32_t* parent, unsigned long long* out_dev) {
  cudaError_t e = cudaMemsetAsync(out_dev, 0, 8, g->stream);
  if (e != cudaSuccess) return e;
  k_wcc_count_roots<<<wcc_grid(g, g->V), WCC_BLOCK, 0, g->stream>>>(parent, g->V, out_dev);
  g->launches++;
  return cudaGetLastError();
}

}  // namespace mk
