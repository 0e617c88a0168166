// tc.cu — the Count kernel of dynamic triangle counting (P:2060-2115,
// P:1643-1656, Algorithm tc-count):
//   Count(G1, G2, edges) = sum over (u, v) in edges of |adjacency_G1(u) ∩ adjacency_G2(v)|.
// The paper walks adjacency(v) in G2 with a warp (SlabIterator) and searches each neighbour adj_v
// in u's table of G1.  The intersection is symmetric in which side is walked, so here
// the walked side is the endpoint with the smaller degree (degree tables counted on demand by
// launch_degrees) and the other side is probed; the result is the same number.
//
// B200 design:
//  * plan: one thread per edge picks the walked side and writes its slab-list (bucket) count;
//    an exclusive scan (cub) turns the counts into item offsets, so a hub's buckets become
//    independent work items (the paper's <v, i> work list) spread over the GPU;
//  * count: an 8-lane group per (edge, bucket) item walks that slab list (one LDG.128 per lane per
//    slab); each lane then probes ITS live keys in the other graph's table independently (hash of
//    the key -> bucket -> whole-slab reads, early exit at the first slab holding an EMPTY cell,
//    the EMPTY-suffix invariant of §4.2), so 8 probes of a group are in flight at once;
//  * warp / block reduction, one 64-bit atomicAdd per block.
#include <cub/cub.cuh>

#include <algorithm>

#include "graph.h"

namespace mk {

constexpr int TC_BLOCK = 256;

// Per edge: walked side (side[e] = 1: walk G2's row of v and probe G1's row of u; 0: the reverse)
// and the number of slab lists of the walked row (0: nothing to intersect).
__global__ void k_tc_plan(GraphDev G1, GraphDev G2, const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst,
                          uint64_t n, uint32_t* __restrict__ side, uint64_t* __restrict__ cnt) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t u = src[e], v = dst[e];
    uint64_t c = 0;
    uint32_t sd = 0;
    if (u < G1.V && v < G2.V) {
      const uint32_t du = G1.deg[u], dv = G2.deg[v];
      if (du && dv) {
        sd = dv < du ? 1u : 0u;
        const uint2 m = sd ? G2.vmeta[v] : G1.vmeta[u];
        c = m.x == INVALID_SLAB ? 0 : m.y;
      }
    }
    side[e] = sd;
    cnt[e] = c;
  }
}

// Is key x in row w of store P?  (whole-slab reads by one lane; chains end at the first slab
// that still holds an EMPTY cell, or at INVALID_SLAB)
template <bool MAP>
__device__ __forceinline__ bool lane_probe(const GraphDev& P, uint32_t w, uint32_t x) {
  const uint2 m = __ldg(P.vmeta + w);
  if (m.x == INVALID_SLAB) return false;
  uint32_t s = m.x + bucket_of(x, m.y, P.seed);
  for (uint32_t guard = 0; guard < (1u << 24); guard++) {
    const uint4* p = reinterpret_cast<const uint4*>(slab_ptr(P, s));
    uint4 q[8];
#pragma unroll
    for (int i = 0; i < 8; i++) q[i] = ld_slab_ro(reinterpret_cast<const uint32_t*>(p + i), 0);
    bool hit = false, empty = false;
#pragma unroll
    for (int i = 0; i < 8; i++) {
#pragma unroll
      for (int k = 0; k < Frag<MAP>::NK; k++) {
        if (!Frag<MAP>::valid_cell(i, k)) continue;
        const uint32_t key = Frag<MAP>::key(q[i], k);
        hit |= key == x;
        empty |= key == EMPTY_KEY;
      }
    }
    if (hit) return true;
    const uint32_t nxt = q[7].w;
    if (empty || nxt == INVALID_SLAB) return false;
    s = nxt;
  }
  return false;
}

template <bool MAP1, bool MAP2>
__global__ void __launch_bounds__(TC_BLOCK) k_tc_count(GraphDev G1, GraphDev G2, const uint32_t* __restrict__ src,
                                                       const uint32_t* __restrict__ dst, uint64_t n,
                                                       const uint32_t* __restrict__ side,
                                                       const uint64_t* __restrict__ off, uint64_t total,
                                                       unsigned long long* __restrict__ out) {
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const uint32_t gmask = 0xFFu << (lane & 24);
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  uint64_t tally = 0;
  for (uint64_t j = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP; j < total; j += ng) {
    // edge of item j: the last e with off[e] <= j (off = exclusive scan of the bucket counts)
    uint64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const uint64_t mid = (lo + hi) / 2;
      if (__ldg(off + mid) <= j) lo = mid; else hi = mid;
    }
    const uint64_t e = lo;
    const uint32_t u = __ldg(src + e), v = __ldg(dst + e), sd = __ldg(side + e);
    const GraphDev& Wk = sd ? G2 : G1;   // walked
    const GraphDev& Pr = sd ? G1 : G2;   // probed
    const uint32_t wv = sd ? v : u, pv = sd ? u : v;
    const bool wmap = sd ? MAP2 : MAP1, pmap = sd ? MAP1 : MAP2;
    uint32_t s = __ldg(&Wk.vmeta[wv].x) + (uint32_t)(j - __ldg(off + e));
    for (uint32_t guard = 0; guard < (1u << 24); guard++) {
      const uint4 d = ld_slab_ro(slab_ptr(Wk, s), l8);
      uint32_t keys[4];
      int nk = 0;
      if (wmap) {
        keys[0] = d.x; keys[1] = l8 == GROUP - 1 ? EMPTY_KEY : d.z; nk = 2;
      } else {
        keys[0] = d.x; keys[1] = d.y; keys[2] = d.z; keys[3] = l8 == GROUP - 1 ? EMPTY_KEY : d.w; nk = 4;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (k >= nk) break;
        const uint32_t x = keys[k];
        if (x >= Pr.Vg) continue;   // EMPTY / TOMBSTONE
        tally += pmap ? lane_probe<true>(Pr, pv, x) : lane_probe<false>(Pr, pv, x);
      }
      const uint32_t nxt = __shfl_sync(gmask, d.w, GROUP - 1, GROUP);   // groups of a warp diverge here
      if (nxt == INVALID_SLAB) break;
      s = nxt;
    }
  }
  // block reduction, one atomic per block
  __shared__ unsigned long long acc;
  if (threadIdx.x == 0) acc = 0;
  __syncthreads();
  for (int o = 16; o; o >>= 1) tally += __shfl_down_sync(0xFFFFFFFFu, tally, o);
  if (lane == 0 && tally) atomicAdd(&acc, tally);
  __syncthreads();
  if (threadIdx.x == 0 && acc) atomicAdd(out, acc);
}

// Count(G1, G2, edges) into *out_dev (device u64, accumulated).  src/dst are device arrays.
cudaError_t launch_tc_count(meerkat_graph* g1, meerkat_graph* g2, const uint32_t* src, const uint32_t* dst,
                            uint64_t n, unsigned long long* out_dev) {
  if (!n) return cudaSuccess;
  cudaStream_t st = g1->stream;
  uint32_t* side = nullptr;
  uint64_t *cnt = nullptr, *off = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  uint64_t total = 0;
  cudaError_t e;
#define CK(x) do { e = (x); if (e != cudaSuccess) goto out; } while (0)
  // degree tables (walked-side choice), counted when a graph changed since the last count
  CK(launch_degrees(g1, g1->out));
  if (g2 != g1) {
    CK(launch_degrees(g2, g2->out));
    if (g2->stream != st) CK(cudaStreamSynchronize(g2->stream));
  }
  CK(cudaMallocAsync(&side, n * 4, st));
  CK(cudaMallocAsync(&cnt, (n + 1) * 8, st));
  CK(cudaMallocAsync(&off, (n + 1) * 8, st));
  {
    const unsigned gb = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)g1->sm_count * 16);
    k_tc_plan<<<gb, 256, 0, st>>>(g1->out.dev, g2->out.dev, src, dst, n, side, cnt);
    g1->launches++;
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(cnt + n, 0, 8, st));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, n + 1, st));
    CK(cudaMallocAsync(&tmp, tmp_bytes, st));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, n + 1, st));
    g1->launches++;
    CK(cudaMemcpyAsync(&total, off + n, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (total) {
      const uint64_t per_block = TC_BLOCK / GROUP;
      const unsigned gc = (unsigned)std::min<uint64_t>((total + per_block - 1) / per_block,
                                                       (uint64_t)g1->sm_count * 8);
      const bool m1 = g1->weighted, m2 = g2->weighted;
      auto fn = m1 ? (m2 ? k_tc_count<true, true> : k_tc_count<true, false>)
                   : (m2 ? k_tc_count<false, true> : k_tc_count<false, false>);
      fn<<<gc, TC_BLOCK, 0, st>>>(g1->out.dev, g2->out.dev, src, dst, n, side, off, total, out_dev);
      g1->launches++;
      CK(cudaGetLastError());
    }
  }
out:
#undef CK
  if (side) cudaFreeAsync(side, st);
  if (cnt) cudaFreeAsync(cnt, st);
  if (off) cudaFreeAsync(off, st);
  if (tmp) cudaFreeAsync(tmp, st);
  return e;
}

}  // namespace mk
