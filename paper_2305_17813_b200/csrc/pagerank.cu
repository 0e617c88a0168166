// pagerank.cu — static and dynamic PageRank over the in-edge slab store.
//
// Method (§Dynamic PageRank; Eq. (1)):
//   PR_i[v] = (1-d)/N + d * sum_{u->v} PR_{i-1}[u] / out[u]
// plus, when some vertex v_z has out-degree 0, the teleport term d * sum_{v_z} PR_{i-1}[v_z] / N
// added to every vertex (FindTeleportProb; reading C27: scaled by d), iterated until
// the L1 norm delta = sum_v |PR_i[v] - PR_{i-1}[v]| is <= the error margin or max_iter super-steps
// have run.  Static: PR_0 = 1/N.  Dynamic (incremental / decremental):
// "the same static-PageRank algorithm is applied on the entire graph after performing
// insertion/deletion", starting from the values before the batch.
// FindContributionPerVertex caches Contribution[u] = PR_{i-1}[u]/out[u] so the
// accumulation reads one array per in-edge.  Arithmetic in double precision (the paper states
// none; BASELINE.json asks 1e-6 relative L1 against the oracle).
//
// B200 design:
//  * ONE persistent cooperative launch runs every super-step; two grid barriers per super-step
//    (after the accumulation, after the per-vertex update) and the convergence test is read on
//    the device, so there is no host round trip per super-step;
//  * the Compute kernel's per-vertex in-edge walk becomes an address-order STREAM
//    over the in-edge store's slab array (owner[] names each slab's destination vertex v): an
//    8-lane group reads a slab with one LDG.128 per lane, gathers Contribution[u] of its live
//    keys, reduces in-group, and runs of slabs with the same owner within a warp are combined
//    before ONE fp64 atomicAdd into acc[v] — hubs' thousands of slab lists spread over the whole
//    GPU instead of serialising on one warp, and no chain is chased;
//  * out[u] is the store's per-vertex degree table, counted by a slab stream (launch_degrees) when
//    the graph changed since the last count;
//  * the per-vertex update fuses Eq. (1), the teleport term, the L1 delta, the next super-step's
//    contributions and the dangling mass, one coalesced pass over the vertex arrays.
#include <cooperative_groups.h>

#include "graph.h"
#include "stream.cuh"

namespace cg = cooperative_groups;

namespace mk {

constexpr int PR_BLOCK = 512;
#ifndef MEERKAT_PR_MINB
#define MEERKAT_PR_MINB 2   // resident blocks per SM k_pagerank is compiled for (A/B)
#endif
constexpr int PR_MINB = MEERKAT_PR_MINB;
#ifndef MEERKAT_PR_UNROLL
#define MEERKAT_PR_UNROLL 2
#endif
constexpr int PR_UNROLL = MEERKAT_PR_UNROLL;   // slabs in flight per group (register double-buffered)
using contrib_t = double;   // Contribution[] in fp64 (an fp32 cache was 5.5 % faster and broke the
                            // closed-form pins' tolerance: DESIGN.md §10)
size_t pagerank_contrib_bytes() { return sizeof(contrib_t); }
#ifndef MEERKAT_PR_BULK
#define MEERKAT_PR_BULK 0   // 1: the slab / owner stream moves by bulk copies through shared memory (stream.cuh; A/B: slower)
#endif

struct PRArgs {
  GraphDev R;               // in-edge store: owner[s] = v, keys = sources u
  const uint32_t* outdeg;   // out-store degree table: out[u]
  double* pr;
  contrib_t* contrib;   // Contribution[u] = PR[u] / out[u] (FindContributionPerVertex)
  double* acc;
  PRCtrl* ctrl;
  uint32_t V;
  uint32_t max_iter;
  uint32_t warm;            // 0: static start 1/N; 1: start from pr[] (dynamic)
  double d, eps;
};

// Block-wide sum of two doubles, one atomicAdd per block and value (all threads call).
__device__ __forceinline__ void block_add2(double a, double b, double* da, double* db) {
  __shared__ double sa[PR_BLOCK / 32], sb[PR_BLOCK / 32];
  for (int o = 16; o; o >>= 1) {
    a += __shfl_down_sync(0xFFFFFFFFu, a, o);
    b += __shfl_down_sync(0xFFFFFFFFu, b, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sa[w] = a; sb[w] = b; }
  __syncthreads();
  if (threadIdx.x < 32) {
    a = threadIdx.x < blockDim.x / 32 ? sa[threadIdx.x] : 0.0;
    b = threadIdx.x < blockDim.x / 32 ? sb[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_down_sync(0xFFFFFFFFu, a, o);
      b += __shfl_down_sync(0xFFFFFFFFu, b, o);
    }
    if (threadIdx.x == 0) {
      if (da && a != 0.0) atomicAdd(da, a);
      if (db && b != 0.0) atomicAdd(db, b);
    }
  }
  __syncthreads();
}

// Compute for one in-edge slab of owner o (this lane's fragment d): gather Contribution[u]
// of its live keys, reduce in the group, combine runs of one owner over the warp's four groups (four
// consecutive slabs), one fp64 atomicAdd into acc[o] per run.  Warp-collective.
// Two slabs per call (two chunks of the bulk stream): every gather of both is issued first.
template <bool MAP>
__device__ __forceinline__ void pr_gather(const PRArgs& A, const uint4& d, bool count, unsigned long long& keys,
                                          double (&cs)[Frag<MAP>::NK]) {
  using F = Frag<MAP>;
  const int l8 = threadIdx.x & 7;
#pragma unroll
  for (int k = 0; k < F::NK; k++) {
    const uint32_t u = F::key(d, k);
    const bool live = u < A.V && (MAP || F::valid_cell(l8, k));   // sentinels are >= V
    cs[k] = live ? (double)__ldcg(A.contrib + u) : 0.0;
    if (count && live) keys++;
  }
}

template <bool MAP>
__device__ __forceinline__ void pr_combine(const PRArgs& A, const double (&cs)[Frag<MAP>::NK], uint32_t o, bool count,
                                           unsigned long long& atomics) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NK; k++) s += cs[k];
  s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
  s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
  s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
  const uint32_t po = __shfl_up_sync(0xFFFFFFFFu, o, GROUP);
  const bool head = lane < GROUP || po != o;
  double tot = s;
  bool run = true;
#pragma unroll
  for (int k = 1; k < 4; k++) {
    const double sk = __shfl_down_sync(0xFFFFFFFFu, s, GROUP * k);
    const uint32_t ok = __shfl_down_sync(0xFFFFFFFFu, o, GROUP * k);
    run = run && lane + GROUP * k < 32 && ok == o;
    if (run) tot += sk;
  }
  if (l8 == 0 && head && o != NO_OWNER && tot != 0.0) {
    atomicAdd(A.acc + o, tot);
    if (count) atomics++;
  }
}

// Compute as a stream over the in-edge slabs [0, n_slabs): acc[v] += Contribution[u]
// for every live in-edge u -> v.  count: also tally live keys / atomics (first super-step only).
template <bool MAP>
__device__ __forceinline__ void pr_accumulate(const PRArgs& A, uint32_t n_slabs, bool count,
                                              unsigned long long& keys, unsigned long long& atomics) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  constexpr int U = PR_UNROLL;
  const GraphDev& R = A.R;
  const uint32_t V = A.V;
  const int lane = threadIdx.x & 31, l8 = lane & 7;
  const uint32_t ng = (gridDim.x * blockDim.x) / GROUP;
  const uint32_t g0 = (blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint32_t span = ng * U;
  const uint32_t trips = (n_slabs + span - 1) / span;   // warp-uniform
  const uint4* __restrict__ base = reinterpret_cast<const uint4*>(R.slabs) + l8;
  uint4 nd[U];
  uint32_t nown[U];
  auto load_trip = [&](uint32_t t, uint4 (&dst)[U], uint32_t (&own)[U]) {
#pragma unroll
    for (int q = 0; q < U; q++) {
      const uint32_t s = t * span + g0 + q * ng;
      dst[q] = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
      own[q] = NO_OWNER;
      if (s < n_slabs) {
        dst[q] = ld_slab_ro(reinterpret_cast<const uint32_t*>(base + (size_t)s * 8), 0);
        own[q] = __ldg(R.owner + s);
      }
    }
  };
  if (trips) load_trip(0, nd, nown);
  for (uint32_t t = 0; t < trips; t++) {
    uint4 d[U];
    uint32_t own[U];
#pragma unroll
    for (int q = 0; q < U; q++) { d[q] = nd[q]; own[q] = nown[q]; }
    if (t + 1 < trips) load_trip(t + 1, nd, nown);
    // gathers of every live key of both slabs first (independent loads in flight), then sums
    double c[U][NK];
#pragma unroll
    for (int q = 0; q < U; q++)
#pragma unroll
      for (int k = 0; k < NK; k++) {
        const uint32_t u = F::key(d[q], k);
        const bool live = u < V && (MAP || F::valid_cell(l8, k));   // sentinels are >= V
        c[q][k] = live ? (double)__ldcg(A.contrib + u) : 0.0;
        if (count && live) keys++;
      }
#pragma unroll
    for (int q = 0; q < U; q++) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < NK; k++) s += c[q][k];
      s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
      s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
      s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
      // the warp's 4 groups hold 4 consecutive slabs: combine runs with the same owner
      const uint32_t o = own[q];
      const uint32_t po = __shfl_up_sync(0xFFFFFFFFu, o, GROUP);
      const bool head = lane < GROUP || po != o;
      double tot = s;
      bool run = true;
#pragma unroll
      for (int k = 1; k < 4; k++) {
        const double sk = __shfl_down_sync(0xFFFFFFFFu, s, GROUP * k);
        const uint32_t ok = __shfl_down_sync(0xFFFFFFFFu, o, GROUP * k);
        run = run && lane + GROUP * k < 32 && ok == o;
        if (run) tot += sk;
      }
      if (l8 == 0 && head && o != NO_OWNER && tot != 0.0) {
        atomicAdd(A.acc + o, tot);
        if (count) atomics++;
      }
    }
  }
}

template <bool MAP>
__global__ void __launch_bounds__(PR_BLOCK, PR_MINB) k_pagerank(const __grid_constant__ PRArgs A) {
  cg::grid_group grid = cg::this_grid();
#if MEERKAT_PR_BULK
  __shared__ StreamSmem sm;
  uint32_t seq = 0;
  stream_init(sm);
#endif
  PRCtrl* C = A.ctrl;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t V = A.V;
  const double invN = 1.0 / (double)V;
  // initial vector and the first super-step's contributions / dangling mass
  {
    double dang = 0.0;
    for (uint64_t v = tid; v < V; v += nt) {
      double p;
      if (A.warm) p = A.pr[v];
      else { p = invN; A.pr[v] = p; }
      const uint32_t o = A.outdeg[v];
      A.contrib[v] = (contrib_t)(o ? p / (double)o : 0.0);
      if (!o) dang += p;
      A.acc[v] = 0.0;
    }
    block_add2(dang, 0.0, &C->dangling[0], nullptr);
  }
  grid.sync();
  const uint32_t n_slabs = A.R.H + (uint32_t)min((unsigned long long)A.R.P, __ldcg(&A.R.ctrl->pool_top));
  unsigned long long keys = 0, atomics = 0;
  const double base = (1.0 - A.d) / (double)V;
  uint32_t i = 0;
  for (;; i++) {
    // Compute: acc[v] = sum over in-edges of Contribution[u]
#if MEERKAT_PR_BULK
    stream_slabs<2>(sm, seq, A.R.slabs, A.R.owner, n_slabs,
                    [&](const uint4& d0, uint32_t o0, uint32_t, const uint4& d1, uint32_t o1, uint32_t) {
                      double c0[Frag<MAP>::NK], c1[Frag<MAP>::NK];
                      pr_gather<MAP>(A, d0, i == 0, keys, c0);
                      pr_gather<MAP>(A, d1, i == 0, keys, c1);
                      pr_combine<MAP>(A, c0, o0, i == 0, atomics);
                      pr_combine<MAP>(A, c1, o1, i == 0, atomics);
                    });
#else
    pr_accumulate<MAP>(A, n_slabs, i == 0, keys, atomics);
#endif
    grid.sync();
    // PR_i = (1-d)/N + d*acc (+ teleport), delta, next contributions and dangling mass
    const double teleport = A.d * __ldcg(&C->dangling[i % 3]) / (double)V;
    double dl = 0.0, dn = 0.0;
    for (uint64_t v = tid; v < V; v += nt) {
      const double old = A.pr[v];
      double p = base + A.d * __ldcg(A.acc + v);   // acc was summed by L2 atomics: bypass L1
      p += teleport;
      dl += fabs(p - old);
      A.pr[v] = p;
      const uint32_t o = A.outdeg[v];
      A.contrib[v] = (contrib_t)(o ? p / (double)o : 0.0);   // gathered next super-step
      if (!o) dn += p;
      A.acc[v] = 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // slots read one super-step ago
      C->delta[(i + 2) % 3] = 0.0;
      C->dangling[(i + 2) % 3] = 0.0;
    }
    block_add2(dl, dn, &C->delta[i % 3], &C->dangling[(i + 1) % 3]);
    grid.sync();
    const double delta = __ldcg(&C->delta[i % 3]);
    if (!(delta > A.eps) || i + 1 >= A.max_iter) {
      if (tid == 0) { C->iters = i + 1; C->last_delta = delta; C->slabs = n_slabs; }
      break;
    }
  }
  // per-super-step work counters (taken in the first super-step)
  keys = __reduce_add_sync(0xFFFFFFFFu, (unsigned)keys);
  atomics = __reduce_add_sync(0xFFFFFFFFu, (unsigned)atomics);
  if ((threadIdx.x & 31) == 0) {
    if (keys) atomicAdd(&C->keys, keys);
    if (atomics) atomicAdd(&C->atomics, atomics);
  }
}

cudaError_t pagerank_occupancy(bool weighted, int* blocks_per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      blocks_per_sm, weighted ? (const void*)k_pagerank<true> : (const void*)k_pagerank<false>, PR_BLOCK, 0);
}

cudaError_t launch_pagerank(meerkat_graph* g, meerkat_pagerank* p, bool warm) {
  cudaError_t e = launch_degrees(g, g->out);   // out[u], counted when the graph changed
  if (e == cudaSuccess) e = cudaMemsetAsync(p->ctrl, 0, sizeof(PRCtrl), g->stream);
  if (e != cudaSuccess) return e;
  PRArgs A;
  A.R = g->in.dev;
  A.outdeg = g->out.dev.deg;
  A.pr = p->pr; A.contrib = reinterpret_cast<contrib_t*>(p->contrib); A.acc = p->acc;
  A.ctrl = p->ctrl;
  A.V = g->V;
  A.max_iter = p->max_iter;
  A.warm = warm ? 1u : 0u;
  A.d = p->d; A.eps = p->eps;
  dim3 grid((unsigned)(p->blocks_per_sm * g->sm_count)), block(PR_BLOCK);
  void* args[] = {&A};
  e = cudaLaunchCooperativeKernel(g->weighted ? (void*)k_pagerank<true> : (void*)k_pagerank<false>, grid, block,
                                  args, 0, g->stream);
  if (e == cudaSuccess) g->launches++;
  return e;
}

}  // namespace mk
