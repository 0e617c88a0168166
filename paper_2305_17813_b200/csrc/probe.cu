// probe.cu — latency microbenchmarks behind the latency floor that bench.py reports beside the
// HBM roofline of the latency-bound tree calls (SURVEY §8(d) "latency term", §7 H2).
//
// A frontier round of a tree call is a chain of dependent memory operations (item fetch -> slab ->
// node[x] atomicMin -> stamp / vmeta -> enqueue) closed by a grid-wide barrier; its floor is
// (barrier + chain x per-access latency), whatever the bytes.  These probes measure the terms on
// the device the graph lives on, with the graph's own cooperative launch shape:
//  * dependent loads (one thread, a full-period LCG permutation so every hop is a new random line)
//    in a buffer far larger than L2 (DRAM latency) and in one that fits L2 (L2 hit latency);
//  * dependent 64-bit atomicMin round trips on random lines of the large buffer;
//  * cooperative-groups grid.sync() on the tree kernels' grid (blocks per SM x SMs x 512 threads).
#include <cooperative_groups.h>

#include <algorithm>

#include "graph.h"
#include "tree_common.cuh"

namespace cg = cooperative_groups;

namespace mk {

__global__ void k_probe_fill(uint32_t* buf, uint64_t n_words, uint64_t mask) {
  // word index i -> next index (a * i + c) mod 2^k restricted to line starts: one full-period cycle
  // over all lines (c odd, a = 1 mod 4), each hop to a pseudo-random line
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_words; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t line = i >> 5;
    buf[i] = (uint32_t)(((line * 0x9E3779B1ull + 0x7F4A7C15ull) & mask) << 5);
  }
}

__global__ void k_probe_chase(const uint32_t* buf, uint32_t steps, int atomic, unsigned long long* out) {
  uint32_t x = 0;
  unsigned long long t0, t1;
  for (int warm = 0; warm < 2; warm++) {   // pass 0 warms the TLB / instruction path, pass 1 is timed
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (uint32_t i = 0; i < steps; i++) {
      if (atomic) {
        // the returned old value is the next index: a chain of dependent atomic round trips
        unsigned long long* p = reinterpret_cast<unsigned long long*>(const_cast<uint32_t*>(buf) + x);
        x = (uint32_t)atomicMin(p, ~0ull);
      } else {
        x = __ldcg(buf + x);
      }
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  }
  out[0] = t1 - t0;
  out[1] = x;   // keeps the chain live
}

__global__ void __launch_bounds__(TREE_BLOCK, TREE_MINB) k_probe_gridsync(uint32_t reps, unsigned long long* out) {
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t i = 0; i < reps; i++) grid.sync();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) out[2] = t1 - t0;
}

}  // namespace mk

using namespace mk;

extern "C" meerkat_status meerkat_probe_latency(meerkat_graph* g, meerkat_latency* out) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  const uint64_t big_lines = 1ull << 24, small_lines = 1ull << 15;   // 2 GiB (>> L2), 4 MiB (<< L2)
  uint32_t* buf = nullptr;
  unsigned long long* res = nullptr;
  unsigned long long h[3] = {0, 0, 0};
  const uint32_t steps = 4096, reps = 200;
  double ns[3] = {0, 0, 0};
  cudaError_t e = cudaMallocAsync(&buf, big_lines * 128, g->stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&res, 3 * 8, g->stream);
  const int order[3][2] = {{1, 0}, {0, 0}, {1, 1}};   // (big buffer?, atomic?): DRAM load, L2 load, DRAM atomic
  for (int k = 0; k < 3 && e == cudaSuccess; k++) {
    const uint64_t lines = order[k][0] ? big_lines : small_lines;
    k_probe_fill<<<g->sm_count * 8, 256, 0, g->stream>>>(buf, lines * 32, lines - 1);
    k_probe_chase<<<1, 1, 0, g->stream>>>(buf, steps, order[k][1], res);
    e = cudaMemcpyAsync(h, res, 16, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    ns[k] = (double)h[0] / steps;
  }
  if (e == cudaSuccess) {
    void* args[] = {(void*)&reps, (void*)&res};
    int bps = g->tree_blocks_per_sm[MODE_DECREMENTAL];
    if (g->latency_bps > 0) bps = std::min(bps, g->latency_bps);
    e = cudaLaunchCooperativeKernel((void*)k_probe_gridsync, dim3((unsigned)(bps * g->sm_count)), dim3(TREE_BLOCK),
                                    args, 0, g->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, res, 24, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    out->grid_blocks = (uint32_t)(bps * g->sm_count);
  }
  cudaFreeAsync(buf, g->stream);
  cudaFreeAsync(res, g->stream);
  cudaStreamSynchronize(g->stream);
  if (prev >= 0) cudaSetDevice(prev);
  if (e != cudaSuccess) { cudaGetLastError(); return MEERKAT_E_CUDA; }
  out->dram_load_ns = ns[0];
  out->l2_load_ns = ns[1];
  out->dram_atomic_ns = ns[2];
  out->grid_sync_us = (double)h[2] / reps / 1e3;
  return MEERKAT_OK;
}
