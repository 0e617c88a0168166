// stream.cuh — address-order streaming of a slab array through shared memory with bulk copies
// (cp.async.bulk + mbarrier), for the kernels that read the WHOLE store once: PageRank's Compute
// and the paper's valid->invalid scan.
//
// A block owns chunks blockIdx.x, blockIdx.x + gridDim.x, ... of SC_SLABS consecutive slabs.  One
// thread keeps SC_STAGES chunks in flight: it arms a stage's mbarrier with the chunk's byte count and
// issues one bulk copy for the slabs and one for their owner[] entries (the copy engine, not the
// SMs' load slots, moves the stream); every thread waits on the stage's barrier, its 8-lane group
// handles slab g of the chunk (one 16-B shared-memory read per lane, as the register stream read it),
// and after a block barrier the stage is refilled with the chunk SC_STAGES ahead.
#pragma once
#include "internal.cuh"

namespace mk {

constexpr int SC_SLABS = 64;    // slabs per chunk: one per 8-lane group of a 512-thread block (8 KiB)
constexpr int SC_STAGES = 4;    // chunks in flight per block (32 KiB + owners)

struct StreamSmem {
  uint4 slab[SC_STAGES][SC_SLABS * 8];
  uint32_t owner[SC_STAGES][SC_SLABS];
  unsigned long long bar[SC_STAGES];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t phase) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

// Once per kernel, all threads: initialise the stage barriers (seq = 0 afterwards).
__device__ __forceinline__ void stream_init(StreamSmem& sm) {
  if (threadIdx.x == 0) {
    for (int st = 0; st < SC_STAGES; st++) mbar_init(&sm.bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Stream slabs [0, n_slabs) of (slabs, owner) through shared memory; body(slab16, owner, s) is called
// by every thread for its group's slab of each chunk (slab16 = this lane's 16-B fragment; past
// n_slabs the fragment is EMPTY and owner NO_OWNER).  Warp-uniform trip count: every lane calls body
// the same number of times (collectives inside body are allowed).  All threads of the block call it,
// blockDim.x == SC_SLABS * 8.  seq: chunks this block streamed so far in the kernel (stage / phase
// of the barriers), identical in every thread.
// PAIRS = 2: body(d0, o0, s0, d1, o1, s1) gets this group's slabs of TWO chunks per call (two stages
// waited for together), so a body with dependent gathers keeps twice the requests in flight.
template <int PAIRS = 1, class Body>
__device__ __forceinline__ void stream_slabs(StreamSmem& sm, uint32_t& seq, const uint32_t* slabs,
                                             const uint32_t* owner, uint32_t n_slabs, Body&& body) {
  static_assert(PAIRS == 1 || PAIRS == 2, "one or two chunks per body call");
  static_assert(SC_STAGES % PAIRS == 0, "stages come in pairs");
  const uint32_t n_chunks = (n_slabs + SC_SLABS - 1) / SC_SLABS;
  const uint32_t mine = n_chunks > blockIdx.x ? (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int g = threadIdx.x >> 3, l8 = threadIdx.x & 7;
  auto issue = [&](uint32_t j) {   // thread 0: chunk j of this block into stage (seq + j) % SC_STAGES
    const int st = (seq + j) % SC_STAGES;
    const uint32_t s0 = (blockIdx.x + j * gridDim.x) * SC_SLABS;
    const uint32_t k = min((uint32_t)SC_SLABS, n_slabs - s0);
    const bool full = k == SC_SLABS;   // owners of a partial chunk are read by the threads themselves
    // the stage was last read through the generic proxy (ordered by the block barrier): order those
    // reads before the async-proxy writes of the copy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&sm.bar[st], k * 128u + (full ? SC_SLABS * 4u : 0u));
    bulk_copy_g2s(sm.slab[st], slabs + (size_t)s0 * SLAB_WORDS, k * 128u, &sm.bar[st]);
    if (full) bulk_copy_g2s(sm.owner[st], owner + s0, SC_SLABS * 4u, &sm.bar[st]);
  };
  if (threadIdx.x == 0)
    for (uint32_t j = 0; j < mine && j < (uint32_t)SC_STAGES; j++) issue(j);
  auto fetch = [&](uint32_t j, uint4& d, uint32_t& own, uint32_t& s) {   // this group's slab of chunk j
    d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    own = NO_OWNER;
    s = n_slabs;
    if (j >= mine) return;
    const int st = (seq + j) % SC_STAGES;
    mbar_wait(&sm.bar[st], ((seq + j) / SC_STAGES) & 1);
    const uint32_t c0 = (blockIdx.x + j * gridDim.x) * SC_SLABS;
    s = c0 + g;
    if (s < n_slabs) {
      d = sm.slab[st][g * 8 + l8];
      own = c0 + SC_SLABS <= n_slabs ? sm.owner[st][g] : __ldg(owner + s);
    }
  };
  for (uint32_t j = 0; j < mine; j += PAIRS) {
    uint4 d0, d1;
    uint32_t o0, o1, s0, s1;
    fetch(j, d0, o0, s0);
    if constexpr (PAIRS == 2) {
      fetch(j + 1, d1, o1, s1);
      body(d0, o0, s0, d1, o1, s1);
    } else {
      body(d0, o0, s0);
    }
    __syncthreads();   // every thread is done with these stages
    if (threadIdx.x == 0)
      for (uint32_t q = 0; q < (uint32_t)PAIRS; q++)
        if (j + q + SC_STAGES < mine) issue(j + q + SC_STAGES);
  }
  seq += mine;
  __syncthreads();
}

}  // namespace mk
