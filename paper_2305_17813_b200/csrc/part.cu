// part.cu — vertex-partitioned (multi-GPU) graphs: owner-routed batches and
// device-driven SSSP / BFS exchange units.
//
// Placement.  Rank r holds every vertex v with owner(v) == r at row(v) (pm_place, internal.cuh: a
// bijective mix of v, so unscrambled R-MAT ids land balanced): its out-edges (keys stay global ids),
// with `reverse` its in-edges, and its tree nodes.
//
// Batches (insert / delete / query).  Any rank may pass any edges.  One kernel
// validates them and counts 16-B rows per (destination rank, section); the counts are exchanged; a
// scatter kernel packs the rows; one all-to-all-v moves them; a split kernel lays the received rows
// out for the single-GPU store kernels (store.cu).  An insert sends (u, v, w) to owner(u) for the
// out-store and, with the mirror, to owner(v) for the in-store (one row when both are the same rank);
// a delete always sends the edge to owner(v) as well -- the decremental tree call tests
// parent(v) == u there.  The routed rows stay on the device for the tree call that must
// follow with the same batch (ordering contract, checked by fingerprint).
//
// Tree updates run as UNITS: one cooperative kernel (k_part_unit), then one
// exchange of fixed-size per-peer blocks (grouped ncclSend/ncclRecv over NVLink / NVSwitch, or the
// caller's host transport).  A unit
//   (A) applies the messages of the last exchange -- relaxation candidates <x, <d, p>> (packed
//       atomicMin), invalidation requests <x, expected parent> (CAS), pull
//       requests <u, (w, x)> (the valid->invalid frontier through the in-edge mirror) and
//       invalid-vertex marks (the same frontier by the paper's scan);
//   (B) runs LOCAL frontier rounds to a fixpoint: a relaxation of a vertex held here is applied in
//       place, any other becomes a message in the ring of its owner;
//   (C) packs up to `cap` messages per peer into the send blocks, each with a header <messages in
//       this block, messages this rank sent, messages still pending here>.
// Every rank receives every rank's header, so every rank sees the same totals: an exchange that
// carried nothing with nothing pending anywhere ends the current phase on all ranks at the same
// unit, and the next unit starts the next phase (propagation -> valid->invalid frontier ->
// relaxation -> done) with no host involvement.  The host launches units and reads a per-unit mode
// word from mapped memory PIPE units behind, so the device never waits for the host between rounds.
// The fixpoint does not depend on the order of relaxations: results are
// bit-identical to one GPU.  On one rank the whole call is one launch (no messages exist).
#include <dlfcn.h>
#include <sched.h>

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <new>

#include <nccl.h>   // types and prototypes only: libnccl.so.2 is opened at run time (nccl_api)

#include "tree_common.cuh"

namespace mk {

enum MsgKind : uint32_t { MSG_RELAX = 0, MSG_PROP = 1, MSG_PULLREQ = 2, MSG_MARK = 3 };
enum PartMode : uint32_t {
  PM_DONE = 0, PM_SEED_STATIC = 1, PM_SEED_INC = 2, PM_SEED_DEC = 3, PM_RELAX = 4, PM_PROP = 5, PM_MARKS = 6,
  PM_CHECK = 7,     // ordering contract: fingerprint the batch this rank was given (no tree is touched)
  PM_VERDICT = 8    // every rank's verdict (exchanged in the headers): all good -> seed, else done
};
constexpr uint64_t HDR = 4;           // header messages (64 B) at the start of every exchange block
constexpr uint32_t FLAG_RING = 64;    // per-unit mode words in mapped host memory
constexpr uint32_t MAX_PIPE = 8;      // event ring: units in flight before the host reads one's mode word
#ifndef MEERKAT_PART_PIPE
#define MEERKAT_PART_PIPE 2
#endif
constexpr uint32_t PIPE = MEERKAT_PART_PIPE;   // <= MAX_PIPE; PIPE - 1 no-op units run past the last
constexpr uint64_t MAX_UNITS = 1ull << 22;
constexpr uint64_t DEFAULT_CAP = 16384;
constexpr int STATIC_CAP_MULT = 16;

struct PartCtrl {
  uint32_t mode, pad;
  unsigned long long fill;                          // index of the (empty) frontier after the last round
  unsigned long long units;                         // units run on this graph
  unsigned long long size[MAX_TREES][3];            // rotating frontier sizes (tree.cu's protocol)
  unsigned long long head[2][MEERKAT_MAX_RANKS];    // ring heads, double-buffered by unit parity
  unsigned long long tail[MEERKAT_MAX_RANKS];
  unsigned long long pull_n[MAX_TREES];
  unsigned long long local_rounds, prop_rounds;     // of the current call
  unsigned long long fp[2];                         // fingerprint of the batch given to the call (PM_CHECK)
};

struct PArgs {
  GraphDev G, R;                 // out-store; in-edge mirror (R.slabs == nullptr without one)
  TreeDev T[MAX_TREES];
  uint64_t* pull[MAX_TREES];     // pull item buffers
  uint32_t ntrees, start_mode, scan, pad;
  PartCtrl* pc;
  uint32_t* flags;               // device view of the mapped mode ring
  uint4* q;                      // per-peer message rings, q_cap messages each
  uint64_t q_cap;
  uint4* send;                   // ws blocks of blk messages
  uint4* recv;
  uint64_t blk, cap;             // block size; messages per block this call
  const uint32_t* bs;            // seed rows (incremental: routed out-rows; decremental: in-rows)
  const uint32_t* bd;
  const uint32_t* bw;
  uint64_t bn;
  const uint32_t* fs;            // the batch the caller passed to the tree call (ordering contract)
  const uint32_t* fd;
  const uint32_t* fw;
  uint64_t fn;
  unsigned long long fp_expect[2];   // fingerprint of the last mutation's batch on this rank
  uint32_t fp_w;                 // compare the weighted half too
  uint32_t fn_bad;               // the batch size differs from the mutation's
  uint32_t seed_mode;            // PM_SEED_INC / PM_SEED_DEC after a good verdict
  uint32_t chain;                // one rank: chain the phases in one launch (0: one unit per phase, as P > 1)
  uint32_t self_send;            // the own block goes to send (exchanged through NCCL) instead of recv
};

// A message: x = target row at the destination, y = tag (kind << 1 | tree), z/w = payload lo/hi.
__device__ __forceinline__ uint64_t hdr_word(const uint4* blk, int i) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(blk) + i);
}

// Warp-aggregated append to the per-peer rings: lanes with the same destination share one atomicAdd.
__device__ __forceinline__ void warp_emit(const PArgs& A, const unsigned long long* s_head, bool has, uint32_t peer,
                                          uint32_t row, uint32_t tag, uint64_t payload, Counters& c) {
  const uint32_t m = __ballot_sync(FULL, has);
  if (!m || !has) return;
  const uint32_t same = __match_any_sync(m, peer);
  const int lane = lane_id(), leader = __ffs(same) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&A.pc->tail[peer], (unsigned long long)__popc(same));
  base = __shfl_sync(same, base, leader);
  const unsigned long long pos = base + __popc(same & ((1u << lane) - 1u));
  if (pos - s_head[peer] >= A.q_cap) { c.err |= ERR_CAPACITY; return; }
  A.q[(uint64_t)peer * A.q_cap + pos % A.q_cap] = make_uint4(row, tag, (uint32_t)payload, (uint32_t)(payload >> 32));
}

__device__ __forceinline__ bool relax_packed(const TreeDev& T, uint32_t x, uint64_t cand, uint32_t epoch, Counters& c) {
  if (cand >= ld_cg_u64(T.node + x)) return false;
  const unsigned long long old = atomicMin(reinterpret_cast<unsigned long long*>(T.node + x), cand);
  if (cand >= old) return false;
  c.improved++;
  return atomicExch(T.stamp + x, epoch) != epoch;
}

__device__ __forceinline__ void count_hit(Counters& c, uint32_t k) {
  if (k == 0) c.hits[0]++;
  else c.hits[MAX_TREES - 1]++;
}

// The frontier slot a fill writes: buffer fr[f & 1], size slot f % 3.
#define FR_OF(A, k, f) (A).T[k].fr[(f) & 1]
#define SZ_OF(A, k, f) (&(A).pc->size[k][(f) % 3])

// ---- (A) received messages
__device__ void apply_recv(const PArgs& A, uint64_t f, uint32_t epoch, const unsigned long long* s_head, Counters& c) {
  const GraphDev& G = A.G;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t p = 0; p < G.ws; p++) {
    const uint4* blk = A.recv + (uint64_t)p * A.blk;
    const uint64_t n = hdr_word(blk, 0);
    const uint64_t trips = (n + nt - 1) / nt;
    for (uint64_t t = 0; t < trips; t++) {
      const uint64_t i = tid + t * nt;
      bool enq[MAX_TREES] = {}, inv[MAX_TREES] = {};
      bool emit = false;
      uint32_t row = 0, xg = 0, peer = 0, erow = 0, etag = 0;
      uint64_t epay = 0;
      if (i < n) {
        const uint4 msg = __ldcg(blk + HDR + i);
        row = msg.x;
        const uint32_t k = msg.y & 1u, kind = msg.y >> 1;
        const uint64_t pay = ((uint64_t)msg.w << 32) | msg.z;
        if (k >= A.ntrees || (kind != MSG_MARK && row >= G.V)) {
          c.err |= ERR_PARTITION;
        } else {
          const TreeDev& T = A.T[k];
          if (kind == MSG_RELAX) {
            enq[k] = relax_packed(T, row, pay, epoch, c);
          } else if (kind == MSG_PROP) {   // invalidate x if its parent is still the sender's vertex
            xg = g_global(G, row);
            const uint64_t cur = ld_cg_u64(T.node + row);
            if (cur != UNREACHED && (uint32_t)cur == (uint32_t)pay && xg != T.source &&
                atomicCAS(reinterpret_cast<unsigned long long*>(T.node + row), (unsigned long long)cur,
                          (unsigned long long)UNREACHED) == cur) {
              inv[k] = enq[k] = true;
            }
          } else if (kind == MSG_PULLREQ) {   // u = row is valid and reached: relax its edge into x
            const uint32_t ug = g_global(G, row);
            if (!bit_test(T.inval_bits, ug)) {
              const uint64_t nu = ld_cg_u64(T.node + row);
              if (nu != UNREACHED) {
                const uint64_t dist = (nu >> 32) + (uint32_t)(pay >> 32);
                if (dist >= INF_DIST) {
                  c.err |= ERR_OVERFLOW;
                } else {
                  count_hit(c, k);
                  peer = g_place(G, (uint32_t)pay, erow);
                  etag = (MSG_RELAX << 1) | k;
                  epay = (dist << 32) | ug;
                  emit = true;
                }
              }
            }
          } else {   // MSG_MARK: another rank's invalid vertex (scan frontier)
            const uint32_t x = (uint32_t)pay;
            if (x < G.Vg) atomicOr(T.inval_bits + (x >> 5), 1u << (x & 31));
          }
        }
      }
#pragma unroll
      for (int k = 0; k < MAX_TREES; k++) {
        if (k >= (int)A.ntrees) break;
        const bool h1[1] = {inv[k]};
        const uint32_t x1[1] = {xg};
        warp_mark_invalid<1>(A.T[k], h1, x1);
        warp_enqueue(G, A.T[k], FR_OF(A, k, f), SZ_OF(A, k, f), enq[k], row, c);
      }
      warp_emit(A, s_head, emit, peer, erow, etag, epay, c);
    }
  }
}

// ---- seeds
__device__ void seed_static(const PArgs& A, uint64_t f, uint32_t epoch, Counters& c) {
  const GraphDev& G = A.G;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t l = tid; l < G.V; l += nt) {
    const uint32_t vg = g_global(G, (uint32_t)l);
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++)
      if (k < (int)A.ntrees) A.T[k].node[l] = vg == A.T[k].source ? (uint64_t)vg : UNREACHED;
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {   // frontier = {SRC} on its owner
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (k >= (int)A.ntrees) break;
      uint32_t row = 0;
      const bool has = threadIdx.x == 0 && g_place(G, A.T[k].source, row) == G.rank;
      if (has) A.T[k].stamp[row] = epoch;
      warp_enqueue(G, A.T[k], FR_OF(A, k, f), SZ_OF(A, k, f), has, row, c);
    }
  }
}

// Incremental prologue over the routed rows (u, v, w) with u held here.
__device__ void seed_inc(const PArgs& A, uint64_t f, uint32_t epoch, const unsigned long long* s_head, Counters& c) {
  const GraphDev& G = A.G;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (A.bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    uint32_t u = 0, v = 0, w = 1, lu = 0, lv = 0, pv = 0;
    bool ok = false;
    if (i < A.bn) {
      u = A.bs[i];
      v = A.bd[i];
      if (A.bw) w = A.bw[i];
      c.batch++;
      ok = g_place(G, u, lu) == G.rank;
      pv = g_place(G, v, lv);
    }
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (k >= (int)A.ntrees) break;
      const TreeDev& T = A.T[k];
      bool enq = false, emit = false;
      uint64_t cand = 0;
      if (ok) {
        const uint64_t nu = ld_cg_u64(T.node + lu);
        if (nu != UNREACHED) {
          const uint64_t dist = (nu >> 32) + (T.unit ? 1u : w);
          if (pv == G.rank) enq = relax(T, lv, dist, u, epoch, c);
          else if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
          else { emit = true; cand = (dist << 32) | u; }
        }
      }
      warp_enqueue(G, T, FR_OF(A, k, f), SZ_OF(A, k, f), enq, lv, c);
      warp_emit(A, s_head, emit, pv, lv, (MSG_RELAX << 1) | k, cand, c);
    }
  }
}

// Decremental Invalidate (C4) over the routed rows (v, u) with v held here.
__device__ void seed_dec(const PArgs& A, uint64_t f, Counters& c) {
  const GraphDev& G = A.G;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t trips = (A.bn + nt - 1) / nt;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t i = tid + t * nt;
    uint32_t v = 0, u = 0, lv = 0;
    bool ok = false;
    if (i < A.bn) {
      v = A.bs[i];
      u = A.bd[i];
      c.batch++;
      ok = g_place(G, v, lv) == G.rank;
    }
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++) {
      if (k >= (int)A.ntrees) break;
      const TreeDev& T = A.T[k];
      bool has = false;
      if (ok && v != T.source) {
        const uint64_t cur = ld_cg_u64(T.node + lv);
        has = cur != UNREACHED && (uint32_t)cur == u &&
              atomicCAS(reinterpret_cast<unsigned long long*>(T.node + lv), (unsigned long long)cur,
                        (unsigned long long)UNREACHED) == cur;
        c.direct[k] += has;
      }
      const bool h1[1] = {has};
      const uint32_t x1[1] = {v};
      warp_mark_invalid<1>(T, h1, x1);
      warp_enqueue(G, T, FR_OF(A, k, f), SZ_OF(A, k, f), has, lv, c);
    }
  }
}

// ---- (B) one local round: expand both trees' frontier items (one 8-lane group per item)
template <bool MAP, int VISIT>
__device__ void p_expand(const PArgs& A, uint64_t r, uint64_t n0, uint64_t n1, const unsigned long long* s_head,
                         Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t N = n0 + n1;
  const uint64_t fn = r + 1;
  const uint32_t epoch = (uint32_t)fn;
  uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  uint32_t v = 0, vg = 0, slab = 0, du = 0, k = 0;
  auto fetch = [&]() -> bool {
    for (; it < N; it += ng) {
      k = it >= n0 ? 1u : 0u;
      const uint64_t item = A.T[k].fr[r & 1][it - (k ? n0 : 0)];
      v = (uint32_t)item;
      slab = (uint32_t)(item >> 32);
      if (l8 == 0) c.items++;
      if (VISIT == PROPAGATE) { vg = g_global(G, v); return true; }
      uint64_t nv = 0;
      if (l8 == 0) nv = ld_cg_u64(A.T[k].node + v);
      nv = __shfl_sync(0xFFu << (lane & 24), nv, 0, GROUP);
      if (nv != UNREACHED) { du = (uint32_t)(nv >> 32); vg = g_global(G, v); return true; }
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
    // phase-wise over the slab's keys (as tree.cu's expand): placement, then every load / atomic of
    // a phase for all keys before any result is consumed, then one enqueue per tree and the messages
    const TreeDev& T = A.T[k];
    uint32_t xs[NK], rows[NK], peer[NK];
    bool loc[NK], rem[NK], has[NK];
    uint64_t pay[NK];
    uint2 mv[NK];
#pragma unroll
    for (int kk = 0; kk < NK; kk++) {
      xs[kk] = F::key(d, kk);
      const bool live = active && F::valid_cell(l8, kk) && xs[kk] < G.Vg;
      peer[kk] = 0; rows[kk] = 0; pay[kk] = 0; has[kk] = false;
      mv[kk] = make_uint2(INVALID_SLAB, 0);
      if (live) { c.visited++; peer[kk] = g_place(G, xs[kk], rows[kk]); }
      loc[kk] = live && peer[kk] == G.rank;
      rem[kk] = live && peer[kk] != G.rank;
      if (VISIT == RELAX && live) {
        const uint64_t dist = (uint64_t)du + (T.unit ? 1u : F::weight(d, kk));
        if (dist >= INF_DIST) { c.err |= ERR_OVERFLOW; loc[kk] = rem[kk] = false; }
        pay[kk] = (dist << 32) | vg;
      } else if (VISIT == PROPAGATE) {
        pay[kk] = vg;
      }
    }
    uint64_t cur[NK];
#pragma unroll
    for (int kk = 0; kk < NK; kk++) cur[kk] = loc[kk] ? ld_cg_u64(T.node + rows[kk]) : UNREACHED;
    if (VISIT == RELAX) {
      // probe passed -> atomicMin, stamp exchange and vmeta together (enqueue iff the stamp was won;
      // tree.cu's expand explains why that enqueues an improved x exactly once)
      unsigned long long old[NK];
      uint32_t st[NK];
      bool go[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        go[kk] = loc[kk] && pay[kk] < cur[kk];
        old[kk] = go[kk] ? atomicMin(reinterpret_cast<unsigned long long*>(T.node + rows[kk]),
                                     (unsigned long long)pay[kk]) : 0ull;
        st[kk] = go[kk] ? atomicExch(T.stamp + rows[kk], epoch) : epoch;
        if (go[kk]) mv[kk] = __ldcg(G.vmeta + rows[kk]);
      }
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        if (go[kk] && pay[kk] < old[kk]) c.improved++;
        has[kk] = st[kk] != epoch;
      }
    } else {   // children of the invalid vertex v
      unsigned long long oc[NK];
      bool child[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) {
        child[kk] = loc[kk] && cur[kk] != UNREACHED && (uint32_t)cur[kk] == vg && xs[kk] != T.source;
        oc[kk] = child[kk] ? atomicCAS(reinterpret_cast<unsigned long long*>(T.node + rows[kk]),
                                       (unsigned long long)cur[kk], (unsigned long long)UNREACHED) : 0ull;
        if (child[kk]) mv[kk] = __ldcg(G.vmeta + rows[kk]);
      }
#pragma unroll
      for (int kk = 0; kk < NK; kk++) has[kk] = child[kk] && oc[kk] == cur[kk];
    }
#pragma unroll
    for (int k2 = 0; k2 < MAX_TREES; k2++) {
      if (k2 >= (int)A.ntrees) break;
      const bool mine = k == (uint32_t)k2;
      bool h2[NK];
#pragma unroll
      for (int kk = 0; kk < NK; kk++) h2[kk] = has[kk] && mine;
      if (VISIT == PROPAGATE) warp_mark_enqueue_multi<NK>(A.T[k2], FR_OF(A, k2, fn), SZ_OF(A, k2, fn), h2, xs, rows, mv, c);
      else warp_enqueue_multi<NK>(A.T[k2], FR_OF(A, k2, fn), SZ_OF(A, k2, fn), h2, rows, mv, c);
    }
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
      warp_emit(A, s_head, rem[kk], peer[kk], rows[kk], ((VISIT == RELAX ? MSG_RELAX : MSG_PROP) << 1) | k, pay[kk], c);
    const uint32_t nxt = __shfl_sync(FULL, d.w, (lane & 24) + GROUP - 1);
    if (active) {
      if (nxt != INVALID_SLAB) slab = nxt;
      else { it += ng; active = fetch(); }
    }
  }
}

// ---- valid->invalid frontier through the mirror: items (invalid x, in-bucket)
__device__ void pull_enqueue(const PArgs& A, Counters& c) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) {
    if (k >= (int)A.ntrees) break;
    const uint64_t n = __ldcg(&A.T[k].ctrl->inval_n);
    const uint64_t trips = (n + nt - 1) / nt;
    for (uint64_t t = 0; t < trips; t++) {
      const uint64_t i = tid + t * nt;
      uint32_t row = 0;
      const bool has = i < n;
      if (has) g_place(A.G, A.T[k].inval_list[i], row);
      warp_enqueue(A.R, A.T[k], A.pull[k], &A.pc->pull_n[k], has, row, c);
    }
  }
}

// In-edges (u -> x) of the invalid x: u held here -> relax now (the group's candidates min-reduced,
// one atomicMin per slab, as tree.cu's PULL); else a pull request to owner(u).
template <bool MAP>
__device__ void pull_walk(const PArgs& A, uint64_t f, const unsigned long long* s_head, Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t n0 = __ldcg(&A.pc->pull_n[0]), n1 = A.ntrees > 1 ? __ldcg(&A.pc->pull_n[1]) : 0;
  const uint64_t N = n0 + n1;
  const uint32_t epoch = (uint32_t)f;
  uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  uint32_t x = 0, xg = 0, slab = 0, k = 0;
  auto fetch = [&]() -> bool {
    for (; it < N; it += ng) {
      k = it >= n0 ? 1u : 0u;
      const uint64_t item = A.pull[k][it - (k ? n0 : 0)];
      x = (uint32_t)item;
      slab = (uint32_t)(item >> 32);
      xg = g_global(G, x);
      if (l8 == 0) c.items++;
      return true;
    }
    return false;
  };
  bool active = fetch();
  while (__any_sync(FULL, active)) {
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    const TreeDev& T = A.T[k];
    uint64_t nx = 0;
    uint32_t sx = 0;
    if (active) {
      d = ld_slab_ro(slab_ptr(A.R, slab), l8);
      if (l8 == 0) { c.slabs++; nx = ld_cg_u64(T.node + x); sx = __ldcg(T.stamp + x); }
    }
    uint32_t us[NK], urow[NK], peer[NK], w[NK], bw[NK];
    bool loc[NK], rem[NK];
    uint64_t nu[NK];
#pragma unroll
    for (int kk = 0; kk < NK; kk++) {
      us[kk] = F::key(d, kk);
      const bool live = active && F::valid_cell(l8, kk) && us[kk] < G.Vg;
      w[kk] = T.unit ? 1u : (MAP ? F::weight(d, kk) : 1u);
      peer[kk] = 0; urow[kk] = 0;
      if (live) { c.visited++; peer[kk] = g_place(G, us[kk], urow[kk]); }
      loc[kk] = live && peer[kk] == G.rank;
      rem[kk] = live && peer[kk] != G.rank;
      bw[kk] = loc[kk] ? __ldcg(T.inval_bits + (us[kk] >> 5)) : 0u;
      nu[kk] = loc[kk] ? ld_cg_u64(T.node + urow[kk]) : UNREACHED;
    }
    uint64_t best = UNREACHED;
#pragma unroll
    for (int kk = 0; kk < NK; kk++) {
      if (loc[kk] && !((bw[kk] >> (us[kk] & 31)) & 1u) && nu[kk] != UNREACHED) {   // valid and reached (C15)
        count_hit(c, k);
        const uint64_t dist = (nu[kk] >> 32) + w[kk];
        if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
        else best = min(best, (dist << 32) | us[kk]);
      }
    }
    best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 1));
    best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 2));
    best = min(best, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)best, 4));
    bool hv[1] = {false};
    uint32_t xv[1] = {x};
    uint2 m1[1] = {make_uint2(INVALID_SLAB, 0)};
    if (l8 == 0 && best != UNREACHED && best < nx) {   // atomicMin, stamp and vmeta together
      const unsigned long long o = atomicMin(reinterpret_cast<unsigned long long*>(T.node + x),
                                             (unsigned long long)best);
      const uint32_t st = sx != epoch ? atomicExch(T.stamp + x, epoch) : epoch;
      if (sx != epoch) m1[0] = __ldcg(G.vmeta + x);
      if (best < o) c.improved++;
      hv[0] = st != epoch;
    }
#pragma unroll
    for (int k2 = 0; k2 < MAX_TREES; k2++) {
      if (k2 >= (int)A.ntrees) break;
      const bool h2[1] = {hv[0] && k == (uint32_t)k2};
      warp_enqueue_multi<1>(A.T[k2], FR_OF(A, k2, f), SZ_OF(A, k2, f), h2, xv, m1, c);
    }
#pragma unroll
    for (int kk = 0; kk < NK; kk++)
      warp_emit(A, s_head, rem[kk], peer[kk], urow[kk], (MSG_PULLREQ << 1) | k, ((uint64_t)w[kk] << 32) | xg, c);
    const uint32_t nxt = __shfl_sync(FULL, d.w, (lane & 24) + GROUP - 1);
    if (active) {
      if (nxt != INVALID_SLAB) slab = nxt;
      else { it += ng; active = fetch(); }
    }
  }
}

// ---- valid->invalid frontier by the paper's scan: this rank's invalid vertices go to
// every other rank as marks; then every rank streams its own slabs against the union.
__device__ void emit_marks(const PArgs& A, const unsigned long long* s_head, Counters& c) {
  const GraphDev& G = A.G;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) {
    if (k >= (int)A.ntrees) break;
    const uint64_t n = __ldcg(&A.T[k].ctrl->inval_n);
    const uint64_t total = n * (G.ws - 1);
    const uint64_t trips = (total + nt - 1) / nt;
    for (uint64_t t = 0; t < trips; t++) {
      const uint64_t i = tid + t * nt;
      const bool has = i < total;
      uint32_t peer = 0, x = 0;
      if (has) {
        x = A.T[k].inval_list[i / (G.ws - 1)];
        peer = (uint32_t)(i % (G.ws - 1));
        if (peer >= G.rank) peer++;
      }
      warp_emit(A, s_head, has, peer, 0, (MSG_MARK << 1) | k, x, c);
    }
  }
}

template <bool MAP>
__device__ void p_scan(const PArgs& A, uint64_t f, const unsigned long long* s_head, Counters& c) {
  using F = Frag<MAP>;
  constexpr int NK = F::NK;
  const GraphDev& G = A.G;
  const int lane = lane_id(), l8 = lane & 7;
  const uint64_t ng = ((uint64_t)gridDim.x * blockDim.x) / GROUP;
  const uint64_t n_slabs = G.H + min((unsigned long long)G.P, __ldcg(&G.ctrl->pool_top));
  const uint32_t epoch = (uint32_t)f;
  const uint64_t g0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / GROUP;
  const uint64_t trips = (n_slabs + ng - 1) / ng;
  for (uint64_t t = 0; t < trips; t++) {
    const uint64_t s = g0 + t * ng;
    uint4 d = make_uint4(EMPTY_KEY, EMPTY_KEY, EMPTY_KEY, INVALID_SLAB);
    uint32_t ul = NO_OWNER;
    if (s < n_slabs) {
      d = ld_slab_ro(slab_ptr(G, (uint32_t)s), l8);
      ul = __ldg(G.owner + s);
      if (l8 == 0) c.scan_slabs++;
    }
    const uint32_t ug = ul == NO_OWNER ? NO_OWNER : g_global(G, ul);
#pragma unroll
    for (int kk = 0; kk < NK; kk++) {
      const uint32_t x = F::key(d, kk);
      const bool live = ul != NO_OWNER && F::valid_cell(l8, kk) && x < G.Vg;
#pragma unroll
      for (int k = 0; k < MAX_TREES; k++) {
        if (k >= (int)A.ntrees) break;
        const TreeDev& T = A.T[k];
        bool enq = false, emit = false;
        uint32_t row = 0, peer = 0;
        uint64_t pay = 0;
        if (live && bit_test(T.inval_bits, x) && !bit_test(T.inval_bits, ug)) {
          const uint64_t nu = ld_cg_u64(T.node + ul);
          if (nu != UNREACHED) {
            c.hits[k]++;
            const uint64_t dist = (nu >> 32) + (T.unit ? 1u : F::weight(d, kk));
            peer = g_place(G, x, row);
            if (peer == G.rank) enq = relax(T, row, dist, ug, epoch, c);
            else if (dist >= INF_DIST) c.err |= ERR_OVERFLOW;
            else { emit = true; pay = (dist << 32) | ug; }
          }
        }
        warp_enqueue(G, T, FR_OF(A, k, f), SZ_OF(A, k, f), enq, row, c);
        warp_emit(A, s_head, emit, peer, row, (MSG_RELAX << 1) | k, pay, c);
      }
    }
  }
}

// End of a decremental call: clear the invalid marks (own list; with the scan, every rank's).
__device__ void p_finish(const PArgs& A) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) {
    if (k >= (int)A.ntrees) break;
    const TreeDev& T = A.T[k];
    if (A.scan) {
      const uint64_t words = ((uint64_t)A.G.Vg + 31) / 32;
      for (uint64_t i = tid; i < words; i += nt) T.inval_bits[i] = 0;
    } else {
      const uint64_t n = __ldcg(&T.ctrl->inval_n);
      for (uint64_t i = tid; i < n; i += nt) {
        const uint32_t x = T.inval_list[i];
        atomicAnd(T.inval_bits + (x >> 5), ~(1u << (x & 31)));
      }
    }
  }
}

// ---- the unit
template <bool MAP>
__global__ void __launch_bounds__(TREE_BLOCK, TREE_MINB) k_part_unit(const __grid_constant__ PArgs A) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long s_head[MEERKAT_MAX_RANKS];
  Counters c;
  PartCtrl* pc = A.pc;
  const GraphDev& G = A.G;
  const uint32_t ws = G.ws;
  const unsigned long long unit = __ldcg(&pc->units);
  const uint32_t hpar = (uint32_t)(unit & 1);
  for (uint32_t p = threadIdx.x; p < ws; p += blockDim.x) s_head[p] = __ldcg(&pc->head[hpar][p]);
  __syncthreads();
  uint32_t mode = A.start_mode ? A.start_mode : __ldcg(&pc->mode);
  unsigned long long r = __ldcg(&pc->fill);
  bool have_recv = A.start_mode == 0, synced = false;
  uint32_t lrounds = 0, prounds = 0;
  uint32_t verdict = 0;   // this rank's ordering-contract verdict (ERR_STATE: a different batch)
  while (mode != PM_DONE) {
    const uint64_t f = r + 1;   // the slot this fill writes (zero by the round protocol)
    const uint32_t epoch = (uint32_t)f;
    if (mode == PM_CHECK) {   // the batch must be the one this rank's last mutation applied
      const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
      uint64_t fa = 0, fb = 0;
      for (uint64_t i = tid; i < A.fn; i += nt) fp_edge(A.fs[i], A.fd[i], A.fw ? A.fw[i] : 0u, fa, fb);
      block_add2_u64(&pc->fp[0], fa, fb);
      grid.sync();
      synced = true;
      const bool bad = A.fn_bad || __ldcg(&pc->fp[0]) != A.fp_expect[0] ||
                       (A.fp_w && __ldcg(&pc->fp[1]) != A.fp_expect[1]);
      verdict = bad ? (uint32_t)ERR_STATE : 0u;
      mode = PM_VERDICT;
      if (ws > 1 || !A.chain) break;   // the verdicts travel in the headers
      continue;
    }
    if (mode == PM_VERDICT) {
      uint32_t any = verdict;
      if (have_recv)
        for (uint32_t p = 0; p < ws; p++) any |= (uint32_t)hdr_word(A.recv + (uint64_t)p * A.blk, 4);
      have_recv = false;
      if (any) {   // some rank was given another batch: no tree is touched anywhere
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&G.ctrl->err, (unsigned)ERR_STATE);
        mode = PM_DONE;
        break;
      }
      mode = A.seed_mode;
    }
    if (mode == PM_SEED_STATIC || mode == PM_SEED_INC || mode == PM_SEED_DEC) {
      if (blockIdx.x == 0 && threadIdx.x < MAX_TREES) pc->pull_n[threadIdx.x] = 0;
      if (mode == PM_SEED_STATIC) seed_static(A, f, epoch, c);
      else if (mode == PM_SEED_INC) seed_inc(A, f, epoch, s_head, c);
      else seed_dec(A, f, c);
      mode = mode == PM_SEED_DEC ? PM_PROP : PM_RELAX;
    } else {
      bool quiet = true;
      if (have_recv) {
        unsigned long long tot = 0;
        for (uint32_t p = 0; p < ws; p++) {
          const uint4* blk = A.recv + (uint64_t)p * A.blk;
          tot += hdr_word(blk, 1) + hdr_word(blk, 2);
        }
        quiet = tot == 0;
        if (!quiet) apply_recv(A, f, epoch, s_head, c);
        have_recv = false;
      }
      if (quiet) {   // the phase is over on every rank
        if (mode == PM_PROP) {
          if (!A.scan) {
            pull_enqueue(A, c);
            grid.sync();
            pull_walk<MAP>(A, f, s_head, c);
            mode = PM_RELAX;
          } else if (ws > 1) {
            emit_marks(A, s_head, c);
            mode = PM_MARKS;
          } else {
            p_scan<MAP>(A, f, s_head, c);
            mode = PM_RELAX;
          }
        } else if (mode == PM_MARKS) {
          p_scan<MAP>(A, f, s_head, c);
          mode = PM_RELAX;
        } else {
          p_finish(A);
          mode = PM_DONE;
          break;
        }
      }
    }
    grid.sync();
    synced = true;
    r = f;
    for (;;) {   // (B) local rounds to a fixpoint
      const uint64_t n0 = __ldcg(SZ_OF(A, 0, r));
      const uint64_t n1 = A.ntrees > 1 ? __ldcg(SZ_OF(A, 1, r)) : 0;
      if (blockIdx.x == 0 && threadIdx.x < A.ntrees) pc->size[threadIdx.x][(r + 2) % 3] = 0;
      if (n0 + n1 == 0) break;
      if (mode == PM_PROP) { p_expand<MAP, PROPAGATE>(A, r, n0, n1, s_head, c); prounds++; }
      else { p_expand<MAP, RELAX>(A, r, n0, n1, s_head, c); lrounds++; }
      grid.sync();
      r++;
    }
    if (ws > 1 || !A.chain) break;   // an exchange must follow; one rank: nothing was sent, the phase is over
  }
  if (!synced) grid.sync();   // every block has read pc before block 0 rewrites it
  // (C) pack up to cap messages per peer
  unsigned long long sent = 0, pend = 0;
  for (uint32_t p = 0; p < ws; p++) {
    const unsigned long long t = __ldcg(&pc->tail[p]), h = s_head[p];
    const unsigned long long m = min((unsigned long long)A.cap, t - h);
    sent += m;
    pend += t - h - m;
  }
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint32_t p = 0; p < ws; p++) {
    const unsigned long long t = __ldcg(&pc->tail[p]), h = s_head[p];
    const unsigned long long m = min((unsigned long long)A.cap, t - h);
    uint4* dst = (p == G.rank && !A.self_send ? A.recv : A.send) + (uint64_t)p * A.blk + HDR;
    const uint4* ring = A.q + (uint64_t)p * A.q_cap;
    for (uint64_t j = tid; j < m; j += nt) dst[j] = ring[(h + j) % A.q_cap];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (uint32_t p = 0; p < ws; p++) {
      const unsigned long long t = __ldcg(&pc->tail[p]), h = s_head[p];
      const unsigned long long m = min((unsigned long long)A.cap, t - h);
      unsigned long long* hd =
          reinterpret_cast<unsigned long long*>((p == G.rank && !A.self_send ? A.recv : A.send) + (uint64_t)p * A.blk);
      hd[0] = m; hd[1] = sent; hd[2] = pend; hd[3] = mode; hd[4] = verdict;
      pc->head[hpar ^ 1][p] = h + m;
    }
    pc->mode = mode;
    pc->fill = r;
    pc->units = unit + 1;
    if (A.start_mode) { pc->local_rounds = lrounds; pc->prop_rounds = prounds; }
    else { pc->local_rounds += lrounds; pc->prop_rounds += prounds; }
#pragma unroll
    for (int k = 0; k < MAX_TREES; k++)
      if (k < (int)A.ntrees) { A.T[k].ctrl->rounds = pc->local_rounds; A.T[k].ctrl->prop_rounds = pc->prop_rounds; }
    __threadfence_system();
    *reinterpret_cast<volatile uint32_t*>(A.flags + unit % FLAG_RING) = mode;
  }
  // counters: the per-call ones into tree 0, the per-tree ones (frontier edges, direct) into each
#pragma unroll
  for (int k = 0; k < MAX_TREES; k++) {
    if (k >= (int)A.ntrees) break;
    flush_counters(G, A.T[k], c, k, false, 0, 0);
    c.items = c.slabs = c.visited = c.improved = c.scan_slabs = c.batch = 0;
    c.err = 0;
  }
}

// ---- batch routing
// Sections of a destination's rows: 0 = out-store only, 1 = both stores, 2 = in-store only.
struct RouteArgs {
  const uint32_t* s;
  const uint32_t* d;
  const uint32_t* w;
  uint64_t n;
  uint32_t V, bits, ws, rank;
  uint32_t need_in;     // also send (v, u) rows to owner(v)
  uint32_t check_w;     // weighted insert: w in [1, 2^31)
  uint32_t aux_index;   // query: row.w = input index
  unsigned long long* counts;   // [ws * 3]
  unsigned long long* cursor;   // [ws * 3], scatter
  unsigned long long* fp;       // [2] batch fingerprint
  unsigned int* err;
  uint4* rows;
};

__device__ __forceinline__ bool route_row(const RouteArgs& R, uint64_t i, uint32_t& s, uint32_t& d, uint32_t& w,
                                          uint32_t& po, uint32_t& pi) {
  s = R.s[i];
  d = R.d[i];
  w = R.w ? R.w[i] : 0u;
  if (s >= R.V || d >= R.V) { atomicOr(R.err, (unsigned)ERR_RANGE); return false; }
  if (R.check_w && (w == 0 || w >= W_LIMIT)) { atomicOr(R.err, (unsigned)ERR_WEIGHT); return false; }
  uint32_t row;
  po = pm_place(s, R.V, R.bits, R.ws, row);
  pi = R.need_in ? pm_place(d, R.V, R.bits, R.ws, row) : po;
  return true;
}

__global__ void k_route_count(const RouteArgs R) {
  __shared__ unsigned int h[MEERKAT_MAX_RANKS * 3];
  for (uint32_t i = threadIdx.x; i < R.ws * 3; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint64_t fa = 0, fb = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R.n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s, d, w, po, pi;
    const bool ok = route_row(R, i, s, d, w, po, pi);
    fp_edge(s, d, w, fa, fb);
    if (!ok) continue;
    if (!R.need_in) atomicAdd(&h[po * 3 + 0], 1u);
    else if (po == pi) atomicAdd(&h[po * 3 + 1], 1u);
    else { atomicAdd(&h[po * 3 + 0], 1u); atomicAdd(&h[pi * 3 + 2], 1u); }
  }
  block_add2_u64(R.fp, fa, fb);
  for (uint32_t i = threadIdx.x; i < R.ws * 3; i += blockDim.x)
    if (h[i]) atomicAdd(&R.counts[i], (unsigned long long)h[i]);
}

__global__ void k_route_scatter(const RouteArgs R) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R.n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t s, d, w, po, pi;
    if (!route_row(R, i, s, d, w, po, pi)) continue;
    const uint32_t aux = R.aux_index ? (uint32_t)i : w;
    if (!R.need_in) {
      R.rows[atomicAdd(&R.cursor[po * 3 + 0], 1ull)] = make_uint4(s, d, aux, 0);
    } else if (po == pi) {
      R.rows[atomicAdd(&R.cursor[po * 3 + 1], 1ull)] = make_uint4(s, d, aux, 0);
    } else {
      R.rows[atomicAdd(&R.cursor[po * 3 + 0], 1ull)] = make_uint4(s, d, aux, 0);
      R.rows[atomicAdd(&R.cursor[pi * 3 + 2], 1ull)] = make_uint4(s, d, aux, 0);
    }
  }
}

__global__ void k_fingerprint(const uint32_t* s, const uint32_t* d, const uint32_t* w, uint64_t n,
                              unsigned long long* fp) {
  uint64_t fa = 0, fb = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    fp_edge(s[i], d[i], w ? w[i] : 0u, fa, fb);
  block_add2_u64(fp, fa, fb);
}

// Received rows -> out-store rows (u, v, w) and in-store rows (v, u, w), per source segment
// [section 0 | section 1 | section 2].
struct SplitArgs {
  const uint4* rows;
  uint64_t base[MEERKAT_MAX_RANKS + 1];   // start of each source's segment (rows)
  uint64_t n0[MEERKAT_MAX_RANKS], n1[MEERKAT_MAX_RANKS];
  uint64_t out_base[MEERKAT_MAX_RANKS], in_base[MEERKAT_MAX_RANKS];
  uint32_t ws;
  uint32_t* os; uint32_t* od; uint32_t* ow;
  uint32_t* is; uint32_t* id; uint32_t* iw;
};

__global__ void k_route_split(const __grid_constant__ SplitArgs S) {
  const uint64_t total = S.base[S.ws];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = S.ws;   // source segment of row i: last q with base[q] <= i
    while (hi - lo > 1) { const uint32_t mid = (lo + hi) / 2; if (S.base[mid] <= i) lo = mid; else hi = mid; }
    const uint64_t j = i - S.base[lo];
    const uint4 r = S.rows[i];
    if (j < S.n0[lo] + S.n1[lo]) {
      const uint64_t o = S.out_base[lo] + j;
      S.os[o] = r.x; S.od[o] = r.y; if (S.ow) S.ow[o] = r.z;
    }
    if (j >= S.n0[lo] && S.is) {
      const uint64_t o = S.in_base[lo] + (j - S.n0[lo]);
      S.is[o] = r.y; S.id[o] = r.x; if (S.iw) S.iw[o] = r.z;
    }
  }
}

// Query answers back at the asking rank: rows (found, w, index).
__global__ void k_query_reply(const uint8_t* found, const uint32_t* w, const uint32_t* idx, uint64_t n, uint4* out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = make_uint4(found[i], w[i], idx[i], 0);
}
__global__ void k_query_scatter(const uint4* rows, uint64_t n, uint8_t* found, uint32_t* w) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 r = rows[i];
    found[r.z] = (uint8_t)r.x;
    if (w) w[r.z] = r.y;
  }
}

// Global hints -> this rank's rows.
__global__ void k_gather_rows(const uint32_t* global, uint32_t* local, uint32_t n_local, uint32_t rank, uint32_t V,
                              uint32_t bits, uint32_t ws) {
  for (uint64_t l = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_local; l += (uint64_t)gridDim.x * blockDim.x)
    local[l] = global[pm_global((uint32_t)l, rank, V, bits, ws)];
}

// All ranks' nodes (segment q = rank q's rows) -> global id order.
__global__ void k_unpermute(const uint64_t* in, const uint64_t* base, uint32_t ws, uint32_t V, uint32_t bits,
                            uint64_t* out) {
  const uint64_t total = base[ws];
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = ws;
    while (hi - lo > 1) { const uint32_t mid = (lo + hi) / 2; if (base[mid] <= i) lo = mid; else hi = mid; }
    out[pm_global((uint32_t)(i - base[lo]), lo, V, bits, ws)] = in[i];
  }
}

// ------------------------------------------------------------------ NCCL, opened at run time

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommAbort)(ncclComm_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
};

static NcclApi* nccl_api() {
  static NcclApi a;
  static bool tried = false;
  if (tried) return a.ok ? &a : nullptr;
  tried = true;
  // the process's NCCL when one is loaded (torch's), else MEERKAT_NCCL_LIB, else the loader's search
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) if (const char* p = std::getenv("MEERKAT_NCCL_LIB")) h = dlopen(p, RTLD_NOW);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
  if (!h) return nullptr;
  bool ok = true;
  auto sym = [&](const char* n) { void* f = dlsym(h, n); ok = ok && f; return f; };
  a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
  a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
  a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
  a.CommAbort = (decltype(a.CommAbort))sym("ncclCommAbort");
  a.CommGetAsyncError = (decltype(a.CommGetAsyncError))sym("ncclCommGetAsyncError");
  a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
  a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
  a.Send = (decltype(a.Send))sym("ncclSend");
  a.Recv = (decltype(a.Recv))sym("ncclRecv");
  a.ok = ok;
  return ok ? &a : nullptr;
}

// ------------------------------------------------------------------ host state

struct PartState {
  ncclComm_t comm = nullptr;
  bool nccl_failed = false;
  meerkat_exchange_fn xfn = nullptr;
  void* xctx = nullptr;
  uint64_t cap_dyn = DEFAULT_CAP, cap_static = DEFAULT_CAP * STATIC_CAP_MULT, blk = 0;
  uint4* send = nullptr;
  uint4* recv = nullptr;
  uint4* q = nullptr;
  uint64_t q_cap = 0;
  PartCtrl* pc = nullptr;
  uint32_t* hflags = nullptr;   // mapped host ring
  uint32_t* dflags = nullptr;
  uint64_t units = 0;
  bool dirty = false;
  cudaEvent_t ev[2 * MAX_PIPE] = {};
  int bps = 0;
  // routing
  uint4* rsend = nullptr; uint64_t rsend_cap = 0;   // rows
  uint4* rrecv = nullptr; uint64_t rrecv_cap = 0;
  uint32_t* rows = nullptr; uint64_t rows_cap = 0;  // 6 arrays of rows_cap: out s/d/w, in s/d/w
  uint64_t n_out = 0, n_in = 0;
  unsigned long long* dscr = nullptr;   // counts[3 * 64] | cursor[3 * 64] | fp[2] | err | pad
  unsigned long long* hscr = nullptr;   // pinned mirror
  uint64_t fp_last[2] = {0, 0};
  uint64_t n_last = 0;
  // host transport staging
  char* hsend = nullptr; char* hrecv = nullptr; size_t hbytes = 0;
  // collectives scratch (device)
  uint64_t* dcoll = nullptr; size_t dcoll_bytes = 0;
  uint64_t* hcoll = nullptr;   // pinned, COLL_WORDS
};

constexpr size_t COLL_WORDS = (size_t)MEERKAT_MAX_RANKS * MEERKAT_MAX_RANKS * 3;   // allgather_small capacity
constexpr int SCR_COUNTS = 0, SCR_CURSOR = 3 * MEERKAT_MAX_RANKS, SCR_FP = 6 * MEERKAT_MAX_RANKS,
              SCR_ERR = SCR_FP + 2, SCR_WORDS = SCR_FP + 4;

static meerkat_status st_of(cudaError_t e) { return e == cudaSuccess ? MEERKAT_OK : MEERKAT_E_CUDA; }
static unsigned grid_of(meerkat_graph* g, uint64_t threads) {
  const uint64_t b = (threads + 255) / 256;
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, (uint64_t)g->sm_count * 8));
}
static uint32_t rows_of(const meerkat_graph* g, uint32_t rank) { return (g->V - rank + g->ws - 1) / g->ws; }

static meerkat_status nccl_check(meerkat_graph* g) {   // asynchronous communicator errors
  PartState* ps = g->part;
  if (!ps->comm) return ps->nccl_failed ? MEERKAT_E_NCCL : MEERKAT_OK;
  NcclApi* api = nccl_api();
  ncclResult_t r = ncclSuccess;
  if (api->CommGetAsyncError(ps->comm, &r) != ncclSuccess || (r != ncclSuccess && r != ncclInProgress)) {
    api->CommAbort(ps->comm);
    ps->comm = nullptr;
    ps->nccl_failed = true;
    return MEERKAT_E_NCCL;
  }
  return MEERKAT_OK;
}

static cudaError_t ensure_host(PartState* ps, size_t bytes) {
  if (ps->hbytes >= bytes) return cudaSuccess;
  if (ps->hsend) cudaFreeHost(ps->hsend);
  if (ps->hrecv) cudaFreeHost(ps->hrecv);
  ps->hsend = ps->hrecv = nullptr;
  ps->hbytes = 0;
  const size_t cap = std::max<size_t>(bytes, 1 << 20);
  cudaError_t e = cudaMallocHost(&ps->hsend, cap);
  if (e == cudaSuccess) e = cudaMallocHost(&ps->hrecv, cap);
  if (e == cudaSuccess) ps->hbytes = cap;
  return e;
}

// All-to-all-v of device buffers: segment p of `send` (sb[p] bytes at offset so[p]) goes to rank p and
// lands there as segment `rank`; recv segment q (rb[q] bytes at ro[q]) comes from rank q.  NCCL:
// stream-ordered grouped send/recv.  Host transport: staged through pinned memory (synchronous).
// MEERKAT_PART_NCCL_SELF=1 (tests): a rank's own segments and unit block also go through ncclSend /
// ncclRecv to itself, so a one-GPU box drives every NCCL call of the P > 1 path with real data.
static bool nccl_self() {
  static int on = -1;
  if (on < 0) on = std::getenv("MEERKAT_PART_NCCL_SELF") ? 1 : 0;
  return on == 1;
}

static bool trace_on() {
  static int on = -1;
  if (on < 0) on = std::getenv("MEERKAT_PART_TRACE") ? 1 : 0;
  return on == 1;
}

static meerkat_status xchg(meerkat_graph* g, const void* send, const uint64_t* sb, const uint64_t* so, void* recv,
                           const uint64_t* rb, const uint64_t* ro) {
  PartState* ps = g->part;
  const uint32_t ws = g->ws, me = g->rank;
  if (trace_on()) {
    fprintf(stderr, "[part r%u] xchg sb", me);
    for (uint32_t p = 0; p < ws; p++) fprintf(stderr, " %llu", (unsigned long long)sb[p]);
    fprintf(stderr, " rb");
    for (uint32_t p = 0; p < ws; p++) fprintf(stderr, " %llu", (unsigned long long)rb[p]);
    fprintf(stderr, "\n");
  }
  const char* s8 = static_cast<const char*>(send);
  char* r8 = static_cast<char*>(recv);
  cudaError_t e = cudaSuccess;
  const bool self_nccl = ps->comm && nccl_self();
  if (sb[me] && !self_nccl) e = cudaMemcpyAsync(r8 + ro[me], s8 + so[me], sb[me], cudaMemcpyDeviceToDevice, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (ws == 1 && !self_nccl) return MEERKAT_OK;
  if (ps->comm) {
    NcclApi* api = nccl_api();
    bool ok = api->GroupStart() == ncclSuccess;
    for (uint32_t p = 0; p < ws && ok; p++) {
      if (p == me && !self_nccl) continue;
      if (sb[p]) ok = api->Send(s8 + so[p], sb[p], ncclUint8, (int)p, ps->comm, g->stream) == ncclSuccess;
      if (ok && rb[p]) ok = api->Recv(r8 + ro[p], rb[p], ncclUint8, (int)p, ps->comm, g->stream) == ncclSuccess;
    }
    ok = (api->GroupEnd() == ncclSuccess) && ok;
    return ok ? MEERKAT_OK : MEERKAT_E_NCCL;
  }
  if (!ps->xfn) return MEERKAT_E_NCCL;
  uint64_t hsb[MEERKAT_MAX_RANKS], hrb[MEERKAT_MAX_RANKS], ts = 0, tr = 0;
  for (uint32_t p = 0; p < ws; p++) {
    hsb[p] = p == me ? 0 : sb[p];
    hrb[p] = p == me ? 0 : rb[p];
    ts += hsb[p];
    tr += hrb[p];
  }
  e = ensure_host(ps, std::max(ts, tr));
  uint64_t o = 0;
  for (uint32_t p = 0; p < ws && e == cudaSuccess; p++) {
    if (hsb[p]) e = cudaMemcpyAsync(ps->hsend + o, s8 + so[p], hsb[p], cudaMemcpyDeviceToHost, g->stream);
    o += hsb[p];
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (ps->xfn(ps->xctx, ps->hsend, hsb, ps->hrecv, hrb) != 0) return MEERKAT_E_NCCL;
  o = 0;
  for (uint32_t p = 0; p < ws && e == cudaSuccess; p++) {
    if (hrb[p]) e = cudaMemcpyAsync(r8 + ro[p], ps->hrecv + o, hrb[p], cudaMemcpyHostToDevice, g->stream);
    o += hrb[p];
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  return st_of(e);
}

// Every rank's m values; returns the per-rank rows in ps->hcoll[q * m + i] (synchronises).
static meerkat_status allgather_small(meerkat_graph* g, const uint64_t* vals, uint32_t m) {
  PartState* ps = g->part;
  const uint32_t ws = g->ws;
  if ((size_t)ws * m > COLL_WORDS) return MEERKAT_E_INVALID_ARG;
  uint64_t* d = ps->dcoll;   // [ws * m] send, [ws * m] recv
  for (uint32_t p = 0; p < ws; p++) std::memcpy(ps->hcoll + (size_t)p * m, vals, m * 8);
  cudaError_t e = cudaMemcpyAsync(d, ps->hcoll, (size_t)ws * m * 8, cudaMemcpyHostToDevice, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint64_t sb[MEERKAT_MAX_RANKS], so[MEERKAT_MAX_RANKS];
  for (uint32_t p = 0; p < ws; p++) { sb[p] = m * 8; so[p] = (uint64_t)p * m * 8; }
  meerkat_status st = xchg(g, d, sb, so, d + (size_t)ws * m, sb, so);
  if (st != MEERKAT_OK) return st;
  e = cudaMemcpyAsync(ps->hcoll, d + (size_t)ws * m, (size_t)ws * m * 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  return nccl_check(g);
}

meerkat_status part_allreduce(meerkat_graph* g, uint64_t* vals, uint32_t m) {
  if (m > 16) return MEERKAT_E_INVALID_ARG;
  meerkat_status st = allgather_small(g, vals, m);
  if (st != MEERKAT_OK) return st;
  for (uint32_t i = 0; i < m; i++) {
    uint64_t s = 0;
    for (uint32_t q = 0; q < g->ws; q++) s += g->part->hcoll[(size_t)q * m + i];
    vals[i] = s;
  }
  return MEERKAT_OK;
}

// ------------------------------------------------------------------ lifecycle

meerkat_status part_init(meerkat_graph* g, const meerkat_config* cfg) {
  PartState* ps = new (std::nothrow) PartState();
  if (!ps) return MEERKAT_E_CUDA;
  g->part = ps;
  ps->xfn = cfg->exchange;
  ps->xctx = cfg->exchange_ctx;
  if (cfg->exchange_pairs) ps->cap_dyn = cfg->exchange_pairs;
  ps->cap_static = ps->cap_dyn * STATIC_CAP_MULT;
  ps->blk = HDR + ps->cap_static;
  cudaError_t e = cudaMalloc(&ps->send, (size_t)g->ws * ps->blk * 16);
  if (e == cudaSuccess) e = cudaMalloc(&ps->recv, (size_t)g->ws * ps->blk * 16);
  if (e == cudaSuccess) e = cudaMemsetAsync(ps->recv, 0, (size_t)g->ws * ps->blk * 16, g->stream);
  if (e == cudaSuccess) e = cudaMalloc(&ps->pc, sizeof(PartCtrl));
  if (e == cudaSuccess) e = cudaMemsetAsync(ps->pc, 0, sizeof(PartCtrl), g->stream);
  if (e == cudaSuccess) e = cudaHostAlloc(&ps->hflags, FLAG_RING * 4, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&ps->dflags, ps->hflags, 0);
  if (e == cudaSuccess) e = cudaMalloc(&ps->dscr, SCR_WORDS * 8);
  if (e == cudaSuccess) e = cudaMallocHost(&ps->hscr, SCR_WORDS * 8);
  if (e == cudaSuccess) { ps->dcoll_bytes = COLL_WORDS * 8 * 2; e = cudaMalloc(&ps->dcoll, ps->dcoll_bytes); }
  if (e == cudaSuccess) e = cudaMallocHost(&ps->hcoll, COLL_WORDS * 8);
  for (uint32_t i = 0; i < 2 * MAX_PIPE && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&ps->ev[i], cudaEventDisableTiming);
  if (e == cudaSuccess) {
    std::memset(ps->hflags, 0, FLAG_RING * 4);
    auto fn = g->weighted ? (const void*)k_part_unit<true> : (const void*)k_part_unit<false>;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps->bps, fn, TREE_BLOCK, 0);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (ps->bps < 1) return MEERKAT_E_CUDA;
  ps->bps = std::min(ps->bps, TREE_MINB);
  if (cfg->nccl_id) {
    NcclApi* api = nccl_api();
    if (!api) return MEERKAT_E_NCCL;
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    if (api->CommInitRank(&ps->comm, (int)g->ws, id, (int)g->rank) != ncclSuccess) {
      ps->comm = nullptr;
      return MEERKAT_E_NCCL;
    }
  }
  return MEERKAT_OK;
}

void part_free(meerkat_graph* g) {
  PartState* ps = g->part;
  if (!ps) return;
  if (ps->comm) nccl_api()->CommDestroy(ps->comm);
  cudaFree(ps->send); cudaFree(ps->recv); cudaFree(ps->q); cudaFree(ps->pc);
  cudaFree(ps->rsend); cudaFree(ps->rrecv); cudaFree(ps->rows); cudaFree(ps->dscr); cudaFree(ps->dcoll);
  if (ps->hflags) cudaFreeHost(ps->hflags);
  if (ps->hscr) cudaFreeHost(ps->hscr);
  if (ps->hcoll) cudaFreeHost(ps->hcoll);
  if (ps->hsend) cudaFreeHost(ps->hsend);
  if (ps->hrecv) cudaFreeHost(ps->hrecv);
  for (uint32_t i = 0; i < 2 * MAX_PIPE; i++) if (ps->ev[i]) cudaEventDestroy(ps->ev[i]);
  delete ps;
  g->part = nullptr;
}

meerkat_status part_hints(meerkat_graph* g, const uint32_t* global_hints, const void** local_hints, int slot) {
  *local_hints = nullptr;
  if (!global_hints) return MEERKAT_OK;
  const void* dg = nullptr;
  cudaError_t e = stage_in(g, slot, global_hints, (size_t)g->V * 4, &dg);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint32_t* loc = nullptr;
  e = cudaMalloc(&loc, (size_t)std::max<uint32_t>(g->Vl, 1) * 4);
  if (e == cudaSuccess) {
    k_gather_rows<<<grid_of(g, g->Vl), 256, 0, g->stream>>>((const uint32_t*)dg, loc, g->Vl, g->rank, g->V,
                                                          pm_bits(g->V), g->ws);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);   // the staging slot is reused next
  if (e == cudaSuccess) e = ensure_stage(g, slot, (size_t)std::max<uint32_t>(g->Vl, 1) * 4);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(g->stage[slot], loc, (size_t)g->Vl * 4, cudaMemcpyDeviceToDevice, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(loc);
  *local_hints = g->stage[slot];
  return st_of(e);
}

// ------------------------------------------------------------------ routing

static cudaError_t ensure_rows(PartState* ps, uint64_t rows) {
  if (ps->rows_cap >= rows) return cudaSuccess;
  cudaFree(ps->rows);
  ps->rows = nullptr;
  ps->rows_cap = 0;
  const uint64_t cap = std::max<uint64_t>(rows + rows / 4, 1 << 16);
  cudaError_t e = cudaMalloc(&ps->rows, cap * 6 * 4);
  if (e == cudaSuccess) ps->rows_cap = cap;
  return e;
}
static cudaError_t ensure_buf(uint4** p, uint64_t* cap, uint64_t rows) {
  if (*cap >= rows) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const uint64_t c = std::max<uint64_t>(rows + rows / 4, 1 << 16);
  cudaError_t e = cudaMalloc(p, c * 16);
  if (e == cudaSuccess) *cap = c;
  return e;
}

// Route a batch: kind 1 insert, 2 delete, 3 query.  Leaves the received rows split into
// ps->rows (out s/d/w at [0..3) x rows_cap, in s/d/w at [3..6)), counts n_out / n_in; for queries the
// received rows stay in rrecv (segments) and rc/ro describe them.
struct Routed {
  uint64_t sc[MEERKAT_MAX_RANKS], so[MEERKAT_MAX_RANKS];   // rows sent to each rank, offsets
  uint64_t rc[MEERKAT_MAX_RANKS], ro[MEERKAT_MAX_RANKS];   // rows received from each rank, offsets
  uint64_t total_recv;
  uint32_t err;
};

static meerkat_status route(meerkat_graph* g, int kind, const uint32_t* s, const uint32_t* d, const uint32_t* w,
                            uint64_t n, Routed& out) {
  PartState* ps = g->part;
  const uint32_t ws = g->ws;
  RouteArgs R{};
  R.s = s; R.d = d; R.w = (kind == 1) ? w : nullptr; R.n = n;
  R.V = g->V; R.bits = pm_bits(g->V); R.ws = ws; R.rank = g->rank;
  R.need_in = (kind == 2) || (kind == 1 && g->reverse);
  R.check_w = kind == 1 && g->weighted;
  R.aux_index = kind == 3;
  R.counts = ps->dscr + SCR_COUNTS;
  R.cursor = ps->dscr + SCR_CURSOR;
  R.fp = ps->dscr + SCR_FP;
  R.err = reinterpret_cast<unsigned int*>(ps->dscr + SCR_ERR);
  cudaError_t e = cudaMemsetAsync(ps->dscr, 0, SCR_WORDS * 8, g->stream);
  if (e == cudaSuccess && n) {
    k_route_count<<<grid_of(g, n), 256, 0, g->stream>>>(R);
    e = cudaGetLastError();
    g->launches++;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(ps->hscr, ps->dscr, SCR_WORDS * 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  out.err = (uint32_t)ps->hscr[SCR_ERR];
  ps->fp_last[0] = ps->hscr[SCR_FP];
  ps->fp_last[1] = ps->hscr[SCR_FP + 1];
  // send offsets per (rank, section); rows per destination
  uint64_t cur[MEERKAT_MAX_RANKS * 3], o = 0;
  uint64_t mine[MEERKAT_MAX_RANKS * 3];
  for (uint32_t p = 0; p < ws; p++) {
    out.so[p] = o;
    for (int sct = 0; sct < 3; sct++) { cur[p * 3 + sct] = o; o += ps->hscr[SCR_COUNTS + p * 3 + sct]; }
    out.sc[p] = o - out.so[p];
  }
  // exchange the section counts: rank p gets my 3 counts for p
  uint64_t vals[3 * MEERKAT_MAX_RANKS];
  for (uint32_t i = 0; i < 3 * ws; i++) vals[i] = ps->hscr[SCR_COUNTS + i];
  meerkat_status st = allgather_small(g, vals, 3 * ws);   // rank q's counts for every rank
  if (st != MEERKAT_OK) return st;
  for (uint32_t q = 0; q < ws; q++)
    for (int sct = 0; sct < 3; sct++) mine[q * 3 + sct] = ps->hcoll[(size_t)q * 3 * ws + g->rank * 3 + sct];
  uint64_t ro = 0;
  for (uint32_t q = 0; q < ws; q++) {
    out.ro[q] = ro;
    out.rc[q] = mine[q * 3] + mine[q * 3 + 1] + mine[q * 3 + 2];
    ro += out.rc[q];
  }
  out.total_recv = ro;
  e = ensure_buf(&ps->rsend, &ps->rsend_cap, o);
  if (e == cudaSuccess) e = ensure_buf(&ps->rrecv, &ps->rrecv_cap, ro);
  if (e == cudaSuccess) {
    for (uint32_t i = 0; i < 3 * ws; i++) ps->hscr[SCR_CURSOR + i] = cur[i];
    e = cudaMemcpyAsync(ps->dscr + SCR_CURSOR, ps->hscr + SCR_CURSOR, 3 * ws * 8, cudaMemcpyHostToDevice, g->stream);
  }
  R.rows = ps->rsend;
  if (e == cudaSuccess && n) {
    k_route_scatter<<<grid_of(g, n), 256, 0, g->stream>>>(R);
    e = cudaGetLastError();
    g->launches++;
  }
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint64_t sb[MEERKAT_MAX_RANKS], sob[MEERKAT_MAX_RANKS], rb[MEERKAT_MAX_RANKS], rob[MEERKAT_MAX_RANKS];
  for (uint32_t p = 0; p < ws; p++) {
    sb[p] = out.sc[p] * 16; sob[p] = out.so[p] * 16; rb[p] = out.rc[p] * 16; rob[p] = out.ro[p] * 16;
  }
  st = xchg(g, ps->rsend, sb, sob, ps->rrecv, rb, rob);
  if (st != MEERKAT_OK) return st;
  // split into the local kernels' arrays
  SplitArgs S{};
  S.rows = ps->rrecv;
  S.ws = ws;
  uint64_t ob = 0, ib = 0;
  for (uint32_t q = 0; q < ws; q++) {
    S.base[q] = out.ro[q];
    S.n0[q] = mine[q * 3];
    S.n1[q] = mine[q * 3 + 1];
    S.out_base[q] = ob;
    S.in_base[q] = ib;
    ob += mine[q * 3] + mine[q * 3 + 1];
    ib += mine[q * 3 + 1] + mine[q * 3 + 2];
  }
  S.base[ws] = ro;
  e = ensure_rows(ps, std::max<uint64_t>(std::max(ob, ib), 1));
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint32_t* r = ps->rows;
  const uint64_t c = ps->rows_cap;
  S.os = r; S.od = r + c; S.ow = r + 2 * c;
  S.is = R.need_in ? r + 3 * c : nullptr; S.id = r + 4 * c; S.iw = r + 5 * c;
  ps->n_out = ob;
  ps->n_in = R.need_in ? ib : 0;
  if (ro) {
    k_route_split<<<grid_of(g, ro), 256, 0, g->stream>>>(S);
    g->launches++;
    e = cudaGetLastError();
  }
  return st_of(e);
}

meerkat_status part_mutate(meerkat_graph* g, int kind, const uint32_t* s, const uint32_t* d, const uint32_t* w,
                           uint64_t n, uint64_t* count) {
  PartState* ps = g->part;
  Routed rt;
  meerkat_status st = route(g, kind, s, d, w, n, rt);
  if (st != MEERKAT_OK) return st;
  uint32_t* r = ps->rows;
  const uint64_t c = ps->rows_cap;
  unsigned long long* cnt = kind == 1 ? &g->out.dev.ctrl->n_inserted : &g->out.dev.ctrl->n_deleted;
  cudaError_t e = cudaMemsetAsync(cnt, 0, 8, g->stream);
  if (e == cudaSuccess) {
    if (kind == 1) {
      e = launch_insert(g, &g->out, nullptr, r, r + c, g->weighted ? r + 2 * c : nullptr, ps->n_out);
      if (e == cudaSuccess && g->reverse)
        e = launch_insert(g, &g->in, nullptr, r + 3 * c, r + 4 * c, g->weighted ? r + 5 * c : nullptr, ps->n_in);
    } else {
      e = launch_delete(g, &g->out, nullptr, r, r + c, ps->n_out);
      if (e == cudaSuccess && g->reverse) e = launch_delete(g, &g->in, nullptr, r + 3 * c, r + 4 * c, ps->n_in);
    }
  }
  if (e == cudaSuccess) e = mutated(g, kind, n);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  ps->n_last = n;
  st = collect(g);   // this rank's store errors (capacity) and counters
  uint64_t vals[2] = {kind == 1 ? g->out.hctrl->n_inserted : g->out.hctrl->n_deleted, (uint64_t)rt.err};
  meerkat_status st2 = part_allreduce(g, vals, 1);   // global count (collective even if unused)
  if (st2 != MEERKAT_OK) return st2;
  if (count) *count = vals[0];
  if (st == MEERKAT_OK && rt.err) {
    if (rt.err & ERR_RANGE) return MEERKAT_E_VERTEX_RANGE;
    if (rt.err & ERR_WEIGHT) return MEERKAT_E_WEIGHT;
  }
  return st;
}

meerkat_status part_query(meerkat_graph* g, const uint32_t* s, const uint32_t* d, uint64_t n, uint8_t* found,
                          uint32_t* w_out) {
  PartState* ps = g->part;
  Routed rt;
  meerkat_status st = route(g, 3, s, d, nullptr, n, rt);
  if (st != MEERKAT_OK) return st;
  const uint64_t m = rt.total_recv;
  uint32_t* r = ps->rows;
  const uint64_t c = ps->rows_cap;
  // answers of the received rows (in received order: queries use section 0 only)
  uint8_t* af = reinterpret_cast<uint8_t*>(r + 3 * c);
  uint32_t* aw = r + 4 * c;
  cudaError_t e = launch_query(g, g->out, r, r + c, m, af, aw);
  if (e == cudaSuccess) e = ensure_buf(&ps->rsend, &ps->rsend_cap, std::max<uint64_t>(m, 1));
  if (e == cudaSuccess && m) {
    k_query_reply<<<grid_of(g, m), 256, 0, g->stream>>>(af, aw, r + 2 * c, m, ps->rsend);
    g->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = ensure_buf(&ps->rrecv, &ps->rrecv_cap, std::max<uint64_t>(n, 1));
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint64_t sb[MEERKAT_MAX_RANKS], so[MEERKAT_MAX_RANKS], rb[MEERKAT_MAX_RANKS], ro[MEERKAT_MAX_RANKS];
  for (uint32_t p = 0; p < g->ws; p++) {   // the reverse of the routing exchange
    sb[p] = rt.rc[p] * 16; so[p] = rt.ro[p] * 16; rb[p] = rt.sc[p] * 16; ro[p] = rt.so[p] * 16;
  }
  st = xchg(g, ps->rsend, sb, so, ps->rrecv, rb, ro);
  if (st != MEERKAT_OK) return st;
  const bool host_f = n && !is_device_ptr(found), host_w = n && w_out && !is_device_ptr(w_out);
  uint8_t* df = found;
  uint32_t* dw = w_out;
  if (host_f) { e = ensure_stage(g, 2, n); df = (uint8_t*)g->stage[2]; }
  if (e == cudaSuccess && host_w) { e = ensure_stage(g, 3, n * 4); dw = (uint32_t*)g->stage[3]; }
  if (e == cudaSuccess && n) {
    k_query_scatter<<<grid_of(g, n), 256, 0, g->stream>>>(ps->rrecv, n, df, dw);
    g->launches++;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess && host_f) e = cudaMemcpyAsync(found, df, n, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess && host_w) e = cudaMemcpyAsync(w_out, dw, n * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  st = collect(g);
  if (st == MEERKAT_OK && (rt.err & ERR_RANGE)) st = MEERKAT_E_VERTEX_RANGE;
  return st;
}

// ------------------------------------------------------------------ trees

meerkat_status part_tree_init(meerkat_graph* g, meerkat_tree* t) {
  t->part = true;
  cudaError_t e = cudaMalloc(&t->pull_items, t->dev.fr_cap * 8);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  t->bytes += t->dev.fr_cap * 8;
  meerkat_tree* one[1] = {t};
  return part_trees(g, one, 1, 0, nullptr, nullptr, nullptr, 0);   // collective static tree
}

void part_tree_free(meerkat_tree* t) { cudaFree(t->pull_items); }

// Per-peer ring capacity: at least the messages one unit can emit for a rank's live edges.
static cudaError_t ensure_rings(meerkat_graph* g) {
  PartState* ps = g->part;
  if (g->ws == 1) {
    if (!ps->q) { ps->q_cap = 1; return cudaMalloc(&ps->q, 16); }
    return cudaSuccess;
  }
  const uint64_t live = g->out.hctrl->ins_total - g->out.hctrl->del_total;
  const uint64_t need = std::max<uint64_t>(1 << 18, (live / (g->ws - 1)) * 2 + (1 << 16));
  if (ps->q_cap >= need) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(g->stream);   // rings are empty between calls
  if (e != cudaSuccess) return e;
  cudaFree(ps->q);
  ps->q = nullptr;
  ps->q_cap = 0;
  ps->dirty = true;   // ring positions restart at 0
  const uint64_t cap = need + need / 2;
  e = cudaMalloc(&ps->q, (size_t)g->ws * cap * 16);
  if (e == cudaSuccess) ps->q_cap = cap;
  return e;
}

static cudaError_t launch_unit(meerkat_graph* g, PArgs& A) {
  PartState* ps = g->part;
  void* args[] = {&A};
  const dim3 grid((unsigned)(g->sm_count * ps->bps)), block(TREE_BLOCK);
  auto fn = g->weighted ? (const void*)k_part_unit<true> : (const void*)k_part_unit<false>;
  cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, block, args, 0, g->stream);
  g->launches++;
  return e;
}

// Units until the call is done on every rank.  Every rank launches the same number of units: the
// stop decision reads the mode of unit (launched - PIPE), which every rank computed identically.
// Copies of the graph's and the trees' control blocks, enqueued before a unit loop's final synchronisation.
static cudaError_t enqueue_readback(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k) {
  cudaError_t e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  for (uint32_t i = 0; i < k && e == cudaSuccess; i++)
    e = cudaMemcpyAsync(trees[i]->hctrl, trees[i]->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  return e;
}

static meerkat_status run_units(meerkat_graph* g, PArgs A, meerkat_tree* const* trees, uint32_t k) {
  PartState* ps = g->part;
  const uint32_t ws = g->ws;
  uint64_t sb[MEERKAT_MAX_RANKS], so[MEERKAT_MAX_RANKS];
  const uint64_t bytes = A.blk * 16;
  for (uint32_t p = 0; p < ws; p++) { sb[p] = p == g->rank && !A.self_send ? 0 : bytes; so[p] = (uint64_t)p * bytes; }
  const uint64_t base = ps->units;
  uint64_t launched = 0;
  meerkat_status st = MEERKAT_OK;
  for (;;) {
    if (launched >= MAX_UNITS) return MEERKAT_E_CAPACITY;
    if (launch_unit(g, A) != cudaSuccess) return MEERKAT_E_CUDA;
    A.start_mode = 0;
    const uint64_t u = launched++;
    ps->units++;
    if (A.chain) {   // one rank: one launch chains every phase
      if (enqueue_readback(g, trees, k) != cudaSuccess) return MEERKAT_E_CUDA;
      if (cudaStreamSynchronize(g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
      return ps->hflags[(base + u) % FLAG_RING] == PM_DONE ? MEERKAT_OK : MEERKAT_E_STATE;
    }
    if (!ps->comm) {   // host transport: synchronous units, variable-size blocks
      if (cudaStreamSynchronize(g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
      if (trace_on()) fprintf(stderr, "[part r%u] unit %llu mode %u\n", g->rank, (unsigned long long)(base + u),
                              ps->hflags[(base + u) % FLAG_RING]);
      if (ps->hflags[(base + u) % FLAG_RING] == PM_DONE) {
        if (enqueue_readback(g, trees, k) != cudaSuccess) return MEERKAT_E_CUDA;
        if (cudaStreamSynchronize(g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
        return MEERKAT_OK;
      }
      uint64_t hs[MEERKAT_MAX_RANKS * 4];
      cudaError_t e = cudaSuccess;
      for (uint32_t p = 0; p < ws && e == cudaSuccess; p++)
        e = cudaMemcpyAsync(hs + p * 4, ps->send + (uint64_t)p * A.blk, 32, cudaMemcpyDeviceToHost, g->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
      if (e != cudaSuccess) return MEERKAT_E_CUDA;
      uint64_t n[MEERKAT_MAX_RANKS];
      for (uint32_t p = 0; p < ws; p++) n[p] = p == g->rank ? 0 : hs[p * 4];
      st = allgather_small(g, n, ws);   // block sizes every rank sends to every rank
      if (st != MEERKAT_OK) return st;
      uint64_t vsb[MEERKAT_MAX_RANKS], vrb[MEERKAT_MAX_RANKS];
      for (uint32_t p = 0; p < ws; p++) {
        vsb[p] = p == g->rank ? 0 : (HDR + n[p]) * 16;
        vrb[p] = p == g->rank ? 0 : (HDR + ps->hcoll[(size_t)p * ws + g->rank]) * 16;
      }
      st = xchg(g, A.send, vsb, so, A.recv, vrb, so);
      if (st != MEERKAT_OK) return st;
      continue;
    }
    st = xchg(g, A.send, sb, so, A.recv, sb, so);
    if (st != MEERKAT_OK) return st;
    if (cudaEventRecord(ps->ev[u % (2 * MAX_PIPE)], g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
    if (u + 1 < PIPE) continue;
    const uint64_t v = u + 1 - PIPE;   // the unit whose mode decides
    cudaEvent_t ev = ps->ev[v % (2 * MAX_PIPE)];
    for (;;) {
      const cudaError_t q = cudaEventQuery(ev);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) return MEERKAT_E_CUDA;
      st = nccl_check(g);
      if (st != MEERKAT_OK) return st;
      sched_yield();
    }
    if (ps->hflags[(base + v) % FLAG_RING] == PM_DONE) break;
  }
  if (enqueue_readback(g, trees, k) != cudaSuccess) return MEERKAT_E_CUDA;
  if (cudaStreamSynchronize(g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
  return nccl_check(g);
}

meerkat_status part_trees(meerkat_graph* g, meerkat_tree* const* trees, uint32_t k, int kind, const uint32_t* s,
                          const uint32_t* d, const uint32_t* w, uint64_t n) {
  PartState* ps = g->part;
  if (k == 0 || k > (uint32_t)MAX_TREES) return MEERKAT_E_INVALID_ARG;
  bool weights = false;
  for (uint32_t i = 0; i < k; i++) {
    if (!trees[i] || trees[i]->g != g || !trees[i]->part) return MEERKAT_E_INVALID_ARG;
    for (uint32_t j = 0; j < i; j++) if (trees[j] == trees[i]) return MEERKAT_E_INVALID_ARG;
    weights = weights || !trees[i]->unit;
  }
  // ordering contract, the parts every rank sees alike (the same collective sequence): the
  // call follows a mutation of its kind and each tree is one mutation behind.  The batch itself (size
  // and fingerprint per rank) is judged on the device by the first unit, and the verdicts are
  // exchanged before any tree is touched (PM_CHECK / PM_VERDICT).
  if (kind) {
    if (g->last_kind != kind) return MEERKAT_E_STATE;
    for (uint32_t i = 0; i < k; i++)
      if (trees[i]->version + 1 != g->version) return MEERKAT_E_STATE;
  }
  const bool with_w = kind == 1 && g->weighted && w != nullptr;
  if (kind == 1 && g->weighted && !w && weights && n) return MEERKAT_E_INVALID_ARG;
  cudaError_t e = cudaSuccess;
  const void *ds = nullptr, *dd = nullptr, *dw = nullptr;
  if (kind && n) {
    e = stage_in(g, 0, s, n * 4, &ds);
    if (e == cudaSuccess) e = stage_in(g, 1, d, n * 4, &dd);
    if (e == cudaSuccess && with_w) e = stage_in(g, 2, w, n * 4, &dw);
  }
  if (e == cudaSuccess) e = cudaMemsetAsync(ps->pc->fp, 0, sizeof(ps->pc->fp), g->stream);
  if (e == cudaSuccess && !kind) {   // live-edge count for the rings
    e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  }
  if (e == cudaSuccess) e = ensure_rings(g);
  if (e == cudaSuccess && ps->dirty) {   // a failed call may have left messages and frontier sizes behind
    e = cudaMemsetAsync(ps->pc->size, 0, sizeof(ps->pc->size), g->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(ps->pc->head, 0, sizeof(ps->pc->head) + sizeof(ps->pc->tail), g->stream);
    ps->dirty = false;
  }
  for (uint32_t i = 0; i < k && e == cudaSuccess; i++)
    e = cudaMemsetAsync(trees[i]->dev.ctrl, 0, sizeof(TreeCtrl), g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  PArgs A{};
  A.G = g->out.dev;
  if (g->reverse) A.R = g->in.dev;
  for (uint32_t i = 0; i < k; i++) { A.T[i] = trees[i]->dev; A.pull[i] = trees[i]->pull_items; }
  for (uint32_t i = k; i < (uint32_t)MAX_TREES; i++) { A.T[i] = trees[0]->dev; A.pull[i] = trees[0]->pull_items; }
  A.ntrees = k;
  A.start_mode = kind == 0 ? PM_SEED_STATIC : PM_CHECK;
  A.seed_mode = kind == 1 ? PM_SEED_INC : PM_SEED_DEC;
  A.scan = g->reverse ? 0u : 1u;
  A.pc = ps->pc;
  A.flags = ps->dflags;
  A.q = ps->q;
  A.q_cap = ps->q_cap;
  A.send = ps->send;
  A.recv = ps->recv;
  A.blk = HDR + (kind == 0 ? ps->cap_static : ps->cap_dyn);
  A.cap = A.blk - HDR;
  const uint64_t c = ps->rows_cap;
  if (kind == 1) { A.bs = ps->rows; A.bd = ps->rows + c; A.bw = g->weighted ? ps->rows + 2 * c : nullptr; A.bn = ps->n_out; }
  if (kind == 2) { A.bs = ps->rows + 3 * c; A.bd = ps->rows + 4 * c; A.bn = ps->n_in; }
  A.fs = (const uint32_t*)ds; A.fd = (const uint32_t*)dd; A.fw = (const uint32_t*)dw; A.fn = kind ? n : 0;
  A.fp_expect[0] = ps->fp_last[0];
  A.fp_expect[1] = ps->fp_last[1];
  A.fp_w = with_w ? 1u : 0u;
  A.fn_bad = kind && n != ps->n_last ? 1u : 0u;
  // one rank chains the phases in one launch; MEERKAT_PART_UNITS=1 keeps one unit per phase (the P > 1
  // protocol, host pipeline included) so a one-GPU box exercises it
  static const bool force_units = std::getenv("MEERKAT_PART_UNITS") != nullptr;
  A.chain = g->ws == 1 && !force_units ? 1u : 0u;
  A.self_send = ps->comm && nccl_self() && !A.chain ? 1u : 0u;
  const uint64_t units0 = ps->units;
  meerkat_status st = run_units(g, A, trees, k);
  ps->dirty = st != MEERKAT_OK;
  if (st == MEERKAT_E_NCCL || st == MEERKAT_E_CUDA) return st;
  // every rank's status: errors anywhere (capacity, overflow, a refused batch) fail the call everywhere
  uint64_t err[1] = {(uint64_t)g->out.hctrl->err | (st != MEERKAT_OK ? (uint64_t)ERR_STATE : 0)};
  if (g->ws > 1) {
    const meerkat_status s2 = allgather_small(g, err, 1);
    if (s2 != MEERKAT_OK) return s2;
    for (uint32_t q = 0; q < g->ws; q++) err[0] |= ps->hcoll[q];
  }
  if (g->out.hctrl->err) cudaMemsetAsync(&g->out.dev.ctrl->err, 0, 4, g->stream);
  if (err[0] & ERR_STATE) return MEERKAT_E_STATE;   // refused: the trees stay one mutation behind
  for (uint32_t i = 0; i < k; i++) {
    trees[i]->version = g->version;
    trees[i]->last_units = A.chain ? 0 : ps->units - units0;
  }
  if (err[0] & ERR_CAPACITY) return MEERKAT_E_CAPACITY;
  if (err[0] & ERR_OVERFLOW) return MEERKAT_E_OVERFLOW;
  if (err[0] & ERR_PARTITION) return MEERKAT_E_PARTITION;
  if (err[0]) return MEERKAT_E_STATE;
  return MEERKAT_OK;
}

meerkat_status part_tree_nodes(meerkat_tree* t, uint64_t* out) {
  meerkat_graph* g = t->g;
  const uint32_t ws = g->ws;
  uint64_t sb[MEERKAT_MAX_RANKS], so[MEERKAT_MAX_RANKS], rb[MEERKAT_MAX_RANKS], ro[MEERKAT_MAX_RANKS];
  uint64_t base[MEERKAT_MAX_RANKS + 1], o = 0;
  for (uint32_t p = 0; p < ws; p++) {
    sb[p] = (uint64_t)g->Vl * 8;
    so[p] = 0;   // the same rows to every rank
    base[p] = o;
    rb[p] = (uint64_t)rows_of(g, p) * 8;
    ro[p] = o * 8;
    o += rows_of(g, p);
  }
  base[ws] = o;
  uint64_t* tmp = nullptr;
  uint64_t* dbase = nullptr;
  cudaError_t e = cudaMalloc(&tmp, (size_t)std::max<uint64_t>(o, 1) * 8 * 2);
  if (e == cudaSuccess) e = cudaMalloc(&dbase, (MEERKAT_MAX_RANKS + 1) * 8);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dbase, base, (ws + 1) * 8, cudaMemcpyHostToDevice, g->stream);
  meerkat_status st = e == cudaSuccess ? xchg(g, t->dev.node, sb, so, tmp, rb, ro) : MEERKAT_E_CUDA;
  const bool host = !is_device_ptr(out);
  uint64_t* dst = host ? tmp + o : out;
  if (st == MEERKAT_OK) {
    k_unpermute<<<grid_of(g, o), 256, 0, g->stream>>>(tmp, dbase, ws, g->V, pm_bits(g->V), dst);
    g->launches++;
    e = cudaGetLastError();
    if (e == cudaSuccess && host) e = cudaMemcpyAsync(out, dst, (size_t)o * 8, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) st = MEERKAT_E_CUDA;
  }
  cudaStreamSynchronize(g->stream);
  cudaFree(tmp);
  cudaFree(dbase);
  if (st == MEERKAT_OK) st = nccl_check(g);
  return st;
}

}  // namespace mk

extern "C" {

meerkat_status meerkat_nccl_unique_id(void* out, uint64_t bytes) {
  if (!out || bytes < sizeof(ncclUniqueId)) return MEERKAT_E_INVALID_ARG;
  mk::NcclApi* api = mk::nccl_api();
  if (!api) return MEERKAT_E_NCCL;
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != ncclSuccess) return MEERKAT_E_NCCL;
  std::memcpy(out, &id, sizeof(id));
  return MEERKAT_OK;
}

meerkat_status meerkat_owner_map(uint32_t vertex_n, uint32_t world_size, const uint32_t* ids, uint64_t n,
                                 uint32_t* owner, uint32_t* row) {
  if (vertex_n == 0 || world_size == 0 || world_size > MEERKAT_MAX_RANKS || (n && !ids)) return MEERKAT_E_INVALID_ARG;
  const uint32_t bits = mk::pm_bits(vertex_n);
  for (uint64_t i = 0; i < n; i++) {
    if (ids[i] >= vertex_n) return MEERKAT_E_VERTEX_RANGE;
    uint32_t r;
    const uint32_t o = mk::pm_place(ids[i], vertex_n, bits, world_size, r);
    if (owner) owner[i] = o;
    if (row) row[i] = r;
  }
  return MEERKAT_OK;
}

}  // extern "C"
