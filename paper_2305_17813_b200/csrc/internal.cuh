// internal.cuh — device-side layout, sentinels and warp-group primitives shared
// by the store kernels (store.cu) and the traversal kernels (tree.cu).
//
// Slab layout: a slab is 128 B = 32 lanes x 4 B,
// one L1/L2 line.  Lane 31 holds the next slab's index (INVALID_SLAB ends the
// chain).  ConcurrentSet (unweighted) slabs keep 31 keys in lanes 0..30;
// ConcurrentMap (weighted) slabs keep 15 <key, weight> pairs in lanes (2k, 2k+1),
// k < 15, lane 30 permanently EMPTY.  A pair is one aligned 64-bit word whose
// low half is the key, so one 64-bit CAS / atomicMin updates it.
//
// B200 mapping: a slab is read by a GROUP of 8 lanes, each loading 16 B
// (one LDG.128), so one warp instruction reads four independent slabs
// (4 memory requests in flight per warp instead of the paper's one,
// SURVEY §7 H2).  Every group-level collective uses the group's 8-lane mask.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace mk {

constexpr uint32_t EMPTY_KEY = 0xFFFFFFFEu;              // UINT32_MAX-1 (P:1504 footnote)
constexpr uint32_t TOMBSTONE_KEY = 0xFFFFFFFDu;          // UINT32_MAX-2 (P:1506 footnote)
constexpr uint32_t INVALID_SLAB = 0xFFFFFFFFu;           // end of chain / no head slab yet
constexpr uint32_t LINKING = 0xFFFFFFFEu;                // link word locked while one group links a slab
constexpr uint32_t NO_OWNER = 0xFFFFFFFFu;               // owner[] of a slab outside any list
constexpr uint64_t EMPTY_PAIR = 0xFFFFFFFFFFFFFFFEull;   // UINT64_MAX-1 (P:1504 footnote)
constexpr uint64_t TOMB_PAIR = 0xFFFFFFFDFFFFFFFDull;    // <UINT32_MAX-2, UINT32_MAX-2> (P:1506 footnote)
constexpr uint64_t UNREACHED = ~0ull;                    // <INF, INVALID> packed (C3)
constexpr uint32_t INF_DIST = 0xFFFFFFFFu;
constexpr uint32_t W_LIMIT = 0x80000000u;                // weights in [1, 2^31) (C6)
constexpr int SLAB_WORDS = 32;
constexpr int GROUP = 8;                                 // lanes per slab
constexpr int SET_CAP = 31, MAP_CAP = 15;

enum ErrBits : uint32_t { ERR_RANGE = 1, ERR_WEIGHT = 2, ERR_CAPACITY = 4, ERR_OVERFLOW = 8, ERR_STATE = 16,
                        ERR_PARTITION = 32 };

struct GraphCtrl {
  unsigned long long pool_top;    // bump pointer of the growth pool
  unsigned long long n_inserted;  // per-call counters (reset by the host when a count is requested)
  unsigned long long n_deleted;
  unsigned long long ins_total;   // cumulative: live edges = ins_total - del_total
  unsigned long long del_total;
  unsigned long long export_n;
  unsigned long long upd_n;       // update tracking: slab lists queued in updq since the last reset
  unsigned int err;               // sticky ErrBits
  unsigned int pad;
  // batch fingerprints of the last plain mutation (ordering contract, meerkat.h): slot = version & 1,
  // [0] over (src, dst), [1] over (src, dst, w).  A mutation accumulates into its slot and zeroes the other.
  unsigned long long fp[2][2];
};

struct GraphDev {
  uint32_t* slabs;   // (H + P) slabs x 32 words: head arena [0, H) then pool [H, H + P)
  uint32_t* owner;   // source vertex of every slab (the paper's bucket_vertex[])
  uint2* vmeta;      // per vertex {first head slab | INVALID_SLAB, bucket_count}
  unsigned long long* upd;   // update tracking (nullable): per slab list (indexed by its head slab) the
                             // earliest cell written since the last reset, (slab << 5) | cell, or ~0
  uint32_t* updq;            // the slab lists with upd != ~0 (UpdateIterator work list)
  uint32_t* deg;     // per vertex live keys (out-degree in the out store, in-degree in the mirror),
                     // computed on demand by a stream over the slabs (launch_degrees) for PageRank's
                     // out[u] and triangle counting -- not maintained by the update kernels
  GraphCtrl* ctrl;
  uint32_t V, H, P, seed;   // V: vertices held here (vmeta entries); H/P: arena / pool slabs
  uint32_t Vg;              // global vertex count: the key range
  uint32_t ws, rank;        // vertex partition: this store holds the sources u with owner(u) == rank, at row(u)
  uint32_t pbits;           // placement domain [0, 2^pbits) of pm_mix (ws > 1)
};

// ---- Vertex placement of a partitioned graph ("let the library place
// vertices through a bijective mixer"): m = pm_mix(v) is a bijection on [0, V) -- two rounds of
// (multiply by an odd constant, xor-shift) on [0, 2^bits), cycle-walked back into [0, V) -- and
// owner(v) = m % ws, row(v) = m / ws.  Unscrambled R-MAT ids (whose low bits are skewed) land
// balanced; results do not depend on the placement (tree arrays are exported in global id order).
// world_size 1 is the identity.
constexpr uint32_t PM_A1 = 0x9E3779B1u, PM_A2 = 0x85EBCA77u;
__host__ __device__ constexpr uint32_t pm_inv(uint32_t a) {   // inverse of an odd a mod 2^32 (Newton)
  uint32_t x = a;
  for (int i = 0; i < 5; i++) x *= 2u - a * x;
  return x;
}
__host__ __device__ __forceinline__ uint32_t pm_mask(uint32_t bits) { return bits >= 32 ? 0xFFFFFFFFu : (1u << bits) - 1u; }
__host__ __device__ __forceinline__ uint32_t pm_step(uint32_t x, uint32_t a, uint32_t bits) {
  x = (x * a) & pm_mask(bits);
  return x ^ (x >> ((bits + 1) / 2));
}
__host__ __device__ __forceinline__ uint32_t pm_unstep(uint32_t y, uint32_t ainv, uint32_t bits) {
  const uint32_t s = (bits + 1) / 2;
  uint32_t x = y;
  for (uint32_t k = s; k < bits; k += s) x = y ^ (x >> s);   // invert x ^ (x >> s)
  return (x * ainv) & pm_mask(bits);
}
__host__ __device__ __forceinline__ uint32_t pm_mix(uint32_t v, uint32_t V, uint32_t bits) {
  uint32_t x = v;
  do { x = pm_step(pm_step(x, PM_A1, bits), PM_A2, bits); } while (x >= V);
  return x;
}
__host__ __device__ __forceinline__ uint32_t pm_unmix(uint32_t m, uint32_t V, uint32_t bits) {
  constexpr uint32_t I1 = pm_inv(PM_A1), I2 = pm_inv(PM_A2);
  uint32_t x = m;
  do { x = pm_unstep(pm_unstep(x, I2, bits), I1, bits); } while (x >= V);
  return x;
}
__host__ __device__ __forceinline__ uint32_t pm_bits(uint32_t V) {
  uint32_t b = 1;
  while (b < 32 && (1ull << b) < V) b++;
  return b;
}
// owner rank of global id x, and its row there
__host__ __device__ __forceinline__ uint32_t pm_place(uint32_t x, uint32_t V, uint32_t bits, uint32_t ws, uint32_t& row) {
  if (ws <= 1) { row = x; return 0; }
  const uint32_t m = pm_mix(x, V, bits);
  row = m / ws;
  return m % ws;
}
__host__ __device__ __forceinline__ uint32_t pm_global(uint32_t row, uint32_t rank, uint32_t V, uint32_t bits, uint32_t ws) {
  return ws <= 1 ? row : pm_unmix(row * ws + rank, V, bits);
}
__device__ __forceinline__ uint32_t g_place(const GraphDev& G, uint32_t x, uint32_t& row) {
  return pm_place(x, G.Vg, G.pbits, G.ws, row);
}
__device__ __forceinline__ uint32_t g_global(const GraphDev& G, uint32_t row) {
  return pm_global(row, G.rank, G.Vg, G.pbits, G.ws);
}

// Source id -> local row, or INVALID_SLAB if u is not held by this partition.
__device__ __forceinline__ uint32_t local_row(const GraphDev& G, uint32_t u) {
  if (G.ws <= 1) return u;
  uint32_t row;
  return g_place(G, u, row) == G.rank ? row : INVALID_SLAB;
}

__device__ __forceinline__ uint32_t* slab_ptr(const GraphDev& G, uint32_t s) {
  return G.slabs + (size_t)s * SLAB_WORDS;
}

// Bucket hash ("determined by a hashing function", unnamed; reading C21):
// a murmur3 finaliser of the key, range-reduced by a multiply-high.  Storage only.
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ uint32_t bucket_of(uint32_t key, uint32_t count, uint32_t seed) {
  return count <= 1 ? 0u : __umulhi(mix32(key ^ seed), count);
}

// Coherent 16-B slab fragment load for kernels that race with writers (update kernels).
__device__ __forceinline__ uint4 ld_slab_cg(const uint32_t* slab, int l8) {
  return __ldcg(reinterpret_cast<const uint4*>(slab) + l8);
}
// Read-only streaming load for traversal kernels (the store is immutable while a tree kernel runs).
__device__ __forceinline__ uint4 ld_slab_ro(const uint32_t* slab, int l8) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(reinterpret_cast<const uint4*>(slab) + l8));
  return r;
}
__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t* p) {
  return __ldcg(reinterpret_cast<const unsigned long long*>(p));
}

// Keys held by one lane's 16-B fragment: MAP -> 2 pairs (x,y),(z,w); SET -> 4 keys.
// Cell index c = l8 * NK + k.  The last cell of lane 7 is not a key cell
// (MAP: pair 15 = lanes 30/31; SET: lane 31 = next pointer).
template <bool MAP> struct Frag {
  static constexpr int NK = MAP ? 2 : 4;
  __device__ __forceinline__ static uint32_t key(const uint4& d, int k) {
    if (MAP) return k == 0 ? d.x : d.z;
    return k == 0 ? d.x : (k == 1 ? d.y : (k == 2 ? d.z : d.w));
  }
  __device__ __forceinline__ static uint32_t weight(const uint4& d, int k) { return k == 0 ? d.y : d.w; }
  __device__ __forceinline__ static bool valid_cell(int l8, int k) { return !(l8 == GROUP - 1 && k == NK - 1); }
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Batch fingerprint (ordering contract): an order-independent sum over the batch's edges of a
// 64-bit mix of (src, dst) and of (src, dst, w).  Same function on the mutation and the tree side.
__host__ __device__ __forceinline__ uint64_t fp_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ void fp_edge(uint32_t s, uint32_t d, uint32_t w, uint64_t& a, uint64_t& b) {
  const uint64_t h = fp_mix(((uint64_t)s << 32) | d);
  a += h;
  b += fp_mix(h + w);
}

// First cell (in chain order) whose per-lane predicate bits are set.
// bits: NK-bit mask of this lane's cells.  Returns cell index or -1 (group-uniform).
template <int NK>
__device__ __forceinline__ int group_first_cell(uint32_t bits, uint32_t gmask, int gbase) {
  uint32_t any = (__ballot_sync(gmask, bits != 0) >> gbase) & 0xFFu;
  if (!any) return -1;
  int l = __ffs(any) - 1;
  uint32_t lb = __shfl_sync(gmask, bits, l, GROUP);
  return l * NK + (__ffs(lb) - 1);
}

}  // namespace mk
