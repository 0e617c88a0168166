// api.cu — the C ABI declared in include/meerkat.h: argument checking, pointer
// staging, stream ordering, version checks and status translation around the
// launchers in store.cu and tree.cu.  No compute happens here.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>

#include "graph.h"

using namespace mk;

namespace {

meerkat_status from_cuda(cudaError_t e) { return e == cudaSuccess ? MEERKAT_OK : MEERKAT_E_CUDA; }

meerkat_status from_err(uint32_t err) {
  if (err & ERR_PARTITION) return MEERKAT_E_PARTITION;
  if (err & ERR_RANGE) return MEERKAT_E_VERTEX_RANGE;
  if (err & ERR_WEIGHT) return MEERKAT_E_WEIGHT;
  if (err & ERR_CAPACITY) return MEERKAT_E_CAPACITY;
  if (err & ERR_OVERFLOW) return MEERKAT_E_OVERFLOW;
  if (err & ERR_STATE) return MEERKAT_E_STATE;
  return MEERKAT_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) cudaSetDevice(d);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

namespace mk {

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

cudaError_t ensure_stage(meerkat_graph* g, int slot, size_t bytes) {
  g->staged_host[slot] = nullptr;   // the slot's content is about to change
  if (g->stage_bytes[slot] >= bytes) return cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return e;
  cudaFree(g->stage[slot]);
  g->stage[slot] = nullptr;
  g->stage_bytes[slot] = 0;
  size_t cap = std::max<size_t>(bytes, 1 << 16);
  e = cudaMalloc(&g->stage[slot], cap);
  if (e == cudaSuccess) g->stage_bytes[slot] = cap;
  return e;
}

// Device view of a caller array: device pointers pass through, host arrays are
// copied into the graph's staging slot on its stream.
cudaError_t stage_in(meerkat_graph* g, int slot, const void* p, size_t bytes, const void** out) {
  *out = p;
  if (!p || !bytes || is_device_ptr(p)) return cudaSuccess;
  g->staged_host[slot] = nullptr;
  cudaError_t e = ensure_stage(g, slot, bytes);
  if (e != cudaSuccess) return e;
  *out = g->stage[slot];
  return cudaMemcpyAsync(g->stage[slot], p, bytes, cudaMemcpyHostToDevice, g->stream);
}

// A mutation's host batch, staged in `slot`, stays reusable until the slot is overwritten: the tree
// update that must follow with the same batch (ordering contract, meerkat.h) does not copy it again.
void remember_stage(meerkat_graph* g, int slot, const void* p, size_t bytes) {
  if (!p || !bytes || is_device_ptr(p)) return;
  g->staged_host[slot] = p;
  g->staged_len[slot] = bytes;
  g->staged_version[slot] = g->version;
}

}  // namespace mk

namespace {

cudaError_t stage_in_reuse(meerkat_graph* g, int slot, const void* p, size_t bytes, const void** out) {
  if (p && bytes && p == g->staged_host[slot] && bytes == g->staged_len[slot] && g->staged_version[slot] == g->version) {
    *out = g->stage[slot];
    return cudaSuccess;
  }
  return stage_in(g, slot, p, bytes, out);
}

}  // namespace

namespace mk {

// Read the control block back (synchronises); returns and clears the sticky error.
meerkat_status collect(meerkat_graph* g) {
  cudaError_t e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess && g->reverse)
    e = cudaMemcpyAsync(g->in.hctrl, g->in.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  uint32_t err = g->out.hctrl->err;
  if (g->reverse) err |= g->in.hctrl->err;
  if (err) {
    if (cudaMemsetAsync(&g->out.dev.ctrl->err, 0, 4, g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
    if (g->reverse && cudaMemsetAsync(&g->in.dev.ctrl->err, 0, 4, g->stream) != cudaSuccess) return MEERKAT_E_CUDA;
  }
  return from_err(err);
}

// Host bookkeeping of a mutation (ordering contract): version, kind and size of the batch; an empty
// batch launches no kernel, so its (zero) fingerprint slot is written here.
cudaError_t mutated(meerkat_graph* g, int kind, uint64_t n) {
  cudaError_t e = cudaSuccess;
  if (!n) e = cudaMemsetAsync(&g->out.dev.ctrl->fp[0][0], 0, sizeof(g->out.dev.ctrl->fp), g->stream);
  g->version++;
  g->last_kind = kind;
  g->last_n = n;
  if (kind == 2) g->last_delete_version = g->version;
  return e;
}

}  // namespace mk

namespace {

meerkat_status check_batch(meerkat_graph* g, const uint32_t* s, const uint32_t* d, uint64_t n) {
  if (!g) return MEERKAT_E_INVALID_ARG;
  if (n && (!s || !d)) return MEERKAT_E_INVALID_ARG;
  return MEERKAT_OK;
}

}  // namespace

extern "C" {

const char* meerkat_status_string(meerkat_status s) {
  switch (s) {
    case MEERKAT_OK: return "MEERKAT_OK";
    case MEERKAT_E_INVALID_ARG: return "MEERKAT_E_INVALID_ARG";
    case MEERKAT_E_VERTEX_RANGE: return "MEERKAT_E_VERTEX_RANGE";
    case MEERKAT_E_WEIGHT: return "MEERKAT_E_WEIGHT";
    case MEERKAT_E_CAPACITY: return "MEERKAT_E_CAPACITY";
    case MEERKAT_E_OVERFLOW: return "MEERKAT_E_OVERFLOW";
    case MEERKAT_E_STATE: return "MEERKAT_E_STATE";
    case MEERKAT_E_CUDA: return "MEERKAT_E_CUDA";
    case MEERKAT_E_NCCL: return "MEERKAT_E_NCCL";
    case MEERKAT_E_PARTITION: return "MEERKAT_E_PARTITION";
  }
  return "MEERKAT_E_UNKNOWN";
}

meerkat_status meerkat_create(const meerkat_config* cfg, meerkat_graph** out) {
  if (!cfg || !out) return MEERKAT_E_INVALID_ARG;
  *out = nullptr;
  const float lf = cfg->load_factor == 0.0f ? 0.7f : cfg->load_factor;
  if (cfg->vertex_n == 0 || cfg->vertex_n >= 0xFFFFFFFCu || !(lf > 0.0f && lf <= 1.0f) ||
      !(cfg->in_load_factor >= 0.0f && cfg->in_load_factor <= 1.0f))
    return MEERKAT_E_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
    cudaGetLastError();
    return MEERKAT_E_CUDA;
  }
  DeviceGuard dg(cfg->device);
  meerkat_graph* g = new (std::nothrow) meerkat_graph();
  if (!g) return MEERKAT_E_CUDA;
  g->device = cfg->device;
  g->stream = static_cast<cudaStream_t>(cfg->stream);
  g->V = cfg->vertex_n;
  const bool partitioned = cfg->nccl_id != nullptr || cfg->exchange != nullptr;
  g->ws = cfg->world_size > 1 ? cfg->world_size : 1;
  g->rank = g->ws > 1 ? cfg->rank : 0;
  if (g->ws > MEERKAT_MAX_RANKS || g->rank >= g->ws || g->V <= g->rank || (g->ws > 1 && !partitioned)) {
    delete g;
    return MEERKAT_E_INVALID_ARG;
  }
  g->Vl = (g->V - g->rank + g->ws - 1) / g->ws;   // rows m < V with m % ws == rank (pm_place)
  g->weighted = cfg->weighted != 0;
  g->hashing = cfg->hashing != 0;
  g->lf = lf;
  g->lf_in = cfg->in_load_factor == 0.0f ? lf : cfg->in_load_factor;
  g->reverse = cfg->reverse != 0;
  g->out.dev.seed = (uint32_t)(cfg->hash_seed ^ (cfg->hash_seed >> 32)) ^ 0x5bd1e995u;
  g->in.dev.seed = g->out.dev.seed ^ 0x27d4eb2fu;
  cudaError_t e = cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, g->device);
  const void* hints = nullptr;
  // partitioned: the global hint arrays are gathered into this rank's rows
  auto hints_of = [&](const uint32_t* h, int slot) -> cudaError_t {
    if (!partitioned) return stage_in(g, slot, h, (size_t)g->Vl * 4, &hints);
    return part_hints(g, h, &hints, slot) == MEERKAT_OK ? cudaSuccess : cudaErrorUnknown;
  };
  if (e == cudaSuccess) e = hints_of(cfg->degree_hints, 0);
  if (e == cudaSuccess) e = launch_build(g, g->out, static_cast<const uint32_t*>(hints), cfg->pool_slabs);
  if (e == cudaSuccess && g->reverse) {
    e = hints_of(cfg->in_degree_hints, 1);
    if (e == cudaSuccess) e = launch_build(g, g->in, static_cast<const uint32_t*>(hints), cfg->pool_slabs);
  }
  if (e == cudaSuccess && cfg->update_tracking) {   // UpdateIterator metadata
    Store& o = g->out;
    e = cudaMalloc(&o.dev.upd, (size_t)(o.H + o.P) * 8);
    if (e == cudaSuccess) e = cudaMemsetAsync(o.dev.upd, 0xFF, (size_t)(o.H + o.P) * 8, g->stream);
    if (e == cudaSuccess) e = cudaMalloc(&o.dev.updq, (size_t)std::max<uint64_t>(o.buckets, 1) * 4);
    o.bytes += (size_t)(o.H + o.P) * 8 + (size_t)o.buckets * 4;
  }
  if (e == cudaSuccess) e = tree_occupancy(g);
  if (const char* s = std::getenv("MEERKAT_LATENCY_BLOCKS_PER_SM")) g->latency_bps = std::atoi(s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) {
    cudaGetLastError();
    meerkat_destroy(g);
    return MEERKAT_E_CUDA;
  }
  if (partitioned) {   // transport (NCCL communicator: collective), rings, exchange blocks
    const meerkat_status st = part_init(g, cfg);
    if (st != MEERKAT_OK) {
      cudaGetLastError();
      meerkat_destroy(g);
      return st;
    }
  }
  *out = g;
  return MEERKAT_OK;
}

meerkat_status meerkat_destroy(meerkat_graph* g) {
  if (!g) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  cudaStreamSynchronize(g->stream);
  part_free(g);
  free_store(g->out);
  free_store(g->in);
  for (int i = 0; i < 4; i++) cudaFree(g->stage[i]);
  delete g;
  return MEERKAT_OK;
}

meerkat_status meerkat_set_stream(meerkat_graph* g, void* stream) {
  if (!g) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaStreamSynchronize(g->stream);
  g->stream = static_cast<cudaStream_t>(stream);
  return from_cuda(e);
}

meerkat_status meerkat_sync(meerkat_graph* g) {
  if (!g) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  return collect(g);
}

meerkat_status meerkat_insert_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                                    uint64_t n, uint64_t* n_inserted) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  if (n && (g->weighted != (w != nullptr))) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  const void *s, *d, *ww = nullptr;
  cudaError_t e = stage_in(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in(g, 1, dst, n * 4, &d);
  if (e == cudaSuccess && w) e = stage_in(g, 2, w, n * 4, &ww);
  if (e == cudaSuccess && g->part)   // collective: routed by owner (part.cu)
    return part_mutate(g, 1, (const uint32_t*)s, (const uint32_t*)d, (const uint32_t*)ww, n, n_inserted);
  if (e == cudaSuccess && n_inserted) e = cudaMemsetAsync(&g->out.dev.ctrl->n_inserted, 0, 8, g->stream);
  if (e == cudaSuccess)
    e = launch_insert(g, &g->out, g->reverse ? &g->in : nullptr,   // in-edge mirror: (dst, src, w)
                      (const uint32_t*)s, (const uint32_t*)d, (const uint32_t*)ww, n);
  if (e == cudaSuccess) e = mutated(g, 1, n);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  remember_stage(g, 0, src, n * 4);
  remember_stage(g, 1, dst, n * 4);
  if (w) remember_stage(g, 2, w, n * 4);
  if (!n_inserted) return MEERKAT_OK;
  st = collect(g);
  *n_inserted = g->out.hctrl->n_inserted;
  return st;
}

meerkat_status meerkat_delete_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                    uint64_t* n_deleted) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  DeviceGuard dg(g->device);
  const void *s, *d;
  cudaError_t e = stage_in(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in(g, 1, dst, n * 4, &d);
  if (e == cudaSuccess && g->part)   // collective: routed by owner (part.cu)
    return part_mutate(g, 2, (const uint32_t*)s, (const uint32_t*)d, nullptr, n, n_deleted);
  if (e == cudaSuccess && n_deleted) e = cudaMemsetAsync(&g->out.dev.ctrl->n_deleted, 0, 8, g->stream);
  if (e == cudaSuccess)
    e = launch_delete(g, &g->out, g->reverse ? &g->in : nullptr, (const uint32_t*)s, (const uint32_t*)d, n);
  if (e == cudaSuccess) e = mutated(g, 2, n);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  remember_stage(g, 0, src, n * 4);
  remember_stage(g, 1, dst, n * 4);
  if (!n_deleted) return MEERKAT_OK;
  st = collect(g);
  *n_deleted = g->out.hctrl->n_deleted;
  return st;
}

meerkat_status meerkat_query_batch(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                   uint8_t* found, uint32_t* w_out) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  if (n && !found) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  const void *s, *d;
  cudaError_t e = stage_in(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in(g, 1, dst, n * 4, &d);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (g->part) return part_query(g, (const uint32_t*)s, (const uint32_t*)d, n, found, w_out);
  const bool host_f = n && !is_device_ptr(found);
  const bool host_w = n && w_out && !is_device_ptr(w_out);
  uint8_t* df = found;
  uint32_t* dw = w_out;
  if (host_f) { e = ensure_stage(g, 2, n); df = (uint8_t*)g->stage[2]; }
  if (e == cudaSuccess && host_w) { e = ensure_stage(g, 3, n * 4); dw = (uint32_t*)g->stage[3]; }
  if (e == cudaSuccess) e = launch_query(g, g->out, (const uint32_t*)s, (const uint32_t*)d, n, df, dw);
  if (e == cudaSuccess && host_f) e = cudaMemcpyAsync(found, df, n, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess && host_w) e = cudaMemcpyAsync(w_out, dw, n * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (host_f || host_w) return collect(g);
  return MEERKAT_OK;
}

meerkat_status meerkat_export_edges(meerkat_graph* g, uint32_t* src, uint32_t* dst, uint32_t* w, uint64_t capacity,
                                    uint64_t* n_out) {
  if (!g || !n_out || (capacity && (!src || !dst))) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  const bool host = capacity && !is_device_ptr(src);
  uint32_t *ds = src, *dd = dst, *dw = w;
  cudaError_t e = cudaSuccess;
  if (host) {
    e = ensure_stage(g, 0, capacity * 4);
    if (e == cudaSuccess) e = ensure_stage(g, 1, capacity * 4);
    if (e == cudaSuccess && w) e = ensure_stage(g, 2, capacity * 4);
    ds = (uint32_t*)g->stage[0]; dd = (uint32_t*)g->stage[1]; dw = w ? (uint32_t*)g->stage[2] : nullptr;
  }
  if (e == cudaSuccess) e = launch_export(g, g->out, ds, dd, dw, capacity);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  meerkat_status st = collect(g);
  const uint64_t n = g->out.hctrl->export_n;
  *n_out = n;
  if (host) {
    const uint64_t m = std::min(n, capacity);
    e = cudaMemcpyAsync(src, ds, m * 4, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, dd, m * 4, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess && w) e = cudaMemcpyAsync(w, dw, m * 4, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return MEERKAT_E_CUDA;
  }
  if (st != MEERKAT_OK) return st;
  return n > capacity ? MEERKAT_E_CAPACITY : MEERKAT_OK;
}

meerkat_status meerkat_check(meerkat_graph* g, uint64_t* info) {
  if (!g || !info) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 10 * 8);
  if (e == cudaSuccess) e = launch_fsck(g, g->out, d);
  if (e == cudaSuccess && g->reverse) e = launch_fsck(g, g->in, d + 5);
  uint64_t h[10] = {0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d, 10 * 8, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  cudaFree(d);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  for (int i = 0; i < 5; i++) info[i] = h[i] ? h[i] : h[5 + i];
  info[0] = h[0] + (g->reverse ? h[5] : 0);
  return info[0] ? MEERKAT_E_STATE : MEERKAT_OK;
}

meerkat_status meerkat_counters_async(meerkat_graph* g, uint64_t* out) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  const GraphCtrl* c = g->out.dev.ctrl;
  cudaError_t e = cudaMemcpyAsync(out, &c->ins_total, 8, cudaMemcpyDefault, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out + 1, &c->del_total, 8, cudaMemcpyDefault, g->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out + 2, &c->pool_top, 8, cudaMemcpyDefault, g->stream);
  return from_cuda(e);
}

meerkat_status meerkat_stats_get(meerkat_graph* g, meerkat_stats* out) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(g->out.hctrl, g->out.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess && g->reverse)
    e = cudaMemcpyAsync(g->in.hctrl, g->in.dev.ctrl, sizeof(GraphCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  std::memset(out, 0, sizeof(*out));
  const Store& o = g->out;
  out->vertex_n = g->V;
  out->edges = o.hctrl->ins_total - o.hctrl->del_total;
  out->head_slabs = o.H;
  out->buckets = o.buckets;
  out->pool_capacity = o.P;
  out->pool_used = std::min<uint64_t>(o.hctrl->pool_top, o.P);
  out->bytes_device = o.bytes + g->in.bytes;
  if (g->reverse) {
    out->in_head_slabs = g->in.H;
    out->in_pool_used = std::min<uint64_t>(g->in.hctrl->pool_top, g->in.P);
    out->in_edges = g->in.hctrl->ins_total - g->in.hctrl->del_total;
  }
  out->kernel_launches = g->launches;
  out->version = g->version;
  return MEERKAT_OK;
}

// ------------------------------------------------------------------ trees

static meerkat_status tree_create(meerkat_graph* g, uint32_t source, bool unit, meerkat_tree** out,
                                  bool vanilla = false) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  *out = nullptr;
  if (source >= g->V) return MEERKAT_E_VERTEX_RANGE;
  if (!unit && !g->weighted) return MEERKAT_E_STATE;   // SSSP needs weights
  if (g->part && vanilla) return MEERKAT_E_INVALID_ARG;   // single-GPU variant only
  DeviceGuard dg(g->device);
  meerkat_tree* t = new (std::nothrow) meerkat_tree();
  if (!t) return MEERKAT_E_CUDA;
  t->g = g;
  t->unit = unit;
  t->vanilla = vanilla;
  TreeDev& T = t->dev;
  T.source = source;
  T.unit = unit ? 1u : 0u;
  T.fr_cap = std::max<uint64_t>(std::max(g->out.buckets, g->in.buckets), 1);
  // node / stamp / invalid list: the vertices held here; invalid bit set: all vertices (global ids)
  const size_t V = g->Vl, words = ((size_t)g->V + 31) / 32;
  cudaError_t e = cudaMalloc(&T.node, V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&T.stamp, V * 4);
  if (e == cudaSuccess) e = cudaMalloc(&T.inval_bits, words * 4);
  if (e == cudaSuccess) e = cudaMalloc(&T.inval_list, V * 4);
  if (e == cudaSuccess) e = cudaMalloc(&T.fr[0], T.fr_cap * 8);
  if (e == cudaSuccess) e = cudaMalloc(&T.fr[1], T.fr_cap * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->ctrl_base, 2 * sizeof(TreeCtrl));   // double-buffered (tree.cu)
  if (e == cudaSuccess) e = cudaMalloc(&T.bstat, (size_t)STAT_BLOCKS * 8 * 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(T.bstat, 0, (size_t)STAT_BLOCKS * 8 * 8, g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->ctrl_base, 0, 2 * sizeof(TreeCtrl), g->stream);
  T.ctrl = t->ctrl_base;
  if (e == cudaSuccess) e = cudaMalloc(&T.epoch_ptr, 8);   // [0] epoch, [1] stale flag
  if (e == cudaSuccess) e = cudaMallocHost(&t->hctrl, sizeof(TreeCtrl));
  if (e == cudaSuccess) e = cudaMemsetAsync(T.stamp, 0, V * 4, g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(T.inval_bits, 0, words * 4, g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(T.epoch_ptr, 0, 8, g->stream);
  if (e == cudaSuccess) {
    const uint32_t one = 1;
    e = cudaMemcpyAsync(T.epoch_ptr, &one, 4, cudaMemcpyHostToDevice, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  }
  t->bytes = V * 8 + V * 4 + words * 4 + V * 4 + 2 * T.fr_cap * 8 + 2 * sizeof(TreeCtrl) + 4;
  if (e != cudaSuccess) {
    cudaGetLastError();
    meerkat_tree_destroy(t);
    return MEERKAT_E_CUDA;
  }
  if (g->part) {   // collective static tree (part.cu)
    const meerkat_status st = part_tree_init(g, t);
    if (st != MEERKAT_OK) { meerkat_tree_destroy(t); return st; }
  } else {
    e = launch_tree(g, &t, 1, MODE_STATIC, nullptr, nullptr, nullptr, 0);
    if (e != cudaSuccess) {
      cudaGetLastError();
      meerkat_tree_destroy(t);
      return MEERKAT_E_CUDA;
    }
  }
  t->version = g->version;
  if (!vanilla) { g->n_trees++; t->counted = true; }
  *out = t;
  return MEERKAT_OK;
}

meerkat_status meerkat_sssp_create(meerkat_graph* g, uint32_t source, meerkat_tree** out) {
  return tree_create(g, source, false, out);
}

meerkat_status meerkat_bfs_create(meerkat_graph* g, uint32_t source, meerkat_tree** out) {
  return tree_create(g, source, true, out);
}

meerkat_status meerkat_sssp_vanilla_create(meerkat_graph* g, uint32_t source, meerkat_tree** out) {
  return tree_create(g, source, false, out, true);
}

meerkat_status meerkat_bfs_vanilla_create(meerkat_graph* g, uint32_t source, meerkat_tree** out) {
  return tree_create(g, source, true, out, true);
}

meerkat_status meerkat_tree_distances(meerkat_tree* t, uint32_t* out) {
  if (!t || !out || t->part) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = t->g;
  DeviceGuard dg(g->device);
  const bool host = !is_device_ptr(out);
  uint32_t* d = out;
  cudaError_t e = cudaSuccess;
  if (host) {
    e = ensure_stage(g, 3, (size_t)g->Vl * 4);
    d = static_cast<uint32_t*>(g->stage[3]);
  }
  if (e == cudaSuccess) e = launch_node_dist(g, t, d);
  if (e == cudaSuccess && host) e = cudaMemcpyAsync(out, d, (size_t)g->Vl * 4, cudaMemcpyDeviceToHost, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (host) return collect(g);
  return MEERKAT_OK;
}

// Mutation-following update of one or more trees of g with the same batch (fused launch).
static meerkat_status trees_update(meerkat_graph* g, meerkat_tree* const* ts, uint32_t k, int kind, const uint32_t* src,
                                   const uint32_t* dst, const uint32_t* w, uint64_t n) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  if (!ts || k == 0 || k > (uint32_t)MAX_TREES) return MEERKAT_E_INVALID_ARG;
  if (g->part) {   // collective, device-driven exchange units (part.cu)
    DeviceGuard dg(g->device);
    return part_trees(g, ts, k, kind, src, dst, w, n);
  }
  bool need_w = false;
  for (uint32_t i = 0; i < k; i++) {
    meerkat_tree* t = ts[i];
    if (!t || t->g != g) return MEERKAT_E_INVALID_ARG;
    if (t->vanilla) return MEERKAT_E_STATE;   // no dependence tree: static only
    for (uint32_t j = 0; j < i; j++)
      if (ts[j] == t) return MEERKAT_E_INVALID_ARG;
    // ordering contract: the batch must be the mutation just applied -- same kind, the
    // very next version, the same size here; the same edges (fingerprint) on the device
    if (g->last_kind != kind || t->version + 1 != g->version || n != g->last_n) return MEERKAT_E_STATE;
    // seeded by that mutation (insert_batch_trees / delete_batch_trees): all the call's trees or none
    if ((t->seeded != 0) != (ts[0]->seeded != 0) || (t->seeded && t->seeded != kind)) return MEERKAT_E_STATE;
    need_w |= kind == 1 && !t->unit;
  }
  if (need_w && n && !w) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  const void *s, *d, *ww = nullptr;
  cudaError_t e = stage_in_reuse(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in_reuse(g, 1, dst, n * 4, &d);
  if (e == cudaSuccess && need_w) e = stage_in_reuse(g, 2, w, n * 4, &ww);
  if (e == cudaSuccess)
    e = launch_tree(g, ts, k, kind == 1 ? MODE_INCREMENTAL : MODE_DECREMENTAL, (const uint32_t*)s, (const uint32_t*)d,
                    (const uint32_t*)ww, n, ts[0]->seeded != 0,
                    // seeded: the mutation kernel already ran the prologue on the batch it applied, so
                    // the tree call reads no batch and needs no fingerprint
                    ts[0]->seeded ? -1 : (ww ? 1 : 0));
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  for (uint32_t i = 0; i < k; i++) { ts[i]->version = g->version; ts[i]->seeded = 0; }
  return MEERKAT_OK;
}

static meerkat_status tree_update(meerkat_graph* g, meerkat_tree* t, bool unit, int kind, const uint32_t* src,
                                  const uint32_t* dst, const uint32_t* w, uint64_t n) {
  if (!t || t->unit != unit) return MEERKAT_E_INVALID_ARG;
  return trees_update(g, &t, 1, kind, src, dst, unit ? nullptr : w, n);
}

// Mutation that also seeds the trees' next call (P:24-26 order: the batch is applied, then the
// trees follow): the trees' batch prologue (relaxation of the inserted edges / invalidation of the
// deleted tree edges) runs inside the insert / delete kernel; the trees_* call that must follow
// with the same batch starts at its first frontier round.
static meerkat_status batch_seed(meerkat_graph* g, int kind, const uint32_t* src, const uint32_t* dst,
                                 const uint32_t* w, uint64_t n, meerkat_tree* const* ts, uint32_t k,
                                 uint64_t* n_changed) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  if (kind == 1 && n && (g->weighted != (w != nullptr))) return MEERKAT_E_INVALID_ARG;
  if (!ts || k == 0 || k > (uint32_t)MAX_TREES || g->part) return MEERKAT_E_INVALID_ARG;
  for (uint32_t i = 0; i < k; i++) {
    meerkat_tree* t = ts[i];
    if (!t || t->g != g) return MEERKAT_E_INVALID_ARG;
    if (t->vanilla) return MEERKAT_E_STATE;   // no dependence tree: static only
    for (uint32_t j = 0; j < i; j++)
      if (ts[j] == t) return MEERKAT_E_INVALID_ARG;
    if (t->version != g->version || t->seeded) return MEERKAT_E_STATE;   // must be current, not seeded
  }
  DeviceGuard dg(g->device);
  const void *s, *d, *ww = nullptr;
  cudaError_t e = stage_in(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in(g, 1, dst, n * 4, &d);
  if (e == cudaSuccess && kind == 1 && w) e = stage_in(g, 2, w, n * 4, &ww);
  unsigned long long* cnt = kind == 1 ? &g->out.dev.ctrl->n_inserted : &g->out.dev.ctrl->n_deleted;
  if (e == cudaSuccess && n_changed) e = cudaMemsetAsync(cnt, 0, 8, g->stream);
  TreePro P;
  tree_pro_fill(ts, k, P);
  Store* mirror = g->reverse ? &g->in : nullptr;
  if (e == cudaSuccess)
    e = kind == 1 ? launch_insert(g, &g->out, mirror, (const uint32_t*)s, (const uint32_t*)d, (const uint32_t*)ww, n, &P)
                  : launch_delete(g, &g->out, mirror, (const uint32_t*)s, (const uint32_t*)d, n, &P);
  if (e == cudaSuccess) e = mutated(g, kind, n);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  remember_stage(g, 0, src, n * 4);
  remember_stage(g, 1, dst, n * 4);
  if (ww) remember_stage(g, 2, w, n * 4);
  for (uint32_t i = 0; i < k; i++) ts[i]->seeded = kind;
  if (!n_changed) return MEERKAT_OK;
  st = collect(g);
  *n_changed = kind == 1 ? g->out.hctrl->n_inserted : g->out.hctrl->n_deleted;
  return st;
}

meerkat_status meerkat_insert_batch_trees(meerkat_graph* g, const uint32_t* src, const uint32_t* dst,
                                          const uint32_t* w, uint64_t n, meerkat_tree* const* trees,
                                          uint32_t n_trees, uint64_t* n_inserted) {
  return batch_seed(g, 1, src, dst, w, n, trees, n_trees, n_inserted);
}

meerkat_status meerkat_delete_batch_trees(meerkat_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                                          meerkat_tree* const* trees, uint32_t n_trees, uint64_t* n_deleted) {
  return batch_seed(g, 2, src, dst, nullptr, n, trees, n_trees, n_deleted);
}

meerkat_status meerkat_trees_incremental(meerkat_graph* g, meerkat_tree* const* trees, uint32_t n_trees,
                                         const uint32_t* src, const uint32_t* dst, const uint32_t* w, uint64_t n) {
  return trees_update(g, trees, n_trees, 1, src, dst, w, n);
}

meerkat_status meerkat_trees_decremental(meerkat_graph* g, meerkat_tree* const* trees, uint32_t n_trees,
                                         const uint32_t* src, const uint32_t* dst, uint64_t n) {
  return trees_update(g, trees, n_trees, 2, src, dst, nullptr, n);
}

meerkat_status meerkat_sssp_incremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src, const uint32_t* dst,
                                        const uint32_t* w, uint64_t n) {
  return tree_update(g, t, false, 1, src, dst, w, n);
}

meerkat_status meerkat_bfs_incremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src, const uint32_t* dst,
                                       uint64_t n) {
  return tree_update(g, t, true, 1, src, dst, nullptr, n);
}

meerkat_status meerkat_sssp_decremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src, const uint32_t* dst,
                                        uint64_t n) {
  return tree_update(g, t, false, 2, src, dst, nullptr, n);
}

meerkat_status meerkat_bfs_decremental(meerkat_graph* g, meerkat_tree* t, const uint32_t* src, const uint32_t* dst,
                                       uint64_t n) {
  return tree_update(g, t, true, 2, src, dst, nullptr, n);
}

// A seeded tree whose trees_* call never came (the graph moved on): drop the seeded frontier,
// counters and V_invalid marks before a static re-run.
static cudaError_t unseed(meerkat_graph* g, meerkat_tree* t) {
  if (!t->seeded) return cudaSuccess;
  t->seeded = 0;
  cudaError_t e = cudaMemsetAsync(t->ctrl_base + t->parity, 0, sizeof(TreeCtrl), g->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(t->dev.inval_bits, 0, ((size_t)g->V + 31) / 32 * 4, g->stream);
  return e;
}

meerkat_status meerkat_tree_recompute_scheme(meerkat_graph* g, meerkat_tree* t, uint32_t iteration_scheme) {
  if (!g || !t || t->g != g || t->part || (iteration_scheme != 1 && iteration_scheme != 2))
    return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  t->dev.scheme1 = iteration_scheme == 1 ? 1u : 0u;
  cudaError_t e = unseed(g, t);
  if (e == cudaSuccess) e = launch_tree(g, &t, 1, MODE_STATIC, nullptr, nullptr, nullptr, 0);
  t->dev.scheme1 = 0;   // dynamic updates always use <vertex, bucket> items
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  t->version = g->version;
  return MEERKAT_OK;
}

meerkat_status meerkat_tree_recompute(meerkat_graph* g, meerkat_tree* t) {
  if (!g || !t || t->g != g) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  if (t->part) return part_trees(g, &t, 1, 0, nullptr, nullptr, nullptr, 0);
  cudaError_t e = unseed(g, t);
  if (e == cudaSuccess) e = launch_tree(g, &t, 1, MODE_STATIC, nullptr, nullptr, nullptr, 0);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  t->version = g->version;
  return MEERKAT_OK;
}

meerkat_status meerkat_tree_nodes(meerkat_tree* t, uint64_t* out) {
  if (!t || !out) return MEERKAT_E_INVALID_ARG;
  if (t->vanilla) return MEERKAT_E_STATE;   // distances only: meerkat_tree_distances
  meerkat_graph* g = t->g;
  DeviceGuard dg(g->device);
  if (t->part) return part_tree_nodes(t, out);   // collective all-gather, global id order
  const bool host = !is_device_ptr(out);
  cudaError_t e = cudaMemcpyAsync(out, t->dev.node, (size_t)g->Vl * 8,
                                  host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (host) return collect(g);
  return MEERKAT_OK;
}

meerkat_status meerkat_tree_invalidated(meerkat_tree* t, uint32_t* out, uint64_t capacity, uint64_t* n_out) {
  if (!t || !n_out || (capacity && !out)) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = t->g;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(t->hctrl, t->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  const uint64_t n = t->hctrl->inval_n;
  *n_out = n;
  const uint64_t m = std::min(n, capacity);
  if (m) {
    const bool host = !is_device_ptr(out);
    e = cudaMemcpyAsync(out, t->dev.inval_list, m * 4, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                        g->stream);
    if (e == cudaSuccess && host) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return MEERKAT_E_CUDA;
  }
  return n > capacity ? MEERKAT_E_CAPACITY : MEERKAT_OK;
}

meerkat_status meerkat_tree_stats_get(meerkat_tree* t, meerkat_tree_stats* out) {
  if (!t || !out) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = t->g;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(t->hctrl, t->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  // the last single-GPU call's per-block slots (its finish stored them instead of adding)
  if (t->stat_blocks && !t->part) {
    static thread_local unsigned long long slots[STAT_BLOCKS * 8];
    e = cudaMemcpyAsync(slots, t->dev.bstat, (size_t)t->stat_blocks * 8 * 8, cudaMemcpyDeviceToHost, g->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
    if (e != cudaSuccess) return MEERKAT_E_CUDA;
    unsigned long long* dst[8] = {&t->hctrl->items, &t->hctrl->slabs_read, &t->hctrl->visited, &t->hctrl->improved,
                                  &t->hctrl->scan_slabs, &t->hctrl->scan_hits, &t->hctrl->batch_edges,
                                  &t->hctrl->direct_n};
    for (uint32_t b = 0; b < t->stat_blocks; b++)
      for (int i = 0; i < 8; i++) *dst[i] += slots[(size_t)b * 8 + i];
  }
  const TreeCtrl& c = *t->hctrl;
  std::memset(out, 0, sizeof(*out));
  out->rounds = c.rounds;
  out->propagate_rounds = c.prop_rounds;
  out->direct_invalid = c.direct_n;
  out->invalidated = c.inval_n;
  out->frontier_edges = c.scan_hits;
  out->items = c.items;
  out->slabs_read = c.slabs_read;
  out->scan_slabs = c.scan_slabs;
  out->improved = c.improved;
  // algorithmic bytes: item read + vmeta + node[v] + item write (32 B),
  // 128 B per slab walked or streamed, 8 B node[x] probe per visited edge, 12 B (atomicMin + stamp) per
  // improvement, 16 B (owner + node[u] + bit) per scan hit, 20 B per batch edge (src, dst, w, node[u]).
  out->alg_bytes = c.items * 32 + (c.slabs_read + c.scan_slabs) * 128 + c.visited * 8 + c.improved * 12 +
                   c.scan_hits * 16 + c.batch_edges * 20;
  out->version = t->version;
  out->source = t->dev.source;
  out->unit_weights = t->unit ? 1 : 0;
  out->exchanges = t->last_units;
  return MEERKAT_OK;
}

meerkat_status meerkat_tree_timeline(meerkat_tree* t, uint64_t* out, uint64_t* items, uint64_t capacity,
                                     uint64_t* n_out) {
  if (!t || !n_out || (capacity && !out)) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = t->g;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(t->hctrl, t->dev.ctrl, sizeof(TreeCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  const uint64_t n = std::min<uint64_t>(t->hctrl->nts, 48);
  *n_out = n;
  for (uint64_t i = 0; i < n && i < capacity; i++) {
    out[i] = t->hctrl->tstamp[i];
    if (items) items[i] = t->hctrl->titems[i];
  }
  return MEERKAT_OK;
}

meerkat_status meerkat_tree_destroy(meerkat_tree* t) {
  if (!t) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(t->g->device);
  cudaStreamSynchronize(t->g->stream);
  TreeDev& T = t->dev;
  cudaFree(T.node); cudaFree(T.stamp); cudaFree(T.inval_bits); cudaFree(T.inval_list);
  cudaFree(T.fr[0]); cudaFree(T.fr[1]); cudaFree(t->ctrl_base); cudaFree(T.epoch_ptr); cudaFree(T.bstat);
  if (t->hctrl) cudaFreeHost(t->hctrl);
  part_tree_free(t);
  if (t->counted) t->g->n_trees--;
  delete t;
  return MEERKAT_OK;
}

/* ------------------------------------------------------------------ PageRank (pagerank.cu) */

static meerkat_status pagerank_run(meerkat_graph* g, meerkat_pagerank* p, bool warm) {
  DeviceGuard dg(g->device);
  cudaError_t e = launch_pagerank(g, p, warm);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->hctrl, p->ctrl, sizeof(PRCtrl), cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) { cudaGetLastError(); return MEERKAT_E_CUDA; }
  p->version = g->version;
  p->warm_last = warm;
  return MEERKAT_OK;
}

meerkat_status meerkat_pagerank_create(meerkat_graph* g, double damping, double error_margin, uint32_t max_iter,
                                       meerkat_pagerank** out) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  *out = nullptr;
  if (!(damping > 0.0 && damping < 1.0) || !(error_margin > 0.0) || max_iter == 0) return MEERKAT_E_INVALID_ARG;
  if (!g->reverse || g->part) return MEERKAT_E_STATE;   // Compute walks in-edges
  DeviceGuard dg(g->device);
  meerkat_pagerank* p = new (std::nothrow) meerkat_pagerank();
  if (!p) return MEERKAT_E_CUDA;
  p->g = g;
  p->d = damping; p->eps = error_margin; p->max_iter = max_iter;
  const size_t V = g->V;
  cudaError_t e = cudaMalloc(&p->pr, V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&p->contrib, V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&p->acc, V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&p->ctrl, sizeof(PRCtrl));
  if (e == cudaSuccess) e = cudaMallocHost(&p->hctrl, sizeof(PRCtrl));
  if (e == cudaSuccess) e = pagerank_occupancy(g->weighted, &p->blocks_per_sm);
  if (e != cudaSuccess || p->blocks_per_sm <= 0) {
    cudaGetLastError();
    meerkat_pagerank_destroy(p);
    return MEERKAT_E_CUDA;
  }
  const meerkat_status st = pagerank_run(g, p, false);
  if (st != MEERKAT_OK) { meerkat_pagerank_destroy(p); return st; }
  *out = p;
  return MEERKAT_OK;
}

meerkat_status meerkat_pagerank_update(meerkat_graph* g, meerkat_pagerank* p) {
  if (!g || !p || p->g != g) return MEERKAT_E_INVALID_ARG;
  return pagerank_run(g, p, true);
}

meerkat_status meerkat_pagerank_recompute(meerkat_graph* g, meerkat_pagerank* p) {
  if (!g || !p || p->g != g) return MEERKAT_E_INVALID_ARG;
  return pagerank_run(g, p, false);
}

meerkat_status meerkat_pagerank_values(meerkat_pagerank* p, double* out) {
  if (!p || !out) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = p->g;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(out, p->pr, (size_t)g->V * 8, cudaMemcpyDefault, g->stream);
  if (e == cudaSuccess && !is_device_ptr(out)) e = cudaStreamSynchronize(g->stream);
  return from_cuda(e);
}

meerkat_status meerkat_pagerank_stats_get(meerkat_pagerank* p, meerkat_pagerank_stats* out) {
  if (!p || !out) return MEERKAT_E_INVALID_ARG;
  const PRCtrl& c = *p->hctrl;   // copied back at the end of every run
  std::memset(out, 0, sizeof(*out));
  out->iterations = c.iters;
  out->delta = c.last_delta;
  out->slabs = c.slabs;
  out->in_edges = c.keys;
  out->atomics = c.atomics;
  // algorithmic bytes: per super-step 128 B per slab + 4 B owner, 8 B Contribution
  // gather per in-edge, 8 B atomicAdd per combined slab run, 44 B per vertex update (acc r/w, PR r/w,
  // out[] r, Contribution w); plus the start, 28 B per vertex (PR r/w, out[] r, Contribution w, acc w)
  const uint64_t V = p->g->V;
  // per super-step: slab + owner per in-slab, one Contribution gather per in-edge, one fp64 atomic per
  // combined run, per vertex acc r/w + PR r/w + out r + Contribution w; once: the initial pass
  const uint64_t cb = pagerank_contrib_bytes();
  out->alg_bytes = c.iters * (c.slabs * 132 + c.keys * cb + c.atomics * 8 + V * (36 + cb)) + V * (20 + cb);
  out->version = p->version;
  out->warm = p->warm_last ? 1u : 0u;
  return MEERKAT_OK;
}

meerkat_status meerkat_pagerank_destroy(meerkat_pagerank* p) {
  if (!p) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(p->g->device);
  cudaStreamSynchronize(p->g->stream);
  cudaFree(p->pr); cudaFree(p->contrib); cudaFree(p->acc); cudaFree(p->ctrl);
  if (p->hctrl) cudaFreeHost(p->hctrl);
  delete p;
  return MEERKAT_OK;
}

/* ------------------------------------------------------------------ triangle counting (tc.cu) */

static meerkat_status tc_check(meerkat_graph* a, meerkat_graph* b) {
  if (!a || !b) return MEERKAT_E_INVALID_ARG;
  if (a->device != b->device || a->V != b->V) return MEERKAT_E_INVALID_ARG;
  if (a->part || b->part) return MEERKAT_E_STATE;
  return MEERKAT_OK;
}

// Count into a device scratch word and read it back (synchronises g1's stream).
static meerkat_status tc_count_sync(meerkat_graph* g1, meerkat_graph* g2, const uint32_t* src, const uint32_t* dst,
                                    uint64_t n, uint64_t* out) {
  DeviceGuard dg(g1->device);
  if (g2 != g1 && cudaStreamSynchronize(g2->stream) != cudaSuccess) return MEERKAT_E_CUDA;   // g2's updates done
  const void *s, *d;
  cudaError_t e = stage_in(g1, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in(g1, 1, dst, n * 4, &d);
  unsigned long long* acc = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(&acc, 8, g1->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(acc, 0, 8, g1->stream);
  if (e == cudaSuccess) e = launch_tc_count(g1, g2, (const uint32_t*)s, (const uint32_t*)d, n, acc);
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, acc, 8, cudaMemcpyDeviceToHost, g1->stream);
  if (acc) cudaFreeAsync(acc, g1->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g1->stream);
  if (e != cudaSuccess) { cudaGetLastError(); return MEERKAT_E_CUDA; }
  *out = h;
  return MEERKAT_OK;
}

meerkat_status meerkat_tc_count(meerkat_graph* g1, meerkat_graph* g2, const uint32_t* src, const uint32_t* dst,
                                uint64_t n, uint64_t* count) {
  meerkat_status st = tc_check(g1, g2);
  if (st != MEERKAT_OK) return st;
  if (!count || (n && (!src || !dst))) return MEERKAT_E_INVALID_ARG;
  return tc_count_sync(g1, g2, src, dst, n, count);
}

meerkat_status meerkat_tc_static(meerkat_graph* g, uint64_t* triangles) {
  meerkat_status st = tc_check(g, g);
  if (st != MEERKAT_OK) return st;
  if (!triangles) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  st = collect(g);
  if (st != MEERKAT_OK) return st;
  const uint64_t m = g->out.hctrl->ins_total - g->out.hctrl->del_total;   // live edges
  uint32_t *s = nullptr, *d = nullptr;
  cudaError_t e = cudaMemsetAsync(&g->out.dev.ctrl->export_n, 0, 8, g->stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&s, (m + 1) * 4, g->stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&d, (m + 1) * 4, g->stream);
  if (e == cudaSuccess) e = launch_export(g, g->out, s, d, nullptr, m);   // every directed edge (u, v)
  uint64_t c = 0;
  if (e == cudaSuccess) st = tc_count_sync(g, g, s, d, m, &c);
  if (s) cudaFreeAsync(s, g->stream);
  if (d) cudaFreeAsync(d, g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  if (st != MEERKAT_OK) return st;
  if (c % 6) return MEERKAT_E_STATE;   // not an undirected (symmetric) graph
  *triangles = c / 6;                  // each triangle is found six times
  return MEERKAT_OK;
}

static meerkat_status tc_delta(meerkat_graph* after, meerkat_graph* upd, const uint32_t* src, const uint32_t* dst,
                               uint64_t n, bool insert, uint64_t* delta, uint64_t* s3) {
  meerkat_status st = tc_check(after, upd);
  if (st != MEERKAT_OK) return st;
  if (!delta || (n && (!src || !dst))) return MEERKAT_E_INVALID_ARG;
  uint64_t s[3] = {0, 0, 0};
  st = tc_count_sync(after, after, src, dst, n, &s[0]);
  if (st == MEERKAT_OK) st = tc_count_sync(after, upd, src, dst, n, &s[1]);
  if (st == MEERKAT_OK) st = tc_count_sync(upd, upd, src, dst, n, &s[2]);
  if (st != MEERKAT_OK) return st;
  if (s3) { s3[0] = s[0]; s3[1] = s[1]; s3[2] = s[2]; }
  // added = S1/2 - S2/2 + S3/6, removed = S1/2 + S2/2 + S3/6, in exact integers
  const int64_t num = insert ? 3 * (int64_t)s[0] - 3 * (int64_t)s[1] + (int64_t)s[2]
                             : 3 * (int64_t)s[0] + 3 * (int64_t)s[1] + (int64_t)s[2];
  if (num < 0 || num % 6) return MEERKAT_E_STATE;   // broken precondition (DivisibilityViolation)
  *delta = (uint64_t)(num / 6);
  return MEERKAT_OK;
}

meerkat_status meerkat_tc_incremental(meerkat_graph* g_after, meerkat_graph* g_update, const uint32_t* src,
                                      const uint32_t* dst, uint64_t n, uint64_t* added, uint64_t* s) {
  return tc_delta(g_after, g_update, src, dst, n, true, added, s);
}

meerkat_status meerkat_tc_decremental(meerkat_graph* g_after, meerkat_graph* g_update, const uint32_t* src,
                                      const uint32_t* dst, uint64_t n, uint64_t* removed, uint64_t* s) {
  return tc_delta(g_after, g_update, src, dst, n, false, removed, s);
}

/* ------------------------------------------------------------------ weakly connected components (wcc.cu) */

meerkat_status meerkat_wcc_create(meerkat_graph* g, meerkat_wcc** out) {
  if (!g || !out) return MEERKAT_E_INVALID_ARG;
  *out = nullptr;
  if (g->part) return MEERKAT_E_STATE;
  DeviceGuard dg(g->device);
  meerkat_wcc* c = new (std::nothrow) meerkat_wcc();
  if (!c) return MEERKAT_E_CUDA;
  c->g = g;
  cudaError_t e = cudaMalloc(&c->parent, (size_t)g->V * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->scratch, 16);
  if (e == cudaSuccess) e = cudaMallocHost(&c->hscratch, 16);
  if (e == cudaSuccess) e = cudaMemsetAsync(c->scratch, 0, 16, g->stream);
  if (e == cudaSuccess) e = launch_wcc_static(g, c->parent, c->scratch);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) { cudaGetLastError(); meerkat_wcc_destroy(c); return MEERKAT_E_CUDA; }
  c->version = g->version;
  *out = c;
  return MEERKAT_OK;
}

meerkat_status meerkat_wcc_recompute(meerkat_graph* g, meerkat_wcc* c) {
  if (!g || !c || c->g != g) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(g->device);
  cudaError_t e = launch_wcc_static(g, c->parent, c->scratch);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  c->version = g->version;
  return MEERKAT_OK;
}

meerkat_status meerkat_wcc_incremental(meerkat_graph* g, meerkat_wcc* c, const uint32_t* src, const uint32_t* dst,
                                       uint64_t n) {
  meerkat_status st = check_batch(g, src, dst, n);
  if (st != MEERKAT_OK) return st;
  if (!c || c->g != g) return MEERKAT_E_INVALID_ARG;
  // the labels must be current up to the insert batch just applied (there is no decremental WCC)
  if (g->last_kind != 1 || c->version + 1 != g->version || n != g->last_n) return MEERKAT_E_STATE;
  DeviceGuard dg(g->device);
  const void *s, *d;
  cudaError_t e = stage_in_reuse(g, 0, src, n * 4, &s);
  if (e == cudaSuccess) e = stage_in_reuse(g, 1, dst, n * 4, &d);
  if (e == cudaSuccess) e = launch_wcc_batch(g, c->parent, (const uint32_t*)s, (const uint32_t*)d, n);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  c->version = g->version;
  return MEERKAT_OK;
}

meerkat_status meerkat_wcc_incremental_tracked(meerkat_graph* g, meerkat_wcc* c) {
  if (!g || !c || c->g != g) return MEERKAT_E_INVALID_ARG;
  if (!g->out.dev.upd) return MEERKAT_E_STATE;   // the graph keeps no update tracking
  // the tracked cells cover every insert since the labels were computed; a delete since then
  // cannot be undone by unions (there is no decremental WCC): recompute instead
  if (g->last_delete_version > c->version) return MEERKAT_E_STATE;
  DeviceGuard dg(g->device);
  const cudaError_t e = launch_wcc_tracked(g, c->parent);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  c->version = g->version;
  return MEERKAT_OK;
}

meerkat_status meerkat_wcc_labels(meerkat_wcc* c, uint32_t* out) {
  if (!c || !out) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = c->g;
  DeviceGuard dg(g->device);
  cudaError_t e = cudaMemcpyAsync(out, c->parent, (size_t)g->V * 4, cudaMemcpyDefault, g->stream);
  if (e == cudaSuccess && !is_device_ptr(out)) e = cudaStreamSynchronize(g->stream);
  return from_cuda(e);
}

meerkat_status meerkat_wcc_components(meerkat_wcc* c, uint64_t* n_components) {
  if (!c || !n_components) return MEERKAT_E_INVALID_ARG;
  meerkat_graph* g = c->g;
  DeviceGuard dg(g->device);
  cudaError_t e = launch_wcc_roots(g, c->parent, c->scratch + 1);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c->hscratch, c->scratch, 16, cudaMemcpyDeviceToHost, g->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return MEERKAT_E_CUDA;
  *n_components = c->hscratch[1];
  return MEERKAT_OK;
}

meerkat_status meerkat_wcc_destroy(meerkat_wcc* c) {
  if (!c) return MEERKAT_E_INVALID_ARG;
  DeviceGuard dg(c->g->device);
  cudaStreamSynchronize(c->g->stream);
  cudaFree(c->parent);
  cudaFree(c->scratch);
  if (c->hscratch) cudaFreeHost(c->hscratch);
  delete c;
  return MEERKAT_OK;
}

}  // extern "C"
