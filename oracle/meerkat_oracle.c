/*
 * oracle/meerkat_oracle.c — CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (the CUDA
 * library behind include/meerkat.h) never calls it, and the two share no
 * code, headers or constants: status codes and sentinels below are restated
 * from the paper / SURVEY, not included from the product.
 *
 * What it computes is the PLAIN DEFINITION the method reaches:
 *  - the edge store is a set of directed edges (a map (src,dst) -> w when
 *    weighted): P:634-641 InsertEdge/DeleteEdge/SearchEdge; an insert of a
 *    present edge keeps the minimum weight (reading C8), only absent keys are
 *    counted; a delete of an absent edge is a no-op (C11);
 *  - SSSP: for every vertex the lexicographically smallest
 *    <distance, parent> (packing footnote P:28-30, readings C1-C3):
 *      node[SRC] = (0, SRC); reachable v: (dist(v), min{u : (u,v) in E,
 *      dist(u) + w(u,v) = dist(v)}); unreachable: UINT64_MAX.
 *    Computed by textbook binary-heap Dijkstra plus one min-parent pass.
 *  - BFS: the same with hop counts (C18), by FIFO BFS.
 *  - decremental intermediates: the directly
 *    invalidated set, its descendants in the old tree T_G, and the
 *    valid->invalid frontier.
 *
 * Data: one array of edge keys (src << 32 | dst) kept sorted, with a parallel
 * weight array.  A batch is sorted once and merged (set union / difference),
 * which is the same as applying its edges one by one because set membership
 * and min() do not depend on order (C8, C11).
 *
 * Status codes (restated from SURVEY §8(b)): 0 OK, 1 INVALID_ARG,
 * 2 VERTEX_RANGE, 3 WEIGHT, 4 CAPACITY, 5 OVERFLOW, 6 STATE.
 * Invalid edges are skipped and never counted; VERTEX_RANGE takes precedence
 * over WEIGHT when a batch holds both.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

enum { ORC_OK = 0, ORC_E_INVALID_ARG = 1, ORC_E_VERTEX_RANGE = 2, ORC_E_WEIGHT = 3,
       ORC_E_CAPACITY = 4, ORC_E_OVERFLOW = 5, ORC_E_STATE = 6 };

#define ORC_UNREACHED UINT64_MAX          /* (INF, INVALID) packed, C3 */
#define ORC_INF_DIST 0xFFFFFFFFull        /* INF = INVALID = 2^32-1, C3 */
#define ORC_W_LIMIT 0x80000000u           /* weights in [1, 2^31), C6 */

typedef struct {
  uint32_t V;
  int weighted;
  uint64_t m;     /* live edges */
  uint64_t* key;  /* sorted ascending, src << 32 | dst */
  uint32_t* w;    /* weight of key[i] (1 when unweighted) */
} orc_graph;

typedef struct { uint64_t key; uint32_t w; } kw;

static int cmp_kw(const void* a, const void* b) {
  const kw* x = (const kw*)a; const kw* y = (const kw*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->w < y->w ? -1 : (x->w > y->w);
}

orc_graph* orc_create(uint32_t V, int weighted) {
  orc_graph* g = (orc_graph*)calloc(1, sizeof(orc_graph));
  g->V = V; g->weighted = weighted;
  return g;
}

void orc_destroy(orc_graph* g) {
  if (!g) return;
  free(g->key); free(g->w); free(g);
}

uint64_t orc_num_edges(const orc_graph* g) { return g->m; }

/* Validate a batch (SURVEY §8(b) Errors) and return the valid edges sorted by key. */
static kw* valid_sorted(const orc_graph* g, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                        uint64_t n, int check_w, uint64_t* nv, int* status) {
  kw* b = (kw*)malloc((n ? n : 1) * sizeof(kw));
  int range = 0, wbad = 0;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; i++) {
    if (src[i] >= g->V || dst[i] >= g->V) { range = 1; continue; }
    uint32_t wi = 1;
    if (check_w) {
      wi = w[i];
      if (wi == 0 || wi >= ORC_W_LIMIT) { wbad = 1; continue; }
    }
    b[k].key = ((uint64_t)src[i] << 32) | dst[i];
    b[k].w = wi;
    k++;
  }
  qsort(b, k, sizeof(kw), cmp_kw);
  *nv = k;
  *status = range ? ORC_E_VERTEX_RANGE : (wbad ? ORC_E_WEIGHT : ORC_OK);
  return b;
}

/* InsertEdges: set union; present key keeps min weight (C8). */
int orc_insert(orc_graph* g, const uint32_t* src, const uint32_t* dst, const uint32_t* w, uint64_t n,
               uint64_t* n_inserted) {
  if (g->weighted && !w && n) return ORC_E_INVALID_ARG;
  int status; uint64_t nb;
  kw* b = valid_sorted(g, src, dst, w, n, g->weighted, &nb, &status);
  uint64_t* nk = (uint64_t*)malloc((g->m + nb + 1) * sizeof(uint64_t));
  uint32_t* nw = (uint32_t*)malloc((g->m + nb + 1) * sizeof(uint32_t));
  uint64_t i = 0, j = 0, o = 0, added = 0;
  while (i < g->m || j < nb) {
    if (j >= nb || (i < g->m && g->key[i] < b[j].key)) { nk[o] = g->key[i]; nw[o] = g->w[i]; o++; i++; continue; }
    /* b[j] is the smallest-weight copy of its key within the batch (sorted by key, then w) */
    uint64_t k = b[j].key; uint32_t wmin = b[j].w;
    while (j < nb && b[j].key == k) j++;
    if (i < g->m && g->key[i] == k) {
      nk[o] = k; nw[o] = g->w[i] < wmin ? g->w[i] : wmin; o++; i++;
    } else {
      nk[o] = k; nw[o] = wmin; o++; added++;
    }
  }
  free(b);
  free(g->key); free(g->w);
  g->key = nk; g->w = nw; g->m = o;
  if (n_inserted) *n_inserted = added;
  return status;
}

/* DeleteEdges: set difference; absent edges are no-ops (C11). */
int orc_delete(orc_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n, uint64_t* n_deleted) {
  int status; uint64_t nb;
  kw* b = valid_sorted(g, src, dst, NULL, n, 0, &nb, &status);
  uint64_t i = 0, j = 0, o = 0, removed = 0;
  while (i < g->m) {
    while (j < nb && b[j].key < g->key[i]) j++;
    if (j < nb && b[j].key == g->key[i]) { removed++; i++; continue; }
    g->key[o] = g->key[i]; g->w[o] = g->w[i]; o++; i++;
  }
  g->m = o;
  free(b);
  if (n_deleted) *n_deleted = removed;
  return status;
}

static int64_t find(const orc_graph* g, uint64_t k) {
  uint64_t lo = 0, hi = g->m;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (g->key[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < g->m && g->key[lo] == k) ? (int64_t)lo : -1;
}

/* SearchEdge: found flag and stored weight (0 when absent or out of range). */
int orc_query(const orc_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n, uint8_t* found,
              uint32_t* w_out) {
  int status = ORC_OK;
  for (uint64_t i = 0; i < n; i++) {
    found[i] = 0;
    if (w_out) w_out[i] = 0;
    if (src[i] >= g->V || dst[i] >= g->V) { status = ORC_E_VERTEX_RANGE; continue; }
    int64_t p = find(g, ((uint64_t)src[i] << 32) | dst[i]);
    if (p >= 0) { found[i] = 1; if (w_out) w_out[i] = g->weighted ? g->w[p] : 0; }
  }
  return status;
}

/* Sorted edge dump (src, dst, w). */
void orc_export(const orc_graph* g, uint32_t* src, uint32_t* dst, uint32_t* w) {
  for (uint64_t i = 0; i < g->m; i++) {
    src[i] = (uint32_t)(g->key[i] >> 32);
    dst[i] = (uint32_t)g->key[i];
    if (w) w[i] = g->w[i];
  }
}

/* CSR row offsets of the sorted key array: edges of u are [off[u], off[u+1]). */
static uint64_t* row_offsets(const orc_graph* g) {
  uint64_t* off = (uint64_t*)calloc((size_t)g->V + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < g->m; i++) off[(g->key[i] >> 32) + 1]++;
  for (uint32_t v = 0; v < g->V; v++) off[v + 1] += off[v];
  return off;
}

/* ---------------- binary heap of (dist, vertex) with lazy deletion ---------------- */
typedef struct { uint64_t d; uint32_t v; } hent;
typedef struct { hent* a; uint64_t n, cap; } heap;

static void hpush(heap* h, uint64_t d, uint32_t v) {
  if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 1024; h->a = (hent*)realloc(h->a, h->cap * sizeof(hent)); }
  uint64_t i = h->n++;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (h->a[p].d <= d) break;
    h->a[i] = h->a[p]; i = p;
  }
  h->a[i].d = d; h->a[i].v = v;
}

static hent hpop(heap* h) {
  hent top = h->a[0], last = h->a[--h->n];
  uint64_t i = 0;
  for (;;) {
    uint64_t c = 2 * i + 1;
    if (c >= h->n) break;
    if (c + 1 < h->n && h->a[c + 1].d < h->a[c].d) c++;
    if (h->a[c].d >= last.d) break;
    h->a[i] = h->a[c]; i = c;
  }
  if (h->n) h->a[i] = last;
  return top;
}

/* Pack distances and the min tight parent (C1-C3): node[v] = dist << 32 | parent. */
static int pack_min_parent(const orc_graph* g, uint32_t SRC, int unit, const uint64_t* dist, uint64_t* node) {
  uint32_t* par = (uint32_t*)malloc((size_t)g->V * sizeof(uint32_t));
  for (uint32_t v = 0; v < g->V; v++) par[v] = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < g->m; i++) {
    uint32_t u = (uint32_t)(g->key[i] >> 32), v = (uint32_t)g->key[i];
    uint64_t w = unit ? 1 : g->w[i];
    if (dist[u] != UINT64_MAX && dist[u] + w == dist[v] && u < par[v]) par[v] = u;
  }
  par[SRC] = SRC;
  int status = ORC_OK;
  for (uint32_t v = 0; v < g->V; v++) {
    if (dist[v] == UINT64_MAX) { node[v] = ORC_UNREACHED; continue; }
    if (dist[v] >= ORC_INF_DIST) { status = ORC_E_OVERFLOW; node[v] = ORC_UNREACHED; continue; } /* C5 */
    node[v] = (dist[v] << 32) | par[v];
  }
  free(par);
  return status;
}

/* Static SSSP (P:88-112 computes it by frontier iteration; the definition is
 * the shortest-path distance): binary-heap Dijkstra, then min-parent pass.
 * unit != 0 uses w = 1 for every edge.  Requires a weighted graph unless unit. */
int orc_sssp(const orc_graph* g, uint32_t SRC, int unit, uint64_t* node) {
  if (SRC >= g->V) return ORC_E_VERTEX_RANGE;
  if (!g->weighted && !unit) return ORC_E_STATE;
  uint64_t* off = row_offsets(g);
  uint64_t* dist = (uint64_t*)malloc((size_t)g->V * sizeof(uint64_t));
  uint8_t* done = (uint8_t*)calloc(g->V, 1);
  for (uint32_t v = 0; v < g->V; v++) dist[v] = UINT64_MAX;
  heap h = {0, 0, 0};
  dist[SRC] = 0;
  hpush(&h, 0, SRC);
  while (h.n) {
    hent e = hpop(&h);
    if (done[e.v]) continue;
    done[e.v] = 1;
    for (uint64_t i = off[e.v]; i < off[e.v + 1]; i++) {
      uint32_t x = (uint32_t)g->key[i];
      uint64_t nd = e.d + (unit ? 1 : g->w[i]);
      if (nd < dist[x]) { dist[x] = nd; hpush(&h, nd, x); }
    }
  }
  int st = pack_min_parent(g, SRC, unit, dist, node);
  free(h.a); free(done); free(dist); free(off);
  return st;
}

/* Static BFS (C18): FIFO level order on hop counts, then min parent at level-1. */
int orc_bfs(const orc_graph* g, uint32_t SRC, uint64_t* node) {
  if (SRC >= g->V) return ORC_E_VERTEX_RANGE;
  uint64_t* off = row_offsets(g);
  uint64_t* level = (uint64_t*)malloc((size_t)g->V * sizeof(uint64_t));
  uint32_t* q = (uint32_t*)malloc((size_t)g->V * sizeof(uint32_t));
  for (uint32_t v = 0; v < g->V; v++) level[v] = UINT64_MAX;
  uint64_t head = 0, tail = 0;
  level[SRC] = 0; q[tail++] = SRC;
  while (head < tail) {
    uint32_t u = q[head++];
    for (uint64_t i = off[u]; i < off[u + 1]; i++) {
      uint32_t x = (uint32_t)g->key[i];
      if (level[x] == UINT64_MAX) { level[x] = level[u] + 1; q[tail++] = x; }
    }
  }
  int st = pack_min_parent(g, SRC, 1, level, node);
  free(q); free(level); free(off);
  return st;
}

/*
 * Decremental intermediates (P:144-147 Invalidate; P:149-154
 * PropagateInvalidation; P:156-164 valid->invalid frontier; readings C4, C14, C15).
 * Inputs: the OLD tree node_old[V] and the deleted batch.
 *  direct   = { v != SRC : node_old[v] reached, (parent_old(v), v) in batch }
 *  invalid  = direct plus all its descendants in the old tree T_G
 * Outputs: invalid_flag[v] in {0,1}; returns |invalid|; *n_direct = |direct|.
 */
uint64_t orc_invalidated(uint32_t V, uint32_t SRC, const uint64_t* node_old, const uint32_t* src,
                         const uint32_t* dst, uint64_t n, uint8_t* invalid_flag, uint64_t* n_direct) {
  memset(invalid_flag, 0, V);
  uint32_t* q = (uint32_t*)malloc(((size_t)V + 1) * sizeof(uint32_t));
  uint64_t tail = 0, nd = 0;
  for (uint64_t i = 0; i < n; i++) {
    uint32_t u = src[i], v = dst[i];
    if (u >= V || v >= V || v == SRC) continue;
    if (node_old[v] == ORC_UNREACHED) continue;
    if ((uint32_t)node_old[v] == u && !invalid_flag[v]) { invalid_flag[v] = 1; q[tail++] = v; nd++; }
  }
  /* children lists of the old tree */
  uint64_t* coff = (uint64_t*)calloc((size_t)V + 1, sizeof(uint64_t));
  for (uint32_t v = 0; v < V; v++)
    if (v != SRC && node_old[v] != ORC_UNREACHED) coff[(uint32_t)node_old[v] + 1]++;
  for (uint32_t v = 0; v < V; v++) coff[v + 1] += coff[v];
  uint32_t* child = (uint32_t*)malloc((coff[V] + 1) * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)malloc(((size_t)V + 1) * sizeof(uint64_t));
  memcpy(fill, coff, ((size_t)V + 1) * sizeof(uint64_t));
  for (uint32_t v = 0; v < V; v++)
    if (v != SRC && node_old[v] != ORC_UNREACHED) child[fill[(uint32_t)node_old[v]]++] = v;
  for (uint64_t head = 0; head < tail; head++) {
    uint32_t p = q[head];
    for (uint64_t i = coff[p]; i < coff[p + 1]; i++) {
      uint32_t c = child[i];
      if (!invalid_flag[c]) { invalid_flag[c] = 1; q[tail++] = c; }
    }
  }
  free(child); free(fill); free(coff); free(q);
  if (n_direct) *n_direct = nd;
  return tail;
}

/* Valid->invalid frontier size (C15): edges (u,x) of the CURRENT graph
 * with u reached in the old tree, u not invalid, x invalid. */
uint64_t orc_dec_frontier_count(const orc_graph* g, const uint64_t* node_old, const uint8_t* invalid_flag) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < g->m; i++) {
    uint32_t u = (uint32_t)(g->key[i] >> 32), x = (uint32_t)g->key[i];
    if (node_old[u] != ORC_UNREACHED && !invalid_flag[u] && invalid_flag[x]) c++;
  }
  return c;
}

/*
 * Certificate check of a claimed tree against this graph, valid at any size
 * (used where a full recompute would be too slow).  With every w >= 1 (C6) the
 * Bellman equations  node[SRC] = (0,SRC),  node[v] = min over in-edges (u,v)
 * with node[u] reached of ((d(u)+w) << 32 | u),  node[v] = UINT64_MAX when no
 * such edge exists, have exactly one solution, the definition above; a vertex
 * whose value differs is counted.  Returns the number of mismatching vertices
 * and the first one in *first_bad (UINT32_MAX if none).
 */
uint64_t orc_check_tree(const orc_graph* g, uint32_t SRC, int unit, const uint64_t* node, uint32_t* first_bad) {
  uint64_t* best = (uint64_t*)malloc((size_t)g->V * sizeof(uint64_t));
  for (uint32_t v = 0; v < g->V; v++) best[v] = ORC_UNREACHED;
  for (uint64_t i = 0; i < g->m; i++) {
    uint32_t u = (uint32_t)(g->key[i] >> 32), v = (uint32_t)g->key[i];
    if (node[u] == ORC_UNREACHED) continue;
    uint64_t d = (node[u] >> 32) + (unit ? 1 : g->w[i]);
    if (d >= ORC_INF_DIST) continue;
    uint64_t cand = (d << 32) | u;
    if (cand < best[v]) best[v] = cand;
  }
  best[SRC] = (uint64_t)SRC;
  uint64_t bad = 0;
  uint32_t fb = 0xFFFFFFFFu;
  for (uint32_t v = 0; v < g->V; v++)
    if (best[v] != node[v]) { if (!bad) fb = v; bad++; }
  free(best);
  if (first_bad) *first_bad = fb;
  return bad;
}

/*
 * PageRank, static and dynamic ("Dynamic PageRank",
 * Eq. (1) contribution-change P:834-836, Algorithm pr-all as narrated P:852-880;
 * d = 0.85 and error margin 0.00001 are the paper's experimental values P:1559-1560).
 * Double precision throughout (the paper states none; BASELINE.json asks 1e-6 relative L1).
 *
 * pr[] (in/out, length V) holds the starting vector: 1/vertex_n for every vertex in the
 * static case, the values computed before the batch in the incremental /
 * decremental case ("the same static-PageRank algorithm is applied on
 * the entire graph after performing insertion/deletion").  One super-step i, in the paper's order:
 *   FindContributionPerVertex: Contribution[u] = PR_{i-1}[u] / out[u] for out[u] > 0;
 *   Compute (Eq. 1): PR_i[v] = (1-d)/N + d * sum over in-edges u->v of
 *     Contribution[u];
 *   FindTeleportProb (reading C27: the sum is scaled by d): if some vertex v_z has
 *     out-degree 0, every PR_i[v] += d * (sum over such v_z of PR_{i-1}[v_z]) / N;
 *   delta = sum_v |PR_i[v] - PR_{i-1}[v]| (the L1 norm).
 * Super-steps repeat while delta > eps and fewer than max_iter have run (at least
 * one).  Out-degrees count stored edges (self-loops included, C12).
 * Returns ORC_E_INVALID_ARG for d not in (0,1), eps <= 0 or max_iter == 0 (SPEC BadDamping /
 * BadEpsilon); *iters = super-steps run, *delta_out = the last delta.
 */
int orc_pagerank(const orc_graph* g, double d, double eps, uint32_t max_iter, double* pr, uint32_t* iters,
                 double* delta_out) {
  if (!(d > 0.0 && d < 1.0) || !(eps > 0.0) || max_iter == 0) return ORC_E_INVALID_ARG;
  const uint32_t N = g->V;
  uint32_t* out = (uint32_t*)calloc((size_t)N + 1, sizeof(uint32_t));
  for (uint64_t i = 0; i < g->m; i++) out[g->key[i] >> 32]++;
  int has_zero = 0;
  for (uint32_t v = 0; v < N; v++) if (out[v] == 0) has_zero = 1;
  double* contribution = (double*)malloc(((size_t)N + 1) * sizeof(double));
  double* next = (double*)malloc(((size_t)N + 1) * sizeof(double));
  uint32_t it = 0;
  double delta = 0.0;
  do {
    /* FindContributionPerVertex */
    for (uint32_t u = 0; u < N; u++) contribution[u] = out[u] ? pr[u] / (double)out[u] : 0.0;
    /* Compute: (1-d)/N + d * sum over in-edges */
    double* sum = next;
    for (uint32_t v = 0; v < N; v++) sum[v] = 0.0;
    for (uint64_t i = 0; i < g->m; i++) sum[(uint32_t)g->key[i]] += contribution[g->key[i] >> 32];
    for (uint32_t v = 0; v < N; v++) next[v] = (1.0 - d) / (double)N + d * sum[v];
    /* FindTeleportProb, added to every vertex */
    if (has_zero) {
      double z = 0.0;
      for (uint32_t v = 0; v < N; v++) if (out[v] == 0) z += pr[v];
      const double teleport = d * z / (double)N;
      for (uint32_t v = 0; v < N; v++) next[v] += teleport;
    }
    /* L1 norm between PR_i and PR_{i-1} */
    delta = 0.0;
    for (uint32_t v = 0; v < N; v++) delta += fabs(next[v] - pr[v]);
    memcpy(pr, next, (size_t)N * sizeof(double));
    it++;
  } while (delta > eps && it < max_iter);
  free(next); free(contribution); free(out);
  if (iters) *iters = it;
  if (delta_out) *delta_out = delta;
  return ORC_OK;
}

/*
 * Dynamic triangle counting ("Dynamic Triangle Counting",
 * P:1643-1656; the Count kernel of Algorithm tc-count).
 *   Count(G1, G2, edges) = sum over (u, v) in edges of |adjacency_G1(u) ∩ adjacency_G2(v)|
 * ("the cardinality of the intersection of the adjacency(u) in G1 and adjacency(v)
 * in G2").  Adjacencies are the stored out-neighbour sets (graphs are undirected, i.e. store both
 * orientations, for triangle counting).  Plain definition: a merge of the two sorted rows.
 */
static uint64_t row_begin(const orc_graph* g, uint32_t u) {
  uint64_t lo = 0, hi = g->m, k = (uint64_t)u << 32;
  while (lo < hi) { uint64_t mid = lo + (hi - lo) / 2; if (g->key[mid] < k) lo = mid + 1; else hi = mid; }
  return lo;
}

uint64_t orc_tc_count(const orc_graph* g1, const orc_graph* g2, const uint32_t* src, const uint32_t* dst,
                      uint64_t n) {
  uint64_t total = 0;
  for (uint64_t e = 0; e < n; e++) {
    const uint32_t u = src[e], v = dst[e];
    if (u >= g1->V || v >= g2->V) continue;
    uint64_t i = row_begin(g1, u), j = row_begin(g2, v);
    while (i < g1->m && (g1->key[i] >> 32) == u && j < g2->m && (g2->key[j] >> 32) == v) {
      const uint32_t a = (uint32_t)g1->key[i], b = (uint32_t)g2->key[j];
      if (a == b) { total++; i++; j++; }
      else if (a < b) i++;
      else j++;
    }
  }
  return total;
}

/*
 * Weakly connected components ("Incremental WCC", supplementary
 * P:381-395 static SamplingWCC).  A WCC of a directed graph is a maximal set of vertices connected
 * when edge directions are ignored.  Labels are canonical: label[v] = the smallest
 * vertex id in v's component (what a union-find that always hooks the larger root under the
 * smaller one ends with after full path compression).  Plain definition: BFS over the
 * undirected version of the edge set, vertices visited in increasing id order.
 */
uint64_t orc_wcc(const orc_graph* g, uint32_t* label) {
  const uint32_t V = g->V;
  /* undirected adjacency: CSR over both orientations */
  uint64_t* off = (uint64_t*)calloc((size_t)V + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < g->m; i++) { off[(g->key[i] >> 32) + 1]++; off[(uint32_t)g->key[i] + 1]++; }
  for (uint32_t v = 0; v < V; v++) off[v + 1] += off[v];
  uint32_t* adj = (uint32_t*)malloc((off[V] + 1) * sizeof(uint32_t));
  uint64_t* fill = (uint64_t*)malloc(((size_t)V + 1) * sizeof(uint64_t));
  memcpy(fill, off, ((size_t)V + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < g->m; i++) {
    const uint32_t u = (uint32_t)(g->key[i] >> 32), v = (uint32_t)g->key[i];
    adj[fill[u]++] = v;
    adj[fill[v]++] = u;
  }
  uint32_t* q = (uint32_t*)malloc(((size_t)V + 1) * sizeof(uint32_t));
  for (uint32_t v = 0; v < V; v++) label[v] = 0xFFFFFFFFu;
  uint64_t comps = 0;
  for (uint32_t r = 0; r < V; r++) {   /* r is the smallest id of a not yet labelled component */
    if (label[r] != 0xFFFFFFFFu) continue;
    comps++;
    uint64_t head = 0, tail = 0;
    label[r] = r; q[tail++] = r;
    while (head < tail) {
      const uint32_t x = q[head++];
      for (uint64_t i = off[x]; i < off[x + 1]; i++)
        if (label[adj[i]] == 0xFFFFFFFFu) { label[adj[i]] = r; q[tail++] = adj[i]; }
    }
  }
  free(q); free(fill); free(adj); free(off);
  return comps;
}
