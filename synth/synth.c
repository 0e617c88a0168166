/*
 * synth/synth.c — seeded synthetic input generators (plumbing, not the method).
 *
 * This module is shared by the CPU oracle side (tests, bench cpu_baseline) and
 * the CUDA side (bench, GPU tests) as the ONE common input source.  It holds
 * none of the method's arithmetic: no slab layout, no hashing into buckets, no
 * min-weight upsert, no shortest-path logic.  Duplicate (src,dst) draws are
 * removed by keeping the FIRST draw (lowest draw index), a generator choice
 * independent of the store's min-weight rule.
 *
 * Recipe (SURVEY §8(d) "Generator specification"):
 *  - counter-based RNG: splitmix64(seed ^ (stream << 56) ^ counter), so every
 *    draw is independent of thread count and order;
 *  - R-MAT / Kronecker, Graph500 initiator (a,b,c,d) = (0.57,0.19,0.19,0.05),
 *    one uniform per bit level, no per-level noise;
 *  - vertex ids scrambled by a bijective xorshift-multiply mixer on `scale`
 *    bits (an affine map would keep R-MAT's low-bit skew);
 *  - weights w = 1 + (splitmix64(...) mod 64)  (S:595 uses U[1,64]);
 *  - self-loops dropped (C12), duplicates dropped keeping the first draw.
 *
 * Build: gcc -O3 -fopenmp -shared -fPIC synth.c -o libsynth.so
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return splitmix64(splitmix64(seed) ^ (stream << 56) ^ ctr);
}

/* uniform double in [0,1) from the top 53 bits */
static inline double unif(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }


/* R-MAT draw i: one uniform per bit level picks a quadrant (a | b | c | d), MSB first. */
static inline void rmat_edge(uint32_t scale, double a, double ab, double abc, uint64_t seed,
                             uint64_t i, uint32_t* pu, uint32_t* pv) {
  uint32_t u = 0, v = 0;
  for (uint32_t l = 0; l < scale; l++) {
    double r = unif(draw(seed, 1, i * 64 + l));
    uint32_t sb = r >= ab;                       /* quadrants c, d: src bit 1 */
    uint32_t db = (r >= a && r < ab) || r >= abc; /* quadrants b, d: dst bit 1 */
    u = (u << 1) | sb;
    v = (v << 1) | db;
  }
  *pu = u; *pv = v;
}

uint64_t synth_draw(uint64_t seed, uint64_t stream, uint64_t ctr) { return draw(seed, stream, ctr); }

/* Bijective mixer on `bits` bits: x^=x>>h; x=(x*M1)&mask; x^=x>>h; x=(x*M2)&mask; x^=x>>h */
uint32_t synth_scramble(uint32_t v, uint32_t bits, uint64_t seed) {
  if (bits == 0) return v;
  uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  uint32_t h = (bits + 1) / 2;
  uint64_t m1 = draw(seed, 7, 1) | 1ull, m2 = draw(seed, 7, 2) | 1ull;
  uint64_t x = v & mask;
  x ^= x >> h; x = (x * m1) & mask;
  x ^= x >> h; x = (x * m2) & mask;
  x ^= x >> h;
  return (uint32_t)x;
}

/* ---------------- parallel stable LSD radix sort of (key, payload) ---------------- */
static void radix_sort_kv(uint64_t* key, uint32_t* val, uint64_t n, int key_bits) {
  if (n < 2) return;
  const int RB = 11, R = 1 << RB;
  uint64_t* k2 = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint32_t* v2 = (uint32_t*)malloc(n * sizeof(uint32_t));
  int nth = 1;
#ifdef _OPENMP
  nth = omp_get_max_threads();
#endif
  uint64_t* hist = (uint64_t*)malloc((size_t)nth * R * sizeof(uint64_t));
  for (int shift = 0; shift < key_bits; shift += RB) {
    memset(hist, 0, (size_t)nth * R * sizeof(uint64_t));
#pragma omp parallel num_threads(nth)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      uint64_t lo = n * t / nth, hi = n * (t + 1) / nth;
      uint64_t* h = hist + (size_t)t * R;
      for (uint64_t i = lo; i < hi; i++) h[(key[i] >> shift) & (R - 1)]++;
#pragma omp barrier
#pragma omp single
      {
        uint64_t run = 0;
        for (int d = 0; d < R; d++)
          for (int tt = 0; tt < nth; tt++) {
            uint64_t c = hist[(size_t)tt * R + d];
            hist[(size_t)tt * R + d] = run;
            run += c;
          }
      }
      for (uint64_t i = lo; i < hi; i++) {
        uint64_t p = h[(key[i] >> shift) & (R - 1)]++;
        k2[p] = key[i];
        v2[p] = val[i];
      }
    }
    memcpy(key, k2, n * sizeof(uint64_t));
    memcpy(val, v2, n * sizeof(uint32_t));
  }
  free(k2); free(v2); free(hist);
}

/*
 * R-MAT graph: 2^scale vertices, ef * 2^scale draws.  Writes the unique edges
 * (self-loops dropped, first draw kept) sorted by (src, dst) into the caller's
 * arrays (capacity ef * 2^scale each); returns the unique edge count.
 * a,b,c: initiator probabilities (d = 1-a-b-c).  Ids are scrambled iff scramble.
 */
uint64_t synth_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                    uint64_t seed_graph, uint64_t seed_w, int scramble,
                    uint32_t* out_src, uint32_t* out_dst, uint32_t* out_w) {
  uint64_t n = (uint64_t)ef << scale;
  uint64_t* key = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint32_t* idx = (uint32_t*)malloc(n * sizeof(uint32_t));
  const double ab = a + b, abc = a + b + c;
  /* draw; key = src << scale | dst, payload = draw index */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; i++) {
    uint32_t u = 0, v = 0;
    rmat_edge(scale, a, ab, abc, seed_graph, (uint64_t)i, &u, &v);
    if (scramble) { u = synth_scramble(u, scale, seed_graph); v = synth_scramble(v, scale, seed_graph); }
    key[i] = ((uint64_t)u << scale) | v;
    idx[i] = (uint32_t)i;
  }
  radix_sort_kv(key, idx, n, 2 * (int)scale);
  uint64_t m = 0;
  const uint64_t vmask = (1ull << scale) - 1;
  for (uint64_t i = 0; i < n; i++) {
    if (i > 0 && key[i] == key[i - 1]) continue; /* stable sort: first draw kept */
    uint32_t u = (uint32_t)(key[i] >> scale), v = (uint32_t)(key[i] & vmask);
    if (u == v) continue;
    out_src[m] = u;
    out_dst[m] = v;
    out_w[m] = 1 + (uint32_t)(draw(seed_w, 2, idx[i]) % 64);
    m++;
  }
  free(key); free(idx);
  return m;
}

/* Uniform random directed graph G(n, m): first m distinct non-loop draws, in draw order. */
uint64_t synth_uniform(uint32_t n, uint64_t m, uint64_t seed_graph, uint64_t seed_w,
                       uint32_t* out_src, uint32_t* out_dst, uint32_t* out_w) {
  if (n < 2) return 0;
  uint64_t maxm = (uint64_t)n * (n - 1);
  if (m > maxm) m = maxm;
  uint64_t cap = 1; while (cap < 2 * m + 16) cap <<= 1;
  uint64_t* table = (uint64_t*)malloc(cap * sizeof(uint64_t));
  memset(table, 0xFF, cap * sizeof(uint64_t));
  uint64_t got = 0;
  for (uint64_t i = 0; got < m; i++) {
    uint64_t r = draw(seed_graph, 3, i);
    uint32_t u = (uint32_t)((r & 0xFFFFFFFFull) % n), v = (uint32_t)((r >> 32) % n);
    if (u == v) continue;
    uint64_t k = ((uint64_t)u << 32) | v;
    uint64_t h = splitmix64(k) & (cap - 1);
    int dup = 0;
    while (table[h] != ~0ull) { if (table[h] == k) { dup = 1; break; } h = (h + 1) & (cap - 1); }
    if (dup) continue;
    table[h] = k;
    out_src[got] = u; out_dst[got] = v;
    out_w[got] = 1 + (uint32_t)(draw(seed_w, 2, got) % 64);
    got++;
  }
  free(table);
  return got;
}

/* k distinct indices in [0, m), in seeded draw order (rejection on a bitmap). */
int synth_sample_distinct(uint64_t m, uint64_t k, uint64_t seed, uint64_t* out) {
  if (k > m) return 1;
  uint64_t words = (m + 63) / 64;
  uint64_t* bits = (uint64_t*)calloc(words, sizeof(uint64_t));
  if (!bits) return 2;
  if (2 * k > m) {
    /* dense: partial Fisher-Yates over an explicit index array */
    uint64_t* p = (uint64_t*)malloc(m * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; i++) p[i] = i;
    for (uint64_t i = 0; i < k; i++) {
      uint64_t j = i + draw(seed, 4, i) % (m - i);
      uint64_t t = p[i]; p[i] = p[j]; p[j] = t;
      out[i] = p[i];
    }
    free(p);
  } else {
    uint64_t got = 0;
    for (uint64_t i = 0; got < k; i++) {
      uint64_t j = draw(seed, 4, i) % m;
      if (bits[j >> 6] & (1ull << (j & 63))) continue;
      bits[j >> 6] |= 1ull << (j & 63);
      out[got++] = j;
    }
  }
  free(bits);
  return 0;
}

/* Fresh R-MAT draws (not deduplicated against anything): for config-2 insert sweeps.  The draws
 * come from seed_graph's stream; ids are scrambled with seed_scramble (pass the base graph's seed
 * so the fresh edges follow the base graph's vertex labelling: its hubs are their hubs). */
void synth_rmat_draws(uint32_t scale, uint64_t n, double a, double b, double c, uint64_t seed_graph,
                      uint64_t seed_w, int scramble, uint64_t seed_scramble, uint64_t first,
                      uint32_t* out_src, uint32_t* out_dst, uint32_t* out_w) {
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < (int64_t)n; i++) {
    uint64_t gi = first + (uint64_t)i;
    uint32_t u = 0, v = 0;
    rmat_edge(scale, a, ab, abc, seed_graph, gi, &u, &v);
    if (scramble) { u = synth_scramble(u, scale, seed_scramble); v = synth_scramble(v, scale, seed_scramble); }
    out_src[i] = u; out_dst[i] = v;
    out_w[i] = 1 + (uint32_t)(draw(seed_w, 2, gi) % 64);
  }
}
