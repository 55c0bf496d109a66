/*
 * graphgen/gen.c — seeded synthetic graph generators (inputs only).
 *
 * This module holds NO arithmetic of the Atos method (arxiv 2112.00132).  It
 * produces CSR graphs shaped like the paper's workloads (tbl:dataset, PAPER.md
 * P:740-757): scale-free RMAT/Kronecker graphs (soc-LiveJournal1-like) and
 * high-diameter 2-D grids / road-like meshes (road_usa-like).  Both the CUDA
 * path and the oracle consume its output; neither is imported here.
 *
 * Determinism: every random draw is a pure function of (seed, index) through
 * splitmix64, so results do not depend on the OpenMP thread count.  Rows are
 * sorted and de-duplicated, self-loops are dropped (SPEC.md S:126 design
 * decision: simple directed graphs).
 *
 * Layout of every produced graph: int64 row_offsets[n+1], int32 col[m].
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

typedef struct {
  int64_t n, m;
  int64_t* off;
  int32_t* col;
} gg_graph;

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t hash2(uint64_t seed, uint64_t i) {
  return splitmix64(splitmix64(seed ^ 0x5851F42D4C957F2Dull) ^ i);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* Build a CSR from a directed edge list (src[i] -> dst[i]).  Drops self-loops
 * (unless keep_loops), sorts each row, removes duplicates.  Consumes nothing;
 * returns a freshly allocated graph or NULL on allocation failure. */
static gg_graph* build_csr(int64_t n, int64_t ne, const uint32_t* src, const uint32_t* dst,
                           int symmetrize) {
  gg_graph* g = (gg_graph*)calloc(1, sizeof(gg_graph));
  if (!g) return NULL;
  g->n = n;
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) { free(g); return NULL; }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < ne; i++) {
    uint32_t u = src[i], v = dst[i];
    if (u == v) continue;
#pragma omp atomic
    cnt[u + 1]++;
    if (symmetrize) {
#pragma omp atomic
      cnt[v + 1]++;
    }
  }
  for (int64_t v = 0; v < n; v++) cnt[v + 1] += cnt[v];
  int64_t total = cnt[n];
  int32_t* tmp = (int32_t*)malloc((size_t)(total > 0 ? total : 1) * sizeof(int32_t));
  int64_t* pos = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!tmp || !pos) { free(cnt); free(tmp); free(pos); free(g); return NULL; }
  memcpy(pos, cnt, ((size_t)n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < ne; i++) {
    uint32_t u = src[i], v = dst[i];
    if (u == v) continue;
    int64_t p;
#pragma omp atomic capture
    p = pos[u]++;
    tmp[p] = (int32_t)v;
    if (symmetrize) {
#pragma omp atomic capture
      p = pos[v]++;
      tmp[p] = (int32_t)u;
    }
  }
  free(pos);
  /* sort + dedup each row in place; record unique counts */
  int64_t* uniq = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!uniq) { free(cnt); free(tmp); free(g); return NULL; }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; v++) {
    int64_t b = cnt[v], e = cnt[v + 1];
    if (e - b > 1) qsort(tmp + b, (size_t)(e - b), sizeof(int32_t), cmp_i32);
    int64_t k = 0;
    for (int64_t i = b; i < e; i++)
      if (k == 0 || tmp[b + k - 1] != tmp[i]) tmp[b + k++] = tmp[i];
    uniq[v + 1] = k;
  }
  for (int64_t v = 0; v < n; v++) uniq[v + 1] += uniq[v];
  g->m = uniq[n];
  g->off = uniq;
  g->col = (int32_t*)malloc((size_t)(g->m > 0 ? g->m : 1) * sizeof(int32_t));
  if (!g->col) { free(cnt); free(tmp); free(uniq); free(g); return NULL; }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; v++)
    memcpy(g->col + uniq[v], tmp + cnt[v], (size_t)(uniq[v + 1] - uniq[v]) * sizeof(int32_t));
  free(cnt);
  free(tmp);
  return g;
}

/* ---- public API (ctypes) ---------------------------------------------- */

int64_t gg_n(const gg_graph* g) { return g ? g->n : -1; }
int64_t gg_m(const gg_graph* g) { return g ? g->m : -1; }
void gg_copy(const gg_graph* g, int64_t* off, int32_t* col) {
  memcpy(off, g->off, ((size_t)g->n + 1) * sizeof(int64_t));
  if (g->m) memcpy(col, g->col, (size_t)g->m * sizeof(int32_t));
}
void gg_free(gg_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->col);
  free(g);
}
void gg_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }

/* 2-D lattice, 4-neighbourhood, both directions, row-major ids v = i*cols + j
 * (SPEC.md S:65-73 gen_grid).  drop_prob > 0 deletes each undirected edge
 * independently with that probability (seeded) — the "road-like" variant
 * (avg degree ≈ 2.4 like road_usa). */
gg_graph* gg_grid(int64_t rows, int64_t cols, double drop_prob, uint64_t seed) {
  if (rows < 0 || cols < 0) return NULL;
  int64_t n = rows * cols;
  if (n >= 2147483647LL) return NULL;
  gg_graph* g = (gg_graph*)calloc(1, sizeof(gg_graph));
  if (!g) return NULL;
  g->n = n;
  g->off = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
  if (!g->off) { free(g); return NULL; }
  const uint64_t thr = drop_prob <= 0 ? 0 : (drop_prob >= 1 ? UINT64_MAX : (uint64_t)(drop_prob * 18446744073709551616.0));
  /* an undirected edge {a<b} is kept iff hash(seed, a*2 + dir) >= thr, dir 0 = right, 1 = down */
#define KEEP(a, dir) (thr == 0 || hash2(seed, (uint64_t)(a) * 2u + (dir)) >= thr)
  g->off[0] = 0;
  /* degrees */
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int64_t i = v / cols, j = v % cols, d = 0;
    if (i > 0 && KEEP(v - cols, 1)) d++;
    if (j > 0 && KEEP(v - 1, 0)) d++;
    if (j + 1 < cols && KEEP(v, 0)) d++;
    if (i + 1 < rows && KEEP(v, 1)) d++;
    g->off[v + 1] = d;
  }
  for (int64_t v = 0; v < n; v++) g->off[v + 1] += g->off[v];
  g->m = g->off[n];
  g->col = (int32_t*)malloc((size_t)(g->m > 0 ? g->m : 1) * sizeof(int32_t));
  if (!g->col) { free(g->off); free(g); return NULL; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; v++) {
    int64_t i = v / cols, j = v % cols, p = g->off[v];
    if (i > 0 && KEEP(v - cols, 1)) g->col[p++] = (int32_t)(v - cols);
    if (j > 0 && KEEP(v - 1, 0)) g->col[p++] = (int32_t)(v - 1);
    if (j + 1 < cols && KEEP(v, 0)) g->col[p++] = (int32_t)(v + 1);
    if (i + 1 < rows && KEEP(v, 1)) g->col[p++] = (int32_t)(v + cols);
  }
#undef KEEP
  return g;
}

/* RMAT / Kronecker generator (Graph500 partition probabilities a,b,c,d; SPEC
 * S:75-83).  2^scale vertices, edge_factor * 2^scale generated directed tuples.
 * Tuple t, level l draws a 16-bit uniform from field (l % 4) of
 * hash2(seed, t * ceil(scale/4) + l/4); quadrant 0 (a) keeps both bits 0,
 * 1 (b) sets the column bit, 2 (c) the row bit, 3 (d) both.
 * symmetrize: emit both directions before de-duplication (colouring input).
 * perm_seed != 0: relabel vertices by a seeded uniform permutation
 * ("randomly permuted vertex IDs"). */
gg_graph* gg_rmat(int scale, int64_t edge_factor, uint64_t seed, double a, double b, double c,
                  int symmetrize, uint64_t perm_seed) {
  if (scale < 0 || scale > 30 || edge_factor < 0) return NULL;
  int64_t n = (int64_t)1 << scale;
  int64_t ne = edge_factor * n;
  uint32_t* src = (uint32_t*)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(uint32_t));
  uint32_t* dst = (uint32_t*)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(uint32_t));
  if (!src || !dst) { free(src); free(dst); return NULL; }
  const uint32_t ta = (uint32_t)(a * 65536.0), tb = (uint32_t)((a + b) * 65536.0),
                 tc = (uint32_t)((a + b + c) * 65536.0);
  const int words = (scale + 3) / 4;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < ne; t++) {
    uint32_t u = 0, v = 0;
    uint64_t h = 0;
    for (int l = 0; l < scale; l++) {
      if ((l & 3) == 0) h = hash2(seed, (uint64_t)t * (uint64_t)words + (uint64_t)(l >> 2));
      uint32_t r = (uint32_t)((h >> (16 * (l & 3))) & 0xFFFFu);
      uint32_t q = r < ta ? 0u : (r < tb ? 1u : (r < tc ? 2u : 3u));
      u = (u << 1) | (q >> 1);
      v = (v << 1) | (q & 1u);
    }
    src[t] = u;
    dst[t] = v;
  }
  if (perm_seed) {
    uint32_t* perm = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!perm) { free(src); free(dst); return NULL; }
    for (int64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    for (int64_t i = n - 1; i > 0; i--) { /* Fisher–Yates, counter-based draws */
      uint64_t j = hash2(perm_seed, (uint64_t)i) % (uint64_t)(i + 1);
      uint32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
    }
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < ne; t++) { src[t] = perm[src[t]]; dst[t] = perm[dst[t]]; }
    free(perm);
  }
  gg_graph* g = build_csr(n, ne, src, dst, symmetrize);
  free(src);
  free(dst);
  return g;
}

/* Generic builder from an explicit edge list (tests; tiny graphs). */
gg_graph* gg_from_edges(int64_t n, int64_t ne, const uint32_t* src, const uint32_t* dst,
                        int symmetrize) {
  for (int64_t i = 0; i < ne; i++)
    if ((int64_t)src[i] >= n || (int64_t)dst[i] >= n) return NULL;
  return build_csr(n, ne, src, dst, symmetrize);
}

/* Relabel an existing CSR by a seeded permutation; returns the new graph and
 * writes forward[v] (old id -> new id) if forward != NULL. */
gg_graph* gg_permute(int64_t n, const int64_t* off, const int32_t* col, uint64_t perm_seed,
                     int32_t* forward) {
  int64_t m = off[n];
  uint32_t* perm = (uint32_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(uint32_t));
  uint32_t* src = (uint32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint32_t));
  uint32_t* dst = (uint32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint32_t));
  if (!perm || !src || !dst) { free(perm); free(src); free(dst); return NULL; }
  for (int64_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
  for (int64_t i = n - 1; i > 0; i--) {
    uint64_t j = hash2(perm_seed, (uint64_t)i) % (uint64_t)(i + 1);
    uint32_t tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
  }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; v++)
    for (int64_t e = off[v]; e < off[v + 1]; e++) { src[e] = perm[v]; dst[e] = perm[col[e]]; }
  if (forward) for (int64_t v = 0; v < n; v++) forward[v] = (int32_t)perm[v];
  gg_graph* g = build_csr(n, m, src, dst, 0);
  free(perm);
  free(src);
  free(dst);
  return g;
}
