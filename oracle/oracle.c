/*
 * oracle/oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU definitions of what the Atos hot path
 * (arxiv 2112.00132, "Atos: A Task-Parallel GPU Dynamic Scheduling Framework
 * for Dynamic Irregular Computations") computes.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this file's library.  It shares no code, header or constant with
 * paper_2112_00132_b200/ (the CUDA path), and the CUDA path never calls it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (not available at run time),
 * S:n = SPEC.md line n.  Readings of garbled or silent passages are numbered
 * as in DESIGN.md §3 ("R#").
 *
 * Pinned by tests/test_oracle_pins.py (closed forms, brute force, dense solve,
 * invariants).  Parity status per function:
 *   or_bfs            pinned (closed forms, Floyd–Warshall brute force)
 *   or_pagerank_jacobi pinned (closed forms, numpy dense solve)
 *   or_pagerank_push  pinned (error bound vs Jacobi, conservation invariant)
 *   or_greedy_color   pinned (closed forms, brute-force chromatic bound)
 *   validators        pinned (planted violations)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define OR_UNREACHED 0xFFFFFFFFu /* "vertex.dist = MAX_UINT32" */

/* ---------------------------------------------------------------------- */
/* BFS: serial FIFO breadth-first search (the BSP BFS of Alg. 1,  */
/* which "is exactly Dijkstra's algorithm").  depth[src] = 0 (R1);    */
/* depth[w] = depth[v] + 1 at first discovery; unreachable = MAX_UINT32.     */
/* Returns 0, or -1 on bad arguments / allocation failure.                   */
/* ---------------------------------------------------------------------- */
int or_bfs(int64_t n, const int64_t* off, const int32_t* col, int64_t src, uint32_t* depth) {
  if (n < 0 || src < 0 || src >= n) return -1;
  int64_t* fifo = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  if (!fifo) return -1;
  for (int64_t v = 0; v < n; v++) depth[v] = OR_UNREACHED;
  int64_t qh = 0, qt = 0;
  depth[src] = 0;
  fifo[qt++] = src;
  while (qh < qt) {
    int64_t v = fifo[qh++];
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      int64_t w = col[e];
      if (depth[w] == OR_UNREACHED) {
        depth[w] = depth[v] + 1;
        fifo[qt++] = w;
      }
    }
  }
  free(fifo);
  return 0;
}

/* ---------------------------------------------------------------------- */
/* PageRank fixed point (Alg. 3, reading R4/R5/R8):     */
/*   x = (1-a)*1 + a*P*x,   (P x)_w = sum_{v->w} x_v / deg(v),              */
/* dangling columns (deg 0) are zero.  Synchronous Jacobi in fp64 from       */
/* x0 = (1-a)*1 until ||x_{k+1}-x_k||_1 <= tol*||x_{k+1}||_1.               */
/* Computed as a pull over in-edges; each x_new[w] sums its in-edges in      */
/* ascending source order serially, so the result is bit-identical for any   */
/* OpenMP thread count (threads<=0: library default).                        */
/* Returns the number of iterations, or -1 on failure.                       */
/* ---------------------------------------------------------------------- */
int or_pagerank_jacobi(int64_t n, const int64_t* off, const int32_t* col, double alpha, double tol,
                       int max_iter, int threads, double* x) {
  if (n < 0 || !(alpha > 0 && alpha < 1)) return -1;
  if (threads > 0) omp_set_num_threads(threads);
  int64_t m = n ? off[n] : 0;
  /* transpose: in-edge lists, sources ascending (stable counting sort by target) */
  int64_t* ioff = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int32_t* isrc = (int32_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
  double* xn = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  double* contrib = (double*)malloc((size_t)(n > 0 ? n : 1) * sizeof(double));
  if (!ioff || !isrc || !xn || !contrib) { free(ioff); free(isrc); free(xn); free(contrib); return -1; }
  for (int64_t e = 0; e < m; e++) ioff[col[e] + 1]++;
  for (int64_t w = 0; w < n; w++) ioff[w + 1] += ioff[w];
  {
    int64_t* pos = (int64_t*)malloc(((size_t)n + 1) * sizeof(int64_t));
    if (!pos) { free(ioff); free(isrc); free(xn); free(contrib); return -1; }
    memcpy(pos, ioff, ((size_t)n + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < n; v++)
      for (int64_t e = off[v]; e < off[v + 1]; e++) isrc[pos[col[e]]++] = (int32_t)v;
    free(pos);
  }
  for (int64_t v = 0; v < n; v++) x[v] = 1.0 - alpha;
  int it = 0;
  for (it = 1; it <= max_iter; it++) {
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; v++) {
      int64_t d = off[v + 1] - off[v];
      contrib[v] = d ? x[v] / (double)d : 0.0;
    }
    double diff = 0, norm = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : diff, norm)
    for (int64_t w = 0; w < n; w++) {
      double s = 0.0;
      for (int64_t e = ioff[w]; e < ioff[w + 1]; e++) s += contrib[isrc[e]];
      double nv = (1.0 - alpha) + alpha * s;
      xn[w] = nv;
      diff += fabs(nv - x[w]);
      norm += fabs(nv);
    }
    memcpy(x, xn, (size_t)n * sizeof(double));
    if (diff <= tol * norm) break;
  }
  free(ioff); free(isrc); free(xn); free(contrib);
  return it > max_iter ? max_iter : it;
}

/* ---------------------------------------------------------------------- */
/* Serial push PageRank, fp64, FIFO order — the asynchronous PageRank of     */
/* Alg. 4 executed by one worker, with:                          */
/*   init (Alg. 3 lines 3-7, reading R4): rank = 1-a; residue = 0; for each  */
/*     edge v->w: residue[w] += (1-a)*a/deg(v); queue = all v in id order;   */
/*   pop v: r = residue[v]; residue[v] = 0; rank[v] += r; if deg(v) > 0 (R5):*/
/*     c = a*r/deg(v); for each w: old = residue[w]; residue[w] = old + c;   */
/*     push w iff old <= eps < old + c   (threshold-crossing activation, R6/R7).
/* Outputs rank, residue; *pushes = edge pushes performed, *pops = pops.      */
/* Returns 0, or -1 on failure / queue overflow.                             */
/* ---------------------------------------------------------------------- */
int or_pagerank_push(int64_t n, const int64_t* off, const int32_t* col, double alpha, double eps,
                     double* rank, double* residue, int64_t* pops, int64_t* pushes) {
  if (n < 0 || !(alpha > 0 && alpha < 1) || !(eps > 0)) return -1;
  int64_t cap = 2 * n + 1; /* at most 2 live copies per vertex (initial + one crossing) */
  int64_t* ring = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  if (!ring) return -1;
  for (int64_t v = 0; v < n; v++) { rank[v] = 1.0 - alpha; residue[v] = 0.0; }
  for (int64_t v = 0; v < n; v++) {
    int64_t d = off[v + 1] - off[v];
    for (int64_t e = off[v]; e < off[v + 1]; e++) residue[col[e]] += (1.0 - alpha) * alpha / (double)d;
  }
  int64_t qh = 0, qt = 0, np = 0, ne = 0;
  for (int64_t v = 0; v < n; v++) ring[(qt++) % cap] = v;
  while (qh < qt) {
    int64_t v = ring[(qh++) % cap];
    np++;
    double r = residue[v];
    residue[v] = 0.0;
    rank[v] += r;
    int64_t d = off[v + 1] - off[v];
    if (d == 0 || r == 0.0) continue;
    double c = alpha * r / (double)d;
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      int64_t w = col[e];
      double old = residue[w];
      residue[w] = old + c;
      ne++;
      if (old <= eps && old + c > eps) {
        if (qt - qh >= cap) { free(ring); return -1; }
        ring[(qt++) % cap] = w;
      }
    }
  }
  free(ring);
  if (pops) *pops = np;
  if (pushes) *pushes = ne;
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Greedy colouring: serial first-fit in vertex-id order (the speculative    */
/* greedy scheme of Alg. 5/6, executed without concurrency, where */
/* no conflict can arise).  color[v] = smallest c >= 0 not used by an        */
/* already-coloured neighbour (R11: colours in [0, deg(v)], self-loops       */
/* ignored).  Returns the number of colours used, or -1.                     */
/* ---------------------------------------------------------------------- */
int or_greedy_color(int64_t n, const int64_t* off, const int32_t* col, int32_t* color) {
  int64_t maxd = 0;
  for (int64_t v = 0; v < n; v++)
    if (off[v + 1] - off[v] > maxd) maxd = off[v + 1] - off[v];
  unsigned char* forbidden = (unsigned char*)calloc((size_t)maxd + 2, 1);
  if (!forbidden) return -1;
  for (int64_t v = 0; v < n; v++) color[v] = -1;
  int32_t ncolors = 0;
  for (int64_t v = 0; v < n; v++) {
    int64_t d = off[v + 1] - off[v];
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      int32_t c = col[e] == v ? -1 : color[col[e]];
      if (c >= 0 && c <= d) forbidden[c] = 1;
    }
    int32_t c = 0;
    while (forbidden[c]) c++;
    color[v] = c;
    if (c + 1 > ncolors) ncolors = c + 1;
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      int32_t cc = col[e] == v ? -1 : color[col[e]];
      if (cc >= 0 && cc <= d) forbidden[cc] = 0;
    }
  }
  free(forbidden);
  return ncolors;
}

/* ---------------------------------------------------------------------- */
/* Validators.                                                   */
/* ---------------------------------------------------------------------- */

/* BFS depth certificate: depth[src] == 0; for every edge v->w with finite   */
/* depth[v]: depth[w] <= depth[v]+1; every finite depth[w] > 0 has an        */
/* in-neighbour with depth[w]-1; unreachable vertices have no finite         */
/* in-neighbour.  Returns the number of violations (first one in *bad_v).    */
int64_t or_check_bfs(int64_t n, const int64_t* off, const int32_t* col, int64_t src,
                     const uint32_t* depth, int64_t* bad_v) {
  int64_t bad = 0;
  unsigned char* has_parent = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!has_parent) return -1;
#define FLAG(v) do { if (!bad && bad_v) *bad_v = (v); bad++; } while (0)
  if (src < 0 || src >= n || depth[src] != 0) FLAG(src);
  for (int64_t v = 0; v < n; v++) {
    if (depth[v] == OR_UNREACHED) continue;
    for (int64_t e = off[v]; e < off[v + 1]; e++) {
      int64_t w = col[e];
      if (depth[w] == OR_UNREACHED || depth[w] > depth[v] + 1) FLAG(w);
      else if (depth[w] == depth[v] + 1) has_parent[w] = 1;
    }
  }
  for (int64_t v = 0; v < n; v++)
    if (v != src && depth[v] != OR_UNREACHED && !has_parent[v]) FLAG(v);
#undef FLAG
  free(has_parent);
  return bad;
}

/* Colouring check: counts edges u->w (u != w) with color[u] == color[w],    */
/* plus vertices with color < 0 or color > deg(v).  *ncolors = max+1.        */
int64_t or_check_coloring(int64_t n, const int64_t* off, const int32_t* col, const int32_t* color,
                          int32_t* ncolors, int64_t* bad_v) {
  int64_t bad = 0;
  int32_t mx = -1;
  for (int64_t v = 0; v < n; v++) {
    int64_t d = off[v + 1] - off[v];
    if (color[v] < 0 || color[v] > d) { if (!bad && bad_v) *bad_v = v; bad++; }
    if (color[v] > mx) mx = color[v];
    for (int64_t e = off[v]; e < off[v + 1]; e++)
      if (col[e] != v && color[col[e]] == color[v]) { if (!bad && bad_v) *bad_v = v; bad++; }
  }
  if (ncolors) *ncolors = mx + 1;
  return bad;
}
