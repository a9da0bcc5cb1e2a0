/*
 * graphs.c -- seeded synthetic graph generators (INPUT GENERATION ONLY).
 *
 * The paper's MaxCut workloads are Gset and DIMACS10;
 * neither is available here, so these generators produce graphs of the
 * same shape:
 *   family 0  Erdos-Renyi G(n, p)                      (configs[0], Gset-like)
 *   family 1  2-D torus rows x cols, weights +-1       (configs[1], Gset toroidal)
 *   family 2  ER + Chung-Lu with Zipf(2.1) degrees      (configs[2], DIMACS10 skewed)
 *   family 3  mutual k-NN random geometric, Morton id  (configs[3], rgg_n_2_24 / road)
 *   family 4  Morton ring + random perfect matching    (configs[4], 3-regular + geometric)
 * Output is the weighted combinatorial Laplacian
 *   L = sum_{ij in E} w_ij (e_i - e_j)(e_i - e_j)^T
 * as CSR with the diagonal stored in place, columns ascending.  Duplicate
 * edges are merged (family 0-3 unit weights: kept once; family 4: weights
 * summed), self-loops dropped.  All randomness is the counter-based stream of
 * scg_rng.h, so the output depends only on (family, size, seed).
 *
 * Nothing here is solver arithmetic.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include "include/scg_rng.h"

typedef struct {
  int64_t n;
  int64_t nnz;
  int64_t *row_ptr; /* n+1 */
  int32_t *col;     /* nnz */
  double *val;      /* nnz */
} scg_graph;

typedef struct {
  int64_t m, cap;
  int32_t *i, *j;
  double *w;
} edge_list;

static int el_push(edge_list *e, int32_t a, int32_t b, double w) {
  if (a == b) return 0; /* self-loops dropped */
  if (e->m == e->cap) {
    int64_t nc = e->cap ? e->cap * 2 : 1024;
    int32_t *ni = (int32_t *)realloc(e->i, nc * sizeof(int32_t));
    int32_t *nj = (int32_t *)realloc(e->j, nc * sizeof(int32_t));
    double *nw = (double *)realloc(e->w, nc * sizeof(double));
    if (!ni || !nj || !nw) return -1;
    e->i = ni; e->j = nj; e->w = nw; e->cap = nc;
  }
  if (a > b) { int32_t t = a; a = b; b = t; }
  e->i[e->m] = a; e->j[e->m] = b; e->w[e->m] = w; e->m++;
  return 0;
}

static void el_free(edge_list *e) { free(e->i); free(e->j); free(e->w); memset(e, 0, sizeof(*e)); }

typedef struct { int32_t c; double v; } cv_pair;

static int cmp_cv(const void *a, const void *b) {
  const cv_pair *x = (const cv_pair *)a, *y = (const cv_pair *)b;
  return (x->c > y->c) - (x->c < y->c);
}

/* Edge list -> Laplacian CSR with diagonal.  dedupe: 1 keep duplicates once, 0 sum them. */
static scg_graph *laplacian_from_edges(int64_t n, const edge_list *e, int dedupe) {
  int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) return NULL;
  for (int64_t k = 0; k < e->m; ++k) { cnt[e->i[k] + 1]++; cnt[e->j[k] + 1]++; }
  for (int64_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r] + 0;
  /* cnt is prefix of off-diagonal counts without the diagonal */
  int64_t tot = cnt[n];
  cv_pair *tmp = (cv_pair *)malloc((size_t)(tot > 0 ? tot : 1) * sizeof(cv_pair));
  int64_t *pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  if (!tmp || !pos) { free(cnt); free(tmp); free(pos); return NULL; }
  for (int64_t r = 0; r < n; ++r) pos[r] = cnt[r];
  for (int64_t k = 0; k < e->m; ++k) {
    int32_t a = e->i[k], b = e->j[k];
    double w = e->w[k];
    tmp[pos[a]].c = b; tmp[pos[a]].v = w; pos[a]++;
    tmp[pos[b]].c = a; tmp[pos[b]].v = w; pos[b]++;
  }
  free(pos);
  /* sort + merge each row; count merged lengths */
  int64_t *len = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  if (!len) { free(cnt); free(tmp); return NULL; }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    cv_pair *row = tmp + cnt[r];
    int64_t l = cnt[r + 1] - cnt[r];
    if (l > 1) {
      if (l <= 16) { /* insertion sort (stable) */
        for (int64_t a = 1; a < l; ++a) {
          cv_pair x = row[a];
          int64_t b = a - 1;
          while (b >= 0 && row[b].c > x.c) { row[b + 1] = row[b]; --b; }
          row[b + 1] = x;
        }
      } else {
        qsort(row, (size_t)l, sizeof(cv_pair), cmp_cv);
      }
    }
    int64_t o = 0;
    for (int64_t a = 0; a < l; ++a) {
      if (o > 0 && row[o - 1].c == row[a].c) {
        if (!dedupe) row[o - 1].v += row[a].v;
      } else {
        row[o++] = row[a];
      }
    }
    len[r] = o + 1; /* + diagonal */
  }
  scg_graph *g = (scg_graph *)calloc(1, sizeof(scg_graph));
  g->n = n;
  g->row_ptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
  g->row_ptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) g->row_ptr[r + 1] = g->row_ptr[r] + len[r];
  g->nnz = g->row_ptr[n];
  g->col = (int32_t *)malloc((size_t)g->nnz * sizeof(int32_t));
  g->val = (double *)malloc((size_t)g->nnz * sizeof(double));
  if (!g->col || !g->val) { free(cnt); free(tmp); free(len); free(g->row_ptr); free(g->col); free(g->val); free(g); return NULL; }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) {
    const cv_pair *row = tmp + cnt[r];
    int64_t l = len[r] - 1;
    double deg = 0.0;
    for (int64_t a = 0; a < l; ++a) deg += row[a].v;
    int64_t o = g->row_ptr[r];
    int placed = 0;
    for (int64_t a = 0; a < l; ++a) {
      if (!placed && row[a].c > r) { g->col[o] = (int32_t)r; g->val[o] = deg; ++o; placed = 1; }
      g->col[o] = row[a].c; g->val[o] = -row[a].v; ++o;
    }
    if (!placed) { g->col[o] = (int32_t)r; g->val[o] = deg; ++o; }
  }
  free(cnt); free(tmp); free(len);
  return g;
}

/* ---- family 0: Erdos-Renyi ---- */
static scg_graph *gen_er(int64_t n, double p, uint64_t seed) {
  edge_list e = {0};
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j)
      if (scg_uniform(seed, SCG_STREAM_GRAPH, 0u, (uint64_t)(i * n + j)) < p)
        if (el_push(&e, (int32_t)i, (int32_t)j, 1.0)) { el_free(&e); return NULL; }
  scg_graph *g = laplacian_from_edges(n, &e, 1);
  el_free(&e);
  return g;
}

/* ---- family 1: torus with +-1 weights ---- */
static scg_graph *gen_torus(int64_t rows, int64_t cols, uint64_t seed) {
  edge_list e = {0};
  int64_t n = rows * cols;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      int64_t id = r * cols + c;
      int64_t down = ((r + 1) % rows) * cols + c;
      int64_t right = r * cols + (c + 1) % cols;
      double w0 = scg_uniform(seed, SCG_STREAM_GRAPH, 1u, (uint64_t)(2 * id)) < 0.5 ? 1.0 : -1.0;
      double w1 = scg_uniform(seed, SCG_STREAM_GRAPH, 1u, (uint64_t)(2 * id + 1)) < 0.5 ? 1.0 : -1.0;
      if (el_push(&e, (int32_t)id, (int32_t)down, w0) || el_push(&e, (int32_t)id, (int32_t)right, w1)) {
        el_free(&e); return NULL;
      }
    }
  scg_graph *g = laplacian_from_edges(n, &e, 0);
  el_free(&e);
  return g;
}

/* ---- family 2: ER(avg deg 4) + Chung-Lu with Zipf(2.1) on {1..kmax} (avg deg 4) ---- */
static int64_t lower_bound_d(const double *a, int64_t n, double x) { /* first idx with a[idx] > x */
  int64_t lo = 0, hi = n;
  while (lo < hi) { int64_t mid = (lo + hi) / 2; if (a[mid] > x) hi = mid; else lo = mid + 1; }
  return lo < n ? lo : n - 1;
}

static scg_graph *gen_powerlaw(int64_t n, uint64_t seed) {
  const int kmax = 10000;
  const double expo = 2.1;
  double *zcdf = (double *)malloc(sizeof(double) * kmax);
  double acc = 0.0;
  for (int k = 1; k <= kmax; ++k) { acc += pow((double)k, -expo); zcdf[k - 1] = acc; }
  for (int k = 0; k < kmax; ++k) zcdf[k] /= acc;
  double *kcdf = (double *)malloc(sizeof(double) * (size_t)n);
  double ks = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double u = scg_uniform(seed, SCG_STREAM_GRAPH, 3u, (uint64_t)i);
    int64_t k = lower_bound_d(zcdf, kmax, u) + 1;
    ks += (double)k;
    kcdf[i] = ks;
  }
  for (int64_t i = 0; i < n; ++i) kcdf[i] /= ks;
  free(zcdf);
  edge_list e = {0};
  int64_t m1 = 2 * n, m2 = 2 * n;
  for (int64_t k = 0; k < m1; ++k) {
    int64_t a = (int64_t)(scg_uniform(seed, SCG_STREAM_GRAPH, 2u, (uint64_t)(2 * k)) * (double)n);
    int64_t b = (int64_t)(scg_uniform(seed, SCG_STREAM_GRAPH, 2u, (uint64_t)(2 * k + 1)) * (double)n);
    if (el_push(&e, (int32_t)a, (int32_t)b, 1.0)) { el_free(&e); free(kcdf); return NULL; }
  }
  for (int64_t k = 0; k < m2; ++k) {
    int64_t a = lower_bound_d(kcdf, n, scg_uniform(seed, SCG_STREAM_GRAPH, 4u, (uint64_t)(2 * k)));
    int64_t b = lower_bound_d(kcdf, n, scg_uniform(seed, SCG_STREAM_GRAPH, 4u, (uint64_t)(2 * k + 1)));
    if (el_push(&e, (int32_t)a, (int32_t)b, 1.0)) { el_free(&e); free(kcdf); return NULL; }
  }
  free(kcdf);
  scg_graph *g = laplacian_from_edges(n, &e, 1);
  el_free(&e);
  return g;
}

/* ---- family 3: mutual k-NN random geometric graph in Morton order ---- */
/* 21-bit coordinate -> its bits at the even positions 0, 2, ..., 40 (2-D Z-order;
 * code = spread21(qx) | spread21(qy) << 1 < 2^42, sorted in full by the 48-bit radix sort) */
static uint64_t spread21(uint64_t x) {
  x &= 0x1fffffull;
  x = (x | (x << 16)) & 0x0000ffff0000ffffull;
  x = (x | (x << 8)) & 0x00ff00ff00ff00ffull;
  x = (x | (x << 4)) & 0x0f0f0f0f0f0f0f0full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

static void radix_sort_u64(uint64_t *key, int64_t *val, int64_t n) {
  uint64_t *k2 = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  int64_t *v2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  for (int pass = 0; pass < 6; ++pass) { /* 6 x 8 = 48 bits (keys < 2^42) */
    int sh = pass * 8;
    int64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[((key[i] >> sh) & 0xff) + 1]++;
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (int64_t i = 0; i < n; ++i) {
      int64_t d = cnt[(key[i] >> sh) & 0xff]++;
      k2[d] = key[i]; v2[d] = val[i];
    }
    memcpy(key, k2, sizeof(uint64_t) * (size_t)n);
    memcpy(val, v2, sizeof(int64_t) * (size_t)n);
  }
  free(k2); free(v2);
}

#define KNN_K 4
static scg_graph *gen_rgg(int64_t n, uint64_t seed) {
  double *px = (double *)malloc(sizeof(double) * (size_t)n);
  double *py = (double *)malloc(sizeof(double) * (size_t)n);
  uint64_t *code = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double x = scg_uniform(seed, SCG_STREAM_GRAPH, 5u, (uint64_t)(2 * i));
    double y = scg_uniform(seed, SCG_STREAM_GRAPH, 5u, (uint64_t)(2 * i + 1));
    px[i] = x; py[i] = y;
    uint64_t qx = (uint64_t)(x * 2097152.0), qy = (uint64_t)(y * 2097152.0);
    code[i] = spread21(qx) | (spread21(qy) << 1);
    perm[i] = i;
  }
  radix_sort_u64(code, perm, n); /* stable: ties keep original index order */
  free(code);
  /* relabel points in Morton order */
  double *x = (double *)malloc(sizeof(double) * (size_t)n);
  double *y = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t v = 0; v < n; ++v) { x[v] = px[perm[v]]; y[v] = py[perm[v]]; }
  free(px); free(py); free(perm);
  /* grid buckets */
  int64_t G = (int64_t)floor(sqrt((double)n / 2.0));
  if (G < 1) G = 1;
  int64_t ncell = G * G;
  int64_t *cstart = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
  int32_t *cell = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int32_t *items = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t v = 0; v < n; ++v) {
    int64_t cx = (int64_t)(x[v] * (double)G), cy = (int64_t)(y[v] * (double)G);
    if (cx >= G) cx = G - 1;
    if (cy >= G) cy = G - 1;
    cell[v] = (int32_t)(cy * G + cx);
    cstart[cell[v] + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) cstart[c + 1] += cstart[c];
  {
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)ncell);
    memcpy(fill, cstart, sizeof(int64_t) * (size_t)ncell);
    for (int64_t v = 0; v < n; ++v) items[fill[cell[v]]++] = (int32_t)v;
    free(fill);
  }
  int32_t *nb = (int32_t *)malloc(sizeof(int32_t) * (size_t)n * KNN_K);
  double h = 1.0 / (double)G;
#pragma omp parallel for schedule(dynamic, 8192)
  for (int64_t v = 0; v < n; ++v) {
    double bd[KNN_K];
    int32_t bi[KNN_K];
    int cntb = 0;
    int64_t cx = cell[v] % G, cy = cell[v] / G;
    for (int64_t r = 0;; ++r) {
      for (int64_t yy = cy - r; yy <= cy + r; ++yy) {
        if (yy < 0 || yy >= G) continue;
        for (int64_t xx = cx - r; xx <= cx + r; ++xx) {
          if (xx < 0 || xx >= G) continue;
          if (r > 0 && yy != cy - r && yy != cy + r && xx != cx - r && xx != cx + r) continue;
          int64_t c = yy * G + xx;
          for (int64_t a = cstart[c]; a < cstart[c + 1]; ++a) {
            int32_t u = items[a];
            if (u == v) continue;
            double dx = x[u] - x[v], dy = y[u] - y[v];
            double d = dx * dx + dy * dy;
            /* insert into sorted top-K by (d, u) */
            if (cntb == KNN_K && (d > bd[KNN_K - 1] || (d == bd[KNN_K - 1] && u > bi[KNN_K - 1]))) continue;
            int p = cntb < KNN_K ? cntb++ : KNN_K - 1;
            while (p > 0 && (bd[p - 1] > d || (bd[p - 1] == d && bi[p - 1] > u))) {
              bd[p] = bd[p - 1]; bi[p] = bi[p - 1]; --p;
            }
            bd[p] = d; bi[p] = u;
          }
        }
      }
      double reach = (double)r * h;
      if (cntb == KNN_K && bd[KNN_K - 1] <= reach * reach) break;
      if (r > G) break;
    }
    for (int a = 0; a < KNN_K; ++a) nb[v * KNN_K + a] = a < cntb ? bi[a] : -1;
  }
  free(cstart); free(cell); free(items); free(x); free(y);
  /* per-vertex k in {2,3,4} w.p. (0.2, 0.3, 0.5) */
  uint8_t *kk = (uint8_t *)malloc((size_t)n);
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    double u = scg_uniform(seed, SCG_STREAM_GRAPH, 6u, (uint64_t)v);
    kk[v] = (uint8_t)(u < 0.2 ? 2 : (u < 0.5 ? 3 : 4));
  }
  edge_list e = {0};
  for (int64_t v = 0; v < n; ++v) {
    for (int a = 0; a < kk[v]; ++a) {
      int32_t u = nb[v * KNN_K + a];
      if (u < 0 || u <= v) continue;
      int mutual = 0;
      for (int b = 0; b < kk[u]; ++b) if (nb[(int64_t)u * KNN_K + b] == (int32_t)v) mutual = 1;
      if (mutual && el_push(&e, (int32_t)v, u, 1.0)) { el_free(&e); free(nb); free(kk); return NULL; }
    }
  }
  free(nb); free(kk);
  scg_graph *g = laplacian_from_edges(n, &e, 1);
  el_free(&e);
  return g;
}

/* ---- family 4: ring (Morton order) + random perfect matching, w ~ U[0.5, 1.5] ---- */
static scg_graph *gen_ring_matching(int64_t n, uint64_t seed) {
  edge_list e = {0};
  e.cap = n + n / 2 + 16;
  e.i = (int32_t *)malloc(sizeof(int32_t) * (size_t)e.cap);
  e.j = (int32_t *)malloc(sizeof(int32_t) * (size_t)e.cap);
  e.w = (double *)malloc(sizeof(double) * (size_t)e.cap);
  for (int64_t i = 0; i < n; ++i)
    el_push(&e, (int32_t)i, (int32_t)((i + 1) % n), 0.5 + scg_uniform(seed, SCG_STREAM_GRAPH, 7u, (uint64_t)i));
  int32_t *perm = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) perm[i] = (int32_t)i;
  for (int64_t i = n - 1; i > 0; --i) { /* Fisher-Yates */
    int64_t j = (int64_t)(scg_uniform(seed, SCG_STREAM_GRAPH, 8u, (uint64_t)i) * (double)(i + 1));
    if (j > i) j = i;
    int32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
  }
  for (int64_t k = 0; k + 1 < n; k += 2)
    el_push(&e, perm[k], perm[k + 1], 0.5 + scg_uniform(seed, SCG_STREAM_GRAPH, 9u, (uint64_t)(k / 2)));
  free(perm);
  scg_graph *g = laplacian_from_edges(n, &e, 0);
  el_free(&e);
  return g;
}

/* ---- exported ---- */
void *scg_gen_graph(int family, int64_t a, int64_t b, double p, uint64_t seed) {
  switch (family) {
    case 0: return gen_er(a, p, seed);
    case 1: return gen_torus(a, b, seed);
    case 2: return gen_powerlaw(a, seed);
    case 3: return gen_rgg(a, seed);
    case 4: return gen_ring_matching(a, seed);
    default: return NULL;
  }
}

/* Laplacian from a caller edge list (i, j, w); dedupe=0 sums duplicates (A16). */
void *scg_graph_from_edges(int64_t n, int64_t m, const int32_t *i, const int32_t *j, const double *w, int dedupe) {
  edge_list e = {0};
  for (int64_t k = 0; k < m; ++k)
    if (el_push(&e, i[k], j[k], w[k])) { el_free(&e); return NULL; }
  scg_graph *g = laplacian_from_edges(n, &e, dedupe);
  el_free(&e);
  return g;
}

void scg_graph_info(const void *gp, int64_t *n, int64_t *nnz) {
  const scg_graph *g = (const scg_graph *)gp;
  *n = g->n; *nnz = g->nnz;
}

void scg_graph_copy(const void *gp, int64_t *row_ptr, int32_t *col, double *val) {
  const scg_graph *g = (const scg_graph *)gp;
  memcpy(row_ptr, g->row_ptr, sizeof(int64_t) * (size_t)(g->n + 1));
  memcpy(col, g->col, sizeof(int32_t) * (size_t)g->nnz);
  memcpy(val, g->val, sizeof(double) * (size_t)g->nnz);
}

void scg_graph_free(void *gp) {
  scg_graph *g = (scg_graph *)gp;
  if (!g) return;
  free(g->row_ptr); free(g->col); free(g->val); free(g);
}

/* Bulk Gaussian draws (for tests / host-side inputs): out[i] = scg_normal(seed, stream, sub, first + i). */
void scg_fill_normal(uint64_t seed, uint32_t stream, uint32_t sub, uint64_t first, int64_t count, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) out[i] = scg_normal(seed, stream, sub, first + (uint64_t)i);
}

void scg_fill_uniform(uint64_t seed, uint32_t stream, uint32_t sub, uint64_t first, int64_t count, double *out) {
  for (int64_t i = 0; i < count; ++i) out[i] = scg_uniform(seed, stream, sub, first + (uint64_t)i);
}

void scg_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1, uint32_t *out4) {
  scg_philox_out o = scg_philox4x32_10(c0, c1, c2, c3, k0, k1);
  for (int a = 0; a < 4; ++a) out4[a] = o.w[a];
}
