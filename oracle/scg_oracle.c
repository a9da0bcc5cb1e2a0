/*
 * scg_oracle.c -- CPU ORACLE for the SketchyCGAL MaxCut hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1912_02949_b200/) never imports, links or calls it,
 * and this file shares no code with the CUDA path; the only common source is
 * the seeded input stream scg_inputs/include/scg_rng.h (random inputs only).
 *
 * Plain, slow, fp64.  OpenMP only splits independent row loops and the exact sums
 * (CAC-2 sums are exact integers, so any split gives the same bits; the thread count
 * never changes a result -- tests/test_oracle_pins.py checks 1 vs all threads).
 * Every function follows the paper
 * (arXiv 1912.02949, /root/reference/PAPER.md, cited as P:<line>) step by step,
 * in the paper's order and notation, with the readings and the Canonical
 * Arithmetic Contract (CAC) written down in DESIGN.md section 3.  The CAC
 * only fixes *how each written operation is rounded* (the paper's Lanczos
 * method has no reorthogonalization, so any two implementations
 * that round differently diverge):
 *   CAC-1  one IEEE fp64 round-to-nearest operation per written +,-,*,/,sqrt;
 *          fma() only where written (compiled with -ffp-contract=off).
 *   CAC-2  global sums are EXACT: xsum(p_1..p_N) = RNE(sum_r Q(p_r)), with
 *          Q(p) = p truncated toward zero to a multiple of 2^-200 (|p| < 2^100).
 *          dot(a, b) = xsum(fl(a_r * b_r)).
 *   CAC-3  (D x)_r = d_r x_r + sum_{j in N(r), ascending} m_rj x_j, left to right,
 *          acc = fl(d_r * x_r); acc = fma(m_rj, x_j, acc); rows of more than 32
 *          entries: 32 (rows of more than 1024 entries: 256) strided partial chains
 *          combined by halving (reading R27).
 *   CAC-4  Alg. 2 as printed, two-pass, with readings R1-R5; a
 *          normalization v / rho is evaluated as v * fl(1/rho) (reading R26).
 *   CAC-5  tridiagonal min eigenpair by Sturm multisection + inverse iteration.
 *   CAC-6  scalar schedules evaluated as written in DESIGN.md.
 *
 * Parity pins: tests/test_oracle_*.py (closed forms, dense eigensolvers,
 * math.fsum, loop invariants, brute-force cuts).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../scg_inputs/include/scg_rng.h"

/* ------------------------------------------------------------------------- */
/* CAC-2: exact summation.  Big integer in base 2^32, value = sum d[i] 2^(32 i - 200). */
#define XS_LIMBS 12
#define XS_LSB_EXP (-200)

typedef struct {
  int64_t d[XS_LIMBS];
  int64_t adds;
  int err; /* 1: |p| >= 2^100 or non-finite summand */
} xsum_t;

static void xs_init(xsum_t *a) { memset(a, 0, sizeof(*a)); }

static void xs_carry(xsum_t *a) {
  for (int i = 0; i < XS_LIMBS - 1; ++i) {
    int64_t c = a->d[i] >> 32; /* floor division by 2^32 */
    a->d[i] -= c * ((int64_t)1 << 32);
    a->d[i + 1] += c;
  }
}

static void xs_add(xsum_t *a, double p) {
  if (p == 0.0) return;
  if (!isfinite(p) || fabs(p) >= 0x1p100) { a->err = 1; return; }
  union { double f; uint64_t u; } b;
  b.f = p;
  int neg = (int)(b.u >> 63);
  int e = (int)((b.u >> 52) & 0x7ff);
  uint64_t m = b.u & 0x000fffffffffffffull;
  if (e == 0) e = 1; else m |= 0x0010000000000000ull;
  /* p = m * 2^(e - 1075);  shift relative to 2^-200 */
  int s = e - 1075 - XS_LSB_EXP;
  if (s < 0) { m = (-s >= 64) ? 0 : (m >> (-s)); s = 0; } /* Q: truncate toward zero */
  if (m == 0) return;
  int q = s / 32, r = s % 32;
  unsigned __int128 x = (unsigned __int128)m << r;
  int64_t d0 = (int64_t)(uint64_t)(x & 0xffffffffu);
  int64_t d1 = (int64_t)(uint64_t)((x >> 32) & 0xffffffffu);
  int64_t d2 = (int64_t)(uint64_t)((x >> 64) & 0xffffffffu);
  if (neg) { a->d[q] -= d0; a->d[q + 1] -= d1; a->d[q + 2] -= d2; }
  else { a->d[q] += d0; a->d[q + 1] += d1; a->d[q + 2] += d2; }
  if (++a->adds >= (1 << 20)) { xs_carry(a); a->adds = 0; }
}

/* Round the exact sum to the nearest double (ties to even). */
static double xs_round(xsum_t *a) {
  xs_carry(a);
  uint32_t mag[XS_LIMBS];
  int neg = a->d[XS_LIMBS - 1] < 0;
  if (neg) { /* magnitude of a negative number: two's complement across digits */
    int64_t borrow = 0;
    for (int i = 0; i < XS_LIMBS; ++i) {
      int64_t v = -a->d[i] - borrow;
      borrow = 0;
      while (v < 0) { v += ((int64_t)1 << 32); borrow += 1; }
      mag[i] = (uint32_t)v;
    }
  } else {
    for (int i = 0; i < XS_LIMBS; ++i) mag[i] = (uint32_t)a->d[i];
  }
  int top = -1;
  for (int i = XS_LIMBS - 1; i >= 0; --i) if (mag[i]) { top = i; break; }
  if (top < 0) return 0.0;
  int hb = 31;
  while (!((mag[top] >> hb) & 1u)) --hb;
  int B = top * 32 + hb; /* index of the highest set bit */
  /* gather bits [B-63, B] into M64, sticky = any set bit below B-63 */
  uint64_t M64 = 0;
  int sticky = 0;
  for (int bit = B; bit >= 0; --bit) {
    int v = (mag[bit / 32] >> (bit % 32)) & 1u;
    if (B - bit < 64) M64 = (M64 << 1) | (uint64_t)v;
    else if (v) { sticky = 1; break; }
  }
  int nbits = B + 1 < 64 ? B + 1 : 64; /* bits collected */
  double res;
  if (nbits <= 53) {
    res = ldexp((double)M64, XS_LSB_EXP);
  } else {
    int drop = nbits - 53;
    uint64_t keep = M64 >> drop;
    uint64_t rem = M64 & (((uint64_t)1 << drop) - 1); /* drop <= 11 */
    uint64_t half = (uint64_t)1 << (drop - 1);
    int round_up;
    if (rem > half) round_up = 1;
    else if (rem < half) round_up = 0;
    else round_up = sticky ? 1 : (int)(keep & 1u); /* tie: to even */
    keep += (uint64_t)round_up;
    /* value = keep * 2^(B - 52 + XS_LSB_EXP) */
    res = ldexp((double)keep, B - 52 + XS_LSB_EXP);
  }
  return neg ? -res : res;
}

/* Add the exact value of b into a (integers: exact; both carried first so no digit overflows). */
static void xs_merge(xsum_t *a, xsum_t *b) {
  xs_carry(a);
  xs_carry(b);
  for (int i = 0; i < XS_LIMBS; ++i) a->d[i] += b->d[i];
  a->err |= b->err;
  a->adds = 0;
}

/* CAC-2 dot product: the exact sum of the rounded products fl(a_r b_r), rounded once.
 * b == NULL: the exact sum of a.  Threads sum disjoint row ranges exactly and the partial
 * integers are added exactly, so the result does not depend on the thread count. */
static double o_dot(const double *a, const double *b, int64_t n, int *err) {
  xsum_t s;
  xs_init(&s);
#pragma omp parallel if (n > 65536)
  {
    xsum_t part;
    xs_init(&part);
#pragma omp for schedule(static)
    for (int64_t r = 0; r < n; ++r) xs_add(&part, b ? a[r] * b[r] : a[r]);
#pragma omp critical
    xs_merge(&s, &part);
  }
  if (s.err && err) *err = 1;
  return xs_round(&s);
}

double oracle_xsum(const double *p, int64_t n, int *err) {
  int e = 0;
  double r = o_dot(p, NULL, n, &e);
  if (err) *err = e;
  return r;
}

/* Threads of the OpenMP loops (n <= 0: all cores); returns the count in effect. */
int oracle_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  else omp_set_num_threads(omp_get_num_procs());
  return omp_get_max_threads();
}

double oracle_dot(const double *a, const double *b, int64_t n) { return o_dot(a, b, n, NULL); }

/* ------------------------------------------------------------------------- */
/* CAC-3: D = offdiag(m) + diag(d), rows ascending.  Primitive 1 + 2 of
 * eqn:primitives, MaxCut instance P:609-614. */
typedef struct {
  int64_t n;
  const int64_t *rp;   /* off-diagonal CSR */
  const int32_t *col;
  const double *m;     /* off-diagonal values of C (or of M) */
} o_off;

/* CAC-3 row of D x.  Rows with at most 32 off-diagonal entries: one chain from fl(d_r x_r).
 * Longer rows (reading R27): W strided partial chains, W = 32 for
 * rows of 33..1024 entries and W = 256 for rows of more than 1024 entries; partial chain l
 * (l = 0..W-1) runs over the entries k = l, l+W, l+2W, ... of the row (ascending column order)
 * by fma from 0; the W partials combine by halving, L[l] = L[l] + L[l+off] for
 * off = W/2, ..., 2, 1 and l < off; the row is fl(fl(d_r x_r) + L[0]). */
#define O_LONG_ROW 32
#define O_HEAVY_ROW 1024
static void o_apply(const o_off *A, const double *d, const double *x, double *y) {
#pragma omp parallel for schedule(static, 4096) if (A->n > 65536)
  for (int64_t r = 0; r < A->n; ++r) {
    const int64_t a = A->rp[r], b = A->rp[r + 1];
    if (b - a <= O_LONG_ROW) {
      double acc = d[r] * x[r];
      for (int64_t k = a; k < b; ++k) acc = fma(A->m[k], x[A->col[k]], acc);
      y[r] = acc;
    } else {
      const int W = b - a > O_HEAVY_ROW ? 256 : 32;
      double L[256];
      for (int l = 0; l < W; ++l) L[l] = 0.0;
      for (int64_t k = a; k < b; ++k) {
        const int l = (int)((k - a) % W);
        L[l] = fma(A->m[k], x[A->col[k]], L[l]);
      }
      for (int off = W / 2; off >= 1; off /= 2)
        for (int l = 0; l < off; ++l) L[l] = L[l] + L[l + off];
      y[r] = d[r] * x[r] + L[0];
    }
  }
}

void oracle_apply(int64_t n, const int64_t *rp, const int32_t *col, const double *m, const double *d,
                  const double *x, double *y) {
  o_off A = {n, rp, col, m};
  o_apply(&A, d, x, y);
}

/* ------------------------------------------------------------------------- */
/* CAC-5: minimum eigenpair of T = tridiag(rho_{1:k-1}, omega_{1:k}, rho_{1:k-1})
 * (Alg. 2 lines 11-12; "exploit tridiagonal form").  Sturm count =
 * number of sign changes of the characteristic-polynomial sequence. */
static int o_sturm(const double *om, const double *rho2, int k, double x) {
  double pprev = 1.0, p = om[0] - x;
  int sprev = 1;
  int s = p > 0.0 ? 1 : (p < 0.0 ? -1 : -sprev);
  int cnt = (s != sprev);
  for (int j = 1; j < k; ++j) {
    double pn = fma(om[j] - x, p, -(rho2[j - 1] * pprev));
    int sn = pn > 0.0 ? 1 : (pn < 0.0 ? -1 : -s);
    cnt += (sn != s);
    pprev = p; p = pn; s = sn;
    double ap = fabs(p), aq = fabs(pprev);
    if (ap > 0x1p500) { p *= 0x1p-500; pprev *= 0x1p-500; }
    else if (ap < 0x1p-500 && aq < 0x1p-500) { p *= 0x1p500; pprev *= 0x1p500; }
  }
  return cnt;
}

static double o_pow2_of(double a) { /* 2^floor(log2 a) for normal a > 0 (exact) */
  union { double f; uint64_t u; } b;
  b.f = a;
  b.u &= 0x7ff0000000000000ull;
  return b.f;
}

int oracle_tridiag_mineig(const double *om, const double *rho, int k, double *theta, double *s) {
  if (k <= 0) return -1;
  if (k == 1) { *theta = om[0]; s[0] = 1.0; return 0; }
  double *rho2 = (double *)malloc(sizeof(double) * (size_t)k * 8);
  double *u0 = rho2 + k, *u1 = u0 + k, *u2 = u1 + k, *mul = u2 + k, *x = mul + k;
  int *swp = (int *)malloc(sizeof(int) * (size_t)k);
  double lo = 0.0, hi = 0.0, NT = 0.0;
  for (int j = 0; j < k - 1; ++j) rho2[j] = rho[j] * rho[j];
  for (int j = 0; j < k; ++j) {
    double rl = j > 0 ? rho[j - 1] : 0.0;
    double rr = j < k - 1 ? rho[j] : 0.0;
    double rj = rl + rr;
    double a = om[j] - rj, b = om[j] + rj;
    if (j == 0 || a < lo) lo = a;
    if (j == 0 || b > hi) hi = b;
  }
  NT = fabs(lo) > fabs(hi) ? fabs(lo) : fabs(hi);
  if (NT == 0.0) {
    *theta = 0.0;
    for (int j = 0; j < k; ++j) s[j] = j == 0 ? 1.0 : 0.0;
    free(rho2); free(swp);
    return 0;
  }
  double pad = NT * 0x1p-20;
  lo = lo - pad;
  hi = hi + pad;
  /* 12 rounds of 32-point multisection: keep count(lo) = 0, count(hi) >= 1 */
  for (int round = 0; round < 12; ++round) {
    double h = (hi - lo) / 33.0;
    double prev = lo;
    double nlo = lo, nhi = hi;
    int found = 0;
    for (int j = 1; j <= 32; ++j) {
      double x = fma((double)j, h, lo);
      if (o_sturm(om, rho2, k, x) >= 1) { nlo = prev; nhi = x; found = 1; break; }
      prev = x;
    }
    if (!found) nlo = prev;
    lo = nlo; hi = nhi;
  }
  double th = (lo + hi) * 0.5;
  *theta = th;
  /* inverse iteration: Gaussian elimination with partial pivoting of T - theta I
   * (rows swapped when the sub-diagonal entry is larger), U has three diagonals. */
  double tiny = NT * 0x1p-60;
  double c0 = om[0] - th, c1 = k > 1 ? rho[0] : 0.0, c2 = 0.0;
  for (int i = 0; i < k - 1; ++i) {
    double nb = rho[i], na = om[i + 1] - th, nc = (i + 1 < k - 1) ? rho[i + 1] : 0.0;
    if (fabs(c0) >= fabs(nb)) {
      double m = c0 != 0.0 ? nb / c0 : 0.0;
      u0[i] = c0; u1[i] = c1; u2[i] = c2; swp[i] = 0; mul[i] = m;
      c0 = na - m * c1; c1 = nc - m * c2; c2 = 0.0;
    } else {
      double m = c0 / nb;
      u0[i] = nb; u1[i] = na; u2[i] = nc; swp[i] = 1; mul[i] = m;
      double t0 = c1 - m * na, t1 = c2 - m * nc;
      c0 = t0; c1 = t1; c2 = 0.0;
    }
  }
  u0[k - 1] = c0; u1[k - 1] = 0.0; u2[k - 1] = 0.0;
  for (int i = 0; i < k; ++i)
    if (fabs(u0[i]) < tiny) u0[i] = u0[i] < 0.0 ? -tiny : tiny;
  for (int j = 0; j < k; ++j) s[j] = (double)(j % 5 + 1) * 0.25;
  for (int it = 0; it < 3; ++it) {
    for (int j = 0; j < k; ++j) x[j] = s[j];
    for (int i = 0; i < k - 1; ++i) {
      if (swp[i]) { double t = x[i]; x[i] = x[i + 1]; x[i + 1] = t; }
      x[i + 1] = fma(-mul[i], x[i], x[i + 1]);
    }
    for (int i = k - 1; i >= 0; --i) {
      double t = x[i];
      if (i + 1 < k) t = fma(-u1[i], x[i + 1], t);
      if (i + 2 < k) t = fma(-u2[i], x[i + 2], t);
      x[i] = t / u0[i];
    }
    double mx = 0.0;
    for (int j = 0; j < k; ++j) if (fabs(x[j]) > mx) mx = fabs(x[j]);
    double sc = 1.0 / o_pow2_of(mx); /* exact power of two */
    for (int j = 0; j < k; ++j) s[j] = x[j] * sc;
  }
  int jm = 0;
  for (int j = 1; j < k; ++j) if (fabs(s[j]) > fabs(s[jm])) jm = j;
  if (s[jm] < 0.0) for (int j = 0; j < k; ++j) s[j] = -s[j];
  free(rho2); free(swp);
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Alg. 2 ApproxMinEvec, two passes.
 * g: the randn start vector of line 1; q: the iteration bound (callers pass
 * min{q_t, n-1}, line 3; there is no other cap).  Outputs theta (xi of line 12 = Ritz
 * value), v (line 13, explicitly normalized: reading A6), k, omega[k], rho[k-1].
 * div_norm = 0: a normalization "v / rho" is evaluated as v * fl(1/rho) (reading R26, the
 * contract the GPU path shares); div_norm = 1: as the printed division v / rho per entry
 * (tests pin R26 against this literal form). */
typedef struct {
  double theta;
  int k;
  int err;
  double *omega, *rho, *svec; /* q entries each */
} o_lanczos_res;

static void o_res_alloc(o_lanczos_res *res, int q) {
  memset(res, 0, sizeof(*res));
  res->omega = (double *)calloc((size_t)q + 1, sizeof(double));
  res->rho = (double *)calloc((size_t)q + 1, sizeof(double));
  res->svec = (double *)calloc((size_t)q + 1, sizeof(double));
}
static void o_res_free(o_lanczos_res *res) { free(res->omega); free(res->rho); free(res->svec); }

/* v[r] / rho for the chosen normalization form */
#define O_NORM(v, rho, rrho, div_norm) ((div_norm) ? (v) / (rho) : (v) * (rrho))

static void o_lanczos(const o_off *A, const double *d, const double *g, int q, double *v,
                      double *w1, double *w2, double *w3, double *a, o_lanczos_res *res, int div_norm) {
  int64_t n = A->n;
  int err = 0;
  double *vprev = w1, *vcur = w2, *vnext = w3;
  /* lines 1-2: v1 = randn / ||randn|| */
  double nu0 = sqrt(o_dot(g, g, n, &err));
  double rnu0 = 1.0 / nu0;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) vcur[r] = O_NORM(g[r], nu0, rnu0, div_norm);
  int k = q;
  for (int i = 1; i <= q; ++i) {
    o_apply(A, d, vcur, a);                            /* M v_i */
    res->omega[i - 1] = o_dot(vcur, a, n, &err);       /* line 5 */
    if (i == q) { k = q; break; }                       /* reading A2: last step needs no v_{i+1} */
    double om = res->omega[i - 1];
    double rp = i >= 2 ? res->rho[i - 2] : 0.0;
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) {                   /* line 6: three-term recurrence */
      double w = fma(-om, vcur[r], a[r]);
      if (i >= 2) w = fma(-rp, vprev[r], w);
      vnext[r] = w;
    }
    double rho = sqrt(o_dot(vnext, vnext, n, &err));    /* line 7 (reading A1) */
    res->rho[i - 1] = rho;
    if (rho <= 0x1p-45 * (fabs(om) + rp)) { k = i; break; } /* line 8 (reading A3) */
    double rrho = 1.0 / rho;
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) vnext[r] = O_NORM(vnext[r], rho, rrho, div_norm); /* line 9 */
    double *t = vprev; vprev = vcur; vcur = vnext; vnext = t;
  }
  res->k = k;
  /* lines 11-12 */
  oracle_tridiag_mineig(res->omega, res->rho, k, &res->theta, res->svec);
  /* line 13, regenerating v_2..v_k (second pass) */
  vprev = w1; vcur = w2; vnext = w3;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) {
    vcur[r] = O_NORM(g[r], nu0, rnu0, div_norm);
    v[r] = res->svec[0] * vcur[r];
  }
  for (int i = 1; i < k; ++i) {
    o_apply(A, d, vcur, a);
    double om = res->omega[i - 1];
    double rp = i >= 2 ? res->rho[i - 2] : 0.0;
    double rho = res->rho[i - 1];
    double rrho = 1.0 / rho;
    double si = res->svec[i];
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) {
      double w = fma(-om, vcur[r], a[r]);
      if (i >= 2) w = fma(-rp, vprev[r], w);
      vnext[r] = O_NORM(w, rho, rrho, div_norm);
      v[r] = fma(si, vnext[r], v[r]);
    }
    double *t = vprev; vprev = vcur; vcur = vnext; vnext = t;
  }
  double nx = sqrt(o_dot(v, v, n, &err));
  double rnx = 1.0 / nx;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) v[r] = O_NORM(v[r], nx, rnx, div_norm);
  res->err = err;
}

/* Standalone Alg. 2 on a general symmetric matrix (tests): offdiag CSR + diagonal d. */
int oracle_lanczos(int64_t n, const int64_t *rp, const int32_t *col, const double *m, const double *d,
                   const double *g, int q, double *v, double *theta, int *k, double *omega, double *rho,
                   double *svec) {
  if (q < 1) return -1;
  o_off A = {n, rp, col, m};
  double *buf = (double *)malloc(sizeof(double) * (size_t)n * 4);
  o_lanczos_res res;
  o_res_alloc(&res, q);
  o_lanczos(&A, d, g, q, v, buf, buf + n, buf + 2 * n, buf + 3 * n, &res, 0);
  free(buf);
  *theta = res.theta;
  *k = res.k;
  for (int j = 0; j < res.k; ++j) { omega[j] = res.omega[j]; svec[j] = res.svec[j]; }
  for (int j = 0; j + 1 < res.k; ++j) rho[j] = res.rho[j];
  int rc = res.err ? -2 : 0;
  o_res_free(&res);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* CAC-6 schedules (Alg. 4 lines 5-6). */
int oracle_qt(int64_t t, int64_t n) {
  double lnN = log((double)n);
  double x = sqrt(sqrt((double)t)) * lnN;
  int64_t q = (int64_t)ceil(x);
  if (q < 2) q = 2;
  if (q > n - 1) q = n - 1;
  return (int)q;
}

/* Dual step size, eqn:sketchy-cgal-dual-step, ||A|| = 1 for diag. */
double oracle_gamma(int64_t t, double alpha, double beta0, double nz) {
  if (nz == 0.0) return beta0;
  double sq = sqrt((double)(t + 1));
  double num = 4.0 * alpha;
  num = num * alpha;
  num = num * beta0;
  double den = ((double)(t + 1) * sq) * nz;
  double g = num / den;
  return g < beta0 ? g : beta0;
}

/* ------------------------------------------------------------------------- */
/* Alg. 4 SketchyCGAL for the MaxCut SDP. */
#define O_LOGW 12 /* t, q, k, theta, xi, c, p, ||z-b||, gamma, tau, gap, bound */
typedef struct {
  int64_t n;
  int32_t R;
  double alpha_orig, alpha, beta0, bval, nrmL;
  int scale;
  int trace_le; /* tr X <= alpha: H = alpha v v* if xi < 0, else 0 */
  int ineq;     /* general template with a box K = {lo <= u <= hi} */
  double lo, hi; /* scaled units; bit 1 of the mode (SCG_INEQ): lo = -inf, hi = b */
  int div_norm; /* bit 2 of the mode: normalizations as printed divisions (R26 pin, see o_lanczos) */
  int ball;      /* K = {u : ||u - b|| <= delta} (norm constraint): 1 l2 (R34), 2 l1 (R35) */
  double delta;  /* scaled units */
  double *pw, *pe; /* projection work arrays */
  uint64_t seed;
  int qfix; /* test-only: fixed Lanczos bound (may be n); 0 = schedule */
  int64_t t; /* iterations done */
  /* off-diagonal part of C and its diagonal (scaled) */
  int64_t *rp;
  int32_t *col;
  double *m;
  double *cdiag;
  double *z, *y, *S, *Omega, *v, *g, *d;
  double *ones; /* all-ones vector: xsum(y) = dot(y, 1) exactly */
  double *w1, *w2, *w3, *a, *cv;
  double p, tau;
  int err;
  /* per-iteration log */
  int64_t logcap;
  double *log; /* 10 per iteration: t q k theta xi c p znorm gamma tau */
  double *vhist; /* optional: T x n */
  int64_t vhist_cap;
} oracle_t;

void *oracle_create(int64_t n, const int64_t *rp_L, const int32_t *col_L, const double *val_L, int32_t R,
                    double alpha, double beta0, uint64_t seed, int scale, int qfix, int64_t logcap,
                    int64_t vhist_cap, int trace_le) {
  oracle_t *o = (oracle_t *)calloc(1, sizeof(oracle_t));
  o->n = n; o->R = R; o->beta0 = beta0; o->seed = seed; o->scale = scale; o->qfix = qfix;
  o->trace_le = trace_le & 1;      /* bit 0: trace-bounded set */
  o->ineq = (trace_le >> 1) & 1;    /* bit 1: inequality constraints A X <= b */
  o->div_norm = (trace_le >> 2) & 1; /* bit 2: literal division v / rho (test-only, reading R26) */
  o->alpha_orig = alpha;
  /* ||C||_F = ||L||_F over all stored entries (CAC-2), scaling P:1805-1814 (reading A13) */
  int err = 0;
  {
    xsum_t s;
    xs_init(&s);
    for (int64_t k = 0; k < rp_L[n]; ++k) xs_add(&s, val_L[k] * val_L[k]);
    err |= s.err;
    o->nrmL = sqrt(xs_round(&s));
  }
  if (scale) { o->alpha = alpha / (double)n; o->bval = 1.0 / (double)n; } /* X~ = X / n (A13) */
  else { o->alpha = alpha; o->bval = 1.0; }
  o->lo = -INFINITY;
  o->hi = o->bval;
  /* split L into off-diagonal C entries and diagonal: C = -L, scaled C / ||C||_F */
  int64_t nnz_off = 0;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t k = rp_L[r]; k < rp_L[r + 1]; ++k) if (col_L[k] != r) nnz_off++;
  o->rp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  o->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz_off ? nnz_off : 1));
  o->m = (double *)malloc(sizeof(double) * (size_t)(nnz_off ? nnz_off : 1));
  o->cdiag = (double *)calloc((size_t)n, sizeof(double));
  int64_t o_k = 0;
  o->rp[0] = 0;
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t k = rp_L[r]; k < rp_L[r + 1]; ++k) {
      double c = -val_L[k];
      if (scale) c = c / o->nrmL;
      if (col_L[k] == r) o->cdiag[r] = c;
      else { o->col[o_k] = col_L[k]; o->m[o_k] = c; o_k++; }
    }
    o->rp[r + 1] = o_k;
  }
  o->z = (double *)calloc((size_t)n, sizeof(double));
  o->ones = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) o->ones[i] = 1.0;
  o->y = (double *)calloc((size_t)n, sizeof(double));
  o->d = (double *)calloc((size_t)n, sizeof(double));
  o->v = (double *)calloc((size_t)n, sizeof(double));
  o->g = (double *)calloc((size_t)n, sizeof(double));
  o->w1 = (double *)calloc((size_t)n, sizeof(double));
  o->w2 = (double *)calloc((size_t)n, sizeof(double));
  o->w3 = (double *)calloc((size_t)n, sizeof(double));
  o->a = (double *)calloc((size_t)n, sizeof(double));
  o->cv = (double *)calloc((size_t)n, sizeof(double));
  o->pw = (double *)calloc((size_t)n, sizeof(double));
  o->pe = (double *)calloc((size_t)n, sizeof(double));
  o->S = (double *)calloc((size_t)n * R, sizeof(double));
  o->Omega = (double *)malloc(sizeof(double) * (size_t)n * R);
  /* NystromSketch.Init (Alg. 3 line 2): Omega column-major, reading A8 */
  for (int32_t kk = 0; kk < R; ++kk)
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t i = 0; i < n; ++i) o->Omega[(int64_t)kk * n + i] = scg_omega(seed, i, kk);
  o->logcap = logcap;
  o->log = (double *)calloc((size_t)(logcap > 0 ? logcap : 1) * O_LOGW, sizeof(double));
  o->vhist_cap = vhist_cap;
  o->vhist = vhist_cap > 0 ? (double *)calloc((size_t)vhist_cap * n, sizeof(double)) : NULL;
  o->err = err;
  return o;
}

void oracle_destroy(void *h) {
  oracle_t *o = (oracle_t *)h;
  if (!o) return;
  free(o->rp); free(o->col); free(o->m); free(o->cdiag);
  free(o->z); free(o->y); free(o->d); free(o->v); free(o->g);
  free(o->w1); free(o->w2); free(o->w3); free(o->a); free(o->cv);
  free(o->S); free(o->Omega); free(o->log); free(o->vhist); free(o->ones); free(o->pw); free(o->pe);
  free(o);
}

/* The exact value S - c a - delta, rounded once (its sign is exact): S an exact sum, c a an exact
 * product by the error-free transformation hi = fl(c a), lo = fma(c, a, -hi) (CAC-2 summands). */
static double o_l1_g(const xsum_t *S, double c, double a, double delta) {
  xsum_t g = *S;
  const double hi = c * a, lo = fma(c, a, -hi);
  xs_add(&g, -hi);
  xs_add(&g, -lo);
  xs_add(&g, -delta);
  return xs_round(&g);
}

static int o_desc(const void *x, const void *y) {
  const double a = *(const double *)x, b = *(const double *)y;
  return a < b ? 1 : (a > b ? -1 : 0);
}

/* Euclidean projection onto the l1 ball {||u - b||_1 <= delta} (reading R35), in place on
 * the points w = p:  e_r = fl(p_r - b), a_r = |e_r|.
 *   sum_r a_r - delta <= 0 (exact): w = p (already in K).  Else delta = 0: w = b.
 *   Else soft thresholding w_r = fl(b + sign(e_r) max(fl(a_r - theta), 0)) with the threshold of the
 *   sorted a_(1) >= a_(2) >= ... : rho = max{j : S_j - j a_(j) - delta < 0} (S_j = a_(1) + ... + a_(j),
 *   decided exactly; S_j - j a_(j) grows with j), theta = fl(fl(S_rho - delta) / rho) (S_rho - delta
 *   summed exactly, rounded once). */
static void o_proj_l1(oracle_t *o, double *w, int *err) {
  const int64_t n = o->n;
  double *e = o->pe;
  double *a = (double *)malloc(sizeof(double) * (size_t)n);
  for (int64_t r = 0; r < n; ++r) {
    e[r] = w[r] - o->bval;
    a[r] = fabs(e[r]);
  }
  xsum_t S;
  xs_init(&S);
  for (int64_t r = 0; r < n; ++r) xs_add(&S, a[r]);
  if (S.err && err) *err = 1;
  if (o_l1_g(&S, 0.0, 0.0, o->delta) <= 0.0) { /* inside: w = p */
    free(a);
    return;
  }
  if (o->delta == 0.0) {
    for (int64_t r = 0; r < n; ++r) w[r] = o->bval;
    free(a);
    return;
  }
  qsort(a, (size_t)n, sizeof(double), o_desc);
  xs_init(&S);
  xsum_t Srho;
  int64_t rho = 0;
  for (int64_t j = 1; j <= n; ++j) {
    xs_add(&S, a[j - 1]);
    if (!(o_l1_g(&S, (double)j, a[j - 1], o->delta) < 0.0)) break;
    rho = j;
    Srho = S;
  }
  /* rho >= 1: S_1 - a_(1) - delta = -delta < 0 */
  const double theta = o_l1_g(&Srho, 0.0, 0.0, o->delta) / (double)rho;
  for (int64_t r = 0; r < n; ++r) w[r] = o->bval + copysign(fmax(fabs(e[r]) - theta, 0.0), e[r]);
  free(a);
}

/* Projection onto K of the points p_r = fl(z_r + fl(y_r / beta)), into w.
 *   box K = {lo <= u <= hi}: w_r = min(max(p_r, lo), hi) (reading R32);
 *   l2 ball K = {||u - b|| <= delta}: e_r = fl(p_r - b), N = sqrt(xsum(e^2)) (exact sum, CAC-2);
 *     N <= delta: w = p (already in K); else w_r = fl(b + fl(s e_r)), s = fl(delta / N) (reading R34). */
static void o_proj(oracle_t *o, const double *z, const double *y, double beta, double *w, int *err) {
  const int64_t n = o->n;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) w[r] = z[r] + y[r] / beta;
  if (!o->ball) {
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) w[r] = fmin(fmax(w[r], o->lo), o->hi);
    return;
  }
  if (o->ball == 2) {
    o_proj_l1(o, w, err);
    return;
  }
  double *e = o->pe;
#pragma omp parallel for schedule(static) if (n > 65536)
  for (int64_t r = 0; r < n; ++r) e[r] = w[r] - o->bval;
  const double N = sqrt(o_dot(e, e, n, err));
  if (N > o->delta) {
    const double s = o->delta / N;
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) w[r] = o->bval + s * e[r];
  }
}

/* l2 ball K = {||u - 1|| <= delta} in original units (norm constraint); before the first
 * step.  (Scaled units: delta / n, like b = 1/n.) */
int oracle_set_ball(void *h, double delta) {
  oracle_t *o = (oracle_t *)h;
  if (o->t != 0 || !(delta >= 0.0)) return -1;
  o->ineq = 1;
  o->ball = 1;
  o->delta = o->scale ? delta / (double)o->n : delta;
  return 0;
}

/* proj_K(z + y / beta) of the constraint set in effect, scaled units (test access to o_proj). */
int oracle_proj(void *h, const double *z, const double *y, double beta, double *w) {
  oracle_t *o = (oracle_t *)h;
  int err = 0;
  if (!o->ineq) return -1;
  o_proj(o, z, y, beta, w, &err);
  return err ? -2 : 0;
}

/* l1 ball K = {||u - 1||_1 <= delta} in original units (reading R35); before the first
 * step.  (Scaled units: delta / n.) */
int oracle_set_l1_ball(void *h, double delta) {
  oracle_t *o = (oracle_t *)h;
  if (o->t != 0 || !(delta >= 0.0)) return -1;
  o->ineq = 1;
  o->ball = 2;
  o->delta = o->scale ? delta / (double)o->n : delta;
  return 0;
}

/* Box K = {lo <= u <= hi} in original units; before the first step. */
int oracle_set_box(void *h, double lo, double hi) {
  oracle_t *o = (oracle_t *)h;
  if (o->t != 0 || !(lo <= hi)) return -1;
  o->ineq = 1;
  o->lo = o->scale ? lo / (double)o->n : lo;
  o->hi = o->scale ? hi / (double)o->n : hi;
  return 0;
}

int oracle_step(void *h, int64_t T) {
  oracle_t *o = (oracle_t *)h;
  int64_t n = o->n;
  o_off A = {n, o->rp, o->col, o->m};
  int R = o->R;
  for (int64_t it = 0; it < T; ++it) {
    int64_t t = o->t + 1;
    /* line 5: beta = beta0 sqrt(t+1), eta = 2/(t+1) */
    double sq = sqrt((double)(t + 1));
    double beta = o->beta0 * sq;
    double eta = 2.0 / (double)(t + 1);
    int q = o->qfix > 0 ? o->qfix : oracle_qt(t, n);
    if (o->qfix <= 0 && q > n - 1) q = (int)(n - 1);
    /* Surrogate duality gap g_t(X_t) (eqn:cgal-gap, as P:1550-1554) and the
     * posterior suboptimality bound (eqn:scgal-posterior-error-bd), which is
     * also the numerator of the stopping rule:
     *   gap   = p_t + <y_t, z_t> + beta_t <z_t - b, z_t> - alpha lambda_min(D_t)
     *   bound = p_t + <y_t, b> + beta_t/2 <z_t - b, z_t + b> - alpha lambda_min(D_t)
     * with lambda_min(D_t) ~ xi_t (reading A22 puts alpha in front), the inner
     * products from exact sums of the state before this iteration's update, evaluated in
     * the order written in DESIGN.md CAC-6.  xi_t is known after the monitor below. */
    int gerr = 0;
    const double S_y = o_dot(o->y, o->ones, n, &gerr);
    const double S_yz = o_dot(o->y, o->z, n, &gerr);
    const double S_zz = o_dot(o->z, o->z, n, &gerr);
    const double S_z = o_dot(o->z, o->ones, n, &gerr);
    /* General template (A X in K): the same two quantities with the slack w_t = proj_K(z_t + y_t /
     * beta_t) in place of b (reading R33): f_t(X) = <C, X> + min_{w in K} <y, A X - w> +
     * beta/2 ||A X - w||^2 is convex with gradient D_t and f_t(X_star) <= p_star, so the derivation of
     * P:3100-3140 gives
     *   gap   = p_t + <y_t, z_t> + beta_t <z_t - w_t, z_t> - alpha xi_t
     *   bound = p_t + <y_t, w_t> + beta_t/2 <z_t - w_t, z_t + w_t> - alpha xi_t
     * (w_t = b gives the equality formulas above) */
    double S_ez = 0.0, S_yw = 0.0, S_ezw = 0.0;
    double *wt = o->cv; /* w_t = proj_K(z_t + y_t / beta_t) (general template); free until the monitor */
    if (o->ineq) {
      double *e = o->a, *zw = o->w1; /* free until the Lanczos call below */
      o_proj(o, o->z, o->y, beta, wt, &gerr);
#pragma omp parallel for schedule(static) if (n > 65536)
      for (int64_t r = 0; r < n; ++r) {
        e[r] = o->z[r] - wt[r];
        zw[r] = o->z[r] + wt[r];
      }
      S_ez = o_dot(e, o->z, n, &gerr);
      S_yw = o_dot(o->y, wt, n, &gerr);
      S_ezw = o_dot(e, zw, n, &gerr);
    }
    const double p_t = o->p;
    o->err |= gerr;
    /* line 6: D = C + A*(y + beta (z - b)) ; diagonal of D (primitive 2).
     * General template, K = {u <= b}: b is replaced by the slack
     * w_t = proj_K(z_t + y_t / beta_t) = min(max(z_t + y_t / beta_t, lo), hi), elementwise (R32). */
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) {
      const double wr = o->ineq ? wt[r] : o->bval;
      o->d[r] = fma(beta, o->z[r] - wr, o->y[r]) + o->cdiag[r];
      o->g[r] = scg_lanczos_start(o->seed, t, r);
    }
    o_lanczos_res res;
    o_res_alloc(&res, q);
    o_lanczos(&A, o->d, o->g, q, o->v, o->w1, o->w2, o->w3, o->a, &res, o->div_norm);
    o->err |= res.err;
    /* monitors: xi = v* D v (eqn 5.1), c = v* C v (p update) */
    int err = 0;
    o_apply(&A, o->d, o->v, o->a);
    double xi = o_dot(o->v, o->a, n, &err);
    o_apply(&A, o->cdiag, o->v, o->cv);
    double cval = o_dot(o->v, o->cv, n, &err);
    double one_m_eta = 1.0 - eta;
    /* LMO: H = alpha v v*; for the trace-bounded set tr X <= alpha, H = 0 when xi >= 0
     * (xi is the Rayleigh quotient approximating lambda_min) */
    const int hoff = o->trace_le && !(xi < 0.0);
    /* line 7: z <- (1 - eta) z + eta A(H)  (primitive 3) */
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) {
      double h = o->alpha * (o->v[r] * o->v[r]);
      o->z[r] = hoff ? one_m_eta * o->z[r] : fma(eta, h, one_m_eta * o->z[r]);
    }
    /* line 8: gamma from ||z - b||^2, y <- y + gamma (z - b).  General template:
     * b is replaced by wbar_t = proj_K(z_{t+1} + y_t / beta_{t+1}) and the step rule keeps the
     * form gamma ||z - wbar||^2 <= beta_t eta_t^2 alpha^2 ||A||^2 (reading R32). */
    const double beta1 = o->beta0 * sqrt((double)(t + 2));
    if (o->ineq) o_proj(o, o->z, o->y, beta1, o->pw, &err);
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) {
      const double wb = o->ineq ? o->pw[r] : o->bval;
      o->a[r] = o->z[r] - wb;
    }
    double nz = o_dot(o->a, o->a, n, &err);
    double gamma = oracle_gamma(t, o->alpha, o->beta0, nz);
#pragma omp parallel for schedule(static) if (n > 65536)
    for (int64_t r = 0; r < n; ++r) o->y[r] = fma(gamma, o->a[r], o->y[r]);
    /* line 9: NystromSketch.RankOneUpdate(sqrt(alpha) v, eta): S <- (1-eta) S + eta alpha v (v* Omega) */
    for (int kk = 0; kk < R; ++kk) {
      double gk = o_dot(o->v, o->Omega + (int64_t)kk * n, n, &err);
      double c = hoff ? 0.0 : (eta * o->alpha) * gk;
      double *Sk = o->S + (int64_t)kk * n;
#pragma omp parallel for schedule(static) if (n > 65536)
      for (int64_t r = 0; r < n; ++r) Sk[r] = fma(c, o->v[r], one_m_eta * Sk[r]);
    }
    /* tau, p */
    double vv = o_dot(o->v, o->v, n, &err);
    if (hoff) {
      o->tau = one_m_eta * o->tau;
      o->p = one_m_eta * o->p;
    } else {
      o->tau = fma(eta * o->alpha, vv, one_m_eta * o->tau);
      o->p = fma(eta * o->alpha, cval, one_m_eta * o->p);
    }
    o->err |= err;
    if (t - 1 < o->logcap) {
      double *L = o->log + (t - 1) * O_LOGW;
      L[0] = (double)t; L[1] = (double)q; L[2] = (double)res.k; L[3] = res.theta; L[4] = xi;
      L[5] = cval; L[6] = o->p; L[7] = sqrt(nz); L[8] = gamma; L[9] = o->tau;
      /* min over the set of <D, H>: alpha xi (tr X = alpha) or alpha min(xi, 0) (tr X <= alpha) */
      const double ax = o->alpha * ((o->trace_le && xi > 0.0) ? 0.0 : xi);
      const double nbb = ((double)n * o->bval) * o->bval;
      if (o->ineq) { /* general template (reading R33) */
        L[10] = ((p_t + S_yz) + beta * S_ez) - ax;
        L[11] = ((p_t + S_yw) + (0.5 * beta) * S_ezw) - ax;
      } else {
        L[10] = ((p_t + S_yz) + beta * (S_zz - o->bval * S_z)) - ax;
        L[11] = ((p_t + o->bval * S_y) + (0.5 * beta) * (S_zz - nbb)) - ax;
      }
    }
    if (o->vhist && t - 1 < o->vhist_cap) memcpy(o->vhist + (t - 1) * n, o->v, sizeof(double) * (size_t)n);
    o_res_free(&res);
    o->t = t;
  }
  return o->err ? -2 : 0;
}

/* getters */
int64_t oracle_t_done(void *h) { return ((oracle_t *)h)->t; }
double oracle_scalar(void *h, int which) {
  oracle_t *o = (oracle_t *)h;
  switch (which) {
    case 0: return o->p;
    case 1: return o->tau;
    case 2: return o->nrmL;
    case 3: return o->alpha;
    case 4: return o->bval;
    default: return NAN;
  }
}
void oracle_get(void *h, int which, double *out) {
  oracle_t *o = (oracle_t *)h;
  int64_t n = o->n;
  switch (which) {
    case 0: memcpy(out, o->z, sizeof(double) * (size_t)n); break;
    case 1: memcpy(out, o->y, sizeof(double) * (size_t)n); break;
    case 2: memcpy(out, o->S, sizeof(double) * (size_t)n * o->R); break;
    case 3: memcpy(out, o->Omega, sizeof(double) * (size_t)n * o->R); break;
    case 4: memcpy(out, o->v, sizeof(double) * (size_t)n); break;
    case 5: memcpy(out, o->log, sizeof(double) * (size_t)o->logcap * O_LOGW); break;
    case 6: if (o->vhist) memcpy(out, o->vhist, sizeof(double) * (size_t)o->vhist_cap * n); break;
    case 7: memcpy(out, o->cdiag, sizeof(double) * (size_t)n); break;
    case 8: memcpy(out, o->d, sizeof(double) * (size_t)n); break;
    default: break;
  }
}
