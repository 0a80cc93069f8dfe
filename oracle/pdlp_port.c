/*
 * pdlp_port.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference PDLP path (see pdlp_port.h).  Each function names the reference
 * lines it follows; arithmetic order is the reference's, expression by
 * expression, so results are bit-identical on x86-64 without FMA.
 */
#define _POSIX_C_SOURCE 200809L
#include "pdlp_port.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

#define TRY(expr)            \
  do {                       \
    int rc_ = (expr);        \
    if (rc_ != FOLP_OK) return rc_; \
  } while (0)

static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */

/* ------------------------------------------------------- summation order
 * g_order selects how scalar reductions are folded.  0 (default) is the
 * reference's sequential fold, bit-identical to the compiled reference.  The
 * other orders exist ONLY to measure the reference's own reduction-order
 * noise floor (tests/test_noise_floor.py, tools/noise_floor.py): same
 * algorithm, same per-element terms, only the association of the sums
 * changes, exactly what any parallel implementation must do.
 *   1  pairwise tree over the terms (leaves of 8, sequential inside)
 *   2  reversed sequential fold
 *   3  like 1, and segment dots longer than 256 entries (K x rows / K'y
 *      columns) summed as 256-entry sequential parts whose sums are then
 *      folded in part order (a warp/part split of long segments)
 */
static int g_order = 0;

static double psum(const double* t, int64_t n) {
  if (n <= 8) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += t[i];
    return s;
  }
  const int64_t h = n / 2;
  return psum(t, h) + psum(t + h, n - h);
}

/* Fold of n terms t[i] in the order g_order selects (t is scratch). */
static double fold(const double* t, int64_t n) {
  if (g_order == 1 || g_order == 3) return psum(t, n);
  double s = 0.0;
  if (g_order == 2) {
    for (int64_t i = n - 1; i >= 0; --i) s += t[i];
  } else {
    for (int64_t i = 0; i < n; ++i) s += t[i];
  }
  return s;
}

void folp_port_set_sum_order(int order) { g_order = order; }

/* ---------------------------------------------------------------- mt19937_64 */
typedef struct {
  uint64_t mt[312];
  int idx;
} Mt64;

static void mt_seed(Mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

static uint64_t mt_next(Mt64* g) {
  static const uint64_t mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
  if (g->idx >= 312) {
    int i;
    uint64_t x;
    for (i = 0; i < 312 - 156; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
      g->mt[i] = g->mt[i + 156] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    for (; i < 311; ++i) {
      x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[i + 1] & 0x7FFFFFFFULL);
      g->mt[i] = g->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1ULL];
    }
    x = (g->mt[311] & 0xFFFFFFFF80000000ULL) | (g->mt[0] & 0x7FFFFFFFULL);
    g->mt[311] = g->mt[155] ^ (x >> 1) ^ mag[x & 1ULL];
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* ---------------------------------------------------------------- problem */
typedef struct {
  int64_t m, n, m1, nnz;
  int64_t *rs, *rc, *cs, *cr;
  double *rv, *cv;
  double *c, *q, *l, *u;
  double cst;
} Lp;

static void* xmalloc(size_t bytes) {
  void* p = malloc(bytes ? bytes : 1);
  if (!p) {
    fprintf(stderr, "pdlp_port: out of memory\n");
    abort();
  }
  return p;
}

static double* dvec(int64_t n) { return (double*)xmalloc((size_t)n * sizeof(double)); }
static double* dzero(int64_t n) { return (double*)calloc((size_t)(n ? n : 1), sizeof(double)); }
static double* dcopy(const double* s, int64_t n) {
  double* d = dvec(n);
  if (n) memcpy(d, s, (size_t)n * sizeof(double));
  return d;
}

/* Column mirror by a counting pass (sparse_matrix.cpp:82-102). */
static void build_csc(Lp* p) {
  p->cs = (int64_t*)calloc((size_t)p->n + 1, sizeof(int64_t));
  p->cr = (int64_t*)xmalloc((size_t)p->nnz * sizeof(int64_t));
  p->cv = dvec(p->nnz);
  for (int64_t k = 0; k < p->nnz; ++k) p->cs[p->rc[k] + 1]++;
  for (int64_t c = 0; c < p->n; ++c) p->cs[c + 1] += p->cs[c];
  int64_t* cur = (int64_t*)xmalloc((size_t)(p->n + 1) * sizeof(int64_t));
  memcpy(cur, p->cs, (size_t)(p->n + 1) * sizeof(int64_t));
  for (int64_t r = 0; r < p->m; ++r) {
    for (int64_t k = p->rs[r]; k < p->rs[r + 1]; ++k) {
      int64_t slot = cur[p->rc[k]]++;
      p->cr[slot] = r;
      p->cv[slot] = p->rv[k];
    }
  }
  free(cur);
}

static int lp_load(const folp_lp_c* in, Lp* p) {
  memset(p, 0, sizeof *p);
  p->m = in->num_rows;
  p->n = in->num_cols;
  p->m1 = in->num_inequality_rows;
  p->nnz = in->nnz;
  for (int64_t r = 0; r < p->m; ++r) {
    for (int64_t k = in->row_start[r]; k < in->row_start[r + 1]; ++k) {
      if (in->row_values[k] == 0.0 || (k > in->row_start[r] && in->row_cols[k] <= in->row_cols[k - 1]))
        return fail(FOLP_E_INVALID_ARGUMENT, "port: CSR must be canonical (sorted, no zeros)");
    }
  }
  p->rs = (int64_t*)xmalloc((size_t)(p->m + 1) * sizeof(int64_t));
  memcpy(p->rs, in->row_start, (size_t)(p->m + 1) * sizeof(int64_t));
  p->rc = (int64_t*)xmalloc((size_t)(p->nnz ? p->nnz : 1) * sizeof(int64_t));
  if (p->nnz) memcpy(p->rc, in->row_cols, (size_t)p->nnz * sizeof(int64_t));
  p->rv = dcopy(in->row_values, p->nnz);
  p->c = dcopy(in->objective, p->n);
  p->q = dcopy(in->right_hand_side, p->m);
  p->l = dcopy(in->variable_lower, p->n);
  p->u = dcopy(in->variable_upper, p->n);
  p->cst = in->objective_constant;
  build_csc(p);
  return FOLP_OK;
}

static void lp_free(Lp* p) {
  free(p->rs); free(p->rc); free(p->rv); free(p->cs); free(p->cr); free(p->cv);
  free(p->c); free(p->q); free(p->l); free(p->u);
  memset(p, 0, sizeof *p);
}

/* sparse_matrix.cpp:106-119 */
static double seg_dot(const int64_t* idx, const double* val, int64_t b, int64_t e,
                      const double* v) {
  if (g_order == 3 && e - b > 256) {  /* 256-entry parts, part sums in order */
    double s = 0.0;
    for (int64_t p0 = b; p0 < e; p0 += 256) {
      double ps = 0.0;
      const int64_t p1 = p0 + 256 < e ? p0 + 256 : e;
      for (int64_t k = p0; k < p1; ++k) ps += val[k] * v[idx[k]];
      s += ps;
    }
    return s;
  }
  double s = 0.0;
  for (int64_t k = b; k < e; ++k) s += val[k] * v[idx[k]];
  return s;
}

static void kx(const Lp* p, const double* x, double* out) {
  for (int64_t r = 0; r < p->m; ++r) out[r] = seg_dot(p->rc, p->rv, p->rs[r], p->rs[r + 1], x);
}

/* sparse_matrix.cpp:127-140 */
static void kty(const Lp* p, const double* y, double* out) {
  for (int64_t c = 0; c < p->n; ++c) out[c] = seg_dot(p->cr, p->cv, p->cs[c], p->cs[c + 1], y);
}

/* linalg.hpp:25-60 */
static void* xmalloc(size_t bytes);
static double dot(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  if (g_order) {
    double* t = (double*)xmalloc((size_t)(n ? n : 1) * sizeof(double));
    for (int64_t i = 0; i < n; ++i) t[i] = a[i] * b[i];
    s = fold(t, n);
    free(t);
    return s;
  }
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nsq(const double* v, int64_t n) { return dot(v, v, n); }
static double dsq_folded(const double* a, const double* b, int64_t n) {
  double* t = (double*)xmalloc((size_t)(n ? n : 1) * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    const double d = a[i] - b[i];
    t[i] = d * d;
  }
  const double s = fold(t, n);
  free(t);
  return s;
}
static double dnorm(const double* a, const double* b, int64_t n) {
  double s = 0.0;
  if (g_order) return sqrt(dsq_folded(a, b, n));
  for (int64_t i = 0; i < n; ++i) {
    const double d = a[i] - b[i];
    s += d * d;
  }
  return sqrt(s);
}
static int finite_all(const double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* ---------------------------------------------------------------- scaling */
/* axis_norms (sparse_matrix.cpp:156-186) for one axis of a value array. */
static void axis_norms(const int64_t* start, const double* val, int64_t S, double p, double* out) {
  for (int64_t i = 0; i < S; ++i) {
    double acc = 0.0;
    for (int64_t k = start[i]; k < start[i + 1]; ++k) {
      const double a = fabs(val[k]);
      if (p == 0.0) acc += 1.0;
      else if (isinf(p)) acc = dmax(acc, a);
      else if (p == 1.0) acc += a;
      else if (p == 2.0) acc += a * a;
      else acc += pow(a, p);
    }
    if (p == 2.0) acc = sqrt(acc);
    else if (isfinite(p) && p > 1.0 && p != 2.0) acc = pow(acc, 1.0 / p);
    out[i] = acc;
  }
}

/* reciprocal_sqrt (scaling.cpp:23-28) */
static void recip_sqrt(double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) v[i] = v[i] > 0.0 ? 1.0 / sqrt(v[i]) : 1.0;
}

/* SparseMatrix::scaled (sparse_matrix.cpp:222-242) into dst value arrays. */
static void scale_values(const Lp* p, const double* srv, const double* scv, double* drv,
                         double* dcv, const double* rsc, const double* csc) {
  for (int64_t r = 0; r < p->m; ++r)
    for (int64_t k = p->rs[r]; k < p->rs[r + 1]; ++k) drv[k] = srv[k] * (rsc[r] * csc[p->rc[k]]);
  for (int64_t c = 0; c < p->n; ++c)
    for (int64_t k = p->cs[c]; k < p->cs[c + 1]; ++k) dcv[k] = scv[k] * (csc[c] * rsc[p->cr[k]]);
}

/* rescale_problem (scaling.cpp:48-96): fills w (sharing the structure of p)
 * and the cumulative diagonals. */
static int rescale(const Lp* p, int64_t ruiz, int pc, double alpha, Lp* w, double* d1,
                   double* d2) {
  if (pc) {
    if (!(alpha >= 0.0 && alpha <= 2.0))
      return fail(FOLP_E_INVALID_ARGUMENT, "pock_chambolle_step: alpha must be in [0,2]");
    const double ps[2] = {2.0 - alpha, alpha};
    for (int i = 0; i < 2; ++i)
      if (isnan(ps[i]) || (ps[i] < 1.0 && ps[i] != 0.0))
        return fail(FOLP_E_UNSUPPORTED_NORM, "axis_norms: p must be 0, in [1, inf), or +inf");
  }
  for (int64_t i = 0; i < p->m; ++i) d1[i] = 1.0;
  for (int64_t j = 0; j < p->n; ++j) d2[j] = 1.0;
  double* wr = dcopy(p->rv, p->nnz);
  double* wc = dcopy(p->cv, p->nnz);
  double* s1 = dvec(p->m);
  double* s2 = dvec(p->n);
  const int64_t steps = ruiz + (pc ? 1 : 0);
  for (int64_t it = 0; it < steps; ++it) {
    const int is_pc = it == ruiz;
    axis_norms(p->rs, wr, p->m, is_pc ? 2.0 - alpha : INFINITY, s1);
    axis_norms(p->cs, wc, p->n, is_pc ? alpha : INFINITY, s2);
    recip_sqrt(s1, p->m);
    recip_sqrt(s2, p->n);
    scale_values(p, wr, wc, wr, wc, s1, s2);
    for (int64_t i = 0; i < p->m; ++i) d1[i] *= s1[i];
    for (int64_t j = 0; j < p->n; ++j) d2[j] *= s2[j];
  }
  *w = *p;  /* structure shared, arrays below are new */
  w->rs = p->rs; w->rc = p->rc; w->cs = p->cs; w->cr = p->cr;
  w->rv = dvec(p->nnz);
  w->cv = dvec(p->nnz);
  scale_values(p, p->rv, p->cv, w->rv, w->cv, d1, d2);
  w->c = dvec(p->n); w->l = dvec(p->n); w->u = dvec(p->n); w->q = dvec(p->m);
  for (int64_t j = 0; j < p->n; ++j) {
    w->c[j] = p->c[j] * d2[j];
    w->l[j] = p->l[j] / d2[j];
    w->u[j] = p->u[j] / d2[j];
  }
  for (int64_t i = 0; i < p->m; ++i) w->q[i] = p->q[i] * d1[i];
  free(wr); free(wc); free(s1); free(s2);
  return FOLP_OK;
}

static void free_working(Lp* w) {
  free(w->rv); free(w->cv); free(w->c); free(w->l); free(w->u); free(w->q);
}

/* ---------------------------------------------------------------- KKT */
/* convergence_info (termination.cpp:23-73) */
static int conv_info(const Lp* p, const double* x, const double* y, folp_info_c* info) {
  if (!finite_all(x, p->n) || !finite_all(y, p->m))
    return fail(FOLP_E_NONFINITE, "convergence_info: point has NaN or inf entries");
  double* kxv = dvec(p->m);
  double* ktyv = dvec(p->n);
  double* res = dvec(p->n);
  double* lam = dvec(p->n);
  kx(p, x, kxv);
  kty(p, y, ktyv);
  info->primal_objective = dot(p->c, x, p->n) + p->cst;
  for (int64_t i = 0; i < p->n; ++i) res[i] = p->c[i] - ktyv[i];
  for (int64_t i = 0; i < p->n; ++i) { /* lp_model.cpp:129-148 */
    const int lo = p->l[i] > -INFINITY, hi = p->u[i] < INFINITY;
    lam[i] = (!lo && !hi) ? 0.0 : (!lo ? dmin(res[i], 0.0) : (!hi ? dmax(res[i], 0.0) : res[i]));
  }
  double v = dot(p->q, y, p->m) + p->cst; /* lp_model.cpp:150-165 */
  int bad = 0;
  for (int64_t i = 0; i < p->n; ++i) {
    if (lam[i] == 0.0) continue;
    const double b = lam[i] > 0.0 ? p->l[i] : p->u[i];
    if (!isfinite(b)) { bad = 1; break; }
    v += b * lam[i];
  }
  int rc = FOLP_OK;
  if (bad) {
    rc = fail(FOLP_E_INFINITE_PRODUCT, "dual_objective: lambda outside its sign cone");
  } else {
    info->dual_objective = v;
    info->gap_abs = fabs(info->dual_objective - info->primal_objective);
    double ps = 0.0;
    double* tt = g_order ? dvec(p->m > p->n ? p->m : p->n) : NULL;
    for (int64_t r = 0; r < p->m; ++r) {
      double t = p->q[r] - kxv[r];
      if (r < p->m1) t = dmax(t, 0.0);
      if (g_order) tt[r] = t * t; else ps += t * t;
    }
    if (g_order) ps = fold(tt, p->m);
    info->primal_residual_norm = sqrt(ps);
    double ds = 0.0;
    for (int64_t i = 0; i < p->n; ++i) {
      const double t = res[i] - lam[i];
      if (g_order) tt[i] = t * t; else ds += t * t;
    }
    if (g_order) ds = fold(tt, p->n);
    free(tt);
    info->dual_residual_norm = sqrt(ds);
    info->norm_q = sqrt(nsq(p->q, p->m));
    info->norm_c = sqrt(nsq(p->c, p->n));
  }
  free(kxv); free(ktyv); free(res); free(lam);
  return rc;
}

/* check_termination (termination.cpp:75-83) */
static int converged(const folp_info_c* i, double eps) {
  const int gap = i->gap_abs <= eps * (1.0 + fabs(i->dual_objective) + fabs(i->primal_objective));
  const int pr = i->primal_residual_norm <= eps * (1.0 + i->norm_q);
  const int du = i->dual_residual_norm <= eps * (1.0 + i->norm_c);
  return gap && pr && du;
}

/* normalized_duality_gap (solver.cpp:277-370) */
static double ndg(const Lp* p, const double* x, const double* y, double radius, double omega) {
  const int64_t n = p->n, m = p->m, tot = n + m;
  double* ktyv = dvec(n);
  double* kxv = dvec(m);
  kty(p, y, ktyv);
  kx(p, x, kxv);
  double *g = dvec(tot), *w = dvec(tot), *lo = dvec(tot), *hi = dvec(tot), *d = dvec(tot);
  for (int64_t i = 0; i < n; ++i) {
    g[i] = ktyv[i] - p->c[i];
    w[i] = omega;
    lo[i] = dmin(0.0, p->l[i] - x[i]);
    hi[i] = dmax(0.0, p->u[i] - x[i]);
  }
  for (int64_t j = 0; j < m; ++j) {
    g[n + j] = p->q[j] - kxv[j];
    w[n + j] = 1.0 / omega;
    lo[n + j] = j < p->m1 ? dmin(0.0, -y[j]) : -INFINITY;
    hi[n + j] = INFINITY;
  }
  double gsq = 0.0;
  int any = 0;
  double* tt = g_order ? dvec(tot) : NULL;
  for (int64_t s = 0; s < tot; ++s) {
    if (g[s] != 0.0) any = 1;
    if (g_order) tt[s] = g[s] * g[s] / w[s]; else gsq += g[s] * g[s] / w[s];
  }
  if (g_order) gsq = fold(tt, tot);
  double result = 0.0;
  if (any) {
    int bounded = 1;
    for (int64_t s = 0; s < tot; ++s) {
      d[s] = g[s] > 0.0 ? hi[s] : (g[s] < 0.0 ? lo[s] : 0.0);
      if (!isfinite(d[s])) { bounded = 0; break; }
    }
    int done = 0;
    if (bounded) {
      double ns = 0.0;
      for (int64_t s = 0; s < tot; ++s) {
        if (g_order) tt[s] = w[s] * d[s] * d[s]; else ns += w[s] * d[s] * d[s];
      }
      if (g_order) ns = fold(tt, tot);
      if (sqrt(ns) <= radius * (1.0 + 1e-12)) {
        result = dot(g, d, tot) / radius;
        done = 1;
      }
    }
    if (!done) {
      double nlo = 0.0, nhi = sqrt(gsq) / radius;
      const double r2 = radius * radius;
      for (int it = 0; it < 200; ++it) {
        const double nu = 0.5 * (nlo + nhi);
        double ns = 0.0;
        for (int64_t s = 0; s < tot; ++s) {
          const double un = g[s] / (nu * w[s]);
          d[s] = dmin(dmax(un, lo[s]), hi[s]);
          if (g_order) tt[s] = w[s] * d[s] * d[s]; else ns += w[s] * d[s] * d[s];
        }
        if (g_order) ns = fold(tt, tot);
        if (fabs(sqrt(ns) - radius) <= 1e-10 * radius) break;
        if (ns > r2) nlo = nu; else nhi = nu;
      }
      result = dot(g, d, tot) / radius;
    }
  }
  free(ktyv); free(kxv); free(g); free(w); free(lo); free(hi); free(d); free(tt);
  return result;
}

/* ---------------------------------------------------------------- steps */
typedef struct {
  double *xn, *yn, *kxn;
  double movement, cross;
} Trial;

/* pdhg_trial (solver.cpp:48-95) */
static int trial(const Lp* w, const double* x, const double* y, const double* kxv,
                 const double* ktyv, double eta, double omega, Trial* t) {
  const double tau = eta / omega, sigma = eta * omega;
  for (int64_t i = 0; i < w->n; ++i) {
    const double v = x[i] - tau * (w->c[i] - ktyv[i]);
    t->xn[i] = dmin(dmax(v, w->l[i]), w->u[i]);
  }
  kx(w, t->xn, t->kxn);
  double cross = 0.0, mv = 0.0;
  double* tc = g_order ? dvec(w->m) : NULL;
  double* tm = g_order ? dvec(w->m > w->n ? w->m : w->n) : NULL;
  for (int64_t j = 0; j < w->m; ++j) {
    const double ex = 2.0 * t->kxn[j] - kxv[j];
    double v = y[j] + sigma * (w->q[j] - ex);
    if (j < w->m1) v = dmax(v, 0.0);
    t->yn[j] = v;
    const double dy = v - y[j];
    if (g_order) {
      tc[j] = dy * (kxv[j] - t->kxn[j]);
      tm[j] = dy * dy;
      continue;
    }
    cross += dy * (kxv[j] - t->kxn[j]);
    mv += dy * dy;
  }
  if (g_order) {
    cross = fold(tc, w->m);
    mv = fold(tm, w->m);
  }
  mv /= omega;
  if (g_order) {
    for (int64_t i = 0; i < w->n; ++i) {
      const double dx = t->xn[i] - x[i];
      tm[i] = omega * dx * dx;
    }
    mv += fold(tm, w->n);
    free(tc);
    free(tm);
  } else {
    for (int64_t i = 0; i < w->n; ++i) {
      const double dx = t->xn[i] - x[i];
      mv += omega * dx * dx;
    }
  }
  t->movement = mv;
  t->cross = cross;
  if (!finite_all(t->xn, w->n) || !finite_all(t->yn, w->m))
    return fail(FOLP_E_NONFINITE, "pdhg step produced a NaN or infinite iterate");
  return FOLP_OK;
}

typedef struct {
  double eta_used, eta_next, movement, cross;
  int64_t trials;
} StepInfo;

/* adaptive_step (solver.cpp:154-200); on success x,y hold the next point. */
static int adaptive(const Lp* w, double* x, double* y, double omega, double eta_hat, int64_t k,
                    int64_t* lk, int64_t* lkt, StepInfo* out) {
  double* ktyv = dvec(w->n);
  double* kxv = dvec(w->m);
  kty(w, y, ktyv);
  kx(w, x, kxv);
  *lkt += 1;
  *lk += 1;
  const double kp1 = (double)(k + 1);
  const double red = 1.0 - pow(kp1, -0.3);
  const double grow = 1.0 + pow(kp1, -0.6);
  Trial t = {dvec(w->n), dvec(w->m), dvec(w->m), 0, 0};
  double eta = eta_hat;
  int rc = FOLP_OK;
  out->trials = 0;
  for (;;) {
    ++out->trials;
    rc = trial(w, x, y, kxv, ktyv, eta, omega, &t);
    *lk += 1;
    if (rc != FOLP_OK) break;
    const double eta_bar = t.cross > 0.0 ? t.movement / (2.0 * t.cross) : INFINITY;
    const double eta_next = dmin(red * eta_bar, grow * eta);
    if (eta <= eta_bar) {
      memcpy(x, t.xn, (size_t)w->n * sizeof(double));
      memcpy(y, t.yn, (size_t)w->m * sizeof(double));
      out->eta_used = eta;
      out->eta_next = eta_next;
      out->movement = t.movement;
      out->cross = t.cross;
      break;
    }
    eta = eta_next;
    if (eta < 1e-300) {
      rc = fail(FOLP_E_STEP_UNDERFLOW, "adaptive_step: step size underflow");
      break;
    }
  }
  free(ktyv); free(kxv); free(t.xn); free(t.yn); free(t.kxn);
  return rc;
}

/* pdhg_step (solver.cpp:127-141) */
static int constant_step(const Lp* w, double* x, double* y, double eta, double omega,
                         int64_t* lk, int64_t* lkt) {
  double* ktyv = dvec(w->n);
  double* kxv = dvec(w->m);
  kty(w, y, ktyv);
  kx(w, x, kxv);
  *lkt += 1;
  *lk += 1;
  Trial t = {dvec(w->n), dvec(w->m), dvec(w->m), 0, 0};
  int rc = trial(w, x, y, kxv, ktyv, eta, omega, &t);
  *lk += 1;
  if (rc == FOLP_OK) {
    memcpy(x, t.xn, (size_t)w->n * sizeof(double));
    memcpy(y, t.yn, (size_t)w->m * sizeof(double));
  }
  free(ktyv); free(kxv); free(t.xn); free(t.yn); free(t.kxn);
  return rc;
}

/* malitsky_pock_step (solver.cpp:202-275) */
static int mp_step(const Lp* w, double* x, double* y, double omega, double* eta_io,
                   double* theta_io, const folp_params_c* prm, int64_t* lk, int64_t* lkt,
                   int64_t* trials) {
  const int64_t n = w->n, m = w->m;
  double* ktyv = dvec(n);
  kty(w, y, ktyv);
  *lkt += 1;
  double* xn = dvec(n);
  const double eta_prev = *eta_io, theta_prev = *theta_io;
  const double tau = eta_prev / omega;
  for (int64_t i = 0; i < n; ++i) {
    const double v = x[i] - tau * (w->c[i] - ktyv[i]);
    xn[i] = dmin(dmax(v, w->l[i]), w->u[i]);
  }
  int rc = FOLP_OK;
  double *ext = dvec(n), *yh = dvec(m), *dy = dvec(m), *kw = dvec(m), *ktdy = dvec(n);
  if (!finite_all(xn, n)) {
    rc = fail(FOLP_E_NONFINITE, "malitsky_pock_step: non-finite primal iterate");
    goto out;
  }
  double eta_hat = eta_prev + prm->mp_interpolation_coefficient * (sqrt(1.0 + theta_prev) - 1.0) * eta_prev;
  *trials = 0;
  for (;;) {
    ++*trials;
    const double theta_hat = eta_prev / eta_hat;
    for (int64_t i = 0; i < n; ++i) ext[i] = xn[i] + theta_hat * (xn[i] - x[i]);
    kx(w, ext, kw);
    *lk += 1;
    const double sigma = omega * eta_hat;
    for (int64_t j = 0; j < m; ++j) {
      double v = y[j] + sigma * (w->q[j] - kw[j]);
      if (j < w->m1) v = dmax(v, 0.0);
      yh[j] = v;
      dy[j] = v - y[j];
    }
    if (!finite_all(yh, m)) {
      rc = fail(FOLP_E_NONFINITE, "malitsky_pock_step: non-finite dual iterate");
      goto out;
    }
    kty(w, dy, ktdy);
    *lkt += 1;
    if (eta_hat * sqrt(nsq(ktdy, n)) <= prm->mp_breaking_factor * sqrt(nsq(dy, m))) {
      memcpy(x, xn, (size_t)n * sizeof(double));
      memcpy(y, yh, (size_t)m * sizeof(double));
      *eta_io = eta_hat;
      *theta_io = theta_hat;
      break;
    }
    eta_hat *= prm->mp_downscaling_factor;
    if (eta_hat < 1e-300) {
      rc = fail(FOLP_E_STEP_UNDERFLOW, "malitsky_pock_step: step size underflow");
      goto out;
    }
  }
out:
  free(ktyv); free(xn); free(ext); free(yh); free(dy); free(kw); free(ktdy);
  return rc;
}

/* ---------------------------------------------------------------- driver */
typedef struct {
  int64_t* v;
  int64_t len, cap;
} IVec;
static void ipush(IVec* a, int64_t x) {
  if (a->len == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 16;
    a->v = (int64_t*)realloc(a->v, (size_t)a->cap * sizeof(int64_t));
  }
  a->v[a->len++] = x;
}

typedef struct {
  const folp_params_c* prm;
  double eps_nec, eps_suf;
  Lp pre, w;
  double *d1, *d2;
  double *x, *y, *lx, *ly, *ax, *ay;
  double avg_w, omega, eta_hat, eta_const, mp_eta, mp_theta, last_eta;
  double ref_gap, last_cand;
  int has_last_cand;
  int64_t k, t, outer, lk, lkt, trials, viol;
  IVec restarts;
  folp_result_c* out;
  struct timespec t0;
} Solver;

static double passes(const Solver* s) { return 0.5 * (double)(s->lk + s->lkt); }
static double elapsed(const Solver* s) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)(t.tv_sec - s->t0.tv_sec) + 1e-9 * (double)(t.tv_nsec - s->t0.tv_nsec);
}

static void trace_push(Solver* s, const folp_info_c* cur, const folp_info_c* avg) {
  folp_result_c* o = s->out;
  const int64_t i = o->num_trace++;
  if (i < o->trace_capacity) {
    if (o->trace_iteration) o->trace_iteration[i] = s->k;
    if (o->trace_kkt_passes) o->trace_kkt_passes[i] = passes(s);
    if (o->trace_current) o->trace_current[i] = *cur;
    if (o->trace_average) o->trace_average[i] = *avg;
  }
}

/* reduced_point + convergence_info (solver.cpp:495-507) */
static int evaluate(Solver* s, const double* xs, const double* ys, folp_info_c* info) {
  double* x = dvec(s->pre.n);
  double* y = dvec(s->pre.m);
  for (int64_t i = 0; i < s->pre.n; ++i) x[i] = dmin(dmax(xs[i] * s->d2[i], s->pre.l[i]), s->pre.u[i]);
  for (int64_t j = 0; j < s->pre.m; ++j) y[j] = ys[j] * s->d1[j];
  int rc = conv_info(&s->pre, x, y, info);
  if (rc == FOLP_OK || rc == FOLP_E_INFINITE_PRODUCT) {
    s->lk += 1;
    s->lkt += 1;
  }
  free(x);
  free(y);
  return rc;
}

/* materialize_average (solver.cpp:509-528) into (ox, oy) */
static void average(const Solver* s, double* ox, double* oy) {
  if (s->avg_w <= 0.0) {
    memcpy(ox, s->x, (size_t)s->w.n * sizeof(double));
    memcpy(oy, s->y, (size_t)s->w.m * sizeof(double));
    return;
  }
  const double inv = 1.0 / s->avg_w;
  for (int64_t i = 0; i < s->w.n; ++i) ox[i] = dmin(dmax(s->ax[i] * inv, s->w.l[i]), s->w.u[i]);
  for (int64_t j = 0; j < s->w.m; ++j) {
    double v = s->ay[j] * inv;
    if (j < s->w.m1) v = dmax(v, 0.0);
    oy[j] = v;
  }
}

/* finish (solver.cpp:647-676); presolve is the identity here */
static int finish(Solver* s, int reason, const double* xs, const double* ys,
                  const folp_info_c* info) {
  folp_result_c* o = s->out;
  o->termination_reason = reason;
  o->final_info = *info;
  o->iterations = s->k;
  o->restarts = s->outer;
  const int64_t n = s->pre.n, m = s->pre.m;
  double* x = dvec(n);
  double* y = dvec(m);
  for (int64_t i = 0; i < n; ++i) x[i] = dmin(dmax(xs[i] * s->d2[i], s->pre.l[i]), s->pre.u[i]);
  for (int64_t j = 0; j < m; ++j) y[j] = ys[j] * s->d1[j];
  double* r = dvec(n);
  kty(&s->pre, y, r);
  s->lkt += 1;
  for (int64_t i = 0; i < n; ++i) r[i] = s->pre.c[i] - r[i];
  if (o->primal_solution) memcpy(o->primal_solution, x, (size_t)n * sizeof(double));
  if (o->dual_solution) memcpy(o->dual_solution, y, (size_t)m * sizeof(double));
  if (o->reduced_costs) {
    for (int64_t i = 0; i < n; ++i) {
      const int lo = s->pre.l[i] > -INFINITY, hi = s->pre.u[i] < INFINITY;
      o->reduced_costs[i] = (!lo && !hi) ? 0.0 : (!lo ? dmin(r[i], 0.0) : (!hi ? dmax(r[i], 0.0) : r[i]));
    }
  }
  o->kkt_passes = passes(s);
  o->wall_seconds = elapsed(s);
  o->step_trials = s->trials;
  o->step_condition_violations = s->viol;
  o->num_restart_iterations = s->restarts.len;
  for (int64_t i = 0; i < s->restarts.len && i < o->restart_capacity; ++i)
    o->restart_iterations[i] = s->restarts.v[i];
  free(x); free(y); free(r);
  return FOLP_OK;
}

static double violation(const folp_info_c* i) { /* solver.cpp:469-475 */
  const double gap = i->gap_abs / (1.0 + fabs(i->primal_objective) + fabs(i->dual_objective));
  const double pr = i->primal_residual_norm / (1.0 + i->norm_q);
  const double du = i->dual_residual_norm / (1.0 + i->norm_c);
  return dmax(gap, dmax(pr, du));
}

static double primal_weight(const Solver* s, const double* nx, const double* ny,
                            const double* ox, const double* oy, double omega_prev) {
  const double th = s->prm->theta_smoothing;  /* solver.cpp:429-443 */
  if (th == 0.0) return omega_prev;
  const double dx = dnorm(nx, ox, s->w.n), dy = dnorm(ny, oy, s->w.m);
  if (dx > s->prm->eps_zero && dy > s->prm->eps_zero)
    return exp(th * log(dy / dx) + (1.0 - th) * log(omega_prev));
  return omega_prev;
}

static double wnorm_diff(const Solver* s, const double* ax_, const double* ay_, const double* bx,
                         const double* by, double omega) {
  double sx = 0.0, sy = 0.0; /* weighted_norm of the difference (lp_model.cpp:167-173) */
  if (g_order) {
    sx = dsq_folded(ax_, bx, s->w.n);
    sy = dsq_folded(ay_, by, s->w.m);
    return sqrt(omega * sx + sy / omega);
  }
  for (int64_t i = 0; i < s->w.n; ++i) {
    const double d = ax_[i] - bx[i];
    sx += d * d;
  }
  for (int64_t j = 0; j < s->w.m; ++j) {
    const double d = ay_[j] - by[j];
    sy += d * d;
  }
  return sqrt(omega * sx + sy / omega);
}

static int finish_numerical(Solver* s) { /* solver.cpp:728-749 */
  double* cx = dvec(s->w.n);
  double* cy = dvec(s->w.m);
  average(s, cx, cy);
  if (!finite_all(cx, s->w.n) || !finite_all(cy, s->w.m)) {
    memcpy(cx, s->lx, (size_t)s->w.n * sizeof(double));
    memcpy(cy, s->ly, (size_t)s->w.m * sizeof(double));
  }
  folp_info_c info;
  int rc = evaluate(s, cx, cy, &info);
  if (rc == FOLP_E_NONFINITE) {
    memcpy(cx, s->lx, (size_t)s->w.n * sizeof(double));
    memcpy(cy, s->ly, (size_t)s->w.m * sizeof(double));
    rc = evaluate(s, cx, cy, &info);
  }
  if (rc == FOLP_OK) {
    trace_push(s, &info, &info);
    rc = finish(s, converged(&info, s->prm->eps_optimal) ? FOLP_TERM_OPTIMAL : FOLP_TERM_NUMERICAL_ERROR,
                cx, cy, &info);
  }
  free(cx); free(cy);
  return rc;
}

static int finish_limit(Solver* s, int reason) { /* solver.cpp:703-726 */
  double* axp = dvec(s->w.n);
  double* ayp = dvec(s->w.m);
  folp_info_c ic, ia;
  int rc = evaluate(s, s->x, s->y, &ic);
  if (rc == FOLP_OK) {
    average(s, axp, ayp);
    rc = evaluate(s, axp, ayp, &ia);
  }
  if (rc == FOLP_E_NONFINITE) {
    free(axp); free(ayp);
    return finish_numerical(s);
  }
  if (rc == FOLP_OK) {
    trace_push(s, &ic, &ia);
    if (converged(&ic, s->prm->eps_optimal)) rc = finish(s, FOLP_TERM_OPTIMAL, s->x, s->y, &ic);
    else if (converged(&ia, s->prm->eps_optimal)) rc = finish(s, FOLP_TERM_OPTIMAL, axp, ayp, &ia);
    else if (violation(&ic) <= violation(&ia)) rc = finish(s, reason, s->x, s->y, &ic);
    else rc = finish(s, reason, axp, ayp, &ia);
  }
  free(axp); free(ayp);
  return rc;
}

/* evaluate_and_maybe_restart (solver.cpp:751-816): 1 = terminated */
static int eval_restart(Solver* s, int* terminated) {
  const int64_t n = s->w.n, m = s->w.m;
  double* axp = dvec(n);
  double* ayp = dvec(m);
  average(s, axp, ayp);
  folp_info_c ic, ia;
  int rc = evaluate(s, s->x, s->y, &ic);
  if (rc == FOLP_OK) rc = evaluate(s, axp, ayp, &ia);
  if (rc != FOLP_OK) goto out;
  trace_push(s, &ic, &ia);
  if (converged(&ic, s->prm->eps_optimal)) {
    *terminated = 1;
    rc = finish(s, FOLP_TERM_OPTIMAL, s->x, s->y, &ic);
    goto out;
  }
  if (converged(&ia, s->prm->eps_optimal)) {
    *terminated = 1;
    rc = finish(s, FOLP_TERM_OPTIMAL, axp, ayp, &ia);
    goto out;
  }
  if (s->prm->restart_scheme == FOLP_RESTART_NONE) {
    if ((double)s->t >= s->prm->beta_artificial * (double)s->k) {
      s->omega = primal_weight(s, s->x, s->y, s->lx, s->ly, s->omega);
      memcpy(s->lx, s->x, (size_t)n * sizeof(double));
      memcpy(s->ly, s->y, (size_t)m * sizeof(double));
      s->t = 0;
    }
    goto out;
  }
  {
    const double rcur = wnorm_diff(s, s->x, s->y, s->lx, s->ly, s->omega);
    const double mu_c = rcur == 0.0 ? 0.0 : ndg(&s->w, s->x, s->y, rcur, s->omega);
    if (rcur != 0.0) { s->lk += 1; s->lkt += 1; }
    const double ravg = wnorm_diff(s, axp, ayp, s->lx, s->ly, s->omega);
    const double mu_a = ravg == 0.0 ? 0.0 : ndg(&s->w, axp, ayp, ravg, s->omega);
    if (ravg != 0.0) { s->lk += 1; s->lkt += 1; }
    const int pick_cur = mu_c < mu_a;
    const double mu = pick_cur ? mu_c : mu_a;
    const double* cx = pick_cur ? s->x : axp;
    const double* cy = pick_cur ? s->y : ayp;
    /* should_restart (solver.cpp:395-419) */
    const double strong = dmin(s->eps_nec, s->eps_suf);
    const double gate = dmax(s->eps_nec, s->eps_suf);
    int restart = 0;
    if (mu <= strong * s->ref_gap) restart = 1;
    else if (mu <= gate * s->ref_gap && s->has_last_cand && mu > s->last_cand) restart = 1;
    else if ((double)s->t >= s->prm->beta_artificial * (double)s->k) restart = 1;
    if (!restart) {
      s->has_last_cand = 1;
      s->last_cand = mu;
      goto out;
    }
    s->outer++;
    ipush(&s->restarts, s->k);
    const double om = primal_weight(s, cx, cy, s->lx, s->ly, s->omega);
    const double rad = wnorm_diff(s, cx, cy, s->lx, s->ly, om);
    if (rad > 0.0) {
      s->ref_gap = ndg(&s->w, cx, cy, rad, om);
      s->lk += 1;
      s->lkt += 1;
    } else {
      s->ref_gap = 0.0;
    }
    s->omega = om;
    if (cx != s->x) {
      memcpy(s->x, cx, (size_t)n * sizeof(double));
      memcpy(s->y, cy, (size_t)m * sizeof(double));
    }
    memcpy(s->lx, s->x, (size_t)n * sizeof(double));
    memcpy(s->ly, s->y, (size_t)m * sizeof(double));
    memset(s->ax, 0, (size_t)n * sizeof(double));
    memset(s->ay, 0, (size_t)m * sizeof(double));
    s->avg_w = 0.0;
    s->has_last_cand = 0;
    s->t = 0;
  }
out:
  free(axp); free(ayp);
  return rc;
}

static int run(Solver* s, const double* x0, const double* y0) { /* solver.cpp:818-946 */
  const folp_params_c* p = s->prm;
  const int64_t n = s->pre.n, m = s->pre.m;
  if (n == 0 || m == 0) return fail(FOLP_E_INVALID_ARGUMENT, "port: empty LP not restated");
  s->d1 = dvec(m);
  s->d2 = dvec(n);
  TRY(rescale(&s->pre, p->ruiz_iterations, p->use_pock_chambolle, p->pc_alpha, &s->w, s->d1, s->d2));
  s->x = dvec(n); s->y = dvec(m); s->lx = dvec(n); s->ly = dvec(m);
  s->ax = dzero(n); s->ay = dzero(m);
  for (int64_t i = 0; i < n; ++i) {
    const double v = (x0 ? x0[i] : 0.0) / s->d2[i];
    s->x[i] = dmin(dmax(v, s->w.l[i]), s->w.u[i]);
  }
  for (int64_t j = 0; j < m; ++j) {
    double v = (y0 ? y0[j] : 0.0) / s->d1[j];
    if (j < s->w.m1) v = dmax(v, 0.0);
    s->y[j] = v;
  }
  memcpy(s->lx, s->x, (size_t)n * sizeof(double));
  memcpy(s->ly, s->y, (size_t)m * sizeof(double));
  s->omega = 1.0;
  if (p->scale_invariant_initial_primal_weight) {
    const double nc = sqrt(nsq(s->w.c, n)), nq = sqrt(nsq(s->w.q, m));
    if (nc > p->eps_zero && nq > p->eps_zero) s->omega = nc / nq;
  }
  const int has = s->w.nnz > 0;
  if (p->step_policy == FOLP_STEP_CONSTANT) {
    double norm = 0.0;
    if (has) { /* estimate_spectral_norm (sparse_matrix.cpp:188-220) */
      Mt64 g;
      mt_seed(&g, 1);
      double* v = dvec(n);
      double* wv = dvec(m);
      double* sv = dvec(n);
      for (int64_t i = 0; i < n; ++i) v[i] = 2.0 * ((double)(mt_next(&g) >> 11) * 0x1.0p-53) - 1.0;
      double vn = sqrt(nsq(v, n));
      if (vn == 0.0) { v[0] = 1.0; vn = 1.0; }
      const double sc = 1.0 / vn;
      for (int64_t i = 0; i < n; ++i) v[i] *= sc;
      double lambda = 0.0;
      int64_t mult = 0;
      int zero = 0;
      for (int64_t it = 0; it < 1000; ++it) {
        kx(&s->w, v, wv);
        kty(&s->w, wv, sv);
        mult += 2;
        const double next = dot(v, sv, n);
        const double sn = sqrt(nsq(sv, n));
        if (sn == 0.0) { zero = 1; break; }
        for (int64_t i = 0; i < n; ++i) v[i] = sv[i] / sn;
        const int conv = it > 0 && fabs(next - lambda) <= 1e-4 * fabs(next);
        lambda = next;
        if (conv) break;
      }
      norm = zero ? 0.0 : sqrt(dmax(lambda, 0.0));
      s->lk += mult / 2;
      s->lkt += mult / 2;
      free(v); free(wv); free(sv);
    }
    s->eta_const = norm > 0.0 ? 0.9 / norm : 1.0;
  } else {
    double mx = 0.0;
    for (int64_t k = 0; k < s->w.nnz; ++k) mx = dmax(mx, fabs(s->w.rv[k]));
    s->eta_hat = 1.0 / (has ? mx : 1.0);
    s->mp_eta = s->eta_hat;
    s->mp_theta = 1.0;
  }
  {
    folp_info_c i0;
    TRY(evaluate(s, s->x, s->y, &i0));
    trace_push(s, &i0, &i0);
    if (converged(&i0, p->eps_optimal)) return finish(s, FOLP_TERM_OPTIMAL, s->x, s->y, &i0);
  }
  folp_result_c* o = s->out;
  for (;;) {
    if (s->k >= p->iteration_limit) return finish_limit(s, FOLP_TERM_ITERATION_LIMIT);
    if (passes(s) >= p->kkt_pass_limit) return finish_limit(s, FOLP_TERM_KKT_PASS_LIMIT);
    if (elapsed(s) >= p->time_limit_seconds) return finish_limit(s, FOLP_TERM_TIME_LIMIT);
    int rc = FOLP_OK;
    if (p->step_policy == FOLP_STEP_ADAPTIVE) {
      StepInfo si;
      rc = adaptive(&s->w, s->x, s->y, s->omega, s->eta_hat, s->k + 1, &s->lk, &s->lkt, &si);
      s->trials += si.trials;
      if (rc == FOLP_OK) {
        if (si.cross > 0.0 && 2.0 * si.eta_used * si.cross > si.movement * (1.0 + 1e-9)) s->viol++;
        s->eta_hat = si.eta_next;
        s->last_eta = si.eta_used;
      }
    } else if (p->step_policy == FOLP_STEP_CONSTANT) {
      rc = constant_step(&s->w, s->x, s->y, s->eta_const, s->omega, &s->lk, &s->lkt);
      if (rc == FOLP_OK) {
        s->trials += 1;
        s->last_eta = s->eta_const;
      }
    } else {
      int64_t tr = 0;
      rc = mp_step(&s->w, s->x, s->y, s->omega, &s->mp_eta, &s->mp_theta, p, &s->lk, &s->lkt, &tr);
      s->trials += tr;
      if (rc == FOLP_OK) s->last_eta = s->mp_eta;
    }
    if (rc == FOLP_E_NONFINITE || rc == FOLP_E_STEP_UNDERFLOW) return finish_numerical(s);
    TRY(rc);
    s->k++;
    s->t++;
    for (int64_t i = 0; i < n; ++i) s->ax[i] += s->last_eta * s->x[i];
    for (int64_t j = 0; j < m; ++j) s->ay[j] += s->last_eta * s->y[j];
    s->avg_w += s->last_eta;
    if (p->record_iterate_trace) {
      const int64_t i = o->num_iterates++;
      o->iterate_n = n;
      o->iterate_m = m;
      if (i < o->iterate_capacity) {
        if (o->iterate_iteration) o->iterate_iteration[i] = s->k;
        if (o->iterate_eta) o->iterate_eta[i] = s->last_eta;
        if (o->iterate_primal) memcpy(o->iterate_primal + i * n, s->x, (size_t)n * sizeof(double));
        if (o->iterate_dual) memcpy(o->iterate_dual + i * m, s->y, (size_t)m * sizeof(double));
      }
    }
    if (s->t % p->evaluation_cadence == 0) {
      int term = 0;
      rc = eval_restart(s, &term);
      if (rc == FOLP_E_NONFINITE) return finish_numerical(s);
      TRY(rc);
      if (term) return FOLP_OK;
    }
  }
}

static int check_params(const folp_params_c* p) { /* solver.cpp:447-467 */
  if (!(p->eps_optimal > 0.0)) return fail(FOLP_E_INVALID_ARGUMENT, "solve: eps_optimal must be > 0");
  if (!(p->beta_necessary > 0.0 && p->beta_necessary < p->beta_sufficient && p->beta_sufficient < 1.0))
    return fail(FOLP_E_INVALID_ARGUMENT, "solve: betas must satisfy 0 < nec < suf < 1");
  if (!(p->beta_artificial > 0.0 && p->beta_artificial < 1.0))
    return fail(FOLP_E_INVALID_ARGUMENT, "solve: beta_artificial must be in (0,1)");
  if (!(p->theta_smoothing >= 0.0 && p->theta_smoothing <= 1.0))
    return fail(FOLP_E_INVALID_ARGUMENT, "solve: theta must be in [0,1]");
  if (p->evaluation_cadence < 1) return fail(FOLP_E_INVALID_ARGUMENT, "solve: evaluation cadence must be >= 1");
  if (p->ruiz_iterations < 0) return fail(FOLP_E_INVALID_ARGUMENT, "solve: ruiz_iterations must be >= 0");
  return FOLP_OK;
}

/* presolve would change this LP?  (presolve.cpp:83-156 rule triggers) */
static int presolve_is_identity(const Lp* p) {
  for (int64_t j = 0; j < p->n; ++j) {
    if (p->l[j] >= p->u[j]) return 0;
    if (p->cs[j + 1] == p->cs[j]) return 0;
  }
  for (int64_t i = 0; i < p->m; ++i)
    if (p->rs[i + 1] == p->rs[i]) return 0;
  return 1;
}

void folp_port_params_default(folp_params_c* p) {
  memset(p, 0, sizeof *p);
  p->eps_optimal = 1e-8;
  p->beta_sufficient = 0.9;
  p->beta_necessary = 0.1;
  p->beta_artificial = 0.5;
  p->theta_smoothing = 0.5;
  p->eps_zero = 1e-10;
  p->mp_breaking_factor = 1.0;
  p->mp_downscaling_factor = 0.5;
  p->mp_interpolation_coefficient = 0.4;
  p->evaluation_cadence = 40;
  p->kkt_pass_limit = INFINITY;
  p->iteration_limit = INT64_MAX;
  p->time_limit_seconds = INFINITY;
  p->ruiz_iterations = 10;
  p->use_pock_chambolle = 1;
  p->pc_alpha = 1.0;
  p->scale_invariant_initial_primal_weight = 1;
  p->use_presolve = 1;
}

int folp_port_solve(const folp_lp_c* lp, const folp_params_c* p, const double* x0,
                    const double* y0, folp_result_c* out) {
  TRY(check_params(p));
  Solver s;
  memset(&s, 0, sizeof s);
  clock_gettime(CLOCK_MONOTONIC, &s.t0);
  s.prm = p;
  s.eps_suf = p->restart_scheme == FOLP_RESTART_THEORY ? 0.37 : p->beta_sufficient;
  s.eps_nec = p->restart_scheme == FOLP_RESTART_THEORY ? 0.37 : p->beta_necessary;
  s.ref_gap = INFINITY;
  s.out = out;
  out->num_trace = out->num_iterates = out->num_restart_iterations = 0;
  TRY(lp_load(lp, &s.pre));
  int rc;
  if (p->use_presolve && !presolve_is_identity(&s.pre)) {
    rc = fail(FOLP_E_INVALID_ARGUMENT, "port: presolve would reduce this LP (not restated)");
  } else {
    rc = run(&s, x0, y0);
  }
  if (s.w.rv) free_working(&s.w);
  free(s.d1); free(s.d2); free(s.x); free(s.y); free(s.lx); free(s.ly); free(s.ax); free(s.ay);
  free(s.restarts.v);
  lp_free(&s.pre);
  return rc;
}

int folp_port_multiply(const folp_lp_c* lp, const double* x, double* out) {
  Lp p;
  TRY(lp_load(lp, &p));
  kx(&p, x, out);
  lp_free(&p);
  return FOLP_OK;
}

int folp_port_multiply_transpose(const folp_lp_c* lp, const double* y, double* out) {
  Lp p;
  TRY(lp_load(lp, &p));
  kty(&p, y, out);
  lp_free(&p);
  return FOLP_OK;
}

int folp_port_rescale(const folp_lp_c* lp, int64_t ruiz, int32_t pc, double alpha, double* d1,
                      double* d2, double* vals, double* c, double* q, double* l, double* u) {
  Lp p, w;
  TRY(lp_load(lp, &p));
  double* a = dvec(p.m);
  double* b = dvec(p.n);
  int rc = rescale(&p, ruiz, pc, alpha, &w, a, b);
  if (rc == FOLP_OK) {
    if (d1) memcpy(d1, a, (size_t)p.m * sizeof(double));
    if (d2) memcpy(d2, b, (size_t)p.n * sizeof(double));
    if (vals) memcpy(vals, w.rv, (size_t)p.nnz * sizeof(double));
    if (c) memcpy(c, w.c, (size_t)p.n * sizeof(double));
    if (q) memcpy(q, w.q, (size_t)p.m * sizeof(double));
    if (l) memcpy(l, w.l, (size_t)p.n * sizeof(double));
    if (u) memcpy(u, w.u, (size_t)p.n * sizeof(double));
    free_working(&w);
  }
  free(a); free(b);
  lp_free(&p);
  return rc;
}

int folp_port_convergence_info(const folp_lp_c* lp, const double* x, const double* y,
                               folp_info_c* info) {
  Lp p;
  TRY(lp_load(lp, &p));
  int rc = conv_info(&p, x, y, info);
  lp_free(&p);
  return rc;
}

int folp_port_normalized_duality_gap(const folp_lp_c* lp, const double* x, const double* y,
                                     double radius, double omega, double* gap) {
  if (!(radius > 0.0)) return fail(FOLP_E_NONPOSITIVE_RADIUS, "normalized_duality_gap: radius must be > 0");
  if (!(omega > 0.0)) return fail(FOLP_E_NONPOSITIVE_WEIGHT, "normalized_duality_gap: omega must be > 0");
  Lp p;
  TRY(lp_load(lp, &p));
  *gap = ndg(&p, x, y, radius, omega);
  lp_free(&p);
  return FOLP_OK;
}

int folp_port_adaptive_step(const folp_lp_c* lp, const double* x, const double* y, double omega,
                            double eta_hat, int64_t k, double* x_next, double* y_next,
                            double* eta_used, double* eta_hat_next, int64_t* trials,
                            double* movement_sq, double* cross_term) {
  if (k < 1) return fail(FOLP_E_INVALID_ARGUMENT, "adaptive_step: counter k is 1-based");
  if (!(eta_hat > 0.0)) return fail(FOLP_E_INVALID_ARGUMENT, "adaptive_step: eta_hat must be > 0");
  Lp p;
  TRY(lp_load(lp, &p));
  double* xs = dcopy(x, p.n);
  double* ys = dcopy(y, p.m);
  int64_t lk = 0, lkt = 0;
  StepInfo si;
  int rc = adaptive(&p, xs, ys, omega, eta_hat, k, &lk, &lkt, &si);
  if (rc == FOLP_OK) {
    memcpy(x_next, xs, (size_t)p.n * sizeof(double));
    memcpy(y_next, ys, (size_t)p.m * sizeof(double));
    *eta_used = si.eta_used;
    *eta_hat_next = si.eta_next;
    *trials = si.trials;
    *movement_sq = si.movement;
    *cross_term = si.cross;
  }
  free(xs); free(ys);
  lp_free(&p);
  return rc;
}

int folp_port_malitsky_pock_step(const folp_lp_c* lp, const double* x, const double* y,
                                 double omega, double eta_prev, double theta_prev,
                                 const folp_params_c* p, double* x_next, double* y_next,
                                 double* eta_next, double* theta_next, int64_t* trials) {
  if (!(eta_prev > 0.0) || !(theta_prev > 0.0))
    return fail(FOLP_E_INVALID_ARGUMENT,
                "malitsky_pock_step: needs positive previous step size and ratio");
  Lp w;
  TRY(lp_load(lp, &w));
  double* xs = dcopy(x, w.n);
  double* ys = dcopy(y, w.m);
  int64_t lk = 0, lkt = 0;
  double eta = eta_prev, theta = theta_prev;
  int rc = mp_step(&w, xs, ys, omega, &eta, &theta, p, &lk, &lkt, trials);
  if (rc == FOLP_OK) {
    memcpy(x_next, xs, (size_t)w.n * sizeof(double));
    memcpy(y_next, ys, (size_t)w.m * sizeof(double));
    *eta_next = eta;
    *theta_next = theta;
  }
  free(xs);
  free(ys);
  lp_free(&w);
  return rc;
}

const char* folp_port_last_error(void) { return g_err; }
