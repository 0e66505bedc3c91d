/*
 * condkit_oracle.c -- TEST INFRASTRUCTURE ONLY (see condkit_oracle.h).
 *
 * A sequential plain-C restatement of the reference algorithm for the
 * Projected-Adam kappa_2 estimator. Every function names the reference
 * file:line it follows (paths relative to /root/reference/proj/include/condkit).
 * Operation order is kept identical to the reference so that, compiled with
 * -ffp-contract=off, results match the reference bit for bit; that is checked
 * against oracle/_ref (the reference itself) by tests/test_oracle.py.
 */
#include "condkit_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_DIM = 1, E_ARG = 2, E_LOGIC = 3, E_SSING = 4, E_NSING = 5, E_ZRHS = 6, E_ZSOL = 7,
       E_DEGEN = 100 };

/* ---------------------------------------------------------------- rng.hpp */

/* std::mt19937_64 (the standard fixes its output sequence). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt_seed(mt64* g, uint64_t s) {
  g->mt[0] = s;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* rng.hpp:23-28 */
uint64_t cko_mix_seed(uint64_t base, uint64_t stream) {
  uint64_t z = base + 0x9E3779B97F4A7C15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* rng.hpp:31-33: top 53 bits of one draw */
static double u01(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }

/* rng.hpp:61-65: Box-Muller, 1-u1 keeps the log argument in (0, 1] */
static double std_normal(mt64* g) {
  double u1 = 1.0 - u01(g);
  double u2 = u01(g);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

double cko_two_norm(int64_t n, const double* v);

/* rng.hpp:68-77 */
static void rand_unit(mt64* g, int64_t n, double* x) {
  double nrm = 0.0;
  while (nrm == 0.0) {
    for (int64_t i = 0; i < n; ++i) x[i] = std_normal(g);
    nrm = cko_two_norm(n, x);
  }
  for (int64_t i = 0; i < n; ++i) x[i] /= nrm;
}

void cko_mt_draws(uint64_t seed, int64_t count, uint64_t* out) {
  mt64 g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt_next(&g);
}

void cko_random_unit_vectors(uint64_t seed, int64_t n, int64_t count, double* out) {
  mt64 g;
  mt_seed(&g, seed);
  for (int64_t c = 0; c < count; ++c) rand_unit(&g, n, out + c * n);
}

/* rng.hpp:36-38 */
void cko_uniform_in(uint64_t seed, int64_t count, double lo, double hi, double* out) {
  mt64 g;
  mt_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * u01(&g);
}

/* ------------------------------------------------------------- sparse.hpp */

/* sparse.hpp:175-186: amax pass, then scaled sum of squares */
double cko_two_norm(int64_t n, const double* v) {
  double amax = 0.0;
  for (int64_t i = 0; i < n; ++i) amax = fmax(amax, fabs(v[i]));
  if (amax == 0.0) return 0.0;
  if (!isfinite(amax)) return amax;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double q = v[i] / amax;
    s += q * q;
  }
  return amax * sqrt(s);
}

/* sparse.hpp:200-205 */
double cko_dot(int64_t n, const double* a, const double* b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* condest.hpp:158-171: Neumaier-compensated sum of squares */
double cko_compensated_norm(int64_t n, const double* v) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double q = v[i] * v[i];
    double t = s + q;
    if (fabs(s) >= fabs(q))
      c += (s - t) + q;
    else
      c += (q - t) + s;
    s = t;
  }
  return sqrt(s + c);
}

/* sparse.hpp:212-226: row sums in stored order */
void cko_matvec(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                const double* va, const double* x, double* y) {
  (void)ncols;
  for (int64_t i = 0; i < nrows; ++i) {
    double s = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += va[k] * x[ci[k]];
    y[i] = s;
  }
}

/* sparse.hpp:230-242: scatter, each output accumulates in increasing row order */
void cko_transpose_matvec(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                          const double* va, const double* x, double* y) {
  for (int64_t j = 0; j < ncols; ++j) y[j] = 0.0;
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) y[ci[k]] += va[k] * x[i];
}

/* column_norms, sparse.hpp:244-268: per-column max magnitude, then the
 * scaled sum of squares accumulated row by row. */
void cko_column_norms(int64_t nrows, int64_t ncols, const int64_t* rp, const int32_t* ci,
                      const double* va, double* out) {
  double* amax = (double*)calloc((size_t)(ncols ? ncols : 1), sizeof(double));
  double* sums = (double*)calloc((size_t)(ncols ? ncols : 1), sizeof(double));
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const double a = fabs(va[k]);
      if (amax[ci[k]] < a) amax[ci[k]] = a;
    }
  for (int64_t i = 0; i < nrows; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t j = ci[k];
      if (amax[j] == 0.0) continue;
      const double q = va[k] / amax[j];
      sums[j] += q * q;
    }
  for (int64_t j = 0; j < ncols; ++j) out[j] = amax[j] * sqrt(sums[j]);
  free(amax);
  free(sums);
}

/* two_norm of every row (the row_scale factors, sparse.hpp:295-311). */
void cko_row_norms(int64_t nrows, const int64_t* rp, const double* va, double* out) {
  for (int64_t i = 0; i < nrows; ++i) out[i] = cko_two_norm(rp[i + 1] - rp[i], va + rp[i]);
}

/* ------------------------------------------------------------- lu.hpp */

struct cko_lu {
  int64_t n;
  int64_t *l_rp, *u_rp, *perm;
  int32_t *l_ci, *u_ci;
  double *l_va, *u_va;
  double pivot_min;
};

typedef struct {
  int64_t* idx;
  double* val;
  int64_t len, cap;
} pvec;

static void pv_push(pvec* p, int64_t i, double v) {
  if (p->len == p->cap) {
    p->cap = p->cap ? 2 * p->cap : 8;
    p->idx = (int64_t*)realloc(p->idx, (size_t)p->cap * sizeof(int64_t));
    p->val = (double*)realloc(p->val, (size_t)p->cap * sizeof(double));
  }
  p->idx[p->len] = i;
  p->val[p->len] = v;
  p->len++;
}

/* lu.hpp:146-169: CSR assembly traversing columns in ascending order */
static void assemble(int64_t n, pvec* cols, const int64_t* remap, int64_t** rp_out,
                     int32_t** ci_out, double** va_out) {
  int64_t* rp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t q = 0; q < cols[j].len; ++q) {
      int64_t i = remap ? remap[cols[j].idx[q]] : cols[j].idx[q];
      rp[i + 1]++;
    }
  for (int64_t i = 0; i < n; ++i) rp[i + 1] += rp[i];
  int64_t* nx = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(nx, rp, (size_t)n * sizeof(int64_t));
  int32_t* ci = (int32_t*)malloc((size_t)(rp[n] + 1) * sizeof(int32_t));
  double* va = (double*)malloc((size_t)(rp[n] + 1) * sizeof(double));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t q = 0; q < cols[j].len; ++q) {
      int64_t i = remap ? remap[cols[j].idx[q]] : cols[j].idx[q];
      int64_t s = nx[i]++;
      ci[s] = (int32_t)j;
      va[s] = cols[j].val[q];
    }
  free(nx);
  *rp_out = rp;
  *ci_out = ci;
  *va_out = va;
}

/* lu.hpp:55-177: left-looking LU with row partial pivoting, natural order */
int cko_lu_factorize(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                     double pivot_tol, cko_lu** out, int64_t* fail_col, double* fail_pivot) {
  const int64_t NONE = -1;
  int64_t nnz = rp[n];
  /* column view (lu.hpp:61-78) */
  int64_t* cp = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int64_t* crow = (int64_t*)malloc((size_t)(nnz + 1) * sizeof(int64_t));
  double* cval = (double*)malloc((size_t)(nnz + 1) * sizeof(double));
  for (int64_t k = 0; k < nnz; ++k) cp[ci[k] + 1]++;
  for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
  {
    int64_t* nx = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
    memcpy(nx, cp, (size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        int64_t s = nx[ci[k]]++;
        crow[s] = i;
        cval[s] = va[k];
      }
    free(nx);
  }
  pvec* lcols = (pvec*)calloc((size_t)n + 1, sizeof(pvec));
  pvec* ucols = (pvec*)calloc((size_t)n + 1, sizeof(pvec));
  int64_t* perm = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  int64_t* pinv = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  double* work = (double*)calloc((size_t)n + 1, sizeof(double));
  char* inwork = (char*)calloc((size_t)n + 1, 1);
  int64_t* touched = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) perm[i] = pinv[i] = NONE;
  double pivot_min = INFINITY;
  int status = OK;

  for (int64_t j = 0; j < n && status == OK; ++j) {
    int64_t nt = 0;
    for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
      int64_t r = crow[p];
      work[r] = cval[p];
      inwork[r] = 1;
      touched[nt++] = r;
    }
    /* lu.hpp:97-110: apply earlier pivot columns in pivot order */
    for (int64_t k = 0; k < j; ++k) {
      int64_t prow = perm[k];
      if (!inwork[prow] || work[prow] == 0.0) continue;
      double ukj = work[prow];
      pv_push(&ucols[j], k, ukj);
      for (int64_t q = 0; q < lcols[k].len; ++q) {
        int64_t r = lcols[k].idx[q];
        if (!inwork[r]) {
          inwork[r] = 1;
          work[r] = 0.0;
          touched[nt++] = r;
        }
        work[r] -= lcols[k].val[q] * ukj;
      }
    }
    /* lu.hpp:112-129: pivot choice and singularity tests */
    int64_t best = NONE;
    double best_mag = 0.0, col_max = 0.0;
    int has_cand = 0;
    for (int64_t q = 0; q < nt; ++q) {
      int64_t r = touched[q];
      double mag = fabs(work[r]);
      col_max = fmax(col_max, mag);
      if (pinv[r] == NONE) {
        has_cand = 1;
        if (mag > best_mag) {
          best_mag = mag;
          best = r;
        }
      }
    }
    if (!has_cand) {
      status = E_SSING;
      if (fail_col) *fail_col = j;
      if (fail_pivot) *fail_pivot = 0.0;
    } else if (best == NONE || best_mag == 0.0 || best_mag < pivot_tol * col_max) {
      status = E_NSING;
      if (fail_col) *fail_col = j;
      if (fail_pivot) *fail_pivot = best_mag;
    } else {
      /* lu.hpp:130-141 */
      pivot_min = fmin(pivot_min, best_mag);
      perm[j] = best;
      pinv[best] = j;
      pv_push(&ucols[j], j, work[best]);
      double piv = work[best];
      for (int64_t q = 0; q < nt; ++q) {
        int64_t r = touched[q];
        if (pinv[r] == NONE && work[r] != 0.0) pv_push(&lcols[j], r, work[r] / piv);
      }
    }
    for (int64_t q = 0; q < nt; ++q) {
      work[touched[q]] = 0.0;
      inwork[touched[q]] = 0;
    }
  }

  if (status == OK) {
    cko_lu* f = (cko_lu*)calloc(1, sizeof(cko_lu));
    f->n = n;
    assemble(n, lcols, pinv, &f->l_rp, &f->l_ci, &f->l_va); /* L rows in pivot coordinates */
    assemble(n, ucols, NULL, &f->u_rp, &f->u_ci, &f->u_va);
    f->perm = perm;
    perm = NULL;
    f->pivot_min = pivot_min;
    *out = f;
  }
  for (int64_t j = 0; j < n; ++j) {
    free(lcols[j].idx);
    free(lcols[j].val);
    free(ucols[j].idx);
    free(ucols[j].val);
  }
  free(lcols);
  free(ucols);
  free(perm);
  free(pinv);
  free(work);
  free(inwork);
  free(touched);
  free(cp);
  free(crow);
  free(cval);
  return status;
}

void cko_lu_free(cko_lu* f) {
  if (!f) return;
  free(f->l_rp);
  free(f->l_ci);
  free(f->l_va);
  free(f->u_rp);
  free(f->u_ci);
  free(f->u_va);
  free(f->perm);
  free(f);
}

void cko_lu_info(const cko_lu* f, int64_t* n, int64_t* nnz_l, int64_t* nnz_u, double* pmin) {
  *n = f->n;
  *nnz_l = f->l_rp[f->n];
  *nnz_u = f->u_rp[f->n];
  *pmin = f->pivot_min;
}

void cko_lu_export(const cko_lu* f, int64_t* l_rp, int32_t* l_ci, double* l_va, int64_t* u_rp,
                   int32_t* u_ci, double* u_va, int64_t* row_perm) {
  int64_t n = f->n;
  memcpy(l_rp, f->l_rp, (size_t)(n + 1) * sizeof(int64_t));
  memcpy(u_rp, f->u_rp, (size_t)(n + 1) * sizeof(int64_t));
  memcpy(l_ci, f->l_ci, (size_t)f->l_rp[n] * sizeof(int32_t));
  memcpy(l_va, f->l_va, (size_t)f->l_rp[n] * sizeof(double));
  memcpy(u_ci, f->u_ci, (size_t)f->u_rp[n] * sizeof(int32_t));
  memcpy(u_va, f->u_va, (size_t)f->u_rp[n] * sizeof(double));
  memcpy(row_perm, f->perm, (size_t)n * sizeof(int64_t));
}

/* lu.hpp:180-202 */
int cko_lu_solve(const cko_lu* f, const double* b, double* y) {
  int64_t n = f->n;
  for (int64_t k = 0; k < n; ++k) y[k] = b[f->perm[k]];
  for (int64_t i = 0; i < n; ++i) {
    double s = y[i];
    for (int64_t k = f->l_rp[i]; k < f->l_rp[i + 1]; ++k) s -= f->l_va[k] * y[f->l_ci[k]];
    y[i] = s;
  }
  for (int64_t i = n; i-- > 0;) {
    int64_t r0 = f->u_rp[i];
    double s = y[i];
    for (int64_t k = r0 + 1; k < f->u_rp[i + 1]; ++k) s -= f->u_va[k] * y[f->u_ci[k]];
    y[i] = s / f->u_va[r0];
  }
  return OK;
}

/* lu.hpp:207-227 */
int cko_lu_transpose_solve(const cko_lu* f, const double* b, double* x) {
  int64_t n = f->n;
  double* w = (double*)malloc((size_t)(n + 1) * sizeof(double));
  memcpy(w, b, (size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) {
    int64_t r0 = f->u_rp[i];
    w[i] /= f->u_va[r0];
    for (int64_t k = r0 + 1; k < f->u_rp[i + 1]; ++k) w[f->u_ci[k]] -= f->u_va[k] * w[i];
  }
  for (int64_t i = n; i-- > 0;)
    for (int64_t k = f->l_rp[i]; k < f->l_rp[i + 1]; ++k) w[f->l_ci[k]] -= f->l_va[k] * w[i];
  for (int64_t k = 0; k < n; ++k) x[f->perm[k]] = w[k];
  free(w);
  return OK;
}

/* ------------------------------------------------------------- condest.hpp */

/* GradientOracle (condest.hpp:78-85) as a function table */
typedef struct {
  int64_t n, apply_dim;
  const void* ctx;
  int (*loss)(const void*, const double*, double*);
  int (*grad)(const void*, const double*, double*);
  void (*apply)(const void*, const double*, double*);
} oracle_t;

typedef struct {
  int64_t nrows, ncols;
  const int64_t* rp;
  const int32_t* ci;
  const double* va;
} csr_t;

/* condest.hpp:88-93 */
static int ex_loss(const void* c, const double* x, double* out) {
  const csr_t* a = (const csr_t*)c;
  double* av = (double*)malloc((size_t)(a->nrows + 1) * sizeof(double));
  cko_matvec(a->nrows, a->ncols, a->rp, a->ci, a->va, x, av);
  double num = cko_two_norm(a->ncols, x);
  double den = cko_two_norm(a->nrows, av);
  free(av);
  if (den == 0.0) return E_DEGEN;
  *out = log(num) - log(den);
  return OK;
}

/* condest.hpp:96-107 */
static int ex_grad(const void* c, const double* v, double* g) {
  const csr_t* a = (const csr_t*)c;
  double* av = (double*)malloc((size_t)(a->nrows + 1) * sizeof(double));
  cko_matvec(a->nrows, a->ncols, a->rp, a->ci, a->va, v, av);
  double vn = cko_two_norm(a->ncols, v);
  double avn = cko_two_norm(a->nrows, av);
  if (avn == 0.0) {
    free(av);
    return E_DEGEN;
  }
  double* atav = (double*)malloc((size_t)(a->ncols + 1) * sizeof(double));
  cko_transpose_matvec(a->nrows, a->ncols, a->rp, a->ci, a->va, av, atav);
  double inv_v2 = 1.0 / (vn * vn);
  double inv_av2 = 1.0 / (avn * avn);
  for (int64_t i = 0; i < a->ncols; ++i) g[i] = v[i] * inv_v2 - atav[i] * inv_av2;
  free(av);
  free(atav);
  return OK;
}

static void ex_apply(const void* c, const double* x, double* y) {
  const csr_t* a = (const csr_t*)c;
  cko_matvec(a->nrows, a->ncols, a->rp, a->ci, a->va, x, y);
}

/* condest.hpp:142-146 */
static int inv_loss(const void* c, const double* x, double* out) {
  const cko_lu* f = (const cko_lu*)c;
  double* r = (double*)malloc((size_t)(f->n + 1) * sizeof(double));
  cko_lu_solve(f, x, r);
  double rn = cko_two_norm(f->n, r);
  free(r);
  if (rn == 0.0) return E_DEGEN;
  *out = log(cko_two_norm(f->n, x)) - log(rn);
  return OK;
}

/* condest.hpp:112-123 */
static int inv_grad(const void* c, const double* x, double* g) {
  const cko_lu* f = (const cko_lu*)c;
  int64_t n = f->n;
  double* r = (double*)malloc((size_t)(n + 1) * sizeof(double));
  cko_lu_solve(f, x, r);
  double rn = cko_two_norm(n, r);
  if (rn == 0.0) {
    free(r);
    return E_DEGEN;
  }
  double* s = (double*)malloc((size_t)(n + 1) * sizeof(double));
  cko_lu_transpose_solve(f, r, s);
  double xn = cko_two_norm(n, x);
  double inv_x2 = 1.0 / (xn * xn);
  double inv_r2 = 1.0 / (rn * rn);
  for (int64_t i = 0; i < n; ++i) g[i] = x[i] * inv_x2 - s[i] * inv_r2;
  free(r);
  free(s);
  return OK;
}

static void inv_apply(const void* c, const double* x, double* y) {
  cko_lu_solve((const cko_lu*)c, x, y);
}

/* condest.hpp:184-297 */
static int projected_adam(const oracle_t* o, const cko_adam_cfg* cfg, cko_norm_result* res,
                          double* witness, double* loss_trace) {
  const int64_t n = o->n;
  if (n == 0) return E_ARG;
  mt64 gen;
  mt_seed(&gen, cfg->seed);
  double* x = (double*)malloc((size_t)n * sizeof(double));
  double* m = (double*)calloc((size_t)n, sizeof(double));
  double* v = (double*)calloc((size_t)n, sizeof(double));
  double* xmin = (double*)malloc((size_t)n * sizeof(double));
  double* g = (double*)malloc((size_t)n * sizeof(double));
  double* delta = (double*)malloc((size_t)n * sizeof(double));
  rand_unit(&gen, n, x);
  memcpy(xmin, x, (size_t)n * sizeof(double));
  uint64_t t = 0, since = 0, budget = 16;
  double loss_min = INFINITY, b1p = 1.0, b2p = 1.0;
  int plateaued = 0, status = OK;
  if (loss_trace)
    for (uint64_t i = 0; i < cfg->max_iter; ++i) loss_trace[i] = NAN;

#define RESTART()                                            \
  do {                                                       \
    rand_unit(&gen, n, x);                                   \
    memset(m, 0, (size_t)n * sizeof(double));                \
    memset(v, 0, (size_t)n * sizeof(double));                \
    b1p = 1.0;                                               \
    b2p = 1.0;                                               \
  } while (0)

  while (t < cfg->max_iter) {
    ++t;
    if (o->grad(o->ctx, x, g) != OK) {
      if (budget-- == 0) break;
      RESTART();
      continue;
    }
    b1p *= cfg->beta1;
    b2p *= cfg->beta2;
    double mc = 1.0 / (1.0 - b1p);
    double vc = 1.0 / (1.0 - b2p);
    for (int64_t i = 0; i < n; ++i) {
      m[i] = cfg->beta1 * m[i] + (1.0 - cfg->beta1) * g[i];
      v[i] = cfg->beta2 * v[i] + (1.0 - cfg->beta2) * g[i] * g[i];
      delta[i] = cfg->alpha * (m[i] * mc) / (sqrt(v[i] * vc) + cfg->eps_stab);
    }
    double radial = cko_dot(n, x, delta);
    for (int64_t i = 0; i < n; ++i) delta[i] -= radial * x[i];
    for (int64_t i = 0; i < n; ++i) x[i] -= delta[i];
    double nrm = cko_compensated_norm(n, x);
    if (nrm == 0.0 || !isfinite(nrm)) {
      if (budget-- == 0) break;
      RESTART();
      continue;
    }
    for (int64_t i = 0; i < n; ++i) x[i] /= nrm;
    double loss;
    if (o->loss(o->ctx, x, &loss) != OK) {
      if (budget-- == 0) break;
      RESTART();
      continue;
    }
    if (loss_trace) loss_trace[t - 1] = loss;
    int improved = !isfinite(loss_min) || loss_min - loss > cfg->rel_tol * fabs(loss_min);
    since = improved ? 0 : since + 1;
    if (loss < loss_min) {
      loss_min = loss;
      memcpy(xmin, x, (size_t)n * sizeof(double));
    }
    if (since >= cfg->patience) {
      plateaued = 1;
      break;
    }
  }
#undef RESTART

  res->iterations = t;
  res->converged = plateaued;
  if (isfinite(loss_min)) {
    res->value = exp(-loss_min);
    /* condest.hpp:284-289: witness re-check */
    double* ax = (double*)malloc((size_t)(o->apply_dim + 1) * sizeof(double));
    o->apply(o->ctx, xmin, ax);
    double chk = cko_two_norm(o->apply_dim, ax);
    free(ax);
    if (!(fabs(chk - res->value) <= 1e-12 * fmax(res->value, chk))) status = E_LOGIC;
  } else {
    res->value = 0.0;
    res->converged = 0;
  }
  if (witness) memcpy(witness, xmin, (size_t)n * sizeof(double));
  free(x);
  free(m);
  free(v);
  free(xmin);
  free(g);
  free(delta);
  return status;
}

/* condest.hpp:301-312: best of `restarts` seeded runs */
static int estimate_norm(const oracle_t* o, const cko_adam_cfg* cfg, uint64_t restarts,
                         cko_norm_result* res, double* witness) {
  if (restarts == 0) return E_ARG;
  double* w = (double*)malloc((size_t)(o->n + 1) * sizeof(double));
  int status = OK;
  for (uint64_t r = 0; r < restarts; ++r) {
    cko_adam_cfg c = *cfg;
    c.seed = r == 0 ? cfg->seed : cko_mix_seed(cfg->seed, r);
    cko_norm_result e;
    status = projected_adam(o, &c, &e, w, NULL);
    if (status != OK) break;
    if (r == 0 || e.value > res->value) {
      *res = e;
      if (witness) memcpy(witness, w, (size_t)o->n * sizeof(double));
    }
  }
  free(w);
  return status;
}

static oracle_t make_explicit(const csr_t* a) {
  oracle_t o = {a->ncols, a->nrows, a, ex_loss, ex_grad, ex_apply};
  return o;
}

static oracle_t make_inverse(const cko_lu* f) {
  oracle_t o = {f->n, f->n, f, inv_loss, inv_grad, inv_apply};
  return o;
}

int cko_loss_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                      const double* va, const double* x, double* loss) {
  csr_t a = {nr, nc, rp, ci, va};
  return ex_loss(&a, x, loss);
}

int cko_grad_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                      const double* va, const double* x, double* g) {
  csr_t a = {nr, nc, rp, ci, va};
  return ex_grad(&a, x, g);
}

int cko_projected_adam_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                                const double* va, const cko_adam_cfg* cfg, cko_norm_result* res,
                                double* witness, double* loss_trace) {
  csr_t a = {nr, nc, rp, ci, va};
  oracle_t o = make_explicit(&a);
  return projected_adam(&o, cfg, res, witness, loss_trace);
}

int cko_estimate_norm_explicit(int64_t nr, int64_t nc, const int64_t* rp, const int32_t* ci,
                               const double* va, const cko_adam_cfg* cfg, uint64_t restarts,
                               cko_norm_result* res, double* witness) {
  csr_t a = {nr, nc, rp, ci, va};
  oracle_t o = make_explicit(&a);
  return estimate_norm(&o, cfg, restarts, res, witness);
}

int cko_loss_inverse(const cko_lu* f, const double* x, double* loss) {
  return inv_loss(f, x, loss);
}

int cko_grad_inverse(const cko_lu* f, const double* x, double* g) { return inv_grad(f, x, g); }

int cko_projected_adam_inverse(const cko_lu* f, const cko_adam_cfg* cfg, cko_norm_result* res,
                               double* witness, double* loss_trace) {
  oracle_t o = make_inverse(f);
  return projected_adam(&o, cfg, res, witness, loss_trace);
}

int cko_estimate_norm_inverse(const cko_lu* f, const cko_adam_cfg* cfg, uint64_t restarts,
                              cko_norm_result* res, double* witness) {
  oracle_t o = make_inverse(f);
  return estimate_norm(&o, cfg, restarts, res, witness);
}

/* condest.hpp:341-365 */
int cko_cond2(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
              const cko_adam_cfg* cfg, uint64_t restarts, double pivot_tol, double* kappa,
              cko_norm_result* fwd, cko_norm_result* inv, int32_t* has_factors) {
  csr_t a = {n, n, rp, ci, va};
  oracle_t o = make_explicit(&a);
  memset(inv, 0, sizeof(*inv));
  int st = estimate_norm(&o, cfg, restarts, fwd, NULL);
  if (st != OK) return st;
  cko_lu* f = NULL;
  st = cko_lu_factorize(n, rp, ci, va, pivot_tol, &f, NULL, NULL);
  *has_factors = 0;
  if (st == E_SSING || st == E_NSING) {
    inv->value = INFINITY;
    *kappa = INFINITY;
    return OK;
  }
  if (st != OK) return st;
  cko_adam_cfg ci_cfg = *cfg;
  ci_cfg.seed = cko_mix_seed(cfg->seed, 0x1234);
  oracle_t oi = make_inverse(f);
  st = estimate_norm(&oi, &ci_cfg, restarts, inv, NULL);
  *kappa = fwd->value * inv->value;
  *has_factors = 1;
  cko_lu_free(f);
  return st;
}

/* ------------------------------------------------------------- error_bounds.hpp */

/* error_bounds.hpp:59-68 */
int cko_loose_bounds(double rn, double bn, double kappa, double* lo, double* hi) {
  if (!(rn >= 0.0)) return E_ARG;
  if (!(kappa >= 1.0)) return E_ARG;
  if (bn == 0.0) return E_ZRHS;
  if (!(bn > 0.0)) return E_ARG;
  double rho = rn / bn;
  if (rho == 0.0) {
    *lo = 0.0;
    *hi = 0.0;
    return OK;
  }
  *lo = rho / kappa;
  *hi = kappa * rho;
  return OK;
}

/* error_bounds.hpp:71-80 */
int cko_tight_bounds(double rn, double an, double xn, double kappa, double* lo, double* hi) {
  if (!(rn >= 0.0)) return E_ARG;
  if (!(kappa >= 1.0)) return E_ARG;
  if (xn == 0.0) return E_ZSOL;
  if (!(xn > 0.0)) return E_ARG;
  if (!(an > 0.0)) return E_ARG;
  double rho = rn / (an * xn);
  if (rho == 0.0) {
    *lo = 0.0;
    *hi = 0.0;
    return OK;
  }
  *lo = rho;
  *hi = kappa * rho;
  return OK;
}

/* error_bounds.hpp:84-88 */
int cko_propagate_bound(double e, double* out) {
  if (!(e >= 0.0)) return E_ARG;
  *out = e >= 1.0 ? INFINITY : e / (1.0 - e);
  return OK;
}

/* error_bounds.hpp:93-99 */
int cko_singularity_bound(double kappa, double eps, double* out) {
  if (!(kappa >= 1.0)) return E_ARG;
  if (!(eps > 0.0)) return E_ARG;
  double ke = kappa * eps;
  *out = ke >= 1.0 ? INFINITY : 2.0 * ke / (1.0 - ke);
  return OK;
}

/* error_bounds.hpp:166-217 */
int cko_verify_solution(int64_t n, const int64_t* rp, const int32_t* ci, const double* va,
                        const double* xhat, const double* b, const cko_verify_options* opt,
                        cko_bounds_report* rep) {
  if (!(opt->threshold > 0.0)) return E_ARG;
  memset(rep, 0, sizeof(*rep));
  rep->threshold = opt->threshold;
  rep->eps_mach = opt->eps_mach;
  rep->xhat_norm = cko_two_norm(n, xhat);
  if (rep->xhat_norm == 0.0) return E_ZSOL;
  rep->b_norm = cko_two_norm(n, b);
  if (rep->b_norm == 0.0) return E_ZRHS;
  double* r = (double*)malloc((size_t)(n + 1) * sizeof(double));
  cko_matvec(n, n, rp, ci, va, xhat, r);
  for (int64_t i = 0; i < n; ++i) r[i] -= b[i];
  rep->residual_norm = cko_two_norm(n, r);
  free(r);
  int st;
  if (opt->has_kappa) {
    if (!(opt->kappa >= 1.0)) return E_ARG;
    rep->kappa = opt->kappa;
    rep->kappa_supplied = 1;
    if (opt->has_a_norm) {
      rep->a_norm = opt->a_norm;
    } else {
      cko_norm_result e;
      st = cko_estimate_norm_explicit(n, n, rp, ci, va, &opt->adam, opt->restarts, &e, NULL);
      if (st != OK) return st;
      rep->a_norm = e.value;
    }
  } else {
    double kappa;
    cko_norm_result fwd, inv;
    int32_t hf;
    st = cko_cond2(n, rp, ci, va, &opt->adam, opt->restarts, opt->pivot_tol, &kappa, &fwd, &inv,
                   &hf);
    if (st != OK) return st;
    rep->kappa = fmax(1.0, kappa);
    rep->a_norm = opt->has_a_norm ? opt->a_norm : fwd.value;
  }
  if (!(rep->a_norm > 0.0)) return E_ARG;
  st = cko_loose_bounds(rep->residual_norm, rep->b_norm, rep->kappa, &rep->loose_lower,
                        &rep->loose_upper);
  if (st != OK) return st;
  st = cko_tight_bounds(rep->residual_norm, rep->a_norm, rep->xhat_norm, rep->kappa,
                        &rep->tight_lower, &rep->tight_upper);
  if (st != OK) return st;
  cko_propagate_bound(rep->tight_upper, &rep->true_error_cap);
  st = cko_singularity_bound(rep->kappa, rep->eps_mach, &rep->singularity_cap);
  if (st != OK) return st;
  if (rep->kappa >= 1.0 / rep->eps_mach)
    rep->verdict = 2;
  else
    rep->verdict = rep->tight_upper <= rep->threshold ? 0 : 1;
  return OK;
}
