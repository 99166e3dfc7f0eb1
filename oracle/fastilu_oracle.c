/*
 * fastilu_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the FastILU hot path of
 * arXiv 2506.05793 (ShyLU-node), Section 5 ("FastILU").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product (the CUDA
 * library under paper_2506_05793_b200/) shares no code with this file.
 *
 * Arithmetic: IEEE binary64, compiled with -O2 -ffp-contract=off so that no
 * multiply-subtract is fused; every per-entry sum is accumulated left to right
 * in the order stated next to it.  The residual r(s-1) (a sum of nnz(S)
 * squares) is summed EXACTLY and rounded once (orc_fsum_*, Shewchuk's
 * partials, the algorithm of Python's math.fsum), so its value does not
 * depend on any summation order.
 *
 * Threads: orc_set_threads(T) runs the per-row loops (scale/init, sweep,
 * Jacobi sweeps) with OpenMP over rows.  Every row/entry is computed by one
 * thread with the sequential arithmetic above and the exact residual sum is
 * order independent, so T threads give results bitwise equal to 1 thread
 * (tests/test_oracle_numeric.py::test_threads_bitwise).  Default: 1 thread.
 *
 * Readings of the paper (listed in DESIGN.md, "Readings"):
 *   R1 (Fig. algo:fastILU_comp line 3): the printed l-update
 *      "(1-w) + w(a_ij - sum)/u_ij" is read as
 *      l_ij <- (1-w) l_ij + w (a_ij - sum_{k<j} l_ik u_kj) / u_jj.
 *   R2: both sums run over k < min(i,j).
 *   R3 (PAPER.md:717 vs BASELINE north_star): sweeps are synchronous
 *      (Jacobi): every right-hand value, the divisor u_jj included, is taken
 *      from iterate s-1.
 *   R4: initial guess l0_ij = ahat_ij/ahat_jj, u0_ij = ahat_ij,
 *      fill entries +0.0.
 *   R5 (north_star): symmetric diagonal scaling s_i = 1/sqrt(|a_ii|),
 *      ahat_ij = (a_ij s_i) s_j; apply returns s o U^-1 L^-1 (s o b).
 *   R6 (Fig. FastSpTRSV): Jacobi sweeps from x0 = 0,
 *      out of place; L is unit lower (no division), the U sweep divides by
 *      u_ii.
 *   R7 level-of-fill: sum rule lev(i,j) = min(lev(i,j), lev(i,k)+lev(k,j)+1)
 *      over pivots k < min(i,j) processed in ascending order, keep lev <= K.
 *   R9 Manteuffel shift alpha >= 0: the factors are those of
 *      A' = A + alpha diag(|a_ii|), i.e. a'_ii = a_ii + alpha |a_ii| (rounded product, then
 *      sum); alpha = 0 leaves A unchanged.
 *   R8 zero pivot: FASTILU_ERR_ZERO_PIVOT when any iterate 0..nsweeps has a
 *      diagonal u_ii that is 0 or non-finite; the error index is the smallest
 *      such row over all iterates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* status codes mirror include/fastilu.h by VALUE only (no shared header) */
enum {
  ORC_OK = 0,
  ORC_ERR_INVALID_ARG = 1,
  ORC_ERR_BAD_MATRIX = 2,
  ORC_ERR_MISSING_DIAG = 3,
  ORC_ERR_ZERO_DIAG = 4,
  ORC_ERR_ZERO_PIVOT = 5,
  ORC_ERR_OOM = 9
};

void orc_free(void *p) { free(p); }

static int g_threads = 1;
/* number of OpenMP threads for the per-row loops (1 = sequential); returns the value in use */
int orc_set_threads(int t) {
#ifdef _OPENMP
  g_threads = t > 0 ? t : 1;
#else
  (void)t;
  g_threads = 1;
#endif
  return g_threads;
}

/* ------------------------------------------------------------------------ */
/* Exactly rounded summation (Shewchuk, "Adaptive precision floating-point   */
/* arithmetic", 1997; the algorithm of Python's math.fsum).  The running sum */
/* is held as a list of non-overlapping partials whose exact sum is the exact */
/* sum of every term added so far (each two-sum below is error free).         */
/* Finite terms only (squares of finite defects here).                        */
/* ------------------------------------------------------------------------ */
typedef struct { double p[80]; int n; } orc_fsum_t;

static void orc_fsum_add(orc_fsum_t *s, double x) {
  int i = 0;
  for (int j = 0; j < s->n; j++) {
    double y = s->p[j];
    if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
    double hi = x + y;           /* two-sum with |x| >= |y|: hi + lo == x + y exactly */
    double lo = y - (hi - x);
    if (lo != 0.0) s->p[i++] = lo;
    x = hi;
  }
  s->p[i++] = x;
  s->n = i;
}

/* the exact sum rounded to nearest (ties to even), from the partials */
static double orc_fsum_result(const orc_fsum_t *s) {
  int n = s->n;
  if (n == 0) return 0.0;
  double hi = s->p[--n], lo = 0.0;
  while (n > 0) {               /* add partials from the largest down until inexact */
    double x = hi, y = s->p[--n];
    hi = x + y;
    double yr = hi - x;
    lo = y - yr;
    if (lo != 0.0) break;
  }
  /* half-way case: the remaining partials decide the rounding direction */
  if (n > 0 && ((lo < 0.0 && s->p[n - 1] < 0.0) || (lo > 0.0 && s->p[n - 1] > 0.0))) {
    double y = lo * 2.0, x = hi + y;
    if (y == x - hi) hi = x;
  }
  return hi;
}

/* exposed for its pin (tests: == math.fsum bitwise on adversarial inputs) */
double orc_fsum(int64_t n, const double *x) {
  orc_fsum_t s;
  s.n = 0;
  for (int64_t i = 0; i < n; i++) orc_fsum_add(&s, x[i]);
  return orc_fsum_result(&s);
}

static void orc_fsum_merge(orc_fsum_t *into, const orc_fsum_t *from) {
  for (int j = 0; j < from->n; j++) orc_fsum_add(into, from->p[j]);
}

/* ------------------------------------------------------------------------ */
/* Validation (SPEC.md:26-31 CSR invariants; SPEC.md:357-359 structural      */
/* diagonal).                                                                */
/* ------------------------------------------------------------------------ */
int orc_validate(int64_t n, const int64_t *rp, const int32_t *ci,
                 int64_t *bad) {
  *bad = -1;
  if (n < 0 || rp == NULL) return ORC_ERR_INVALID_ARG;
  if (rp[0] != 0) { *bad = 0; return ORC_ERR_BAD_MATRIX; }
  for (int64_t i = 0; i < n; i++) {
    if (rp[i + 1] < rp[i]) { *bad = i; return ORC_ERR_BAD_MATRIX; }
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      if (ci[q] < 0 || (int64_t)ci[q] >= n) { *bad = i; return ORC_ERR_BAD_MATRIX; }
      if (q > rp[i] && ci[q] <= ci[q - 1]) { *bad = i; return ORC_ERR_BAD_MATRIX; }
    }
  }
  for (int64_t i = 0; i < n; i++) {
    int found = 0;
    for (int64_t q = rp[i]; q < rp[i + 1]; q++)
      if (ci[q] == i) found = 1;
    if (!found) { *bad = i; return ORC_ERR_MISSING_DIAG; }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Symbolic ILU(K) (reading R7; "level-based ILU", SPEC.md:341-  */
/* 344, 355-363).  Row by row; pivots k < i of row i popped in ascending      */
/* order from a binary min-heap, fill created during the row included.        */
/* ------------------------------------------------------------------------ */
static void heap_push(int32_t *h, int64_t *hn, int32_t v) {
  int64_t c = (*hn)++;
  h[c] = v;
  while (c > 0) {
    int64_t p = (c - 1) / 2;
    if (h[p] <= h[c]) break;
    int32_t t = h[p]; h[p] = h[c]; h[c] = t;
    c = p;
  }
}
static int32_t heap_pop(int32_t *h, int64_t *hn) {
  int32_t top = h[0];
  (*hn)--;
  h[0] = h[*hn];
  int64_t c = 0;
  for (;;) {
    int64_t l = 2 * c + 1, r = l + 1, m = c;
    if (l < *hn && h[l] < h[m]) m = l;
    if (r < *hn && h[r] < h[m]) m = r;
    if (m == c) break;
    int32_t t = h[m]; h[m] = h[c]; h[c] = t;
    c = m;
  }
  return top;
}
static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

int orc_symbolic(int64_t n, const int64_t *rp, const int32_t *ci, int K,
                 int64_t **out_rp, int32_t **out_ci, int32_t **out_lev,
                 int64_t *bad) {
  int st = orc_validate(n, rp, ci, bad);
  if (st != ORC_OK) return st;
  if (K < 0) return ORC_ERR_INVALID_ARG;
  const int32_t UNSET = INT32_MAX;
  int32_t *lev = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t *list = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int32_t *heap = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  int64_t *dpos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t *srp = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t cap = rp[n] > 16 ? rp[n] : 16;
  int32_t *sci = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  int32_t *slev = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  if (!lev || !list || !heap || !dpos || !srp || !sci || !slev) return ORC_ERR_OOM;
  for (int64_t j = 0; j < n; j++) lev[j] = UNSET;
  srp[0] = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t nl = 0, hn = 0;
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      int32_t j = ci[q];
      lev[j] = 0; /* entries of A (explicit zeros included) have level 0 */
      list[nl++] = j;
      if (j < i) heap_push(heap, &hn, j);
    }
    while (hn > 0) {
      int32_t k = heap_pop(heap, &hn);
      /* strict upper part of row k of S: columns j > k */
      for (int64_t q = dpos[k] + 1; q < srp[k + 1]; q++) {
        int32_t j = sci[q];
        int32_t l = lev[k] + slev[q] + 1;
        if (l > K) continue;
        if (lev[j] == UNSET) {
          lev[j] = l;
          list[nl++] = j;
          if (j < i) heap_push(heap, &hn, j);
        } else if (l < lev[j]) {
          lev[j] = l;
        }
      }
    }
    qsort(list, (size_t)nl, sizeof(int32_t), cmp_i32);
    if (srp[i] + nl > cap) {
      while (srp[i] + nl > cap) cap *= 2;
      sci = (int32_t *)realloc(sci, sizeof(int32_t) * (size_t)cap);
      slev = (int32_t *)realloc(slev, sizeof(int32_t) * (size_t)cap);
      if (!sci || !slev) return ORC_ERR_OOM;
    }
    for (int64_t t = 0; t < nl; t++) {
      int32_t j = list[t];
      sci[srp[i] + t] = j;
      slev[srp[i] + t] = lev[j];
      if (j == i) dpos[i] = srp[i] + t;
      lev[j] = UNSET;
    }
    srp[i + 1] = srp[i] + nl;
  }
  free(lev); free(list); free(heap); free(dpos);
  *out_rp = srp; *out_ci = sci; *out_lev = slev;
  return ORC_OK;
}

/* position of column j in row r of a sorted CSR pattern, -1 if absent */
static int64_t find_in_row(const int64_t *rp, const int32_t *ci, int64_t r,
                           int32_t j) {
  int64_t lo = rp[r], hi = rp[r + 1] - 1;
  while (lo <= hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (ci[mid] == j) return mid;
    if (ci[mid] < j) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* ------------------------------------------------------------------------ */
/* Diagonal scaling + initial guess (readings R4, R5).                        */
/*   s_i = 1/sqrt(|a_ii|);  ahat_ij = (a_ij * s_i) * s_j  (on S, 0 for fill)  */
/*   vals: l0_ij = ahat_ij / ahat_jj (j < i), u0_ij = ahat_ij (i <= j).       */
/* ------------------------------------------------------------------------ */
static double shifted(double aii, double shift) {  /* reading R9 */
  double t = shift * fabs(aii);
  return aii + t;
}

int orc_scale_init(int64_t n, const int64_t *rp, const int32_t *ci,
                   const double *a, const int64_t *srp, const int32_t *sci, double shift,
                   double *s, double *ahat, double *vals, int64_t *bad) {
  *bad = -1;
  for (int64_t i = 0; i < n; i++) {
    int64_t q = find_in_row(rp, ci, i, (int32_t)i);
    if (q < 0) { *bad = i; return ORC_ERR_MISSING_DIAG; }
    double aii = shifted(a[q], shift);
    if (aii == 0.0) { *bad = i; return ORC_ERR_ZERO_DIAG; }
    s[i] = 1.0 / sqrt(fabs(aii));
  }
  for (int64_t p = 0; p < srp[n]; p++) ahat[p] = 0.0;
  int missing = 0;
#pragma omp parallel for schedule(static) num_threads(g_threads) reduction(| : missing)
  for (int64_t i = 0; i < n; i++) {
    for (int64_t q = rp[i]; q < rp[i + 1]; q++) {
      int32_t j = ci[q];
      int64_t p = find_in_row(srp, sci, i, j);
      if (p < 0) { missing = 1; continue; } /* S must contain A */
      double aij = (j == i) ? shifted(a[q], shift) : a[q];
      ahat[p] = (aij * s[i]) * s[j];
    }
  }
  if (missing) return ORC_ERR_BAD_MATRIX;
#pragma omp parallel for schedule(static) num_threads(g_threads)
  for (int64_t i = 0; i < n; i++) {
    for (int64_t p = srp[i]; p < srp[i + 1]; p++) {
      int32_t j = sci[p];
      if (j < i) {
        int64_t pjj = find_in_row(srp, sci, j, j);
        vals[p] = ahat[p] / ahat[pjj];
      } else {
        vals[p] = ahat[p];
      }
    }
  }
  return ORC_OK;
}

/* smallest row whose diagonal in `vals` is 0 or non-finite, else -1 */
int64_t orc_bad_diagonal(int64_t n, const int64_t *srp, const int32_t *sci,
                         const double *vals) {
  for (int64_t i = 0; i < n; i++) {
    int64_t p = find_in_row(srp, sci, i, (int32_t)i);
    double d = vals[p];
    if (d == 0.0 || !isfinite(d)) return i;
  }
  return -1;
}

/* ------------------------------------------------------------------------ */
/* One synchronous FastILU sweep (PAPER.md:543-551 Fig. algo:fastILU_comp,    */
/* readings R1-R3).  For every (i,j) in S, row-major order:                   */
/*   acc = ahat_ij;                                                           */
/*   for k in S_i ascending with k < min(i,j) and (k,j) in S:                 */
/*       acc = acc - l_ik * u_kj            (rounded product, then difference) */
/*   i > j:  l_ij = w == 1 ? acc/u_jj : (1-w) l_ij + w (acc/u_jj)             */
/*   i <= j: u_ij = w == 1 ? acc      : (1-w) u_ij + w acc                    */
/* all right-hand values from `old` (iterate s-1).  *resid receives           */
/*   r(s-1) = sqrt( sum_L (acc - l_ij u_jj)^2 + sum_U (acc - u_ij)^2 )        */
/*         = ||(Ahat - L U)|_S||_F at iterate s-1,          */
/* each square a rounded product, their sum exact and rounded once (fsum).    */
/* ------------------------------------------------------------------------ */
void orc_sweep(int64_t n, const int64_t *srp, const int32_t *sci,
               const double *ahat, const double *old, double *out,
               double omega, double *resid) {
  orc_fsum_t total;
  total.n = 0;
#pragma omp parallel num_threads(g_threads)
  {
    orc_fsum_t r2; /* this thread's exact partial sum of squares */
    r2.n = 0;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; i++) {
      for (int64_t p = srp[i]; p < srp[i + 1]; p++) {
        int32_t j = sci[p];
        int64_t m = (j < i) ? j : i; /* min(i,j) */
        double acc = ahat[p];
        for (int64_t q = srp[i]; q < srp[i + 1] && sci[q] < m; q++) {
          int32_t k = sci[q];
          int64_t pkj = find_in_row(srp, sci, k, j);
          if (pkj < 0) continue;
          double prod = old[q] * old[pkj];
          acc = acc - prod;
        }
        if (j < i) {
          int64_t pjj = find_in_row(srp, sci, j, j);
          double ujj = old[pjj];
          double e = acc - old[p] * ujj;
          orc_fsum_add(&r2, e * e);
          double l = acc / ujj;
          out[p] = (omega == 1.0) ? l : (1.0 - omega) * old[p] + omega * l;
        } else {
          double e = acc - old[p];
          orc_fsum_add(&r2, e * e);
          out[p] = (omega == 1.0) ? acc : (1.0 - omega) * old[p] + omega * acc;
        }
      }
    }
#pragma omp critical
    orc_fsum_merge(&total, &r2);
  }
  *resid = sqrt(orc_fsum_result(&total));
}

/* ------------------------------------------------------------------------ */
/* FastILU compute: scale/init, then nsweeps synchronous sweeps (R8 for the   */
/* zero-pivot rule).  resid_hist[s-1] = r(s-1), s = 1..nsweeps.               */
/* ------------------------------------------------------------------------ */
int orc_compute(int64_t n, const int64_t *rp, const int32_t *ci,
                const double *a, const int64_t *srp, const int32_t *sci,
                int nsweeps, double omega, double shift, double *s, double *ahat,
                double *vals, double *resid_hist, int64_t *bad) {
  int st = orc_scale_init(n, rp, ci, a, srp, sci, shift, s, ahat, vals, bad);
  if (st != ORC_OK) return st;
  int64_t nnz = srp[n];
  double *tmp = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  if (!tmp) return ORC_ERR_OOM;
  int64_t worst = orc_bad_diagonal(n, srp, sci, vals);
  for (int sw = 1; sw <= nsweeps; sw++) {
    orc_sweep(n, srp, sci, ahat, vals, tmp, omega, &resid_hist[sw - 1]);
    memcpy(vals, tmp, sizeof(double) * (size_t)nnz);
    int64_t b = orc_bad_diagonal(n, srp, sci, vals);
    if (b >= 0 && (worst < 0 || b < worst)) worst = b;
  }
  free(tmp);
  if (worst >= 0) { *bad = worst; return ORC_ERR_ZERO_PIVOT; }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Exact ILU on S (the fixed point of the sweep map):        */
/* row-wise IKJ Gaussian elimination of `ahat` restricted to S, pivots k in   */
/* ascending order, the same operation order as orc_sweep.                    */
/* ------------------------------------------------------------------------ */
int orc_exact_ilu(int64_t n, const int64_t *srp, const int32_t *sci,
                  const double *ahat, double *vals, int64_t *bad) {
  *bad = -1;
  for (int64_t p = 0; p < srp[n]; p++) vals[p] = ahat[p];
  for (int64_t i = 0; i < n; i++) {
    for (int64_t q = srp[i]; q < srp[i + 1] && sci[q] < i; q++) {
      int32_t k = sci[q];
      int64_t pkk = find_in_row(srp, sci, k, k);
      double ukk = vals[pkk];
      if (ukk == 0.0 || !isfinite(ukk)) { *bad = k; return ORC_ERR_ZERO_PIVOT; }
      vals[q] = vals[q] / ukk; /* l_ik */
      for (int64_t r = pkk + 1; r < srp[k + 1]; r++) {
        int32_t j = sci[r];
        int64_t pij = find_in_row(srp, sci, i, j);
        if (pij < 0) continue;
        double prod = vals[q] * vals[r];
        vals[pij] = vals[pij] - prod;
      }
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* FastSpTRSV (reading R6).                            */
/* Lower: z0 = 0; z(t)_i = y_i - sum_{j<i, ascending} l_ij z(t-1)_j.          */
/* Upper: w0 = 0; w(t)_i = (z_i - sum_{j>i, ascending} u_ij w(t-1)_j) / u_ii. */
/* Damped: x(t) = (1-w) x(t-1) + w * (update) when w != 1.                    */
/* ------------------------------------------------------------------------ */
void orc_jacobi_lower(int64_t n, const int64_t *srp, const int32_t *sci,
                      const double *vals, const double *y, int ntri,
                      double omega, double *z) {
  double *zo = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t i = 0; i < n; i++) z[i] = 0.0;
  for (int t = 1; t <= ntri; t++) {
    memcpy(zo, z, sizeof(double) * (size_t)n);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) {
      double acc = y[i];
      for (int64_t p = srp[i]; p < srp[i + 1] && sci[p] < i; p++) {
        double prod = vals[p] * zo[sci[p]];
        acc = acc - prod;
      }
      z[i] = (omega == 1.0) ? acc : (1.0 - omega) * zo[i] + omega * acc;
    }
  }
  free(zo);
}

void orc_jacobi_upper(int64_t n, const int64_t *srp, const int32_t *sci,
                      const double *vals, const double *z, int ntri,
                      double omega, double *w) {
  double *wo = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  for (int64_t i = 0; i < n; i++) w[i] = 0.0;
  for (int t = 1; t <= ntri; t++) {
    memcpy(wo, w, sizeof(double) * (size_t)n);
#pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t i = 0; i < n; i++) {
      double acc = z[i];
      double d = 0.0;
      for (int64_t p = srp[i]; p < srp[i + 1]; p++) {
        int32_t j = sci[p];
        if (j == i) d = vals[p];
        if (j <= i) continue;
        double prod = vals[p] * wo[j];
        acc = acc - prod;
      }
      double upd = acc / d;
      w[i] = (omega == 1.0) ? upd : (1.0 - omega) * wo[i] + omega * upd;
    }
  }
  free(wo);
}

/* x = s o U^-1 L^-1 (s o b), both inverses replaced by ntri Jacobi sweeps */
void orc_apply(int64_t n, const int64_t *srp, const int32_t *sci,
               const double *vals, const double *s, const double *b, int ntri,
               double omega_tri, double *x) {
  double *y = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *z = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double *w = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; i++) y[i] = s[i] * b[i];
  orc_jacobi_lower(n, srp, sci, vals, y, ntri, omega_tri, z);
  orc_jacobi_upper(n, srp, sci, vals, z, ntri, omega_tri, w);
  for (int64_t i = 0; i < n; i++) x[i] = s[i] * w[i];
  free(y); free(z); free(w);
}

/* exact forward / backward substitution with the same per-row order */
void orc_subst_lower(int64_t n, const int64_t *srp, const int32_t *sci,
                     const double *vals, const double *y, double *z) {
  for (int64_t i = 0; i < n; i++) {
    double acc = y[i];
    for (int64_t p = srp[i]; p < srp[i + 1] && sci[p] < i; p++) {
      double prod = vals[p] * z[sci[p]];
      acc = acc - prod;
    }
    z[i] = acc;
  }
}

void orc_subst_upper(int64_t n, const int64_t *srp, const int32_t *sci,
                     const double *vals, const double *z, double *w) {
  for (int64_t i = n - 1; i >= 0; i--) {
    double acc = z[i];
    double d = 0.0;
    for (int64_t p = srp[i]; p < srp[i + 1]; p++) {
      int32_t j = sci[p];
      if (j == i) d = vals[p];
      if (j <= i) continue;
      double prod = vals[p] * w[j];
      acc = acc - prod;
    }
    w[i] = acc / d;
  }
}
