/*
 * Plain-C oracle of the ILUt preconditioner of S and of its triangular solves
 * (the paper's "Sparsification method as a preconditioner",
 * "sparsified and factorized with ILUt decomposition").
 * TEST INFRASTRUCTURE ONLY (oracle/__init__.py): nothing here is part of, or
 * shared with, the CUDA path.
 *
 * The paper names ILUt and its drop tolerance tau but
 * does not define it; reading 25 takes Saad's ILUT(tau, p)
 * ("Iterative Methods for Sparse Linear Systems", Algorithm 10.6, IKJ
 * variant, with its dual dropping rule), written out here step by step:
 *
 *   for i = 0 .. n-1:
 *     tau_i := tau * ||a_i*||_2        (row 2-norm, summed in column order)
 *     w := a_i*
 *     for k = 0 .. i-1 with w_k present:
 *       w_k := w_k / u_kk
 *       rule 1: drop w_k if |w_k| < tau_i or w_k == 0
 *       if w_k kept: w := w - w_k * u_k*   (u_k* = strict upper part of U row k)
 *     rule 2: drop w_j (j != i) if |w_j| < tau_i or w_j == 0; then keep only
 *             the p largest |w_j| of the L part (j < i) and the p largest of
 *             the strict U part (j > i); ties go to the smaller column
 *             (reading 25); p < 0 keeps all.  The diagonal is always kept.
 *     l_ij := w_j (j < i, unit diagonal implied); u_ii := w_i; u_ij := w_j (j > i)
 *
 * Every update is the two-rounding w_j - (w_k * u_kj) (no fused multiply-add:
 * compile with -ffp-contract=off), in increasing k, the order of the
 * algorithm.  The "w_k present" scan is a plain linear scan over k.
 *
 * Outputs: L (strict lower, CSR, ascending columns), U (strict upper, CSR,
 * ascending columns) and diag = u_ii.  Return: 0 ok, 1 capacity too small,
 * 2 zero pivot (u_ii == 0 at row *bad_row).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double v;
  int32_t c;
} ent;

/* (|v| descending, column ascending) */
static int by_mag(const void *a, const void *b) {
  const ent *x = (const ent *)a, *y = (const ent *)b;
  const double ax = fabs(x->v), ay = fabs(y->v);
  if (ax > ay) return -1;
  if (ax < ay) return 1;
  return (x->c > y->c) - (x->c < y->c);
}

static int by_col(const void *a, const void *b) {
  const ent *x = (const ent *)a, *y = (const ent *)b;
  return (x->c > y->c) - (x->c < y->c);
}

/* keep the p largest of e[0..m) (all if p < 0 or m <= p); returns the count
 * kept, sorted by column */
static int64_t keep_largest(ent *e, int64_t m, int p) {
  if (p >= 0 && m > p) {
    qsort(e, (size_t)m, sizeof(ent), by_mag);
    m = p;
  }
  qsort(e, (size_t)m, sizeof(ent), by_col);
  return m;
}

int oracle_ilut(int64_t n, const int64_t *rp, const int32_t *ci, const double *av, double tau, int p,
                int64_t *lrp, int32_t *lci, double *lv, int64_t lcap, int64_t *urp, int32_t *uci, double *uv,
                int64_t ucap, double *diag, int64_t *bad_row) {
  double *w = (double *)calloc((size_t)n, sizeof(double));
  char *present = (char *)calloc((size_t)n, 1);
  int32_t *touched = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  ent *cand = (ent *)malloc((size_t)n * sizeof(ent));
  int rc = 0;
  lrp[0] = 0;
  urp[0] = 0;
  for (int64_t i = 0; i < n && rc == 0; i++) {
    int64_t nt = 0;
    double s = 0.0;
    for (int64_t e = rp[i]; e < rp[i + 1]; e++) s = s + av[e] * av[e];
    const double taui = tau * sqrt(s);
    for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
      w[ci[e]] = av[e];
      present[ci[e]] = 1;
      touched[nt++] = ci[e];
    }
    for (int64_t k = 0; k < i; k++) {
      if (!present[k]) continue;
      const double wk = w[k] / diag[k];
      if (fabs(wk) < taui || wk == 0.0) {  /* rule 1 */
        w[k] = 0.0;
        present[k] = 0;
        continue;
      }
      w[k] = wk;
      for (int64_t e = urp[k]; e < urp[k + 1]; e++) {
        const int32_t j = uci[e];
        const double prod = wk * uv[e];
        w[j] = w[j] - prod;
        if (!present[j]) {
          present[j] = 1;
          touched[nt++] = j;
        }
      }
    }
    /* rule 2, L part */
    int64_t m = 0;
    for (int64_t k = 0; k < i; k++)
      if (present[k]) {
        cand[m].v = w[k];
        cand[m].c = (int32_t)k;
        m++;
      }
    m = keep_largest(cand, m, p);
    if (lrp[i] + m > lcap) {
      rc = 1;
      break;
    }
    for (int64_t a = 0; a < m; a++) {
      lci[lrp[i] + a] = cand[a].c;
      lv[lrp[i] + a] = cand[a].v;
    }
    lrp[i + 1] = lrp[i] + m;
    /* rule 2, U part */
    m = 0;
    for (int64_t j = i + 1; j < n; j++)
      if (present[j] && !(fabs(w[j]) < taui || w[j] == 0.0)) {
        cand[m].v = w[j];
        cand[m].c = (int32_t)j;
        m++;
      }
    m = keep_largest(cand, m, p);
    if (urp[i] + m > ucap) {
      rc = 1;
      break;
    }
    for (int64_t a = 0; a < m; a++) {
      uci[urp[i] + a] = cand[a].c;
      uv[urp[i] + a] = cand[a].v;
    }
    urp[i + 1] = urp[i] + m;
    diag[i] = w[i];
    if (w[i] == 0.0) {
      rc = 2;
      *bad_row = i;
    }
    for (int64_t a = 0; a < nt; a++) {
      w[touched[a]] = 0.0;
      present[touched[a]] = 0;
    }
  }
  free(w);
  free(present);
  free(touched);
  free(cand);
  return rc;
}

/* x = (L U)^{-1} b: forward substitution with the unit lower L, then backward
 * substitution with U (diagonal diag); plain row loops in column order. */
void oracle_ilu_solve(int64_t n, const int64_t *lrp, const int32_t *lci, const double *lv, const int64_t *urp,
                      const int32_t *uci, const double *uv, const double *diag, const double *b, double *x) {
  for (int64_t i = 0; i < n; i++) {
    double s = b[i];
    for (int64_t e = lrp[i]; e < lrp[i + 1]; e++) s = s - lv[e] * x[lci[e]];
    x[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; i--) {
    double s = x[i];
    for (int64_t e = urp[i]; e < urp[i + 1]; e++) s = s - uv[e] * x[uci[e]];
    x[i] = s / diag[i];
  }
}
