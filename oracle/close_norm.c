/*
 * Plain-C helper of the CPU oracle: squared Frobenius norms of close blocks
 * C_ts[i][j] = K(x_{tB+i}, x_{sB+j}) evaluated from the points (the kernels
 * of BASELINE.json configs, readings 14-15; the same definitions as
 * h2gen.kernel_matrix), for pin P5 at sizes where the blocks are never stored
 * (config 5: ~1e11 entries).  TEST INFRASTRUCTURE ONLY (oracle/__init__.py):
 * nothing here is part of, or shared with, the CUDA path.
 *
 * out[p] = sum_i sum_j C_{t_p s_p}[i][j]^2 in the plain loop order; the pairs
 * are independent (OpenMP over p, one owner per output), so the result does
 * not depend on the thread count.
 */
#include <math.h>
#include <stdint.h>

/* kind 1: exp(-r / p0) + p1 [same point]; 2: 1 / (r + p0) + p1 [same];
 * 3: 1 / (4 pi r), p1 at the same point. */
static double kern(int kind, double r, int same, double p0, double p1) {
  if (kind == 1) return exp(-r / p0) + (same ? p1 : 0.0);
  if (kind == 2) return 1.0 / (r + p0) + (same ? p1 : 0.0);
  return same ? p1 : 1.0 / (4.0 * M_PI * r);
}

void oracle_close_frob_sq(const double *x, int dim, int B, const int32_t *pt, const int32_t *ps, int64_t npairs,
                          int kind, double p0, double p1, double *out) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t p = 0; p < npairs; p++) {
    const double *xt = x + (int64_t)pt[p] * B * dim, *xs = x + (int64_t)ps[p] * B * dim;
    double acc = 0.0;
    for (int i = 0; i < B; i++)
      for (int j = 0; j < B; j++) {
        double r2 = 0.0;
        for (int a = 0; a < dim; a++) {
          const double d = xt[i * dim + a] - xs[j * dim + a];
          r2 += d * d;
        }
        const double v = kern(kind, sqrt(r2), pt[p] == ps[p] && i == j, p0, p1);
        acc += v * v;
      }
    out[p] = acc;
  }
}
