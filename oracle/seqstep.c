/*
 * seqstep.c — ORACLE / CPU baseline only (test infrastructure; see oracle/__init__.py).
 *
 * Plain sequential time stepping u^{n+1} = Phi u^n, u^0 = u0 for an explicit
 * Runge-Kutta scheme over a periodic upwind stencil, in the Runge-Kutta stage form of
 * oracle/discretization.py (RKPhi.__call__, Lemma 1):
 *     k_i = Z (u + sum_{l<i, a_il != 0} a_il k_l),   Phi u = u + sum_{i, b_i != 0} b_i k_i,
 *     (Z y)_j = sum_d z_d y_{(j+d) mod nx}, d ascending,
 * with the same operation order as the numpy oracle and no FMA contraction (built with
 * -ffp-contract=off), so its result is bitwise the numpy oracle's sequential() (pinned in
 * tests/test_oracle_seqstep.py).  The coefficients (z_d, A, b) are passed in by the caller
 * from oracle.discretization.  OpenMP splits each stage over space (the only parallelism
 * sequential stepping has); `threads` = 1 is the single-core baseline.
 *
 * This is the paper's serial baseline ("sequential time-stepping"), timed by
 * bench.py as `cpu_sequential` on the GPU box's host cores.
 */
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXS 6

/* Returns 0 on success, -1 on bad arguments / allocation failure.  u (nx doubles) is
 * advanced in place by nsteps steps. */
int seq_steps(int nx, long long nsteps, int s, const double *A /* s x s row-major */,
              const double *b, int zlo, int zn, const double *z, double *u, int threads) {
  if (nx < 1 || s < 1 || s > MAXS || zn < 1 || !A || !b || !z || !u || nsteps < 0) return -1;
  double *k = (double *)malloc(sizeof(double) * (size_t)nx * (size_t)s);
  double *y = (double *)malloc(sizeof(double) * (size_t)nx);
  if (!k || !y) {
    free(k);
    free(y);
    return -1;
  }
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#else
  (void)threads;
#endif
  for (long long n = 0; n < nsteps; ++n) {
    for (int i = 0; i < s; ++i) {
      double *ki = k + (size_t)i * nx;
#pragma omp parallel for schedule(static)
      for (int j = 0; j < nx; ++j) {
        double yj = u[j];
        for (int l = 0; l < i; ++l)
          if (A[i * s + l] != 0.0) yj = yj + A[i * s + l] * k[(size_t)l * nx + j];
        y[j] = yj;
      }
#pragma omp parallel for schedule(static)
      for (int j = 0; j < nx; ++j) {
        int q = (j + zlo) % nx;
        if (q < 0) q += nx;
        double acc = z[0] * y[q];
        for (int d = 1; d < zn; ++d) {
          q = (q + 1 == nx) ? 0 : q + 1;
          acc = acc + z[d] * y[q];
        }
        ki[j] = acc;
      }
    }
#pragma omp parallel for schedule(static)
    for (int j = 0; j < nx; ++j) {
      double o = u[j];
      for (int i = 0; i < s; ++i)
        if (b[i] != 0.0) o = o + b[i] * k[(size_t)i * nx + j];
      u[j] = o;
    }
  }
  free(k);
  free(y);
  return 0;
}
