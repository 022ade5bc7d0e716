/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Plain-C restatement of the reference's
 * native GEPP kernel; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, as the checker.  The product never links it.
 *
 * Restates rlra/_lu_cython.pyx:14-55 (twin: rlra/_lu_numpy.py:14-40),
 * loop for loop:
 *   - pivot = FIRST maximum of |a[i,j]| over i >= j (strict '>' scan, :24-30)
 *   - colmax spans the WHOLE column, rows < j included (:31-35)
 *   - zero pivot (amax <= 1e-14 * colmax): zero L below the diagonal, no swap,
 *     no update (:36-39)
 *   - full-row swap and piv swap (:40-48)
 *   - divide by the pivot, not reciprocal-multiply (:49-51)
 *   - rank-1 update, multiply then subtract, no FMA (:52-55; built with
 *     -ffp-contract=off exactly like pkg/setup.py:27)
 * Storage is column-major with leading dimension ld (>= m).
 */
#include <math.h>
#include <stdint.h>

static const double ZERO_PIVOT_RTOL = 1e-14; /* rlra/_lu_cython.pyx:11 */

#define A(i, j) lu[(int64_t)(i) + (int64_t)(j) * ld]

void oracle_plu_inplace(double* lu, int64_t m, int64_t n, int64_t ld, int64_t* piv) {
  int64_t r = m < n ? m : n;
  for (int64_t j = 0; j < r; j++) {
    double amax = -1.0;
    int64_t rel = j;
    for (int64_t i = j; i < m; i++) {
      double v = fabs(A(i, j));
      if (v > amax) { amax = v; rel = i; }
    }
    double colmax = amax;
    for (int64_t i = 0; i < j; i++) {
      double v = fabs(A(i, j));
      if (v > colmax) colmax = v;
    }
    if (amax <= ZERO_PIVOT_RTOL * colmax) {
      for (int64_t i = j + 1; i < m; i++) A(i, j) = 0.0;
      continue;
    }
    int64_t prow = rel;
    if (prow != j) {
      for (int64_t jj = 0; jj < n; jj++) {
        double t = A(j, jj); A(j, jj) = A(prow, jj); A(prow, jj) = t;
      }
      int64_t pt = piv[j]; piv[j] = piv[prow]; piv[prow] = pt;
    }
    double ljj = A(j, j);
    for (int64_t i = j + 1; i < m; i++) A(i, j) = A(i, j) / ljj;
    for (int64_t jj = j + 1; jj < n; jj++) {
      double ujj = A(j, jj);
      for (int64_t i = j + 1; i < m; i++) A(i, jj) = A(i, jj) - A(i, j) * ujj;
    }
  }
}
