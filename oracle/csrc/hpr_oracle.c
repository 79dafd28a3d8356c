/* HPR-LP oracle kernels -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain-C restatement of the reference's per-iteration arithmetic, used as the
 * parity checker's fast path and as the timed CPU baseline:
 *   orc_matvec  -- SparseMatrix.apply / t_apply (reference sparse.py:102-108),
 *                  i.e. scipy csr_matvec: sum starts at 0.0 and adds the
 *                  separately rounded products left to right; no FMA.
 *   orc_xphase  -- core.py:168-169 (v, xb) and core.py:149-153 (x update)
 *   orc_yphase  -- core.py:170-172 (yb, dual-cone clamp) and core.py:149-153
 * Rows are independent, so OpenMP across rows keeps every row's summation order
 * and the result is bit-identical for any thread count.
 * Build: oracle/Makefile (-O2 -ffp-contract=off, no -march: no FMA is emitted).
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* numpy's maximum/minimum/clip semantics: NaN in the first operand wins, ties
 * return the second operand (matters only for the sign of zero). */
static inline double np_max(double a, double b) { return (isnan(a) || a > b) ? a : b; }
static inline double np_min(double a, double b) { return (isnan(a) || a < b) ? a : b; }

int orc_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

static inline double row_dot(const int64_t *rp, const int64_t *ci, const double *v,
                             const double *x, int64_t i) {
  double s = 0.0;
  for (int64_t k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
  return s;
}

void orc_matvec(int64_t nrows, const int64_t *rp, const int64_t *ci, const double *v,
                const double *x, double *out) {
#pragma omp parallel for schedule(static, 2048)
  for (int64_t i = 0; i < nrows; ++i) out[i] = row_dot(rp, ci, v, x, i);
}

/* variant: 0 = DR, 1 = HDR family, 2 = HPR.  Returns 1 if any new x is non-finite. */
int orc_xphase(int64_t n, const int64_t *rpt, const int64_t *cit, const double *vt,
               const double *y, const double *x, const double *c, const double *lo,
               const double *up, const double *anc_x, double *xb_out, double *w_out,
               double *xn_out, double sigma, int64_t t, int variant) {
  const double t2 = (double)t + 2.0;
  const double wn = ((double)t + 1.0) / t2;
  const double wa = 1.0 / t2;
  int bad = 0;
#pragma omp parallel for schedule(static, 2048) reduction(| : bad)
  for (int64_t j = 0; j < n; ++j) {
    double aty = row_dot(rpt, cit, vt, y, j);
    double v = x[j] + sigma * (aty - c[j]);
    double xb = np_min(np_max(v, lo[j]), up[j]);
    double w = 2.0 * xb - x[j];
    double xn;
    if (variant == 0) xn = xb;
    else if (variant == 1) xn = wa * anc_x[j] + wn * xb;
    else xn = wa * anc_x[j] + wn * w;
    xb_out[j] = xb;
    w_out[j] = w;
    xn_out[j] = xn;
    bad |= !isfinite(xn);
  }
  return bad;
}

int orc_yphase(int64_t m, int64_t m1, const int64_t *rp, const int64_t *ci, const double *v,
               const double *w, const double *y, const double *b, const double *anc_y,
               double *yb_out, double *yn_out, double lamsig, int64_t t, int variant) {
  const double t2 = (double)t + 2.0;
  const double wn = ((double)t + 1.0) / t2;
  const double wa = 1.0 / t2;
  int bad = 0;
#pragma omp parallel for schedule(static, 2048) reduction(| : bad)
  for (int64_t i = 0; i < m; ++i) {
    double s = row_dot(rp, ci, v, w, i);
    double yb = y[i] + (b[i] - s) / lamsig;
    if (i >= m1) yb = np_max(yb, 0.0);
    double yn;
    if (variant == 0) yn = yb;
    else if (variant == 1) yn = wa * anc_y[i] + wn * yb;
    else yn = wa * anc_y[i] + wn * (2.0 * yb - y[i]);
    yb_out[i] = yb;
    yn_out[i] = yn;
    bad |= !isfinite(yn);
  }
  return bad;
}
