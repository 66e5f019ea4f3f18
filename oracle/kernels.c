/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle, never linked into libaqp.
 *
 * Plain-C restatement of the reference's compiled kernels
 * (/root/reference/pkg/src/anchorqp/_kernels/_core.pyx).  Every loop runs
 * in the same fixed order as the Cython source and the file is compiled
 * with gcc -O2 -ffp-contract=off, so results are bit-identical to the
 * reference's Cython backend (checked in tests/test_oracle.py against the
 * committed golden vectors).  Built by oracle/build_oracle.sh into
 * oracle/_build/liboracle.so.
 */
#include <math.h>
#include <stdint.h>

/* _core.pyx:21-26 */
static inline double clip(double v, double lo, double hi) {
  if (v < lo) return lo;
  if (v > hi) return hi;
  return v;
}

/* _core.pyx:29-42: row-sequential A x */
void orc_csr_matvec(const int64_t *ptr, const int64_t *idx, const double *val, const double *x, int64_t rows,
                    double *out) {
  for (int64_t i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) acc += val[k] * x[idx[k]];
    out[i] = acc;
  }
}

/* _core.pyx:45-59: A' x by row scatter, rows with x_i == 0 skipped */
void orc_csr_matvec_t(const int64_t *ptr, const int64_t *idx, const double *val, const double *x, int64_t rows,
                      int64_t cols, double *out) {
  for (int64_t j = 0; j < cols; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < rows; ++i) {
    const double xi = x[i];
    if (xi == 0.0) continue;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) out[idx[k]] += val[k] * xi;
  }
}

/* _core.pyx:62-80: symmetric product from the upper triangle; the row dot
 * is accumulated privately and added after the mirrored scatters */
void orc_sym_matvec(const int64_t *ptr, const int64_t *idx, const double *val, const double *x, int64_t n,
                    double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k) {
      const int64_t j = idx[k];
      acc += val[k] * x[j];
      if (j != i) out[j] += val[k] * x[i];
    }
    out[i] += acc;
  }
}

/* _core.pyx:83-92 */
void orc_clamp(const double *x, const double *lo, const double *hi, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = clip(x[i], lo[i], hi[i]);
}

/* _core.pyx:95-115; codes ZERO=0 NONNEG=1 NONPOS=2 FREE=3 */
void orc_cone_project(const double *z, const int8_t *codes, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) {
    const double v = z[i];
    switch (codes[i]) {
      case 0: out[i] = 0.0; break;
      case 1: out[i] = v > 0.0 ? v : 0.0; break;
      case 2: out[i] = v < 0.0 ? v : 0.0; break;
      default: out[i] = v;
    }
  }
}

/* _core.pyx:118-128 */
void orc_diag_prox_step(const double *xk, const double *q, const double *lin, double tau, const double *lo,
                        const double *hi, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = clip((xk[i] - tau * lin[i]) / (1.0 + tau * q[i]), lo[i], hi[i]);
}

/* _core.pyx:131-142 */
double orc_natural_res_sq(const double *x, const double *g, const double *lo, const double *hi, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = x[i] - clip(x[i] - g[i], lo[i], hi[i]);
    acc += d * d;
  }
  return acc;
}

/* _core.pyx:145-157 */
void orc_dual_step(const double *y, const double *ax, double sigma, const double *lo, const double *hi, int64_t m,
                   double *out) {
  for (int64_t i = 0; i < m; ++i) {
    const double w = y[i] / sigma + ax[i];
    out[i] = sigma * (w - clip(w, lo[i], hi[i]));
  }
}

/* _core.pyx:160-170 */
void orc_lincomb3(double a, const double *x, double b, const double *y, double c, const double *z, int64_t n,
                  double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = a * x[i] + b * y[i] + c * z[i];
}

/* _core.pyx:173-182 */
void orc_axpby(double a, const double *x, double b, const double *y, int64_t n, double *out) {
  for (int64_t i = 0; i < n; ++i) out[i] = a * x[i] + b * y[i];
}
