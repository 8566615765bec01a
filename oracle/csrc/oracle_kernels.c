/*
 * ORACLE — test infrastructure only.  CPU restatement of the reference's seven
 * data-parallel sweep kernels (reference: pkg/src/patchbeam/_kernels.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It is never the product path.
 *
 * Every loop nest and reduction order mirrors the reference line by line so
 * that, compiled without FP contraction (-ffp-contract=off), results are
 * bit-identical to the reference's Numba kernels:
 *   - per-patch loops are independent (OpenMP over patches),
 *   - cross-patch reductions use fixed 512-patch blocks whose partials are
 *     merged in block order (_kernels.py:15, 42-61, 116-130).
 *
 * Layouts are the reference's: row-major (N,P) values/observed/resid,
 * (N,K) usage/weights, (K,P) atoms; f64 everywhere, observed/usage as uint8.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_BLOCK 512 /* _kernels.py:15 */

/* _kernels.py:18-31 */
void oracle_residual_full(const double *values, const uint8_t *observed,
                          const uint8_t *usage, const double *weights,
                          const double *atoms, double *out, int64_t n,
                          int64_t p_len, int64_t k_len) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    const double *x = values + i * p_len;
    const uint8_t *o = observed + i * p_len;
    double *r = out + i * p_len;
    for (int64_t p = 0; p < p_len; ++p) r[p] = o[p] ? x[p] : 0.0;
    for (int64_t k = 0; k < k_len; ++k) {
      if (usage[i * k_len + k]) {
        double w = weights[i * k_len + k];
        const double *d = atoms + k * p_len;
        for (int64_t p = 0; p < p_len; ++p)
          if (o[p]) r[p] -= w * d[p];
      }
    }
  }
}

/* _kernels.py:34-62 */
void oracle_atom_moments(const double *resid, const uint8_t *observed,
                         const double *w_col, double *a, double *c, int64_t n,
                         int64_t p_len) {
  int64_t nblocks = (n + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
  double *part_a = (double *)calloc((size_t)(nblocks * p_len), sizeof(double));
  double *part_c = (double *)calloc((size_t)(nblocks * p_len), sizeof(double));
  int64_t b;
#pragma omp parallel for schedule(static)
  for (b = 0; b < nblocks; ++b) {
    int64_t lo = b * ORACLE_BLOCK;
    int64_t hi = lo + ORACLE_BLOCK < n ? lo + ORACLE_BLOCK : n;
    double *pa = part_a + b * p_len, *pc = part_c + b * p_len;
    for (int64_t i = lo; i < hi; ++i) {
      double w = w_col[i];
      if (w != 0.0) {
        double w2 = w * w;
        const uint8_t *o = observed + i * p_len;
        const double *r = resid + i * p_len;
        for (int64_t p = 0; p < p_len; ++p) {
          if (o[p]) {
            pa[p] += w2;
            pc[p] += w * r[p];
          }
        }
      }
    }
  }
  for (int64_t p = 0; p < p_len; ++p) { a[p] = 0.0; c[p] = 0.0; }
  for (b = 0; b < nblocks; ++b)
    for (int64_t p = 0; p < p_len; ++p) {
      a[p] += part_a[b * p_len + p];
      c[p] += part_c[b * p_len + p];
    }
  free(part_a);
  free(part_c);
}

/* _kernels.py:65-74 */
void oracle_shift_atom(double *resid, const uint8_t *observed,
                       const double *w_col, const double *delta, int64_t n,
                       int64_t p_len) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double w = w_col[i];
    if (w != 0.0) {
      const uint8_t *o = observed + i * p_len;
      double *r = resid + i * p_len;
      for (int64_t p = 0; p < p_len; ++p)
        if (o[p]) r[p] += w * delta[p];
    }
  }
}

/* _kernels.py:77-97 */
void oracle_code_moments(const double *resid, const uint8_t *observed,
                         const double *atom, double *u, double *v, int64_t n,
                         int64_t p_len) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double acc_u = 0.0, acc_v = 0.0;
    const uint8_t *o = observed + i * p_len;
    const double *r = resid + i * p_len;
    for (int64_t p = 0; p < p_len; ++p) {
      if (o[p]) {
        double d = atom[p];
        acc_u += d * d;
        acc_v += d * r[p];
      }
    }
    u[i] = acc_u;
    v[i] = acc_v;
  }
}

/* _kernels.py:100-109 */
void oracle_shift_codes(double *resid, const uint8_t *observed,
                        const double *atom, const double *dw, int64_t n,
                        int64_t p_len) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double d = dw[i];
    if (d != 0.0) {
      const uint8_t *o = observed + i * p_len;
      double *r = resid + i * p_len;
      for (int64_t p = 0; p < p_len; ++p)
        if (o[p]) r[p] += d * atom[p];
    }
  }
}

/* _kernels.py:112-130 */
double oracle_masked_sq_norm(const double *resid, int64_t n, int64_t p_len) {
  int64_t nblocks = (n + ORACLE_BLOCK - 1) / ORACLE_BLOCK;
  double *part = (double *)calloc((size_t)nblocks, sizeof(double));
  int64_t b;
#pragma omp parallel for schedule(static)
  for (b = 0; b < nblocks; ++b) {
    int64_t lo = b * ORACLE_BLOCK;
    int64_t hi = lo + ORACLE_BLOCK < n ? lo + ORACLE_BLOCK : n;
    double acc = 0.0;
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t p = 0; p < p_len; ++p) {
        double r = resid[i * p_len + p];
        acc += r * r;
      }
    part[b] = acc;
  }
  double total = 0.0;
  for (b = 0; b < nblocks; ++b) total += part[b];
  free(part);
  return total;
}

/* _kernels.py:133-145 */
void oracle_compose_estimates(const uint8_t *usage, const double *weights,
                              const double *atoms, double *out, int64_t n,
                              int64_t k_len, int64_t p_len) {
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    double *e = out + i * p_len;
    for (int64_t p = 0; p < p_len; ++p) e[p] = 0.0;
    for (int64_t k = 0; k < k_len; ++k) {
      if (usage[i * k_len + k]) {
        double w = weights[i * k_len + k];
        const double *d = atoms + k * p_len;
        for (int64_t p = 0; p < p_len; ++p) e[p] += w * d[p];
      }
    }
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
