/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library,
 * and only as the checker or the CPU baseline -- never on the product path.
 *
 * Plain-C restatement of the reference's CPU MTTKRP kernels
 * (pkg/src/cpkern/_kernels.py, numba @njit):
 *
 *   orc_mttkrp_ref   -- ref_kernel (_kernels.py:39-57): serial, elements in
 *                       linear order, div/mod ind2sub per element, all R
 *                       columns, p = lam[j]*y*A_0*A_1*... (modes ascending,
 *                       k skipped), out[row, j] += p.  The canonical order.
 *   orc_mttkrp_tile  -- tile_kernel + accum_tile (_kernels.py:96-174) with the
 *                       reference's private-copy merge (mttkrp.py:279-286):
 *                       tiles enumerated slice-major, odometer walk, column
 *                       blocks of width F, per-thread private output copies
 *                       summed in thread order.  OpenMP replaces numba's prange.
 *   orc_mttkrp_rows  -- ref_kernel restricted to chosen output rows: walks
 *                       each requested slice in first-mode-fastest order (the
 *                       single-slice sub-tensor trick of SURVEY.md 8(c)),
 *                       for row-sampled parity at sizes the serial oracle
 *                       cannot finish in full.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_MAX_MODES 16

/* factors: array of d row-major (I_m x R) pointers; lam may be NULL (unit). */
int orc_mttkrp_ref(const double* data, int d, const int64_t* dims, int k, const double* const* fac,
                   const double* lam, int64_t R, double* out) {
  if (d < 1 || d > ORC_MAX_MODES || k < 0 || k >= d) return 1;
  int64_t n = 1;
  for (int m = 0; m < d; ++m) n *= dims[m];
  int64_t sub[ORC_MAX_MODES];
  for (int64_t i = 0; i < n; ++i) {
    int64_t rem = i;
    for (int m = 0; m < d; ++m) {
      sub[m] = rem % dims[m];
      rem /= dims[m];
    }
    const double y = data[i];
    double* row = out + sub[k] * R;
    for (int64_t j = 0; j < R; ++j) {
      double p = (lam ? lam[j] : 1.0) * y;
      for (int m = 0; m < d; ++m)
        if (m != k) p *= fac[m][sub[m] * R + j];
      row[j] += p;
    }
  }
  return 0;
}

/* accum_tile (_kernels.py:96-150): one tile = slice n, in-slice offsets
 * [t0, t0 + tlen), column blocks of width f_cols; block sums land in grow. */
static void accum_tile(const double* data, int d, const int64_t* dims, const int64_t* strides, int k,
                       const double* const* fac, const double* lam, int64_t R, int64_t f_cols, int64_t n,
                       int64_t t0, int64_t tlen, double* grow, double* pi) {
  int64_t dig0[ORC_MAX_MODES], dig[ORC_MAX_MODES];
  int64_t rem = t0, flat0 = n * strides[k];
  for (int m = 0; m < d; ++m) {
    if (m == k) {
      dig0[m] = 0;
    } else {
      dig0[m] = rem % dims[m];
      rem /= dims[m];
      flat0 += dig0[m] * strides[m];
    }
  }
  for (int64_t jj = 0; jj < R; jj += f_cols) {
    const int64_t fw = (R - jj < f_cols) ? R - jj : f_cols;
    for (int64_t f = 0; f < fw; ++f) pi[f] = 0.0;
    memcpy(dig, dig0, sizeof(int64_t) * d);
    int64_t flat = flat0;
    for (int64_t ii = 0; ii < tlen; ++ii) {
      const double y = data[flat];
      for (int64_t f = 0; f < fw; ++f) {
        const int64_t j = jj + f;
        double p = (lam ? lam[j] : 1.0) * y;
        for (int m = 0; m < d; ++m)
          if (m != k) p *= fac[m][dig[m] * R + j];
        pi[f] += p;
      }
      if (ii + 1 < tlen) {
        for (int m = 0; m < d; ++m) {
          if (m == k) continue;
          dig[m] += 1;
          flat += strides[m];
          if (dig[m] < dims[m]) break;
          flat -= dig[m] * strides[m];
          dig[m] = 0;
        }
      }
    }
    for (int64_t f = 0; f < fw; ++f) grow[jj + f] += pi[f];
  }
}

/* tile_kernel (_kernels.py:162-174) + _run_private_copy (mttkrp.py:279-286).
 * workers <= 0: all OpenMP threads.  Returns the worker count used. */
int orc_mttkrp_tile(const double* data, int d, const int64_t* dims, int k, const double* const* fac,
                    const double* lam, int64_t R, int64_t f_cols, int64_t n_t, int workers, double* out) {
  if (d < 1 || d > ORC_MAX_MODES || k < 0 || k >= d || f_cols < 1 || n_t < 1) return -1;
  int64_t strides[ORC_MAX_MODES], n = 1;
  for (int m = 0; m < d; ++m) {
    strides[m] = n;
    n *= dims[m];
  }
  const int64_t i_k = dims[k], n_s = n / i_k;
  if (n_t > n_s) n_t = n_s;
  const int64_t tps = (n_s + n_t - 1) / n_t;
  int w = 1;
#ifdef _OPENMP
  w = workers > 0 ? workers : omp_get_max_threads();
#endif
  double* gp = (double*)calloc((size_t)w * (size_t)(i_k * R), sizeof(double));
  if (!gp) return -2;
#ifdef _OPENMP
#pragma omp parallel num_threads(w)
#endif
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* pi = (double*)malloc(sizeof(double) * (size_t)f_cols);
    double* mine = gp + (size_t)tid * (size_t)(i_k * R);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
    for (int64_t wi = 0; wi < i_k * tps; ++wi) {
      const int64_t nn = wi / tps, t0 = (wi % tps) * n_t;
      const int64_t tlen = (n_t < n_s - t0) ? n_t : n_s - t0;
      accum_tile(data, d, dims, strides, k, fac, lam, R, f_cols, nn, t0, tlen, mine + nn * R, pi);
    }
    free(pi);
  }
  memset(out, 0, sizeof(double) * (size_t)(i_k * R));
  for (int t = 0; t < w; ++t)
    for (int64_t e = 0; e < i_k * R; ++e) out[e] += gp[(size_t)t * (size_t)(i_k * R) + e];
  free(gp);
  return w;
}

/* Rows `rows[0..nr)` of G only: out is nr x R.  Each requested slice is
 * walked in the reference's in-slice order (slice_ind2sub, dtensor.py:97-122),
 * so out[r] equals G[rows[r]] of orc_mttkrp_ref bit for bit. */
int orc_mttkrp_rows(const double* data, int d, const int64_t* dims, int k, const double* const* fac,
                    const double* lam, int64_t R, const int64_t* rows, int64_t nr, double* out) {
  if (d < 1 || d > ORC_MAX_MODES || k < 0 || k >= d) return 1;
  int64_t strides[ORC_MAX_MODES], n = 1;
  for (int m = 0; m < d; ++m) {
    strides[m] = n;
    n *= dims[m];
  }
  const int64_t n_s = n / dims[k];
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t r = 0; r < nr; ++r) {
    int64_t dig[ORC_MAX_MODES];
    for (int m = 0; m < d; ++m) dig[m] = 0;
    dig[k] = rows[r];
    int64_t flat = rows[r] * strides[k];
    double* row = out + r * R;
    for (int64_t j = 0; j < R; ++j) row[j] = 0.0;
    for (int64_t ii = 0; ii < n_s; ++ii) {
      const double y = data[flat];
      for (int64_t j = 0; j < R; ++j) {
        double p = (lam ? lam[j] : 1.0) * y;
        for (int m = 0; m < d; ++m)
          if (m != k) p *= fac[m][dig[m] * R + j];
        row[j] += p;
      }
      for (int m = 0; m < d; ++m) {
        if (m == k) continue;
        dig[m] += 1;
        flat += strides[m];
        if (dig[m] < dims[m]) break;
        flat -= dig[m] * strides[m];
        dig[m] = 0;
      }
    }
  }
  return 0;
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
