/*
 * mmref.c — the CPU ORACLE for the dense product C = A·B.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA path under
 * paper_2408_15384_b200/, and neither side includes the other.
 *
 * What it computes (§III, the displayed equation):
 *     C[i][j] = sum_{k=1..n} A[i][k] * B[k][j],   A m×n, B n×p, C m×p,
 * element by element as the dot product of row i of A with column j of B
 * (§III itemize), repeated for all i, j.
 * Storage is dense row-major: (i,j) at i*cols + j.
 *
 * The oracle IS that definition written out: one accumulator per element,
 * k ascending (the paper's k = 1..n shifted to 0..n-1), each step
 * `s = s + a*b` with a separately rounded multiply and add (built with
 * -ffp-contract=off; reading R5).
 *
 *  - mmref_f64_ijk : the literal i-j-k loop of the definition.
 *  - mmref_f64     : the same per-element arithmetic with the j loop inside
 *                    the k loop (i-k-j).  Every C[i][j] still sees exactly
 *                    s=0; s=s+A[i][0]B[0][j]; s=s+A[i][1]B[1][j]; ... so the
 *                    result is bit-identical to the i-j-k form; the test
 *                    suite pins that identity (tests/test_oracle.py).
 *  - mmref_bf16    : bf16 inputs decoded exactly, accumulated in double
 *                    (reading R4: "FP32 accumulate" is a property
 *                    of the GPU path; the reference is near-exact).
 *  - mmref_s8      : int8 inputs, int64 accumulation (exact).
 *  - *_absden      : D[i][j] = sum_k |A[i][k]*B[k][j]|, the normaliser of the
 *                    tolerance in BASELINE.json north_star.
 *  - *_rows / *_cols : the same loops restricted to chosen rows / columns
 *                    (for shapes whose full product is too slow).
 *
 * OpenMP parallelises over output rows only (the paper's own parallel
 * method, §III-B1 "one line of code above the algorithm");
 * it never splits a sum.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int mmref_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* exact bf16 -> double: a bf16 bit pattern is the high half of an IEEE fp32 */
static inline double bf16_to_double(uint16_t b) {
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return (double)f;
}

/* ------------------------------ FP64 ------------------------------ */

void mmref_f64_ijk(int64_t m, int64_t n, int64_t p, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < p; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < n; ++k) s = s + A[i * n + k] * B[k * p + j];
      C[i * p + j] = s;
    }
}

void mmref_f64(int64_t m, int64_t n, int64_t p, const double* A, const double* B, double* C) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    double* c = C + i * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = A[i * n + k];
      const double* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) c[j] = c[j] + a * b[j];
    }
  }
}

void mmref_f64_absden(int64_t m, int64_t n, int64_t p, const double* A, const double* B, double* D) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    double* d = D + i * p;
    for (int64_t j = 0; j < p; ++j) d[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = A[i * n + k];
      const double* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) d[j] = d[j] + fabs(a * b[j]);
    }
  }
}

/* rows[r] selects output row i = rows[r]; C, D are nrows × p */
void mmref_f64_rows(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                    int64_t nrows, const int64_t* rows, double* C, double* D) {
  (void)m;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    double* c = C + r * p;
    double* d = D + r * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0.0, d[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = A[i * n + k];
      const double* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) {
        c[j] = c[j] + a * b[j];
        d[j] = d[j] + fabs(a * b[j]);
      }
    }
  }
}

/* cols[c] selects output column j = cols[c]; C, D are m × ncols */
void mmref_f64_cols(int64_t m, int64_t n, int64_t p, const double* A, const double* B,
                    int64_t ncols, const int64_t* cols, double* C, double* D) {
  /* gather the selected columns of B once (a copy, no arithmetic); the
   * per-element sum is still s = s + A[i][k]*B[k][j], k ascending */
  double* Bc = (double*)malloc((size_t)(n * ncols) * sizeof(double));
  for (int64_t k = 0; k < n; ++k)
    for (int64_t c = 0; c < ncols; ++c) Bc[k * ncols + c] = B[k * p + cols[c]];
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    double* c_ = C + i * ncols;
    double* d_ = D + i * ncols;
    for (int64_t c = 0; c < ncols; ++c) c_[c] = 0.0, d_[c] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = A[i * n + k];
      for (int64_t c = 0; c < ncols; ++c) {
        c_[c] = c_[c] + a * Bc[k * ncols + c];
        d_[c] = d_[c] + fabs(a * Bc[k * ncols + c]);
      }
    }
  }
  free(Bc);
}

/* ------------------------------ BF16 ------------------------------ */
/* A, B are raw bf16 bit patterns.  Products of two bf16 values are exact in
 * double (8+8 significant bits), so only the additions round. */

void mmref_bf16(int64_t m, int64_t n, int64_t p, const uint16_t* A, const uint16_t* B, double* C, double* D) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    double* c = C + i * p;
    double* d = D + i * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0.0, d[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = bf16_to_double(A[i * n + k]);
      const uint16_t* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) {
        const double ab = a * bf16_to_double(b[j]);
        c[j] = c[j] + ab;
        d[j] = d[j] + fabs(ab);
      }
    }
  }
}

void mmref_bf16_rows(int64_t m, int64_t n, int64_t p, const uint16_t* A, const uint16_t* B,
                     int64_t nrows, const int64_t* rows, double* C, double* D) {
  (void)m;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    double* c = C + r * p;
    double* d = D + r * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0.0, d[j] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = bf16_to_double(A[i * n + k]);
      const uint16_t* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) {
        const double ab = a * bf16_to_double(b[j]);
        c[j] = c[j] + ab;
        d[j] = d[j] + fabs(ab);
      }
    }
  }
}

void mmref_bf16_cols(int64_t m, int64_t n, int64_t p, const uint16_t* A, const uint16_t* B,
                     int64_t ncols, const int64_t* cols, double* C, double* D) {
  /* gather the selected columns of B once (a copy, no arithmetic) so the
   * inner loop streams; the per-element sum is still k ascending */
  double* Bc = (double*)malloc((size_t)(n * ncols) * sizeof(double));
  for (int64_t k = 0; k < n; ++k)
    for (int64_t c = 0; c < ncols; ++c) Bc[k * ncols + c] = bf16_to_double(B[k * p + cols[c]]);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    double* c_ = C + i * ncols;
    double* d_ = D + i * ncols;
    for (int64_t c = 0; c < ncols; ++c) c_[c] = 0.0, d_[c] = 0.0;
    for (int64_t k = 0; k < n; ++k) {
      const double a = bf16_to_double(A[i * n + k]);
      for (int64_t c = 0; c < ncols; ++c) {
        const double ab = a * Bc[k * ncols + c];
        c_[c] = c_[c] + ab;
        d_[c] = d_[c] + fabs(ab);
      }
    }
  }
  free(Bc);
}

/* ------------------------------ INT8 ------------------------------ */
/* int8 × int8 products fit in int32 (|ab| <= 128^2); sums kept in int64,
 * so the result is the exact integer (no wrap). */

void mmref_s8(int64_t m, int64_t n, int64_t p, const int8_t* A, const int8_t* B, int64_t* C) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = 0; i < m; ++i) {
    int64_t* c = C + i * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t a = A[i * n + k];
      const int8_t* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) c[j] = c[j] + a * (int64_t)b[j];
    }
  }
}

void mmref_s8_rows(int64_t m, int64_t n, int64_t p, const int8_t* A, const int8_t* B,
                   int64_t nrows, const int64_t* rows, int64_t* C) {
  (void)m;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nrows; ++r) {
    const int64_t i = rows[r];
    int64_t* c = C + r * p;
    for (int64_t j = 0; j < p; ++j) c[j] = 0;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t a = A[i * n + k];
      const int8_t* b = B + k * p;
      for (int64_t j = 0; j < p; ++j) c[j] = c[j] + a * (int64_t)b[j];
    }
  }
}
