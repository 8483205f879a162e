/* Extended-precision (x87 80-bit long double) matrix product for the oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): called by oracle/xprec.py
 * (mm_ld) to form the long-double products of the reference-element build
 * (DESIGN.md R-A24). numpy's longdouble matmul has no BLAS and holds the GIL;
 * this is the same textbook loop, C[i][j] = sum_k A[i][k] B[k][j] with k
 * ascending from C[i][j] = 0 -- the order numpy's non-BLAS matmul uses, so the
 * results are bitwise identical (tests/test_oracle_xprec.py) -- with rows of C
 * spread over OpenMP threads. Row-major, contiguous operands.
 */
#include <stdint.h>

void ld_gemm(const long double* A, const long double* B, long double* C, int64_t m, int64_t k, int64_t n) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t i = 0; i < m; ++i) {
    long double* c = C + i * n;
    for (int64_t j = 0; j < n; ++j) c[j] = 0.0L;
    const long double* a = A + i * k;
    for (int64_t l = 0; l < k; ++l) {
      const long double ail = a[l];
      const long double* b = B + l * n;
      for (int64_t j = 0; j < n; ++j) c[j] += ail * b[j];
    }
  }
}
