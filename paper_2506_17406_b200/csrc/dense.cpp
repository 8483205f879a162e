// Host dense SPD inverse of the patch matrices (R-A15, the patch factorisation
// of P:2284-2288 done once at setup): A^-1 = L^-T L^-1 from the Cholesky
// factor A = L L^T. Every O(n^3) step is cast as dot products of contiguous
// rows, evaluated four rows by two rows at a time with AVX2 FMA (8 vector
// accumulators), so the setup of config 3 (4913 patches of ~1140 dofs,
// ~7e12 flop) runs at tens of GFLOP/s per core instead of streaming each row
// pair from memory.
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "dense.hpp"

namespace rdr {

namespace {

inline double hsum(__m256d v) {
  __m128d lo = _mm256_castpd256_pd128(v), hi = _mm256_extractf128_pd(v, 1);
  lo = _mm_add_pd(lo, hi);
  return _mm_cvtsd_f64(_mm_add_sd(lo, _mm_unpackhi_pd(lo, lo)));
}

// out[r][c] = sum_{k in [k0,k1)} a[r][k] * b[c][k] for 4 rows a, 2 rows b
inline void dot4x2(const double* const a[4], const double* const b[2], int k0, int k1, double out[4][2]) {
  __m256d s00 = _mm256_setzero_pd(), s01 = s00, s10 = s00, s11 = s00, s20 = s00, s21 = s00, s30 = s00, s31 = s00;
  int k = k0;
  for (; k + 4 <= k1; k += 4) {
    const __m256d b0 = _mm256_loadu_pd(b[0] + k), b1 = _mm256_loadu_pd(b[1] + k);
    __m256d x = _mm256_loadu_pd(a[0] + k);
    s00 = _mm256_fmadd_pd(x, b0, s00);
    s01 = _mm256_fmadd_pd(x, b1, s01);
    x = _mm256_loadu_pd(a[1] + k);
    s10 = _mm256_fmadd_pd(x, b0, s10);
    s11 = _mm256_fmadd_pd(x, b1, s11);
    x = _mm256_loadu_pd(a[2] + k);
    s20 = _mm256_fmadd_pd(x, b0, s20);
    s21 = _mm256_fmadd_pd(x, b1, s21);
    x = _mm256_loadu_pd(a[3] + k);
    s30 = _mm256_fmadd_pd(x, b0, s30);
    s31 = _mm256_fmadd_pd(x, b1, s31);
  }
  double r[4][2] = {{hsum(s00), hsum(s01)}, {hsum(s10), hsum(s11)}, {hsum(s20), hsum(s21)}, {hsum(s30), hsum(s31)}};
  for (; k < k1; ++k)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 2; ++j) r[i][j] += a[i][k] * b[j][k];
  std::memcpy(out, r, sizeof(r));
}

inline double dot1(const double* a, const double* b, int k0, int k1) {
  __m256d s0 = _mm256_setzero_pd(), s1 = s0, s2 = s0, s3 = s0;  // 4 chains hide the FMA latency
  int k = k0;
  for (; k + 16 <= k1; k += 16) {
    s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + k), _mm256_loadu_pd(b + k), s0);
    s1 = _mm256_fmadd_pd(_mm256_loadu_pd(a + k + 4), _mm256_loadu_pd(b + k + 4), s1);
    s2 = _mm256_fmadd_pd(_mm256_loadu_pd(a + k + 8), _mm256_loadu_pd(b + k + 8), s2);
    s3 = _mm256_fmadd_pd(_mm256_loadu_pd(a + k + 12), _mm256_loadu_pd(b + k + 12), s3);
  }
  for (; k + 4 <= k1; k += 4) s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + k), _mm256_loadu_pd(b + k), s0);
  double r = hsum(_mm256_add_pd(_mm256_add_pd(s0, s1), _mm256_add_pd(s2, s3)));
  for (; k < k1; ++k) r += a[k] * b[k];
  return r;
}

// C[i][j] -= sum_{k in [k0,k1)} R[i][k] S[j][k] for i in [i0,i1), j in [j0,j1),
// j <= i only when `lower` (row-major, leading dimension ld)
void dot_update(double* C, const double* R, const double* S, int ld, int i0, int i1, int j0, int j1, int k0, int k1,
                bool lower, double sign, bool par = false) {
  const int nblk = (i1 - i0) / 4;
#pragma omp parallel for schedule(dynamic, 4) if (par)
  for (int ib = 0; ib < nblk; ++ib) {
    const int i = i0 + 4 * ib;
    const double* a[4] = {R + (size_t)i * ld, R + (size_t)(i + 1) * ld, R + (size_t)(i + 2) * ld,
                          R + (size_t)(i + 3) * ld};
    const int jend = lower ? std::min(j1, i + 4) : j1;
    int j = j0;
    for (; j + 2 <= jend; j += 2) {
      const double* b[2] = {S + (size_t)j * ld, S + (size_t)(j + 1) * ld};
      double o[4][2];
      dot4x2(a, b, k0, k1, o);
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 2; ++c)
          if (!lower || j + c <= i + r) C[(size_t)(i + r) * ld + j + c] += sign * o[r][c];
    }
    for (; j < jend; ++j)
      for (int r = 0; r < 4; ++r)
        if (!lower || j <= i + r) C[(size_t)(i + r) * ld + j] += sign * dot1(a[r], S + (size_t)j * ld, k0, k1);
  }
  for (int i = i0 + 4 * nblk; i < i1; ++i) {
    const int jend = lower ? std::min(j1, i + 1) : j1;
    for (int j = j0; j < jend; ++j)
      C[(size_t)i * ld + j] += sign * dot1(R + (size_t)i * ld, S + (size_t)j * ld, k0, k1);
  }
}

}  // namespace

bool spd_inverse(double* A, int n, std::vector<double>& work) {
  constexpr int NB = 64;
  // one large matrix (the coarse space) outside a parallel region: threads
  // inside each step; the patch matrices are inverted one per thread instead
  const bool par = n >= 1024 && !omp_in_parallel();
  // ---- 1. Cholesky, lower, row-major, left-looking by block columns
  for (int jb = 0; jb < n; jb += NB) {
    const int je = std::min(n, jb + NB);
    // block column update with the finished columns [0, jb)
    if (jb > 0) dot_update(A, A, A, n, jb, n, jb, je, 0, jb, /*lower=*/true, -1.0, par);
    // diagonal block and the panel below, column by column within the block
    for (int j = jb; j < je; ++j) {
      double d = A[(size_t)j * n + j] - dot1(A + (size_t)j * n, A + (size_t)j * n, jb, j);
      if (!(d > 0)) return false;
      const double l = std::sqrt(d), inv = 1.0 / l;
      A[(size_t)j * n + j] = l;
#pragma omp parallel for schedule(static) if (par && n - j > 4096)
      for (int i = j + 1; i < n; ++i)
        A[(size_t)i * n + j] = (A[(size_t)i * n + j] - dot1(A + (size_t)i * n, A + (size_t)j * n, jb, j)) * inv;
    }
  }
  // ---- 2. W = L^-T stored row-major as Wt[i][k] = (L^-1)[k][i] (upper triangular):
  // column k of L^-1 solves L w = e_k; row i of Wt is column i of L^-1.
  // Computed as Y = L^-1 by rows (Y[i][:i] = -(1/L_ii) sum_{k<i} L[i][k] Y[k][:i])
  // with the row-by-row dot form on the transposed factor: Y[i][j] for j < i is
  // -(1/L_ii) sum_{k=j}^{i-1} L[i][k] Y[k][j]; with Yt[j][k] = Y[k][j] this is a
  // dot product of row i of L and row j of Yt over k in [j, i).
  work.assign((size_t)n * n, 0.0);
  double* Yt = work.data();
  for (int i = 0; i < n; ++i) Yt[(size_t)i * n + i] = 1.0 / A[(size_t)i * n + i];
  for (int i = 0; i < n; ++i) {
    const double* Li = A + (size_t)i * n;
    const double inv = Yt[(size_t)i * n + i];
#pragma omp parallel for schedule(static) if (par && i > 2048)
    for (int j = 0; j < i; ++j) {
      // sum_{k=j}^{i-1} L[i][k] * Yt[j][k]   (Yt[j][k] = 0 for k < j)
      const double s = dot1(Li, Yt + (size_t)j * n, j, i);
      Yt[(size_t)j * n + i] = -s * inv;
    }
  }
  // ---- 3. A^-1[i][j] = sum_{k >= max(i,j)} Y[k][i] Y[k][j] = dot(Yt row i, Yt row j), j <= i;
  // row i of Yt vanishes below k = i, so a block of rows [i0, i0+4) starts at k = i0
#pragma omp parallel for schedule(dynamic, 2) if (par)
  for (int i0 = 0; i0 < n; i0 += 4) {
    const int i1 = std::min(n, i0 + 4);
    for (int i = i0; i < i1; ++i)
      for (int j = 0; j <= i; ++j) A[(size_t)i * n + j] = 0.0;
    dot_update(A, Yt, Yt, n, i0, i1, 0, i1, i0, n, /*lower=*/true, 1.0);
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) A[(size_t)i * n + j] = A[(size_t)j * n + i];
  return true;
}

}  // namespace rdr
