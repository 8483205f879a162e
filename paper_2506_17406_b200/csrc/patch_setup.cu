// Device-side assembly and inversion of the star-patch matrices (SURVEY §8(f)
// NEXT-4; the patch factorisation of P:2284-2288, R-A15). See patch_setup.hpp.
//
// One CTA per patch at a time (persistent grid, patches claimed largest
// first). The patch matrix lives in a per-CTA global scratch (lower triangle
// in 64x64 tiles, leading dimension ld = n rounded up to 64, padded with the
// identity so that every pivot block is full) and is inverted in place by the
// block sweep (Gauss-Jordan) operator: sweeping pivot block K maps
//   A_KK -> -A_KK^-1,  A_IK -> A_IK A_KK^-1,  A_IJ -> A_IJ - A_IK A_KK^-1 A_KJ,
// and sweeping every block leaves -A^-1. For an SPD matrix each pivot block is
// a Schur complement of the unswept part, hence SPD: no pivoting, and a
// non-positive pivot flags a matrix that is not SPD (RDR_ENOTSPD). The sweep
// keeps the matrix symmetric, so only the tiles I >= J are updated. The
// rank-64 updates are 64x64x64 tile products on the FP64 tensor cores
// (mma.sync m8n8k4 DMMA, 16x32 per warp, operands staged in shared memory). The last
// step packs -(-A^-1) into the stored tile layout (setup.hpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "patch_setup.hpp"

namespace rdr {

namespace {

constexpr int kB = 64;         // pivot block / tile
constexpr int kThreads = 256;  // 8 warps, 16 x 32 outputs each
constexpr int kSs = kB + 8;    // stride of the pivot block (= kXs: it doubles as the second V buffer)
constexpr int kXs = kB + 8;    // stride of the staged operands: == 16 words (mod 32), so the DMMA
                               // fragment loads (rows k..k+3, 8 lanes each) take the minimum 2 wavefronts

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// dst[k][c] (stride kXs) <- src[k * ld + c], a 64 x 64 tile, asynchronously (16-byte copies)
__device__ __forceinline__ void tile_load_async(double* dst, const double* src, int64_t ld, int tid) {
#pragma unroll
  for (int u = 0; u < kB * kB / 2 / kThreads; ++u) {
    const int e = tid + u * kThreads, k = e / (kB / 2), c = 2 * (e % (kB / 2));
    cp_async16(dst + k * kXs + c, src + (int64_t)k * ld + c);
  }
  cp_async_commit();
}

// 64x64x64 tile product on the FP64 tensor cores (DMMA.8x8x4):
//   acc = sum_k X[k][row] * Y[k][col]
// Warp w owns rows (w&3)*16 + [0,16) and columns (w>>2)*32 + [0,32). Element
// (m, q, i) of acc is at row acc_row(w, lane, m), column acc_col(w, lane, q, i).
__device__ __forceinline__ int acc_row(int warp, int lane, int m) { return (warp & 3) * 16 + m * 8 + (lane >> 2); }
__device__ __forceinline__ int acc_col(int warp, int lane, int q, int i) {
  return (warp >> 2) * 32 + q * 8 + 2 * (lane & 3) + i;
}
__device__ __forceinline__ void tile_product(const double* X, const double* Y, int warp, int lane,
                                             double acc[2][4][2]) {
  const int g = lane >> 2, t = lane & 3;
  const int r0 = (warp & 3) * 16 + g, c0 = (warp >> 2) * 32 + g;
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
#pragma unroll 4
  for (int k = 0; k < kB; k += 4) {
    const double* xk = X + (k + t) * kXs;
    const double* yk = Y + (k + t) * kXs;
    const double a0 = xk[r0], a1 = xk[r0 + 8];
    double b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) b[q] = yk[c0 + q * 8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      dmma884(acc[0][q][0], acc[0][q][1], a0, b[q]);
      dmma884(acc[1][q][0], acc[1][q][1], a1, b[q]);
    }
  }
}

// A[rows i0.., cols j0..] -= acc (row-major, leading dimension ld). The
// reductions are performed at L2, so every later read of A in the same kernel
// goes through L2 too (__ldcg): an L1 line of a reused scratch address could
// otherwise be stale.
__device__ __forceinline__ void tile_subtract(double* A, int64_t ld, int i0, int j0, int warp, int lane,
                                              const double acc[2][4][2]) {
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // fire-and-forget reductions (RED.ADD.F64): no load latency on the product's critical
      // path; each element has exactly one writer here, so the order cannot change the result
      double* a = A + (int64_t)(i0 + acc_row(warp, lane, m)) * ld + j0 + acc_col(warp, lane, q, 0);
      atomicAdd(a, -acc[m][q][0]);
      atomicAdd(a + 1, -acc[m][q][1]);
    }
}

// Scalar sweep of the 64 pivots of the symmetric block S (stride kSs) in
// place: S -> -S^-1. A non-positive pivot sets *status = flag (if still 0).
__device__ void sweep_pivot_block(double* S, int tid, int32_t* status, int32_t flag) {
  for (int p = 0; p < kB; ++p) {
    const double d = S[p * kSs + p];
    const double inv = 1.0 / d;
    double nv[kB * kB / kThreads];
#pragma unroll
    for (int u = 0; u < kB * kB / kThreads; ++u) {
      const int e = tid + u * kThreads, i = e / kB, j = e % kB;
      const double a = S[i * kSs + j];
      if (i == p && j == p)
        nv[u] = -inv;
      else if (i == p || j == p)
        nv[u] = a * inv;
      else
        nv[u] = fma(-S[i * kSs + p] * inv, S[p * kSs + j], a);
    }
    if (tid == 0 && !(d > 0.0)) atomicCAS(status, 0, flag);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kB * kB / kThreads; ++u) {
      const int e = tid + u * kThreads;
      S[(e / kB) * kSs + e % kB] = nv[u];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kThreads, 2) patch_setup_kernel(DevPatchSetup s) {
  extern __shared__ double4 smem_raw[];
  double* S = reinterpret_cast<double*>(smem_raw);  // [kB][kSs] pivot block, then the second V buffer
  double* X = S + kB * kSs;                         // [kB][kXs] (16-byte aligned)
  double* Y = X + kB * kXs;                         // [kB][kXs]
  __shared__ int64_t claim;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* A = s.scratch + (int64_t)blockIdx.x * (s.ld_max * s.ld_max + 2 * kB * s.ld_max);
  for (;;) {
    __syncthreads();
    if (tid == 0) claim = atomicAdd(s.queue, 1);
    __syncthreads();
    const int64_t m = claim;
    if (m >= s.np) break;
    const int n = s.pn[m];
    const int ld = (n + kB - 1) / kB * kB, nb = ld / kB;
    double* Wp = A + (int64_t)ld * ld;  // [kB][ld]: W_I = A_IK A_KK^-1, transposed
    double* Vp = Wp + (int64_t)kB * ld;  // [kB][ld]: V_I = A_IK (before the sweep of K), transposed

    // ---- 1. zero, identity padding, assembly of the lower triangle
    for (int64_t e = tid; e < (int64_t)ld * ld; e += kThreads) {
      const int i = (int)(e / ld), j = (int)(e % ld);
      A[e] = (i == j && i >= n) ? 1.0 : 0.0;
    }
    __syncthreads();
    {
      const int kind = s.pkind[m];
      const double* R = s.R[kind];
      const double* cf = s.coef[kind];
      const int nl = s.nl[kind], nm = s.nm[kind];
      for (int64_t rc = s.rec_ptr[m]; rc < s.rec_ptr[m + 1]; ++rc) {
        const int64_t e0 = s.rec_off[rc];
        const int cnt = (int)(s.rec_off[rc + 1] - e0);
        const double* c = cf + (int64_t)s.rec_cell[rc] * nm;
        // the entries of one cell hit distinct (pa, pb): no two threads add to one entry
        for (int q = tid; q < cnt * cnt; q += kThreads) {
          const uint32_t ea = s.ent[e0 + q / cnt], eb = s.ent[e0 + q % cnt];
          const int pa = (int)(ea & 0xffffu), pb = (int)(eb & 0xffffu);
          if (pa < pb) continue;
          const int64_t la = ea >> 16, lb = eb >> 16;
          double v = 0.0;
          for (int t = 0; t < nm; ++t) v = fma(c[t], R[((int64_t)t * nl + la) * nl + lb], v);
          A[(int64_t)pa * ld + pb] = __ldcg(A + (int64_t)pa * ld + pb) + v;
        }
        __syncthreads();
      }
    }

    // ---- 2. block sweep
    for (int K = 0; K < nb; ++K) {
      const int k0 = K * kB;
      // 2a. pivot block, symmetric, then the scalar sweep of its 64 pivots: S = -A_KK^-1
      for (int e = tid; e < kB * kB; e += kThreads) {
        const int i = e / kB, j = e % kB;
        S[i * kSs + j] = i >= j ? __ldcg(A + (int64_t)(k0 + i) * ld + k0 + j) : __ldcg(A + (int64_t)(k0 + j) * ld + k0 + i);
      }
      __syncthreads();
      sweep_pivot_block(S, tid, s.status, (int32_t)(m + 1));
      if (nb == 1) {
        for (int e = tid; e < kB * kB; e += kThreads) {
          const int i = e / kB, j = e % kB;
          if (i >= j) A[(int64_t)i * ld + j] = S[i * kSs + j];
        }
        __syncthreads();
        break;
      }
      // 2b. V_I = A_IK and W_I = A_IK A_KK^-1 = -V_I S for every I != K
      for (int e = tid; e < kB * kB; e += kThreads) Y[(e / kB) * kXs + e % kB] = S[(e / kB) * kSs + e % kB];
      for (int I = 0; I < nb; ++I) {
        if (I == K) continue;
        const int i0 = I * kB;
        if (I > K) {  // tile (I, K): row-major rows i, columns k -> X[k][i]
          for (int e = tid; e < kB * kB; e += kThreads) {
            const int r = e / kB, k = e % kB;
            X[k * kXs + r] = __ldcg(A + (int64_t)(i0 + r) * ld + k0 + k);
          }
        } else {  // tile (K, I) = A_KI = A_IK^T: rows k, columns i -> X[k][i]
          for (int e = tid; e < kB * kB; e += kThreads) {
            const int k = e / kB, r = e % kB;
            X[k * kXs + r] = __ldcg(A + (int64_t)(k0 + k) * ld + i0 + r);
          }
        }
        __syncthreads();
        for (int e = tid; e < kB * kB; e += kThreads) {
          const int k = e / kB, r = e % kB;
          Vp[(int64_t)k * ld + i0 + r] = X[k * kXs + r];
        }
        double acc[2][4][2];
        tile_product(X, Y, warp, lane, acc);
#pragma unroll
        for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < 2; ++i)
              Wp[(int64_t)acc_col(warp, lane, q, i) * ld + i0 + acc_row(warp, lane, m2)] = -acc[m2][q][i];
        __syncthreads();
      }
      // A_KK = S now: from here on S is the second V buffer of 2c
      for (int e = tid; e < kB * kB; e += kThreads) {
        const int i = e / kB, j = e % kB;
        if (i >= j) A[(int64_t)(k0 + i) * ld + k0 + j] = S[i * kSs + j];
      }
      // 2c. A_IJ -= W_I V_J^T for I >= J, I, J != K; the next V_J streams into
      // the other buffer (cp.async) while the current tile product runs
      for (int I = 0; I < nb; ++I) {
        if (I == K) continue;
        const int i0 = I * kB;
        __syncthreads();  // the previous I's products are done with X and both V buffers
        for (int e = tid; e < kB * kB; e += kThreads) {
          const int k = e / kB, r = e % kB;
          X[k * kXs + r] = Wp[(int64_t)k * ld + i0 + r];
        }
        double *cur = Y, *nxt = S;
        int J = K == 0 ? 1 : 0;
        if (J <= I) tile_load_async(cur, Vp + J * kB, ld, tid);
        while (J <= I) {
          int Jn = J + 1;
          if (Jn == K) ++Jn;
          cp_async_wait_all();
          __syncthreads();  // V_J (and X) visible; everyone is done with the buffer refilled next
          if (Jn <= I) tile_load_async(nxt, Vp + Jn * kB, ld, tid);
          double acc[2][4][2];
          tile_product(X, cur, warp, lane, acc);
          tile_subtract(A, ld, i0, J * kB, warp, lane, acc);
          double* t2 = cur;
          cur = nxt;
          nxt = t2;
          J = Jn;
        }
      }
      __syncthreads();
      // 2d. the swept block row / column: A_IK = W_I (I > K), A_KI = W_I^T (I < K)
      for (int I = 0; I < nb; ++I) {
        if (I == K) continue;
        const int i0 = I * kB;
        if (I > K) {
          for (int e = tid; e < kB * kB; e += kThreads) {
            const int r = e / kB, k = e % kB;
            A[(int64_t)(i0 + r) * ld + k0 + k] = Wp[(int64_t)k * ld + i0 + r];
          }
        } else {
          for (int e = tid; e < kB * kB; e += kThreads) {
            const int k = e / kB, r = e % kB;
            A[(int64_t)(k0 + k) * ld + i0 + r] = Wp[(int64_t)k * ld + i0 + r];
          }
        }
      }
      __syncthreads();
    }

    // ---- 3. pack A^-1 = -(swept A), lower triangle, into the stored layout (setup.hpp)
    double* out = s.tiles + s.tile_off[m];
    const int nbk = (n + 31) / 32;
    for (int I = 0; I < nbk; ++I) {
      const int rows = min(32, n - 32 * I);
      const int64_t base = 512LL * I * I + 16LL * I;
      const int full = I * 32 * rows, total = full + rows * (rows + 1) / 2;
      for (int w = tid; w < total; w += kThreads) {
        int i, col;
        if (w < full) {
          const int J = w / (32 * rows), q = w % (32 * rows);
          int kk;
          if (s.layout == 0) {
            i = (q >> 2) % rows;
            kk = ((q >> 2) / rows) * 4 + (q & 3);
          } else {
            i = q >> 5;
            kk = ((((q & 31) >> 1) ^ (i & 7)) << 1) | (q & 1);
          }
          col = 32 * J + kk;
        } else {  // diagonal tile by columns: (i, kk), kk <= i, at kk*rows - kk(kk-1)/2 + (i-kk)
          int q = w - full, kk = 0;
          while (q >= rows - kk) {
            q -= rows - kk;
            ++kk;
          }
          i = kk + q;
          col = 32 * I + kk;
        }
        out[base + w] = -__ldcg(A + (int64_t)(32 * I + i) * ld + col);
      }
    }
    const int64_t exact = (int64_t)n * (n + 1) / 2, stored = s.tile_off[m + 1] - s.tile_off[m];
    for (int64_t w = exact + tid; w < stored; w += kThreads) out[w] = 0.0;
  }
}

// ---- one large SPD matrix (the hybrid's Whitney coarse space): the same block
// sweep with each phase spread over the grid, three launches per pivot block.
// A: ld x ld row-major lower tiles, rows/columns >= n zero (identity pivots).

// phase 1 (one CTA): S = -A_KK^-1 into Sg (64 x 64) and into A_KK
__global__ void __launch_bounds__(kThreads) dense_pivot_kernel(double* A, int64_t ld, int n, int K, double* Sg,
                                                              int32_t* status) {
  __shared__ double S[kB * kSs];
  const int tid = threadIdx.x, k0 = K * kB;
  for (int e = tid; e < kB * kB; e += kThreads) {
    const int i = e / kB, j = e % kB;
    double v = i >= j ? A[(int64_t)(k0 + i) * ld + k0 + j] : A[(int64_t)(k0 + j) * ld + k0 + i];
    if (k0 + i >= n || k0 + j >= n) v = (i == j) ? 1.0 : 0.0;  // identity padding
    S[i * kSs + j] = v;
  }
  __syncthreads();
  sweep_pivot_block(S, tid, status, K + 1);
  for (int e = tid; e < kB * kB; e += kThreads) {
    const int i = e / kB, j = e % kB;
    Sg[e] = S[i * kSs + j];
    if (i >= j) A[(int64_t)(k0 + i) * ld + k0 + j] = S[i * kSs + j];
  }
}

// phase 2 (one CTA per I != K): V_I = A_IK -> Vp, W_I = -V_I S -> Wp and into A's block row/column K
__global__ void __launch_bounds__(kThreads, 2) dense_panel_kernel(double* A, int64_t ld, int K, const double* Sg,
                                                                 double* Wp, double* Vp) {
  extern __shared__ double4 smem_raw[];
  double* X = reinterpret_cast<double*>(smem_raw);
  double* Y = X + kB * kXs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int I = blockIdx.x < (unsigned)K ? blockIdx.x : blockIdx.x + 1;
  const int i0 = I * kB, k0 = K * kB;
  for (int e = tid; e < kB * kB; e += kThreads) Y[(e / kB) * kXs + e % kB] = Sg[e];
  if (I > K) {
    for (int e = tid; e < kB * kB; e += kThreads) {
      const int r = e / kB, k = e % kB;
      X[k * kXs + r] = A[(int64_t)(i0 + r) * ld + k0 + k];
    }
  } else {
    for (int e = tid; e < kB * kB; e += kThreads) {
      const int k = e / kB, r = e % kB;
      X[k * kXs + r] = A[(int64_t)(k0 + k) * ld + i0 + r];
    }
  }
  __syncthreads();
  for (int e = tid; e < kB * kB; e += kThreads) {
    const int k = e / kB, r = e % kB;
    Vp[(int64_t)k * ld + i0 + r] = X[k * kXs + r];
  }
  double acc[2][4][2];
  tile_product(X, Y, warp, lane, acc);
#pragma unroll
  for (int m2 = 0; m2 < 2; ++m2)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int i = i0 + acc_row(warp, lane, m2), k = acc_col(warp, lane, q, c);
        Wp[(int64_t)k * ld + i] = -acc[m2][q][c];
        if (I > K)
          A[(int64_t)i * ld + k0 + k] = -acc[m2][q][c];
        else
          A[(int64_t)(k0 + k) * ld + i] = -acc[m2][q][c];
      }
}

// phase 3 (grid-stride over the lower tiles I >= J, I, J != K): A_IJ -= W_I V_J^T
__global__ void __launch_bounds__(kThreads, 2) dense_update_kernel(double* A, int64_t ld, int nb, int K,
                                                                  const double* Wp, const double* Vp) {
  extern __shared__ double4 smem_raw[];
  double* X = reinterpret_cast<double*>(smem_raw);
  double* Y = X + kB * kXs;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m = nb - 1, ntiles = m * (m + 1) / 2;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int64_t a = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) / 2.0);
    while (a * (a + 1) / 2 > t) --a;
    while ((a + 1) * (a + 2) / 2 <= t) ++a;
    const int Ip = (int)a, Jp = (int)(t - a * (a + 1) / 2);
    const int I = Ip < K ? Ip : Ip + 1, J = Jp < K ? Jp : Jp + 1;
    const int i0 = I * kB, j0 = J * kB;
    __syncthreads();
    for (int e = tid; e < kB * kB; e += kThreads) {
      const int k = e / kB, r = e % kB;
      X[k * kXs + r] = Wp[(int64_t)k * ld + i0 + r];
      Y[k * kXs + r] = Vp[(int64_t)k * ld + j0 + r];
    }
    __syncthreads();
    double acc[2][4][2];
    tile_product(X, Y, warp, lane, acc);
    tile_subtract(A, ld, i0, j0, warp, lane, acc);
  }
}

// pack -(swept A) = A^-1 (n x n) into the stored tile layout, one CTA per 32-row block row
__global__ void dense_pack_kernel(const double* A, int64_t ld, int n, double* out, int layout) {
  const int I = blockIdx.x, tid = threadIdx.x;
  const int rows = min(32, n - 32 * I);
  const int64_t base = 512LL * I * I + 16LL * I;
  const int full = I * 32 * rows, total = full + rows * (rows + 1) / 2;
  for (int w = tid; w < total; w += blockDim.x) {
    int i, col;
    if (w < full) {
      const int J = w / (32 * rows), q = w % (32 * rows);
      int kk;
      if (layout == 0) {
        i = (q >> 2) % rows;
        kk = ((q >> 2) / rows) * 4 + (q & 3);
      } else {
        i = q >> 5;
        kk = ((((q & 31) >> 1) ^ (i & 7)) << 1) | (q & 1);
      }
      col = 32 * J + kk;
    } else {
      int q = w - full, kk = 0;
      while (q >= rows - kk) {
        q -= rows - kk;
        ++kk;
      }
      i = kk + q;
      col = 32 * I + kk;
    }
    out[base + w] = -A[(int64_t)(32 * I + i) * ld + col];
  }
}

}  // namespace

cudaError_t dense_spd_inverse_packed(double* A, int64_t ld, int n, double* work, int32_t* status, double* tiles,
                                     int layout, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int nb = (int)(ld / kB);
  double* Sg = work;
  double* Wp = Sg + kB * kB;
  double* Vp = Wp + (int64_t)kB * ld;
  const size_t smem = sizeof(double) * 2 * kB * kXs;
  cudaError_t e = cudaFuncSetAttribute(dense_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dense_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int K = 0; K < nb; ++K) {
    dense_pivot_kernel<<<1, kThreads, 0, stream>>>(A, ld, n, K, Sg, status);
    if (nb > 1) {
      dense_panel_kernel<<<nb - 1, kThreads, smem, stream>>>(A, ld, K, Sg, Wp, Vp);
      const int64_t ntiles = (int64_t)(nb - 1) * nb / 2;
      const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * 16);
      dense_update_kernel<<<grid, kThreads, smem, stream>>>(A, ld, nb, K, Wp, Vp);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  dense_pack_kernel<<<(n + 31) / 32, kThreads, 0, stream>>>(A, ld, n, tiles, layout);
  return cudaGetLastError();
}

int64_t patch_setup_scratch_doubles(int64_t ld_max) { return ld_max * ld_max + 2 * kB * ld_max; }

size_t patch_setup_smem() { return sizeof(double) * (kB * kSs + 2 * kB * kXs); }

cudaError_t launch_patch_setup(const DevPatchSetup& s, int n_ctas, cudaStream_t stream) {
  const size_t smem = patch_setup_smem();
  cudaError_t e = cudaFuncSetAttribute(patch_setup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  patch_setup_kernel<<<n_ctas, kThreads, smem, stream>>>(s);
  return cudaGetLastError();
}

}  // namespace rdr
