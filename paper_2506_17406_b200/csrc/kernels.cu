// sm_100a kernels of the Riesz-map PCG hot path.
//
//  * apply_kernel      : gather x_e -> y_e = sum_s c_{e,s} R_s x_e -> scatter-add
//                        (north_star operator apply; matrix-free action P:2267-2275)
//  * precond_init      : interior point-Jacobi z_I = r_I / A_II (Thm 5.1)
//  * patch_kernel      : additive star patches z += E_m A_m^{-1} E_m^T r with the
//                        stored packed inverses streamed from HBM (Eq. 5.4 / 5.12)
//  * gather_grad / scatter_grad : the discrete gradient of the H(curl) potential
//                        patches (R-A12, Lemma 4.3)
//  * pcg_*             : fused PCG vector updates and reductions (R-A16)
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace rdr {

namespace {

constexpr int kVecThreads = 256;

__device__ __forceinline__ bool stopped(const PcgScalars* g) {
  return g != nullptr && *((volatile const int32_t*)&g->done) != 0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum, result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
    s = warp_sum(s);
  }
  __syncthreads();
  return s;
}

// 32-byte streaming load (sm_100: LDG.E.NA.EFL2.256): no L1 allocation, L2 evict-first
__device__ __forceinline__ double4 ld_stream4(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------- operator apply
// One CTA = TC cells. Thread i owns output rows i, i+blockDim, ...; for each
// reference matrix s it forms t_c = sum_j R_s[j][i] X[c][j] for its TC cells
// (R_s symmetric, so the [j][i] read is coalesced over i) and accumulates
// y[c][i] += c_{c,s} t_c. Gather/scatter through the masked dof map.
template <int TC>
__global__ void __launch_bounds__(128) apply_kernel(DevOperator op, const double* __restrict__ x,
                                                   double* __restrict__ y, double* pq_acc,
                                                   const PcgScalars* guard) {
  if (stopped(guard)) return;
  extern __shared__ double smem[];
  const int n = op.n_loc, nm = op.n_mat, ldr = op.n_pad;
  double* X = smem;                         // [TC][n]
  double* C = X + TC * n;                   // [TC][nm]
  int* D = reinterpret_cast<int*>(C + TC * nm);  // [TC][n]
  const int64_t c0 = (int64_t)blockIdx.x * TC;
  const int64_t rem = op.n_cells - c0;
  const int nc = rem < TC ? (int)rem : TC;
  for (int k = threadIdx.x; k < TC * n; k += blockDim.x) {
    int c = k / n;
    int g = (c < nc) ? op.dofmap_m[(c0 + c) * n + (k - c * n)] : -1;
    D[k] = g;
    X[k] = (g >= 0) ? x[g] : 0.0;
  }
  for (int k = threadIdx.x; k < TC * nm; k += blockDim.x) {
    int c = k / nm;
    C[k] = (c < nc) ? op.coef[(c0 + c) * nm + (k - c * nm)] : 0.0;
  }
  __syncthreads();
  double pq = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double acc[TC];
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[c] = 0;
    for (int s = 0; s < nm; ++s) {
      const double* Rs = op.R + (size_t)s * n * ldr + i;
      double t[TC];
#pragma unroll
      for (int c = 0; c < TC; ++c) t[c] = 0;
      for (int j = 0; j < n; ++j) {
        double r = __ldg(Rs + (size_t)j * ldr);
#pragma unroll
        for (int c = 0; c < TC; ++c) t[c] = fma(r, X[c * n + j], t[c]);
      }
#pragma unroll
      for (int c = 0; c < TC; ++c) acc[c] = fma(C[c * nm + s], t[c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      int g = D[c * n + i];
      if (g >= 0) {
        atomicAdd(y + g, acc[c]);
        pq = fma(X[c * n + i], acc[c], pq);
      }
    }
  }
  if (pq_acc) {
    __shared__ double sh[32];
    double s = block_sum(pq, sh);
    if (threadIdx.x == 0) atomicAdd(pq_acc, s);
  }
}

// ---------------------------------------------------------------- operator apply on FP64 tensor cores
// Y[c][i] = sum_s sum_j (c_{c,s} X[c][j]) R_s[j][i]: one GEMM with M = cells,
// N = n_loc, K = n_mat * n_loc, on DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4;
// sm_100a has no tcgen05 kind::f64). CTA = TM cells (TM/8 m-tiles),
// 4 warps split the n8-tiles of N; the A fragment (X scaled by c_s in registers)
// comes from shared memory, the B fragment (R_s, zero-padded [KP][LDN], L2/L1
// resident and shared by all CTAs) straight from global memory.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int TM, int NTW>
__global__ void __launch_bounds__(128) apply_dmma_kernel(DevOperator op, const double* __restrict__ x,
                                                         double* __restrict__ y, double* pq_acc,
                                                         const PcgScalars* guard) {
  if (stopped(guard)) return;
  constexpr int MT = TM / 8;
  extern __shared__ double smem[];
  const int n = op.n_loc, nm = op.n_mat, KP = op.kp, LDN = op.ldn;
  double* X = smem;                              // [TM][KP], zero padded
  double* C = X + TM * KP;                       // [TM][nm]
  int* D = reinterpret_cast<int*>(C + TM * nm);  // [TM][n]
  const int64_t c0 = (int64_t)blockIdx.x * TM;
  const int64_t rem = op.n_cells - c0;
  const int nc = rem < TM ? (int)rem : TM;
  for (int k = threadIdx.x; k < TM * KP; k += blockDim.x) {
    const int c = k / KP, j = k - c * KP;
    int g = (c < nc && j < n) ? op.dofmap_m[(c0 + c) * n + j] : -1;
    if (j < n) D[c * n + j] = g;
    X[k] = (g >= 0) ? x[g] : 0.0;
  }
  for (int k = threadIdx.x; k < TM * nm; k += blockDim.x) {
    const int c = k / nm;
    C[k] = (c < nc) ? op.coef[(c0 + c) * nm + (k - c * nm)] : 0.0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int NT = LDN / 8;
  double acc[MT][NTW][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < NTW; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
  int ncol[NTW];
#pragma unroll
  for (int q = 0; q < NTW; ++q) {
    const int tile = warp + 4 * q;
    ncol[q] = (tile < NT) ? tile * 8 + g : -1;
  }
  for (int s = 0; s < nm; ++s) {
    double cs[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) cs[m] = C[(m * 8 + g) * nm + s];
    const double* __restrict__ Rs = op.Rt + (size_t)s * KP * LDN;
#pragma unroll 4
    for (int k0 = 0; k0 < KP; k0 += 4) {
      const int kk = k0 + t;
      double b[NTW];
#pragma unroll
      for (int q = 0; q < NTW; ++q) b[q] = (ncol[q] >= 0) ? __ldg(Rs + (size_t)kk * LDN + ncol[q]) : 0.0;
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = cs[m] * X[(m * 8 + g) * KP + kk];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int q = 0; q < NTW; ++q)
          if (warp + 4 * q < NT) dmma884(acc[m][q][0], acc[m][q][1], a[m], b[q]);
    }
  }
  // epilogue: C fragment (row g, cols 2t, 2t+1) -> scatter-add, fused p.(Ap)
  double pq = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < NTW; ++q) {
      const int tile = warp + 4 * q;
      if (tile >= NT) continue;
      const int cell = m * 8 + g;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = tile * 8 + 2 * t + i;
        if (col < n && cell < nc) {
          const int gd = D[cell * n + col];
          if (gd >= 0) {
            atomicAdd(y + gd, acc[m][q][i]);
            pq = fma(X[cell * KP + col], acc[m][q][i], pq);
          }
        }
      }
    }
  if (pq_acc) {
    __shared__ double sh[32];
    double sum = block_sum(pq, sh);
    if (threadIdx.x == 0) atomicAdd(pq_acc, sum);
  }
}

template <int TM, int NTW>
cudaError_t launch_apply_dmma(const DevOperator& op, const double* x, double* y, double* pq_acc,
                              const PcgScalars* guard, cudaStream_t s) {
  size_t sm = (size_t)TM * op.kp * sizeof(double) + (size_t)TM * op.n_mat * sizeof(double) +
              (size_t)TM * op.n_loc * sizeof(int);
  static bool configured = false;  // first call happens in rdr_setup (outside stream capture)
  if (!configured) {
    cudaFuncSetAttribute(apply_dmma_kernel<TM, NTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  unsigned grid = (unsigned)((op.n_cells + TM - 1) / TM);
  apply_dmma_kernel<TM, NTW><<<grid, 128, sm, s>>>(op, x, y, pq_acc, guard);
  return cudaGetLastError();
}

template <int TC>
cudaError_t launch_apply_tc(const DevOperator& op, const double* x, double* y, double* pq_acc,
                            const PcgScalars* guard, cudaStream_t s) {
  size_t sm = (size_t)TC * op.n_loc * (sizeof(double) + sizeof(int)) + (size_t)TC * op.n_mat * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(apply_kernel<TC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  unsigned grid = (unsigned)((op.n_cells + TC - 1) / TC);
  apply_kernel<TC><<<grid, 128, sm, s>>>(op, x, y, pq_acc, guard);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- preconditioner
__global__ void precond_init_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ z,
                                    double* rz_acc, const PcgScalars* guard) {
  if (stopped(guard)) return;
  double part = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_total; i += stride) {
    if (i < pc.off3) {
      z[i] = 0.0;
    } else {
      double ri = r[i];
      double zi = pc.dinv[i - pc.off3] * ri;
      z[i] = zi;
      part = fma(ri, zi, part);
    }
  }
  if (pc.ubuf)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_cg_iface; i += stride) pc.ubuf[i] = 0.0;
  if (rz_acc) {
    __shared__ double sh[32];
    double s = block_sum(part, sh);
    if (threadIdx.x == 0) atomicAdd(rz_acc, s);
  }
}

__global__ void gather_grad_kernel(DevPrecond pc, const double* __restrict__ r, const PcgScalars* guard) {
  if (stopped(guard)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < pc.n_cg_iface; c += stride) {
    double s = 0;
    for (int64_t k = pc.g_ptr[c]; k < pc.g_ptr[c + 1]; ++k) s = fma(pc.g_val[k], r[pc.g_col[k]], s);
    pc.gbuf[c] = s;
  }
}

__global__ void scatter_grad_kernel(DevPrecond pc, double* __restrict__ z, const PcgScalars* guard) {
  if (stopped(guard)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < pc.n_cg_iface; c += stride) {
    double u = pc.ubuf[c];
    if (u == 0.0) continue;
    for (int64_t k = pc.g_ptr[c]; k < pc.g_ptr[c + 1]; ++k) atomicAdd(z + pc.g_col[k], pc.g_val[k] * u);
  }
}

// Sum over the 32 lanes of v[lane'][k], delivered to lane k (recursive halving, 31 shuffles).
template <int S>
__device__ __forceinline__ void transpose_reduce_stage(double (&v)[32], int lane) {
  const bool upper = (lane & S) != 0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    double send = upper ? v[k] : v[k + S];
    double keep = upper ? v[k + S] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, S);
  }
}

// One CTA per patch (patches sorted by decreasing size). The packed lower
// tiles of A_m^{-1} (32x32, element (i,k) at ((k>>2)*32+i)*4+(k&3)) are
// streamed once with 32-byte non-allocating loads; a warp owns a tile: row
// products go to z_I, the transposed products (off-diagonal tiles) to z_J.
constexpr int kPatchThreads = 256;
__global__ void __launch_bounds__(kPatchThreads) patch_kernel(DevPrecond pc, const double* __restrict__ r,
                                                             double* __restrict__ z, double* rz_acc,
                                                             const PcgScalars* guard) {
  if (stopped(guard)) return;
  extern __shared__ double smem[];
  const int pid = blockIdx.x;
  const int n = pc.pn[pid];
  const int nb = (n + 31) >> 5, npad = nb * 32;
  const bool pot = pc.pkind[pid] != 0;
  const double* __restrict__ rin = pot ? pc.gbuf : r;
  double* __restrict__ zout = pot ? pc.ubuf : z;
  double* rl = smem;
  double* zl = smem + npad;
  const int32_t* id = pc.idx + pc.idx_off[pid];
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    int g = id[i];
    rl[i] = (g >= 0) ? rin[g] : 0.0;
    zl[i] = 0.0;
  }
  __syncthreads();
  const double* T = pc.tiles + pc.tile_off[pid];
  const int ntiles = nb * (nb + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  int I = 0, J = 0, tcur = 0;
  for (int t = warp; t < ntiles; t += nwarps) {
    while (tcur < t) {  // advance (I,J) in tile order I(I+1)/2 + J
      ++J;
      if (J > I) { ++I; J = 0; }
      ++tcur;
    }
    const double4* tp = reinterpret_cast<const double4*>(T + (size_t)t * 1024) + lane;
    double a[32];
#pragma unroll
    for (int k4 = 0; k4 < 8; ++k4) {
      double4 v = ld_stream4(tp + k4 * 32);
      a[4 * k4] = v.x;
      a[4 * k4 + 1] = v.y;
      a[4 * k4 + 2] = v.z;
      a[4 * k4 + 3] = v.w;
    }
    const double* rJ = rl + J * 32;
    double row = 0;
#pragma unroll
    for (int k = 0; k < 32; ++k) row = fma(a[k], rJ[k], row);
    atomicAdd(zl + I * 32 + lane, row);
    if (I != J) {
      const double ri = rl[I * 32 + lane];
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] *= ri;
      transpose_reduce_stage<16>(a, lane);
      transpose_reduce_stage<8>(a, lane);
      transpose_reduce_stage<4>(a, lane);
      transpose_reduce_stage<2>(a, lane);
      transpose_reduce_stage<1>(a, lane);
      atomicAdd(zl + J * 32 + lane, a[0]);
    }
  }
  __syncthreads();
  double part = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    int g = id[i];
    double zi = zl[i];
    atomicAdd(zout + g, zi);
    part = fma(rl[i], zi, part);
  }
  if (rz_acc) {
    __shared__ double sh[32];
    double s = block_sum(part, sh);
    if (threadIdx.x == 0) atomicAdd(rz_acc, s);
  }
}

// ---------------------------------------------------------------- PCG vector kernels
__global__ void pcg_init_kernel(const double* __restrict__ b, const uint8_t* __restrict__ cons, int64_t n,
                                double* __restrict__ x, double* __restrict__ r, double* __restrict__ q) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    x[i] = 0.0;
    q[i] = 0.0;
    r[i] = cons[i] ? 0.0 : b[i];
  }
}

// last-block finalisation of a grid reduction into sc->zz
__device__ __forceinline__ bool last_block(PcgScalars* sc, double part) {
  __shared__ double sh[32];
  __shared__ bool last;
  double s = block_sum(part, sh);
  if (threadIdx.x == 0) {
    atomicAdd(&sc->zz, s);
    __threadfence();
    unsigned t = atomicAdd(&sc->ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  return last;
}

__global__ void pcg_start_kernel(PcgScalars* sc, const double* __restrict__ z, double* __restrict__ p, int64_t n,
                                 double rtol, int maxit) {
  double part = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double zi = z[i];
    p[i] = zi;
    part = fma(zi, zi, part);
  }
  if (last_block(sc, part) && threadIdx.x == 0) {
    __threadfence();
    volatile PcgScalars* v = sc;
    double zz = v->zz;
    sc->z0 = sqrt(zz);
    sc->rz = v->rz_new;
    sc->rz_new = 0;
    sc->zz = 0;
    sc->pq = 0;
    sc->ticket = 0;
    sc->iters = 0;
    sc->rtol = rtol;
    sc->maxit = maxit;
    sc->converged = (zz == 0.0);
    sc->done = (zz == 0.0) || (maxit <= 0);
    sc->beta = 0;
  }
}

__global__ void pcg_update_kernel(PcgScalars* sc, const double* __restrict__ p, const double* __restrict__ q,
                                  double* __restrict__ x, double* __restrict__ r, int64_t n) {
  if (stopped(sc)) return;
  const double alpha = sc->rz / sc->pq;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    x[i] = fma(alpha, p[i], x[i]);
    r[i] = fma(-alpha, q[i], r[i]);
  }
}

__global__ void pcg_finish_kernel(PcgScalars* sc, const double* __restrict__ z, int64_t n) {
  if (stopped(sc)) return;
  double part = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double zi = z[i];
    part = fma(zi, zi, part);
  }
  if (last_block(sc, part) && threadIdx.x == 0) {
    __threadfence();
    volatile PcgScalars* v = sc;
    double zn = sqrt(v->zz);
    int it = v->iters + 1;
    sc->iters = it;
    if (zn <= v->rtol * v->z0) {
      sc->done = 1;
      sc->converged = 1;
    } else if (it >= v->maxit) {
      sc->done = 1;
      sc->converged = 0;
    } else {
      sc->beta = v->rz_new / v->rz;
      sc->rz = v->rz_new;
    }
    sc->rz_new = 0;
    sc->zz = 0;
    sc->pq = 0;
    sc->ticket = 0;
  }
}

__global__ void pcg_direction_kernel(PcgScalars* sc, const double* __restrict__ z, double* __restrict__ p,
                                     double* __restrict__ q, int64_t n) {
  if (stopped(sc)) return;
  const double beta = sc->beta;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    p[i] = fma(beta, p[i], z[i]);
    q[i] = 0.0;
  }
}

unsigned vec_grid(int64_t n) {
  int64_t g = (n + kVecThreads - 1) / kVecThreads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

cudaError_t launch_apply(const DevOperator& op, const double* x, double* y, double* pq_acc,
                         const PcgScalars* guard, cudaStream_t s) {
  if (!op.Rt) {  // CUDA-core reference kernel (RDR_KERNEL=simple)
    if (op.n_loc <= 64) return launch_apply_tc<16>(op, x, y, pq_acc, guard, s);
    if (op.n_loc <= 400) return launch_apply_tc<8>(op, x, y, pq_acc, guard, s);
    return launch_apply_tc<4>(op, x, y, pq_acc, guard, s);
  }
  const int nt = (op.ldn / 8 + 3) / 4;  // n8-tiles per warp
  const int64_t cells = op.n_cells;
#define RDR_DMMA_CASE(NTW)                                                                     \
  if (nt <= NTW) {                                                                             \
    if (NTW <= 6 && cells >= 32 * 296) return launch_apply_dmma<32, NTW>(op, x, y, pq_acc, guard, s); \
    if (NTW <= 12 && cells >= 16 * 296) return launch_apply_dmma<16, NTW>(op, x, y, pq_acc, guard, s); \
    return launch_apply_dmma<8, NTW>(op, x, y, pq_acc, guard, s);                              \
  }
  RDR_DMMA_CASE(1)
  RDR_DMMA_CASE(2)
  RDR_DMMA_CASE(3)
  RDR_DMMA_CASE(4)
  RDR_DMMA_CASE(6)
  RDR_DMMA_CASE(8)
  RDR_DMMA_CASE(10)
  RDR_DMMA_CASE(12)
  RDR_DMMA_CASE(15)
  RDR_DMMA_CASE(19)
  RDR_DMMA_CASE(25)
#undef RDR_DMMA_CASE
  return cudaErrorInvalidValue;
}

int count_precond_launches(const DevPrecond& pc) {
  return 1 + (pc.n_patches > 0 ? 1 : 0) + (pc.gbuf ? 2 : 0);
}

cudaError_t launch_precond_part(int part, const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                                const PcgScalars* guard, cudaStream_t s) {
  switch (part) {
    case 0:
      precond_init_kernel<<<vec_grid(pc.n_total), kVecThreads, 0, s>>>(pc, r, z, rz_acc, guard);
      break;
    case 1:
      if (pc.gbuf) gather_grad_kernel<<<vec_grid(pc.n_cg_iface), kVecThreads, 0, s>>>(pc, r, guard);
      break;
    case 2:
      if (pc.n_patches > 0) {
        const int npad = ((pc.max_n + 31) / 32) * 32;  // the largest patch (grid sorted by size)
        const size_t sm = (size_t)2 * npad * sizeof(double);
        patch_kernel<<<(unsigned)pc.n_patches, kPatchThreads, sm, s>>>(pc, r, z, rz_acc, guard);
      }
      break;
    case 3:
      if (pc.gbuf) scatter_grad_kernel<<<vec_grid(pc.n_cg_iface), kVecThreads, 0, s>>>(pc, z, guard);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_precond(const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                           const PcgScalars* guard, cudaStream_t s) {
  for (int part = 0; part < 4; ++part) {
    cudaError_t e = launch_precond_part(part, pc, r, z, rz_acc, guard, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_pcg_init(const double* b, const uint8_t* constrained, int64_t n, double* x, double* r,
                            double* q, cudaStream_t s) {
  pcg_init_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(b, constrained, n, x, r, q);
  return cudaGetLastError();
}
cudaError_t launch_pcg_start(PcgScalars* sc, const double* z, double* p, int64_t n, double rtol, int maxit,
                             cudaStream_t s) {
  pcg_start_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, z, p, n, rtol, maxit);
  return cudaGetLastError();
}
cudaError_t launch_pcg_update(PcgScalars* sc, const double* p, const double* q, double* x, double* r, int64_t n,
                              cudaStream_t s) {
  pcg_update_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, p, q, x, r, n);
  return cudaGetLastError();
}
cudaError_t launch_pcg_finish(PcgScalars* sc, const double* z, int64_t n, cudaStream_t s) {
  pcg_finish_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, z, n);
  return cudaGetLastError();
}
cudaError_t launch_pcg_direction(PcgScalars* sc, const double* z, double* p, double* q, int64_t n, cudaStream_t s) {
  pcg_direction_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, z, p, q, n);
  return cudaGetLastError();
}

}  // namespace rdr

namespace rdr {
void configure_kernels() {
  cudaFuncSetAttribute(apply_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(apply_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(apply_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(patch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
}
}  // namespace rdr
