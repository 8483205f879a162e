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

#include <algorithm>
#include <cstdint>
#include <cstdlib>

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

__device__ __forceinline__ double ld_stream1(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
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

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// smem row strides chosen so a warp's 8x4 fragment reads hit each bank pair at most twice
__host__ __device__ __forceinline__ int apply_x_stride(int kp) { return kp + ((4 - kp % 16) + 16) % 16; }
__host__ __device__ __forceinline__ int apply_b_stride(int ncol) { return ncol + 8; }

constexpr int kApplyKC = 16;      // K rows per pipeline stage
constexpr int kApplyStages = 3;   // cp.async ring depth

template <int TM, int NTW>
__global__ void __launch_bounds__(128) apply_dmma_kernel(DevOperator op, const double* __restrict__ x,
                                                         double* __restrict__ y, double* pq_acc,
                                                         const PcgScalars* guard) {
  if (stopped(guard)) return;
  constexpr int MT = TM / 8;
  constexpr int NCOL = 32 * NTW;  // columns of this CTA's group: 4 warps x NTW n8-tiles
  extern __shared__ double smem[];
  const int n = op.n_loc, nm = op.n_mat, KP = op.kp, LDN = op.ldn;
  const int XS = apply_x_stride(KP), BS = apply_b_stride(NCOL);
  double* Bs = smem;                               // [stages][KC][BS]
  double* X = Bs + kApplyStages * kApplyKC * BS;   // [TM][XS], zero padded
  double* C = X + TM * XS;                         // [TM][nm]
  int* D = reinterpret_cast<int*>(C + TM * nm);    // [TM][n]
  const int col0 = blockIdx.y * NCOL;
  const int ncols = min(NCOL, LDN - col0);         // multiple of 8
  const int ktot = nm * KP;                        // rows of the concatenated [R_0; ...; R_{nm-1}]
  const int nchunks = (ktot + kApplyKC - 1) / kApplyKC;
  const double* __restrict__ Rcat = op.Rt;

  auto issue = [&](int c) {
    if (c < nchunks) {
      double* dst = Bs + (c % kApplyStages) * kApplyKC * BS;
      const int pieces_per_row = ncols / 2;  // 16-byte pieces
      for (int p = threadIdx.x; p < kApplyKC * pieces_per_row; p += blockDim.x) {
        const int r = p / pieces_per_row, q = p - r * pieces_per_row;
        const int krow = c * kApplyKC + r;
        if (krow < ktot) cp_async16(dst + r * BS + 2 * q, Rcat + (size_t)krow * LDN + col0 + 2 * q);
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);

  const int64_t c0 = (int64_t)blockIdx.x * TM;
  const int64_t rem = op.n_cells - c0;
  const int nc = rem < TM ? (int)rem : TM;
  for (int k = threadIdx.x; k < TM * XS; k += blockDim.x) {
    const int c = k / XS, j = k - c * XS;
    const int gd = (c < nc && j < n) ? op.dofmap_m[(c0 + c) * n + j] : -1;
    if (j < n) D[c * n + j] = gd;
    X[k] = (gd >= 0) ? x[gd] : 0.0;
  }
  for (int k = threadIdx.x; k < TM * nm; k += blockDim.x) {
    const int c = k / nm;
    C[k] = (c < nc) ? op.coef[(c0 + c) * nm + (k - c * nm)] : 0.0;
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double acc[MT][NTW][2];
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < NTW; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
  bool live[NTW];
#pragma unroll
  for (int q = 0; q < NTW; ++q) live[q] = (warp + 4 * q) * 8 < ncols;

  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<kApplyStages - 2>();
    __syncthreads();  // chunk c landed for everyone; slot (c+2)%3 is free again
    issue(c + kApplyStages - 1);
    const double* Bc = Bs + (c % kApplyStages) * kApplyKC * BS;
#pragma unroll
    for (int k4 = 0; k4 < kApplyKC / 4; ++k4) {
      const int kg = c * kApplyKC + k4 * 4;  // first K row of this k-step (KP is a multiple of 4)
      if (kg >= ktot) break;
      const int s = kg / KP, j = kg - s * KP + t;
      double a[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) a[m] = C[(m * 8 + g) * nm + s] * X[(m * 8 + g) * XS + j];
      double b[NTW];
#pragma unroll
      for (int q = 0; q < NTW; ++q) b[q] = Bc[(k4 * 4 + t) * BS + (warp + 4 * q) * 8 + g];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int q = 0; q < NTW; ++q)
          if (live[q]) dmma884(acc[m][q][0], acc[m][q][1], a[m], b[q]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C fragment (row g, cols 2t, 2t+1) -> scatter-add, fused p.(Ap)
  double pq = 0;
#pragma unroll
  for (int m = 0; m < MT; ++m)
#pragma unroll
    for (int q = 0; q < NTW; ++q) {
      if (!live[q]) continue;
      const int cell = m * 8 + g;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int col = col0 + (warp + 4 * q) * 8 + 2 * t + i;
        if (col < n && cell < nc) {
          const int gd = D[cell * n + col];
          if (gd >= 0) {
            atomicAdd(y + gd, acc[m][q][i]);
            pq = fma(X[cell * XS + col], acc[m][q][i], pq);
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

// B-stationary variant for n_mat * n_loc * 8 columns that fit in shared memory:
// a CTA owns NTC n8-tiles (8*NTC output columns) and keeps the matching slice
// of the stacked reference matrices [R_0; ...; R_{nm-1}] resident in smem for
// its whole range of cells; each warp loops over m-tiles of 8 cells: gather x
// (8 x n), K-loop of DMMA.8x8x4 with A = c_s X (scaled in registers) and B from
// the resident slice, scatter-add. R is read from L2 once per CTA.
constexpr int kBstStride = 8;  // smem row stride (doubles) of the B slice: 4 K rows x 8 cols -> 2 wavefronts
__host__ __device__ __forceinline__ int bst_x_stride(int kp) { return kp + ((4 - kp % 16) + 16) % 16; }

// B-stationary apply: a CTA owns one n8-tile (8 output columns) and keeps the
// matching K x 8 slice of the stacked reference matrices [R_0; ...; R_{nm-1}]
// resident in shared memory for its whole range of cells (R read from L2 once
// per CTA). Per m-tile of 8 cells: cooperative gather of x (8 x n), split-K
// DMMA.8x8x4 over the 4 warps (A = c_s X scaled in registers, B from the
// resident slice), cross-warp reduction in smem, scatter-add.
//
// PCG mode (fused PCG step): the gathered vector is the new search
// direction p_k = z_k + beta_k p_{k-1} (beta_k = (r_k.z_k)/(r_{k-1}.z_{k-1}),
// beta_0 = 0), written once per dof by its owner cell; ||z_k||^2 (owners) and
// p_k.A p_k are reduced, and the last CTA applies the stopping test of R-A16 to
// z_k and advances the iteration counter.
template <bool PCG>
__global__ void __launch_bounds__(128) apply_bst_kernel(DevOperator op, const double* __restrict__ x,
                                                        double* __restrict__ y, double* pq_acc,
                                                        const PcgScalars* guard, int cells_per_cta,
                                                        PcgScalars* sc, double* pbuf0, double* pbuf1) {
  if (stopped(guard)) return;
  extern __shared__ double smem[];
  double beta = 0.0;
  const double* p_old = nullptr;
  double* p_new = nullptr;
  int kit = 0;
  if (PCG) {
    volatile PcgScalars* v = sc;
    kit = v->k;
    beta = kit == 0 ? 0.0 : v->rz_acc / v->rz_old;
    p_old = (kit & 1) ? pbuf0 : pbuf1;
    p_new = (kit & 1) ? pbuf1 : pbuf0;
  }
  double zz = 0.0;
  const int n = op.n_loc, nm = op.n_mat, KP = op.kp, LDN = op.ldn;
  const int XS = bst_x_stride(KP);
  const int ktot = nm * KP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double* Bst = smem;                              // [ktot][8]
  double* X = Bst + (size_t)ktot * kBstStride;     // [8][XS]
  double* C = X + 8 * XS;                          // [8][nm]
  double* red = C + 8 * nm;                        // [4 warps][32 lanes][2]
  int* D = reinterpret_cast<int*>(red + 4 * 64);   // [8][8] dofs of this CTA's columns
  const int col0 = blockIdx.y * 8;
  for (int e = threadIdx.x; e < ktot * 4; e += blockDim.x) {
    const int k = e >> 2, c2 = e & 3;
    const double2 v = __ldg(reinterpret_cast<const double2*>(op.Rt + (size_t)k * LDN + col0 + 2 * c2));
    Bst[k * kBstStride + 2 * c2] = v.x;
    Bst[k * kBstStride + 2 * c2 + 1] = v.y;
  }
  // split-K: warp w owns k-steps [ks0, ks1) of the ktot/4 steps
  const int nsteps = ktot / 4;
  const int ks0 = (warp * nsteps) / 4, ks1 = ((warp + 1) * nsteps) / 4;
  const int64_t cbeg = (int64_t)blockIdx.x * cells_per_cta;
  const int64_t cend = min((int64_t)op.n_cells, cbeg + cells_per_cta);
  double pq = 0;
  for (int64_t cb = cbeg; cb < cend; cb += 8) {
    const int nc = (int)min((int64_t)8, cend - cb);
    __syncthreads();  // previous m-tile fully consumed (and the B slice loaded)
    // gather in batches of 8 elements per thread: all dof-map loads, then all
    // vector loads, then the smem stores (8 independent loads in flight per thread)
    constexpr int GB = 8;
    for (int e0 = 0; e0 < 8 * XS; e0 += GB * 128) {
      int gd[GB], cc[GB], jj[GB];
#pragma unroll
      for (int i = 0; i < GB; ++i) {
        const int e = e0 + i * 128 + threadIdx.x;
        const int c = e / XS, j = e - c * XS;
        cc[i] = c;
        jj[i] = j;
        gd[i] = (e < 8 * XS && c < nc && j < n) ? op.dofmap_m[(cb + c) * n + j] : -1;
      }
      double val[GB], zv[GB];
#pragma unroll
      for (int i = 0; i < GB; ++i) {
        zv[i] = gd[i] >= 0 ? x[gd[i]] : 0.0;
        val[i] = (PCG && gd[i] >= 0) ? p_old[gd[i]] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < GB; ++i) {
        const int e = e0 + i * 128 + threadIdx.x;
        if (e >= 8 * XS) continue;
        double v = zv[i];
        if (PCG && gd[i] >= 0) {
          v = fma(beta, val[i], zv[i]);
          if (blockIdx.y == 0 && op.owner[(cb + cc[i]) * n + jj[i]]) {
            p_new[gd[i]] = v;
            zz = fma(zv[i], zv[i], zz);
          }
        }
        X[e] = v;
        const int j = jj[i];
        if (j >= col0 && j < col0 + 8) D[cc[i] * 8 + (j - col0)] = (j < n) ? gd[i] : -1;
      }
    }
    for (int e = threadIdx.x; e < 8 * nm; e += blockDim.x) {
      const int c = e / nm;
      C[e] = (c < nc) ? op.coef[(cb + c) * nm + (e - c * nm)] : 0.0;
    }
    __syncthreads();
    // two independent accumulator chains (even / odd k-steps) hide the DMMA latency
    double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
    int s = (ks0 * 4) / KP, j = ks0 * 4 - s * KP;
    double cs = C[g * nm + s];
    const double* xr = X + g * XS + t;
    const double* br = Bst + (size_t)(ks0 * 4 + t) * kBstStride + g;
    auto advance = [&]() {
      br += 4 * kBstStride;
      j += 4;
      if (j >= KP) {
        j = 0;
        ++s;
        cs = (s < nm) ? C[g * nm + s] : 0.0;
      }
    };
    int ks = ks0;
#pragma unroll 2
    for (; ks + 1 < ks1; ks += 2) {
      dmma884(c0, c1, cs * xr[j], *br);
      advance();
      dmma884(d0, d1, cs * xr[j], *br);
      advance();
    }
    if (ks < ks1) dmma884(c0, c1, cs * xr[j], *br);
    red[(warp * 32 + lane) * 2] = c0 + d0;
    red[(warp * 32 + lane) * 2 + 1] = c1 + d1;
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        double v = red[lane * 2 + i] + red[(32 + lane) * 2 + i] + red[(64 + lane) * 2 + i] + red[(96 + lane) * 2 + i];
        const int col = 2 * t + i;  // row g = cell, column col0 + col
        const int gd = (g < nc && col0 + col < n) ? D[g * 8 + col] : -1;
        if (gd >= 0) {
          atomicAdd(y + gd, v);
          pq = fma(X[g * XS + col0 + col], v, pq);
        }
      }
    }
  }
  if (PCG) {
    __shared__ double sh[32];
    __shared__ bool last;
    const double spq = block_sum(pq, sh);
    const double szz = block_sum(zz, sh);
    if (threadIdx.x == 0) {
      atomicAdd(&sc->pq2[kit & 1], spq);
      atomicAdd(&sc->zz, szz);
      __threadfence();
      const unsigned nblocks = gridDim.x * gridDim.y;
      last = atomicAdd(&sc->ticket, 1u) == nblocks - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {  // stopping test on z_k (R-A16), then advance k
      __threadfence();
      volatile PcgScalars* v = sc;
      const double zn = sqrt(v->zz);
      if (kit == 0) {
        sc->z0 = zn;
        sc->iters = 0;
        if (zn == 0.0) {
          sc->done = 1;
          sc->converged = 1;
        } else if (v->maxit <= 0) {
          sc->done = 1;
        }
      } else {
        sc->iters = kit;
        if (zn <= v->rtol * v->z0) {
          sc->done = 1;
          sc->converged = 1;
        } else if (kit >= v->maxit) {
          sc->done = 1;
        }
      }
      sc->rz_old = v->rz_acc;
      sc->pq2[(kit + 1) & 1] = 0.0;  // accumulator of the next fused apply
      sc->rz_acc = 0.0;
      sc->zz = 0.0;
      sc->ticket = 0;
      sc->k = kit + 1;
    }
  } else if (pq_acc) {
    __shared__ double sh[32];
    double sum = block_sum(pq, sh);
    if (threadIdx.x == 0) atomicAdd(pq_acc, sum);
  }
}

size_t bst_smem_bytes(const DevOperator& op) {
  return sizeof(double) * ((size_t)op.n_mat * op.kp * kBstStride + 8 * (size_t)bst_x_stride(op.kp) + 8 * op.n_mat + 256) +
         sizeof(int) * 64;
}

template <bool PCG>
cudaError_t launch_apply_bst(const DevOperator& op, const double* x, double* y, double* pq_acc,
                             const PcgScalars* guard, cudaStream_t s, PcgScalars* sc = nullptr,
                             double* pbuf0 = nullptr, double* pbuf1 = nullptr) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(apply_bst_kernel<PCG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    configured = true;
  }
  const size_t sm = bst_smem_bytes(op);
  const int groups = op.ldn / 8;
  const int per_sm = (int)std::min<size_t>(4, (220 * 1024) / (sm + 1024));
  int64_t gx = (148 * std::max(1, per_sm) + groups - 1) / groups;
  int64_t cpc = (op.n_cells + gx - 1) / gx;
  cpc = (cpc + 7) / 8 * 8;
  gx = (op.n_cells + cpc - 1) / cpc;
  dim3 grid((unsigned)gx, (unsigned)groups);
  apply_bst_kernel<PCG><<<grid, 128, sm, s>>>(op, x, y, pq_acc, guard, (int)cpc, sc, pbuf0, pbuf1);
  return cudaGetLastError();
}
template <int TM, int NTW>
cudaError_t launch_apply_dmma(const DevOperator& op, const double* x, double* y, double* pq_acc,
                              const PcgScalars* guard, cudaStream_t s) {
  const int ncol = 32 * NTW;
  size_t sm = sizeof(double) * ((size_t)kApplyStages * kApplyKC * apply_b_stride(ncol) +
                                (size_t)TM * apply_x_stride(op.kp) + (size_t)TM * op.n_mat) +
              sizeof(int) * (size_t)TM * op.n_loc;
  static bool configured = false;  // first call happens in rdr_setup (outside stream capture)
  if (!configured) {
    cudaFuncSetAttribute(apply_dmma_kernel<TM, NTW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  dim3 grid((unsigned)((op.n_cells + TM - 1) / TM), (unsigned)((op.ldn + ncol - 1) / ncol));
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
    // exact packed layout (setup.hpp: patch_tile_offset): rows valid rows in block row I
    const int rows = min(32, n - 32 * I);
    const double* tb = T + 512LL * I * I + 16LL * I + (int64_t)J * 32 * rows;
    double a[32];
    const double ri = rl[I * 32 + lane];
    double row = 0;
    if (J < I) {
      if (lane < rows) {
        const double4* tp = reinterpret_cast<const double4*>(tb) + lane;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          double4 v = ld_stream4(tp + k4 * rows);
          a[4 * k4] = v.x;
          a[4 * k4 + 1] = v.y;
          a[4 * k4 + 2] = v.z;
          a[4 * k4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 32; ++k) a[k] = 0.0;
      }
      const double* rJ = rl + J * 32;
#pragma unroll
      for (int k = 0; k < 32; ++k) row = fma(a[k], rJ[k], row);
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] *= ri;
    } else {
      // diagonal tile, lower triangle packed by columns: (i,k), k <= i, at k*rows - k(k-1)/2 + i - k
#pragma unroll
      for (int k = 0; k < 32; ++k)
        a[k] = (k <= lane && lane < rows) ? ld_stream1(tb + k * rows - k * (k - 1) / 2 + (lane - k)) : 0.0;
      const double* rI = rl + I * 32;
#pragma unroll
      for (int k = 0; k < 32; ++k) row = fma(a[k], rI[k], row);
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] = (k < lane) ? a[k] * ri : 0.0;  // strict lower part, transposed
    }
    atomicAdd(zl + I * 32 + lane, row);
    transpose_reduce_stage<16>(a, lane);
    transpose_reduce_stage<8>(a, lane);
    transpose_reduce_stage<4>(a, lane);
    transpose_reduce_stage<2>(a, lane);
    transpose_reduce_stage<1>(a, lane);
    atomicAdd(zl + J * 32 + lane, a[0]);
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

// fused path, after the fused apply of iteration k: alpha = (r.z)/(p.Ap),
// x += alpha p, r -= alpha q, q = 0, then the interior point-Jacobi part of
// P^-1 on the new r (z_I = r_I / A_II, z_Gamma = 0; Thm 5.1) with
// its share of r.z.
__global__ void pcg_update_jacobi_kernel(PcgScalars* sc, DevPrecond pc, const double* __restrict__ p0,
                                         const double* __restrict__ p1, double* __restrict__ q,
                                         double* __restrict__ x, double* __restrict__ r, double* __restrict__ z) {
  if (stopped(sc)) return;
  const int kk = *((volatile int32_t*)&sc->k) - 1;  // iteration of the apply that just ran
  const double* __restrict__ p = (kk & 1) ? p1 : p0;
  const double alpha = sc->rz_old / sc->pq2[kk & 1];
  double part = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_total; i += stride) {
    x[i] = fma(alpha, p[i], x[i]);
    const double rn = fma(-alpha, q[i], r[i]);
    r[i] = rn;
    q[i] = 0.0;
    if (i < pc.off3) {
      z[i] = 0.0;
    } else {
      const double zi = pc.dinv[i - pc.off3] * rn;
      z[i] = zi;
      part = fma(rn, zi, part);
    }
  }
  if (pc.ubuf)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_cg_iface; i += stride) pc.ubuf[i] = 0.0;
  __shared__ double sh[32];
  const double s = block_sum(part, sh);
  if (threadIdx.x == 0) atomicAdd(&sc->rz_acc, s);
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
  // B-stationary kernel when the stacked reference-matrix slice fits in shared memory
  static const bool force_stream = std::getenv("RDR_APPLY_STREAM") != nullptr;
  if (bst_smem_bytes(op) <= 220 * 1024 && !force_stream) return launch_apply_bst<false>(op, x, y, pq_acc, guard, s);
  // n8-tiles per warp (column groups of 4*NTW tiles go to gridDim.y); cells per CTA
  // chosen so the grid covers the 148 SMs about twice
  const int per_warp = (op.ldn / 8 + 3) / 4;
  const int ntw = per_warp <= 1 ? 1 : per_warp <= 2 ? 2 : per_warp <= 3 ? 3 : 4;
  const int64_t groups = (op.ldn / 8 + 4 * ntw - 1) / (4 * ntw);
  const int64_t ctas32 = (op.n_cells + 31) / 32 * groups, ctas16 = (op.n_cells + 15) / 16 * groups;
  const int tm = ctas32 >= 296 ? 32 : (ctas16 >= 296 ? 16 : 8);
#define RDR_DMMA_CASE(TM, NTW) \
  if (tm == TM && ntw == NTW) return launch_apply_dmma<TM, NTW>(op, x, y, pq_acc, guard, s);
  RDR_DMMA_CASE(8, 1) RDR_DMMA_CASE(8, 2) RDR_DMMA_CASE(8, 3) RDR_DMMA_CASE(8, 4)
  RDR_DMMA_CASE(16, 1) RDR_DMMA_CASE(16, 2) RDR_DMMA_CASE(16, 3) RDR_DMMA_CASE(16, 4)
  RDR_DMMA_CASE(32, 1) RDR_DMMA_CASE(32, 2) RDR_DMMA_CASE(32, 3) RDR_DMMA_CASE(32, 4)
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

bool fused_pcg_supported(const DevOperator& op) {
  static const bool off = std::getenv("RDR_PCG_UNFUSED") != nullptr || std::getenv("RDR_APPLY_STREAM") != nullptr;
  return op.Rt && op.owner && !off && bst_smem_bytes(op) <= 220 * 1024;
}

cudaError_t launch_pcg_fused_apply(const DevOperator& op, PcgScalars* sc, const double* z, double* p0, double* p1,
                                   double* q, cudaStream_t s) {
  return launch_apply_bst<true>(op, z, q, nullptr, sc, s, sc, p0, p1);
}

cudaError_t launch_pcg_update_jacobi(PcgScalars* sc, const DevPrecond& pc, const double* p0, const double* p1,
                                     double* q, double* x, double* r, double* z, cudaStream_t s) {
  pcg_update_jacobi_kernel<<<vec_grid(pc.n_total), kVecThreads, 0, s>>>(sc, pc, p0, p1, q, x, r, z);
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
