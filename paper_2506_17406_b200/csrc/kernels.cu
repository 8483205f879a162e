// sm_100a kernels of the Riesz-map PCG hot path.
//
//  * apply_tc_kernel   : gather x_e -> y_e = sum_s c_{e,s} R_s x_e on DMMA -> scatter-add
//                        (north_star operator apply; matrix-free action P:2267-2275)
//  * precond_init      : interior point-Jacobi z_I = r_I / A_II (Thm 5.1)
//  * patch_ldg_kernel / patch_warp_kernel: additive star patches
//                        z += E_m A_m^{-1} E_m^T r with the stored packed inverses
//                        streamed from HBM (Eq. 5.4 / 5.12)
//  * gather_grad / scatter_grad : the discrete gradient of the H(curl) potential
//                        patches (R-A12, Lemma 4.3)
//  * pcg_*             : fused PCG vector updates and reductions (R-A16)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.hpp"

namespace rdr {

namespace {

constexpr int kVecThreads = 256;

// Kernels are launched with the programmatic stream-serialization attribute
// (PDL, see pdl_wait). Every kernel launched this way calls pdl_wait() before
// it reads anything a predecessor kernel writes.
constexpr bool pdl_enabled() { return true; }
constexpr bool pdl_patch_enabled() { return true; }
template <typename... Params, typename... Args>
cudaError_t launch_kx(bool pdl, void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                      Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<Params>(args)...);
}
template <typename... Params, typename... Args>
cudaError_t launch_k(void (*kernel)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  return launch_kx(true, kernel, grid, block, smem, s, args...);
}

// The PCG stop flag, read once the previous kernel's writes are visible (after
// griddepcontrol.wait): a relaxed GPU-scope load (a volatile read compiles to a
// system-scope LDG.STRONG.SYS, which every thread of a large grid then pays).
__device__ __forceinline__ bool stopped(const PcgScalars* g) {
  if (g == nullptr) return false;
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(&g->done) : "memory");
  return v != 0;
}

// Programmatic dependent launch (PDL): a kernel launched with the programmatic
// stream-serialization attribute may start while its predecessor drains; it
// loads only constant data (dof maps, patch metadata, reference stack) before
// griddepcontrol.wait, which returns once the predecessor grid has completed
// and its memory is visible. Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// dependents may launch once every CTA has finished its main loop (an early
// trigger let waiting dependent CTAs take SM slots from the patch kernel)
__device__ __forceinline__ bool pdl_late() { return true; }

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

// ---------------------------------------------------------------- operator apply on FP64 tensor cores
// Y[c][i] = sum_s c_{c,s} sum_j X[c][j] R_s[j][i]: one GEMM with M = cells,
// N = n_loc, K = n_mat * kp (the stacked reference matrices), on DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; sm_100a has no tcgen05 kind::f64,
// SURVEY F1/F2).
//
// CTA = BM cells x one 32-column group of N. The CTA's B operand (the group's
// K x 32 slice of the stack, stored swizzled in HBM/L2) streams through an
// 8-slot shared-memory ring by cp.async.bulk (TMA bulk copies) completing on
// mbarriers; a dedicated producer warp refills slots as consumers release them.
// Consumer warps own 16 cells x 32 columns (2 x 4 DMMA tiles, 16 FP64
// accumulators per lane: every A fragment is reused 4x and every B fragment
// 2x from registers) and split K in KS groups (chunk c -> group c % KS); the
// groups' partial sums are reduced through shared memory. A = c_s X is scaled
// in registers (c_s changes every kp/4 k-steps). The gathered X tile (BM x kp)
// stays in shared memory for the whole K loop; the epilogue scatter-adds with
// red.global.add.f64 and accumulates p.(Ap) (or, in PCG mode, runs the fused
// direction update and stopping test).
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Release a TMA ring slot: the CTA-scope fence makes this thread's earlier
// shared-memory loads of the slot complete before the arrive (ptxas issues a
// plain mbarrier.arrive right behind still-outstanding LDS, and the TMA refill
// it unblocks then races those loads).
__device__ __forceinline__ void mbar_release(uint64_t* bar) {
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

constexpr int kApplyCols = 32;   // N columns per work unit: one 32-column group of the stack
constexpr int kLutShift = 9;     // op.lut[i] = (local entity << 9) | position inside the entity's block

// smem row stride of X: == 4 (mod 16) doubles, so a warp's 8x4 A-fragment read is conflict-free
__host__ __device__ __forceinline__ int apply_x_stride(int kp) { return kp + ((4 - kp % 16) + 16) % 16; }

// Warp layout: BM cells per work unit, warp tile 16 cells x 8*NQ columns,
// MW = BM/16 warps along M, NW = 32/(8 NQ) along N, KS K-split groups:
// MW*NW*KS MMA warps plus one TMA producer warp.
__host__ __device__ constexpr int apply_mma_warps(int BM, int NQ, int KS) { return (BM / 16) * (32 / (8 * NQ)) * KS; }

// One ring chunk = one 4-row step j4 of all NM reference matrices: rows
// (j4, s, t) = R_s[4 j4 + t][group columns], t = 0..3, 4 NM x 32 doubles.
__host__ __device__ constexpr int apply_chunk_doubles(int nm) { return 4 * nm * kApplyCols; }

struct ApplySmem {
  size_t ring, x, red, c, eb, lut, own, total;
};
__host__ __device__ inline ApplySmem apply_smem_layout(int BM, int NQ, int KS, int S, int kp, int nm) {
  ApplySmem L;
  const int MW = BM / 16, NW = 32 / (8 * NQ);
  L.ring = sizeof(uint64_t) * 2 * S;
  L.x = L.ring + sizeof(double) * (size_t)S * apply_chunk_doubles(nm);
  L.red = L.x + sizeof(double) * (size_t)BM * apply_x_stride(kp);
  L.c = L.red + sizeof(double) * (size_t)(KS - 1) * MW * NW * 16 * 8 * NQ;
  L.eb = L.c + sizeof(double) * (size_t)BM * nm;
  L.lut = L.eb + sizeof(int32_t) * (size_t)BM * 16;
  L.own = L.lut + sizeof(uint16_t) * (size_t)((kp + 3) & ~3);
  L.total = L.own + sizeof(uint16_t) * (size_t)((BM + 3) & ~3);
  return L;
}

__device__ __forceinline__ void mma_bar_sync(int nthreads) {  // named barrier 1: the MMA warps only
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// Operator apply y += A x on FP64 tensor cores:
// Y[c][i] = sum_s c_{c,s} sum_j X[c][j] R_s[j][i], one GEMM with M = cells,
// N = n_loc, K = n_mat * kp (the stacked reference matrices), on DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4; sm_100a has no tcgen05 kind::f64,
// SURVEY F1/F2).
//
// Persistent work split: the output is cut into units (a tile of BM cells) x
// (a 32-column group), ntiles * ngroups of them in tile-major order, and CTA b
// takes the contiguous range [U b / G, U (b+1) / G): balanced to one unit, and
// a CTA gathers each tile once for all the column groups it covers (a tile
// split between two CTAs is gathered by both). The producer warp streams the
// group slices of the reference stack for all the CTA's units back to back
// through an S-slot ring of cp.async.bulk (TMA) copies completing on
// mbarriers, so the ring never drains between units. The stack is stored
// j-major: chunk j4 holds rows 4 j4 .. 4 j4 + 3 of every R_s, so a chunk's K
// loop is NM branch-free k-steps that reuse one pair of X values and the
// cells' NM coefficients held in registers (A = c_s X is formed with one DMUL
// per fragment). MMA warps own 16 cells x 8*NQ columns and split the chunks
// in KS groups (chunk j4 -> group j4 % KS) reduced through shared memory.
// The gather reads x (PCG mode: z and p_{k-1}) through per-cell entity bases
// (ebase: first global dof of each of the 15 local entities, R-A9 numbering)
// and the element's (entity, position) table, so no per-cell dof map is
// stored; the epilogue scatter-adds with red.global.add.f64 and accumulates
// p.(Ap). In PCG mode the gather also forms p_k = z_k + beta_k p_{k-1}, which
// the owner cell of each entity writes once (the CTA holding the tile's
// column group 0), and the last CTA performs the stopping test (R-A16).
template <int BM, int NQ, int KS, int NM, int NM0, int MINB, bool PCG>
__global__ void __launch_bounds__((apply_mma_warps(BM, NQ, KS) + 1) * 32, MINB)
    apply_tc_kernel(DevOperator op, int S, const double* __restrict__ x, double* __restrict__ y, double* pq_acc,
                    const PcgScalars* guard, PcgScalars* sc, double* pbuf0, double* pbuf1) {
  constexpr int MW = BM / 16, NW = 32 / (8 * NQ), NWARP = apply_mma_warps(BM, NQ, KS);
  constexpr int NT = NWARP * 32;
  constexpr int kChunk = apply_chunk_doubles(NM);
  constexpr uint32_t kChunkBytes = kChunk * sizeof(double);
  // H(curl) / H(div) (NM0 = 6 < NM): the curl (div-div) matrices s >= NM0 vanish outside the
  // leading ncb rows / columns of the lut_tc order, so chunks of rows >= ncb or groups of
  // columns >= ncb carry, copy and multiply only the NM0 mass matrices (0.70 of the flops
  // for H(curl) at p >= 8, 0.87 for H(div)); H(grad): NM0 = NM
  constexpr uint32_t kChunkBytes0 = apply_chunk_doubles(NM0) * sizeof(double);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int n = op.n_loc, kp = op.kp;
  const int XS = apply_x_stride(kp);
  const ApplySmem L = apply_smem_layout(BM, NQ, KS, S, kp, NM);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + S;
  double* ring = reinterpret_cast<double*>(smem_raw + L.ring);  // [S][4 NM][32] swizzled
  double* X = reinterpret_cast<double*>(smem_raw + L.x);        // [BM][XS]
  double* red = reinterpret_cast<double*>(smem_raw + L.red);    // [KS-1][MW*NW][16 * 8NQ] per lane
  double* C = reinterpret_cast<double*>(smem_raw + L.c);        // [BM][NM]
  int32_t* EB = reinterpret_cast<int32_t*>(smem_raw + L.eb);    // [BM][16]
  uint16_t* LUT = reinterpret_cast<uint16_t*>(smem_raw + L.lut);
  uint16_t* OWN = reinterpret_cast<uint16_t*>(smem_raw + L.own);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp == NWARP;
  const int nchunks = kp / 4;
  const int64_t U = (int64_t)op.ntiles * op.ngroups;
  const int64_t u0 = U * blockIdx.x / gridDim.x, u1 = U * (blockIdx.x + 1) / gridDim.x;
  const int64_t total_chunks = (u1 - u0) * nchunks;

  // ---- prologue on constant data only (overlaps the previous kernel under PDL)
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MW * NW * 32);  // every lane of the chunk's K group releases its own reads
    }
    mbar_fence_init();
  }
  for (int i = threadIdx.x; i < kp; i += blockDim.x) LUT[i] = i < n ? op.lut_tc[i] : 0;
  __syncthreads();
  const int prefilled = (int)min((int64_t)S, total_chunks);
  // producer cursor over the CTA's chunk sequence: unit group / chunk / ring slot,
  // advanced incrementally (no 64-bit divisions on the issue path)
  int p_grp = (int)(u0 % op.ngroups), p_c = 0, p_slot = 0;
  auto issue_next = [&]() {
    const double* src = op.Bsw + ((size_t)p_grp * nchunks + p_c) * kChunk;
    const uint32_t bytes = (NM0 == NM || (4 * p_c < op.ncb && 32 * p_grp < op.ncb)) ? kChunkBytes : kChunkBytes0;
    mbar_expect_tx(&full[p_slot], bytes);
    bulk_g2s(ring + p_slot * kChunk, src, bytes, &full[p_slot]);
    if (++p_c == nchunks) {
      p_c = 0;
      if (++p_grp == op.ngroups) p_grp = 0;
    }
    if (++p_slot == S) p_slot = 0;
  };
  if (producer && lane == 0)
    for (int q = 0; q < prefilled; ++q) issue_next();

  pdl_wait();
  if (stopped(guard)) {  // drain the prefilled ring before the CTA's shared memory goes away
    if (producer && lane == 0)
      for (int q = 0; q < prefilled; ++q) mbar_wait(&full[q], 0);
    return;
  }

  double pq = 0.0, zz = 0.0;
  int kit = 0;
  if (producer) {
    if (lane == 0) {
      uint32_t ph = 0;  // parity of the slot's previous use
      for (int64_t q = prefilled; q < total_chunks; ++q) {
        if (p_slot == 0 && q > prefilled) ph ^= 1u;
        mbar_wait(&empty[p_slot], ph);
        issue_next();
      }
    }
  } else {
    // ---- PCG mode: direction update p_k = z_k + beta_k p_{k-1} folded into the gather
    double beta = 0.0;
    const double* p_old = nullptr;
    double* p_new = nullptr;
    if (PCG) {  // the scalars once per CTA (shared), not one strong load per thread
      __shared__ double s_beta;
      __shared__ int s_kit;
      if (threadIdx.x == 0) {
        volatile PcgScalars* v = sc;
        s_kit = v->k;
        const double rz_old = v->rz_old;  // 0 only before the first direction (or in a timing loop)
        s_beta = (s_kit == 0 || rz_old == 0.0) ? 0.0 : v->rz_acc / rz_old;
      }
      mma_bar_sync(NT);
      kit = s_kit;
      beta = s_beta;
      p_old = (kit & 1) ? pbuf0 : pbuf1;
      p_new = (kit & 1) ? pbuf1 : pbuf0;
    }
    const int tid = threadIdx.x;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int kg = warp / (MW * NW), wmn = warp % (MW * NW), mw = wmn % MW, nw = wmn / MW;
    int boff[NQ];  // B fragment (k, col) of a 4-row k-step at k*32 + (col ^ ((k & 3) << 2))
#pragma unroll
    for (int q = 0; q < NQ; ++q) boff[q] = t4 * kApplyCols + ((nw * 8 * NQ + q * 8 + g8) ^ (t4 << 2));
    const double* xr0 = X + (mw * 16 + g8) * XS + t4;
    const double* xr1 = xr0 + 8 * XS;
    double cs0[NM], cs1[NM];  // the two fragment rows' cell coefficients
    int64_t tile_cur = -1;
    int64_t qbase = 0;
    for (int64_t u = u0; u < u1; ++u, qbase += nchunks) {
      const int64_t tile = u / op.ngroups;
      const int grp = (int)(u % op.ngroups);
      if (tile != tile_cur) {
        // ---- gather the tile (once per CTA): entity bases, coefficients, owner bits, then X
        mma_bar_sync(NT);  // every read of the previous tile's X / C / EB is done
        const int64_t c0 = tile * BM;
        const int nc = (int)min((int64_t)BM, op.n_cells - c0);
        for (int e = tid; e < BM * 16; e += NT) EB[e] = (e >> 4) < nc ? op.ebase[c0 * 16 + e] : -1;
        for (int e = tid; e < BM * NM; e += NT) C[e] = e / NM < nc ? op.coef[c0 * NM + e] : 0.0;
        for (int e = tid; e < BM; e += NT) OWN[e] = e < nc ? op.own[c0 + e] : 0;
        mma_bar_sync(NT);
        const bool writer = PCG && grp == 0;  // the CTA that holds column group 0 of the tile
        constexpr int GB = 4;
        const int total = BM * XS;
        for (int e0 = 0; e0 < total; e0 += GB * NT) {
          int gid[GB];
          bool own[GB];
#pragma unroll
          for (int i = 0; i < GB; ++i) {
            const int e = e0 + i * NT + tid;
            const int c = e / XS, j = e - c * XS;
            gid[i] = -1;
            own[i] = false;
            if (e < total && j < n) {
              const int l = LUT[j];
              const int b = EB[c * 16 + (l >> kLutShift)];
              if (b >= 0) {
                gid[i] = b + (l & ((1 << kLutShift) - 1));
                own[i] = (OWN[c] >> (l >> kLutShift)) & 1;
              }
            }
          }
          double xv[GB], pv[GB];
#pragma unroll
          for (int i = 0; i < GB; ++i) {
            xv[i] = gid[i] >= 0 ? x[gid[i]] : 0.0;
            pv[i] = (PCG && gid[i] >= 0) ? p_old[gid[i]] : 0.0;
          }
#pragma unroll
          for (int i = 0; i < GB; ++i) {
            const int e = e0 + i * NT + tid;
            if (e >= total) continue;
            double v = xv[i];
            if (PCG && gid[i] >= 0) {
              v = fma(beta, pv[i], xv[i]);
              if (writer && own[i]) {
                p_new[gid[i]] = v;
                zz = fma(xv[i], xv[i], zz);
              }
            }
            X[e] = v;
          }
        }
        mma_bar_sync(NT);
#pragma unroll
        for (int s = 0; s < NM; ++s) {
          cs0[s] = C[(mw * 16 + g8) * NM + s];
          cs1[s] = C[(mw * 16 + 8 + g8) * NM + s];
        }
        tile_cur = tile;
      }

      // ---- K loop of the unit: chunk j4 (rows 4 j4.. of every R_s) by K group j4 % KS
      double acc[2][NQ][2];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
      // ring position of this warp's first chunk of the unit (one division per unit)
      int slot = (int)((qbase + kg) % S);
      uint32_t par = (uint32_t)(((qbase + kg) / S) & 1);
      const int cfull = (NM0 == NM || 32 * grp < op.ncb) ? op.ncb : 0;  // chunks c with 4 c < cfull: all NM
      for (int c = kg; c < nchunks; c += KS) {
        mbar_wait(&full[slot], par);
        const double* Bs = ring + slot * kChunk;
        const double x0 = xr0[4 * c], x1 = xr1[4 * c];
        auto kstep = [&](const int s) {
          const double a0 = cs0[s] * x0, a1 = cs1[s] * x1;
          double b[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) b[q] = Bs[s * 4 * kApplyCols + boff[q]];
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            dmma884(acc[0][q][0], acc[0][q][1], a0, b[q]);
            dmma884(acc[1][q][0], acc[1][q][1], a1, b[q]);
          }
        };
#pragma unroll
        for (int s = 0; s < NM0; ++s) kstep(s);
        if (NM0 < NM && 4 * c < cfull) {
#pragma unroll
          for (int s = NM0; s < NM; ++s) kstep(s);
        }
        // every lane releases the slot after its own loads of it completed (DESIGN.md §6:
        // an arrive right behind the LDS let the TMA refill race the loads)
        mbar_release(&empty[slot]);
        slot += KS;
        while (slot >= S) {
          slot -= S;
          par ^= 1u;
        }
      }

      // ---- K-split reduction, then scatter-add from K group 0
      if (KS > 1) {
        if (kg > 0) {
          double* dst = red + (((kg - 1) * MW * NW + wmn) * 16 * 8 * NQ) + lane;
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int q = 0; q < NQ; ++q)
#pragma unroll
              for (int i = 0; i < 2; ++i) dst[((m * NQ + q) * 2 + i) * 32] = acc[m][q][i];
        }
        mma_bar_sync(NT);
        if (kg == 0)
          for (int h = 1; h < KS; ++h) {
            const double* src = red + (((h - 1) * MW * NW + wmn) * 16 * 8 * NQ) + lane;
#pragma unroll
            for (int m = 0; m < 2; ++m)
#pragma unroll
              for (int q = 0; q < NQ; ++q)
#pragma unroll
                for (int i = 0; i < 2; ++i) acc[m][q][i] += src[((m * NQ + q) * 2 + i) * 32];
          }
      }
      if (kg == 0) {
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          const int row = mw * 16 + m * 8 + g8;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int col = grp * kApplyCols + nw * 8 * NQ + q * 8 + 2 * t4 + i;
              if (col < n) {
                const int l = LUT[col];
                const int b = EB[row * 16 + (l >> kLutShift)];
                if (b >= 0) {
                  atomicAdd(y + b + (l & ((1 << kLutShift) - 1)), acc[m][q][i]);
                  pq = fma(X[row * XS + col], acc[m][q][i], pq);
                }
              }
            }
        }
      }
      if (KS > 1) mma_bar_sync(NT);  // the reduction buffer is reused by the next unit
    }
  }
  if (pdl_late()) pdl_trigger();

  if (PCG) {
    __shared__ double sh[32];
    __shared__ bool last;
    const double spq = block_sum(pq, sh);
    const double szz = block_sum(zz, sh);
    if (threadIdx.x == 0) {
      atomicAdd(&sc->pq2[kit & 1], spq);
      atomicAdd(&sc->zz, szz);
      __threadfence();
      last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {  // stopping test on z_k (R-A16), then advance k
      __threadfence();
      volatile PcgScalars* v = sc;
      const double zn = sqrt(v->zz);
      if (kit == 0) {
        sc->z0 = zn;
        sc->z_last = zn;
        sc->iters = 0;
        if (zn == 0.0) {
          sc->done = 1;
          sc->converged = 1;
        } else if (v->maxit <= 0) {
          sc->done = 1;
        }
      } else {
        sc->iters = kit;
        sc->z_last = zn;
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
    const double sum = block_sum(pq, sh);
    if (threadIdx.x == 0) atomicAdd(pq_acc, sum);
  }
}

// ---------------------------------------------------------------- factored apply (H(curl), H(div))
// The reference matrices factor through L2-orthonormal bases of P_p (values) and
// P_{p-1} (curls): M^{ab} = FaM FbM^T, K^{ab} = FaK FbK^T (refelem.cpp, RefElement::F).
// The cell operator is y_e = F (Gm ⊗ I) F^T x_e on the value block plus the same with
// Gk on the curl block, i.e. two GEMMs per cell tile with a per-cell 3 x 3 mix between:
//   stage A (fact_stage_a_kernel): gather x_e (PCG mode: the direction update and
//            ||z||^2 as in apply_tc_kernel), U = X F  (K = n_loc, N = nf) -> op.ubuf;
//   stage B (fact_stage_b_kernel): V = mix(U) (and p.Ap = sum u.v), Y = V F^T
//            (K = nf, N = n_loc), scatter-add.
// 4 (n_loc + 3) (nf) flops per cell against 2 n_mat n_loc^2: 3.1x fewer for Ned1_6.
// DMMA.8x8x4 with A from shared memory and B = F read through L1/L2 (op.F is
// [kp][nfp], zero-padded, ~0.8 MB for Ned1_6). 8 warps, 16 cells per CTA, each warp
// 16 cells x 32 columns per pass.
constexpr int kFactWarps = 8, kFactNQ = 4;
// cells per tile of (stage A, stage B): op.fact 1 (16, 16), 2 (32, 32), 3 (32, 24: the V tile
// of stage B small enough for two CTAs per SM up to Ned1_6 / RT_7)
__host__ __device__ inline int fact_bm_a(int fact) { return fact == 1 ? 16 : 32; }
__host__ __device__ inline int fact_bm_b(int fact) { return fact == 1 ? 16 : fact == 2 ? 32 : 24; }

struct FactSmem {
  size_t x, eb, lut, own, total;
};
__host__ __device__ inline FactSmem fact_a_layout(int kp, int bm) {
  FactSmem L;
  L.x = 0;
  L.eb = L.x + sizeof(double) * (size_t)bm * apply_x_stride(kp);
  L.lut = L.eb + sizeof(int32_t) * bm * 16;
  L.own = L.lut + sizeof(uint16_t) * (size_t)((kp + 3) & ~3);
  L.total = L.own + sizeof(uint16_t) * bm;
  return L;
}
__host__ __device__ inline size_t fact_vs(int nfp) { return (size_t)nfp + 4; }  // V row stride (== 4 mod 16)
__host__ __device__ inline FactSmem fact_b_layout(int kp, int nfp, int bm) {
  FactSmem L;
  L.x = 0;  // V [bm][nfp + 4]
  L.eb = L.x + sizeof(double) * (size_t)bm * fact_vs(nfp);
  L.lut = L.eb + sizeof(int32_t) * bm * 16;
  L.own = L.lut + sizeof(uint16_t) * (size_t)((kp + 3) & ~3);  // coefficients [bm][n_mat <= 12] doubles
  L.total = L.own + sizeof(double) * bm * 12;
  return L;
}

template <int BM, bool PCG>
__global__ void __launch_bounds__(kFactWarps * 32)
    fact_stage_a_kernel(DevOperator op, const double* __restrict__ x, const PcgScalars* guard, PcgScalars* sc,
                        double* pbuf0, double* pbuf1) {
  extern __shared__ __align__(128) unsigned char fsm_raw[];
  constexpr int NT = kFactWarps * 32;
  const int n = op.n_loc, kp = op.kp, XS = apply_x_stride(kp), nfp = op.nfp;
  constexpr int MB = BM / 8;  // 8-row DMMA blocks per warp tile
  const FactSmem L = fact_a_layout(kp, BM);
  double* X = reinterpret_cast<double*>(fsm_raw + L.x);
  int32_t* EB = reinterpret_cast<int32_t*>(fsm_raw + L.eb);
  uint16_t* LUT = reinterpret_cast<uint16_t*>(fsm_raw + L.lut);
  uint16_t* OWN = reinterpret_cast<uint16_t*>(fsm_raw + L.own);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, t4 = lane & 3;
  // gridDim.y column splits per cell tile (op.fact_nsa): split sp takes the 32-column blocks
  // sp, sp + ns, ... of U; every split gathers the tile, split 0 writes the direction
  const int ns = gridDim.y, sp = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * BM;
  const int nc = (int)min((int64_t)BM, op.n_cells - c0);
  for (int i = tid; i < kp; i += NT) LUT[i] = i < n ? op.lut[i] : 0;
  for (int e = tid; e < BM * 16; e += NT) EB[e] = (e >> 4) < nc ? op.ebase[c0 * 16 + e] : -1;
  for (int e = tid; e < BM; e += NT) OWN[e] = e < nc ? op.own[c0 + e] : 0;
  pdl_wait();
  if (stopped(guard)) return;
  double beta = 0.0;
  int kit = 0;
  const double* p_old = nullptr;
  double* p_new = nullptr;
  if (PCG) {
    __shared__ double s_beta;
    __shared__ int s_kit;
    if (tid == 0) {
      volatile PcgScalars* v = sc;
      s_kit = v->k;
      const double rz_old = v->rz_old;
      s_beta = (s_kit == 0 || rz_old == 0.0) ? 0.0 : v->rz_acc / rz_old;
    }
    __syncthreads();
    kit = s_kit;
    beta = s_beta;
    p_old = (kit & 1) ? pbuf0 : pbuf1;
    p_new = (kit & 1) ? pbuf1 : pbuf0;
  } else {
    __syncthreads();
  }
  // ---- gather the tile (PCG mode: p_k = z_k + beta p_{k-1}, the owner cell writes it, ||z||^2;
  // a version issuing 8 elements' loads before any store measured slower:
  // profiles/round2/experiments/fact_apply_batched_gather_ab.jsonl)
  double zz = 0.0;
  const int total = BM * XS;
  for (int e = tid; e < total; e += NT) {
    const int c = e / XS, j = e - c * XS;
    double v = 0.0;
    if (j < n) {
      const int l = LUT[j];
      const int b = EB[c * 16 + (l >> kLutShift)];
      if (b >= 0) {
        const int g = b + (l & ((1 << kLutShift) - 1));
        const double xv = x[g];
        v = xv;
        if (PCG) {
          v = fma(beta, p_old[g], xv);
          if (sp == 0 && ((OWN[c] >> (l >> kLutShift)) & 1)) {
            p_new[g] = v;
            zz = fma(xv, xv, zz);
          }
        }
      }
    }
    X[e] = v;
  }
  __syncthreads();
  // ---- stage A: U = X F, warp = 32-column block, BM cells
  const double* xr = X + g8 * XS + t4;
  const int nblk = nfp / 32;
  for (int blk = sp + ns * warp; blk < nblk; blk += ns * kFactWarps) {
    double acc[MB][kFactNQ][2];
#pragma unroll
    for (int m = 0; m < MB; ++m)
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
    const double* fb = op.F + (size_t)t4 * nfp + blk * 32 + g8;
#pragma unroll 4
    for (int k0 = 0; k0 < kp; k0 += 4) {
      double a[MB];
#pragma unroll
      for (int m = 0; m < MB; ++m) a[m] = xr[m * 8 * XS + k0];
      const double* fr = fb + (size_t)k0 * nfp;
      double b[kFactNQ];
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q) b[q] = __ldg(fr + q * 8);
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q)
#pragma unroll
        for (int m = 0; m < MB; ++m) dmma884(acc[m][q][0], acc[m][q][1], a[m], b[q]);
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const int row = m * 8 + g8;
      if (row < nc) {
        double* ur = op.ubuf + (size_t)(c0 + row) * nfp + blk * 32 + 2 * t4;
#pragma unroll
        for (int q = 0; q < kFactNQ; ++q) *reinterpret_cast<double2*>(ur + q * 8) = make_double2(acc[m][q][0], acc[m][q][1]);
      }
    }
  }
  if (pdl_late()) pdl_trigger();
  if (PCG) {  // ||z||^2, then the stopping test in the last CTA (as apply_tc_kernel's PCG mode)
    __shared__ double sh[32];
    __shared__ bool last;
    const double szz = block_sum(zz, sh);
    if (tid == 0) {
      atomicAdd(&sc->zz, szz);
      __threadfence();
      last = atomicAdd(&sc->ticket, 1u) == gridDim.x * gridDim.y - 1;
    }
    __syncthreads();
    if (last && tid == 0) {
      __threadfence();
      volatile PcgScalars* v = sc;
      const double zn = sqrt(v->zz);
      if (kit == 0) {
        sc->z0 = zn;
        sc->z_last = zn;
        sc->iters = 0;
        if (zn == 0.0) {
          sc->done = 1;
          sc->converged = 1;
        } else if (v->maxit <= 0) {
          sc->done = 1;
        }
      } else {
        sc->iters = kit;
        sc->z_last = zn;
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
  }
}

// stage B: V = mix(U) with the cells' 3 x 3 coefficient matrices (value block: coef 0..5 =
// Gm_00, Gm_11, Gm_22, Gm_01, Gm_02, Gm_12; curl block: coef 6..11 likewise), p.Ap =
// sum over the tile of u.v (PCG mode: into pq2 of the iteration stage A just ran), then
// Y = V F^T and the scatter-add.
template <int BM, bool PCG>
__global__ void __launch_bounds__(kFactWarps * 32)
    fact_stage_b_kernel(DevOperator op, double* __restrict__ y, double* pq_acc, const PcgScalars* guard,
                        PcgScalars* sc) {
  extern __shared__ __align__(128) unsigned char fsm_raw[];
  constexpr int NT = kFactWarps * 32;
  const int n = op.n_loc, kp = op.kp, nfp = op.nfp, VS = (int)fact_vs(nfp);
  constexpr int MB = BM / 8;
  const FactSmem L = fact_b_layout(kp, nfp, BM);
  double* V = reinterpret_cast<double*>(fsm_raw + L.x);
  int32_t* EB = reinterpret_cast<int32_t*>(fsm_raw + L.eb);
  uint16_t* LUT = reinterpret_cast<uint16_t*>(fsm_raw + L.lut);
  double* C = reinterpret_cast<double*>(fsm_raw + L.own);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g8 = lane >> 2, t4 = lane & 3;
  // gridDim.y column splits per cell tile (op.fact_nsb): split sp takes the 32-column blocks
  // sp, sp + ns, ... of Y; every split loads and mixes the U tile, split 0 accumulates p.Ap
  const int ns = gridDim.y, sp = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * BM;
  const int nc = (int)min((int64_t)BM, op.n_cells - c0);
  for (int i = tid; i < kp; i += NT) LUT[i] = i < n ? op.lut[i] : 0;
  for (int e = tid; e < BM * 16; e += NT) EB[e] = (e >> 4) < nc ? op.ebase[c0 * 16 + e] : -1;
  const int nm = op.n_mat;
  for (int e = tid; e < BM * nm; e += NT) C[e] = e / nm < nc ? op.coef[c0 * nm + e] : 0.0;
  pdl_wait();
  if (stopped(guard)) return;
  for (int e = tid; e < BM * (nfp / 2); e += NT) {  // U tile -> smem (16-byte loads)
    const int c = e / (nfp / 2), j = 2 * (e - c * (nfp / 2));
    const double2 u = c < nc ? *reinterpret_cast<const double2*>(op.ubuf + (size_t)(c0 + c) * nfp + j)
                             : make_double2(0.0, 0.0);
    V[c * VS + j] = u.x;
    V[c * VS + j + 1] = u.y;
  }
  __syncthreads();
  double pq = 0.0;
  const int npm = op.nfm / 3, npk = (op.nf - op.nfm) / op.fck;
  for (int e = tid; e < BM * (npm + npk); e += NT) {
    const int c = e / (npm + npk), k = e - c * (npm + npk);
    const bool val = k < npm;
    const int np3 = val ? npm : npk, off = val ? k : op.nfm + (k - npm);
    const double* g = C + c * nm + (val ? 0 : 6);
    double* vr = V + c * VS + off;
    if (!val && op.fck == 1) {  // H(div): the div-div block is scalar, coefficient alpha / |det J|
      const double u = vr[0], v = g[0] * u;
      vr[0] = v;
      pq = fma(u, v, pq);
      continue;
    }
    const double u0 = vr[0], u1 = vr[np3], u2 = vr[2 * np3];
    const double v0 = g[0] * u0 + g[3] * u1 + g[4] * u2;
    const double v1 = g[3] * u0 + g[1] * u1 + g[5] * u2;
    const double v2 = g[4] * u0 + g[5] * u1 + g[2] * u2;
    vr[0] = v0;
    vr[np3] = v1;
    vr[2 * np3] = v2;
    pq = fma(u0, v0, fma(u1, v1, fma(u2, v2, pq)));
  }
  __syncthreads();
  if (sp != 0) pq = 0.0;
  // ---- stage B: Y = V F^T, warp = 32 output columns, BM cells
  const double* vrow = V + g8 * VS + t4;
  const int nblk = (kp + 31) / 32;
  for (int blk = sp + ns * warp; blk < nblk; blk += ns * kFactWarps) {
    double acc[MB][kFactNQ][2];
#pragma unroll
    for (int m = 0; m < MB; ++m)
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;
    int colr[kFactNQ];  // F row of this lane's B fragment column (clamped: rows >= kp read as zero)
#pragma unroll
    for (int q = 0; q < kFactNQ; ++q) colr[q] = min(blk * 32 + q * 8 + g8, kp - 1);
    bool colok[kFactNQ];
#pragma unroll
    for (int q = 0; q < kFactNQ; ++q) colok[q] = blk * 32 + q * 8 + g8 < kp;
#pragma unroll 4
    for (int k0 = 0; k0 < op.nf; k0 += 4) {
      double a[MB];
#pragma unroll
      for (int m = 0; m < MB; ++m) a[m] = vrow[m * 8 * VS + k0];
      double b[kFactNQ];
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q) b[q] = colok[q] ? __ldg(op.F + (size_t)colr[q] * nfp + k0 + t4) : 0.0;
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q)
#pragma unroll
        for (int m = 0; m < MB; ++m) dmma884(acc[m][q][0], acc[m][q][1], a[m], b[q]);
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const int row = m * 8 + g8;
#pragma unroll
      for (int q = 0; q < kFactNQ; ++q)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int col = blk * 32 + q * 8 + 2 * t4 + i;
          if (row < nc && col < n) {
            const int l = LUT[col];
            const int b = EB[row * 16 + (l >> kLutShift)];
            if (b >= 0) atomicAdd(y + b + (l & ((1 << kLutShift) - 1)), acc[m][q][i]);
          }
        }
    }
  }
  if (pdl_late()) pdl_trigger();
  __shared__ double sh[32];
  const double spq = block_sum(pq, sh);
  if (tid == 0) {
    if (PCG) {
      const int kit = ((volatile PcgScalars*)sc)->k - 1;  // stage A of this iteration advanced k
      atomicAdd(&sc->pq2[kit & 1], spq);
    } else if (pq_acc) {
      atomicAdd(pq_acc, spq);
    }
  }
}

template <int BMA, int BMB, bool PCG>
cudaError_t launch_fact_apply_bm(const DevOperator& op, const double* x, double* y, double* pq_acc,
                                 const PcgScalars* guard, PcgScalars* sc, double* p0, double* p1, cudaStream_t s) {
  const dim3 block(kFactWarps * 32);
  const unsigned nsa = (unsigned)std::max(1, op.fact_nsa), nsb = (unsigned)std::max(1, op.fact_nsb);
  cudaError_t e = launch_k(fact_stage_a_kernel<BMA, PCG>, dim3((unsigned)((op.n_cells + BMA - 1) / BMA), nsa), block,
                           fact_a_layout(op.kp, BMA).total, s, op, x, guard, sc, p0, p1);
  if (e != cudaSuccess) return e;
  return launch_k(fact_stage_b_kernel<BMB, PCG>, dim3((unsigned)((op.n_cells + BMB - 1) / BMB), nsb), block,
                  fact_b_layout(op.kp, op.nfp, BMB).total, s, op, y, pq_acc, guard, sc);
}
template <bool PCG>
cudaError_t launch_fact_apply(const DevOperator& op, const double* x, double* y, double* pq_acc,
                              const PcgScalars* guard, PcgScalars* sc, double* p0, double* p1, cudaStream_t s) {
  switch (op.fact) {
    case 1: return launch_fact_apply_bm<16, 16, PCG>(op, x, y, pq_acc, guard, sc, p0, p1, s);
    case 2: return launch_fact_apply_bm<32, 32, PCG>(op, x, y, pq_acc, guard, sc, p0, p1, s);
    default: return launch_fact_apply_bm<32, 24, PCG>(op, x, y, pq_acc, guard, sc, p0, p1, s);
  }
}

constexpr size_t kMaxSmem = 226 * 1024;  // 227 KB opt-in minus the static reduction scratch

// The warp layouts built (BM, NQ, KS), each for NM = 7, NM0 = 7 (H(grad)), NM = 12,
// NM0 = 6 (H(curl)) and NM = 7, NM0 = 6 (H(div)). The ring depth is sized per operator
// (apply_configure_variant).
struct ApplyVariant {
  int bm, nq, ks, nm, nm0;
  const void* fn[2];  // plain, PCG
};
template <int BM, int NQ, int KS, int NM, int MINB = 1, int NM0 = (NM == 12 ? 6 : NM)>
ApplyVariant apply_variant() {
  return {BM, NQ, KS, NM, NM0,
          {(const void*)apply_tc_kernel<BM, NQ, KS, NM, NM0, MINB, false>,
           (const void*)apply_tc_kernel<BM, NQ, KS, NM, NM0, MINB, true>}};
}
const ApplyVariant* apply_variants(int* count) {
  static const ApplyVariant v[] = {
      apply_variant<32, 4, 2, 7>(),  apply_variant<32, 4, 2, 12>(),   // 4 MMA warps
      apply_variant<32, 4, 4, 7>(),  apply_variant<32, 4, 4, 12>(),   // 8 MMA warps
      apply_variant<32, 2, 2, 7>(),  apply_variant<32, 2, 2, 12>(),   // 8 MMA warps, 16 x 16 warp tiles
      apply_variant<16, 4, 4, 7>(),  apply_variant<16, 4, 4, 12>(),   // 4 MMA warps, 16 cells per unit
      apply_variant<32, 4, 4, 7, 2>(), apply_variant<32, 4, 4, 12, 2>(),  // 8 MMA warps, registers for 2 CTAs/SM
      apply_variant<16, 2, 4, 7>(),  apply_variant<16, 2, 4, 12>(),   // 8 MMA warps, 16 cells (large n_loc)
      // the same six layouts for H(div) (the div-div matrix skipped beyond ncb)
      apply_variant<32, 4, 2, 7, 1, 6>(), apply_variant<32, 4, 4, 7, 1, 6>(), apply_variant<32, 2, 2, 7, 1, 6>(),
      apply_variant<16, 4, 4, 7, 1, 6>(), apply_variant<32, 4, 4, 7, 2, 6>(), apply_variant<16, 2, 4, 7, 1, 6>(),
  };
  *count = (int)(sizeof(v) / sizeof(v[0]));
  return v;
}

size_t apply_variant_smem(const ApplyVariant& v, const DevOperator& op) {
  return apply_smem_layout(v.bm, v.nq, v.ks, op.apply_slots, op.kp, op.n_mat).total;
}

inline int apply_threads(const ApplyVariant& v) { return (apply_mma_warps(v.bm, v.nq, v.ks) + 1) * 32; }

template <bool PCG>
cudaError_t launch_apply_tc(const DevOperator& op, const double* x, double* y, double* pq_acc,
                            const PcgScalars* guard, cudaStream_t s, PcgScalars* sc = nullptr,
                            double* p0 = nullptr, double* p1 = nullptr) {
  int cnt = 0;
  const ApplyVariant& v = apply_variants(&cnt)[op.av];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)op.apply_grid);
  cfg.blockDim = dim3(apply_threads(v));
  cfg.dynamicSmemBytes = apply_variant_smem(v, op);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  int S = op.apply_slots;
  DevOperator o = op;
  void* args[] = {(void*)&o, (void*)&S, (void*)&x, (void*)&y, (void*)&pq_acc, (void*)&guard, (void*)&sc, (void*)&p0,
                  (void*)&p1};
  return cudaLaunchKernelExC(&cfg, v.fn[PCG ? 1 : 0], args);
}

// ---------------------------------------------------------------- preconditioner
__global__ void precond_init_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ z,
                                    double* rz_acc, const PcgScalars* guard) {
  pdl_wait();
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
  if (rz_acc) {
    __shared__ double sh[32];
    double s = block_sum(part, sh);
    if (threadIdx.x == 0) atomicAdd(rz_acc, s);
  }
}


// Star-patch kernel (Eq. 5.4 P:1763-1774 / Eq. 5.12 P:1956-1970 with exact
// local solvers, R-A15): z += E_m A_m^{-1} E_m^T r. One CTA per patch, patches in decreasing size
// order, so the hardware block scheduler hands out the work longest-first.
// Full tiles are stored row-major in 32-byte groups ((i,k) at
// ((k>>2)*rows + i)*4 + (k&3)): a warp owns a tile and reads it in two
// 16-column halves with coalesced 32-byte non-allocating loads, lane = row.
// Half-tiles keep the kernel at <= 64 registers, i.e. 4 CTAs = 32 warps per
// SM streaming. Row products (-> z_I) are dot products with r_J; transposed
// products (-> z_J) are a 16-value transpose reduction across the warp.
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

// H(curl) potential patches (kind 1, Eq. 5.12): the patch's dofs are
// CG_p interface dofs c embedded by the discrete gradient G (R-A12), so the
// patch residual is (G^T r)_c = sum_k G[k][c] r_k and the correction is
// scattered as z_k += G[k][c] u_c, both straight from the CSR rows of G^T
// (one entry per CG edge / face dof, the incident Whitney edges per vertex).
__device__ __forceinline__ double patch_residual(const DevPrecond& pc, bool pot, const double* __restrict__ r,
                                                 int g) {
  if (g < 0) return 0.0;
  if (!pot) return r[g];
  double s = 0.0;
  for (int64_t k = pc.g_ptr[g]; k < pc.g_ptr[g + 1]; ++k) s = fma(pc.g_val[k], r[pc.g_col[k]], s);
  return s;
}
__device__ __forceinline__ void patch_scatter(const DevPrecond& pc, bool pot, double* __restrict__ z, int g,
                                              double u) {
  if (!pot) {
    atomicAdd(z + g, u);
    return;
  }
  for (int64_t k = pc.g_ptr[g]; k < pc.g_ptr[g + 1]; ++k) atomicAdd(z + pc.g_col[k], pc.g_val[k] * u);
}

// v[k] over 32 lanes -> lane l holds sum_{lanes} v[l & 15] (16-value transpose reduction)
constexpr int kSmallPatch = 128;  // patches of at most this size take the warp-per-patch path

template <int S>
__device__ __forceinline__ void treduce_stage(double (&v)[16], int lane) {
  const bool upper = (lane & S) != 0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const double send = upper ? v[k] : v[k + S];
    const double keep = upper ? v[k + S] : v[k];
    v[k] = keep + __shfl_xor_sync(0xffffffffu, send, S);
  }
}
__device__ __forceinline__ double treduce16(double (&v)[16], int lane) {
  __syncwarp();  // converged: plain SHFL (not the WARPSYNC.COLLECTIVE sequence ptxas emits otherwise)
  treduce_stage<8>(v, lane);
  treduce_stage<4>(v, lane);
  treduce_stage<2>(v, lane);
  treduce_stage<1>(v, lane);
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}
// The same reduction for a half tile held in lane-permuted order: position
// 4 g' + j holds column 4 (g' ^ G) + j, G = (lane >> 2) & 3 (patch_ldg_kernel
// loads its four 4-column groups in that order). Then at the 8- and
// 4-exchanges every lane keeps its low positions and sends its high ones --
// the partner (lane ^ 8, lane ^ 4) holds the matching columns there -- so 12 of
// the 15 exchanges need no select (the stage-8 and stage-4 selects were most of
// the kernel's instructions); lane l ends with column l & 15 as before.
__device__ __forceinline__ double treduce16p(double (&v)[16], int lane) {
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k + 8], 8);
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k + 4], 4);
  treduce_stage<2>(v, lane);
  treduce_stage<1>(v, lane);
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// One star patch solved by one warp (the lane = row half-tile stream of
// patch_ldg_kernel without block barriers): z += E_m A_m^-1 E_m^T r for patch
// pid, rl / zl = npad doubles of warp-private shared memory each. `ready()` is
// called once the first half tile is in flight and before r is read (the PDL
// wait of a kernel launched behind the producer of r); it returns false to
// abandon the patch. Returns this lane's share of r.z (0 if abandoned).
template <class Ready>
__device__ __forceinline__ double warp_patch_solve(const DevPrecond& pc, int64_t pid, const double* __restrict__ r,
                                                   double* __restrict__ z, double* rl, double* zl, int lane,
                                                   Ready ready) {
  const int n = pc.pn[pid];
  const int nb = (n + 31) >> 5, npad = nb * 32;
  const bool pot = pc.pkind[pid] != 0;
  const int32_t* id = pc.idx + pc.idx_off[pid];
  long long* rli = reinterpret_cast<long long*>(rl);
  for (int i = lane; i < npad; i += 32) {
    rli[i] = id[i];
    zl[i] = 0.0;
  }
  const double* T = pc.tiles + pc.tile_off[pid];
  const int ntiles = nb * (nb + 1) / 2;
  int I = 0, J = 0, h = 0, t = 0;
  auto load_half = [&](double(&a)[16]) {
    const int rows = min(32, n - 32 * I);
    const double* tb = T + 512LL * I * I + 16LL * I + (int64_t)J * 32 * rows;
    if (J < I) {
      if (lane < rows) {
        const double4* tp = reinterpret_cast<const double4*>(tb) + lane + 4 * h * rows;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const double4 v = ld_stream4(tp + k4 * rows);
          a[4 * k4] = v.x;
          a[4 * k4 + 1] = v.y;
          a[4 * k4 + 2] = v.z;
          a[4 * k4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = 0.0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = 16 * h + q;
        a[q] = (k <= lane && lane < rows) ? ld_stream1(tb + k * rows - k * (k - 1) / 2 + (lane - k)) : 0.0;
      }
    }
  };
  double a[16];
  load_half(a);
  if (!ready()) return 0.0;
  for (int i = lane; i < npad; i += 32) rl[i] = patch_residual(pc, pot, r, (int)rli[i]);
  __syncwarp();
  double row = 0.0;
  while (t < ntiles) {
    const double ri = rl[I * 32 + lane];
    if (J < I) {
      const double* rJ = rl + J * 32 + 16 * h;
#pragma unroll
      for (int q = 0; q < 16; ++q) row = fma(a[q], rJ[q], row);
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] *= ri;
    } else {
      const double* rI = rl + I * 32 + 16 * h;
#pragma unroll
      for (int q = 0; q < 16; ++q) row = fma(a[q], rI[q], row);
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] = (16 * h + q < lane) ? a[q] * ri : 0.0;  // strict lower, transposed
    }
    const double col = treduce16(a, lane);
    if (lane < 16) atomicAdd(zl + J * 32 + 16 * h + lane, col);
    if (h == 1) {
      atomicAdd(zl + I * 32 + lane, row);
      row = 0.0;
      h = 0;
      ++t;
      if (++J > I) {
        J = 0;
        ++I;
      }
    } else {
      h = 1;
    }
    if (t < ntiles) load_half(a);
  }
  __syncwarp();
  double part = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double zi = zl[i];
    patch_scatter(pc, pot, z, id[i], pc.out_scale * zi);
    part = fma(rl[i], zi, part);
  }
  __syncwarp();  // rl / zl may be reused by the warp's next patch
  return part;
}

// Small patches (n <= 128, at most 4 block rows: the H(div) and H(curl) edge
// stars, sorted last, [n_big, n_patches)) one per warp, kLdgWarps per CTA, so
// a small patch's gather / scatter / reduction latency overlaps the other
// warps' tile streams instead of serialising on __syncthreads.
template <int kLdgWarps>
__global__ void __launch_bounds__(kLdgWarps * 32, 32 / kLdgWarps)
    patch_warp_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ z, double* rz_acc,
                      const PcgScalars* guard) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t pid = pc.n_big + (int64_t)blockIdx.x * kLdgWarps + warp;
  if (pid >= pc.n_patches) {
    pdl_wait();  // warps without a patch still order the CTA after the previous kernel
    return;
  }
  double* rl = smem + warp * 2 * kSmallPatch;
  double* zl = rl + kSmallPatch;
  bool live = true;
  double part = warp_patch_solve(pc, pid, r, z, rl, zl, lane, [&] {
    pdl_wait();
    live = !stopped(guard);
    return live;
  });
  if (!live) return;
  if (pdl_late()) pdl_trigger();
  part = warp_sum(part);
  if (rz_acc && lane == 0) atomicAdd(rz_acc, part);
}

// Small patches (every patch <= 128 dofs, as the H(div) edge stars), persistent
// form: a grid of resident CTAs whose warps each walk a strided sequence of
// patches (pid = gw, gw + GW, ...). After a patch's last tile, the warp issues
// the next patch's dof ids and first half tile, then scatters the finished
// patch (its atomics and shared-memory reads overlap those loads), then
// gathers the next r: the per-patch latency chain of patch_warp_kernel
// (ids -> first tile, ids -> r, the scatter) is half hidden. Shared memory:
// two (r, z) buffer pairs per warp.
struct SmallPatch {
  int64_t pid;
  int n, nb, ntiles;
  bool pot;
  const double* T;
  const int32_t* id;
};

template <int kLdgWarps>
__global__ void __launch_bounds__(kLdgWarps * 32, 24 / kLdgWarps)
    patch_warp_loop_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ z, double* rz_acc,
                           const PcgScalars* guard) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kLdgWarps + warp, GW = (int64_t)gridDim.x * kLdgWarps;
  double* wbuf = smem + (size_t)warp * 4 * kSmallPatch;  // [2 buffers][r, z][128]
  auto meta = [&](int64_t pid) {
    SmallPatch m;
    m.pid = pid;
    m.n = pc.pn[pid];
    m.nb = (m.n + 31) >> 5;
    m.ntiles = m.nb * (m.nb + 1) / 2;
    m.pot = pc.pkind[pid] != 0;
    m.T = pc.tiles + pc.tile_off[pid];
    m.id = pc.idx + pc.idx_off[pid];
    return m;
  };
  auto load_half = [&](double(&a)[16], const SmallPatch& m, int I, int J, int h) {
    const int rows = min(32, m.n - 32 * I);
    const double* tb = m.T + 512LL * I * I + 16LL * I + (int64_t)J * 32 * rows;
    if (J < I) {
      if (lane < rows) {
        const double4* tp = reinterpret_cast<const double4*>(tb) + lane + 4 * h * rows;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const double4 v = ld_stream4(tp + k4 * rows);
          a[4 * k4] = v.x;
          a[4 * k4 + 1] = v.y;
          a[4 * k4 + 2] = v.z;
          a[4 * k4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = 0.0;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int k = 16 * h + q;
        a[q] = (k <= lane && lane < rows) ? ld_stream1(tb + k * rows - k * (k - 1) / 2 + (lane - k)) : 0.0;
      }
    }
  };
  int64_t pid = pc.n_big + gw;
  if (pid >= pc.n_patches) {
    pdl_wait();
    return;
  }
  SmallPatch m = meta(pid);
  int buf = 0;
  int ids[4];  // this lane's dof ids of the patch (npad <= 128)
#pragma unroll
  for (int q = 0; q < 4; ++q) ids[q] = 32 * q + lane < m.nb * 32 ? m.id[32 * q + lane] : -1;
  double a[16];
  load_half(a, m, 0, 0, 0);
  pdl_wait();
  if (stopped(guard)) return;
  double part = 0.0;
  for (;;) {
    double* rl = wbuf + buf * 2 * kSmallPatch;
    double* zl = rl + kSmallPatch;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (32 * q < m.nb * 32) {
        rl[32 * q + lane] = patch_residual(pc, m.pot, r, ids[q]);
        zl[32 * q + lane] = 0.0;
      }
    __syncwarp();
    // the patch's tiles (lane = row, half tiles), as patch_warp_kernel
    int I = 0, J = 0, h = 0, t = 0;
    double row = 0.0;
    while (t < m.ntiles) {
      const double ri = rl[I * 32 + lane];
      if (J < I) {
        const double* rJ = rl + J * 32 + 16 * h;
#pragma unroll
        for (int q = 0; q < 16; ++q) row = fma(a[q], rJ[q], row);
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] *= ri;
      } else {
        const double* rI = rl + I * 32 + 16 * h;
#pragma unroll
        for (int q = 0; q < 16; ++q) row = fma(a[q], rI[q], row);
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = (16 * h + q < lane) ? a[q] * ri : 0.0;
      }
      const double col = treduce16(a, lane);
      if (lane < 16) atomicAdd(zl + J * 32 + 16 * h + lane, col);
      if (h == 1) {
        atomicAdd(zl + I * 32 + lane, row);
        row = 0.0;
        h = 0;
        ++t;
        if (++J > I) {
          J = 0;
          ++I;
        }
      } else {
        h = 1;
      }
      if (t < m.ntiles) load_half(a, m, I, J, h);
    }
    // the next patch's ids and first half tile are issued before this one is scattered
    const int64_t next = pid + GW;
    const bool more = next < pc.n_patches;
    SmallPatch mn = m;
    int nids[4];
    if (more) {
      mn = meta(next);
#pragma unroll
      for (int q = 0; q < 4; ++q) nids[q] = 32 * q + lane < mn.nb * 32 ? mn.id[32 * q + lane] : -1;
      load_half(a, mn, 0, 0, 0);
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = 32 * q + lane;
      if (i < m.n) {
        const double zi = zl[i];
        patch_scatter(pc, m.pot, z, ids[q], pc.out_scale * zi);
        part = fma(rl[i], zi, part);
      }
    }
    if (!more) break;
    pid = next;
    m = mn;
#pragma unroll
    for (int q = 0; q < 4; ++q) ids[q] = nids[q];
    buf ^= 1;
  }
  if (pdl_late()) pdl_trigger();
  part = warp_sum(part);
  if (rz_acc && lane == 0) atomicAdd(rz_acc, part);
}

template <int kLdgWarps>
__global__ void __launch_bounds__(kLdgWarps * 32, 32 / kLdgWarps)
    patch_ldg_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ z, double* rz_acc,
                     const PcgScalars* guard) {
  extern __shared__ double smem[];
  const int pid = blockIdx.x;
  const int n = pc.pn[pid];
  const int nb = (n + 31) >> 5, npad = nb * 32;
  const bool pot = pc.pkind[pid] != 0;
  double* rl = smem;
  double* zl = smem + npad;
  const int32_t* id = pc.idx + pc.idx_off[pid];
  // prologue on constant data (overlaps the previous kernel under PDL): the
  // patch's dof ids go into the r slots, replaced by r in place after the wait
  long long* rli = reinterpret_cast<long long*>(rl);
  for (int i = threadIdx.x; i < npad; i += blockDim.x) {
    rli[i] = id[i];
    zl[i] = 0.0;
  }
  const double* T = pc.tiles + pc.tile_off[pid];
  const int ntiles = nb * (nb + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G4 = ((lane >> 2) & 3) << 2;  // lane-permuted column order (treduce16p)
  int I = 0, J = warp, h = 0, t = warp;
  while (J > I) {
    J -= I + 1;
    ++I;
  }
  // half tile (I, J, h) -> a[16] (row `lane`; diagonal tiles: lower triangle only), position
  // q holding column 16 h + (q ^ G4)
  auto load_half = [&](double(&a)[16]) {
    const int rows = min(32, n - 32 * I);
    const double* tb = T + 512LL * I * I + 16LL * I + (int64_t)J * 32 * rows;
    if (J < I) {
      if (lane < rows) {
        const double4* tp = reinterpret_cast<const double4*>(tb) + lane + 4 * h * rows;
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const double4 v = ld_stream4(tp + (k4 ^ (G4 >> 2)) * rows);
          a[4 * k4] = v.x;
          a[4 * k4 + 1] = v.y;
          a[4 * k4 + 2] = v.z;
          a[4 * k4 + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = 0.0;
      }
    } else {
      // diagonal tile, lower triangle packed by columns: (i,k), k <= i at k*rows - k(k-1)/2 + i - k
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int c0 = 16 * h + ((4 * g) ^ G4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int k = c0 + j;
          a[4 * g + j] = (k <= lane && lane < rows) ? ld_stream1(tb + k * rows - k * (k - 1) / 2 + (lane - k)) : 0.0;
        }
      }
    }
  };
  double a[16];
  if (t < ntiles) load_half(a);  // the first half tile is in flight during the r gather
  pdl_wait();
  if (stopped(guard)) return;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) rl[i] = patch_residual(pc, pot, r, (int)rli[i]);
  __syncthreads();
  double row = 0.0;
  while (t < ntiles) {
    const double ri = rl[I * 32 + lane];
    if (J < I) {
      const double* rJ = rl + J * 32 + 16 * h;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const double* rg = rJ + ((4 * g) ^ G4);  // the group's columns (4-aligned: ^ == +)
#pragma unroll
        for (int j = 0; j < 4; ++j) row = fma(a[4 * g + j], rg[j], row);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) a[q] *= ri;
    } else {
      const double* rI = rl + I * 32 + 16 * h;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int c0 = (4 * g) ^ G4;
        const double* rg = rI + c0;
#pragma unroll
        for (int j = 0; j < 4; ++j) row = fma(a[4 * g + j], rg[j], row);
#pragma unroll
        for (int j = 0; j < 4; ++j)  // strict lower, transposed
          a[4 * g + j] = (16 * h + c0 + j < lane) ? a[4 * g + j] * ri : 0.0;
      }
    }
    const double col = treduce16p(a, lane);
    if (lane < 16) atomicAdd(zl + J * 32 + 16 * h + lane, col);
    if (h == 1) {  // tile done: this warp's next tile; row products flushed when the block row changes
      h = 0;
      t += kLdgWarps;
      J += kLdgWarps;
      const int I0 = I;
      while (J > I) {
        J -= I + 1;
        ++I;
      }
      if (I != I0 || t >= ntiles) {
        atomicAdd(zl + I0 * 32 + lane, row);
        row = 0.0;
      }
    } else {
      h = 1;
    }
    if (t < ntiles) load_half(a);
  }
  if (pdl_late()) pdl_trigger();
  __syncthreads();
  double part = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = zl[i];
    patch_scatter(pc, pot, z, id[i], pc.out_scale * zi);
    part = fma(rl[i], zi, part);
  }
  if (rz_acc) {
    __shared__ double sh[32];
    const double s = block_sum(part, sh);
    if (threadIdx.x == 0) atomicAdd(rz_acc, s);
  }
}

// ---------------------------------------------------------------- hybrid Schwarz
// Symmetric multiplicative sweep J, P, C, P, J: helpers.
// e = s * dinv .* r on the interior dofs (set: e = 0 elsewhere and the sweep's
// A e accumulator hy = 0; add: e += ...). Every sweep kernel returns at once
// once the PCG has stopped (guard), like the patch and apply kernels.
__global__ void hyb_jacobi_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ e, double s,
                                  int add, const PcgScalars* guard) {
  pdl_wait();
  if (stopped(guard)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_total; i += stride) {
    const double v = i >= pc.off3 ? s * pc.dinv[i - pc.off3] * r[i] : 0.0;
    e[i] = add ? e[i] + v : v;
    if (!add) pc.hy[i] = 0.0;
  }
}

// t = r - y (y = A e, constrained rows already 0), then y = 0 for the next
// stage's apply; also clears the coarse accumulators
__global__ void hyb_residual_kernel(DevPrecond pc, const double* __restrict__ r, double* __restrict__ y,
                                    double* __restrict__ t, const PcgScalars* guard) {
  pdl_wait();
  if (stopped(guard)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.n_total; i += stride) {
    t[i] = r[i] - y[i];
    y[i] = 0.0;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pc.nc; i += stride) pc.czc[i] = 0.0;
}

// coarse solve e += E_c A_c^-1 E_c^T t: the stored packed inverse of the
// Whitney-space matrix (setup.hpp tile layout "groups", one n_c x n_c patch),
// tiles spread over the whole grid (one warp per tile, half tiles as in
// patch_ldg_kernel), row and transposed products accumulated into czc with
// red.global.add; the coarse residual is read through cidx.
__global__ void __launch_bounds__(256) coarse_symv_kernel(DevPrecond pc, const double* __restrict__ t,
                                                           const PcgScalars* guard) {
  pdl_wait();
  if (stopped(guard)) return;
  const int n = (int)pc.nc, nb = (n + 31) >> 5;
  const int64_t ntiles = (int64_t)nb * (nb + 1) / 2;
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tt = gw; tt < ntiles; tt += nw) {
    // (I, J) of tile tt in order I(I+1)/2 + J
    int I = (int)((sqrt(8.0 * (double)tt + 1.0) - 1.0) * 0.5);
    while ((int64_t)(I + 1) * (I + 2) / 2 <= tt) ++I;
    while ((int64_t)I * (I + 1) / 2 > tt) --I;
    const int J = (int)(tt - (int64_t)I * (I + 1) / 2);
    const int rows = min(32, n - 32 * I);
    const double* tb = pc.ctiles + 512LL * I * I + 16LL * I + (int64_t)J * 32 * rows;
    const int gi = 32 * I + lane;
    const double ri = (lane < rows) ? t[pc.cidx[gi]] : 0.0;
    double row = 0.0;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      double a[16];
      const int gj0 = 32 * J + 16 * h;
      if (J < I) {
        if (lane < rows) {
          const double4* tp = reinterpret_cast<const double4*>(tb) + lane + 4 * h * rows;
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4) {
            const double4 v = ld_stream4(tp + k4 * rows);
            a[4 * k4] = v.x;
            a[4 * k4 + 1] = v.y;
            a[4 * k4 + 2] = v.z;
            a[4 * k4 + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) a[q] = 0.0;
        }
        // r_J from the broadcast of lane-held values: lane q holds t at column gj0 + q
        const double rjl = (gj0 + (lane & 15) < n) ? t[pc.cidx[gj0 + (lane & 15)]] : 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) row = fma(a[q], __shfl_sync(0xffffffffu, rjl, q), row);
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] *= ri;
      } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int k = 16 * h + q;
          a[q] = (k <= lane && lane < rows) ? ld_stream1(tb + k * rows - k * (k - 1) / 2 + (lane - k)) : 0.0;
        }
        const double ril = __shfl_sync(0xffffffffu, ri, (16 * h + (lane & 15)) & 31);
#pragma unroll
        for (int q = 0; q < 16; ++q) row = fma(a[q], __shfl_sync(0xffffffffu, ril, q), row);
#pragma unroll
        for (int q = 0; q < 16; ++q) a[q] = (16 * h + q < lane) ? a[q] * ri : 0.0;
      }
      const double col = treduce16(a, lane);
      if (lane < 16 && gj0 + lane < n) atomicAdd(pc.czc + gj0 + lane, col);
    }
    if (lane < rows) atomicAdd(pc.czc + gi, row);
  }
}

// e[cidx[k]] += czc[k]
__global__ void coarse_scatter_kernel(DevPrecond pc, double* __restrict__ e, const PcgScalars* guard) {
  pdl_wait();
  if (stopped(guard)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < pc.nc; k += stride) e[pc.cidx[k]] += pc.czc[k];
}

// device-side PCG loop: the graph's while node runs another body only while
// the stopping test has not fired (one thread, once per body)
__global__ void pcg_loop_condition_kernel(const PcgScalars* sc, cudaGraphConditionalHandle loop) {
  pdl_wait();
  cudaGraphSetConditional(loop, *((volatile const int32_t*)&sc->done) ? 0u : 1u);
}

// r.z into sc->rz_new (the hybrid preconditioner does not accumulate it itself)
__global__ void pcg_rz_kernel(PcgScalars* sc, const double* __restrict__ r, const double* __restrict__ z, int64_t n) {
  pdl_wait();
  if (stopped(sc)) return;
  double part = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) part = fma(r[i], z[i], part);
  __shared__ double sh[32];
  const double s = block_sum(part, sh);
  if (threadIdx.x == 0) atomicAdd(&sc->rz_new, s);
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
    sc->z_last = sc->z0;
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

// r != nullptr (hybrid preconditioner, which does not accumulate r.z itself): r.z into
// sc->rz_new in the same pass, each block before it takes its ticket
__global__ void pcg_finish_kernel(PcgScalars* sc, const double* __restrict__ z, const double* __restrict__ r,
                                  int64_t n) {
  if (stopped(sc)) return;
  double part = 0, rz = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double zi = z[i];
    part = fma(zi, zi, part);
    if (r) rz = fma(r[i], zi, rz);
  }
  if (r) {
    __shared__ double shr[32];
    const double s = block_sum(rz, shr);
    if (threadIdx.x == 0) atomicAdd(&sc->rz_new, s);
    __syncthreads();
  }
  if (last_block(sc, part) && threadIdx.x == 0) {
    __threadfence();
    volatile PcgScalars* v = sc;
    double zn = sqrt(v->zz);
    int it = v->iters + 1;
    sc->iters = it;
    sc->z_last = zn;
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
  pdl_wait();
  // the scalars once per block (strong loads by every thread cost ~25 us on config 4)
  __shared__ double s_alpha;
  __shared__ int s_kk, s_stop;
  if (threadIdx.x == 0) {
    volatile const PcgScalars* v = sc;
    s_stop = v->done;
    s_kk = v->k - 1;  // iteration of the apply that just ran
    s_alpha = s_stop ? 0.0 : v->rz_old / v->pq2[s_kk & 1];
  }
  __syncthreads();
  if (s_stop) return;
  const int kk = s_kk;
  const double* __restrict__ p = (kk & 1) ? p1 : p0;
  const double alpha = s_alpha;
  double part = 0;
  // two dofs per thread with 16-byte accesses (the slab vectors are 256-byte aligned)
  const int64_t n2 = pc.n_total >> 1, stride = (int64_t)gridDim.x * blockDim.x;
  const double2* __restrict__ p2 = reinterpret_cast<const double2*>(p);
  double2* __restrict__ q2 = reinterpret_cast<double2*>(q);
  double2* __restrict__ x2 = reinterpret_cast<double2*>(x);
  double2* __restrict__ r2 = reinterpret_cast<double2*>(r);
  double2* __restrict__ z2 = reinterpret_cast<double2*>(z);
  auto jacobi = [&](int64_t i, double rn) {
    if (i < pc.off3) return 0.0;
    const double zi = pc.dinv[i - pc.off3] * rn;
    part = fma(rn, zi, part);
    return zi;
  };
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += stride) {
    const double2 pv = p2[k], qv = q2[k], rv = r2[k];
    double2 xv = x2[k];
    xv.x = fma(alpha, pv.x, xv.x);
    xv.y = fma(alpha, pv.y, xv.y);
    const double2 rn = make_double2(fma(-alpha, qv.x, rv.x), fma(-alpha, qv.y, rv.y));
    x2[k] = xv;
    r2[k] = rn;
    q2[k] = make_double2(0.0, 0.0);
    z2[k] = make_double2(jacobi(2 * k, rn.x), jacobi(2 * k + 1, rn.y));
  }
  if ((pc.n_total & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd length: the last dof
    const int64_t i = pc.n_total - 1;
    x[i] = fma(alpha, p[i], x[i]);
    const double rn = fma(-alpha, q[i], r[i]);
    r[i] = rn;
    q[i] = 0.0;
    z[i] = jacobi(i, rn);
  }
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

// ---------------------------------------------------------------- persistent PCG (small problems)
// Small problems are launch-latency bound in the 3-kernel iteration (config 5 at
// p <= 4: ~20-38 us per iteration for a few us of work). This kernel runs a whole
// solve (R-A16, the fused order of the 3-kernel path) in one cooperative launch,
// with a grid barrier between its phases.
// grid-wide barrier of the cooperative launch: cooperative_groups' grid sync
// (1.2 us on this B200 with 148-296 CTAs, vs 2.3-2.5 us for a counter +
// generation barrier in global memory; tools/grid_barrier_probe.cu)
__device__ __forceinline__ void grid_barrier() { cooperative_groups::this_grid().sync(); }

__device__ __forceinline__ void block_add(double v, double* dst, double* sh) {
  const double s = block_sum(v, sh);
  if (threadIdx.x == 0 && s != 0.0) atomicAdd(dst, s);
}

struct PersistentArgs {
  const double* b;
  const uint8_t* cons;
  double *x, *r, *z, *p0, *p1, *q;
};

__global__ void __launch_bounds__(512, 1)
    pcg_persistent_kernel(DevOperator op, DevPrecond pc, PcgScalars* sc, PersistentArgs a, int wb) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double sh[32];
  const int n = op.n_loc, nm = op.n_mat;
  double* R = reinterpret_cast<double*>(smem_raw);  // [nm][n][n], symmetric: R_s[j][i] = R_s[i][j]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double* w0 = R + (size_t)nm * n * n + (size_t)warp * 2 * wb;  // warp scratch: x_e / r_m
  double* w1 = w0 + wb;                                         // dof ids / z_m
  for (int i = threadIdx.x; i < nm * n * n; i += blockDim.x) R[i] = op.R[i];
  const int64_t N = pc.n_total, gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int gwarp = blockIdx.x * nw + warp, nwarps = gridDim.x * nw;
  const double rtol = sc->rtol;
  const int maxit = sc->maxit;
  auto all_patches = [&](double* rz_dst) {  // z += sum_m E_m A_m^-1 E_m^T r
    double part = 0.0;
    for (int64_t pid = gwarp; pid < pc.n_patches; pid += nwarps)
      part += warp_patch_solve(pc, pid, a.r, a.z, w0, w1, lane, [] { return true; });
    block_add(part, rz_dst, sh);
  };

  // ---- start: x0 = 0, r0 = b (masked), z0 = P^-1 r0, r0.z0 (into prz[0])
  double part = 0.0;
  for (int64_t i = gtid; i < N; i += gstride) {
    const double ri = a.cons[i] ? 0.0 : a.b[i];
    a.x[i] = 0.0;
    a.q[i] = 0.0;
    a.p0[i] = 0.0;
    a.p1[i] = 0.0;
    a.r[i] = ri;
    const double zi = i >= pc.off3 ? pc.dinv[i - pc.off3] * ri : 0.0;
    a.z[i] = zi;
    part = fma(ri, zi, part);
  }
  block_add(part, &sc->prz[0], sh);
  grid_barrier();
  all_patches(&sc->prz[0]);
  grid_barrier();

  double z0 = 0.0;
  for (int k = 0;; ++k) {
    // ---- fused apply: p_k = z_k + beta_k p_{k-1} (owners write it), ||z_k||^2, q = A p_k, p.q
    volatile PcgScalars* v = sc;
    const double rz = v->prz[k % 3];
    const double beta = k == 0 ? 0.0 : rz / v->prz[(k + 2) % 3];
    const double* p_old = (k & 1) ? a.p0 : a.p1;
    double* p_new = (k & 1) ? a.p1 : a.p0;
    if (gtid == 0) sc->prz[(k + 1) % 3] = 0.0;  // accumulated from the update on, after the barrier
    double zz = 0.0, pq = 0.0;
    long long* ids = reinterpret_cast<long long*>(w1);
    for (int64_t c = gwarp; c < op.n_cells; c += nwarps) {
      const int own = op.own[c];
      for (int i = lane; i < n; i += 32) {
        const int l = op.lut[i];
        const int bse = op.ebase[c * 16 + (l >> 9)];
        double val = 0.0;
        long long id = -1;
        if (bse >= 0) {
          id = bse + (l & 511);
          const double zi = a.z[id];
          val = fma(beta, p_old[id], zi);
          if ((own >> (l >> 9)) & 1) {
            p_new[id] = val;
            zz = fma(zi, zi, zz);
          }
        }
        w0[i] = val;
        ids[i] = id;
      }
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        double acc = 0.0;
        for (int s = 0; s < nm; ++s) {
          const double* Rs = R + (size_t)s * n * n + i;
          double t = 0.0;
          for (int j = 0; j < n; ++j) t = fma(Rs[j * n], w0[j], t);
          acc = fma(op.coef[c * nm + s], t, acc);
        }
        if (ids[i] >= 0) {
          atomicAdd(a.q + ids[i], acc);
          pq = fma(w0[i], acc, pq);
        }
      }
      __syncwarp();
    }
    block_add(zz, &sc->pzz[k & 1], sh);
    block_add(pq, &sc->ppq[k & 1], sh);
    grid_barrier();

    // ---- stopping test on z_k (R-A16): every thread takes the same decision
    const double zn = sqrt(v->pzz[k & 1]);
    bool stop = false, conv = false;
    if (k == 0) {
      z0 = zn;
      conv = zn == 0.0;
      stop = conv || maxit <= 0;
    } else {
      conv = zn <= rtol * z0;
      stop = conv || k >= maxit;
    }
    if (stop) {
      if (gtid == 0) {
        sc->iters = k;
        sc->z0 = z0;
        sc->z_last = zn;
        sc->converged = conv;
        sc->done = 1;
        sc->k = k + 1;
      }
      break;
    }

    // ---- x += alpha p_k, r -= alpha q, q = 0, interior Jacobi z_I = D r_I, z_Gamma = 0, r.z
    const double alpha = rz / v->ppq[k & 1];
    if (gtid == 0) {  // last read after the previous barrier; accumulated again in the next apply
      sc->pzz[(k + 1) & 1] = 0.0;
      sc->ppq[(k + 1) & 1] = 0.0;
    }
    part = 0.0;
    for (int64_t i = gtid; i < N; i += gstride) {
      a.x[i] = fma(alpha, p_new[i], a.x[i]);
      const double rn = fma(-alpha, a.q[i], a.r[i]);
      a.r[i] = rn;
      a.q[i] = 0.0;
      double zi = 0.0;
      if (i >= pc.off3) {
        zi = pc.dinv[i - pc.off3] * rn;
        part = fma(rn, zi, part);
      }
      a.z[i] = zi;
    }
    block_add(part, &sc->prz[(k + 1) % 3], sh);
    grid_barrier();
    // ---- star patches
    all_patches(&sc->prz[(k + 1) % 3]);
    grid_barrier();
  }
}

unsigned vec_grid(int64_t n) {
  int64_t g = (n + kVecThreads - 1) / kVecThreads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace

PersistentPcg plan_persistent_pcg(const DevOperator& op, const DevPrecond& pc) {
  PersistentPcg plan;
  if (pc.hybrid || pc.npad_max > 256 || op.n_loc > 128) return plan;
  plan.wb = std::max(pc.npad_max, (op.n_loc + 31) / 32 * 32);
  const size_t rbytes = sizeof(double) * (size_t)op.n_mat * op.n_loc * op.n_loc;
  for (int w : {16, 8, 4}) {
    const size_t sm = rbytes + sizeof(double) * 2 * (size_t)plan.wb * w;
    if (sm <= kMaxSmem) {
      plan.warps = w;
      plan.smem = sm;
      break;
    }
  }
  if (!plan.warps) return plan;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaFuncSetAttribute(pcg_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.smem) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pcg_persistent_kernel, plan.warps * 32, plan.smem) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    plan.warps = 0;
    return plan;
  }
  plan.grid = sms * std::min(per_sm, 2);
  return plan;
}

cudaError_t launch_persistent_pcg(const PersistentPcg& plan, const DevOperator& op, const DevPrecond& pc,
                                  PcgScalars* sc, const double* b, const uint8_t* cons, double* x, double* r,
                                  double* z, double* p0, double* p1, double* q, cudaStream_t s) {
  PersistentArgs a{b, cons, x, r, z, p0, p1, q};
  DevOperator o = op;
  DevPrecond c = pc;
  int wb = plan.wb;
  void* args[] = {(void*)&o, (void*)&c, (void*)&sc, (void*)&a, (void*)&wb};
  return cudaLaunchCooperativeKernel((const void*)pcg_persistent_kernel, dim3(plan.grid), dim3(plan.warps * 32), args,
                                     plan.smem, s);
}

cudaError_t launch_apply(const DevOperator& op, const double* x, double* y, double* pq_acc,
                         const PcgScalars* guard, cudaStream_t s) {
  if (op.fact) return launch_fact_apply<false>(op, x, y, pq_acc, guard, nullptr, nullptr, nullptr, s);
  return launch_apply_tc<false>(op, x, y, pq_acc, guard, s);
}

size_t max_kernel_smem() { return kMaxSmem; }

int count_precond_launches(const DevPrecond& pc) {
  const int patch_launches = pc.n_patches == 0 ? 0 : (pc.n_big > 0) + (pc.n_big < pc.n_patches);
  return 1 + patch_launches;
}

cudaError_t launch_precond_part(int part, const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                                const PcgScalars* guard, cudaStream_t s) {
  switch (part) {
    case 0:
      return launch_k(precond_init_kernel, dim3(vec_grid(pc.n_total)), dim3(kVecThreads), 0, s, pc, r, z, rz_acc,
                      guard);
    case 1:
      if (pc.n_patches > 0) {
        const int W = pc.ldg_warps;
        cudaError_t e = cudaSuccess;
        if (pc.n_big > 0) {  // one CTA per patch
          const size_t sm = 2 * sizeof(double) * pc.npad_max;
          e = W == 4 ? launch_kx(pdl_patch_enabled(), patch_ldg_kernel<4>, dim3((unsigned)pc.n_big), dim3(4 * 32), sm,
                                 s, pc, r, z, rz_acc, guard)
                     : launch_kx(pdl_patch_enabled(), patch_ldg_kernel<8>, dim3((unsigned)pc.n_big), dim3(8 * 32), sm,
                                 s, pc, r, z, rz_acc, guard);
          if (e != cudaSuccess) return e;
        }
        if (pc.n_big < pc.n_patches) {  // one warp per small patch
          if (pc.small_grid > 0) {  // persistent warps walking the small patches
            const size_t sm = 4 * sizeof(double) * kSmallPatch * W;
            e = W == 4 ? launch_kx(pdl_patch_enabled(), patch_warp_loop_kernel<4>, dim3(pc.small_grid), dim3(4 * 32),
                                   sm, s, pc, r, z, rz_acc, guard)
                       : launch_kx(pdl_patch_enabled(), patch_warp_loop_kernel<8>, dim3(pc.small_grid), dim3(8 * 32),
                                   sm, s, pc, r, z, rz_acc, guard);
          } else {
            const size_t sm = 2 * sizeof(double) * kSmallPatch * W;
            const dim3 grid((unsigned)((pc.n_patches - pc.n_big + W - 1) / W));
            e = W == 4 ? launch_kx(pdl_patch_enabled(), patch_warp_kernel<4>, grid, dim3(4 * 32), sm, s, pc, r, z,
                                   rz_acc, guard)
                       : launch_kx(pdl_patch_enabled(), patch_warp_kernel<8>, grid, dim3(8 * 32), sm, s, pc, r, z,
                                   rz_acc, guard);
          }
        }
        return e;
      }
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_precond_hybrid(const DevOperator& op, const DevPrecond& pc, const double* r, double* z,
                                  const PcgScalars* guard, cudaStream_t s) {
  // symmetric multiplicative sweep X_I (Jacobi), X_Gamma (patches), W (coarse), X_Gamma, X_I
  const dim3 vg(vec_grid(pc.n_total)), vb(kVecThreads);
  cudaError_t e = launch_k(hyb_jacobi_kernel, vg, vb, 0, s, pc, r, z, pc.s1, 0, guard);  // also hy = 0
  if (e != cudaSuccess) return e;
  DevPrecond pp = pc;
  pp.out_scale = pc.s2;
  for (int stage = 1; stage < 5; ++stage) {
    if ((e = launch_apply(op, z, pc.hy, nullptr, guard, s)) != cudaSuccess) return e;
    if ((e = launch_k(hyb_residual_kernel, vg, vb, 0, s, pc, r, pc.hy, pc.ht, guard)) != cudaSuccess) return e;
    if (stage == 1 || stage == 3) {  // interface star patches, weight 1/rho_2
      if ((e = launch_precond_part(1, pp, pc.ht, z, nullptr, guard, s)) != cudaSuccess) return e;
    } else if (stage == 2) {         // exact coarse solve on W^k
      if (pc.nc > 0) {
        if ((e = launch_k(coarse_symv_kernel, dim3(148 * 4), dim3(256), 0, s, pc, (const double*)pc.ht, guard)) !=
            cudaSuccess)
          return e;
        if ((e = launch_k(coarse_scatter_kernel, dim3(vec_grid(pc.nc)), vb, 0, s, pc, z, guard)) != cudaSuccess)
          return e;
      }
    } else {                         // interior Jacobi, weight 1/rho_1
      if ((e = launch_k(hyb_jacobi_kernel, vg, vb, 0, s, pc, (const double*)pc.ht, z, pc.s1, 1, guard)) != cudaSuccess)
        return e;
    }
  }
  return cudaSuccess;
}

int count_hybrid_launches(const DevPrecond& pc) {
  const int patches = count_precond_launches(pc) - 1;
  return 1 + 4 * 2 + 2 * patches + (pc.nc > 0 ? 2 : 0) + 1;
}

cudaError_t launch_pcg_loop_condition(const PcgScalars* sc, cudaGraphConditionalHandle loop, cudaStream_t s) {
  return launch_k(pcg_loop_condition_kernel, dim3(1), dim3(1), 0, s, sc, loop);
}

cudaError_t launch_pcg_rz(PcgScalars* sc, const double* r, const double* z, int64_t n, cudaStream_t s) {
  return launch_k(pcg_rz_kernel, dim3(vec_grid(n)), dim3(kVecThreads), 0, s, sc, r, z, n);
}

cudaError_t launch_precond(const DevPrecond& pc, const double* r, double* z, double* rz_acc,
                           const PcgScalars* guard, cudaStream_t s) {
  for (int part = 0; part < 2; ++part) {
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
cudaError_t launch_pcg_finish(PcgScalars* sc, const double* z, const double* r, int64_t n, cudaStream_t s) {
  pcg_finish_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, z, r, n);
  return cudaGetLastError();
}
cudaError_t launch_pcg_direction(PcgScalars* sc, const double* z, double* p, double* q, int64_t n, cudaStream_t s) {
  pcg_direction_kernel<<<vec_grid(n), kVecThreads, 0, s>>>(sc, z, p, q, n);
  return cudaGetLastError();
}

bool fused_pcg_supported(const DevOperator& op) { return op.Bsw && op.own; }

// Variant k's cell tiles and persistent grid for this operator (occupancy from
// the PCG instance's registers and shared memory); -1 if it cannot run.
// Variant k with ring mode `ring`: 0 the default rule below, 1 the deepest ring
// that still fits two CTAs per SM (at least KS + 1 chunks), 2 the deepest ring
// for one CTA per SM (the setup autotuner tries all three).
int apply_configure_variant_ring(DevOperator& op, int k, int ring) {
  int cnt = 0;
  const ApplyVariant* vs = apply_variants(&cnt);
  if (k < 0 || k >= cnt || vs[k].nm != op.n_mat || vs[k].nm0 != op.nm0) return -1;
  const ApplyVariant& v = vs[k];
  // Ring depth: each K group consumes every KS-th chunk, so the ring holds S / KS
  // chunks ahead per group; take the deepest ring (up to 4 per group) that keeps
  // two CTAs per SM if the registers allow two, else one CTA per SM.
  const size_t base = apply_smem_layout(v.bm, v.nq, v.ks, 0, op.kp, op.n_mat).total;
  const size_t chunk = sizeof(double) * apply_chunk_doubles(op.n_mat);
  int dev = 0, sms = 148, regs_occ = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&regs_occ, v.fn[1], apply_threads(v), 0) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  const size_t two_per_sm = 228 * 1024 / 2 - 1024;
  const int s_max = 4 * v.ks;
  int S = 0;
  if (ring == 1) {
    if (regs_occ >= 2 && base + chunk * (v.ks + 1) <= two_per_sm)
      S = (int)std::min<size_t>(s_max, (two_per_sm - base) / chunk);
  } else if (ring == 2) {
    if (base + chunk * (v.ks + 2) <= kMaxSmem) S = (int)std::min<size_t>(s_max, (kMaxSmem - base) / chunk);
  } else if (regs_occ >= 2 && base + chunk * 2 * v.ks <= two_per_sm) {
    S = (int)std::min<size_t>(s_max, (two_per_sm - base) / chunk);
  } else if (base + chunk * (v.ks + 2) <= kMaxSmem) {
    S = (int)std::min<size_t>(s_max, (kMaxSmem - base) / chunk);
  }
  if (S == 0) return -1;
  op.apply_slots = S;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn[1], apply_threads(v), apply_variant_smem(v, op)) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return -1;
  }
  op.av = k;
  op.ntiles = (int)((op.n_cells + v.bm - 1) / v.bm);
  const int64_t units = (int64_t)op.ntiles * op.ngroups;
  op.apply_grid = (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * sms));
  return 0;
}

int apply_configure_variant(DevOperator& op, int k) { return apply_configure_variant_ring(op, k, 0); }

// Variant k with an explicit ring depth (slots >= KS + 1) and grid (0: the persistent grid of
// resident CTAs), e.g. to reproduce the configuration another setup's timing chose.
int apply_configure_exact(DevOperator& op, int k, int slots, int grid) {
  DevOperator t = op;
  if (apply_configure_variant_ring(t, k, 0)) return -1;
  int cnt = 0;
  const ApplyVariant& v = apply_variants(&cnt)[k];
  if (slots < v.ks + 1 || apply_smem_layout(v.bm, v.nq, v.ks, slots, t.kp, t.n_mat).total > kMaxSmem) return -1;
  t.apply_slots = slots;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn[1], apply_threads(v), apply_variant_smem(v, t)) !=
          cudaSuccess ||
      per_sm < 1) {
    cudaGetLastError();
    return -1;
  }
  const int64_t units = (int64_t)t.ntiles * t.ngroups;
  t.apply_grid = grid > 0 ? (int)std::min<int64_t>(grid, units)
                          : (int)std::max<int64_t>(1, std::min<int64_t>(units, (int64_t)per_sm * sms));
  op = t;
  return 0;
}

int apply_variant_count() {
  int cnt = 0;
  apply_variants(&cnt);
  return cnt;
}

// Setup-time autotuning of the apply's warp layout: every variant that fits is
// timed on this operator (one warm-up, then `reps` plain applies between CUDA
// events on `s`) and the fastest is kept.
// Setup-time choice for workloads of small patches only (patch_warp_kernel, one
// warp per patch, vs patch_warp_loop_kernel, resident warps walking the
// patches with the next patch's loads in flight): both timed on r (reps launches
// each), the faster kept in pc.small_grid.
int tune_small_patches(DevPrecond& pc, const double* r, double* z, cudaStream_t s, int reps) {
  pc.small_grid = 0;
  if (pc.n_big >= pc.n_patches) return 0;
  const int W = pc.ldg_warps;
  const void* fn = W == 4 ? (const void*)patch_warp_loop_kernel<4> : (const void*)patch_warp_loop_kernel<8>;
  const size_t sm = 4 * sizeof(double) * kSmallPatch * W;
  int dev = 0, sms = 148, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, W * 32, sm) != cudaSuccess || per_sm < 1) {
    cudaGetLastError();
    return 0;
  }
  const int64_t needed = (pc.n_patches - pc.n_big + W - 1) / W;
  const int grid = (int)std::min<int64_t>(needed, (int64_t)per_sm * sms);
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1;
  float t[2] = {0.f, 0.f};
  for (int mode = 0; mode < 2; ++mode) {
    pc.small_grid = mode ? grid : 0;
    launch_precond_part(1, pc, r, z, nullptr, nullptr, s);
    cudaEventRecord(e0, s);
    for (int k = 0; k < reps; ++k) launch_precond_part(1, pc, r, z, nullptr, nullptr, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t[mode], e0, e1);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  pc.small_grid = t[1] < t[0] ? grid : 0;
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// Setup-time autotuning of the apply's warp layout. Every (layout, ring depth,
// grid) candidate that fits is timed on the kernel the solve runs -- the
// PCG-mode apply (sc: scalars with rtol 0 and a huge maxit, so the stopping
// test never fires; x != 0; p0, p1: scratch direction buffers), or the plain
// apply when the operator has no PCG mode -- in three interleaved rounds of
// `reps` launches after a warm-up, each candidate scored by its best round.
// (Timing each candidate once, back to back, let the clock drift right after
// the patch-setup kernel pick a layout that ran the config-3 solve at 167
// instead of 177 PCG it/s: profiles/round2/experiments/apply_layout_bench_ab.jsonl.)
int tune_apply(DevOperator& op, const double* x, double* y, PcgScalars* sc, double* p0, double* p1, cudaStream_t s,
               int reps) {
  const int cnt = apply_variant_count();
  const bool pcg = sc && fused_pcg_supported(op);
  std::vector<DevOperator> cand;
  for (int kr = 0; kr < 3 * cnt; ++kr) {
    const int k = kr / 3, ring = kr % 3;
    DevOperator t = op;
    if (apply_configure_variant_ring(t, k, ring)) continue;
    if (ring > 0) {  // skip ring modes that give the default's depth
      DevOperator d = op;
      if (!apply_configure_variant_ring(d, k, 0) && d.apply_slots == t.apply_slots) continue;
    }
    // the persistent grid (resident CTAs, each a contiguous range of units), and
    // for problems with fewer units than twice that, one CTA per unit (waves)
    const int64_t units = (int64_t)t.ntiles * t.ngroups;
    const int grids[2] = {t.apply_grid, units < 2 * (int64_t)t.apply_grid ? (int)units : 0};
    for (int gi = 0; gi < 2; ++gi) {
      if (grids[gi] <= 0 || (gi == 1 && grids[1] == grids[0])) continue;
      t.apply_grid = grids[gi];
      cand.push_back(t);
    }
  }
  auto launch = [&](const DevOperator& t) {
    return pcg ? launch_apply_tc<1>(t, x, y, nullptr, sc, s, sc, p0, p1) : launch_apply_tc<0>(t, x, y, nullptr, nullptr, s);
  };
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1;
  std::vector<float> best_ms(cand.size(), -1.f);
  for (int round = 0; round < 3; ++round)
    for (size_t c = 0; c < cand.size(); ++c) {
      if (launch(cand[c]) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      cudaEventRecord(e0, s);
      for (int r = 0; r < reps; ++r) launch(cand[c]);
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (best_ms[c] < 0.f || ms < best_ms[c]) best_ms[c] = ms;
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGetLastError();
  int best = -1;
  for (size_t c = 0; c < cand.size(); ++c)
    if (best_ms[c] >= 0.f && (best < 0 || best_ms[c] < best_ms[best])) best = (int)c;
  if (best < 0) return -1;
  op = cand[best];
  return 0;
}

cudaError_t launch_pcg_fused_apply(const DevOperator& op, PcgScalars* sc, const double* z, double* p0, double* p1,
                                   double* q, cudaStream_t s) {
  if (op.fact) return launch_fact_apply<true>(op, z, q, nullptr, sc, sc, p0, p1, s);
  return launch_apply_tc<true>(op, z, q, nullptr, sc, s, sc, p0, p1);
}

// Setup-time choice between the DMMA apply (op.fact = 0, its tuned layout) and the
// factored two-stage apply (op.fact = 1, 2, 3: its tile sizes), timed on the iteration the
// solve runs: for each candidate a PCG on b is started (x = 0, r = b, z = P^-1 r; sc_init:
// the scalars with rtol 0 and a huge maxit, so the stopping test never fires) and `reps`
// whole iterations (fused apply, update + Jacobi, patch solves) are timed after a warm-up
// one, in three interleaved rounds, best round each. The factored stages lose up to
// 0.15 ms per apply inside the iteration which a loop of applies alone does not show (RT_9:
// 0.345 ms alone, 0.499 ms in the solve; experiments/fact_in_solve.jsonl), and a loop of
// patch solves + apply without the vector update reproduced only part of that: on close
// calls (RT_9, Ned1_5) it picked the slower iteration in some setups.
int tune_fact(DevOperator& op, const DevPrecond& pc, const double* b, const uint8_t* cons, double* x, double* r,
              double* z, double* q, PcgScalars* sc, const PcgScalars* sc_init, double* p0, double* p1,
              cudaStream_t s, int reps) {
  op.fact = 0;
  // Only meshes of >= kFactMinCells cells are considered: below that the two timings are
  // within noise, and a timing-dependent choice would make the rounding of small solves
  // (the iteration count of an ill-conditioned one) vary from setup to setup.
  if (!fact_apply_fits(op, 1) || op.n_cells < kFactMinCells || !fused_pcg_supported(op)) return 0;
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1;
  const int64_t n = pc.n_total;
  // candidates: the DMMA apply, the factored apply with op.fact = 1, 2, 3 and, for the 32-cell
  // tiles, column splits (stage A, stage B) that leave every CTA >= 3 column blocks (the stages
  // launch one CTA per cell tile otherwise: 96 and 128 CTAs on the 8^3 x 6 mesh, 1.1 and 1.5
  // waves on config 4; experiments/fact_split_in_solve.jsonl)
  struct Cand {
    int f, nsa, nsb;
  };
  std::vector<Cand> cand = {{0, 1, 1}, {1, 1, 1}};
  const int nblk_a = op.nfp / 32, nblk_b = (op.kp + 31) / 32;
  for (int f = 2; f <= 3; ++f)
    for (const Cand& c : {Cand{f, 1, 1}, Cand{f, 2, 1}, Cand{f, 2, 2}, Cand{f, 3, 1}, Cand{f, 3, 2}, Cand{f, 4, 2}})
      if ((c.nsa == 1 || nblk_a / c.nsa >= 3) && (c.nsb == 1 || nblk_b / c.nsb >= 3)) cand.push_back(c);
  const int kNF = (int)cand.size();
  std::vector<float> best(kNF, -1.f);
  for (int round = 0; round < 3; ++round)
    for (int f = 0; f < kNF; ++f) {
      if (cand[f].f > 0 && !fact_apply_fits(op, cand[f].f)) continue;
      DevOperator t = op;
      t.fact = cand[f].f;
      t.fact_nsa = cand[f].nsa;
      t.fact_nsb = cand[f].nsb;
      auto iteration = [&]() {
        cudaError_t e = launch_pcg_fused_apply(t, sc, z, p0, p1, q, s);
        if (e == cudaSuccess) e = launch_pcg_update_jacobi(sc, pc, p0, p1, q, x, r, z, s);
        if (e == cudaSuccess) e = launch_precond_part(1, pc, r, z, &sc->rz_acc, sc, s);
        return e;
      };
      bool ok = cudaMemcpyAsync(sc, sc_init, sizeof(PcgScalars), cudaMemcpyHostToDevice, s) == cudaSuccess &&
                cudaMemsetAsync(p0, 0, sizeof(double) * n, s) == cudaSuccess &&
                cudaMemsetAsync(p1, 0, sizeof(double) * n, s) == cudaSuccess &&
                launch_pcg_init(b, cons, n, x, r, q, s) == cudaSuccess &&
                launch_precond(pc, r, z, &sc->rz_acc, nullptr, s) == cudaSuccess && iteration() == cudaSuccess;
      if (!ok) {
        cudaGetLastError();
        continue;
      }
      cudaEventRecord(e0, s);
      for (int k = 0; k < reps; ++k) iteration();
      cudaEventRecord(e1, s);
      if (cudaEventSynchronize(e1) != cudaSuccess) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (best[f] < 0.f || ms < best[f]) best[f] = ms;
    }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGetLastError();
  int f = 0;
  for (int k = 1; k < kNF; ++k)
    if (best[k] >= 0.f && (best[f] < 0.f || best[k] < best[f])) f = k;
  op.fact = cand[f].f;
  op.fact_nsa = cand[f].nsa;
  op.fact_nsb = cand[f].nsb;
  return 0;
}

bool fact_apply_fits(const DevOperator& op, int fact) {
  return op.F && fact >= 1 && fact <= 3 && fact_a_layout(op.kp, fact_bm_a(fact)).total <= kMaxSmem &&
         fact_b_layout(op.kp, op.nfp, fact_bm_b(fact)).total <= kMaxSmem;
}

cudaError_t launch_pcg_update_jacobi(PcgScalars* sc, const DevPrecond& pc, const double* p0, const double* p1,
                                     double* q, double* x, double* r, double* z, cudaStream_t s) {
  return launch_k(pcg_update_jacobi_kernel, dim3(vec_grid((pc.n_total + 1) / 2)), dim3(kVecThreads), 0, s, sc, pc, p0,
                  p1, q, x, r, z);
}

// FP64 tensor-core peak microbenchmark (roofline denominator of the apply,
// bench.py): 4 independent DMMA.8x8x4 chains per warp, issue-bound.
__global__ void dmma_peak_kernel(double* out, int n) {
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  const double a = threadIdx.x * 1e-3, b = 1.0;
  for (int i = 0; i < n; ++i) {
    dmma884(c0, c1, a, b);
    dmma884(d0, d1, a, b);
    dmma884(e0, e1, a, b);
    dmma884(f0, f1, a, b);
  }
  if (c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1 == 1.2345) out[0] = 1.0;
}

// SM clock probe (rdr_debug_profile_clocks): one thread spins `ns` nanoseconds of the
// global timer and adds the SM cycles per microsecond it saw (MHz) to acc[0], 1 to acc[1]
__global__ void sm_clock_probe_kernel(double* acc, unsigned ns) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  const long long c0 = clock64();
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (t1 - t0 < ns);
  const long long c1 = clock64();
  acc[0] += (double)(c1 - c0) * 1e3 / (double)(t1 - t0);
  acc[1] += 1.0;
}
cudaError_t launch_sm_clock_probe(double* acc, unsigned ns, cudaStream_t s) {
  sm_clock_probe_kernel<<<1, 1, 0, s>>>(acc, ns);
  return cudaGetLastError();
}

cudaError_t launch_dmma_peak(double* out, int n, int blocks, int threads, cudaStream_t s) {
  dmma_peak_kernel<<<blocks, threads, 0, s>>>(out, n);
  return cudaGetLastError();
}

}  // namespace rdr

namespace rdr {
void configure_kernels() {  // errors here would surface as a later launch's cudaGetLastError
  cudaFuncSetAttribute(fact_stage_a_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_a_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_a_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_a_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<24, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<24, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(fact_stage_b_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(patch_ldg_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaFuncSetAttribute(patch_ldg_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  int cnt = 0;
  const ApplyVariant* v = apply_variants(&cnt);
  for (int k = 0; k < cnt; ++k)
    for (const void* fn : v[k].fn) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  cudaGetLastError();
}
}  // namespace rdr
