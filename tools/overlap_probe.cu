// Microbenchmark: can an HBM read stream (the patch solves) and a DMMA-bound
// kernel (the operator apply) run at the same time on one B200 without slowing
// each other down? (A) a TMA bulk-copy ring streaming a 4 GiB buffer, (B) a
// register-only DMMA.8x8x4 loop. Each alone, then both launched on two streams,
// either on disjoint SM sets (A's shared memory excludes B from its SMs) or
// co-resident on every SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/overlap_probe.cu -o tools/overlap_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred P;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra W_%=;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// A: CTA b streams tiles b, b+G, ... (passes over the buffer); nw consumer warps
__global__ void ring_kernel(const double* src, int64_t ntiles, int passes, int tile, int S, int nw, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + S;
  unsigned char* ring = sm + 16 * S + 128;
  ring = (unsigned char*)(((uintptr_t)ring + 127) & ~(uintptr_t)127);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t per = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t mine = per * passes;
  if (warp == nw) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0; bool first = true;
      for (int64_t j = 0; j < mine; ++j) {
        if (!first) mbar_wait(&empty[slot], ph ^ 1u);
        mbar_expect_tx(&full[slot], tile);
        const int64_t t = blockIdx.x + (j % per) * gridDim.x;
        bulk_g2s(ring + (size_t)slot * tile, (const char*)src + t * (int64_t)tile, tile, &full[slot]);
        if (++slot == S) { slot = 0; ph ^= 1u; first = false; }
      }
    }
    return;
  }
  double acc = 0;
  int slot = warp; uint32_t ph = 0;
  for (int64_t j = warp; j < mine; j += nw) {
    mbar_wait(&full[slot], ph);
    const double* t = (const double*)(ring + (size_t)slot * tile);
    for (int k = lane; k < tile / 8; k += 32) acc += t[k];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    slot += nw; if (slot >= S) { slot -= S; ph ^= 1u; }
  }
  if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ double4 ld4(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
// A': each warp streams 8 KB tiles with 8 x 32 B loads per lane (the patch kernel's loads)
__global__ void ldg_kernel(const double* src, int64_t ntiles, int passes, double* out) {
  extern __shared__ unsigned char pad[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nwt = (int64_t)gridDim.x * (blockDim.x >> 5);
  double acc = 0;
  for (int ps = 0; ps < passes; ++ps)
    for (int64_t t = gw; t < ntiles; t += nwt) {
      const double4* p = (const double4*)(src + t * 1024) + lane;
      double4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = ld4(p + 32 * k);
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
    }
  if (acc == 12345.0) out[0] = acc + pad[0];
}

// B: DMMA.8x8x4 issue loop, 4 independent accumulators per warp
__global__ void dmma_kernel(double* out, int n) {
  extern __shared__ unsigned char pad[];
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  double a = threadIdx.x * 1e-3, b = 1.0;
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
  }
  if (c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1 == 1.2345) out[0] = 1 + pad[0];
}

int main() {
  const size_t bytes = 4ull << 30;
  double *src, *out;
  cudaMalloc(&src, bytes); cudaMalloc(&out, 8);
  cudaMemset(src, 0, bytes);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaFuncSetAttribute(ldg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaStream_t sa, sb; cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  cudaEvent_t a0, a1, b0, b1, j0;
  cudaEventCreate(&a0); cudaEventCreate(&a1); cudaEventCreate(&b0); cudaEventCreate(&b1); cudaEventCreate(&j0);
  const int passes = 5;  // 20 GiB per run of A
  const int tile = 16384;
  const int64_t nt = bytes / tile;
  struct Res { float ams, bms; };
  // kind 0: TMA ring (S slots of 16 KB, 4 consumer warps), kind 1: LDG warps
  auto run = [&](int kind, int na, int a_smem_kb, int a_warps, int nb, int b_warps, int b_smem_kb, int n, bool doA, bool doB) {
    cudaDeviceSynchronize();
    cudaEventRecord(j0, 0);
    cudaStreamWaitEvent(sa, j0, 0); cudaStreamWaitEvent(sb, j0, 0);
    if (doA) {
      cudaEventRecord(a0, sa);
      if (kind == 0) {
        const int S = (a_smem_kb * 1024 - 512) / tile;
        ring_kernel<<<na, (a_warps + 1) * 32, a_smem_kb * 1024, sa>>>(src, nt, passes, tile, S, a_warps, out);
      } else {
        ldg_kernel<<<na, a_warps * 32, a_smem_kb * 1024, sa>>>(src, bytes / 8192, passes, out);
      }
      cudaEventRecord(a1, sa);
    }
    if (doB) {
      cudaEventRecord(b0, sb);
      dmma_kernel<<<nb, b_warps * 32, b_smem_kb * 1024, sb>>>(out, n);
      cudaEventRecord(b1, sb);
    }
    cudaDeviceSynchronize();
    Res r{0, 0};
    if (doA) cudaEventElapsedTime(&r.ams, a0, a1);
    if (doB) cudaEventElapsedTime(&r.bms, b0, b1);
    return r;
  };
  auto report = [&](const char* what, int kind, int na, int a_smem_kb, int a_warps, int nb, int b_warps, int b_smem_kb, int n) {
    run(kind, na, a_smem_kb, a_warps, nb, b_warps, b_smem_kb, n, true, true);  // warm
    Res A = run(kind, na, a_smem_kb, a_warps, nb, b_warps, b_smem_kb, n, true, false);
    Res B = run(kind, na, a_smem_kb, a_warps, nb, b_warps, b_smem_kb, n, false, true);
    Res C = run(kind, na, a_smem_kb, a_warps, nb, b_warps, b_smem_kb, n, true, true);
    const double abytes = (double)bytes * passes;
    const double bflop = 512.0 * 4 * nb * b_warps * (double)n;
    printf("%-34s A %3d CTA x %2d warps %3d KB | B %3d CTA x %2d warps | alone A %6.0f GB/s (%.2f ms) B %5.2f TF (%.2f ms) | "
           "together A %6.0f GB/s (%.2f ms) B %5.2f TF (%.2f ms)\n",
           what, na, a_warps, a_smem_kb, nb, b_warps, abytes / (A.ams / 1e3) / 1e9, A.ams, bflop / (B.bms / 1e3) / 1e12, B.bms,
           abytes / (C.ams / 1e3) / 1e9, C.ams, bflop / (C.bms / 1e3) / 1e12, C.bms);
  };
  const int n = 1 << 16;
  // disjoint SM sets: A takes >= 120 KB (one per SM), B 120 KB (cannot share an SM with A)
  for (int na : {148, 120, 110, 100, 90, 80}) {
    const int nb = 148 - na;
    if (nb == 0) { report("TMA alone, 1 CTA/SM", 0, na, 200, 4, 1, 4, 4, 1 << 10); continue; }
    report("TMA | DMMA on disjoint SMs", 0, na, 200, 4, nb, 16, 120, n);
  }
  for (int na : {148, 120, 100}) {
    const int nb = 148 - na;
    report("LDG | DMMA on disjoint SMs", 1, na, 120, 32, nb > 0 ? nb : 1, 16, 120, nb > 0 ? n : 1 << 10);
  }
  // co-resident: A small ring + B DMMA warps on every SM
  for (int bw : {4, 8, 16})
    for (int kb : {64, 96}) report("TMA + DMMA co-resident", 0, 148, kb, 2, 148, bw, 1, n);
  for (int aw : {8, 16})
    for (int bw : {4, 8}) report("LDG + DMMA co-resident", 1, 148, 1, aw, 148, bw, 1, n);
  return 0;
}
