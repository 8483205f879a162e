// Microbenchmark: HBM streaming rate of (A) a TMA bulk-copy ring (one producer
// thread, consumer warps that only touch the data) vs (B) plain 32-byte
// non-allocating loads, over a 1 GiB buffer. Sizes the patch-kernel pipeline.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/stream_probe.cu -o tools/stream_probe
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

// A: grid-stride over tiles of `tile` bytes; CTA b handles tiles b, b+G, ...
__global__ void ring_kernel(const double* src, int64_t ntiles, int tile, int S, int nw, double* out, int hold = 0,
                            int after = 0) {
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
  const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (warp == nw) {
    if (lane == 0) {
      int slot = 0; uint32_t ph = 0; bool first = true;
      for (int64_t j = 0; j < mine; ++j) {
        if (!first) mbar_wait(&empty[slot], ph ^ 1u);
        mbar_expect_tx(&full[slot], tile);
        bulk_g2s(ring + (size_t)slot * tile, (const char*)src + (blockIdx.x + j * gridDim.x) * (int64_t)tile, tile, &full[slot]);
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
    acc += t[lane] + t[tile / 8 - 1 - lane];
    if (hold && !after) { const long long c0 = clock64(); while (clock64() - c0 < hold) {} }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (hold && after) { const long long c0 = clock64(); while (clock64() - c0 < hold) {} }
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
// B: each warp streams 8 KB tiles with 8 x 32 B loads per lane
__global__ void ldg_kernel(const double* src, int64_t ntiles, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp, nwt = (int64_t)gridDim.x * (blockDim.x >> 5);
  double acc = 0;
  for (int64_t t = gw; t < ntiles; t += nwt) {
    const double4* p = (const double4*)(src + t * 1024) + lane;
    double4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld4(p + 32 * k);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 12345.0) out[0] = acc;
}

int main() {
  const size_t bytes = 1ull << 30;
  double *src, *out;
  cudaMalloc(&src, bytes); cudaMalloc(&out, 8);
  cudaMemset(src, 0, bytes);
  cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto f) {
    f(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i = 0; i < 5; ++i) f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); return bytes * 5 / (ms / 1e3) / 1e9;
  };
  for (int hold : {0, 500, 1000, 2000, 4000})
    for (int after : {0, 1})
      for (int cfg = 0; cfg < 3; ++cfg) {
        const int c = cfg == 0 ? 2 : 1, S = cfg == 0 ? 8 : (cfg == 1 ? 16 : 24), nw = 8, tile = 8192;
        size_t smem = (size_t)S * tile + 16 * S + 256;
        int64_t nt = bytes / tile;
        double gbs = timeit([&] { ring_kernel<<<148 * c, (nw + 1) * 32, smem>>>(src, nt, tile, S, nw, out, hold, after); });
        printf("hold %4d %s ctas/SM %d slots %2d consumers %d : %7.1f GB/s\n", hold, after ? "after " : "before", c, S, nw, gbs);
      }
  for (int w : {8, 16, 32, 48, 64}) {
    int threads = 256, blocks = 148 * w / 8;
    double gbs = timeit([&] { ldg_kernel<<<blocks, threads>>>(src, bytes / 8192, out); });
    printf("ldg warps/SM %2d : %7.1f GB/s\n", w, gbs);
  }
  return 0;
}
