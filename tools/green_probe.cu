// Probe: green contexts (driver SM partitions) for running the HBM-bound patch
// solves and the DMMA-bound apply at the same time on disjoint SM sets.
// Checks: runtime-API launches on green-context streams, the SMs each launch
// lands on, runtime-allocated memory visible from both partitions, concurrent
// throughput, and stream capture of a fork/join over the two partitions.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/green_probe.cu -o tools/green_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CKD(x)                                                                 \
  do {                                                                         \
    CUresult e_ = (x);                                                         \
    if (e_ != CUDA_SUCCESS) {                                                  \
      const char* s_ = nullptr;                                                \
      cuGetErrorString(e_, &s_);                                               \
      printf("%s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, (int)e_, s_);      \
      return 1;                                                                \
    }                                                                          \
  } while (0)
#define CKR(x)                                                                 \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__global__ void where_kernel(int* sm_of_block, int spin) {
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0) sm_of_block[blockIdx.x] = (int)smid();
}
__device__ __forceinline__ double4 ld4(const double4* p) {
  double4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__global__ void ldg_kernel(const double* src, int64_t ntiles, int passes, double* out) {
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
  if (acc == 12345.0) out[0] = acc;
}
__global__ void dmma_kernel(double* out, int n) {
  double c0 = 0, c1 = 0, d0 = 0, d1 = 0, e0 = 0, e1 = 0, f0 = 0, f1 = 0;
  double a = threadIdx.x * 1e-3, b = 1.0;
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(e0), "+d"(e1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1},{%2},{%3},{%0,%1};" : "+d"(f0), "+d"(f1) : "d"(a), "d"(b));
  }
  if (c0 + d0 + e0 + f0 + c1 + d1 + e1 + f1 == 1.2345) out[0] = 1;
}
// consumer waits (bounded) on a flag the producer sets: cross-partition signalling
__global__ void producer_kernel(int* flag, int spin) {
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    __threadfence();
    atomicExch(flag, 1);
  }
}
__global__ void consumer_kernel(const int* flag, int* result) {
  const long long t0 = clock64();
  int v = 0;
  while (true) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v || clock64() - t0 > 4000000000LL) break;
    __nanosleep(200);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) *result = v ? 1 : -1;
}

int main() {
  CKD(cuInit(0));
  CKR(cudaSetDevice(0));
  CKR(cudaFree(0));  // primary context (as torch makes it)
  CUdevice dev;
  CKD(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CKD(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  const size_t bytes = 4ull << 30;
  double *src, *out;
  CKR(cudaMalloc(&src, bytes));
  CKR(cudaMalloc(&out, 64));
  CKR(cudaMemset(src, 0, bytes));
  int* d_sm;
  CKR(cudaMalloc(&d_sm, 4096 * sizeof(int)));
  cudaEvent_t e0, e1, e2, e3, j;
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3); cudaEventCreate(&j);
  for (unsigned na : {40u, 48u, 56u, 64u}) {
    CUdevResource parts[2];
    unsigned nparts = 1;
    CUdevResource rest;
    CKD(cuDevSmResourceSplitByCount(&parts[0], &nparts, &all, &rest, 0, na));
    parts[1] = rest;
    CUdevResourceDesc da, dp;
    CKD(cuDevResourceGenerateDesc(&da, &parts[0], 1));
    CKD(cuDevResourceGenerateDesc(&dp, &parts[1], 1));
    CUgreenCtx ga, gp;
    CKD(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CKD(cuGreenCtxCreate(&gp, dp, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sa, sp;
    CKD(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
    CKD(cuGreenCtxStreamCreate(&sp, gp, CU_STREAM_NON_BLOCKING, 0));
    printf("split %u: apply partition %u SMs, patch partition %u SMs\n", na, parts[0].sm.smCount, parts[1].sm.smCount);
    // where do launches land?
    for (int w = 0; w < 2; ++w) {
      CKR(cudaMemset(d_sm, 0xff, 4096 * sizeof(int)));
      where_kernel<<<1024, 128, 0, w ? (cudaStream_t)sp : (cudaStream_t)sa>>>(d_sm, 20000);
      CKR(cudaGetLastError());
      CKR(cudaDeviceSynchronize());
      std::vector<int> h(1024);
      cudaMemcpy(h.data(), d_sm, 1024 * sizeof(int), cudaMemcpyDeviceToHost);
      std::vector<int> used(256, 0);
      int distinct = 0, lo = 999, hi = -1;
      for (int v : h) {
        if (v >= 0 && v < 256 && !used[v]++) ++distinct;
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
      }
      printf("  %s stream: 1024 blocks on %d distinct SMs (smid %d..%d)\n", w ? "patch" : "apply", distinct, lo, hi);
    }
    // throughput alone and together
    const int passes = 4, n = 1 << 16;
    auto run = [&](bool A, bool B, float* ta, float* tb) {
      cudaDeviceSynchronize();
      cudaEventRecord(j, 0);
      cudaStreamWaitEvent((cudaStream_t)sp, j, 0);
      cudaStreamWaitEvent((cudaStream_t)sa, j, 0);
      if (A) {
        cudaEventRecord(e0, (cudaStream_t)sp);
        ldg_kernel<<<parts[1].sm.smCount * 4, 256, 0, (cudaStream_t)sp>>>(src, bytes / 8192, passes, out);
        cudaEventRecord(e1, (cudaStream_t)sp);
      }
      if (B) {
        cudaEventRecord(e2, (cudaStream_t)sa);
        dmma_kernel<<<parts[0].sm.smCount, 512, 0, (cudaStream_t)sa>>>(out, n);
        cudaEventRecord(e3, (cudaStream_t)sa);
      }
      cudaDeviceSynchronize();
      if (A) cudaEventElapsedTime(ta, e0, e1);
      if (B) cudaEventElapsedTime(tb, e2, e3);
    };
    float ta = 0, tb = 0, ta2 = 0, tb2 = 0, dummy;
    run(true, true, &dummy, &dummy);
    run(true, false, &ta, &dummy);
    run(false, true, &dummy, &tb);
    run(true, true, &ta2, &tb2);
    const double flop = 512.0 * 4 * parts[0].sm.smCount * 16 * (double)n;
    printf("  LDG on patch SMs: alone %.0f GB/s, together %.0f GB/s | DMMA on apply SMs: alone %.2f TF, together %.2f TF\n",
           (double)bytes * passes / (ta / 1e3) / 1e9, (double)bytes * passes / (ta2 / 1e3) / 1e9, flop / (tb / 1e3) / 1e12,
           flop / (tb2 / 1e3) / 1e12);
    CKR(cudaGetLastError());
    // cross-partition flag: consumer launched FIRST on the apply partition, producer after
    int *flag, *res;
    cudaMalloc(&flag, 4); cudaMalloc(&res, 4);
    cudaMemset(flag, 0, 4); cudaMemset(res, 0, 4);
    cudaDeviceSynchronize();
    consumer_kernel<<<parts[0].sm.smCount * 2, 128, 0, (cudaStream_t)sa>>>(flag, res);
    producer_kernel<<<8, 32, 0, (cudaStream_t)sp>>>(flag, 100000);
    CKR(cudaDeviceSynchronize());
    int hres = 0;
    cudaMemcpy(&hres, res, 4, cudaMemcpyDeviceToHost);
    printf("  consumer-first flag handoff: %s\n", hres == 1 ? "ok" : "TIMED OUT");
    // graph capture of a fork/join over both partitions
    cudaStream_t cs;
    cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaEvent_t f1, f2, f3;
    cudaEventCreateWithFlags(&f1, cudaEventDisableTiming); cudaEventCreateWithFlags(&f2, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&f3, cudaEventDisableTiming);
    cudaError_t ce = cudaStreamBeginCapture((cudaStream_t)sp, cudaStreamCaptureModeRelaxed);
    if (ce == cudaSuccess) {
      cudaEventRecord(f1, (cudaStream_t)sp);
      cudaStreamWaitEvent((cudaStream_t)sa, f1, 0);
      where_kernel<<<1024, 128, 0, (cudaStream_t)sa>>>(d_sm, 20000);
      where_kernel<<<1024, 128, 0, (cudaStream_t)sp>>>(d_sm + 1024, 20000);
      cudaEventRecord(f2, (cudaStream_t)sa);
      cudaStreamWaitEvent((cudaStream_t)sp, f2, 0);
      ce = cudaStreamEndCapture((cudaStream_t)sp, &g);
    }
    if (ce == cudaSuccess) ce = cudaGraphInstantiate(&ge, g, 0);
    if (ce == cudaSuccess) {
      cudaMemset(d_sm, 0xff, 4096 * sizeof(int));
      ce = cudaGraphLaunch(ge, cs);
      cudaDeviceSynchronize();
    }
    if (ce == cudaSuccess) {
      std::vector<int> h(2048);
      cudaMemcpy(h.data(), d_sm, 2048 * sizeof(int), cudaMemcpyDeviceToHost);
      int lo[2] = {999, 999}, hi[2] = {-1, -1};
      std::vector<int> used[2] = {std::vector<int>(256, 0), std::vector<int>(256, 0)};
      int distinct[2] = {0, 0};
      for (int k = 0; k < 2048; ++k) {
        const int w = k / 1024, v = h[k];
        if (v >= 0 && v < 256 && !used[w][v]++) ++distinct[w];
        lo[w] = v < lo[w] ? v : lo[w];
        hi[w] = v > hi[w] ? v : hi[w];
      }
      int overlap = 0;
      for (int v = 0; v < 256; ++v) overlap += used[0][v] && used[1][v];
      printf("  graph replay: apply node on %d SMs, patch node on %d SMs, shared SMs %d\n", distinct[0], distinct[1], overlap);
    } else {
      printf("  graph capture over green streams: %s\n", cudaGetErrorString(ce));
      cudaGetLastError();
    }
  }
  return 0;
}
