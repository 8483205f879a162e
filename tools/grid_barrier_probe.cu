// Microbenchmark: cost of one grid-wide barrier in a cooperative launch on this
// GPU (sense-reversal counter barrier with and without __nanosleep backoff, and
// cooperative_groups grid sync), for the persistent PCG kernel's design.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Bar { unsigned count, gen; };

template <int SLEEP>
__global__ void bar_kernel(Bar* b, int n, double* acc) {
  for (int k = 0; k < n; ++k) {
    __syncthreads();
    if (threadIdx.x == 0) {
      volatile unsigned* gen = &b->gen;
      const unsigned g = *gen;
      __threadfence();
      if (atomicAdd(&b->count, 1u) == gridDim.x - 1) {
        b->count = 0;
        __threadfence();
        atomicAdd(&b->gen, 1u);
      } else {
        while (*gen == g) if (SLEEP) __nanosleep(SLEEP);
      }
      __threadfence();
    }
    __syncthreads();
    if (acc && threadIdx.x == 0) atomicAdd(acc + (k & 1), 1.0);  // a block reduction's atomic per phase
  }
}

__global__ void cg_kernel(int n) {
  cg::grid_group g = cg::this_grid();
  for (int k = 0; k < n; ++k) g.sync();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Bar* b;
  double* acc;
  cudaMalloc(&b, sizeof(Bar));
  cudaMalloc(&acc, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 2000;
  for (int per_sm : {1, 2}) {
    for (int threads : {256, 512}) {
      dim3 grid(sms * per_sm), block(threads);
      auto run = [&](const void* fn, void** args, const char* name) {
        cudaMemset(b, 0, sizeof(Bar));
        cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(fn, grid, block, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-28s grid %4d x %3d: %.3f us per barrier (%s)\n", name, grid.x, threads, 1e3 * ms / n,
               cudaGetErrorString(cudaGetLastError()));
      };
      int nn = n;
      double* nul = nullptr;
      void* a0[] = {&b, &nn, &nul};
      void* a1[] = {&b, &nn, &acc};
      void* a2[] = {&nn};
      run((const void*)bar_kernel<0>, a0, "counter, spin");
      run((const void*)bar_kernel<32>, a0, "counter, nanosleep(32)");
      run((const void*)bar_kernel<0>, a1, "counter, spin + 1 atomic");
      run((const void*)cg_kernel, a2, "cooperative_groups sync");
    }
  }
  return 0;
}
