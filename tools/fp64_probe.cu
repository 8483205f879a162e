// Microbenchmark: DFMA latency (dependent chain) and throughput (independent
// chains) per SM on this GPU; DMMA.8x8x4 throughput. Sizes FP64 kernels.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, int n, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = (double)(t1 - t0) / n; }
}
template <int C>
__global__ void thr(double* out, int n, double a, double b) {
  double x[C];
  for (int c = 0; c < C; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
  for (int c = 0; c < C; ++c) s += x[c];
  if (s == 1.2345) out[0] = s;
}
__global__ void dmma(double* out, int n) {
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
int main() {
  double* out; cudaMalloc(&out, 64);
  double h[2];
  lat<<<1, 32>>>(out, 1 << 16, 1.0000001, 1e-9); cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cyc\n", h[1]);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n = 1 << 14; float ms;
  for (int warps : {4, 8, 16, 32}) {
    thr<8><<<148, warps * 32>>>(out, n, 1.0000001, 1e-9);
    cudaEventRecord(e0); thr<8><<<148, warps * 32>>>(out, n, 1.0000001, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA throughput, %2d warps/SM x 8 chains: %.2f TFLOP/s\n", warps, 2.0 * 148 * warps * 32 * 8 * (double)n / (ms / 1e3) / 1e12);
  }
  for (int warps : {4, 8, 16}) {
    dmma<<<148, warps * 32>>>(out, n);
    cudaEventRecord(e0); dmma<<<148, warps * 32>>>(out, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA.884 throughput, %2d warps/SM x 4 chains: %.2f TFLOP/s\n", warps, 512.0 * 4 * 148 * warps * (double)n / (ms / 1e3) / 1e12);
  }
  return 0;
}
