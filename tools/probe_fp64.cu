// Microbenchmark: FP64 DFMA throughput and device attributes on the B200 box.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int smemOptin; cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  int smemSM; cudaDeviceGetAttribute(&smemSM, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("name=%s sms=%d smem_optin=%d smem_per_sm=%d l2=%d clock_khz=%d regs_per_sm=%d\n", p.name,
         p.multiProcessorCount, smemOptin, smemSM, p.l2CacheSize, clk, p.regsPerMultiprocessor);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4000;
  for (int rep = 0; rep < 3; ++rep) {
    dfma_loop<<<148 * 8, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_loop<<<148 * 8, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 148 * 8 * 256 * (double)iters * 16 * 8;
    printf("dfma: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  size_t n = (size_t)1 << 27;  // 4 GiB of double4
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32); cudaMemset(a, 0, n * 32);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_k<<<148 * 16, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.3f ms  %.1f GB/s\n", ms, 2.0 * n * 32 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
