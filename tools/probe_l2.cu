// probe_l2.cu -- how much freshly written data survives in L2 for a later read.
// Kernel k_write stores S bytes of Y (optionally while streaming R bytes of a
// second buffer with evict-first loads); k_read then reads Y back. Run under
//   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ./probe_l2
// and compare k_read's DRAM reads with S (0 = all hits).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_l2 tools/probe_l2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pol_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

__global__ void k_write(double* y, long long n, const double* w, long long nw, double* sink) {
  const unsigned long long pol = pol_first();
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = j; i < n; i += stride) {
    y[i] = (double)i;
    if (nw) {
      double v;
      const double* p = w + (i % nw);
      asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
      acc += v;
    }
  }
  if (acc == 12345.0) sink[0] = acc;
}

__global__ void k_read(const double* y, long long n, double* sink) {
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) acc += y[i];
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const long long maxn = 160ll << 20;   // 160 MB of doubles per buffer
  double *y, *w, *sink;
  cudaMalloc(&y, maxn);
  cudaMalloc(&w, 4ll << 30);
  cudaMalloc(&sink, 64);
  cudaMemset(w, 0, 4ll << 30);
  const int mbs[] = {16, 32, 48, 64, 80, 96, 112};
  for (int stream_w = 0; stream_w < 2; ++stream_w) {
    for (int mb : mbs) {
      const long long n = ((long long)mb << 20) / 8;
      // flush: stream 512 MB through L2
      k_read<<<148 * 4, 512>>>(w + (1ll << 28), (512ll << 20) / 8, sink);
      k_write<<<148 * 4, 512>>>(y, n, w, stream_w ? n : 0, sink);
      k_read<<<148 * 4, 512>>>(y, n, sink);
      cudaDeviceSynchronize();
      printf("case stream_w=%d size=%d MB done\n", stream_w, mb);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
