// Microbenchmark: bandwidth of "tile gather" access patterns on B200.
// Reads a (rows x cols) row-major fp64 matrix in tiles of W consecutive
// columns x all rows (chunks of 8W bytes at row stride), writes them back in
// place -- the access pattern of the strided DST passes.
#include <cstdio>
#include <cuda_runtime.h>
template <int W>
__global__ void tile_rw(double* a, long long rows, long long cols, int ntile_c) {
  const long long ntiles = (long long)ntile_c;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long c0 = t * W;
    for (long long i = threadIdx.x; i < rows * W; i += blockDim.x) {
      const long long r = i / W, c = c0 + (i % W);
      if (c < cols) a[r * cols + c] = a[r * cols + c] * 1.0000001;
    }
  }
}
__global__ void contig_rw(double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = a[i] * 1.0000001;
}
int main() {
  const long long rows = 511, cols = 513LL * 511;  // like y (levels*511 lines) transposed roles
  const long long n = rows * cols;                 // 134M doubles
  double* a; cudaMalloc(&a, n * 8); cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); contig_rw<<<148 * 8, 256>>>(a, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); printf("contig rw: %.3f ms %.0f GB/s\n", ms, 16.0 * n / ms / 1e6);
  }
#define RUN(WW)                                                                                   \
  for (int rep = 0; rep < 2; ++rep) {                                                             \
    int nt = (int)((cols + WW - 1) / WW);                                                         \
    cudaEventRecord(e0); tile_rw<WW><<<148 * 4, 256>>>(a, rows, cols, nt); cudaEventRecord(e1);   \
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);                                  \
    printf("tile W=%3d (%4d B chunks): %.3f ms %.0f GB/s\n", WW, WW * 8, ms, 16.0 * n / ms / 1e6);  \
  }
  RUN(4) RUN(8) RUN(16) RUN(32) RUN(64)
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
