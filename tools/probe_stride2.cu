// Microbenchmark: in-place read-modify-write of column blocks of a level-major
// (levels, 511, 511) fp64 array, staged through shared memory with cp.async
// (all loads of a tile in flight), for column-block widths W = 8..64 doubles;
// plus the contiguous-row equivalent. Bounds the strided DST pass.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int M = 511;
template <int W>
__global__ void blk_rw(double* a, int levels, int nblk) {
  extern __shared__ double sm[];
  const int ntiles = levels * nblk;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int lev = t / nblk, cb = t - lev * nblk;
    double* base = a + (long long)lev * M * M + cb * W;
    const int wv = min(W, M - cb * W);
    __syncthreads();
    for (int i = threadIdx.x; i < M * W; i += blockDim.x) {
      const int r = i / W, c = i - r * W;
      if (c < wv) {
        unsigned s = (unsigned)__cvta_generic_to_shared(sm + i);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(base + (long long)r * M + c));
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::);
    __syncthreads();
    for (int i = threadIdx.x; i < M * W; i += blockDim.x) {
      const int r = i / W, c = i - r * W;
      if (c < wv) base[(long long)r * M + c] = sm[i] * 1.0000001;
    }
  }
}
__global__ void __launch_bounds__(512) rows_rw(double* a, long long n, int chunk) {
  extern __shared__ double sm[];
  const long long ntiles = (n + chunk - 1) / chunk;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    double* base = a + t * chunk;
    const int cv = (int)min((long long)chunk, n - t * chunk);
    __syncthreads();
    for (int i = threadIdx.x; i < cv; i += blockDim.x) {
      unsigned s = (unsigned)__cvta_generic_to_shared(sm + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(base + i));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_all;\n" ::);
    __syncthreads();
    for (int i = threadIdx.x; i < cv; i += blockDim.x) base[i] = sm[i] * 1.0000001;
  }
}
int main() {
  const int levels = 513;
  const long long n = (long long)levels * M * M;
  double* a;
  cudaMalloc(&a, n * 8);
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  int nsm = 148;
#define RUNB(WW)                                                                                           \
  {                                                                                                        \
    const int nblk = (M + WW - 1) / WW;                                                                    \
    const size_t smb = (size_t)M * WW * 8;                                                                 \
    cudaFuncSetAttribute(blk_rw<WW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);               \
    int per = 0;                                                                                           \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, blk_rw<WW>, 512, smb);                             \
    for (int rep = 0; rep < 3; ++rep) {                                                                    \
      cudaEventRecord(e0);                                                                                 \
      blk_rw<WW><<<nsm * per, 512, smb>>>(a, levels, nblk);                                                \
      cudaEventRecord(e1);                                                                                 \
      cudaEventSynchronize(e1);                                                                            \
      cudaEventElapsedTime(&ms, e0, e1);                                                                   \
      if (rep) printf("colblock W=%3d (%4d B chunks, %d CTA/SM): %.3f ms %.0f GB/s\n", WW, WW * 8, per, ms, \
                      16.0 * n / ms / 1e6);                                                                \
    }                                                                                                      \
  }
  RUNB(8) RUNB(16) RUNB(24) RUNB(32) RUNB(48)
  // emulate the k_dst_blk2 MODE 1 shape: 256 threads, smem forcing 3 CTAs/SM
  for (int thr : {256, 512}) for (size_t smb : {(size_t)73 * 1024, (size_t)110 * 1024, (size_t)48 * 1024}) {
    const int nblk = (M + 7) / 8;
    cudaFuncSetAttribute(blk_rw<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, blk_rw<8>, thr, smb);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      blk_rw<8><<<nsm * per, thr, smb>>>(a, levels, nblk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("colblock W=8 T=%d smem=%zuK (%d CTA/SM): %.3f ms %.0f GB/s\n", thr, smb / 1024, per, ms, 16.0 * n / ms / 1e6);
    }
  }
  for (int chunk : {4096, 8192, 16384}) {
    const size_t smb = (size_t)chunk * 8;
    cudaFuncSetAttribute(rows_rw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, rows_rw, 512, smb);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      rows_rw<<<nsm * per, 512, smb>>>(a, n, chunk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("contig chunk %6d doubles (%d CTA/SM): %.3f ms %.0f GB/s\n", chunk, per, ms, 16.0 * n / ms / 1e6);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
