// wax_dst.cuh -- strided spatial axes of the fused solve, in place on the
// blocked W, moved by the TMA unit in both directions.
//
// The blocked W (fast_kernels.cuh, kTBL = 8 levels per block) is
//   W[k1][level tile][k2 .. kd][8 levels]
// so along any spatial axis but the last, the elements of one "line"
// (fixed other indices and level) sit at a constant stride, and the lines
// that differ only in the faster indices form a contiguous run between two
// consecutive elements. Every such axis is a 3D view
//   {Li lines (contiguous), m elements (stride As), No outer blocks (stride Os)}
// whose strides are all multiples of 64 B, which is what a TMA tensor map
// needs (the level-major y, with a 511-double row, is not). k_dst_wax
// transforms LW adjacent lines x m elements per tile:
//   TMA tensor load (box LW x 256 rows, one or more per tile) into one of
//   NBUF shared-memory buffers, completion on an mbarrier;
//   half-length real DST-I in place (the k_dst_cols3 algorithm: pre-step
//   u_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2, one N-point complex
//   FFT per line pair, even outputs -Im U_k, odd outputs a prefix sum);
//   TMA tensor store of the tile back to the same place.
// One persistent CTA per SM keeps NBUF - 1 tile loads in flight while it
// transforms the current tile, and its stores drain asynchronously: no
// thread spends instructions or registers on moving the tile.
// Because the DSTs along different axes commute, the solve runs these
// passes on W before the contiguous-axis pass k_dst_blk2 (W -> y).
// Reference: the two DSTs of space.py:163-177 per level (pint.py:94-96).
#pragma once
#include <cuda.h>
#include "static_fft.cuh"

namespace bhcp {
namespace wax {

using namespace sfft;

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                          unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(su32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store3(const CUtensorMap* tm, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(tm), "r"(c0),
               "r"(c1), "r"(c2), "r"(su32(src))
               : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}

// S sequences (LW = 2S lines, LW * 8 B per row chunk), T threads, NBUF tile
// buffers of N * S complex slots (row e of the tile in slot e; the rows a box
// covers past m are zero-filled by the TMA unit and never read), first radix R1.
template <int N_, int S_, int T_, int NBUF_, int MINB_, int R1_, int R2_, int R3_>
struct CfgWX {
  static constexpr int N = N_, S = S_, T = T_, NBUF = NBUF_, MINB = MINB_, R1 = R1_;
  template <class Lay> using F = Fft<N_, S_, T_, Lay, R1_, R2_, R3_>;
};
// Measured on c2 (N = 512): 128 B rows beat 64 B rows (0.53 vs 0.73-0.85 ms);
// N = 512 now runs the warp-per-line-pair k_dst_wax2 (wax2_dst.cuh, 0.45 ms),
// N = 1024 (c3) the y-side k_dst_cols3 (64 B rows here: 7.45 vs 6.5 ms).
// N = 256 (c4): 32-line tiles (256 B rows), 17.8 ms per axis vs 20-22 ms.
template <int N> struct PlanWX;
// c4, per pass: 256 threads (156 registers, no spills) 14.9-15.2 ms; 512 threads
// (106 registers) 16.6-16.9; 128 / 384 / 1024 threads 16.8 / 17.3 / 22.8;
// 16-line tiles at 2 CTAs per SM 17.4-18.6
template <> struct PlanWX<256> : CfgWX<256, 16, 256, 3, 1, 4, 8, 8> {};

constexpr int kBoxRows = 256;   // TMA box height (<= 256)

template <class P> constexpr size_t smem_bytes() {
  constexpr int N = P::N;
  return sizeof(double2) * (size_t)P::NBUF * N * P::S + sizeof(double) * (N + 2 * (P::T / 32) * P::S) +
         sizeof(unsigned long long) * P::NBUF + 128;
}

struct ArgsWX {
  const double2* tw;   // exp(-2 pi i k / N)
  const double* sn;    // sin(pi j / N)
  double scale;        // sqrt(2 / N)
  int lchunks;         // ceil(Li / LW): tiles per outer block
  int ntiles;          // lchunks * No
  // padding levels of the last level tile (W holds NT * 8 >= nlev levels;
  // pass A leaves the padding unwritten). A padding line shares its complex
  // FFT with a valid line, so it is zeroed after the load:
  int vlast;           // valid levels in level tile NT - 1 (8: no padding)
  int nt;              // NT
  int llast;           // axis 0: first line of level tile NT - 1; else -1 (level tile = outer % NT)
};

template <class P>
__global__ void __launch_bounds__(P::T, P::MINB) k_dst_wax(const __grid_constant__ CUtensorMap tm, ArgsWX a) {
  constexpr int N = P::N;
  constexpr int S = P::S, T = P::T, NBUF = P::NBUF, LW = 2 * S;
  constexpr int NW = T / 32;
  constexpr int KK = 32 / S;        // k values per warp step
  constexpr int KW = (N / 2) / NW;  // k values per warp
  constexpr int STEPS = KW / KK;
  constexpr int NBOX = (N + kBoxRows - 1) / kBoxRows;
  constexpr int SLOTS = N;
  constexpr unsigned TILE_BYTES = (unsigned)(NBOX * kBoxRows * LW * sizeof(double));
  static_assert(STEPS >= 1 && KW % KK == 0, "post-processing shape");
  static_assert(NBOX * kBoxRows == N, "boxes cover the slots exactly");
  using Lay = Interleaved<S>;
  extern __shared__ __align__(128) double2 smem[];
  double* sn = reinterpret_cast<double*>(smem + NBUF * SLOTS * S);
  double* tot = sn + N;   // [NW warps][S q][2 lines]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(tot + 2 * NW * S);
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
    for (int b = 0; b < NBUF; ++b) mbar_init(full + b, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  // tile -> (outer block o, line chunk c); row e lands in slot e
  auto load = [&](int tile, int b) {
    const int o = tile / a.lchunks, c = tile - o * a.lchunks;
    double2* dst = smem + b * SLOTS * S;
    mbar_expect(full + b, TILE_BYTES);
#pragma unroll
    for (int x = 0; x < NBOX; ++x) tma_load3(dst + x * kBoxRows * S, &tm, c * LW, x * kBoxRows, o, full + b);
  };
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NBUF; ++i) {
      const int tile = blockIdx.x + i * G;
      if (tile < a.ntiles) load(tile, i);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane % S, kk = lane / S;
  int it = 0;
  for (int tile = blockIdx.x; tile < a.ntiles; tile += G, ++it) {
    const int b = it % NBUF;
    double2* buf = smem + b * SLOTS * S;
    mbar_wait(full + b, (unsigned)((it / NBUF) & 1));
    if (a.vlast < 8) {
      // does this tile hold lines of the last level tile? (uniform across the CTA)
      const int o = tile / a.lchunks, c = tile - o * a.lchunks;
      const int l0 = c * LW;
      const bool last_lo = a.llast >= 0 ? l0 >= a.llast : (o % a.nt == a.nt - 1);
      const bool last_hi = a.llast >= 0 ? l0 + LW - 1 >= a.llast : last_lo;
      if (last_lo || last_hi) {
        double* bd = reinterpret_cast<double*>(buf);
        for (int i = threadIdx.x; i < N * LW; i += T) {
          const int l = i % LW;
          const bool last = a.llast >= 0 ? l0 + l >= a.llast : last_lo;
          if (last && (l & 7) >= a.vlast) bd[i] = 0.0;
        }
        __syncthreads();
      }
    }
    auto gen = [&](int qg, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      const double2 p = buf[Lay::addr(qg, j - 1)];       // x_j (lines 2q, 2q+1), slot j-1
      const double2 r = buf[Lay::addr(qg, N - j - 1)];   // x_{N-j}
      const double s = sn[j];
      return make_double2(fma(s, p.x + r.x, 0.5 * (p.x - r.x)), fma(s, p.y + r.y, 0.5 * (p.y - r.y)));
    };
    using Ff = typename P::template F<Lay>;
    Stage<N, S, T, Lay, P::R1, 1>::first_inplace(buf, gen);
    // Every thread is past the previous tile (barriers inside the first
    // stage): once its store has read the buffer, refill that buffer.
    if (threadIdx.x == 0 && it >= 1) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      const int nt = tile + (NBUF - 1) * G;
      if (nt < a.ntiles) load(nt, (it - 1) % NBUF);
    }
    auto sink = [&](int qs, int idx, double2 X) { buf[Lay::addr(qs, idx)] = X; };
    FftTail<Ff>::run(buf, a.tw, sink);
    __syncthreads();
    // post-processing: warp w covers k in [w*KW, (w+1)*KW), lane (q, kk)
    const double2 U0 = buf[Lay::addr(q, 0)];
    double ca = 0.0, cb = 0.0;
    double oa[STEPS], ob[STEPS], ea[STEPS], eb[STEPS];
#pragma unroll
    for (int u = 0; u < STEPS; ++u) {
      const int k = warp * KW + u * KK + kk;
      const double2 A = buf[Lay::addr(q, k)];
      const double2 Bv = buf[Lay::addr(q, (N - k) & (N - 1))];
      double ia = 0.5 * (A.x + Bv.x), ib = 0.5 * (A.y + Bv.y);
      ea[u] = -0.5 * (A.y - Bv.y);
      eb[u] = 0.5 * (A.x - Bv.x);
#pragma unroll
      for (int off = S; off < 32; off <<= 1) {
        const double va = __shfl_up_sync(0xffffffffu, ia, off);
        const double vb = __shfl_up_sync(0xffffffffu, ib, off);
        if (lane >= off) { ia += va; ib += vb; }
      }
      oa[u] = ca + ia;
      ob[u] = cb + ib;
      ca += __shfl_sync(0xffffffffu, ia, q + 32 - S);
      cb += __shfl_sync(0xffffffffu, ib, q + 32 - S);
    }
    if (kk == 0) { tot[(warp * S + q) * 2] = ca; tot[(warp * S + q) * 2 + 1] = cb; }
    __syncthreads();   // all U reads done; warp totals visible
    double pa = 0.0, pb = 0.0;
    for (int w = 0; w < warp; ++w) { pa += tot[(w * S + q) * 2]; pb += tot[(w * S + q) * 2 + 1]; }
    const double ha = 0.5 * U0.x, hb = 0.5 * U0.y;
    // output e lands in slot e (e = 0..m-1)
#pragma unroll
    for (int u = 0; u < STEPS; ++u) {
      const int k = warp * KW + u * KK + kk;
      if (k >= 1) buf[Lay::addr(q, 2 * k - 1)] = make_double2(a.scale * ea[u], a.scale * eb[u]);
      buf[Lay::addr(q, 2 * k)] = make_double2(a.scale * ((pa + oa[u]) - ha), a.scale * ((pb + ob[u]) - hb));
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int o = tile / a.lchunks, c = tile - o * a.lchunks;
#pragma unroll
      for (int x = 0; x < NBOX; ++x) tma_store3(&tm, c * LW, x * kBoxRows, o, buf + x * kBoxRows * S);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

}  // namespace wax
}  // namespace bhcp
