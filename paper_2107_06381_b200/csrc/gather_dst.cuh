// gather_dst.cuh -- first level pass of the fused solve (2D / 3D).
//
// The modes kernels store W blocked: 8 consecutive levels of every mode of a
// k1 plane form one contiguous block, so one spatial line for 8 levels is a
// single contiguous run. k_dst_blk2 stages that run with cp.async (the next
// tile is prefetched while the current one is transformed), computes the
// inverse DST-I along the last spatial axis for the 8 levels with the
// half-length real-DST algorithm and writes the rows of the level-major
// trajectory y.
#pragma once
#include "static_fft.cuh"

namespace bhcp {
namespace gdst {

using namespace sfft;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Levels per contiguous W block (fastk::kTBL).
constexpr int kTB = 8;

// ---------------------------------------------------------------------------
// k_dst_blk2: first level pass from the blocked W. DST-I of two real lines
// a, b (length N-1) through ONE complex FFT of length N (not the 2N-point
// odd extension), the classic real-sine algorithm:
//   u_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2,  j = 0..N-1
//   U = FFT_N(u^a + i u^b);  U^a_k = (U_k + conj U_{N-k})/2, U^b_k = (U_k - conj U_{N-k})/(2i)
//   S_{2k}   = -Im U_k                       (k = 1 .. N/2-1)
//   S_{2k+1} = sum_{i<=k} Re U_i - Re U_0/2   (k = 0 .. N/2-1, prefix sum)
// since Re U_k = S_{2k+1} - S_{2k-1} and -Im U_k = S_{2k}. A per-warp pass
// (one warp per output line) splits U^a/U^b, runs the prefix sum with warp
// shuffles and writes the row of y directly.
template <int N> struct PlanB2;
template <> struct PlanB2<256> { static constexpr int T = 256, R1 = 4; template <class Lay> using F = Fft<256, 4, T, Lay, 4, 8, 8>; };
template <> struct PlanB2<512> { static constexpr int T = 256, R1 = 8; template <class Lay> using F = Fft<512, 4, T, Lay, 8, 8, 8>; };
template <> struct PlanB2<1024> { static constexpr int T = 256, R1 = 16; template <class Lay> using F = Fft<1024, 4, T, Lay, 16, 8, 8>; };

struct ArgsB2 {
  const double* in;
  double* out;
  const double2* tw;      // exp(-2 pi i k / N)
  const double* sn;       // sin(pi j / N)
  double scale;           // sqrt(2/N)
  const long long* koff;
  long long NT, P1, idiv, P, nlev;
};

template <int N>
__global__ void __launch_bounds__(PlanB2<N>::T, 3) k_dst_blk2(ArgsB2 a) {
  constexpr int S = 4, T = PlanB2<N>::T, m = N - 1;
  constexpr int RUN = m * kTB;
  constexpr int KU = (N / 2) / 32;   // k values per lane (k = u*32 + lane)
  using Lay = Interleaved<S, PlanB2<N>::R1>;
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* stage = reinterpret_cast<double*>(smem + Lay::words(N));
  double* sn = stage + RUN;
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);
  const long long ntiles = a.P * a.NT;
  auto issue = [&](long long tile) {
    const long long o = tile / a.NT, tt = tile - o * a.NT;
    const long long k1 = o / a.idiv, r2 = o - k1 * a.idiv;
    const long long kb = a.koff ? __ldg(a.koff + k1) : k1 * a.NT * a.P1 * kTB;
    const double2* src = reinterpret_cast<const double2*>(a.in + kb + tt * a.P1 * kTB + r2 * (long long)m * kTB);
    double2* dst = reinterpret_cast<double2*>(stage);
    for (int i = threadIdx.x; i < RUN / 2; i += T) {
      const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + i));
    }
    cp_async_commit();
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long tile = blockIdx.x;
  if (tile < ntiles) issue(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const long long o = tile / a.NT, tt = tile - o * a.NT;
    cp_async_wait_all();
    __syncthreads();
    const long long tvalid = a.nlev - tt * kTB;
    auto gen = [&](int q, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      double2 p = *reinterpret_cast<const double2*>(stage + (j - 1) * kTB + 2 * q);      // x_j
      double2 r = *reinterpret_cast<const double2*>(stage + (N - j - 1) * kTB + 2 * q);  // x_{N-j}
      if (2 * q >= tvalid) { p.x = 0.0; r.x = 0.0; }
      if (2 * q + 1 >= tvalid) { p.y = 0.0; r.y = 0.0; }
      const double s = sn[j];
      return make_double2(fma(s, p.x + r.x, 0.5 * (p.x - r.x)), fma(s, p.y + r.y, 0.5 * (p.y - r.y)));
    };
    using Ff = typename PlanB2<N>::template F<Lay>;
    Stage<N, S, T, Lay, PlanB2<N>::R1, 1>::first(buf, gen);
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    FftTail<Ff>::run(buf, a.tw, sink);
    __syncthreads();
    // one warp per output line; k = u*32 + lane, running prefix across u
    for (int li = warp; li < kTB; li += T / 32) {
      const long long t = tt * kTB + li;
      if (t >= a.nlev) continue;
      const int q = li >> 1;
      const bool isb = li & 1;
      double* __restrict__ dst = a.out + (t * a.P + o) * m;
      double carry = 0.0, c0 = 0.0;
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = u * 32 + lane;
        const double2 A = buf[Lay::addr(q, k)];
        const double2 Bv = buf[Lay::addr(q, (N - k) & (N - 1))];
        double ur, ui;
        if (!isb) { ur = 0.5 * (A.x + Bv.x); ui = 0.5 * (A.y - Bv.y); }
        else { ur = 0.5 * (A.y + Bv.y); ui = -0.5 * (A.x - Bv.x); }
        if (u == 0) c0 = __shfl_sync(0xffffffffu, ur, 0);
        double incl = ur;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double v = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += v;
        }
        const double odd = carry + incl - 0.5 * c0;       // S_{2k+1}
        carry += __shfl_sync(0xffffffffu, incl, 31);
        if (k >= 1) dst[2 * k - 1] = a.scale * (-ui);     // S_{2k}
        dst[2 * k] = a.scale * odd;
      }
    }
  }
}

template <int N> constexpr size_t smemB2_bytes() {
  using Lay = Interleaved<4, PlanB2<N>::R1>;
  return sizeof(double2) * Lay::words(N) + sizeof(double) * ((N - 1) * kTB + N);
}

}  // namespace gdst
}  // namespace bhcp
