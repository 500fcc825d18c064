// gather_dst.cuh -- staged, persistent DST-I passes over strided real lines.
//
// Both level-pass kernels of the fused solve read lines whose elements are
// strided in memory but whose *neighbouring lines* are contiguous:
//   MODE 0 (first level pass): W is mode-major (each mode's time series is
//     contiguous, written that way by the modes kernel), so for a fixed
//     spatial line the consecutive levels t are adjacent. The kernel reads a
//     tile (one spatial line o, 2S consecutive levels) and writes the DST
//     along the last spatial axis into the level-major trajectory y.
//   MODE 1 (remaining axes, in place on y): element e of line (o, i) at
//     o*os + e*es + i with consecutive inner lines i adjacent.
// A tile is 2S real lines = S complex FFT sequences of length L = 2N (odd
// extension, two real lines per complex sequence). Its input is prefetched
// into a shared staging buffer with cp.async while the previous tile's FFT
// runs (one tile in flight per CTA), so the global-load latency is off the
// FFT's critical path; the result goes through shared memory and is stored
// with the lines' contiguous axis across threads.
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

template <int L> struct Plan;
template <> struct Plan<512> { static constexpr int S = 8, T = 256, R1 = 8; template <class Lay> using F = Fft<512, S, T, Lay, 8, 8, 8>; };
template <> struct Plan<1024> { static constexpr int S = 4, T = 256, R1 = 16; template <class Lay> using F = Fft<1024, S, T, Lay, 16, 8, 8>; };
template <> struct Plan<2048> { static constexpr int S = 2, T = 256, R1 = 16; template <class Lay> using F = Fft<2048, S, T, Lay, 16, 16, 8>; };
template <> struct Plan<8192> { static constexpr int S = 1, T = 512, R1 = 16; template <class Lay> using F = Fft<8192, S, T, Lay, 16, 16, 8, 4>; };

struct Args {
  const double* in;
  double* out;
  const double2* tw;
  double f;          // sqrt(2/N)/2
  int m;             // line length N-1
  long long ni;      // inner (contiguous) line count
  long long no;      // outer line count
  // MODE 0: input (o, e, i) at koff[o / idiv] + (o % idiv) * m * Lin + e * Lin + i
  //         (koff null: koff[k1] = k1 * idiv * m * Lin, i.e. one mode-major block)
  //         output level-major: ((i + ibase) * P + o) * m + e
  const long long* koff;
  long long idiv;    // m^(d-2) (1 in 2D; lines per k1 value)
  long long Lin;     // levels per mode in the input block (element stride)
  long long P;       // lines per level (m^(d-1))
  long long ibase;   // level offset of inner index 0 in the output
  int ishift;        // 1 if inner index 0 is an odd global level: tiles start at -1 so
                     // level pairs (2u, 2u+1) match the single-GPU solve bit for bit
  // MODE 1: input/output (o, e, i) at o * os + e * es + i
  long long os, es;
};

template <int L, int MODE>
struct Geo {
  // element (o, e, i) of the input at in_base(o) + e * in_es + i
  static __device__ __forceinline__ long long in_base(const Args& a, long long o) {
    if (MODE == 0) {
      const long long k1 = o / a.idiv, r2 = o - k1 * a.idiv;
      const long long base = a.koff ? __ldg(a.koff + k1) : k1 * a.idiv * (long long)a.m * a.Lin;
      return base + r2 * (long long)a.m * a.Lin;
    }
    return o * a.os;
  }
  static __device__ __forceinline__ long long in_es(const Args& a) { return MODE == 0 ? a.Lin : a.es; }
};

// staging row stride (doubles) for one element e of the 2S lines: odd -> conflict-light
template <int S> struct Stg { static constexpr int W = 2 * S + 1; };

template <int L, int MODE>
__global__ void __launch_bounds__(Plan<L>::T, (L <= 2048 ? 2 : 1)) k_dst_gather(Args a) {
  constexpr int S = Plan<L>::S, T = Plan<L>::T, N = L / 2;
  constexpr int SW = Stg<S>::W;
  using Lay = SeqMajorPad<L, Plan<L>::R1>;
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* stage = reinterpret_cast<double*>(smem + Lay::words(S));
  const int m = a.m;
  const int shift = MODE == 0 ? a.ishift : 0;
  const long long ntile_i = (a.ni + shift + 2 * S - 1) / (2 * S);
  const long long ntiles = ntile_i * a.no;

  const long long es = Geo<L, MODE>::in_es(a);
  auto issue = [&](long long tile) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * (2 * S) - shift;
    const double* src = a.in + Geo<L, MODE>::in_base(a, o) + i0;
    // lane li of every element row e; rows beyond the valid level range are zero
    const int li = threadIdx.x % (2 * S);
    const bool ok = (i0 + li >= 0) && (i0 + li < a.ni);
    for (int e = threadIdx.x / (2 * S); e < m; e += T / (2 * S)) {
      double* dst = stage + e * SW + li;
      if (ok) cp_async8(dst, src + e * es + li);
      else *dst = 0.0;
    }
    cp_async_commit();
  };

  long long tile = blockIdx.x;
  if (tile < ntiles) issue(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * (2 * S) - shift;
    cp_async_wait_all();
    __syncthreads();
    // first stage reads the staged lines (odd extension, two real lines per sequence)
    auto gen = [&](int q, int idx) -> double2 {
      if (idx == 0 || idx == N) return make_double2(0.0, 0.0);
      const bool neg = idx > N;
      const int e = neg ? (L - idx - 1) : (idx - 1);
      const double* p = stage + e * SW + 2 * q;
      const double2 x = make_double2(p[0], p[1]);
      return neg ? make_double2(-x.x, -x.y) : x;
    };
    using Fft = typename Plan<L>::template F<Lay>;
    Stage<L, S, T, Lay, Plan<L>::R1, 1>::first(buf, gen);
    // staging buffer is free: prefetch the next tile behind the remaining stages
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    FftTail<Fft>::run(buf, a.tw, sink);
    __syncthreads();
    // store: DST coefficient e of real line li = S_{e+1}; contiguous axis across threads
    if (MODE == 0) {
      // line (level i0+li, spatial line o) is contiguous in the level-major output
      for (int idx = threadIdx.x; idx < 2 * S * m; idx += T) {
        const int li = idx / m, e = idx - li * m;
        const long long i = i0 + li;
        if (i < 0 || i >= a.ni) continue;
        const double2 X = buf[Lay::addr(li >> 1, e + 1)];
        const double c = (li & 1) ? a.f * X.x : -a.f * X.y;
        a.out[((i + a.ibase) * a.P + o) * m + e] = c;
      }
    } else {
      double* dst = a.out + o * a.os + i0;
      const int li = threadIdx.x % (2 * S);
      const bool ok = i0 + li < a.ni;
      const double2* col = buf + Lay::addr(li >> 1, 0);
      for (int e = threadIdx.x / (2 * S); e < m; e += T / (2 * S)) {
        if (!ok) continue;
        const double2 X = col[(e + 1) + (e + 1) / Plan<L>::R1];
        const double c = (li & 1) ? a.f * X.x : -a.f * X.y;
        dst[e * a.es + li] = c;
      }
    }
  }
}

template <int L> constexpr size_t smem_bytes() {
  using Lay = SeqMajorPad<L, Plan<L>::R1>;
  return sizeof(double2) * Lay::words(Plan<L>::S) + sizeof(double) * (L / 2 - 1) * Stg<Plan<L>::S>::W;
}

}  // namespace gdst
}  // namespace bhcp
