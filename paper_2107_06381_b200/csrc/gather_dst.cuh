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
  constexpr int m = N - 1;
  const int shift = MODE == 0 ? a.ishift : 0;
  const long long ntile_i = (a.ni + shift + 2 * S - 1) / (2 * S);
  const long long ntiles = ntile_i * a.no;

  const long long es = Geo<L, MODE>::in_es(a);
  // thread -> (lane li of the 2S lines, first element row); pointer walks the rows
  constexpr int ROWS = T / (2 * S);
  const int my_li = threadIdx.x % (2 * S);
  const int my_e0 = threadIdx.x / (2 * S);
  auto issue = [&](long long tile) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * (2 * S) - shift;
    const bool ok = (i0 + my_li >= 0) && (i0 + my_li < a.ni);
    const double* src = a.in + Geo<L, MODE>::in_base(a, o) + i0 + my_li + my_e0 * es;
    const long long step = ROWS * es;
    double* dst = stage + my_e0 * SW + my_li;
    for (int e = my_e0; e < m; e += ROWS) {
      if (ok) cp_async8(dst, src);
      else *dst = 0.0;
      src += step;
      dst += ROWS * SW;
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
      // one warp per output line (level i0+li, spatial line o): contiguous run of m
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int li = warp; li < 2 * S; li += T / 32) {
        const long long i = i0 + li;
        if (i < 0 || i >= a.ni) continue;
        double* __restrict__ dst = a.out + ((i + a.ibase) * a.P + o) * m;
        const double2* col = buf + Lay::addr(li >> 1, 0);
        const bool odd = li & 1;
        for (int e = lane; e < m; e += 32) {
          const double2 X = col[(e + 1) + (e + 1) / Plan<L>::R1];
          dst[e] = odd ? a.f * X.x : -a.f * X.y;
        }
      }
    } else {
      const bool ok = i0 + my_li < a.ni;
      double* __restrict__ dst = a.out + o * a.os + i0 + my_li + my_e0 * a.es;
      const long long step = ROWS * a.es;
      const double2* col = buf + Lay::addr(my_li >> 1, 0);
      const bool odd = my_li & 1;
      if (ok) {
        for (int e = my_e0; e < m; e += ROWS) {
          const double2 X = col[(e + 1) + (e + 1) / Plan<L>::R1];
          *dst = odd ? a.f * X.x : -a.f * X.y;
          dst += step;
        }
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

namespace bhcp {
namespace gdst {

// ---------------------------------------------------------------------------
// k_dst2: the same level passes with a half-length transform.
// DST-I of two real lines a, b (length N-1) through ONE complex FFT of length
// N (instead of the 2N-point odd extension), the classic real-sine algorithm:
//   u_j = sin(pi j/N)(x_j + x_{N-j}) + (x_j - x_{N-j})/2,  j = 0..N-1
//   U = FFT_N(u^a + i u^b);  U^a_k = (U_k + conj U_{N-k})/2, U^b_k = (U_k - conj U_{N-k})/(2i)
//   S_{2k}   = -Im U_k                      (k = 1 .. N/2-1)
//   S_{2k+1} = sum_{i<=k} Re U_i - Re U_0/2  (k = 0 .. N/2-1, prefix sum)
// (C_k = Re U_k = S_{2k+1} - S_{2k-1}, D_k = -Im U_k = S_{2k}). Half the FFT
// flops and half the shared-memory traffic of the odd-extension kernel; the
// prefix sum runs as a per-lane serial scan plus a warp shuffle scan.
template <int N> struct Plan2;
template <> struct Plan2<256> { static constexpr int S = 8, T = 512, MINB = 1; template <class Lay> using F = Fft<256, S, T, Lay, 4, 8, 8>; static constexpr int R1 = 4; };
template <> struct Plan2<512> { static constexpr int S = 4, T = 256, MINB = 2; template <class Lay> using F = Fft<512, S, T, Lay, 8, 8, 8>; static constexpr int R1 = 8; };
template <> struct Plan2<1024> { static constexpr int S = 4, T = 256, MINB = 2; template <class Lay> using F = Fft<1024, S, T, Lay, 16, 8, 8>; static constexpr int R1 = 16; };
template <> struct Plan2<4096> { static constexpr int S = 1, T = 256, MINB = 2; template <class Lay> using F = Fft<4096, S, T, Lay, 16, 16, 16>; static constexpr int R1 = 16; };

struct Args2 {
  const double* in;
  double* out;
  const double2* tw;     // exp(-2 pi i k / N), k < N
  const double* sn;      // sin(pi j / N), j < N
  double scale;          // sqrt(2/N)
  long long ni, no;
  const long long* koff;
  long long idiv, Lin, P, ibase;
  int ishift;
  long long os, es;
};

template <int N, int MODE>
__global__ void __launch_bounds__(Plan2<N>::T, Plan2<N>::MINB) k_dst2(Args2 a) {
  constexpr int S = Plan2<N>::S, T = Plan2<N>::T, m = N - 1, NL = 2 * S;
  constexpr int SW = NL + 1;        // staging row stride (doubles)
  constexpr int OW = m + 2;         // output staging row stride (doubles), MODE 1
  constexpr int K = (N / 2) / 32;   // k values per lane in the scan
  static_assert(T / 32 >= NL || MODE == 0 || true, "");
  using Lay = SeqMajorPad<N, Plan2<N>::R1>;
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* stage = reinterpret_cast<double*>(smem + Lay::words(S));
  double* sn = stage + m * SW;
  double* ob = sn + N;              // MODE 1 only
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);

  const int shift = MODE == 0 ? a.ishift : 0;
  const long long ntile_i = (a.ni + shift + NL - 1) / NL;
  const long long ntiles = ntile_i * a.no;
  const long long es_in = MODE == 0 ? a.Lin : a.es;
  constexpr int ROWS = T / NL;
  const int my_li = threadIdx.x % NL;
  const int my_e0 = threadIdx.x / NL;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto in_base = [&](long long o) -> long long {
    if (MODE == 0) {
      const long long k1 = o / a.idiv, r2 = o - k1 * a.idiv;
      const long long base = a.koff ? __ldg(a.koff + k1) : k1 * a.idiv * (long long)m * a.Lin;
      return base + r2 * (long long)m * a.Lin;
    }
    return o * a.os;
  };
  auto issue = [&](long long tile) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * NL - shift;
    const bool ok = (i0 + my_li >= 0) && (i0 + my_li < a.ni);
    const double* src = a.in + in_base(o) + i0 + my_li + my_e0 * es_in;
    const long long step = ROWS * es_in;
    double* dst = stage + my_e0 * SW + my_li;
    for (int e = my_e0; e < m; e += ROWS) {
      if (ok) cp_async8(dst, src);
      else *dst = 0.0;
      src += step;
      dst += ROWS * SW;
    }
    cp_async_commit();
  };

  long long tile = blockIdx.x;
  if (tile < ntiles) issue(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * NL - shift;
    cp_async_wait_all();
    __syncthreads();
    auto gen = [&](int q, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      const double* p = stage + (j - 1) * SW + 2 * q;        // x_j
      const double* r = stage + (N - j - 1) * SW + 2 * q;    // x_{N-j}
      const double s = sn[j];
      const double pa = p[0], pb = p[1], ra = r[0], rb = r[1];
      return make_double2(fma(s, pa + ra, 0.5 * (pa - ra)), fma(s, pb + rb, 0.5 * (pb - rb)));
    };
    using F = typename Plan2<N>::template F<Lay>;
    Stage<N, S, T, Lay, Plan2<N>::R1, 1>::first(buf, gen);
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    FftTail<F>::run(buf, a.tw, sink);
    __syncthreads();
    // post-processing + prefix sum: one warp per real line
    for (int li = warp; li < NL; li += T / 32) {
      const int q = li >> 1;
      const bool isb = li & 1;
      double C[K], D[K];
      double run = 0.0;
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int k = lane * K + u;
        const double2 A = buf[Lay::addr(q, k)];
        const double2 B = buf[Lay::addr(q, (N - k) & (N - 1))];
        // U^a = (A + conj B)/2 ; U^b = (A - conj B)/(2i)
        double ur, ui;
        if (!isb) { ur = 0.5 * (A.x + B.x); ui = 0.5 * (A.y - B.y); }
        else { ur = 0.5 * (A.y + B.y); ui = -0.5 * (A.x - B.x); }
        C[u] = ur;
        D[u] = -ui;
        run += ur;
      }
      // exclusive warp scan of the lane totals
      double incl = run;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
      }
      const double c0 = __shfl_sync(0xffffffffu, C[0], 0);
      double acc = incl - run - 0.5 * c0;
      const long long i = i0 + li;
      const bool valid = i >= 0 && i < a.ni;
      if (MODE == 0) {
        double* __restrict__ dst = a.out + ((i + a.ibase) * a.P + o) * m;
#pragma unroll
        for (int u = 0; u < K; ++u) {
          const int k = lane * K + u;
          acc += C[u];
          if (valid) {
            if (k >= 1) dst[2 * k - 1] = a.scale * D[u];   // S_{2k}
            dst[2 * k] = a.scale * acc;                    // S_{2k+1}
          }
        }
      } else {
        double* row = ob + li * OW;
#pragma unroll
        for (int u = 0; u < K; ++u) {
          const int k = lane * K + u;
          acc += C[u];
          if (k >= 1) row[2 * k - 1] = a.scale * D[u];
          row[2 * k] = a.scale * acc;
        }
      }
    }
    if (MODE == 1) {
      __syncthreads();
      const bool ok = i0 + my_li < a.ni;
      double* __restrict__ dst = a.out + o * a.os + i0 + my_li + my_e0 * a.es;
      const long long step = ROWS * a.es;
      const double* row = ob + my_li * OW;
      if (ok) {
        for (int e = my_e0; e < m; e += ROWS) {
          *dst = row[e];
          dst += step;
        }
      }
    }
  }
}

template <int N> constexpr size_t smem2_bytes(int mode) {
  using Lay = SeqMajorPad<N, Plan2<N>::R1>;
  constexpr int NL = 2 * Plan2<N>::S;
  return sizeof(double2) * Lay::words(Plan2<N>::S) + sizeof(double) * ((N - 1) * (NL + 1) + N) +
         (mode == 1 ? sizeof(double) * NL * (N + 1) : 0);
}

}  // namespace gdst
}  // namespace bhcp

namespace bhcp {
namespace gdst {

// ---------------------------------------------------------------------------
// k_dst_blk: first level pass from the BLOCKED W layout.
// The modes kernel stores W in blocks of TB = 8 consecutive levels:
//   block (k1, level tile tt) = P1 x 8 doubles, mode (k1, rr) at rr*8,
// so one tile of this kernel -- one spatial line (k1, r2) for 8 levels -- is
// a single contiguous m*8*8-byte run: it is staged with 16-byte cp.async
// (coalesced, long DRAM bursts) while the previous tile is transformed.
constexpr int kTB = 8;

template <int L> struct PlanB;
template <> struct PlanB<512> { static constexpr int T = 256, R1 = 8; template <class Lay> using F = Fft<512, 4, T, Lay, 8, 8, 8>; };
template <> struct PlanB<1024> { static constexpr int T = 256, R1 = 16; template <class Lay> using F = Fft<1024, 4, T, Lay, 16, 8, 8>; };
template <> struct PlanB<2048> { static constexpr int T = 512, R1 = 16; template <class Lay> using F = Fft<2048, 4, T, Lay, 16, 16, 8>; };

struct ArgsB {
  const double* in;       // blocked W (receive buffer on a rank)
  double* out;            // level-major y (nlev, n_space)
  const double2* tw;
  double f;               // sqrt(2/N)/2
  const long long* koff;  // start of k1's first block, null: k1 * NT * P1 * TB
  long long NT;           // level tiles in this W (slab)
  long long P1;           // modes per k1 value (m^(d-1))
  long long idiv;         // m^(d-2): lines per k1 value
  long long P;            // lines per level (m^(d-1))
  long long nlev;         // valid levels
};

template <int L>
__global__ void __launch_bounds__(PlanB<L>::T, (L <= 1024 ? 2 : 1)) k_dst_blk(ArgsB a) {
  constexpr int S = 4, T = PlanB<L>::T, N = L / 2, m = N - 1;
  constexpr int RUN = m * kTB;        // doubles per tile (contiguous)
  using Lay = Interleaved<S, PlanB<L>::R1>;
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* stage = reinterpret_cast<double*>(smem + Lay::words(L));
  const long long ntiles = a.P * a.NT;
  auto src_of = [&](long long tile) -> const double* {
    const long long o = tile / a.NT, tt = tile - o * a.NT;
    const long long k1 = o / a.idiv, r2 = o - k1 * a.idiv;
    const long long kb = a.koff ? __ldg(a.koff + k1) : k1 * a.NT * a.P1 * kTB;
    return a.in + kb + tt * a.P1 * kTB + r2 * (long long)m * kTB;
  };
  auto issue = [&](long long tile) {
    const double2* src = reinterpret_cast<const double2*>(src_of(tile));
    double2* dst = reinterpret_cast<double2*>(stage);
    for (int i = threadIdx.x; i < RUN / 2; i += T) {
      const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst + i));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + i));
    }
    cp_async_commit();
  };
  long long tile = blockIdx.x;
  if (tile < ntiles) issue(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    const long long o = tile / a.NT, tt = tile - o * a.NT;
    cp_async_wait_all();
    __syncthreads();
    // staged tile: element e of level tl at stage[e*8 + tl]; sequence q = levels (2q, 2q+1).
    // Levels past nlev (padding of the last tile) are never read: they hold
    // no data and must not leak into the partner level through the FFT.
    const long long tvalid = a.nlev - tt * kTB;
    auto gen = [&](int q, int idx) -> double2 {
      if (idx == 0 || idx == N) return make_double2(0.0, 0.0);
      const bool neg = idx > N;
      const int e = neg ? (L - idx - 1) : (idx - 1);
      double2 x = *reinterpret_cast<const double2*>(stage + e * kTB + 2 * q);
      if (2 * q >= tvalid) x.x = 0.0;
      if (2 * q + 1 >= tvalid) x.y = 0.0;
      return neg ? make_double2(-x.x, -x.y) : x;
    };
    using Ff = typename PlanB<L>::template F<Lay>;
    Stage<L, S, T, Lay, PlanB<L>::R1, 1>::first(buf, gen);
    if (tile + gridDim.x < ntiles) issue(tile + gridDim.x);
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    FftTail<Ff>::run(buf, a.tw, sink);
    __syncthreads();
    // one warp per output line (level t0 + li): contiguous run of m in y
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int li = warp; li < kTB; li += T / 32) {
      const long long t = tt * kTB + li;
      if (t >= a.nlev) continue;
      double* __restrict__ dst = a.out + (t * a.P + o) * m;
      const bool odd = li & 1;
      for (int e = lane; e < m; e += 32) {
        const double2 X = buf[Lay::addr(li >> 1, e + 1)];
        dst[e] = odd ? a.f * X.x : -a.f * X.y;
      }
    }
  }
}

template <int L> constexpr size_t smemB_bytes() {
  using Lay = Interleaved<4, PlanB<L>::R1>;
  return sizeof(double2) * Lay::words(L) + sizeof(double) * (L / 2 - 1) * kTB;
}

}  // namespace gdst
}  // namespace bhcp

namespace bhcp {
namespace gdst {

// ---------------------------------------------------------------------------
// k_dst_blk2: first level pass from the blocked W with the half-length real
// DST (see k_dst2): one complex FFT of length N = m+1 per two levels, then a
// per-warp post-processing pass (U^a/U^b split, prefix sum for the odd
// coefficients) that writes the output row directly.
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

namespace bhcp {
namespace gdst {

// ---------------------------------------------------------------------------
// k_lines2<N, S, MODE>: level-pass DST over 2S real lines per CTA with the
// half-length real DST (one N-point complex FFT per two lines), wide tiles
// and no CTA-wide barrier in the post-processing:
//   * first FFT stage loads the lines straight from global memory, thread
//     mapping sequence-fastest, so 2S consecutive lines give 16*S-byte runs;
//   * warp q post-processes sequence q (both of its lines: U^a/U^b split and
//     the prefix sums) and writes the DST coefficients back into its own
//     shared-memory region;
//   * one coalesced store phase.
// MODE 0: input = blocked W (lines = levels of one spatial line, 8 levels per
//         contiguous block), output = rows of the level-major y.
// MODE 1: strided in place on y: element e of line (o, i) at o*os + e*es + i.
template <int L, int LD>
struct SeqMajorQ {  // sequence-major, odd stride LD, thread mapping sequence-fastest
  static constexpr int words(int S) { return LD * S; }
  static __device__ __forceinline__ int addr(int q, int idx) { return q * LD + idx; }
  template <int STRIDE>
  static __device__ __forceinline__ int addr_r(int q, int j, int r) { return q * LD + j + r * STRIDE; }
  template <int R>
  static __device__ __forceinline__ int addr_first(int q, int base, int r) { return q * LD + base + r; }
  static __device__ __forceinline__ void split(int b, int nb, int& q, int& j);
};

template <int N, int S> struct PlanL2;
template <> struct PlanL2<256, 16> { template <class Lay> using F = Fft<256, 16, 512, Lay, 4, 8, 8>; };
template <> struct PlanL2<512, 16> { template <class Lay> using F = Fft<512, 16, 512, Lay, 8, 8, 8>; };
template <> struct PlanL2<1024, 8> { template <class Lay> using F = Fft<1024, 8, 256, Lay, 16, 8, 8>; };

template <int S> struct QSplit {
  static __device__ __forceinline__ void split(int b, int nb, int& q, int& j) { q = b % S; j = b / S; }
};
template <int L, int LD, int S>
struct SeqMajorQS : SeqMajorQ<L, LD> {
  static __device__ __forceinline__ void split(int b, int nb, int& q, int& j) { q = b % S; j = b / S; }
};

struct ArgsL2 {
  const double* in;
  double* out;
  const double2* tw;
  const double* sn;
  double scale;
  long long ni, no;            // lines per outer index (levels for MODE 0), outer count
  // MODE 0
  const long long* koff;
  long long NT, P1, idiv, P;
  // MODE 1
  long long os, es;
};

template <int N, int S, int MODE>
__global__ void __launch_bounds__(32 * S, 1) k_lines2(ArgsL2 a) {
  constexpr int T = 32 * S, m = N - 1, NL = 2 * S;
  constexpr int LD = N + 1;  // odd stride (double2 units)
  constexpr int KU = (N / 2) / 32;
  using Lay = SeqMajorQS<N, LD, S>;
  using Ff = typename PlanL2<N, S>::template F<Lay>;
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* sn = reinterpret_cast<double*>(smem + Lay::words(S));
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long ntile_i = (a.ni + NL - 1) / NL;
  const long long ntiles = ntile_i * a.no;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long o = tile / ntile_i;
    const long long i0 = (tile - o * ntile_i) * NL;
    const long long valid = a.ni - i0;  // lines li < valid exist
    long long base0 = 0;
    if (MODE == 0) {
      const long long k1 = o / a.idiv, r2 = o - k1 * a.idiv;
      const long long kb = a.koff ? __ldg(a.koff + k1) : k1 * a.NT * a.P1 * kTB;
      base0 = kb + r2 * (long long)m * kTB;  // + (tt*P1 + e)*8 + tl with level i = tt*8 + tl
    } else {
      base0 = o * a.os + i0;
    }
    __syncthreads();  // previous tile's store phase done with buf
    auto gen = [&](int q, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      double2 p = make_double2(0.0, 0.0), r = make_double2(0.0, 0.0);
      const int li = 2 * q;
      if (li < valid) {
        if (MODE == 0) {
          const long long i = i0 + li;  // even level: its pair lies in the same 8-level block
          const long long blk = base0 + ((i >> 3) * a.P1) * kTB + (i & 7);
          p = __ldg(reinterpret_cast<const double2*>(a.in + blk + (long long)(j - 1) * kTB));
          r = __ldg(reinterpret_cast<const double2*>(a.in + blk + (long long)(N - j - 1) * kTB));
        } else {
          const double* src = a.in + base0 + li;
          p.x = __ldg(src + (long long)(j - 1) * a.es);
          r.x = __ldg(src + (long long)(N - j - 1) * a.es);
          if (li + 1 < valid) {
            p.y = __ldg(src + 1 + (long long)(j - 1) * a.es);
            r.y = __ldg(src + 1 + (long long)(N - j - 1) * a.es);
          }
        }
        if (MODE == 0 && li + 1 >= valid) { p.y = 0.0; r.y = 0.0; }
      }
      const double s = sn[j];
      return make_double2(fma(s, p.x + r.x, 0.5 * (p.x - r.x)), fma(s, p.y + r.y, 0.5 * (p.y - r.y)));
    };
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    Ff::run(buf, a.tw, gen, sink);
    __syncthreads();
    // post-processing: warp q owns sequence q = lines (2q, 2q+1)
    {
      const int q = warp;
      double Ca[KU], Da[KU], Cb[KU], Db[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = u * 32 + lane;
        const double2 A = buf[Lay::addr(q, k)];
        const double2 B = buf[Lay::addr(q, (N - k) & (N - 1))];
        Ca[u] = 0.5 * (A.x + B.x);
        Da[u] = -0.5 * (A.y - B.y);
        Cb[u] = 0.5 * (A.y + B.y);
        Db[u] = 0.5 * (A.x - B.x);
      }
      __syncwarp();
      double* reg = reinterpret_cast<double*>(buf + Lay::addr(q, 0));  // 2*LD doubles
      const double c0a = __shfl_sync(0xffffffffu, Ca[0], 0), c0b = __shfl_sync(0xffffffffu, Cb[0], 0);
      double carry_a = 0.0, carry_b = 0.0;
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        const int k = u * 32 + lane;
        double ia = Ca[u], ib = Cb[u];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double va = __shfl_up_sync(0xffffffffu, ia, off);
          const double vb = __shfl_up_sync(0xffffffffu, ib, off);
          if (lane >= off) { ia += va; ib += vb; }
        }
        const double oa = carry_a + ia - 0.5 * c0a, ob = carry_b + ib - 0.5 * c0b;
        carry_a += __shfl_sync(0xffffffffu, ia, 31);
        carry_b += __shfl_sync(0xffffffffu, ib, 31);
        // line a at reg[0 .. m), line b at reg[m .. 2m): coefficient e = 2k (odd S), 2k-1 (even S)
        reg[2 * k] = a.scale * oa;
        reg[m + 2 * k] = a.scale * ob;
        if (k >= 1) {
          reg[2 * k - 1] = a.scale * Da[u];
          reg[m + 2 * k - 1] = a.scale * Db[u];
        }
      }
    }
    __syncthreads();
    if (MODE == 0) {
      // output rows: line li = level i0+li, contiguous in y
      for (int li = warp; li < NL; li += T / 32) {
        if (li >= valid) continue;
        const double* reg = reinterpret_cast<const double*>(buf + Lay::addr(li >> 1, 0)) + (li & 1) * m;
        double* __restrict__ dst = a.out + ((i0 + li) * a.P + o) * m;
        for (int e = lane; e < m; e += 32) dst[e] = reg[e];
      }
    } else {
      const int li = threadIdx.x % NL;
      const double* reg = reinterpret_cast<const double*>(buf + Lay::addr(li >> 1, 0)) + (li & 1) * m;
      double* __restrict__ dst = a.out + base0 + li;
      if (li < valid) {
        for (int e = threadIdx.x / NL; e < m; e += T / NL) dst[(long long)e * a.es] = reg[e];
      }
    }
  }
}

template <int N, int S> constexpr size_t smemL2_bytes() {
  return sizeof(double2) * (N + 1) * S + sizeof(double) * N;
}

}  // namespace gdst
}  // namespace bhcp
