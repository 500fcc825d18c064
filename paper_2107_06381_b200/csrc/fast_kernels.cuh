// fast_kernels.cuh -- specialised kernels for the BASELINE lengths.
//
// k_dst_rows_fast / k_dst_cols_fast: orthonormal DST-I (space.py:163-177) of
//   length N-1 through an odd-extension FFT of length L = 2N, for
//   N in {256, 512, 1024, 4096}; first stage reads global memory, last stage
//   writes the coefficients straight back (one shared-memory round trip per
//   middle stage only).
// k_modes_fast: pass A of the fused solve for n = 513 time levels:
//   generator = 1/(s_j + mu_k) computed in registers, sink = Gamma^-1, Re,
//   norms and the coalesced store of W[t, k].
// Included by bhcp_b200.cu (single translation unit).
#pragma once
#include "static_fft.cuh"

namespace bhcp {
namespace fastk {

using namespace sfft;

// radix plans for the odd-extension DST lengths (L = 2N)
template <int L> struct DstPlan;
template <> struct DstPlan<512> { template <int S, int T, class Lay> using F = Fft<512, S, T, Lay, 8, 8, 8>; static constexpr int R1 = 8; };
template <> struct DstPlan<1024> { template <int S, int T, class Lay> using F = Fft<1024, S, T, Lay, 16, 8, 8>; static constexpr int R1 = 16; };
template <> struct DstPlan<2048> { template <int S, int T, class Lay> using F = Fft<2048, S, T, Lay, 16, 16, 8>; static constexpr int R1 = 16; };
template <> struct DstPlan<8192> { template <int S, int T, class Lay> using F = Fft<8192, S, T, Lay, 16, 16, 8, 4>; static constexpr int R1 = 16; };

// CTA shapes: sequences per CTA (S) and threads (T), rows / cols kernels
template <int L> struct RowsShape;
template <> struct RowsShape<512> { static constexpr int S = 8, T = 256; };
template <> struct RowsShape<1024> { static constexpr int S = 4, T = 256; };
template <> struct RowsShape<2048> { static constexpr int S = 2, T = 256; };
template <> struct RowsShape<8192> { static constexpr int S = 1, T = 512; };
template <int L> struct ColsShape;
template <> struct ColsShape<512> { static constexpr int S = 8, T = 256; };
template <> struct ColsShape<1024> { static constexpr int S = 4, T = 256; };
template <> struct ColsShape<2048> { static constexpr int S = 4, T = 512; };
template <> struct ColsShape<8192> { static constexpr int S = 1, T = 512; };

struct FastDstArgs {
  const double* in;
  double* out;
  long long nseqs;   // rows: number of FFT sequences (complex lines or real pairs)
  long long nlines;  // rows: number of lines
  long long ni, no, es, os;  // cols geometry
  const double2* tw;
  double f;          // sqrt(2/N)/2
  int m;
  // rows, blocked input (see DstArgs in bhcp_b200.cu); null koff = contiguous
  const long long* koff;
  const long long* kstride;
  long long lines_per_level, inner_div;
};

__device__ __forceinline__ long long fast_line_base(const FastDstArgs& a, long long l) {
  if (!a.koff) return l * a.m;
  const long long t = l / a.lines_per_level;
  const long long rem = l - t * a.lines_per_level;
  const long long k1 = rem / a.inner_div;
  const long long r2 = rem - k1 * a.inner_div;
  return __ldg(a.koff + k1) + t * __ldg(a.kstride + k1) + r2 * a.m;
}

// ---------------------------------------------------------------- rows
template <int L, int CPLX>
struct RowsGen {
  const double* in;
  long long s0, nlines;
  const long long* base;  // shared: start of each line of the CTA (2 per sequence)
  __device__ __forceinline__ double2 operator()(int q, int idx) const {
    constexpr int N = L / 2, m = N - 1;
    if (idx == 0 || idx == N) return make_double2(0.0, 0.0);
    const bool neg = idx > N;
    const int e = neg ? (L - idx - 1) : (idx - 1);
    const long long s = s0 + q;
    double2 x = make_double2(0.0, 0.0);
    if (CPLX) {
      if (s < nlines) x = __ldg(reinterpret_cast<const double2*>(in) + s * m + e);
    } else {
      const long long l0 = 2 * s;
      if (l0 < nlines) x.x = __ldg(in + base[2 * q] + e);
      if (l0 + 1 < nlines) x.y = __ldg(in + base[2 * q + 1] + e);
    }
    return neg ? make_double2(-x.x, -x.y) : x;
  }
};

template <int L, int CPLX>
struct RowsSink {
  double* out;
  long long s0, nlines;
  double f;
  __device__ __forceinline__ void operator()(int q, int idx, double2 X) const {
    constexpr int N = L / 2, m = N - 1;
    if (idx < 1 || idx >= N) return;
    const long long s = s0 + q;
    const int e = idx - 1;
    const double2 c = make_double2(-f * X.y, f * X.x);
    if (CPLX) {
      if (s < nlines) reinterpret_cast<double2*>(out)[s * m + e] = c;
    } else {
      const long long l0 = 2 * s;
      if (l0 < nlines) out[l0 * m + e] = c.x;
      if (l0 + 1 < nlines) out[(l0 + 1) * m + e] = c.y;
    }
  }
};

template <int L, int CPLX>
__global__ void __launch_bounds__(RowsShape<L>::T) k_dst_rows_fast(FastDstArgs a) {
  constexpr int S = RowsShape<L>::S, T = RowsShape<L>::T;
  using Lay = SeqMajorPad<L, DstPlan<L>::R1>;
  extern __shared__ double2 smem[];
  __shared__ long long s_base[2 * S];
  const long long s0 = (long long)blockIdx.x * S;
  if (!CPLX && threadIdx.x < 2 * S) {
    const long long l = 2 * s0 + threadIdx.x;
    s_base[threadIdx.x] = l < a.nlines ? fast_line_base(a, l) : 0;
  }
  __syncthreads();
  RowsGen<L, CPLX> gen{a.in, s0, a.nlines, s_base};
  RowsSink<L, CPLX> sink{a.out, s0, a.nlines, a.f};
  DstPlan<L>::template F<S, T, Lay>::run(smem, a.tw, gen, sink);
}

// ---------------------------------------------------------------- cols
template <int L, int CPLX>
struct ColsGen {
  const double* base;  // line origin for outer index o
  long long i0, ni, es;
  __device__ __forceinline__ double2 operator()(int q, int idx) const {
    constexpr int N = L / 2;
    if (idx == 0 || idx == N) return make_double2(0.0, 0.0);
    const bool neg = idx > N;
    const long long e = neg ? (L - idx - 1) : (idx - 1);
    double2 x = make_double2(0.0, 0.0);
    if (CPLX) {
      const long long i = i0 + q;
      if (i < ni) x = __ldg(reinterpret_cast<const double2*>(base) + i + e * es);
    } else {
      const long long i = i0 + 2 * q;
      if (i < ni) x.x = __ldg(base + i + e * es);
      if (i + 1 < ni) x.y = __ldg(base + i + 1 + e * es);
    }
    return neg ? make_double2(-x.x, -x.y) : x;
  }
};

template <int L, int CPLX>
struct ColsSink {
  double* base;
  long long i0, ni, es;
  double f;
  __device__ __forceinline__ void operator()(int q, int idx, double2 X) const {
    constexpr int N = L / 2;
    if (idx < 1 || idx >= N) return;
    const long long e = idx - 1;
    const double2 c = make_double2(-f * X.y, f * X.x);
    if (CPLX) {
      const long long i = i0 + q;
      if (i < ni) reinterpret_cast<double2*>(base)[i + e * es] = c;
    } else {
      const long long i = i0 + 2 * q;
      if (i < ni) base[i + e * es] = c.x;
      if (i + 1 < ni) base[i + 1 + e * es] = c.y;
    }
  }
};

template <int L, int CPLX>
__global__ void __launch_bounds__(ColsShape<L>::T) k_dst_cols_fast(FastDstArgs a) {
  constexpr int S = ColsShape<L>::S, T = ColsShape<L>::T;
  using Lay = Interleaved<S>;
  extern __shared__ double2 smem[];
  constexpr int lines_per_cta = CPLX ? S : 2 * S;
  const long long ntile = (a.ni + lines_per_cta - 1) / lines_per_cta;
  const long long o = blockIdx.x / ntile;
  const long long i0 = (blockIdx.x - o * ntile) * lines_per_cta;
  const long long off = (CPLX ? 2 : 1) * (o * a.os);
  ColsGen<L, CPLX> gen{a.in + off, i0, a.ni, a.es};
  ColsSink<L, CPLX> sink{a.out + off, i0, a.ni, a.es, a.f};
  DstPlan<L>::template F<S, T, Lay>::run(smem, a.tw, gen, sink);
}

// ---------------------------------------------------------------- modes
template <int N> struct ModesPlan;
template <> struct ModesPlan<513> {
  static constexpr int S = 8, T = 256;
  template <class Lay> using F = Fft<513, S, T, Lay, 19, 9, 3>;
};

struct FastModesArgs {
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  long long w_ld;
  int m, dim;
  const double2* tw;
  StatusDev* st;
};

template <int S>
struct ModesGen {
  const double2* shifts;
  const double* smu;  // shared: per-sequence mu
  const bool* valid;
  StatusDev* st;
  __device__ __forceinline__ double2 operator()(int q, int j) const {
    const double2 s = __ldg(shifts + j);
    if (!valid[q]) return make_double2(0.0, 0.0);
    const double dr = s.x + smu[q], di = s.y;
    const double den2 = dr * dr + di * di;
    if (den2 <= 1e-28 * (s.x * s.x + s.y * s.y)) flag_singular(st, j);
    const double inv = 1.0 / den2;
    return make_double2(dr * inv, -di * inv);
  }
};

template <int S>
struct ModesSink {
  const double2* gaminv;
  const double* sc;  // shared: per-sequence ghat * cscale
  const bool* valid;
  double* W;
  long long w_ld, kl0;
  double sre, sim;
  __device__ __forceinline__ void operator()(int q, int t, double2 X) {
    if (!valid[q]) return;
    const double2 g = __ldg(gaminv + t);
    const double c = sc[q];
    const double wr = c * (X.x * g.x - X.y * g.y);
    const double wi = c * (X.x * g.y + X.y * g.x);
    sre = fma(wr, wr, sre);
    sim = fma(wi, wi, sim);
    W[(long long)t * w_ld + kl0 + q] = wr;
  }
};

template <int N>
__global__ void __launch_bounds__(ModesPlan<N>::T) k_modes_fast(FastModesArgs a) {
  constexpr int S = ModesPlan<N>::S, T = ModesPlan<N>::T;
  using Lay = Interleaved<S>;
  extern __shared__ double2 smem[];
  __shared__ double s_mu[S], s_c[S], red[2 * (T / 32)];
  __shared__ bool s_valid[S];
  const long long kl0 = (long long)blockIdx.x * S;
  if (threadIdx.x < S) {
    const int q = threadIdx.x;
    const long long kl = kl0 + q;
    const bool v = kl < a.k_count;
    s_valid[q] = v;
    const long long k = a.k_begin + (v ? kl : 0);
    s_mu[q] = mode_mu(a.mu1, a.m, a.dim, k);
    s_c[q] = v ? a.ghat[k] * a.cscale : 0.0;
  }
  __syncthreads();
  ModesGen<S> gen{a.shifts, s_mu, s_valid, a.st};
  ModesSink<S> sink{a.gaminv, s_c, s_valid, a.W, a.w_ld, kl0, 0.0, 0.0};
  ModesPlan<N>::template F<Lay>::run(smem, a.tw, gen, sink);
  double sre = sink.sre, sim = sink.sim;
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
  }
}

// smem bytes for each kernel
template <int L> constexpr size_t rows_smem() {
  return sizeof(double2) * SeqMajorPad<L, DstPlan<L>::R1>::LD * RowsShape<L>::S;
}
template <int L> constexpr size_t cols_smem() { return sizeof(double2) * L * ColsShape<L>::S; }
template <int N> constexpr size_t modes_smem() { return sizeof(double2) * N * ModesPlan<N>::S; }

}  // namespace fastk
}  // namespace bhcp
