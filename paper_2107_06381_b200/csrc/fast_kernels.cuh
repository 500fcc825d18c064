// fast_kernels.cuh -- specialised kernels for the BASELINE lengths.
//
// k_dst_rows_fast / k_dst_cols_fast: orthonormal DST-I (space.py:163-177) of
//   length N-1 through an odd-extension FFT of length L = 2N, for
//   N in {256, 512, 1024, 4096}; the first stage reads global memory, the last
//   stage writes the coefficients straight back.
// k_modes_fast: pass A of the fused solve for n = 513 levels:
//   generator = 1/(s_j + mu_k) computed in registers, sink = Gamma^-1, Re,
//   residue norms and the coalesced store of W[t, k]. In 2D the CTA works on
//   a 4x4 tile (k1, k2) of the upper triangle k1 <= k2 and also stores the
//   mirrored tile: mu(k1,k2) = mu1[k1] + mu1[k2] is bit-identical to
//   mu(k2,k1), so the time transform of one mode serves both.
// Included by bhcp_b200.cu (single translation unit).
#pragma once
#include "static_fft.cuh"

namespace bhcp {
namespace fastk {

using namespace sfft;

// fp64 reciprocal: hardware approximation + two Newton steps (<= 1 ulp).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Layout of W written by the modes kernels.
//   mode_major = 0: level-major, W[t * w_ld + k]                      (1D)
//   mode_major = 2: blocked, per level slab s (levels [c_s, c_{s+1}),
//     NT_s = ceil(L_s / 8) tiles of 8 levels):                        (2D / 3D)
//       W[off_s + ((k1 * NT_s + tl / 8) * P1 + r) * 8 + tl % 8],
//       k = k1 * P1 + r (local mode), tl = t - c_s, off_s = nmodes * 8 * sum NT_{s'<s}
//     so a spatial line of 8 levels is contiguous for the level pass and
//     each destination slab is one contiguous all-to-all chunk.
//   sl_base[s]: where slab s starts -- W + off_s for a local W, or a chunk of
//     another GPU's receive buffer (peer memory over NVLink) when pass A
//     stores straight into the destination rank (bhcp_pint_modes_to).
constexpr int kTBL = 8;
struct WLayout {
  int mode_major;
  int nsl;
  int sl_c[9];
  long long sl_off[8];
  long long sl_nt[8];
  double* sl_base[8];
  const long long* sl_koff[8];   // optional: k1 row -> offset from sl_base[s] (receiver block tables)
  long long nmodes;
  long long w_ld;
  long long P1;
  __host__ __device__ __forceinline__ double* ptr(long long k, int t) const {
    if (!mode_major) return sl_base[0] + (long long)t * w_ld + k;
    int s = 0;
    while (s + 1 < nsl && t >= sl_c[s + 1]) ++s;
    const long long tl = t - sl_c[s];
    const long long k1 = k / P1, r = k - k1 * P1;
    return sl_base[s] + row_off(s, k1) + ((tl / kTBL) * P1 + r) * kTBL + (tl % kTBL);
  }
  // offset of k1 row's first block in slab s
  __host__ __device__ __forceinline__ long long row_off(int s, long long k1) const {
    return sl_koff[s] ? sl_koff[s][k1] : k1 * sl_nt[s] * P1 * kTBL;
  }
  // local W: slab s starts at W + sl_off[s]
  __host__ __device__ __forceinline__ void bind(double* W) {
    for (int s = 0; s < 8; ++s) sl_base[s] = (mode_major && s < nsl) || s == 0 ? W + (mode_major ? sl_off[s] : 0) : nullptr;
  }
  __host__ __device__ __forceinline__ long long total(int n) const {
    if (!mode_major) return (long long)n * w_ld;
    long long nt = 0;
    for (int s = 0; s < nsl; ++s) nt += sl_nt[s];
    return nmodes * kTBL * nt;
  }
};

// radix plans for the odd-extension DST lengths (L = 2N)
template <int L> struct DstPlan;
template <> struct DstPlan<512> { template <int S, int T, class Lay> using F = Fft<512, S, T, Lay, 8, 8, 8>; static constexpr int R1 = 8; };
template <> struct DstPlan<1024> { template <int S, int T, class Lay> using F = Fft<1024, S, T, Lay, 16, 8, 8>; static constexpr int R1 = 16; };
template <> struct DstPlan<2048> { template <int S, int T, class Lay> using F = Fft<2048, S, T, Lay, 16, 16, 8>; static constexpr int R1 = 16; };
template <> struct DstPlan<8192> { template <int S, int T, class Lay> using F = Fft<8192, S, T, Lay, 16, 16, 8, 4>; static constexpr int R1 = 16; };

// CTA shapes: sequences per CTA (S), threads (T), min CTAs per SM
template <int L> struct RowsShape;
template <> struct RowsShape<512> { static constexpr int S = 8, T = 256, MINB = 2; };
template <> struct RowsShape<1024> { static constexpr int S = 4, T = 256, MINB = 2; };
template <> struct RowsShape<2048> { static constexpr int S = 2, T = 256, MINB = 2; };
template <> struct RowsShape<8192> { static constexpr int S = 1, T = 512, MINB = 1; };
template <int L> struct ColsShape;
template <> struct ColsShape<512> { static constexpr int S = 8, T = 256, MINB = 2; };
template <> struct ColsShape<1024> { static constexpr int S = 8, T = 512, MINB = 1; };
template <> struct ColsShape<2048> { static constexpr int S = 4, T = 512, MINB = 1; };
template <> struct ColsShape<8192> { static constexpr int S = 1, T = 512, MINB = 1; };

struct FastDstArgs {
  const double* in;
  double* out;
  long long nseqs;   // rows: number of FFT sequences
  long long nlines;  // rows: number of lines
  long long lpl;     // rows, real data: lines per level (>1: pair lines inside a level)
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

// Real-data rows: FFT sequence s carries lines (l0, l1). With lpl > 1 the two
// lines are taken inside one level (lines (t, 2u), (t, 2u+1)), so the result
// of a level never depends on which other levels share the launch (slab
// decomposition stays bit-identical); with lpl == 1 (1D) consecutive levels
// are paired. l1 = -1 when the partner line does not exist.
__host__ __device__ __forceinline__ void pair_lines(long long s, long long nlines, long long lpl, long long& l0,
                                                    long long& l1) {
  if (lpl > 1) {
    const long long ppl = (lpl + 1) / 2;
    const long long t = s / ppl, u = s - t * ppl;
    l0 = t * lpl + 2 * u;
    l1 = (2 * u + 1 < lpl) ? l0 + 1 : -1;
  } else {
    l0 = 2 * s;
    l1 = 2 * s + 1;
  }
  if (l0 >= nlines) l0 = -1;
  if (l1 >= nlines) l1 = -1;
}
__host__ __device__ __forceinline__ long long real_row_seqs(long long nlines, long long lpl) {
  return lpl > 1 ? (nlines / lpl) * ((lpl + 1) / 2) : (nlines + 1) / 2;
}

// ---------------------------------------------------------------- rows
template <int L, int CPLX>
struct RowsGen {
  const double* in;
  long long s0, nseqs;
  const long long* base;  // shared: input start of each line of the CTA (2 per sequence), -1 = none
  __device__ __forceinline__ double2 operator()(int q, int idx) const {
    constexpr int N = L / 2, m = N - 1;
    if (idx == 0 || idx == N) return make_double2(0.0, 0.0);
    const bool neg = idx > N;
    const int e = neg ? (L - idx - 1) : (idx - 1);
    const long long s = s0 + q;
    double2 x = make_double2(0.0, 0.0);
    if (CPLX) {
      if (s < nseqs) x = __ldg(reinterpret_cast<const double2*>(in) + s * m + e);
    } else {
      const long long b0 = base[2 * q], b1 = base[2 * q + 1];
      if (b0 >= 0) x.x = __ldg(in + b0 + e);
      if (b1 >= 0) x.y = __ldg(in + b1 + e);
    }
    return neg ? make_double2(-x.x, -x.y) : x;
  }
};

template <int L, int CPLX>
struct RowsSink {
  double* out;
  long long s0, nseqs;
  const long long* obase;  // shared: output start of each line (2 per sequence), -1 = none
  double f;
  __device__ __forceinline__ void operator()(int q, int idx, double2 X) const {
    constexpr int N = L / 2, m = N - 1;
    if (idx < 1 || idx >= N) return;
    const long long s = s0 + q;
    const int e = idx - 1;
    const double2 c = make_double2(-f * X.y, f * X.x);
    if (CPLX) {
      if (s < nseqs) reinterpret_cast<double2*>(out)[s * m + e] = c;
    } else {
      const long long b0 = obase[2 * q], b1 = obase[2 * q + 1];
      if (b0 >= 0) out[b0 + e] = c.x;
      if (b1 >= 0) out[b1 + e] = c.y;
    }
  }
};

// twiddle table: global (L1-cached); set TwSmem<L>::on to stage it in shared memory
template <int L> struct TwSmem { static constexpr bool on = false; static constexpr int n = on ? L : 0; };

template <int L>
__device__ __forceinline__ const double2* stage_twiddles(const double2* tw_g, double2* tw_s) {
  if constexpr (TwSmem<L>::on) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) tw_s[i] = __ldg(tw_g + i);
    return tw_s;
  } else {
    return tw_g;
  }
}

// Persistent: each CTA loops over tiles of S sequences (grid = resident CTAs).
template <int L, int CPLX>
__global__ void __launch_bounds__(RowsShape<L>::T, RowsShape<L>::MINB) k_dst_rows_fast(FastDstArgs a) {
  constexpr int S = RowsShape<L>::S, T = RowsShape<L>::T;
  using Lay = SeqMajorPad<L, DstPlan<L>::R1>;
  extern __shared__ double2 smem[];
  __shared__ long long s_base[2 * S], s_obase[2 * S];
  double2* buf = smem;
  const double2* tw = stage_twiddles<L>(a.tw, smem + Lay::words(S));
  const long long ntiles = (a.nseqs + S - 1) / S;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long s0 = tile * S;
    __syncthreads();  // previous tile done with buf / s_base
    if (!CPLX && threadIdx.x < S) {
      long long l0, l1;
      pair_lines(s0 + threadIdx.x, a.nlines, a.lpl, l0, l1);
      if (s0 + threadIdx.x >= a.nseqs) l0 = l1 = -1;
      s_base[2 * threadIdx.x] = l0 >= 0 ? fast_line_base(a, l0) : -1;
      s_base[2 * threadIdx.x + 1] = l1 >= 0 ? fast_line_base(a, l1) : -1;
      s_obase[2 * threadIdx.x] = l0 >= 0 ? l0 * a.m : -1;
      s_obase[2 * threadIdx.x + 1] = l1 >= 0 ? l1 * a.m : -1;
    }
    __syncthreads();
    RowsGen<L, CPLX> gen{a.in, s0, a.nseqs, s_base};
    RowsSink<L, CPLX> sink{a.out, s0, a.nseqs, s_obase, a.f};
    DstPlan<L>::template F<S, T, Lay>::run(buf, tw, gen, sink);
  }
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
__global__ void __launch_bounds__(ColsShape<L>::T, ColsShape<L>::MINB) k_dst_cols_fast(FastDstArgs a) {
  constexpr int S = ColsShape<L>::S, T = ColsShape<L>::T;
  using Lay = Interleaved<S, DstPlan<L>::R1>;
  extern __shared__ double2 smem[];
  constexpr int lines_per_cta = CPLX ? S : 2 * S;
  double2* buf = smem;
  const double2* tw = stage_twiddles<L>(a.tw, smem + Lay::words(L));
  const long long ntile = (a.ni + lines_per_cta - 1) / lines_per_cta;
  const long long total = ntile * a.no;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const long long o = tile / ntile;
    const long long i0 = (tile - o * ntile) * lines_per_cta;
    const long long off = (CPLX ? 2 : 1) * (o * a.os);
    __syncthreads();
    ColsGen<L, CPLX> gen{a.in + off, i0, a.ni, a.es};
    ColsSink<L, CPLX> sink{a.out + off, i0, a.ni, a.es, a.f};
    DstPlan<L>::template F<S, T, Lay>::run(buf, tw, gen, sink);
  }
}

// ---------------------------------------------------------------- modes
template <int N> struct ModesPlan;
// 2D symmetric tiles: kSymTile x kSymTile modes, one warp each (16 warps at 128
// registers; 3 x 3 tiles, 9 warps at 168 registers, measured 0.65 vs 0.51 ms on c2)
constexpr int kSymTile = 4;
template <> struct ModesPlan<513> {
  static constexpr int S = kSymTile * kSymTile, T = 32 * S, MINB = 1;
  using WF = WarpFft<513, 19, 9, 3>;
};

struct FastModesArgs {
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  int m, dim;
  const double2* tw;
  StatusDev* st;
  const int2* tiles;  // SYM: upper-triangle 4x4 tile coordinates (a, b), a <= b
  long long ntiles;
  WLayout wl;
};

// Warp-per-mode pass A, persistent: a CTA loads the shift and 1/gamma tables
// once and loops over tiles of S = 16 modes (a 4x4 upper-triangle tile in
// 2D, SYM, or 16 consecutive modes); warp q transforms mode q of the tile in
// its own shared-memory region with warp-synchronous stages and writes that
// mode's time series (and the mirrored mode's) itself. No CTA barrier inside
// the tile loop: warps progress independently.
template <int N, bool SYM>
__global__ void __launch_bounds__(ModesPlan<N>::T, ModesPlan<N>::MINB) k_modes_fast(FastModesArgs a) {
  constexpr int S = ModesPlan<N>::S, T = ModesPlan<N>::T;
  static_assert(T == 32 * S, "one warp per mode");
  constexpr int LDW = N;  // per-warp region (odd length: conflict-light)
  extern __shared__ double2 smem[];
  __shared__ double red[2 * (T / 32)];
  __shared__ double2 s_gi[N], s_sh[N];
  __shared__ double s_thr[N];   // singular-shift threshold 1e-28 |s_j|^2 (space.py:237-240)
  for (int i = threadIdx.x; i < N; i += T) {
    s_gi[i] = __ldg(a.gaminv + i);
    const double2 sh = __ldg(a.shifts + i);
    s_sh[i] = sh;
    s_thr[i] = 1e-28 * (sh.x * sh.x + sh.y * sh.y);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* buf = smem + warp * LDW;
  StatusDev* st = a.st;
  const fastk::WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long ntiles = SYM ? a.ntiles : (a.k_count + S - 1) / S;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    // this warp's mode: destination (k1, r) = (kd / P1, kd % P1), mirror, mu, coefficients
    bool valid;
    long long kd, km = -1;
    int k1d = 0, k1m = 0;
    long long rd = 0, rm = 0;
    if (SYM) {
      const int2 tb = __ldg(a.tiles + tile);
      const int k1 = kSymTile * tb.x + warp / kSymTile, k2 = kSymTile * tb.y + warp % kSymTile;
      valid = (k1 < a.m) && (k2 < a.m) && (tb.x != tb.y || k1 <= k2);
      kd = valid ? (long long)k1 * a.m + k2 : 0;
      if (valid && k1 != k2) km = (long long)k2 * a.m + k1;
      k1d = k1; rd = k2; k1m = k2; rm = k1;   // 2D: P1 = m
    } else {
      const long long kl = tile * S + warp;
      valid = kl < a.k_count;
      kd = a.k_begin + (valid ? kl : 0);
      const long long local = valid ? kl : 0;
      if (wl.mode_major) { k1d = (int)(local / wl.P1); rd = local - (long long)k1d * wl.P1; }
    }
    // 2D symmetric tiles know (k1, k2): mu1[k1] + mu1[k2] directly (the same sum
    // mode_mu forms, without its 64-bit division of the flat index)
    const double mu = SYM ? (valid ? __ldg(a.mu1 + k1d) + __ldg(a.mu1 + rd) : __ldg(a.mu1) + __ldg(a.mu1))
                          : mode_mu(a.mu1, a.m, a.dim, kd);
    const double c = valid ? __ldg(a.ghat + kd) * a.cscale : 0.0;
    const double c2 = (SYM && km >= 0) ? __ldg(a.ghat + km) * a.cscale : 0.0;
    {
      const double2* shifts = s_sh;
      auto gen = [&](int j) -> double2 {
        const double2 s = shifts[j];
        if (!valid) return make_double2(0.0, 0.0);
        const double dr = s.x + mu, di = s.y;
        const double den2 = dr * dr + di * di;
        if (den2 <= s_thr[j]) flag_singular(st, j);
        const double inv = fast_rcp(den2);
        return make_double2(dr * inv, -di * inv);
      };
      ModesPlan<N>::WF::run(buf, lane, a.tw, gen);
    }
    if (!valid) continue;
    // W layout a.wl: blocked slabs (runs of 8 levels at stride P1*8) or level-major (stride w_ld)
    // residue norms: sum over this warp's modes of (c^2 + c2^2) * sum_t zr^2 (zi^2)
    double zr2 = 0.0, zi2 = 0.0;
    const double2* X = buf;
    const int nsl = wl.mode_major ? wl.nsl : 1;
    for (int sl = 0; sl < nsl; ++sl) {
      const int t0 = wl.mode_major ? wl.sl_c[sl] : 0;
      const int t1 = wl.mode_major ? wl.sl_c[sl + 1] : N;
      long long pd, pm, step;
      if (wl.mode_major) {
        pd = wl.row_off(sl, k1d) + rd * kTBL;
        pm = wl.row_off(sl, k1m) + rm * kTBL;
        // t = t0 + lane + 32 i  ->  (tl >> 3) * P1*8 + (tl & 7), t0 a multiple of 8
        const long long lo = (long long)(lane >> 3) * wl.P1 * kTBL + (lane & 7);
        pd += lo; pm += lo;
        step = 4 * wl.P1 * kTBL;
      } else {
        pd = kd - a.k_begin + (long long)lane * wl.w_ld;
        pm = km + (long long)lane * wl.w_ld;
        step = 32 * wl.w_ld;
      }
      double* __restrict__ wd = wl.sl_base[sl] + pd;
      double* __restrict__ wm = wl.sl_base[sl] + pm;
      for (int t = t0 + lane; t < t1; t += 32, wd += step, wm += step) {
        const double2 x = X[t];
        const double2 g = s_gi[t];
        const double zr = x.x * g.x - x.y * g.y;
        const double zi = x.x * g.y + x.y * g.x;
        zr2 = fma(zr, zr, zr2);
        zi2 = fma(zi, zi, zi2);
        *wd = c * zr;
        if (SYM && km >= 0) *wm = c2 * zr;
      }
    }
    const double cc = c * c + c2 * c2;
    sre = fma(cc, zr2, sre);
    sim = fma(cc, zi2, sim);
    __syncwarp();   // the store loop's trip count differs across lanes; buf is rewritten by the next mode
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
  }
}

// smem bytes for each kernel
template <int L> constexpr size_t rows_smem() {
  return sizeof(double2) * (SeqMajorPad<L, DstPlan<L>::R1>::words(RowsShape<L>::S) + TwSmem<L>::n);
}
template <int L> constexpr size_t cols_smem() {
  return sizeof(double2) * (Interleaved<ColsShape<L>::S, DstPlan<L>::R1>::words(L) + TwSmem<L>::n);
}
template <int N> constexpr size_t modes_smem() { return sizeof(double2) * N * ModesPlan<N>::S; }

}  // namespace fastk
}  // namespace bhcp

namespace bhcp {
namespace fastk {

// ---------------------------------------------------------------------------
// k_modes_blue<n>: pass A for n = 2^p + 1 time levels (BASELINE n = 257,
// 1025, 4097). With M = n - 1 = 2^p the DFT
//   X_t = sum_{j<M} v_j w^{jt} + v_M w^{Mt},  w = exp(-2 pi i / n),
// has its first sum as a chirp-z transform whose linear convolution spans
// exactly 2M = 2^(p+1) points (inputs j < M, lags -(M-1)..M), so Bluestein
// runs on power-of-two FFTs of length L = 2M instead of the smooth length
// >= 2n-1 a general Bluestein needs:
//   X_t = c_t * IFFT_L( FFT_L(v c) * FFT_L(b) )_t + v_M w^{Mt},
//   c_j = exp(-i pi j^2 / n), b_d = conj(c_d) for d in [-(M-1), M].
// Tables (host, long double): chirp c (n), bhat = FFT_L(b)/L (L), w^{Mt} (n),
// twiddles of length L.
struct BlueTables {
  const double2* tw;     // exp(-2 pi i k / L)
  const double2* chirp;  // c_j, j < n
  const double2* bhat;   // FFT_L(b) / L
  const double2* wM;     // w^{M t}, t < n
  const double2* cg;     // chirp_t / gamma_t
  const double2* wg;     // w^{M t} / gamma_t
  const double2* thr;    // (1e-28 |s_j|^2, 0)
};

template <int NL> struct BluePlan;
template <> struct BluePlan<257> { static constexpr int L = 512, S = 8, T = 256, R1 = 8, MINB = 2; template <class Lay> using F = Fft<512, S, T, Lay, 8, 8, 8>; };
template <> struct BluePlan<1025> { static constexpr int L = 2048, S = 2, T = 256, R1 = 16, MINB = 2; template <class Lay> using F = Fft<2048, S, T, Lay, 16, 16, 8>; };
template <> struct BluePlan<4097> { static constexpr int L = 8192, S = 1, T = 512, R1 = 16, MINB = 1; template <class Lay> using F = Fft<8192, S, T, Lay, 16, 16, 8, 4>; };

struct BlueModesArgs {
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  int m, dim;
  StatusDev* st;
  BlueTables bt;
  WLayout wl;
  const int4* tiles;   // SYM: (k1, k2-or-segment start, k3 segment start)
  long long ntiles;
};

// Second FFT of the Bluestein pair: all stages read shared memory.
template <int L, int S, int T, class Lay, int R1, int... Rest>
struct FftAllSmem {
  template <class Sink>
  static __device__ __forceinline__ void run(double2* buf, const double2* tw, Sink& sink) {
    Runner<L, S, T, Lay, 1, R1, Rest...>::tail(buf, tw, sink);
  }
};
template <class F> struct AllSmemOf;
template <int L, int S, int T, class Lay, int R1, int... Rest>
struct AllSmemOf<Fft<L, S, T, Lay, R1, Rest...>> { using type = FftAllSmem<L, S, T, Lay, R1, Rest...>; };

template <int NL, bool SYM>
__global__ void __launch_bounds__(BluePlan<NL>::T, BluePlan<NL>::MINB) k_modes_blue(BlueModesArgs a) {
  using P = BluePlan<NL>;
  constexpr int L = P::L, S = P::S, T = P::T, M = NL - 1;
  using Lay = SeqMajorPad<L, P::R1>;
  using F1 = typename P::template F<Lay>;
  using F2 = typename AllSmemOf<F1>::type;
  extern __shared__ double2 smem[];
  __shared__ double s_mu[S], s_c[S], s_cm[S], red[2 * (T / 32)];
  __shared__ int s_k1d[S], s_k1m[S];
  __shared__ long long s_rd[S], s_rm[S];
  __shared__ bool s_valid[S], s_hasm[S];
  __shared__ double2 s_vM[S];
  double2* buf = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long ntiles = SYM ? a.ntiles : (a.k_count + S - 1) / S;
  // Persistent: each CTA loops over tiles of S modes.
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    __syncthreads();   // previous tile's stores done with buf / per-mode data
    if (threadIdx.x < S) {
      const int q = threadIdx.x;
      bool v, hm = false;
      long long kd;
      int k1d = 0, k1m = 0;
      long long rd = 0, rm = 0, km = 0;
      if (SYM) {
        const int4 tb = a.tiles[tile];
        if (a.dim == 2) {
          const int k1 = tb.x, k2 = tb.y + q;
          v = k2 < a.m && k2 >= k1;
          kd = (long long)k1 * a.m + k2;
          hm = v && k2 != k1;
          km = (long long)k2 * a.m + k1;
          k1d = k1; rd = k2; k1m = k2; rm = k1;                       // P1 = m
        } else {
          const int k1 = tb.x, k2 = tb.y, k3 = tb.z + q;
          v = k3 < a.m;
          kd = ((long long)k1 * a.m + k2) * a.m + k3;
          hm = v && k1 != k2;
          km = ((long long)k2 * a.m + k1) * a.m + k3;
          k1d = k1; rd = (long long)k2 * a.m + k3; k1m = k2; rm = (long long)k1 * a.m + k3;   // P1 = m^2
        }
        if (!v) kd = 0;
      } else {
        const long long kl = tile * S + q;
        v = kl < a.k_count;
        kd = a.k_begin + (v ? kl : 0);
        const long long local = v ? kl : 0;
        if (wl.mode_major) { k1d = (int)(local / wl.P1); rd = local - (long long)k1d * wl.P1; }
        else rd = local;
      }
      s_valid[q] = v;
      s_hasm[q] = hm;
      const double mu = mode_mu(a.mu1, a.m, a.dim, kd);
      s_mu[q] = mu;
      s_c[q] = v ? a.ghat[kd] * a.cscale : 0.0;
      s_cm[q] = hm ? a.ghat[km] * a.cscale : 0.0;
      s_k1d[q] = k1d; s_rd[q] = rd; s_k1m[q] = k1m; s_rm[q] = rm;
      // last input v_M = 1/(s_M + mu)
      const double2 s = __ldg(a.shifts + M);
      const double dr = s.x + mu, di = s.y;
      const double den2 = dr * dr + di * di;
      if (v && den2 <= 1e-28 * (s.x * s.x + s.y * s.y)) flag_singular(a.st, M);
      const double inv = fast_rcp(den2);
      s_vM[q] = v ? make_double2(dr * inv, -di * inv) : make_double2(0.0, 0.0);
    }
    __syncthreads();
    // FFT 1: a_j = v_j c_j (j < M), zero padded to L
    auto gen = [&](int q, int j) -> double2 {
      if (j >= M || !s_valid[q]) return make_double2(0.0, 0.0);
      const double2 s = __ldg(a.shifts + j);
      const double dr = s.x + s_mu[q], di = s.y;
      const double den2 = dr * dr + di * di;
      if (den2 <= __ldg(&a.bt.thr[j].x)) flag_singular(a.st, j);
      const double inv = fast_rcp(den2);
      return cmul(make_double2(dr * inv, -di * inv), __ldg(a.bt.chirp + j));
    };
    auto sink1 = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = cconj(cmul(X, __ldg(a.bt.bhat + idx))); };
    F1::run(buf, a.bt.tw, gen, sink1);
    __syncthreads();
    // FFT 2 (conjugated inverse): conv_t = conj(X_t); X_t of the DFT = c_t conv_t + v_M w^{Mt}
    auto sink2 = [&](int q, int idx, double2 X) {
      if (idx > M) return;
      // Gamma^-1 X_t = conj(X) chirp_t / gamma_t + v_M w^{Mt} / gamma_t (tables cg, wg)
      buf[Lay::addr(q, idx)] = cadd(cmul(cconj(X), __ldg(a.bt.cg + idx)), cmul(s_vM[q], __ldg(a.bt.wg + idx)));
    };
    F2::run(buf, a.bt.tw, sink2);
    __syncthreads();
    // store: warps loop over the S modes; lanes run along t
    for (int q = warp; q < S; q += T / 32) {
      if (!s_valid[q]) continue;
      const bool hm = SYM && s_hasm[q];
      const double c = s_c[q], c2 = s_cm[q];
      const int nsl = wl.mode_major ? wl.nsl : 1;
      double zr2 = 0.0, zi2 = 0.0;
      for (int sl = 0; sl < nsl; ++sl) {
        const int t0 = wl.mode_major ? wl.sl_c[sl] : 0;
        const int t1 = wl.mode_major ? wl.sl_c[sl + 1] : NL;
        long long pd, pm, step;
        if (wl.mode_major) {
          const long long lo = (long long)(lane >> 3) * wl.P1 * kTBL + (lane & 7);
          pd = wl.row_off(sl, s_k1d[q]) + s_rd[q] * kTBL + lo;
          pm = wl.row_off(sl, s_k1m[q]) + s_rm[q] * kTBL + lo;
          step = 4 * wl.P1 * kTBL;
        } else {
          pd = s_rd[q] + (long long)lane * wl.w_ld;
          pm = pd;
          step = 32 * wl.w_ld;
        }
        double* __restrict__ wd = wl.sl_base[sl] + pd;
        double* __restrict__ wm = wl.sl_base[sl] + pm;
        for (int t = t0 + lane; t < t1; t += 32, wd += step, wm += step) {
          const double2 z = buf[Lay::addr(q, t)];
          zr2 = fma(z.x, z.x, zr2);
          zi2 = fma(z.y, z.y, zi2);
          *wd = c * z.x;
          if (hm) *wm = c2 * z.x;
        }
      }
      const double cc = c * c + (hm ? c2 * c2 : 0.0);
      sre = fma(cc, zr2, sre);
      sim = fma(cc, zi2, sim);
    }
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
  }
}

// ---------------------------------------------------------------- Rader
// k_modes_rader<n>: pass A for a prime n with n - 1 = NP a power of two
// (BASELINE n = 257: c1, c4). With j = g^p, t = g^-q (g a primitive root),
//   X_0 = sum_j v_j,   X_{g^-q} = v_0 + sum_p v_{g^p} w^{g^(p-q)} = v_0 + (a (*) b)_q
// a cyclic convolution of length NP (a_p = v_{g^p}, b_m = w^{g^-m}), done as
//   A = FFT(a);  conv = conj(FFT(conj(A * bhat)))   (bhat = FFT(b) / NP)
// so each mode costs two NP-point FFTs instead of the two 2NP-point FFTs of
// the power-of-two Bluestein, and X_0 = v_0 + A_0. One warp per mode
// (warp-synchronous, no CTA barrier in the tile loop), persistent CTAs.
template <int NL> struct RaderPlan;
template <> struct RaderPlan<257> {
  // 12 warps at 168 registers (no spills): c4 pass A 14.7 ms, against 16.5 ms
  // for 16 warps at 128 registers with spills (20 / 24 warps: 20.3 / 23.0 ms)
  static constexpr int NP = 256, S = 12, T = 32 * S, MINB = 1;
  using WF = WarpFftPad<256, 8, 8, 8, 4>;
};

struct RaderModesArgs {
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  int m, dim;
  StatusDev* st;
  const double2* tw;    // exp(-2 pi i k / NP)
  const double2* bhat;  // FFT(b) / NP
  const int* perm;      // g^p mod n
  const int* qidx;      // q with g^-q = t
  WLayout wl;
  const int4* tiles;    // SYM: seg tiles of S modes (see k_modes_blue)
  long long ntiles;
  int sym6;             // 3D: tiles of sorted triples k1 <= k2 <= k3, one FFT for all their permutations
};

template <int NL, bool SYM>
__global__ void __launch_bounds__(RaderPlan<NL>::T, RaderPlan<NL>::MINB) k_modes_rader(RaderModesArgs a) {
  using P = RaderPlan<NL>;
  constexpr int NP = P::NP, S = P::S, T = P::T;
  using WF = typename P::WF;
  static_assert(T == 32 * S, "one warp per mode");
  extern __shared__ double2 smem[];
  __shared__ double red[2 * (T / 32)];
  // shifts and singular thresholds in the permuted order p (j = g^p), so the
  // generator reads consecutive slots; index 0 of s_sh0 / s_thr0 is j = 0.
  __shared__ double2 s_shp[NP], s_gi[NL], s_bh[NP];
  __shared__ double s_thrp[NP];
  __shared__ short s_q[NL];
  __shared__ double2 s_sh0;
  __shared__ double s_thr0;
  for (int i = threadIdx.x; i < NL; i += T) {
    s_gi[i] = __ldg(a.gaminv + i);
    s_q[i] = (short)__ldg(a.qidx + i);
    if (i < NP) {
      const int j = __ldg(a.perm + i);
      const double2 sh = __ldg(a.shifts + j);
      s_shp[i] = sh;
      s_thrp[i] = 1e-28 * (sh.x * sh.x + sh.y * sh.y);   // space.py:237-240
      s_bh[i] = __ldg(a.bhat + i);
    }
    if (i == 0) {
      const double2 sh = __ldg(a.shifts);
      s_sh0 = sh;
      s_thr0 = 1e-28 * (sh.x * sh.x + sh.y * sh.y);
    }
  }
  __syncthreads();
  const int* perm = a.perm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* buf = smem + warp * WF::words;
  StatusDev* st = a.st;
  const WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long ntiles = SYM ? a.ntiles : (a.k_count + S - 1) / S;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    bool valid, hm = false;
    long long kd, km = 0;
    int k1d = 0, k1m = 0;
    long long rd = 0, rm = 0;
    if (SYM) {
      const int4 tb = __ldg(a.tiles + tile);
      if (a.dim == 2) {
        const int k1 = tb.x, k2 = tb.y + warp;
        valid = k2 < a.m && k2 >= k1;
        kd = (long long)k1 * a.m + k2;
        hm = valid && k2 != k1;
        km = (long long)k2 * a.m + k1;
        k1d = k1; rd = k2; k1m = k2; rm = k1;
      } else if (a.sym6) {
        // sorted triple (k1 <= k2 <= k3): every permutation of it has the same
        // mu = (mu1[k1] + mu1[k2]) + mu1[k3] (the sum in sorted order; within an
        // ulp of the C-order sum of the other permutations), so one FFT serves
        // all of them
        const int k1 = tb.x, k2 = tb.y, k3 = tb.z + warp;
        valid = k3 < a.m && k3 >= k2;
        kd = ((long long)k1 * a.m + k2) * a.m + k3;
        k1d = k1; rd = (long long)k2 * a.m + k3; k1m = k2; rm = (long long)k1 * a.m + k3;
      } else {
        const int k1 = tb.x, k2 = tb.y, k3 = tb.z + warp;
        valid = k3 < a.m;
        kd = ((long long)k1 * a.m + k2) * a.m + k3;
        hm = valid && k1 != k2;
        km = ((long long)k2 * a.m + k1) * a.m + k3;
        k1d = k1; rd = (long long)k2 * a.m + k3; k1m = k2; rm = (long long)k1 * a.m + k3;
      }
      if (!valid) kd = 0;
    } else {
      const long long kl = tile * S + warp;
      valid = kl < a.k_count;
      kd = a.k_begin + (valid ? kl : 0);
      const long long local = valid ? kl : 0;
      if (wl.mode_major) { k1d = (int)(local / wl.P1); rd = local - (long long)k1d * wl.P1; }
      else rd = local;
    }
    if (!valid) continue;
    const bool six = SYM && a.sym6;
    double mu;
    if (six) {
      const int4 tb = __ldg(a.tiles + tile);
      mu = (__ldg(a.mu1 + tb.x) + __ldg(a.mu1 + tb.y)) + __ldg(a.mu1 + tb.z + warp);
    } else {
      mu = mode_mu(a.mu1, a.m, a.dim, kd);
    }
    const double c = __ldg(a.ghat + kd) * a.cscale;
    const double c2 = hm ? __ldg(a.ghat + km) * a.cscale : 0.0;
    // 1 / (s + mu) with the singular test of space.py:237-240 (column j reported)
    auto vinv = [&](double2 s, double thr, auto col) -> double2 {
      const double dr = s.x + mu, di = s.y;
      const double den2 = dr * dr + di * di;
      if (den2 <= thr) flag_singular(st, col());
      const double inv = fast_rcp(den2);
      return make_double2(dr * inv, -di * inv);
    };
    const double2 v0 = vinv(s_sh0, s_thr0, [] { return 0; });
    auto gen = [&](int p) -> double2 { return vinv(s_shp[p], s_thrp[p], [&] { return __ldg(perm + p); }); };
    WF::run(buf, lane, a.tw, gen);                     // A = FFT(a)
    const double2 A0 = buf[WF::pi(0)];
    __syncwarp();
    for (int k = lane; k < NP; k += 32) {             // conj(A * bhat), in place
      const int i = WF::pi(k);
      buf[i] = cconj(cmul(buf[i], s_bh[k]));
    }
    __syncwarp();
    WF::run_inplace(buf, lane, a.tw);                  // conv_q = conj(buf[q])
    // store: t along lanes; X_0 = v0 + A0, X_t = v0 + conv_{qidx[t]}
    const int nsl = wl.mode_major ? wl.nsl : 1;
    double zr2 = 0.0, zi2 = 0.0;
    if (six) {
      // the distinct permutations (p1, p2, p3) of the sorted triple (x, y, z):
      // 0 (x,y,z) 1 (x,z,y) 2 (y,x,z) 3 (y,z,x) 4 (z,x,y) 5 (z,y,x)
      const int4 tb = __ldg(a.tiles + tile);
      const int x = tb.x, yv = tb.y, z = tb.z + warp;
      const unsigned mask = (x == yv && yv == z) ? 0x01u : (x == yv) ? 0x13u : (yv == z) ? 0x0du : 0x3fu;
      const int P1[6] = {x, x, yv, yv, z, z}, P2[6] = {yv, z, x, z, x, yv}, P3[6] = {z, yv, z, x, yv, x};
      double cf[6];
      double cc = 0.0;
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        cf[p] = ((mask >> p) & 1u) ? __ldg(a.ghat + ((long long)P1[p] * a.m + P2[p]) * a.m + P3[p]) * a.cscale : 0.0;
        cc = fma(cf[p], cf[p], cc);
      }
      for (int sl = 0; sl < nsl; ++sl) {
        const int t0 = wl.sl_c[sl], t1 = wl.sl_c[sl + 1];
        const long long lo = (long long)(lane >> 3) * wl.P1 * kTBL + (lane & 7);
        const long long step = 4 * wl.P1 * kTBL;
        double* w6[6];
#pragma unroll
        for (int p = 0; p < 6; ++p)
          w6[p] = wl.sl_base[sl] + wl.row_off(sl, P1[p]) + ((long long)P2[p] * a.m + P3[p]) * kTBL + lo;
        for (int t = t0 + lane; t < t1; t += 32) {
          double2 X;
          if (t == 0) X = cadd(v0, A0);
          else X = cadd(v0, cconj(buf[WF::pi(s_q[t])]));
          const double2 g = s_gi[t];
          const double zr = X.x * g.x - X.y * g.y;
          const double zi = X.x * g.y + X.y * g.x;
          zr2 = fma(zr, zr, zr2);
          zi2 = fma(zi, zi, zi2);
#pragma unroll
          for (int p = 0; p < 6; ++p) {
            if ((mask >> p) & 1u) *w6[p] = cf[p] * zr;
            w6[p] += step;
          }
        }
      }
      sre = fma(cc, zr2, sre);
      sim = fma(cc, zi2, sim);
      __syncwarp();
      continue;
    }
    for (int sl = 0; sl < nsl; ++sl) {
      const int t0 = wl.mode_major ? wl.sl_c[sl] : 0;
      const int t1 = wl.mode_major ? wl.sl_c[sl + 1] : NL;
      long long pd, pm, step;
      if (wl.mode_major) {
        const long long lo = (long long)(lane >> 3) * wl.P1 * kTBL + (lane & 7);
        pd = wl.row_off(sl, k1d) + rd * kTBL + lo;
        pm = wl.row_off(sl, k1m) + rm * kTBL + lo;
        step = 4 * wl.P1 * kTBL;
      } else {
        pd = rd + (long long)lane * wl.w_ld;
        pm = pd;
        step = 32 * wl.w_ld;
      }
      double* __restrict__ wd = wl.sl_base[sl] + pd;
      double* __restrict__ wmr = wl.sl_base[sl] + pm;
      for (int t = t0 + lane; t < t1; t += 32, wd += step, wmr += step) {
        double2 X;
        if (t == 0) X = cadd(v0, A0);
        else X = cadd(v0, cconj(buf[WF::pi(s_q[t])]));
        const double2 g = s_gi[t];
        const double zr = X.x * g.x - X.y * g.y;
        const double zi = X.x * g.y + X.y * g.x;
        zr2 = fma(zr, zr, zr2);
        zi2 = fma(zi, zi, zi2);
        *wd = c * zr;
        if (hm) *wmr = c2 * zr;
      }
    }
    const double cc = c * c + c2 * c2;
    sre = fma(cc, zr2, sre);
    sim = fma(cc, zi2, sim);
    __syncwarp();   // buf is rewritten by the next mode
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
  }
}
template <int NL> constexpr size_t rader_smem() { return sizeof(double2) * RaderPlan<NL>::WF::words * RaderPlan<NL>::S; }

template <int NL> constexpr size_t blue_smem() {
  using P = BluePlan<NL>;
  return sizeof(double2) * SeqMajorPad<P::L, P::R1>::words(P::S);
}

}  // namespace fastk
}  // namespace bhcp
