// bhcp_b200.cu -- sm_100a kernels and the C ABI (include/bhcp_b200.h) of the
// PinT QBVM/MQBVM direct solver.
//
// Reference path (pkg/src/bhcp): solve_pint (pint.py:69-110) =
//   (a) to_eigenspace: ifft_ortho(rhs * gamma) along time   (circulant.py:99-106)
//   (b) per level j: DST, divide by s_j + mu_k, DST          (pint.py:26-66, space.py:249-283)
//   (c) from_eigenspace: fft_ortho / gamma, residue, Re      (circulant.py:108-115, 167-190)
// Kernels here:
//   k_time        general time-axis transforms (steps (a)/(c), any layout)
//   k_dst_rows    DST-I along the contiguous spatial axis (+ fused 1D shifted solve)
//   k_dst_cols    DST-I along a strided spatial axis (+ fused divide on the outer axis)
//   k_modes       fused solve pass A: shifts -> time FFT -> Gamma^-1 -> Re, per mode
//   k_rhs, k_transpose, k_scale helpers
// All arithmetic is fp64; no tensor cores (the work is FFT/elementwise).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <mutex>
#include <string>
#include <vector>
#include <algorithm>

#include "../../include/bhcp_b200.h"
#include "fft_engine.cuh"
#include "plan.h"

namespace bhcp {

struct StatusDev {
  unsigned long long bad_col;  // first singular column, ULLONG_MAX if none
  double sum_re2;              // sum of (Re Y)^2
  double sum_im2;              // sum of (Im Y)^2
  unsigned long long work;     // pass-A work counter (dynamic scheduling; 0 between launches)
  unsigned long long done;     // CTAs finished (the last one resets work and done)
  double pad[3];
};
static_assert(sizeof(StatusDev) == 64, "status block is 64 bytes");

constexpr size_t kSmemBudget = 200 * 1024;

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// Block-wide sum of two doubles; result valid in thread 0. Deterministic tree.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) { red[2 * w] = a; red[2 * w + 1] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int i = 0; i < nw; ++i) { s0 += red[2 * i]; s1 += red[2 * i + 1]; }
    a = s0; b = s1;
  }
}

__device__ __forceinline__ void flag_singular(StatusDev* st, long long col) {
  atomicMin(&st->bad_col, (unsigned long long)col);
}

// mu for flattened mode index (C order, first axis outermost) -- same
// association as numpy add.outer (space.py:215). 3D (no reference; restated):
// the sum of the sorted triple, (mu1[lo] + mu1[mid]) + mu1[hi], so all six
// permutations of a mode share one bit-identical mu (one time FFT serves them,
// k_modes_rader sym6); within an ulp of the C-order sum.
__device__ __forceinline__ double mode_mu(const double* __restrict__ mu1, int m, int dim, long long k) {
  if (dim == 1) return __ldg(mu1 + k);
  if (dim == 2) {
    const int k1 = (int)(k / m), k2 = (int)(k - (long long)k1 * m);
    return __ldg(mu1 + k1) + __ldg(mu1 + k2);
  }
  const long long mm = (long long)m * m;
  int k1 = (int)(k / mm);
  const long long r = k - k1 * mm;
  int k2 = (int)(r / m), k3 = (int)(r - (long long)k2 * m);
  if (k1 > k2) { const int t = k1; k1 = k2; k2 = t; }
  if (k2 > k3) { const int t = k2; k2 = k3; k3 = t; }
  if (k1 > k2) { const int t = k1; k1 = k2; k2 = t; }
  return (__ldg(mu1 + k1) + __ldg(mu1 + k2)) + __ldg(mu1 + k3);
}

// Divide by (s + mu) the way numpy does complex / complex for these operands:
// x * conj(den) / |den|^2. Flags the column when |s + mu| <= 1e-14 |s|
// (space.py:237-240).
__device__ __forceinline__ double2 shifted_divide(double2 x, double2 s, double mu, StatusDev* st,
                                                  long long col) {
  const double dr = s.x + mu, di = s.y;
  const double den2 = dr * dr + di * di;
  const double s2 = s.x * s.x + s.y * s.y;
  if (den2 <= 1e-28 * s2) flag_singular(st, col);
  const double inv = 1.0 / den2;
  return make_double2((x.x * dr + x.y * di) * inv, (x.y * dr - x.x * di) * inv);
}

}  // namespace bhcp
#include "fast_kernels.cuh"
#include "gather_dst.cuh"
#include "gt_modes.cuh"
#include "pf_modes.cuh"
#include "wax_dst.cuh"
#include "wax2_dst.cuh"
#include "lvl_dst.cuh"
#include <cudaTypedefs.h>
namespace bhcp {

template <int V> struct VT;
template <> struct VT<V256> { static constexpr int T = 256, CAP = 16, MINB = 2; };
template <> struct VT<V512> { static constexpr int T = 512, CAP = 16, MINB = 1; };
template <> struct VT<V768> { static constexpr int T = 768, CAP = 12, MINB = 1; };

// ------------------------------------------------------------------ DST helpers
// Orthonormal DST-I of length m via a complex FFT of length L = 2(m+1) of the
// odd extension [0, x_1..x_m, 0, -x_m..-x_1]: X_k = -2i sum_j x_j sin(pi jk/(m+1)),
// so DST_k = sqrt(2/(m+1)) * (i/2) X_k. Real data are packed two lines per
// complex sequence (DST is real-linear), complex lines one per sequence.
__device__ __forceinline__ void dst_put(const FftPlanDev& p, double2* buf, int ld, int seq, int m,
                                        int e, double2 x) {
  if (p.blue) {
    buf[seq * ld + e + 1] = cmul(x, __ldg(p.chirp + e + 1));
    buf[seq * ld + p.L - 1 - e] = cmul(make_double2(-x.x, -x.y), __ldg(p.chirp + p.L - 1 - e));
  } else {
    buf[seq * ld + e + 1] = x;
    buf[seq * ld + p.L - 1 - e] = make_double2(-x.x, -x.y);
  }
}
__device__ __forceinline__ void dst_put_zeros(const FftPlanDev& p, double2* buf, int ld, int nseq, int m) {
  // positions 0 and m+1 of each sequence, plus the Bluestein tail
  for (int q = threadIdx.x; q < nseq; q += blockDim.x) {
    buf[q * ld] = make_double2(0.0, 0.0);
    buf[q * ld + m + 1] = make_double2(0.0, 0.0);
  }
  if (p.blue) {
    const int pad = p.Lc - p.L;
    for (int i = threadIdx.x; i < nseq * pad; i += blockDim.x) {
      const int q = i / pad;
      buf[q * ld + p.L + (i - q * pad)] = make_double2(0.0, 0.0);
    }
  }
}
__device__ __forceinline__ double2 gen_get(const FftPlanDev& p, const double2* buf, int ld, int seq, int k) {
  double2 x = buf[seq * ld + k];
  if (p.blue) x = cmul(cconj(x), __ldg(p.chirp + k));
  return x;
}
__device__ __forceinline__ void gen_put(const FftPlanDev& p, double2* buf, int ld, int seq, int j, double2 x) {
  if (p.blue) x = cmul(x, __ldg(p.chirp + j));
  buf[seq * ld + j] = x;
}
__device__ __forceinline__ void gen_zero_tail(const FftPlanDev& p, double2* buf, int ld, int nseq) {
  if (!p.blue) return;
  const int pad = p.Lc - p.L;
  for (int i = threadIdx.x; i < nseq * pad; i += blockDim.x) {
    const int q = i / pad;
    buf[q * ld + p.L + (i - q * pad)] = make_double2(0.0, 0.0);
  }
}

// Stockham core over nseq sequences of stride ld. V768 only instantiates the
// {2,3,4,5} stages (its plans are factored with those radices only) to keep
// the register budget of 768-thread CTAs.
template <int V, int CAP> struct BigStage {
  static __device__ __forceinline__ void run(int R, double2* buf, int nseq, int Lc, int ld, int Ns,
                                             const double2* tw) {
    switch (R) {
      case 7: fft_stage_ld<7, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 8: fft_stage_ld<8, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 11: fft_stage_ld<11, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 13: fft_stage_ld<13, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 17: fft_stage_ld<17, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 19: fft_stage_ld<19, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      case 23: fft_stage_ld<23, CAP>(buf, nseq, Lc, ld, Ns, tw); break;
      default: __trap();
    }
  }
};
template <int CAP> struct BigStage<V768, CAP> {
  static __device__ __forceinline__ void run(int, double2*, int, int, int, int, const double2*) { __trap(); }
};

template <int V>
__device__ __forceinline__ void fft_run(const FftPlanDev& p, double2* buf, int ld, int nseq) {
  constexpr int CAP = VT<V>::CAP;
  int Ns = 1;
  for (int s = 0; s < p.nst; ++s) {
    const int R = p.radix[s];
    switch (R) {
      case 2: fft_stage_ld<2, CAP>(buf, nseq, p.Lc, ld, Ns, p.tw); break;
      case 3: fft_stage_ld<3, CAP>(buf, nseq, p.Lc, ld, Ns, p.tw); break;
      case 4: fft_stage_ld<4, CAP>(buf, nseq, p.Lc, ld, Ns, p.tw); break;
      case 5: fft_stage_ld<5, CAP>(buf, nseq, p.Lc, ld, Ns, p.tw); break;
      default: BigStage<V, CAP>::run(R, buf, nseq, p.Lc, ld, Ns, p.tw);
    }
    Ns *= R;
  }
}

template <int V>
__device__ __forceinline__ void fft_exec_ld(const FftPlanDev& p, double2* buf, int ld, int nseq) {
  fft_run<V>(p, buf, ld, nseq);
  if (p.blue) {
    for (int i = threadIdx.x; i < nseq * p.Lc; i += blockDim.x) {
      const int q = i / p.Lc;
      const int k = i - q * p.Lc;
      double2* x = buf + q * ld + k;
      *x = cconj(cmul(*x, __ldg(p.bhat + k)));
    }
    __syncthreads();
    fft_run<V>(p, buf, ld, nseq);
  }
}

// ------------------------------------------------------------------ k_time
// MODE 0 (step a): out = ifft_ortho(in * gamma)   -- circulant.py:99-106
// MODE 1 (step c): Y = fft_ortho(in) * gamma_inv  -- circulant.py:108-115, 182-190
struct TimeArgs {
  FftPlanDev p;
  int ld, nseq, n;
  const double* in;
  int in_cplx;
  long long B, in_sb, in_st;
  double* out;
  int out_cplx;
  long long out_sb, out_st;
  const double2* gam;  // gamma (MODE 0) or gamma_inv (MODE 1)
  double scale;        // 1/sqrt(n)
  StatusDev* st;
};

template <int V, int MODE>
__global__ void __launch_bounds__(VT<V>::T, VT<V>::MINB) k_time(TimeArgs a) {
  extern __shared__ double2 smem[];
  __shared__ double red[64];
  const int n = a.n, nseq = a.nseq;
  const long long q0 = (long long)blockIdx.x * nseq;
  const bool rows_in = (a.in_st == 1);
  gen_zero_tail(a.p, smem, a.ld, nseq);
  for (int i = threadIdx.x; i < nseq * n; i += blockDim.x) {
    int q, t;
    if (rows_in) { q = i / n; t = i - q * n; } else { t = i / nseq; q = i - t * nseq; }
    const long long qq = q0 + q;
    double2 x = make_double2(0.0, 0.0);
    if (qq < a.B) {
      const long long off = qq * a.in_sb + (long long)t * a.in_st;
      if (a.in_cplx) x = ld2(a.in + 2 * off); else x = make_double2(a.in[off], 0.0);
    }
    if (MODE == 0) {
      x = cconj(cmul(x, __ldg(a.gam + t)));  // inverse DFT via conj(FFT(conj))
    }
    gen_put(a.p, smem, a.ld, q, t, x);
  }
  __syncthreads();
  fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  const bool rows_out = (a.out_st == 1);
  double sre = 0.0, sim = 0.0;
  for (int i = threadIdx.x; i < nseq * n; i += blockDim.x) {
    int q, t;
    if (rows_out) { q = i / n; t = i - q * n; } else { t = i / nseq; q = i - t * nseq; }
    const long long qq = q0 + q;
    if (qq >= a.B) continue;
    double2 X = gen_get(a.p, smem, a.ld, q, t);
    const long long off = qq * a.out_sb + (long long)t * a.out_st;
    if (MODE == 0) {
      X = cconj(X);
      X.x *= a.scale; X.y *= a.scale;
      reinterpret_cast<double2*>(a.out)[off] = X;
    } else {
      X.x *= a.scale; X.y *= a.scale;
      const double2 Y = cmul(X, __ldg(a.gam + t));
      sre = fma(Y.x, Y.x, sre);
      sim = fma(Y.y, Y.y, sim);
      if (a.out_cplx) reinterpret_cast<double2*>(a.out)[off] = Y; else a.out[off] = Y.x;
    }
  }
  if (MODE == 1) {
    block_sum2(sre, sim, red);
    if (threadIdx.x == 0) {
      atomicAdd(&a.st->sum_re2, sre);
      atomicAdd(&a.st->sum_im2, sim);
    }
  }
}

// ------------------------------------------------------------------ DST kernels
// EPI 0: plain orthonormal DST.
// EPI 1: DST, divide by (shift[level] + mu[mode]), DST  (fused shifted solve on
//        the outermost spatial axis; level/mode from the line geometry).
struct DstArgs {
  FftPlanDev p;
  int ld, nseq, m, dim;
  const double* in;
  double* out;
  long long nlines;      // rows kernel: number of lines (real or complex)
  long long nseqs;       // rows kernel: number of FFT sequences
  long long lpl;         // rows kernel, real data: lines per level (pairing, see fastk::pair_lines)
  long long ni, no;      // cols kernel: inner / outer line counts
  long long es, os;      // cols kernel: element / outer strides (elements)
  double f;              // sqrt(2/(m+1)) / 2
  const double2* shifts; // EPI 1
  const double* mu1;     // EPI 1
  int axis_depth;        // cols kernel: 1 = axis -2, 2 = axis -3
  StatusDev* st;
  // rows kernel, blocked input (slab all-to-all buffer): line (t, k1, r) at
  // koff[k1] + t * kstride[k1] + r * m; null koff = contiguous lines
  const long long* koff;
  const long long* kstride;
  long long lines_per_level, inner_div;
};

__device__ __forceinline__ long long line_base(const DstArgs& a, long long l) {
  if (!a.koff) return l * a.m;
  const long long t = l / a.lines_per_level;
  const long long rem = l - t * a.lines_per_level;
  const long long k1 = rem / a.inner_div;
  const long long r2 = rem - k1 * a.inner_div;
  return __ldg(a.koff + k1) + t * __ldg(a.kstride + k1) + r2 * a.m;
}

// k-th DST coefficient (1-based k) of sequence seq from the FFT buffer.
__device__ __forceinline__ double2 dst_coef(const DstArgs& a, const double2* buf, int seq, int k) {
  const double2 X = gen_get(a.p, buf, a.ld, seq, k);
  return make_double2(-a.f * X.y, a.f * X.x);
}

// Rows: lines are contiguous; line l occupies [l*m, (l+1)*m).
template <int V, int CPLX, int EPI>
__global__ void __launch_bounds__(VT<V>::T, VT<V>::MINB) k_dst_rows(DstArgs a) {
  extern __shared__ double2 smem[];
  constexpr int CAP = VT<V>::CAP;
  const int m = a.m, nseq = a.nseq;
  const long long s0 = (long long)blockIdx.x * nseq;  // first sequence of the CTA
  dst_put_zeros(a.p, smem, a.ld, nseq, m);
  for (int i = threadIdx.x; i < nseq * m; i += blockDim.x) {
    const int q = i / m, e = i - q * m;
    const long long s = s0 + q;
    double2 x = make_double2(0.0, 0.0);
    if (CPLX) {
      if (s < a.nlines) x = ld2(a.in + 2 * (s * m + e));
    } else if (s < a.nseqs) {
      long long l0, l1;
      fastk::pair_lines(s, a.nlines, a.lpl, l0, l1);
      if (l0 >= 0) x.x = a.in[line_base(a, l0) + e];
      if (l1 >= 0) x.y = a.in[line_base(a, l1) + e];
    }
    dst_put(a.p, smem, a.ld, q, m, e, x);
  }
  __syncthreads();
  fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  if (EPI == 1) {
    // divide in registers, then rebuild the odd extension and transform again
    constexpr int MAXI = CAP / 2 + 1;
    double2 hold[MAXI];
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      if (i < nseq * m) {
        const int q = i / m, e = i - q * m;
        const long long s = s0 + q;
        double2 c = dst_coef(a, smem, q, e + 1);
        if (s < a.nlines) c = shifted_divide(c, a.shifts[s], __ldg(a.mu1 + e), a.st, s);
        hold[u] = c;
      }
    }
    __syncthreads();
    dst_put_zeros(a.p, smem, a.ld, nseq, m);
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      if (i < nseq * m) {
        const int q = i / m, e = i - q * m;
        dst_put(a.p, smem, a.ld, q, m, e, hold[u]);
      }
    }
    __syncthreads();
    fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  }
  for (int i = threadIdx.x; i < nseq * m; i += blockDim.x) {
    const int q = i / m, e = i - q * m;
    const long long s = s0 + q;
    const double2 c = dst_coef(a, smem, q, e + 1);
    if (CPLX) {
      if (s < a.nlines) reinterpret_cast<double2*>(a.out)[s * m + e] = c;
    } else if (s < a.nseqs) {
      long long l0, l1;
      fastk::pair_lines(s, a.nlines, a.lpl, l0, l1);
      if (l0 >= 0) a.out[l0 * m + e] = c.x;
      if (l1 >= 0) a.out[l1 * m + e] = c.y;
    }
  }
}

// Cols: element e of line (o, i) at o*os + i + e*es; the CTA takes one outer
// index and a tile of consecutive inner indices (coalesced loads/stores).
template <int V, int CPLX, int EPI>
__global__ void __launch_bounds__(VT<V>::T, VT<V>::MINB) k_dst_cols(DstArgs a) {
  extern __shared__ double2 smem[];
  constexpr int CAP = VT<V>::CAP;
  const int m = a.m, nseq = a.nseq;
  const int lines_per_cta = CPLX ? nseq : 2 * nseq;
  const long long ntile = (a.ni + lines_per_cta - 1) / lines_per_cta;
  const long long o = blockIdx.x / ntile;
  const long long i0 = (blockIdx.x - o * ntile) * lines_per_cta;
  const double* base_in = a.in + (CPLX ? 2 : 1) * (o * a.os);
  double* base_out = a.out + (CPLX ? 2 : 1) * (o * a.os);
  dst_put_zeros(a.p, smem, a.ld, nseq, m);
  for (int idx = threadIdx.x; idx < nseq * m; idx += blockDim.x) {
    const int e = idx / nseq, q = idx - e * nseq;
    double2 x = make_double2(0.0, 0.0);
    if (CPLX) {
      const long long i = i0 + q;
      if (i < a.ni) x = ld2(base_in + 2 * (i + e * a.es));
    } else {
      const long long i = i0 + 2 * q;
      if (i < a.ni) x.x = base_in[i + e * a.es];
      if (i + 1 < a.ni) x.y = base_in[i + 1 + e * a.es];
    }
    dst_put(a.p, smem, a.ld, q, m, e, x);
  }
  __syncthreads();
  fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  if (EPI == 1) {
    constexpr int MAXI = CAP / 2 + 1;
    double2 hold[MAXI];
    const double2 sh = a.shifts[o];  // outermost axis: o enumerates levels
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int idx = threadIdx.x + u * blockDim.x;
      if (idx < nseq * m) {
        const int e = idx / nseq, q = idx - e * nseq;
        const long long i = i0 + q;
        double2 c = dst_coef(a, smem, q, e + 1);
        if (i < a.ni) {
          double mu;
          if (a.axis_depth == 1) {
            mu = __ldg(a.mu1 + e) + __ldg(a.mu1 + i);
          } else {
            const int k2 = (int)(i / m), k3 = (int)(i - (long long)k2 * m);
            mu = (__ldg(a.mu1 + e) + __ldg(a.mu1 + k2)) + __ldg(a.mu1 + k3);
          }
          c = shifted_divide(c, sh, mu, a.st, o);
        }
        hold[u] = c;
      }
    }
    __syncthreads();
    dst_put_zeros(a.p, smem, a.ld, nseq, m);
#pragma unroll
    for (int u = 0; u < MAXI; ++u) {
      const int idx = threadIdx.x + u * blockDim.x;
      if (idx < nseq * m) {
        const int e = idx / nseq, q = idx - e * nseq;
        dst_put(a.p, smem, a.ld, q, m, e, hold[u]);
      }
    }
    __syncthreads();
    fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  }
  for (int idx = threadIdx.x; idx < nseq * m; idx += blockDim.x) {
    const int e = idx / nseq, q = idx - e * nseq;
    const double2 c = dst_coef(a, smem, q, e + 1);
    if (CPLX) {
      const long long i = i0 + q;
      if (i < a.ni) reinterpret_cast<double2*>(base_out)[i + e * a.es] = c;
    } else {
      const long long i = i0 + 2 * q;
      if (i < a.ni) base_out[i + e * a.es] = c.x;
      if (i + 1 < a.ni) base_out[i + 1 + e * a.es] = c.y;
    }
  }
}

// ------------------------------------------------------------------ k_modes
// Fused solve, pass A: for spatial mode k,
//   W[t, k] = ghat_k * Re( gamma_inv_t * sum_j exp(-2 pi i jt/n) / (s_j + mu_k) )
// ghat already carries DST(g) / (divisor * n).
struct ModesArgs {
  FftPlanDev p;
  int ld, nseq, n, m, dim;
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;         // 1 / (divisor * n) applied to ghat
  long long k_begin, k_count;
  double* W;
  fastk::WLayout wl;
  StatusDev* st;
};

template <int V>
__global__ void __launch_bounds__(VT<V>::T, VT<V>::MINB) k_modes(ModesArgs a) {
  extern __shared__ double2 smem[];
  __shared__ double red[64];
  __shared__ double s_mu[64];
  __shared__ double s_c[64];
  const int n = a.n, nseq = a.nseq;
  const long long kl0 = (long long)blockIdx.x * nseq;  // local mode offset
  for (int q = threadIdx.x; q < nseq; q += blockDim.x) {
    const long long kl = kl0 + q;
    if (kl < a.k_count) {
      const long long k = a.k_begin + kl;
      s_mu[q] = mode_mu(a.mu1, a.m, a.dim, k);
      s_c[q] = a.ghat[k] * a.cscale;
    } else {
      s_mu[q] = 0.0;
      s_c[q] = 0.0;
    }
  }
  gen_zero_tail(a.p, smem, a.ld, nseq);
  __syncthreads();
  for (int i = threadIdx.x; i < nseq * n; i += blockDim.x) {
    const int q = i / n, j = i - q * n;
    const double2 s = __ldg(a.shifts + j);
    double2 v = make_double2(0.0, 0.0);
    if (kl0 + q < a.k_count) {
      const double dr = s.x + s_mu[q], di = s.y;
      const double den2 = dr * dr + di * di;
      if (den2 <= 1e-28 * (s.x * s.x + s.y * s.y)) flag_singular(a.st, j);
      const double inv = 1.0 / den2;
      v = make_double2(dr * inv, -di * inv);
    }
    gen_put(a.p, smem, a.ld, q, j, v);
  }
  __syncthreads();
  fft_exec_ld<V>(a.p, smem, a.ld, nseq);
  double sre = 0.0, sim = 0.0;
  for (int i = threadIdx.x; i < nseq * n; i += blockDim.x) {
    const int t = i / nseq, q = i - t * nseq;
    const long long kl = kl0 + q;
    if (kl >= a.k_count) continue;
    const double2 X = gen_get(a.p, smem, a.ld, q, t);
    const double2 Z = cmul(X, __ldg(a.gaminv + t));
    const double c = s_c[q];
    const double wr = c * Z.x, wi = c * Z.y;
    sre = fma(wr, wr, sre);
    sim = fma(wi, wi, sim);
    *a.wl.ptr(kl, t) = wr;
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
  }
}

// ------------------------------------------------------------------ small kernels
__global__ void k_status_reset_n(StatusDev* st, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    st[i].bad_col = ~0ull;
    st[i].sum_re2 = 0.0;
    st[i].sum_im2 = 0.0;
    st[i].work = 0;
    st[i].done = 0;
  }
}
__global__ void k_status_reset(StatusDev* st) {
  if (threadIdx.x == 0) {
    st->bad_col = ~0ull;
    st->sum_re2 = 0.0;
    st->sum_im2 = 0.0;
    st->work = 0;
    st->done = 0;
  }
}

// rhs block of methods.py:158-162: zeros with row 0 = g / divisor.
__global__ void k_rhs(const double* __restrict__ g, double inv_divisor_mul, double divisor, long long nx,
                      long long total, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    out[i] = (i < nx) ? g[i] / divisor : 0.0;
  }
}

__global__ void k_scale(const double* __restrict__ in, double s, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i] * s;
}

// out[c * rows + r] = in[r * ld + c], r < rows, c < cols (32x32 tiles through shared memory)
__global__ void k_transpose_ld(const double* __restrict__ in, long long ld, double* __restrict__ out, long long rows,
                               long long cols) {
  __shared__ double tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * ld + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][dy];
  }
}

// k_transpose_ld over a batch of matrices (blockIdx.z): in + z * in_stride -> out + z * rows * cols
__global__ void k_transpose_ld_batch(const double* __restrict__ in, long long ld, long long in_stride,
                                     double* __restrict__ out, long long rows, long long cols) {
  __shared__ double tile[32][33];
  const double* src = in + (long long)blockIdx.z * in_stride;
  double* dst = out + (long long)blockIdx.z * rows * cols;
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = src[r * ld + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][dy];
  }
}

template <typename E>
__global__ void k_transpose(const E* __restrict__ in, E* __restrict__ out, long long rows, long long cols) {
  __shared__ E tile[32][33];
  const long long c0 = (long long)blockIdx.x * 32, r0 = (long long)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const long long c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][dy];
  }
}

// ------------------------------------------------------------------ residual
// Relative residual of the all-at-once system for the pint kinds
// (methods.py:164-171, 239-247, residual_norm 281-285): r = rhs - A y with
//   (A y)_0 = y_0 / tau + corner * y_N - lap y_0,   (A y)_t = (y_t - y_{t-1}) / tau - lap y_t,
//   rhs_0 = g / divisor, rhs_t = 0, corner = 1 / divisor.
// 3/5/7-point Dirichlet Laplacian on the interior grid. Each CTA writes the
// partial sums of |r|^2 and |rhs|^2; k_residual_finish reduces them in a
// fixed order (deterministic).
struct ResidualArgs {
  const double* y;
  const double* g;
  long long n, nx;
  int m, dim;
  double inv_tau, corner, inv_div, inv_h2;
  double* partial;  // 2 * gridDim.x
};

__device__ __forceinline__ double lap_at(const double* __restrict__ f, long long x, int m, int dim, double inv_h2) {
  // x = flattened interior index (C order)
  double s;
  if (dim == 1) {
    const int i = (int)x;
    s = -2.0 * f[x];
    if (i > 0) s += f[x - 1];
    if (i + 1 < m) s += f[x + 1];
  } else if (dim == 2) {
    const int i1 = (int)(x / m), i2 = (int)(x - (long long)i1 * m);
    s = -4.0 * f[x];
    if (i2 > 0) s += f[x - 1];
    if (i2 + 1 < m) s += f[x + 1];
    if (i1 > 0) s += f[x - m];
    if (i1 + 1 < m) s += f[x + m];
  } else {
    const long long mm = (long long)m * m;
    const int i1 = (int)(x / mm);
    const long long r = x - i1 * mm;
    const int i2 = (int)(r / m), i3 = (int)(r - (long long)i2 * m);
    s = -6.0 * f[x];
    if (i3 > 0) s += f[x - 1];
    if (i3 + 1 < m) s += f[x + 1];
    if (i2 > 0) s += f[x - m];
    if (i2 + 1 < m) s += f[x + m];
    if (i1 > 0) s += f[x - mm];
    if (i1 + 1 < m) s += f[x + mm];
  }
  return s * inv_h2;
}

__global__ void __launch_bounds__(256) k_residual(ResidualArgs a) {
  __shared__ double red[16];
  double rr = 0.0, bb = 0.0;
  const long long total = a.n * a.nx;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (long long)gridDim.x * 256) {
    const long long t = i / a.nx, x = i - t * a.nx;
    const double* yt = a.y + t * a.nx;
    double ay = (t == 0) ? yt[x] * a.inv_tau + a.corner * a.y[(a.n - 1) * a.nx + x]
                         : (yt[x] - yt[x - a.nx]) * a.inv_tau;
    ay -= lap_at(yt, x, a.m, a.dim, a.inv_h2);
    const double rhs = (t == 0) ? a.g[x] * a.inv_div : 0.0;
    const double r = rhs - ay;
    rr = fma(r, r, rr);
    bb = fma(rhs, rhs, bb);
  }
  block_sum2(rr, bb, red);
  if (threadIdx.x == 0) {
    a.partial[2 * blockIdx.x] = rr;
    a.partial[2 * blockIdx.x + 1] = bb;
  }
}

__global__ void k_residual_finish(const double* __restrict__ partial, int nblk, double* out) {
  __shared__ double red[64];
  double rr = 0.0, bb = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    rr += partial[2 * i];
    bb += partial[2 * i + 1];
  }
  block_sum2(rr, bb, red);
  if (threadIdx.x == 0) {
    out[0] = rr;
    out[1] = bb;
  }
}

// ------------------------------------------------------------------ closed form
// Device form of the reference's per-mode closed-form solver
// solve_spectral_oracle (baseline.py:67-112) and of march_forward's per-mode
// identity (baseline.py:115-129): W(k, t) = amp_k * rho_k^t in the blocked
// layout, then the same level passes as the solve. kind: 0 qbvm, 1 mqbvm,
// 2 pint-qbvm, 3 pint-mqbvm (baseline.py:92-99 denominators).
struct SpectralArgs {
  const double* ghat;    // DST(data)
  const double* mu1;
  int m, dim, kind;
  double alpha, tau;
  long long num_steps, n;  // N and n = N + 1 (levels written: n)
  double* W;
  fastk::WLayout wl;
};

__global__ void k_spectral_w(SpectralArgs a, long long nx) {
  for (long long k = blockIdx.x * (long long)blockDim.y + threadIdx.y; k < nx; k += (long long)gridDim.x * blockDim.y) {
    const double mu = mode_mu(a.mu1, a.m, a.dim, k);
    const double rho = 1.0 / (1.0 + a.tau * mu);
    const double decay = pow(rho, (double)a.num_steps);
    double denom;
    if (a.kind == 0) denom = a.alpha + decay;
    else if (a.kind == 1) denom = a.alpha * mu * rho + decay;
    else if (a.kind == 2) denom = a.alpha * (1.0 + a.tau * mu) + decay;
    else denom = a.alpha * (mu + 1.0 / a.tau) + decay;
    const double amp = a.ghat[k] / denom;
    for (long long t = threadIdx.x; t < a.n; t += blockDim.x)
      *a.wl.ptr(k, (int)t) = amp * pow(rho, (double)t);
  }
}

// x_k <- x_k * rho_k^N  (march_forward in per-mode form, in place)
__global__ void k_decay(double* x, const double* __restrict__ mu1, int m, int dim, double tau, double N, long long nx) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nx; k += (long long)gridDim.x * blockDim.x) {
    const double rho = 1.0 / (1.0 + tau * mode_mu(mu1, m, dim, k));
    x[k] *= pow(rho, N);
  }
}

}  // namespace bhcp

// ====================================================================== host
using namespace bhcp;

struct bhcp_space_plan {
  int device, dim, num_cells, m;
  long long nx;          // m^dim interior unknowns
  double* mu1_dev;       // m doubles
  FftPlanHost dst;       // FFT of length 2(m+1)
  int2* tiles_dev;       // 2D: upper-triangle 4x4 mode tiles (a, b), a <= b
  long long ntiles;
  double2* twN;          // exp(-2 pi i k / N), N = m + 1 (half-length DST kernels)
  double* snN;           // sin(pi j / N)
  double mu_lo, mu_hi;   // range of the mode eigenvalues: dim * mu1_min, dim * mu1_max (host)
  int4* seg_tiles[9];    // symmetric segment tiles of the Bluestein / Rader / Good-Thomas modes kernels,
  long long seg_count[9];   // one slot per segment length seg_len[slot]
  int seg_len[9];
};

struct bhcp_time_plan {
  int device, n;
  double2* tables;       // gamma | gamma_inv | shifts  (3n double2)
  FftPlanHost fft;       // FFT of length n
  double2* blue;         // n = 2^p + 1 fast path: tw (L) | chirp (n) | bhat (L) | wM (n), L = 2(n-1)
  double2* rader;        // prime n = 2^p + 1: tw (n-1) | bhat (n-1)
  int* rader_idx;        //                    perm (n-1) | qidx (n)
  double2* gt;           // n = 1025: plan.h kGt2* layout (generator shifts, twiddles, 1/gamma, bhat40)
  int* gt_idx;           //           stage-C lane map | row slots | powers of g
  std::vector<double2> shifts_h;   // host copy of the shifts (may_be_singular)
  double2* pf;           // n = 4097: w240 | bhat240 | shifts in prime-factor order (4097)
  int* pf_idx;           //           tq241 (240): g^-q mod 241
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(const char* what) {
  cudaError_t e = cudaGetLastError();
  return fail(BHCP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

std::mutex g_init_mutex;
bool g_init_done[64] = {false};

int g_smem_optin = 0;

template <typename K>
void allow_smem(K kernel) {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kernel) != cudaSuccess) return;
  const int dyn = g_smem_optin - (int)fa.sharedSizeBytes;
  if (dyn > 0) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
}

#define BHCP_FOR_VARIANTS(X) X(V256) X(V512) X(V768)

void set_all_attributes() {
#define BHCP_ATTR(VV)                                   \
  allow_smem(k_time<VV, 0>);                            \
  allow_smem(k_time<VV, 1>);                            \
  allow_smem(k_dst_rows<VV, 0, 0>);                     \
  allow_smem(k_dst_rows<VV, 1, 0>);                     \
  allow_smem(k_dst_rows<VV, 1, 1>);                     \
  allow_smem(k_dst_cols<VV, 0, 0>);                     \
  allow_smem(k_dst_cols<VV, 1, 0>);                     \
  allow_smem(k_dst_cols<VV, 1, 1>);                     \
  allow_smem(k_modes<VV>);
  BHCP_FOR_VARIANTS(BHCP_ATTR)
#undef BHCP_ATTR
#define BHCP_FATTR(LL)                                  \
  allow_smem(fastk::k_dst_rows_fast<LL, 0>);            \
  allow_smem(fastk::k_dst_rows_fast<LL, 1>);            \
  allow_smem(fastk::k_dst_cols_fast<LL, 0>);            \
  allow_smem(fastk::k_dst_cols_fast<LL, 1>);
  BHCP_FATTR(512) BHCP_FATTR(1024) BHCP_FATTR(2048) BHCP_FATTR(8192)
#undef BHCP_FATTR
  allow_smem(fastk::k_modes_blue<257, false>);
  allow_smem(fastk::k_modes_blue<257, true>);
  allow_smem(fastk::k_modes_blue<1025, false>);
  allow_smem(fastk::k_modes_blue<1025, true>);
  allow_smem(fastk::k_modes_blue<4097, false>);
  allow_smem(fastk::k_modes_blue<4097, true>);
  allow_smem(gdst::k_dst_blk2<256>);
  allow_smem(gdst::k_dst_blk2<512>);
  allow_smem(gdst::k_dst_blk2<1024>);
  allow_smem(gdst::k_dst_cols3<256>);
  allow_smem(gdst::k_dst_cols3<512>);
  allow_smem(gdst::k_dst_cols3<1024>);
  allow_smem(wax::k_dst_wax<wax::PlanWX<256>>);
  allow_smem(wax2::k_dst_wax2<512>);
  allow_smem(wax2::k_dst_blk3<512>);
  allow_smem(wax2::k_dst_blk3<256>);
  allow_smem(wax2::k_dst_blk4);
  allow_smem(lvl::k_dst_lvl4);

  allow_smem(fastk::k_modes_pf<false>);
  allow_smem(fastk::k_modes_pf<true>);
  allow_smem(fastk::k_modes_pf<false, true>);
  allow_smem(fastk::k_modes_gt<false, false, false>);
  allow_smem(fastk::k_modes_gt<true, false, false>);
  allow_smem(fastk::k_modes_gt<false, true, false>);
  allow_smem(fastk::k_modes_gt<true, true, false>);
  allow_smem(fastk::k_modes_gt<false, false, true>);
  allow_smem(fastk::k_modes_gt<true, false, true>);
  allow_smem(fastk::k_modes_gt<false, true, true>);
  allow_smem(fastk::k_modes_gt<true, true, true>);
  allow_smem(fastk::k_modes_rader<257, false>);
  allow_smem(fastk::k_modes_rader<257, true>);
  allow_smem(fastk::k_modes_fast<513, false>);
  allow_smem(fastk::k_modes_fast<513, true>);
}

// --- specialised fast paths (fast_kernels.cuh) ---------------------------------
int g_num_sms = 148;

// CTAs of `kernel` that fit on the device at once (persistent-grid size).
template <typename K>
long long resident_ctas(K kernel, int threads, size_t smem) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return (long long)per_sm * g_num_sms;
}
struct Blocked;
template <int L, class B>
void rows_fast(const bhcp_space_plan* sp, const double* in, double* out, int cplx, long long nlines,
               cudaStream_t s, const B& blk, long long lpl) {
  using namespace fastk;
  FastDstArgs a{};
  a.in = in; a.out = out; a.nlines = nlines; a.tw = sp->dst.d.tw; a.m = sp->m; a.lpl = lpl;
  a.koff = blk.koff; a.kstride = blk.kstride; a.lines_per_level = blk.lines_per_level; a.inner_div = blk.inner_div;
  a.f = sqrt(2.0 / (L / 2)) * 0.5;
  const long long seqs = cplx ? nlines : real_row_seqs(nlines, lpl);
  a.nseqs = seqs;
  long long grid = (seqs + RowsShape<L>::S - 1) / RowsShape<L>::S;
  grid = std::min<long long>(grid, cplx ? resident_ctas(k_dst_rows_fast<L, 1>, RowsShape<L>::T, rows_smem<L>())
                                        : resident_ctas(k_dst_rows_fast<L, 0>, RowsShape<L>::T, rows_smem<L>()));
  if (cplx) k_dst_rows_fast<L, 1><<<(unsigned)grid, RowsShape<L>::T, rows_smem<L>(), s>>>(a);
  else k_dst_rows_fast<L, 0><<<(unsigned)grid, RowsShape<L>::T, rows_smem<L>(), s>>>(a);
}

template <int L>
void cols_fast(const bhcp_space_plan* sp, const double* in, double* out, int cplx, long long ni, long long no,
               cudaStream_t s) {
  using namespace fastk;
  FastDstArgs a{};
  a.in = in; a.out = out; a.ni = ni; a.no = no; a.es = ni; a.os = (long long)sp->m * ni; a.tw = sp->dst.d.tw;
  a.f = sqrt(2.0 / (L / 2)) * 0.5;
  const int lines_per_cta = cplx ? ColsShape<L>::S : 2 * ColsShape<L>::S;
  long long grid = ((ni + lines_per_cta - 1) / lines_per_cta) * no;
  grid = std::min<long long>(grid, cplx ? resident_ctas(k_dst_cols_fast<L, 1>, ColsShape<L>::T, cols_smem<L>())
                                        : resident_ctas(k_dst_cols_fast<L, 0>, ColsShape<L>::T, cols_smem<L>()));
  if (cplx) k_dst_cols_fast<L, 1><<<(unsigned)grid, ColsShape<L>::T, cols_smem<L>(), s>>>(a);
  else k_dst_cols_fast<L, 0><<<(unsigned)grid, ColsShape<L>::T, cols_smem<L>(), s>>>(a);
}

bool fast_dst_length(int L) { return L == 512 || L == 1024 || L == 2048 || L == 8192; }
bool g_disable_fast = false;
int g_lvl4 = 1;          // BHCP_LVL4=0: c3 level phase as two sweeps (k_dst_blk4 + k_dst_cols3)
int g_lvl4_kfirst = -1;  // BHCP_LVL4_KFIRST: row-task pairs of a phase before its column tasks (default: grid)

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

size_t smem_bytes(const FftPlanHost& p, int nseq) { return size_t(nseq) * p.ld * sizeof(double2); }

// --- DST pass launchers --------------------------------------------------------
struct Blocked {
  const long long* koff = nullptr;
  const long long* kstride = nullptr;
  long long lines_per_level = 1, inner_div = 1;
};

int launch_rows(const bhcp_space_plan* sp, const double* in, double* out, int cplx, long long nlines,
                int epi, const double2* shifts, StatusDev* st, cudaStream_t s, const Blocked& blk = Blocked(),
                long long lpl = 1) {
  const FftPlanHost& P = sp->dst;
  if (!epi && !g_disable_fast && fast_dst_length(2 * (sp->m + 1)) && nlines > 0) {
    switch (2 * (sp->m + 1)) {
      case 512: rows_fast<512>(sp, in, out, cplx, nlines, s, blk, lpl); break;
      case 1024: rows_fast<1024>(sp, in, out, cplx, nlines, s, blk, lpl); break;
      case 2048: rows_fast<2048>(sp, in, out, cplx, nlines, s, blk, lpl); break;
      case 8192: rows_fast<8192>(sp, in, out, cplx, nlines, s, blk, lpl); break;
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_rows_fast launch");
    return BHCP_OK;
  }
  const int nseq_max = P.max_seqs(kSmemBudget);
  if (nseq_max < 1) return fail(BHCP_ERR_INVALID, "DST length does not fit the FFT engine");
  const long long seqs = cplx ? nlines : fastk::real_row_seqs(nlines, lpl);
  const int nseq = (int)(seqs < nseq_max ? seqs : nseq_max);
  if (seqs == 0) return BHCP_OK;
  DstArgs a{};
  a.p = P.d; a.ld = P.ld; a.nseq = nseq; a.m = sp->m; a.dim = sp->dim;
  a.in = in; a.out = out; a.nlines = nlines; a.nseqs = seqs; a.lpl = lpl;
  a.f = sqrt(2.0 / (sp->m + 1)) * 0.5;
  a.shifts = shifts; a.mu1 = sp->mu1_dev; a.st = st;
  a.koff = blk.koff; a.kstride = blk.kstride; a.lines_per_level = blk.lines_per_level; a.inner_div = blk.inner_div;
  const long long grid = (seqs + nseq - 1) / nseq;
  const size_t sm = smem_bytes(P, nseq);
#define BHCP_ROWS(VV)                                                                  \
  case VV:                                                                             \
    if (epi) k_dst_rows<VV, 1, 1><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);            \
    else if (cplx) k_dst_rows<VV, 1, 0><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);      \
    else k_dst_rows<VV, 0, 0><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);                \
    break;
  switch (P.variant) { BHCP_FOR_VARIANTS(BHCP_ROWS) }
#undef BHCP_ROWS
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_rows launch");
  return BHCP_OK;
}

int cols_blk2(const bhcp_space_plan* sp, const double* in, double* out, long long ni, long long no,
              cudaStream_t s);

int launch_cols(const bhcp_space_plan* sp, const double* in, double* out, int cplx, long long ni,
                long long no, int depth, int epi, const double2* shifts, StatusDev* st, cudaStream_t s) {
  const FftPlanHost& P = sp->dst;
  const int Lfull = 2 * (sp->m + 1);
  if (!epi && !cplx && !g_disable_fast && ni > 0 && no > 0 &&
      (Lfull == 512 || Lfull == 1024 || Lfull == 2048))
    return cols_blk2(sp, in, out, ni, no, s);
  if (!epi && !g_disable_fast && fast_dst_length(2 * (sp->m + 1)) && ni > 0 && no > 0) {
    switch (2 * (sp->m + 1)) {
      case 512: cols_fast<512>(sp, in, out, cplx, ni, no, s); break;
      case 1024: cols_fast<1024>(sp, in, out, cplx, ni, no, s); break;
      case 2048: cols_fast<2048>(sp, in, out, cplx, ni, no, s); break;
      case 8192: cols_fast<8192>(sp, in, out, cplx, ni, no, s); break;
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_cols_fast launch");
    return BHCP_OK;
  }
  const int nseq_max = P.max_seqs(kSmemBudget);
  if (nseq_max < 1) return fail(BHCP_ERR_INVALID, "DST length does not fit the FFT engine");
  const long long lines_needed = ni;
  long long seqs_needed = cplx ? lines_needed : (lines_needed + 1) / 2;
  const int nseq = (int)(seqs_needed < nseq_max ? seqs_needed : nseq_max);
  if (ni == 0 || no == 0) return BHCP_OK;
  DstArgs a{};
  a.p = P.d; a.ld = P.ld; a.nseq = nseq; a.m = sp->m; a.dim = sp->dim;
  a.in = in; a.out = out; a.ni = ni; a.no = no; a.es = ni; a.os = (long long)sp->m * ni;
  a.f = sqrt(2.0 / (sp->m + 1)) * 0.5;
  a.shifts = shifts; a.mu1 = sp->mu1_dev; a.axis_depth = depth; a.st = st;
  const int lines_per_cta = cplx ? nseq : 2 * nseq;
  const long long ntile = (ni + lines_per_cta - 1) / lines_per_cta;
  const long long grid = ntile * no;
  if (grid > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "grid too large");
  const size_t sm = smem_bytes(P, nseq);
#define BHCP_COLS(VV)                                                                  \
  case VV:                                                                             \
    if (epi) k_dst_cols<VV, 1, 1><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);            \
    else if (cplx) k_dst_cols<VV, 1, 0><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);      \
    else k_dst_cols<VV, 0, 0><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);                \
    break;
  switch (P.variant) { BHCP_FOR_VARIANTS(BHCP_COLS) }
#undef BHCP_COLS
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_cols launch");
  return BHCP_OK;
}

long long ipow(long long b, int e) {
  long long r = 1;
  while (e-- > 0) r *= b;
  return r;
}

// Orthonormal DST over all spatial axes of `batch` fields: axis -1, -2, -3.
int sine_passes(const bhcp_space_plan* sp, const double* in, double* out, int cplx, long long batch,
                cudaStream_t s) {
  const int d = sp->dim, m = sp->m;
  int rc = launch_rows(sp, in, out, cplx, batch * ipow(m, d - 1), 0, nullptr, nullptr, s, Blocked(),
                       ipow(m, d - 1));
  if (rc) return rc;
  for (int depth = 1; depth < d; ++depth) {
    rc = launch_cols(sp, out, out, cplx, ipow(m, depth), batch * ipow(m, d - 1 - depth), depth, 0,
                     nullptr, nullptr, s);
    if (rc) return rc;
  }
  return BHCP_OK;
}

// Step (b) on level-major complex fields: forward DST on the inner axes, a
// fused DST-divide-DST on the outermost axis, inverse DST on the inner axes.
int step_b_passes(const bhcp_space_plan* sp, const double* in, double* out, long long batch,
                  const double2* shifts, StatusDev* st, cudaStream_t s) {
  const int d = sp->dim, m = sp->m;
  if (d == 1) return launch_rows(sp, in, out, 1, batch, 1, shifts, st, s);
  int rc = launch_rows(sp, in, out, 1, batch * ipow(m, d - 1), 0, nullptr, nullptr, s);
  if (rc) return rc;
  for (int depth = 1; depth < d - 1; ++depth) {
    rc = launch_cols(sp, out, out, 1, ipow(m, depth), batch * ipow(m, d - 1 - depth), depth, 0, nullptr,
                     nullptr, s);
    if (rc) return rc;
  }
  rc = launch_cols(sp, out, out, 1, ipow(m, d - 1), batch, d - 1, 1, shifts, st, s);
  if (rc) return rc;
  for (int depth = d - 2; depth >= 1; --depth) {
    rc = launch_cols(sp, out, out, 1, ipow(m, depth), batch * ipow(m, d - 1 - depth), depth, 0, nullptr,
                     nullptr, s);
    if (rc) return rc;
  }
  return launch_rows(sp, out, out, 1, batch * ipow(m, d - 1), 0, nullptr, nullptr, s);
}

int launch_time(const bhcp_time_plan* tp, int mode, const double* in, int in_cplx, long long B, long long in_sb,
                long long in_st, double* out, int out_cplx, long long out_sb, long long out_st, StatusDev* st,
                cudaStream_t s) {
  if (B == 0) return BHCP_OK;
  if (in_st != 1 && in_sb != 1) return fail(BHCP_ERR_INVALID, "one input stride must be 1");
  const FftPlanHost& P = tp->fft;
  int nseq = P.max_seqs(kSmemBudget);
  if (nseq < 1) return fail(BHCP_ERR_INVALID, "time length does not fit the FFT engine");
  if (nseq > 32) nseq = 32;
  if (B < nseq) nseq = (int)B;
  TimeArgs a{};
  a.p = P.d; a.ld = P.ld; a.nseq = nseq; a.n = tp->n;
  a.in = in; a.in_cplx = in_cplx; a.B = B; a.in_sb = in_sb; a.in_st = in_st;
  a.out = out; a.out_cplx = out_cplx; a.out_sb = out_sb; a.out_st = out_st;
  a.gam = mode == 0 ? tp->tables : tp->tables + tp->n;
  a.scale = 1.0 / sqrt((double)tp->n);
  a.st = st;
  const long long grid = (B + nseq - 1) / nseq;
  const size_t sm = smem_bytes(P, nseq);
#define BHCP_TIME(VV)                                                             \
  case VV:                                                                        \
    if (mode == 0) k_time<VV, 0><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);        \
    else k_time<VV, 1><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a);                  \
    break;
  switch (P.variant) { BHCP_FOR_VARIANTS(BHCP_TIME) }
#undef BHCP_TIME
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_time launch");
  return BHCP_OK;
}


// Symmetric work list of the Bluestein modes kernel: 2D tiles (k1, k2a) cover
// k2 in [k2a, k2a+S) with k2 >= k1; 3D tiles (k1, k2, k3a) with k1 <= k2 cover
// k3 in [k3a, k3a+S). Each computed mode also writes its (k1 <-> k2) mirror.
// Optional window [begin, end) of the symmetric tile list of the modes kernel
// (multi-GPU: each rank computes a share of the upper triangle and stores
// both mirrors straight into their owners through per-slab block tables).
struct SymRange {
  bool on = false;
  long long begin = 0, end = -1;
};

// six = true (3D): tiles (k1, k2, k3a) of sorted triples k1 <= k2 <= k3, k3 in
// [k3a, k3a + S) with k3a stepping from k2 rounded down to S (k_modes_rader's
// one-FFT-per-permutation-class work list)
std::vector<int4> seg_list(int dim, int m, int S, bool six) {
  std::vector<int4> t;
  if (six && dim == 3) {
    for (int k1 = 0; k1 < m; ++k1)
      for (int k2 = k1; k2 < m; ++k2)
        for (int k3a = k2 - k2 % S; k3a < m; k3a += S) t.push_back(make_int4(k1, k2, k3a, 0));
  } else if (dim == 2) {
    for (int k1 = 0; k1 < m; ++k1)
      for (int k2a = k1 - k1 % S; k2a < m; k2a += S) t.push_back(make_int4(k1, k2a, 0, 0));
  } else {
    for (int k1 = 0; k1 < m; ++k1)
      for (int k2 = k1; k2 < m; ++k2)
        for (int k3a = 0; k3a < m; k3a += S) t.push_back(make_int4(k1, k2, k3a, 0));
  }
  return t;
}

// Number of tiles of seg_list without building it.
long long seg_list_count(int dim, int m, int S, bool six) {
  long long c = 0;
  if (six && dim == 3) {
    for (int k1 = 0; k1 < m; ++k1)
      for (int k2 = k1; k2 < m; ++k2) c += (m - (k2 - k2 % S) + S - 1) / S;
  } else if (dim == 2) {
    for (int k1 = 0; k1 < m; ++k1) c += (m - (k1 - k1 % S) + S - 1) / S;
  } else {
    c = (long long)m * (m + 1) / 2 * ((m + S - 1) / S);
  }
  return c;
}

// Symmetric work lists are built once, at space-plan creation (plans are
// immutable afterwards: no allocation or synchronous copy on the enqueue path,
// so a solve can be captured into a CUDA graph on a fresh plan). The segment
// lengths are those of the symmetric pass-A kernels: Good-Thomas / Rader (12,
// 3D Rader: sorted triples), prime-factor (1), Bluestein (8, 2, 1). A list
// above kSegCapBytes is not built; its kernel then runs the non-symmetric
// variant (every mode its own FFT).
constexpr long long kSegCapBytes = 64LL << 20;
struct SegKey { int S; bool six; };
constexpr SegKey kSegKeys[] = {{12, false}, {12, true}, {10, false}, {1, false}, {8, false}, {2, false}};

constexpr bool seg_key_listed(int S, bool six) {
  for (const SegKey& k : kSegKeys)
    if (k.S == S && k.six == six) return true;
  return false;
}

int build_seg_tiles(bhcp_space_plan* sp) {
  if (sp->dim < 2) return BHCP_OK;
  int slot = 0;
  for (const SegKey& k : kSegKeys) {
    if (k.six && sp->dim != 3) continue;
    if (slot >= 9) break;
    if (seg_list_count(sp->dim, sp->m, k.S, k.six) * (long long)sizeof(int4) > kSegCapBytes) continue;
    const std::vector<int4> t = seg_list(sp->dim, sp->m, k.S, k.six);
    if (t.empty()) continue;
    if (cudaMalloc(&sp->seg_tiles[slot], sizeof(int4) * t.size()) != cudaSuccess) return cuda_fail("cudaMalloc seg tiles");
    if (cudaMemcpy(sp->seg_tiles[slot], t.data(), sizeof(int4) * t.size(), cudaMemcpyHostToDevice) != cudaSuccess)
      return cuda_fail("seg tiles upload");
    sp->seg_len[slot] = k.six ? k.S + 1000 : k.S;
    sp->seg_count[slot] = (long long)t.size();
    ++slot;
  }
  return BHCP_OK;
}

// lookup only (built by build_seg_tiles); nullptr when the plan has no such list
const int4* seg_tiles(const bhcp_space_plan* sp, int S, long long* count, bool six = false) {
  const int key = six ? S + 1000 : S;
  for (int slot = 0; slot < 9; ++slot)
    if (sp->seg_tiles[slot] && sp->seg_len[slot] == key) {
      *count = sp->seg_count[slot];
      return sp->seg_tiles[slot];
    }
  return nullptr;
}

// apply a tile window to a symmetric work list
inline void window(const SymRange& sr, const int4*& tiles, long long& cnt) {
  if (!sr.on) return;
  const long long e = sr.end < 0 || sr.end > cnt ? cnt : sr.end;
  const long long b = sr.begin < 0 ? 0 : (sr.begin > e ? e : sr.begin);
  tiles += b;
  cnt = e - b;
}
inline void window(const SymRange& sr, const int2*& tiles, long long& cnt) {
  if (!sr.on) return;
  const long long e = sr.end < 0 || sr.end > cnt ? cnt : sr.end;
  const long long b = sr.begin < 0 ? 0 : (sr.begin > e ? e : sr.begin);
  tiles += b;
  cnt = e - b;
}

static_assert(seg_key_listed(fastk::GtPlan::S, false) && seg_key_listed(fastk::RaderPlan<257>::S, false) &&
                  seg_key_listed(fastk::RaderPlan<257>::S, true) && seg_key_listed(1, false) &&
                  seg_key_listed(fastk::BluePlan<257>::S, false) && seg_key_listed(fastk::BluePlan<1025>::S, false) &&
                  seg_key_listed(fastk::BluePlan<4097>::S, false),
              "every symmetric pass-A kernel's segment length has a prebuilt list");

// Could some shift s_j lie within 1e-14 |s_j| of a mode eigenvalue of this
// plan (space.py:237-240)? mu ranges over [dim mu1_min, dim mu1_max]; the
// nearest point of that interval to -s_j is tested with a 2x margin for the
// rounding of the device's den2. If not, the pass-A generator skips the test.
bool may_be_singular(const bhcp_space_plan* sp, const bhcp_time_plan* tp) {
  const double lo = sp->mu_lo * (1.0 - 1e-12), hi = sp->mu_hi * (1.0 + 1e-12);
  for (const double2& s : tp->shifts_h) {
    const double x = std::min(std::max(-s.x, lo), hi);
    const double d = std::hypot(s.x + x, s.y);
    if (d <= 2e-14 * std::hypot(s.x, s.y)) return true;
  }
  return false;
}

template <bool CHECK, bool FAST>
int gt_launch(const fastk::GtModesArgs& a, bool sym, size_t sm, cudaStream_t s) {
  using namespace fastk;
  if (sym) {
    const long long grid = std::min<long long>(a.ntiles, resident_ctas(k_modes_gt<true, CHECK, FAST>, GtPlan::T, sm));
    k_modes_gt<true, CHECK, FAST><<<(unsigned)grid, GtPlan::T, sm, s>>>(a);
  } else {
    const long long work = (a.k_count + GtPlan::S - 1) / GtPlan::S;
    const long long grid = std::min<long long>(work, resident_ctas(k_modes_gt<false, CHECK, FAST>, GtPlan::T, sm));
    k_modes_gt<false, CHECK, FAST><<<(unsigned)grid, GtPlan::T, sm, s>>>(a);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_gt launch");
  return BHCP_OK;
}

int gt_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat, double cscale,
             long long k_begin, long long k_end, double* W, const fastk::WLayout& wl, StatusDev* st, cudaStream_t s,
             const SymRange& sr = SymRange()) {
  using namespace fastk;
  GtModesArgs a{};
  a.mu1 = sp->mu1_dev; a.ghat = ghat;
  a.cscale = cscale; a.k_begin = k_begin; a.k_count = k_end - k_begin; a.W = W; a.m = sp->m; a.dim = sp->dim;
  a.st = st; a.wl = wl; a.tab = tp->gt; a.itab = tp->gt_idx;
  const size_t sm = gt_smem();
  const bool want_sym = sr.on || (sp->dim >= 2 && k_begin == 0 && k_end == sp->nx && wl.nmodes == sp->nx);
  long long cnt = 0;
  a.tiles = want_sym ? seg_tiles(sp, GtPlan::S, &cnt) : nullptr;
  if (want_sym && !a.tiles && sr.on) return fail(BHCP_ERR_INVALID, "symmetric tile list not built for this plan");
  if (a.tiles) {
    window(sr, a.tiles, cnt);
    if (cnt == 0) return BHCP_OK;
    a.ntiles = cnt;
  }
  const bool sym = a.tiles != nullptr;
  const bool fast = wl.mode_major && wl.nsl == 1 && !wl.sl_koff[0] && wl.P1 * fastk::kTBL * 129 < (1LL << 31);
  if (may_be_singular(sp, tp))
    return fast ? gt_launch<true, true>(a, sym, sm, s) : gt_launch<true, false>(a, sym, sm, s);
  return fast ? gt_launch<false, true>(a, sym, sm, s) : gt_launch<false, false>(a, sym, sm, s);
}

int pf_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat, double cscale,
             long long k_begin, long long k_end, double* W, const fastk::WLayout& wl, StatusDev* st, cudaStream_t s,
             const SymRange& sr = SymRange()) {
  using namespace fastk;
  PfModesArgs a{};
  a.shg = tp->pf + 2 * kPfNp; a.gaminv = tp->tables + tp->n;
  a.mu1 = sp->mu1_dev; a.ghat = ghat; a.cscale = cscale; a.k_begin = k_begin; a.k_count = k_end - k_begin;
  a.m = sp->m; a.dim = sp->dim; a.st = st; a.tab = tp->pf; a.tq = tp->pf_idx; a.wl = wl;
  const size_t sm = pf_smem();
  const bool sym = sr.on || (sp->dim >= 2 && k_begin == 0 && k_end == sp->nx && wl.nmodes == sp->nx);
  long long cnt = 0;
  a.tiles = sym ? seg_tiles(sp, 1, &cnt) : nullptr;
  if (sym && !a.tiles && sr.on) return fail(BHCP_ERR_INVALID, "symmetric tile list not built for this plan");
  if (a.tiles) {
    window(sr, a.tiles, cnt);
    if (cnt == 0) return BHCP_OK;
    a.ntiles = cnt;
    const long long grid = std::min<long long>(cnt, resident_ctas(k_modes_pf<true>, PfPlan::T, sm));
    k_modes_pf<true><<<(unsigned)grid, PfPlan::T, sm, s>>>(a, PfPairs{});
  } else {
    const long long grid = std::min<long long>(a.k_count, resident_ctas(k_modes_pf<false>, PfPlan::T, sm));
    k_modes_pf<false><<<(unsigned)grid, PfPlan::T, sm, s>>>(a, PfPairs{});
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_pf launch");
  return BHCP_OK;
}

// Pass A of nb independent solves (one launch per kPfMaxPairs pairs): 1D,
// n = 4097 (BASELINE config 5). Pair i: time plan tps[i], coefficient scale
// cscales[i], status sts[i], W at W + i * w_stride.
int pf_modes_batch(const bhcp_space_plan* sp, const bhcp_time_plan* const* tps, int nb, const double* ghat,
                   const double* cscales, const fastk::WLayout& wl, long long w_stride, StatusDev* sts,
                   cudaStream_t s) {
  using namespace fastk;
  const bhcp_time_plan* tp = tps[0];
  double* W = wl.sl_base[0];
  for (int p0 = 0; p0 < nb; p0 += kPfMaxPairs) {
    const int np = std::min(kPfMaxPairs, nb - p0);
    PfModesArgs a{};
    a.shg = tp->pf + 2 * kPfNp; a.gaminv = tp->tables + tp->n;
    a.mu1 = sp->mu1_dev; a.ghat = ghat; a.cscale = cscales[p0]; a.k_begin = 0; a.k_count = sp->nx;
    a.m = sp->m; a.dim = sp->dim; a.st = sts + p0; a.tab = tp->pf; a.tq = tp->pf_idx;
    a.wl = wl;
    a.wl.sl_base[0] = W + (long long)p0 * w_stride;
    PfPairs pp{};
    pp.n = np;
    pp.w_stride = w_stride;
    for (int i = 0; i < np; ++i) {
      const bhcp_time_plan* t = tps[p0 + i];
      pp.shg[i] = t->pf + 2 * kPfNp; pp.gaminv[i] = t->tables + t->n;
      pp.cscale[i] = cscales[p0 + i]; pp.st[i] = sts + p0 + i;
    }
    const size_t sm = pf_smem();
    const long long grid = std::min<long long>(a.k_count * np, resident_ctas(k_modes_pf<false, true>, PfPlan::T, sm));
    k_modes_pf<false, true><<<(unsigned)grid, PfPlan::T, sm, s>>>(a, pp);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_pf (batch) launch");
  }
  return BHCP_OK;
}

template <int NL>
int rader_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat, double cscale,
                long long k_begin, long long k_end, double* W, const fastk::WLayout& wl, StatusDev* st,
                cudaStream_t s, const SymRange& sr = SymRange()) {
  using namespace fastk;
  using Pl = RaderPlan<NL>;
  RaderModesArgs a{};
  a.shifts = tp->tables + 2 * tp->n; a.gaminv = tp->tables + tp->n; a.mu1 = sp->mu1_dev; a.ghat = ghat;
  a.cscale = cscale; a.k_begin = k_begin; a.k_count = k_end - k_begin; a.W = W; a.m = sp->m; a.dim = sp->dim;
  a.st = st; a.wl = wl;
  a.tw = tp->rader; a.bhat = tp->rader + Pl::NP; a.perm = tp->rader_idx; a.qidx = tp->rader_idx + Pl::NP;
  const size_t sm = rader_smem<NL>();
  const bool sym = sr.on || (sp->dim >= 2 && k_begin == 0 && k_end == sp->nx && wl.nmodes == sp->nx);
  long long cnt = 0;
  a.sym6 = sp->dim == 3 ? 1 : 0;
  a.tiles = sym ? seg_tiles(sp, Pl::S, &cnt, a.sym6 != 0) : nullptr;
  if (sym && !a.tiles && sr.on) return fail(BHCP_ERR_INVALID, "symmetric tile list not built for this plan");
  if (a.tiles) {
    window(sr, a.tiles, cnt);
    if (cnt == 0) return BHCP_OK;
    a.ntiles = cnt;
    const long long grid = std::min<long long>(cnt, resident_ctas(k_modes_rader<NL, true>, Pl::T, sm));
    k_modes_rader<NL, true><<<(unsigned)grid, Pl::T, sm, s>>>(a);
  } else {
    const long long work = (a.k_count + Pl::S - 1) / Pl::S;
    const long long grid = std::min<long long>(work, resident_ctas(k_modes_rader<NL, false>, Pl::T, sm));
    k_modes_rader<NL, false><<<(unsigned)grid, Pl::T, sm, s>>>(a);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_rader launch");
  return BHCP_OK;
}

template <int NL>
int blue_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat, double cscale,
               long long k_begin, long long k_end, double* W, const fastk::WLayout& wl, StatusDev* st,
               cudaStream_t s, const SymRange& sr = SymRange()) {
  using namespace fastk;
  using Pl = BluePlan<NL>;
  BlueModesArgs a{};
  a.shifts = tp->tables + 2 * tp->n; a.gaminv = tp->tables + tp->n; a.mu1 = sp->mu1_dev; a.ghat = ghat;
  a.cscale = cscale; a.k_begin = k_begin; a.k_count = k_end - k_begin; a.W = W; a.m = sp->m; a.dim = sp->dim;
  a.st = st; a.wl = wl;
  const int L = Pl::L;
  a.bt.tw = tp->blue; a.bt.chirp = tp->blue + L; a.bt.bhat = tp->blue + L + NL; a.bt.wM = tp->blue + 2 * L + NL;
  a.bt.cg = tp->blue + 2 * L + 2 * NL; a.bt.wg = tp->blue + 2 * L + 3 * NL; a.bt.thr = tp->blue + 2 * L + 4 * NL;
  const size_t sm = blue_smem<NL>();
  const bool sym = sr.on || (sp->dim >= 2 && k_begin == 0 && k_end == sp->nx && wl.nmodes == sp->nx);
  long long cnt = 0;
  a.tiles = sym ? seg_tiles(sp, Pl::S, &cnt) : nullptr;
  if (sym && !a.tiles && sr.on) return fail(BHCP_ERR_INVALID, "symmetric tile list not built for this plan");
  if (a.tiles) {
    window(sr, a.tiles, cnt);
    if (cnt == 0) return BHCP_OK;
    a.ntiles = cnt;
    const long long grid = std::min<long long>(cnt, resident_ctas(k_modes_blue<NL, true>, Pl::T, sm));
    k_modes_blue<NL, true><<<(unsigned)grid, Pl::T, sm, s>>>(a);
  } else {
    const long long work = (a.k_count + Pl::S - 1) / Pl::S;
    const long long grid = std::min<long long>(work, resident_ctas(k_modes_blue<NL, false>, Pl::T, sm));
    k_modes_blue<NL, false><<<(unsigned)grid, Pl::T, sm, s>>>(a);
  }
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_blue launch");
  return BHCP_OK;
}

int launch_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat, double cscale,
                 long long k_begin, long long k_end, double* W, const fastk::WLayout& wl_in, StatusDev* st,
                 cudaStream_t s, const SymRange& sr = SymRange()) {
  fastk::WLayout wl = wl_in;
  if (!wl.sl_base[0]) wl.bind(W);   // local W unless the caller set per-slab destinations
  const long long kc = k_end - k_begin;
  if (kc <= 0) return BHCP_OK;
  const FftPlanHost& P = tp->fft;
  if (!g_disable_fast && tp->rader && tp->n == 257)
    return rader_modes<257>(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
  if (!g_disable_fast && tp->gt && tp->n == 1025)
    return gt_modes(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
  if (!g_disable_fast && tp->pf && tp->n == 4097)
    return pf_modes(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
  if (!g_disable_fast && tp->blue) {
    switch (tp->n) {
      case 257: return blue_modes<257>(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
      case 1025: return blue_modes<1025>(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
      case 4097: return blue_modes<4097>(sp, tp, ghat, cscale, k_begin, k_end, W, wl, st, s, sr);
    }
  }
  if (!g_disable_fast && tp->n == 513) {
    using namespace fastk;
    FastModesArgs f{};
    f.shifts = tp->tables + 2 * tp->n; f.gaminv = tp->tables + tp->n; f.mu1 = sp->mu1_dev; f.ghat = ghat;
    f.cscale = cscale; f.k_begin = k_begin; f.k_count = kc; f.W = W; f.m = sp->m; f.dim = sp->dim;
    f.tw = P.d.tw; f.st = st; f.wl = wl;
    // symmetric 4x4 tiles need the whole mode range with global column indices
    const bool sym = sp->dim == 2 && sp->tiles_dev &&
                     (sr.on || (k_begin == 0 && k_end == sp->nx && wl.nmodes == sp->nx));
    if (sym) {
      const int2* tl = sp->tiles_dev;
      long long cnt = sp->ntiles;
      window(sr, tl, cnt);
      if (cnt == 0) return BHCP_OK;
      f.tiles = tl;
      f.ntiles = cnt;
      const long long grid = std::min<long long>(cnt, resident_ctas(k_modes_fast<513, true>, ModesPlan<513>::T,
                                                                   modes_smem<513>()));
      k_modes_fast<513, true><<<(unsigned)grid, ModesPlan<513>::T, modes_smem<513>(), s>>>(f);
    } else {
      const long long work = (kc + ModesPlan<513>::S - 1) / ModesPlan<513>::S;
      const long long grid = std::min<long long>(work, resident_ctas(k_modes_fast<513, false>, ModesPlan<513>::T,
                                                                     modes_smem<513>()));
      k_modes_fast<513, false><<<(unsigned)grid, ModesPlan<513>::T, modes_smem<513>(), s>>>(f);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes_fast launch");
    return BHCP_OK;
  }
  int nseq = P.max_seqs(kSmemBudget);
  if (nseq < 1) return fail(BHCP_ERR_INVALID, "time length does not fit the FFT engine");
  if (nseq > 64) nseq = 64;
  if (kc < nseq) nseq = (int)kc;
  ModesArgs a{};
  a.p = P.d; a.ld = P.ld; a.nseq = nseq; a.n = tp->n; a.m = sp->m; a.dim = sp->dim;
  a.shifts = tp->tables + 2 * tp->n; a.gaminv = tp->tables + tp->n; a.mu1 = sp->mu1_dev;
  a.ghat = ghat; a.cscale = cscale; a.k_begin = k_begin; a.k_count = kc; a.W = W; a.wl = wl; a.st = st;
  const long long grid = (kc + nseq - 1) / nseq;
  const size_t sm = smem_bytes(P, nseq);
#define BHCP_MODES(VV) \
  case VV: k_modes<VV><<<(unsigned)grid, VT<VV>::T, sm, s>>>(a); break;
  switch (P.variant) { BHCP_FOR_VARIANTS(BHCP_MODES) }
#undef BHCP_MODES
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_modes launch");
  return BHCP_OK;
}

// W layout of the single-GPU fused solve: level-major in 1D, one blocked slab otherwise.
fastk::WLayout make_blocked(const bhcp_space_plan* sp, long long k_count, int nsl, const long long* bounds) {
  fastk::WLayout wl{};
  wl.mode_major = 2;
  wl.nsl = nsl;
  wl.nmodes = k_count;
  wl.P1 = ipow(sp->m, sp->dim - 1);
  long long off = 0;
  for (int s = 0; s < nsl; ++s) {
    wl.sl_c[s] = (int)bounds[s];
    wl.sl_nt[s] = (bounds[s + 1] - bounds[s] + fastk::kTBL - 1) / fastk::kTBL;
    wl.sl_off[s] = off;
    off += k_count * fastk::kTBL * wl.sl_nt[s];
  }
  wl.sl_c[nsl] = (int)bounds[nsl];
  return wl;
}

fastk::WLayout native_layout(const bhcp_space_plan* sp, long long k_count, int n) {
  // 1D: P1 = 1, i.e. mode-major with row stride NT*8 (each mode's time series contiguous)
  const long long b[2] = {0, n};
  return make_blocked(sp, k_count, 1, b);
}

long long native_w_elems(const bhcp_space_plan* sp, int n) {
  return sp->nx * fastk::kTBL * ((n + fastk::kTBL - 1) / fastk::kTBL);
}

// --- level passes ----------------------------------------------------------------
__global__ void k_unpack_blocked(const double* __restrict__ in, const long long* __restrict__ koff, long long NT,
                                 long long P1, long long nx, long long nlev, double* __restrict__ out) {
  const long long total = nx * nlev;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / nx, k = i - t * nx;
    const long long k1 = k / P1, r = k - k1 * P1;
    const long long base = koff ? koff[k1] : k1 * NT * P1 * fastk::kTBL;
    out[i] = in[base + ((t / fastk::kTBL) * P1 + r) * fastk::kTBL + (t % fastk::kTBL)];
  }
}

template <int N>
int blk2_launch(const bhcp_space_plan* sp, gdst::ArgsB2 a, cudaStream_t s) {
  using namespace gdst;
  const long long tiles = a.P * a.NT;
  if (tiles == 0) return BHCP_OK;
  if (tiles > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  const size_t sm = gdst::smemB2_bytes<N>();
  const long long grid = std::min<long long>(tiles, resident_ctas(k_dst_blk2<N>, PlanB2<N>::T, sm));
  k_dst_blk2<N><<<(unsigned)grid, PlanB2<N>::T, sm, s>>>(a);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_blk2 launch");
  return BHCP_OK;
}

template <int N>
int cols3_launch(const bhcp_space_plan* sp, gdst::ArgsB2 a, cudaStream_t s) {
  using namespace gdst;
  const long long tiles = a.no * ((a.ni + 2 * PlanC3<N>::S - 1) / (2 * PlanC3<N>::S));
  if (tiles == 0) return BHCP_OK;
  if (tiles > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  const size_t sm = gdst::smemC3_bytes<N>();
  const long long grid = std::min<long long>(tiles, resident_ctas(k_dst_cols3<N>, PlanC3<N>::T, sm));
  k_dst_cols3<N><<<(unsigned)grid, PlanC3<N>::T, sm, s>>>(a);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_cols3 launch");
  return BHCP_OK;
}

// Real-field DST along a strided axis, in place capable (k_dst_cols3).
int cols_blk2(const bhcp_space_plan* sp, const double* in, double* out, long long ni, long long no,
              cudaStream_t s) {
  gdst::ArgsB2 b{};
  b.in = in; b.out = out; b.tw = sp->twN; b.sn = sp->snN; b.scale = sqrt(2.0 / (sp->m + 1));
  b.ni = ni; b.no = no;
  switch (2 * (sp->m + 1)) {
    case 512: return cols3_launch<256>(sp, b, s);
    case 1024: return cols3_launch<512>(sp, b, s);
    case 2048: return cols3_launch<1024>(sp, b, s);
  }
  return fail(BHCP_ERR_INVALID, "cols_blk2 length");
}

int blk3_launch(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, cudaStream_t s);

// One level pass of the fused solve on `nlev` levels. pass 0: W (1D:
// level-major; else blocked, k1's first block at koff[k1] or k1*NT*P1*8) ->
// y (level-major) with the DST along the last axis; pass p >= 1: DST along
// axis -(p+1) in place on y.
int level_pass(const bhcp_space_plan* sp, const double* in, const long long* koff, double* y, long long nlev,
               int pass, cudaStream_t s) {
  const int d = sp->dim, m = sp->m;
  const int L = 2 * (m + 1);
  if (pass == 0 && d == 1) {
    // 1D: W mode-major (row stride NT*8) -> transpose to level-major y -> rows DST in place
    const long long NT1 = (nlev + fastk::kTBL - 1) / fastk::kTBL;
    dim3 grid((unsigned)((nlev + 31) / 32), (unsigned)((m + 31) / 32));
    k_transpose_ld<<<grid, dim3(32, 8), 0, s>>>(in, NT1 * fastk::kTBL, y, m, nlev);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_transpose_ld");
    return launch_rows(sp, y, y, 0, nlev, 0, nullptr, nullptr, s, Blocked(), 1);
  }
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  const long long P1 = ipow(m, d - 1);
  if (pass >= 1)
    return launch_cols(sp, y, y, 0, ipow(m, pass), nlev * ipow(m, d - 1 - pass), pass, 0, nullptr, nullptr, s);
  if (!g_disable_fast && (L == 512 || L == 1024 || L == 2048) && d <= 3 && !koff) return blk3_launch(sp, in, y, nlev, s);
  if (!g_disable_fast && (L == 512 || L == 1024 || L == 2048)) {
    gdst::ArgsB2 b{};
    b.in = in; b.out = y; b.tw = sp->twN; b.sn = sp->snN; b.scale = sqrt(2.0 / (m + 1));
    b.koff = koff; b.NT = NT; b.P1 = P1; b.idiv = ipow(m, d - 2); b.P = P1; b.nlev = nlev;
    switch (L) {
      case 512: return blk2_launch<256>(sp, b, s);
      case 1024: return blk2_launch<512>(sp, b, s);
      case 2048: return blk2_launch<1024>(sp, b, s);
    }
  }
  const long long total = nlev * sp->nx;
  k_unpack_blocked<<<(unsigned)std::min<long long>((total + 255) / 256, 65535), 256, 0, s>>>(in, koff, NT, P1, sp->nx,
                                                                                          nlev, y);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_unpack_blocked");
  return launch_rows(sp, y, y, 0, nlev * P1, 0, nullptr, nullptr, s, Blocked(), P1);
}

// ---- strided axes in place on the blocked W (wax_dst.cuh), TMA tensor maps
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
std::mutex g_encode_mutex;

int tensor_map_3d(CUtensorMap* tm, double* base, long long Li, long long m, long long No, long long as_elems,
                  long long os_elems, int box_lines, int swizzle_bytes = 0) {
  {
    std::lock_guard<std::mutex> lk(g_encode_mutex);
    if (!g_encode_tiled) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return fail(BHCP_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
      g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
  }
  const cuuint64_t dims[3] = {(cuuint64_t)Li, (cuuint64_t)m, (cuuint64_t)No};
  const cuuint64_t strides[2] = {(cuuint64_t)as_elems * sizeof(double), (cuuint64_t)os_elems * sizeof(double)};
  const cuuint32_t box[3] = {(cuuint32_t)box_lines, (cuuint32_t)wax::kBoxRows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode_tiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE,
                              swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                              : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BHCP_ERR_INVALID, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return BHCP_OK;
}

template <class P>
int wax_launch(const bhcp_space_plan* sp, double* W, long long Li, long long No, long long nlev, long long lpl,
               cudaStream_t s) {
  constexpr int N = P::N;
  constexpr int LW = 2 * P::S;
  const long long m = N - 1;
  const long long lchunks = (Li + LW - 1) / LW;
  const long long tiles = lchunks * No;
  if (tiles == 0) return BHCP_OK;
  if (tiles > 0x7fffffffLL || Li > 0x7fffffffLL || No > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  if (reinterpret_cast<uintptr_t>(W) % 16 != 0) return fail(BHCP_ERR_INVALID, "W must be 16-byte aligned");
  alignas(64) CUtensorMap tm;
  int rc = tensor_map_3d(&tm, W, Li, m, No, Li, Li * m, LW);
  if (rc) return rc;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  wax::ArgsWX a{sp->twN, sp->snN, sqrt(2.0 / N), (int)lchunks, (int)tiles,
                (int)(nlev - (NT - 1) * fastk::kTBL), (int)NT, lpl > 0 ? (int)((NT - 1) * lpl) : -1};
  const size_t sm = wax::smem_bytes<P>();
  const long long grid = std::min<long long>(tiles, resident_ctas(wax::k_dst_wax<P>, P::T, sm));
  wax::k_dst_wax<P><<<(unsigned)grid, P::T, sm, s>>>(tm, a);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_wax launch");
  return BHCP_OK;
}

template <int N>
int wax2_launch(const bhcp_space_plan* sp, double* W, long long Li, long long No, long long nlev, long long lpl,
                cudaStream_t s) {
  constexpr int LW = wax2::kLW;
  const long long m = N - 1;
  const long long lchunks = (Li + LW - 1) / LW;
  const long long tiles = lchunks * No;
  if (tiles == 0) return BHCP_OK;
  if (tiles > 0x7fffffffLL || Li > 0x7fffffffLL || No > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  if (reinterpret_cast<uintptr_t>(W) % 16 != 0) return fail(BHCP_ERR_INVALID, "W must be 16-byte aligned");
  alignas(64) CUtensorMap tm;
  int rc = tensor_map_3d(&tm, W, Li, m, No, Li, Li * m, LW, 128);
  if (rc) return rc;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  wax::ArgsWX a{sp->twN, sp->snN, sqrt(2.0 / N), (int)lchunks, (int)tiles,
                (int)(nlev - (NT - 1) * fastk::kTBL), (int)NT, lpl > 0 ? (int)((NT - 1) * lpl) : -1};
  const size_t sm = wax2::smem_bytes<N>();
  const int threads = (wax2::kCW + 1) * 32;
  const long long grid = std::min<long long>(tiles, resident_ctas(wax2::k_dst_wax2<N>, threads, sm));
  wax2::k_dst_wax2<N><<<(unsigned)grid, threads, sm, s>>>(tm, a);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_wax2 launch");
  return BHCP_OK;
}

// last spatial axis, blocked W -> y, N = m + 1 in {256, 512} (k_dst_blk3, wax2_dst.cuh)
template <int N>
int blk3_launch_n(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, cudaStream_t s) {
  const long long m = sp->m, d = sp->dim;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  const long long idiv = ipow(m, d - 2);
  const long long No = m * NT * idiv;   // W blocks (k1, level tile, r2)
  if (No == 0) return BHCP_OK;
  if (No > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  if (reinterpret_cast<uintptr_t>(W) % 16 != 0) return fail(BHCP_ERR_INVALID, "W must be 16-byte aligned");
  alignas(64) CUtensorMap tm;
  // view {8 levels, m elements (64 B rows), No blocks}
  int rc = tensor_map_3d(&tm, const_cast<double*>(W), fastk::kTBL, m, No, fastk::kTBL, fastk::kTBL * m,
                         fastk::kTBL, 64);
  if (rc) return rc;
  wax2::ArgsB3 a{sp->twN, sp->snN, sqrt(2.0 / N), y, (int)No, (int)NT, (int)idiv, (int)nlev, (int)m};
  const size_t sm = wax2::smem_bytes_b3<N>();
  const int threads = (wax2::kCW + 1) * 32;
  const long long grid = std::min<long long>(No, resident_ctas(wax2::k_dst_blk3<N>, threads, sm));
  wax2::k_dst_blk3<N><<<(unsigned)grid, threads, sm, s>>>(tm, a);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_blk3 launch");
  return BHCP_OK;
}

int q4_blk_launch(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, cudaStream_t s);

int blk3_launch(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, cudaStream_t s) {
  switch (sp->m + 1) {
    case 256: return blk3_launch_n<256>(sp, W, y, nlev, s);
    case 512: return blk3_launch_n<512>(sp, W, y, nlev, s);
    case 1024: return q4_blk_launch(sp, W, y, nlev, s);
  }
  return fail(BHCP_ERR_INVALID, "blk3 length");
}

// Strided axes on W: k_dst_wax (m + 1 = 256, c4), k_dst_wax2 (512, c2).
// m + 1 = 1024 (c3) last axis: k_dst_blk4 (two warps per line pair, 64 B row tiles)
int q4_blk_launch(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, cudaStream_t s) {
  constexpr int N = 1024;
  const long long m = sp->m, d = sp->dim;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  const long long idiv = ipow(m, d - 2);
  const long long No = m * NT * idiv;
  if (No == 0) return BHCP_OK;
  if (No > 0x7fffffffLL) return fail(BHCP_ERR_INVALID, "too many tiles");
  if (reinterpret_cast<uintptr_t>(W) % 16 != 0) return fail(BHCP_ERR_INVALID, "W must be 16-byte aligned");
  alignas(64) CUtensorMap tm;
  int rc = tensor_map_3d(&tm, const_cast<double*>(W), fastk::kTBL, m, No, fastk::kTBL, fastk::kTBL * m,
                         fastk::kTBL, 64);
  if (rc) return rc;
  wax2::ArgsB3 b3{sp->twN, sp->snN, sqrt(2.0 / N), y, (int)No, (int)NT, (int)idiv, (int)nlev, (int)m};
  const size_t sm = wax2::smem_bytes_4();
  const int threads = (wax2::kCW + 1) * 32;
  const long long grid = std::min<long long>(No, resident_ctas(wax2::k_dst_blk4, threads, sm));
  wax2::k_dst_blk4<<<(unsigned)grid, threads, sm, s>>>(tm, b3);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_dst_blk4 launch");
  return BHCP_OK;
}

// m + 1 = 1024 (c3) keeps the strided axis on y (k_dst_cols3, 6.6 ms): a W-side
// tile of that length fits the smem budget only with 64 B rows, which measured
// 7.5 ms (DRAM efficiency of 64 B rows at an 8 MB stride). Its last axis runs
// k_dst_blk4 (3.8 ms vs 5.4 for k_dst_blk2).
bool wax_ok(const bhcp_space_plan* sp) {
  const int L = 2 * (sp->m + 1);
  return !g_disable_fast && sp->dim >= 2 && sp->dim <= 3 && (L == 512 || L == 1024);
}

// In-place inverse DST of the blocked W (single-slab layout with NT level
// tiles, or an all-to-all receive buffer, whose k1 blocks sit at the same
// uniform stride NT * P1 * 8) along spatial axis `axis` < dim - 1.
//   axis 0 (k1):  lines = a whole k1 block (NT * P1 * 8 contiguous doubles)
//   axis 1 (k2, 3D): lines = (k3, level) runs of 8m doubles, outer = (k1, level tile)
int w_pass(const bhcp_space_plan* sp, double* W, long long nlev, int axis, cudaStream_t s) {
  if (!wax_ok(sp)) return fail(BHCP_ERR_INVALID, "w_pass: unsupported length or dimension");
  if (axis < 0 || axis > sp->dim - 2) return fail(BHCP_ERR_INVALID, "w_pass: axis out of range");
  const long long m = sp->m, d = sp->dim;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  const long long P1 = ipow(m, d - 1);
  if (nlev == 0) return BHCP_OK;
  long long Li, No, lpl;
  if (axis == 0) { Li = NT * P1 * fastk::kTBL; No = 1; lpl = P1 * fastk::kTBL; }
  else { Li = ipow(m, d - 1 - axis) * fastk::kTBL; No = m * NT * ipow(m, axis - 1); lpl = 0; }
  switch (m + 1) {
    // N = 256 (c4): the CTA-synchronous 32-line tiles (256 B rows) measured faster than
    // k_dst_wax2<256> with 16-line tiles (17.8 / 17.5 vs 19.4 / 18.3 ms per axis)
    case 256: return wax_launch<wax::PlanWX<256>>(sp, W, Li, No, nlev, lpl, s);
    case 512: return wax2_launch<512>(sp, W, Li, No, nlev, lpl, s);   // warp per line pair (wax2_dst.cuh)
  }
  return fail(BHCP_ERR_INVALID, "w_pass length");
}

// m + 1 = 1024 in 2D (c3): the whole level phase as one persistent kernel over
// L2-resident level tiles (k_dst_lvl4, lvl_dst.cuh): row tasks W -> y, then
// column tasks in place on y while the level tile is still in L2. gsync: one
// counter per level tile, zeroed on the stream before the launch.
bool lvl4_ok(const bhcp_space_plan* sp) {
  return g_lvl4 != 0 && !g_disable_fast && sp->dim == 2 && sp->m + 1 == 1024;
}
// scratch of the level-group pass: per-level-tile counters, then the two Z
// slots (8 levels x m rows x 1024 doubles each)
size_t lvl4_counter_bytes(long long nlev) {
  return (2 * sizeof(unsigned) * (size_t)((nlev + fastk::kTBL - 1) / fastk::kTBL + 1) + 255) & ~size_t(255);
}
size_t lvl4_sync_bytes(long long nlev) {
  return lvl4_counter_bytes(nlev) + sizeof(double) * 2 * 8 * (size_t)1023 * lvl::kZPitch;
}

int lvl4_launch(const bhcp_space_plan* sp, const double* W, double* y, long long nlev, unsigned* gsync,
                cudaStream_t s) {
  const long long m = sp->m;
  const long long NT = (nlev + fastk::kTBL - 1) / fastk::kTBL;
  if (NT == 0) return BHCP_OK;
  const long long No = m * NT;                // W blocks
  const long long nct = (m + 7) / 8;          // column tiles per level (128)
  const long long ntasks = NT * lvl::kRowTasks + nlev * nct;
  if (ntasks > 0x7fffffffLL || m != 1023) return fail(BHCP_ERR_INVALID, "level-group pass: bad shape");
  if (reinterpret_cast<uintptr_t>(W) % 16 != 0 || reinterpret_cast<uintptr_t>(gsync) % 256 != 0)
    return fail(BHCP_ERR_INVALID, "W must be 16-byte and the scratch 256-byte aligned");
  double* z = reinterpret_cast<double*>(reinterpret_cast<char*>(gsync) + lvl4_counter_bytes(nlev));
  alignas(64) CUtensorMap tm, tz;
  int rc = tensor_map_3d(&tm, const_cast<double*>(W), fastk::kTBL, m, No, fastk::kTBL, fastk::kTBL * m,
                         fastk::kTBL, 64);
  if (rc) return rc;
  // Z: {1024 columns, m rows, 16 slot levels}, box 8 columns x 256 rows (64 B rows)
  rc = tensor_map_3d(&tz, z, lvl::kZPitch, m, 16, lvl::kZPitch, lvl::kZPitch * m, 8, 64);
  if (rc) return rc;
  // y row pairs: {2046 = parity x 1023 + column, floor(rows / 2) pairs}, pitch 2 * 1023 doubles
  if (reinterpret_cast<uintptr_t>(y) % 16 != 0) return fail(BHCP_ERR_INVALID, "y must be 16-byte aligned");
  alignas(64) CUtensorMap ty256, ty255;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)(2 * m), (cuuint64_t)(nlev * m / 2)};
    const cuuint64_t strides[1] = {(cuuint64_t)(2 * m * sizeof(double))};
    const cuuint32_t estr[2] = {1, 1};
    for (int k = 0; k < 2; ++k) {
      const cuuint32_t box[2] = {8, (cuuint32_t)(k ? 255 : 256)};
      CUresult r = g_encode_tiled(k ? &ty255 : &ty256, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, y, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(BHCP_ERR_INVALID, "cuTensorMapEncodeTiled (y pairs) failed (code " + std::to_string((int)r) + ")");
    }
  }
  const size_t sm = lvl::smem_bytes();
  // every CTA must be resident at once (column tasks wait for row tasks of other CTAs)
  const long long grid = std::min<long long>((ntasks + 1) / 2, resident_ctas(lvl::k_dst_lvl4, lvl::kThreads, sm));
  if (cudaMemsetAsync(gsync, 0, lvl4_counter_bytes(nlev), s) != cudaSuccess) return cuda_fail("lvl4 sync reset");
  const int kfirst = g_lvl4_kfirst >= 0 ? g_lvl4_kfirst : (int)grid;
  lvl::ArgsLV a{sp->twN, sp->snN, sqrt(2.0 / 1024), y, z, gsync, gsync + (NT + 1), (int)m, (int)NT, (int)nlev,
                (int)nct, (int)ntasks, kfirst};
  // cooperative launch: the driver schedules the whole grid at once or refuses,
  // so a concurrent kernel can never leave part of it waiting on CTAs that
  // cannot become resident
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(lvl::kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, lvl::k_dst_lvl4, tm, tz, ty256, ty255, a) != cudaSuccess)
    return cuda_fail("k_dst_lvl4 launch");
  return BHCP_OK;
}

// All spatial passes of the fused solve: W (blocked) -> y.
// koff == null: k1 blocks at the uniform stride NT * P1 * 8 (the single-slab
// W and every slab receive buffer). Fast lengths in 2D/3D then run the strided
// axes in place on W (k_dst_wax / k_dst_wax2; W is consumed) and the last
// axis W -> y (k_dst_blk3 / k_dst_blk4), all on TMA views that need that one
// stride. koff != null: an explicit k1 -> block offset table, honoured by the
// general passes (pass 0 into y by k_dst_blk2 / unpack + rows, then the
// strided axes in place on y); W is left untouched.
int levels_all(const bhcp_space_plan* sp, double* W, const long long* koff, double* y, long long nlev,
               cudaStream_t s, unsigned* gsync = nullptr) {
  if (!koff && gsync && lvl4_ok(sp)) return lvl4_launch(sp, W, y, nlev, gsync, s);
  if (!koff && wax_ok(sp)) {
    for (int a = 0; a < sp->dim - 1; ++a) {
      int rc = w_pass(sp, W, nlev, a, s);
      if (rc) return rc;
    }
    return blk3_launch(sp, W, y, nlev, s);
  }
  for (int p = 0; p < sp->dim; ++p) {
    // m + 1 = 1024: the last axis by k_dst_blk4 (uniform k1 stride), then y-side passes
    const bool blk4 = p == 0 && !koff && !g_disable_fast && sp->dim >= 2 && sp->dim <= 3 && sp->m + 1 == 1024;
    int rc = blk4 ? blk3_launch(sp, W, y, nlev, s) : level_pass(sp, W, koff, y, nlev, p, s);
    if (rc) return rc;
  }
  return BHCP_OK;
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

namespace bhcp {
bool ensure_device_constants(int device, std::string* err) {
  std::lock_guard<std::mutex> lk(g_init_mutex);
  if (device < 0 || device >= 64) { *err = "bad device"; return false; }
  if (g_init_done[device]) return true;
  double cs[kOddRootsTotal], sn[kOddRootsTotal];
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int R : {3, 5, 7, 11, 13, 17, 19, 23}) {
    const int off = odd_root_offset(R);
    for (int q = 0; q < R; ++q) {
      long double ang = 2.0L * pi * (long double)q / (long double)R;
      cs[off + q] = (double)cosl(ang);
      sn[off + q] = (double)sinl(ang);
    }
  }
  if (cudaMemcpyToSymbol(c_root_cos, cs, sizeof(cs)) != cudaSuccess ||
      cudaMemcpyToSymbol(c_root_sin, sn, sizeof(sn)) != cudaSuccess) {
    *err = std::string("cudaMemcpyToSymbol: ") + cudaGetErrorString(cudaGetLastError());
    return false;
  }
  cudaDeviceGetAttribute(&g_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, device);
  {
    const char* e = getenv("BHCP_DISABLE_FAST");
    g_disable_fast = (e && e[0] == '1');
    const char* l4 = getenv("BHCP_LVL4");
    if (l4) g_lvl4 = atoi(l4);
    const char* kf = getenv("BHCP_LVL4_KFIRST");
    if (kf) g_lvl4_kfirst = atoi(kf);

  }
  set_all_attributes();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    *err = std::string("kernel attribute setup: ") + cudaGetErrorString(e);
    return false;
  }
  g_init_done[device] = true;
  return true;
}
}  // namespace bhcp

// ====================================================================== C ABI
extern "C" {

int bhcp_version(void) { return 100; }
const char* bhcp_last_error(void) { return g_last_error.c_str(); }
size_t bhcp_status_bytes(void) { return sizeof(StatusDev); }

int bhcp_space_plan_create(int device, int dim, int num_cells, const double* mu1_host, bhcp_space_plan** out) {
  if (!out || !mu1_host) return fail(BHCP_ERR_INVALID, "null argument");
  if (dim < 1 || dim > 3) return fail(BHCP_ERR_INVALID, "dim must be 1, 2 or 3");
  if (num_cells < 2) return fail(BHCP_ERR_INVALID, "need at least 2 cells per edge");
  DeviceGuard g(device);
  std::string err;
  if (!ensure_device_constants(device, &err)) return fail(BHCP_ERR_CUDA, err);
  auto* sp = new bhcp_space_plan();
  sp->device = device; sp->dim = dim; sp->num_cells = num_cells; sp->m = num_cells - 1;
  sp->nx = ipow(sp->m, dim);
  if (!build_fft_plan(2 * num_cells, &sp->dst, &err)) { delete sp; return fail(BHCP_ERR_INVALID, err); }
  if (cudaMalloc(&sp->mu1_dev, sizeof(double) * sp->m) != cudaSuccess) {
    free_fft_plan(&sp->dst); delete sp; return cuda_fail("cudaMalloc mu1");
  }
  cudaMemcpy(sp->mu1_dev, mu1_host, sizeof(double) * sp->m, cudaMemcpyHostToDevice);
  sp->mu_lo = dim * *std::min_element(mu1_host, mu1_host + sp->m);
  sp->mu_hi = dim * *std::max_element(mu1_host, mu1_host + sp->m);
  sp->tiles_dev = nullptr;
  sp->ntiles = 0;
  for (int i = 0; i < 9; ++i) { sp->seg_tiles[i] = nullptr; sp->seg_count[i] = 0; sp->seg_len[i] = 0; }
  {
    const int N = num_cells;
    std::vector<double2> tw(N);
    std::vector<double> sn(N);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < N; ++k) {
      const long double a = -2.0L * pi * (long double)k / (long double)N;
      tw[k] = make_double2((double)cosl(a), (double)sinl(a));
      sn[k] = (double)sinl(pi * (long double)k / (long double)N);
    }
    if (cudaMalloc(&sp->twN, sizeof(double2) * N) != cudaSuccess || cudaMalloc(&sp->snN, sizeof(double) * N) != cudaSuccess) {
      free_fft_plan(&sp->dst); cudaFree(sp->mu1_dev); delete sp; return cuda_fail("cudaMalloc DST tables");
    }
    cudaMemcpy(sp->twN, tw.data(), sizeof(double2) * N, cudaMemcpyHostToDevice);
    cudaMemcpy(sp->snN, sn.data(), sizeof(double) * N, cudaMemcpyHostToDevice);
  }
  if (dim == 2) {
    const int mt = (sp->m + fastk::kSymTile - 1) / fastk::kSymTile;
    std::vector<int2> tiles;
    for (int a = 0; a < mt; ++a)
      for (int b = a; b < mt; ++b) tiles.push_back(make_int2(a, b));
    sp->ntiles = (long long)tiles.size();
    if (cudaMalloc(&sp->tiles_dev, sizeof(int2) * tiles.size()) != cudaSuccess) {
      free_fft_plan(&sp->dst); cudaFree(sp->mu1_dev); delete sp; return cuda_fail("cudaMalloc tiles");
    }
    cudaMemcpy(sp->tiles_dev, tiles.data(), sizeof(int2) * tiles.size(), cudaMemcpyHostToDevice);
  }
  if (const int rc = build_seg_tiles(sp); rc != BHCP_OK) {
    const std::string msg = g_last_error;
    bhcp_space_plan_destroy(sp);
    return fail(rc, msg);
  }
  if (const cudaError_t e = cudaGetLastError(); e != cudaSuccess) {   // a failed table upload
    bhcp_space_plan_destroy(sp);
    return fail(BHCP_ERR_CUDA, std::string("space plan upload: ") + cudaGetErrorString(e));
  }
  *out = sp;
  return BHCP_OK;
}

void bhcp_space_plan_destroy(bhcp_space_plan* sp) {
  if (!sp) return;
  DeviceGuard g(sp->device);
  free_fft_plan(&sp->dst);
  cudaFree(sp->mu1_dev);
  if (sp->tiles_dev) cudaFree(sp->tiles_dev);
  cudaFree(sp->twN);
  cudaFree(sp->snN);
  for (int i = 0; i < 9; ++i)
    if (sp->seg_tiles[i]) cudaFree(sp->seg_tiles[i]);
  delete sp;
}

int bhcp_time_plan_create(int device, int n_levels, const double* gamma_host, const double* gamma_inv_host,
                          const double* shifts_host, bhcp_time_plan** out) {
  if (!out || !gamma_host || !gamma_inv_host || !shifts_host) return fail(BHCP_ERR_INVALID, "null argument");
  if (n_levels < 1) return fail(BHCP_ERR_INVALID, "n_levels must be >= 1");
  DeviceGuard g(device);
  std::string err;
  if (!ensure_device_constants(device, &err)) return fail(BHCP_ERR_CUDA, err);
  auto* tp = new bhcp_time_plan();
  tp->device = device; tp->n = n_levels;
  if (!build_fft_plan(n_levels, &tp->fft, &err)) { delete tp; return fail(BHCP_ERR_INVALID, err); }
  const size_t nb = sizeof(double2) * n_levels;
  if (cudaMalloc(&tp->tables, 3 * nb) != cudaSuccess) {
    free_fft_plan(&tp->fft); delete tp; return cuda_fail("cudaMalloc time tables");
  }
  cudaMemcpy(tp->tables, gamma_host, nb, cudaMemcpyHostToDevice);
  cudaMemcpy(tp->tables + n_levels, gamma_inv_host, nb, cudaMemcpyHostToDevice);
  cudaMemcpy(tp->tables + 2 * n_levels, shifts_host, nb, cudaMemcpyHostToDevice);
  tp->blue = nullptr;
  if (n_levels == 257 || n_levels == 1025 || n_levels == 4097) {
    std::vector<double2> tabs;
    if (!build_blue_tables(n_levels, &tabs, &err)) {
      free_fft_plan(&tp->fft); cudaFree(tp->tables); delete tp; return fail(BHCP_ERR_INVALID, err);
    }
    // fused sink / generator tables: cg_t = chirp_t / gamma_t, wg_t = w^{Mt} / gamma_t,
    // thr_j = 1e-28 |s_j|^2 (space.py:237-240), products rounded once from long double
    {
      const int L = 2 * (n_levels - 1);
      const double2* chirp = tabs.data() + L;
      const double2* wM = tabs.data() + 2 * L + n_levels;
      for (int t = 0; t < n_levels; ++t) {
        const long double gr = gamma_inv_host[2 * t], gi = gamma_inv_host[2 * t + 1];
        const long double cr = chirp[t].x, ci = chirp[t].y, wr = wM[t].x, wi = wM[t].y;
        tabs.push_back(make_double2((double)(cr * gr - ci * gi), (double)(cr * gi + ci * gr)));
      }
      for (int t = 0; t < n_levels; ++t) {
        const long double gr = gamma_inv_host[2 * t], gi = gamma_inv_host[2 * t + 1];
        const long double wr = wM[t].x, wi = wM[t].y;
        tabs.push_back(make_double2((double)(wr * gr - wi * gi), (double)(wr * gi + wi * gr)));
      }
      for (int j = 0; j < n_levels; ++j) {
        const double sr = shifts_host[2 * j], si = shifts_host[2 * j + 1];
        tabs.push_back(make_double2(1e-28 * (sr * sr + si * si), 0.0));
      }
    }
    if (cudaMalloc(&tp->blue, sizeof(double2) * tabs.size()) != cudaSuccess) {
      free_fft_plan(&tp->fft); cudaFree(tp->tables); delete tp; return cuda_fail("cudaMalloc blue tables");
    }
    cudaMemcpy(tp->blue, tabs.data(), sizeof(double2) * tabs.size(), cudaMemcpyHostToDevice);
  }
  tp->rader = nullptr;
  tp->rader_idx = nullptr;
  tp->gt = nullptr;
  tp->gt_idx = nullptr;
  tp->pf = nullptr;
  tp->pf_idx = nullptr;
  if (n_levels == 4097) {
    std::vector<double2> pc;
    std::vector<int> tq, perm;
    if (!build_pf_tables(&pc, &tq, &perm, &err)) { bhcp_time_plan_destroy(tp); return fail(BHCP_ERR_INVALID, err); }
    // shifts in prime-factor input order (row, slot); the kernel derives the
    // singular thresholds and, when one fires, the time index from them and tq
    for (int i = 0; i < 4097; ++i) {
      const int row = i / 241, slot = i - row * 241;
      const int j2 = slot ? perm[slot - 1] : 0;
      const int j = (241 * row + 17 * j2) % 4097;
      pc.push_back(make_double2(shifts_host[2 * j], shifts_host[2 * j + 1]));
    }
    if (cudaMalloc(&tp->pf, sizeof(double2) * pc.size()) != cudaSuccess ||
        cudaMalloc(&tp->pf_idx, sizeof(int) * tq.size()) != cudaSuccess) {
      bhcp_time_plan_destroy(tp); return cuda_fail("cudaMalloc pf tables");
    }
    cudaMemcpy(tp->pf, pc.data(), sizeof(double2) * pc.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(tp->pf_idx, tq.data(), sizeof(int) * tq.size(), cudaMemcpyHostToDevice);
  }
  tp->shifts_h.resize(n_levels);
  for (int j = 0; j < n_levels; ++j) tp->shifts_h[j] = make_double2(shifts_host[2 * j], shifts_host[2 * j + 1]);
  if (n_levels == 1025) {
    std::vector<double2> gc;
    std::vector<int> gi;
    if (!build_gt2_tables(shifts_host, gamma_inv_host, &gc, &gi, &err)) {
      bhcp_time_plan_destroy(tp); return fail(BHCP_ERR_INVALID, err);
    }
    if (cudaMalloc(&tp->gt, sizeof(double2) * gc.size()) != cudaSuccess ||
        cudaMalloc(&tp->gt_idx, sizeof(int) * gi.size()) != cudaSuccess) {
      bhcp_time_plan_destroy(tp); return cuda_fail("cudaMalloc gt tables");
    }
    cudaMemcpy(tp->gt, gc.data(), sizeof(double2) * gc.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(tp->gt_idx, gi.data(), sizeof(int) * gi.size(), cudaMemcpyHostToDevice);
  }
  if (n_levels == 257) {
    std::vector<double2> rc;
    std::vector<int> ri;
    if (!build_rader_tables(n_levels, &rc, &ri, &err)) {
      bhcp_time_plan_destroy(tp); return fail(BHCP_ERR_INVALID, err);
    }
    if (cudaMalloc(&tp->rader, sizeof(double2) * rc.size()) != cudaSuccess ||
        cudaMalloc(&tp->rader_idx, sizeof(int) * ri.size()) != cudaSuccess) {
      bhcp_time_plan_destroy(tp); return cuda_fail("cudaMalloc rader tables");
    }
    cudaMemcpy(tp->rader, rc.data(), sizeof(double2) * rc.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(tp->rader_idx, ri.data(), sizeof(int) * ri.size(), cudaMemcpyHostToDevice);
  }
  if (const cudaError_t e = cudaGetLastError(); e != cudaSuccess) {   // a failed table upload
    bhcp_time_plan_destroy(tp);
    return fail(BHCP_ERR_CUDA, std::string("time plan upload: ") + cudaGetErrorString(e));
  }
  *out = tp;
  return BHCP_OK;
}

void bhcp_time_plan_destroy(bhcp_time_plan* tp) {
  if (!tp) return;
  DeviceGuard g(tp->device);
  free_fft_plan(&tp->fft);
  cudaFree(tp->tables);
  if (tp->blue) cudaFree(tp->blue);
  if (tp->rader) cudaFree(tp->rader);
  if (tp->rader_idx) cudaFree(tp->rader_idx);
  if (tp->gt) cudaFree(tp->gt);
  if (tp->gt_idx) cudaFree(tp->gt_idx);
  if (tp->pf) cudaFree(tp->pf);
  if (tp->pf_idx) cudaFree(tp->pf_idx);
  delete tp;
}

int bhcp_status_reset(void* status_dev, void* stream) {
  if (!status_dev) return fail(BHCP_ERR_INVALID, "null status");
  k_status_reset<<<1, 32, 0, as_stream(stream)>>>(reinterpret_cast<StatusDev*>(status_dev));
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("status reset");
  return BHCP_OK;
}

int bhcp_read_status(const void* status_dev, double tol, bhcp_status* st, void* stream) {
  if (!status_dev || !st) return fail(BHCP_ERR_INVALID, "null argument");
  if (cudaStreamSynchronize(as_stream(stream)) != cudaSuccess) return cuda_fail("stream sync");
  StatusDev h;
  if (cudaMemcpy(&h, status_dev, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_fail("status copy");
  st->bad_column = h.bad_col == ~0ull ? -1 : (int64_t)h.bad_col;
  st->norm = sqrt(h.sum_re2 + h.sum_im2);
  st->residue = sqrt(h.sum_im2);
  st->code = BHCP_OK;
  if (st->bad_column >= 0) st->code = BHCP_ERR_SINGULAR_SHIFT;
  else if (st->residue > tol * fmax(st->norm, 2.2250738585072014e-308)) st->code = BHCP_ERR_IMAGINARY_RESIDUE;
  return BHCP_OK;
}

int bhcp_sine_transform(const bhcp_space_plan* sp, const void* in, void* out, int is_complex, int64_t batch,
                        void* stream) {
  if (!sp || !in || !out || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  return sine_passes(sp, (const double*)in, (double*)out, is_complex ? 1 : 0, batch, as_stream(stream));
}

int bhcp_sine_axis(const bhcp_space_plan* sp, const void* in, void* out, int is_complex, int64_t batch, int axis,
                   void* stream) {
  if (!sp || !in || !out || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  if (axis < 0 || axis >= sp->dim) return fail(BHCP_ERR_INVALID, "axis out of range");
  DeviceGuard g(sp->device);
  const int d = sp->dim, m = sp->m;
  const int cplx = is_complex ? 1 : 0;
  if (axis == 0)
    return launch_rows(sp, (const double*)in, (double*)out, cplx, batch * ipow(m, d - 1), 0, nullptr, nullptr,
                       as_stream(stream), Blocked(), ipow(m, d - 1));
  return launch_cols(sp, (const double*)in, (double*)out, cplx, ipow(m, axis), batch * ipow(m, d - 1 - axis), axis,
                     0, nullptr, nullptr, as_stream(stream));
}

int bhcp_step_b(const bhcp_space_plan* sp, const void* in, void* out, const double* shifts_dev, int64_t batch,
                void* status_dev, void* stream) {
  if (!sp || !in || !out || !shifts_dev || !status_dev || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  return step_b_passes(sp, (const double*)in, (double*)out, batch, (const double2*)shifts_dev,
                       (StatusDev*)status_dev, as_stream(stream));
}

int bhcp_to_eigenspace(const bhcp_time_plan* tp, const void* in, int in_is_complex, int64_t batch, int64_t in_sb,
                       int64_t in_st, void* out, int64_t out_sb, int64_t out_st, void* stream) {
  if (!tp || !in || !out || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(tp->device);
  return launch_time(tp, 0, (const double*)in, in_is_complex ? 1 : 0, batch, in_sb, in_st, (double*)out, 1,
                     out_sb, out_st, nullptr, as_stream(stream));
}

int bhcp_from_eigenspace(const bhcp_time_plan* tp, const void* in, int64_t batch, int64_t in_sb, int64_t in_st,
                         void* out, int out_is_complex, int64_t out_sb, int64_t out_st, void* status_dev,
                         void* stream) {
  if (!tp || !in || !out || !status_dev || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(tp->device);
  return launch_time(tp, 1, (const double*)in, 1, batch, in_sb, in_st, (double*)out, out_is_complex ? 1 : 0,
                     out_sb, out_st, (StatusDev*)status_dev, as_stream(stream));
}

size_t bhcp_pint_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp) {
  if (!sp || !tp) return 0;
  return align256(sizeof(StatusDev)) + align256(sizeof(double) * sp->nx) +
         align256(sizeof(double) * (size_t)native_w_elems(sp, tp->n)) +
         (lvl4_ok(sp) ? align256(lvl4_sync_bytes(tp->n)) : 0);
}

void* bhcp_pint_status_ptr(const bhcp_space_plan*, const bhcp_time_plan*, void* ws) { return ws; }

int bhcp_pint_ghat(const bhcp_space_plan* sp, const double* g_dev, double scale, double* ghat_dev, void* stream) {
  if (!sp || !g_dev || !ghat_dev) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  int rc = sine_passes(sp, g_dev, ghat_dev, 0, 1, s);
  if (rc) return rc;
  if (scale != 1.0) {
    k_scale<<<(unsigned)((sp->nx + 255) / 256 < 4096 ? (sp->nx + 255) / 256 : 4096), 256, 0, s>>>(ghat_dev, scale,
                                                                                                  sp->nx, ghat_dev);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_scale");
  }
  return BHCP_OK;
}

int bhcp_pint_modes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat_dev, int64_t k_begin,
                    int64_t k_end, double* w_dev, int nslabs, const int64_t* slab_bounds, void* status_dev,
                    void* stream) {
  if (!sp || !tp || !ghat_dev || !w_dev || !status_dev) return fail(BHCP_ERR_INVALID, "bad argument");
  if (k_begin < 0 || k_end > sp->nx || k_begin > k_end) return fail(BHCP_ERR_INVALID, "bad mode range");
  if (nslabs < 0 || nslabs > 8) return fail(BHCP_ERR_INVALID, "nslabs must be in [0, 8]");
  DeviceGuard g(sp->device);
  fastk::WLayout wl = native_layout(sp, k_end - k_begin, tp->n);
  if (nslabs > 0) {
    if (sp->dim < 2) return fail(BHCP_ERR_INVALID, "level slabs need dim >= 2");
    const long long P1 = ipow(sp->m, sp->dim - 1);
    if (k_begin % P1 || k_end % P1) return fail(BHCP_ERR_INVALID, "mode range must hold whole k1 planes");
    if (!slab_bounds || slab_bounds[0] != 0 || slab_bounds[nslabs] != tp->n)
      return fail(BHCP_ERR_INVALID, "slab bounds must cover [0, n_levels)");
    for (int i = 1; i <= nslabs; ++i) {
      if (slab_bounds[i] < slab_bounds[i - 1]) return fail(BHCP_ERR_INVALID, "slab bounds not sorted");
      if (i < nslabs && slab_bounds[i] % fastk::kTBL && slab_bounds[i] != tp->n)
        return fail(BHCP_ERR_INVALID, "slab bounds must be multiples of 8");
    }
    wl = make_blocked(sp, k_end - k_begin, nslabs, (const long long*)slab_bounds);
  }
  return launch_modes(sp, tp, ghat_dev, 1.0, k_begin, k_end, w_dev, wl, (StatusDev*)status_dev,
                      as_stream(stream));
}

int bhcp_pint_modes_to(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat_dev, int64_t k_begin,
                       int64_t k_end, double* const* slab_dst, int nslabs, const int64_t* slab_bounds,
                       void* status_dev, void* stream) {
  if (!sp || !tp || !ghat_dev || !slab_dst || !status_dev) return fail(BHCP_ERR_INVALID, "bad argument");
  if (nslabs < 1 || nslabs > 8) return fail(BHCP_ERR_INVALID, "nslabs must be in [1, 8]");
  for (int s = 0; s < nslabs; ++s)
    if (!slab_dst[s]) return fail(BHCP_ERR_INVALID, "null slab destination");
  if (k_begin < 0 || k_end > sp->nx || k_begin > k_end) return fail(BHCP_ERR_INVALID, "bad mode range");
  if (sp->dim < 2) return fail(BHCP_ERR_INVALID, "level slabs need dim >= 2");
  const long long P1 = ipow(sp->m, sp->dim - 1);
  if (k_begin % P1 || k_end % P1) return fail(BHCP_ERR_INVALID, "mode range must hold whole k1 planes");
  if (!slab_bounds || slab_bounds[0] != 0 || slab_bounds[nslabs] != tp->n)
    return fail(BHCP_ERR_INVALID, "slab bounds must cover [0, n_levels)");
  for (int i = 1; i <= nslabs; ++i) {
    if (slab_bounds[i] < slab_bounds[i - 1]) return fail(BHCP_ERR_INVALID, "slab bounds not sorted");
    if (i < nslabs && slab_bounds[i] % fastk::kTBL && slab_bounds[i] != tp->n)
      return fail(BHCP_ERR_INVALID, "slab bounds must be multiples of 8");
  }
  DeviceGuard g(sp->device);
  fastk::WLayout wl = make_blocked(sp, k_end - k_begin, nslabs, (const long long*)slab_bounds);
  for (int s = 0; s < nslabs; ++s) wl.sl_base[s] = slab_dst[s];
  return launch_modes(sp, tp, ghat_dev, 1.0, k_begin, k_end, slab_dst[0], wl, (StatusDev*)status_dev,
                      as_stream(stream));
}

int64_t bhcp_pint_sym_tiles(const bhcp_space_plan* sp, const bhcp_time_plan* tp) {
  if (!sp || !tp || sp->dim < 2 || g_disable_fast) return 0;
  DeviceGuard g(sp->device);
  long long cnt = 0;
  const int4* t = nullptr;
  if (tp->rader && tp->n == 257) t = seg_tiles(sp, fastk::RaderPlan<257>::S, &cnt, sp->dim == 3);
  else if (tp->gt && tp->n == 1025) t = seg_tiles(sp, fastk::GtPlan::S, &cnt);
  else if (tp->pf && tp->n == 4097) t = seg_tiles(sp, 1, &cnt);
  else if (tp->blue && tp->n == 4097) t = seg_tiles(sp, fastk::BluePlan<4097>::S, &cnt);
  else if (tp->blue && tp->n == 257) t = seg_tiles(sp, fastk::BluePlan<257>::S, &cnt);
  else if (tp->blue && tp->n == 1025) t = seg_tiles(sp, fastk::BluePlan<1025>::S, &cnt);
  else if (tp->n == 513 && sp->dim == 2 && sp->tiles_dev) return sp->ntiles;
  return t ? cnt : 0;
}

int bhcp_pint_modes_sym_to(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* ghat_dev,
                           int64_t tile_begin, int64_t tile_end, double* const* slab_dst,
                           const int64_t* const* slab_koff, int nslabs, const int64_t* slab_bounds,
                           void* status_dev, void* stream) {
  if (!sp || !tp || !ghat_dev || !slab_dst || !slab_koff || !status_dev) return fail(BHCP_ERR_INVALID, "bad argument");
  if (nslabs < 1 || nslabs > 8) return fail(BHCP_ERR_INVALID, "nslabs must be in [1, 8]");
  const int64_t total = bhcp_pint_sym_tiles(sp, tp);
  if (total <= 0) return fail(BHCP_ERR_INVALID, "no symmetric work list for this grid / time length");
  if (tile_begin < 0 || tile_end < tile_begin || tile_end > total) return fail(BHCP_ERR_INVALID, "bad tile range");
  for (int s = 0; s < nslabs; ++s)
    if (!slab_dst[s] || !slab_koff[s]) return fail(BHCP_ERR_INVALID, "null slab destination or table");
  if (!slab_bounds || slab_bounds[0] != 0 || slab_bounds[nslabs] != tp->n)
    return fail(BHCP_ERR_INVALID, "slab bounds must cover [0, n_levels)");
  for (int i = 1; i <= nslabs; ++i) {
    if (slab_bounds[i] < slab_bounds[i - 1]) return fail(BHCP_ERR_INVALID, "slab bounds not sorted");
    if (i < nslabs && slab_bounds[i] % fastk::kTBL && slab_bounds[i] != tp->n)
      return fail(BHCP_ERR_INVALID, "slab bounds must be multiples of 8");
  }
  DeviceGuard g(sp->device);
  fastk::WLayout wl = make_blocked(sp, sp->nx, nslabs, (const long long*)slab_bounds);
  for (int s = 0; s < nslabs; ++s) {
    wl.sl_base[s] = slab_dst[s];
    wl.sl_koff[s] = (const long long*)slab_koff[s];
  }
  SymRange sr;
  sr.on = true;
  sr.begin = tile_begin;
  sr.end = tile_end;
  return launch_modes(sp, tp, ghat_dev, 1.0, 0, sp->nx, slab_dst[0], wl, (StatusDev*)status_dev,
                      as_stream(stream), sr);
}

int bhcp_pint_level_pass(const bhcp_space_plan* sp, const double* in_dev, const int64_t* koff_dev, double* y_dev,
                         int64_t nlev, int pass, void* stream) {
  if (!sp || !in_dev || !y_dev || nlev < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  if (pass < 0 || pass >= sp->dim) return fail(BHCP_ERR_INVALID, "pass out of range");
  DeviceGuard g(sp->device);
  return level_pass(sp, in_dev, (const long long*)koff_dev, y_dev, nlev, pass, as_stream(stream));
}

int bhcp_pint_w_pass(const bhcp_space_plan* sp, double* w_dev, int64_t nlev, int axis, void* stream) {
  if (!sp || !w_dev || nlev < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  return w_pass(sp, w_dev, nlev, axis, as_stream(stream));
}

int bhcp_pint_w_passes_supported(const bhcp_space_plan* sp) { return sp && wax_ok(sp) ? 1 : 0; }

int bhcp_pint_levels(const bhcp_space_plan* sp, double* in_dev, double* out_dev, int64_t batch,
                     void* stream) {
  if (!sp || !in_dev || !out_dev || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  return levels_all(sp, in_dev, nullptr, out_dev, batch, as_stream(stream));
}

int bhcp_pint_solve(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* g_dev, double divisor,
                    double* y_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!sp || !tp || !g_dev || !y_dev || !ws) return fail(BHCP_ERR_INVALID, "null argument");
  if (ws_bytes < bhcp_pint_workspace_bytes(sp, tp)) return fail(BHCP_ERR_INVALID, "workspace too small");
  if (sp->device != tp->device) return fail(BHCP_ERR_INVALID, "plans on different devices");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  char* w = (char*)ws;
  StatusDev* st = (StatusDev*)w;
  double* ghat = (double*)(w + align256(sizeof(StatusDev)));
  double* W = (double*)(w + align256(sizeof(StatusDev)) + align256(sizeof(double) * sp->nx));
  unsigned* gsync = (unsigned*)((char*)W + align256(sizeof(double) * (size_t)native_w_elems(sp, tp->n)));
  k_status_reset<<<1, 32, 0, s>>>(st);
  int rc = sine_passes(sp, g_dev, ghat, 0, 1, s);
  if (rc) return rc;
  const double cscale = 1.0 / (divisor * (double)tp->n);
  rc = launch_modes(sp, tp, ghat, cscale, 0, sp->nx, W, native_layout(sp, sp->nx, tp->n), st, s);
  if (rc) return rc;
  return levels_all(sp, W, nullptr, y_dev, tp->n, s, gsync);
}

size_t bhcp_pint_batch_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp, int nb) {
  if (!sp || !tp || nb < 1) return 0;
  return align256(sizeof(double) * sp->nx) + (size_t)nb * align256(sizeof(double) * (size_t)native_w_elems(sp, tp->n));
}

int bhcp_pint_solve_batch(const bhcp_space_plan* sp, const bhcp_time_plan* const* tps, int nb, const double* g_dev,
                          const double* divisors, double* y_dev, void* status_dev, void* ws, size_t ws_bytes,
                          void* stream) {
  if (!sp || !tps || nb < 1 || !g_dev || !divisors || !y_dev || !status_dev || !ws)
    return fail(BHCP_ERR_INVALID, "null argument");
  const bhcp_time_plan* tp0 = tps[0];
  for (int i = 0; i < nb; ++i) {
    if (!tps[i]) return fail(BHCP_ERR_INVALID, "null time plan");
    if (tps[i]->n != tp0->n) return fail(BHCP_ERR_INVALID, "time plans of different lengths");
    if (tps[i]->device != sp->device) return fail(BHCP_ERR_INVALID, "plans on different devices");
    if (!(divisors[i] != 0.0)) return fail(BHCP_ERR_INVALID, "divisor must be nonzero");
  }
  if (ws_bytes < bhcp_pint_batch_workspace_bytes(sp, tp0, nb)) return fail(BHCP_ERR_INVALID, "workspace too small");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  StatusDev* st = (StatusDev*)status_dev;
  double* ghat = (double*)ws;
  double* W = (double*)((char*)ws + align256(sizeof(double) * sp->nx));
  const long long w_stride = (long long)(align256(sizeof(double) * (size_t)native_w_elems(sp, tp0->n)) / sizeof(double));
  const long long n = tp0->n, nx = sp->nx;
  k_status_reset_n<<<1, 128, 0, s>>>(st, nb);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("status reset");
  int rc = sine_passes(sp, g_dev, ghat, 0, 1, s);   // one DST of g serves every pair
  if (rc) return rc;
  std::vector<double> cs(nb);
  for (int i = 0; i < nb; ++i) cs[i] = 1.0 / (divisors[i] * (double)n);
  if (sp->dim == 1 && !g_disable_fast && n == 4097 && tp0->pf) {
    for (int i = 0; i < nb; ++i)
      if (!tps[i]->pf) return fail(BHCP_ERR_INVALID, "time plan without prime-factor tables");
    fastk::WLayout wl = native_layout(sp, nx, n);
    wl.sl_base[0] = W;
    rc = pf_modes_batch(sp, tps, nb, ghat, cs.data(), wl, w_stride, st, s);
    if (rc) return rc;
    // level phase of every pair at once: mode-major W -> level-major y, then the
    // rows DST over nb * n levels, lines paired inside each solve (lpl = n: the
    // pairs of a single solve, so every trajectory is bitwise the unbatched one)
    const long long NT1 = (n + fastk::kTBL - 1) / fastk::kTBL;
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((sp->m + 31) / 32), (unsigned)nb);
    k_transpose_ld_batch<<<grid, dim3(32, 8), 0, s>>>(W, NT1 * fastk::kTBL, w_stride, y_dev, sp->m, n);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_transpose_ld_batch");
    return launch_rows(sp, y_dev, y_dev, 0, (long long)nb * n, 0, nullptr, nullptr, s, Blocked(), n);
  }
  // other shapes: the single-solve pipeline per pair (W slots of the workspace)
  for (int i = 0; i < nb; ++i) {
    double* Wi = W + (long long)i * w_stride;
    rc = launch_modes(sp, tps[i], ghat, cs[i], 0, nx, Wi, native_layout(sp, nx, n), st + i, s);
    if (rc) return rc;
    rc = levels_all(sp, Wi, nullptr, y_dev + (long long)i * n * nx, n, s);
    if (rc) return rc;
  }
  return BHCP_OK;
}

size_t bhcp_pint_levels_sync_bytes(const bhcp_space_plan* sp, int64_t nlev) {
  if (!sp || nlev <= 0 || !lvl4_ok(sp)) return 0;
  return lvl4_sync_bytes(nlev);
}

int bhcp_pint_levels_fused(const bhcp_space_plan* sp, const double* in_dev, double* out_dev, int64_t nlev,
                           void* sync_dev, void* stream) {
  if (!sp || !in_dev || !out_dev || nlev < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  if (lvl4_ok(sp)) {
    if (!sync_dev) return fail(BHCP_ERR_INVALID, "the level-group pass needs a sync buffer");
    return lvl4_launch(sp, in_dev, out_dev, nlev, (unsigned*)sync_dev, s);
  }
  return levels_all(sp, const_cast<double*>(in_dev), nullptr, out_dev, nlev, s);
}

int bhcp_pint_levels_blocked(const bhcp_space_plan* sp, double* in_dev, const int64_t* koff_dev,
                             double* out_dev, int64_t batch, void* stream) {
  if (!sp || !in_dev || !out_dev || batch < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  if (sp->dim < 2) return fail(BHCP_ERR_INVALID, "blocked level input needs dim >= 2");
  DeviceGuard g(sp->device);
  return levels_all(sp, in_dev, (const long long*)koff_dev, out_dev, batch, as_stream(stream));
}

size_t bhcp_pint_unfused_workspace_bytes(const bhcp_space_plan* sp, const bhcp_time_plan* tp) {
  if (!sp || !tp) return 0;
  return align256(sizeof(StatusDev)) + align256(sizeof(double2) * sp->nx * (size_t)tp->n);
}

void* bhcp_pint_unfused_status_ptr(const bhcp_space_plan*, const bhcp_time_plan*, void* ws) { return ws; }

int bhcp_pint_solve_unfused(const bhcp_space_plan* sp, const bhcp_time_plan* tp, const double* g_dev,
                            double divisor, double* y_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!sp || !tp || !g_dev || !y_dev || !ws) return fail(BHCP_ERR_INVALID, "null argument");
  if (ws_bytes < bhcp_pint_unfused_workspace_bytes(sp, tp)) return fail(BHCP_ERR_INVALID, "workspace too small");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  char* w = (char*)ws;
  StatusDev* st = (StatusDev*)w;
  double* S = (double*)(w + align256(sizeof(StatusDev)));
  const long long nx = sp->nx, n = tp->n, total = nx * n;
  k_status_reset<<<1, 32, 0, s>>>(st);
  // rhs assembly (methods.py:158-162) into y, used as scratch
  k_rhs<<<(unsigned)(total / 256 + 1 < 65535 ? total / 256 + 1 : 65535), 256, 0, s>>>(g_dev, 0.0, divisor, nx,
                                                                                      total, y_dev);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_rhs");
  // step (a): sequences are spatial points x, time stride nx
  int rc = launch_time(tp, 0, y_dev, 0, nx, 1, nx, S, 1, 1, nx, nullptr, s);
  if (rc) return rc;
  // step (b): level-major complex fields
  rc = step_b_passes(sp, S, S, n, tp->tables + 2 * n, st, s);
  if (rc) return rc;
  // step (c)
  return launch_time(tp, 1, S, 1, nx, 1, nx, y_dev, 0, 1, nx, st, s);
}

size_t bhcp_spectral_workspace_bytes(const bhcp_space_plan* sp, int64_t n_levels) {
  if (!sp) return 0;
  return align256(sizeof(double) * sp->nx) + align256(sizeof(double) * native_w_elems(sp, (int)n_levels));
}

int bhcp_spectral_solve(const bhcp_space_plan* sp, int kind, double alpha, double tau, int64_t num_steps,
                        const double* g_dev, double* y_dev, void* ws, size_t ws_bytes, void* stream) {
  if (!sp || !g_dev || !y_dev || !ws || kind < 0 || kind > 3 || num_steps < 1) return fail(BHCP_ERR_INVALID, "bad argument");
  const long long n = num_steps + 1;
  if (ws_bytes < bhcp_spectral_workspace_bytes(sp, n)) return fail(BHCP_ERR_INVALID, "workspace too small");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  double* ghat = (double*)ws;
  double* W = (double*)((char*)ws + align256(sizeof(double) * sp->nx));
  int rc = sine_passes(sp, g_dev, ghat, 0, 1, s);
  if (rc) return rc;
  SpectralArgs a{};
  a.ghat = ghat; a.mu1 = sp->mu1_dev; a.m = sp->m; a.dim = sp->dim; a.kind = kind; a.alpha = alpha; a.tau = tau;
  a.num_steps = num_steps; a.n = n; a.W = W; a.wl = native_layout(sp, sp->nx, (int)n);
  a.wl.bind(W);
  k_spectral_w<<<2048, dim3(32, 8), 0, s>>>(a, sp->nx);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_spectral_w");
  for (int p = 0; p < sp->dim; ++p) {
    rc = level_pass(sp, W, nullptr, y_dev, n, p, s);
    if (rc) return rc;
  }
  return BHCP_OK;
}

int bhcp_march_forward(const bhcp_space_plan* sp, double tau, int64_t num_steps, const double* z0_dev,
                       double* g_dev, void* stream) {
  if (!sp || !z0_dev || !g_dev || num_steps < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  int rc = sine_passes(sp, z0_dev, g_dev, 0, 1, s);
  if (rc) return rc;
  k_decay<<<(unsigned)std::min<long long>((sp->nx + 255) / 256, 4096), 256, 0, s>>>(g_dev, sp->mu1_dev, sp->m, sp->dim,
                                                                                   tau, (double)num_steps, sp->nx);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_decay");
  return sine_passes(sp, g_dev, g_dev, 0, 1, s);
}

size_t bhcp_residual_workspace_bytes(void) { return sizeof(double) * (2 * 1184 + 2); }

int bhcp_residual_norm(const bhcp_space_plan* sp, const double* y_dev, int64_t n_levels, double tau, double divisor,
                       double h, const double* g_dev, void* ws, double* result_host, void* stream) {
  if (!sp || !y_dev || !g_dev || !ws || !result_host || n_levels < 1) return fail(BHCP_ERR_INVALID, "bad argument");
  DeviceGuard g(sp->device);
  cudaStream_t s = as_stream(stream);
  ResidualArgs a{};
  a.y = y_dev; a.g = g_dev; a.n = n_levels; a.nx = sp->nx; a.m = sp->m; a.dim = sp->dim;
  a.inv_tau = 1.0 / tau; a.corner = 1.0 / divisor; a.inv_div = 1.0 / divisor; a.inv_h2 = 1.0 / (h * h);
  const int nblk = 1184;  // 8 x 148 SMs, fixed for a deterministic reduction order
  double* part = (double*)ws;
  a.partial = part;
  k_residual<<<nblk, 256, 0, s>>>(a);
  k_residual_finish<<<1, 1024, 0, s>>>(part, nblk, part + 2 * nblk);
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_residual");
  double out[2];
  if (cudaMemcpyAsync(out, part + 2 * nblk, sizeof(out), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return cuda_fail("residual copy");
  result_host[0] = sqrt(out[0]);
  result_host[1] = sqrt(out[1]);
  return BHCP_OK;
}

int bhcp_transpose(const void* in, void* out, int64_t rows, int64_t cols, int elem_bytes, void* stream) {
  if (!in || !out || rows < 0 || cols < 0) return fail(BHCP_ERR_INVALID, "bad argument");
  if (rows == 0 || cols == 0) return BHCP_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) return fail(BHCP_ERR_INVALID, "transpose too tall");
  dim3 block(32, 8);
  if (elem_bytes == 8)
    k_transpose<double><<<grid, block, 0, as_stream(stream)>>>((const double*)in, (double*)out, rows, cols);
  else if (elem_bytes == 16)
    k_transpose<double2><<<grid, block, 0, as_stream(stream)>>>((const double2*)in, (double2*)out, rows, cols);
  else
    return fail(BHCP_ERR_INVALID, "elem_bytes must be 8 or 16");
  if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("k_transpose");
  return BHCP_OK;
}

}  // extern "C"
