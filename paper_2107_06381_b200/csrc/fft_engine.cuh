// fft_engine.cuh -- CTA-cooperative fp64 complex FFT in shared memory (sm_100a).
//
// Replaces the pocketfft transforms the reference reaches through
// numpy.fft.ifft / numpy.fft.fft (pkg/src/bhcp/circulant.py:106,115) and
// scipy.fft.dst (pkg/src/bhcp/space.py:172-176).
//
// Design
//  * A CTA transforms `nseq` independent sequences that live in shared
//    memory, each occupying `Lc` double2 slots (Lc = L for a direct plan,
//    Lc = the Bluestein convolution length otherwise).
//  * Direct plans are mixed-radix Stockham autosort transforms (Govindaraju
//    et al. 2008 formulation): stage s with radix R reads the R inputs of a
//    butterfly at stride L/R, applies twiddles w_{Ns R}^{r k}, runs a radix-R
//    codelet in registers and writes the outputs at stride Ns. Each stage is
//    done in place: every thread first computes all of its butterflies into
//    registers, the CTA synchronises, then the results are stored. A thread
//    holds stage_slots(R, CAP) butterflies, so nseq*Lc <= blockDim.x *
//    min_R stage_capacity(R, CAP) is the capacity rule (checked by the host).
//  * Radices: 2, 4, 8 and the odd primes 3..23 (symmetric real-coefficient
//    codelet, constants in __constant__ memory). Lengths with a larger prime
//    factor use Bluestein's chirp-z algorithm with a smooth convolution length.
//  * Only the forward (e^{-2 pi i}) transform is implemented; callers obtain
//    the inverse as conj(FFT(conj(x))) by conjugating in their load/store.
//  * Twiddle tables are precomputed on the host in long double and rounded
//    once, so the per-transform error stays at pocketfft's ~1e-16 level.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft_types.h"

namespace bhcp {

// cos/sin(2 pi q / R) for the odd-prime codelets, packed per radix.
// Offsets: 3:0 5:3 7:8 11:15 13:26 17:39 19:56 23:75 -> 98 entries.
constexpr int kOddRootsTotal = 98;
__host__ __device__ constexpr int odd_root_offset(int R) {
  return R == 3 ? 0 : R == 5 ? 3 : R == 7 ? 8 : R == 11 ? 15 : R == 13 ? 26
       : R == 17 ? 39 : R == 19 ? 56 : R == 23 ? 75 : -1;
}
// Defined here: only bhcp_b200.cu (a single translation unit) includes this header.
__constant__ double c_root_cos[kOddRootsTotal];
__constant__ double c_root_sin[kOddRootsTotal];

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by -i
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

// ---------------------------------------------------------------- codelets
// Each codelet is split in two phases around the stage barrier:
//   prep(v)            runs before the barrier on the loaded (twiddled) inputs
//   emit(v, out, Ns)   runs after it and writes X_r to out[r * Ns]
// Power-of-two codelets do all the work in prep; the odd-prime codelet keeps
// only the R symmetric combinations live across the barrier and produces the
// outputs straight into shared memory, which halves its register footprint.
template <int R> struct Dft;

template <> struct Dft<2> {
  static __device__ __forceinline__ void prep(double2 (&v)[2]) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
  static __device__ __forceinline__ void emit(const double2 (&v)[2], double2* out, int Ns) {
    out[0] = v[0];
    out[Ns] = v[1];
  }
};

template <> struct Dft<4> {
  static __device__ __forceinline__ void prep(double2 (&v)[4]) {
    double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    double2 a2 = cadd(v[1], v[3]), a3 = cmul_mi(csub(v[1], v[3]));
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, a3);
    v[3] = csub(a1, a3);
  }
  static __device__ __forceinline__ void emit(const double2 (&v)[4], double2* out, int Ns) {
#pragma unroll
    for (int r = 0; r < 4; ++r) out[r * Ns] = v[r];
  }
};

template <> struct Dft<8> {
  static __device__ __forceinline__ void prep(double2 (&v)[8]) {
    const double s = 0.70710678118654752440084436210485;
    double2 a0 = cadd(v[0], v[4]), a1 = csub(v[0], v[4]);
    double2 a2 = cadd(v[2], v[6]), a3 = cmul_mi(csub(v[2], v[6]));
    double2 a4 = cadd(v[1], v[5]), a5 = csub(v[1], v[5]);
    double2 a6 = cadd(v[3], v[7]), a7 = cmul_mi(csub(v[3], v[7]));
    double2 b0 = cadd(a0, a2), b2 = csub(a0, a2), b1 = cadd(a1, a3), b3 = csub(a1, a3);
    double2 c0 = cadd(a4, a6), c2 = csub(a4, a6), c1 = cadd(a5, a7), c3 = csub(a5, a7);
    // w8 = (1 - i)/sqrt2 ; w8^3 = (-1 - i)/sqrt2
    double2 w1c1 = make_double2(s * (c1.x + c1.y), s * (c1.y - c1.x));
    double2 w3c3 = make_double2(s * (c3.y - c3.x), -s * (c3.x + c3.y));
    double2 mic2 = cmul_mi(c2);
    v[0] = cadd(b0, c0);
    v[4] = csub(b0, c0);
    v[2] = cadd(b2, mic2);
    v[6] = csub(b2, mic2);
    v[1] = cadd(b1, w1c1);
    v[5] = csub(b1, w1c1);
    v[3] = cadd(b3, w3c3);
    v[7] = csub(b3, w3c3);
  }
  static __device__ __forceinline__ void emit(const double2 (&v)[8], double2* out, int Ns) {
#pragma unroll
    for (int r = 0; r < 8; ++r) out[r * Ns] = v[r];
  }
};

// Odd prime R: pair inputs j and R-j so every coefficient is real.
//   X_k = A_k - i B_k,  X_{R-k} = A_k + i B_k,
//   A_k = x0 + sum_j (x_j + x_{R-j}) cos(2 pi jk/R),  B_k = sum_j (x_j - x_{R-j}) sin(2 pi jk/R)
// prep leaves v[j] = x_j + x_{R-j}, v[R-j] = x_j - x_{R-j} (j = 1..H).
template <int R> struct Dft {
  static_assert(R % 2 == 1, "odd radix only");
  static __device__ __forceinline__ void prep(double2 (&v)[R]) {
    constexpr int H = (R - 1) / 2;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const double2 p = v[j], q = v[R - j];
      v[j] = cadd(p, q);
      v[R - j] = csub(p, q);
    }
  }
  static __device__ __forceinline__ void emit(const double2 (&v)[R], double2* out, int Ns) {
    constexpr int H = (R - 1) / 2;
    constexpr int off = odd_root_offset(R);
    const double2 x0 = v[0];
    double2 sum = x0;
#pragma unroll
    for (int j = 1; j <= H; ++j) sum = cadd(sum, v[j]);
    out[0] = sum;
#pragma unroll
    for (int k = 1; k <= H; ++k) {
      double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 1; j <= H; ++j) {
        const int q = (j * k) % R;
        const double c = c_root_cos[off + q];
        const double s = c_root_sin[off + q];
        A.x = fma(v[j].x, c, A.x);
        A.y = fma(v[j].y, c, A.y);
        B.x = fma(v[R - j].x, s, B.x);
        B.y = fma(v[R - j].y, s, B.y);
      }
      out[k * Ns] = make_double2(A.x + B.y, A.y - B.x);
      out[(R - k) * Ns] = make_double2(A.x - B.y, A.y + B.x);
    }
  }
};

// ---------------------------------------------------------------- stages
// One in-place Stockham stage over nseq sequences stored with stride ld
// (ld >= Lc; an odd ld keeps the strided smem accesses bank-conflict light).
// Host guarantees nseq * Lc <= blockDim.x * stage_capacity(R, CAP).
template <int R, int CAP>
__device__ __noinline__ void fft_stage_ld(double2* __restrict__ data, int nseq, int Lc, int ld, int Ns,
                                             const double2* __restrict__ tw) {
  constexpr int MAXS = stage_slots(R, CAP);
  const int nb = Lc / R;
  const int total = nseq * nb;
  const int T = blockDim.x;
  const int tw_stride = Lc / (Ns * R);
  double2 v[MAXS][R];
  int obase[MAXS];
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    const int b = threadIdx.x + s * T;
    obase[s] = -1;
    if (b < total) {
      const int seq = b / nb;
      const int j = b - seq * nb;
      const int k = j % Ns;
      const double2* in = data + seq * ld;
#pragma unroll
      for (int r = 0; r < R; ++r) v[s][r] = in[j + r * nb];
      if (Ns > 1) {
        const int step = k * tw_stride;
#pragma unroll
        for (int r = 1; r < R; ++r) v[s][r] = cmul(v[s][r], __ldg(tw + r * step));
      }
      Dft<R>::prep(v[s]);
      obase[s] = seq * ld + (j - k) * R + k;
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < MAXS; ++s) {
    if (obase[s] >= 0) Dft<R>::emit(v[s], data + obase[s], Ns);
  }
  __syncthreads();
}

}  // namespace bhcp
