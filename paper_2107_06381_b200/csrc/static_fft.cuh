// static_fft.cuh -- compile-time specialised fp64 FFTs for the hot lengths.
//
// The generic engine (fft_engine.cuh) handles any length with runtime radix
// plans; its stages are out-of-line calls, which costs registers and calls.
// For the lengths the BASELINE configs hit, this header instantiates fully
// inlined Stockham transforms whose radices, strides and butterfly counts are
// compile-time constants:
//   * every stage keeps exactly ceil(S*L/R / T) radix-R butterflies per thread
//     in registers (in-place stage: load -> barrier -> store),
//   * the first stage takes its inputs from a generator functor (global
//     memory or computed values, no shared-memory round trip) and the last
//     stage hands its outputs to a sink functor (global memory),
//   * shared-memory layouts are chosen per kernel to be bank-conflict free:
//     SeqMajorPad (thread-fastest index = FFT index j, one pad slot every R1
//     elements) and Interleaved (thread-fastest index = sequence q).
#pragma once
#include "fft_engine.cuh"

namespace bhcp {
namespace sfft {

// ------------------------------------------------------------------ codelets
template <int R> struct Cod {
  static __device__ __forceinline__ void run(double2 (&v)[R]) {
    Dft<R>::prep(v);
    if constexpr (R % 2 == 1) {
      // odd primes: finish the symmetric codelet in registers
      constexpr int H = (R - 1) / 2;
      constexpr int off = odd_root_offset(R);
      double2 a[H], b[H];
#pragma unroll
      for (int j = 1; j <= H; ++j) { a[j - 1] = v[j]; b[j - 1] = v[R - j]; }
      const double2 x0 = v[0];
      double2 sum = x0;
#pragma unroll
      for (int j = 0; j < H; ++j) sum = cadd(sum, a[j]);
      v[0] = sum;
#pragma unroll
      for (int k = 1; k <= H; ++k) {
        double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
        for (int j = 1; j <= H; ++j) {
          const int q = (j * k) % R;
          const double c = c_root_cos[off + q];
          const double s = c_root_sin[off + q];
          A.x = fma(a[j - 1].x, c, A.x);
          A.y = fma(a[j - 1].y, c, A.y);
          B.x = fma(b[j - 1].x, s, B.x);
          B.y = fma(b[j - 1].y, s, B.y);
        }
        v[k] = make_double2(A.x + B.y, A.y - B.x);
        v[R - k] = make_double2(A.x - B.y, A.y + B.x);
      }
    }
  }
};

// radix 16 = 4 x 4 with internal twiddles w16^(n1*k2)
template <> struct Cod<16> {
  static __device__ __forceinline__ void run(double2 (&v)[16]) {
    const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
    const double r2 = 0.70710678118654752440;
    // columns: for n1 in 0..3, DFT4 over n2 of x[n1 + 4 n2]
    double2 t[4][4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      double2 u[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
      Dft<4>::prep(u);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) t[n1][k2] = u[k2];
    }
    // twiddles w16^(n1*k2): w^1=(c1,-s1) w^2=(r2,-r2) w^3=(s1,-c1) w^4=(0,-1) w^6=(-r2,-r2) w^9=(-c1,s1)
    t[1][1] = cmul(t[1][1], make_double2(c1, -s1));
    t[1][2] = cmul(t[1][2], make_double2(r2, -r2));
    t[1][3] = cmul(t[1][3], make_double2(s1, -c1));
    t[2][1] = cmul(t[2][1], make_double2(r2, -r2));
    t[2][2] = cmul_mi(t[2][2]);
    t[2][3] = cmul(t[2][3], make_double2(-r2, -r2));
    t[3][1] = cmul(t[3][1], make_double2(s1, -c1));
    t[3][2] = cmul(t[3][2], make_double2(-r2, -r2));
    t[3][3] = cmul(t[3][3], make_double2(-c1, s1));
    // rows: for k2, DFT4 over n1 -> X[k2 + 4 k1]
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      double2 u[4] = {t[0][k2], t[1][k2], t[2][k2], t[3][k2]};
      Dft<4>::prep(u);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = u[k1];
    }
  }
};
template <> struct Cod<2> { static __device__ __forceinline__ void run(double2 (&v)[2]) { Dft<2>::prep(v); } };
template <> struct Cod<4> { static __device__ __forceinline__ void run(double2 (&v)[4]) { Dft<4>::prep(v); } };
template <> struct Cod<8> { static __device__ __forceinline__ void run(double2 (&v)[8]) { Dft<8>::prep(v); } };

// radix 9 = 3 x 3 with internal twiddles w9^(n1*k2)
template <> struct Cod<9> {
  static __device__ __forceinline__ void run(double2 (&v)[9]) {
    // w9^1, w9^2, w9^4 (cos, -sin)
    const double c1 = 0.76604444311897803520, s1 = 0.64278760968653932632;
    const double c2 = 0.17364817766693034885, s2 = 0.98480775301220805936;
    const double c4 = -0.93969262078590838405, s4 = 0.34202014332566873304;
    double2 t[3][3];
#pragma unroll
    for (int n1 = 0; n1 < 3; ++n1) {
      double2 u[3] = {v[n1], v[n1 + 3], v[n1 + 6]};
      Cod<3>::run(u);
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2) t[n1][k2] = u[k2];
    }
    t[1][1] = cmul(t[1][1], make_double2(c1, -s1));
    t[1][2] = cmul(t[1][2], make_double2(c2, -s2));
    t[2][1] = cmul(t[2][1], make_double2(c2, -s2));
    t[2][2] = cmul(t[2][2], make_double2(c4, -s4));
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) {
      double2 u[3] = {t[0][k2], t[1][k2], t[2][k2]};
      Cod<3>::run(u);
#pragma unroll
      for (int k1 = 0; k1 < 3; ++k1) v[k2 + 3 * k1] = u[k1];
    }
  }
};

// ------------------------------------------------------------------ layouts
// Interleaved: element idx of sequence q at idx*S + q + idx/P (thread-fastest
// = q); the pad slot every P indices breaks the stride-R*S pattern of the
// first-stage stores (P = first radix).
template <int S, int P = 1 << 30> struct Interleaved {
  static constexpr int words(int L) { return L * S + L / P + 1; }
  static __device__ __forceinline__ int addr(int q, int idx) { return idx * S + q + idx / P; }
  // addr(q, j + r * STRIDE) with the per-r part folded to a compile-time offset
  template <int STRIDE>
  static __device__ __forceinline__ int addr_r(int q, int j, int r) {
    if constexpr (STRIDE % P == 0) return addr(q, j) + r * (STRIDE * S + STRIDE / P);
    else return addr(q, j + r * STRIDE);
  }
  // addr(q, base + r), r < R, base a multiple of R (first-stage stores)
  template <int R>
  static __device__ __forceinline__ int addr_first(int q, int base, int r) {
    if constexpr (P % R == 0) return addr(q, base) + r * S;
    else return addr(q, base + r);
  }
  // butterfly b -> (q, j): q fastest
  static __device__ __forceinline__ void split(int b, int nb, int& q, int& j) { q = b % S; j = b / S; }
};
// SeqMajorPad: element idx of sequence q at q*LD + idx + idx/P (thread-fastest = j).
template <int L, int P> struct SeqMajorPad {
  static constexpr int LD = L + L / P + 1;
  static constexpr int words(int S) { return LD * S; }
  static __device__ __forceinline__ int addr(int q, int idx) { return q * LD + idx + idx / P; }
  template <int STRIDE>
  static __device__ __forceinline__ int addr_r(int q, int j, int r) {
    if constexpr (STRIDE % P == 0) return addr(q, j) + r * (STRIDE + STRIDE / P);
    else return addr(q, j + r * STRIDE);
  }
  template <int R>
  static __device__ __forceinline__ int addr_first(int q, int base, int r) {
    if constexpr (P % R == 0) return addr(q, base) + r;
    else return addr(q, base + r);
  }
  static __device__ __forceinline__ void split(int b, int nb, int& q, int& j) { q = b / nb; j = b - q * nb; }
};

// ------------------------------------------------------------------ stages
// Multiply v[r] by w^r, r = 1..R-1, from the single table value w = w_L^(k*TWS)
// (running product, depth R-2 <= 7 for the radices used after stage 1, so
// the twiddle error stays within a few ulp) -- one table load per butterfly
// instead of R-1.
template <int R>
__device__ __forceinline__ void apply_twiddles(double2 (&v)[R], double2 w) {
  double2 p = w;
  v[1] = cmul(v[1], p);
#pragma unroll
  for (int r = 2; r < R; ++r) {
    p = cmul(p, w);
    v[r] = cmul(v[r], p);
  }
}

template <int L, int S, int T, class Lay, int R, int Ns>
struct Stage {
  static constexpr int NB = S * L / R;            // butterflies in the CTA
  static constexpr int PER = (NB + T - 1) / T;    // per thread
  static constexpr bool FULL = (NB % T) == 0;
  static constexpr int TWS = L / (Ns * R);        // twiddle stride in the length-L table

  // middle stage: smem -> smem
  static __device__ __forceinline__ void mid(double2* buf, const double2* __restrict__ tw) {
    double2 v[PER][R];
    int qq[PER], jj[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
        int q, j;
        Lay::split(b, L / R, q, j);
        qq[i] = q; jj[i] = j;
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = buf[Lay::template addr_r<L / R>(q, j, r)];
        if (Ns > 1) apply_twiddles<R>(v[i], tw[(j % Ns) * TWS]);
        Cod<R>::run(v[i]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
        const int q = qq[i], j = jj[i];
        const int k = j % Ns;
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[Lay::template addr_r<Ns>(q, base, r)] = v[i][r];
      }
    }
    __syncthreads();
  }

  // first stage (Ns == 1): inputs from gen(q, idx) instead of smem.
  // The caller must have synchronised if buf still holds a previous transform.
  template <class Gen>
  static __device__ __forceinline__ void first(double2* buf, Gen& gen) {
    static_assert(Ns == 1, "first stage");
    double2 v[PER][R];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
        int q, j;
        Lay::split(b, L / R, q, j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = gen(q, j + r * (L / R));
        Cod<R>::run(v[i]);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[Lay::template addr_first<R>(q, j * R, r)] = v[i][r];
      }
    }
    __syncthreads();
  }

  // first stage in place: gen reads buf itself, so all loads finish (CTA
  // barrier) before any store.
  template <class Gen>
  static __device__ __forceinline__ void first_inplace(double2* buf, Gen& gen) {
    static_assert(Ns == 1, "first stage");
    double2 v[PER][R];
    int qq[PER], jj[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
        int q, j;
        Lay::split(b, L / R, q, j);
        qq[i] = q; jj[i] = j;
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = gen(q, j + r * (L / R));
        Cod<R>::run(v[i]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
#pragma unroll
        for (int r = 0; r < R; ++r) buf[Lay::template addr_first<R>(qq[i], jj[i] * R, r)] = v[i][r];
      }
    }
    __syncthreads();
  }

  // last stage (Ns * R == L): outputs to sink(q, idx, value)
  template <class Sink>
  static __device__ __forceinline__ void last(double2* buf, const double2* __restrict__ tw, Sink& sink) {
    static_assert(Ns * R == L, "last stage");
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = threadIdx.x + i * T;
      if (FULL || b < NB) {
        int q, j;
        Lay::split(b, L / R, q, j);
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = buf[Lay::template addr_r<L / R>(q, j, r)];
        if (Ns > 1) apply_twiddles<R>(v, tw[j * TWS]);
        Cod<R>::run(v);
        // k = j (j < Ns), outputs at j + r*Ns
#pragma unroll
        for (int r = 0; r < R; ++r) sink(q, j + r * Ns, v[r]);
      }
    }
  }
};

// Run a full transform: first stage from gen, middle stages in smem, last to sink.
template <int L, int S, int T, class Lay, int Ns, int R, int... Rest>
struct Runner {
  template <class Sink>
  static __device__ __forceinline__ void tail(double2* buf, const double2* tw, Sink& sink) {
    if constexpr (sizeof...(Rest) == 0) {
      Stage<L, S, T, Lay, R, Ns>::last(buf, tw, sink);
    } else {
      Stage<L, S, T, Lay, R, Ns>::mid(buf, tw);
      Runner<L, S, T, Lay, Ns * R, Rest...>::tail(buf, tw, sink);
    }
  }
};

template <int L, int S, int T, class Lay, int R1, int... Rest>
struct Fft {
  template <class Gen, class Sink>
  static __device__ __forceinline__ void run(double2* buf, const double2* tw, Gen& gen, Sink& sink) {
    static_assert(sizeof...(Rest) >= 1, "need at least two stages");
    Stage<L, S, T, Lay, R1, 1>::first(buf, gen);
    Runner<L, S, T, Lay, R1, Rest...>::tail(buf, tw, sink);
  }
  // stages 2..k only (after the caller ran Stage<..., R1, 1>::first itself)
  template <class Sink>
  static __device__ __forceinline__ void tail(double2* buf, const double2* tw, Sink& sink) {
    Runner<L, S, T, Lay, R1, Rest...>::tail(buf, tw, sink);
  }
};

template <class F> struct FftTail {
  template <class Sink>
  static __device__ __forceinline__ void run(double2* buf, const double2* tw, Sink& sink) { F::tail(buf, tw, sink); }
};

}  // namespace sfft
}  // namespace bhcp

namespace bhcp {
namespace sfft {

// ------------------------------------------------------------------ warp FFT
// One warp owns one length-L sequence in its own shared-memory region and runs
// the Stockham stages with __syncwarp() only: warps of a CTA progress
// independently (no CTA-wide barrier inside the transform), which is what
// hides the latency of the FP64 / shared-memory chains at 16 warps per SM.
// Stage s in place: every lane computes its ceil(L/R / 32) butterflies into
// registers, the warp synchronises, then stores.
template <int L, int R, int Ns, int PAD = 0>
struct WStage {
  static constexpr int NB = L / R;
  static constexpr int PER = (NB + 31) / 32;
  static constexpr int TWS = L / (Ns * R);
  // element i of the per-warp region (PAD > 0: one spare slot every PAD elements)
  static __device__ __forceinline__ int pi(int i) { return PAD ? i + i / PAD : i; }

  template <class Gen>
  static __device__ __forceinline__ void first(double2* buf, int lane, Gen& gen) {
    static_assert(Ns == 1, "first stage");
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane + 32 * i;
      if (b < NB) {
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = gen(b + r * NB);
        Cod<R>::run(v);
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pi(b * R + r)] = v[r];
      }
    }
    __syncwarp();
  }

  static __device__ __forceinline__ void mid(double2* buf, int lane, const double2* __restrict__ tw) {
    double2 v[PER][R];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane + 32 * i;
      if (b < NB) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = buf[pi(b + r * NB)];
        if (Ns > 1) apply_twiddles<R>(v[i], __ldg(tw + (b % Ns) * TWS));
        Cod<R>::run(v[i]);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = lane + 32 * i;
      if (b < NB) {
        const int k = b % Ns;
        const int base = (b - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pi(base + r * Ns)] = v[i][r];
      }
    }
    __syncwarp();
  }
};

template <int L, int PAD, int Ns, int R, int... Rest>
struct WRunner {
  static __device__ __forceinline__ void tail(double2* buf, int lane, const double2* tw) {
    WStage<L, R, Ns, PAD>::mid(buf, lane, tw);
    if constexpr (sizeof...(Rest) > 0) WRunner<L, PAD, Ns * R, Rest...>::tail(buf, lane, tw);
  }
};

// Full transform, natural-order result left in buf (per-warp region).
template <int L, int R1, int... Rest>
struct WarpFft {
  template <class Gen>
  static __device__ __forceinline__ void run(double2* buf, int lane, const double2* tw, Gen& gen) {
    WStage<L, R1, 1>::first(buf, lane, gen);
    if constexpr (sizeof...(Rest) > 0) WRunner<L, 0, R1, Rest...>::tail(buf, lane, tw);
  }
};

// Same with a padded per-warp region (element i at i + i/PAD) and a variant
// whose first stage also reads the region (in place).
template <int L, int PAD, int R1, int... Rest>
struct WarpFftPad {
  static __device__ __forceinline__ int pi(int i) { return WStage<L, R1, 1, PAD>::pi(i); }
  static constexpr int words = L + L / PAD + 1;
  template <class Gen>
  static __device__ __forceinline__ void run(double2* buf, int lane, const double2* tw, Gen& gen) {
    WStage<L, R1, 1, PAD>::first(buf, lane, gen);
    if constexpr (sizeof...(Rest) > 0) WRunner<L, PAD, R1, Rest...>::tail(buf, lane, tw);
  }
  static __device__ __forceinline__ void run_inplace(double2* buf, int lane, const double2* tw) {
    WRunner<L, PAD, 1, R1, Rest...>::tail(buf, lane, tw);
  }
};

}  // namespace sfft
}  // namespace bhcp
