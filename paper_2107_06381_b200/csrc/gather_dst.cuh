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

// 1D bulk copy global -> shared on the TMA unit, completion tracked by an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
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
// INPL: the W tile is staged straight into the (padded) FFT buffer and the
// first stage runs in place -- no separate staging buffer, no prefetch of the
// next tile, more CTAs per SM. Otherwise a staging buffer lets the next tile
// load while this one is transformed.
template <int N> struct PlanB2;
template <> struct PlanB2<256> { static constexpr int T = 256, R1 = 4, MINB = 3; static constexpr bool INPL = false; template <class Lay> using F = Fft<256, 4, T, Lay, 4, 8, 8>; };
template <> struct PlanB2<512> { static constexpr int T = 256, R1 = 8, MINB = 3; static constexpr bool INPL = false; template <class Lay> using F = Fft<512, 4, T, Lay, 8, 8, 8>; };  // in place: 0.70 vs 0.61 ms (c2)
template <> struct PlanB2<1024> { static constexpr int T = 256, R1 = 16, MINB = 1; static constexpr bool INPL = false; template <class Lay> using F = Fft<1024, 4, T, Lay, 16, 8, 8>; };

struct ArgsB2 {
  const double* in;
  double* out;
  const double2* tw;      // exp(-2 pi i k / N)
  const double* sn;       // sin(pi j / N)
  double scale;           // sqrt(2/N)
  // k_dst_blk2 (blocked W -> rows of y)
  const long long* koff;
  long long NT, P1, idiv, P, nlev;
  // k_dst_cols3 (columns, in place capable): lines i in [0, ni) adjacent,
  // element stride ni, outer blocks o in [0, no) at stride m * ni
  long long ni, no;
};

__device__ __forceinline__ void cp_async8_zfill(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0));
}

// First level pass from the blocked W: a tile is one spatial line (k1, r2)
// x 8 levels, a contiguous 8*m-double run of W; the 8 output lines are rows
// of y.
template <int N>
__global__ void __launch_bounds__(PlanB2<N>::T, PlanB2<N>::MINB) k_dst_blk2(ArgsB2 a) {
  constexpr int S = 4, T = PlanB2<N>::T, m = N - 1;
  constexpr bool INPL = PlanB2<N>::INPL;
  constexpr int RUN = m * kTB;
  constexpr int KU = (N / 2) / 32;   // k values per lane (k = u*32 + lane)
  using Lay = Interleaved<S, 2>;   // pad every 2: conflict-free for q-fastest stages and lane-per-k reads
  extern __shared__ double2 smem[];
  double2* buf = smem;
  double* stage = reinterpret_cast<double*>(smem + Lay::words(N));
  double* sn = INPL ? stage : stage + RUN + 16;
  double* carry = sn + N;           // 8 doubles: lower-half running sums per line
  __shared__ alignas(8) unsigned long long tile_bar;   // TMA bulk-copy completion of the staged tile
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);
  if (!INPL && threadIdx.x == 0) {
    mbar_init(&tile_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // Tiles are walked with 32-bit incremental counters (o, tt) = (line, level tile).
  const int NT = (int)a.NT;
  const int idiv = (int)a.idiv;
  const int ntiles = (int)(a.P * a.NT);
  const int gstep = gridDim.x, step_o = gstep / NT, step_t = gstep - step_o * NT;
  // Staged path: one thread hands the tile (a contiguous 8m-double run) to
  // the TMA unit as a single bulk copy (cp.async.bulk, completion on an
  // mbarrier); the next tile is issued once the first FFT stage has read the
  // current one. In-place path: 16 B cp.async chunks into the padded slots.
  auto src_of = [&](int o, int tt) -> const double* {
    const int k1 = o / idiv, r2 = o - k1 * idiv;
    const long long kb = a.koff ? __ldg(a.koff + k1) : (long long)k1 * a.NT * a.P1 * kTB;
    return a.in + kb + (long long)tt * a.P1 * kTB + (long long)r2 * m * kTB;
  };
  auto issue = [&](const double* src_d) {
    if (INPL) {
      // 16 B chunk i = (element j-1 = i/4, line pair q = i%4) -> slot (q, j)
      const double2* src = reinterpret_cast<const double2*>(src_d);
      for (int i = threadIdx.x; i < RUN / 2; i += T) {
        const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(buf + Lay::addr(i & 3, (i >> 2) + 1)));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src + i));
      }
      cp_async_commit();
      return 0;
    }
    // one thread hands the contiguous 8 m doubles of the tile to the TMA unit
    if (threadIdx.x == 0) bulk_load(stage, src_d, (unsigned)(RUN * sizeof(double)), &tile_bar);
    return 0;
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int tile = blockIdx.x;
  int o = tile / NT, tt = tile - o * NT;
  int soff = 0;
  unsigned phase = 0;
  if (!INPL && tile < ntiles) soff = issue(src_of(o, tt));
  for (; tile < ntiles; tile += gstep) {
    int no = o + step_o, ntt = tt + step_t;
    if (ntt >= NT) { ntt -= NT; ++no; }
    if (INPL) {
      __syncthreads();   // the previous tile's post-processing is done with buf
      issue(src_of(o, tt));
    }
    if (INPL) {
      cp_async_wait_all();
    } else {
      mbar_wait(&tile_bar, phase);
      phase ^= 1u;
    }
    __syncthreads();
    const long long tvalid = a.nlev - (long long)tt * kTB;
    const double* st = stage + soff;
    auto gen = [&](int q, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      double2 p, r;
      if (INPL) {
        p = buf[Lay::addr(q, j)];        // x_j
        r = buf[Lay::addr(q, N - j)];    // x_{N-j}
      } else {
        p = *reinterpret_cast<const double2*>(st + (j - 1) * kTB + 2 * q);
        r = *reinterpret_cast<const double2*>(st + (N - j - 1) * kTB + 2 * q);
      }
      if (2 * q >= tvalid) { p.x = 0.0; r.x = 0.0; }
      if (2 * q + 1 >= tvalid) { p.y = 0.0; r.y = 0.0; }
      const double s = sn[j];
      return make_double2(fma(s, p.x + r.x, 0.5 * (p.x - r.x)), fma(s, p.y + r.y, 0.5 * (p.y - r.y)));
    };
    using Ff = typename PlanB2<N>::template F<Lay>;
    if (INPL) Stage<N, S, T, Lay, PlanB2<N>::R1, 1>::first_inplace(buf, gen);
    else Stage<N, S, T, Lay, PlanB2<N>::R1, 1>::first(buf, gen);
    const int cur_o = o, cur_tt = tt;
    if (!INPL && tile + gstep < ntiles) soff = issue(src_of(no, ntt));
    o = no; tt = ntt;
    auto sink = [&](int q, int idx, double2 X) { buf[Lay::addr(q, idx)] = X; };
    FftTail<Ff>::run(buf, a.tw, sink);
    __syncthreads();
    // Post-processing: warp w takes sequence q = w & 3 (lines 2q, 2q+1) and
    // the half h = w >> 2 of the k range; k = (h*KH + u)*32 + lane. Each U_k,
    // U_{N-k} load serves both lines. The upper half waits for the lower
    // half's running sums (named barrier 1+q).
    {
      static_assert(T == 256, "post-processing assumes 8 warps");
      constexpr int KH = KU / 2;
      const int q = warp & 3, h = warp >> 2;
      const double2 U0 = buf[Lay::addr(q, 0)];
      const double c0a = U0.x, c0b = U0.y;       // Re U^a_0, Re U^b_0
      double ca = 0.0, cb = 0.0;
      double oa[KH], ob[KH], ea[KH], eb[KH];
#pragma unroll
      for (int u = 0; u < KH; ++u) {
        const int k = (h * KH + u) * 32 + lane;
        const double2 A = buf[Lay::addr(q, k)];
        const double2 Bv = buf[Lay::addr(q, (N - k) & (N - 1))];
        double ia = 0.5 * (A.x + Bv.x), ib = 0.5 * (A.y + Bv.y);   // Re U^a_k, Re U^b_k
        ea[u] = -0.5 * (A.y - Bv.y);                                 // S^a_{2k}
        eb[u] = 0.5 * (A.x - Bv.x);                                  // S^b_{2k}
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const double va = __shfl_up_sync(0xffffffffu, ia, off);
          const double vb = __shfl_up_sync(0xffffffffu, ib, off);
          if (lane >= off) { ia += va; ib += vb; }
        }
        oa[u] = ca + ia;
        ob[u] = cb + ib;
        ca += __shfl_sync(0xffffffffu, ia, 31);
        cb += __shfl_sync(0xffffffffu, ib, 31);
      }
      if (h == 0) {
        if (lane == 0) { carry[2 * q] = ca; carry[2 * q + 1] = cb; }
        __threadfence_block();
        asm volatile("bar.arrive %0, 64;\n" ::"r"(1 + q) : "memory");
        ca = 0.0; cb = 0.0;
      } else {
        asm volatile("bar.sync %0, 64;\n" ::"r"(1 + q) : "memory");
        ca = carry[2 * q]; cb = carry[2 * q + 1];
      }
      const double ha = 0.5 * c0a, hb = 0.5 * c0b;
      {
#pragma unroll
        for (int line = 0; line < 2; ++line) {
          const long long t = (long long)cur_tt * kTB + 2 * q + line;
          if (t >= a.nlev) continue;
          double* __restrict__ dst = a.out + (t * a.P + cur_o) * m;
          const double cc = line ? cb : ca, hc = line ? hb : ha;
#pragma unroll
          for (int u = 0; u < KH; ++u) {
            const int k = (h * KH + u) * 32 + lane;
            const double odd = (cc + (line ? ob[u] : oa[u])) - hc;   // S_{2k+1}
            if (k >= 1) dst[2 * k - 1] = a.scale * (line ? eb[u] : ea[u]);
            dst[2 * k] = a.scale * odd;
          }
        }
      }
    }
  }
}

template <int N> struct PlanC3;
// S sequences (2S lines) per tile, T threads, NBUF tile buffers (2: the next
// tile's rows load while this one is transformed), MINB CTAs per SM. Measured
// on c2: one 64 KB buffer of 16 lines (128 B row chunks) at 2 CTAs/SM beats
// double-buffered 8-line tiles at 3 CTAs/SM (0.71 vs 1.05 ms): the row chunk
// width matters more than overlapping load and transform inside a CTA.
template <> struct PlanC3<256> { static constexpr int S = 16, T = 256, NBUF = 1, MINB = 2, R1 = 4; template <class Lay> using F = Fft<256, 16, T, Lay, 4, 8, 8>; };
template <> struct PlanC3<512> { static constexpr int S = 8, T = 256, NBUF = 1, MINB = 2, R1 = 8; template <class Lay> using F = Fft<512, 8, T, Lay, 8, 8, 8>; };
template <> struct PlanC3<1024> { static constexpr int S = 8, T = 512, NBUF = 1, MINB = 1, R1 = 16; template <class Lay> using F = Fft<1024, 8, T, Lay, 16, 8, 8>; };

template <int N> constexpr size_t smemC3_bytes() {
  using P = PlanC3<N>;
  return sizeof(double2) * (P::NBUF * P::S * N) + sizeof(double) * (N + 2 * (P::T / 32) * P::S);
}

template <int N>
__global__ void __launch_bounds__(PlanC3<N>::T, PlanC3<N>::MINB) k_dst_cols3(ArgsB2 a) {
  using P = PlanC3<N>;
  constexpr int S = P::S, T = P::T, m = N - 1, LW = 2 * S;   // LW lines per tile
  constexpr int NW = T / 32;
  constexpr int KK = 32 / S;                 // k values per warp step
  constexpr int KW = (N / 2) / NW;           // k values per warp
  constexpr int STEPS = KW / KK;
  static_assert(STEPS >= 1 && KW % KK == 0, "post-processing shape");
  using Lay = Interleaved<S>;
  extern __shared__ double2 smem[];
  double* sn = reinterpret_cast<double*>(smem + P::NBUF * S * N);
  double* tot = sn + N;                       // [NW warps][S q][2 lines]
  for (int j = threadIdx.x; j < N; j += T) sn[j] = __ldg(a.sn + j);
  const int NT = (int)((a.ni + LW - 1) / LW);
  const int ntiles = (int)(a.no * NT);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = lane % S, kk = lane / S;
  // thread -> fixed line l, rows e = e0, e0 + T/LW, ... (pointer increments only)
  constexpr int RSTEP = T / LW;
  const int l = threadIdx.x % LW, e0 = threadIdx.x / LW;
  const long long gstep_rows = (long long)RSTEP * a.ni;
  auto tile_off = [&](int tile, int& nval) -> long long {
    const int o = tile / NT, cb = tile - o * NT;
    const long long i0 = (long long)cb * LW;
    nval = (int)min((long long)LW, a.ni - i0);
    return (long long)o * m * a.ni + i0;
  };
  // x(e, l) -> double (e+1)*LW + l of buffer b, i.e. complex slot (l/2, e+1)
  auto issue = [&](int tile, int b) {
    int nval;
    const long long off = tile_off(tile, nval);
    double* sdst = reinterpret_cast<double*>(smem + b * S * N) + (e0 + 1) * LW + l;
    if (l < nval) {
      const double* g = a.in + off + (long long)e0 * a.ni + l;
      for (int e = e0; e < m; e += RSTEP, g += gstep_rows, sdst += RSTEP * LW) cp_async8(sdst, g);
    } else {
      for (int e = e0; e < m; e += RSTEP, sdst += RSTEP * LW) *sdst = 0.0;
    }
    cp_async_commit();
  };
  int it = 0;
  if (P::NBUF == 2 && (int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = P::NBUF == 2 ? (it & 1) : 0;
    if (P::NBUF == 2) {
      if (tile + (int)gridDim.x < ntiles) {
        issue(tile + gridDim.x, b ^ 1);    // buffer b^1 was released at the end of the last iteration
        asm volatile("cp.async.wait_group 1;\n" ::);
      } else {
        cp_async_wait_all();
      }
    } else {
      issue(tile, 0);
      cp_async_wait_all();
    }
    __syncthreads();
    double2* buf = smem + b * S * N;
    double* bufd = reinterpret_cast<double*>(buf);
    auto gen = [&](int qg, int j) -> double2 {
      if (j == 0) return make_double2(0.0, 0.0);
      const double2 p = buf[Lay::addr(qg, j)];       // x_j (lines 2q, 2q+1)
      const double2 r = buf[Lay::addr(qg, N - j)];   // x_{N-j}
      const double s = sn[j];
      return make_double2(fma(s, p.x + r.x, 0.5 * (p.x - r.x)), fma(s, p.y + r.y, 0.5 * (p.y - r.y)));
    };
    using Ff = typename P::template F<Lay>;
    Stage<N, S, T, Lay, P::R1, 1>::first_inplace(buf, gen);
    auto sink = [&](int qs, int idx, double2 X) { buf[Lay::addr(qs, idx)] = X; };
    FftTail<Ff>::run(buf, a.tw, sink);
    __syncthreads();
    // post-processing: warp w covers k in [w*KW, (w+1)*KW), lane (q, kk)
    const double2 U0 = buf[Lay::addr(q, 0)];
    double ca = 0.0, cb2 = 0.0;
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
      ob[u] = cb2 + ib;
      ca += __shfl_sync(0xffffffffu, ia, q + 32 - S);
      cb2 += __shfl_sync(0xffffffffu, ib, q + 32 - S);
    }
    if (kk == 0) { tot[(warp * S + q) * 2] = ca; tot[(warp * S + q) * 2 + 1] = cb2; }
    __syncthreads();   // all U reads done; warp totals visible
    double pa = 0.0, pb = 0.0;
    for (int w = 0; w < warp; ++w) { pa += tot[(w * S + q) * 2]; pb += tot[(w * S + q) * 2 + 1]; }
    const double ha = 0.5 * U0.x, hb = 0.5 * U0.y;
#pragma unroll
    for (int u = 0; u < STEPS; ++u) {
      const int k = warp * KW + u * KK + kk;
      if (k >= 1) buf[Lay::addr(q, 2 * k - 1)] = make_double2(a.scale * ea[u], a.scale * eb[u]);
      buf[Lay::addr(q, 2 * k)] = make_double2(a.scale * ((pa + oa[u]) - ha), a.scale * ((pb + ob[u]) - hb));
    }
    __syncthreads();
    int nval;
    const long long off = tile_off(tile, nval);
    if (l < nval) {
      double* g = a.out + off + (long long)e0 * a.ni + l;
      const double* s = bufd + e0 * LW + l;
      for (int e = e0; e < m; e += RSTEP, g += gstep_rows, s += RSTEP * LW) *g = *s;
    }
    __syncthreads();   // buffer b is refilled by the next iteration's prefetch (NBUF = 2) or load
  }
}

template <int N> constexpr size_t smemB2_bytes() {
  using Lay = Interleaved<4, 2>;
  return sizeof(double2) * Lay::words(N) + sizeof(double) * ((PlanB2<N>::INPL ? 0 : (N - 1) * kTB + 16) + N + 8);
}

}  // namespace gdst
}  // namespace bhcp
