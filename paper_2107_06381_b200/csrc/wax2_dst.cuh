// wax2_dst.cuh -- the level passes of the fused solve with one warp (or two)
// per line pair and no CTA barriers. Kernels:
//   k_dst_wax2<512>  strided axis in place on the blocked W (c2)
//   k_dst_blk3<N>    last axis, W -> y, N = 256 (c4) and 512 (c2)
//   k_dst_blk4       last axis, W -> y, N = 1024 (c3; two warps per line pair)
// Column DSTs: warp_dst512 (three radix-8 stages), warp_dst256 (four radix-4
// stages), warp_dst1024 (radix 8, 16, 8 over two warps with named barriers).
//
// k_dst_wax2 does the job of k_dst_wax (wax_dst.cuh): a tile is 16 adjacent
// lines x 511 elements of a 3D view of W, moved by TMA tensor loads/stores.
// The difference is who works on it:
//   * the tile lands 128B-swizzled (16-byte chunk q of row e at chunk
//     q ^ (e & 7)), so one line pair q -- a column of 16-byte elements -- is
//     read and written conflict-free by a warp whose lanes walk the rows;
//   * each of the 8 consumer warps owns one line pair and runs the whole
//     half-length real DST-I on its own column: pre-step + three radix-8
//     Stockham stages in place, synchronised with __syncwarp only, then the
//     even/odd output split with the odd-output prefix sum as warp shuffles;
//   * a producer warp issues the TMA loads, waits for the 8 consumer warps of
//     a buffer (mbarrier), issues its TMA store and refills it.
// Warps therefore progress independently across tiles (the latency hiding of
// k_modes_fast), and every element is read once by the pre-step (lane u
// takes butterflies u and 64 - u, whose inputs are each other's mirrors
// x_j / x_{N-j}) and the prefix-sum split is fused into the last stage
// (the same pairing holds U_k and U_{N-k}): 8 shared-memory passes per tile
// instead of 11.
// Bank conflicts: stage 1 writes index i = 8a + b; it is stored at row
// 8a + ((a + b) & 7) (a within-octet rotation that stage 2 reads back), so
// both the stride-8 writes of stage 1 and the unit-stride reads of stage 2
// hit 8 distinct chunks per 8 lanes.
// Reference: the DSTs of space.py:163-177 per level (pint.py:94-96).
#pragma once
#include "wax_dst.cuh"

namespace bhcp {
namespace wax2 {

using namespace sfft;
using wax::su32;
using wax::mbar_init;
using wax::mbar_expect;
using wax::mbar_wait;
using wax::tma_load3;
using wax::tma_store3;

constexpr int kCW = 8;      // consumer warps = line pairs per tile
constexpr int kLW = 16;     // lines per tile (128 B rows)

// tile buffers: 192 KB of 16-line tiles (N * 128 bytes each)
template <int N> constexpr int nbuf_wax() { return (192 * 1024) / (N * 128); }
template <int N> constexpr size_t smem_bytes() {
  return 1024 /* alignment slack */ + (size_t)nbuf_wax<N>() * N * 128 + sizeof(double) * N + 16 * nbuf_wax<N>();
}

// try_wait with a suspend-time hint: the thread sleeps in hardware until the
// phase completes (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ void mbar_sleep_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// rows 2k - 1 (pe <- ev) and 2k (po <- od) of one k: lanes with sw store them
// in the other order, so each of the two stores covers 8 distinct chunks per
// 8 lanes (explicit selects; predicated stores would split the warp)
__device__ __forceinline__ void store_pair(bool sw, double2* pe, double2 ev, double2* po, double2 od, bool has_ev) {
  asm volatile(
      "{\n .reg .pred q, h;\n .reg .f64 x1, y1, x2, y2;\n .reg .b32 a1, a2;\n"
      " setp.ne.u32 q, %0, 0;\n setp.ne.u32 h, %1, 0;\n"
      " selp.f64 x1, %2, %4, q;\n selp.f64 y1, %3, %5, q;\n"
      " selp.f64 x2, %4, %2, q;\n selp.f64 y2, %5, %3, q;\n"
      " selp.b32 a1, %6, %7, q;\n selp.b32 a2, %7, %6, q;\n"
      " @h st.shared.v2.f64 [a1], {x1, y1};\n"
      " st.shared.v2.f64 [a2], {x2, y2};\n}\n" ::"r"((unsigned)sw),
      "r"((unsigned)has_ev), "d"(od.x), "d"(od.y), "d"(ev.x), "d"(ev.y), "r"(su32(po)), "r"(su32(pe))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
// Hand a tile buffer back to the TMA producer after the warp rewrote it in
// place through generic-proxy shared-memory stores (padding zeroing, Stockham
// stages): the proxy fence orders those stores before the producer's next
// async-proxy (cp.async.bulk.tensor) write into the buffer, and the release
// arrive publishes them to the producer's acquiring wait.
__device__ __forceinline__ void release_buffer(unsigned long long* bar, int lane) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(bar);
}

// TMA-swizzled tiles of 16-byte chunks (one chunk = one line pair):
//   Sw128: 128 B rows (8 pairs), chunk q of row e at q ^ (e & 7)          (SWIZZLE_128B)
//   Sw64:   64 B rows (4 pairs), chunk q of row e at q ^ ((e >> 1) & 3)   (SWIZZLE_64B)
// Either way the 16-byte bank group of (e, q) is a bijection of e & 7 for a
// fixed q, so 8 lanes on rows with distinct e & 7 are conflict-free.
struct Sw128 {
  static constexpr int RS = 8;
  static __device__ __forceinline__ int key(int e) { return e & 7; }
};
struct Sw64 {
  static constexpr int RS = 4;
  static __device__ __forceinline__ int key(int e) { return (e >> 1) & 3; }
};
template <class L>
__device__ __forceinline__ double2* at(double2* tile, int e, int q) { return tile + e * L::RS + (q ^ L::key(e)); }

// Per-lane constants of warp_dst512.
struct LaneK {
  int u, j1, j2;          // lane; butterflies of stages 1 and 3 (u, 64 - u; lane 0: 0, 32)
  double2 w2, w3a, w3b;   // stage-2 twiddle w^((lane%8)*8), stage-3 twiddles w^j1, w^j2
  double mup[5], mdn[5];  // scan masks: 1 where the shuffled neighbour exists
  double scale;
  __device__ __forceinline__ LaneK(int lane, const double2* tw, double sc) {
    u = lane; j1 = lane; j2 = lane == 0 ? 32 : 64 - lane;
    w2 = __ldg(tw + (lane & 7) * 8);
    w3a = __ldg(tw + j1); w3b = __ldg(tw + j2);
    scale = sc;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      mup[s] = lane >= (1 << s) ? 1.0 : 0.0;
      mdn[s] = lane + (1 << s) < 32 ? 1.0 : 0.0;
    }
  }
};

// The half-length real DST-I of line pair q (a column of the swizzled tile T,
// rows e = 0..N-2 = the m elements, row N-1 zero) in place, by one warp:
// pre-step + three radix-8 Stockham stages + even/odd split with the
// odd-output prefix sum. Output e (scaled) is left in row e.
// Default output sink: rows 2k - 1 / 2k of the column (conflict-free order).
template <class L, int KS = 64>
struct ColumnSink {
  double2 *lo_ev, *lo_od, *hi_ev, *hi_od;
  __device__ __forceinline__ ColumnSink(double2* T, int q, int v, int j1, int j2) {
    // output rows 2k - 1, 2k of k = j + KS r: chunk independent of r (rows step 2 KS)
    lo_ev = at<L>(T, v == 0 ? 2 * KS - 1 : 2 * j1 - 1, q) - (v == 0 ? 2 * KS * L::RS : 0);   // unit 0: row 2 KS r - 1 (r >= 1)
    lo_od = at<L>(T, 2 * j1, q);
    hi_ev = at<L>(T, 2 * j2 - 1, q);
    hi_od = at<L>(T, 2 * j2, q);
  }
  // k = j1 + KS r (hi = false) or j2 + KS r (hi = true); ev = S_{2k} -> element 2k - 1, od = S_{2k+1} -> 2k
  __device__ __forceinline__ void put(int r, bool hi, int v, double2 ev, double2 od) {
    const bool sw = (v & 4) != 0;
    if (!hi) store_pair(sw, lo_ev + 2 * KS * L::RS * r, ev, lo_od + 2 * KS * L::RS * r, od, (v | r) != 0);
    else store_pair(sw, hi_ev + 2 * KS * L::RS * r, ev, hi_od + 2 * KS * L::RS * r, od, true);
  }
};

template <class L, class Sink>
__device__ __forceinline__ void warp_dst512(double2* T, int q, const LaneK& K, const double* sn, Sink& sink) {
  constexpr int N = 512;
  constexpr int R8 = 8 * L::RS, R64 = 64 * L::RS, R128 = 128 * L::RS;   // 8 / 64 / 128 rows
  const int u = K.u, j1 = K.j1, j2 = K.j2;
  const double2 w2 = K.w2, w3a = K.w3a, w3b = K.w3b;
  const double scale = K.scale;
  const int lane = u;
    // ---- stage 1: u_i = s_i (x_i + x_{N-i}) + (x_i - x_{N-i})/2 for the 16 indices
    // i = j1 + 64 r, j2 + 64 r; x_i is tile row i - 1 (x_0 = 0)
    double2 A[8], B[8];
    {
      double2 xa[8], xb[8];
      // x_i sits in row i - 1; row (j + 64 r - 1) & 7 does not depend on r. Lane 0's
      // x_0 (= 0) is read from row N - 1, the row past m that the TMA unit zero-fills.
      const double2* pa0 = at<L>(T, u == 0 ? N - 1 : j1 - 1, q);
      const double2* pa1 = at<L>(T, j1 + 63, q) - R64;   // rows j1 - 1 + 64 r, r >= 1
      const double2* pb = at<L>(T, j2 - 1, q);
      xa[0] = *pa0;
#pragma unroll
      for (int r = 1; r < 8; ++r) xa[r] = pa1[R64 * r];
#pragma unroll
      for (int r = 0; r < 8; ++r) xb[r] = pb[R64 * r];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        // partner of index j1 + 64 r: u >= 1 -> j2 + 64 (7 - r); u == 0 -> j1 + 64 (8 - r) (mod N)
        const double2 pa = u == 0 ? xa[(8 - r) & 7] : xb[7 - r];
        const double2 pb = u == 0 ? xb[7 - r] : xa[7 - r];
        const double sa = sn[j1 + 64 * r], sb = sn[j2 + 64 * r];
        A[r] = make_double2(fma(sa, xa[r].x + pa.x, 0.5 * (xa[r].x - pa.x)), fma(sa, xa[r].y + pa.y, 0.5 * (xa[r].y - pa.y)));
        B[r] = make_double2(fma(sb, xb[r].x + pb.x, 0.5 * (xb[r].x - pb.x)), fma(sb, xb[r].y + pb.y, 0.5 * (xb[r].y - pb.y)));
      }
    }
    Cod<8>::run(A);
    Cod<8>::run(B);
    __syncwarp();   // every lane has read its inputs
    // outputs of butterfly j at index 8 j + r, stored at row 8 j + ((j + r) & 7)
    {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        *at<L>(T, 8 * j1 + ((j1 + r) & 7), q) = A[r];
        *at<L>(T, 8 * j2 + ((j2 + r) & 7), q) = B[r];
      }
    }
    __syncwarp();
    // ---- stage 2: butterflies j = lane, lane + 32; read index j + 64 r (rotated rows),
    // twiddle w^((j%8) * 8 * r), write index 64 (j/8) + j%8 + 8 r (natural rows)
    {
      double2 v[2][8];
      // index i = j + 64 r = 8 a + b (a = j/8 + 8 r, b = j%8) is at row
      // 8 a + ((a + b) & 7) = 64 r + 8 (j/8) + ((j/8 + j%8) & 7): r-independent chunk
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        const double2* p = at<L>(T, 8 * (j >> 3) + (((j >> 3) + (j & 7)) & 7), q);
#pragma unroll
        for (int r = 0; r < 8; ++r) v[h][r] = p[R64 * r];
      }
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        apply_twiddles<8>(v[h], w2);
        Cod<8>::run(v[h]);
        double2* p = at<L>(T, 64 * (j >> 3) + (j & 7), q);   // rows base + 8 r: chunk fixed
#pragma unroll
        for (int r = 0; r < 8; ++r) p[R8 * r] = v[h][r];
      }
    }
    __syncwarp();
    // ---- stage 3: butterflies j1, j2: read j + 64 r, twiddle w^(j r), outputs U_{j + 64 r}
    {
      const double2* pa = at<L>(T, j1, q);
      const double2* pb = at<L>(T, j2, q);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        A[r] = pa[R64 * r];
        B[r] = pb[R64 * r];
      }
    }
    apply_twiddles<8>(A, w3a);
    apply_twiddles<8>(B, w3b);
    Cod<8>::run(A);
    Cod<8>::run(B);
    __syncwarp();   // all of U read before the outputs overwrite the column
    // ---- split: for k < N/2, U^a_k = (U_k + conj U_{N-k})/2, U^b_k = (U_k - conj U_{N-k})/(2i);
    // S_{2k} = -Im U_k per line, S_{2k+1} = sum_{i<=k} Re U_i - Re U_0 / 2.
    // Block r (k in [64 r, 64 r + 64)): lane u holds position u ("lo", k = j1 + 64 r)
    // and position 64 - u ("hi", k = j2 + 64 r; lane 0: position 32).
    const double2 U0 = make_double2(__shfl_sync(0xffffffffu, A[0].x, 0), __shfl_sync(0xffffffffu, A[0].y, 0));
    double offa = -0.5 * U0.x, offb = -0.5 * U0.y;   // running block offsets minus Re U_0 / 2
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const double2 P = A[r], Q = u == 0 ? A[(8 - r) & 7] : B[7 - r];     // U_k, U_{N-k}, k = j1 + 64 r
      const double2 Ph = B[r], Qh = u == 0 ? B[7 - r] : A[7 - r];         // k = j2 + 64 r
      double la = 0.5 * (P.x + Q.x), lb = 0.5 * (P.y + Q.y);
      double ha = 0.5 * (Ph.x + Qh.x), hb = 0.5 * (Ph.y + Qh.y);
      const double ela = -0.5 * (P.y - Q.y), elb = 0.5 * (P.x - Q.x);     // S_{2k}, k = j1 + 64 r
      const double eha = -0.5 * (Ph.y - Qh.y), ehb = 0.5 * (Ph.x - Qh.x); // S_{2k}, k = j2 + 64 r
      // inclusive scan of lo over lanes; suffix scan of hi over lanes 1..31
      const double h0a = __shfl_sync(0xffffffffu, ha, 0), h0b = __shfl_sync(0xffffffffu, hb, 0);
      if (u == 0) { ha = 0.0; hb = 0.0; }
#pragma unroll
      for (int s = 0; s < 5; ++s) {
        const int off = 1 << s;
        const double va = __shfl_up_sync(0xffffffffu, la, off), vb = __shfl_up_sync(0xffffffffu, lb, off);
        const double wa = __shfl_down_sync(0xffffffffu, ha, off), wb = __shfl_down_sync(0xffffffffu, hb, off);
        la = fma(K.mup[s], va, la);
        lb = fma(K.mup[s], vb, lb);
        ha = fma(K.mdn[s], wa, ha);
        hb = fma(K.mdn[s], wb, hb);
      }
      const double tla = __shfl_sync(0xffffffffu, la, 31), tlb = __shfl_sync(0xffffffffu, lb, 31);
      const double tha = __shfl_sync(0xffffffffu, ha, 0), thb = __shfl_sync(0xffffffffu, hb, 0);
      const double mida = tla + h0a, midb = tlb + h0b;   // prefix through position 32
      const double oloa = offa + la, olob = offb + lb;                                      // S_{2k+1}, lo
      const double ohia = offa + mida + (u == 0 ? 0.0 : ha), ohib = offb + midb + (u == 0 ? 0.0 : hb);  // hi
      offa += mida + tha;
      offb += midb + thb;
      sink.put(r, false, u, make_double2(scale * ela, scale * elb), make_double2(scale * oloa, scale * olob));
      sink.put(r, true, u, make_double2(scale * eha, scale * ehb), make_double2(scale * ohia, scale * ohib));
    }
}

// Per-lane constants of warp_dst256 (N = 256 = 4^4, four radix-4 stages).
struct LaneK256 {
  int u, j1, j2;          // lane; butterflies of stages 1 and 4 (u, 64 - u; lane 0: 0, 32)
  double2 w2, w3, w4a, w4b;   // stage twiddles w^(16 (j%4)), w^(4 (j%16)), w^j1, w^j2
  double mup[5], mdn[5];
  double scale;
  __device__ __forceinline__ LaneK256(int lane, const double2* tw, double sc) {
    u = lane; j1 = lane; j2 = lane == 0 ? 32 : 64 - lane;
    w2 = __ldg(tw + 16 * (lane & 3));
    w3 = __ldg(tw + 4 * (lane & 15));
    w4a = __ldg(tw + j1); w4b = __ldg(tw + j2);
    scale = sc;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      mup[s] = lane >= (1 << s) ? 1.0 : 0.0;
      mdn[s] = lane + (1 << s) < 32 ? 1.0 : 0.0;
    }
  }
};

// N = 256 version of warp_dst512: pre-step + four radix-4 Stockham stages
// (butterfly j reads j + 64 r, writes (j - j%Ns) 4 + j%Ns + Ns r) + split.
// Stage 1 and 4 pair butterflies u / 64 - u as before. Two in-octet row
// permutations keep stages 1 -> 2 and 2 -> 3 conflict-free:
//   after stage 1: index i at row (i & ~7) | ((i & 7) ^ ((i >> 3) & 3))
//   after stage 2: index i at row (i & ~7) | ((i & 7) ^ (((i >> 4) & 1) << 2))
// Output e (scaled) ends in row e, through the sink.
__device__ __forceinline__ int perm1(int i) { return (i & ~7) | ((i & 7) ^ ((i >> 3) & 3)); }
__device__ __forceinline__ int perm2(int i) { return (i & ~7) | ((i & 7) ^ (((i >> 4) & 1) << 2)); }

template <class L, class Sink>
__device__ __forceinline__ void warp_dst256(double2* T, int q, const LaneK256& K, const double* sn, Sink& sink) {
  constexpr int N = 256;
  constexpr int R64 = 64 * L::RS;
  const int u = K.u, j1 = K.j1, j2 = K.j2, lane = u;
  const double scale = K.scale;
  double2 A[4], B[4];
  {
    // ---- stage 1 inputs: x_i (row i - 1) for i = j1 + 64 r, j2 + 64 r; lane 0's x_0
    // from row N - 1 (zero-filled by the TMA unit)
    double2 xa[4], xb[4];
    const double2* pa0 = at<L>(T, u == 0 ? N - 1 : j1 - 1, q);
    const double2* pa1 = at<L>(T, j1 + 63, q) - R64;
    const double2* pb = at<L>(T, j2 - 1, q);
    xa[0] = *pa0;
#pragma unroll
    for (int r = 1; r < 4; ++r) xa[r] = pa1[R64 * r];
#pragma unroll
    for (int r = 0; r < 4; ++r) xb[r] = pb[R64 * r];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      // partner of j1 + 64 r: u >= 1 -> j2 + 64 (3 - r); u == 0 -> j1 + 64 (4 - r) (mod N)
      const double2 pa = u == 0 ? xa[(4 - r) & 3] : xb[3 - r];
      const double2 pb2 = u == 0 ? xb[3 - r] : xa[3 - r];
      const double sa = sn[j1 + 64 * r], sb = sn[j2 + 64 * r];
      A[r] = make_double2(fma(sa, xa[r].x + pa.x, 0.5 * (xa[r].x - pa.x)), fma(sa, xa[r].y + pa.y, 0.5 * (xa[r].y - pa.y)));
      B[r] = make_double2(fma(sb, xb[r].x + pb2.x, 0.5 * (xb[r].x - pb2.x)), fma(sb, xb[r].y + pb2.y, 0.5 * (xb[r].y - pb2.y)));
    }
  }
  Cod<4>::run(A);
  Cod<4>::run(B);
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    *at<L>(T, perm1(4 * j1 + r), q) = A[r];
    *at<L>(T, perm1(4 * j2 + r), q) = B[r];
  }
  __syncwarp();
  // ---- stage 2 (Ns = 4) and stage 3 (Ns = 16): butterflies j = lane, lane + 32
  {
    double2 v[2][4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      // index j + 64 r: (i >> 3) & 3 and i & 7 do not depend on r
      const double2* p = at<L>(T, perm1(j), q);
#pragma unroll
      for (int r = 0; r < 4; ++r) v[h][r] = p[R64 * r];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      apply_twiddles<4>(v[h], K.w2);
      Cod<4>::run(v[h]);
      const int base = 16 * (j >> 2) + (j & 3);
#pragma unroll
      for (int r = 0; r < 4; ++r) *at<L>(T, perm2(base + 4 * r), q) = v[h][r];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      const double2* p = at<L>(T, perm2(j), q);   // (i >> 4) & 1 and i & 7 do not depend on r
#pragma unroll
      for (int r = 0; r < 4; ++r) v[h][r] = p[R64 * r];
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      apply_twiddles<4>(v[h], K.w3);
      Cod<4>::run(v[h]);
      double2* p = at<L>(T, 64 * (j >> 4) + (j & 15), q);   // rows base + 16 r: key fixed
#pragma unroll
      for (int r = 0; r < 4; ++r) p[16 * L::RS * r] = v[h][r];
    }
  }
  __syncwarp();
  // ---- stage 4 (Ns = 64): butterflies j1, j2, outputs U_{j + 64 r}
  {
    const double2* pa = at<L>(T, j1, q);
    const double2* pb = at<L>(T, j2, q);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      A[r] = pa[R64 * r];
      B[r] = pb[R64 * r];
    }
  }
  apply_twiddles<4>(A, K.w4a);
  apply_twiddles<4>(B, K.w4b);
  Cod<4>::run(A);
  Cod<4>::run(B);
  __syncwarp();
  // ---- split (k < N/2: blocks r = 0, 1; lo k = j1 + 64 r, hi k = j2 + 64 r)
  const double2 U0 = make_double2(__shfl_sync(0xffffffffu, A[0].x, 0), __shfl_sync(0xffffffffu, A[0].y, 0));
  double offa = -0.5 * U0.x, offb = -0.5 * U0.y;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const double2 P = A[r], Q = u == 0 ? A[(4 - r) & 3] : B[3 - r];
    const double2 Ph = B[r], Qh = u == 0 ? B[3 - r] : A[3 - r];
    double la = 0.5 * (P.x + Q.x), lb = 0.5 * (P.y + Q.y);
    double ha = 0.5 * (Ph.x + Qh.x), hb = 0.5 * (Ph.y + Qh.y);
    const double ela = -0.5 * (P.y - Q.y), elb = 0.5 * (P.x - Q.x);
    const double eha = -0.5 * (Ph.y - Qh.y), ehb = 0.5 * (Ph.x - Qh.x);
    const double h0a = __shfl_sync(0xffffffffu, ha, 0), h0b = __shfl_sync(0xffffffffu, hb, 0);
    if (u == 0) { ha = 0.0; hb = 0.0; }
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int off = 1 << s;
      const double va = __shfl_up_sync(0xffffffffu, la, off), vb = __shfl_up_sync(0xffffffffu, lb, off);
      const double wa = __shfl_down_sync(0xffffffffu, ha, off), wb = __shfl_down_sync(0xffffffffu, hb, off);
      la = fma(K.mup[s], va, la);
      lb = fma(K.mup[s], vb, lb);
      ha = fma(K.mdn[s], wa, ha);
      hb = fma(K.mdn[s], wb, hb);
    }
    const double tla = __shfl_sync(0xffffffffu, la, 31), tlb = __shfl_sync(0xffffffffu, lb, 31);
    const double tha = __shfl_sync(0xffffffffu, ha, 0), thb = __shfl_sync(0xffffffffu, hb, 0);
    const double mida = tla + h0a, midb = tlb + h0b;
    const double oloa = offa + la, olob = offb + lb;
    const double ohia = offa + mida + (u == 0 ? 0.0 : ha), ohib = offb + midb + (u == 0 ? 0.0 : hb);
    offa += mida + tha;
    offb += midb + thb;
    sink.put(r, false, u, make_double2(scale * ela, scale * elb), make_double2(scale * oloa, scale * olob));
    sink.put(r, true, u, make_double2(scale * eha, scale * ehb), make_double2(scale * ohia, scale * ohib));
  }
}

// ---------------------------------------------------------------------------
// N = 1024 (c3): the column is 1024 rows, too many for one warp's registers at
// the in-place read-all / write-all points, so TWO warps share a line pair.
// Unit v = 32 h + lane (h = warp half) owns butterflies v and 128 - v (unit 0:
// 0 and 64) in the radix-8 stages 1 and 3 (stride 128) and butterfly v in the
// radix-16 stage 2; the two warps meet at a 64-thread named barrier around
// every in-place write and exchange block totals for the prefix sum.
struct LaneK1024 {
  int u, v, j1, j2;
  double2 w2, w3a, w3b;   // w^(8 (v%8)), w^j1, w^j2
  double mup[5], mdn[5];
  double scale;
  __device__ __forceinline__ LaneK1024(int lane, int h, const double2* tw, double sc) {
    u = lane; v = 32 * h + lane; j1 = v; j2 = v == 0 ? 64 : 128 - v;
    w2 = __ldg(tw + 8 * (v & 7));
    w3a = __ldg(tw + j1); w3b = __ldg(tw + j2);
    scale = sc;
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      mup[s] = lane >= (1 << s) ? 1.0 : 0.0;
      mdn[s] = lane + (1 << s) < 32 ? 1.0 : 0.0;
    }
  }
};

__device__ __forceinline__ void pair_sync(int id) { asm volatile("bar.sync %0, 64;\n" ::"r"(id) : "memory"); }

// The pre-step's sin(pi j / N) factors of a unit's 16 rows: read from the
// shared-memory table per tile (SnTable), or held in registers for the whole
// kernel (SnRegs: k_dst_lvl4, whose consumers have the registers after setmaxnreg).
struct SnTable {
  const double* sn;
  int j1, j2;
  __device__ __forceinline__ double a(int r) const { return sn[j1 + 128 * r]; }
  __device__ __forceinline__ double b(int r) const { return sn[j2 + 128 * r]; }
};
struct SnRegs {
  double va[8], vb[8];
  __device__ __forceinline__ SnRegs(const double* sn, int j1, int j2) {
#pragma unroll
    for (int r = 0; r < 8; ++r) { va[r] = sn[j1 + 128 * r]; vb[r] = sn[j2 + 128 * r]; }
  }
  __device__ __forceinline__ double a(int r) const { return va[r]; }
  __device__ __forceinline__ double b(int r) const { return vb[r]; }
};

// xch: 42 doubles per line pair (block totals and U_0 exchanged between the two warps)
template <class L, class Sink, class Sn>
__device__ __forceinline__ void warp_dst1024(double2* T, int q, int h, const LaneK1024& K, const Sn& sn,
                                             double* xch, int bar, Sink& sink) {
  constexpr int N = 1024;
  constexpr int R128 = 128 * L::RS, R64 = 64 * L::RS;
  const int u = K.u, v = K.v, j1 = K.j1, j2 = K.j2;
  const double scale = K.scale;
  double2 A[8], B[8];
  {
    double2 xa[8], xb[8];
    const double2* pa0 = at<L>(T, v == 0 ? N - 1 : j1 - 1, q);
    const double2* pa1 = at<L>(T, j1 + 127, q) - R128;
    const double2* pb = at<L>(T, j2 - 1, q);
    xa[0] = *pa0;
#pragma unroll
    for (int r = 1; r < 8; ++r) xa[r] = pa1[R128 * r];
#pragma unroll
    for (int r = 0; r < 8; ++r) xb[r] = pb[R128 * r];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const double2 pa = v == 0 ? xa[(8 - r) & 7] : xb[7 - r];
      const double2 pb2 = v == 0 ? xb[7 - r] : xa[7 - r];
      const double sa = sn.a(r), sb = sn.b(r);
      A[r] = make_double2(fma(sa, xa[r].x + pa.x, 0.5 * (xa[r].x - pa.x)), fma(sa, xa[r].y + pa.y, 0.5 * (xa[r].y - pa.y)));
      B[r] = make_double2(fma(sb, xb[r].x + pb2.x, 0.5 * (xb[r].x - pb2.x)), fma(sb, xb[r].y + pb2.y, 0.5 * (xb[r].y - pb2.y)));
    }
  }
  Cod<8>::run(A);
  Cod<8>::run(B);
  pair_sync(bar);   // both warps have read their inputs
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    *at<L>(T, 8 * j1 + ((j1 + r) & 7), q) = A[r];
    *at<L>(T, 8 * j2 + ((j2 + r) & 7), q) = B[r];
  }
  pair_sync(bar);
  // ---- stage 2: radix 16, Ns = 8, butterfly j = v: reads index j + 64 r (rotated rows)
  {
    double2 w[16];
    const int j = v;
    const double2* p = at<L>(T, 8 * (j >> 3) + (((j >> 3) + (j & 7)) & 7), q);
#pragma unroll
    for (int r = 0; r < 16; ++r) w[r] = p[R64 * r];
    apply_twiddles<16>(w, K.w2);
    Cod<16>::run(w);
    pair_sync(bar);
    double2* o = at<L>(T, 128 * (j >> 3) + (j & 7), q);   // rows base + 8 r: key fixed
#pragma unroll
    for (int r = 0; r < 16; ++r) o[8 * L::RS * r] = w[r];
  }
  pair_sync(bar);
  // ---- stage 3: radix 8, Ns = 128: butterflies j1, j2, outputs U_{j + 128 r}
  {
    const double2* pa = at<L>(T, j1, q);
    const double2* pb = at<L>(T, j2, q);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      A[r] = pa[R128 * r];
      B[r] = pb[R128 * r];
    }
  }
  apply_twiddles<8>(A, K.w3a);
  apply_twiddles<8>(B, K.w3b);
  Cod<8>::run(A);
  Cod<8>::run(B);
  // ---- split: blocks r = 0..3 of 128 positions; unit v holds position v (lo,
  // k = j1 + 128 r) and 128 - v (hi, k = j2 + 128 r; unit 0: position 64)
  double la[4], lb[4], ha[4], hb[4], ela[4], elb[4], eha[4], ehb[4], h0a[4], h0b[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double2 P = A[r], Q = v == 0 ? A[(8 - r) & 7] : B[7 - r];
    const double2 Ph = B[r], Qh = v == 0 ? B[7 - r] : A[7 - r];
    la[r] = 0.5 * (P.x + Q.x); lb[r] = 0.5 * (P.y + Q.y);
    ha[r] = 0.5 * (Ph.x + Qh.x); hb[r] = 0.5 * (Ph.y + Qh.y);
    ela[r] = -0.5 * (P.y - Q.y); elb[r] = 0.5 * (P.x - Q.x);
    eha[r] = -0.5 * (Ph.y - Qh.y); ehb[r] = 0.5 * (Ph.x - Qh.x);
    h0a[r] = ha[r]; h0b[r] = hb[r];   // unit 0's value is read from warp 0 lane 0 below
    if (v == 0) { ha[r] = 0.0; hb[r] = 0.0; }
#pragma unroll
    for (int s = 0; s < 5; ++s) {
      const int off = 1 << s;
      const double va = __shfl_up_sync(0xffffffffu, la[r], off), vb = __shfl_up_sync(0xffffffffu, lb[r], off);
      const double wa = __shfl_down_sync(0xffffffffu, ha[r], off), wb = __shfl_down_sync(0xffffffffu, hb[r], off);
      la[r] = fma(K.mup[s], va, la[r]);
      lb[r] = fma(K.mup[s], vb, lb[r]);
      ha[r] = fma(K.mdn[s], wa, ha[r]);
      hb[r] = fma(K.mdn[s], wb, hb[r]);
    }
  }
  // exchange: warp h publishes its lo totals (lane 31) and hi totals (lane 0);
  // warp 0 also publishes unit 0's hi value. xch[h][r][{la, lb, ha, hb}], xch[2][r][{h0a, h0b}]
  if (u == 31) {
#pragma unroll
    for (int r = 0; r < 4; ++r) { xch[(h * 4 + r) * 4 + 0] = la[r]; xch[(h * 4 + r) * 4 + 1] = lb[r]; }
  }
  if (u == 0) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      xch[(h * 4 + r) * 4 + 2] = ha[r]; xch[(h * 4 + r) * 4 + 3] = hb[r];
      if (h == 0) { xch[32 + r * 2] = h0a[r]; xch[32 + r * 2 + 1] = h0b[r]; }
    }
    if (h == 0) { xch[40] = A[0].x; xch[41] = A[0].y; }   // U_0 (unit 0 holds butterfly 0)
  }
  pair_sync(bar);   // totals visible; all stage-3 reads of the column done
  double offa = -0.5 * xch[40], offb = -0.5 * xch[41];   // running block offsets minus Re U_0 / 2
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double lo0a = xch[(0 * 4 + r) * 4 + 0], lo0b = xch[(0 * 4 + r) * 4 + 1];
    const double lo1a = xch[(1 * 4 + r) * 4 + 0], lo1b = xch[(1 * 4 + r) * 4 + 1];
    const double hi0a = xch[(0 * 4 + r) * 4 + 2], hi0b = xch[(0 * 4 + r) * 4 + 3];
    const double hi1a = xch[(1 * 4 + r) * 4 + 2], hi1b = xch[(1 * 4 + r) * 4 + 3];
    const double c0a = xch[32 + r * 2], c0b = xch[32 + r * 2 + 1];
    // prefix through position v (lo): own scan + warp 0's lo total for warp 1
    const double pla = la[r] + (h ? lo0a : 0.0), plb = lb[r] + (h ? lo0b : 0.0);
    // prefix through position 64: all lo + unit 0's hi
    const double mida = lo0a + lo1a + c0a, midb = lo0b + lo1b + c0b;
    // suffix over units v..63 of hi: own suffix + warp 1's hi total for warp 0
    const double sha = ha[r] + (h ? 0.0 : hi1a), shb = hb[r] + (h ? 0.0 : hi1b);
    const double oloa = offa + pla, olob = offb + plb;
    const double ohia = offa + mida + (v == 0 ? 0.0 : sha), ohib = offb + midb + (v == 0 ? 0.0 : shb);
    offa += mida + hi0a + hi1a;
    offb += midb + hi0b + hi1b;
    sink.put(r, false, v, make_double2(scale * ela[r], scale * elb[r]), make_double2(scale * oloa, scale * olob));
    sink.put(r, true, v, make_double2(scale * eha[r], scale * ehb[r]), make_double2(scale * ohia, scale * ohib));
  }
}

// per-N dispatch of the column DST
template <int N> struct ColDst;
template <> struct ColDst<512> {
  using K = LaneK;
  template <class L, class Sink>
  static __device__ __forceinline__ void run(double2* T, int q, const K& k, const double* sn, Sink& s) {
    warp_dst512<L>(T, q, k, sn, s);
  }
};
template <> struct ColDst<256> {
  using K = LaneK256;
  template <class L, class Sink>
  static __device__ __forceinline__ void run(double2* T, int q, const K& k, const double* sn, Sink& s) {
    warp_dst256<L>(T, q, k, sn, s);
  }
};

template <int N>
__global__ void __launch_bounds__((kCW + 1) * 32, 1) k_dst_wax2(const __grid_constant__ CUtensorMap tm,
                                                                 wax::ArgsWX a) {
  static_assert(N == 512 || N == 256, "column DST lengths");
  constexpr int kNBUF = nbuf_wax<N>();
  constexpr int NBOX = N / wax::kBoxRows;
  constexpr unsigned TILE_BYTES = (unsigned)(N * kLW * sizeof(double));
  extern __shared__ unsigned char smem_raw[];
  // TMA 128B swizzle needs 1024-byte aligned tiles
  unsigned char* base = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  double2* tiles = reinterpret_cast<double2*>(base);
  double* sn = reinterpret_cast<double*>(base + (size_t)kNBUF * N * 128);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sn + N);
  unsigned long long* done = full + kNBUF;
  for (int j = threadIdx.x; j < N; j += blockDim.x) sn[j] = __ldg(a.sn + j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
    for (int b = 0; b < kNBUF; ++b) {
      mbar_init(full + b, 1);
      mbar_init(done + b, kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const int ntiles_cta = a.ntiles > (int)blockIdx.x ? (a.ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;

  if (warp == kCW) {
    // ------------------------------------------------------------ producer
    if (lane != 0) return;
    auto load = [&](int it, int b) {
      const int tile = blockIdx.x + it * G;
      const int o = tile / a.lchunks, c = tile - o * a.lchunks;
      double2* dst = tiles + b * N * 8;
      mbar_expect(full + b, TILE_BYTES);
#pragma unroll
      for (int x = 0; x < NBOX; ++x) tma_load3(dst + x * wax::kBoxRows * 8, &tm, c * kLW, x * wax::kBoxRows, o, full + b);
    };
    auto store = [&](int it, int b) {
      const int tile = blockIdx.x + it * G;
      const int o = tile / a.lchunks, c = tile - o * a.lchunks;
      // the producer is not latency critical: back off instead of spinning on
      // the issue slots the consumer warps need
      mbar_sleep_wait(done + b, (unsigned)((it / kNBUF) & 1));
      const double2* src = tiles + b * N * 8;
#pragma unroll
      for (int x = 0; x < NBOX; ++x) tma_store3(&tm, c * kLW, x * wax::kBoxRows, o, src + x * wax::kBoxRows * 8);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    };
    for (int it = 0; it < ntiles_cta; ++it) {
      const int b = it % kNBUF;
      if (it >= kNBUF) {
        store(it - kNBUF, b);
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      }
      load(it, b);
    }
    for (int it = ntiles_cta - kNBUF < 0 ? 0 : ntiles_cta - kNBUF; it < ntiles_cta; ++it) store(it, it % kNBUF);
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    return;
  }

  // -------------------------------------------------------------- consumers
  const int q = warp;   // line pair (lines 2q, 2q+1) of every tile
  const typename ColDst<N>::K K(lane, a.tw, a.scale);
  // tile = blockIdx.x + it * G as (outer o, chunk c), advanced incrementally
  const int dG_o = G / a.lchunks, dG_c = G - dG_o * a.lchunks;
  int to = (int)blockIdx.x / a.lchunks, tc = (int)blockIdx.x - to * a.lchunks;
  for (int it = 0; it < ntiles_cta; ++it) {
    const int b = it % kNBUF;
    const int o = to, c = tc;
    tc += dG_c; to += dG_o;
    if (tc >= a.lchunks) { tc -= a.lchunks; ++to; }
    double2* T = tiles + b * N * 8;
    mbar_sleep_wait(full + b, (unsigned)((it / kNBUF) & 1));
    if (a.vlast < 8) {
      // padding levels of the last level tile share a complex FFT with a
      // valid level: zero them (rare tiles only)
      const int l0 = c * kLW + 2 * q;
      const bool lastA = a.llast >= 0 ? l0 >= a.llast : (o % a.nt == a.nt - 1);
      const bool lastB = a.llast >= 0 ? l0 + 1 >= a.llast : lastA;
      const bool za = lastA && (int)(l0 & 7) >= a.vlast, zb = lastB && (int)((l0 + 1) & 7) >= a.vlast;
      if (za || zb) {
        for (int e = lane; e < N; e += 32) {
          double2* p = at<Sw128>(T, e, q);
          if (za) p->x = 0.0;
          if (zb) p->y = 0.0;
        }
        __syncwarp();
      }
    }
    ColumnSink<Sw128> sink(T, q, K.u, K.j1, K.j2);
    ColDst<N>::template run<Sw128>(T, q, K, sn, sink);
    // hand the buffer to the producer (its TMA store reads it through the async proxy)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(done + b);
  }
}

// ---------------------------------------------------------------------------
// k_dst_blk3: the last spatial axis, W -> y (replaces k_dst_blk2 for N = 512).
// A tile is one W block: 8 levels x m elements of one spatial line, a
// contiguous 32 KB run ([element][8 levels], 64 B rows), loaded by TMA with
// the 64-byte swizzle. Four warps (line pairs = level pairs) transform it
// with warp_dst512 and write their two levels as coalesced rows of y. Eight
// consumer warps = two groups working on alternate tiles; a producer warp
// keeps the other buffers loading.
struct ArgsB3 {
  const double2* tw;
  const double* sn;
  double scale;
  double* y;           // level-major (nlev, n_space)
  int ntiles;          // W blocks = m^(d-2) * NT * m
  int nt;              // NT (level tiles)
  int idiv;            // m^(d-2): spatial lines per (k1, level tile)
  int nlev;
  int m;
};

// Output sink of k_dst_blk3: the two y rows of the line pair, straight from
// registers (elements 2k - 1 and 2k of every k the lane holds).
template <int KS = 64>
struct RowSink {
  double* ya;
  double* yb;
  bool va, vb;
  int j1, j2;
  __device__ __forceinline__ void put(int r, bool hi, int v, double2 ev, double2 od) {
    const int k = (hi ? j2 : j1) + KS * r;
    const bool he = k > 0;
    if (va) {
      if (he) ya[2 * k - 1] = ev.x;
      ya[2 * k] = od.x;
    }
    if (vb) {
      if (he) yb[2 * k - 1] = ev.y;
      yb[2 * k] = od.y;
    }
  }
};

// tile buffers: 192 KB of W blocks (N * 64 bytes each)
template <int N> constexpr int nbuf_b3() { return (192 * 1024) / (N * 64); }
template <int N> constexpr size_t smem_bytes_b3() {
  return 1024 + (size_t)nbuf_b3<N>() * N * 64 + sizeof(double) * N + 16 * nbuf_b3<N>();
}

template <int N>
__global__ void __launch_bounds__((kCW + 1) * 32, 1) k_dst_blk3(const __grid_constant__ CUtensorMap tm, ArgsB3 a) {
  static_assert(N == 512 || N == 256, "column DST lengths");
  constexpr int kB3Buf = nbuf_b3<N>();
  constexpr int NBOX = N / wax::kBoxRows;
  constexpr unsigned TILE_BYTES = (unsigned)(N * 8 * sizeof(double));
  constexpr int TD2 = N * 4;   // double2 per tile
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  double2* tiles = reinterpret_cast<double2*>(base);
  double* sn = reinterpret_cast<double*>(base + (size_t)kB3Buf * N * 64);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sn + N);
  unsigned long long* done = full + kB3Buf;
  for (int j = threadIdx.x; j < N; j += blockDim.x) sn[j] = __ldg(a.sn + j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
    for (int b = 0; b < kB3Buf; ++b) {
      mbar_init(full + b, 1);
      mbar_init(done + b, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const int ntiles_cta = a.ntiles > (int)blockIdx.x ? (a.ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (warp == kCW) {
    if (lane != 0) return;
    for (int it = 0; it < ntiles_cta; ++it) {
      const int b = it % kB3Buf;
      if (it >= kB3Buf) mbar_sleep_wait(done + b, (unsigned)(((it - kB3Buf) / kB3Buf) & 1));
      const int o = blockIdx.x + it * G;
      mbar_expect(full + b, TILE_BYTES);
#pragma unroll
      for (int x = 0; x < NBOX; ++x) tma_load3(tiles + b * TD2 + x * wax::kBoxRows * 4, &tm, 0, x * wax::kBoxRows, o, full + b);
    }
    return;
  }
  const int q = warp & 3, grp = warp >> 2;
  const typename ColDst<N>::K K(lane, a.tw, a.scale);
  const int m = a.m;
  for (int it = grp; it < ntiles_cta; it += 2) {
    const int b = it % kB3Buf;
    double2* T = tiles + b * TD2;
    const int o = blockIdx.x + it * G;
    // o = (k1 * NT + lt) * idiv + r2
    const int o2 = o / a.idiv, r2 = o - o2 * a.idiv;
    const int k1 = o2 / a.nt, lt = o2 - k1 * a.nt;
    const int t0 = lt * 8 + 2 * q;   // levels of lines 2q, 2q + 1
    mbar_sleep_wait(full + b, (unsigned)((it / kB3Buf) & 1));
    if (t0 + 1 >= a.nlev) {
      // padding levels of the last level tile: zero them (their partner in the
      // complex FFT is a valid level)
      const bool za = t0 >= a.nlev, zb = t0 + 1 >= a.nlev;
      for (int e = lane; e < N; e += 32) {
        double2* p = at<Sw64>(T, e, q);
        if (za) p->x = 0.0;
        if (zb) p->y = 0.0;
      }
      __syncwarp();
    }
    // rows of y: level t, spatial line (k1, r2) -> y[((t * m + k1) * idiv + r2) * m + e]
    const long long rowa = ((long long)((long long)t0 * m + k1) * a.idiv + r2) * m;
    const long long rowb = rowa + (long long)m * m * a.idiv;
    RowSink<> sink{a.y + rowa, a.y + rowb, t0 < a.nlev, t0 + 1 < a.nlev, K.j1, K.j2};
    ColDst<N>::template run<Sw64>(T, q, K, sn, sink);
    release_buffer(done + b, lane);
  }
}

// ---------------------------------------------------------------------------
// k_dst_blk4: the last axis W -> y for m + 1 = 1024 (c3). A tile is one 64 KB W
// block (8 levels x 1024 rows, 64 B rows, 64-byte swizzle); two warps per line
// pair (warp w: pair w & 3, half w >> 2) run warp_dst1024 and write the y rows
// from registers; a producer warp streams 3 buffers.
// (A W-side strided variant of the same tiles, TMA load + store, measured 7.5 ms
// on c3 against 6.6 ms for k_dst_cols3 on y -- 64 B rows at an 8 MB stride --
// so c3's strided axis stays on y.)
constexpr int kNB4 = 3;
constexpr size_t smem_bytes_4() { return 1024 + (size_t)kNB4 * 1024 * 64 + sizeof(double) * (1024 + 4 * 42) + 16 * kNB4; }

__global__ void __launch_bounds__((kCW + 1) * 32, 1) k_dst_blk4(const __grid_constant__ CUtensorMap tm, ArgsB3 b3) {
  constexpr int N = 1024, NBOX = N / wax::kBoxRows, TD2 = N * 4;
  constexpr unsigned TILE_BYTES = (unsigned)(N * 8 * sizeof(double));
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  double2* tiles = reinterpret_cast<double2*>(base);
  double* sn = reinterpret_cast<double*>(base + (size_t)kNB4 * TD2 * 16);
  double* xch = sn + N;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xch + 4 * 42);
  unsigned long long* done = full + kNB4;
  for (int j = threadIdx.x; j < N; j += blockDim.x) sn[j] = __ldg(b3.sn + j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
    for (int b = 0; b < kNB4; ++b) {
      mbar_init(full + b, 1);
      mbar_init(done + b, kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  const int ntiles_cta = b3.ntiles > (int)blockIdx.x ? (b3.ntiles - 1 - (int)blockIdx.x) / G + 1 : 0;
  if (warp == kCW) {
    if (lane != 0) return;
    for (int it = 0; it < ntiles_cta; ++it) {
      const int b = it % kNB4;
      if (it >= kNB4) mbar_sleep_wait(done + b, (unsigned)(((it - kNB4) / kNB4) & 1));
      const int o = blockIdx.x + it * G;
      mbar_expect(full + b, TILE_BYTES);
#pragma unroll
      for (int x = 0; x < NBOX; ++x) tma_load3(tiles + b * TD2 + x * wax::kBoxRows * 4, &tm, 0, x * wax::kBoxRows, o, full + b);
    }
    return;
  }
  const int q = warp & 3, h = warp >> 2, bar = 1 + q;
  const LaneK1024 K(lane, h, b3.tw, b3.scale);
  const long long m = b3.m;
  for (int it = 0; it < ntiles_cta; ++it) {
    const int b = it % kNB4;
    double2* T = tiles + b * TD2;
    const int o = blockIdx.x + it * G;
    // o = (k1 * NT + lt) * idiv + r2
    const int o2 = o / b3.idiv, r2 = o - o2 * b3.idiv;
    const int k1 = o2 / b3.nt, lt = o2 - k1 * b3.nt;
    const int t0 = lt * 8 + 2 * q;   // levels of lines 2q, 2q + 1
    mbar_sleep_wait(full + b, (unsigned)((it / kNB4) & 1));
    const bool za = t0 >= b3.nlev, zb = t0 + 1 >= b3.nlev;
    if (za || zb) {
      // padding levels of the last level tile: zero them (they share the complex FFT)
      for (int e = h * 32 + lane; e < N; e += 64) {
        double2* p = at<Sw64>(T, e, q);
        if (za) p->x = 0.0;
        if (zb) p->y = 0.0;
      }
      pair_sync(bar);
    }
    const long long rowa = ((long long)((long long)t0 * m + k1) * b3.idiv + r2) * m;
    const long long rowb = rowa + m * m * b3.idiv;
    RowSink<128> sink{b3.y + rowa, b3.y + rowb, !za, !zb, K.j1, K.j2};
    warp_dst1024<Sw64>(T, q, h, K, SnTable{sn, K.j1, K.j2}, xch + q * 42, bar, sink);
    release_buffer(done + b, lane);
  }
}

}  // namespace wax2
}  // namespace bhcp
