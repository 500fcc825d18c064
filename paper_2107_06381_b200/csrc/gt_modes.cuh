// gt_modes.cuh -- pass A for n = 1025 time levels (BASELINE config 3) by the
// prime-factor (Good-Thomas) algorithm, 1025 = 25 x 41, with Rader's
// algorithm for the 41-point transforms. Included by bhcp_b200.cu.
//
// X_t = sum_j v_j w^{jt}, w = exp(-2 pi i / 1025), v_j = 1 / (s_j + mu).
// With the input map j = (41 j1 + 25 j2) mod 1025 and t1 = t mod 25,
// t2 = t mod 41 the kernel is w25^{j1 t1} w41^{j2 t2}: a 25 x 41 2D DFT with
// no twiddles between the two factors.
//   * 41-point DFTs along j2 (one per row j1) by Rader: with j2 = g^p,
//     t2 = g^-q (g a primitive root of 41),
//       Y_0 = sum y,  Y_{g^-q} = y_0 + (a (*) b)_q,  a_p = y_{g^p}, b_m = w41^{g^-m},
//     a length-40 cyclic convolution done as A = FFT40(a),
//     conv = conj(FFT40(conj(A * bhat))) (bhat = FFT40(b) / 40), and Y_0 = y_0 + A_0.
//   * 25-point DFTs along j1 (one per column t2), radix 5 x 5.
// The per-mode work is about 0.6x the FLOPs of the 2048-point Bluestein
// pair it replaces. One warp per mode (warp-synchronous stages over a
// 25 x 41 region, in rounds of whole rows / columns so every stage can run in
// place), persistent CTAs, symmetric seg tiles as in k_modes_blue.
#pragma once

namespace bhcp {
namespace fastk {

constexpr int kGtRows = 25, kGtLen = 41, kGtN = kGtRows * kGtLen;   // row j1: 41 slots

struct GtModesArgs {
  const double2* shifts;
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  int m, dim;
  StatusDev* st;
  const double2* tab;   // w40 (40) | w25 (25) | bhat40 (40)
  const int* itab;      // perm (40): g^p mod 41 | tq (40): g^-q mod 41
  WLayout wl;
  const int4* tiles;
  long long ntiles;
};

// 12 warps at 168 registers; 8 warps (no spills, 231 registers) measured 12.2 ms
// against 10.0 on c3
struct GtPlan { static constexpr int S = 12, T = 384; };

template <bool SYM>
__global__ void __launch_bounds__(GtPlan::T, 1) k_modes_gt(GtModesArgs a) {   // 12 warps: 197 KB buffers
  constexpr int NL = kGtN, S = GtPlan::S, T = GtPlan::T, RS = kGtLen;
  static_assert(T == 32 * S, "one warp per mode");
  extern __shared__ double2 smem[];
  __shared__ double red[2 * (T / 32)];
  __shared__ double2 s_t40[7][5], s_t25[4][5], s_bh[40];   // twiddles by (r-1, b)
  __shared__ short s_tq[40];
  // shifts and singular thresholds in the Good-Thomas input order (row j1, slot):
  // the generator reads consecutive entries
  __shared__ double2 s_shg[NL];
  __shared__ double s_thrg[NL];
  __shared__ short s_jg[NL];
  __shared__ double2 s_x0[S][kGtRows];
  for (int i = threadIdx.x; i < NL; i += T) {
    const int row = i / RS, slot = i - row * RS;
    const int j2 = slot ? __ldg(a.itab + slot - 1) : 0;
    const int j = (41 * row + 25 * j2) % NL;
    const double2 sh = __ldg(a.shifts + j);
    s_shg[i] = sh;
    s_thrg[i] = 1e-28 * (sh.x * sh.x + sh.y * sh.y);   // space.py:237-240
    s_jg[i] = (short)j;
    if (i < 40) {
      s_bh[i] = __ldg(a.tab + 65 + i);
      s_tq[i] = (short)__ldg(a.itab + 40 + i);
    }
    if (i < 35) s_t40[i / 5][i % 5] = __ldg(a.tab + ((i / 5 + 1) * (i % 5)) % 40);
    if (i < 20) s_t25[i / 5][i % 5] = __ldg(a.tab + 40 + ((i / 5 + 1) * (i % 5)) % 25);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* buf = smem + warp * NL;
  double2* x0 = s_x0[warp];
  StatusDev* st = a.st;
  const WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long ntiles = SYM ? a.ntiles : (a.k_count + S - 1) / S;

  // In-place FFT40 over slots 1..40 of every row: radix 5 (Ns = 1) then
  // radix 8 (Ns = 5). Rounds cover whole rows, so loads of a round finish
  // (syncwarp) before its stores and no round reads what another wrote. Both
  // stages touch consecutive slots across lanes (strides 1 and 5): no bank
  // conflicts with the odd row stride 41. store_out(rowp, q, value) stores
  // output q of the radix-8 stage.
  auto fft40 = [&](auto&& store_out) {
    // radix 5: 8 butterflies per row, 4 rows per round
#pragma unroll 1
    for (int r0 = 0; r0 < kGtRows; r0 += 4) {
      const int row = r0 + (lane >> 3), b = lane & 7;
      const bool act = row < kGtRows;
      double2 v[5];
      double2* rowp = buf + row * RS + 1;
      if (act) {
#pragma unroll
        for (int r = 0; r < 5; ++r) v[r] = rowp[b + 8 * r];
        sfft::Cod<5>::run(v);
      }
      __syncwarp();
      if (act) {
#pragma unroll
        for (int r = 0; r < 5; ++r) rowp[5 * b + r] = v[r];
      }
      __syncwarp();
    }
    // radix 8 with twiddles w40^{b r} (k = b % 5 = b): 5 butterflies per row, 6 rows per round
#pragma unroll 1
    for (int r0 = 0; r0 < kGtRows; r0 += 6) {
      const int row = r0 + lane / 5, b = lane % 5;
      const bool act = lane < 30 && row < kGtRows;
      double2 v[8];
      double2* rowp = buf + row * RS + 1;
      if (act) {
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = rowp[b + 5 * r];
#pragma unroll
        for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], s_t40[r - 1][b]);
        sfft::Cod<8>::run(v);
      }
      __syncwarp();
      if (act) {
#pragma unroll
        for (int r = 0; r < 8; ++r) store_out(rowp, b + 5 * r, v[r]);
      }
      __syncwarp();
    }
  };

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
    const double mu = mode_mu(a.mu1, a.m, a.dim, kd);
    const double c = __ldg(a.ghat + kd) * a.cscale;
    const double c2 = hm ? __ldg(a.ghat + km) * a.cscale : 0.0;
    // 1. generator: row j1, slot 0 -> j2 = 0, slot 1 + p -> j2 = g^p;  j = (41 j1 + 25 j2) mod 1025
    for (int i = lane; i < NL; i += 32) {
      const double2 s = s_shg[i];
      const double dr = s.x + mu, di = s.y;
      const double den2 = dr * dr + di * di;
      if (den2 <= s_thrg[i]) flag_singular(st, s_jg[i]);
      const double inv = fast_rcp(den2);
      buf[i] = make_double2(dr * inv, -di * inv);
    }
    __syncwarp();
    // 2. A = FFT40(a) per row (natural order)
    fft40([](double2* rowp, int q, double2 x) { rowp[q] = x; });
    // 3. Y(row, 0) = y0 + A_0 (kept aside); slots <- conj(A_k * bhat_k)
    for (int i = lane; i < kGtRows * 40; i += 32) {
      const int row = i / 40, k = i - row * 40;
      double2* p = buf + row * RS + 1 + k;
      const double2 A = *p;
      if (k == 0) x0[row] = cadd(buf[row * RS], A);
      *p = cconj(cmul(A, s_bh[k]));
    }
    __syncwarp();
    // 4. FFT40 again; conv_q = conj(out_q); Y(row, t2 = g^-q) = y0 + conv_q, stored at slot t2
    //    (rounds hold whole rows, so the permuted stores stay inside the round's rows)
    fft40([&](double2* rowp, int q, double2 x) { rowp[s_tq[q] - 1] = cadd(rowp[-1], cconj(x)); });
    // slot 0 <- Y(row, 0)
    if (lane < kGtRows) buf[lane * RS] = x0[lane];
    __syncwarp();
    // 5. 25-point DFTs down each column t2 (stride RS): radix 5 (Ns = 1) then radix 5 (Ns = 5, w25)
#pragma unroll 1
    for (int st2 = 0; st2 < 2; ++st2) {
      for (int c0 = 0; c0 < kGtLen; c0 += 6) {
        const int col = c0 + lane / 5, b = lane % 5;
        const bool act = lane < 30 && col < kGtLen;
        double2 v[5];
        double2* colp = buf + col;
        if (act) {
#pragma unroll
          for (int r = 0; r < 5; ++r) v[r] = colp[(b + 5 * r) * RS];
          if (st2 == 1) {
#pragma unroll
            for (int r = 1; r < 5; ++r) v[r] = cmul(v[r], s_t25[r - 1][b]);
          }
          sfft::Cod<5>::run(v);
        }
        __syncwarp();
        if (act) {
          // Stockham: stage 1 (Ns = 1) writes 5b + r; stage 2 (Ns = 5, k = b) writes b + 5r
#pragma unroll
          for (int r = 0; r < 5; ++r) colp[(st2 == 0 ? 5 * b + r : b + 5 * r) * RS] = v[r];
        }
        __syncwarp();
      }
    }
    // 6. store: X_t at (t mod 25, t mod 41); W = c Re(Gamma^-1 X), residue norms
    const int nsl = wl.mode_major ? wl.nsl : 1;
    double zr2 = 0.0, zi2 = 0.0;
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
        const double2 X = buf[(t % kGtRows) * RS + (t % kGtLen)];
        const double2 g = __ldg(a.gaminv + t);
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

constexpr size_t gt_smem() { return sizeof(double2) * kGtN * GtPlan::S; }

}  // namespace fastk
}  // namespace bhcp
