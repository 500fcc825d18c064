// pf_modes.cuh -- pass A for n = 4097 time levels (BASELINE config 5) by the
// prime-factor algorithm, 4097 = 17 x 241, with Rader's algorithm for the
// 241-point transforms. Included by bhcp_b200.cu after gt_modes.cuh.
//
// Same construction as k_modes_gt (n = 1025 = 25 x 41), one CTA per mode:
//   j = (241 j1 + 17 j2) mod 4097, t1 = t mod 17, t2 = t mod 241,
//   X_t = sum_{j1} w17^{j1 t1} sum_{j2} w241^{j2 t2} v(j1, j2);
//   241-point DFTs along rows by Rader (g a primitive root of 241):
//     Y_0 = y_0 + A_0, Y_{g^-q} = y_0 + conj(FFT240(conj(A * bhat)))_q, A = FFT240(a),
//     a_p = y_{g^p}, FFT240 = radix 4 x 4 x 5 x 3;
//   17-point DFTs down the 241 columns (direct odd codelet).
// About 0.55x the FLOPs of the 8192-point Bluestein pair; 65.5 KB of shared
// memory per mode, so two CTAs share an SM. The 17 rows go one per warp
// (warp-synchronous in-place stages: a lane loads its butterflies, the warp
// synchronises, then it stores); CTA barriers only separate the row, column
// and store phases of a mode.
#pragma once

namespace bhcp {
namespace fastk {

constexpr int kPfRows = 17, kPfLen = 241, kPfN = kPfRows * kPfLen, kPfNp = 240;

struct PfModesArgs {
  const double2* shg;   // shifts in prime-factor input order (row j1, slot)
  const double2* gaminv;
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  int m, dim;
  StatusDev* st;
  const double2* tab;   // w240 (240) | bhat240 (240)
  const int* tq;        // g^-q mod 241 (240)
  WLayout wl;
  const int4* tiles;    // SYM: seg tiles with S = 1
  long long ntiles;
};

// A batch of independent solves of one g on one space grid with n = 4097
// (BASELINE config 5: 64 alpha x 2 kinds): pair p has its own
// shift and 1/gamma tables (its omega), coefficient scale
// 1/(divisor_p n), status block and W. Tiles run over pairs x modes, so one
// launch covers the batch with no per-solve launch tail.
constexpr int kPfMaxPairs = 32;
struct PfPairs {
  int n;                              // pairs in this launch (0: unbatched, use PfModesArgs)
  long long w_stride;                 // doubles between consecutive pairs' W
  const double2* shg[kPfMaxPairs];
  const double2* gaminv[kPfMaxPairs];
  double cscale[kPfMaxPairs];
  StatusDev* st[kPfMaxPairs];
};

// 9 warps (at most two of the 17 rows each) and two CTAs per SM: 96
// registers, some spills, but measured faster (c5: 464 us) than 8 warps with
// a rotating third row (507 us) or 17 warps, one CTA per SM (490 us)
struct PfPlan { static constexpr int T = 288, MINB = 2; };

// One in-place Stockham stage of radix R over slots 1..240 of one row, run by
// one warp: butterfly b < 240/R (lanes b = lane + 32 i) reads slots
// 1 + b + (240/R) r and twiddles them by w240^{TWS k r} (k = b % Ns); the warp
// synchronises, then store(q, x) takes output q = (b - k) R + k + Ns r.
template <int R, int Ns, class Store>
__device__ __forceinline__ void pf_warp_stage(const double2* rowp, int lane, const double2* __restrict__ w240,
                                              Store&& store) {
  constexpr int NB = kPfNp / R, PER = (NB + 31) / 32, TWS = kPfNp / (Ns * R);
  double2 v[PER][R];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int b = lane + 32 * i;
    if (b < NB) {
#pragma unroll
      for (int r = 0; r < R; ++r) v[i][r] = rowp[b + NB * r];
      if (Ns > 1) {
        const int k = b % Ns;
#pragma unroll
        for (int r = 1; r < R; ++r) v[i][r] = cmul(v[i][r], w240[(TWS * k * r) % kPfNp]);
      }
      sfft::Cod<R>::run(v[i]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int b = lane + 32 * i;
    if (b < NB) {
      const int k = b % Ns, base = (b - k) * R + k;
      if constexpr (R == 4 && (Ns == 1 || Ns == 4)) {
        // radix-4 stores land at base + Ns r: with base = 4b (Ns = 1) or
        // 16 (b / 4) + b % 4 (Ns = 4) the 8 lanes of a 16-byte wavefront share 2
        // (resp. 4) bank groups for a common r. Lane b issues its r in the rotated
        // order r = (rr + f) & 3, f = b / 2 (resp. b / 4): 8 distinct bank groups.
        const int f = (Ns == 1 ? (b >> 1) : (b >> 2)) & 3;
        double2 w0 = v[i][0], w1 = v[i][1], w2 = v[i][2], w3 = v[i][3];
        if (f & 1) { const double2 t0 = w0; w0 = w1; w1 = w2; w2 = w3; w3 = t0; }
        if (f & 2) { double2 t0 = w0; w0 = w2; w2 = t0; t0 = w1; w1 = w3; w3 = t0; }
        store(base + Ns * (f & 3), w0);
        store(base + Ns * ((f + 1) & 3), w1);
        store(base + Ns * ((f + 2) & 3), w2);
        store(base + Ns * ((f + 3) & 3), w3);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) store(base + Ns * r, v[i][r]);
      }
    }
  }
  __syncwarp();
}

template <bool SYM, bool BATCH = false>
__global__ void __launch_bounds__(PfPlan::T, PfPlan::MINB) k_modes_pf(PfModesArgs a,
                                                                     const __grid_constant__ PfPairs pp) {
  constexpr int NL = kPfN, T = PfPlan::T;
  extern __shared__ double2 smem[];
  __shared__ double2 s_w[kPfNp], s_bh[kPfNp];
  __shared__ short s_tq[kPfNp];
  __shared__ double2 s_x0[kPfRows];
  __shared__ double red[2 * (T / 32)];
  for (int i = threadIdx.x; i < kPfNp; i += T) {
    s_w[i] = __ldg(a.tab + i);
    s_bh[i] = __ldg(a.tab + kPfNp + i);
    s_tq[i] = (short)__ldg(a.tq + i);
  }
  double2* buf = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  StatusDev* st = a.st;
  const WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long ntiles = SYM ? a.ntiles : (BATCH ? a.k_count * pp.n : a.k_count);
  // batch: the pair of the current tile; residue sums flushed to its status block
  // whenever the CTA moves on to another pair (tiles are uniform across the CTA)
  int pair = -1;
  const double2* shg = a.shg;
  const double2* gaminv = a.gaminv;
  double cscale = a.cscale;
  long long wofs = 0;
  __syncthreads();
  for (long long tile0 = blockIdx.x; tile0 < ntiles; tile0 += gridDim.x) {
    long long tile = tile0;
    if (BATCH) {
      const int pr = (int)(tile0 / a.k_count);
      tile = tile0 - (long long)pr * a.k_count;
      if (pr != pair) {
        if (pair >= 0) {
          block_sum2(sre, sim, red);
          if (threadIdx.x == 0) {
            atomicAdd(&st->sum_re2, sre);
            atomicAdd(&st->sum_im2, sim);
          }
          sre = 0.0; sim = 0.0;
          __syncthreads();   // red is reused
        }
        pair = pr;
        shg = pp.shg[pr]; gaminv = pp.gaminv[pr]; cscale = pp.cscale[pr];
        st = pp.st[pr]; wofs = (long long)pr * pp.w_stride;
      }
    }
    bool valid, hm = false;
    long long kd, km = 0;
    int k1d = 0, k1m = 0;
    long long rd = 0, rm = 0;
    if (SYM) {
      const int4 tb = __ldg(a.tiles + tile);
      if (a.dim == 2) {
        const int k1 = tb.x, k2 = tb.y;
        valid = k2 < a.m && k2 >= k1;
        kd = (long long)k1 * a.m + k2;
        hm = valid && k2 != k1;
        km = (long long)k2 * a.m + k1;
        k1d = k1; rd = k2; k1m = k2; rm = k1;
      } else {
        const int k1 = tb.x, k2 = tb.y, k3 = tb.z;
        valid = k3 < a.m;
        kd = ((long long)k1 * a.m + k2) * a.m + k3;
        hm = valid && k1 != k2;
        km = ((long long)k2 * a.m + k1) * a.m + k3;
        k1d = k1; rd = (long long)k2 * a.m + k3; k1m = k2; rm = (long long)k1 * a.m + k3;
      }
      if (!valid) kd = 0;
    } else {
      valid = true;
      kd = a.k_begin + tile;
      if (wl.mode_major) { k1d = (int)(tile / wl.P1); rd = tile - (long long)k1d * wl.P1; }
      else rd = tile;
    }
    if (!valid) continue;   // uniform across the CTA
    const double mu = mode_mu(a.mu1, a.m, a.dim, kd);
    const double c = __ldg(a.ghat + kd) * cscale;
    const double c2 = hm ? __ldg(a.ghat + km) * cscale : 0.0;
    // 1-4. rows, one warp per row (warp-synchronous, no CTA barrier): the
    // generator in prime-factor order (slot 0: j2 = 0; slot 1 + p: j2 = g^p),
    // A = FFT240(a), Y(row, 0) = y0 + A_0 kept aside, slots <- conj(A_k bhat_k),
    // FFT240 again with the last stage storing y0 + conj(out_q) at slot
    // t2 = g^-q.
    for (int row = warp; row < kPfRows; row += T / 32) {
      double2* rowb = buf + row * kPfLen;
      double2* rowp = rowb + 1;
#pragma unroll
      for (int sl = lane; sl < kPfLen; sl += 32) {
        const int i = row * kPfLen + sl;
        const double2 s = __ldg(shg + i);
        const double dr = s.x + mu, di = s.y;
        const double den2 = dr * dr + di * di;
        // singular-shift threshold 1e-28 |s_j|^2 (space.py:237-240), rounded exactly as
        // the host forms it (no contraction), and the time index j of (row, slot)
        // only when it fires: j2 = g^(slot - 1) = tq[(241 - slot) % 240] (tq = g^-q)
        const double thr = __dmul_rn(1e-28, __dadd_rn(__dmul_rn(s.x, s.x), __dmul_rn(s.y, s.y)));
        if (den2 <= thr) {
          const int j2 = sl ? (int)s_tq[(241 - sl) % kPfNp] : 0;
          flag_singular(st, (kPfLen * row + kPfRows * j2) % kPfN);
        }
        const double inv = fast_rcp(den2);
        rowb[sl] = make_double2(dr * inv, -di * inv);
      }
      __syncwarp();
      auto natural = [&](int q, double2 x) { rowp[q] = x; };
      pf_warp_stage<4, 1>(rowp, lane, s_w, natural);
      pf_warp_stage<4, 4>(rowp, lane, s_w, natural);
      pf_warp_stage<5, 16>(rowp, lane, s_w, natural);
      pf_warp_stage<3, 80>(rowp, lane, s_w, [&](int q, double2 x) {
        if (q == 0) s_x0[row] = cadd(rowb[0], x);
        rowp[q] = cconj(cmul(x, s_bh[q]));
      });
      pf_warp_stage<4, 1>(rowp, lane, s_w, natural);
      pf_warp_stage<4, 4>(rowp, lane, s_w, natural);
      pf_warp_stage<5, 16>(rowp, lane, s_w, natural);
      pf_warp_stage<3, 80>(rowp, lane, s_w, [&](int q, double2 x) { rowp[s_tq[q] - 1] = cadd(rowb[0], cconj(x)); });
      if (lane == 0) rowb[0] = s_x0[row];
    }
    __syncthreads();
    // 5. 17-point DFT down each of the 241 columns (one per thread), the
    //    symmetric odd-prime codelet with outputs stored as they are formed
    //    (only the 8 pair sums / differences stay in registers)
    {
      const int col = threadIdx.x;
      if (col < kPfLen) {
        constexpr int R = kPfRows, H = (R - 1) / 2, off = odd_root_offset(R);
        double2* colp = buf + col;
        const double2 x0 = colp[0];
        double2 sa[H], sb[H];
        double2 sum = x0;
#pragma unroll
        for (int j = 1; j <= H; ++j) {
          const double2 p = colp[j * kPfLen], q = colp[(R - j) * kPfLen];
          sa[j - 1] = cadd(p, q);
          sb[j - 1] = csub(p, q);
          sum = cadd(sum, sa[j - 1]);
        }
        colp[0] = sum;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
          double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
          for (int j = 1; j <= H; ++j) {
            const int qq = (j * k) % R;
            const double cs = c_root_cos[off + qq], sn = c_root_sin[off + qq];
            A.x = fma(sa[j - 1].x, cs, A.x);
            A.y = fma(sa[j - 1].y, cs, A.y);
            B.x = fma(sb[j - 1].x, sn, B.x);
            B.y = fma(sb[j - 1].y, sn, B.y);
          }
          colp[k * kPfLen] = make_double2(A.x + B.y, A.y - B.x);
          colp[(R - k) * kPfLen] = make_double2(A.x - B.y, A.y + B.x);
        }
      }
    }
    __syncthreads();
    // 6. store: X_t at (t mod 17, t mod 241); W = c Re(Gamma^-1 X), residue norms
    const int nsl = wl.mode_major ? wl.nsl : 1;
    double zr2 = 0.0, zi2 = 0.0;
    for (int sl = 0; sl < nsl; ++sl) {
      const int t0 = wl.mode_major ? wl.sl_c[sl] : 0;
      const int t1 = wl.mode_major ? wl.sl_c[sl + 1] : NL;
      // thread -> t = t0 + threadIdx.x + T i: (t / 8) blocks at stride P1*8
      long long pd, pm, step;
      if (wl.mode_major) {
        const long long lo = (long long)(threadIdx.x >> 3) * wl.P1 * kTBL + (threadIdx.x & 7);
        pd = wl.row_off(sl, k1d) + rd * kTBL + lo;
        pm = wl.row_off(sl, k1m) + rm * kTBL + lo;
        step = (T / kTBL) * wl.P1 * kTBL;
      } else {
        pd = rd + (long long)threadIdx.x * wl.w_ld;
        pm = pd;
        step = (long long)T * wl.w_ld;
      }
      double* __restrict__ wd = wl.sl_base[sl] + wofs + pd;
      double* __restrict__ wmr = wl.sl_base[sl] + wofs + pm;
#pragma unroll 4
      for (int t = t0 + threadIdx.x; t < t1; t += T, wd += step, wmr += step) {
        const double2 X = buf[(t % kPfRows) * kPfLen + (t % kPfLen)];
        const double2 g = __ldg(gaminv + t);
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
    __syncthreads();   // buf is rewritten by the next mode
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0 && (!BATCH || pair >= 0)) {
    atomicAdd(&st->sum_re2, sre);
    atomicAdd(&st->sum_im2, sim);
  }
}

constexpr size_t pf_smem() { return sizeof(double2) * kPfN; }

}  // namespace fastk
}  // namespace bhcp
