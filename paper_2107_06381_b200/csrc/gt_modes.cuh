// gt_modes.cuh -- pass A for n = 1025 time levels (BASELINE config 3):
// register-resident Cooley-Tukey 1025 = 41 x 25 with a Rader 41-point first
// stage. Included by bhcp_b200.cu.
//
// X_t = sum_j v_j w^{jt}, w = exp(-2 pi i / 1025), v_j = 1 / (s_j + mu) (the
// shifted divide of space.py:276-278 for one spatial mode, pint.py:52-61).
// With j = 25 j1 + j2 and t = k1 + 41 k2 (j1, k1 in Z41; j2, k2 in Z25):
//   Y(j2, k1) = sum_j1 v_{25 j1 + j2} w41^{j1 k1}                 (41-point, 25 rows)
//   X_{k1 + 41 k2} = sum_j2 [Y(j2, k1) w1025^{j2 k1}] w25^{j2 k2}  (25-point, 41 columns)
// The 41-point transforms use Rader (g a primitive root of 41):
//   Y(j2, 0) = y0 + A_0,  Y(j2, g^-q) = y0 + conj(FFT40(conj(A * bhat)))_q,
//   A = FFT40(a), a_p = v_{25 g^p + j2}, y0 = v_{j2}, bhat = FFT40(b) / 40,
//   b_m = w41^{g^-m}; and FFT40 is the prime-factor 5 x 8 (no twiddles):
//   position (x, y) in Z5 x Z8 holds input index (8x + 5y) mod 40 and output
//   index K = CRT(x mod 5, y mod 8).
//
// One warp per mode; its 25 rows live in shared memory (row stride 43,
// slot 5y + x for FFT40 position (x, y), slot 40 = y0, slot 41 = Y(j2, 0)),
// and every small DFT runs in registers:
//   R1  (4 rounds, pencils (x, j2)): generator 1/(s_j + mu) -> DFT8 over y
//   R2  (7 rounds, lane = (y, j2 mod 4)): DFT5 over x -> * bhat, conj -> DFT5
//   R3  (4 rounds, pencils (x, j2)): DFT8 over y -> y0 + conj
//   C   (2 rounds, lane = column k1): twiddle, DFT25 (5 x 5) over j2,
//       Gamma^-1, Re, residue norms, and the store of W[t] straight from
//       registers (t = k1 + 41 k2: consecutive lanes, consecutive levels).
// Each stage reads what the previous one wrote through one shared-memory
// pass (4 passes per mode instead of 16 in a stage-per-round layout); the
// pencil orders and the stage-C lane positions make every 16-byte access
// conflict-free. Persistent CTAs of 10 warps, no CTA barrier in the mode loop.
#pragma once

namespace bhcp {
namespace fastk {

constexpr int kGtRS = 43;                 // row stride (odd: consecutive rows hit distinct banks)
constexpr int kGtRowWords = 25 * kGtRS;   // one warp's mode: 25 rows

struct GtModesArgs {
  const double* mu1;
  const double* ghat;
  double cscale;
  long long k_begin, k_count;
  double* W;
  int m, dim;
  StatusDev* st;
  const double2* tab;   // plan.h kGt2* layout
  const int* itab;      // ck1 [41] | csl [41] | gpw [40]
  WLayout wl;
  const int4* tiles;
  long long ntiles;
};

struct GtPlan { static constexpr int S = 10, T = 32 * S; };

// w25^e = cos(2 pi e / 25) - i sin(2 pi e / 25), e = 0..16 (DFT25 internal twiddles)
__constant__ double c_cos25[17] = {1.0, 0.96858316112863111949, 0.876306680043863587308, 0.728968627421411523147,
                                   0.535826794978996618271, 0.309016994374947424102, 0.0627905195293133760762,
                                   -0.187381314585724630543, -0.425779291565072648863, -0.637423989748689710177,
                                   -0.809016994374947424102, -0.929776485888251403661, -0.99211470131447783105,
                                   -0.99211470131447783105, -0.929776485888251403661, -0.809016994374947424102,
                                   -0.637423989748689710177};
__constant__ double c_sin25[17] = {0.0, 0.248689887164854788242, 0.481753674101715274987, 0.684547105928688673732,
                                   0.844327925502015078549, 0.951056516295153572116, 0.998026728428271561952,
                                   0.982287250728688681086, 0.904827052466019527714, 0.770513242775789230803,
                                   0.587785252292473129169, 0.368124552684677959157, 0.125333233564304245373,
                                   -0.125333233564304245373, -0.368124552684677959157, -0.587785252292473129169,
                                   -0.770513242775789230803};

__device__ __forceinline__ double2 cmulc(double2 a, double c, double s) {   // a * (c + i s)
  return make_double2(fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c));
}

// 1/(s + mu) with the singular-shift test of space.py:237-240 when CHECK
template <bool CHECK>
__device__ __forceinline__ double2 gen_inv(double2 s, double mu, StatusDev* st, long long j) {
  const double dr = s.x + mu, di = s.y;
  const double den2 = fma(dr, dr, di * di);
  if (CHECK) {
    if (den2 <= 1e-28 * fma(s.x, s.x, s.y * s.y)) flag_singular(st, j);
  }
  const double inv = fast_rcp(den2);
  return make_double2(dr * inv, -di * inv);
}

// W address of level t for destination (row k1, in-row index r) of layout wl
__device__ __forceinline__ double* w_level_ptr(const WLayout& wl, int k1, long long r, int t) {
  if (!wl.mode_major) return wl.sl_base[0] + (long long)t * wl.w_ld + r;
  int s = 0;
  while (s + 1 < wl.nsl && t >= wl.sl_c[s + 1]) ++s;
  const int tl = t - wl.sl_c[s];
  return wl.sl_base[s] + wl.row_off(s, k1) + (((long long)(tl >> 3)) * wl.P1 + r) * kTBL + (tl & 7);
}

// One work item = one warp-mode: SYM (2D/3D mirror tiles): item = tile * S + w,
// the w-th mode of tile `tile` (invalid off the triangle / past m: skipped);
// otherwise item = local mode index.
struct GtItem {
  bool valid, hm;
  long long kd, km, rd, rm;
  int k1d, k1m;
};

template <bool SYM>
__device__ __forceinline__ GtItem gt_decode(const GtModesArgs& a, long long item, int4 tb) {
  GtItem it{};
  constexpr int S = GtPlan::S;
  if (SYM) {
    const int w = (int)(item % S);
    if (a.dim == 2) {
      const int k1 = tb.x, k2 = tb.y + w;
      it.valid = k2 < a.m && k2 >= k1;
      it.kd = (long long)k1 * a.m + k2;
      it.hm = it.valid && k2 != k1;
      it.km = (long long)k2 * a.m + k1;
      it.k1d = k1; it.rd = k2; it.k1m = k2; it.rm = k1;
    } else {
      const int k1 = tb.x, k2 = tb.y, k3 = tb.z + w;
      it.valid = k3 < a.m;
      it.kd = ((long long)k1 * a.m + k2) * a.m + k3;
      it.hm = it.valid && k1 != k2;
      it.km = ((long long)k2 * a.m + k1) * a.m + k3;
      it.k1d = k1; it.rd = (long long)k2 * a.m + k3; it.k1m = k2; it.rm = (long long)k1 * a.m + k3;
    }
  } else {
    it.valid = item < a.k_count;
    const long long local = it.valid ? item : 0;
    it.kd = a.k_begin + local;
    if (a.wl.mode_major) { it.k1d = (int)(local / a.wl.P1); it.rd = local - (long long)it.k1d * a.wl.P1; }
    else it.rd = local;
  }
  return it;
}

// FAST: one level slab without a block table (the single-GPU blocked W): the
// store offset of level t is (t / 8) * P1 * 8 + t % 8 from the mode's base;
// otherwise w_level_ptr walks the slabs (multi-GPU layouts, 1D level-major W).
template <bool SYM, bool CHECK, bool FAST>
__global__ void __launch_bounds__(GtPlan::T, 1) k_modes_gt(GtModesArgs a) {
  constexpr int S = GtPlan::S, T = GtPlan::T, RS = kGtRS;
  extern __shared__ double2 smem[];
  __shared__ double red[2 * S];
  __shared__ int s_ck1[41], s_csl[41], s_gpw[40];
  // generic (multi-slab / block-table) W stores: level tile -> slab, and per warp
  // the mode's (and its mirror's) base pointer in every slab, biased so that
  // level t lands at base[slab(t)] + (t >> 3) * P1 * 8 + (t & 7) (slabs start at
  // multiples of 8 levels)
  __shared__ unsigned char s_slab[FAST ? 1 : 136];
  __shared__ double* s_sb[FAST ? 1 : S][2][8];
  double2* s_sg = smem;                       // [8][128] + y0 [32]
  double2* s_tw = smem + kGt2Tw;              // [25][41]
  double2* s_gi = smem + kGt2Gi;              // [25][41]
  double2* s_bh = smem + kGt2Bh;              // [8][5]
  for (int i = threadIdx.x; i < kGt2Total; i += T) smem[i] = __ldg(a.tab + i);
  for (int i = threadIdx.x; i < 41; i += T) {
    s_ck1[i] = __ldg(a.itab + i);
    s_csl[i] = __ldg(a.itab + 41 + i);
    if (i < 40) s_gpw[i] = __ldg(a.itab + 82 + i);
  }
  if (!FAST && a.wl.mode_major) {
    for (int i = threadIdx.x; i < 136; i += T) {
      int sl = 0;
      while (sl + 1 < a.wl.nsl && 8 * i >= a.wl.sl_c[sl + 1]) ++sl;
      s_slab[i] = (unsigned char)sl;
    }
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* Y = smem + kGt2Total + warp * kGtRowWords;
  StatusDev* st = a.st;
  const WLayout& wl = a.wl;
  double sre = 0.0, sim = 0.0;
  const long long nitems = SYM ? a.ntiles * S : a.k_count;

  // Dynamic per-warp scheduling (atomic counter in the status block, reset by the
  // last CTA): warps finish together whatever their share of off-triangle items.
  // Depth-2 prefetch: while mode i is transformed, item i+2 is claimed and item
  // i+1's tile, mu and ghat loads are in flight.
  auto claim = [&]() -> long long {
    unsigned long long v = 0;
    if (lane == 0) v = atomicAdd(&st->work, 1ull);
    return (long long)__shfl_sync(0xffffffffu, v, 0);
  };
  long long cur = claim();
  long long nxt = claim();
  int4 tb_cur = make_int4(0, 0, 0, 0);
  if (SYM && cur < nitems) tb_cur = __ldg(a.tiles + cur / S);
  while (cur < nitems) {
    const GtItem it = gt_decode<SYM>(a, cur, tb_cur);
    // next item's tile (consumed at the next iteration) and the claim after it
    int4 tb_nxt = make_int4(0, 0, 0, 0);
    if (SYM && nxt < nitems) tb_nxt = __ldg(a.tiles + nxt / S);
    const long long nxt2 = claim();
    if (!it.valid) {   // warp-uniform
      cur = nxt; nxt = nxt2; tb_cur = tb_nxt;
      continue;
    }
    const double mu = (SYM && a.dim == 2) ? __ldg(a.mu1 + it.k1d) + __ldg(a.mu1 + it.rd)
                                          : mode_mu(a.mu1, a.m, a.dim, it.kd);
    const double c = __ldg(a.ghat + it.kd) * a.cscale;
    const double c2 = it.hm ? __ldg(a.ghat + it.km) * a.cscale : 0.0;

    // ---- R1: generator + DFT8 over y, pencils p = x * 25 + j2 (x = alpha), two per lane at a time
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int pa = lane + 64 * h, pb = pa + 32;
      const bool okb = pb < 125;
      double2 va[8], vb[8];
      const int xa = pa / 25, ja = pa - xa * 25, xb = pb / 25, jb = pb - xb * 25;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const long long jja = CHECK ? 25LL * s_gpw[(8 * xa + 5 * y) % 40] + ja : 0;
        const long long jjb = CHECK ? 25LL * s_gpw[(8 * xb + 5 * y) % 40] + jb : 0;
        va[y] = gen_inv<CHECK>(s_sg[y * 128 + pa], mu, st, jja);
        vb[y] = okb ? gen_inv<CHECK>(s_sg[y * 128 + pb], mu, st, jjb) : make_double2(0.0, 0.0);
      }
      Dft<8>::prep(va);
      Dft<8>::prep(vb);
      double2* rowa = Y + ja * RS;
      double2* rowb = Y + jb * RS;
#pragma unroll
      for (int k = 0; k < 8; ++k) rowa[5 * k + xa] = va[k];
      if (okb) {
#pragma unroll
        for (int k = 0; k < 8; ++k) rowb[5 * k + xb] = vb[k];
      }
    }
    if (lane < 25) Y[lane * RS + 40] = gen_inv<CHECK>(s_sg[1024 + lane], mu, st, lane);   // y0 = v_{j2}
    __syncwarp();
    // ---- R2: DFT5 over x, * bhat, conj, DFT5. Lane l keeps y = l % 8 (its five
    // bhat factors stay in registers) and takes rows j2 = l / 8 + 4 r, two rows at a time
    {
      const int y = lane & 7;
      double2 bh[5];
#pragma unroll
      for (int x = 0; x < 5; ++x) bh[x] = s_bh[y * 5 + x];
#pragma unroll 1
      for (int r = 0; r < 7; r += 2) {
        const int ja = (lane >> 3) + 4 * r, jb = ja + 4;
        const bool oka = ja < 25, okb = jb < 25 && r + 1 < 7;
        double2* rowa = Y + ja * RS;
        double2* rowb = Y + jb * RS;
        double2 ua[5], ub[5];
#pragma unroll
        for (int x = 0; x < 5; ++x) {
          ua[x] = oka ? rowa[5 * y + x] : make_double2(0.0, 0.0);
          ub[x] = okb ? rowb[5 * y + x] : make_double2(0.0, 0.0);
        }
        sfft::Cod<5>::run(ua);
        sfft::Cod<5>::run(ub);
        if (y == 0) {   // Y(j2, 0) = y0 + A_0
          if (oka) rowa[41] = cadd(rowa[40], ua[0]);
          if (okb) rowb[41] = cadd(rowb[40], ub[0]);
        }
#pragma unroll
        for (int x = 0; x < 5; ++x) {
          ua[x] = cconj(cmul(ua[x], bh[x]));
          ub[x] = cconj(cmul(ub[x], bh[x]));
        }
        sfft::Cod<5>::run(ua);
        sfft::Cod<5>::run(ub);
        if (oka) {
#pragma unroll
          for (int x = 0; x < 5; ++x) rowa[5 * y + x] = ua[x];
        }
        if (okb) {
#pragma unroll
          for (int x = 0; x < 5; ++x) rowb[5 * y + x] = ub[x];
        }
      }
    }
    __syncwarp();
    // ---- R3: DFT8 over y, conv = conj, Y = y0 + conv; pencils p = x * 25 + j2, two per lane at a time
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int pa = lane + 64 * h, pb = pa + 32;
      const bool okb = pb < 125;
      const int xa = pa / 25, ja = pa - xa * 25, xb = pb / 25, jb = pb - xb * 25;
      double2* rowa = Y + ja * RS;
      double2* rowb = Y + jb * RS;
      double2 va[8], vb[8];
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        va[y] = rowa[5 * y + xa];
        vb[y] = okb ? rowb[5 * y + xb] : make_double2(0.0, 0.0);
      }
      const double2 y0a = rowa[40];
      const double2 y0b = okb ? rowb[40] : make_double2(0.0, 0.0);
      Dft<8>::prep(va);
      Dft<8>::prep(vb);
#pragma unroll
      for (int y = 0; y < 8; ++y) rowa[5 * y + xa] = make_double2(y0a.x + va[y].x, y0a.y - va[y].y);
      if (okb) {
#pragma unroll
        for (int y = 0; y < 8; ++y) rowb[5 * y + xb] = make_double2(y0b.x + vb[y].x, y0b.y - vb[y].y);
      }
    }
    __syncwarp();
    // ---- C: column k1 per lane: twiddle, DFT25 over j2, Gamma^-1, Re, norms, stores
    if (!FAST && wl.mode_major) {
      if (lane < wl.nsl) {
        const long long bias = (long long)(wl.sl_c[lane] >> 3) * wl.P1 * kTBL;
        s_sb[FAST ? 0 : warp][0][lane] = wl.sl_base[lane] + (wl.row_off(lane, it.k1d) + it.rd * kTBL - bias);
        if (it.hm) s_sb[FAST ? 0 : warp][1][lane] = wl.sl_base[lane] + (wl.row_off(lane, it.k1m) + it.rm * kTBL - bias);
      }
      __syncwarp();
    }
    double zr2 = 0.0, zi2 = 0.0;
    const int dstride = FAST ? (int)(wl.P1 * kTBL) : 0;
    double* const based = FAST ? wl.sl_base[0] + wl.row_off(0, it.k1d) + it.rd * kTBL : nullptr;
    double* const basem = FAST ? wl.sl_base[0] + wl.row_off(0, it.k1m) + it.rm * kTBL : nullptr;
#pragma unroll 1
    for (int cp = lane; cp < 41; cp += 32) {
      const int k1 = s_ck1[cp];
      const double2* col = Y + s_csl[cp];
      double2 z[25];
      z[0] = col[0];
#pragma unroll
      for (int j2 = 1; j2 < 25; ++j2) z[j2] = cmul(col[j2 * RS], s_tw[j2 * 41 + cp]);
      // DFT25, j2 = 5 a + b, k2 = q + 5 d: DFT5 over a, twiddle w25^{b q}, DFT5 over b
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        double2 u[5] = {z[b], z[5 + b], z[10 + b], z[15 + b], z[20 + b]};
        sfft::Cod<5>::run(u);
        z[b] = u[0];
#pragma unroll
        for (int q = 1; q < 5; ++q) {
          if (b == 0) z[5 * q + b] = u[q];
          else z[5 * q + b] = cmulc(u[q], c_cos25[b * q], -c_sin25[b * q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        double2 u[5] = {z[5 * q], z[5 * q + 1], z[5 * q + 2], z[5 * q + 3], z[5 * q + 4]};
        sfft::Cod<5>::run(u);
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int k2 = q + 5 * d;
          const int t = k1 + 41 * k2;
          const double2 gi = s_gi[k2 * 41 + cp];
          const double zr = fma(u[d].x, gi.x, -u[d].y * gi.y);
          const double zi = fma(u[d].x, gi.y, u[d].y * gi.x);
          zr2 = fma(zr, zr, zr2);
          zi2 = fma(zi, zi, zi2);
          if (FAST) {
            const int off = (t >> 3) * dstride + (t & 7);
            based[off] = c * zr;
            if (it.hm) basem[off] = c2 * zr;
          } else if (wl.mode_major) {
            const int sl = s_slab[t >> 3];
            const long long off = (long long)(t >> 3) * wl.P1 * kTBL + (t & 7);
            s_sb[FAST ? 0 : warp][0][sl][off] = c * zr;
            if (it.hm) s_sb[FAST ? 0 : warp][1][sl][off] = c2 * zr;
          } else {
            *w_level_ptr(wl, it.k1d, it.rd, t) = c * zr;
            if (it.hm) *w_level_ptr(wl, it.k1m, it.rm, t) = c2 * zr;
          }
        }
      }
    }
    const double cc = c * c + c2 * c2;
    sre = fma(cc, zr2, sre);
    sim = fma(cc, zi2, sim);
    __syncwarp();   // Y (and the warp's slab base pointers) are rewritten by the next mode
    cur = nxt; nxt = nxt2; tb_cur = tb_nxt;
  }
  block_sum2(sre, sim, red);
  if (threadIdx.x == 0) {
    atomicAdd(&a.st->sum_re2, sre);
    atomicAdd(&a.st->sum_im2, sim);
    // the last CTA out resets the work counter for the next launch on this status block
    __threadfence();
    if (atomicAdd(&st->done, 1ull) == gridDim.x - 1) {
      st->work = 0;
      st->done = 0;
      __threadfence();
    }
  }
}

constexpr size_t gt_smem() { return sizeof(double2) * ((size_t)kGt2Total + (size_t)kGtRowWords * GtPlan::S); }

}  // namespace fastk
}  // namespace bhcp
