// lvl_dst.cuh -- the whole level phase of the fused 2D solve for m + 1 = 1024
// (c3) as ONE persistent kernel that walks the levels in groups small enough
// to stay in the 126 MB L2 (k_dst_lvl4).
//
// The two spatial DSTs of every level (space.py:163-177, per level as in
// pint.py:94-96) used to be two full sweeps of HBM: k_dst_blk4 (last axis,
// blocked W -> y, 16 B/DOF) and k_dst_cols3 (strided axis in place on y,
// 16 B/DOF, 2.6 TB/s because its 64 B row chunks sit 8 KB apart). Here one
// W level tile (8 levels, 67 MB) is a group:
//   row task    B(g, k1): one 64 KB W block (k1, level tile g) -> 8 rows of
//               the scratch Z (the k_dst_blk4 work; W read from HBM by TMA
//               with an evict-first hint). Z holds one level tile per slot
//               (two slots) with a 1024-double row pitch, so unlike y
//               (1023-double rows) it is a TMA tensor. Element e of a row
//               sits at Z column e + 1 (column 0 is a zero pad), so a lane's
//               outputs S_2k, S_2k+1 are one aligned 16-byte store.
//   column task C(g, t, c): 8 adjacent Z columns of level t (elements
//               8c - 1 .. 8c + 6), all 1023 rows, loaded from Z by TMA (still
//               in L2), transformed into a row-parity-split tile (at_par) and
//               stored to y: the rows whose 64 B chunk is 16-byte aligned (odd
//               global rows) by two TMA boxes of the row-pair view of y, the
//               others by 8-byte stores (a TMA box must start 16-byte
//               aligned; the first column tile and the last level entirely
//               by 8-byte stores); after the odd column tile of a
//               pair (both on one CTA) the Z lines are discarded from L2
//               (discard.global.L2) instead of being written back.
// W is read and y written once; Z lines that L2 evicts before their discard
// are the only extra traffic (c3: 11.5 GB read + 14.1 GB written by this
// kernel against 17.2 + 17.1 GB for k_dst_blk4 + k_dst_cols3).
//
// Order. Task pairs (two row tasks k1 = 2i, 2i + 1; or the even and odd
// column tile of one 128-byte Z column pair), 1024 row tasks per level tile
// (the last one empty), in one global order (decode): phase 0 = B(0); phase p
// = the first `kfirst` B(p) pairs, all of C(p - 1), the rest of B(p); phase
// NT = C(NT - 1). CTA c takes the pairs c, c + G, ... (all CTAs co-resident,
// one per SM) and runs its tasks in increasing order. A column task of level
// tile g waits for g's row-task counter, and a row task of g >= 2 for the
// column-task counter of g - 2 (its Z slot); both point to lower task
// indices, so the lowest unfinished task never waits and the kernel cannot
// deadlock. The look-ahead row tasks keep every CTA busy while the last row
// tasks of level tile p - 1 drain.
//
// Measured on a B200 (c3, 1025 levels): 9.3-9.5 ms against 10.2 ms for the
// two sweeps. Variants that lost: 4-level groups (half W blocks: 32 B of each
// 64 B row, so DRAM reads W twice); column tiles gathered straight from y
// (8-byte cp.async by one warp: 15 us per tile); C(p - 1) spread over all of
// phase p (two level tiles of Z resident: L2 hit rate 42%, 15 GB written);
// strictly sequential phases (every CTA idles while the last row tasks
// drain: 9.8 ms); Z rows stored with an evict-last hint (the hinted 8-byte
// stores cost the consumers 20% more issue time). A kernel's freshly written
// lines survive in L2 for the next reader up to about 64 MB
// (tools/probe_l2.cu), which is what one 67 MB level tile leans on.
//
// Warps: 8 consumers (4 line pairs x 2 halves: warp_dst1024; two warpgroups at
// 232 registers after setmaxnreg), 1 producer (TMA loads of both task kinds,
// after the counters), 1 storer (the TMA half of a column tile to y, Z
// discards, the release increments of the counters) and two idle warps that
// only donate their registers. Three 64 KB buffers, per buffer the mbarriers
// full (producer -> consumers), done (consumers -> storer) and free (storer ->
// producer). Variants that lost (round 2): an FP64 ping-pong between line
// pairs through named barriers (no change); two consumer teams of 8 warps at
// 112 registers on alternate tiles (each team twice as slow: 9.4 ms); the
// misaligned y rows stored by three / two storer warps instead of the consumers
// (storers become the bottleneck: 9.9 / 10.2 ms); a product tree for the
// twiddle powers (no change). What bounds the consumers (round-2 ablations,
// DESIGN.md section 7): not the butterflies (removing them: -0.4 ms) but the
// LSU / shared-memory pipe -- 3.6 K LDS/STS wavefronts, 1.4 K shuffles of the
// odd-output prefix sums and the global stores per 7.7 K-cycle tile.
#pragma once
#include "wax2_dst.cuh"

namespace bhcp {
namespace lvl {

using namespace sfft;
using wax::su32;
using wax::mbar_init;
using wax::mbar_expect;
using wax2::mbar_sleep_wait;
using wax2::Sw64;
using wax2::at;

// -DLVL4_PROF: per-role clock64 accounting, printed by a few CTAs at the end
// (diagnostics only; never in the shipped build)
#ifdef LVL4_PROF
#define LP_T0(v) const long long v = clock64()
#define LP_ADD(slot, t0) atomicAdd(&prof[slot], (unsigned long long)(clock64() - (t0)))
#else
#define LP_T0(v)
#define LP_ADD(slot, t0)
#endif

constexpr int kN = 1024;
constexpr int kNB = 3;        // tile buffers
constexpr int kCW = 8;        // consumer warps
constexpr int kSW = 1;        // storer warps
// Warpgroups 0, 1 = the consumers; warpgroup 2 = producer, storer, two idle warps.
// The kernel launches at 168 registers per thread (384 threads); the auxiliary
// warpgroup then drops to kRegsAux and the consumers rise to kRegsCons
// (setmaxnreg moves registers inside the CTA's allocation: 256 x 232 + 128 x 40
// = 384 x 168), so the consumers' 16 complex values, twiddles and addresses stay
// in registers with room for the scheduler to hoist loads.
constexpr int kThreads = 384;
constexpr int kRegsCons = 232, kRegsAux = 40;
constexpr int kTD2 = kN * 4;  // double2 per tile (8 lines x 1024 rows)

constexpr size_t smem_bytes() {
  return 1024 + (size_t)kNB * kTD2 * 16 + sizeof(double) * (kN + 4 * 42) + 8 * 3 * kNB;
}

struct ArgsLV {
  const double2* tw;   // exp(-2 pi i k / N)
  const double* sn;    // sin(pi j / N)
  double scale;        // sqrt(2 / N)
  double* y;           // (nlev, m, m) level-major
  double* z;           // scratch: [2 slots][8 levels][m rows][1024]
  unsigned* gdone;     // per level tile: row tasks finished (zeroed before the launch)
  unsigned* cdone;     // per level tile: column tasks finished (Z slot free again)
  int m;               // 1023
  int nt;              // level tiles (groups)
  int nlev;
  int nct;             // column tiles per level: ceil(m / 8), even
  int ntasks;
  int kfirst;          // row-task pairs of phase p before the column tasks of level tile p - 1
};

constexpr int kRowTasks = 1024;   // row tasks per group (k1 = m .. 1023 empty)
constexpr int kZPitch = 1024;     // doubles per Z row

struct Task {
  int kind;   // 0 row task, 1 column task
  int g;      // level tile
  int idx;    // row task: k1; column task: (level within the tile) * nct + column tile
};

// Task pairs (two row tasks k1 = 2i, 2i + 1, or the even and odd column tile of
// one 128-byte Z column pair) in one global order: phase 0 = B(0); phase p =
// the first `kfirst` B(p) pairs (work for every CTA while the last row tasks
// of level tile p - 1 drain), then all of C(p - 1), then the rest of B(p);
// phase NT = C(NT - 1).
__device__ __forceinline__ Task decode(const ArgsLV& a, int i) {
  const int pi = i >> 1, u = i & 1;
  const int nb = kRowTasks / 2, nc = 4 * a.nct, per = nb + nc;
  Task t;
  int pidx;
  if (pi < nb) { t.kind = 0; t.g = 0; pidx = pi; }
  else {
    const int p = 1 + (int)((unsigned)(pi - nb) / (unsigned)per);
    const int j = pi - nb - (p - 1) * per;
    const int kf = a.kfirst < nb ? a.kfirst : nb;
    if (p >= a.nt) { t.kind = 1; t.g = a.nt - 1; pidx = j; }
    else if (j < kf) { t.kind = 0; t.g = p; pidx = j; }
    else if (j < kf + nc) { t.kind = 1; t.g = p - 1; pidx = j - kf; }
    else { t.kind = 0; t.g = p; pidx = j - nc; }
  }
  t.idx = 2 * pidx + u;
  return t;
}
// task of CTA c's it-th slot: pairs 2c + 2Gk + {0, 1}
__device__ __forceinline__ int task_of(int c, int G, int it) { return 2 * c + 2 * G * (it >> 1) + (it & 1); }

__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load3_hint(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                               unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(su32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void st_hint(double* p, double v, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void discard_l2(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(p) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void tma_store2_hint(const CUtensorMap* tm, int c0, int c1, const void* src,
                                                unsigned long long pol) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;\n" ::"l"(tm),
               "r"(c0), "r"(c1), "r"(su32(src)), "l"(pol)
               : "memory");
}

// Column-task output layout: the rows of the tile split by parity, plane p =
// e & 1 holding rows e = 2 j + p at 64-byte row j (64-byte swizzle), so that
// each plane is what one TMA box of the parity view of y stores (y rows are
// 1023 doubles, so only row PAIRS have a 16-byte multiple pitch: the view is
// {2046 = (row parity s) x 1023 + column, row pairs}).
__device__ __forceinline__ double2* at_par(double2* T, int e, int q) {
  const int j = e >> 1;
  return T + ((e & 1) * 512 + j) * 4 + (q ^ ((j >> 1) & 3));
}
// Row-task output sink: the two Z rows of the line pair, straight from
// registers. Z stores element e of a row at column e + 1, so a unit's outputs
// S_{2k} (element 2k - 1) and S_{2k+1} (element 2k) are ONE aligned 16-byte
// store at column 2k, consecutive lanes writing consecutive chunks (k = 0:
// the pad column 0 gets the zero the column tasks read as element -1).
struct ZRowSink {
  double* za;
  double* zb;
  bool va, vb;
  int j1, j2;
  __device__ __forceinline__ void put(int r, bool hi, int v, double2 ev, double2 od) {
    const int k = (hi ? j2 : j1) + 128 * r;
    const bool he = k > 0;
    if (va) *reinterpret_cast<double2*>(za + 2 * k) = make_double2(he ? ev.x : 0.0, od.x);
    if (vb) *reinterpret_cast<double2*>(zb + 2 * k) = make_double2(he ? ev.y : 0.0, od.y);
  }
};
struct ParitySink {
  double2* T;
  int q;
  int j1, j2;
  // k = j1 + 128 r (lo) or j2 + 128 r (hi); ev = S_{2k} -> element 2k - 1, od = S_{2k+1} -> 2k
  __device__ __forceinline__ void put(int r, bool hi, int v, double2 ev, double2 od) {
    const int k = (hi ? j2 : j1) + 128 * r;
    if (k > 0) *at_par(T, 2 * k - 1, q) = ev;
    *at_par(T, 2 * k, q) = od;
  }
};

__global__ void __launch_bounds__(kThreads, 1) k_dst_lvl4(const __grid_constant__ CUtensorMap tm,
                                                          const __grid_constant__ CUtensorMap tz,
                                                          const __grid_constant__ CUtensorMap ty256,
                                                          const __grid_constant__ CUtensorMap ty255, ArgsLV a) {
  constexpr int NBOX = kN / wax::kBoxRows;
  constexpr unsigned TILE_BYTES = (unsigned)(kN * 8 * sizeof(double));
  extern __shared__ unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  double2* tiles = reinterpret_cast<double2*>(base);
  double* sn = reinterpret_cast<double*>(base + (size_t)kNB * kTD2 * 16);
  double* xch = sn + kN;
  unsigned long long* full = reinterpret_cast<unsigned long long*>(xch + 4 * 42);
  unsigned long long* done = full + kNB;
  unsigned long long* freeb = done + kNB;
#ifdef LVL4_PROF
  __shared__ unsigned long long prof[16];
  __shared__ long long issue_t[kNB];
  if (threadIdx.x < 16) prof[threadIdx.x] = 0;
  const long long k_t0 = clock64();
#endif
  for (int j = threadIdx.x; j < kN; j += blockDim.x) sn[j] = __ldg(a.sn + j);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tm) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tz) : "memory");
    for (int b = 0; b < kNB; ++b) {
      mbar_init(full + b, 1);
      mbar_init(done + b, kCW);
      mbar_init(freeb + b, kSW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int G = gridDim.x;
  int ntiles_cta = 0;   // slots it with task_of(c, G, it) < ntasks (increasing in it)
  {
    const int c2 = 2 * (int)blockIdx.x;
    if (a.ntasks > c2) {
      const int full_pairs = (a.ntasks - c2) / (2 * G), rem = (a.ntasks - c2) - full_pairs * 2 * G;
      ntiles_cta = 2 * full_pairs + (rem >= 2 ? 2 : rem);
    }
  }
  const long long m = a.m, lvl = m * m;
  if (warp >= kCW) {
  // the auxiliary warpgroup hands its registers to the two consumer warpgroups
  // (no path from here joins the consumers' code again: ptxas allocates each
  // region for the register count set on every path into it)
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegsAux));
  if (warp > kCW + kSW) return;
  if (warp == kCW) {
    // ---------------------------------------------------------------- producer
    if (lane != 0) return;
    const unsigned long long pol = evict_first_policy();
    for (int it = 0; it < ntiles_cta; ++it) {
      const int b = it % kNB;
      LP_T0(tw0);
      if (it >= kNB) mbar_sleep_wait(freeb + b, (unsigned)(((it - kNB) / kNB) & 1));
      LP_ADD(0, tw0);
      const Task tk = decode(a, task_of((int)blockIdx.x, G, it));
      double2* T = tiles + b * kTD2;
      if (tk.kind == 0) {
        // Z slot g & 1 is free once every column task of level tile g - 2 has loaded it
        if (tk.g >= 2) {
          LP_T0(tg0);
          while (ld_acquire(a.cdone + tk.g - 2) < (unsigned)(8 * a.nct)) __nanosleep(128);
          LP_ADD(12, tg0);
        }
#ifdef LVL4_PROF
        issue_t[b] = clock64();
#endif
        const int o = tk.idx * a.nt + tk.g;   // W block (k1, level tile); k1 >= m: out of range, zero fill
        mbar_expect(full + b, TILE_BYTES);
#pragma unroll
        for (int x = 0; x < NBOX; ++x)
          tma_load3_hint(T + x * wax::kBoxRows * 4, &tm, 0, x * wax::kBoxRows, o, full + b, pol);
      } else {
        // column task: wait until every row task of the level tile has stored its Z rows
        LP_T0(td0);
        while (ld_acquire(a.gdone + tk.g) < (unsigned)kRowTasks) __nanosleep(128);
        LP_ADD(1, td0);
#ifdef LVL4_PROF
        issue_t[b] = clock64();
#endif
        asm volatile("fence.proxy.async.global;\n" ::: "memory");   // generic Z stores -> TMA reads
        const int lev = tk.idx / a.nct, c0 = (tk.idx % a.nct) * 8;
        mbar_expect(full + b, TILE_BYTES);
        // Z view {1024 columns, m rows (row m: zero fill = the DST's row N - 1), 16 slot levels}
#pragma unroll
        for (int x = 0; x < NBOX; ++x)
          // (no evict-first mark: the other half of each 128 B line is the next column tile's)
          wax::tma_load3(T + x * wax::kBoxRows * 4, &tz, c0, x * wax::kBoxRows, (tk.g & 1) * 8 + lev, full + b);
      }
    }
    return;
  }
  if (warp > kCW) {
    // ----------------------------------------------------------------- storers
    const int sw = warp - kCW - 1;
    const unsigned long long pol = evict_first_policy();
    for (int it = 0; it < ntiles_cta; ++it) {
      const int b = it % kNB;
      LP_T0(ts0);
      mbar_sleep_wait(done + b, (unsigned)((it / kNB) & 1));
      if (sw == 0 && lane == 0) LP_ADD(2, ts0);
      LP_T0(ts1);
      const Task tk = decode(a, task_of((int)blockIdx.x, G, it));
      if (tk.kind == 0) {
        // the consumers' Z rows (observed through the done barrier) before the count
        if (sw == 0 && lane == 0) {
          __threadfence();
          atomicAdd(a.gdone + tk.g, 1u);
        }
      } else {
        const double2* T = tiles + b * kTD2;
        const int lev = tk.idx / a.nct, ct = tk.idx % a.nct, c0 = ct * 8;
        const int t = tk.g * 8 + lev;
        const long long R0 = (long long)t * m;
        if (t < a.nlev - 1 && ct > 0 && sw == 0 && lane == 0) {
          // the tile's 8 lines are elements c0 - 1 .. c0 + 6 (Z column = element + 1).
          // The plane whose rows are ODD in y (their 64 B chunk at column c0 - 1 is
          // 16-byte aligned) leaves by two TMA boxes of the row-pair view, second row
          // of each pair: inner coordinate 1023 + c0 - 1 (the second box 255 rows if
          // it is plane 1: row e = 1023 is the DST's zero row); the consumers stored
          // the other plane, and every row of the first column tile (its line 0 is
          // the pad column)
          const int pe = (int)(R0 & 1) ^ 1;   // plane with (R0 + pe) odd
          const int P0 = (int)((R0 + pe - 1) >> 1);
          tma_store2_hint(&ty256, 1022 + c0, P0, T + (pe * 512) * 4, pol);
          tma_store2_hint(pe ? &ty255 : &ty256, 1022 + c0, P0 + 256, T + (pe * 512 + 256) * 4, pol);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        }
        if ((ct & 1) && sw == kSW - 1) {
          // both column tiles of this 128-byte Z column pair are loaded (same CTA, in
          // order): drop the lines from L2 without writing them back
          const double* zc = a.z + ((long long)((tk.g & 1) * 8 + lev) * m) * kZPitch + (ct >> 1) * 16;
          for (int r = lane; r < a.m; r += 32) discard_l2(zc + (long long)r * kZPitch);
        }
        if (sw == kSW - 1 && lane == 0) {
          // this tile's Z reads (complete: the consumers saw its data) and discards
          // before the count that lets row tasks of level tile g + 2 rewrite the slot
          __threadfence();
          atomicAdd(a.cdone + tk.g, 1u);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (sw == 0) LP_ADD(tk.kind == 0 ? 3 : 4, ts1);
        wax2::mbar_arrive(freeb + b);
      }
    }
    if (sw == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    return;
  }
  return;
  }
  // ------------------------------------------------------------------ consumers
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegsCons));
  // warp w: half w >> 2 of line pair w (w < 4) or (w + 2) & 3: each scheduler
  // hosts halves of two different line pairs (warps w and w + 4), which are not
  // in lockstep at the pair barriers
  const int q = warp >= 4 ? ((warp + 2) & 3) : warp, h = warp >> 2, bar = 1 + q;
  const wax2::LaneK1024 K(lane, h, a.tw, a.scale);
  const wax2::SnRegs snr(sn, K.j1, K.j2);
  for (int it = 0; it < ntiles_cta; ++it) {
    const int b = it % kNB;
    double2* T = tiles + b * kTD2;
    const Task tk = decode(a, task_of((int)blockIdx.x, G, it));
    LP_T0(tc0);
    mbar_sleep_wait(full + b, (unsigned)((it / kNB) & 1));
#ifdef LVL4_PROF
    if (warp == 0 && lane == 0) {
      LP_ADD(5, tc0);
      atomicAdd(&prof[tk.kind == 0 ? 6 : 7], (unsigned long long)(clock64() - issue_t[b]));
      atomicAdd(&prof[tk.kind == 0 ? 10 : 11], 1ull);
    }
#endif
    LP_T0(tc1);
    if (tk.kind == 0) {
      const int k1 = tk.idx;
      const int t0 = tk.g * 8 + 2 * q;   // levels of lines 2q, 2q + 1
      const bool za = t0 >= a.nlev, zb = t0 + 1 >= a.nlev;
      if (za || zb) {
        // padding levels of the last level tile: zero them (they share the complex FFT)
        for (int e = h * 32 + lane; e < kN; e += 64) {
          double2* p = at<Sw64>(T, e, q);
          if (za) p->x = 0.0;
          if (zb) p->y = 0.0;
        }
        wax2::pair_sync(bar);
      }
      // Z rows (slot, level t0 & 7, k1) and (.., t0 + 1, k1); k1 >= m (the empty last task): none
      const bool kv = k1 < a.m;
      const long long rowa = ((long long)((tk.g & 1) * 8 + 2 * q) * m + k1) * kZPitch;
      double* za_row = a.z + rowa;
      double* zb_row = za_row + m * kZPitch;
      ZRowSink sink{za_row, zb_row, kv && !za, kv && !zb, K.j1, K.j2};
      wax2::warp_dst1024<Sw64>(T, q, h, K, snr, xch + q * 42, bar, sink);
    } else {
      ParitySink sink{T, q, K.j1, K.j2};
      wax2::warp_dst1024<Sw64>(T, q, h, K, snr, xch + q * 42, bar, sink);
      // all four line pairs are in the tile: the consumers store the rows TMA cannot
      // (chunks 8 bytes off 16-byte alignment; every row for the last column tile
      // and the last level) with 8-byte stores, 8 lanes per row
      asm volatile("bar.sync 5, %0;\n" ::"r"(kCW * 32) : "memory");
      const int lev = tk.idx / a.nct, c0 = (tk.idx % a.nct) * 8;
      const int t = tk.g * 8 + lev;
      const long long R0 = (long long)t * m;
      const int l = lane & 7, rr = 4 * warp + (lane >> 3);   // 32 rows per round over the 8 warps
      const bool lv = c0 + l >= 1;   // tile line l = Z column c0 + l = element c0 + l - 1 (Z column 0: pad)
      double* dst = a.y + R0 * m + (lv ? c0 + l - 1 : 0);
      if (t < a.nlev - 1 && c0 > 0) {
        const int po = (int)(R0 & 1);   // the plane whose y rows (even global row, column c0 - 1) start 8 bytes off
#pragma unroll 4
        for (int j = rr; j < 512; j += 32) {
          const int e = 2 * j + po;
          const double v = reinterpret_cast<const double*>(at_par(T, e, l >> 1))[l & 1];
          if (e < a.m) dst[(long long)e * m] = v;
        }
      } else {
        for (int e = rr; e < a.m; e += 32) {
          const double v = reinterpret_cast<const double*>(at_par(T, e, l >> 1))[l & 1];
          if (lv) dst[(long long)e * m] = v;
        }
      }
    }
#ifdef LVL4_PROF
    if (warp == 0 && lane == 0) LP_ADD(tk.kind == 0 ? 8 : 9, tc1);
#endif
    wax2::release_buffer(done + b, lane);
  }
#ifdef LVL4_PROF
  __syncwarp();
  if (warp == 0 && lane == 0 && (blockIdx.x % 37) == 0) {
    const double nb = (double)prof[10] + 1e-9, nc = (double)prof[11] + 1e-9;
    printf("lvl4 prof cta %d: total %.0f kcyc; tasks B %d C %d | per task (cyc): prod wait free %.0f dep %.0f |"
           " storer wait done %.0f busy B %.0f C %.0f | cons wait full %.0f, load lat B %.0f C %.0f, busy B %.0f C %.0f"
           " | prod slot guard %.0f\n",
           (int)blockIdx.x, (clock64() - k_t0) / 1e3, (int)prof[10], (int)prof[11], prof[0] / (nb + nc),
           prof[1] / nc, prof[2] / (nb + nc), prof[3] / nb, prof[4] / nc, prof[5] / (nb + nc), prof[6] / nb,
           prof[7] / nc, prof[8] / nb, prof[9] / nc, prof[12] / nb);
  }
#endif
}

}  // namespace lvl
}  // namespace bhcp
