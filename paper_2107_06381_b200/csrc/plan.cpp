// plan.cpp -- host construction of FFT plans: factorisation, twiddles, and
// Bluestein chirp/filter tables, all computed in long double and rounded once.
#include "plan.h"

#include <map>
#include <mutex>

#include <cmath>
#include <complex>
#include <cstring>

namespace bhcp {

namespace {

using cld = std::complex<long double>;
const long double kPi = 3.141592653589793238462643383279502884L;

bool is_direct_prime(int p) {
  return p == 2 || p == 3 || p == 5 || p == 7 || p == 11 || p == 13 || p == 17 || p == 19 || p == 23;
}

// Factor L into Stockham radices. restricted: only {2,3,4,5} (V768 register budget).
bool factor_direct(int L, bool restricted, std::vector<int>* radices) {
  radices->clear();
  int a = 0;
  while (L % 2 == 0) { L /= 2; ++a; }
  if (restricted) {
    while (a >= 2) { radices->push_back(4); a -= 2; }
  } else {
    while (a >= 3) { radices->push_back(8); a -= 3; }
    if (a == 2) { radices->push_back(4); a = 0; }
  }
  if (a == 1) radices->push_back(2);
  for (int p = 3; L > 1; p += 2) {
    while (L % p == 0) {
      if (!is_direct_prime(p)) return false;
      if (restricted && p > 5) return false;
      radices->push_back(p);
      L /= p;
    }
    if (p > 23 && L > 1) return false;
  }
  return true;
}

bool smooth235(int n) {
  for (int p : {2, 3, 5}) while (n % p == 0) n /= p;
  return n == 1;
}

// Simple recursive mixed-radix DFT in long double (host; smooth sizes only),
// forward sign exp(-2 pi i jk / n).
void host_dft(std::vector<cld>& x) {
  const int n = (int)x.size();
  if (n <= 1) return;
  int p = 2;
  while (n % p) ++p;
  const int m = n / p;
  std::vector<std::vector<cld>> sub(p, std::vector<cld>(m));
  for (int r = 0; r < p; ++r)
    for (int j = 0; j < m; ++j) sub[r][j] = x[j * p + r];
  for (int r = 0; r < p; ++r) host_dft(sub[r]);
  for (int k = 0; k < n; ++k) {
    cld acc = 0;
    for (int r = 0; r < p; ++r) {
      long long e = ((long long)r * k) % n;
      long double ang = -2.0L * kPi * (long double)e / (long double)n;
      acc += sub[r][k % m] * cld(cosl(ang), sinl(ang));
    }
    x[k] = acc;
  }
}

double2 to_d2(cld z) { return make_double2((double)z.real(), (double)z.imag()); }

}  // namespace

int variant_capacity(const std::vector<int>& rad, int variant) {
  int c = 1 << 30;
  for (int R : rad) {
    const int s = stage_capacity(R, kVariantCap[variant]);
    if (s < c) c = s;
  }
  if (rad.empty()) c = kVariantCap[variant];
  return c * kVariantThreads[variant];
}

bool smooth23(int n) {
  for (int p : {2, 3}) while (n % p == 0) n /= p;
  return n == 1;
}

bool build_fft_plan(int L, FftPlanHost* out, std::string* err) {
  if (L < 1) { *err = "FFT length must be >= 1"; return false; }
  FftPlanHost p;
  std::vector<int> rad;
  int Lc = L;
  bool blue = false;
  bool ok = false;
  // 1) direct mixed-radix plan on a 256/512-thread CTA
  if (factor_direct(L, false, &rad)) {
    for (int v : {V256, V512}) {
      if (variant_capacity(rad, v) >= L) { p.variant = v; ok = true; break; }
    }
  }
  // 2) direct plan with the small radix set on a 768-thread CTA
  if (!ok && factor_direct(L, true, &rad) && variant_capacity(rad, V768) >= L) {
    p.variant = V768;
    ok = true;
  }
  // 3) Bluestein with a 5-smooth length, then a 3-smooth one on 768 threads
  if (!ok) {
    blue = true;
    Lc = 2 * L - 1;
    while (!smooth235(Lc)) ++Lc;
    factor_direct(Lc, false, &rad);
    for (int v : {V256, V512}) {
      if (variant_capacity(rad, v) >= Lc) { p.variant = v; ok = true; break; }
    }
    if (!ok) {
      Lc = 2 * L - 1;
      while (!smooth23(Lc)) ++Lc;
      factor_direct(Lc, true, &rad);
      if (variant_capacity(rad, V768) >= Lc) { p.variant = V768; ok = true; }
    }
  }
  if (!ok) {
    *err = "transform length " + std::to_string(L) + " is beyond the shared-memory FFT engine";
    return false;
  }
  p.cap_elems = variant_capacity(rad, p.variant);
  if ((int)rad.size() > kMaxStages) { *err = "too many FFT stages"; return false; }
  if (L == 1) rad.clear();
  p.d.L = L;
  p.d.Lc = Lc;
  p.d.blue = blue ? 1 : 0;
  p.d.nst = (int)rad.size();
  for (size_t i = 0; i < rad.size(); ++i) p.d.radix[i] = rad[i];
  p.ld = (Lc % 2 == 0) ? Lc + 1 : Lc;

  // Host tables (depend on L only: computed once per length and cached; the
  // long-double DFT of the Bluestein kernel is O(Lc^2))
  struct Tabs { std::vector<double2> tw, chirp, bhat; };
  static std::mutex tabs_mutex;
  static std::map<std::pair<int, int>, Tabs> tabs_cache;
  Tabs tb;
  {
    std::lock_guard<std::mutex> lk(tabs_mutex);
    auto it = tabs_cache.find({L, Lc});
    if (it != tabs_cache.end()) tb = it->second;
  }
  if (tb.tw.empty()) {
    tb.tw.resize(Lc);
    for (int k = 0; k < Lc; ++k) {
      long double ang = -2.0L * kPi * (long double)k / (long double)Lc;
      tb.tw[k] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    if (blue) {
      tb.chirp.resize(L);
      std::vector<cld> cl(L);
      for (int j = 0; j < L; ++j) {
        long long e = ((long long)j * j) % (2LL * L);
        long double ang = -kPi * (long double)e / (long double)L;
        cl[j] = cld(cosl(ang), sinl(ang));
        tb.chirp[j] = to_d2(cl[j]);
      }
      std::vector<cld> b(Lc, cld(0, 0));
      for (int j = 0; j < L; ++j) b[j] = std::conj(cl[j]);
      for (int j = 1; j < L; ++j) b[Lc - j] = std::conj(cl[j]);
      host_dft(b);
      tb.bhat.resize(Lc);
      for (int k = 0; k < Lc; ++k) tb.bhat[k] = to_d2(b[k] / (long double)Lc);
    }
    std::lock_guard<std::mutex> lk(tabs_mutex);
    tabs_cache[{L, Lc}] = tb;
  }
  const std::vector<double2>& tw = tb.tw;
  const std::vector<double2>& chirp = tb.chirp;
  const std::vector<double2>& bhat = tb.bhat;
  size_t bytes = (tw.size() + chirp.size() + bhat.size()) * sizeof(double2);
  cudaGetLastError();  // clear any stale error before checking our own calls
  if (cudaMalloc(&p.mem, bytes) != cudaSuccess) { *err = "cudaMalloc failed for FFT plan"; return false; }
  double2* base = (double2*)p.mem;
  cudaMemcpy(base, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice);
  p.d.tw = base;
  if (blue) {
    cudaMemcpy(base + Lc, chirp.data(), chirp.size() * sizeof(double2), cudaMemcpyHostToDevice);
    cudaMemcpy(base + Lc + L, bhat.data(), bhat.size() * sizeof(double2), cudaMemcpyHostToDevice);
    p.d.chirp = base + Lc;
    p.d.bhat = base + Lc + L;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { *err = std::string("FFT plan upload: ") + cudaGetErrorString(e); return false; }
  *out = p;
  return true;
}

// Power-of-two Bluestein tables for n = 2^p + 1 (see fastk::k_modes_blue):
// tw (L) | chirp (n) | bhat (L) | wM (n), L = 2(n-1).
bool build_blue_tables_uncached(int n, std::vector<double2>* out, std::string* err);

bool build_blue_tables(int n, std::vector<double2>* out, std::string* err) {
  static std::mutex mu;
  static std::map<int, std::vector<double2>> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(n);
    if (it != cache.end()) { *out = it->second; return true; }
  }
  if (!build_blue_tables_uncached(n, out, err)) return false;
  std::lock_guard<std::mutex> lk(mu);
  cache[n] = *out;
  return true;
}

bool build_blue_tables_uncached(int n, std::vector<double2>* out, std::string* err) {
  const int M = n - 1, L = 2 * M;
  if (M < 2 || (M & (M - 1))) { *err = "n - 1 must be a power of two"; return false; }
  out->assign(2 * L + 2 * n, make_double2(0.0, 0.0));
  double2* tw = out->data();
  double2* chirp = tw + L;
  double2* bhat = chirp + n;
  double2* wM = bhat + L;
  for (int k = 0; k < L; ++k) {
    const long double a = -2.0L * kPi * (long double)k / (long double)L;
    tw[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  std::vector<cld> cl(n);
  for (int j = 0; j < n; ++j) {
    const long long e = ((long long)j * j) % (2LL * n);
    const long double a = -kPi * (long double)e / (long double)n;
    cl[j] = cld(cosl(a), sinl(a));
    chirp[j] = to_d2(cl[j]);
    const long long f = ((long long)M * j) % n;
    const long double b = -2.0L * kPi * (long double)f / (long double)n;
    wM[j] = make_double2((double)cosl(b), (double)sinl(b));
  }
  std::vector<cld> bb(L, cld(0, 0));
  for (int d = 0; d <= M; ++d) bb[d] = std::conj(cl[d]);
  for (int d = 1; d < M; ++d) bb[L - d] = std::conj(cl[d]);
  host_dft(bb);
  for (int k = 0; k < L; ++k) bhat[k] = to_d2(bb[k] / (long double)L);
  return true;
}

bool build_rader_tables(int n, std::vector<double2>* cplx, std::vector<int>* idx, std::string* err) {
  const int NP = n - 1;
  if (n < 3 || (NP & (NP - 1))) { *err = "n - 1 must be a power of two"; return false; }
  for (int d = 2; (long long)d * d <= n; ++d)
    if (n % d == 0) { *err = "n must be prime"; return false; }
  // smallest primitive root: g^(NP/2) != 1 suffices since NP is a power of two
  auto powmod = [n](long long b, long long e) {
    long long r = 1;
    b %= n;
    while (e) { if (e & 1) r = r * b % n; b = b * b % n; e >>= 1; }
    return r;
  };
  int g = 2;
  while (powmod(g, NP / 2) == 1) ++g;
  const long long ginv = powmod(g, n - 2);
  cplx->assign(2 * NP, make_double2(0.0, 0.0));
  idx->assign(NP + n, 0);
  double2* tw = cplx->data();
  double2* bhat = tw + NP;
  int* perm = idx->data();
  int* qidx = perm + NP;
  for (int k = 0; k < NP; ++k) {
    const long double a = -2.0L * kPi * (long double)k / (long double)NP;
    tw[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  // b_m = w^(g^-m), w = exp(-2 pi i / n); bhat = DFT_NP(b) / NP
  std::vector<cld> bb(NP);
  long long gp = 1, gm = 1;
  for (int p = 0; p < NP; ++p) {
    perm[p] = (int)gp;
    qidx[gm] = p;                      // g^-p = gm
    const long double a = -2.0L * kPi * (long double)gm / (long double)n;
    bb[p] = cld(cosl(a), sinl(a));
    gp = gp * g % n;
    gm = gm * ginv % n;
  }
  host_dft(bb);
  for (int k = 0; k < NP; ++k) bhat[k] = to_d2(bb[k] / (long double)NP);
  return true;
}

// n = 1025 = 41 x 25, Cooley-Tukey with a Rader 41-point first stage (gt_modes.cuh).
// Layout (double2): sgen [8][128] shifts of the generator (beta, pencil p =
// alpha * 25 + j2: j = 25 * g^((8 alpha + 5 beta) mod 40) + j2) | y0 shifts [32]
// (j = j2) | tw [25][41] w1025^(j2 * k1(cpos)) | gi [25][41] 1/gamma_(k1(cpos) +
// 41 k2) | bh [8][5] bhat40[K], K = CRT(k1' mod 5, k2 mod 8).
// int: ck1 [41] k1 per stage-C lane position | csl [41] slot of Y(j2, k1) in a
// row | gpw [40] g^e mod 41 (generator index recovery on the singular path).
// Stage-C lane positions: 5 groups of 8 (k1 = 1..40) whose row slots are
// distinct mod 8 (conflict-free 16-byte reads), then k1 = 0 (slot 41 = y0 + A0).
bool build_gt2_tables(const double* shifts, const double* gaminv, std::vector<double2>* cplx, std::vector<int>* idx,
                      std::string* err) {
  const int p = 41, NP = 40;
  auto powmod = [p](long long b, long long e) {
    long long r = 1;
    b %= p;
    while (e) { if (e & 1) r = r * b % p; b = b * b % p; e >>= 1; }
    return r;
  };
  int g = 2;   // smallest primitive root: g^(40/2) != 1 and g^(40/5) != 1
  while (powmod(g, NP / 2) == 1 || powmod(g, NP / 5) == 1) ++g;
  const long long ginv = powmod(g, p - 2);
  cplx->assign(kGt2Total, make_double2(0.0, 0.0));
  idx->assign(41 + 41 + 40, 0);
  // generator order
  for (int beta = 0; beta < 8; ++beta)
    for (int pc = 0; pc < 125; ++pc) {
      const int alpha = pc / 25, j2 = pc % 25;
      const int j = 25 * (int)powmod(g, (8 * alpha + 5 * beta) % 40) + j2;
      (*cplx)[kGt2Sg + beta * 128 + pc] = make_double2(shifts[2 * j], shifts[2 * j + 1]);
    }
  for (int j2 = 0; j2 < 25; ++j2) (*cplx)[kGt2Sg + 1024 + j2] = make_double2(shifts[2 * j2], shifts[2 * j2 + 1]);
  // row slot of Y(j2, k1): the second FFT40's output (q1, q2) sits at 5 q2 + q1, q = (8 q1 + 5 q2) mod 40,
  // k1 = g^-q; k1 = 0 at slot 41
  std::vector<int> sigma(41, 41);
  for (int q1 = 0; q1 < 5; ++q1)
    for (int q2 = 0; q2 < 8; ++q2) {
      const int q = (8 * q1 + 5 * q2) % 40;
      sigma[powmod(ginv, q)] = 5 * q2 + q1;
    }
  // stage-C lane positions: the i-th k1 of each residue class (slot mod 8) goes to group i
  std::vector<int> ck1(41, 0);
  {
    std::vector<int> cnt(8, 0);
    for (int k1 = 1; k1 <= 40; ++k1) {
      const int r = sigma[k1] % 8;
      const int grp = cnt[r]++;
      if (grp >= 5) { *err = "gt2: slot classes unbalanced"; return false; }
      ck1[8 * grp + r] = k1;
    }
    ck1[40] = 0;
  }
  for (int c = 0; c < 41; ++c) {
    (*idx)[c] = ck1[c];
    (*idx)[41 + c] = sigma[ck1[c]];
  }
  for (int e = 0; e < 40; ++e) (*idx)[82 + e] = (int)powmod(g, e);
  for (int j2 = 0; j2 < 25; ++j2)
    for (int c = 0; c < 41; ++c) {
      const long long e = (long long)j2 * ck1[c] % 1025;
      const long double a = -2.0L * kPi * (long double)e / 1025.0L;
      (*cplx)[kGt2Tw + j2 * 41 + c] = make_double2((double)cosl(a), (double)sinl(a));
      const int t = ck1[c] + 41 * j2;   // here j2 plays k2
      (*cplx)[kGt2Gi + j2 * 41 + c] = make_double2(gaminv[2 * t], gaminv[2 * t + 1]);
    }
  // bhat40 = DFT40(b) / 40, b_m = w41^(g^-m)
  std::vector<cld> bb(NP);
  long long gm = 1;
  for (int q = 0; q < NP; ++q) {
    const long double a = -2.0L * kPi * (long double)gm / (long double)p;
    bb[q] = cld(cosl(a), sinl(a));
    gm = gm * ginv % p;
  }
  host_dft(bb);
  for (int k2 = 0; k2 < 8; ++k2)
    for (int k1 = 0; k1 < 5; ++k1) {
      int K = 0;
      while (K % 5 != k1 || K % 8 != k2) ++K;
      (*cplx)[kGt2Bh + k2 * 5 + k1] = to_d2(bb[K] / (long double)NP);
    }
  return true;
}

bool build_pf_tables(std::vector<double2>* cplx, std::vector<int>* tq, std::vector<int>* perm, std::string* err) {
  const int p = 241, NP = 240;
  auto powmod = [p](long long b, long long e) {
    long long r = 1;
    b %= p;
    while (e) { if (e & 1) r = r * b % p; b = b * b % p; e >>= 1; }
    return r;
  };
  int g = 2;   // smallest primitive root: g^(240/q) != 1 for q = 2, 3, 5
  while (powmod(g, NP / 2) == 1 || powmod(g, NP / 3) == 1 || powmod(g, NP / 5) == 1) ++g;
  const long long ginv = powmod(g, p - 2);
  cplx->assign(2 * NP, make_double2(0.0, 0.0));
  tq->assign(NP, 0);
  perm->assign(NP, 0);
  for (int k = 0; k < NP; ++k) {
    const long double a = -2.0L * kPi * (long double)k / (long double)NP;
    (*cplx)[k] = make_double2((double)cosl(a), (double)sinl(a));
  }
  std::vector<cld> bb(NP);
  long long gp = 1, gm = 1;
  for (int q = 0; q < NP; ++q) {
    (*perm)[q] = (int)gp;
    (*tq)[q] = (int)gm;
    const long double a = -2.0L * kPi * (long double)gm / (long double)p;
    bb[q] = cld(cosl(a), sinl(a));   // b_q = w241^(g^-q)
    gp = gp * g % p;
    gm = gm * ginv % p;
  }
  host_dft(bb);
  for (int k = 0; k < NP; ++k) (*cplx)[NP + k] = to_d2(bb[k] / (long double)NP);
  (void)err;
  return true;
}

void free_fft_plan(FftPlanHost* p) {
  if (p->mem) cudaFree(p->mem);
  p->mem = nullptr;
}

}  // namespace bhcp
