// plan.h -- host-side FFT / DST / time plans (built once, immutable afterwards).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "fft_types.h"

namespace bhcp {

// Kernel variants: threads per CTA and per-thread register capacity (complex
// values held per Stockham stage). The host picks the smallest variant whose
// CAP*T covers one sequence of the core length.
enum Variant { V256 = 0, V512 = 1, V768 = 2 };
constexpr int kVariantThreads[3] = {256, 512, 768};
constexpr int kVariantCap[3] = {16, 16, 12};

struct FftPlanHost {
  FftPlanDev d{};
  int ld = 0;           // shared-memory stride per sequence (odd -> conflict-light)
  int variant = 0;
  int cap_elems = 0;    // complex elements one CTA can transform (all stages)
  void* mem = nullptr;  // device allocation (twiddles, chirp, bhat)
  int capacity() const { return cap_elems; }
  int threads() const { return kVariantThreads[variant]; }
  // max sequences per CTA given the register capacity and a shared-memory budget
  int max_seqs(size_t smem_budget) const {
    int a = capacity() / d.Lc;
    int b = (int)(smem_budget / (size_t(ld) * sizeof(double2)));
    return a < b ? a : b;
  }
};

// Builds the plan on the current device; returns false and sets err on failure.
bool build_fft_plan(int L, FftPlanHost* out, std::string* err);
void free_fft_plan(FftPlanHost* p);

// tw (L) | chirp (n) | bhat (L) | wM (n) for the power-of-two Bluestein, n = 2^p + 1.
bool build_blue_tables(int n, std::vector<double2>* out, std::string* err);

// Rader tables for a prime n with n - 1 a power of two (see fastk::k_modes_rader):
// cplx = tw (n-1) | bhat (n-1); idx = perm (n-1) | qidx (n), perm[p] = g^p mod n,
// qidx[t] = q with g^-q = t (t >= 1), g the smallest primitive root.
bool build_rader_tables(int n, std::vector<double2>* cplx, std::vector<int>* idx, std::string* err);

// Good-Thomas / Rader tables for n = 1025 = 25 x 41 (see fastk::k_modes_gt):
// cplx = w40 (40) | w25 (25) | bhat40 (40); idx = perm (40) g^p mod 41 | tq (40) g^-q mod 41.

// Prime-factor / Rader tables for n = 4097 = 17 x 241 (see fastk::k_modes_pf):
// cplx = w240 (240) | bhat240 (240); tq (240) = g^-q mod 241; perm (240) = g^p mod 241.
// n = 1025 tables of k_modes_gt (gt_modes.cuh); offsets in double2
constexpr int kGt2Sg = 0, kGt2Tw = 1056, kGt2Gi = kGt2Tw + 1025, kGt2Bh = kGt2Gi + 1025, kGt2Total = kGt2Bh + 40;
bool build_gt2_tables(const double* shifts, const double* gaminv, std::vector<double2>* cplx, std::vector<int>* idx,
                      std::string* err);
bool build_pf_tables(std::vector<double2>* cplx, std::vector<int>* tq, std::vector<int>* perm, std::string* err);

// Upload the odd-radix codelet constants to the current device (idempotent).
bool ensure_device_constants(int device, std::string* err);

}  // namespace bhcp
