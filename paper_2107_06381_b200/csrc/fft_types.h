// fft_types.h -- plan descriptor shared by host planning code and kernels.
#pragma once
#include <cuda_runtime.h>

namespace bhcp {

constexpr int kMaxStages = 16;

#ifdef __CUDACC__
#define BHCP_HD __host__ __device__
#else
#define BHCP_HD
#endif

// Per-thread butterfly slots of a radix-R stage for a register budget of CAP
// complex values, and the resulting per-thread element capacity.
BHCP_HD constexpr int stage_slots(int R, int CAP) { return CAP / R > 0 ? CAP / R : 1; }
BHCP_HD constexpr int stage_capacity(int R, int CAP) { return R * stage_slots(R, CAP); }

struct FftPlanDev {
  int L;                   // logical transform length
  int Lc;                  // core (Stockham) length: L, or the Bluestein length
  int nst;                 // number of Stockham stages of the core
  int blue;                // 1 = Bluestein
  int radix[kMaxStages];   // radix of each stage (product == Lc)
  const double2* tw;       // exp(-2 pi i k / Lc), k < Lc
  const double2* chirp;    // Bluestein: exp(-i pi j^2 / L), j < L
  const double2* bhat;     // Bluestein: FFT_Lc(conj chirp filter) / Lc
};

}  // namespace bhcp
