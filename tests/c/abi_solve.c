/* C caller of the library's ABI (no Python): a 2D pint-mqbvm solve through
 * bhcp_pint_solve against the closed-form per-mode solution (baseline.py:67-112
 * restated here with dense sine matrices), the status read-back, and the
 * BHCP_ERR_INVALID contract. Built and run by tests/test_capi_c.py. */
#include <complex.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>
#include "bhcp_b200.h"

#define M 8          /* cells per axis */
#define MI (M - 1)   /* interior points per axis */
#define NX (MI * MI)
#define NSTEPS 16
#define NL (NSTEPS + 1)

static void dst2(const double* in, double* out) {   /* orthonormal DST-I on both axes */
  double tmp[NX];
  const double s = sqrt(2.0 / M);
  for (int a = 0; a < MI; ++a)
    for (int k = 0; k < MI; ++k) {
      double acc = 0.0;
      for (int i = 0; i < MI; ++i) acc += s * sin(M_PI * (k + 1) * (i + 1) / M) * in[a * MI + i];
      tmp[a * MI + k] = acc;
    }
  for (int k = 0; k < MI; ++k)
    for (int b = 0; b < MI; ++b) {
      double acc = 0.0;
      for (int i = 0; i < MI; ++i) acc += s * sin(M_PI * (k + 1) * (i + 1) / M) * tmp[i * MI + b];
      out[k * MI + b] = acc;
    }
}

#define CHECK(x) do { int rc_ = (x); if (rc_) { fprintf(stderr, "%s -> %d (%s)\n", #x, rc_, bhcp_last_error()); return 1; } } while (0)

int main(void) {
  const double L = 1.0, T = 0.1, alpha = 1e-2;
  const double tau = T / NSTEPS, h = L / M;
  const double divisor = alpha;                 /* pint-mqbvm (methods.py:85-96) */
  const double omega = -tau / divisor;
  double mu1[MI], gam[2 * NL], gami[2 * NL], shifts[2 * NL];
  for (int k = 1; k <= MI; ++k) mu1[k - 1] = (4.0 / (h * h)) * pow(sin(k * M_PI / (2.0 * M)), 2);
  for (int t = 0; t < NL; ++t) {                /* gamma_t = omega^(t/n), principal branch */
    double complex g = cpow((double complex)omega, (double)t / NL);
    double complex gi = 1.0 / g;
    gam[2 * t] = creal(g); gam[2 * t + 1] = cimag(g);
    gami[2 * t] = creal(gi); gami[2 * t + 1] = cimag(gi);
  }
  double complex g1 = gam[2] + I * gam[3];
  for (int j = 0; j < NL; ++j) {                /* s_j = (1 - gamma_1 e^{2 pi i j / n}) / tau */
    double complex d = 1.0 - g1 * cexp(2.0 * M_PI * I * j / NL);
    shifts[2 * j] = creal(d) / tau; shifts[2 * j + 1] = cimag(d) / tau;
  }
  double g[NX];
  for (int i = 0; i < NX; ++i) g[i] = sin(0.7 * i) + 0.1 * cos(1.3 * i);

  /* closed form: y_t = DST(DST(g)_k rho_k^t / D_k), D = alpha (mu + 1/tau) + rho^N */
  double ghat[NX], ref[NL * NX];
  dst2(g, ghat);
  for (int t = 0; t < NL; ++t) {
    double amp[NX];
    for (int k1 = 0; k1 < MI; ++k1)
      for (int k2 = 0; k2 < MI; ++k2) {
        const double mu = mu1[k1] + mu1[k2], rho = 1.0 / (1.0 + tau * mu);
        const double D = alpha * (mu + 1.0 / tau) + pow(rho, NSTEPS);
        amp[k1 * MI + k2] = ghat[k1 * MI + k2] / D * pow(rho, t);
      }
    dst2(amp, ref + t * NX);
  }

  bhcp_space_plan* sp = NULL;
  bhcp_time_plan* tp = NULL;
  if (bhcp_space_plan_create(0, 4, M, mu1, &sp) != BHCP_ERR_INVALID) { fprintf(stderr, "dim 4 accepted\n"); return 1; }
  CHECK(bhcp_space_plan_create(0, 2, M, mu1, &sp));
  CHECK(bhcp_time_plan_create(0, NL, gam, gami, shifts, &tp));
  const size_t wsb = bhcp_pint_workspace_bytes(sp, tp);
  double *g_dev, *y_dev;
  void* ws;
  if (cudaMalloc((void**)&g_dev, sizeof g) || cudaMalloc((void**)&y_dev, sizeof(double) * NL * NX) ||
      cudaMalloc(&ws, wsb)) { fprintf(stderr, "cudaMalloc\n"); return 1; }
  cudaMemcpy(g_dev, g, sizeof g, cudaMemcpyHostToDevice);
  if (bhcp_pint_solve(sp, tp, g_dev, divisor, y_dev, ws, 16, NULL) != BHCP_ERR_INVALID) {
    fprintf(stderr, "short workspace accepted\n"); return 1;
  }
  CHECK(bhcp_pint_solve(sp, tp, g_dev, divisor, y_dev, ws, wsb, NULL));
  bhcp_status st;
  CHECK(bhcp_read_status(bhcp_pint_status_ptr(sp, tp, ws), 1e-8, &st, NULL));
  if (st.code != BHCP_OK || st.bad_column != -1) { fprintf(stderr, "status %d %lld\n", st.code, (long long)st.bad_column); return 1; }
  static double y[NL * NX];
  cudaMemcpy(y, y_dev, sizeof y, cudaMemcpyDeviceToHost);
  double num = 0.0, den = 0.0;
  for (int i = 0; i < NL * NX; ++i) { num += (y[i] - ref[i]) * (y[i] - ref[i]); den += ref[i] * ref[i]; }
  const double rel = sqrt(num / den);
  printf("rel-L2 vs closed form %.3e, residue %.3e of %.3e\n", rel, st.residue, st.norm);
  if (!(rel <= 1e-10)) return 1;
  bhcp_time_plan_destroy(tp);
  bhcp_space_plan_destroy(sp);
  cudaFree(g_dev); cudaFree(y_dev); cudaFree(ws);
  printf("C_ABI_OK\n");
  return 0;
}
