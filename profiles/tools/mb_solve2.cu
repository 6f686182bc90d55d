// standalone timing of solve2_kernel (two-sided) on a synthetic banded SPD system (nb=299, BW=10)
#ifndef NOPROF
#define DBA_SOLVE_PROF
#endif
#ifndef DBA_NOPRODUCER
#define DBA_NOPRODUCER 0
#endif
#include <cstdio>
#include <vector>
#include <random>
#include <cstdlib>
#include <cmath>
#include <algorithm>
#include <cuda_runtime.h>
#include "../../paper_2411_17660_b200/csrc/dba_solve.cuh"
using namespace dba;
#if defined(NOPROF) && !defined(DBA_CRIT_PROF)
__device__ long long g_prof[16];
#endif
int main(int argc, char** argv) {
  const int nb = 299, BW = 10, W1 = BW + 1;
  std::vector<double> band((size_t)nb * W1 * 36, 0.0), rband(band.size(), 0.0), y(6 * nb + 4, 1.0);
  std::mt19937 g(0); std::normal_distribution<double> n;
  for (int a = 0; a < nb; ++a) for (int pos = 0; pos < W1; ++pos) {
    int c = a - BW + pos; if (c < 0) continue;
    for (int e = 0; e < 36; ++e) band[((size_t)a * W1 + pos) * 36 + e] = (pos == BW) ? ((e / 6 == e % 6) ? 200.0 : 0.0) : 0.5 * n(g);
  }
  for (int a = 0; a < nb; ++a) for (int pos = 0; pos < W1; ++pos) {  // reversed copy
    int c = a - BW + pos; if (c < 0) continue;
    int ar = nb - 1 - c;
    for (int r = 0; r < 6; ++r) for (int cc = 0; cc < 6; ++cc)
      rband[((size_t)ar * W1 + pos) * 36 + 6 * r + cc] = band[((size_t)a * W1 + pos) * 36 + 6 * cc + r];
  }
  double *dband, *drband, *dy, *dL, *drL, *dmid, *ddel, *dcond, *dlam; int* dst;
  cudaMalloc(&dband, band.size() * 8); cudaMalloc(&drband, band.size() * 8); cudaMalloc(&dy, y.size() * 8);
  cudaMalloc(&dL, band.size() * 8); cudaMalloc(&drL, band.size() * 8); cudaMalloc(&dmid, solve_mid_len(BW) * 8);
  cudaMalloc(&ddel, y.size() * 8); cudaMalloc(&dcond, 8); cudaMalloc(&dst, 16); cudaMalloc(&dlam, 8);
  cudaMemcpy(dband, band.data(), band.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(drband, rband.data(), band.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y.data(), y.size() * 8, cudaMemcpyHostToDevice);
  double lam = 1e-4; cudaMemcpy(dlam, &lam, 8, cudaMemcpyHostToDevice);
  SolveArgs a; a.nb = nb; a.BW = BW; a.calib = 0; a.lambda = dlam; a.status = dst; a.band = dband; a.rband = drband;
  a.theta = dband; a.thth = dband; a.y = dy; a.Lband = dL; a.rLband = drL; a.mid = dmid; a.delta = ddel; a.cond = dcond;
  a.m_top = (nb - BW) / 2;
  a.nspec = 1; a.refine = 0; a.spec_Lband = a.spec_rLband = a.spec_mid = a.spec_delta = 0; a.scalefix = 0;
  for (int k = 0; k < kMaxSpec; ++k) { a.spec_status[k] = dst; a.spec_cond[k] = dcond; }
  SolveSmem s = solve_smem_layout(nb, BW, 0);
  cudaFuncSetAttribute(solve2_kernel<2, kRing>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s.total);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int it = 0; it < (argc > 1 ? atoi(argv[1]) : 3); ++it) {
    cudaMemset(dst, 0, 16);
    long long z[16] = {0}; cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    void* args[] = {&a};
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)solve2_kernel<2, kRing>, dim3(2), dim3(kSolveThreads), args, s.total, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long pr[16]; cudaMemcpyFromSymbol(pr, g_prof, sizeof(pr));
    const int piv = a.m_top + BW;  // CTA0 forward steps incl. the middle
    printf("solve2 %.1f us   per-pivot cycles (CTA0, ~%d steps):", ms * 1e3, piv);
    const char* nm[3] = {"crit", "trail0", "stage"};
    for (int w = 0; w < 3; ++w) printf("  %s work %.0f wait %.0f", nm[w], pr[2*w] / (double)piv, pr[2*w+1] / (double)piv);
    printf("  trail panel %.0f bar %.0f\n   phases (us): fwd %.1f mid %.1f bwd %.1f  sweep: wait/row %.0f total %.1f us endsync %.1f us", pr[6] / (double)piv, pr[7] / (double)piv, pr[10] / 1965.0, pr[11] / 1965.0, pr[12] / 1965.0, pr[13] / 154.0, pr[14] / 1965.0, pr[15] / 1965.0);
    printf("\n   crit: L %.0f S11 %.0f inv %.0f export %.0f barrier %.0f\n", pr[8] / (double)piv, pr[9] / (double)piv, pr[10] / (double)piv, pr[11] / (double)piv, pr[12] / (double)piv);
  }
  // residual of the last solve: (S + lam I) x = y with S symmetric from the lower band
  std::vector<double> x(6 * nb + 4);
  cudaMemcpy(x.data(), ddel, x.size() * 8, cudaMemcpyDeviceToHost);
  double rn = 0.0, yn = 0.0;
  for (int a = 0; a < nb; ++a)
    for (int r = 0; r < 6; ++r) {
      double acc = lam * x[6 * a + r];
      for (int c = std::max(0, a - BW); c <= std::min(nb - 1, a + BW); ++c)
        for (int cc = 0; cc < 6; ++cc) {
          const double v = c <= a ? band[((size_t)a * W1 + (c - a + BW)) * 36 + 6 * r + cc]
                                  : band[((size_t)c * W1 + (a - c + BW)) * 36 + 6 * cc + r];
          acc += v * x[6 * c + cc];
        }
      rn += (acc - y[6 * a + r]) * (acc - y[6 * a + r]);
      yn += y[6 * a + r] * y[6 * a + r];
    }
  printf("relative residual %.3e\n", std::sqrt(rn / yn));
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
