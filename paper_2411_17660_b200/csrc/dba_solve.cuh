// K3b: damped Cholesky solve of the reduced pose (+intrinsics) system (float64).
//
// The Schur-reduced system of a covisibility graph is block-banded: a source
// frame couples the poses {i} U out(i), so with the (free-pose) ordering used
// by the plan every nonzero 6x6 block (a, c) satisfies |a - c| <= BW.  The
// intrinsics (4 rows, "global block") form a dense border that is
// eliminated last.  One CTA factors the band right-looking with a sliding
// window of BW+1 block rows resident in shared memory; the forward solve rides
// along as an extra column, the backward solve streams L from global memory
// with a one-step prefetch.  A non-positive pivot aborts with status 1 (the host
// raises lambda).  Pivot ratio of the theta block -> A9 estimate.
#pragma once

#include "dba_common.cuh"

namespace dba {

constexpr int kSolveThreads = 512;

struct SolveArgs {
  int nb, BW, calib;
  double lambda;
  int* status;
  const double* band;   // nb*(BW+1)*36, block (a,c) at (a*(BW+1) + c-a+BW)*36
  const double* theta;  // nb*24 (4x6 per block)  [+16 theta-theta after]
  const double* thth;   // 16
  const double* y;      // 6 nb + 4 calib
  double* Lband;        // output factor rows (same layout as band)
  double* delta;        // 6 nb + 4 calib
  double* cond;         // theta pivot ratio
};

struct SolveSmem {
  size_t win, th, z, lbb, total;
};
__host__ __device__ inline SolveSmem solve_smem_layout(int nb, int BW, int calib) {
  SolveSmem s;
  size_t o = 0;
  s.win = o; o += sizeof(double) * (size_t)(BW + 1) * (BW + 1) * 36;
  s.th = o; o += sizeof(double) * (calib ? (size_t)nb * 24 + 16 : 0);
  s.z = o; o += sizeof(double) * ((size_t)6 * nb + 4);
  s.lbb = o; o += sizeof(double) * 48;
  s.total = o;
  return s;
}

__device__ __forceinline__ double* win_block(double* win, int BW, int a, int c) {
  return win + ((size_t)(a % (BW + 1)) * (BW + 1) + (c - a + BW)) * 36;
}

__global__ void __launch_bounds__(kSolveThreads, 1) solve_kernel(const SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveSmem Ls = solve_smem_layout(A.nb, A.BW, A.calib);
  double* win = reinterpret_cast<double*>(smem + Ls.win);
  double* th = reinterpret_cast<double*>(smem + Ls.th);
  double* z = reinterpret_cast<double*>(smem + Ls.z);
  double* lbb = reinterpret_cast<double*>(smem + Ls.lbb);  // 36 L_bb + 6 1/diag
  __shared__ int fail;
  const int tid = threadIdx.x, nb = A.nb, BW = A.BW, W1 = BW + 1;
  const double lam = A.lambda;
  const int nz = 6 * nb + (A.calib ? 4 : 0);
  if (tid == 0) fail = 0;

  // ---- load: rows 0..min(BW, nb-1), theta border, rhs
  const int r0 = min(BW, nb - 1);
  for (int x = tid; x < (r0 + 1) * W1 * 36; x += kSolveThreads) {
    const int a = x / (W1 * 36), rem = x % (W1 * 36), pos = rem / 36, e = rem % 36;
    double v = A.band[(size_t)a * W1 * 36 + rem];
    if (pos == BW && (e / 6) == (e % 6)) v += lam;
    win[((size_t)(a % W1) * W1 + pos) * 36 + e] = v;
  }
  if (A.calib) {
    for (int x = tid; x < nb * 24; x += kSolveThreads) th[x] = A.theta[x];
    if (tid < 16) th[nb * 24 + tid] = A.thth[tid] + ((tid / 4 == tid % 4) ? lam : 0.0);
  }
  for (int x = tid; x < nz; x += kSolveThreads) z[x] = A.y[x];
  __syncthreads();

  for (int b = 0; b < nb; ++b) {
    const int amax = min(nb - 1, b + BW);
    const int na = amax - b;
    // (1) factor the diagonal block, forward-substitute z_b
    if (tid == 0) {
      double* D = win_block(win, BW, b, b);
      double L[36];
      for (int x = 0; x < 36; ++x) L[x] = 0.0;
      bool ok = true;
      for (int c = 0; c < 6; ++c) {
        double s = D[6 * c + c];
        for (int d = 0; d < c; ++d) s -= L[6 * c + d] * L[6 * c + d];
        if (!(s > 0.0) || !isfinite(s)) ok = false;
        const double l = sqrt(fmax(s, 1e-300));
        L[6 * c + c] = l;
        const double il = 1.0 / l;
        for (int r = c + 1; r < 6; ++r) {
          double t = D[6 * r + c];
          for (int d = 0; d < c; ++d) t -= L[6 * r + d] * L[6 * c + d];
          L[6 * r + c] = t * il;
        }
      }
      for (int x = 0; x < 36; ++x) lbb[x] = L[x];
      for (int c = 0; c < 6; ++c) lbb[36 + c] = 1.0 / L[6 * c + c];
      double* zb = z + 6 * b;
      for (int c = 0; c < 6; ++c) {
        double s = zb[c];
        for (int d = 0; d < c; ++d) s -= L[6 * c + d] * zb[d];
        zb[c] = s * lbb[36 + c];
      }
      if (!ok) fail = 1;
    }
    __syncthreads();
    if (fail) break;
    // (2) panel L_ab = S_ab L_bb^-T (thread per scalar row) + write row b of L
    const int prow = 6 * na + (A.calib ? 4 : 0);
    for (int x = tid; x < prow; x += kSolveThreads) {
      double* row;
      if (x < 6 * na) {
        const int a = b + 1 + x / 6;
        row = win_block(win, BW, a, b) + 6 * (x % 6);
      } else {
        row = th + (size_t)b * 24 + 6 * (x - 6 * na);
      }
      double v[6];
      for (int c = 0; c < 6; ++c) v[c] = row[c];
      for (int c = 0; c < 6; ++c) {
        double s = v[c];
        for (int d = 0; d < c; ++d) s -= v[d] * lbb[6 * c + d];
        v[c] = s * lbb[36 + c];
      }
      for (int c = 0; c < 6; ++c) row[c] = v[c];
    }
    for (int x = tid; x < W1 * 36; x += kSolveThreads) {
      const int pos = x / 36, e = x % 36;
      const int c = b - BW + pos;
      double v = 0.0;
      if (c >= 0) v = (pos == BW) ? lbb[e] : win_block(win, BW, b, c)[e];
      A.Lband[(size_t)b * W1 * 36 + x] = v;
    }
    __syncthreads();
    // (3) trailing update of the window + border + rhs, and load row b+BW+1
    {
      const int npair = na * (na + 1) / 2;
      const int n1 = npair * 36;
      const int n2 = A.calib ? na * 24 : 0;
      const int n3 = A.calib ? 16 : 0;
      const int n4 = 6 * na + (A.calib ? 4 : 0);
      const int nl = (b + BW + 1 < nb) ? W1 * 36 : 0;
      const int ntot = n1 + n2 + n3 + n4 + nl;
      const double* zb = z + 6 * b;
      for (int x = tid; x < ntot; x += kSolveThreads) {
        if (x < n1) {
          int pi = x / 36;
          const int e = x % 36, r = e / 6, c = e % 6;
          int ao = 0;
          while (pi > ao) {
            pi -= ao + 1;
            ++ao;
          }
          const int a = b + 1 + ao, cc = b + 1 + pi;  // cc <= a
          const double* La = win_block(win, BW, a, b) + 6 * r;
          const double* Lc = win_block(win, BW, cc, b) + 6 * c;
          double s = 0.0;
          for (int d = 0; d < 6; ++d) s += La[d] * Lc[d];
          win_block(win, BW, a, cc)[e] -= s;
        } else if (x < n1 + n2) {
          const int y2 = x - n1, co = y2 / 24, e = y2 % 24, t = e / 6, c = e % 6;
          const int cc = b + 1 + co;
          const double* Lt = th + (size_t)b * 24 + 6 * t;
          const double* Lc = win_block(win, BW, cc, b) + 6 * c;
          double s = 0.0;
          for (int d = 0; d < 6; ++d) s += Lt[d] * Lc[d];
          th[(size_t)cc * 24 + e] -= s;
        } else if (x < n1 + n2 + n3) {
          const int e = x - n1 - n2, t = e / 4, u = e % 4;
          const double* Lt = th + (size_t)b * 24 + 6 * t;
          const double* Lu = th + (size_t)b * 24 + 6 * u;
          double s = 0.0;
          for (int d = 0; d < 6; ++d) s += Lt[d] * Lu[d];
          th[(size_t)nb * 24 + e] -= s;
        } else if (x < n1 + n2 + n3 + n4) {
          const int q = x - n1 - n2 - n3;
          const double* Lr;
          double* zt;
          if (q < 6 * na) {
            Lr = win_block(win, BW, b + 1 + q / 6, b) + 6 * (q % 6);
            zt = z + 6 * (b + 1) + q;
          } else {
            Lr = th + (size_t)b * 24 + 6 * (q - 6 * na);
            zt = z + 6 * nb + (q - 6 * na);
          }
          double s = 0.0;
          for (int d = 0; d < 6; ++d) s += Lr[d] * zb[d];
          *zt -= s;
        } else {
          const int q = x - n1 - n2 - n3 - n4, pos = q / 36, e = q % 36;
          const int a = b + BW + 1;
          double v = A.band[(size_t)a * W1 * 36 + q];
          if (pos == BW && (e / 6) == (e % 6)) v += lam;
          win[((size_t)(a % W1) * W1 + pos) * 36 + e] = v;
        }
      }
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) A.status[0] = 1;
    return;
  }
  // ---- theta block: factor, forward, condition estimate, backward
  if (A.calib && tid == 0) {
    double* T = th + (size_t)nb * 24;
    double L[16];
    bool ok = true;
    double pmax = 0.0, pmin = 1e300;
    for (int x = 0; x < 16; ++x) L[x] = 0.0;
    for (int c = 0; c < 4; ++c) {
      double s = T[4 * c + c];
      for (int d = 0; d < c; ++d) s -= L[4 * c + d] * L[4 * c + d];
      if (!(s > 0.0) || !isfinite(s)) ok = false;
      pmax = fmax(pmax, s);
      pmin = fmin(pmin, s);
      const double l = sqrt(fmax(s, 1e-300));
      L[4 * c + c] = l;
      for (int r = c + 1; r < 4; ++r) {
        double t = T[4 * r + c];
        for (int d = 0; d < c; ++d) t -= L[4 * r + d] * L[4 * c + d];
        L[4 * r + c] = t / l;
      }
    }
    double* zt = z + 6 * nb;
    for (int c = 0; c < 4; ++c) {
      double s = zt[c];
      for (int d = 0; d < c; ++d) s -= L[4 * c + d] * zt[d];
      zt[c] = s / L[4 * c + c];
    }
    for (int c = 3; c >= 0; --c) {
      double s = zt[c];
      for (int d = c + 1; d < 4; ++d) s -= L[4 * d + c] * zt[d];
      zt[c] = s / L[4 * c + c];
    }
    A.cond[0] = pmax / fmax(pmin, 1e-300);
    if (!ok) fail = 1;
  }
  __syncthreads();
  if (fail) {
    if (tid == 0) A.status[0] = 1;
    return;
  }
  // ---- backward: x_b = L_bb^-T (z_b - sum_a L_ab^T x_a - L_tb^T x_t), z overwritten by x
  __shared__ double tmp[8];
  const int warp = tid >> 5, lane = tid & 31;
  double Lv[3] = {0.0, 0.0, 0.0};
  auto fetch = [&](int b, double (&out)[3]) {
    if (warp >= 6 || b < 0) return;
    const int na = min(nb - 1, b + BW) - b;
    const int nterm = 6 * na + (A.calib ? 4 : 0);
    for (int s = 0; s < 3; ++s) {
      const int tau = lane + 32 * s;
      double v = 0.0;
      if (tau < 6 * na) {
        const int a = b + 1 + tau / 6, r = tau % 6;
        v = A.Lband[((size_t)a * W1 + (b - a + BW)) * 36 + 6 * r + warp];
      } else if (tau < nterm) {
        v = th[(size_t)b * 24 + 6 * (tau - 6 * na) + warp];
      }
      out[s] = v;
    }
  };
  fetch(nb - 1, Lv);
  for (int b = nb - 1; b >= 0; --b) {
    double Ln[3] = {0.0, 0.0, 0.0};
    fetch(b - 1, Ln);
    if (warp < 6) {
      const int na = min(nb - 1, b + BW) - b;
      double s = 0.0;
      for (int q = 0; q < 3; ++q) {
        const int tau = lane + 32 * q;
        double xv = 0.0;
        if (tau < 6 * na)
          xv = z[6 * (b + 1) + tau];
        else if (tau < 6 * na + (A.calib ? 4 : 0))
          xv = z[6 * nb + tau - 6 * na];
        s += Lv[q] * xv;
      }
      for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) tmp[warp] = s;
    }
    __syncthreads();
    if (tid == 0) {
      const double* D = A.Lband + ((size_t)b * W1 + BW) * 36;
      double v[6];
      for (int c = 0; c < 6; ++c) v[c] = z[6 * b + c] - tmp[c];
      for (int c = 5; c >= 0; --c) {
        double s = v[c];
        for (int d = c + 1; d < 6; ++d) s -= D[6 * d + c] * v[d];
        v[c] = s / D[6 * c + c];
      }
      for (int c = 0; c < 6; ++c) z[6 * b + c] = v[c];
    }
    __syncthreads();
    for (int q = 0; q < 3; ++q) Lv[q] = Ln[q];
  }
  for (int x = tid; x < nz; x += kSolveThreads) A.delta[x] = z[x];
}

}  // namespace dba
