// K3b: damped solve of the reduced pose (+intrinsics) system (float64).
//
// The Schur-reduced system of a covisibility graph is block-banded: a source
// frame couples the poses {i} U out(i), so with the (free-pose) ordering used
// by the plan every nonzero 6x6 block (a, c) satisfies |a - c| <= BW.  The
// intrinsics (4 rows, "global block") form a dense border that is
// eliminated last.  One CTA factors the band as a block LDL^T,
//     L_ab = S_ab D_b^-1,   S_ac -= L_ab S_cb^T,   D_b = S_bb (updated),
// with a sliding window of BW+1 block rows resident in shared memory.  D_b is
// SPD iff the damped system is; D_b^-1 comes from two 3x3 adjugate inverses
// (leading-minor test = the Cholesky pivot test), which keeps only two
// reciprocals on the pivot chain instead of six square roots.
//
// Latency engineering (the factorisation is a chain of nb dependent pivots):
//  * one critical warp (warp 7: the arbiter issues higher warp ids first, and
//    warp 3 that shares its scheduler only issues cp.async) forms the NEXT
//    pivot — L_{b+1,b}, D_{b+1}, D_{b+1}^-1 — with all 32 lanes, while 6 warps
//    apply step b's trailing update: one CTA barrier per step;
//  * rows entering the window are copied global->shared with cp.async a step
//    ahead (the damping of their diagonal block is added when it becomes a pivot);
//  * back-substitution: w_b = D_b^-1 z_b for all b in parallel, then one warp
//    sweeps b = nb-1..0 without CTA barriers, folding x_b = w_b - sum L_ab^T x_a
//    into the BW blocks above it with the next factor row prefetched from L2.
// A non-SPD pivot aborts with status 1 (the host raises lambda).
// The Cholesky pivots of the intrinsics Schur block give the A9 estimate.
#pragma once

#include "dba_common.cuh"

namespace dba {

constexpr int kSolveThreads = 256;
constexpr int kCritWarp = 7;
constexpr int kStageWarp = 3;       // shares the critical warp's scheduler; only issues cp.async
constexpr int kTrailThreads = 192;  // warps 0,1,2,4,5,6
constexpr int kMaxBand = 24;        // compiled limit on BW

#ifdef DBA_SOLVE_PROF
// clock64() phase accounting for the microbenchmark in scratch/ (not in the library build)
#define SPROF(k)                                              \
  do {                                                        \
    prof_sink += *(volatile int*)&fail;                       \
    const long long _t = clock64();                           \
    if (lane == 0 && (warp == kCritWarp || warp == 0 || warp == 3)) \
      prof_acc[k] += _t - prof_t;                             \
    prof_t = _t;                                              \
  } while (0)
__device__ long long g_prof[64];
#else
#define SPROF(k) \
  do {           \
  } while (0)
#endif

struct SolveArgs {
  int nb, BW, calib;
  double lambda;
  int* status;
  const double* band;   // nb*(BW+1)*36, block (a,c) at (a*(BW+1) + c-a+BW)*36
  const double* theta;  // nb*24 (4x6 per block)
  const double* thth;   // 16
  const double* y;      // 6 nb + 4 calib
  double* Lband;        // factor rows: L_ab at (a, c=b); slot BW holds D_a^-1
  double* delta;        // 6 nb + 4 calib
  double* cond;         // theta pivot ratio
};

struct SolveSmem {
  size_t win, th, thL, z, dinv, pbuf, cbuf, tbuf, pairs, total;
};
__host__ __device__ inline SolveSmem solve_smem_layout(int nb, int BW, int calib) {
  SolveSmem s;
  size_t o = 0;
  s.win = o; o += sizeof(double) * (size_t)(BW + 1) * (BW + 1) * 36;
  s.th = o; o += sizeof(double) * (calib ? (size_t)nb * 24 + 16 : 0);
  s.thL = o; o += sizeof(double) * (calib ? (size_t)nb * 24 : 0);
  s.z = o; o += sizeof(double) * ((size_t)6 * nb + 4);
  s.dinv = o; o += sizeof(double) * 2 * 36;
  s.pbuf = o; o += sizeof(double) * (size_t)(BW + 1) * 36;
  s.cbuf = o; o += sizeof(double) * 2 * 36;
  s.tbuf = o; o += sizeof(double) * 24;
  s.pairs = o; o += sizeof(short2) * (size_t)(BW * (BW + 1) / 2 + 1);
  s.total = (o + 15) & ~size_t(15);
  return s;
}

// inverse of a symmetric 3x3 (row-major m) via the adjugate; leading minors check SPD
__device__ __forceinline__ bool inv3_spd(const double m[9], double o[9]) {
  const double c00 = m[4] * m[8] - m[5] * m[7];
  const double c01 = m[5] * m[6] - m[3] * m[8];
  const double c02 = m[3] * m[7] - m[4] * m[6];
  const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  const double m2 = m[0] * m[4] - m[1] * m[3];
  const bool ok = (m[0] > 0.0) && (m2 > 0.0) && (det > 0.0) && isfinite(det);
  const double id = 1.0 / (ok ? det : 1.0);
  o[0] = c00 * id;
  o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  o[3] = c01 * id;
  o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  o[6] = c02 * id;
  o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  return ok;
}

// inverse of a 6x6 SPD block via [A B; B^T C]:  A^-1, T = A^-1 B, C' = C - B^T T,
// D^-1 = [A^-1 + T C'^-1 T^T, -T C'^-1; -C'^-1 T^T, C'^-1].  false if not SPD.
__device__ __forceinline__ bool inv6_spd(const double* D, double* Di) {
  double A[9], B[9], C[9], Ai[9], T[9], Cs[9], Ci[9], U[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[3 * r + c] = 0.5 * (D[6 * r + c] + D[6 * c + r]);
      B[3 * r + c] = D[6 * r + c + 3];
      C[3 * r + c] = 0.5 * (D[6 * (r + 3) + c + 3] + D[6 * (c + 3) + r + 3]);
    }
  bool ok = inv3_spd(A, Ai);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      T[3 * r + c] = Ai[3 * r] * B[c] + Ai[3 * r + 1] * B[3 + c] + Ai[3 * r + 2] * B[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Cs[3 * r + c] = C[3 * r + c] - (B[r] * T[c] + B[3 + r] * T[3 + c] + B[6 + r] * T[6 + c]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = r + 1; c < 3; ++c) {
      const double v = 0.5 * (Cs[3 * r + c] + Cs[3 * c + r]);
      Cs[3 * r + c] = v;
      Cs[3 * c + r] = v;
    }
  ok = inv3_spd(Cs, Ci) && ok;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      U[3 * r + c] = T[3 * r] * Ci[c] + T[3 * r + 1] * Ci[3 + c] + T[3 * r + 2] * Ci[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Di[6 * r + c] = Ai[3 * r + c] + U[3 * r] * T[3 * c] + U[3 * r + 1] * T[3 * c + 1] +
                      U[3 * r + 2] * T[3 * c + 2];
      Di[6 * r + c + 3] = -U[3 * r + c];
      Di[6 * (r + 3) + c] = -U[3 * c + r];
      Di[6 * (r + 3) + c + 3] = Ci[3 * r + c];
    }
  return ok;
}

// 6-vector row times the symmetric D^-1:  out[c] = sum_k v[k] Di[k][c]
__device__ __forceinline__ void row_times(const double* v, const double* Di, double* out) {
  double x[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) x[k] = v[k];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) s = fma(x[k], Di[6 * k + c], s);
    out[c] = s;
  }
}

template <int NS>  // backward-sweep prefetch slots per lane: ceil(6 BW / 32)
__global__ void __launch_bounds__(kSolveThreads, 1) solve_kernel(const SolveArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveSmem Ls = solve_smem_layout(A.nb, A.BW, A.calib);
  double* win = reinterpret_cast<double*>(smem + Ls.win);
  double* th = reinterpret_cast<double*>(smem + Ls.th);
  double* thL = reinterpret_cast<double*>(smem + Ls.thL);
  double* z = reinterpret_cast<double*>(smem + Ls.z);
  double* dinv = reinterpret_cast<double*>(smem + Ls.dinv);
  double* pbuf = reinterpret_cast<double*>(smem + Ls.pbuf);
  double* cbuf = reinterpret_cast<double*>(smem + Ls.cbuf);
  double* tbuf = reinterpret_cast<double*>(smem + Ls.tbuf);
  short2* pairs = reinterpret_cast<short2*>(smem + Ls.pairs);
  __shared__ int fail;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = A.nb, BW = A.BW, W1 = BW + 1, NR = W1 * 36;
  const double lam = A.lambda;
  const int nz = 6 * nb + (A.calib ? 4 : 0);
  const bool crit = warp == kCritWarp;
  const bool trail = (warp & 3) != 3;
  const int gt = (warp - (warp >> 2)) * 32 + lane;  // index within the trailing group
  if (tid == 0) fail = 0;
#ifdef DBA_SOLVE_PROF
  long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long prof_t = clock64();
  int prof_sink = 0;
#endif

  // ---- load: rows 0..min(BW, nb-1), theta border, rhs, pair table
  const int r0 = min(BW, nb - 1);
  for (int x = tid; x < (r0 + 1) * NR; x += kSolveThreads) {
    const int rem = x % NR, pos = rem / 36, e = rem % 36;
    double v = A.band[x];
    if (pos == BW && (e / 6) == (e % 6)) v += lam;
    win[x] = v;  // slot(a) = a for a <= BW
  }
  if (A.calib) {
    for (int x = tid; x < nb * 24; x += kSolveThreads) th[x] = A.theta[x];
    if (tid < 16) th[nb * 24 + tid] = A.thth[tid] + ((tid / 4 == tid % 4) ? lam : 0.0);
  }
  for (int x = tid; x < nz; x += kSolveThreads) z[x] = A.y[x];
  if (tid == 0) {
    int q = 0;
    for (int ao = 0; ao < BW; ++ao)
      for (int pi = 0; pi <= ao; ++pi) pairs[q++] = make_short2((short)ao, (short)pi);
  }
  __syncthreads();
  if (nb > 0 && crit && lane == 0) {
    double Di[36];
    if (!inv6_spd(win + (size_t)BW * 36, Di)) fail = 1;  // block (0,0)
    for (int x = 0; x < 36; ++x) dinv[x] = Di[x];
  }
  // rows entering the window: warp 3 issues cp.async for row b+BW+1 during step b
  auto row_stage = [&](int a, int slot) {
    if (warp != kStageWarp || a >= nb) return;
    const char* src = reinterpret_cast<const char*>(A.band + (size_t)a * NR);
    const unsigned dst = (unsigned)__cvta_generic_to_shared(win + (size_t)slot * NR);
    for (int q = lane; q < NR / 2; q += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * q), "l"(src + 16 * q));
    asm volatile("cp.async.commit_group;");
  };
  __syncthreads();

  int sb = 0;  // slot of block row b (= b % W1)
  for (int b = 0; b < nb && !fail; ++b) {
    const int amax = min(nb - 1, b + BW);
    const int na = amax - b;
    const double* Db = dinv + 36 * (b & 1);  // D_b^-1
    auto wb = [&](int a, int c) -> double* {
      int sl = sb + (a - b);
      sl = sl >= W1 ? sl - W1 : sl;
      return win + ((size_t)sl * W1 + (c - a + BW)) * 36;
    };
    const double* zb = z + 6 * b;
    SPROF(0);
    if (crit) {
      // ---- next pivot: L_{b+1,b} = S_{b+1,b} D_b^-1, D_{b+1} = S_{b+1,b+1} - L S^T, D_{b+1}^-1
      if (na > 0) {
        const double* S1 = wb(b + 1, b);
        const double* S11 = wb(b + 1, b + 1);
        for (int e = lane; e < 36; e += 32) {
          const int r = e / 6, c = e % 6;
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < 6; ++k) s = fma(S1[6 * r + k], Db[6 * k + c], s);
          cbuf[e] = s;  // L_{b+1,b}
        }
        __syncwarp();
        SPROF(1);
        double* Dn = cbuf + 36;
        const double dl = (b + 1 > BW) ? lam : 0.0;  // rows staged by cp.async carry no damping
        for (int e = lane; e < 36; e += 32) {
          const int r = e / 6, c = e % 6;
          double s = S11[e] + ((r == c) ? dl : 0.0);
#pragma unroll
          for (int k = 0; k < 6; ++k) s = fma(-cbuf[6 * r + k], S1[6 * c + k], s);
          Dn[e] = s;
        }
        if (lane < 6) {
          double s = z[6 * (b + 1) + lane];
#pragma unroll
          for (int k = 0; k < 6; ++k) s = fma(-cbuf[6 * lane + k], zb[k], s);
          z[6 * (b + 1) + lane] = s;
        }
        __syncwarp();
        SPROF(2);
        if (lane == 0) {
          double Di[36];
          if (!inv6_spd(Dn, Di)) fail = 1;
          double* Dnx = dinv + 36 * ((b + 1) & 1);
#pragma unroll
          for (int x = 0; x < 36; ++x) Dnx[x] = Di[x];
        }
      }
      SPROF(3);
      for (int e = lane; e < 36; e += 32) A.Lband[((size_t)b * W1 + BW) * 36 + e] = Db[e];
    } else if (trail) {
      // ---- panels L_ab = S_ab D_b^-1 (a in (b, amax]), L_tb = S_tb D_b^-1
      const int prow = 6 * na + (A.calib ? 4 : 0);
      for (int x = gt; x < prow; x += kTrailThreads) {
        if (x < 6 * na) {
          const int ao = x / 6, r = x % 6;
          double o[6];
          row_times(wb(b + 1 + ao, b) + 6 * r, Db, o);
          double* pb = pbuf + 36 * ao + 6 * r;
          double* lb = A.Lband + ((size_t)(b + 1 + ao) * W1 + (BW - 1 - ao)) * 36 + 6 * r;
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            pb[c] = o[c];
            lb[c] = o[c];
          }
        } else {
          const int tt = x - 6 * na;
          row_times(th + (size_t)b * 24 + 6 * tt, Db, tbuf + 6 * tt);
        }
      }
      SPROF(1);
      asm volatile("bar.sync 1, %0;" ::"n"(kTrailThreads) : "memory");
      SPROF(2);
      // ---- trailing update S_ac -= L_ab S_cb^T (except (b+1,b+1)), border, rhs
      const int npair = na * (na + 1) / 2;
      const int n1 = npair * 3;
      const int n2 = A.calib ? na * 4 : 0;
      const int n3 = A.calib ? 4 : 0;
      const int n4 = 6 * (na > 0 ? na - 1 : 0) + (A.calib ? 4 : 0);
      const int ntot = n1 + n2 + n3 + n4;
      for (int x = gt; x < ntot; x += kTrailThreads) {
        if (x < n1) {
          const int pidx = x / 3, rr = 2 * (x % 3);
          if (pidx == 0) continue;  // (b+1, b+1): critical warp
          const short2 pr = pairs[pidx];
          const int a = b + 1 + pr.x, cc = b + 1 + pr.y;
          const double* La = pbuf + 36 * pr.x + 6 * rr;
          const double2* Sc = reinterpret_cast<const double2*>(wb(cc, b));
          double2* O = reinterpret_cast<double2*>(wb(a, cc) + 6 * rr);
          double ar[2][6], o[2][6];
#pragma unroll
          for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int d = 0; d < 6; ++d) ar[r][d] = La[6 * r + d];
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const double2 v = O[q];
            o[(2 * q) / 6][(2 * q) % 6] = v.x;
            o[(2 * q + 1) / 6][(2 * q + 1) % 6] = v.y;
          }
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            double sc[6];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const double2 v = Sc[3 * c + q];
              sc[2 * q] = v.x;
              sc[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
              for (int d = 0; d < 6; ++d) o[r][c] = fma(-ar[r][d], sc[d], o[r][c]);
          }
#pragma unroll
          for (int q = 0; q < 6; ++q)
            O[q] = make_double2(o[(2 * q) / 6][(2 * q) % 6], o[(2 * q + 1) / 6][(2 * q + 1) % 6]);
        } else if (x < n1 + n2) {
          const int y2 = x - n1, co = y2 / 4, tt = y2 % 4;
          const int cc = b + 1 + co;
          const double* Lt = tbuf + 6 * tt;
          const double* Sc = wb(cc, b);
          double* O = th + (size_t)cc * 24 + 6 * tt;
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            double s = O[c];
#pragma unroll
            for (int d = 0; d < 6; ++d) s = fma(-Lt[d], Sc[6 * c + d], s);
            O[c] = s;
          }
        } else if (x < n1 + n2 + n3) {
          const int tt = x - n1 - n2;
          const double* Lt = tbuf + 6 * tt;
          double* O = th + (size_t)nb * 24 + 4 * tt;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* Su = th + (size_t)b * 24 + 6 * u;
            double s = O[u];
#pragma unroll
            for (int d = 0; d < 6; ++d) s = fma(-Lt[d], Su[d], s);
            O[u] = s;
          }
        } else {
          const int q = x - n1 - n2 - n3;
          const double* Lr;
          double* zt;
          if (q < 6 * (na - 1)) {
            Lr = pbuf + 36 + 6 * q;  // rows a >= b+2
            zt = z + 6 * (b + 2) + q;
          } else {
            const int tt = q - 6 * (na > 0 ? na - 1 : 0);
            Lr = tbuf + 6 * tt;
            zt = z + 6 * nb + tt;
          }
          double s = *zt;
#pragma unroll
          for (int d = 0; d < 6; ++d) s = fma(-Lr[d], zb[d], s);
          *zt = s;
        }
      }
      if (A.calib && gt < 24) thL[(size_t)b * 24 + gt] = tbuf[gt];  // L_tb for the backward sweep
    } else {
      // ---- warp 3: copy row b+BW+1 into row b's slot (free during step b)
      if (b + BW + 1 < nb) {
        row_stage(b + BW + 1, sb);
        asm volatile("cp.async.wait_all;" ::: "memory");
      }
    }
    SPROF(4);
    __syncthreads();
    SPROF(5);
    sb = (sb + 1 == W1) ? 0 : sb + 1;
  }
  if (fail) {
    if (tid == 0) A.status[0] = 1;
    return;
  }
  // ---- theta block: Cholesky pivots (A9), solve
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
  // ---- backward (block LDL^T): x_b = D_b^-1 z_b - L_tb^T x_t - sum_{a>b} L_ab^T x_a.
  // w_b = D_b^-1 z_b - L_tb^T x_t for all b in parallel (staged through delta), then
  // one warp sweeps b = nb-1..0 folding x_b into the BW blocks above it.
  for (int x = tid; x < 6 * nb; x += kSolveThreads) {
    const int b = x / 6, s = x % 6;
    const double* Di = A.Lband + ((size_t)b * W1 + BW) * 36 + 6 * s;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) v = fma(Di[k], z[6 * b + k], v);
    if (A.calib) {
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) v = fma(-thL[(size_t)b * 24 + 6 * tt + s], z[6 * nb + tt], v);
    }
    A.delta[x] = v;
  }
  __syncthreads();
  for (int x = tid; x < 6 * nb; x += kSolveThreads) z[x] = A.delta[x];
  __syncthreads();
  if (crit && nb > 0) {
    // register-prefetched factor row b: slot j of lane q = lane + 32 j (q < 6 BW)
    // holds column s = q % 6 of L_{b, b-1-q/6}
    double lc[NS][6], ln[NS][6];
    auto fetch = [&](int b, double (&p)[NS][6]) {
      const double* row = A.Lband + (size_t)(b < 0 ? 0 : b) * NR;
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const int q = lane + 32 * j;
        const bool ok = b >= 0 && q < 6 * BW && b - 1 - q / 6 >= 0;
        const int pos = BW - 1 - q / 6, sc = q % 6;
#pragma unroll
        for (int k = 0; k < 6; ++k) p[j][k] = ok ? row[pos * 36 + 6 * k + sc] : 0.0;
      }
    };
    fetch(nb - 1, lc);
    for (int b = nb - 1; b >= 0; --b) {
      fetch(b - 1, ln);
      double xr[6];
#pragma unroll
      for (int r = 0; r < 6; ++r) xr[r] = z[6 * b + r];
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const int q = lane + 32 * j;
        if (q < 6 * BW && b - 1 - q / 6 >= 0) {
          double acc = 0.0;
#pragma unroll
          for (int r = 0; r < 6; ++r) acc = fma(lc[j][r], xr[r], acc);
          z[6 * (b - 1 - q / 6) + q % 6] -= acc;
        }
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < NS; ++j)
#pragma unroll
        for (int k = 0; k < 6; ++k) lc[j][k] = ln[j][k];
    }
  }
  SPROF(6);
  __syncthreads();
  SPROF(7);
  for (int x = tid; x < nz; x += kSolveThreads) A.delta[x] = z[x];
#ifdef DBA_SOLVE_PROF
  if (lane == 0 && (warp == kCritWarp || warp == 0 || warp == 3)) {
    const int base = warp == kCritWarp ? 0 : (warp == 0 ? 8 : 16);
    for (int k = 0; k < 8; ++k) g_prof[base + k] = prof_acc[k] + (prof_sink == 12345);
  }
#endif
}

}  // namespace dba
