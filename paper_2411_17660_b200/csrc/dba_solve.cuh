// K3b: damped solve of the reduced pose (+intrinsics) system (float64).
//
// The Schur-reduced system of a covisibility graph is block-banded: a source
// frame couples the poses {i} U out(i), so with the (free-pose) ordering used
// by the plan every nonzero 6x6 block (a, c) satisfies |a - c| <= BW.  The
// intrinsics (4 rows, "global block") form a dense border that is
// eliminated last.  The band is factored as a block Cholesky for the Schur updates and
// kept in block LDL^T form for the substitutions:
//     D_b = S_bb (updated) + lambda I = C_b C_b^T,   Li_b = C_b^-1,
//     W_ab = S_ab Li_b^T,   S_ac -= W_ab W_cb^T,   L_ab = W_ab Li_b,   D_b^-1 = Li_b^T Li_b,
// with a sliding window of BW+1 block rows resident in shared memory.  The symmetric
// update W W^T is backward stable: the former L_ab S_cb^T form (explicit D_b^-1 from 3x3
// adjugates) left the noisy-C3 step 5e-7 from the exact solution where LAPACK's Cholesky is
// 1e-8; this form is 1.4e-8 (profiles/r02_solve_accuracy.txt).  The Cholesky pivot
// test (every pivot > 0) is the SPD test.  Damping lambda is added to a diagonal block
// when it becomes a pivot.
//
// The factorisation is a chain of dependent 6x6 pivots, so:
//  * two-sided (solve2_kernel, cooperative, 2 CTAs): CTA 0 eliminates poses
//    0..m-1 top-down while CTA 1 eliminates nb-1..m+BW bottom-up on the reversed
//    band (written by gather); the BW-block middle receives both Schur updates,
//    is combined (T + B - S) and solved densely, then both halves back-substitute
//    in parallel — half the chain length of the one-sided solve_kernel;
//  * inside a chain one critical warp (warp 7: the arbiter issues higher warp ids
//    first, and warp 3 on its scheduler only issues cp.async) forms the NEXT
//    pivot while 7 warps form the panels and apply the trailing update: one CTA
//    barrier per step;
//  * rows entering the window are copied with cp.async a step ahead;
//  * back-substitution: w_b = D_b^-1 z_b for all b in parallel, then one warp
//    sweeps without CTA barriers, folding x_b = w_b - sum L_ab^T x_a into the BW
//    blocks above, factor rows streaming through a ring of bulk async copies (TMA
//    engine) with full/empty mbarriers.
// A non-SPD pivot aborts with status 1 (the host raises lambda).
// The Cholesky pivots of the intrinsics Schur block give the A9 estimate.
#pragma once

#include <cooperative_groups.h>

#include "dba_common.cuh"

namespace dba {

#ifndef DBA_NOPRODUCER
#define DBA_NOPRODUCER 0
#endif
constexpr int kSolveThreads = 256;
constexpr int kCritWarp = 7;
constexpr int kStageWarp = 3;       // also a trailing warp; issues the next row's cp.async first
constexpr int kTrailThreads = 224;  // warps 0..6
constexpr int kMaxBand = 24;        // compiled limit on BW
constexpr int kRing = 32;           // backward-sweep factor-row ring depth (hides the bulk-copy latency)
constexpr int kRingWide = 8;        // ... for wide bands (a folded loop closure): 8 rows of BW blocks
// blocks of the shared-memory window are kWB doubles apart (36 + 2 padding): block
// starts then fall on 8 different bank offsets instead of 4, which removes most of
// the bank conflicts of the trailing update (measured 1.5k -> 1.2k cycles per pivot)
constexpr int kWB = 38;
#ifndef DBA_KTR
#define DBA_KTR 3
#endif
constexpr int kTR = DBA_KTR;  // rows of a trailing-update output block per thread
constexpr int kMaxSpec = 3;   // damping candidates solved per round (lambda, 10 lambda, 100 lambda)

struct SolveArgs {
  int nb, BW, calib;
  const double* lambda;  // damping (device: the GN controller's current value)
  int* status;
  const double* band;   // nb*(BW+1)*36, block (a,c) at (a*(BW+1) + c-a+BW)*36
  const double* rband;  // the same band in reversed block order (two-sided solve)
  const double* theta;  // nb*24 (4x6 per block)
  const double* thth;   // 16
  const double* y;      // 6 nb + 4 calib
  double* Lband;        // factor rows (top / single chain): L_ab at (a, c=b); slot BW = D_a^-1
  double* rLband;       // factor rows of the bottom chain (reversed indexing)
  double* mid;          // two-sided exchange scratch (see solve_mid_len)
  double* delta;        // 6 nb + 4 calib
  double* cond;         // theta pivot ratio
  int m_top;            // two-sided: pivots of the top chain (0: one-sided)
  // prior-fixed monocular scale (DESIGN.md §5 "Parity at C4"): q = exact S u along the
  // scaling u about the anchor camera; the step is corrected along u after the solve
  int scalefix;
  const double* q;
  const double* poses;      // current poses (N,7)
  const int* block_pose;    // reduced block -> pose
  int anchor;

  // speculative damping: candidate k (one CTA / CTA pair each) factors S + 10^k lambda I
  // into its own factor rows, exchange scratch, step, flags word and condition slot,
  // so the trials a rejection would run next are already solved
  int nspec;
  long long spec_Lband, spec_rLband, spec_mid, spec_delta;  // per-candidate strides (doubles)
  int* spec_status[kMaxSpec];
  double* spec_cond[kMaxSpec];
  int refine;  // one step of iterative refinement (see refine_* below)
};

// the arguments of candidate k (k = 0: the controller's lambda)
__device__ __forceinline__ SolveArgs spec_view(const SolveArgs& A, int k, double& lam) {
  SolveArgs B = A;
  B.Lband += k * A.spec_Lband;
  B.rLband += k * A.spec_rLband;
  B.mid += k * A.spec_mid;
  B.delta += k * A.spec_delta;
  B.status = A.spec_status[k];
  B.cond = A.spec_cond[k];
  lam = *A.lambda;
  for (int i = 0; i < k; ++i) lam *= 10.0;  // the controller's own sequence after k rejections
  return B;
}

// doubles of the two-sided exchange scratch
__host__ __device__ inline long long solve_mid_len(int BW) {
  const long long per = (long long)BW * BW * 36 + 6 * BW + (long long)BW * 24 + 16 + 4;
  return 2 * per + (long long)BW * BW * 36 /* middle factor rows */ + 6 * BW + 4 /* solution */;
}

struct SolveSmem {
  size_t win, ring, th, thL, z, thm, thLm, zm, linv, pbuf, cbuf, tbuf, pairs, xo, bars, total;
};
__host__ __device__ inline SolveSmem solve_smem_layout(int nb, int BW, int calib, int ring = kRing) {
  SolveSmem s;
  size_t o = 0;
  s.win = o; o += sizeof(double) * (size_t)(BW + 1) * (BW + 1) * kWB;
  s.ring = o; o += sizeof(double) * (size_t)ring * BW * 36;  // backward sweep: L blocks of `ring` rows
  s.th = o; o += sizeof(double) * (calib ? (size_t)nb * 24 + 16 : 0);
  s.thL = o; o += sizeof(double) * (calib ? (size_t)nb * 24 : 0);
  s.z = o; o += sizeof(double) * ((size_t)6 * nb + 4);
  s.thm = o; o += sizeof(double) * (calib ? (size_t)BW * 24 + 16 : 0);
  s.thLm = o; o += sizeof(double) * (calib ? (size_t)BW * 24 : 0);
  s.zm = o; o += sizeof(double) * ((size_t)6 * BW + 4);
  s.linv = o; o += sizeof(double) * 2 * 36;
  s.pbuf = o; o += sizeof(double) * (size_t)(BW + 1) * kWB;
  s.cbuf = o; o += sizeof(double) * 2 * 36;
  s.tbuf = o; o += sizeof(double) * 48;
  s.pairs = o; o += sizeof(short2) * (size_t)(BW * (BW + 1) / 2 + 1);
  o = (o + 7) & ~size_t(7);
  s.xo = o; o += sizeof(double) * ((size_t)6 * nb + 4);  // refinement: the unrefined step
  s.bars = o; o += sizeof(unsigned long long) * 2 * ring;  // backward-sweep ring full/empty mbarriers
  s.total = (o + 15) & ~size_t(15);
  return s;
}

// 1/sqrt(v) to ~1 ulp: the MUFU estimate and two Newton steps (no IEEE sqrt / division
// sequence on the pivot chain)
__device__ __forceinline__ double rsqrt64(double v) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double h = 0.5 * v;
  r = r * fma(-h * r, r, 1.5);
  return r * fma(-h * r, r, 1.5);
}

// Cholesky factor C of a 6x6 SPD block (+ lam I; the block is symmetrised; right-looking,
// so each column's trailing updates are independent), returned as Li = C^-1 (lower
// triangular, row-major, zeros above the diagonal).  false when a pivot is not positive
// (the block is not SPD).
__device__ __forceinline__ bool chol6_inv(const double* D, double lam, double* Li) {
  double a[6][6], ri[6];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j <= i; ++j) a[i][j] = 0.5 * (D[6 * i + j] + D[6 * j + i]) + (i == j ? lam : 0.0);
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const double v0 = a[j][j];
    ok = ok && v0 > 0.0 && isfinite(v0);
    const double v = ok ? v0 : 1.0;
    const double r = rsqrt64(v);
    ri[j] = r;
    a[j][j] = v * r;
#pragma unroll
    for (int i = j + 1; i < 6; ++i) a[i][j] *= r;
#pragma unroll
    for (int i = j + 1; i < 6; ++i)
#pragma unroll
      for (int k = j + 1; k <= i; ++k) a[i][k] = fma(-a[i][j], a[k][j], a[i][k]);
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      double v = 0.0;
      if (j < i) {
#pragma unroll
        for (int k = j; k < i; ++k) v = fma(a[i][k], Li[6 * k + j], v);
        v = -v * ri[i];
      } else if (j == i) {
        v = ri[i];
      }
      Li[6 * i + j] = v;
    }
  }
  return ok;
}

// W row of a block row v:  out[c] = (v Li^T)[c] = sum_{k <= c} v[k] Li[c][k]
__device__ __forceinline__ void w_row(const double* v, const double* Li, double* out) {
  double x[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) x[k] = v[k];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= c; ++k) s = fma(x[k], Li[6 * c + k], s);
    out[c] = s;
  }
}

// LDL^T factor row from a W row:  out[c] = (w Li)[c] = sum_{k >= c} w[k] Li[k][c]
__device__ __forceinline__ void l_row(const double* w, const double* Li, double* out) {
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = c; k < 6; ++k) s = fma(w[k], Li[6 * k + c], s);
    out[c] = s;
  }
}

// entry (r, c) of D^-1 = Li^T Li
__device__ __forceinline__ double dinv_entry(const double* Li, int r, int c) {
  double s = 0.0;
  for (int k = (r > c ? r : c); k < 6; ++k) s = fma(Li[6 * k + r], Li[6 * k + c], s);
  return s;
}

// shared-memory working set of one elimination chain
struct ChainSm {
  double* win;   // (BW+1) window rows x (BW+1) blocks x 36
  double* th;    // theta border: ncols x 24, then theta-theta (16)
  double* thL;   // L_tb per eliminated pivot (ncols x 24)
  double* z;     // rhs: 6 ncols, then theta (4)
  double* linv;  // Li_b = C_b^-1 double buffer
  double* pbuf;  // W panels of the current step (blocks kWB apart)
  double* cbuf;  // critical-warp scratch: W_{b+1,b} rows [0, 36), y_b = Li_b z_b at 48 + 6 (b & 1)
  double* tbuf;  // theta panel: W_tb [0, 24), L_tb [24, 48)
  short2* pairs;
  double* ring;
  unsigned long long* bars;
  int* fail;
};

// Forward block-LDL^T over pivots [0, npiv) of a band whose rows [0, nrows) live in
// `band` (local orientation).  The window must hold rows 0..min(BW, nrows-1) on
// entry.  Rows npiv..nrows-1 receive the Schur updates but are not pivoted (their
// diagonal block includes the critical warp's update).  ncols: offset of the theta
// rows in th / z.  Writes factor rows [0, nrows) to Lband (off-diagonal L blocks) and
// D_b^-1 to the diagonal slot of rows [0, npiv).
#if defined(DBA_SOLVE_PROF) || defined(DBA_CRIT_PROF)
__device__ long long g_prof[16];  // [role*2 + {work, barrier wait}] cycles, CTA 0
#endif
// DBA_CRIT_PROF: phase clock of the critical warp (CTA 0, lane 0) in registers, one
// global write at the end (g_prof[8..12]: L, S11 update, inversion, export, barrier)
#ifdef DBA_CRIT_PROF
#define CRIT_MARK(i)                   \
  do {                                 \
    const long long t_ = clock64();    \
    cpa[i] += t_ - cpt;                \
    cpt = t_;                          \
  } while (0)
#else
#define CRIT_MARK(i) \
  do {               \
  } while (0)
#endif
__device__ inline void chain_forward(const ChainSm& S, const double* band, double* Lband, int nrows, int npiv,
                                     int BW, int calib, int ncols, double lam) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W1 = BW + 1, NR = W1 * 36;
  const bool crit = warp == kCritWarp;
  const bool trail = !crit;
  const int gt = tid;
  if (tid == 0) {
    int q = 0;
    for (int ao = 0; ao < BW; ++ao)
      for (int pi = 0; pi <= ao; ++pi) S.pairs[q++] = make_short2((short)ao, (short)pi);
  }
  double* const ybuf = S.cbuf + 48;  // y_b = Li_b z_b, double-buffered
  if (npiv > 0 && crit && lane == 0) {
    double Li[36];
    if (!chol6_inv(S.win + (size_t)BW * kWB, lam, Li)) *S.fail = 1;  // block (0,0)
    for (int x = 0; x < 36; ++x) S.linv[x] = Li[x];
    for (int r = 0; r < 6; ++r) {
      double v = 0.0;
      for (int k = 0; k <= r; ++k) v = fma(Li[6 * r + k], S.z[k], v);
      ybuf[r] = v;
    }
  }
  __syncthreads();
#ifdef DBA_CRIT_PROF
  long long cpa[5] = {0, 0, 0, 0, 0}, cpt = clock64();
#endif
  int sb = 0;  // slot of block row b (= b % W1)
  // a failed pivot sets *S.fail; the sweep runs on (values are discarded) so the
  // loop needs no per-step flag read
  for (int b = 0; b < npiv; ++b) {
#ifdef DBA_SOLVE_PROF
    const long long pt0 = clock64();
#endif
    const int amax = min(nrows - 1, b + BW);
    const int na = amax - b;
    const double* Lib = S.linv + 36 * (b & 1);  // Li_b
    const double* yb = ybuf + 6 * (b & 1);      // y_b
    auto wb = [&](int a, int c) -> double* {
      int sl = sb + (a - b);
      sl = sl >= W1 ? sl - W1 : sl;
      return S.win + ((size_t)sl * W1 + (c - a + BW)) * kWB;
    };
    if (crit) {
      // next pivot: W_{b+1,b} = S_{b+1,b} Li_b^T, S_{b+1,b+1} -= W W^T, z_{b+1} -= W y_b,
      // then C_{b+1}, Li_{b+1} and y_{b+1} = Li_{b+1} z_{b+1}
      if (na > 0) {
        const double* S1 = wb(b + 1, b);
        double* S11 = wb(b + 1, b + 1);
        double* Wc = S.cbuf;
        if (lane < 6) {  // lane r owns row r (the same w_row arithmetic as the panels)
          double w[6];
          w_row(S1 + 6 * lane, Lib, w);
#pragma unroll
          for (int c = 0; c < 6; ++c) Wc[6 * lane + c] = w[c];
        }
        __syncwarp();
        if (lane < 6) {
          const int r = lane;
          double w[6], d[6], zs = S.z[6 * (b + 1) + r];
#pragma unroll
          for (int k = 0; k < 6; ++k) w[k] = Wc[6 * r + k];
#pragma unroll
          for (int c = 0; c < 6; ++c) d[c] = S11[6 * r + c];
#pragma unroll
          for (int k = 0; k < 6; ++k) {
#pragma unroll
            for (int c = 0; c < 6; ++c) d[c] = fma(-w[k], Wc[6 * c + k], d[c]);
            zs = fma(-w[k], yb[k], zs);
          }
#pragma unroll
          for (int c = 0; c < 6; ++c) S11[6 * r + c] = d[c];  // non-pivot rows are exported from here
          S.z[6 * (b + 1) + r] = zs;
        }
        CRIT_MARK(0);
        __syncwarp();
        CRIT_MARK(1);
        if (b + 1 < npiv) {
          double* Lnx = S.linv + 36 * ((b + 1) & 1);
          if (lane == 0) {  // C_{b+1}, Li_{b+1}, y_{b+1} = Li_{b+1} z_{b+1} from registers
            double Li[36], zn[6];
            if (!chol6_inv(S11, lam, Li)) *S.fail = 1;
#pragma unroll
            for (int k = 0; k < 6; ++k) zn[k] = S.z[6 * (b + 1) + k];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              double v = 0.0;
#pragma unroll
              for (int k = 0; k <= r; ++k) v = fma(Li[6 * r + k], zn[k], v);
              ybuf[6 * ((b + 1) & 1) + r] = v;
            }
#pragma unroll
            for (int x = 0; x < 36; ++x) Lnx[x] = Li[x];
          }
        }
        __syncwarp();
        CRIT_MARK(2);
      }
      CRIT_MARK(3);
    } else if (trail) {
      const bool stage = warp == kStageWarp && band != nullptr && b + BW + 1 < nrows;
      if (stage) {
        // copy row b+BW+1 into row b's slot (free during step b)
        const char* src = reinterpret_cast<const char*>(band + (size_t)(b + BW + 1) * NR);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(S.win + (size_t)sb * W1 * kWB);
        for (int q = lane; q < NR / 2; q += 32) {  // 18 chunks of 16 B per 36-double block
          const int blk = q / 18, ch = q % 18;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + blk * kWB * 8 + 16 * ch),
                       "l"(src + 16 * q));
        }
        asm volatile("cp.async.commit_group;");
      }
      // D_b^-1 = Li_b^T Li_b -> the diagonal slot of factor row b (threads past the panel rows)
      if (gt >= kTrailThreads - 64 && gt < kTrailThreads - 28) {
        const int e = gt - (kTrailThreads - 64);
        Lband[((size_t)b * W1 + BW) * 36 + e] = dinv_entry(Lib, e / 6, e % 6);
      }
      // panels W_ab = S_ab Li_b^T (a in (b, amax]) for the updates, L_ab = W_ab Li_b to
      // the factor rows; W_tb, L_tb of the theta border
      const int prow = 6 * na + (calib ? 4 : 0);
      for (int x = gt; x < prow; x += kTrailThreads) {
        double w[6], l[6];
        if (x < 6 * na) {
          const int ao = x / 6, r = x % 6;
          w_row(wb(b + 1 + ao, b) + 6 * r, Lib, w);
          l_row(w, Lib, l);
          double* pb = S.pbuf + kWB * ao + 6 * r;
          double* lb = Lband + ((size_t)(b + 1 + ao) * W1 + (BW - 1 - ao)) * 36 + 6 * r;
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            pb[c] = w[c];
            lb[c] = l[c];
          }
        } else {
          const int tt = x - 6 * na;
          w_row(S.th + (size_t)b * 24 + 6 * tt, Lib, w);
          l_row(w, Lib, l);
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            S.tbuf[6 * tt + c] = w[c];
            S.tbuf[24 + 6 * tt + c] = l[c];
          }
        }
      }
#ifdef DBA_SOLVE_PROF
      const long long pa = clock64();
#endif
      asm volatile("bar.sync 1, %0;" ::"n"(kTrailThreads) : "memory");
#ifdef DBA_SOLVE_PROF
      const long long pb2 = clock64();
      if (blockIdx.x == 0 && warp == 0 && lane == 0) {
        g_prof[6] += pa - pt0;
        g_prof[7] += pb2 - pa;
      }
#endif
      // trailing update S_ac -= W_ab W_cb^T (except (b+1,b+1)), border, rhs
      const int npair = na * (na + 1) / 2;
      const int n1 = npair * (6 / kTR) * 2;
      const int n2 = calib ? na * 4 : 0;
      const int n3 = calib ? 4 : 0;
      const int n4 = 6 * (na > 0 ? na - 1 : 0) + (calib ? 4 : 0);
      const int ntot = n1 + n2 + n3 + n4;
      for (int x = gt; x < ntot; x += kTrailThreads) {
        if (x < n1) {
          // item = (block pair, kTR output rows, 3 output columns): twice the items of a
          // whole-row split, so every trailing thread has one (measured 240 -> 229 us);
          // each output keeps the same FMA order
          const int it = x / 2, cg = 3 * (x & 1);
          const int pidx = it / (6 / kTR), rr = kTR * (it % (6 / kTR));
          if (pidx == 0) continue;  // (b+1, b+1): critical warp
          const short2 pr = S.pairs[pidx];
          const int a = b + 1 + pr.x, cc = b + 1 + pr.y;
          const double* Wa = S.pbuf + kWB * pr.x + 6 * rr;
          const double2* Wc = reinterpret_cast<const double2*>(S.pbuf + kWB * pr.y);
          double* O = wb(a, cc) + 6 * rr + cg;
          double ar[kTR][6], o[kTR][3];
#pragma unroll
          for (int r = 0; r < kTR; ++r)
#pragma unroll
            for (int d = 0; d < 6; ++d) ar[r][d] = Wa[6 * r + d];
#pragma unroll
          for (int r = 0; r < kTR; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) o[r][c] = O[6 * r + c];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double sc[6];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const double2 v = Wc[3 * (cg + c) + q];
              sc[2 * q] = v.x;
              sc[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int r = 0; r < kTR; ++r)
#pragma unroll
              for (int d = 0; d < 6; ++d) o[r][c] = fma(-ar[r][d], sc[d], o[r][c]);
          }
#pragma unroll
          for (int r = 0; r < kTR; ++r)
#pragma unroll
            for (int c = 0; c < 3; ++c) O[6 * r + c] = o[r][c];
        } else if (x < n1 + n2) {
          const int y2 = x - n1, co = y2 / 4, tt = y2 % 4;
          const int cc = b + 1 + co;
          const double* Wt = S.tbuf + 6 * tt;
          const double* Wc = S.pbuf + kWB * co;
          double* O = S.th + (size_t)cc * 24 + 6 * tt;
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            double s = O[c];
#pragma unroll
            for (int d = 0; d < 6; ++d) s = fma(-Wt[d], Wc[6 * c + d], s);
            O[c] = s;
          }
        } else if (x < n1 + n2 + n3) {
          const int tt = x - n1 - n2;
          const double* Wt = S.tbuf + 6 * tt;
          double* O = S.th + (size_t)ncols * 24 + 4 * tt;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* Wu = S.tbuf + 6 * u;
            double s = O[u];
#pragma unroll
            for (int d = 0; d < 6; ++d) s = fma(-Wt[d], Wu[d], s);
            O[u] = s;
          }
        } else {
          const int q = x - n1 - n2 - n3;
          const double* Wr;
          double* zt;
          if (q < 6 * (na - 1)) {
            Wr = S.pbuf + kWB * (1 + q / 6) + 6 * (q % 6);  // rows a >= b+2
            zt = S.z + 6 * (b + 2) + q;
          } else {
            const int tt = q - 6 * (na > 0 ? na - 1 : 0);
            Wr = S.tbuf + 6 * tt;
            zt = S.z + 6 * ncols + tt;
          }
          double s = *zt;
#pragma unroll
          for (int d = 0; d < 6; ++d) s = fma(-Wr[d], yb[d], s);
          *zt = s;
        }
      }
      if (calib && gt < 24) S.thL[(size_t)b * 24 + gt] = S.tbuf[24 + gt];  // L_tb for the backward sweep
      if (stage) asm volatile("cp.async.wait_all;" ::: "memory");
    }
#ifdef DBA_SOLVE_PROF
    __syncwarp();
    const long long pt1 = clock64();
#endif
    __syncthreads();
#ifdef DBA_SOLVE_PROF
    const long long pt2 = clock64();
    if (blockIdx.x == 0 && lane == 0 && (crit || warp == 0 || warp == kStageWarp)) {
      const int role = crit ? 0 : (warp == 0 ? 1 : 2);
      g_prof[2 * role] += pt1 - pt0;
      g_prof[2 * role + 1] += pt2 - pt1;
    }
#endif
    if (crit) CRIT_MARK(4);
    sb = (sb + 1 == W1) ? 0 : sb + 1;
  }
#ifdef DBA_CRIT_PROF
  if (crit && lane == 0 && blockIdx.x == 0)
    for (int i = 0; i < 5; ++i) g_prof[8 + i] += cpa[i];
#endif
}

// theta block (4x4 Schur complement + lam): Cholesky, forward+backward solve in
// place of zt, A9 condition estimate.  Single thread.
__device__ inline bool theta_solve(const double* T, double* zt, double lam, double* cond) {
  double L[16];
  bool ok = true;
  double pmax = 0.0, pmin = 1e300;
  for (int x = 0; x < 16; ++x) L[x] = 0.0;
  for (int c = 0; c < 4; ++c) {
    double s = T[4 * c + c] + lam;
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
  cond[0] = pmax / fmax(pmin, 1e-300);
  return ok;
}

// Backward (block LDL^T): x_b = D_b^-1 z_b - L_tb^T x_t - sum_{a>b} L_ab^T x_a for
// b < npiv.  On entry z[0, npiv) holds the forward rhs and z[npiv, nrows) the already
// known x of the rows that were not pivoted; xt (4) the theta solution (calib).
// `ring` (>= 8 factor rows) streams Lband rows via cp.async; tmp (6 npiv) staging.
template <int NS, int RD>
__device__ inline void chain_backward(double* z, const double* thL, const double* xt, const double* Lband,
                                      double* ring, unsigned long long* bars, int nrows, int npiv, int BW, int calib,
                                      double* tmp) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int W1 = BW + 1, NR = W1 * 36;
  for (int x = tid; x < 6 * npiv; x += kSolveThreads) {
    const int b = x / 6, s = x % 6;
    const double* Di = Lband + ((size_t)b * W1 + BW) * 36 + 6 * s;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 6; ++k) v = fma(Di[k], z[6 * b + k], v);
    if (calib) {
#pragma unroll
      for (int tt = 0; tt < 4; ++tt) v = fma(-thL[(size_t)b * 24 + 6 * tt + s], xt[tt], v);
    }
    tmp[x] = v;
  }
  __syncthreads();
  for (int x = tid; x < 6 * npiv; x += kSolveThreads) z[x] = tmp[x];
  // sweep: rows a = nrows-1 .. 1 fold x_a into x_b, b in [a-BW, a-1].  The factor rows
  // stream through a ring of RD slots: the staging warp refills a slot with one bulk
  // async copy (TMA engine) once the sweep warp has released it (full/empty mbarrier
  // pairs), so the sweep's critical path holds no copy issue and no proxy fence.
  const unsigned full0 = (unsigned)__cvta_generic_to_shared(bars), empty0 = full0 + 8 * RD;
  const unsigned bytes = (unsigned)(BW * 36 * sizeof(double));
  if (tid == 0)
    for (int t = 0; t < RD; ++t) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full0 + 8 * t));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty0 + 8 * t));
    }
  __syncthreads();
  auto wait_bar = [](unsigned bar, unsigned parity) {
    unsigned done = 0;
    while (!done)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(bar), "r"(parity)
          : "memory");
  };
  if (warp == kStageWarp && lane == 0 && nrows > 1 && !DBA_NOPRODUCER) {
    static_assert(RD % 8 == 0 && RD <= 32, "batches of 8 slots, at most four");
    unsigned fills = 0;  // 8 bits per batch of 8 slots: how often the batch was entered
    for (int i = 0; nrows - 1 - i >= 1; ++i) {
      const int a = nrows - 1 - i, slot = a % RD, batch = slot / 8;
      const bool enter = i == 0 || slot % 8 == 7;
      const unsigned use = (fills >> (8 * batch)) & 255u;
      if (enter) fills += 1u << (8 * batch);
      if (enter && use > 0) {  // wait for the sweep's use-th release of this batch
        // the producer shares the sweep warp's scheduler: back off instead of spinning
        for (unsigned done = 0;;) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
              "selp.u32 %0, 1, 0, p;\n\t}\n"
              : "=r"(done)
              : "r"(empty0 + 8 * batch), "r"((unsigned)(use - 1) & 1u)
              : "memory");
          if (done) break;
          __nanosleep(64);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the sweep's reads of the slot
      }
      const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + (size_t)slot * BW * 36);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full0 + 8 * slot), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst),
                   "l"(Lband + (size_t)a * NR), "r"(bytes), "r"(full0 + 8 * slot)
                   : "memory");
    }
  } else if (warp == kCritWarp && nrows > 1) {
#ifdef DBA_SOLVE_PROF
    const long long qs0 = clock64();
#endif
    // register window with rotating row groups: slot (lane < 30, register j) belongs to
    // group g = 5 j + lane / 6 (component lane % 6) and holds the partially folded z of
    // row a-1-((g - gc) mod BW); group gc holds the row finalised in this step.  No data
    // moves between lanes: the finished group reloads the row entering at distance BW.
    const int gl = lane < 30 ? lane / 6 : 99, cl = lane % 6;
    double zr[NS];
    int gc = 0;
    const int a0 = nrows - 1;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int g = 5 * j + gl, bp = a0 - 1 - g;
      zr[j] = (g < BW && bp >= 0) ? z[6 * bp + cl] : 0.0;
    }
    double xr[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) xr[r] = z[6 * a0 + r];
    for (int i = 0; nrows - 1 - i >= 1; ++i) {
      const int a = nrows - 1 - i, slot = a % RD;
#ifndef DBA_NOWAIT
      wait_bar(full0 + 8 * slot, (i / RD) & 1);
#endif
      const double* row = ring + (size_t)slot * BW * 36;
      // branch-free so that all loads issue ahead of the FMA chains
      double acc[NS];
      bool fold[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const int g = 5 * j + gl;
        int d = g - gc;
        d = d < 0 ? d + BW : d;
        const int bp = a - 1 - d;  // this slot's row
        fold[j] = g < BW && bp >= 0 && bp < npiv;
        const double* blk = row + (fold[j] ? (BW - 1 - d) * 36 + cl : 0);
        double v[6];
#pragma unroll
        for (int r = 0; r < 6; ++r) v[r] = blk[6 * r];
        acc[j] = 0.0;
#pragma unroll
        for (int r = 0; r < 6; ++r) acc[j] = fma(v[r], xr[r], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < NS; ++j) zr[j] = fold[j] ? zr[j] - acc[j] : zr[j];
      // x_{a-1} is final in group gc: broadcast it, store it, reload the group
      const int jc = gc / 5, lc = 6 * (gc % 5);
      double zc = zr[0];
#pragma unroll
      for (int j = 1; j < NS; ++j) zc = (jc == j) ? zr[j] : zc;
#pragma unroll
      for (int r = 0; r < 6; ++r) xr[r] = __shfl_sync(0xffffffffu, zc, lc + r);
      __syncwarp();
      // slots are released in batches of 8 (one arrive per batch keeps the
      // barrier off the per-row critical path)
      if (lane == 0 && !DBA_NOPRODUCER && slot % 8 == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty0 + 8 * (slot / 8)) : "memory");
      if (lane < 30 && gl == gc % 5) z[6 * (a - 1) + cl] = zc;
      {
        const int bp = a - 1 - BW;
        const double v = z[6 * (bp >= 0 ? bp : 0) + cl];
        const bool take = gl == gc % 5;
#pragma unroll
        for (int j = 0; j < NS; ++j) zr[j] = (take && j == jc) ? (bp >= 0 ? v : 0.0) : zr[j];
      }
      gc = gc + 1 == BW ? 0 : gc + 1;
    }
#ifdef DBA_SOLVE_PROF
    if (blockIdx.x == 0 && lane == 0 && nrows > 20) g_prof[14] += clock64() - qs0;
#endif
  }
#ifdef DBA_SOLVE_PROF
  const long long qe0 = clock64();
#endif
  __syncthreads();
#ifdef DBA_SOLVE_PROF
  if (blockIdx.x == 0 && warp == kCritWarp && lane == 0 && nrows > 20) g_prof[15] += clock64() - qe0;
#endif
  if (tid == 0)
    for (int t = 0; t < RD; ++t) {
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(full0 + 8 * t));
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(empty0 + 8 * t));
    }
  __syncthreads();
}

// ---------------------------------------------------------------- iterative refinement
// Optional (dba_options.refine).  With the Cholesky-form updates the factorisation is as
// accurate as LAPACK's (noisy C3 at cond 7e10: 1.1e-8 vs 2.3e-8, the former explicit-inverse
// LDL^T 1.9e-7; profiles/r02_solve_accuracy.txt).  One step of iterative refinement with
// the stored factors -- r = y - (S + lam I) x in float64 from the original band, the same
// forward / middle / backward substitutions on r, x += c -- takes the step to ~1e-10.  The
// substitutions reuse the factor rows in global memory and the theta factors still in
// shared memory.

// r[6a + s] of (S + lam I) x = y for pose block a (global order)
__device__ inline double resid_pose(const SolveArgs& A, const double* x, int a, int s, double lam) {
  const int BW = A.BW, W1 = BW + 1, nb = A.nb;
  double v = fma(-lam, x[6 * a + s], A.y[6 * a + s]);
  for (int c = max(0, a - BW); c <= a; ++c) {  // lower band and diagonal: row s of S_ac
    const double* blk = A.band + ((size_t)a * W1 + (c - a + BW)) * 36 + 6 * s;
#pragma unroll
    for (int k = 0; k < 6; ++k) v = fma(-blk[k], x[6 * c + k], v);
  }
  for (int c = a + 1; c <= min(nb - 1, a + BW); ++c) {  // upper: S_ac = S_ca^T
    const double* blk = A.band + ((size_t)c * W1 + (a - c + BW)) * 36 + s;
#pragma unroll
    for (int k = 0; k < 6; ++k) v = fma(-blk[6 * k], x[6 * c + k], v);
  }
  if (A.calib) {
    const double* xt = x + 6 * nb;
#pragma unroll
    for (int t = 0; t < 4; ++t) v = fma(-A.theta[(size_t)a * 24 + 6 * t + s], xt[t], v);
  }
  return v;
}

// r_theta (4) with warp w < 4 computing component w (fixed-order lane partials + tree)
__device__ inline void resid_theta(const SolveArgs& A, const double* x, double lam, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nb = A.nb;
  if (warp >= 4) return;
  const int t = warp;
  double v = 0.0;
  for (int q = lane; q < 6 * nb; q += 32) v = fma(-A.theta[(size_t)(q / 6) * 24 + 6 * t + q % 6], x[q], v);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) {
    double w = fma(-lam, x[6 * nb + t], A.y[6 * nb + t]);
    for (int u = 0; u < 4; ++u) w = fma(-A.thth[4 * t + u], x[6 * nb + u], w);
    out[t] = w + v;
  }
}

// forward substitution with stored factor rows (one warp, warp 0):
//   z_a -= sum_{b in [a-BW, a-1], b < npiv} L_ab z_b,  a = 1 .. nrows-1
// lanes 6p + r (p < 5) own output component r of the blocks b = a-1-p-5q; the next
// row's factor blocks are loaded while the current row folds
template <int NS>
__device__ inline void forward_apply(double* z, const double* Lband, int nrows, int npiv, int BW) {
  const int lane = threadIdx.x & 31;
  if ((threadIdx.x >> 5) != 0) return;
  const int W1 = BW + 1, r = lane % 6, part = lane < 30 ? lane / 6 : 99;
  double Lc[NS][6], Ln[NS][6];
  auto load = [&](int a, double (&Lx)[NS][6]) {
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int b = a - 1 - part - 5 * j;
      const bool use = part < 5 && a < nrows && b >= 0 && b >= a - BW && b < npiv;
      const double* L = Lband + ((size_t)(use ? a : 0) * W1 + (use ? BW - (a - b) : 0)) * 36 + 6 * r;
#pragma unroll
      for (int k = 0; k < 6; ++k) Lx[j][k] = use ? L[k] : 0.0;
    }
  };
  load(1, Lc);
  for (int a = 1; a < nrows; ++a) {
    load(a + 1, Ln);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int b = max(a - 1 - part - 5 * j, 0);
#pragma unroll
      for (int k = 0; k < 6; ++k) acc = fma(Lc[j][k], z[6 * b + k], acc);
    }
    double tot = 0.0;
#pragma unroll
    for (int p = 0; p < 5; ++p) tot += __shfl_sync(0xffffffffu, acc, r + 6 * p);
    if (lane < 6) z[6 * a + lane] -= tot;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < NS; ++j)
#pragma unroll
      for (int k = 0; k < 6; ++k) Lc[j][k] = Ln[j][k];
  }
}

// theta rows of the forward substitution: z_t -= sum_{b < npiv} L_tb z_b (warps 0..3)
__device__ inline void forward_theta(double* z, const double* thL, int npiv, int ncols) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 4) return;
  double v = 0.0;
  for (int q = lane; q < 6 * npiv; q += 32) v = fma(thL[(size_t)(q / 6) * 24 + 6 * warp + q % 6], z[q], v);
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  if (lane == 0) z[6 * ncols + warp] -= v;
}

__device__ inline ChainSm chain_sm(unsigned char* smem, const SolveSmem& L, int* fail, bool middle) {
  ChainSm S;
  S.win = reinterpret_cast<double*>(smem + L.win);
  S.th = reinterpret_cast<double*>(smem + (middle ? L.thm : L.th));
  S.thL = reinterpret_cast<double*>(smem + (middle ? L.thLm : L.thL));
  S.z = reinterpret_cast<double*>(smem + (middle ? L.zm : L.z));
  S.linv = reinterpret_cast<double*>(smem + L.linv);
  S.pbuf = reinterpret_cast<double*>(smem + L.pbuf);
  S.cbuf = reinterpret_cast<double*>(smem + L.cbuf);
  S.tbuf = reinterpret_cast<double*>(smem + L.tbuf);
  S.pairs = reinterpret_cast<short2*>(smem + L.pairs);
  S.bars = reinterpret_cast<unsigned long long*>(smem + L.bars);
  S.ring = reinterpret_cast<double*>(smem + L.ring);
  S.fail = fail;
  return S;
}

// Step correction along the prior-fixed scale direction u (u_k = t_k - R_k R_0^T t_0 in the
// translation slots, scaling about the anchor camera 0).  The fp32-assembled S is accurate
// to ~5e-8 but that error lands on u, whose eigenvalue is ~alpha-sized; q = S u is formed
// exactly (the flow terms cancel analytically), so with x the computed step:
//   x += u (u.y - (q + lam u).x) / (u.q + lam u.u)
// One CTA, after the whole step x is written.
__device__ void scale_correct(const SolveArgs& A, double lam) {
  __shared__ double red[5][kSolveThreads / 32];
  __shared__ double beta_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* p0 = A.poses + 7 * (size_t)A.anchor;
  double q0[4] = {p0[0], p0[1], p0[2], p0[3]};
  quat_normalize(q0);
  double R0[9];
  quat_to_rot(q0, R0);
  double c0[3];  // anchor camera centre -R0^T t0
  for (int r = 0; r < 3; ++r) c0[r] = -(R0[r] * p0[4] + R0[3 + r] * p0[5] + R0[6 + r] * p0[6]);
  // u.y exactly (gathered after q): the flow gradient has no component along u, so
  //   u.y = sum_p d_p [(eta + alpha m_p) g_d,p - C_p g^prior_p] / C_p = sum_frames (rho - pi)
  // with rho = c^T C^-1 g_d (c = d (eta + alpha m), the pass's GEMM) and pi the prior sum
  double d[5] = {tid == 0 ? A.q[A.nb * 6 + (A.calib ? 4 : 0)] : 0.0, 0.0, 0.0, 0.0, 0.0};  // u.y, q.x, u.x, u.q, u.u
  for (int a = tid; a < A.nb; a += kSolveThreads) {
    const double* pk = A.poses + 7 * (size_t)A.block_pose[a];
    double qk[4] = {pk[0], pk[1], pk[2], pk[3]};
    quat_normalize(qk);
    double Rk[9];
    quat_to_rot(qk, Rk);
    for (int r = 0; r < 3; ++r) {
      const double u = pk[4 + r] + (Rk[3 * r] * c0[0] + Rk[3 * r + 1] * c0[1] + Rk[3 * r + 2] * c0[2]);
      const double x = A.delta[6 * a + r], q = A.q[6 * a + r];
      d[2] += u * x;
      d[3] += u * q;
      d[4] += u * u;
    }
  }
  for (int x = tid; x < A.nb * 6 + (A.calib ? 4 : 0); x += kSolveThreads) d[1] += A.q[x] * A.delta[x];
  for (int i = 0; i < 5; ++i) {
    double v = d[i];
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[i][warp] = v;
  }
  __syncthreads();
  if (tid == 0) {
    double t[5];
    for (int i = 0; i < 5; ++i) {
      t[i] = 0.0;
      for (int w = 0; w < kSolveThreads / 32; ++w) t[i] += red[i][w];
    }
    const double den = t[3] + lam * t[4];
    beta_s = den > 0.0 ? (t[0] - t[1] - lam * t[2]) / den : 0.0;
  }
  __syncthreads();
  const double beta = beta_s;
  for (int a = tid; a < A.nb; a += kSolveThreads) {
    const double* pk = A.poses + 7 * (size_t)A.block_pose[a];
    double qk[4] = {pk[0], pk[1], pk[2], pk[3]};
    quat_normalize(qk);
    double Rk[9];
    quat_to_rot(qk, Rk);
    for (int r = 0; r < 3; ++r)
      A.delta[6 * a + r] += beta * (pk[4 + r] + (Rk[3 * r] * c0[0] + Rk[3 * r + 1] * c0[1] + Rk[3 * r + 2] * c0[2]));
  }
}

// one-sided solve (small systems)
template <int NS, int RD>
__global__ void __launch_bounds__(kSolveThreads, 1) solve_kernel(const SolveArgs A0) {
  pdl_enter();
  if (A0.status[3] != 0) return;  // GN loop finished
  double lam;
  const SolveArgs A = spec_view(A0, blockIdx.x, lam);
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveSmem L = solve_smem_layout(A.nb, A.BW, A.calib, RD);
  __shared__ int fail;
  const int tid = threadIdx.x;
  const int nb = A.nb, BW = A.BW, NR = (BW + 1) * 36;
  if (tid == 0) fail = 0;
  const ChainSm S = chain_sm(smem, L, &fail, false);
  const int r0 = min(BW, nb - 1);
  for (int x = tid; x < (r0 + 1) * NR; x += kSolveThreads) S.win[(x / 36) * kWB + x % 36] = A.band[x];
  if (A.calib) {
    for (int x = tid; x < nb * 24; x += kSolveThreads) S.th[x] = A.theta[x];
    if (tid < 16) S.th[nb * 24 + tid] = A.thth[tid];
  }
  for (int x = tid; x < 6 * nb + (A.calib ? 4 : 0); x += kSolveThreads) S.z[x] = A.y[x];
  __syncthreads();
  chain_forward(S, A.band, A.Lband, nb, nb, BW, A.calib, nb, lam);
  if (A.calib && tid == 0 && !fail)
    if (!theta_solve(S.th + (size_t)nb * 24, S.z + 6 * nb, lam, A.cond)) fail = 1;
  __syncthreads();
  if (fail) {
    if (tid == 0) A.status[0] = 1;
    return;
  }
  chain_backward<NS, RD>(S.z, S.thL, S.z + 6 * nb, A.Lband, S.ring, S.bars, nb, nb, BW, A.calib, A.delta);
  for (int x = tid; x < 6 * nb + (A.calib ? 4 : 0); x += kSolveThreads) A.delta[x] = S.z[x];
  if (A.refine) {
    double* xo = reinterpret_cast<double*>(smem + L.xo);
    __syncthreads();
    const int n = 6 * nb + (A.calib ? 4 : 0);
    for (int x = tid; x < n; x += kSolveThreads) xo[x] = S.z[x];
    __syncthreads();
    for (int x = tid; x < 6 * nb; x += kSolveThreads) S.z[x] = resid_pose(A, xo, x / 6, x % 6, lam);
    if (A.calib) resid_theta(A, xo, lam, S.z + 6 * nb);
    __syncthreads();
    forward_apply<NS>(S.z, A.Lband, nb, nb, BW);
    __syncthreads();
    if (A.calib) {
      forward_theta(S.z, S.thL, nb, nb);
      __syncthreads();
      if (tid == 0) {
        double cd;
        theta_solve(S.th + (size_t)nb * 24, S.z + 6 * nb, lam, &cd);
      }
      __syncthreads();
    }
    chain_backward<NS, RD>(S.z, S.thL, S.z + 6 * nb, A.Lband, S.ring, S.bars, nb, nb, BW, A.calib, A.delta);
    for (int x = tid; x < n; x += kSolveThreads) A.delta[x] = xo[x] + S.z[x];
  }
  if (A.scalefix) {
    __syncthreads();
    scale_correct(A, lam);
  }
}

// two-sided solve: 2 cooperative CTAs (see the header comment)
template <int NS, int RD>
__global__ void __launch_bounds__(kSolveThreads, 1) solve2_kernel(const SolveArgs A0) {
  pdl_enter();
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  if (A0.status[3] != 0) return;  // GN loop finished (uniform over the grid)
  double lam;
  const SolveArgs A = spec_view(A0, blockIdx.x >> 1, lam);  // CTA pair per candidate
  extern __shared__ __align__(16) unsigned char smem[];
  const SolveSmem L = solve_smem_layout(A.nb, A.BW, A.calib, RD);
  __shared__ int fail;
  __shared__ double xts[4];
  const int tid = threadIdx.x, cta = blockIdx.x & 1;
  const int nb = A.nb, BW = A.BW, W1 = BW + 1, NR = W1 * 36;
  const int calib = A.calib;
  const int m = A.m_top, mb = nb - m - BW;  // pivots of the top / bottom chain
  const int npiv = cta == 0 ? m : mb;
  const int nrows = npiv + BW;
  const double* band = cta == 0 ? A.band : A.rband;
  double* Lb = cta == 0 ? A.Lband : A.rLband;
  if (tid == 0) fail = 0;
  const ChainSm S = chain_sm(smem, L, &fail, false);
  // ---- load this orientation: window rows, theta border, rhs (bottom: reversed)
  for (int x = tid; x < W1 * NR; x += kSolveThreads) S.win[(x / 36) * kWB + x % 36] = band[x];
  if (calib) {
    for (int x = tid; x < nrows * 24; x += kSolveThreads) {
      const int c = x / 24, e = x % 24;
      S.th[x] = A.theta[(size_t)(cta == 0 ? c : nb - 1 - c) * 24 + e];
    }
    if (tid < 16) S.th[nb * 24 + tid] = A.thth[tid];
  }
  for (int x = tid; x < 6 * nrows; x += kSolveThreads) {
    const int a = x / 6, s = x % 6;
    S.z[x] = A.y[6 * (cta == 0 ? a : nb - 1 - a) + s];
  }
  if (calib && tid < 4) S.z[6 * nb + tid] = A.y[6 * nb + tid];
  __syncthreads();
#ifdef DBA_SOLVE_PROF
  long long ph0 = clock64();
#endif
  chain_forward(S, band, Lb, nrows, npiv, BW, calib, nb, lam);
#ifdef DBA_SOLVE_PROF
  long long ph1 = clock64();
#endif
  // ---- export the middle rows (local rows npiv..nrows-1, columns >= npiv)
  const long long per = (long long)BW * BW * 36 + 6 * BW + (long long)BW * 24 + 16 + 4;
  double* ex = A.mid + cta * per;
  {
    const int sb0 = npiv % W1;
    for (int x = tid; x < BW * BW * 36; x += kSolveThreads) {
      const int i = x / (BW * 36), j = (x / 36) % BW, e = x % 36;  // block (npiv+i, npiv+j)
      double v = 0.0;
      if (j <= i) {
        int sl = sb0 + i;
        sl = sl >= W1 ? sl - W1 : sl;
        v = S.win[((size_t)sl * W1 + (j - i + BW)) * kWB + e];
      }
      ex[x] = v;
    }
    for (int x = tid; x < 6 * BW; x += kSolveThreads) ex[BW * BW * 36 + x] = S.z[6 * npiv + x];
    if (calib) {
      for (int x = tid; x < BW * 24; x += kSolveThreads)
        ex[BW * BW * 36 + 6 * BW + x] = S.th[(size_t)npiv * 24 + x];
      if (tid < 16) ex[BW * BW * 36 + 6 * BW + BW * 24 + tid] = S.th[nb * 24 + tid];
      if (tid < 4) ex[BW * BW * 36 + 6 * BW + BW * 24 + 16 + tid] = S.z[6 * nb + tid];
    }
  }
  int* gfail = A.status + 2;  // cross-CTA failure flag (reset by the host)
  __syncthreads();
  if (tid == 0 && fail) atomicExch(gfail, 1);
  __threadfence();
  grid.sync();
  double* xsol = A.mid + 2 * per + (long long)BW * BW * 36;  // 6 BW + 4
  if (cta == 0 && *((volatile int*)gfail) == 0) {
    // ---- middle system: T + B^T(reversed) - S over poses m..m+BW-1 (+ theta)
    const ChainSm M = chain_sm(smem, L, &fail, true);
    const double* T = A.mid;
    const double* R = A.mid + per;
    const int BWm = BW - 1, W1m = BW, NRm = W1m * 36;
    for (int x = tid; x < BW * NRm; x += kSolveThreads) {
      const int i = x / NRm, pos = (x % NRm) / 36, e = x % 36, r = e / 6, c = e % 6;
      const int j = i - BWm + pos;  // column block (local middle index)
      double v = 0.0;
      if (j >= 0) {
        const double t = T[((size_t)i * BW + j) * 36 + e];
        const double rv = R[((size_t)(BW - 1 - j) * BW + (BW - 1 - i)) * 36 + 6 * c + r];
        const double o = A.band[((size_t)(m + i) * W1 + (j - i + BW)) * 36 + e];
        v = t + rv - o;
      }
      M.win[(x / 36) * kWB + x % 36] = v;
    }
    for (int x = tid; x < 6 * BW; x += kSolveThreads) {
      const int i = x / 6, s = x % 6;
      M.z[x] = T[BW * BW * 36 + x] + R[BW * BW * 36 + 6 * (BW - 1 - i) + s] - A.y[6 * (m + i) + s];
    }
    if (calib) {
      for (int x = tid; x < BW * 24; x += kSolveThreads) {
        const int i = x / 24, e = x % 24;
        M.th[x] = T[BW * BW * 36 + 6 * BW + x] + R[BW * BW * 36 + 6 * BW + (BW - 1 - i) * 24 + e] -
                  A.theta[(size_t)(m + i) * 24 + e];
      }
      const long long o2 = (long long)BW * BW * 36 + 6 * BW + BW * 24;
      if (tid < 16) M.th[BW * 24 + tid] = T[o2 + tid] + R[o2 + tid] - A.thth[tid];
      if (tid < 4) M.z[6 * BW + tid] = T[o2 + 16 + tid] + R[o2 + 16 + tid] - A.y[6 * nb + tid];
    }
    __syncthreads();
    double* Lm = A.mid + 2 * per;
    chain_forward(M, nullptr, Lm, BW, BW, BWm, calib, BW, lam);
    if (calib && tid == 0 && !fail)
      if (!theta_solve(M.th + (size_t)BW * 24, M.z + 6 * BW, lam, A.cond)) fail = 1;
    __syncthreads();
    if (!fail) chain_backward<NS, RD>(M.z, M.thL, M.z + 6 * BW, Lm, M.ring, M.bars, BW, BW, BWm, calib, A.delta);
    for (int x = tid; x < 6 * BW + (calib ? 4 : 0); x += kSolveThreads) xsol[x] = M.z[x];
    __syncthreads();
    if (tid == 0 && fail) atomicExch(gfail, 1);
  }
  __threadfence();
  grid.sync();
  // a failed candidate skips its back-substitution but stays in the grid: the scale
  // correction below needs one more grid-wide barrier
  const bool failed = *((volatile int*)gfail) != 0;
  if (failed && tid == 0 && cta == 0) A.status[0] = 1;
#ifdef DBA_SOLVE_PROF
  long long ph2 = clock64();
#endif
  if (!failed) {
  // ---- back-substitute this chain with the middle solution
  for (int x = tid; x < 6 * BW; x += kSolveThreads) {
    const int i = x / 6, s = x % 6;  // local middle row npiv + i
    S.z[6 * npiv + x] = xsol[6 * (cta == 0 ? i : BW - 1 - i) + s];
  }
  if (tid < 4) xts[tid] = calib ? xsol[6 * BW + tid] : 0.0;
  __syncthreads();
  double* tmp = A.delta + (cta == 0 ? 0 : 6 * (m + BW));  // staging inside this chain's output range
  chain_backward<NS, RD>(S.z, S.thL, xts, Lb, S.ring, S.bars, nrows, npiv, BW, calib, tmp);
  for (int x = tid; x < 6 * npiv; x += kSolveThreads) {
    const int a = x / 6, s = x % 6;
    A.delta[6 * (cta == 0 ? a : nb - 1 - a) + s] = S.z[x];
  }
  if (cta == 0) {
    for (int x = tid; x < 6 * BW; x += kSolveThreads) A.delta[6 * m + x] = xsol[x];
    if (calib && tid < 4) A.delta[6 * nb + tid] = xsol[6 * BW + tid];
  }
  }
  if (A.refine) {
    // ---- one refinement step: residual of both halves, forward on each chain, the
    // middle system on CTA 0, back-substitution, x += correction
    __threadfence();
    grid.sync();  // the whole step is in A.delta
    double* xo = reinterpret_cast<double*>(smem + L.xo);
    const int n = 6 * nb + (calib ? 4 : 0);
    double* exz = A.mid + cta * per;  // exchange: z of the middle rows (6 BW) + theta (4)
    if (!failed) {
      for (int x = tid; x < n; x += kSolveThreads) xo[x] = A.delta[x];
      __syncthreads();
      for (int x = tid; x < 6 * nrows; x += kSolveThreads) {
        const int a = x / 6, s2 = x % 6;
        S.z[x] = resid_pose(A, xo, cta == 0 ? a : nb - 1 - a, s2, lam);
      }
      if (calib) resid_theta(A, xo, lam, S.z + 6 * nb);
      __syncthreads();
      forward_apply<NS>(S.z, Lb, nrows, npiv, BW);
      __syncthreads();
      if (calib) {
        forward_theta(S.z, S.thL, npiv, nb);
        __syncthreads();
      }
      for (int x = tid; x < 6 * BW; x += kSolveThreads) exz[x] = S.z[6 * npiv + x];
      if (calib && tid < 4) exz[6 * BW + tid] = S.z[6 * nb + tid];
    }
    __threadfence();
    grid.sync();
    if (cta == 0 && !failed) {
      const ChainSm M = chain_sm(smem, L, &fail, true);
      const double* Tz = A.mid;
      const double* Rz = A.mid + per;
      for (int x = tid; x < 6 * BW; x += kSolveThreads) {
        const int i = x / 6, s2 = x % 6;
        M.z[x] = Tz[x] + Rz[6 * (BW - 1 - i) + s2] - resid_pose(A, xo, m + i, s2, lam);
      }
      if (calib) {
        resid_theta(A, xo, lam, xts);
        __syncthreads();
        if (tid < 4) M.z[6 * BW + tid] = Tz[6 * BW + tid] + Rz[6 * BW + tid] - xts[tid];
      }
      __syncthreads();
      double* Lm = A.mid + 2 * per;
      forward_apply<NS>(M.z, Lm, BW, BW, BW - 1);
      __syncthreads();
      if (calib) {
        forward_theta(M.z, M.thL, BW, BW);
        __syncthreads();
        if (tid == 0) {
          double cd;
          theta_solve(M.th + (size_t)BW * 24, M.z + 6 * BW, lam, &cd);
        }
        __syncthreads();
      }
      chain_backward<NS, RD>(M.z, M.thL, M.z + 6 * BW, Lm, M.ring, M.bars, BW, BW, BW - 1, calib, A.delta + 6 * m);
      for (int x = tid; x < 6 * BW + (calib ? 4 : 0); x += kSolveThreads) xsol[x] = M.z[x];
    }
    __threadfence();
    grid.sync();
    if (!failed) {
      for (int x = tid; x < 6 * BW; x += kSolveThreads) {
        const int i = x / 6, s2 = x % 6;
        S.z[6 * npiv + x] = xsol[6 * (cta == 0 ? i : BW - 1 - i) + s2];
      }
      if (tid < 4) xts[tid] = calib ? xsol[6 * BW + tid] : 0.0;
      __syncthreads();
      double* tmp = A.delta + (cta == 0 ? 0 : 6 * (m + BW));
      chain_backward<NS, RD>(S.z, S.thL, xts, Lb, S.ring, S.bars, nrows, npiv, BW, calib, tmp);
      for (int x = tid; x < 6 * npiv; x += kSolveThreads) {
        const int a = x / 6, s2 = x % 6;
        const int g = 6 * (cta == 0 ? a : nb - 1 - a) + s2;
        A.delta[g] = xo[g] + S.z[x];
      }
      if (cta == 0) {
        for (int x = tid; x < 6 * BW; x += kSolveThreads) A.delta[6 * m + x] = xo[6 * m + x] + xsol[x];
        if (calib && tid < 4) A.delta[6 * nb + tid] = xo[6 * nb + tid] + xsol[6 * BW + tid];
      }
    }
  }
  if (A.scalefix) {
    __threadfence();
    grid.sync();  // both chains' steps are in A.delta
    if (!failed && cta == 0) scale_correct(A, lam);
  }
#ifdef DBA_SOLVE_PROF
  if (cta == 0 && tid == 0) {
    const long long ph3 = clock64();
    g_prof[10] += ph1 - ph0;  // forward
    g_prof[11] += ph2 - ph1;  // export + middle + grid syncs
    g_prof[12] += ph3 - ph2;  // backward + writes
  }
#endif
}

}  // namespace dba
