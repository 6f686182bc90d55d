// Small per-pose / per-edge / per-frame kernels around the fused pass:
//   prep_kernel      K4: clamped tangent step -> retraction exp(xi) o G (float64),
//                    per-edge constants for the next pass (both states)
//   assemble_kernel  per source frame: split partials -> frame factor F_i over the
//                    local variables [i, j_e..., theta] (float64):
//                    F_i = sum_e B_e - T M T^T,  f_i = sum_e g_e - T w
//   gather_kernel    deterministic scatter-free assembly of the banded reduced
//                    system from the frame factors (host-built contribution lists)
//   finalize_kernel  fixed-order energy reduction
//   gauge kernels    A5 scale gauge at the end of a solve
#pragma once

#include <climits>

#include "dba_common.cuh"

namespace dba {

// ---------------------------------------------------------------- prep (K4)

struct PrepArgs {
  int N, EL, init, calib, theta_off;
  int phase;  // 0: per-pose retraction (+ intrinsics), 1: per-edge constants from both states
  double tmax;
  const int* status;
  const int* ridx;
  const int* slot_i;
  const int* slot_j;
  const double* poses_c;
  double* poses_n;
  const double* intr_c;
  double* intr_n;
  const double* delta;
  double* xi_out;  // (N,6) clamped steps actually applied
  EdgeLin* lin;
  EdgeBack* back;
  double* adj;  // (EL,36) Ad(G_ij) at x_n
  const int* slot_edge;
  int* bad_edge;  // smallest edge whose x_n constants are non-finite (flags word [1])
};

__device__ inline void clamped_xi(const PrepArgs& A, int k, double xi[6]) {
  for (int c = 0; c < 6; ++c) xi[c] = 0.0;
  if (A.init) return;
  const int r = A.ridx[k];
  if (r < 0) return;
  double n2 = 0.0;
  for (int c = 0; c < 6; ++c) {
    xi[c] = A.delta[6 * r + c];
    n2 += xi[c] * xi[c];
  }
  const double n = sqrt(n2);
  if (n > A.tmax) {
    const double s = A.tmax / n;
    for (int c = 0; c < 6; ++c) xi[c] *= s;
  }
}

__device__ inline Pose64 stepped_pose(const PrepArgs& A, int k, const double xi[6]) {
  const Pose64 pc = load_pose(A.poses_c + 7 * k);
  if (A.init || A.ridx[k] < 0) return pc;
  return compose(se3_exp(xi), pc);
}

__global__ void prep_kernel(const PrepArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x + (A.phase == 1 ? A.N : 0);
  if (A.phase == 0 && t == A.N) {  // intrinsics
    for (int c = 0; c < 4; ++c) {
      const double d = (A.calib && !A.init) ? A.delta[A.theta_off + c] : 0.0;
      A.intr_n[c] = A.intr_c[c] + d;
    }
    return;
  }
  if (A.phase == 0 ? t > A.N : t >= A.N + A.EL) return;
  if (t < A.N) {
    double xi[6];
    clamped_xi(A, t, xi);
    for (int c = 0; c < 6; ++c) A.xi_out[6 * t + c] = xi[c];
    if (A.init || A.ridx[t] < 0) {
      for (int c = 0; c < 7; ++c) A.poses_n[7 * t + c] = A.poses_c[7 * t + c];
    } else {
      store_pose(stepped_pose(A, t, xi), A.poses_n + 7 * t);
    }
  } else if (t < A.N + A.EL) {
    const int s = t - A.N;
    const int i = A.slot_i[s], j = A.slot_j[s];
    double xi_i[6], xi_j[6];
    for (int c = 0; c < 6; ++c) {  // clamped steps and stepped poses from phase 0
      xi_i[c] = A.xi_out[6 * i + c];
      xi_j[c] = A.xi_out[6 * j + c];
    }
    const Pose64 ci = load_pose(A.poses_c + 7 * i), cj = load_pose(A.poses_c + 7 * j);
    const Pose64 gc = compose(cj, inverse(ci));
    const Pose64 gn = compose(load_pose(A.poses_n + 7 * j), inverse(load_pose(A.poses_n + 7 * i)));
    double Rn[9], Rc[9], Ac[36], An[36];
    quat_to_rot(gn.q, Rn);
    quat_to_rot(gc.q, Rc);
    adjoint(Rn, gn.t, An);
    adjoint(Rc, gc.t, Ac);
    EdgeLin el;
    EdgeBack eb;
    for (int c = 0; c < 9; ++c) {
      el.R[c] = Rn[c];
      eb.R[c] = Rc[c];
    }
    for (int c = 0; c < 3; ++c) {
      el.t[c] = gn.t[c];
      eb.t[c] = gc.t[c];
    }
    for (int r = 0; r < 6; ++r) {
      double s2 = xi_j[r];
      for (int c = 0; c < 6; ++c) s2 -= Ac[6 * r + c] * xi_i[c];
      eb.dlt[r] = s2;
    }
    // a non-finite trial pose or intrinsics: the energy-only trial pass cannot see it
    // (invalid projections contribute zero), so flag the edge here
    bool ok = true;
    for (int c = 0; c < 9; ++c) ok = ok && isfinite(Rn[c]);
    for (int c = 0; c < 3; ++c) ok = ok && isfinite(gn.t[c]);
    for (int c = 0; c < 4; ++c) ok = ok && isfinite(A.intr_n[c]);
    if (!ok && A.bad_edge) atomicMin(A.bad_edge, A.slot_edge[s]);
    A.lin[s] = el;
    A.back[s] = eb;
    for (int c = 0; c < 36; ++c) A.adj[36 * (size_t)s + c] = An[c];
  }
}

// ---------------------------------------------------------------- assemble

struct AsmArgs {
  int calib, nve;
  const int* status;
  const int* csr_off;
  const int* slot_edge;
  const int* frame_seg;  // local frame -> segment range
  const double* adj;
  const double* part_edge;
  const double* part_M;
  const double* part_w;
  const double* part_frame;
  const long long* seg_off_edge;
  const long long* seg_off_M;
  const long long* seg_off_w;
  double* Fbuf;
  const long long* off_F;
  const long long* off_f;
  int* bad_edge;
  int gauge_frame;        // A5 (global frame id) or -1
  int scalefix;           // write the frame's exact scale-direction row q after f
  const int* frame_of;
  double* gstate;         // out: [gamma, rho, h] for the gauge frame
};

__device__ __forceinline__ int tri6(int r, int c) {
  if (r > c) {
    const int t = r;
    r = c;
    c = t;
  }
  return r * 6 - r * (r - 1) / 2 + (c - r);
}
__device__ __forceinline__ int tri4(int r, int c) {
  if (r > c) {
    const int t = r;
    r = c;
    c = t;
  }
  return r * 4 - r * (r - 1) / 2 + (c - r);
}

// dynamic shared memory of assemble_kernel: the frame's M (mu x mu float64)
__host__ __device__ inline size_t assemble_smem_bytes(int kmax, bool calib) {
  const size_t mu = 6 * (size_t)kmax + (calib ? 4 : 0);
  return sizeof(double) * mu * mu;
}

__global__ void __launch_bounds__(512) assemble_kernel(const AsmArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  extern __shared__ double Ms[];  // M = sum_p v_p v_p^T / C_p over u-space (mu x mu)
  __shared__ double Ad[kMaxOutDegree * 36];
  __shared__ double hs[kMaxOutDegree * (kEdgeVals + kCalibVals)];
  __shared__ double ws[6 * kMaxOutDegree + 4];
  __shared__ double fs[kFrameVals];
  __shared__ double Nm[6 * (6 * kMaxOutDegree + 4)];
  __shared__ double hg[6 * kMaxOutDegree + 4];
  __shared__ double Th[6 * kMaxOutDegree + 10];
  __shared__ double Tb[kMaxOutDegree * 36];  // per-edge Ad_e^T H_e
  __shared__ double Tc[kMaxOutDegree * 36];  // per-edge pose-block terms
  __shared__ int t6[36];                      // tri6(r, c) of the packed 6x6 Hessians
  const int fl = blockIdx.x, tid = threadIdx.x;
  const int s0 = A.csr_off[fl], k = A.csr_off[fl + 1] - s0;
  if (k == 0) return;
  const int nve = A.nve;
  const int mu = 6 * k + (A.calib ? 4 : 0), m = mu + 6;
  double* F = A.Fbuf + A.off_F[fl];
  double* fv = A.Fbuf + A.off_f[fl];
  const int sg0 = A.frame_seg[fl], sg1 = A.frame_seg[fl + 1];

  if (tid < 36) t6[tid] = tri6(tid / 6, tid % 6);
  // segment partials, summed in segment order; each pass over x issues its loads
  // independently (unrolled) so the loop is bandwidth-, not latency-bound
  for (int x = tid; x < k * 36; x += blockDim.x) Ad[x] = A.adj[36 * (size_t)s0 + x];
  const bool gauge = A.frame_of[fl] == A.gauge_frame;
  for (int sg = sg0; sg < sg1; ++sg) {
    const bool first = sg == sg0;
    const double* pe = A.part_edge + A.seg_off_edge[sg];
    const double* pw = A.part_w + A.seg_off_w[sg];
    const double* pm = A.part_M + A.seg_off_M[sg];
#pragma unroll 4
    for (int x = tid; x < k * nve; x += blockDim.x) hs[x] = first ? pe[x] : hs[x] + pe[x];
#pragma unroll 2
    for (int x = tid; x < mu; x += blockDim.x) {
      ws[x] = first ? pw[x] : ws[x] + pw[x];
      hg[x] = first ? pw[mu + x] : hg[x] + pw[mu + x];
    }
    if (tid < kFrameVals) {
      const double v = A.part_frame[(long long)sg * kFrameVals + tid];
      fs[tid] = first ? v : fs[tid] + v;
    }
#pragma unroll 8
    for (int x = tid; x < mu * mu; x += blockDim.x) Ms[x] = first ? pm[x] : Ms[x] + pm[x];
  }
  __syncthreads();
  if (tid < k) {
    bool ok = true;
    for (int x = 0; x < nve; ++x) ok = ok && isfinite(hs[tid * nve + x]);
    if (!ok) atomicMin(A.bad_edge, A.slot_edge[s0 + tid]);
  }
  // N = sum_e Ad_e^T M[e, :]   (6 x mu)
  for (int x = tid; x < 6 * mu; x += blockDim.x) {
    const int r = x / mu, c = x % mu;
    double s = 0.0;
    for (int e = 0; e < k; ++e)
      for (int q = 0; q < 6; ++q) s += Ad[36 * e + 6 * q + r] * Ms[(6 * e + q) * mu + c];
    Nm[x] = s;
  }
  // (Ad_e^T H_e) per edge, 6x6 each
  for (int x = tid; x < k * 36; x += blockDim.x) {
    const int e = x / 36, r = (x / 6) % 6, q = x % 6;
    const double* Ae = Ad + 36 * e;
    const double* He = hs + e * nve;
    double hq = 0.0;
    for (int u = 0; u < 6; ++u) hq += Ae[6 * u + r] * He[t6[6 * u + q]];
    Tb[x] = hq;
  }
  __syncthreads();
  // pose-block terms per edge: (Ad_e^T H_e - N_e) Ad_e; N_e = Nm[:, 6e..6e+5]
  for (int x = tid; x < k * 36; x += blockDim.x) {
    const int e = x / 36, r = (x / 6) % 6, c = x % 6;
    const double* Ae = Ad + 36 * e;
    double t = 0.0;
    for (int q = 0; q < 6; ++q) t += (Tb[36 * e + 6 * r + q] - Nm[r * mu + 6 * e + q]) * Ae[6 * q + c];
    Tc[x] = t;
  }
  __syncthreads();
  const int th0 = 6 * k;  // theta offset in u-space
  // F row by row: warp w takes rows w, w + 16, ..., lanes the columns (no per-entry
  // division by m); packed 6x6 indices from the shared tri6 table
  const int lane = tid & 31, nwarp = blockDim.x >> 5;
  for (int r = tid >> 5; r < m; r += nwarp) {
    const int ru = r - 6;
    const int rb = ru / 6, rs = ru - 6 * rb;  // (ru >= 0) block and slot of row r in u-space
    for (int c = lane; c < m; c += 32) {
      double v;
      if (r >= 6 && c >= 6) {
        const int cu = c - 6;
        const int cb = cu / 6, cs = cu - 6 * cb;
        double b = 0.0;
        const bool rt = A.calib && ru >= th0, ct = A.calib && cu >= th0;
        if (!rt && !ct) {
          if (rb == cb) b = hs[rb * nve + t6[6 * rs + cs]];
        } else if (rt && !ct) {
          b = hs[cb * nve + 32 + 6 * (ru - th0) + cs];
        } else if (!rt && ct) {
          b = hs[rb * nve + 32 + 6 * (cu - th0) + rs];
        } else {
          b = fs[1 + tri4(ru - th0, cu - th0)];
        }
        v = b - Ms[ru * mu + cu];
      } else if (r < 6 && c < 6) {
        v = 0.0;
        for (int e = 0; e < k; ++e) v += Tc[36 * e + 6 * r + c];  // fixed edge order
      } else {
        const int rr = r < 6 ? r : c;          // pose-i row (0..5)
        const int cu = r < 6 ? c - 6 : r - 6;  // u-space column
        double b = 0.0;
        if (A.calib && cu >= th0) {
          const int t = cu - th0;
          for (int e = 0; e < k; ++e)
            for (int q = 0; q < 6; ++q) b -= hs[e * nve + 32 + 6 * t + q] * Ad[36 * e + 6 * q + rr];
        } else {
          const int e = cu / 6, cc = cu - 6 * e;
#pragma unroll
          for (int q = 0; q < 6; ++q) b -= Ad[36 * e + 6 * q + rr] * hs[e * nve + t6[6 * q + cc]];
        }
        v = b + Nm[rr * mu + cu];  // B_iu - (T M T^T)_iu with T_i = -Ad^T
      }
      F[r * m + c] = v;
    }
  }
  for (int x = tid; x < m; x += blockDim.x) {
    double v;
    if (x < 6) {
      v = 0.0;
      for (int e = 0; e < k; ++e)
        for (int q = 0; q < 6; ++q) v += Ad[36 * e + 6 * q + x] * (ws[6 * e + q] - hs[e * nve + 21 + q]);
    } else {
      const int cu = x - 6;
      if (A.calib && cu >= th0)
        v = fs[11 + cu - th0] - ws[cu];
      else
        v = hs[(cu / 6) * nve + 21 + cu % 6] - ws[cu];
    }
    fv[x] = v;
  }
  if (A.scalefix) {
    // exact S u along the prior-fixed monocular scale u (the flow terms cancel analytically):
    // T h with h = E C^-1 c, c = d (eta + alpha m); stored after f for the gather
    double* qv = fv + m;
    // u.y of this frame: rho (= c^T C^-1 g_d with the scale column c) minus the prior sum
    if (tid == 0) qv[m] = fs[16] - fs[17];
    for (int x = tid; x < m; x += blockDim.x) {
      double v;
      if (x < 6) {
        v = 0.0;
        for (int e = 0; e < k; ++e)
          for (int q = 0; q < 6; ++q) v -= Ad[36 * e + 6 * q + x] * hg[6 * e + q];
      } else {
        v = hg[x - 6];
      }
      qv[x] = v;
    }
  }
  if (!gauge) return;
  // A5 gauge constraint (Sherman-Morrison): F += (T h)(T h)^T / gamma, f += (T h) rho / gamma
  __syncthreads();
  const double gam = fs[15], rho = fs[16];
  for (int x = tid; x < m; x += blockDim.x) {
    double v;
    if (x < 6) {
      v = 0.0;
      for (int e = 0; e < k; ++e)
        for (int q = 0; q < 6; ++q) v -= Ad[36 * e + 6 * q + x] * hg[6 * e + q];
    } else {
      v = hg[x - 6];
    }
    Th[x] = v;
  }
  if (tid == 0) {
    A.gstate[0] = gam;
    A.gstate[1] = rho;
  }
  for (int x = tid; x < mu; x += blockDim.x) A.gstate[2 + x] = hg[x];
  __syncthreads();
  for (int x = tid; x < m * m; x += blockDim.x) F[x] += Th[x / m] * Th[x % m] / gam;
  for (int x = tid; x < m; x += blockDim.x) fv[x] += Th[x] * rho / gam;
}

// ---------------------------------------------------------------- gather

struct GatherUnit {
  long long dst;
  int rows, cols, c0, c1;
  int trans = 0;  // square block written transposed (reversed band)
  int pad = 0;
};
struct Contrib {
  long long src;
  int stride, pad;
};

struct GatherArgs {
  int n_units;
  const int* status;
  const GatherUnit* units;
  const Contrib* contrib;
  const double* Fbuf;
  double* sys;
};

__global__ void gather_kernel(const GatherArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= A.n_units) return;
  const GatherUnit u = A.units[wid];
  const int n = u.rows * u.cols;
  if (n <= 64) {
    // every unit of the band (6x6, 4x6, 4x4 blocks, rhs rows): a lane owns elements lane and
    // lane + 32; the contribution list is read coalesced, 32 at a time, and broadcast by
    // shuffles, so the Fbuf loads of successive contributions are independent (the sum
    // order per element is the list order, as before)
    const int e0 = lane, e1 = lane + 32;
    const int r0 = e0 / u.cols, k0 = e0 - r0 * u.cols, r1 = e1 / u.cols, k1 = e1 - r1 * u.cols;
    double s0 = 0.0, s1 = 0.0;
    for (int q0 = u.c0; q0 < u.c1; q0 += 32) {
      const int nq = min(32, u.c1 - q0);
      long long src = 0;
      int stride = 0;
      if (lane < nq) {
        const Contrib cb = A.contrib[q0 + lane];
        src = cb.src;
        stride = cb.stride;
      }
#pragma unroll 4
      for (int j = 0; j < nq; ++j) {
        const long long sj = __shfl_sync(0xffffffffu, src, j);
        const long long tj = __shfl_sync(0xffffffffu, stride, j);
        if (e0 < n) s0 += A.Fbuf[sj + (u.trans ? k0 * tj + r0 : r0 * tj + k0)];
        if (e1 < n) s1 += A.Fbuf[sj + (u.trans ? k1 * tj + r1 : r1 * tj + k1)];
      }
    }
    if (e0 < n) A.sys[u.dst + e0] = s0;
    if (e1 < n) A.sys[u.dst + e1] = s1;
    return;
  }
  for (int e = lane; e < n; e += 32) {
    const int r = e / u.cols, c = e % u.cols;
    double s = 0.0;
#pragma unroll 4
    for (int q = u.c0; q < u.c1; ++q) {
      const Contrib cb = A.contrib[q];
      s += u.trans ? A.Fbuf[cb.src + (long long)c * cb.stride + r] : A.Fbuf[cb.src + (long long)r * cb.stride + c];
    }
    A.sys[u.dst + e] = s;
  }
}

// ---------------------------------------------------------------- finalize

struct FinalArgs {
  int n;       // number of partial rows (pass segments or energy CTAs)
  int stride;  // doubles between rows; the energy is the first value of a row
  const int* status;
  const double* part_frame;
  double* energy_out;
};


// fixed-order sum of the partial rows: strided per-thread sums, warp butterfly, then
// the warp sums in order (kFinalThreads threads)
constexpr int kFinalThreads = 1024;
__device__ __forceinline__ void finalize_energy(const FinalArgs& A) {
  __shared__ double sh[kFinalThreads / 32];
  double s = 0.0;
#pragma unroll 4
  for (int x = threadIdx.x; x < A.n; x += kFinalThreads) s += A.part_frame[(long long)x * A.stride];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kFinalThreads / 32; ++w) t += sh[w];
    A.energy_out[0] = t;
  }
}

__global__ void __launch_bounds__(kFinalThreads) finalize_kernel(const FinalArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  finalize_energy(A);
}

// ---------------------------------------------------------------- gauge (A5)

// sum of log d over one frame (fixed-order tree); out[0] = sum (0 if frame < 0)
// float32 boundary disparities <-> the float64 solver state
__global__ void __launch_bounds__(256) widen_kernel(const float* src, double* dst, long long n) {
  pdl_enter();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) dst[t] = (double)src[t];
}
__global__ void __launch_bounds__(256) narrow_kernel(const double* src, float* dst, long long n) {
  pdl_enter();
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) dst[t] = (float)src[t];
}

__global__ void __launch_bounds__(256) logsum_kernel(const float* d, int frame, int P, double* out) {
  pdl_enter();
  __shared__ double sh[256];
  double s = 0.0;
  if (frame >= 0)
    for (int x = threadIdx.x; x < P; x += 256) s += log((double)d[(size_t)frame * P + x]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int off = 128; off >= 1; off >>= 1) {
    if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

struct GaugeArgs {
  int N, P, g, f0, f1;
  double d_min;
  const double* ref_sum;  // sum log d_g at the input state
  const double* cur_sum;  // sum log d_g at the final state
  double* scale_out;
  float* d;
  double* poses;
};

// d <- max(s d, d_min) on this rank's frames; every pose moved by the similarity
// about camera g that keeps G_g:  t_k <- (t_k - c_k)/s + c_k,  c_k = R_k R_g^T t_g
__global__ void gauge_apply_kernel(const GaugeArgs A) {
  pdl_enter();
  const double s = exp((A.ref_sum[0] - A.cur_sum[0]) / (double)A.P);
  const long long n_d = (long long)(A.f1 - A.f0) * A.P;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) A.scale_out[0] = s;
  if (t < n_d) {
    float* dp = A.d + (long long)A.f0 * A.P + t;
    *dp = fmaxf(*dp * (float)s, (float)A.d_min);
  }
  if (t < A.N && t != A.g) {
    const Pose64 pg = load_pose(A.poses + 7 * A.g);
    const Pose64 pk = load_pose(A.poses + 7 * t);
    double Rg[9], Rk[9], w[3], c[3];
    quat_to_rot(pg.q, Rg);
    quat_to_rot(pk.q, Rk);
    for (int r = 0; r < 3; ++r) w[r] = Rg[r] * pg.t[0] + Rg[3 + r] * pg.t[1] + Rg[6 + r] * pg.t[2];
    for (int r = 0; r < 3; ++r) c[r] = Rk[3 * r] * w[0] + Rk[3 * r + 1] * w[1] + Rk[3 * r + 2] * w[2];
    for (int r = 0; r < 3; ++r) A.poses[7 * t + 4 + r] = (pk.t[r] - c[r]) / s + c[r];
  }
}

}  // namespace dba

namespace dba {

// ---------------------------------------------------------------- GN controller
// The Levenberg-Marquardt schedule (A1) runs on the device so that a
// whole solve is enqueued without host round trips: state slot 0 is the current
// iterate, slot 1 the trial; the decision (finalize_decide_kernel, or decide_kernel
// after the all-reduce) copies accepted poses/intrinsics to slot 0, and the gated
// linearisation of an accepted trial writes slot 0's disparities, system and gauge
// state.
constexpr int kTraceMax = 64;  // == DBA_TRACE_MAX
constexpr int kMaxSpecD = 3;   // == kMaxSpec (dba_solve.cuh)

struct Control {
  double lam, Ec, cond;
  int it, trials, result, converged, bad_edge, accept, done, pad;
  int rounds, cands, lins, pad2;  // executed rounds / candidate decisions / linearisations
  double trace[kTraceMax];
};

struct DecideArgs {
  int iters, calib;
  double lam_min, lam_max, cond_max;
  int* status;          // flags word of this damping candidate ([0] failed, [1] bad edge, [3] skip)
  int* loop;            // the loop's flags word ([3] finished; == status for candidate 0)
  int* next;            // flags word of the next candidate, or null
  int* gate;            // flags word of the kernels that linearise an accepted trial
  double* cond;         // theta pivot ratio of the last solve
  const double* energy; // energy of the trial state (slot 1)
  Control* ctl;
  // acceptance: the trial poses / intrinsics (slot 1) become the iterate (slot 0);
  // disparities, system and gauge state are written to slot 0 by the gated
  // linearisation of the accepted trial
  double* poses_dst;
  const double* poses_src;
  int pose_words;
  double* intr_dst;
  const double* intr_src;
  // graph mode (dba_solve's device-driven loop): the decision also steers the
  // conditional nodes -- the next candidate's IF, the linearisation IF, the WHILE
  int graph, cand, nspec;
  unsigned long long h_cand[kMaxSpecD], h_lin, h_loop;
};

// One LM decision on the trial of one damping candidate.  Candidates are decided in
// order (lambda, 10 lambda, ...) exactly as the sequential schedule would run them:
// candidate k is only evaluated when every earlier one was rejected or failed, so
// the decisions, lambda sequence, trial count and trace are those of one-at-a-time
// trials.  Returns false when the candidate was not needed (no state change beyond
// propagating the skip).
__device__ bool gn_decide(const DecideArgs& A) {
  Control* cg = A.ctl;
  int* st = A.status;
  int* lp = A.loop;
  const bool first = st == lp;
  // flags and controller scalars are read once into registers (the flags words may
  // alias nothing in Control, but the compiler cannot know): one round of loads
  const int s0 = st[0], s1 = st[1], s3 = st[3], l3 = lp[3];
  if (l3 != 0 || (!first && s3 != 0)) {  // finished, or an earlier candidate decided
    if (!first) {
      st[0] = 0;
      st[1] = INT_MAX;
      st[2] = 0;
    }
    if (A.next) {
      A.next[3] = 1;
      A.next[0] = 0;
      A.next[2] = 0;
    }
    return false;
  }
  double lam = cg->lam, Ec = cg->Ec, cond = cg->cond;
  int it = cg->it, trials = cg->trials, result = cg->result, converged = cg->converged;
  int bad_edge = cg->bad_edge;
  const double E = *A.energy;
  const double cin = *A.cond;
  int accept = 0, done = 0;
  if (s0 != 0) {  // factorisation failed: more damping, same iterate
    lam *= 10.0;
    if (lam > A.lam_max) {
      result = 1;  // DBA_ESOLVER (mapped by the host)
      done = 1;
    }
  } else {
    trials++;
    if (A.calib) {
      cond = cin;
      if (A.cond_max > 0.0 && cond > A.cond_max) {
        result = 2;  // DBA_ECALIB
        done = 1;
      }
    }
    if (!done && (s1 != INT_MAX || !isfinite(E))) {
      bad_edge = s1 != INT_MAX ? s1 : -1;
      result = 3;  // DBA_ENONFINITE
      done = 1;
    }
    if (!done) {
      if (E <= Ec) {
        accept = 1;
        Ec = E;
        lam = fmax(lam / 10.0, A.lam_min);
        if (it < kTraceMax) cg->trace[it] = E;
        it++;
        if (it >= A.iters) done = 1;
      } else {
        lam *= 10.0;
        if (lam > A.lam_max) {
          converged = 1;
          done = 1;
        }
      }
    }
  }
  cg->lam = lam;
  cg->Ec = Ec;
  cg->cond = cond;
  cg->it = it;
  cg->trials = trials;
  cg->result = result;
  cg->converged = converged;
  cg->bad_edge = bad_edge;
  cg->accept = accept;
  cg->done = done;
  cg->cands++;
  if (first) cg->rounds++;
  if (accept && !done) cg->lins++;
  if (A.gate) {  // [0]: rejected, [3]: finished -> trial_skipped
    A.gate[0] = !accept;
    A.gate[3] = done;
  }
  st[0] = 0;
  st[1] = INT_MAX;
  st[2] = 0;
  st[3] = first ? done : 0;
  lp[3] = done;
  if (A.next) {  // the next candidate runs only after a rejection / failure
    const int skip = accept || done;
    A.next[3] = skip;
    A.next[1] = INT_MAX;
    if (skip) {
      A.next[0] = 0;
      A.next[2] = 0;
    }
  }
  *A.cond = 0.0;
  return true;
}

// the LM decision (thread 0) and, on acceptance, the pose/intrinsics copy by the
// whole block
__device__ void decide_block(const DecideArgs& A) {
  __shared__ int acc;
  if (threadIdx.x == 0) {
    const bool decided = gn_decide(A);
    acc = decided && A.ctl->accept;
    if (A.graph && decided) {
      const Control* c = A.ctl;
      const int go_next = !c->accept && !c->done;
      for (int m = A.cand + 1; m < A.nspec; ++m) cudaGraphSetConditional(A.h_cand[m], m == A.cand + 1 ? go_next : 0);
      cudaGraphSetConditional(A.h_lin, c->accept && !c->done);
      cudaGraphSetConditional(A.h_loop, !c->done);
    }
  }
  __syncthreads();
  if (acc) {
    for (int x = threadIdx.x; x < A.pose_words; x += blockDim.x) A.poses_dst[x] = A.poses_src[x];
    if (threadIdx.x < 4) A.intr_dst[threadIdx.x] = A.intr_src[threadIdx.x];
  }
}

__global__ void decide_kernel(const DecideArgs A) {
  pdl_enter();
  decide_block(A);
}

// single rank: the trial energy and the LM decision in one launch
__global__ void __launch_bounds__(kFinalThreads) finalize_decide_kernel(const FinalArgs F, const DecideArgs D) {
  pdl_enter();
  if (!trial_skipped(F.status)) finalize_energy(F);  // uniform over the block
  decide_block(D);
}

}  // namespace dba
