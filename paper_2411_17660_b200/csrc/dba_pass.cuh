// K1+K2+K3a(+K5): the fused per-frame pass of one Gauss-Newton trial.
//
// A CTA (16 warps) walks a list of segments; a segment is (source frame i, a
// run of 256-pixel sub-tiles) and owns ALL out-edges of frame i, so every
// per-pixel disparity term (C_p, g_d,p and the pose/disparity couplings
// E_e,p) stays on chip.  Per sub-tile:
//
//   phase A (back-substitution at x_c, skipped on the first pass), edge-major:
//       unit (edge e, 64-px slice) -> per-pixel parts of C_p, g_d,p and
//       E_e,p . delta_e recomputed at x_c from the flow record;
//       per pixel: delta d_p = (g_d,p - sum_e E_e,p . delta_e) / C_p,
//       d_n = max(d + delta d, d_min)
//   phase B (linearisation at x_n = trial state), edge-major:
//       residual, validity (geometry.py:235-250), J_j, J_d, [J_theta];
//       energy, per-edge H_jj / g_j accumulated in registers of the warp that
//       owns the units (one warp transpose-reduce per edge per sub-tile);
//       E_e,p -> shared U[p][6e..6e+5]; per-edge parts of C_p, g_d,p
//   per pixel: C_p, g_d,p (+ Eq. 4 prior), U[p] row extended by [g_d,p, C_p/d_p]
//   phase C (K3a): M_ext += V V^T with V = U_ext / sqrt(C), a shared-memory SIMT
//       GEMM in 4x8 register tiles split over pixels across warp groups.  The two extra rows give, in the
//       same GEMM, w = E C^-1 g_d (Schur rhs) and the A5 gauge terms
//       h = E C^-1 c, rho = c^T C^-1 g_d, gamma = c^T C^-1 c with c = C/d.
//
// The flow record (tu, tv, wu, wv) is one coalesced float4 per edge-pixel (the
// 16 B of algorithmic traffic); phase B re-reads it from L1/L2.  Jacobians use
// homogeneous coordinates X~ = R q + t d (q = ((u-cx)/fx, (v-cy)/fy, 1)):
//   J_u = fx [d/Z, 0, -d x/Z, -x y, 1 + x^2, -y]
//   J_v = fy [0, d/Z, -d y/Z, -(1 + y^2), x y, x]
//   J_d = (fx (t_x - x t_z)/Z, fy (t_y - y t_z)/Z)
// equal to the oracle's J_j = J_pi(X_j)[I | -[X_j]x], J_d = J_pi(X_j) R (-X_i/d)
// (oracle/dba.py edge_terms).  J_i = -J_j Ad(G_ij) is applied per edge in
// assemble.  Partials leave in float64; every reduction has a fixed order.
#pragma once

#include "dba_common.cuh"

namespace dba {

constexpr int kPassThreads = 512;
constexpr int kPassWarps = 16;
constexpr int kSub = 256;    // pixels per sub-tile
constexpr int kSlice = 32;   // pixels per phase-B edge unit (1 per lane)
constexpr int kSlices = kSub / kSlice;
constexpr int kEdgeSlots = 2;  // distinct edges per warp per segment (4k units / 16 warps)

struct PassArgs {
  int H, W, P, n_tiles, kmax;
  int backsub;  // run phase A
  int freeze;   // disparity block frozen (motion-only / pose stage): no Schur fill-in, d unchanged
  int system;   // produce system partials (0: energy only)
  int stage;    // flow records of the next sub-tile are staged in smem with cp.async
  int scalefix; // prior-fixed monocular scale: the A5 column carries c = d (eta + alpha m) instead
  const int* status;  // see trial_skipped
  unsigned long long* runs;  // counts executed launches (profiling of gated passes) or null
  const int* csr_off;
  const int* slot_flow;
  const int* frame_of;
  const int* seg_frame;  // segment -> local frame
  const int* seg_t0;     // segment -> first 256-px tile
  const int* seg_t1;     // segment -> end tile
  const int* cta_seg;    // CTA -> segment range
  const EdgeLin* lin;
  const EdgeBack* back;
  const float4* flow;
  const float* d_cur;
  float* d_new;
  const float* prior;
  const uint8_t* pmask;
  const float* pweight;  // (N,) per-frame multiplier of alpha (Eq. 5 stage A: s_i^2) or null
  float alpha, eta, d_min;
  const double* intr_c;
  const double* intr_n;
  int gauge_frame;         // A5 mono gauge frame (global id) or -1
  const double* gstate_c;  // [gamma, rho, h(u-space)] of the x_c linearisation
  double* part_edge;
  double* part_M;
  double* part_w;
  double* part_frame;
  const long long* seg_off_edge;
  const long long* seg_off_M;
  const long long* seg_off_w;
};

// 32 values per lane -> lane l ends with the warp sum of value l (31 shuffles).
__device__ __forceinline__ float transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const float send = up ? v[i] : v[i + off];
      const float keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

__host__ __device__ inline int pass_mu(int k, bool calib) { return 6 * k + (calib ? 4 : 0); }
// GEMM rows: U (mu) + [g_d, C/d], padded to a multiple of 8 (4x8 register tiles)
__host__ __device__ inline int pass_mext(int k, bool calib) { return pass_mu(k, calib) + 2; }
__host__ __device__ inline int pass_mpad(int k, bool calib) { return (pass_mext(k, calib) + 7) & ~7; }
// row stride = 2 (mod 8): float2 accesses by 16 lanes of consecutive pixel rows are
// conflict-free; the GEMM reads rows with 8-byte loads
__host__ __device__ inline int pass_ustride(int k, bool calib) { return pass_mpad(k, calib) + 2; }
// number of 4x8 tiles touching the upper triangle of an (mpad x mpad) matrix
__host__ __device__ inline int pass_ntiles(int mpad) {
  const int nr = mpad / 4, nc = mpad / 8;
  int n = 0;
  for (int tj = 0; tj < nc; ++tj) n += (2 * tj + 2 < nr) ? 2 * tj + 2 : nr;
  return n;
}

struct PassSmem {
  size_t fbuf, U, parts, dcs, dns, qc, qn, ebuf, ethb, red, emap, sflow, sl, sb, total;
};
__host__ __device__ inline PassSmem pass_smem_layout(int kmax, bool calib, bool stage) {
  PassSmem s;
  size_t o = 0;
  s.fbuf = o; o += stage ? sizeof(float4) * (size_t)kmax * kSub : 0;
  const int nparts = calib ? 6 : 2;  // phase B: C, gd (+ E_theta x4)
  s.ethb = o; o += calib ? sizeof(double) * kPassWarps * kEdgeSlots * 32 : 0;
  s.red = o; o += sizeof(double) * kPassWarps * 16;
  s.U = o; o += sizeof(float) * (size_t)kSub * pass_ustride(kmax, calib);
  {  // the segment-end GEMM partials reuse U: 32 floats per thread
    const size_t need = sizeof(float) * 32 * kPassThreads;
    const size_t have = sizeof(float) * (size_t)kSub * pass_ustride(kmax, calib);
    if (need > have) o += need - have;
  }
  s.parts = o; o += sizeof(float) * (size_t)nparts * kmax * kSub;
  s.dcs = o; o += sizeof(float) * kSub;
  s.dns = o; o += sizeof(float) * kSub;
  s.qc = o; o += sizeof(float2) * kSub;
  s.qn = o; o += sizeof(float2) * kSub;
  s.ebuf = o; o += sizeof(double) * kPassWarps * kEdgeSlots * 32;
  s.emap = o; o += sizeof(int) * kPassWarps * kEdgeSlots;
  s.sflow = o; o += sizeof(int) * kmax;
  o = (o + 15) & ~size_t(15);
  s.sl = o; o += sizeof(EdgeLin) * kmax;
  s.sb = o; o += sizeof(EdgeBack) * kmax;
  s.total = (o + 15) & ~size_t(15);
  return s;
}

// packed fp32x2 FMA (sm_100): lanes (lo, hi) each fmaf-rounded
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long splat2(float a) {
  const unsigned long long u = __float_as_uint(a);
  return u | (u << 32);
}
__device__ __forceinline__ unsigned long long pack2(float2 v) {
  return (unsigned long long)__float_as_uint(v.x) | ((unsigned long long)__float_as_uint(v.y) << 32);
}

// per edge-pixel geometry at one state
struct PixTerms {
  bool ok;
  float xt, yt, iz, ru, rv, wu, wv;
};

__device__ __forceinline__ PixTerms pix_terms(const float R[9], const float t[3], float qx, float qy, float d,
                                              float fx, float fy, float cx, float cy, float Wf, float Hf,
                                              const float4& fw, bool in) {
  PixTerms o;
  const float X = fmaf(R[0], qx, fmaf(R[1], qy, R[2])) + t[0] * d;
  const float Y = fmaf(R[3], qx, fmaf(R[4], qy, R[5])) + t[1] * d;
  const float Z = fmaf(R[6], qx, fmaf(R[7], qy, R[8])) + t[2] * d;
  bool ok = in && Z > 1e-4f * d;
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(Z));  // <= 1 ulp; Z > 0 here
  o.iz = ok ? r : 0.f;
  o.xt = X * o.iz;
  o.yt = Y * o.iz;
  const float pu = fmaf(fx, o.xt, cx), pv = fmaf(fy, o.yt, cy);
  ok = ok && pu >= -1e-9f && pu <= Wf + 1e-9f && pv >= -1e-9f && pv <= Hf + 1e-9f;
  o.ok = ok;
  o.wu = ok ? fw.z : 0.f;
  o.wv = ok ? fw.w : 0.f;
  o.ru = ok ? fw.x - pu : 0.f;
  o.rv = ok ? fw.y - pv : 0.f;
  return o;
}

template <bool CALIB>
__global__ void __launch_bounds__(kPassThreads, 1) pass_kernel(const PassArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  if (A.runs && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(A.runs, 1ull);
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NVE = kEdgeVals + (CALIB ? kCalibVals : 0);
  const PassSmem L = pass_smem_layout(A.kmax, CALIB, A.stage != 0);
  float4* fbuf = reinterpret_cast<float4*>(smem + L.fbuf);  // [k][kSub] flow records
  float* U = reinterpret_cast<float*>(smem + L.U);
  float* Mg = reinterpret_cast<float*>(smem + L.U);  // segment end only: [32][kPassThreads]
  float* parts = reinterpret_cast<float*>(smem + L.parts);
  float* dcs = reinterpret_cast<float*>(smem + L.dcs);
  float* dns = reinterpret_cast<float*>(smem + L.dns);
  float2* qcs = reinterpret_cast<float2*>(smem + L.qc);  // normalised pixel rays at x_c
  float2* qns = reinterpret_cast<float2*>(smem + L.qn);  // ... at x_n
  double* ebuf = reinterpret_cast<double*>(smem + L.ebuf);
  double* ethb = reinterpret_cast<double*>(smem + L.ethb);
  double* red = reinterpret_cast<double*>(smem + L.red);
  int* emap = reinterpret_cast<int*>(smem + L.emap);
  int* sflow = reinterpret_cast<int*>(smem + L.sflow);
  EdgeLin* sl = reinterpret_cast<EdgeLin*>(smem + L.sl);
  EdgeBack* sb = reinterpret_cast<EdgeBack*>(smem + L.sb);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int P = A.P, KM = A.kmax;
  const float Wf = (float)A.W, Hf = (float)A.H;
  const float fxn = (float)A.intr_n[0], fyn = (float)A.intr_n[1];
  const float cxn = (float)A.intr_n[2], cyn = (float)A.intr_n[3];
  const float fxc = (float)A.intr_c[0], fyc = (float)A.intr_c[1];
  const float cxc = (float)A.intr_c[2], cyc = (float)A.intr_c[3];
  const float dth[4] = {(float)(A.intr_n[0] - A.intr_c[0]), (float)(A.intr_n[1] - A.intr_c[1]),
                        (float)(A.intr_n[2] - A.intr_c[2]), (float)(A.intr_n[3] - A.intr_c[3])};

  for (int sg = A.cta_seg[blockIdx.x]; sg < A.cta_seg[blockIdx.x + 1]; ++sg) {
    const int fl = A.seg_frame[sg];
    const int s0 = A.csr_off[fl];
    const int k = A.csr_off[fl + 1] - s0;
    const int f = A.frame_of[fl];
    const int mu = pass_mu(k, CALIB);
    const int mext = mu + 2;
    const int mpad = (mext + 7) & ~7;
    const int ustride = mpad + 2;
    float* Pa0 = parts;                  // [k][kSub]  C part
    float* Pa1 = parts + KM * kSub;      // [k][kSub]  g_d part
    float* Pth = parts + 2 * KM * kSub;  // [4][k][kSub] E_theta parts (phase B, calib)

    // ---- stage per-edge constants, unit -> edge slots
    for (int x = tid; x < k * (int)(sizeof(EdgeLin) / 4); x += kPassThreads)
      reinterpret_cast<float*>(sl)[x] = reinterpret_cast<const float*>(A.lin + s0)[x];
    if (A.backsub)
      for (int x = tid; x < k * (int)(sizeof(EdgeBack) / 4); x += kPassThreads)
        reinterpret_cast<float*>(sb)[x] = reinterpret_cast<const float*>(A.back + s0)[x];
    for (int x = tid; x < k; x += kPassThreads) sflow[x] = A.slot_flow[s0 + x];
    const int nunit = k * kSlices;
    const int u0 = (nunit * warp) / kPassWarps, u1 = (nunit * (warp + 1)) / kPassWarps;
    const int e0 = u0 / kSlices;  // slot s holds edge e0 + s
    if (lane < kEdgeSlots) {
      const int e = e0 + lane;
      emap[warp * kEdgeSlots + lane] = (u1 > u0 && e * kSlices < u1 && e < k) ? e : -1;
    }
    for (int x = tid; x < kPassWarps * kEdgeSlots * 32; x += kPassThreads) {
      ebuf[x] = 0.0;
      if (CALIB) ethb[x] = 0.0;
    }
    // GEMM assignment: 4x8 tiles touching the upper triangle x pixel groups
    const int nr = mpad >> 2;
    const int ntiles = pass_ntiles(mpad);
    const int G = A.system ? max(1, min(16, kPassThreads / max(ntiles, 1))) : 0;
    int tI = -1, tJ = -1, gk0 = 0, gk1 = 0;
    if (A.system && tid < G * ntiles) {
      int t = tid % ntiles;
      const int g = tid / ntiles;
      int tj = 0;
      while (t >= min(2 * tj + 2, nr)) {
        t -= min(2 * tj + 2, nr);
        ++tj;
      }
      tI = t;
      tJ = tj;
      gk0 = (kSub * g) / G;
      gk1 = (kSub * (g + 1)) / G;
    }
    // GEMM accumulators as float pairs: Macc2[4 r + q] = (M[r][2q], M[r][2q+1]) of the
    // thread's 4x8 tile, updated with packed FFMA2 (two fp32 FMAs per instruction,
    // each rounded exactly like FFMA)
    unsigned long long Macc2[16];
#pragma unroll
    for (int x = 0; x < 16; ++x) Macc2[x] = 0ull;
    float hacc[kEdgeSlots][28];  // per-edge H_jj, g_j, energy of this warp's units (whole segment)
#pragma unroll
    for (int s = 0; s < kEdgeSlots; ++s)
#pragma unroll
      for (int x = 0; x < 28; ++x) hacc[s][x] = 0.f;
    float facc[15];  // energy, H_tt (10), g_t (4)
#pragma unroll
    for (int x = 0; x < 15; ++x) facc[x] = 0.f;
    float fpri = 0.f;  // scalefix: sum_p d_p alpha m_p (d*_p - d_p) (the prior's gradient along the scale)
    // A5: kappa = (rho - h . delta_local) / gamma from the x_c linearisation
    const bool gauge = (f == A.gauge_frame) && k > 0;
    __syncthreads();
    double kappa = 0.0;
    if (gauge && A.backsub) {
      const double* gs = A.gstate_c;
      double hd = 0.0;
      for (int a = 0; a < k; ++a)
        for (int q = 0; q < 6; ++q) hd += gs[2 + 6 * a + q] * (double)sb[a].dlt[q];
      if (CALIB)
        for (int q = 0; q < 4; ++q) hd += gs[2 + 6 * k + q] * (A.intr_n[q] - A.intr_c[q]);
      kappa = (gs[1] - hd) / gs[0];
    }

    // cp.async staging of a sub-tile's flow records (16 B each) and disparities;
    // out-of-range pixels are zero-filled
    auto prefetch = [&](int tile) {
      const int pb = tile * kSub;
      for (int x = tid; x < k * kSub; x += kPassThreads) {
        const int a = x >> 8, pl = x & (kSub - 1), p = pb + pl;
        const float4* src = A.flow + (size_t)sflow[a] * P + (p < P ? p : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(fbuf + x);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                     "r"(p < P ? 16 : 0));
      }
      if (tid < kSub) {
        const int p = pb + tid;
        const float* src = A.d_cur + (size_t)f * P + (p < P ? p : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(dcs + tid);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(p < P ? 4 : 0));
      }
      asm volatile("cp.async.commit_group;");
    };
    if (A.stage) prefetch(A.seg_t0[sg]);

    for (int tile = A.seg_t0[sg]; tile < A.seg_t1[sg]; ++tile) {
      const int pbase = tile * kSub;
      if (A.stage) asm volatile("cp.async.wait_all;" ::: "memory");
      if (tid < kSub) {
        const int p = pbase + tid;
        if (!A.stage) dcs[tid] = p < P ? A.d_cur[(size_t)f * P + p] : 0.f;
        const float pu = (float)(p % A.W), pv = (float)(p / A.W);
        qcs[tid] = make_float2((pu - cxc) / fxc, (pv - cyc) / fyc);
        qns[tid] = make_float2((pu - cxn) / fxn, (pv - cyn) / fyn);
      }
      __syncthreads();
      // ------------------------------------------------------------ phase A
      // pixel-major: a half-warp per 16 pixels, the two halves split the edges; the
      // per-pixel sums close with one shuffle, so d_n needs no block barrier
      if (A.backsub && !A.freeze) {
        const int pl = 16 * warp + (lane & 15), p = pbase + pl, eg = lane >> 4;
        const bool in = p < P;
        const float dc = dcs[pl];
        const float2 q = qcs[pl];
        const float qx = q.x, qy = q.y;
        float Cp = 0.f, gdp = 0.f, accp = 0.f;
#ifndef DBA_PASS_SKIP_A
        for (int a = eg; a < k; a += 2) {
          const EdgeBack& e = sb[a];
          const float4 fw = A.stage ? fbuf[a * kSub + pl]
                                    : (in ? __ldg(A.flow + (size_t)sflow[a] * P + p) : make_float4(0.f, 0.f, 0.f, 0.f));
          const PixTerms T = pix_terms(e.R, e.t, qx, qy, dc, fxc, fyc, cxc, cyc, Wf, Hf, fw, in);
          const float fxi = fxc * T.iz, fyi = fyc * T.iz;
          const float Jdu = fxi * (e.t[0] - T.xt * e.t[2]);
          const float Jdv = fyi * (e.t[1] - T.yt * e.t[2]);
          const float* dl = e.dlt;
          float ju = fxi * dc * (dl[0] - T.xt * dl[2]) +
                     fxc * (-T.xt * T.yt * dl[3] + (1.f + T.xt * T.xt) * dl[4] - T.yt * dl[5]);
          float jv = fyi * dc * (dl[1] - T.yt * dl[2]) +
                     fyc * (-(1.f + T.yt * T.yt) * dl[3] + T.xt * T.yt * dl[4] + T.xt * dl[5]);
          if (CALIB) {
            const float cu0 = T.iz * (e.R[0] - T.xt * e.R[6]), cu1 = T.iz * (e.R[1] - T.xt * e.R[7]);
            const float cv0 = T.iz * (e.R[3] - T.yt * e.R[6]), cv1 = T.iz * (e.R[4] - T.yt * e.R[7]);
            ju += (T.xt - cu0 * qx) * dth[0] + (-cu1 * qy * fxc / fyc) * dth[1] + (1.f - cu0) * dth[2] +
                  (-cu1 * fxc / fyc) * dth[3];
            jv += (-cv0 * qx * fyc / fxc) * dth[0] + (T.yt - cv1 * qy) * dth[1] +
                  (-cv0 * fyc / fxc) * dth[2] + (1.f - cv1) * dth[3];
          }
          const float au = T.wu * Jdu, av = T.wv * Jdv;
          Cp += fmaf(au, Jdu, av * Jdv);
          gdp += fmaf(au, T.ru, av * T.rv);
          accp += fmaf(au, ju, av * jv);
        }
#endif
        // edge-group halves in fixed order: (even edges) + (odd edges)
        const float Co = __shfl_xor_sync(0xffffffffu, Cp, 16);
        const float go = __shfl_xor_sync(0xffffffffu, gdp, 16);
        const float ao = __shfl_xor_sync(0xffffffffu, accp, 16);
        if (eg == 0) {
          if (in) {
            float C = A.eta + (Cp + Co), gd = gdp + go, acc = accp + ao;
            if (A.prior != nullptr) {
              const size_t fp = (size_t)f * P + p;
              const float ap = A.alpha * (A.pweight ? A.pweight[f] : 1.f) * (float)A.pmask[fp];
              C += ap;
              gd += ap * (A.prior[fp] - dc);
            }
            float dd = (gd - acc) / C;
            if (gauge) dd -= (float)(kappa / (double)dc);  // A5: r/C - kappa/d
            const float dn = fmaxf(dc + dd, A.d_min);
            dns[pl] = dn;
            A.d_new[(size_t)f * P + p] = dn;
          } else {
            dns[pl] = 1.f;
          }
        }
      } else if (tid < kSub) {
        const int p = pbase + tid;
        dns[tid] = dcs[tid];
        if (p < P) A.d_new[(size_t)f * P + p] = dcs[tid];
      }
      __syncthreads();
      // ------------------------------------------------------------ phase B
#ifdef DBA_PASS_SKIP_B
      for (int u = u0; u < u0; ++u) {
#else
      for (int u = u0; u < u1; ++u) {
#endif
        const int a = u / kSlices, sl0 = (u % kSlices) * kSlice;
        const int slot = a - e0;
        (void)sl0;
        const EdgeLin& e = sl[a];
        const float4* fl4 = A.flow + (size_t)sflow[a] * P;
        float ct[24];
        if (CALIB) {
#pragma unroll
          for (int x = 0; x < 24; ++x) ct[x] = 0.f;
        }
        {
          const int pl = sl0 + lane, p = pbase + pl;
          const bool in = p < P;
          const float4 fw = A.stage ? fbuf[a * kSub + pl]
                                    : (in ? __ldg(fl4 + p) : make_float4(0.f, 0.f, 0.f, 0.f));
          const float dn = dns[pl];
          const float2 q = qns[pl];
          const float qx = q.x, qy = q.y;
          const PixTerms T = pix_terms(e.R, e.t, qx, qy, dn, fxn, fyn, cxn, cyn, Wf, Hf, fw, in);
          const float en = T.wu * T.ru * T.ru + T.wv * T.rv * T.rv;
          facc[0] += en;
          if (!A.system) continue;
          const float fxi = fxn * T.iz, fyi = fyn * T.iz;
          float Ju[6], Jv[6];
          Ju[0] = fxi * dn;
          Ju[1] = 0.f;
          Ju[2] = -fxi * dn * T.xt;
          Ju[3] = -fxn * T.xt * T.yt;
          Ju[4] = fxn * (1.f + T.xt * T.xt);
          Ju[5] = -fxn * T.yt;
          Jv[0] = 0.f;
          Jv[1] = fyi * dn;
          Jv[2] = -fyi * dn * T.yt;
          Jv[3] = -fyn * (1.f + T.yt * T.yt);
          Jv[4] = fyn * T.xt * T.yt;
          Jv[5] = fyn * T.xt;
          const float Jdu = fxi * (e.t[0] - T.xt * e.t[2]);
          const float Jdv = fyi * (e.t[1] - T.yt * e.t[2]);
          const float au = T.wu * Jdu, av = T.wv * Jdv;
          Pa0[a * kSub + pl] = fmaf(au, Jdu, av * Jdv);
          Pa1[a * kSub + pl] = fmaf(au, T.ru, av * T.rv);
          float2* U2 = reinterpret_cast<float2*>(U + pl * ustride + 6 * a);
          U2[0] = make_float2(fmaf(au, Ju[0], av * Jv[0]), fmaf(au, Ju[1], av * Jv[1]));
          U2[1] = make_float2(fmaf(au, Ju[2], av * Jv[2]), fmaf(au, Ju[3], av * Jv[3]));
          U2[2] = make_float2(fmaf(au, Ju[4], av * Jv[4]), fmaf(au, Ju[5], av * Jv[5]));
          // per-edge H_jj (upper 21), g_j (6), energy into this slot's registers
#pragma unroll
          for (int s = 0; s < kEdgeSlots; ++s) {
            if (s != slot) continue;
            // J_u[1] = 0 and J_v[0] = 0: the structurally zero terms are skipped
            // (H_01 has none), which leaves every other sum unchanged bit for bit
            int o = 0;
#pragma unroll
            for (int r = 0; r < 6; ++r)
#pragma unroll
              for (int c = r; c < 6; ++c) {
                const bool zu = r == 1 || c == 1, zv = r == 0 || c == 0;
                if (!zu && !zv)
                  hacc[s][o] = fmaf(T.wu * Ju[r], Ju[c], fmaf(T.wv * Jv[r], Jv[c], hacc[s][o]));
                else if (!zu)
                  hacc[s][o] = fmaf(T.wu * Ju[r], Ju[c], hacc[s][o]);
                else if (!zv)
                  hacc[s][o] = fmaf(T.wv * Jv[r], Jv[c], hacc[s][o]);
                ++o;
              }
#pragma unroll
            for (int r = 0; r < 6; ++r) {
              if (r == 0)
                hacc[s][21 + r] = fmaf(T.wu * T.ru, Ju[r], hacc[s][21 + r]);
              else if (r == 1)
                hacc[s][21 + r] = fmaf(T.wv * T.rv, Jv[r], hacc[s][21 + r]);
              else
                hacc[s][21 + r] = fmaf(T.wu * T.ru, Ju[r], fmaf(T.wv * T.rv, Jv[r], hacc[s][21 + r]));
            }
            hacc[s][27] += en;
          }
          if (CALIB) {
            // J_theta = d(u,v)/d(fx,fy,cx,cy) through unprojection and projection
            const float cu0 = T.iz * (e.R[0] - T.xt * e.R[6]), cu1 = T.iz * (e.R[1] - T.xt * e.R[7]);
            const float cv0 = T.iz * (e.R[3] - T.yt * e.R[6]), cv1 = T.iz * (e.R[4] - T.yt * e.R[7]);
            float Tu[4], Tv[4];
            Tu[0] = T.xt - cu0 * qx;
            Tu[1] = -cu1 * qy * fxn / fyn;
            Tu[2] = 1.f - cu0;
            Tu[3] = -cu1 * fxn / fyn;
            Tv[0] = -cv0 * qx * fyn / fxn;
            Tv[1] = T.yt - cv1 * qy;
            Tv[2] = -cv0 * fyn / fxn;
            Tv[3] = 1.f - cv1;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = 0; c < 6; ++c)
                ct[6 * r + c] = fmaf(T.wu * Tu[r], Ju[c], fmaf(T.wv * Tv[r], Jv[c], ct[6 * r + c]));
            int q = 1;
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
              for (int c = r; c < 4; ++c) {
                facc[q] = fmaf(T.wu * Tu[r], Tu[c], fmaf(T.wv * Tv[r], Tv[c], facc[q]));
                ++q;
              }
#pragma unroll
            for (int r = 0; r < 4; ++r)
              facc[11 + r] = fmaf(T.wu * T.ru, Tu[r], fmaf(T.wv * T.rv, Tv[r], facc[11 + r]));
#pragma unroll
            for (int r = 0; r < 4; ++r) Pth[(r * KM + a) * kSub + pl] = fmaf(au, Tu[r], av * Tv[r]);
          }
        }
        if (CALIB && A.system) {
          float v32[32];
#pragma unroll
          for (int x = 0; x < 24; ++x) v32[x] = ct[x];
#pragma unroll
          for (int x = 24; x < 32; ++x) v32[x] = 0.f;
          const float rs = transpose_reduce32(v32, lane);
          ethb[(warp * kEdgeSlots + slot) * 32 + lane] += (double)rs;
        }
      }
      __syncthreads();
      if (A.stage && tile + 1 < A.seg_t1[sg]) prefetch(tile + 1);  // overlaps the GEMM
      // ------------------------------------------------------------ per pixel
      // two threads per pixel: both form C_p, g_d,p; each scales half of the row
      {
        const int pl = tid & (kSub - 1), half = tid >> 8;
        const int p = pbase + pl;
        const bool in = p < P;
        float* Urow = U + pl * ustride;
        float C = A.eta, gd = 0.f;
        if (A.system) {
          for (int a = 0; a < k; ++a) {
            C += Pa0[a * kSub + pl];
            gd += Pa1[a * kSub + pl];
          }
        }
        const float dn = dns[pl];
        float ap = 0.f;
        if (A.prior != nullptr && in) {
          const size_t fp = (size_t)f * P + p;
          ap = A.alpha * (A.pweight ? A.pweight[f] : 1.f) * (float)A.pmask[fp];
          const float dd = A.prior[fp] - dn;
          C += ap;
          gd += ap * dd;
          if (half == 0) {
            facc[0] += ap * dd * dd;
            fpri = fmaf(dn * ap, dd, fpri);
          }
        }
        if (A.system) {
          // V = U_ext / sqrt(C): the GEMM below is then M_ext = V V^T
          const float sq = (in && !A.freeze) ? rsqrtf(C) : 0.f;  // frozen d: no fill-in
          float2* U2 = reinterpret_cast<float2*>(Urow);
          const int ne = 3 * k;  // float2 columns of the edge rows
          const int c0 = half ? ne / 2 : 0, c1 = half ? ne : ne / 2;
          for (int c = c0; c < c1; ++c) {
            const float2 v = U2[c];
            U2[c] = make_float2(v.x * sq, v.y * sq);
          }
          if (half) {
            if (CALIB) {
              float Et[4] = {0.f, 0.f, 0.f, 0.f};
              for (int a = 0; a < k; ++a)
#pragma unroll
                for (int r = 0; r < 4; ++r) Et[r] += Pth[(r * KM + a) * kSub + pl];
              U2[ne] = make_float2(Et[0] * sq, Et[1] * sq);
              U2[ne + 1] = make_float2(Et[2] * sq, Et[3] * sq);
            }
            // second extra column: A5 gauge c = C/d, or (scalefix) c = d (eta + alpha m), whose
            // E C^-1 c is the reduced system's exact row along the monocular scale direction
            const float cx = A.scalefix ? dn * (A.eta + ap) : C / dn;
            U2[mu >> 1] = make_float2(gd * sq, in ? cx * sq : 0.f);
            for (int c = (mext >> 1); c < (mpad >> 1); ++c) U2[c] = make_float2(0.f, 0.f);
          }
        }
      }
      __syncthreads();
      if (!A.system) continue;
      // ------------------------------------------------------------ phase C (K3a)
#ifdef DBA_PASS_SKIP_GEMM
      if (tI >= 0 && tI < -1) {
#else
      if (tI >= 0) {
#endif
        const int ca = 4 * tI, cb = 8 * tJ;
#pragma unroll 2
        for (int pp = gk0; pp < gk1; ++pp) {
          const float2* row = reinterpret_cast<const float2*>(U + pp * ustride);
          const float2 a0 = row[(ca >> 1)], a1 = row[(ca >> 1) + 1];
          const float2 b0 = row[(cb >> 1)], b1 = row[(cb >> 1) + 1], b2 = row[(cb >> 1) + 2],
                       b3 = row[(cb >> 1) + 3];
          const float av[4] = {a0.x, a0.y, a1.x, a1.y};
          const unsigned long long bp[4] = {pack2(b0), pack2(b1), pack2(b2), pack2(b3)};
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 4; ++q) Macc2[4 * r + q] = ffma2(splat2(av[r]), bp[q], Macc2[4 * r + q]);
        }
      }
      __syncthreads();
    }

    // ------------------------------------------------------------ segment outputs
    if (A.system) {
      // per-edge register accumulators: one transpose-reduce per slot per segment
#pragma unroll
      for (int s = 0; s < kEdgeSlots; ++s) {
        float v32[32];
#pragma unroll
        for (int x = 0; x < 28; ++x) v32[x] = hacc[s][x];
#pragma unroll
        for (int x = 28; x < 32; ++x) v32[x] = 0.f;
        const float rs = transpose_reduce32(v32, lane);
        ebuf[(warp * kEdgeSlots + s) * 32 + lane] = (double)rs;
      }
      // GEMM partials of every (tile, pixel group) thread -> Mg[x][tid] (aliases U)
      if (tI >= 0) {
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          const unsigned long long v = Macc2[x >> 1];
          Mg[x * kPassThreads + tid] = __uint_as_float((unsigned)((x & 1) ? (v >> 32) : v));
        }
      }
    }
    // per-frame values: fixed-order block reduction (float64 across warps)
#pragma unroll
    for (int x = 0; x < 15; ++x) {
      float v = facc[x];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[warp * 16 + x] = (double)v;
    }
    {
      double v = (double)fpri;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[warp * 16 + 15] = v;
    }
    __syncthreads();
    double* pf = A.part_frame + (long long)sg * kFrameVals;
    if (tid < kFrameVals) {
      double v = 0.0;
      if (tid < 15)
        for (int w = 0; w < kPassWarps; ++w) v += red[w * 16 + tid];
      if (tid == 17)
        for (int w = 0; w < kPassWarps; ++w) v += red[w * 16 + 15];
      pf[tid] = v;  // [15], [16] (gamma, rho) are overwritten below when system
    }
    if (A.system) {
      double* pe = A.part_edge + A.seg_off_edge[sg];
      for (int x = tid; x < k * NVE; x += kPassThreads) {
        const int a = x / NVE, l = x % NVE;
        double v = 0.0;
        for (int ws = 0; ws < kPassWarps * kEdgeSlots; ++ws)
          if (emap[ws] == a) v += (l < 32) ? ebuf[ws * 32 + l] : ethb[ws * 32 + (l - 32)];
        pe[x] = v;
      }
      // unpack: M (mu x mu), w = column mu, h = column mu+1, rho, gamma;
      // each entry sums its tile's pixel groups in fixed order (float64)
      double* pM = A.part_M + A.seg_off_M[sg];
      double* pw = A.part_w + A.seg_off_w[sg];
      for (int x = tid; x < mext * mext; x += kPassThreads) {
        const int R = x / mext, Cc = x % mext;
        const int lo = min(R, Cc), hi = max(R, Cc);
        const int ti = lo >> 2, tj = hi >> 3;
        // tiles are enumerated column block by column block: sum_{j<tj} min(2j+2, nr)
        const int full = min(tj, (nr - 1) / 2);  // blocks with 2j+2 <= nr
        const int t = ti + full * (full + 1) + (tj - full) * nr;
        const int e = 8 * (lo & 3) + (hi & 7);
        double v = 0.0;
        for (int g = 0; g < G; ++g) v += (double)Mg[e * kPassThreads + g * ntiles + t];
        if (R < mu && Cc < mu)
          pM[(long long)R * mu + Cc] = v;
        else if (R < mu && Cc == mu)
          pw[R] = v;
        else if (R < mu && Cc == mu + 1)
          pw[mu + R] = v;
        else if (R == mu && Cc == mu + 1)
          pf[16] = v;  // rho
        else if (R == mu + 1 && Cc == mu + 1)
          pf[15] = v;  // gamma
      }
    }
    __syncthreads();
  }  // segments
}

}  // namespace dba
