// K1+K2+K3a(+K5): the fused per-frame pass of one Gauss-Newton trial.
//
// One CTA owns (source frame i, a contiguous range of 256-pixel sub-tiles) and
// ALL out-edges of frame i, so every per-pixel disparity term (C_p, g_d,p and
// the pose/disparity couplings E_e,p) stays on chip:
//
//   phase A (back-substitution at x_c, skipped on the first pass):
//       for e in out(i): recompute J_d, J_j.delta_e at x_c from the flow record
//       delta d_p = (g_d,p - sum_e E_e,p . delta_e) / C_p ;  d_n = max(d + delta d, d_min)
//   phase B (linearisation at x_n = trial state):
//       for e in out(i): residual, validity (geometry.py:235-250), J_j, J_d,
//       [J_theta]; energy; per-edge H_jj / g_j (warp transpose-reduce);
//       E_e,p -> shared U[p][6e..6e+5]; C_p, g_d,p
//   phase C (Schur fill-in, K3a): M += U^T diag(1/C) U,  w += U^T (g_d / C)
//       as a shared-memory SIMT GEMM over the sub-tile's pixels.
//
// The flow record (tu, tv, wu, wv) is read as one coalesced float4 per
// edge-pixel (16 B, the algorithmic traffic of the path); phase B re-reads it
// from L1/L2.  Pose-block Jacobians use homogeneous coordinates
// X~ = R q + t d (q = ((u-cx)/fx, (v-cy)/fy, 1)):
//   J_u = fx [d/Z, 0, -d x/Z, -x y, 1 + x^2, -y]
//   J_v = fy [0, d/Z, -d y/Z, -(1 + y^2), x y, x]
//   J_d = (fx (t_x - x t_z)/Z, fy (t_y - y t_z)/Z)
// which equal the oracle's non-homogeneous J_j = J_pi(X_j)[I | -[X_j]x] and
// J_d = J_pi(X_j) R (-X_i/d) (oracle/dba.py edge_terms).  J_i = -J_j Ad(G_ij)
// is never formed per pixel; the adjoint is applied per edge in assemble.
// Partials leave the CTA in float64; every reduction has a fixed order.
#pragma once

#include "dba_common.cuh"

namespace dba {

struct PassArgs {
  int H, W, P, n_tiles, kmax;
  int backsub;  // run phase A
  int system;   // produce system partials (0: energy only)
  const int* status;  // abort when status[0] != 0 (failed factorisation)
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
__host__ __device__ inline int pass_mpad(int k, bool calib) { return (pass_mu(k, calib) + 3) & ~3; }
__host__ __device__ inline int pass_ustride(int k, bool calib) { return pass_mpad(k, calib) + 2; }

// dynamic shared memory layout (bytes), identical on host and device
struct PassSmem {
  size_t eacc, stage, U, cinv, gdc, hcs, red, sl, sb, total;
};
__host__ __device__ inline PassSmem pass_smem_layout(int kmax, bool calib) {
  PassSmem s;
  const int nve = kEdgeVals + (calib ? kCalibVals : 0);
  size_t o = 0;
  s.eacc = o; o += sizeof(double) * (size_t)kmax * nve;
  s.red = o; o += sizeof(double) * 8 * kFrameVals;
  s.stage = o; o += sizeof(float) * 8 * (size_t)kmax * nve;
  s.U = o; o += sizeof(float) * (size_t)kBlock * pass_ustride(kmax, calib);
  s.cinv = o; o += sizeof(float) * kBlock;
  s.gdc = o; o += sizeof(float) * kBlock;
  s.hcs = o; o += sizeof(float) * kBlock;
  o = (o + 15) & ~size_t(15);
  s.sl = o; o += sizeof(EdgeLin) * kmax;
  s.sb = o; o += sizeof(EdgeBack) * kmax;
  s.total = (o + 15) & ~size_t(15);
  return s;
}

template <bool CALIB, int MT>
__global__ void __launch_bounds__(kBlock, 1) pass_kernel(const PassArgs A) {
  if (A.status != nullptr && A.status[0] != 0) return;
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NVE = kEdgeVals + (CALIB ? kCalibVals : 0);
  const PassSmem L = pass_smem_layout(A.kmax, CALIB);
  double* eacc = reinterpret_cast<double*>(smem + L.eacc);
  double* red = reinterpret_cast<double*>(smem + L.red);
  float* stage = reinterpret_cast<float*>(smem + L.stage);
  float* U = reinterpret_cast<float*>(smem + L.U);
  float* cinv = reinterpret_cast<float*>(smem + L.cinv);
  float* gdc = reinterpret_cast<float*>(smem + L.gdc);
  float* hcs = reinterpret_cast<float*>(smem + L.hcs);
  EdgeLin* sl = reinterpret_cast<EdgeLin*>(smem + L.sl);
  EdgeBack* sb = reinterpret_cast<EdgeBack*>(smem + L.sb);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int sg = A.cta_seg[blockIdx.x]; sg < A.cta_seg[blockIdx.x + 1]; ++sg) {
  const int fl = A.seg_frame[sg];
  const int s0 = A.csr_off[fl];
  const int k = A.csr_off[fl + 1] - s0;
  const int f = A.frame_of[fl];
  const int mu = pass_mu(k, CALIB);
  const int mpad = pass_mpad(k, CALIB);
  const int ustride = mpad + 2;
  const int P = A.P;
  const float Wf = (float)A.W, Hf = (float)A.H;

  // stage per-edge constants
  for (int x = tid; x < k * (int)(sizeof(EdgeLin) / 4); x += kBlock)
    reinterpret_cast<float*>(sl)[x] = reinterpret_cast<const float*>(A.lin + s0)[x];
  if (A.backsub)
    for (int x = tid; x < k * (int)(sizeof(EdgeBack) / 4); x += kBlock)
      reinterpret_cast<float*>(sb)[x] = reinterpret_cast<const float*>(A.back + s0)[x];
  if (A.system)
    for (int x = tid; x < k * NVE; x += kBlock) eacc[x] = 0.0;
  __syncthreads();

  const float fxn = (float)A.intr_n[0], fyn = (float)A.intr_n[1];
  const float cxn = (float)A.intr_n[2], cyn = (float)A.intr_n[3];
  const float fxc = (float)A.intr_c[0], fyc = (float)A.intr_c[1];
  const float cxc = (float)A.intr_c[2], cyc = (float)A.intr_c[3];
  const float dfx = (float)(A.intr_n[0] - A.intr_c[0]);
  const float dfy = (float)(A.intr_n[1] - A.intr_c[1]);
  const float dcx = (float)(A.intr_n[2] - A.intr_c[2]);
  const float dcy = (float)(A.intr_n[3] - A.intr_c[3]);

  // upper-triangular 4x4 tiles of the (mpad x mpad) Schur block owned by this thread
  const int nt = mpad >> 2;
  const int ntiles = nt * (nt + 1) / 2;
  int tI[MT], tJ[MT];
#pragma unroll
  for (int s = 0; s < MT; ++s) {
    int t = tid + kBlock * s;
    tI[s] = -1;
    tJ[s] = -1;
    if (t < ntiles && A.system) {
      int r = 0;
      while (t >= nt - r) {
        t -= nt - r;
        ++r;
      }
      tI[s] = r;
      tJ[s] = r + t;
    }
  }
  double Macc[MT][16];
#pragma unroll
  for (int s = 0; s < MT; ++s)
#pragma unroll
    for (int x = 0; x < 16; ++x) Macc[s][x] = 0.0;
  double wacc = 0.0, hacc = 0.0;
  const bool gauge = (f == A.gauge_frame) && k > 0;
  // A5: kappa = (rho - h . delta_local) / gamma from the x_c linearisation
  double kappa = 0.0;
  if (gauge && A.backsub) {
    const double* gs = A.gstate_c;
    double hd = 0.0;
    for (int a = 0; a < k; ++a)
      for (int q = 0; q < 6; ++q) hd += gs[2 + 6 * a + q] * (double)sb[a].dlt[q];
    if (CALIB) {
      hd += gs[2 + 6 * k + 0] * (A.intr_n[0] - A.intr_c[0]) + gs[2 + 6 * k + 1] * (A.intr_n[1] - A.intr_c[1]) +
            gs[2 + 6 * k + 2] * (A.intr_n[2] - A.intr_c[2]) + gs[2 + 6 * k + 3] * (A.intr_n[3] - A.intr_c[3]);
    }
    kappa = (gs[1] - hd) / gs[0];
  }
  double facc[kFrameVals];
#pragma unroll
  for (int x = 0; x < kFrameVals; ++x) facc[x] = 0.0;
  __syncthreads();

  const int t0 = A.seg_t0[sg], t1 = A.seg_t1[sg];
  const float4* flow_f = A.flow;

  for (int tile = t0; tile < t1; ++tile) {
    const int p = tile * kBlock + tid;
    const bool in = p < P;
    const float pu0 = in ? (float)(p % A.W) : 0.f;
    const float pv0 = in ? (float)(p / A.W) : 0.f;
    const size_t fp = (size_t)f * P + (in ? p : 0);
    const float dc = in ? A.d_cur[fp] : 1.f;
    float dstar = 0.f, pm = 0.f;
    if (A.prior != nullptr && in) {
      dstar = A.prior[fp];
      pm = (float)A.pmask[fp];
    }
    float dn = dc;

    // ------------------------------------------------------------ phase A
    if (A.backsub) {
      const float qx = (pu0 - cxc) / fxc, qy = (pv0 - cyc) / fyc;
      float C = A.eta, gd = 0.f, acc = 0.f;
      for (int a = 0; a < k; ++a) {
        const EdgeBack& e = sb[a];
        const float4 fw = in ? __ldg(flow_f + (size_t)A.slot_flow[s0 + a] * P + p)
                             : make_float4(0.f, 0.f, 0.f, 0.f);
        const float X = fmaf(e.R[0], qx, fmaf(e.R[1], qy, e.R[2])) + e.t[0] * dc;
        const float Y = fmaf(e.R[3], qx, fmaf(e.R[4], qy, e.R[5])) + e.t[1] * dc;
        const float Z = fmaf(e.R[6], qx, fmaf(e.R[7], qy, e.R[8])) + e.t[2] * dc;
        bool ok = in && Z > 1e-4f * dc;
        const float iz = ok ? 1.f / Z : 0.f;
        const float xt = X * iz, yt = Y * iz;
        const float pu = fmaf(fxc, xt, cxc), pv = fmaf(fyc, yt, cyc);
        ok = ok && pu >= -1e-9f && pu <= Wf + 1e-9f && pv >= -1e-9f && pv <= Hf + 1e-9f;
        const float wu = ok ? fw.z : 0.f, wv = ok ? fw.w : 0.f;
        const float ru = ok ? fw.x - pu : 0.f, rv = ok ? fw.y - pv : 0.f;
        const float fxi = fxc * iz, fyi = fyc * iz;
        const float Jdu = fxi * (e.t[0] - xt * e.t[2]);
        const float Jdv = fyi * (e.t[1] - yt * e.t[2]);
        const float* dl = e.dlt;
        float ju = fxi * dc * (dl[0] - xt * dl[2]) +
                   fxc * (-xt * yt * dl[3] + (1.f + xt * xt) * dl[4] - yt * dl[5]);
        float jv = fyi * dc * (dl[1] - yt * dl[2]) +
                   fyc * (-(1.f + yt * yt) * dl[3] + xt * yt * dl[4] + xt * dl[5]);
        if (CALIB) {
          const float cu0 = iz * (e.R[0] - xt * e.R[6]), cu1 = iz * (e.R[1] - xt * e.R[7]);
          const float cv0 = iz * (e.R[3] - yt * e.R[6]), cv1 = iz * (e.R[4] - yt * e.R[7]);
          // J_theta rows at x_c (see phase B for the derivation)
          ju += (xt - cu0 * qx) * dfx + (-cu1 * qy * fxc / fyc) * dfy + (1.f - cu0) * dcx +
                (-cu1 * fxc / fyc) * dcy;
          jv += (-cv0 * qx * fyc / fxc) * dfx + (yt - cv1 * qy) * dfy +
                (-cv0 * fyc / fxc) * dcx + (1.f - cv1) * dcy;
        }
        const float au = wu * Jdu, av = wv * Jdv;
        C = fmaf(au, Jdu, fmaf(av, Jdv, C));
        gd = fmaf(au, ru, fmaf(av, rv, gd));
        acc = fmaf(au, ju, fmaf(av, jv, acc));
      }
      C += A.alpha * pm;
      gd += A.alpha * pm * (dstar - dc);
      float dd = (gd - acc) / C;
      if (gauge) dd -= (float)(kappa / (double)dc);  // A5: r/C - kappa/d
      if (in) dn = fmaxf(dc + dd, A.d_min);
    }
    if (in) A.d_new[fp] = dn;

    // ------------------------------------------------------------ phase B
    const float qx = (pu0 - cxn) / fxn, qy = (pv0 - cyn) / fyn;
    float C = A.eta, gd = 0.f;
    float Et[4] = {0.f, 0.f, 0.f, 0.f};
    float* Urow = U + tid * ustride;
    for (int a = 0; a < k; ++a) {
      const EdgeLin& e = sl[a];
      const float4 fw = in ? __ldg(flow_f + (size_t)A.slot_flow[s0 + a] * P + p)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      const float X = fmaf(e.R[0], qx, fmaf(e.R[1], qy, e.R[2])) + e.t[0] * dn;
      const float Y = fmaf(e.R[3], qx, fmaf(e.R[4], qy, e.R[5])) + e.t[1] * dn;
      const float Z = fmaf(e.R[6], qx, fmaf(e.R[7], qy, e.R[8])) + e.t[2] * dn;
      bool ok = in && Z > 1e-4f * dn;
      const float iz = ok ? 1.f / Z : 0.f;
      const float xt = X * iz, yt = Y * iz;
      const float pu = fmaf(fxn, xt, cxn), pv = fmaf(fyn, yt, cyn);
      ok = ok && pu >= -1e-9f && pu <= Wf + 1e-9f && pv >= -1e-9f && pv <= Hf + 1e-9f;
      const float wu = ok ? fw.z : 0.f, wv = ok ? fw.w : 0.f;
      const float ru = ok ? fw.x - pu : 0.f, rv = ok ? fw.y - pv : 0.f;
      const float en = wu * ru * ru + wv * rv * rv;
      facc[0] += (double)en;
      if (!A.system) continue;
      const float fxi = fxn * iz, fyi = fyn * iz;
      float Ju[6], Jv[6];
      Ju[0] = fxi * dn;
      Ju[1] = 0.f;
      Ju[2] = -fxi * dn * xt;
      Ju[3] = -fxn * xt * yt;
      Ju[4] = fxn * (1.f + xt * xt);
      Ju[5] = -fxn * yt;
      Jv[0] = 0.f;
      Jv[1] = fyi * dn;
      Jv[2] = -fyi * dn * yt;
      Jv[3] = -fyn * (1.f + yt * yt);
      Jv[4] = fyn * xt * yt;
      Jv[5] = fyn * xt;
      const float Jdu = fxi * (e.t[0] - xt * e.t[2]);
      const float Jdv = fyi * (e.t[1] - yt * e.t[2]);
      const float au = wu * Jdu, av = wv * Jdv;
      C = fmaf(au, Jdu, fmaf(av, Jdv, C));
      gd = fmaf(au, ru, fmaf(av, rv, gd));
      // E_e,p -> shared (conflict-free float2 stores: ustride = 2 * odd)
      float Ee[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) Ee[c] = fmaf(au, Ju[c], av * Jv[c]);
      float2* U2 = reinterpret_cast<float2*>(Urow + 6 * a);
      U2[0] = make_float2(Ee[0], Ee[1]);
      U2[1] = make_float2(Ee[2], Ee[3]);
      U2[2] = make_float2(Ee[4], Ee[5]);
      // per-edge H_jj (upper 21), g_j (6), energy -> warp transpose-reduce
      float v[32];
      int o = 0;
#pragma unroll
      for (int r = 0; r < 6; ++r)
#pragma unroll
        for (int c = r; c < 6; ++c) v[o++] = fmaf(wu * Ju[r], Ju[c], wv * Jv[r] * Jv[c]);
#pragma unroll
      for (int r = 0; r < 6; ++r) v[21 + r] = fmaf(wu * ru, Ju[r], wv * rv * Jv[r]);
      v[27] = en;
      v[28] = v[29] = v[30] = v[31] = 0.f;
      const float rs = transpose_reduce32(v, lane);
      stage[(warp * A.kmax + a) * NVE + lane] = rs;
      if (CALIB) {
        // J_theta = d(u,v)/d(fx,fy,cx,cy) through unprojection and projection:
        //   u = fx x + cx with X~ = R q(theta) + t d,  dq/dfx = (-qx/fx, 0, 0), ...
        const float cu0 = iz * (e.R[0] - xt * e.R[6]), cu1 = iz * (e.R[1] - xt * e.R[7]);
        const float cv0 = iz * (e.R[3] - yt * e.R[6]), cv1 = iz * (e.R[4] - yt * e.R[7]);
        float Tu[4], Tv[4];
        Tu[0] = xt - cu0 * qx;
        Tu[1] = -cu1 * qy * fxn / fyn;
        Tu[2] = 1.f - cu0;
        Tu[3] = -cu1 * fxn / fyn;
        Tv[0] = -cv0 * qx * fyn / fxn;
        Tv[1] = yt - cv1 * qy;
        Tv[2] = -cv0 * fyn / fxn;
        Tv[3] = 1.f - cv1;
        float c32[32];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 6; ++c) c32[6 * r + c] = fmaf(wu * Tu[r], Ju[c], wv * Tv[r] * Jv[c]);
#pragma unroll
        for (int x = 24; x < 32; ++x) c32[x] = 0.f;
        const float rc = transpose_reduce32(c32, lane);
        stage[(warp * A.kmax + a) * NVE + 32 + lane] = rc;
        // frame-level theta blocks
        int q = 1;
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = r; c < 4; ++c) facc[q++] += (double)fmaf(wu * Tu[r], Tu[c], wv * Tv[r] * Tv[c]);
#pragma unroll
        for (int r = 0; r < 4; ++r) facc[11 + r] += (double)fmaf(wu * ru, Tu[r], wv * rv * Tv[r]);
#pragma unroll
        for (int r = 0; r < 4; ++r) Et[r] = fmaf(au, Tu[r], fmaf(av, Tv[r], Et[r]));
      }
    }
    // disparity prior (Eq. 4)
    {
      const float dd = dstar - dn;
      const float ap = A.alpha * pm;
      C += ap;
      gd += ap * dd;
      facc[0] += (double)(ap * dd * dd);
    }
    if (!A.system) continue;
    if (CALIB) {
      float2* U2 = reinterpret_cast<float2*>(Urow + 6 * k);
      U2[0] = make_float2(Et[0], Et[1]);
      U2[1] = make_float2(Et[2], Et[3]);
    }
    for (int c = mu; c < mpad; ++c) Urow[c] = 0.f;
    if (!in) {
      for (int c = 0; c < mu; ++c) Urow[c] = 0.f;
    }
    cinv[tid] = in ? 1.f / C : 0.f;
    gdc[tid] = in ? gd / C : 0.f;
    if (gauge) {  // A5 with c = C/d: h = U^T (1/d), gamma = sum C/d^2, rho = sum g_d/d
      const float id = in ? 1.f / dn : 0.f;
      hcs[tid] = id;
      facc[15] += (double)(C * id * id);
      facc[16] += (double)(gd * id);
    }
    __syncthreads();

    // per-edge partials: sum the 8 warp rows, accumulate in float64
    for (int x = tid; x < k * NVE; x += kBlock) {
      const int a = x / NVE, l = x % NVE;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += stage[(w * A.kmax + a) * NVE + l];
      eacc[x] += (double)s;
    }

    // ------------------------------------------------------------ phase C (K3a)
#pragma unroll
    for (int s = 0; s < MT; ++s) {
      if (tI[s] < 0) continue;
      float acc[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) acc[x] = 0.f;
      const int ca = 4 * tI[s], cb = 4 * tJ[s];
#pragma unroll 4
      for (int pp = 0; pp < kBlock; ++pp) {
        const float* row = U + pp * ustride;
        const float2 a01 = *reinterpret_cast<const float2*>(row + ca);
        const float2 a23 = *reinterpret_cast<const float2*>(row + ca + 2);
        const float2 b01 = *reinterpret_cast<const float2*>(row + cb);
        const float2 b23 = *reinterpret_cast<const float2*>(row + cb + 2);
        const float ci = cinv[pp];
        const float av4[4] = {a01.x, a01.y, a23.x, a23.y};
        const float bv4[4] = {b01.x * ci, b01.y * ci, b23.x * ci, b23.y * ci};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[4 * r + c] = fmaf(av4[r], bv4[c], acc[4 * r + c]);
      }
#pragma unroll
      for (int x = 0; x < 16; ++x) Macc[s][x] += (double)acc[x];
    }
    if (tid < mu) {
      float s = 0.f, sh = 0.f;
      if (gauge) {
        for (int pp = 0; pp < kBlock; ++pp) {
          const float u = U[pp * ustride + tid];
          s = fmaf(u, gdc[pp], s);
          sh = fmaf(u, hcs[pp], sh);
        }
      } else {
        for (int pp = 0; pp < kBlock; ++pp) s = fmaf(U[pp * ustride + tid], gdc[pp], s);
      }
      wacc += (double)s;
      hacc += (double)sh;
    }
    __syncthreads();
  }

  // ------------------------------------------------------------ write partials
  if (A.system) {
    const int NV = NVE;
    double* pe = A.part_edge + A.seg_off_edge[sg];
    for (int x = tid; x < k * NV; x += kBlock) pe[x] = eacc[x];
    double* pM = A.part_M + A.seg_off_M[sg];
#pragma unroll
    for (int s = 0; s < MT; ++s) {
      if (tI[s] < 0) continue;
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int R = 4 * tI[s] + r, Cc = 4 * tJ[s] + c;
          if (R < mu && Cc < mu) {
            pM[(long long)R * mu + Cc] = Macc[s][4 * r + c];
            pM[(long long)Cc * mu + R] = Macc[s][4 * r + c];
          }
        }
    }
    if (tid < mu) {
      A.part_w[A.seg_off_w[sg] + tid] = wacc;
      A.part_w[A.seg_off_w[sg] + mu + tid] = hacc;
    }
  }
  // per-frame values: fixed-order block reduction in float64
#pragma unroll
  for (int x = 0; x < kFrameVals; ++x) {
    double v = facc[x];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp * kFrameVals + x] = v;
  }
  __syncthreads();
  if (tid < kFrameVals) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w * kFrameVals + tid];
    A.part_frame[(long long)sg * kFrameVals + tid] = v;
  }
  __syncthreads();
  }  // segments
}

}  // namespace dba
