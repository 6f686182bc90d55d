// Energy-only trial pass: back-substitution at x_c and the Eq. 3 (+ Eq. 4) energy at
// the trial state x_n, without Jacobians of x_n, per-edge Hessians or the Schur
// fill-in.  The LM controller only needs the trial energy to accept or reject; the
// full pass (pass_kernel) then linearises an ACCEPTED trial, so a rejected trial
// costs one solve plus this kernel.
//
// One thread per source-frame pixel, a CTA per 256-pixel tile of one frame: the
// thread walks the frame's out-edges twice (flow records staged in shared memory), first
// for delta d_p = (g_d,p - sum_e E_e,p . delta_e) / C_p (the
// same terms as pass_kernel phase A), then for the residual energy at
// (x_n, d_n).  No shared-memory pixel staging and no block barriers inside the
// pixel loop.  Per-CTA partial energies (float64, fixed-order tree) are summed by
// finalize in CTA order, so every energy the controller compares (including the
// initial one) comes from this kernel with one summation order.
#pragma once

#include "dba_pass.cuh"

namespace dba {

constexpr int kEnergyTile = 256;                   // pixels per CTA (one tile of one frame)
// pixels per thread: 2 and 4 (independent chains, fewer CTA-setup instructions) measured
// no faster than 1 (65.5 / 80.6 us vs 65.6 us on C3: fewer resident warps)
constexpr int kEnergyPx = 1;
constexpr int kEnergyThreads = kEnergyTile / kEnergyPx;

struct EnergyArgs {
  int H, W, P, tiles;  // tiles = ceil(P / kEnergyTile) per frame
  int kmax;
  int backsub, freeze;
  const int* status;
  const int* csr_off;
  const int* slot_flow;
  const int* frame_of;
  const EdgeLin* lin;
  const EdgeBack* back;
  const float4* flow;
  const float* d_cur;
  float* d_new;
  const float* prior;
  const uint8_t* pmask;
  const float* pweight;
  float alpha, eta, d_min;
  const double* intr_c;
  const double* intr_n;
  int gauge_frame;
  const double* gstate_c;
  double* part;  // (NL * tiles) per-CTA energies
};

// flow records of the thread's pixel are staged in shared memory (cp.async, one burst
// per CTA; reading them through L1 in both walks measured 72 us vs 66 us on C3); the
// compiled out-degree limit keeps the stage within 64 KB
static_assert(kMaxOutDegree <= 16, "energy_kernel stages kMaxOutDegree x 256 flow records");

__host__ __device__ inline size_t energy_smem_bytes(int kmax) {
  const size_t k = (size_t)(kmax > 0 ? kmax : 1);
  return (sizeof(float4) * kEnergyTile + sizeof(EdgeLin) + sizeof(EdgeBack) + sizeof(float4*)) * k;
}

// pix_terms with the hardware reciprocal (rcp.approx, <= 1 ulp): the energy walk
// only needs the residual and validity
__device__ __forceinline__ PixTerms pix_terms_e(const EdgeLin& e, float qx, float qy, float d, float fx, float fy,
                                                float cx, float cy, float Wf, float Hf, const float4& fw) {
  PixTerms o;
  const float X = fmaf(e.R[0], qx, fmaf(e.R[1], qy, e.R[2])) + e.t[0] * d;
  const float Y = fmaf(e.R[3], qx, fmaf(e.R[4], qy, e.R[5])) + e.t[1] * d;
  const float Z = fmaf(e.R[6], qx, fmaf(e.R[7], qy, e.R[8])) + e.t[2] * d;
  bool ok = Z > 1e-4f * d;
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(Z));
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
__global__ void __launch_bounds__(kEnergyThreads) energy_kernel(const EnergyArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[kEnergyThreads / 32];
  __shared__ double kappa_s;
  const int fl = blockIdx.x / A.tiles, tile = blockIdx.x % A.tiles;
  const int s0 = A.csr_off[fl], k = A.csr_off[fl + 1] - s0;
  const int f = A.frame_of[fl];
  float4* fs = reinterpret_cast<float4*>(smem);  // [kmax][256]
  EdgeLin* sl = reinterpret_cast<EdgeLin*>(smem + sizeof(float4) * kEnergyTile * A.kmax);
  EdgeBack* sb = reinterpret_cast<EdgeBack*>(sl + k);
  const float4** fp0 = reinterpret_cast<const float4**>(sb + k);
  const int tid = threadIdx.x;
  const bool phaseA = A.backsub && !A.freeze;
  const int P = A.P;
  for (int x = tid; x < k * (int)(sizeof(EdgeLin) / 16); x += kEnergyThreads)
    reinterpret_cast<float4*>(sl)[x] = reinterpret_cast<const float4*>(A.lin + s0)[x];
  if (phaseA)
    for (int x = tid; x < k * (int)(sizeof(EdgeBack) / 16); x += kEnergyThreads)
      reinterpret_cast<float4*>(sb)[x] = reinterpret_cast<const float4*>(A.back + s0)[x];
  for (int x = tid; x < k; x += kEnergyThreads) fp0[x] = A.flow + (size_t)A.slot_flow[s0 + x] * P;
  __syncthreads();
  const bool gauge = phaseA && f == A.gauge_frame && k > 0;
  if (gauge && tid == 0) {  // A5: kappa = (rho - h . delta_local) / gamma, as pass_kernel
    const double* gs = A.gstate_c;
    double hd = 0.0;
    for (int a = 0; a < k; ++a)
      for (int q = 0; q < 6; ++q) hd += gs[2 + 6 * a + q] * (double)sb[a].dlt[q];
    if (CALIB)
      for (int q = 0; q < 4; ++q) hd += gs[2 + 6 * k + q] * (A.intr_n[q] - A.intr_c[q]);
    kappa_s = (gs[1] - hd) / gs[0];
  }
  __syncthreads();

  // the thread's pixels p_j = tile*256 + j*kEnergyThreads + tid, each with its k flow
  // records staged in shared memory in one burst (each thread reads back only its own,
  // so no barrier)
  bool in[kEnergyPx];
  int pc[kEnergyPx];
#pragma unroll
  for (int j = 0; j < kEnergyPx; ++j) {
    const int p = tile * kEnergyTile + j * kEnergyThreads + tid;
    in[j] = p < P;
    pc[j] = in[j] ? p : 0;  // clamped: out-of-range pixels read pixel 0 and contribute nothing
  }
  for (int a = 0; a < k; ++a)
#pragma unroll
    for (int j = 0; j < kEnergyPx; ++j) {
      const unsigned dst = (unsigned)__cvta_generic_to_shared(fs + a * kEnergyTile + j * kEnergyThreads + tid);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(fp0[a] + pc[j]));
    }
  asm volatile("cp.async.commit_group;");
  auto record = [&](int a, int j) -> float4 { return fs[a * kEnergyTile + j * kEnergyThreads + tid]; };
  const float Wf = (float)A.W, Hf = (float)A.H;
  const float fxn = (float)A.intr_n[0], fyn = (float)A.intr_n[1];
  const float cxn = (float)A.intr_n[2], cyn = (float)A.intr_n[3];
  float pu[kEnergyPx], pv[kEnergyPx], dc[kEnergyPx], dn[kEnergyPx], ap[kEnergyPx];
#pragma unroll
  for (int j = 0; j < kEnergyPx; ++j) {
    pu[j] = (float)(pc[j] % A.W);
    pv[j] = (float)(pc[j] / A.W);
    const size_t fpx = (size_t)f * P + pc[j];
    dc[j] = A.d_cur[fpx];
    dn[j] = dc[j];
    ap[j] = A.prior != nullptr ? A.alpha * (A.pweight ? A.pweight[f] : 1.f) * (float)A.pmask[fpx] : 0.f;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (phaseA) {
    const float fxc = (float)A.intr_c[0], fyc = (float)A.intr_c[1];
    const float cxc = (float)A.intr_c[2], cyc = (float)A.intr_c[3];
    const float dth[4] = {(float)(A.intr_n[0] - A.intr_c[0]), (float)(A.intr_n[1] - A.intr_c[1]),
                          (float)(A.intr_n[2] - A.intr_c[2]), (float)(A.intr_n[3] - A.intr_c[3])};
    float qx[kEnergyPx], qy[kEnergyPx], Cp[kEnergyPx], gdp[kEnergyPx], accp[kEnergyPx];
#pragma unroll
    for (int j = 0; j < kEnergyPx; ++j) {
      qx[j] = (pu[j] - cxc) / fxc;
      qy[j] = (pv[j] - cyc) / fyc;
      Cp[j] = gdp[j] = accp[j] = 0.f;
    }
    for (int a = 0; a < k; ++a) {
      const EdgeBack& e = sb[a];
#pragma unroll
      for (int j = 0; j < kEnergyPx; ++j) {
        const float4 fw = record(a, j);
        const PixTerms T =
            pix_terms_e(reinterpret_cast<const EdgeLin&>(e), qx[j], qy[j], dc[j], fxc, fyc, cxc, cyc, Wf, Hf, fw);
        const float fxi = fxc * T.iz, fyi = fyc * T.iz;
        const float Jdu = fxi * (e.t[0] - T.xt * e.t[2]);
        const float Jdv = fyi * (e.t[1] - T.yt * e.t[2]);
        const float* dl = e.dlt;
        float ju = fxi * dc[j] * (dl[0] - T.xt * dl[2]) +
                   fxc * (-T.xt * T.yt * dl[3] + (1.f + T.xt * T.xt) * dl[4] - T.yt * dl[5]);
        float jv = fyi * dc[j] * (dl[1] - T.yt * dl[2]) +
                   fyc * (-(1.f + T.yt * T.yt) * dl[3] + T.xt * T.yt * dl[4] + T.xt * dl[5]);
        if (CALIB) {
          const float cu0 = T.iz * (e.R[0] - T.xt * e.R[6]), cu1 = T.iz * (e.R[1] - T.xt * e.R[7]);
          const float cv0 = T.iz * (e.R[3] - T.yt * e.R[6]), cv1 = T.iz * (e.R[4] - T.yt * e.R[7]);
          ju += (T.xt - cu0 * qx[j]) * dth[0] + (-cu1 * qy[j] * fxc / fyc) * dth[1] + (1.f - cu0) * dth[2] +
                (-cu1 * fxc / fyc) * dth[3];
          jv += (-cv0 * qx[j] * fyc / fxc) * dth[0] + (T.yt - cv1 * qy[j]) * dth[1] +
                (-cv0 * fyc / fxc) * dth[2] + (1.f - cv1) * dth[3];
        }
        const float au = T.wu * Jdu, av = T.wv * Jdv;
        Cp[j] += fmaf(au, Jdu, av * Jdv);
        gdp[j] += fmaf(au, T.ru, av * T.rv);
        accp[j] += fmaf(au, ju, av * jv);
      }
    }
#pragma unroll
    for (int j = 0; j < kEnergyPx; ++j) {
      float C = A.eta + Cp[j], gd = gdp[j];
      if (A.prior != nullptr) {
        C += ap[j];
        gd += ap[j] * (A.prior[(size_t)f * P + pc[j]] - dc[j]);
      }
      float dd = (gd - accp[j]) / C;
      if (gauge) dd -= (float)(kappa_s / (double)dc[j]);  // A5: r/C - kappa/d
      dn[j] = fmaxf(dc[j] + dd, A.d_min);
    }
  }
  // residual energy at (x_n, d_n)
  float qx[kEnergyPx], qy[kEnergyPx], en[kEnergyPx];
#pragma unroll
  for (int j = 0; j < kEnergyPx; ++j) {
    if (in[j]) A.d_new[(size_t)f * P + pc[j]] = dn[j];
    qx[j] = (pu[j] - cxn) / fxn;
    qy[j] = (pv[j] - cyn) / fyn;
    en[j] = 0.f;
  }
  for (int a = 0; a < k; ++a) {
    const EdgeLin& e = sl[a];
#pragma unroll
    for (int j = 0; j < kEnergyPx; ++j) {
      const PixTerms T = pix_terms_e(e, qx[j], qy[j], dn[j], fxn, fyn, cxn, cyn, Wf, Hf, record(a, j));
      en[j] += T.wu * T.ru * T.ru + T.wv * T.rv * T.rv;
    }
  }
  double ed = 0.0;
#pragma unroll
  for (int j = 0; j < kEnergyPx; ++j) {
    if (!in[j]) continue;
    ed += (double)en[j];
    if (A.prior != nullptr) {
      const float dd = A.prior[(size_t)f * P + pc[j]] - dn[j];
      ed += (double)(ap[j] * dd * dd);
    }
  }
  // fixed-order block reduction
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) ed += __shfl_xor_sync(0xffffffffu, ed, off);
  if ((tid & 31) == 0) red[tid >> 5] = ed;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kEnergyThreads / 32; ++w) s += red[w];
    A.part[blockIdx.x] = s;
  }
}

}  // namespace dba
