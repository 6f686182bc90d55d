// Energy-only trial pass (float64): back-substitution at x_c and the Eq. 3 (+ Eq. 4) energy at
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
constexpr int kEnergyThreads = kEnergyTile;  // one thread per pixel

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
  const double* d_cur;
  double* d_new;
  const float* prior;
  const uint8_t* pmask;
  const float* pweight;
  double alpha, eta, d_min;
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

template <bool CALIB>
__global__ void __launch_bounds__(kEnergyThreads, 4) energy_kernel(const EnergyArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[kEnergyThreads / 32];
  __shared__ double kappa_s;
  __shared__ double rcp_s[8];  // 1/fx_c, 1/fy_c, 1/fx_n, 1/fy_n, fx_c/fy_c, fy_c/fx_c, 1/W (one thread)
  const int fl = blockIdx.y, tile = blockIdx.x;  // grid (tiles, frames)
  const int s0 = A.csr_off[fl], k = A.csr_off[fl + 1] - s0;
  const int f = A.frame_of[fl];
  float4* fs = reinterpret_cast<float4*>(smem);  // [kmax][256]
  EdgeLin* sl = reinterpret_cast<EdgeLin*>(smem + sizeof(float4) * kEnergyTile * A.kmax);
  EdgeBack* sb = reinterpret_cast<EdgeBack*>(sl + k);
  const float4** fp0 = reinterpret_cast<const float4**>(sb + k);
  const int tid = threadIdx.x;
  const bool phaseA = A.backsub && !A.freeze;
  const int P = A.P;
  for (int x = tid; x < k * (int)(sizeof(EdgeLin) / 8); x += kEnergyThreads)
    reinterpret_cast<double*>(sl)[x] = reinterpret_cast<const double*>(A.lin + s0)[x];
  if (phaseA)
    for (int x = tid; x < k * (int)(sizeof(EdgeBack) / 8); x += kEnergyThreads)
      reinterpret_cast<double*>(sb)[x] = reinterpret_cast<const double*>(A.back + s0)[x];
  for (int x = tid; x < k; x += kEnergyThreads) fp0[x] = A.flow + (size_t)A.slot_flow[s0 + x] * P;
  if (tid == 0) {
    rcp_s[0] = 1.0 / A.intr_c[0];
    rcp_s[1] = 1.0 / A.intr_c[1];
    rcp_s[2] = 1.0 / A.intr_n[0];
    rcp_s[3] = 1.0 / A.intr_n[1];
    rcp_s[4] = A.intr_c[0] * rcp_s[1];
    rcp_s[5] = A.intr_c[1] * rcp_s[0];
    rcp_s[6] = 1.0 / (double)A.W;
  }
  __syncthreads();
  const double dth[4] = {A.intr_n[0] - A.intr_c[0], A.intr_n[1] - A.intr_c[1], A.intr_n[2] - A.intr_c[2],
                         A.intr_n[3] - A.intr_c[3]};
  const bool gauge = phaseA && f == A.gauge_frame && k > 0;
  if (gauge && tid == 0) {  // A5: kappa = (rho - h . delta_local) / gamma, as pass_kernel
    const double* gs = A.gstate_c;
    double hd = 0.0;
    for (int a = 0; a < k; ++a)
      for (int q = 0; q < 6; ++q) hd += gs[2 + 6 * a + q] * sb[a].dlt[q];
    if (CALIB)
      for (int q = 0; q < 4; ++q) hd += gs[2 + 6 * k + q] * dth[q];
    kappa_s = (gs[1] - hd) / gs[0];
  }
  __syncthreads();

  // the thread's pixel p = tile*256 + tid, its k flow records staged in shared memory in
  // one burst (each thread reads back only its own, so no barrier)
  const int p = tile * kEnergyTile + tid;
  const bool in = p < P;
  const int pc = in ? p : 0;  // clamped: out-of-range pixels read pixel 0 and contribute nothing
  for (int a = 0; a < k; ++a) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(fs + a * kEnergyTile + tid);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(fp0[a] + pc));
  }
  asm volatile("cp.async.commit_group;");
  const double Wf = (double)A.W, Hf = (double)A.H;
  const double fxn = A.intr_n[0], fyn = A.intr_n[1], cxn = A.intr_n[2], cyn = A.intr_n[3];
  const double pd = (double)pc;
  const double pv = floor((pd + 0.5) * rcp_s[6]), pu = fma(-pv, Wf, pd);  // exact: p < 2^40
  const size_t fpx = (size_t)f * P + pc;
  const double dc = A.d_cur[fpx];
  double dn = dc;
  const double ap =
      A.prior != nullptr ? A.alpha * (A.pweight ? (double)A.pweight[f] : 1.0) * (double)A.pmask[fpx] : 0.0;
  asm volatile("cp.async.wait_all;" ::: "memory");
  if (phaseA) {
    const double fxc = A.intr_c[0], fyc = A.intr_c[1], cxc = A.intr_c[2], cyc = A.intr_c[3];
    const double qx = (pu - cxc) * rcp_s[0], qy = (pv - cyc) * rcp_s[1];
    double Cp = 0.0, gdp = 0.0, accp = 0.0;
    for (int a = 0; a < k; ++a) {
      const EdgeBack& e = sb[a];
      const float4 fw = fs[a * kEnergyTile + tid];
      const PixTerms T = pix_terms(e.R, e.t, qx, qy, dc, fxc, fyc, cxc, cyc, Wf, Hf, fw, true);
      const double fxi = fxc * T.iz, fyi = fyc * T.iz;
      const double Jdu = fxi * (e.t[0] - T.xt * e.t[2]);
      const double Jdv = fyi * (e.t[1] - T.yt * e.t[2]);
      const double* dl = e.dlt;
      double ju = fxi * dc * (dl[0] - T.xt * dl[2]) +
                  fxc * (-T.xt * T.yt * dl[3] + (1.0 + T.xt * T.xt) * dl[4] - T.yt * dl[5]);
      double jv = fyi * dc * (dl[1] - T.yt * dl[2]) +
                  fyc * (-(1.0 + T.yt * T.yt) * dl[3] + T.xt * T.yt * dl[4] + T.xt * dl[5]);
      if (CALIB) {
        double Tu[4], Tv[4];
        theta_jac(e.R, T, qx, qy, rcp_s[4], rcp_s[5], Tu, Tv);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          ju += Tu[r] * dth[r];
          jv += Tv[r] * dth[r];
        }
      }
      const double au = T.wu * Jdu, av = T.wv * Jdv;
      Cp += fma(au, Jdu, av * Jdv);
      gdp += fma(au, T.ru, av * T.rv);
      accp += fma(au, ju, av * jv);
    }
    double C = A.eta + Cp, gd = gdp;
    if (A.prior != nullptr) {
      C += ap;
      gd += ap * ((double)A.prior[fpx] - dc);
    }
    double dd = (gd - accp) / C;
    if (gauge) dd -= kappa_s / dc;  // A5: r/C - kappa/d
    dn = fmax(dc + dd, A.d_min);
  }
  // residual energy at (x_n, d_n)
  if (in) A.d_new[fpx] = dn;
  const double qx = (pu - cxn) * rcp_s[2], qy = (pv - cyn) * rcp_s[3];
  double ed = 0.0;
  for (int a = 0; a < k; ++a) {
    const EdgeLin& e = sl[a];
    const PixTerms T = pix_terms(e.R, e.t, qx, qy, dn, fxn, fyn, cxn, cyn, Wf, Hf, fs[a * kEnergyTile + tid], true);
    ed += T.wu * T.ru * T.ru + T.wv * T.rv * T.rv;
  }
  if (A.prior != nullptr) {
    const double dd = (double)A.prior[fpx] - dn;
    ed += ap * dd * dd;
  }
  if (!in) ed = 0.0;
  // fixed-order block reduction
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) ed += __shfl_xor_sync(0xffffffffu, ed, off);
  if ((tid & 31) == 0) red[tid >> 5] = ed;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kEnergyThreads / 32; ++w) s += red[w];
    A.part[blockIdx.y * A.tiles + blockIdx.x] = s;
  }
}

}  // namespace dba
