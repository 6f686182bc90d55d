// K1+K2+K3a: the fused per-frame linearisation pass of one Gauss-Newton trial, float64.
//
// A CTA (8 warps, one per SM, persistent) walks a list of segments; a segment is
// (source frame i, a run of `sub`-pixel tiles, sub = 128 or 64) and owns ALL out-edges
// of frame i, so every per-pixel disparity term (C_p, g_d,p and the pose/disparity
// couplings E_e,p) stays on chip.  Per tile:
//
//   phase A (back-substitution at x_c; only the dba_debug_trial hook runs it -- the
//       solve loop takes d_n from energy_kernel), pixel-major:
//       delta d_p = (g_d,p - sum_e E_e,p . delta_e) / C_p, d_n = max(d + delta d, d_min)
//
//   phase B (linearisation at x_n), edge-major units (edge e, 32-pixel slice), a lane
//       per pixel: residual, validity (geometry.py:235-250), J_j, J_d, [J_theta];
//       energy; per-edge H_jj / g_j accumulated in registers of the warp that owns the
//       units (two edge slots per warp, reduced once per segment); E_e,p -> the
//       column-major shared matrix U[6e..6e+5][p]; per-edge parts of C_p, g_d,p
//   per pixel: C_p, g_d,p (+ Eq. 4 prior), 1/C_p; U_ext = U extended by the columns
//       [g_d,p, c_p] (c = C/d: A5 gauge; c = d (eta + alpha m): scalefix)
//   phase C (K3a): M_ext += U_ext C^-1 U_ext^T over the tile's pixels on the FP64 TENSOR CORES
//       (mma.sync m8n8k4 f64, DMMA): the upper triangle of M_ext in 8x8 blocks, a
//       fixed block list per warp, accumulators in registers for the whole segment.
//       The extra columns give, in the same product, w = E C^-1 g_d (Schur rhs) and the
//       A5 gauge terms h = E C^-1 c, rho = c^T C^-1 g_d, gamma = c^T C^-1 c.
//
// Everything after the float32 flow record is float64, like the oracle: parity with
// oracle/dba.py is then limited by float64 rounding (~1e-12 relative), not by the
// conditioning of the monocular chain -- a float32 per-pixel chain measured pose-step
// errors of 7e-5 on C3 and amplified them past 1e-4 in near-cancelling back-substitutions.
// Tensor cores: tcgen05 has no float64 kind; DMMA reaches the B200 FP64 peak
// (18.5 TFMA/s measured, the same as DFMA) while issuing one instruction per 256 FMAs,
// which leaves the issue slots to the phase-B geometry.
//
// The flow record (tu, tv, wu, wv) is one coalesced float4 per edge-pixel (the 16 B of
// algorithmic traffic), staged into shared memory with cp.async one tile ahead.
// Jacobians use homogeneous coordinates X~ = R q + t d (q = ((u-cx)/fx, (v-cy)/fy, 1)):
//   J_u = fx [d/Z, 0, -d x/Z, -x y, 1 + x^2, -y]
//   J_v = fy [0, d/Z, -d y/Z, -(1 + y^2), x y, x]
//   J_d = (fx (t_x - x t_z)/Z, fy (t_y - y t_z)/Z)
// equal to the oracle's J_j = J_pi(X_j)[I | -[X_j]x], J_d = J_pi(X_j) R (-X_i/d)
// (oracle/dba.py edge_terms).  J_i = -J_j Ad(G_ij) is applied per edge in assemble.
// Every reduction has a fixed order (bitwise-deterministic results).
#pragma once

#include "dba_common.cuh"

namespace dba {

constexpr int kPassThreads = 256;  // linearisation (geometry) threads
constexpr int kPassWarps = 8;
constexpr int kGemmWarps = 8;      // two warpgroups: the tensor-core Schur product
constexpr int kGemmThreads = 32 * kGemmWarps;
constexpr int kPassCTA = kGemmThreads + kPassThreads;
// named barriers: geometry warps only; U-ring slot b full (geometry -> product warps),
// slot b empty (product -> geometry)
constexpr int kMaxSlots = 4;  // U-ring depth limit (named barriers 2..9)
constexpr int kBarGeo = 1, kBarFull = 2, kBarEmpty = 2 + kMaxSlots;
// register split between the roles (setmaxnreg; 256 * R_gemm + 256 * R_geo <= 512 * 128):
// product warps 72 registers for up to 2 items (measured: 64 spills in the k-loop, 88 costs
// the linearisation warps theirs), more for the rare high-degree shapes
__host__ __device__ constexpr int pass_gemm_regs(int qmax) { return qmax <= 2 ? 72 : qmax <= 3 ? 80 : 96; }
__host__ __device__ constexpr int pass_geo_regs(int qmax) {
  return ((kPassCTA * 128 - kGemmThreads * pass_gemm_regs(qmax)) / kPassThreads) & ~7;
}
constexpr int kSlice = 32;     // pixels per phase-B edge unit (1 per lane)
constexpr int kEdgeSlots = 2;  // distinct edges per warp per segment (see pass_units)

struct PassArgs {
  int H, W, P, n_tiles, kmax, sub;
  int nslot;    // U-ring depth (2..kMaxSlots)
  int backsub;  // run phase A
  int freeze;   // disparity block frozen (motion-only / pose stage): no Schur fill-in, d unchanged
  int scalefix; // prior-fixed monocular scale: the A5 column carries c = d (eta + alpha m) instead
  const int* status;  // see trial_skipped
  unsigned long long* runs;  // counts executed launches (profiling of gated passes) or null
  const int* csr_off;
  const int* slot_flow;
  const int* frame_of;
  const int* seg_frame;  // segment -> local frame
  const int* seg_t0;     // segment -> first tile
  const int* seg_t1;     // segment -> end tile
  const int* cta_seg;    // CTA -> segment range
  const EdgeLin* lin;
  const EdgeBack* back;
  const float4* flow;
  const double* d_cur;
  double* d_new;
  const float* prior;
  const uint8_t* pmask;
  const float* pweight;  // (N,) per-frame multiplier of alpha (Eq. 5 stage A: s_i^2) or null
  double alpha, eta, d_min;
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
template <typename T>
__device__ __forceinline__ T transpose_reduce32(T (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < off; ++i) {
      const T send = up ? v[i] : v[i + off];
      const T keep = up ? v[i + off] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

__host__ __device__ inline int pass_mu(int k, bool calib) { return 6 * k + (calib ? 4 : 0); }
// GEMM rows: U (mu) + [g_d, c], padded to pairs of 8x8 tensor-core blocks
__host__ __device__ inline int pass_mext(int k, bool calib) { return pass_mu(k, calib) + 2; }
__host__ __device__ inline int pass_mpad(int k, bool calib) { return (pass_mext(k, calib) + 15) & ~15; }
// column stride of the column-major U (doubles): = 4 (mod 16) makes both the phase-B
// stores (a lane per pixel) and the m8n8k4 fragment loads (4 pixels x 8 rows per
// half-warp pair) bank-conflict free
__host__ __device__ constexpr int pass_ustride(int sub) { return sub + 4; }

// Work split of the symmetric product M_ext = V C^-1 V^T (upper triangle, 8x8 blocks).
// The np = mpad/16 row PAIRS of blocks give two kinds of items:
//   cross (r < c): the 2x2 block square {2r, 2r+1} x {2c, 2c+1}: 4 fragments, 4 DMMAs
//   diag  (r = c): (2r,2r), (2r,2r+1), (2r+1,2r+1): 2 fragments, 3 DMMAs
// (A and B fragments of one block row are the same shared-memory words.)  Items go to
// the kGemmWarps product warps longest-first onto the least-loaded warp, lowest index on
// ties (np = 4, radius-5 graphs: 4,4,4,4,4,4,6,6 DMMAs per k-step; splitting the diagonal
// items for an exact balance measured no faster and needs more accumulator registers).
// Every thread evaluates the same deterministic assignment.  Returns the number of items
// of warp `w`, their pairs and kinds (0 cross, 3 diag) in (qr, qc, qk) when non-null.
template <int QMAX>
__host__ __device__ inline int pass_quads(int np, int w, int* qr, int* qc, int* qk) {
  constexpr int nw = kGemmWarps;
  int load[nw];
  for (int x = 0; x < nw; ++x) load[x] = 0;
  int n = 0;
  for (int kind = 0; kind < 4; kind += 3)
    for (int r = 0; r < np; ++r)
      for (int c = r; c < np; ++c) {
        if ((kind == 0) != (r < c)) continue;
        int best = 0;
        for (int x = 1; x < nw; ++x)
          if (load[x] < load[best]) best = x;
        load[best] += kind == 0 ? 4 : 3;
        if (best == w) {
          if (qr) {
#pragma unroll
            for (int s = 0; s < QMAX; ++s)  // compile-time register index
              if (s == n) {
                qr[s] = r;
                qc[s] = c;
                qk[s] = kind;
              }
          }
          ++n;
        }
      }
  return n;
}
// largest per-warp item count for np row pairs (the plan picks QMAX from it)
__host__ __device__ inline int pass_qmax(int np) {
  int m = 0;
  for (int w = 0; w < kGemmWarps; ++w) {
    const int n = pass_quads<1>(np, w, nullptr, nullptr, nullptr);
    m = n > m ? n : m;
  }
  return m;
}

// phase-B unit range of warp w: contiguous, at most kEdgeSlots distinct edges
__device__ __forceinline__ void pass_units(int k, int slices, int w, int& u0, int& u1) {
  const int n = k * slices;
  int L = (n + kPassWarps - 1) / kPassWarps;
  for (;; ++L) {  // L = 2 * slices always satisfies it for k <= 2 * kPassWarps
    bool ok = true;
    for (int x = 0; x < kPassWarps && ok; ++x) {
      const int a = x * L, b = min(a + L, n);
      if (a < n) ok = (b - 1) / slices - a / slices < kEdgeSlots;
    }
    if (ok) break;
  }
  u0 = min(w * L, n);
  u1 = min(u0 + L, n);
}

struct PassSmem {
  size_t fbuf, U, parts, dcs, dns, icv, qc, qn, ebuf, ethb, red, emap, sflow, sl, sb, total;
};
__host__ __device__ inline PassSmem pass_smem_layout(int kmax, bool calib, int sub, int nslot) {
  PassSmem s;
  size_t o = 0;
  const int nparts = calib ? 6 : 2;  // phase B: C, gd (+ E_theta x4)
  s.fbuf = o; o += 2 * sizeof(float4) * (size_t)kmax * sub;  // double-buffered: tile t+1 lands under tile t
  s.U = o; o += nslot * sizeof(double) * (size_t)pass_mpad(kmax, calib) * pass_ustride(sub);  // tile ring
  s.parts = o; o += sizeof(double) * (size_t)nparts * kmax * sub;
  s.dcs = o; o += 2 * sizeof(double) * sub;
  s.dns = o; o += sizeof(double) * sub;
  s.icv = o; o += nslot * sizeof(double) * sub;
  s.qc = o; o += sizeof(double2) * sub;
  s.qn = o; o += sizeof(double2) * sub;
  s.ebuf = o; o += sizeof(double) * kPassWarps * kEdgeSlots * 32;
  s.ethb = o; o += calib ? sizeof(double) * kPassWarps * kEdgeSlots * 32 : 0;
  s.red = o; o += sizeof(double) * kPassWarps * 16;
  s.emap = o; o += sizeof(int) * kPassWarps * kEdgeSlots;
  s.sflow = o; o += sizeof(int) * kmax;
  o = (o + 15) & ~size_t(15);
  s.sl = o; o += sizeof(EdgeLin) * kmax;
  s.sb = o; o += sizeof(EdgeBack) * kmax;
  s.total = (o + 15) & ~size_t(15);
  return s;
}


// per edge-pixel geometry at one state
struct PixTerms {
  bool ok;
  double xt, yt, iz, ru, rv, wu, wv;
};

__device__ __forceinline__ PixTerms pix_terms(const double R[9], const double t[3], double qx, double qy, double d,
                                              double fx, double fy, double cx, double cy, double Wf, double Hf,
                                              const float4& fw, bool in) {
  PixTerms o;
  const double X = fma(R[0], qx, fma(R[1], qy, R[2])) + t[0] * d;
  const double Y = fma(R[3], qx, fma(R[4], qy, R[5])) + t[1] * d;
  const double Z = fma(R[6], qx, fma(R[7], qy, R[8])) + t[2] * d;
  bool ok = in && Z > 1e-4 * d;  // Z_MIN on the non-homogeneous depth (geometry.py:17)
  o.iz = ok ? rcp64(Z) : 0.0;
  o.xt = X * o.iz;
  o.yt = Y * o.iz;
  const double pu = fma(fx, o.xt, cx), pv = fma(fy, o.yt, cy);
  ok = ok && pu >= -1e-9 && pu <= Wf + 1e-9 && pv >= -1e-9 && pv <= Hf + 1e-9;
  o.ok = ok;
  o.wu = ok ? (double)fw.z : 0.0;
  o.wv = ok ? (double)fw.w : 0.0;
  o.ru = ok ? (double)fw.x - pu : 0.0;
  o.rv = ok ? (double)fw.y - pv : 0.0;
  return o;
}

// J_theta = d(u,v)/d(fx,fy,cx,cy) through unprojection and projection; fxy = fx / fy and
// fyx = fy / fx are formed once per thread by the caller (four divisions per edge-pixel
// otherwise)
__device__ __forceinline__ void theta_jac(const double R[9], const PixTerms& T, double qx, double qy, double fxy,
                                          double fyx, double Tu[4], double Tv[4]) {
  const double cu0 = T.iz * (R[0] - T.xt * R[6]), cu1 = T.iz * (R[1] - T.xt * R[7]);
  const double cv0 = T.iz * (R[3] - T.yt * R[6]), cv1 = T.iz * (R[4] - T.yt * R[7]);
  Tu[0] = T.xt - cu0 * qx;
  Tu[1] = -cu1 * qy * fxy;
  Tu[2] = 1.0 - cu0;
  Tu[3] = -cu1 * fxy;
  Tv[0] = -cv0 * qx * fyx;
  Tv[1] = T.yt - cv1 * qy;
  Tv[2] = -cv0 * fyx;
  Tv[3] = 1.0 - cv1;
}


// The product warp's k-loop for a compile-time item shape: NC cross items then ND
// diagonal items, k-step outer and items inner, so every accumulator chain of the warp is
// in flight at once (a lone product warp per SM sub-partition has no other warp to hide
// the DMMA latency behind) with no branches inside the loop.
template <int QMAX, int US, int NC, int ND>
__device__ __forceinline__ void gemm_shape(double (&macc)[QMAX][4][2], const double* Ub, const double* icl,
                                           const int (&fo_r)[QMAX], const int (&fo_c)[QMAX]) {
  constexpr int kRB = 8 * US;
  constexpr int nks = (US - 4) / 4;
  constexpr int NI = NC + ND;
  // fragments of k-step ks + 1 are loaded while the DMMAs of ks issue (explicit double
  // buffering: the LDS -> DMUL -> DMMA chain of one k-step would otherwise serialise)
  double ic = icl[0], r0[NI > 0 ? NI : 1], r1[NI > 0 ? NI : 1], c0[NC > 0 ? NC : 1], c1[NC > 0 ? NC : 1];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    r0[i] = Ub[fo_r[i]];
    r1[i] = Ub[fo_r[i] + kRB];
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    c0[i] = Ub[fo_c[i]];
    c1[i] = Ub[fo_c[i] + kRB];
  }
#pragma unroll 2
  for (int ks = 0; ks < nks; ++ks) {
    // the last step prefetches the 4 padding columns of the slot (US = SUB + 4) and the
    // shared words after its 1/C_p row: unused, and no per-step clamp
    const int pn = 4 * (ks + 1);
    const double icn = icl[pn];
    double r0n[NI > 0 ? NI : 1], r1n[NI > 0 ? NI : 1], c0n[NC > 0 ? NC : 1], c1n[NC > 0 ? NC : 1];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      r0n[i] = Ub[fo_r[i] + pn];
      r1n[i] = Ub[fo_r[i] + kRB + pn];
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      c0n[i] = Ub[fo_c[i] + pn];
      c1n[i] = Ub[fo_c[i] + kRB + pn];
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const double a0 = r0[i] * ic, a1 = r1[i] * ic;
      dmma884(macc[i][0], a0, c0[i]);
      dmma884(macc[i][1], a0, c1[i]);
      dmma884(macc[i][2], a1, c0[i]);
      dmma884(macc[i][3], a1, c1[i]);
    }
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const double a0 = r0[NC + j] * ic;
      dmma884(macc[NC + j][0], a0, r0[NC + j]);
      dmma884(macc[NC + j][1], a0, r1[NC + j]);
      dmma884(macc[NC + j][3], r1[NC + j] * ic, r1[NC + j]);
    }
    ic = icn;
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      r0[i] = r0n[i];
      r1[i] = r1n[i];
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      c0[i] = c0n[i];
      c1[i] = c1n[i];
    }
  }
}
// runs gemm_shape<NC', ND'> for the runtime (nc, nd); false when the shape is not covered
template <int QMAX, int US, int NC, int ND>
__device__ __forceinline__ bool gemm_dispatch(int nc, int nd, double (&macc)[QMAX][4][2], const double* Ub,
                                              const double* icl, const int (&fo_r)[QMAX], const int (&fo_c)[QMAX]) {
  if (nc == NC && nd == ND) {
    gemm_shape<QMAX, US, NC, ND>(macc, Ub, icl, fo_r, fo_c);
    return true;
  }
  if constexpr (NC + ND + 1 <= QMAX && QMAX <= 4) {
    if (gemm_dispatch<QMAX, US, NC, ND + 1>(nc, nd, macc, Ub, icl, fo_r, fo_c)) return true;
    if constexpr (ND == 0)
      if (gemm_dispatch<QMAX, US, NC + 1, 0>(nc, nd, macc, Ub, icl, fo_r, fo_c)) return true;
  }
  return false;
}

__device__ __forceinline__ void nbar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Warp-specialised: warpgroups 0-1 (kGemmWarps warps) run the tensor-core product, the
// other 8 warps the per-pixel linearisation.  Per tile the geometry warps fill U-ring
// slot b (tile sequence number mod the ring depth) and hand it over (kBarFull + b); the product warps
// drain it and hand it back (kBarEmpty + b).  DMMA and DFMA share the fp64 datapath
// (profiles/tools/mb_fp64pipes.cu), so the point is that every SM sub-partition always has
// a warp with fp64 work ready: two product warps next to two linearisation warps (one lone
// product warp per sub-partition issued a DMMA only every ~32 cycles).
// DBA_PASS_TIMING (diagnostic build, profiles/tools/pass_balance.py): per CTA the
// globaltimer at entry and when its last product / linearisation warp finishes, and its SM
#ifdef DBA_PASS_TIMING
__device__ unsigned long long g_pass_t[4 * 1024];
__device__ __forceinline__ unsigned long long pass_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PASS_T_MARK(slot)                                                                   \
  do {                                                                                      \
    if ((threadIdx.x & 31) == 0) atomicMax(&g_pass_t[4 * blockIdx.x + (slot)], pass_now()); \
  } while (0)
#else
#define PASS_T_MARK(slot) \
  do {                    \
  } while (0)
#endif
template <bool CALIB, int QMAX, int SUB>
__global__ void __launch_bounds__(kPassCTA, 1) pass_kernel(const PassArgs A) {
  pdl_enter();
  if (trial_skipped(A.status)) return;
  if (A.runs && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(A.runs, 1ull);
#ifdef DBA_PASS_TIMING
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_pass_t[4 * blockIdx.x] = pass_now();
    g_pass_t[4 * blockIdx.x + 3] = smid;
  }
#endif
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NVE = kEdgeVals + (CALIB ? kCalibVals : 0);
  constexpr int SL = SUB / kSlice, US = pass_ustride(SUB);
  const int NS = A.nslot;
  const PassSmem L = pass_smem_layout(A.kmax, CALIB, SUB, NS);
  float4* const fbufb = reinterpret_cast<float4*>(smem + L.fbuf);  // 2 x [k][SUB] flow records
  double* const Ubuf = reinterpret_cast<double*>(smem + L.U);  // U ring: two [mpad][US] slots
  const int ulen = pass_mpad(A.kmax, CALIB) * US;
  double* const icvb = reinterpret_cast<double*>(smem + L.icv);  // 1 / C_p, per ring slot
  const int sg0 = A.cta_seg[blockIdx.x], sg1 = A.cta_seg[blockIdx.x + 1];
  int ntot = 0;  // tiles of this CTA: the ring handshakes
  for (int sg = sg0; sg < sg1; ++sg) ntot += A.seg_t1[sg] - A.seg_t0[sg];
  constexpr int nks = SUB / 4;

  if (threadIdx.x < kGemmThreads) {
    // ============================================================== product warps
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(pass_gemm_regs(QMAX)));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int tau = 0, slot = 0;  // tile sequence number and its ring slot (tau mod NS)
    for (int sg = sg0; sg < sg1; ++sg) {
      const int fl = A.seg_frame[sg];
      const int k = A.csr_off[fl + 1] - A.csr_off[fl];
      const int mu = pass_mu(k, CALIB);
      const int mext = mu + 2;
      const int np = ((mext + 15) & ~15) >> 4;
      double* pf = A.part_frame + (long long)sg * kFrameVals;
      // product items of this warp (pass_quads): fragment pointers into a ring slot are
      // U + fo_r[q] (rows of block 2r; block 2r+1 is kRB doubles further) and U + fo_c[q]
      int qr[QMAX], qc[QMAX], qk[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) qr[q] = qc[q] = qk[q] = 0;
      const int nq = pass_quads<QMAX>(np, warp, qr, qc, qk);
      const int lane_off = (lane >> 2) * US + (lane & 3);
      int fo_r[QMAX], fo_c[QMAX];
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        fo_r[q] = 16 * qr[q] * US + lane_off;
        fo_c[q] = 16 * qc[q] * US + lane_off;
      }
      constexpr int kRB = 8 * US;  // doubles between the fragments of blocks 2r and 2r+1
      double macc[QMAX][4][2];
#pragma unroll
      for (int q = 0; q < QMAX; ++q)
#pragma unroll
        for (int b = 0; b < 4; ++b) macc[q][b][0] = macc[q][b][1] = 0.0;
      // M_ext += U C^-1 U^T over the k-steps of one ring slot, item by item: per k-step
      // (4 pixels) the A fragments are the row-pair's U words scaled by the lane's 1/C_p,
      // the B fragments the column-pair's unscaled words (for a diagonal item the same
      // words as A); branch-free inner loops with immediate shared offsets
      int nc = 0;  // items are in kind order: cross (kind 0) first, then diagonal (3)
#pragma unroll
      for (int q = 0; q < QMAX; ++q) nc += (q < nq && qk[q] == 0) ? 1 : 0;
      auto gemm = [&](const double* Ub, const double* ic_b) {
        const double* icl = ic_b + (lane & 3);
        if (QMAX <= 4 && gemm_dispatch<QMAX, US, 0, 0>(nc, nq - nc, macc, Ub, icl, fo_r, fo_c))
          return;
        // generic: item by item, branch-free unrolled k-loops per item
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
          if (q >= nq) break;
          const double* pr = Ub + fo_r[q];
          if (qk[q] == 3) {  // (2r,2r), (2r,2r+1), (2r+1,2r+1)
#pragma unroll 4
            for (int ks = 0; ks < nks; ++ks) {
              const int p0 = 4 * ks;
              const double ic = icl[p0];
              const double b0 = pr[p0], b1 = pr[kRB + p0];
              const double a0 = b0 * ic;
              dmma884(macc[q][0], a0, b0);
              dmma884(macc[q][1], a0, b1);
              dmma884(macc[q][3], b1 * ic, b1);
            }
          } else {
            const double* pc = Ub + fo_c[q];
#pragma unroll 4
            for (int ks = 0; ks < nks; ++ks) {
              const int p0 = 4 * ks;
              const double ic = icl[p0];
              const double a0 = pr[p0] * ic, a1 = pr[kRB + p0] * ic;
              const double b0 = pc[p0], b1 = pc[kRB + p0];
              dmma884(macc[q][0], a0, b0);
              dmma884(macc[q][1], a0, b1);
              dmma884(macc[q][2], a1, b0);
              dmma884(macc[q][3], a1, b1);
            }
          }
        }
      };
      for (int tile = A.seg_t0[sg]; tile < A.seg_t1[sg]; ++tile, ++tau, slot = slot + 1 == NS ? 0 : slot + 1) {
        const int b = slot;
        nbar_sync(kBarFull + b, kPassCTA);
        gemm(Ubuf + b * ulen, icvb + b * SUB);
        if (tau + NS < ntot) nbar_arrive(kBarEmpty + b, kPassCTA);
      }
    // tensor-core blocks -> M (mu x mu, both triangles), w = column mu, h = column mu+1,
    // rho, gamma; lane l holds D[l/4][2(l%4) + i] of each block
    double* pM = A.part_M + A.seg_off_M[sg];
    double* pw = A.part_w + A.seg_off_w[sg];
#pragma unroll
    for (int q = 0; q < QMAX; ++q) {
      if (q >= nq) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        // blocks of the item: cross all four, diag 0, 1 and 3
        if (qk[q] == 3 && b == 2) continue;
        const int bi = 2 * qr[q] + (b >> 1), bj = 2 * qc[q] + (b & 1);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int R = 8 * bi + (lane >> 2), Cc = 8 * bj + 2 * (lane & 3) + i;
          if (R > Cc || Cc >= mext) continue;
          const double v = macc[q][b][i];
          if (Cc < mu) {
            pM[(long long)R * mu + Cc] = v;
            pM[(long long)Cc * mu + R] = v;
          } else if (R < mu && Cc == mu) {
            pw[R] = v;
          } else if (R < mu && Cc == mu + 1) {
            pw[mu + R] = v;
          } else if (R == mu && Cc == mu + 1) {
            pf[16] = v;  // rho
          } else if (R == mu + 1 && Cc == mu + 1) {
            pf[15] = v;  // gamma
          }
        }
      }
    }
    }  // segments
    PASS_T_MARK(1);
    return;
  }

  // ================================================================ linearisation warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(pass_geo_regs(QMAX)));
  double* parts = reinterpret_cast<double*>(smem + L.parts);
  double* const dcsb = reinterpret_cast<double*>(smem + L.dcs);  // 2 x [SUB]
  double* dns = reinterpret_cast<double*>(smem + L.dns);
  double2* qcs = reinterpret_cast<double2*>(smem + L.qc);  // normalised pixel rays at x_c
  double2* qns = reinterpret_cast<double2*>(smem + L.qn);  // ... at x_n
  double* ebuf = reinterpret_cast<double*>(smem + L.ebuf);
  double* ethb = reinterpret_cast<double*>(smem + L.ethb);
  double* red = reinterpret_cast<double*>(smem + L.red);
  int* emap = reinterpret_cast<int*>(smem + L.emap);
  int* sflow = reinterpret_cast<int*>(smem + L.sflow);
  EdgeLin* sl = reinterpret_cast<EdgeLin*>(smem + L.sl);
  EdgeBack* sb = reinterpret_cast<EdgeBack*>(smem + L.sb);

  const int tid = threadIdx.x - kGemmThreads, lane = tid & 31, warp = tid >> 5;
  const int P = A.P, KM = A.kmax;
  const double Wf = (double)A.W, Hf = (double)A.H;
  const double fxn = A.intr_n[0], fyn = A.intr_n[1], cxn = A.intr_n[2], cyn = A.intr_n[3];
  const double fxc = A.intr_c[0], fyc = A.intr_c[1], cxc = A.intr_c[2], cyc = A.intr_c[3];
  // reciprocals and ratios of the intrinsics, once per thread (per-pixel rays, J_theta)
  const double ifxn = 1.0 / fxn, ifyn = 1.0 / fyn, ifxc = 1.0 / fxc, ifyc = 1.0 / fyc;
  const double fxyn = fxn * ifyn, fyxn = fyn * ifxn, fxyc = fxc * ifyc, fyxc = fyc * ifxc;
  const double iW = 1.0 / Wf;  // pixel index -> (u, v) without integer division
  const double dth[4] = {fxn - fxc, fyn - fyc, cxn - cxc, cyn - cyc};
  int tau = 0, slot = 0;  // tile sequence number and its ring slot (tau mod NS)

  for (int sg = sg0; sg < sg1; ++sg) {
    const int fl = A.seg_frame[sg];
    const int s0 = A.csr_off[fl];
    const int k = A.csr_off[fl + 1] - s0;
    const int f = A.frame_of[fl];
    const int mu = pass_mu(k, CALIB);
    const int mext = mu + 2;
    const int mpad = (mext + 15) & ~15;
    double* Pa0 = parts;                 // [k][SUB]  C part
    double* Pa1 = parts + KM * SUB;      // [k][SUB]  g_d part
    double* Pth = parts + 2 * KM * SUB;  // [4][k][SUB] E_theta parts (phase B, calib)

    // ---- stage per-edge constants, unit -> edge slots
    for (int x = tid; x < k * (int)(sizeof(EdgeLin) / 8); x += kPassThreads)
      reinterpret_cast<double*>(sl)[x] = reinterpret_cast<const double*>(A.lin + s0)[x];
    if (A.backsub)
      for (int x = tid; x < k * (int)(sizeof(EdgeBack) / 8); x += kPassThreads)
        reinterpret_cast<double*>(sb)[x] = reinterpret_cast<const double*>(A.back + s0)[x];
    for (int x = tid; x < k; x += kPassThreads) sflow[x] = A.slot_flow[s0 + x];
    int u0, u1;
    pass_units(k, SL, warp, u0, u1);
    const int e0 = u0 / SL;  // slot s holds edge e0 + s
    if (lane < kEdgeSlots) {
      const int e = e0 + lane;
      emap[warp * kEdgeSlots + lane] = (u1 > u0 && e * SL < u1 && e < k) ? e : -1;
    }
    for (int x = tid; x < kPassWarps * kEdgeSlots * 32; x += kPassThreads) {
      ebuf[x] = 0.0;
      if (CALIB) ethb[x] = 0.0;
    }
    double hacc[kEdgeSlots][28];  // per-edge H_jj, g_j, energy of this warp's units (whole segment)
#pragma unroll
    for (int s = 0; s < kEdgeSlots; ++s)
#pragma unroll
      for (int x = 0; x < 28; ++x) hacc[s][x] = 0.0;
    double facc[15];  // energy, H_tt (10), g_t (4)
#pragma unroll
    for (int x = 0; x < 15; ++x) facc[x] = 0.0;
    double fpri = 0.0;  // scalefix: sum_p d_p alpha m_p (d*_p - d_p) (the prior's gradient along the scale)
    // A5: kappa = (rho - h . delta_local) / gamma from the x_c linearisation
    const bool gauge = (f == A.gauge_frame) && k > 0;
    nbar_sync(kBarGeo, kPassThreads);
    double kappa = 0.0;
    if (gauge && A.backsub) {
      const double* gs = A.gstate_c;
      double hd = 0.0;
      for (int a = 0; a < k; ++a)
        for (int q = 0; q < 6; ++q) hd += gs[2 + 6 * a + q] * sb[a].dlt[q];
      if (CALIB)
        for (int q = 0; q < 4; ++q) hd += gs[2 + 6 * k + q] * dth[q];
      kappa = (gs[1] - hd) / gs[0];
    }

    // cp.async staging of a tile's flow records (16 B each) and disparities;
    // out-of-range pixels are zero-filled
    auto prefetch = [&](int tile, int buf) {
      float4* const fbuf = fbufb + buf * KM * SUB;
      double* const dcs = dcsb + buf * SUB;
      const int pb = tile * SUB;
      for (int x = tid; x < k * SUB; x += kPassThreads) {
        const int a = x / SUB, pl = x - a * SUB, p = pb + pl;
        const float4* src = A.flow + (size_t)sflow[a] * P + (p < P ? p : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(fbuf + x);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                     "r"(p < P ? 16 : 0));
      }
      for (int x = tid; x < SUB; x += kPassThreads) {
        const int p = pb + x;
        const double* src = A.d_cur + (size_t)f * P + (p < P ? p : 0);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(dcs + x);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(p < P ? 8 : 0));
      }
      asm volatile("cp.async.commit_group;");
    };
    prefetch(A.seg_t0[sg], tau & 1);

    for (int tile = A.seg_t0[sg]; tile < A.seg_t1[sg]; ++tile, ++tau, slot = slot + 1 == NS ? 0 : slot + 1) {
      const int pbase = tile * SUB;
      const int tb = slot;
      double* const U = Ubuf + tb * ulen;  // this tile's ring slot
      double* const icv = icvb + tb * SUB;
      const float4* const fbuf = fbufb + (tau & 1) * KM * SUB;
      const double* const dcs = dcsb + (tau & 1) * SUB;
      asm volatile("cp.async.wait_all;" ::: "memory");
      for (int x = tid; x < SUB; x += kPassThreads) {
        const double pd = (double)(pbase + x);
        const double pv = floor((pd + 0.5) * iW), pu = fma(-pv, Wf, pd);  // exact: p < 2^40
        if (A.backsub) qcs[x] = make_double2((pu - cxc) * ifxc, (pv - cyc) * ifyc);  // phase A only
        qns[x] = make_double2((pu - cxn) * ifxn, (pv - cyn) * ifyn);
      }
      nbar_sync(kBarGeo, kPassThreads);
      // the next tile's records land in the other buffer under this tile's work (its last
      // reader, tile t-1, is behind the barrier above)
      if (tile + 1 < A.seg_t1[sg]) prefetch(tile + 1, (tau + 1) & 1);
      // ------------------------------------------------------------ phase A
      // pixel-major: a half-warp per 16 pixels, the two halves split the edges; the
      // per-pixel sums close with one shuffle, so d_n needs no block barrier
      if (A.backsub && !A.freeze) {
        for (int pl = 16 * warp + (lane & 15); pl < SUB; pl += 16 * kPassWarps) {
          const int p = pbase + pl, eg = lane >> 4;
          const bool in = p < P;
          const double dc = dcs[pl];
          const double qx = qcs[pl].x, qy = qcs[pl].y;
          double Cp = 0.0, gdp = 0.0, accp = 0.0;
          for (int a = eg; a < k; a += 2) {
            const EdgeBack& e = sb[a];
            const float4 fw = fbuf[a * SUB + pl];
            const PixTerms T = pix_terms(e.R, e.t, qx, qy, dc, fxc, fyc, cxc, cyc, Wf, Hf, fw, in);
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
              theta_jac(e.R, T, qx, qy, fxyc, fyxc, Tu, Tv);
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
          // edge-group halves in fixed order: (even edges) + (odd edges)
          const double Co = __shfl_xor_sync(0xffffffffu, Cp, 16);
          const double go = __shfl_xor_sync(0xffffffffu, gdp, 16);
          const double ao = __shfl_xor_sync(0xffffffffu, accp, 16);
          if (eg == 0) {
            if (in) {
              double C = A.eta + (Cp + Co), gd = gdp + go, acc = accp + ao;
              if (A.prior != nullptr) {
                const size_t fp = (size_t)f * P + p;
                const double ap = A.alpha * (A.pweight ? (double)A.pweight[f] : 1.0) * (double)A.pmask[fp];
                C += ap;
                gd += ap * ((double)A.prior[fp] - dc);
              }
              double dd = (gd - acc) / C;
              if (gauge) dd -= kappa / dc;  // A5: r/C - kappa/d
              const double dn = fmax(dc + dd, A.d_min);
              dns[pl] = dn;
              A.d_new[(size_t)f * P + p] = dn;
            } else {
              dns[pl] = 1.0;
            }
          }
        }
      } else {
        for (int x = tid; x < SUB; x += kPassThreads) {
          const int p = pbase + x;
          dns[x] = dcs[x];
          if (p < P) A.d_new[(size_t)f * P + p] = dcs[x];
        }
      }
      nbar_sync(kBarGeo, kPassThreads);
      // ------------------------------------------------------------ phase B
      if (tau >= NS) nbar_sync(kBarEmpty + tb, kPassCTA);  // the product warps are done with the slot
      for (int u = u0; u < u1; ++u) {
        const int a = u / SL, slot = a - e0;
        const int pl = (u - a * SL) * kSlice + lane, p = pbase + pl;
        const bool in = p < P;
        const EdgeLin& e = sl[a];
        const float4 fw = fbuf[a * SUB + pl];
        const double dn = dns[pl];
        const double qx = qns[pl].x, qy = qns[pl].y;
        const PixTerms T = pix_terms(e.R, e.t, qx, qy, dn, fxn, fyn, cxn, cyn, Wf, Hf, fw, in);
        const double en = T.wu * T.ru * T.ru + T.wv * T.rv * T.rv;
        facc[0] += en;
        const double fxi = fxn * T.iz, fyi = fyn * T.iz;
        double Ju[6], Jv[6];
        Ju[0] = fxi * dn;
        Ju[1] = 0.0;
        Ju[2] = -fxi * dn * T.xt;
        Ju[3] = -fxn * T.xt * T.yt;
        Ju[4] = fxn * (1.0 + T.xt * T.xt);
        Ju[5] = -fxn * T.yt;
        Jv[0] = 0.0;
        Jv[1] = fyi * dn;
        Jv[2] = -fyi * dn * T.yt;
        Jv[3] = -fyn * (1.0 + T.yt * T.yt);
        Jv[4] = fyn * T.xt * T.yt;
        Jv[5] = fyn * T.xt;
        const double Jdu = fxi * (e.t[0] - T.xt * e.t[2]);
        const double Jdv = fyi * (e.t[1] - T.yt * e.t[2]);
        const double au = T.wu * Jdu, av = T.wv * Jdv;
        Pa0[a * SUB + pl] = fma(au, Jdu, av * Jdv);
        Pa1[a * SUB + pl] = fma(au, T.ru, av * T.rv);
        double* Ucol = U + (6 * a) * US + pl;
#pragma unroll
        for (int c = 0; c < 6; ++c) Ucol[c * US] = fma(au, Ju[c], av * Jv[c]);
        const double wu = T.wu, wv = T.wv, wru = T.wu * T.ru, wrv = T.wv * T.rv;
        // per-edge H_jj (upper 21), g_j (6), energy into this slot's registers;
        // J_u[1] = 0 and J_v[0] = 0: the structurally zero terms are skipped
#pragma unroll
        for (int s = 0; s < kEdgeSlots; ++s) {
          if (s != slot) continue;
          int o = 0;
#pragma unroll
          for (int r = 0; r < 6; ++r)
#pragma unroll
            for (int c = r; c < 6; ++c) {
              const bool zu = r == 1 || c == 1, zv = r == 0 || c == 0;
              if (!zu && !zv)
                hacc[s][o] = fma(wu * Ju[r], Ju[c], fma(wv * Jv[r], Jv[c], hacc[s][o]));
              else if (!zu)
                hacc[s][o] = fma(wu * Ju[r], Ju[c], hacc[s][o]);
              else if (!zv)
                hacc[s][o] = fma(wv * Jv[r], Jv[c], hacc[s][o]);
              ++o;
            }
#pragma unroll
          for (int r = 0; r < 6; ++r) {
            if (r == 0)
              hacc[s][21 + r] = fma(wru, Ju[r], hacc[s][21 + r]);
            else if (r == 1)
              hacc[s][21 + r] = fma(wrv, Jv[r], hacc[s][21 + r]);
            else
              hacc[s][21 + r] = fma(wru, Ju[r], fma(wrv, Jv[r], hacc[s][21 + r]));
          }
          hacc[s][27] += en;
        }
        if (CALIB) {
          double Tu[4], Tv[4];
          theta_jac(e.R, T, qx, qy, fxyn, fyxn, Tu, Tv);
          double v32[32];
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 6; ++c) v32[6 * r + c] = fma(wu * Tu[r], Ju[c], wv * Tv[r] * Jv[c]);
#pragma unroll
          for (int x = 24; x < 32; ++x) v32[x] = 0.0;
          int q = 1;
#pragma unroll
          for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = r; c < 4; ++c) {
              facc[q] = fma(wu * Tu[r], Tu[c], fma(wv * Tv[r], Tv[c], facc[q]));
              ++q;
            }
#pragma unroll
          for (int r = 0; r < 4; ++r) facc[11 + r] = fma(wru, Tu[r], fma(wrv, Tv[r], facc[11 + r]));
#pragma unroll
          for (int r = 0; r < 4; ++r) Pth[(r * KM + a) * SUB + pl] = fma(au, Tu[r], av * Tv[r]);
          // H_theta_j of this unit: one transpose-reduce (lane l: value l), fixed order
          const double rs = transpose_reduce32(v32, lane);
          ethb[(warp * kEdgeSlots + slot) * 32 + lane] += rs;
        }
      }
      nbar_sync(kBarGeo, kPassThreads);
      // ------------------------------------------------------------ per pixel
      // C_p, g_d,p (+ Eq. 4 prior), 1/C_p and the extra columns; the 1/C_p scaling is
      // applied to the A fragments of the product (M_ext = sum_p U_p U_p^T / C_p)
      for (int pl = tid; pl < SUB; pl += kPassThreads) {
        const int p = pbase + pl;
        const bool in = p < P;
        double C = A.eta, gd = 0.0;
        for (int a = 0; a < k; ++a) {
          C += Pa0[a * SUB + pl];
          gd += Pa1[a * SUB + pl];
        }
        const double dn = dns[pl];
        double ap = 0.0;
        if (A.prior != nullptr && in) {
          const size_t fp = (size_t)f * P + p;
          ap = A.alpha * (A.pweight ? (double)A.pweight[f] : 1.0) * (double)A.pmask[fp];
          const double dd = (double)A.prior[fp] - dn;
          C += ap;
          gd += ap * dd;
          facc[0] += ap * dd * dd;
          fpri = fma(dn * ap, dd, fpri);
        }
        icv[pl] = (in && !A.freeze) ? rcp64(C) : 0.0;  // frozen d: no fill-in
        if (CALIB) {
          double Et[4] = {0.0, 0.0, 0.0, 0.0};
          for (int a = 0; a < k; ++a)
#pragma unroll
            for (int r = 0; r < 4; ++r) Et[r] += Pth[(r * KM + a) * SUB + pl];
#pragma unroll
          for (int r = 0; r < 4; ++r) U[(6 * k + r) * US + pl] = Et[r];
        }
        // second extra column: A5 gauge c = C/d, or (scalefix) c = d (eta + alpha m), whose
        // E C^-1 c is the reduced system's exact row along the monocular scale direction
        // (only the gauge frame's and the scalefix rows are read by assemble_kernel)
        const double cx = A.scalefix ? dn * (A.eta + ap) : gauge ? C * rcp64(dn) : 0.0;
        U[mu * US + pl] = gd;
        U[(mu + 1) * US + pl] = in ? cx : 0.0;
      }
      // rows mext..mpad of the slot: zero (the product covers whole 16-row pairs)
      for (int x = tid; x < (mpad - mext) * SUB; x += kPassThreads) U[(mext + x / SUB) * US + x % SUB] = 0.0;
      nbar_arrive(kBarFull + tb, kPassCTA);
    }

    // ------------------------------------------------------------ segment outputs
    // per-edge register accumulators: one transpose-reduce per slot per segment
#pragma unroll
    for (int s = 0; s < kEdgeSlots; ++s) {
      double v32[32];
#pragma unroll
      for (int x = 0; x < 28; ++x) v32[x] = hacc[s][x];
#pragma unroll
      for (int x = 28; x < 32; ++x) v32[x] = 0.0;
      const double rs = transpose_reduce32(v32, lane);
      ebuf[(warp * kEdgeSlots + s) * 32 + lane] = rs;
    }
    // per-frame values: fixed-order block reduction
#pragma unroll
    for (int x = 0; x < 15; ++x) {
      double v = facc[x];
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[warp * 16 + x] = v;
    }
    {
      double v = fpri;
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) red[warp * 16 + 15] = v;
    }
    nbar_sync(kBarGeo, kPassThreads);
    double* pf = A.part_frame + (long long)sg * kFrameVals;
    if (tid < kFrameVals) {
      double v = 0.0;
      if (tid < 15)
        for (int w = 0; w < kPassWarps; ++w) v += red[w * 16 + tid];
      if (tid == 17)
        for (int w = 0; w < kPassWarps; ++w) v += red[w * 16 + 15];
      if (tid < 15 || tid == 17) pf[tid] = v;  // [15], [16] (gamma, rho) come from the product
    }
    double* pe = A.part_edge + A.seg_off_edge[sg];
    for (int x = tid; x < k * NVE; x += kPassThreads) {
      const int a = x / NVE, l = x % NVE;
      double v = 0.0;
      for (int ws = 0; ws < kPassWarps * kEdgeSlots; ++ws)
        if (emap[ws] == a) v += (l < 32) ? ebuf[ws * 32 + l] : ethb[ws * 32 + (l - 32)];
      pe[x] = v;
    }
    nbar_sync(kBarGeo, kPassThreads);
  }  // segments
  PASS_T_MARK(2);
}

}  // namespace dba
