// GPU synthetic correspondence provider: the flow records of
// SyntheticProviders.provide_correspondences (providers.py:318-338) for a batch of
// edges, one thread per edge-pixel, written straight into the (E, H, W, 4) layout
// [tu, tv, wu, wv] the BA consumes.
//
// Scene (providers.py:122-218): the camera sits inside an outer sphere of radius R_out
// (every ray hits it) with spherical occluders.  For pixel p of frame i:
//   ray  o = c_i, dir = R_c2w,i (xn, yn, 1)   -> nearest hit s = pinhole depth Z
//   target = project(w2c_j o c2w_i . unproject(p, 1/Z))        (reproject, :265-276)
//   visible = cast(c_j, X_w - c_j) >= 1 - 1e-6  and  X_w projects inside frame j
//   weight = (valid and visible) for both channels; non-finite targets -> 0.
// float64 throughout; pixel noise (pixel_noise > 0) is added by the caller.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/dba_b200.h"

namespace {

constexpr int kMaxOccluders = 64;

struct ProvArgs {
  int H, W, n_edges, n_occ;
  double fx, fy, cx, cy, r_out;
  const double* c2w;  // (F,7)
  const double* w2c;  // (F,7)
  const double* occ;  // (n_occ,4) centre, radius
  const int* ii;
  const int* jj;
  float* out;
};

__device__ void quat_rot(const double* q, double R[9]) {
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  R[0] = 1 - 2 * (y * y + z * z);
  R[1] = 2 * (x * y - w * z);
  R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);
  R[4] = 1 - 2 * (x * x + z * z);
  R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);
  R[7] = 2 * (y * z + w * x);
  R[8] = 1 - 2 * (x * x + y * y);
}

// nearest intersection along o + s d (d unnormalised; s in units of d)  (providers.py:195-218)
__device__ double cast(const ProvArgs& A, const double o[3], const double d[3]) {
  const double dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  const double od = o[0] * d[0] + o[1] * d[1] + o[2] * d[2];
  const double oo = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
  double disc = od * od - dd * (oo - A.r_out * A.r_out);
  double best = (-od + sqrt(fmax(disc, 0.0))) / dd;
  for (int k = 0; k < A.n_occ; ++k) {
    const double* c = A.occ + 4 * k;
    const double oc[3] = {o[0] - c[0], o[1] - c[1], o[2] - c[2]};
    const double ocd = oc[0] * d[0] + oc[1] * d[1] + oc[2] * d[2];
    disc = ocd * ocd - dd * ((oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2]) - c[3] * c[3]);
    const double s = (-ocd - sqrt(fmax(disc, 0.0))) / dd;
    if (disc > 0.0 && s > 1e-9 && s < best) best = s;
  }
  return best;
}

__device__ bool project(const ProvArgs& A, const double X[3], double& u, double& v) {
  const double z = X[2];
  const double zs = fabs(z) > 1e-300 ? z : 1e-300;
  u = A.fx * X[0] / zs + A.cx;
  v = A.fy * X[1] / zs + A.cy;
  const double eps = 1e-9;
  return z > 1e-4 && u >= -eps && u <= A.W + eps && v >= -eps && v <= A.H + eps;
}

__global__ void __launch_bounds__(256) provider_kernel(const ProvArgs A) {
  const int P = A.H * A.W;
  const long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= (long long)A.n_edges * P) return;
  const int e = (int)(x / P), p = (int)(x % P);
  const int i = A.ii[e], j = A.jj[e];
  const double u = p % A.W, v = p / A.W;
  double Rc[9], Rj[9], Rrel[9];
  quat_rot(A.c2w + 7 * (size_t)i, Rc);
  quat_rot(A.w2c + 7 * (size_t)j, Rj);
  const double* ci = A.c2w + 7 * (size_t)i + 4;
  const double* tj = A.w2c + 7 * (size_t)j + 4;
  const double cam[3] = {(u - A.cx) / A.fx, (v - A.cy) / A.fy, 1.0};
  double dir[3];
  for (int r = 0; r < 3; ++r) dir[r] = Rc[3 * r] * cam[0] + Rc[3 * r + 1] * cam[1] + Rc[3 * r + 2] * cam[2];
  const double s = cast(A, ci, dir);
  // reproject through the disparity as the provider does (z = 1 / (1 / depth))
  const double z = 1.0 / (1.0 / s);
  const double Xi[3] = {cam[0] * z, cam[1] * z, z};
  // rel = w2c_j o c2w_i
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      Rrel[3 * r + c] = Rj[3 * r] * Rc[c] + Rj[3 * r + 1] * Rc[3 + c] + Rj[3 * r + 2] * Rc[6 + c];
  double Xj[3];
  for (int r = 0; r < 3; ++r) {
    const double trel = Rj[3 * r] * ci[0] + Rj[3 * r + 1] * ci[1] + Rj[3 * r + 2] * ci[2] + tj[r];
    Xj[r] = Rrel[3 * r] * Xi[0] + Rrel[3 * r + 1] * Xi[1] + Rrel[3 * r + 2] * Xi[2] + trel;
  }
  double tu, tv;
  const bool valid = project(A, Xj, tu, tv);
  // visibility of the surface point from camera j
  const double Xw[3] = {ci[0] + s * dir[0], ci[1] + s * dir[1], ci[2] + s * dir[2]};
  const double* cj_q = A.c2w + 7 * (size_t)j;
  const double cj[3] = {cj_q[4], cj_q[5], cj_q[6]};
  const double d2[3] = {Xw[0] - cj[0], Xw[1] - cj[1], Xw[2] - cj[2]};
  const bool unocc = cast(A, cj, d2) > 1.0 - 1e-6;
  double Xc[3];
  for (int r = 0; r < 3; ++r) Xc[r] = Rj[3 * r] * Xw[0] + Rj[3 * r + 1] * Xw[1] + Rj[3 * r + 2] * Xw[2] + tj[r];
  double uj, vj;
  const bool inview = project(A, Xc, uj, vj);
  const float w = (valid && unocc && inview) ? 1.f : 0.f;
  float4 rec;
  rec.x = isfinite(tu) ? (float)tu : 0.f;
  rec.y = isfinite(tv) ? (float)tv : 0.f;
  rec.z = w;
  rec.w = w;
  reinterpret_cast<float4*>(A.out)[x] = rec;
}

}  // namespace

extern "C" {

int dba_synthetic_flows(int32_t H, int32_t W, const double* intr, double outer_radius, int32_t n_occluders,
                        const double* occluders, const double* c2w, const double* w2c, int32_t n_edges,
                        const int32_t* ii, const int32_t* jj, float* out, void* stream) {
  if (H <= 0 || W <= 0 || n_edges < 0 || n_occluders < 0 || n_occluders > kMaxOccluders || !intr) return DBA_EINVAL;
  if (n_edges == 0) return DBA_OK;
  if (!c2w || !w2c || !ii || !jj || !out || (n_occluders > 0 && !occluders)) return DBA_EINVAL;
  ProvArgs a;
  a.H = H;
  a.W = W;
  a.n_edges = n_edges;
  a.n_occ = n_occluders;
  a.fx = intr[0];
  a.fy = intr[1];
  a.cx = intr[2];
  a.cy = intr[3];
  a.r_out = outer_radius;
  a.c2w = c2w;
  a.w2c = w2c;
  a.occ = occluders;
  a.ii = ii;
  a.jj = jj;
  a.out = out;
  const long long n = (long long)n_edges * H * W;
  provider_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? DBA_OK : DBA_ECUDA;
}

}  // extern "C"
