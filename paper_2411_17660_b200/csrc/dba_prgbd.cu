// P-RGBD block-coordinate descent helpers:
// the per-frame affine prior of Eq. 5, E_reg,m = sum m (d* - (s d + o))^2.
//
//  prior_affine_kernel  stage A (s, o frozen): the term is the Eq. 4 prior of the
//                       fused pass with d*' = (d* - o) / s and weight alpha s^2
//                       (identical value and normal equations).
//  fit_affine_kernel    stage B: closed-form least squares for (s_i, o_i) given the
//                       disparities (2x2 normal equations per frame, float64, fixed
//                       reduction tree), s clamped to >= s_min.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/dba_b200.h"

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) prior_affine_kernel(int N, int P, const float* prior, const double* s,
                                                                const double* o, float* prior_out, float* weight) {
  const int f = blockIdx.y;
  const double sf = s[f], of = o[f];
  for (int p = blockIdx.x * kThreads + threadIdx.x; p < P; p += gridDim.x * kThreads)
    prior_out[(size_t)f * P + p] = (float)(((double)prior[(size_t)f * P + p] - of) / sf);
  if (blockIdx.x == 0 && threadIdx.x == 0) weight[f] = (float)(sf * sf);
}

__global__ void __launch_bounds__(kThreads) fit_affine_kernel(int P, const float* disps, const float* prior,
                                                              const uint8_t* mask, double* s, double* o,
                                                              double s_min) {
  const int f = blockIdx.x, tid = threadIdx.x;
  __shared__ double red[5][kThreads];
  double a = 0.0, b = 0.0, c = 0.0, dd = 0.0, dp = 0.0;  // sum m d^2, m d, m, m d d*, m d*
  for (int p = tid; p < P; p += kThreads) {
    const size_t x = (size_t)f * P + p;
    if (mask[x]) {
      const double d = disps[x], ds = prior[x];
      a += d * d;
      b += d;
      c += 1.0;
      dd += d * ds;
      dp += ds;
    }
  }
  red[0][tid] = a;
  red[1][tid] = b;
  red[2][tid] = c;
  red[3][tid] = dd;
  red[4][tid] = dp;
  __syncthreads();
  for (int off = kThreads / 2; off >= 1; off >>= 1) {
    if (tid < off)
      for (int q = 0; q < 5; ++q) red[q][tid] += red[q][tid + off];
    __syncthreads();
  }
  if (tid != 0) return;
  a = red[0][0];
  b = red[1][0];
  c = red[2][0];
  dd = red[3][0];
  dp = red[4][0];
  if (c <= 0.0) return;  // no valid prior pixel: keep (s, o)
  double sv = s[f], ov;
  const double det = a * c - b * b;
  if (det > 1e-12 * a * c) sv = (c * dd - b * dp) / det;  // else constant disparity: keep s
  if (!(sv >= s_min)) sv = s_min;
  ov = (dp - sv * b) / c;  // optimal offset for the chosen scale
  s[f] = sv;
  o[f] = ov;
}

}  // namespace

extern "C" {

int dba_prior_affine(int32_t n_frames, int32_t n_pixels, const float* prior, const double* scale,
                     const double* offset, float* prior_out, float* weight_out, void* stream) {
  if (n_frames < 0 || n_pixels <= 0) return DBA_EINVAL;
  if (n_frames == 0) return DBA_OK;
  if (!prior || !scale || !offset || !prior_out || !weight_out) return DBA_EINVAL;
  const dim3 grid((unsigned)((n_pixels + kThreads - 1) / kThreads), (unsigned)n_frames);
  prior_affine_kernel<<<grid, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n_frames, n_pixels, prior, scale,
                                                                                      offset, prior_out, weight_out);
  return cudaGetLastError() == cudaSuccess ? DBA_OK : DBA_ECUDA;
}

int dba_fit_affine(int32_t n_frames, int32_t n_pixels, const float* disps, const float* prior, const uint8_t* mask,
                   double* scale, double* offset, double s_min, void* stream) {
  if (n_frames < 0 || n_pixels <= 0) return DBA_EINVAL;
  if (n_frames == 0) return DBA_OK;
  if (!disps || !prior || !mask || !scale || !offset) return DBA_EINVAL;
  fit_affine_kernel<<<n_frames, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(n_pixels, disps, prior, mask,
                                                                                       scale, offset, s_min);
  return cudaGetLastError() == cudaSuccess ? DBA_OK : DBA_ECUDA;
}

}  // extern "C"
