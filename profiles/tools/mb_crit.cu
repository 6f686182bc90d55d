// single-warp replica of the critical-warp step (6-lane L/S11 update + lane-0 inv6)
#include <cstdio>
#include "old_pivot.cuh"
using namespace dba;
template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ __align__(16) double S1[38], S11[38], dinv[72], z[12];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 36) {
    const int r = threadIdx.x / 6, c = threadIdx.x % 6;
    S1[threadIdx.x] = 0.01 * (r + 2 * c);
    S11[threadIdx.x] = (r == c ? 10.0 : 0.0) + 1.0 / (1 + r + c);
    dinv[threadIdx.x] = (r == c ? 0.1 : 0.0);
    dinv[36 + threadIdx.x] = (r == c ? 0.1 : 0.0);
  }
  if (threadIdx.x < 12) z[threadIdx.x] = 1.0;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64(), tl = 0, ti = 0;
  for (int b = 0; b < n; ++b) {
    const double* Db = dinv + 36 * (b & 1);
    long long ta = clock64();
    if (MODE != 1 && lane < 6) {
      const int r = lane;
      double Lr[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
        const double sk = S1[6 * r + kk];
#pragma unroll
        for (int c = 0; c < 6; ++c) Lr[c] = fma(sk, Db[6 * kk + c], Lr[c]);
      }
      double d[6], zs = z[6 + r];
#pragma unroll
      for (int c = 0; c < 6; ++c) d[c] = S11[6 * r + c];
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
#pragma unroll
        for (int c = 0; c < 6; ++c) d[c] = fma(-Lr[kk] * 1e-9, S1[6 * c + kk], d[c]);
        zs = fma(-Lr[kk], z[kk], zs);
      }
#pragma unroll
      for (int c = 0; c < 6; ++c) S11[6 * r + c] = d[c];
      z[6 + r] = zs * 1e-9;
    }
    __syncwarp();
    long long tb = clock64();
    if (MODE != 2 && lane == 0) {
      double Di[36];
      inv6_spd(S11, 1e-4, Di);
      double* Dn = dinv + 36 * ((b + 1) & 1);
#pragma unroll
      for (int x = 0; x < 36; ++x) Dn[x] = Di[x];
    }
    __syncwarp();
    long long tc = clock64();
    tl += tb - ta;
    ti += tc - tb;
  }
  if (lane == 0) {
    cyc[0] = clock64() - t0;
    cyc[1] = tl;
    cyc[2] = ti;
    out[0] = dinv[0];
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  for (int mode = 0; mode < 3; ++mode)
    for (int r = 0; r < 2; ++r) {
      if (mode == 0) k<0><<<1, 64>>>(o, c, 1000);
      if (mode == 1) k<1><<<1, 64>>>(o, c, 1000);
      if (mode == 2) k<2><<<1, 64>>>(o, c, 1000);
      long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
      printf("mode %d: step %.0f  L/S11 %.0f  inv %.0f cycles\n", mode, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0);
    }
}
