// crit-step variant: 6 lanes hold the rows of S11' and invert it by Gauss-Jordan with
// shuffle broadcasts (no lane-0 gather, no serial inverse)
#include <cstdio>
#include "old_pivot.cuh"
using namespace dba;
__device__ __forceinline__ double rcp_d(double x) { return 1.0 / x; }
__global__ void k(double* out, long long* cyc, int n, int variant) {
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
    double* Dn = dinv + 36 * ((b + 1) & 1);
    long long ta = clock64();
    double d[6];
    const int r = lane < 6 ? lane : 0;
    {
      double Lr[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
        const double sk = S1[6 * r + kk];
#pragma unroll
        for (int c = 0; c < 6; ++c) Lr[c] = fma(sk, Db[6 * kk + c], Lr[c]);
      }
      double zs = z[6 + r];
#pragma unroll
      for (int c = 0; c < 6; ++c) d[c] = S11[6 * r + c];
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
#pragma unroll
        for (int c = 0; c < 6; ++c) d[c] = fma(-Lr[kk] * 1e-9, S1[6 * c + kk], d[c]);
        zs = fma(-Lr[kk], z[kk], zs);
      }
      if (lane < 6) z[6 + r] = zs * 1e-9;
    }
    long long tb = clock64();
    if (variant == 0) {
      // reference: rows -> smem, lane 0 inverts (the current kernel)
      if (lane < 6)
#pragma unroll
        for (int c = 0; c < 6; ++c) S11[6 * r + c] = d[c];
      __syncwarp();
      if (lane == 0) {
        double Di[36];
        inv6_spd(S11, 1e-4, Di);
#pragma unroll
        for (int x = 0; x < 36; ++x) Dn[x] = Di[x];
      }
    } else {
      // Gauss-Jordan on [S + lam I | I] by rows, lane r owns row r (lanes >= 6 idle copies)
      double a[6], e[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        a[c] = 0.5 * (d[c] + __shfl_sync(0xffffffffu, d[r], c)) + (c == r ? 1e-4 : 0.0);  // symmetrise
        e[c] = c == r ? 1.0 : 0.0;
      }
#pragma unroll
      for (int kk = 0; kk < 6; ++kk) {
        const double piv = __shfl_sync(0xffffffffu, a[kk], kk);
        const double ip = 1.0 / piv;
        double rk[6], ek[6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          rk[c] = __shfl_sync(0xffffffffu, a[c], kk) * ip;
          ek[c] = __shfl_sync(0xffffffffu, e[c], kk) * ip;
        }
        const double f = a[kk];
        if (r == kk) {
#pragma unroll
          for (int c = 0; c < 6; ++c) { a[c] = rk[c]; e[c] = ek[c]; }
        } else {
#pragma unroll
          for (int c = 0; c < 6; ++c) { a[c] = fma(-f, rk[c], a[c]); e[c] = fma(-f, ek[c], e[c]); }
        }
      }
      if (lane < 6)
#pragma unroll
        for (int c = 0; c < 6; ++c) Dn[6 * r + c] = e[c];
    }
    __syncwarp();
    long long tc = clock64();
    tl += tb - ta;
    ti += tc - tb;
  }
  if (lane == 0) { cyc[0] = clock64() - t0; cyc[1] = tl; cyc[2] = ti; out[0] = dinv[0]; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 24);
  for (int v = 0; v < 2; ++v)
    for (int rr = 0; rr < 2; ++rr) {
      k<<<1, 64>>>(o, c, 1000, v); long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
      double ho; cudaMemcpy(&ho, o, 8, cudaMemcpyDeviceToHost);
      printf("variant %d: step %.0f  L/S11 %.0f  inv %.0f cycles  (Dinv[0] %.12g)\n", v, h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, ho);
    }
}
