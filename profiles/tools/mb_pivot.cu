// isolated single-thread latency of the 6x6 pivot factorisations (operands in shared memory):
// the round-1/2 adjugate inverse (kept here for the comparison) and chol6_inv of dba_solve.cuh.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_pivot mb_pivot.cu
#include <cstdio>
#include "old_pivot.cuh"
using namespace dba;
template <int V>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double D[36], Di[36];
  if (threadIdx.x < 36) {
    const int r = threadIdx.x / 6, c = threadIdx.x % 6;
    D[threadIdx.x] = (r == c ? 10.0 : 0.0) + 1.0 / (1 + r + c);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
      double o[36];
      if (V == 0) inv6_spd(D, 1e-4 * it, o);
      else chol6_inv(D, 1e-4 * it, o);
      for (int x = 0; x < 36; ++x) Di[x] = o[x];
      D[0] += Di[35] * 1e-30;  // dependency between calls
    }
    cyc[0] = clock64() - t0;
    out[0] = Di[0];
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  for (int r = 0; r < 2; ++r) {
    long long h;
    k<0><<<1, 64>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("adjugate inverse: %.0f cycles/call\n", h / 1000.0);
    k<1><<<1, 64>>>(o, c, 1000); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("chol6_inv: %.0f cycles/call\n", h / 1000.0);
  }
}
