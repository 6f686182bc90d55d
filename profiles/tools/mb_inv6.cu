// isolated latency of inv6_spd (one thread, operands in shared memory)
#include <cstdio>
#include "old_pivot.cuh"
using namespace dba;
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
      inv6_spd(D, 1e-4 * it, o);
      for (int x = 0; x < 36; ++x) Di[x] = o[x];
      D[0] += Di[35] * 1e-30;  // dependency
    }
    cyc[0] = clock64() - t0;
    out[0] = Di[0];
  }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
  for (int r = 0; r < 3; ++r) {
    k<<<1, 64>>>(o, c, 1000); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("inv6 isolated: %.0f cycles/call\n", h / 1000.0);
  }
}
