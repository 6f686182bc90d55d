// Dependent-issue latency of DMMA m8n8k4 and DFMA on B200 (one warp, clock64 around a
// chain of 1024 dependent operations).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fp64lat mb_fp64lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, double s) {
  double d[2] = {threadIdx.x * 1e-9, 0.0};
  const double a = s * 0.5, b = s * 0.25;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 1024; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  double f = d[0];
#pragma unroll 16
  for (int i = 0; i < 1024; ++i) f = fma(f, a, b);
  long long t2 = clock64();
  out[threadIdx.x] = d[0] + d[1] + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
  }
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 16);
  for (int it = 0; it < 2; ++it) k<<<1, 32>>>(o, c, 1.0);
  long long h[2];
  cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("dependent DMMA m8n8k4: %.1f cycles each; dependent DFMA: %.1f cycles each\n", h[0] / 1024.0, h[1] / 1024.0);
  return 0;
}
