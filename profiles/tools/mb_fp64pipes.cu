// Are DMMA (fp64 tensor) and DFMA (fp64 FMA pipe) independent on B200?  Times
// DMMA-only, DFMA-only and interleaved kernels with the same per-kind work.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fp64pipes mb_fp64pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool DO_MMA, bool DO_FMA>
__global__ void k(double* out, int iters, double s) {
  double acc[8][2];
  double f[16];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-9;
  for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-7 + i;
  const double a = s * 0.5, b = s * 0.25;
  for (int it = 0; it < iters; ++it) {
    if (DO_MMA) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    }
    if (DO_FMA) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], a, b);
    }
  }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += acc[i][0] + acc[i][1];
  for (int i = 0; i < 16; ++i) t += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <bool M, bool F>
float run(double* o, int blocks, int threads, int iters) {
  k<M, F><<<blocks, threads>>>(o, iters, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<M, F><<<blocks, threads>>>(o, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o;
  cudaMalloc(&o, sizeof(double) * sms * 8 * 1024);
  const int iters = 4096;
  for (int threads : {128, 256, 512}) {
    const int blocks = sms;
    const double warps = (double)blocks * threads / 32;
    const float tm = run<true, false>(o, blocks, threads, iters);
    const float tf = run<false, true>(o, blocks, threads, iters);
    const float tb = run<true, true>(o, blocks, threads, iters);
    const double fma_mma = warps * iters * 8 * 256.0;  // FMAs
    const double fma_f = warps * iters * 64 * 32.0;
    printf("threads %4d: DMMA-only %.3f ms (%.2f TFMA/s)  DFMA-only %.3f ms (%.2f TFMA/s)  both %.3f ms (sum of alone %.3f)\n",
           threads, tm, fma_mma / tm * 1e-9, tf, fma_f / tf * 1e-9, tb, tm + tf);
  }
  return 0;
}
