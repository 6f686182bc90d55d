// Microbenchmark: tcgen05.mma kind::tf32, MN-major SWIZZLE_NONE operands from smem,
// D = Z Z^T over 128 "pixels" (K) with Z rows = 128 (single MMA M=128,N=128) and
// the split form (A = Z[0:128], B = Z[0:256]; A = Z[128:256], B = Z[0:128]).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int KSUB = 128;
constexpr int SBO = (KSUB / 8) * 128;  // bytes between 4-row chunks

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // layout type 0 = SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int ROWS>
__global__ void k_umma(const float* zin, float* out, int split, int reps, long long* cyc, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* Z = reinterpret_cast<float*>(smem);
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // zin: [ROWS][KSUB] row-major -> interleaved MN-major layout
  for (int x = tid; x < ROWS * KSUB; x += blockDim.x) {
    const int r = x / KSUB, p = x % KSUB;
    float v = zin[x];
    uint32_t h;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    if (mode == 3)
      Z[((p >> 5) * (ROWS / 8) * 1024 + (r >> 3) * 1024 + (r & 7) * 128 + ((((p & 31) >> 2) ^ (r & 7)) << 4)) / 4 +
        (p & 3)] = __uint_as_float(h);
    else if (mode == 2)
      Z[((r >> 3) * (KSUB / 4) * 128 + (p >> 2) * 128 + (r & 7) * 16) / 4 + (p & 3)] = __uint_as_float(h);
    else
      Z[((r >> 2) * SBO + (p >> 3) * 128 + (p & 7) * 16) / 4 + (r & 3)] = __uint_as_float(h);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&mbar)));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  {
    // prefill D with 1.0 via tcgen05.st (32x32b.x32): lanes by warp%4, columns by warp/4
    for (int cb = (warp >> 2) * 32; cb < 512; cb += (blockDim.x / 128) * 32) {
      const uint32_t addr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + cb;
      const uint32_t one = __float_as_uint(1.0f);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
          "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr), "r"(one));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  const int accall = reps < 0;
  if (reps < 0) reps = 1;
  const uint32_t zb = (uint32_t)__cvta_generic_to_shared(Z);
  long long t0 = 0, t1 = 0;
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (tid == 0) {
      t0 = clock64();
      for (int ks = 0; ks < KSUB / 8; ++ks) {
        const uint32_t koff = ks * (mode == 2 ? 256 : 128);
        if (!split) {
          uint64_t d = mode == 0 ? sdesc(zb + koff, 128, SBO) : mode == 1 ? sdesc(zb + koff, SBO, 128)
                                                             : sdesc(zb + koff, 128, (KSUB / 4) * 128);
          if (mode == 3)
            d = sdesc(zb + (ks >> 2) * (ROWS / 8) * 1024 + (ks & 3) * 32, 16, 1024) | ((uint64_t)2 << 61);
          uint32_t id = idesc_tf32(128, ROWS);
          if (mode >= 2) id &= ~((1u << 15) | (1u << 16));
          if (ks == 0 && rep == 0) printf("zb=%u desc=%016llx idesc=%08x tmem=%08x\n", zb, (unsigned long long)d, id, tmem);
          mma_tf32(tmem, d, d, id, accall || ks > 0);
        } else if (mode == 3) {
          const uint32_t kb = zb + (ks >> 2) * (ROWS / 8) * 1024 + (ks & 3) * 32;
          const uint64_t sw = (uint64_t)2 << 61;
          const uint32_t id256 = idesc_tf32(128, 256) & ~((1u << 15) | (1u << 16));
          const uint32_t id128 = idesc_tf32(128, 128) & ~((1u << 15) | (1u << 16));
          mma_tf32(tmem, sdesc(kb, 16, 1024) | sw, sdesc(kb, 16, 1024) | sw, id256, ks > 0);
          mma_tf32(tmem + 256, sdesc(kb + 16 * 1024, 16, 1024) | sw, sdesc(kb, 16, 1024) | sw, id128, ks > 0);
        } else {
          // D1 (cols 0..255) = Z[0:128] . Z[0:256]^T ; D2 (cols 256..383) = Z[128:256] . Z[0:128]^T
          mma_tf32(tmem, sdesc(zb + koff, 128, SBO), sdesc(zb + koff, 128, SBO), idesc_tf32(128, 256), ks > 0);
          mma_tf32(tmem + 256, sdesc(zb + 32 * SBO + koff, 128, SBO), sdesc(zb + koff, 128, SBO),
                   idesc_tf32(128, 128), ks > 0);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"l"(
          (unsigned long long)__cvta_generic_to_shared(&mbar)));
    }
    {
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"((uint32_t)__cvta_generic_to_shared(&mbar)), "r"(phase));
      }
      phase ^= 1;
    }
    if (tid == 0) t1 = clock64();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // read D: warp w -> lanes 32*(w%4).., columns 32*(w/4).. (+ 128 per column block)
  const int ncols = split ? 384 : ROWS;
  for (int cb = (warp >> 2) * 32; cb < ncols; cb += (blockDim.x / 128) * 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + cb;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int row = 32 * (warp & 3) + lane;
    for (int j = 0; j < 32; ++j) out[row * ncols + cb + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  if (tid == 0) cyc[0] = t1 - t0;
}

static float tf32r(float v) {  // round-to-nearest-away on 13 dropped bits
  uint32_t u;
  memcpy(&u, &v, 4);
  u = (u + 0x1000u) & ~0x1FFFu;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

template <int ROWS>
int run(int split, int mode = 0) {
  std::vector<float> z(ROWS * KSUB);
  srand(1);
  for (auto& v : z) v = (float)(rand() % 2001 - 1000) / 777.0f;
  float *dz, *dout;
  long long* dc;
  const int ncols = split ? 384 : ROWS;
  cudaMalloc(&dz, z.size() * 4);
  cudaMalloc(&dout, 128 * ncols * 4);
  cudaMalloc(&dc, 8);
  cudaMemcpy(dz, z.data(), z.size() * 4, cudaMemcpyHostToDevice);
  const int smem = ROWS * KSUB * 4;
  cudaFuncSetAttribute(k_umma<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_umma<ROWS><<<1, 512, smem>>>(dz, dout, split == 2 ? 0 : split, split == 2 ? -1 : 20, dc, mode);
  if (split == 2) split = 0;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<float> out(128 * ncols);
  long long cyc;
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0, bias = 0;
  int nb = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < ncols; ++c) {
      int ar = r, bc = c;
      if (split && c >= 256) {
        ar = 128 + r;
        bc = c - 256;
      }
      double s = 0;
      for (int p = 0; p < KSUB; ++p) s += (double)tf32r(z[ar * KSUB + p]) * (double)tf32r(z[bc * KSUB + p]);
      maxerr = fmax(maxerr, fabs(s - out[r * ncols + c]));
      if (ar == bc) { bias += (out[r * ncols + c] - s) / s; ++nb; }
      maxref = fmax(maxref, fabs(s));
    }
  printf("diag mean signed rel err %.3e (n=%d)\n", nb ? bias / nb : 0.0, nb);
  printf("mode=%d ROWS=%d split=%d max|err|=%.3e max|ref|=%.3e rel=%.3e cycles(last rep)=%lld  D[0][0]=%f D[5][77]=%f\n",
         mode, ROWS, split, maxerr, maxref, maxerr / maxref, cyc, out[0], out[5 * ncols + 77]);
  return 0;
}

int main() {
  run<128>(0, 0);
  run<128>(0, 1);
  run<128>(0, 2);
  run<128>(0, 3);
  run<256>(1, 3);
  return 0;
}
