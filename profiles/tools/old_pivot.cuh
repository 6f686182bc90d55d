// The round-1/2 pivot inverse of dba_solve.cuh (3x3 adjugates), kept for the single-warp
// pivot microbenchmarks that compare against it.
#pragma once
#include "../../paper_2411_17660_b200/csrc/dba_solve.cuh"
namespace dba {
// inverse of a symmetric 3x3 (row-major m) via the adjugate; leading minors check SPD
__device__ __forceinline__ bool inv3_spd(const double m[9], double o[9]) {
  const double c00 = m[4] * m[8] - m[5] * m[7];
  const double c01 = m[5] * m[6] - m[3] * m[8];
  const double c02 = m[3] * m[7] - m[4] * m[6];
  const double det = m[0] * c00 + m[1] * c01 + m[2] * c02;
  const double m2 = m[0] * m[4] - m[1] * m[3];
  const bool ok = (m[0] > 0.0) && (m2 > 0.0) && (det > 0.0) && isfinite(det);
  const double id = 1.0 / (ok ? det : 1.0);
  o[0] = c00 * id;
  o[1] = (m[2] * m[7] - m[1] * m[8]) * id;
  o[2] = (m[1] * m[5] - m[2] * m[4]) * id;
  o[3] = c01 * id;
  o[4] = (m[0] * m[8] - m[2] * m[6]) * id;
  o[5] = (m[2] * m[3] - m[0] * m[5]) * id;
  o[6] = c02 * id;
  o[7] = (m[1] * m[6] - m[0] * m[7]) * id;
  o[8] = (m[0] * m[4] - m[1] * m[3]) * id;
  return ok;
}

// inverse of a 6x6 SPD block (+ lam I) via [A B; B^T C]:  A^-1, T = A^-1 B,
// C' = C - B^T T, D^-1 = [A^-1 + T C'^-1 T^T, -T C'^-1; -C'^-1 T^T, C'^-1].
__device__ __forceinline__ bool inv6_spd(const double* D, double lam, double* Di) {
  double A[9], B[9], C[9], Ai[9], T[9], Cs[9], Ci[9], U[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      A[3 * r + c] = 0.5 * (D[6 * r + c] + D[6 * c + r]) + (r == c ? lam : 0.0);
      B[3 * r + c] = D[6 * r + c + 3];
      C[3 * r + c] = 0.5 * (D[6 * (r + 3) + c + 3] + D[6 * (c + 3) + r + 3]) + (r == c ? lam : 0.0);
    }
  bool ok = inv3_spd(A, Ai);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      T[3 * r + c] = Ai[3 * r] * B[c] + Ai[3 * r + 1] * B[3 + c] + Ai[3 * r + 2] * B[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      Cs[3 * r + c] = C[3 * r + c] - (B[r] * T[c] + B[3 + r] * T[3 + c] + B[6 + r] * T[6 + c]);
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = r + 1; c < 3; ++c) {
      const double v = 0.5 * (Cs[3 * r + c] + Cs[3 * c + r]);
      Cs[3 * r + c] = v;
      Cs[3 * c + r] = v;
    }
  ok = inv3_spd(Cs, Ci) && ok;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      U[3 * r + c] = T[3 * r] * Ci[c] + T[3 * r + 1] * Ci[3 + c] + T[3 * r + 2] * Ci[6 + c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      Di[6 * r + c] = Ai[3 * r + c] + U[3 * r] * T[3 * c] + U[3 * r + 1] * T[3 * c + 1] +
                      U[3 * r + 2] * T[3 * c + 2];
      Di[6 * r + c + 3] = -U[3 * r + c];
      Di[6 * (r + 3) + c] = -U[3 * c + r];
      Di[6 * (r + 3) + c + 3] = Ci[3 * r + c];
    }
  return ok;
}

}  // namespace dba
