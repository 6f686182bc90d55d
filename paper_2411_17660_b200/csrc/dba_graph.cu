// Frame-graph construction: the frame
// distance that ranks candidate edges, computed on the GPU, and the frontend /
// backend edge-list builders on the host.  Conventions G1-G4 are written out in
// oracle/graph.py (the CPU restatement these results are compared with bit for
// bit) and DESIGN.md §Graph.
//
// frame_distance_kernel: one warp per ordered pair (a, b).  Lane l walks pixels
// p = l, l+32, ... of frame a, accumulating |flow_full| and |flow_rot| in float64
// with round-to-nearest intrinsics (no contraction into FMA), then a fixed halving
// shuffle tree — the same operation sequence as the oracle, so the distances and
// therefore the edge ranking are bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <set>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/dba_b200.h"

namespace {

constexpr double kZMin = 1e-4;  // geometry.py:17

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// geometry.py:35-41
__device__ void quat_to_matrix(const double* q, double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = sub(1.0, mul(2.0, add(mul(y, y), mul(z, z))));
  R[1] = mul(2.0, sub(mul(x, y), mul(w, z)));
  R[2] = mul(2.0, add(mul(x, z), mul(w, y)));
  R[3] = mul(2.0, add(mul(x, y), mul(w, z)));
  R[4] = sub(1.0, mul(2.0, add(mul(x, x), mul(z, z))));
  R[5] = mul(2.0, sub(mul(y, z), mul(w, x)));
  R[6] = mul(2.0, sub(mul(x, z), mul(w, y)));
  R[7] = mul(2.0, add(mul(y, z), mul(w, x)));
  R[8] = sub(1.0, mul(2.0, add(mul(x, x), mul(y, y))));
}

struct DistArgs {
  int n_pairs, H, W;
  const double* poses;
  const float* disps;
  const double* intr;
  const int* ia;
  const int* ib;
  double beta;
  double* out;
};

__global__ void __launch_bounds__(256) frame_distance_kernel(const DistArgs A) {
  const int pair = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (pair >= A.n_pairs) return;
  const int a = A.ia[pair], b = A.ib[pair];
  double Ra[9], Rb[9], R[9], t[3];
  quat_to_matrix(A.poses + 7 * (size_t)a, Ra);
  quat_to_matrix(A.poses + 7 * (size_t)b, Rb);
  const double* ta = A.poses + 7 * (size_t)a + 4;
  const double* tb = A.poses + 7 * (size_t)b + 4;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      R[3 * r + c] = add(add(mul(Rb[3 * r], Ra[3 * c]), mul(Rb[3 * r + 1], Ra[3 * c + 1])),
                         mul(Rb[3 * r + 2], Ra[3 * c + 2]));
  for (int r = 0; r < 3; ++r)
    t[r] = sub(tb[r], add(add(mul(R[3 * r], ta[0]), mul(R[3 * r + 1], ta[1])), mul(R[3 * r + 2], ta[2])));
  const double fx = A.intr[0], fy = A.intr[1], cx = A.intr[2], cy = A.intr[3];
  const int P = A.H * A.W;
  const float* d_a = A.disps + (size_t)a * P;
  double sf = 0.0, sr = 0.0;
  int nf = 0, nr = 0;
  for (int p = lane; p < P; p += 32) {
    const double u = (double)(p % A.W), v = (double)(p / A.W);
    const double x = __ddiv_rn(sub(u, cx), fx), y = __ddiv_rn(sub(v, cy), fy);
    const double d = (double)d_a[p];
    // homogeneous X~ = R q + t d, q = (x, y, 1); flows in normalised coordinates x f
    const double Xr = add(add(mul(R[0], x), mul(R[1], y)), R[2]);
    const double Yr = add(add(mul(R[3], x), mul(R[4], y)), R[5]);
    const double Zr = add(add(mul(R[6], x), mul(R[7], y)), R[8]);
    if (d > 0.0) {
      const double Xh = add(Xr, mul(t[0], d)), Yh = add(Yr, mul(t[1], d)), Zh = add(Zr, mul(t[2], d));
      if (Zh > mul(kZMin, d)) {
        const double du = mul(fx, sub(__ddiv_rn(Xh, Zh), x));
        const double dv = mul(fy, sub(__ddiv_rn(Yh, Zh), y));
        sf = add(sf, __dsqrt_rn(add(mul(du, du), mul(dv, dv))));
        ++nf;
      }
    }
    if (Zr > kZMin) {
      const double du = mul(fx, sub(__ddiv_rn(Xr, Zr), x));
      const double dv = mul(fy, sub(__ddiv_rn(Yr, Zr), y));
      sr = add(sr, __dsqrt_rn(add(mul(du, du), mul(dv, dv))));
      ++nr;
    }
  }
  // halving tree: lane l (< m) takes lane l + m, the oracle's acc[:m] + acc[m:2m]
  for (int m = 16; m >= 1; m >>= 1) {
    const double of = __shfl_down_sync(0xffffffffu, sf, m), orr = __shfl_down_sync(0xffffffffu, sr, m);
    const int onf = __shfl_down_sync(0xffffffffu, nf, m), onr = __shfl_down_sync(0xffffffffu, nr, m);
    if (lane < m) {
      sf = add(sf, of);
      sr = add(sr, orr);
      nf += onf;
      nr += onr;
    }
  }
  if (lane == 0) {
    const double mf = nf > 0 ? __ddiv_rn(sf, (double)nf) : INFINITY;
    const double mr = nr > 0 ? __ddiv_rn(sr, (double)nr) : INFINITY;
    A.out[pair] = add(mul(A.beta, mf), mul(sub(1.0, A.beta), mr));
  }
}

}  // namespace

extern "C" {

int dba_frame_distance(int32_t n_frames, int32_t H, int32_t W, const double* poses, const float* disps,
                       const double* intr, int32_t n_pairs, const int32_t* ia, const int32_t* ib, double beta,
                       double* out, void* stream) {
  if (n_frames <= 0 || H <= 0 || W <= 0 || n_pairs < 0) return DBA_EINVAL;
  if (n_pairs == 0) return DBA_OK;
  if (!poses || !disps || !intr || !ia || !ib || !out) return DBA_EINVAL;
  DistArgs a{n_pairs, H, W, poses, disps, intr, ia, ib, beta, out};
  const int threads = 256, pairs_per_block = threads / 32;
  frame_distance_kernel<<<(n_pairs + pairs_per_block - 1) / pairs_per_block, threads, 0,
                          reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? DBA_OK : DBA_ECUDA;
}

int dba_frontend_edges(int32_t n_window, const int32_t* window, int32_t radius, int32_t n_existing,
                       const int32_t* ei, const int32_t* ej, const int32_t* age, int32_t max_age, int32_t capacity,
                       int32_t* out_i, int32_t* out_j, int32_t* n_out) {
  if (n_window < 0 || radius < 0 || n_existing < 0 || !n_out || (n_window > 0 && !window) ||
      (n_existing > 0 && (!ei || !ej)))
    return DBA_EINVAL;
  std::set<int> inwin(window, window + n_window);
  std::set<std::pair<int, int>> cand;
  for (int a = 0; a < n_window; ++a)
    for (int b = a + 1; b < std::min(n_window, a + radius + 1); ++b) {
      cand.insert({window[a], window[b]});
      cand.insert({window[b], window[a]});
    }
  std::set<std::pair<int, int>> old_;
  for (int e = 0; e < n_existing; ++e)
    if (ei[e] != ej[e] && inwin.count(ei[e]) && inwin.count(ej[e])) cand.insert({ei[e], ej[e]});
  if (age)
    for (int e = 0; e < n_existing; ++e)
      if (age[e] > max_age) old_.insert({ei[e], ej[e]});
  int n = 0;
  for (const auto& e : cand) {
    if (old_.count(e)) continue;
    if (n < capacity) {
      out_i[n] = e.first;
      out_j[n] = e.second;
    }
    ++n;
  }
  *n_out = n;
  return n <= capacity ? DBA_OK : DBA_ECAPACITY;
}

int dba_backend_edges(int32_t n_frames, const int32_t* frames, const double* dist, int32_t window, int32_t max_edges,
                      int32_t n_loop, const int32_t* li, const int32_t* lj, int32_t capacity, int32_t* out_i,
                      int32_t* out_j, int32_t* n_out) {
  if (n_frames < 0 || window < 0 || max_edges < 0 || n_loop < 0 || !n_out || (n_frames > 0 && (!frames || !dist)) ||
      (n_loop > 0 && (!li || !lj)))
    return DBA_EINVAL;
  std::set<std::pair<int, int>> chosen;
  for (int e = 0; e < n_loop; ++e) chosen.insert({li[e], lj[e]});
  const int w0 = std::max(0, n_frames - window);
  std::vector<std::tuple<double, int, int>> keys;
  for (int a = w0; a < n_frames; ++a)
    for (int b = a + 1; b < n_frames; ++b) {
      const double m = 0.5 * (dist[(size_t)a * n_frames + b] + dist[(size_t)b * n_frames + a]);
      if (std::isfinite(m)) keys.emplace_back(m, frames[a], frames[b]);
    }
  std::sort(keys.begin(), keys.end());
  for (const auto& k : keys) {
    const std::pair<int, int> e1{std::get<1>(k), std::get<2>(k)}, e2{std::get<2>(k), std::get<1>(k)};
    const int add = (chosen.count(e1) ? 0 : 1) + (chosen.count(e2) ? 0 : 1);
    if ((int)chosen.size() + add > max_edges) break;
    chosen.insert(e1);
    chosen.insert(e2);
  }
  int n = 0;
  for (const auto& e : chosen) {
    if (n < capacity) {
      out_i[n] = e.first;
      out_j[n] = e.second;
    }
    ++n;
  }
  *n_out = n;
  return n <= capacity ? DBA_OK : DBA_ECAPACITY;
}

}  // extern "C"
