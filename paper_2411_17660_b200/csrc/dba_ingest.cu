// DSPT flow / prior ingestion: provider tensors on disk -> the pass kernel's
// (E, H, W, 4) float32 layout, host or device.
//
// File format (providers.py:12-15, write_dspt / read_dspt :368-399): "DSPT",
// u32 version (1), u32 H, u32 W, u32 C, then H*W*C little-endian float32,
// row-major.  Flow files are flow_{i:06d}_{j:06d}.dspt with C = 4
// (target u, target v, weight u, weight v); PrecomputedProviders clips the
// weights to [0, 1] (providers.py:415-420), prior_{k:06d}.dspt (C = 1) is
// clamped below at 1e-6 (:422-424).  A flow record is therefore read straight
// into its slot of the output (no repacking): one pread per file, spread over a
// pool of host threads, and for device output streamed through a caller-owned
// pinned staging buffer whose halves alternate between disk reads and async
// host->device copies.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/dba_b200.h"

namespace {

constexpr uint32_t kDsptVersion = 1;
constexpr size_t kHeader = 20;

// read one DSPT file into dst (expected shape H x W x C); returns DBA_OK or DBA_EDATA
int read_record(const char* path, int H, int W, int C, float* dst) {
  const int fd = open(path, O_RDONLY);
  if (fd < 0) return DBA_EDATA;  // missing provider tensor
  unsigned char hdr[kHeader];
  const ssize_t n = pread(fd, hdr, kHeader, 0);
  int status = DBA_OK;
  const size_t payload = sizeof(float) * (size_t)H * W * C;
  if (n < (ssize_t)kHeader || std::memcmp(hdr, "DSPT", 4) != 0) {
    status = DBA_EDATA;  // not a DSPT tensor file
  } else {
    uint32_t f[4];
    std::memcpy(f, hdr + 4, sizeof(f));  // little-endian host
    const off_t size = lseek(fd, 0, SEEK_END);
    if (f[0] != kDsptVersion) {
      status = DBA_EDATA;  // unsupported version
    } else if ((uint64_t)size != kHeader + 4ull * f[1] * f[2] * f[3]) {
      status = DBA_EDATA;  // truncated payload
    } else if (f[3] != (uint32_t)C || f[1] != (uint32_t)H || f[2] != (uint32_t)W) {
      status = DBA_EDATA;  // wrong channel count / resolution
    } else {
      size_t done = 0;
      unsigned char* out = reinterpret_cast<unsigned char*>(dst);
      while (done < payload) {
        const ssize_t r = pread(fd, out + done, payload - done, (off_t)(kHeader + done));
        if (r <= 0) {
          status = DBA_EDATA;
          break;
        }
        done += (size_t)r;
      }
    }
  }
  close(fd);
  return status;
}

// PrecomputedProviders.provide_correspondences: weights clipped to [0, 1]
// (np.clip keeps NaN: the comparisons below are false for NaN)
void clip_weights(float* rec, size_t pixels) {
  for (size_t p = 0; p < pixels; ++p) {
    float* w = rec + 4 * p + 2;
    for (int c = 0; c < 2; ++c) w[c] = w[c] < 0.f ? 0.f : (w[c] > 1.f ? 1.f : w[c]);
  }
}

// provide_depth_prior: max(d, 1e-6) (NaN kept, as np.maximum does)
void clamp_prior(float* rec, size_t pixels) {
  for (size_t p = 0; p < pixels; ++p) rec[p] = rec[p] < 1e-6f ? 1e-6f : rec[p];
}

int pick_threads(int requested, int work) {
  int n = requested > 0 ? requested : (int)std::thread::hardware_concurrency();
  return std::max(1, std::min({n, work, 64}));
}

// records [r0, r1) -> dst + (r - r0) * rec_floats; first failing record -> *bad
template <typename Fn>
int parallel_records(int r0, int r1, int threads, int* bad, Fn&& fn) {
  std::atomic<int> next{r0};
  std::atomic<int> first_bad{INT_MAX};
  auto worker = [&]() {
    for (int r = next++; r < r1; r = next++)
      if (fn(r) != DBA_OK) {
        int cur = first_bad.load();
        while (r < cur && !first_bad.compare_exchange_weak(cur, r)) {
        }
      }
  };
  const int nt = pick_threads(threads, r1 - r0);
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (first_bad.load() != INT_MAX) {
    if (bad) *bad = first_bad.load();
    return DBA_EDATA;
  }
  return DBA_OK;
}

void flow_path(char* buf, size_t n, const char* dir, int i, int j) {
  std::snprintf(buf, n, "%s/flow_%06d_%06d.dspt", dir, i, j);
}

}  // namespace

extern "C" {

int dba_dspt_read_flows(const char* directory, int32_t n_edges, const int32_t* ii, const int32_t* jj, int32_t H,
                        int32_t W, float* out, int32_t n_threads, int32_t* bad_edge) {
  if (bad_edge) *bad_edge = -1;
  if (!directory || n_edges < 0 || (n_edges > 0 && (!ii || !jj || !out)) || H <= 0 || W <= 0) return DBA_EINVAL;
  const size_t P = (size_t)H * W;
  return parallel_records(0, n_edges, n_threads, bad_edge, [&](int e) {
    char path[4096];
    flow_path(path, sizeof(path), directory, ii[e], jj[e]);
    float* rec = out + 4 * P * (size_t)e;
    const int s = read_record(path, H, W, 4, rec);
    if (s == DBA_OK) clip_weights(rec, P);
    return s;
  });
}

int dba_dspt_read_priors(const char* directory, int32_t n_frames, const int32_t* frames, int32_t H, int32_t W,
                         float* out, int32_t n_threads, int32_t* bad_frame) {
  if (bad_frame) *bad_frame = -1;
  if (!directory || n_frames < 0 || (n_frames > 0 && (!frames || !out)) || H <= 0 || W <= 0) return DBA_EINVAL;
  const size_t P = (size_t)H * W;
  return parallel_records(0, n_frames, n_threads, bad_frame, [&](int k) {
    char path[4096];
    std::snprintf(path, sizeof(path), "%s/prior_%06d.dspt", directory, frames[k]);
    float* rec = out + P * (size_t)k;
    const int s = read_record(path, H, W, 1, rec);
    if (s == DBA_OK) clamp_prior(rec, P);
    return s;
  });
}

int dba_dspt_load_flows(const char* directory, int32_t n_edges, const int32_t* ii, const int32_t* jj, int32_t H,
                        int32_t W, float* out_device, void* staging, int64_t staging_bytes, int32_t n_threads,
                        void* stream, int32_t* bad_edge) {
  if (bad_edge) *bad_edge = -1;
  if (!directory || n_edges < 0 || (n_edges > 0 && (!ii || !jj || !out_device || !staging)) || H <= 0 || W <= 0)
    return DBA_EINVAL;
  const size_t P = (size_t)H * W, rec = 4 * P * sizeof(float);
  const int per_half = (int)std::min<int64_t>(staging_bytes / 2 / (int64_t)rec, INT_MAX);
  if (n_edges > 0 && per_half < 1) return DBA_EINVAL;  // staging must hold two records
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaEvent_t done[2];
  for (auto& e : done)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return DBA_ECUDA;
  int status = DBA_OK;
  bool used[2] = {false, false};
  unsigned char* half[2] = {reinterpret_cast<unsigned char*>(staging),
                            reinterpret_cast<unsigned char*>(staging) + (size_t)per_half * rec};
  for (int r0 = 0, h = 0; r0 < n_edges && status == DBA_OK; r0 += per_half, h ^= 1) {
    const int r1 = std::min(n_edges, r0 + per_half);
    // the copy that last read this half must have finished before it is refilled
    if (used[h] && cudaEventSynchronize(done[h]) != cudaSuccess) {
      status = DBA_ECUDA;
      break;
    }
    status = parallel_records(r0, r1, n_threads, bad_edge, [&](int e) {
      char path[4096];
      flow_path(path, sizeof(path), directory, ii[e], jj[e]);
      float* dst = reinterpret_cast<float*>(half[h] + (size_t)(e - r0) * rec);
      const int s = read_record(path, H, W, 4, dst);
      if (s == DBA_OK) clip_weights(dst, P);
      return s;
    });
    if (status != DBA_OK) break;
    if (cudaMemcpyAsync(reinterpret_cast<unsigned char*>(out_device) + (size_t)r0 * rec, half[h],
                        (size_t)(r1 - r0) * rec, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventRecord(done[h], st) != cudaSuccess) {
      status = DBA_ECUDA;
      break;
    }
    used[h] = true;
  }
  for (int h = 0; h < 2; ++h) {
    if (used[h] && cudaEventSynchronize(done[h]) != cudaSuccess && status == DBA_OK) status = DBA_ECUDA;
    cudaEventDestroy(done[h]);
  }
  return status;
}

}  // extern "C"
