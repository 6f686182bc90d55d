/*
 * dba_b200.h — C-ABI of the B200-native dense bundle adjustment (DBA)
 * Gauss-Newton step (DROID-Splat, arXiv 2411.17660).
 *
 * Drop-in boundary.  The reference package declares a `dba` module
 * (/root/reference/pkg/src/flowsplat/__init__.py:8) whose contract is written
 * in /root/reference/SPEC.md:286-394:
 *
 *   energy(problem, state) -> scalar
 *   solve_ba(problem, state) -> state' + BAReport
 *   solve_ba_calib(problem, state) -> state' incl. theta
 *   energy_rgbd(problem, state, d*, alpha) -> scalar
 *
 * (the module file itself is absent from the reference; there is no upstream
 * FFI, so these entry points are what a ctypes/cffi binding of that module
 * would call — see INTEGRATION.md).  `dba_plan_create` replaces the
 * BAProblem's graph half (edges, fixed set, block flags),
 * `dba_solve` replaces solve_ba / solve_ba_calib (+ the prior term of
 * energy_rgbd), `dba_energy` replaces energy / energy_rgbd, and the dba_report
 * struct replaces BAReport.
 *
 * Conventions
 *  - Ownership: the caller owns every buffer (inputs, outputs, workspace).
 *    The library allocates only host-side plan metadata in dba_plan_create
 *    and never allocates device memory.
 *  - All buffer pointers in dba_buffers are DEVICE pointers; the problem
 *    descriptor's ii/jj/fixed are HOST pointers (read once at plan creation).
 *  - Poses: (N,7) float64 rows [qw,qx,qy,qz,tx,ty,tz], world->camera
 *    (geometry.py:72-81).  Disparities: (N,H,W) float32.  Intrinsics:
 *    (4,) float64 [fx,fy,cx,cy] (geometry.py:211-212).  Flow: (E_local,H,W,4)
 *    float32 [target_u, target_v, weight_u, weight_v] — the DSPT flow record
 *    (providers.py:12-15), rows in INPUT edge order restricted to this rank's
 *    edges (all edges when nranks == 1).
 *  - Errors: every entry point returns a DBA_* status; no C++ exception
 *    crosses the ABI.  DBA_ENONFINITE sets report->bad_edge (input edge id).
 *  - Threading: stream-ordered on `stream`.  The Levenberg-Marquardt
 *    accept/reject schedule runs on the device; dba_solve enqueues batches of
 *    trials and synchronises the stream once per batch (once per call when no
 *    trial is rejected) to read the controller state.  Distinct
 *    plans + workspaces may run concurrently on distinct streams; one plan
 *    must not be used concurrently.
 *  - Determinism: fixed reduction trees, no floating-point atomics; results
 *    are bitwise reproducible for a fixed plan (rank count, split count).
 */
#ifndef DBA_B200_H_
#define DBA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DBA_VERSION 1

/* status codes -> flowsplat.errors (errors.py:8-29) */
#define DBA_OK 0
#define DBA_EINVAL 1       /* ValueError / ConfigError */
#define DBA_ECAPACITY 2    /* CapacityError (compiled limits) */
#define DBA_ENONFINITE 3   /* NumericalError, report->bad_edge */
#define DBA_ESOLVER 4      /* SolverFailure */
#define DBA_ECALIB 5       /* CalibrationDegenerateError */
#define DBA_ECUDA 6        /* CUDA runtime failure */
#define DBA_ENCCL 7        /* NCCL failure */
#define DBA_EDATA 8        /* DataError: missing / malformed DSPT provider file */

#define DBA_TRACE_MAX 64

typedef struct dba_plan dba_plan;

/* Graph half of SPEC BAProblem. */
typedef struct {
  int32_t n_frames;            /* N */
  int32_t height, width;       /* H, W (the 1/8-resolution BA grid) */
  int32_t n_edges;             /* E (global) */
  const int32_t* ii;           /* host (E,) source frame per edge */
  const int32_t* jj;           /* host (E,) target frame per edge */
  const uint8_t* fixed;        /* host (N,) 1 = pose held fixed (gauge) */
  int32_t optimize_intrinsics; /* solve_ba_calib */
  int32_t use_prior;           /* energy_rgbd term */
  int32_t scale_gauge;         /* -1 auto (1 fixed pose, no prior), 0 off, 1 on */
  int32_t rank, nranks;        /* edge sharding by source frame */
  int32_t freeze_disparities;  /* disparity block not updated (SPEC BAProblem block flags):
                                  motion-only pose solves, fill_nonkeyframe_poses */
} dba_problem_desc;

/* Solver knobs. */
typedef struct {
  int32_t iters;        /* accepted GN iterations budget (4 frontend, 8 backend) */
  double lambda0;       /* initial damping on the reduced pose system */
  double lambda_min;    /* floor after an accepted step (lambda /= 10) */
  double lambda_max;    /* rejects beyond this stop the solve */
  double eta;           /* disparity-diagonal damping */
  double alpha;         /* prior weight (1e-3) */
  double d_min;         /* disparity floor (1e-6) */
  double tangent_max;   /* per-pose tangent clamp (1) */
  double calib_cond_max;/* A9 degeneracy threshold */
  int32_t damping_candidates; /* lambda values factored per round by dba_solve (lambda, 10 lambda,
                                 ...; 0 = default 3, max 3).  A rejection then costs no new
                                 factorisation; results are identical for every value. */
  int32_t refine;       /* 0 (default): one block factorisation + substitution per damping
                           value; 1: plus one step of iterative refinement (float64 residual
                           from the original band, the stored factors re-applied).  Measured
                           on the committed fixtures: both within the 1e-4 bar (C3 noisy max
                           5.1e-6 without, 5.4e-6 with: the Cholesky-form factorisation is
                           already as accurate as LAPACK's), refinement costs +18 % per C3 call */
} dba_options;

typedef struct {
  const double* poses_in;   /* (N,7) */
  double* poses_out;        /* (N,7) */
  const float* disps_in;    /* (N,H,W) */
  float* disps_out;         /* (N,H,W) (only this rank's frames are written) */
  const double* intr_in;    /* (4,) */
  double* intr_out;         /* (4,) */
  const float* flow;        /* (E_local,H,W,4) */
  const float* prior;       /* (N,H,W) or NULL */
  const uint8_t* prior_mask;/* (N,H,W) or NULL */
  void* workspace;          /* >= dba_plan_workspace_bytes, 256-byte aligned */
  size_t workspace_bytes;
  void* stream;             /* cudaStream_t (NULL = legacy default stream) */
  void* nccl_comm;          /* ncclComm_t for nranks > 1, else NULL */
  const float* prior_weight;/* (N,) per-frame multiplier of alpha, or NULL (= 1); the Eq. 5
                               affine prior s d + o = d* enters as d*' = (d* - o)/s, weight s^2 */
} dba_buffers;

/* SPEC BAReport + diagnostics. */
typedef struct {
  int32_t status;
  int32_t bad_edge;         /* input edge id for DBA_ENONFINITE, else -1 */
  int32_t iterations;       /* accepted GN iterations */
  int32_t trials;           /* linearize+solve+back-substitute passes after the first */
  int32_t converged;        /* 1 if the damping schedule ran out without a decrease */
  int32_t trace_len;
  double initial_energy;
  double final_energy;
  double lambda_final;
  double scale;             /* mono gauge factor applied at the end (1 if off) */
  double calib_condition;   /* A9 estimate of the last solve (0 if not calibrating) */
  double energy_trace[DBA_TRACE_MAX];
} dba_report;

typedef struct {
  int32_t n_reduced;        /* size of the reduced pose(+theta) system */
  int32_t n_free_poses;
  int32_t band_blocks;      /* block bandwidth BW of the reduced system */
  int32_t frame_begin, frame_end;   /* this rank's source frames */
  int32_t n_local_edges;
  int32_t max_out_degree;
  int32_t n_split;          /* pixel splits per frame in the fused pass */
  int32_t gauge_frame;      /* -1 when the scale gauge is off */
  int32_t solve_ctas;       /* 1: one factorisation chain, 2: top/bottom chains */
  int64_t workspace_bytes;
} dba_plan_info;

int dba_version(void);
const char* dba_status_string(int status);

/* Frame partition used for edge sharding: contiguous source-frame ranges with
 * balanced (out-degree + 1) weight.  bounds: (nranks+1,) host output. */
int dba_partition(int32_t n_frames, int32_t n_edges, const int32_t* ii, int32_t nranks,
                  int32_t* bounds);

/* Builds the plan of one graph.  DBA_ECAPACITY (CapacityError) when the graph exceeds
 * the compiled limits: out-degree (edges per source frame) > 16, or a reduced-system
 * block bandwidth > 24 pose blocks AFTER the plan's band ordering (identity, ring fold
 * or reverse Cuthill-McKee, the narrowest wins: a radius-r covisibility graph has
 * 2r, a ring closure of it stays at ~4r).  A workspace holds one plan's metadata;
 * plans may share a workspace (re-uploaded when another plan used it last). */
int dba_plan_create(const dba_problem_desc* desc, dba_plan** out);
void dba_plan_destroy(dba_plan* plan);
int dba_plan_get_info(const dba_plan* plan, dba_plan_info* info);
/* (E_local,) host output: input edge id of each local flow row. */
int dba_plan_local_edges(const dba_plan* plan, int32_t* edge_ids);

/* solve_ba / solve_ba_calib: damped Gauss-Newton with Schur elimination. */
int dba_solve(dba_plan* plan, const dba_options* opt, const dba_buffers* buf,
              dba_report* report);

/* energy / energy_rgbd at the input state (poses_in, disps_in, intr_in). */
int dba_energy(dba_plan* plan, const dba_options* opt, const dba_buffers* buf,
               double* energy);

/* Test hook: the Schur-reduced system at the input state, expanded to a dense
 * host (n_reduced x n_reduced) matrix + host rhs (n_reduced,) + energy.  With
 * nccl_comm == NULL and nranks > 1 this is this rank's PARTIAL system. */
int dba_build_system(dba_plan* plan, const dba_options* opt, const dba_buffers* buf,
                     double* S_host, double* y_host, double* energy);

/* Launch accounting and live kernel timing.  With profiling enabled the library
 * brackets every fused-pass and solve launch with CUDA events on the launching
 * stream and accumulates their durations (resolved at each stream sync). */
typedef struct {
  int64_t launches;        /* all kernels launched by the library */
  int64_t pass_launches;   /* fused linearising passes (system build) */
  int64_t solve_launches;  /* reduced-system factorisations */
  double pass_ms;          /* summed CUDA-event time of the pass launches */
  double solve_ms;         /* summed CUDA-event time of the solve launches */
  int64_t pass_runs;       /* pass launches that ran (the rest were gated off by a rejection) */
  int64_t energy_launches; /* energy-only trial passes (back-substitution + residuals) */
  double energy_ms;        /* summed CUDA-event time of the energy-only passes */
} dba_stats;

int dba_plan_set_profiling(dba_plan* plan, int32_t enable);
int dba_plan_get_stats(dba_plan* plan, dba_stats* stats, int32_t reset);

/* Test hook: linearise at the input state, solve (S + lambda I) once, run one
 * trial pass, and return the step (n_reduced,), the trial poses (N,7), the
 * trial disparities (N,H,W) and intrinsics (4,) (all HOST) and the trial energy. */
int dba_debug_trial(dba_plan* plan, const dba_options* opt, const dba_buffers* buf, double lambda,
                    double* delta, double* poses_n, float* disps_n, double* intr_n, double* energy_n);

/* NCCL bootstrap helpers (the library links NCCL; ids travel as 128 bytes). */
int dba_nccl_unique_id(uint8_t id_out[128]);
int dba_nccl_comm_init(int32_t nranks, const uint8_t id[128], int32_t rank, void** comm_out);
int dba_nccl_comm_destroy(void* comm);

/* Provider-tensor ingestion (replaces PrecomputedProviders, providers.py:401-424).
 * DSPT files (providers.py:12-15, :368-399): "DSPT", u32 version = 1, u32 H, W,
 * C, then H*W*C little-endian float32.  Flow files <dir>/flow_{i:06d}_{j:06d}.dspt
 * (C = 4) land directly in the dba_buffers.flow layout, record e = edge
 * (ii[e], jj[e]), with the weights clipped to [0, 1] as provide_correspondences
 * does (:415-420; NaN kept).  Priors <dir>/prior_{k:06d}.dspt (C = 1) are clamped
 * below at 1e-6 (:422-424).  A missing, malformed (magic, version, length), or
 * wrong-shape file returns DBA_EDATA with the smallest failing index in *bad_*.
 * n_threads <= 0: one reader per hardware thread. */
int dba_dspt_read_flows(const char* directory, int32_t n_edges, const int32_t* ii, const int32_t* jj, int32_t H,
                        int32_t W, float* out_host, int32_t n_threads, int32_t* bad_edge);
int dba_dspt_read_priors(const char* directory, int32_t n_frames, const int32_t* frames, int32_t H, int32_t W,
                         float* out_host, int32_t n_threads, int32_t* bad_frame);
/* Same flow records into DEVICE memory: file reads fill one half of the
 * caller's pinned `staging` buffer while the other half is copied
 * asynchronously on `stream`; staging_bytes must hold >= 2 records
 * (2 * 16 * H * W bytes).  Returns after the last copy has completed. */
int dba_dspt_load_flows(const char* directory, int32_t n_edges, const int32_t* ii, const int32_t* jj, int32_t H,
                        int32_t W, float* out_device, void* staging, int64_t staging_bytes, int32_t n_threads,
                        void* stream, int32_t* bad_edge);

/* Frame-graph construction (the map_state
 * operations that produce ii/jj).  Conventions G1-G4: oracle/graph.py, DESIGN.md.
 *
 * dba_frame_distance: mean_flow_distance for n_pairs ordered
 * pairs (ia[k] -> ib[k]) of frames in poses (N,7) / disps (N,H,W) / intr (4,):
 * beta * mean |full flow| + (1 - beta) * mean |rotation-only flow| over frame
 * ia's pixels in front of the camera.  DEVICE pointers; out (n_pairs,) float64;
 * float64 without contraction in a fixed reduction order (bitwise reproducible).
 * Stream-ordered, no synchronisation. */
int dba_frame_distance(int32_t n_frames, int32_t H, int32_t W, const double* poses, const float* disps,
                       const double* intr, int32_t n_pairs, const int32_t* ia, const int32_t* ib, double beta,
                       double* out, void* stream);
/* build_frontend_edges: ordered pairs of the window at most
 * `radius` apart (window order) plus existing in-window edges, minus edges whose
 * age exceeds max_age; sorted by (i, j).  HOST pointers; age may be NULL.
 * Writes up to `capacity` edges, *n_out = total (DBA_ECAPACITY if larger). */
int dba_frontend_edges(int32_t n_window, const int32_t* window, int32_t radius, int32_t n_existing,
                       const int32_t* ei, const int32_t* ej, const int32_t* age, int32_t max_age, int32_t capacity,
                       int32_t* out_i, int32_t* out_j, int32_t* n_out);
/* build_backend_graph: over the last `window` of the n_frames
 * keyframes `frames` (ascending), unordered pairs ranked by (mean of the two
 * directed distances dist[a*n+b], dist[b*n+a]; frames[a]; frames[b]), each adding
 * both directions, loop edges always kept, at most max_edges edges; sorted by
 * (i, j).  HOST pointers; dist is (n_frames, n_frames) float64. */
int dba_backend_edges(int32_t n_frames, const int32_t* frames, const double* dist, int32_t window, int32_t max_edges,
                      int32_t n_loop, const int32_t* li, const int32_t* lj, int32_t capacity, int32_t* out_i,
                      int32_t* out_j, int32_t* n_out);

/* P-RGBD block-coordinate descent, Eq. 5
 * E_reg,m = alpha sum m (d* - (s_i d + o_i))^2 with per-frame scale/offset.
 * dba_prior_affine: stage A (s, o frozen) input to dba_solve — prior_out =
 *   (d* - o) / s (N,P) and weight_out = s^2 (N,) for dba_buffers.prior /
 *   prior_weight (same energy and normal equations).
 * dba_fit_affine: stage B closed form — per frame the 2x2 least-squares (s, o)
 *   over mask pixels given disps, in place; s clamped to >= s_min; frames with
 *   no mask pixel keep (s, o); constant-disparity frames keep s.
 * DEVICE pointers, stream-ordered; scale/offset are (N,) float64. */
int dba_prior_affine(int32_t n_frames, int32_t n_pixels, const float* prior, const double* scale,
                     const double* offset, float* prior_out, float* weight_out, void* stream);
int dba_fit_affine(int32_t n_frames, int32_t n_pixels, const float* disps, const float* prior, const uint8_t* mask,
                   double* scale, double* offset, double s_min, void* stream);

/* GPU synthetic correspondence provider: flow records of
 * SyntheticProviders.provide_correspondences (providers.py:318-338) for n_edges
 * edges (ii[e] -> jj[e]) of the analytic scene (outer sphere of outer_radius,
 * spherical occluders (n,4) [centre, radius], camera poses c2w / w2c (F,7)),
 * one thread per edge-pixel, float64, into out (E,H,W,4) float32.  intr is a
 * HOST (4,) array; every other pointer is DEVICE.  Pixel noise is not added. */
int dba_synthetic_flows(int32_t H, int32_t W, const double* intr, double outer_radius, int32_t n_occluders,
                        const double* occluders, const double* c2w, const double* w2c, int32_t n_edges,
                        const int32_t* ii, const int32_t* jj, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DBA_B200_H_ */
