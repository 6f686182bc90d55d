"""ctypes binding of the C-ABI in ``include/dba_b200.h`` (libdba_b200.so).

This is exactly the stub a maintainer of the reference's ``flowsplat`` package
would add to bind its ``dba`` module to the library.  There is
no fallback: if the shared library is missing or fails to load, importing the
solver raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_NAME = "libdba_b200.so"
_HERE = Path(__file__).resolve().parent

DBA_OK = 0
DBA_EINVAL = 1
DBA_ECAPACITY = 2
DBA_ENONFINITE = 3
DBA_ESOLVER = 4
DBA_ECALIB = 5
DBA_ECUDA = 6
DBA_ENCCL = 7
DBA_EDATA = 8
TRACE_MAX = 64

c_i32 = ctypes.c_int32
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


class ProblemDesc(ctypes.Structure):
    _fields_ = [
        ("n_frames", c_i32), ("height", c_i32), ("width", c_i32), ("n_edges", c_i32),
        ("ii", ctypes.POINTER(c_i32)), ("jj", ctypes.POINTER(c_i32)),
        ("fixed", ctypes.POINTER(ctypes.c_uint8)),
        ("optimize_intrinsics", c_i32), ("use_prior", c_i32), ("scale_gauge", c_i32),
        ("rank", c_i32), ("nranks", c_i32), ("freeze_disparities", c_i32),
    ]


class Options(ctypes.Structure):
    _fields_ = [
        ("iters", c_i32), ("lambda0", c_dbl), ("lambda_min", c_dbl), ("lambda_max", c_dbl),
        ("eta", c_dbl), ("alpha", c_dbl), ("d_min", c_dbl), ("tangent_max", c_dbl),
        ("calib_cond_max", c_dbl), ("damping_candidates", c_i32), ("refine", c_i32),
    ]


class Buffers(ctypes.Structure):
    _fields_ = [
        ("poses_in", c_vp), ("poses_out", c_vp), ("disps_in", c_vp), ("disps_out", c_vp),
        ("intr_in", c_vp), ("intr_out", c_vp), ("flow", c_vp), ("prior", c_vp),
        ("prior_mask", c_vp), ("workspace", c_vp), ("workspace_bytes", ctypes.c_size_t),
        ("stream", c_vp), ("nccl_comm", c_vp), ("prior_weight", c_vp),
    ]


class Report(ctypes.Structure):
    _fields_ = [
        ("status", c_i32), ("bad_edge", c_i32), ("iterations", c_i32), ("trials", c_i32),
        ("converged", c_i32), ("trace_len", c_i32), ("initial_energy", c_dbl),
        ("final_energy", c_dbl), ("lambda_final", c_dbl), ("scale", c_dbl),
        ("calib_condition", c_dbl), ("energy_trace", c_dbl * TRACE_MAX),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("n_reduced", c_i32), ("n_free_poses", c_i32), ("band_blocks", c_i32),
        ("frame_begin", c_i32), ("frame_end", c_i32), ("n_local_edges", c_i32),
        ("max_out_degree", c_i32), ("n_split", c_i32), ("gauge_frame", c_i32), ("solve_ctas", c_i32),
        ("workspace_bytes", ctypes.c_int64),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("launches", ctypes.c_int64), ("pass_launches", ctypes.c_int64),
        ("solve_launches", ctypes.c_int64), ("pass_ms", c_dbl), ("solve_ms", c_dbl),
        ("pass_runs", ctypes.c_int64), ("energy_launches", ctypes.c_int64), ("energy_ms", c_dbl),
    ]


EXPORTS = (
    "dba_version", "dba_status_string", "dba_partition", "dba_plan_create", "dba_plan_destroy",
    "dba_plan_get_info", "dba_plan_local_edges", "dba_solve", "dba_energy", "dba_build_system",
    "dba_plan_set_profiling", "dba_plan_get_stats", "dba_debug_trial", "dba_nccl_unique_id", "dba_nccl_comm_init", "dba_nccl_comm_destroy",
    "dba_dspt_read_flows", "dba_dspt_read_priors", "dba_dspt_load_flows",
    "dba_frame_distance", "dba_frontend_edges", "dba_backend_edges",
    "dba_prior_affine", "dba_fit_affine", "dba_synthetic_flows",
)

_lib = None


def lib_path() -> Path:
    override = os.environ.get("DBA_B200_LIB")
    return Path(override) if override else _HERE / LIB_NAME


def load():
    """Load libdba_b200.so (built in-tree by ``__graft_entry__.build()``)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise ImportError(
            f"{path} not found: the CUDA library is required (no CPU fallback); "
            "run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(path))
    P = ctypes.POINTER
    lib.dba_version.restype = c_i32
    lib.dba_status_string.restype = ctypes.c_char_p
    lib.dba_status_string.argtypes = [c_i32]
    lib.dba_partition.restype = c_i32
    lib.dba_partition.argtypes = [c_i32, c_i32, P(c_i32), c_i32, P(c_i32)]
    lib.dba_plan_create.restype = c_i32
    lib.dba_plan_create.argtypes = [P(ProblemDesc), P(c_vp)]
    lib.dba_plan_destroy.restype = None
    lib.dba_plan_destroy.argtypes = [c_vp]
    lib.dba_plan_get_info.restype = c_i32
    lib.dba_plan_get_info.argtypes = [c_vp, P(PlanInfo)]
    lib.dba_plan_local_edges.restype = c_i32
    lib.dba_plan_local_edges.argtypes = [c_vp, P(c_i32)]
    for name in ("dba_solve",):
        fn = getattr(lib, name)
        fn.restype = c_i32
        fn.argtypes = [c_vp, P(Options), P(Buffers), P(Report)]
    lib.dba_energy.restype = c_i32
    lib.dba_energy.argtypes = [c_vp, P(Options), P(Buffers), P(c_dbl)]
    lib.dba_build_system.restype = c_i32
    lib.dba_build_system.argtypes = [c_vp, P(Options), P(Buffers), P(c_dbl), P(c_dbl), P(c_dbl)]
    lib.dba_plan_set_profiling.restype = c_i32
    lib.dba_plan_set_profiling.argtypes = [c_vp, c_i32]
    lib.dba_plan_get_stats.restype = c_i32
    lib.dba_plan_get_stats.argtypes = [c_vp, P(Stats), c_i32]
    lib.dba_debug_trial.restype = c_i32
    lib.dba_debug_trial.argtypes = [c_vp, P(Options), P(Buffers), c_dbl, P(c_dbl), P(c_dbl),
                                    P(ctypes.c_float), P(c_dbl), P(c_dbl)]
    lib.dba_nccl_unique_id.restype = c_i32
    lib.dba_nccl_unique_id.argtypes = [P(ctypes.c_uint8)]
    lib.dba_nccl_comm_init.restype = c_i32
    lib.dba_nccl_comm_init.argtypes = [c_i32, P(ctypes.c_uint8), c_i32, P(c_vp)]
    lib.dba_nccl_comm_destroy.restype = c_i32
    lib.dba_nccl_comm_destroy.argtypes = [c_vp]
    Pf = P(ctypes.c_float)
    lib.dba_dspt_read_flows.restype = c_i32
    lib.dba_dspt_read_flows.argtypes = [ctypes.c_char_p, c_i32, P(c_i32), P(c_i32), c_i32, c_i32, Pf, c_i32,
                                        P(c_i32)]
    lib.dba_dspt_read_priors.restype = c_i32
    lib.dba_dspt_read_priors.argtypes = [ctypes.c_char_p, c_i32, P(c_i32), c_i32, c_i32, Pf, c_i32, P(c_i32)]
    lib.dba_dspt_load_flows.restype = c_i32
    lib.dba_dspt_load_flows.argtypes = [ctypes.c_char_p, c_i32, P(c_i32), P(c_i32), c_i32, c_i32, c_vp, c_vp,
                                        ctypes.c_int64, c_i32, c_vp, P(c_i32)]
    lib.dba_frame_distance.restype = c_i32
    lib.dba_frame_distance.argtypes = [c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_dbl, c_vp,
                                       c_vp]
    lib.dba_frontend_edges.restype = c_i32
    lib.dba_frontend_edges.argtypes = [c_i32, P(c_i32), c_i32, c_i32, P(c_i32), P(c_i32), P(c_i32), c_i32,
                                       c_i32, P(c_i32), P(c_i32), P(c_i32)]
    lib.dba_backend_edges.restype = c_i32
    lib.dba_backend_edges.argtypes = [c_i32, P(c_i32), P(c_dbl), c_i32, c_i32, c_i32, P(c_i32), P(c_i32),
                                      c_i32, P(c_i32), P(c_i32), P(c_i32)]
    lib.dba_prior_affine.restype = c_i32
    lib.dba_prior_affine.argtypes = [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]
    lib.dba_fit_affine.restype = c_i32
    lib.dba_fit_affine.argtypes = [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl, c_vp]
    lib.dba_synthetic_flows.restype = c_i32
    lib.dba_synthetic_flows.argtypes = [c_i32, c_i32, P(c_dbl), c_dbl, c_i32, c_vp, c_vp, c_vp, c_i32, c_vp,
                                        c_vp, c_vp, c_vp]
    _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().dba_status_string(int(code)).decode()
