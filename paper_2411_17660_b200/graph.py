"""Frame-graph construction: the edge lists ii/jj fed to the BA.

The map_state operations of ``SPEC.md:134-169`` — ``mean_flow_distance``,
``build_frontend_edges`` and ``build_backend_graph`` — on the C-ABI of
``libdba_b200.so`` (``csrc/dba_graph.cu``): the all-pairs frame distance runs on the
GPU (one warp per ordered pair, float64, fixed reduction order), the ranking and
selection on the host.  Conventions G1-G4 are stated in ``oracle/graph.py`` and
DESIGN.md §Graph; results are bit-identical to that restatement.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import CapacityError, ConfigError

_I32P = ctypes.POINTER(ctypes.c_int32)

BACKEND_WINDOW = 150      # Supp. §1.1 "window of max. 150 frames"
BACKEND_MAX_EDGES = 1500  # "... using up to 1500 edges"
FRONTEND_RADIUS = 3
MAX_EDGE_AGE = 30         # Supp. §1.1 "increase this value from 25 to 30"


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _check(code):
    if code == _lib.DBA_OK:
        return
    if code == _lib.DBA_EINVAL:
        raise ConfigError(_lib.status_string(code))
    if code == _lib.DBA_ECAPACITY:
        raise CapacityError(_lib.status_string(code))
    raise RuntimeError(f"libdba_b200: {_lib.status_string(code)} (status {code})")


def frame_distances(poses, disps, intr, ia, ib, beta=0.5, device=None):
    """mean_flow_distance(ia[k] -> ib[k]) for every requested ordered pair (float64).

    poses (N,7) [qw,qx,qy,qz,tx,ty,tz] world->camera, disps (N,H,W), intr (4,)."""
    import torch

    from .dba import _device
    lib = _lib.load()
    dev = _device(device)
    P7 = torch.as_tensor(poses, dtype=torch.float64, device=dev).contiguous()
    D = torch.as_tensor(disps, dtype=torch.float32, device=dev).contiguous()
    K = torch.as_tensor(intr, dtype=torch.float64, device=dev).contiguous()
    a = torch.as_tensor(_i32(ia), device=dev)
    b = torch.as_tensor(_i32(ib), device=dev)
    n = int(a.numel())
    if b.numel() != n:
        raise ConfigError("ia and ib must have the same length")
    N, H, W = D.shape
    if n and (int(a.min()) < 0 or int(b.min()) < 0 or int(a.max()) >= N or int(b.max()) >= N):
        raise ConfigError("frame index out of range")
    out = torch.empty(n, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream(dev)
    with torch.cuda.device(dev):
        _check(lib.dba_frame_distance(N, H, W, ctypes.c_void_p(P7.data_ptr()), ctypes.c_void_p(D.data_ptr()),
                                      ctypes.c_void_p(K.data_ptr()), n, ctypes.c_void_p(a.data_ptr()),
                                      ctypes.c_void_p(b.data_ptr()), float(beta),
                                      ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(st.cuda_stream)))
    return out.cpu().numpy()


def mean_flow_distance(poses, disps, intr, a, b, beta=0.5, device=None):
    """SPEC.md:140-147 for one ordered pair of frames."""
    return float(frame_distances(poses, disps, intr, [a], [b], beta, device)[0])


def distance_matrix(poses, disps, intr, frames, beta=0.5, device=None):
    """D[a, b] = distance(frames[a] -> frames[b]) for all ordered pairs; diagonal 0."""
    fr = _i32(frames)
    n = len(fr)
    A, B = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    off = A != B
    D = np.zeros((n, n))
    if off.any():
        D[off] = frame_distances(poses, disps, intr, fr[A[off]], fr[B[off]], beta, device)
    return D


def build_frontend_edges(window, radius=FRONTEND_RADIUS, existing=(), ages=None, max_age=MAX_EDGE_AGE):
    """SPEC.md:150-157 (G3) -> (ii, jj) int32, sorted by (i, j)."""
    lib = _lib.load()
    w = _i32(window)
    ex = np.asarray(existing, dtype=np.int32).reshape(-1, 2)
    ei, ej = _i32(ex[:, 0]), _i32(ex[:, 1])
    ag = None if ages is None else _i32(ages)
    if ag is not None and len(ag) != len(ei):
        raise ConfigError("ages must match existing edges")
    cap = len(w) * (len(w) - 1) + len(ei) + 1
    oi = np.empty(cap, np.int32)
    oj = np.empty(cap, np.int32)
    n = ctypes.c_int32(0)
    _check(lib.dba_frontend_edges(len(w), w.ctypes.data_as(_I32P), int(radius), len(ei),
                                  ei.ctypes.data_as(_I32P), ej.ctypes.data_as(_I32P),
                                  None if ag is None else ag.ctypes.data_as(_I32P), int(max_age), cap,
                                  oi.ctypes.data_as(_I32P), oj.ctypes.data_as(_I32P), ctypes.byref(n)))
    return oi[:n.value].copy(), oj[:n.value].copy()


def backend_edges(frames, dist, window=BACKEND_WINDOW, max_edges=BACKEND_MAX_EDGES, loops=()):
    """G4 selection from a precomputed (n, n) distance matrix over ``frames``."""
    lib = _lib.load()
    fr = _i32(frames)
    D = np.ascontiguousarray(dist, dtype=np.float64)
    if D.shape != (len(fr), len(fr)):
        raise ConfigError("dist must be (n_frames, n_frames)")
    lp = np.asarray(loops, dtype=np.int32).reshape(-1, 2)
    li, lj = _i32(lp[:, 0]), _i32(lp[:, 1])
    cap = max(int(max_edges), 0) + len(li) + 2
    oi = np.empty(cap, np.int32)
    oj = np.empty(cap, np.int32)
    n = ctypes.c_int32(0)
    _check(lib.dba_backend_edges(len(fr), fr.ctypes.data_as(_I32P), D.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 int(window), int(max_edges), len(li), li.ctypes.data_as(_I32P),
                                 lj.ctypes.data_as(_I32P), cap, oi.ctypes.data_as(_I32P),
                                 oj.ctypes.data_as(_I32P), ctypes.byref(n)))
    return oi[:n.value].copy(), oj[:n.value].copy()


def build_backend_graph(poses, disps, intr, frames, beta=0.5, window=BACKEND_WINDOW,
                        max_edges=BACKEND_MAX_EDGES, loops=(), device=None):
    """GPU distances over the last `window` keyframes, host ranking (G4)."""
    fr = _i32(frames)
    w0 = max(0, len(fr) - int(window))
    D = np.full((len(fr), len(fr)), np.inf)
    np.fill_diagonal(D, 0.0)
    D[w0:, w0:] = distance_matrix(poses, disps, intr, fr[w0:], beta, device)
    return backend_edges(fr, D, window, max_edges, loops)
