"""Provider-tensor ingestion: DSPT files -> the DBA flow layout.

Replaces ``PrecomputedProviders`` (``providers.py:401-424``) on the BA path.  A DSPT
flow file *is* one (H, W, 4) float32 record ``[tu, tv, wu, wv]`` (``providers.py:12-15``),
so the native reader (``dba_dspt_*`` in ``include/dba_b200.h``, ``csrc/dba_ingest.cu``)
preads each payload straight into its row of the ``(E, H, W, 4)`` array the pass kernel
consumes — on the host, or into device memory through a pinned staging buffer whose two
halves alternate between disk reads and async host->device copies.

Semantics follow the reference adapter exactly:

* file names ``flow_{i:06d}_{j:06d}.dspt`` / ``prior_{k:06d}.dspt`` (``providers.py:415-424``);
* header checks of ``read_dspt`` (``:386-399``): magic, version 1, exact payload length,
  and here also C = 4 (flow) / 1 (prior) and the expected H, W;
* weights clipped to [0, 1] (``np.clip``, NaN kept), priors clamped below at 1e-6.

Values are kept in float32 (the reference upcasts the same float32 payload to float64, so
the two agree exactly); failures raise :class:`DataError` naming the first bad file.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _lib
from .errors import ConfigError, DataError

_I32P = ctypes.POINTER(ctypes.c_int32)
_F32P = ctypes.POINTER(ctypes.c_float)


def flow_name(i: int, j: int) -> str:
    return f"flow_{int(i):06d}_{int(j):06d}.dspt"


def prior_name(k: int) -> str:
    return f"prior_{int(k):06d}.dspt"


def _edges(ii, jj):
    ii = np.ascontiguousarray(ii, dtype=np.int32).reshape(-1)
    jj = np.ascontiguousarray(jj, dtype=np.int32).reshape(-1)
    if ii.shape != jj.shape:
        raise ConfigError("ii and jj must have the same length")
    return ii, jj


def _check(code: int, directory, what: str, bad: int):
    if code == _lib.DBA_OK:
        return
    if code == _lib.DBA_EDATA:
        raise DataError(f"{Path(directory) / what}: missing or malformed DSPT provider tensor "
                        f"(index {bad})")
    if code == _lib.DBA_EINVAL:
        raise ConfigError(_lib.status_string(code))
    raise RuntimeError(f"libdba_b200: {_lib.status_string(code)} (status {code})")


def read_flows(directory, ii, jj, height: int, width: int, out=None, threads: int = 0) -> np.ndarray:
    """All edges' flow records into a host (E, H, W, 4) float32 array.

    ``out`` may be a caller-owned C-contiguous float32 buffer of that shape (e.g. the
    numpy view of a pinned torch tensor) so that a following device copy is DMA."""
    lib = _lib.load()
    ii, jj = _edges(ii, jj)
    E = len(ii)
    if out is None:
        out = np.empty((E, height, width, 4), dtype=np.float32)
    if out.dtype != np.float32 or not out.flags.c_contiguous or out.shape != (E, height, width, 4):
        raise ConfigError("out must be a C-contiguous float32 (E, H, W, 4) array")
    bad = ctypes.c_int32(-1)
    code = lib.dba_dspt_read_flows(os.fsencode(str(directory)), E, ii.ctypes.data_as(_I32P),
                                   jj.ctypes.data_as(_I32P), int(height), int(width),
                                   out.ctypes.data_as(_F32P), int(threads), ctypes.byref(bad))
    b = int(bad.value)
    _check(code, directory, flow_name(ii[b], jj[b]) if 0 <= b < E else "flow_*.dspt", b)
    return out


def read_priors(directory, frames, height: int, width: int, threads: int = 0) -> np.ndarray:
    """Depth priors d* (N, H, W) float32 of ``frames``, clamped below at 1e-6."""
    lib = _lib.load()
    fr = np.ascontiguousarray(frames, dtype=np.int32).reshape(-1)
    out = np.empty((len(fr), height, width), dtype=np.float32)
    bad = ctypes.c_int32(-1)
    code = lib.dba_dspt_read_priors(os.fsencode(str(directory)), len(fr), fr.ctypes.data_as(_I32P),
                                    int(height), int(width), out.ctypes.data_as(_F32P), int(threads),
                                    ctypes.byref(bad))
    b = int(bad.value)
    _check(code, directory, prior_name(fr[b]) if 0 <= b < len(fr) else "prior_*.dspt", b)
    return out


def load_flows(directory, ii, jj, height: int, width: int, device=None, staging_mb: int = 64,
               threads: int = 0, stream=None):
    """All edges' flow records straight into a device (E, H, W, 4) float32 tensor.

    Disk reads (a thread pool) fill one half of a pinned staging buffer while the other
    half is copied on ``stream``; returns once every copy has landed."""
    import torch

    from .dba import _device
    lib = _lib.load()
    dev = _device(device)
    ii, jj = _edges(ii, jj)
    E = len(ii)
    rec = 16 * int(height) * int(width)
    out = torch.empty((E, height, width, 4), dtype=torch.float32, device=dev)
    if E == 0:
        return out
    nbytes = max(2 * rec, (int(staging_mb) << 20) // rec * rec)
    nbytes = min(nbytes, 2 * E * rec)
    staging = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    bad = ctypes.c_int32(-1)
    with torch.cuda.device(dev):
        code = lib.dba_dspt_load_flows(os.fsencode(str(directory)), E, ii.ctypes.data_as(_I32P),
                                       jj.ctypes.data_as(_I32P), int(height), int(width),
                                       ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(staging.data_ptr()),
                                       nbytes, int(threads), ctypes.c_void_p(st.cuda_stream),
                                       ctypes.byref(bad))
    b = int(bad.value)
    _check(code, directory, flow_name(ii[b], jj[b]) if 0 <= b < E else "flow_*.dspt", b)
    return out


def dump_flows(directory, flow, ii, jj):
    """Write (E, H, W, 4) records as DSPT flow files (the layout dump_providers writes,
    ``providers.py:432-447``)."""
    from .scenes import write_dspt
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    ii, jj = _edges(ii, jj)
    for e in range(len(ii)):
        write_dspt(d / flow_name(ii[e], jj[e]), flow[e])
